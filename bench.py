"""Benchmark: shadow-model train samples/s + MMD kernel-pairs/s on B200
(BASELINE.json metric), with the reference CPU path timed beside it.

Default line (configs[1], C2): the mapping-based MMD transfer step of MLP
1024-512-256-10 with a 512 source + 512 target batch and 5-bandwidth
Gaussian MMD on the 256-d hidden layer (CE + lambda*MMD, SGD), for a bank of
G=32 shadow models per GPU (C5's per-GPU, per-paradigm shadow share).  Weak
scaling: every rank trains its own 32 shadows, no data-path collective
(models are independent).  One step = one SGD step of all 32.
The same JSON line carries two sub-objects measured in the same run, each
with its own roofline, clocks, e2e and cpu_baseline:
  "c4"     -- configs[3] MMD stress (65536 x 8192 x 512): kernel pairs/s;
  "attack" -- the attack stage of configs[4] over 2^20 queries: queries/s.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  python bench.py --workload c4|attack|c3|c5   # one workload as the whole line
      c3: configs[2], parameter-based 784-256-10, 8 shadows per GPU, with the
          NCCL feature all-gather inside the timed region
      c5: configs[4], the full sweep (3 paradigms x 256 shadows, 2^20 attack
          queries each) through the native driver

--gpus N without torchrun re-launches itself under torch.distributed.run
(one process per GPU).  Rank 0 prints ONE JSON line (contract in the task).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# NCCL's "NCCL version ..." banner goes to stdout, which must hold exactly one
# JSON line (rank 0); keep NCCL at warnings (env NCCL_DEBUG_BENCH overrides)
os.environ["NCCL_DEBUG"] = os.environ.get("NCCL_DEBUG_BENCH", "WARN")

DIMS = [1024, 512, 256, 10]
G = 32
SRC, TGT = 512, 512
B = SRC + TGT
LAMBDA = 1.0
LR = 0.01
# algorithmic cost
FLOP_SRC = 2_898_944
MMD_PAIRS = (B * (B - 1)) // 2  # 523,776 unique pairs per model per step
MMD_FLOP_PER_PAIR = 4 * DIMS[2]  # fwd 2d + bwd 2d
WORKLOAD = ("C2 mapping-based MMD transfer: MLP 1024-512-256-10, 512 src + 512 tgt, "
            "5-bandwidth Gaussian MMD (lambda=1) on the 256-d hidden layer, SGD; bank of 32 "
            "shadow models per GPU")

C4_M, C4_N, C4_D = 65536, 8192, 512
C4_PAIRS = C4_M * (C4_M - 1) // 2 + C4_N * (C4_N - 1) // 2 + C4_M * C4_N  # 2,717,872,128
C4_CPU_SLICE = 4096
ATT_Q = 1 << 20
# attack stage algorithmic bytes per query: logits 40 + label 1 read, two AUC
# keys written (8); the sort reads and writes the 4-B keys (one pass counted),
# the member count reads label + member key + ~1 probe (9)
ATT_BYTES_Q = 40 + 1 + 8 + 2 * 4 + 9

C3_DIMS = [784, 256, 10]
C3_G = 8            # shadows per GPU (64 over 8 GPUs)
C3_B = 256          # member rows per step (+ as many source rows)
C3_MEMBERS = 2048
C3_EPOCHS = 10
C3_FLOP = 818_176   # per training sample


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("bf16_tflops"), d.get("bf16_tflops_sustained"), d.get("hbm_gbs"), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


def fp32acc_peak():
    """3xTF32 = fp32-accurate tensor rate: tf32 is half the measured bf16
    rate, three MMAs per product."""
    bf16, _, _, src = peaks()
    return bf16 / 6.0, bf16, src


class ClockSampler:
    """SM clock + throttle reasons via NVML, polled every `period` s (1 ms) in a
    thread, for the duration of the `with` block (the timed region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int, period: float = 0.001):
        self.index = index
        self.period = period
        self.samples = []
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)

            def poll():
                while not self._stop.is_set():
                    try:
                        self.samples.append(
                            (pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                             pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)))
                    except Exception:
                        pass
                    time.sleep(self.period)

            self.t = threading.Thread(target=poll, daemon=True)
            self.t.start()
        except Exception:
            self.t = None
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.t:
            self.t.join()

    def summary(self):
        sm = [s for s, _ in self.samples]
        reasons = sorted({n for _, r in self.samples for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(sm), "source": f"nvml, {self.period * 1000:g} ms poll"}


# ----------------------------------------------------------------------------- processes
def self_launch(args) -> None:
    """--gpus N > 1 without torchrun: re-run this command under
    torch.distributed.run, one process per GPU (127.0.0.1 rendezvous)."""
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    raise SystemExit(subprocess.call(cmd))


def dist_setup(n_gpus):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != n_gpus:
        raise SystemExit(f"bench.py: --gpus {n_gpus} but WORLD_SIZE={world}; launch one process per GPU "
                         f"(torchrun --nproc-per-node {n_gpus}) or drop the launcher to self-launch")
    if n_gpus > torch.cuda.device_count():
        raise SystemExit(f"bench.py: --gpus {n_gpus} but only {torch.cuda.device_count()} visible GPU(s)")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed(world, local, steps, fn, stream=None):
    """W warm-up steps are the caller's; here: barrier + synchronize, CUDA
    events on the launching stream around exactly `steps` calls, synchronize,
    max over ranks; NVML clocks sampled during the region."""
    import torch

    stream = stream or torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
    return max_over_ranks(e0.elapsed_time(e1), world), clk.summary()


# ----------------------------------------------------------------------------- CPU arms
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def _ref():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    return po, po.ref()


def _cpu_record(po, R, kind, cores, sample, value, unit, seconds):
    rec = {"value": value, "unit": unit, "cores": cores, "kind": kind, "sample": sample,
           "seconds": seconds}
    rec.update(po.cpu_info())
    if R is not None:
        rec["build"] = R.ref_build_info().decode()
    return rec


def cpu_c2(threads=None, steps=1):
    """Reference CPU path for C2 on the host cores: one model per std::thread
    (tape.hpp:84-85), each running reference-Tape SGD steps with
    the MMD injected into the same Tape; init and data before the timed
    region.  Returns (samples/s, cpu_baseline record)."""
    import ctypes as C

    po, R = _ref()
    threads = threads or cpu_threads()
    sample = (f"{threads} C2 models x {steps} SGD step(s) of {B} samples (512 src + 512 tgt, 5-bw "
              f"MMD over unique pairs injected into the step's Tape), one model per thread")
    if R is not None:
        secs = R.ref_bench_train(threads, 3, (C.c_int * 4)(*DIMS), B, SRC, steps, LAMBDA, 1234)
        kind = "reference"
    else:  # oracle port (C restatement) in Python threads; ctypes drops the GIL
        import numpy as np

        def one(seed):
            r = po.Rng(seed)
            W, b = po.mlp_init(r, DIMS)
            X = r.normals(B * DIMS[0]).reshape(B, DIMS[0])
            y = np.array([r.below(10) for _ in range(B)], dtype=np.int32)
            for _ in range(steps):
                _, H = po.mlp_forward(DIMS, W, b, X)
                _, _, gs, gt = po.mmd_gaussian(H[:SRC], H[SRC:])
                po.mlp_train_step(DIMS, W, b, X, y, lr=LR, dH=LAMBDA * np.concatenate([gs, gt]))

        t0 = time.perf_counter()
        ts = [threading.Thread(target=one, args=(s,)) for s in range(threads)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        secs = time.perf_counter() - t0
        kind = "port"
    v = threads * steps * B / secs
    return v, _cpu_record(po, R, kind, threads, sample, v, "samples/s", secs)


def cpu_c4(threads=None):
    """C4 on the host cores: the unordered pairs whose smaller index lies in
    the first 4,096 source rows (a 4,096-row slice,
    scaled by the stated pair fraction), value + gradient, reference
    mm_acc / mm_tn_acc tiles over threads."""
    import ctypes as C

    po, R = _ref()
    if R is None:
        return None, None
    threads = threads or cpu_threads()
    pairs, sums = C.c_double(), (C.c_double * 3)()
    secs = R.ref_bench_mmd(threads, C4_M, C4_N, C4_D, C4_CPU_SLICE, 7, C.byref(pairs), sums)
    v = pairs.value / secs
    sample = (f"pairs (i < j) with i in the first {C4_CPU_SLICE} of {C4_M + C4_N} rows: "
              f"{pairs.value:.4g} unique pairs = {pairs.value / C4_PAIRS:.4f} of the full C4 "
              f"evaluation (scaled to pairs/s), fwd + bwd, f64")
    return v, _cpu_record(po, R, "reference", threads, sample, v, "pairs/s", secs)


def cpu_attack(threads=None, reps=2):
    """the attack stage on the host cores: Tape softmax -> top-3 -> attack MLP
    (Tape ops) over row chunks on threads, then std::sort + mid-rank AUC"""
    import ctypes as C

    po, R = _ref()
    if R is None:
        return None, None
    threads = threads or cpu_threads()
    auc = C.c_double()
    secs = R.ref_bench_attack(threads, ATT_Q, reps, 5, C.byref(auc))
    v = reps * ATT_Q / secs
    sample = f"{reps} full evaluations of {ATT_Q} queries (scoring on threads, std::sort AUC on one)"
    return v, _cpu_record(po, R, "reference", threads, sample, v, "queries/s", secs)


def cpu_c3(threads=None, steps=2):
    import ctypes as C

    po, R = _ref()
    if R is None:
        return None, None
    threads = threads or cpu_threads()
    secs = R.ref_bench_train_heads(threads, 2, (C.c_int * 3)(*C3_DIMS), 2, 2 * C3_B, C3_B, steps, 0.0, 99)
    v = threads * steps * 2 * C3_B / secs
    sample = (f"{threads} parameter-based 784-256-10 models (two heads) x {steps} SGD steps of "
              f"{C3_B} source + {C3_B} member rows, one model per thread")
    return v, _cpu_record(po, R, "reference", threads, sample, v, "samples/s", secs)


def run_reference_arm(args, world, rank):
    """--impl reference: the reference's own CPU implementation of the path
    (oracle/_ref: the unmodified headers) on the host cores, rank 0 only."""
    if rank != 0:
        return
    wl = args.workload
    if wl == "c2":
        fn, unit, metric = (lambda: cpu_c2()), "samples/s", "shadow-model train samples/s"
    elif wl == "c4":
        fn, unit, metric = (lambda: cpu_c4()), "pairs/s", "MMD kernel-pairs/s"
    elif wl == "attack":
        fn, unit, metric = (lambda: cpu_attack(reps=1)), "queries/s", "membership-attack queries/s"
    elif wl == "c5":
        fn, unit, metric = (lambda: cpu_c1_sample()), "samples/s", "shadow-model train samples/s"
    else:
        fn, unit, metric = (lambda: cpu_c3()), "samples/s", "shadow-model train samples/s"
    for _ in range(min(args.warmup, 1)):
        fn()
    vals, secs, rec = [], 0.0, None
    for _ in range(args.steps):
        v, rec = fn()
        vals.append(v)
        secs += rec["seconds"]
    # each step is a bounded sample of the workload; value = the mean rate
    value = statistics.mean(vals)
    line = {
        "metric": metric, "value": value, "unit": unit,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * secs / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": {"c2": WORKLOAD, "c4": "C4 MMD stress 65536 x 8192 x 512",
                                "attack": "attack stage, 2^20 queries",
                                "c3": "C3 parameter-based 784-256-10",
                                "c5": "C5 sweep model 784-256-10 (sampled steps)"}[wl] + " (CPU, host threads)",
                   "parallelism": f"{rec['cores']} threads"},
        "cpu_baseline": dict(rec, value=value),
        "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def kernel_traffic(phase, key="phases"):
    """DRAM read+write bytes per step of a phase's kernels (the same launches
    `achieved` is timed over), from the newest committed ncu --set full capture
    summary (profiles/rNN_kernels.json).  Returns (bytes or None, source file)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r[0-9]*_kernels.json")))
    for f in reversed(files):
        with open(f) as fh:
            d = json.load(fh)
        ent = d.get(key, {}).get(phase)
        if ent and ent.get("dram_bytes_per_step") is not None:
            return ent.get("dram_bytes_per_step"), os.path.basename(f)
    return None, None


# ----------------------------------------------------------------------------- C4 MMD
def measure_c4(args, world, rank, local, steps, warmup, cpu=True):
    """configs[3]: multi-bandwidth MMD^2 + gradient of Xs [65536, 512] vs Xt
    [8192, 512].  One step = the full evaluation on the materialised-W path
    (each unordered 128x128 tile pair once, W = 21.7 GB, V = W.Z as a GEMM).
    N GPUs: rank r owns an equal range of 128-row tiles
    (mtk_mmd_gaussian_tiles: the tile pairs touching its rows, its rows of W,
    V and the gradient); the [T, 3] tile-row kernel sums are all-gathered
    over NCCL inside the timed region and combined in ascending tile order --
    the gradients and the value are bit-identical to one GPU's."""
    import torch

    from paper_2011_09463_b200 import api

    ctx = api.Context(local)
    gen = torch.Generator(device="cuda").manual_seed(4)
    Nt = C4_M + C4_N
    Z = torch.randn(Nt, C4_D, device="cuda", generator=gen)  # [Xs; Xt] in one block
    Z[C4_M:] += 0.1
    Xs, Xt = Z[:C4_M], Z[C4_M:]
    gZ = torch.empty_like(Z)
    gXs, gXt = gZ[:C4_M], gZ[C4_M:]
    beta = api.mmd_beta(ctx, Xs, Xt)
    lo, hi = api.mmd_tile_ranges(C4_M, C4_N, world)[rank]
    r0, r1 = lo * api.MMD_TILE, min(Nt, hi * api.MMD_TILE)
    full = world == 1
    out = {}
    parts = torch.empty((world, -(-Nt // api.MMD_TILE), 3), dtype=torch.float64, device="cuda")

    def evaluate():
        if full:
            out["v"] = api.mmd_gaussian(ctx, Xs, Xt, beta=beta)[0]
        else:
            import torch.distributed as dist

            part = torch.from_numpy(api.mmd_gaussian_tiles(ctx, Z, C4_M, beta, lo, hi, gZ)).cuda()
            dist.all_gather_into_tensor(parts, part)  # [world, T, 3], one owner per tile row
            out["v"] = api.mmd_value_from_tiles(parts.sum(0).cpu().numpy(), C4_M, C4_N)

    for _ in range(warmup):
        evaluate()
    torch.cuda.synchronize()
    n0 = ctx.launches
    ms, clocks = timed(world, local, steps, evaluate)
    launches = ctx.launches - n0
    # e2e through the C ABI with HOST buffers: the [Xs; Xt] block H2D from
    # pinned memory, the evaluation, the gradient block D2H, every step
    Zh = Z.cpu().pin_memory()
    gh = torch.empty_like(Zh).pin_memory()

    def e2e_step():
        Z.copy_(Zh, non_blocking=True)
        if full:
            v, _, gs, gt = api.mmd_gaussian(ctx, Xs, Xt, beta=beta)
            gh[:C4_M].copy_(gs, non_blocking=True)
            gh[C4_M:].copy_(gt, non_blocking=True)
        else:
            evaluate()
            gh[r0:r1].copy_(gZ[r0:r1], non_blocking=True)

    e2e_step()
    e2e_ms, _ = timed(world, local, max(1, steps // 2), e2e_step)
    e2e_steps = max(1, steps // 2)
    peak, bf16, src = fp32acc_peak()
    pairs_s = C4_PAIRS * steps / (ms / 1000.0)
    achieved = pairs_s / world * 4 * C4_D / 1e12  # per GPU
    traffic, tsrc = kernel_traffic("c4", key="workloads")
    res = {
        "metric": "MMD kernel-pairs/s", "value": pairs_s, "unit": "pairs/s", "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": ms / steps, "higher_is_better": True,
        "scaling": "strong", "dtype": "f32",
        "config": {"workload": "C4 MMD stress: Xs 65536 x 512 vs Xt 8192 x 512 (N(0,1), N(0.1,1)), "
                               "5-bandwidth Gaussian MMD^2 + gradient"
                               + ("" if full else ", 128-row tiles sharded over ranks"),
                   "unique_pairs": C4_PAIRS, "parallelism": f"tiles{world}", "value": out.get("v"),
                   "path": "materialised W (mmd_w + wsum + V GEMM)" + (
                       "" if full else f"; rank tiles [{lo}, {hi}): its tile pairs (cross-rank pairs on both "
                       "ranks, each its own rows), its rows of V; [T,3] partials all-gathered (NCCL)"),
                   "l2": "inputs 151 MB + tf32 planes + 21.7 GB of W > 126 MB L2"},
        "roofline": {"bound": "tensor", "kernel": "mmd_w + V GEMM (+prep)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "peak_note": f"algorithmic 4d flop per unique pair; 3xTF32 peak = {src} bf16 {bf16} / 6"
                                  + ("" if full else f"; per rank {2 - 1 / world:.3f}x the ideal share of "
                                     "pass-1 tile pairs (cross-rank pairs evaluated twice)"),
                     "traffic_note": f"DRAM bytes per evaluation, profiles/{tsrc}" if tsrc else
                     "no ncu capture of this workload committed"},
        "e2e": {"value": C4_PAIRS * e2e_steps / (e2e_ms / 1000.0), "unit": "pairs/s",
                "h2d_bytes_per_step": Nt * C4_D * 4,
                "d2h_bytes_per_step": (Nt if full else r1 - r0) * C4_D * 4 + 8},
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": None,
    }
    del Z, gZ, Zh, gh
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and cpu:
        res["cpu_baseline"] = cpu_c4()[1]
    return res


# ----------------------------------------------------------------------------- attack
def measure_attack(args, world, rank, local, steps, warmup, cpu=True):
    """Attack stage of configs[4] on one paradigm's 2^20 member/non-member
    queries per rank: posterior top-3 features -> attack MLP 3-64-2 -> member
    score -> AUC + accuracy (mtk_attack_auc)."""
    import torch

    from paper_2011_09463_b200 import api

    ctx = api.Context(local)
    gen = torch.Generator(device="cuda").manual_seed(5 + rank)
    logits = torch.randn(ATT_Q, 10, device="cuda", generator=gen)
    labels = (torch.rand(ATT_Q, device="cuda", generator=gen) < 0.5).to(torch.uint8)
    logits[labels.bool(), 0] += 1.0  # members look more confident
    att = api.Bank(ctx, 1, [3, 64, 2])
    att.init_params(0, api.Rng(77))
    out = {}

    def step():
        out["r"] = api.attack_auc(att, logits, labels)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    n0 = ctx.launches
    ms, clocks = timed(world, local, steps, step)
    launches = ctx.launches - n0
    auc, acc = out["r"]
    lh = logits.cpu().pin_memory()
    labh = labels.cpu().pin_memory()

    def e2e_step():  # host posteriors + labels in, AUC / accuracy out (synchronizing)
        logits.copy_(lh, non_blocking=True)
        labels.copy_(labh, non_blocking=True)
        api.attack_auc(att, logits, labels)

    e2e_step()
    e2e_ms, _ = timed(world, local, steps, e2e_step)
    _, _, hbm, src = peaks()
    qps = world * ATT_Q * steps / (ms / 1000.0)
    gbs = qps * ATT_BYTES_Q / world / 1e9
    traffic, tsrc = kernel_traffic("attack", key="workloads")
    res = {
        "metric": "membership-attack queries/s", "value": qps, "unit": "queries/s", "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": ms / steps, "higher_is_better": True,
        "scaling": "weak", "dtype": "f32",
        "config": {"workload": "attack stage: 2^20 queries x 10-class posteriors -> top-3 "
                               "features -> attack MLP 3-64-2 -> score -> AUC/accuracy per rank",
                   "queries_per_gpu": ATT_Q, "parallelism": f"shard{world}", "auc": auc, "accuracy": acc},
        "roofline": {"bound": "hbm", "kernel": "attack_score + AUC (whole stage)", "achieved": gbs,
                     "peak": hbm, "unit": "GB/s", "frac": gbs / hbm if hbm else None, "traffic": traffic,
                     "peak_note": f"{src} HBM copy bandwidth; {ATT_BYTES_Q} algorithmic B/query",
                     "traffic_note": f"DRAM bytes per evaluation, profiles/{tsrc}" if tsrc else
                     "no ncu capture of this workload committed"},
        "e2e": {"value": world * ATT_Q * steps / (e2e_ms / 1000.0), "unit": "queries/s",
                "h2d_bytes_per_step": ATT_Q * (10 * 4 + 1), "d2h_bytes_per_step": 16},
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": None,
    }
    if rank == 0 and world == 1 and cpu:
        res["cpu_baseline"] = cpu_attack()[1]
    return res


# ----------------------------------------------------------------------------- C3
def measure_c3(args, world, rank, local, steps, warmup, cpu=True):
    """configs[2]: parameter-based shared-layer transfer, 8 shadows per GPU
    (784-256-10 trunk + a source and a target head), device-resident pools.
    One step = one rank's whole shadow job: E=10 epochs over 2048 members
    (B = 256 member rows + 256 source rows per step, mtk_bank_train_epoch),
    the posterior top-3 features of its 8 models on 2048 members + 2048
    non-members, and the NCCL all-gather of every rank's features
    (mtk_allgather) -- the collective is inside the timed region."""
    import numpy as np
    import torch

    from paper_2011_09463_b200 import api

    ctx = api.Context(local)
    comm = api.Comm(ctx)
    dev = torch.device("cuda", local)
    C, d = C3_DIMS[-1], C3_DIMS[0]
    rng = np.random.default_rng(20110946)
    mu = torch.tensor(0.1 * rng.standard_normal((C, d)), dtype=torch.float32)
    shift = torch.tensor(0.5 * rng.standard_normal(d), dtype=torch.float32)
    Xt, yt = api.synth_counter(ctx, 20110946, 1, 8192, mu, shift)    # target pool
    Xs, ys = api.synth_counter(ctx, 20110946, 2, 16384, mu, None)    # source pool
    pool = torch.cat([Xs, Xt]).contiguous()
    ypool = torch.cat([ys, yt]).contiguous()
    off = Xs.shape[0]
    bank = api.Bank(ctx, C3_G, C3_DIMS, n_heads=2)
    r = api.Rng(1000 + rank)
    for g in range(C3_G):
        bank.init_params(g, r)
    spe = C3_MEMBERS // C3_B
    nsteps = C3_EPOCHS * spe
    idx = np.empty((nsteps, C3_G, 2 * C3_B), dtype=np.int64)
    qidx = np.empty((C3_G, 2 * C3_MEMBERS), dtype=np.int64)
    for g in range(C3_G):
        perm = rng.permutation(8192)
        mem, non = perm[:C3_MEMBERS], perm[C3_MEMBERS:2 * C3_MEMBERS]
        srcrows = rng.permutation(16384)[:4096]
        qidx[g] = np.concatenate([mem, non])
        for e in range(C3_EPOCHS):
            order = rng.permutation(C3_MEMBERS)
            for t in range(spe):
                s = e * spe + t
                idx[s, g, :C3_B] = srcrows[(s * C3_B + np.arange(C3_B)) % 4096]
                idx[s, g, C3_B:] = off + mem[order[t * C3_B:(t + 1) * C3_B]]
    idx_d = torch.from_numpy(idx).to(dev)
    qidx_d = torch.from_numpy(qidx).to(dev)
    Xq = torch.empty((C3_G, 2 * C3_MEMBERS, d), device=dev)
    feats_all = torch.empty((world, C3_G, 2 * C3_MEMBERS, 3), device=dev)
    kw = dict(lr=0.05, src_rows=C3_B, denom=(float(C3_B), float(C3_B)))

    def job(pool_, ypool_):
        bank.train_epoch(pool_, ypool_, idx_d, None, None, **kw)
        api.gather_rows(ctx, pool_[off:], qidx_d, Xq)
        F = api.posterior_features(ctx, bank.forward(Xq, head=1), 3).reshape(C3_G, 2 * C3_MEMBERS, 3)
        comm.all_gather(F, out=feats_all)

    for _ in range(warmup):
        job(pool, ypool)
    torch.cuda.synchronize()
    n0 = ctx.launches
    ms, clocks = timed(world, local, steps, lambda: job(pool, ypool))
    launches = ctx.launches - n0
    # e2e: the pools + batch indices from pinned host memory, the gathered
    # features of all ranks back to the host, every step
    ph, yph, ih = pool.cpu().pin_memory(), ypool.cpu().pin_memory(), idx_d.cpu().pin_memory()
    fh = torch.empty(feats_all.shape, dtype=torch.float32).pin_memory()

    def e2e_step():
        pool.copy_(ph, non_blocking=True)
        ypool.copy_(yph, non_blocking=True)
        idx_d.copy_(ih, non_blocking=True)
        job(pool, ypool)
        fh.copy_(feats_all, non_blocking=True)

    e2e_step()
    e2e_ms, _ = timed(world, local, steps, e2e_step)
    peak, bf16, src = fp32acc_peak()
    samples = world * C3_G * nsteps * 2 * C3_B
    value = samples * steps / (ms / 1000.0)
    achieved = value / world * C3_FLOP / 1e12
    res = {
        "metric": "shadow-model train samples/s", "value": value, "unit": "samples/s",
        "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": ms / steps,
        "higher_is_better": True, "scaling": "weak", "dtype": "f32",
        "config": {"workload": "C3 parameter-based shared-layer transfer: MLP 784-256-10 trunk + "
                               "source / target heads, 8 shadows per GPU, 10 epochs over 2048 "
                               "members (256 member + 256 source rows per step), top-3 posterior "
                               "features of 4096 queries per model, NCCL all-gather of all ranks' "
                               "features inside the timed region",
                   "models_per_gpu": C3_G, "models_total": world * C3_G,
                   "samples_per_step": samples, "parallelism": f"shard{world}",
                   "nccl": comm.nccl_version(),
                   "allgather_bytes_per_rank": C3_G * 2 * C3_MEMBERS * 3 * 4},
        "roofline": {"bound": "tensor", "kernel": "whole job (train epochs + query + all-gather)",
                     "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": None,
                     "peak_note": f"{C3_FLOP} algorithmic flop per train sample; 3xTF32 peak = {src} "
                                  f"bf16 {bf16} / 6"},
        "e2e": {"value": samples * steps / (e2e_ms / 1000.0), "unit": "samples/s",
                "h2d_bytes_per_step": pool.numel() * 4 + ypool.numel() * 4 + idx_d.numel() * 8,
                "d2h_bytes_per_step": feats_all.numel() * 4},
        "gpu_launches": launches,
        "clocks": clocks,
        "cpu_baseline": None,
    }
    comm.close()
    if rank == 0 and world == 1 and cpu:
        res["cpu_baseline"] = cpu_c3()[1]
    return res


# ----------------------------------------------------------------------------- C5
def measure_c5(args, world, rank, local, steps, warmup, cpu=True):
    """configs[4]: the full privacy sweep -- 3 transfer paradigms x 256 shadow
    models (+ 1 target each), 2048 members + 2048 non-members per model, so
    the attack model trains on 256 x 4096 = 2^20 member / non-member queries
    per paradigm; AUC + accuracy on the target's 4096.  Each paradigm is one
    mtk_sweep_run call (the native C++ driver: host mt::Rng sampling, device
    pools, whole epochs per call, the ranks' features all-gathered over NCCL).
    model / parameter: MLP 784-256-10; mapping: 1024-512-256-10 (configs[1]'s
    model, lambda = 1 MMD).  One step = the whole sweep; timed on the host
    clock (it includes host sampling), max over ranks."""
    import torch

    from paper_2011_09463_b200 import api

    ctx = api.Context(local)
    comm = api.Comm(ctx) if world > 1 else None
    cfgs = [dict(paradigm="model", n_shadows=256), dict(paradigm="mapping", n_shadows=256, dims=(1024, 512, 256, 10)),
            dict(paradigm="parameter", n_shadows=256)]

    def sweep():
        return [api.sweep_run(ctx, c, comm) for c in cfgs]

    res = None
    for _ in range(warmup):
        res = sweep()
    times = []
    # a 10 ms poll: the sweep's host phases use every core (a 1 ms poller
    # thread straggles their parallel sections)
    with ClockSampler(local, period=0.01) as clk:
        for _ in range(steps):
            barrier(world)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = sweep()
            torch.cuda.synchronize()
            times.append(max_over_ranks(time.perf_counter() - t0, world))
    secs = statistics.median(times)
    d = {"model": 784, "mapping": 1024, "parameter": 784}
    # training rows per model: model = 2 pretrain epochs x 4096 source + 10 x 2048 members;
    # mapping / parameter = 10 epochs x (2048 members + 2048 source rows riding along)
    rows = {"model": 2 * 4096 + 10 * 2048, "mapping": 10 * 4096, "parameter": 10 * 4096}
    samples = sum(257 * rows[c["paradigm"]] for c in cfgs)
    flop = sum(257 * rows[c["paradigm"]] * (818_176 if c["paradigm"] != "mapping" else 2_898_944) for c in cfgs)
    peak, bf16, src = fp32acc_peak()
    achieved = flop / secs / world / 1e12
    out = {
        "metric": "shadow-model train samples/s", "value": samples / secs, "unit": "samples/s", "n_gpus": world,
        "steps": steps, "warmup": warmup, "ms_per_step": 1000.0 * secs, "higher_is_better": True,
        "scaling": "strong", "dtype": "f32",
        "config": {"workload": "C5 full privacy sweep: 3 paradigms x (1 target + 256 shadows), 2048 members + "
                               "2048 non-members each, 2^20 attack-training queries per paradigm, attack MLP "
                               "3-64-2, AUC/accuracy on the target (native mtk_sweep_run, host-clock timed)",
                   "paradigms": {c["paradigm"]: {"auc": r["auc"], "accuracy": r["accuracy"],
                                                 "models": r["models"], "seconds": r["seconds"],
                                                 "dims": list(c.get("dims", (784, 256, 10)))}
                                 for c, r in zip(cfgs, res)},
                   "train_samples_per_sweep": samples, "parallelism": f"models{world}",
                   "timing": f"median of {steps} host-clock sweeps"},
        "roofline": {"bound": "tensor", "kernel": "whole sweep (training dominates)", "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                     "peak_note": f"algorithmic train flop per sample (818,176 / 2,898,944); 3xTF32 peak = "
                                  f"{src} bf16 {bf16} / 6"},
        "e2e": {"value": samples / secs, "unit": "samples/s", "h2d_bytes_per_step": None,
                "d2h_bytes_per_step": None,
                "note": "the sweep is end to end by construction: host sampling, pool upload and the AUC "
                        "readback are inside each timed sweep"},
        "gpu_launches": None,
        "clocks": clk.summary(),
        "cpu_baseline": None,
    }
    if comm is not None:
        comm.close()
    if rank == 0 and world == 1 and cpu:
        v, rec = cpu_c1_sample()
        rec["sample"] += f"; the full C5 sweep at this rate would take {samples / v / 3600:.2f} h"
        out["cpu_baseline"] = rec
    return out


def cpu_c1_sample(threads=None, steps=8):
    """784-256-10 SGD steps (B = 128), one model per thread (the C1/C5 model)"""
    import ctypes as C

    po, R = _ref()
    if R is None:
        return None, None
    threads = threads or cpu_threads()
    secs = R.ref_bench_train(threads, 2, (C.c_int * 3)(784, 256, 10), 128, 0, steps, 0.0, 5)
    v = threads * steps * 128 / secs
    sample = f"{threads} 784-256-10 models x {steps} SGD steps of 128 rows, one model per thread"
    return v, _cpu_record(po, R, "reference", threads, sample, v, "samples/s", secs)


# ----------------------------------------------------------------------------- C2 (headline)
def measure_c2(args, world, rank, local):
    import torch

    from paper_2011_09463_b200 import api

    ctx = api.Context(local)
    bank = api.Bank(ctx, G, DIMS)
    rng = api.Rng(20110946 + rank)
    for g in range(G):
        bank.init_params(g, rng)
    gen = torch.Generator(device="cuda").manual_seed(1000 + rank)
    X = torch.randn((G, B, DIMS[0]), device="cuda", generator=gen)
    X[:, SRC:, :] += 0.5  # target-domain shift
    y = torch.randint(0, DIMS[-1], (G, B), device="cuda", dtype=torch.int32, generator=gen)
    step_kw = dict(lr=LR, src_rows=SRC, mmd_lambda=LAMBDA)

    def step():
        bank.train_step(X, y, want_loss=False, **step_kw)

    for _ in range(max(args.warmup, 3)):  # warm-up (device-resident inputs)
        step()
    torch.cuda.synchronize()
    n0 = ctx.launches
    ms, clocks = timed(world, local, args.steps, step)
    launches = ctx.launches - n0
    ms_step = ms / args.steps
    value = world * G * B * args.steps / (ms / 1000.0)

    # per-phase kernel timing (CUDA events on the launching streams)
    ctx.set_timing(True)
    for _ in range(args.steps):
        step()
    ph = ctx.phase_times()
    ctx.set_timing(False)
    # algorithmic flops per step, per phase (target rows are labelled, so every
    # row pays the full 2,898,944 flop/sample of BASELINE.md's C2 source row).
    # The head's DX rides on the MMD gradient GEMM (mmd_pairs phase) and the
    # head's dW runs on the side stream, so dx/dw hold the hidden layers only.
    macs = [DIMS[l] * DIMS[l + 1] for l in range(len(DIMS) - 1)]
    phase_flop = {"fwd_gemm": 2 * G * B * sum(macs), "dx_gemm": 2 * G * B * sum(macs[1:-1]),
                  "dw_gemm": 2 * G * B * sum(macs[:-1]),
                  "mmd_pairs": G * MMD_PAIRS * MMD_FLOP_PER_PAIR}
    step_flop = G * B * FLOP_SRC
    head_flop = 2 * G * B * macs[-1]
    assert phase_flop["fwd_gemm"] + phase_flop["dx_gemm"] + phase_flop["dw_gemm"] + 2 * head_flop == step_flop
    gemm_ms = sum(ph[p][0] for p in ("fwd_gemm", "dx_gemm", "dw_gemm")) / args.steps
    mmd_ms = ph["mmd_pairs"][0] / args.steps
    peak, bf16, src = fp32acc_peak()
    tf32_peak = bf16 / 2.0
    dominant = max(phase_flop, key=lambda p: ph[p][0])
    dom_ms = ph[dominant][0] / args.steps
    achieved = phase_flop[dominant] / (dom_ms / 1000.0) / 1e12

    # e2e through the C ABI with HOST buffers (H2D + loss/MMD D2H in the timed
    # region): mtk_bank_train_step_host_async copies step k's inputs on a copy
    # stream while step k-1 computes; every step's per-model loss and MMD are
    # read back (step k-1's right after step k is enqueued, the last at the end)
    Xh = X.cpu().pin_memory()
    yh = y.cpu().pin_memory()
    for _ in range(2):
        bank.train_step_host_async(Xh, yh, **step_kw)
        bank.step_result(0)
    torch.cuda.synchronize()
    state = {"k": 0}

    def e2e_step():
        bank.train_step_host_async(Xh, yh, **step_kw)
        if state["k"] > 0:
            bank.step_result(1)
        state["k"] += 1

    e2e_ms, _ = timed(world, local, args.steps, e2e_step)
    t0 = time.perf_counter()
    bank.step_result(0)  # the last step's result: host wait, added to the e2e time
    e2e_ms += 1000.0 * (time.perf_counter() - t0)
    e2e_value = world * G * B * args.steps / (e2e_ms / 1000.0)
    traffic, traffic_src = kernel_traffic(dominant)
    line = {
        "metric": "shadow-model train samples/s",
        "value": value,
        "unit": "samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD, "models_per_gpu": G, "global_batch": world * G * B,
                   "batch_per_model": B, "dims": DIMS, "parallelism": f"shard{world}",
                   "l2": "inputs 134 MB per step > 126 MB L2"},
        "mmd": {"pairs_per_s": world * G * MMD_PAIRS * args.steps / (ms / 1000.0),
                "unique_pairs_per_step": world * G * MMD_PAIRS,
                "kernel_ms_per_step": mmd_ms,
                "kernel_tflops": phase_flop["mmd_pairs"] / (mmd_ms / 1000.0) / 1e12 if mmd_ms else None,
                "kernel_frac": (phase_flop["mmd_pairs"] / (mmd_ms / 1000.0) / 1e12 / peak) if mmd_ms else None},
        "phases_ms_per_step": {p: ph[p][0] / args.steps for p in ph},
        "roofline": {"bound": "tensor", "kernel": dominant,
                     "launches_per_step": ph[dominant][1] / args.steps, "achieved": achieved,
                     "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "peak_note": (f"fp32-accurate tensor peak = 3xTF32 = tf32/3 = {src} bf16 "
                                   f"{bf16} TFLOP/s / 6; frac vs plain tf32 "
                                   f"{achieved / tf32_peak:.3f}, vs bf16 {achieved / bf16:.3f}"),
                     "traffic_note": (f"DRAM read+write bytes per step of the {dominant} "
                                      f"phase's {ph[dominant][1] / args.steps:.0f} launch(es), "
                                      f"profiles/{traffic_src} (one ncu --set full capture)")},
        "step_tflops": step_flop / (ms_step / 1000.0) / 1e12,
        "step_frac": step_flop / (ms_step / 1000.0) / 1e12 / peak,
        "gemm_tflops": (step_flop - 2 * head_flop) / (gemm_ms / 1000.0) / 1e12 if gemm_ms else None,
        "cpu_baseline": None,
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": G * B * DIMS[0] * 4 + G * B * 4,
                "d2h_bytes_per_step": 2 * G * 8},
        "gpu_launches": launches,
        "clocks": clocks,
    }
    del bank, X, y, Xh, yh
    torch.cuda.empty_cache()
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="C2 line without the c4 / attack sub-objects")
    ap.add_argument("--workload", default="c2", choices=["c2", "c4", "attack", "c3", "c5"],
                    help="c2 (default, the headline + c4 / attack sub-objects), c4, attack, c3, c5")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference_arm(args, int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")))
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        self_launch(args)
    world, rank, local = dist_setup(args.gpus)
    cpu = not args.no_cpu_baseline
    try:
        if args.workload == "c2":
            line = measure_c2(args, world, rank, local)
            if not args.no_sub:
                line["c4"] = measure_c4(args, world, rank, local, steps=max(3, args.steps // 4),
                                        warmup=3, cpu=cpu)
                line["attack"] = measure_attack(args, world, rank, local, steps=args.steps,
                                                warmup=max(args.warmup, 3), cpu=cpu)
            if rank == 0 and world == 1 and cpu:
                line["cpu_baseline"] = cpu_c2()[1]
        else:
            fn = {"c4": measure_c4, "attack": measure_attack, "c3": measure_c3, "c5": measure_c5}[args.workload]
            line = fn(args, world, rank, local, steps=args.steps, warmup=max(args.warmup, 3), cpu=cpu)
            line.update({"warmup": args.warmup, "vs_baseline": None, "data": "synthetic"})
        if rank == 0:
            print(json.dumps(line), flush=True)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
