"""Benchmark: shadow-model train samples/s (+ MMD pairs/s) on B200.

Workload (BASELINE.json configs[1], C2): mapping-based MMD transfer step of
MLP 1024-512-256-10 with a 512 source + 512 target batch and 5-bandwidth
Gaussian MMD on the 256-d hidden layer (CE + lambda*MMD, SGD), run for a
bank of G=32 shadow models per GPU (C5's per-GPU, per-paradigm shadow
share: 3 x 256 shadows / 8 GPUs / 3).  Weak scaling: every rank trains its
own 32 shadows; no data-path collective (models are independent, SURVEY.md
section 8(e)).  One step = one SGD step of all 32 models.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
  python bench.py --workload c4      # MMD stress (configs[3]): kernel pairs/s, row-sharded
  python bench.py --workload attack  # attack stage over 2^20 queries (configs[4] share)

Prints ONE JSON line on rank 0 (contract in the task description).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = [1024, 512, 256, 10]
G = 32
SRC, TGT = 512, 512
B = SRC + TGT
LAMBDA = 1.0
LR = 0.01
N_BW = 5
# algorithmic cost
FLOP_SRC = 2_898_944
MMD_PAIRS = (B * (B - 1)) // 2  # 523,776 unique pairs per model per step
MMD_FLOP_PER_PAIR = 4 * DIMS[2]  # fwd 2d + bwd 2d
WORKLOAD = ("C2 mapping-based MMD transfer: MLP 1024-512-256-10, 512 src + 512 tgt, "
            "5-bandwidth Gaussian MMD (lambda=1) on the 256-d hidden layer, SGD; bank of 32 "
            "shadow models per GPU")


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d.get("bf16_tflops"), d.get("bf16_tflops_sustained"), d.get("hbm_gbs"), "measured"
    return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """SM clock + throttle reasons via NVML, polled every 1 ms in a thread, for
    the duration of the `with` block (the timed region)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
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
                    time.sleep(0.001)

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
                "reasons": reasons, "samples": len(sm), "source": "nvml, 1 ms poll"}


def dist_setup(n_gpus):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local)
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


# ----------------------------------------------------------------------------- CPU arms
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_reference_sample(steps_per_thread=1, threads=None):
    """Reference CPU path on the host cores: one C2 model per std::thread, each
    running reference-Tape SGD steps (tape.hpp / optim.hpp, headers compiled
    unmodified) + the oracle's f64 MMD injection.  Returns (samples/s, info)."""
    import ctypes as C

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle as po

    threads = threads or cpu_threads()
    R = po.ref()
    dims = (C.c_int * 4)(*DIMS)
    if R is not None:
        secs = R.ref_bench_train(threads, 3, dims, B, SRC, steps_per_thread, LAMBDA, 1234)
        kind = "reference"
    else:  # oracle port (C restatement) in Python threads; ctypes drops the GIL
        import numpy as np

        def one(seed):
            r = po.Rng(seed)
            W, b = po.mlp_init(r, DIMS)
            X = r.normals(B * DIMS[0]).reshape(B, DIMS[0])
            y = np.array([r.below(10) for _ in range(B)], dtype=np.int32)
            for _ in range(steps_per_thread):
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
    samples = threads * steps_per_thread * B
    return samples / secs, {
        "kind": kind, "cores": threads,
        "sample": f"{threads} C2 models x {steps_per_thread} SGD step(s) of {B} samples "
                  f"(512 src + 512 tgt, 5-bw MMD), one model per thread",
        "seconds": secs}


def run_reference_arm(args, world, rank):
    if rank != 0:
        return
    for _ in range(args.warmup if args.warmup < 1 else 1):
        cpu_reference_sample(1)
    t = []
    for _ in range(args.steps):
        v, info = cpu_reference_sample(1)
        t.append(info["seconds"])
    secs = sum(t)
    value = args.steps * info["cores"] * B / secs
    line = {
        "metric": "shadow-model train samples/s", "value": value, "unit": "samples/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * secs / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "impl": "reference",
        "config": {"workload": WORKLOAD + " (CPU: one model per host thread)",
                   "global_batch": info["cores"] * B, "parallelism": "threads"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": info["cores"],
                         "kind": info["kind"], "sample": info["sample"]},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def kernel_traffic(phase):
    """DRAM read+write bytes per step of a phase's kernels (the same launches
    `achieved` is timed over), from the newest committed ncu --set full capture
    summary (profiles/rNN_kernels.json).  Returns (bytes or None, source file)."""
    import glob

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r[0-9]*_kernels.json")))
    if not files:
        return None, None
    with open(files[-1]) as f:
        d = json.load(f)
    ent = d.get("phases", {}).get(phase)
    return (ent.get("dram_bytes_per_step") if ent else None), os.path.basename(files[-1])


# ----------------------------------------------------------------------------- C4 MMD
C4_M, C4_N, C4_D = 65536, 8192, 512
C4_PAIRS = C4_M * (C4_M - 1) // 2 + C4_N * (C4_N - 1) // 2 + C4_M * C4_N  # 2,717,872,128


def run_c4_arm(args, world, rank, local):
    """configs[3]: multi-bandwidth MMD^2 + gradient of Xs [65536, 512] vs Xt
    [8192, 512].  One step = the full evaluation, pair rows sharded over the
    ranks (strong scaling); the ranks' raw sums would be combined in ascending
    rank order (section 8(e))."""
    import torch

    from paper_2011_09463_b200 import api

    torch.cuda.set_device(local)
    ctx = api.Context(local)
    gen = torch.Generator(device="cuda").manual_seed(4)
    Nt = C4_M + C4_N
    Z = torch.randn(Nt, C4_D, device="cuda", generator=gen)  # [Xs; Xt] in one block
    Z[C4_M:] += 0.1
    Xs, Xt = Z[:C4_M], Z[C4_M:]
    gZ = torch.empty_like(Z)
    gXs, gXt = gZ[:C4_M], gZ[C4_M:]
    beta = api.mmd_beta(ctx, Xs, Xt)
    r0, r1 = rank * Nt // world, (rank + 1) * Nt // world
    # one GPU: the full evaluation on the materialised kernel matrix (each
    # unordered 128x128 tile pair once, W = 21.7 GB, then V = W.Z as a GEMM);
    # N GPUs: pair rows sharded over the ranks (fused pair kernel)
    full = world == 1

    def evaluate():
        if full:
            api.mmd_gaussian(ctx, Xs, Xt, beta=beta)
        else:
            api.mmd_gaussian_rows(ctx, Xs, Xt, beta, r0, r1, gXs=gXs, gXt=gXt)

    for _ in range(max(args.warmup, 1)):
        evaluate()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            evaluate()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    launches = ctx.launches - launches0
    if rank != 0:
        return
    bf16, _, _, src = peaks()
    fp32acc_peak = bf16 / 2.0 / 3.0
    pairs_s = C4_PAIRS * args.steps / (ms / 1000.0)
    achieved = pairs_s * 4 * C4_D / 1e12
    line = {
        "metric": "MMD kernel-pairs/s", "value": pairs_s, "unit": "pairs/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": "C4 MMD stress: Xs 65536 x 512 vs Xt 8192 x 512 (N(0,1), N(0.1,1)), "
                               "5-bandwidth Gaussian MMD^2 + gradient, pair rows sharded over ranks",
                   "unique_pairs": C4_PAIRS, "parallelism": f"rows{world}",
                   "path": "materialised W (mmd_w + wsum + V GEMM)" if full else "fused pair kernel, row shards",
                   "l2": "inputs 151 MB + tf32 planes > 126 MB L2"},
        "roofline": {"bound": "tensor", "kernel": "mmd_w + V GEMM (+prep)" if full else "mmd_tc_kernel (+prep, grad finish)",
                     "achieved": achieved, "peak": fp32acc_peak, "unit": "TFLOP/s",
                     "frac": achieved / fp32acc_peak, "traffic": None,
                     "peak_note": f"algorithmic 4d flop per unique pair; 3xTF32 peak = {src} bf16 / 6; "
                                  + ("GEMM1 visits unique pairs, V = W.Z every ordered pair" if full else
                                     "the kernel evaluates ordered pairs (2x the algorithmic work)")},
        "cpu_baseline": None,
        "e2e": None,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- attack
ATT_Q = 1 << 20


def run_attack_arm(args, world, rank, local):
    """Attack stage of configs[4] on one paradigm's 2^20 member/non-member
    queries per rank: posterior top-3 features -> attack MLP 3-64-2 -> member
    score -> AUC + accuracy.  Reports queries/s and the streaming kernels'
    achieved HBM bandwidth on algorithmic bytes."""
    import torch

    from paper_2011_09463_b200 import api

    torch.cuda.set_device(local)
    ctx = api.Context(local)
    gen = torch.Generator(device="cuda").manual_seed(5 + rank)
    logits = torch.randn(ATT_Q, 10, device="cuda", generator=gen)
    labels = (torch.rand(ATT_Q, device="cuda", generator=gen) < 0.5).to(torch.uint8)
    logits[labels.bool(), 0] += 1.0  # members look more confident
    att = api.Bank(ctx, 1, [3, 64, 2])
    rng = api.Rng(77)
    att.init_params(0, rng)

    def step():  # mtk_attack_auc: one streaming scoring kernel + the AUC sort / count
        return api.attack_auc(att, logits, labels)

    for _ in range(max(args.warmup, 1)):
        step()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            auc, acc = step()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    launches = ctx.launches - launches0
    if rank != 0:
        return
    _, _, hbm, src = peaks()
    # algorithmic bytes per query: logits 40 + label 1 read, two AUC keys written (8);
    # the sort reads and writes the 4-B keys (one pass counted), the count reads
    # label + member key + ~1 probe (9)
    bytes_q = 40 + 1 + 8 + 2 * 4 + 9
    qps = world * ATT_Q * args.steps / (ms / 1000.0)
    gbs = qps * bytes_q / world / 1e9
    line = {
        "metric": "membership-attack queries/s", "value": qps, "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "attack stage: 2^20 queries x 10-class posteriors -> top-3 "
                               "features -> attack MLP 3-64-2 -> score -> AUC/accuracy per rank",
                   "queries_per_gpu": ATT_Q, "parallelism": f"shard{world}", "auc": auc,
                   "accuracy": acc},
        "roofline": {"bound": "hbm", "kernel": "attack_score + AUC sort/count (whole stage)",
                     "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm if hbm else None,
                     "traffic": None,
                     "peak_note": f"{src} HBM copy bandwidth; {bytes_q} algorithmic B/query"},
        "cpu_baseline": None,
        "e2e": None,
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def run_gpu_arm(args, world, rank, local):
    import numpy as np
    import torch

    from paper_2011_09463_b200 import api

    torch.cuda.set_device(local)
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

    # warm-up (device-resident inputs)
    for _ in range(max(args.warmup, 3)):
        bank.train_step(X, y, want_loss=False, **step_kw)
    torch.cuda.synchronize()

    # ---- timed region: K steps, inputs resident in HBM ----------------------------
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = ctx.launches
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            bank.train_step(X, y, want_loss=False, **step_kw)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    launches = ctx.launches - launches0
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    ms_step = ms / args.steps
    samples = world * G * B * args.steps
    value = samples / (ms / 1000.0)

    # ---- per-phase kernel timing (CUDA events on the launching stream) ---------------
    ctx.set_timing(True)
    for _ in range(args.steps):
        bank.train_step(X, y, want_loss=False, **step_kw)
    ph = ctx.phase_times()
    ctx.set_timing(False)
    # algorithmic flops per step, per phase (target rows are labelled, so every
    # row pays the full 2,898,944 flop/sample of BASELINE.md's C2 source row)
    # Where the layers' work runs: the head's DX rides on the MMD gradient GEMM
    # (mmd_pairs phase) and the head's dW runs on the side stream (side_stream
    # phase, overlapped), so the dx/dw phases hold the hidden layers only.
    macs = [DIMS[l] * DIMS[l + 1] for l in range(len(DIMS) - 1)]
    phase_flop = {"fwd_gemm": 2 * G * B * sum(macs), "dx_gemm": 2 * G * B * sum(macs[1:-1]),
                  "dw_gemm": 2 * G * B * sum(macs[:-1]),
                  "mmd_pairs": G * MMD_PAIRS * MMD_FLOP_PER_PAIR}
    step_flop = G * B * FLOP_SRC
    head_flop = 2 * G * B * macs[-1]  # each of the head's DX and dW
    assert phase_flop["fwd_gemm"] + phase_flop["dx_gemm"] + phase_flop["dw_gemm"] + 2 * head_flop == step_flop
    gemm_ms = sum(ph[p][0] for p in ("fwd_gemm", "dx_gemm", "dw_gemm")) / args.steps
    mmd_ms = ph["mmd_pairs"][0] / args.steps
    mmd_flop = phase_flop["mmd_pairs"]
    bf16, bf16_s, hbm, src = peaks()
    tf32_peak = bf16 / 2.0  # dense tf32 tensor rate is half the bf16 rate
    fp32acc_peak = tf32_peak / 3.0  # three tf32 MMAs per fp32-accurate product
    dominant = max(phase_flop, key=lambda p: ph[p][0])
    dom_ms = ph[dominant][0] / args.steps  # this phase's launches per step, summed
    achieved = phase_flop[dominant] / (dom_ms / 1000.0) / 1e12

    # ---- e2e: through the C ABI with HOST buffers (H2D + loss D2H in the timed region).
    # mtk_bank_train_step_host_async copies step k's inputs on a copy stream while
    # step k-1 computes; every step's per-model loss and MMD are read back to the
    # host (step k-1's right after step k is enqueued, the last one at the end).
    Xh = X.cpu().pin_memory()
    yh = y.cpu().pin_memory()
    for _ in range(2):
        bank.train_step_host_async(Xh, yh, **step_kw)
        bank.step_result(0)
    torch.cuda.synchronize()
    barrier(world)
    e0.record(stream)
    for k in range(args.steps):
        bank.train_step_host_async(Xh, yh, **step_kw)
        if k > 0:
            bank.step_result(1)
    bank.step_result(0)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks(e0.elapsed_time(e1), world)
    e2e_value = world * G * B * args.steps / (e2e_ms / 1000.0)
    h2d = G * B * DIMS[0] * 4 + G * B * 4
    d2h = 2 * G * 8
    traffic, traffic_src = kernel_traffic(dominant)

    if rank != 0:
        return
    cpu = None
    if not args.no_cpu_baseline:
        cv, info = cpu_reference_sample(1)
        cpu = {"value": cv, "unit": "samples/s", "cores": info["cores"], "kind": info["kind"],
               "sample": info["sample"]}
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
                "kernel_tflops": mmd_flop / (mmd_ms / 1000.0) / 1e12 if mmd_ms else None},
        "phases_ms_per_step": {p: ph[p][0] / args.steps for p in ph},
        "roofline": {"bound": "tensor", "kernel": dominant,
                     "launches_per_step": ph[dominant][1] / args.steps, "achieved": achieved,
                     "peak": fp32acc_peak, "unit": "TFLOP/s", "frac": achieved / fp32acc_peak,
                     "traffic": traffic,
                     "peak_note": (f"fp32-accurate tensor peak = 3xTF32 = tf32/3 = {src} bf16 "
                                   f"{bf16} TFLOP/s / 6; frac vs plain tf32 "
                                   f"{achieved / tf32_peak:.3f}, vs bf16 {achieved / bf16:.3f}"),
                     "traffic_note": (f"DRAM read+write bytes per step of the {dominant} "
                                      f"phase's {ph[dominant][1] / args.steps:.0f} launch(es), "
                                      f"profiles/{traffic_src} (one ncu --set full capture)")},
        "step_tflops": step_flop / (ms_step / 1000.0) / 1e12,
        "gemm_tflops": (step_flop - 2 * head_flop) / (gemm_ms / 1000.0) / 1e12 if gemm_ms else None,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="c2", choices=["c2", "c4", "attack"],
                    help="c2 (default, the headline), c4 MMD stress, attack stage")
    args = ap.parse_args()
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference_arm(args, world, rank)
        return
    world, rank, local = dist_setup(args.gpus)
    try:
        {"c2": run_gpu_arm, "c4": run_c4_arm, "attack": run_attack_arm}[args.workload](
            args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
