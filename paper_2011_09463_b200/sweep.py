"""Shadow-training sweep and membership-inference attack (SURVEY.md section 8
rows a17/a18; Appendix A of SURVEY.md).

The reference has no code for this stage; the definitions pinned here are:

* data: class-conditional Gaussians, y = below(C), x = mu_y + N(0, I) on the
  host RNG (rng.hpp semantics, bit-exact); the target domain adds a fixed
  shift delta (D^S, D^T, N^S >> N^T);
* data_rng = "counter": mu / shift as above, but the
  two pools come from the device counter-based generator (mtk_synth_counter:
  Philox4x64-10 keyed {seed, 1} for the target pool, {seed, 2} for the
  source pool), generated straight into HBM -- the host Box-Muller stream is
  the C5 wall-clock floor otherwise.  A different (documented) stream, so
  "counter" results differ from "host" ones; the oracle backend restates it;
* streams: root = Rng(seed); data = root.split(0); model k (0 = target,
  1..S = shadows) = root.split(k + 1), derived in ascending k on every rank
  (rng.hpp:65-69: split advances the parent);
* per model k: perm = permutation(pool) -> members = perm[:n_mem],
  non-members = perm[n_mem:2 n_mem]; then parameter init; then
  one permutation(n_mem) per epoch for the batch order; a
  short last batch is padded with weight-0 duplicates;
* paradigms:
    model     -- pretrain on a source subset, then fine-tune on the members
                 (optionally with a frozen prefix);
    mapping   -- co-train on [source batch ; member batch] with CE on both and
                 lambda * MMD^2(h_src, h_tgt) on the last hidden layer;
    parameter -- shared trunk, a source head and a target head; each step
                 feeds [source batch ; member batch] (rows split by head);
* attack: top-k sorted posteriors of the target-domain head; an MLP
  k -> 64 -> 2 trained with CE + SGD on the shadows' members (1) and
  non-members (0); it scores the target's members / non-members -> AUC
  (mid-rank Mann-Whitney) and accuracy at 0.5.

The product path is ``GpuBackend`` (libmtk through ``api``).  The driver is
written against a small backend interface so tests can replay it on the CPU
oracle; nothing here imports the oracle.
"""
from __future__ import annotations

import dataclasses
import json
from typing import Any

import numpy as np


@dataclasses.dataclass
class SweepConfig:
    paradigm: str = "model"          # model | mapping | parameter
    dims: tuple = (784, 256, 10)
    n_shadows: int = 4
    pool: int = 8192                 # target-domain population
    members: int = 2048              # per model; as many non-members
    source_pool: int = 16384         # source-domain population (N^S >> N^T)
    source_per_model: int = 4096     # source rows each model sees
    batch: int = 128
    epochs: int = 10
    pretrain_epochs: int = 2         # model-based
    frozen_layers: int = 0           # model-based fine-tuning
    lr: float = 0.05
    optimizer: str = "sgd"           # sgd | adam (optim.hpp:30-68) for target/shadows
    mmd_lambda: float = 1.0          # mapping-based
    mu_scale: float = 0.1
    shift_scale: float = 0.5
    k: int = 3
    attack_hidden: int = 64
    attack_epochs: int = 30
    attack_batch: int = 1024
    attack_lr: float = 0.1
    attack_optimizer: str = "sgd"
    data_rng: str = "host"           # host (mt::Rng, bit-exact) | counter (device Philox)
    seed: int = 20110946

    def validate(self):
        from .errors import ConfigError

        if self.paradigm not in ("model", "mapping", "parameter"):
            raise ConfigError(f"unknown paradigm {self.paradigm!r}")
        if 2 * self.members > self.pool:
            raise ConfigError("members + non-members exceed the pool")
        if self.source_per_model > self.source_pool:
            raise ConfigError("source_per_model exceeds source_pool")
        if len(self.dims) < 2 or (self.paradigm != "model" and len(self.dims) < 3):
            raise ConfigError("transfer paradigms need a hidden layer")
        if not 1 <= self.k <= self.dims[-1]:
            raise ConfigError("k must be in [1, C]")
        for o in (self.optimizer, self.attack_optimizer):
            if o not in ("sgd", "adam"):
                raise ConfigError(f"unknown optimizer {o!r}")
        if self.data_rng not in ("host", "counter"):
            raise ConfigError(f"unknown data_rng {self.data_rng!r} (host | counter)")


# --------------------------------------------------------------------------- data
class Population:
    """Source and target pools: drawn from the host data stream (bit-exact
    mt::Rng), or with data_rng = "counter" by the backend's counter-based
    generator (device pools for the GPU backend)."""

    def __init__(self, cfg: SweepConfig, rng_cls, synth_counter=None):
        from .errors import ConfigError

        C, d = cfg.dims[-1], cfg.dims[0]
        self.root = rng_cls(cfg.seed)
        data = self.root.split(0)
        self.mu = cfg.mu_scale * data.normals(C * d).reshape(C, d)
        self.shift = cfg.shift_scale * data.normals(d)
        if cfg.data_rng == "counter":
            if synth_counter is None:
                raise ConfigError("data_rng 'counter' needs a backend with synth_counter")
            self.Xt, self.yt = synth_counter(cfg.seed, 1, cfg.pool, self.mu, self.shift)
            self.Xs, self.ys = synth_counter(cfg.seed, 2, cfg.source_pool, self.mu, None)
            return
        self.Xt, self.yt = synth(data, C, d, cfg.pool, self.mu, self.shift)
        self.Xs, self.ys = synth(data, C, d, cfg.source_pool, self.mu, None)

    def model_streams(self, n_models: int):
        # ascending k on one root: stream k+1 for model k
        return [self.root.split(k + 1) for k in range(n_models)]


def synth(rng, C, d, n, mu, shift):
    out = rng.synth(C, d, n, mu, shift)
    return out[0], out[1]


def host_gather(parts):
    """[(X_pool, y_pool, idx[G][nb]), ...] -> X [G, sum nb, d], y [G, sum nb] (rows
    concatenated in part order)."""
    Xs = [np.stack([X[i] for i in idx]) for X, _, idx in parts]
    ys = [np.stack([y[i] for i in idx]).astype(np.int32) for _, y, idx in parts]
    return np.concatenate(Xs, axis=1), np.concatenate(ys, axis=1)


def batches(order: np.ndarray, B: int):
    """batch_iter semantics: consecutive slices of the seeded order; the short
    last batch is padded with weight-0 duplicates."""
    out = []
    for s in range(0, len(order), B):
        idx = order[s:s + B]
        w = np.ones(B, dtype=np.float32)
        if len(idx) < B:
            pad = B - len(idx)
            w[len(idx):] = 0.0
            idx = np.concatenate([idx, np.repeat(idx[-1:], pad)])
        out.append((idx.astype(np.int64), w))
    return out


# --------------------------------------------------------------------------- backend
class GpuBackend:
    """The product path: libmtk (CUDA sm_100a) through the C ABI."""

    def __init__(self, device: int = 0):
        import torch

        from . import api

        self.torch, self.api = torch, api
        self.ctx = api.Context(device)
        self.Rng = api.Rng
        self.device = torch.device("cuda", device)

    def bank(self, G, dims, n_heads=1):
        return self.api.Bank(self.ctx, G, list(dims), n_heads=n_heads)

    def init(self, bank, g, rng):
        bank.init_params(g, rng)

    def to_dev(self, a):
        if isinstance(a, self.torch.Tensor):
            return a
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def synth_counter(self, seed, stream, n, mu, shift):
        """pool generated on the device (mtk_synth_counter); stays in HBM"""
        torch = self.torch
        return self.api.synth_counter(self.ctx, seed, stream, n, torch.from_numpy(np.asarray(mu)),
                                      None if shift is None else torch.from_numpy(np.asarray(shift)))

    def _pool(self, X, y):
        if isinstance(X, self.torch.Tensor):  # device-resident pool (counter data, features)
            return X, self.to_dev(np.ascontiguousarray(y, dtype=np.int32)
                                  if not isinstance(y, self.torch.Tensor) else y)
        if not hasattr(self, "_pools"):
            self._pools = {}
        key = (id(X), id(y))
        if key not in self._pools:
            self._pools[key] = (X, y, self.to_dev(np.ascontiguousarray(X, dtype=np.float32)),
                                self.to_dev(np.ascontiguousarray(y, dtype=np.int32)))
        return self._pools[key][2], self._pools[key][3]

    def train_epoch(self, bank, X, y, idx, w, denom0, **kw):
        Xd, yd = self._pool(X, y)
        bank.train_epoch(Xd, yd, self.to_dev(np.ascontiguousarray(idx, dtype=np.int64)),
                         self.to_dev(np.ascontiguousarray(w, dtype=np.float32)), denom0, **kw)

    def gather(self, parts):
        """Batch assembly on the device: parts = [(X_pool, y_pool, idx[G][nb]), ...]
        concatenated along rows; pools are uploaded once (mtk_gather_rows)."""
        torch = self.torch
        G = len(parts[0][2])
        rows = sum(len(p[2][0]) for p in parts)
        d = parts[0][0].shape[1]
        Xo = torch.empty((G, rows, d), device=self.device, dtype=torch.float32)
        yo = torch.empty((G, rows), device=self.device, dtype=torch.int32)
        r0 = 0
        for X, y, idx in parts:
            Xd, yd = self._pool(X, y)
            ix = self.to_dev(np.ascontiguousarray(np.stack(idx), dtype=np.int64))
            self.api.gather_rows(self.ctx, Xd, ix, Xo, r0)
            self.api.gather_rows(self.ctx, yd, ix, yo.view(G, rows, 1), r0)
            r0 += ix.shape[1]
        return Xo, yo

    def step(self, bank, X, y, w, **kw):
        return bank.train_step(self.to_dev(X), self.to_dev(y), self.to_dev(w), want_loss=False,
                               **kw)

    def features(self, bank, X, head, k):
        """[G, rows, k] top-k posteriors; stays on the device"""
        X = self.to_dev(X)
        logits = bank.forward(X, head=head)
        return self.api.posterior_features(self.ctx, logits, k).reshape(X.shape[0], X.shape[1], k)

    def all_gather(self, F):
        """the feature all-gather over NCCL (mtk_allgather), device to device;
        needs an initialised torch.distributed group (used for the NCCL id)"""
        if getattr(self, "comm", None) is None:
            self.comm = self.api.Comm(self.ctx)
        return list(self.comm.all_gather(F.contiguous()).unbind(0))

    def attack_scores(self, bank, F):
        logits = bank.forward(self.to_dev(F)[None].contiguous(), head=0)
        return self.api.posterior_column(self.ctx, logits, 1)

    def auc(self, scores, labels):
        torch = self.torch
        sc = scores if isinstance(scores, torch.Tensor) else self.to_dev(scores.astype(np.float32))
        return self.api.auc(self.ctx, sc, self.to_dev(np.ascontiguousarray(labels, dtype=np.uint8)))


# --------------------------------------------------------------------------- training
def train_bank(be, cfg: SweepConfig, pop: Population, streams, models: list[int]):
    """Train the given models (indices into `streams`) as one bank.
    Returns (bank, members[G], non_members[G])."""
    G = len(models)
    two = cfg.paradigm == "parameter"
    bank = be.bank(G, cfg.dims, n_heads=2 if two else 1)
    mem, non, src = [], [], []
    for g, k in enumerate(models):
        r = streams[k]
        perm = r.permutation(cfg.pool)
        mem.append(perm[:cfg.members])
        non.append(perm[cfg.members:2 * cfg.members])
        be.init(bank, g, r)
        src.append(r.permutation(cfg.source_pool)[:cfg.source_per_model])
    B = cfg.batch
    d = cfg.dims[0]

    gather_parts = getattr(be, "gather", None) or host_gather

    def gather(X, y, idx_per_model):
        return gather_parts([(X, y, idx_per_model)])

    if cfg.paradigm == "model" and cfg.pretrain_epochs > 0:
        for _ in range(cfg.pretrain_epochs):
            orders = [batches(streams[k].permutation(cfg.source_per_model), B) for k in models]
            for t in range(len(orders[0])):
                idx = [src[g][orders[g][t][0]] for g in range(G)]
                w = np.stack([orders[g][t][1] for g in range(G)])
                Xb, yb = gather(pop.Xs, pop.ys, idx)
                be.step(bank, Xb, yb, w, lr=cfg.lr, denom=(float(w[0].sum()), 0.0),
                        optimizer=cfg.optimizer)
    for _ in range(cfg.epochs):
        orders = [batches(streams[k].permutation(cfg.members), B) for k in models]
        for t in range(len(orders[0])):
            idx = [mem[g][orders[g][t][0]] for g in range(G)]
            w = np.stack([orders[g][t][1] for g in range(G)])
            if cfg.paradigm == "model":
                Xb, yb = gather(pop.Xt, pop.yt, idx)
                be.step(bank, Xb, yb, w, lr=cfg.lr, frozen_layers=cfg.frozen_layers,
                        denom=(float(w[0].sum()), 0.0), optimizer=cfg.optimizer)
                continue
            # co-training: a source batch rides along with every member batch
            sidx = [src[g][(t * B + np.arange(B)) % cfg.source_per_model] for g in range(G)]
            Xc, yc = gather_parts([(pop.Xs, pop.ys, sidx), (pop.Xt, pop.yt, idx)])
            wc = np.concatenate([np.ones_like(w), w], axis=1)
            if cfg.paradigm == "mapping":
                be.step(bank, Xc, yc, wc, lr=cfg.lr, src_rows=B, mmd_lambda=cfg.mmd_lambda,
                        denom=(float(wc[0].sum()), 0.0), optimizer=cfg.optimizer)
            else:
                be.step(bank, Xc, yc, wc, lr=cfg.lr, src_rows=B,
                        denom=(float(B), float(w[0].sum())), optimizer=cfg.optimizer)
    return bank, mem, non


def query_features(be, cfg, pop, bank, mem, non):
    """Top-k posteriors of every model on its members and non-members:
    returns feats [G, 2*members, k] and labels [2*members] (1 = member)."""
    head = 1 if cfg.paradigm == "parameter" else 0
    G = len(mem)
    gather_parts = getattr(be, "gather", None) or host_gather
    X, _ = gather_parts([(pop.Xt, pop.yt, [np.concatenate([mem[g], non[g]]) for g in range(G)])])
    F = be.features(bank, X, head, cfg.k)
    lab = np.concatenate([np.ones(cfg.members, np.uint8), np.zeros(cfg.members, np.uint8)])
    return F, lab


def train_attack(be, cfg, F_train, lab_train, rng):
    """Attack MLP k -> hidden -> 2 with CE + SGD on shadow features."""
    bank = be.bank(1, (cfg.k, cfg.attack_hidden, 2))
    be.init(bank, 0, rng)
    n = len(lab_train)
    lab32 = np.ascontiguousarray(lab_train, dtype=np.int32)
    epoch_fn = getattr(be, "train_epoch", None)
    for _ in range(cfg.attack_epochs):
        bl = batches(rng.permutation(n), cfg.attack_batch)
        if epoch_fn is not None:  # the whole epoch in one library call
            idx = np.stack([b[0] for b in bl])[:, None, :]
            w = np.stack([b[1] for b in bl])[:, None, :]
            epoch_fn(bank, F_train, lab32, idx, w,
                     [float(b[1].sum()) for b in bl], lr=cfg.attack_lr,
                     optimizer=cfg.attack_optimizer)
            continue
        for idx, w in bl:
            be.step(bank, F_train[idx][None], lab_train[idx][None].astype(np.int32), w[None],
                    lr=cfg.attack_lr, denom=(float(w.sum()), 0.0), optimizer=cfg.attack_optimizer)
    return bank


def _is_torch(x) -> bool:
    return type(x).__module__.split(".")[0] == "torch"


def _cat(parts):
    if _is_torch(parts[0]):
        import torch

        return torch.cat(list(parts), 0)
    return np.concatenate(parts, axis=0)


def _f32(x):
    if _is_torch(x):
        import torch

        return x.to(torch.float32).contiguous()
    return np.ascontiguousarray(x, dtype=np.float32)


def model_blocks(M: int, world: int):
    """rank r trains the contiguous model block [r M / W, (r + 1) M / W)
    (SURVEY.md 8(e)); every model's RNG stream is root.split(k + 1) whatever
    the rank, so results do not depend on W"""
    return [(r * M // world, (r + 1) * M // world) for r in range(world)]


def gather_features(F, blocks, gather):
    """Combine the ranks' feature blocks [G_r, Q, k] into [M, Q, k] in model
    order with an EQUAL-size collective `gather` (an NCCL all-gather needs
    equal buffers): each block is padded to the largest G_r, gathered, and
    the padding trimmed again."""
    gmax = max(hi - lo for lo, hi in blocks)
    g = F.shape[0]
    if g < gmax:
        pad = (F[:1] * 0).repeat(gmax - g, 1, 1) if _is_torch(F) else np.zeros(
            (gmax - g,) + F.shape[1:], dtype=F.dtype)
        F = _cat([F, pad])
    parts = gather(F)
    if len(parts) != len(blocks):
        raise RuntimeError(f"feature gather returned {len(parts)} blocks for {len(blocks)} ranks")
    return _cat([p[:hi - lo] for p, (lo, hi) in zip(parts, blocks)])


def run_sweep(cfg: SweepConfig, be=None, *, rank: int = 0, world: int = 1,
              all_gather=None) -> dict[str, Any]:
    """One paradigm: train target + shadows (sharded over ranks), attack, AUC.

    Models [0, 1 + n_shadows) are split into contiguous rank blocks; the
    per-rank feature blocks are combined with ``all_gather`` (a callable
    taking this rank's block and returning the list over ranks), by default
    the backend's own (the GPU backend: NCCL over NVLink through
    mtk_allgather, device to device); with one rank it is the identity.
    """
    cfg.validate()
    be = be or GpuBackend()
    pop = Population(cfg, be.Rng, getattr(be, "synth_counter", None))
    M = 1 + cfg.n_shadows
    streams = pop.model_streams(M + 1)  # last stream drives the attack model
    blocks = model_blocks(M, world)
    lo, hi = blocks[rank]
    models = list(range(lo, hi))
    bank, mem, non = train_bank(be, cfg, pop, streams, models)
    F, lab = query_features(be, cfg, pop, bank, mem, non)
    gather = all_gather or (getattr(be, "all_gather", None) if world > 1 else None)
    if world > 1 and gather is None:
        raise RuntimeError("run_sweep: world > 1 needs an all_gather")
    F_all = gather_features(F, blocks, gather) if gather else F  # [M, 2*members, k], model order
    F_target, F_shadow = F_all[0], F_all[1:]
    Ftr = _f32(F_shadow.reshape(-1, cfg.k))
    ltr = np.tile(lab, cfg.n_shadows)
    attack = train_attack(be, cfg, Ftr, ltr, streams[M])
    scores = be.attack_scores(attack, _f32(F_target))
    auc, acc = be.auc(scores, lab)
    return {"paradigm": cfg.paradigm, "auc": auc, "accuracy": acc, "models": M,
            "rank_models": models, "n_queries": int(len(lab)),
            "config": dataclasses.asdict(cfg)}


# --------------------------------------------------------------------------- config / report
# Strict-JSON sweep configuration, metrics report and exit codes (SURVEY.md
# 8(f) f4, after SPEC.md:656-665, 686-697): unknown keys are rejected with a
# nearest-name suggestion, every violation is reported (not just the first),
# the resolved config (defaults injected) is echoed, and the report carries a
# digest of the resolved config.  Exit codes: 0 ok, 2 config, 3 data, 4 other.
REPORT_VERSION = 1


def _edit_distance(a: str, b: str) -> int:
    d = list(range(len(b) + 1))
    for i, ca in enumerate(a, 1):
        prev, d[0] = d[0], i
        for j, cb in enumerate(b, 1):
            prev, d[j] = d[j], min(d[j] + 1, d[j - 1] + 1, prev + (ca != cb))
    return d[-1]


def resolve_config(doc: dict) -> SweepConfig:
    """Strictly validate a JSON document into a SweepConfig (raises
    ConfigError listing every violation)."""
    from .errors import ConfigError

    if not isinstance(doc, dict):
        raise ConfigError("sweep config: the document must be a JSON object")
    fields = {f.name: f for f in dataclasses.fields(SweepConfig)}
    errs = []
    for k in doc:
        if k not in fields:
            near = min(fields, key=lambda f: _edit_distance(k, f))
            errs.append(f"unknown key {k!r} (did you mean {near!r}?)")
    kw = {}
    for name, f in fields.items():
        if name not in doc:
            continue
        v = doc[name]
        default = f.default
        if isinstance(default, bool) or not isinstance(default, (int, float, str, tuple)):
            kw[name] = v
            continue
        if isinstance(default, tuple):
            if not (isinstance(v, list) and all(isinstance(x, int) and not isinstance(x, bool) for x in v)):
                errs.append(f"{name}: expected a list of integers")
                continue
            kw[name] = tuple(v)
        elif isinstance(default, str):
            if not isinstance(v, str):
                errs.append(f"{name}: expected a string")
                continue
            kw[name] = v
        elif isinstance(default, int):
            if not (isinstance(v, int) and not isinstance(v, bool)):
                errs.append(f"{name}: expected an integer")
                continue
            kw[name] = v
        else:
            if not isinstance(v, (int, float)) or isinstance(v, bool):
                errs.append(f"{name}: expected a number")
                continue
            kw[name] = float(v)
    cfg = None
    if not errs:
        cfg = SweepConfig(**kw)
        try:
            cfg.validate()
        except ConfigError as e:
            errs.append(str(e))
    if errs:
        raise ConfigError("sweep config: " + "; ".join(errs))
    return cfg


def resolved_dict(cfg: SweepConfig) -> dict:
    return {k: list(v) if isinstance(v, tuple) else v for k, v in dataclasses.asdict(cfg).items()}


def config_digest(cfg: SweepConfig) -> str:
    import hashlib

    canon = json.dumps(resolved_dict(cfg), sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(canon.encode()).hexdigest()


def metrics_report(cfg: SweepConfig, result: dict, seconds: float) -> dict:
    """Deterministic fields first; only `wall_clock_seconds` varies between runs."""
    return {"report_version": REPORT_VERSION, "paradigm": cfg.paradigm,
            "auc": result["auc"], "accuracy": result["accuracy"], "models": result["models"],
            "n_queries": result["n_queries"], "config_digest": config_digest(cfg),
            "wall_clock_seconds": seconds}


EXIT_OK, EXIT_CONFIG, EXIT_DATA, EXIT_INTERNAL = 0, 2, 3, 4


def main(argv=None) -> int:
    """python -m paper_2011_09463_b200.sweep --config cfg.json [--output DIR]
    (or the quick flags); prints the metrics report; returns the exit code."""
    import argparse
    import os
    import sys
    import time

    from .errors import ConfigError, DataError

    ap = argparse.ArgumentParser(description="shadow-model membership-inference sweep")
    ap.add_argument("--config", help="strict JSON SweepConfig document")
    ap.add_argument("--output", help="directory for metrics.json and resolved_config.json")
    ap.add_argument("--paradigm", choices=["model", "mapping", "parameter"])
    ap.add_argument("--shadows", type=int)
    ap.add_argument("--epochs", type=int)
    ap.add_argument("--seed", type=int)
    a = ap.parse_args(argv)
    try:
        doc = {}
        if a.config:
            try:
                with open(a.config) as f:
                    doc = json.load(f)
            except OSError as e:
                raise DataError(f"sweep config: cannot read {a.config}: {e}") from e
            except json.JSONDecodeError as e:
                raise ConfigError(f"sweep config: not valid JSON: {e}") from e
        for flag, key in (("paradigm", "paradigm"), ("shadows", "n_shadows"), ("epochs", "epochs"),
                          ("seed", "seed")):
            if getattr(a, flag) is not None:  # flag > file > default
                doc[key] = getattr(a, flag)
        cfg = resolve_config(doc)
        # under torchrun: one rank per GPU, contiguous model blocks, the
        # feature all-gather over NCCL (mtk_allgather); rank 0 reports
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        kw = {}
        if world > 1:
            import torch
            import torch.distributed as dist

            local = int(os.environ.get("LOCAL_RANK", "0"))
            torch.cuda.set_device(local)
            if not dist.is_initialized():
                dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            kw = dict(be=GpuBackend(local), rank=rank, world=world)
        t0 = time.perf_counter()
        result = run_sweep(cfg, **kw)
        report = metrics_report(cfg, result, time.perf_counter() - t0)
        if rank != 0:
            return EXIT_OK
        if a.output:
            os.makedirs(a.output, exist_ok=True)
            with open(os.path.join(a.output, "resolved_config.json"), "w") as f:
                json.dump(resolved_dict(cfg), f, indent=1, sort_keys=True)
            with open(os.path.join(a.output, "metrics.json"), "w") as f:
                json.dump(report, f, indent=1)
        print(json.dumps(report))
        return EXIT_OK
    except ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except DataError as e:
        print(f"data error: {e}", file=sys.stderr)
        return EXIT_DATA
    except Exception as e:  # noqa: BLE001 - internal invariant violation
        print(f"internal error: {type(e).__name__}: {e}", file=sys.stderr)
        return EXIT_INTERNAL


if __name__ == "__main__":
    raise SystemExit(main())
