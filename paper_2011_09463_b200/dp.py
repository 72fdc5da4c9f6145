"""Deterministic data-parallel training of a replicated bank
("distributed-trainer").

One process per GPU (torch.distributed over NCCL); every rank holds a
bit-identical replica of the bank and trains on its round-robin shard of each
global batch:

  1. replica check: the order-independent parameter fingerprint of every rank
     is compared; a mismatch raises ConsistencyError;
  2. compute_grads: forward + backward of the shard into the flat gradient
     arena, cross-entropy with denominator global_rows / n so the shard mean
     keeps the large-batch algebra exact (tape.hpp:466-468);
  3. all-gather of the n arenas (one NCCL collective) into [n, arena];
  4. dp_apply: one kernel forms g = (sum over workers in ascending order) / n
     in fp64 and applies one SGD / Adam step.  Every rank
     reduces the same gathered bytes in the same order, so the replicas stay
     bit-identical with no parameter broadcast.

The gather + ordered sum is the reference's fixed-order reduction made
schedule-independent; an all-reduce would let NCCL pick the summation order.
``dp_step_local`` runs the same arithmetic with n simulated workers on one
device (the reference's own execution model).

(The analytic ring all-reduce speed-up model of SPEC.md:623-631 is not on
the north_star path -- SURVEY.md section 2 row 20 -- and is not built.)
"""
from __future__ import annotations


import numpy as np
import torch

from . import errors

# ---- sharding -------------------------------------------


def shard_batches(batch_size: int, n_workers: int) -> list[np.ndarray]:
    """Round-robin example indices per worker: worker r gets r, r+n, r+2n, ...
    (8 examples, n=4 -> {0,4},{1,5},{2,6},{3,7}).  batch_size must be a
    multiple of n_workers (pad_batch pads)."""
    if int(n_workers) < 1:
        raise errors.ConfigError(f"shard_batches: n_workers must be >= 1, got {n_workers}")
    if batch_size < 0 or batch_size % n_workers:
        raise errors.ShapeError(f"shard_batches: batch of {batch_size} is not divisible by "
                                f"{n_workers} workers (pad_batch pads it)")
    idx = np.arange(batch_size, dtype=np.int64)
    return [idx[r::n_workers] for r in range(n_workers)]


def pad_batch(batch_size: int, n_workers: int):
    """(indices, weights) padding a batch to a multiple of n_workers by
    repeating the final example with weight 0, so the shard
    denominators stay global_rows / n and dp equivalence stays exact."""
    if int(n_workers) < 1:
        raise errors.ConfigError(f"pad_batch: n_workers must be >= 1, got {n_workers}")
    if batch_size < 1:
        raise errors.ShapeError("pad_batch: empty batch")
    padded = -(-batch_size // n_workers) * n_workers
    idx = np.concatenate([np.arange(batch_size, dtype=np.int64),
                          np.full(padded - batch_size, batch_size - 1, dtype=np.int64)])
    w = np.ones(padded, dtype=np.float32)
    w[batch_size:] = 0.0
    return idx, w


# ---- replicas ----------------------------------------------------------------


class BankReplica:
    """The GPU bank behind the replica interface DataParallel drives."""

    def __init__(self, bank):
        self.bank = bank
        self.device = torch.device("cuda", bank.ctx.device)

    def grad_size(self) -> int:
        return self.bank.grad_size()

    def compute_grads(self, X, y, w, out, denom, **opts):
        _, loss, _ = self.bank.compute_grads(X, y, w, out=out, denom=denom, **opts)
        return loss

    def apply(self, parts, **opts):
        self.bank.dp_apply(parts, **opts)

    def fingerprint(self) -> int:
        return self.bank.fingerprint()

    def param_tensors(self):
        return self.bank.param_tensors()


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


class DataParallel:
    """dp_step over torch.distributed: every rank calls step() with its own
    shard of the same global batch (shard_batches order)."""

    _STEP_KEYS = ("lr", "optimizer", "adam_betas", "adam_eps", "frozen_layers")

    def __init__(self, replica, *, group=None, check_replicas: bool = True, device=None):
        self.replica = replica
        self.group = group
        d = _dist()
        self.world = d.get_world_size(group) if d else 1
        self.rank = d.get_rank(group) if d else 0
        self.device = device if device is not None else getattr(replica, "device", torch.device("cpu"))
        self.check = check_replicas
        n = replica.grad_size()
        dt = getattr(replica, "grad_dtype", torch.float32)
        self.parts = torch.empty((self.world, n), dtype=dt, device=self.device)
        self.local = self.parts[0] if self.world == 1 else torch.empty(n, dtype=dt,
                                                                       device=self.device)
        self.steps = 0

    def broadcast_params(self, src: int = 0):
        """make every replica bit-identical to rank `src` (initialisation)."""
        d = _dist()
        if d is None or self.world == 1:
            return
        for t in self.replica.param_tensors():
            d.broadcast(t, src=src, group=self.group)

    def check_replicas(self):
        """ConsistencyError unless every rank's parameter fingerprint matches."""
        d = _dist()
        if d is None or self.world == 1:
            return
        fp = self.replica.fingerprint()
        mine = torch.tensor([fp - (1 << 64) if fp >= (1 << 63) else fp], dtype=torch.int64,
                            device=self.device)
        allfp = torch.empty(self.world, dtype=torch.int64, device=self.device)
        d.all_gather_into_tensor(allfp, mine, group=self.group)
        v = allfp.cpu().tolist()
        bad = [r for r in range(self.world) if v[r] != v[0]]
        if bad:
            raise errors.ConsistencyError(
                f"dp_step: replicas diverged before step {self.steps} (ranks {bad} differ from rank 0)")

    def step(self, X, y, w=None, *, global_rows: int | None = None, want_loss: bool = False,
             **opts):
        """One dp_step on this rank's shard X [G, b, d] / y [G, b] / w [G, b]
        (or None).  global_rows = real rows in the global batch (default
        b * n_workers; smaller when pad_batch padded it).  opts: lr,
        optimizer, adam_betas, adam_eps, frozen_layers.  Returns the global
        mean CE loss [G] when want_loss (one small extra gather)."""
        unknown = set(opts) - set(self._STEP_KEYS)
        if unknown:
            raise errors.ConfigError(f"dp_step: unsupported options {sorted(unknown)} "
                                     "(MMD / two-head steps do not shard by rows)")
        b = X.shape[1]
        rows = b * self.world if global_rows is None else int(global_rows)
        if rows < 1 or rows > b * self.world:
            raise errors.ShapeError(f"dp_step: global_rows {rows} outside [1, {b * self.world}]")
        if self.check:
            self.check_replicas()
        denom = rows / self.world
        loss = self.replica.compute_grads(X, y, w, self.local, (denom, denom), **opts)
        d = _dist()
        if d is not None and self.world > 1:
            d.all_gather_into_tensor(self.parts.view(-1), self.local, group=self.group)
        self.replica.apply(self.parts, **opts)
        self.steps += 1
        if not want_loss:
            return None
        # per-shard loss = n * S_r / rows, so the global mean is their average
        lv = torch.as_tensor(np.asarray(loss, dtype=np.float64), device=self.device)
        if d is not None and self.world > 1:
            allv = torch.empty(self.world * lv.numel(), dtype=torch.float64, device=self.device)
            d.all_gather_into_tensor(allv, lv.reshape(-1), group=self.group)
            rows_v = allv.cpu().numpy().reshape(self.world, -1)
        else:
            rows_v = lv.cpu().numpy()[None]
        acc = rows_v[0].copy()
        for r in range(1, rows_v.shape[0]):
            acc = acc + rows_v[r]
        return acc / rows_v.shape[0]


def dp_step_local(bank, X, y, w=None, *, n_workers: int, global_rows: int | None = None,
                  parts: torch.Tensor | None = None, **opts):
    """n simulated workers on one device: the global batch
    X [G, B, d] / y [G, B] is sharded round-robin on the device, each shard's
    gradients go to parts[r], and one dp_apply aggregates in ascending worker
    order and steps.  Same arithmetic as DataParallel.step at n ranks."""
    from . import api

    G, B = X.shape[0], X.shape[1]
    shards = shard_batches(B, n_workers)
    rows = B if global_rows is None else int(global_rows)
    denom = rows / n_workers
    n = bank.grad_size()
    if parts is None:
        parts = torch.empty((n_workers, n), dtype=torch.float32, device=X.device)
    base = (torch.arange(G, device=X.device, dtype=torch.int64) * B)[:, None]
    Xf = X.reshape(G * B, -1)
    for r, sidx in enumerate(shards):
        idx = base + torch.as_tensor(sidx, device=X.device)[None, :]
        Xr = api.gather_rows(bank.ctx, Xf, idx).reshape(G, len(sidx), X.shape[2])
        yr = api.gather_rows(bank.ctx, y.reshape(G * B), idx).reshape(G, len(sidx))
        wr = (api.gather_rows(bank.ctx, w.reshape(G * B), idx).reshape(G, len(sidx))
              if w is not None else None)
        bank.compute_grads(Xr, yr, wr, out=parts[r], denom=(denom, denom), want_loss=False,
                           **opts)
    bank.dp_apply(parts, **opts)
