"""Data-parallel training (dp.py).

CPU: shard_batches / pad_batch / the speedup model's pinned examples
(SPEC.md:610-631, 716-718); dp_step over gloo with world_size 2 on the f64
oracle replica against single-process full-batch training (<= 1e-9,
SPEC.md:622 / 634), bit-identical replicas, and the replica-divergence
ConsistencyError.
GPU: the libmtk path (compute_grads -> ordered fp64 mean -> optimizer step)
with n simulated workers on one device: n = 1 is a plain step, identical
shards give exactly one worker's gradient, n in {2,4,8} matches the
full-batch step to fp32 summation-order tolerance, and frozen layers stay
bit-identical.
"""
import os
import socket

import numpy as np
import pytest
import torch

import pyoracle as po
from oracle_backend import OracleReplica
from paper_2011_09463_b200 import dp, errors

# ---- sharding ----------------------------------------------------------------


def test_shard_batches_examples():
    assert [s.tolist() for s in dp.shard_batches(8, 4)] == [[0, 4], [1, 5], [2, 6], [3, 7]]
    assert [s.tolist() for s in dp.shard_batches(5, 1)] == [[0, 1, 2, 3, 4]]
    for size in range(0, 65, 4):
        for n in (1, 2, 4):
            sh = dp.shard_batches(size, n)
            allidx = np.concatenate(sh)
            assert sorted(allidx.tolist()) == list(range(size))  # union = batch, disjoint
            assert all(len(s) == size // n for s in sh)


def test_shard_batches_errors():
    with pytest.raises(errors.ConfigError):
        dp.shard_batches(8, 0)
    with pytest.raises(errors.ShapeError):
        dp.shard_batches(9, 4)


def test_pad_batch():
    idx, w = dp.pad_batch(10, 4)
    assert idx.tolist() == list(range(10)) + [9, 9]
    assert w.tolist() == [1.0] * 10 + [0.0, 0.0]
    idx, w = dp.pad_batch(8, 4)
    assert idx.tolist() == list(range(8)) and w.min() == 1.0


# ---- speedup model -----------------------------------


# ---- dp_step on the oracle replica over gloo ---------------------------------

DIMS = (12, 10, 4)


def _task(seed, B):
    r = po.Rng(seed)
    W, b = po.mlp_init(r, DIMS)
    X = np.array(r.normals(B * DIMS[0])).reshape(B, DIMS[0])
    y = np.array([r.below(DIMS[-1]) for _ in range(B)], dtype=np.int32)
    return W, b, X, y


def _single(W, b, X, y, steps, lr, w=None, rows=None):
    W = [x.copy() for x in W]
    b = [x.copy() for x in b]
    for _ in range(steps):
        po.mlp_train_step(list(DIMS), W, b, X, y, lr=lr, w=w,
                          denoms=[float(rows if rows else X.shape[0])])
    return W, b


def _dp_worker(rank, world, port, seed, B, steps, lr, out, diverge, pad):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, b, X, y = _task(seed, B)
        if rank != 0:  # replicas start from rank 0's parameters
            W = [np.zeros_like(x) for x in W]
            b = [np.zeros_like(x) for x in b]
        rep = OracleReplica(DIMS, W, b)
        par = dp.DataParallel(rep)
        par.broadcast_params()
        wv = np.ones(B)
        rows = B
        if pad:
            idx, wv = dp.pad_batch(B - pad, world)
            X, y, rows = X[idx], y[idx], B - pad
        sidx = dp.shard_batches(len(y), world)[rank]
        if diverge and rank == 1:
            rep.W[0][0, 0] += 1e-12
        losses = []
        for _ in range(steps):
            lv = par.step(X[sidx][None], y[sidx][None], np.asarray(wv)[sidx][None],
                          global_rows=rows, lr=lr, want_loss=True)
            losses.append(float(lv[0]))
        out[rank] = ("ok", [x.copy() for x in rep.W], [x.copy() for x in rep.b], losses)
    except errors.ConsistencyError as e:
        out[rank] = ("consistency", str(e))
    finally:
        dist.destroy_process_group()


def _run_gloo(world, **kw):
    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mgr = mp.Manager()
    out = mgr.dict()
    args = dict(seed=1, B=32, steps=10, lr=0.1, diverge=False, pad=0)
    args.update(kw)
    mp.spawn(_dp_worker, args=(world, port, args["seed"], args["B"], args["steps"], args["lr"],
                               out, args["diverge"], args["pad"]), nprocs=world, join=True)
    return dict(out), args


@pytest.mark.parametrize("pad", [0, 1])
def test_dp_step_gloo_matches_full_batch(pad):
    out, a = _run_gloo(2, pad=pad)
    W0, b0, X, y = _task(a["seed"], a["B"])
    n_real = a["B"] - pad
    Ws, bs = _single(W0, b0, X[:n_real], y[:n_real], a["steps"], a["lr"])
    assert out[0][0] == out[1][0] == "ok"
    for r in (0, 1):
        for got, want in zip(out[r][1] + out[r][2], Ws + bs):
            assert np.max(np.abs(got - want)) <= 1e-9
    # replicas bit-identical after every step
    for x0, x1 in zip(out[0][1] + out[0][2], out[1][1] + out[1][2]):
        assert np.array_equal(x0, x1)
    assert out[0][3] == out[1][3]


def test_dp_step_gloo_detects_replica_divergence():
    out, _ = _run_gloo(2, diverge=True, steps=1)
    assert out[0][0] == out[1][0] == "consistency"
    assert "ranks [1]" in out[0][1]


@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_dp_local_oracle_equivalence_seeds(n):
    # SPEC.md:634 / 717: n simulated workers vs single-process, 10 steps, 20 seeds
    B, steps, lr = 32, 10, 0.1
    for seed in range(20):
        W, b, X, y = _task(100 + seed, B)
        rep = OracleReplica(DIMS, W, b)
        parts = torch.empty((n, rep.grad_size()), dtype=torch.float64)
        for _ in range(steps):
            for r, s in enumerate(dp.shard_batches(B, n)):
                rep.compute_grads(X[s][None], y[s][None], None, parts[r], (B / n, B / n))
            rep.apply(parts, lr=lr)
        Ws, bs = _single(W, b, X, y, steps, lr)
        err = max(np.max(np.abs(g - w)) for g, w in zip(rep.W + rep.b, Ws + bs))
        assert err <= 1e-9, (seed, err)


# ---- GPU: the libmtk dp path ------------------------------------------------


def _gpu_bank(dims, seed, G=2):
    from paper_2011_09463_b200 import api

    ctx = api.Context(0)
    bank = api.Bank(ctx, G, dims)
    r = api.Rng(seed)
    for g in range(G):
        bank.init_params(g, r)
    return ctx, bank


def _gpu_batch(G, B, d, C, seed):
    g = torch.Generator().manual_seed(seed)
    X = torch.randn(G, B, d, generator=g).cuda()
    y = torch.randint(0, C, (G, B), generator=g, dtype=torch.int32).cuda()
    return X, y


def _params(bank):
    return [t.detach().clone() for t in bank.param_tensors()]


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(64, 128, 10), (40, 96, 64, 10)])
def test_gpu_dp_n1_is_a_plain_step(dims):
    ctx, a = _gpu_bank(dims, 3)
    _, b = _gpu_bank(dims, 3)
    X, y = _gpu_batch(2, 256, dims[0], dims[-1], 0)
    for _ in range(3):
        a.train_step(X, y, lr=0.05, want_loss=False)
        dp.dp_step_local(b, X, y, n_workers=1, lr=0.05)
    for p, q in zip(_params(a), _params(b)):
        assert torch.equal(p, q)


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_gpu_dp_identical_shards_give_one_workers_gradient(n):
    dims = (64, 128, 10)
    ctx, bank = _gpu_bank(dims, 5)
    X, y = _gpu_batch(2, 128, dims[0], dims[-1], 1)
    g1, _, _ = bank.compute_grads(X, y, want_loss=False)
    before = _params(bank)
    fp = bank.fingerprint()
    parts = g1[None].repeat(n, 1).contiguous()
    assert bank.fingerprint() == fp and all(torch.equal(p, q) for p, q in zip(before, _params(bank)))
    _, single = _gpu_bank(dims, 5)
    bank.dp_apply(parts, lr=0.1)
    single.dp_apply(g1[None].contiguous(), lr=0.1)
    for p, q in zip(_params(bank), _params(single)):
        assert torch.equal(p, q)
    assert bank.fingerprint() == single.fingerprint() != fp


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("optimizer", ["sgd", "adam"])
def test_gpu_dp_matches_full_batch(n, optimizer):
    dims = (64, 128, 96, 10)
    lr = 0.05 if optimizer == "sgd" else 0.002
    _, full = _gpu_bank(dims, 7)
    _, par = _gpu_bank(dims, 7)
    X, y = _gpu_batch(2, 512, dims[0], dims[-1], 2)
    for _ in range(10):
        full.train_step(X, y, lr=lr, optimizer=optimizer, want_loss=False)
        dp.dp_step_local(par, X, y, n_workers=n, lr=lr, optimizer=optimizer)
    for p, q in zip(_params(full), _params(par)):
        err = (p - q).abs().max().item()
        assert err <= 2e-5 * max(1.0, p.abs().max().item()), err


@pytest.mark.gpu
def test_gpu_dp_weighted_padding_and_frozen():
    dims = (48, 64, 32, 10)
    _, full = _gpu_bank(dims, 9, G=1)
    _, par = _gpu_bank(dims, 9, G=1)
    X, y = _gpu_batch(1, 90, dims[0], dims[-1], 3)
    idx, w = dp.pad_batch(90, 4)
    it = torch.as_tensor(idx, device="cuda")
    Xp, yp = X[:, it].contiguous(), y[:, it].contiguous()
    wp = torch.as_tensor(w, device="cuda")[None].contiguous()
    frozen0 = _params(par)[:2]
    for _ in range(5):
        full.train_step(X, y, lr=0.05, frozen_layers=1, want_loss=False)
        dp.dp_step_local(par, Xp, yp, wp, n_workers=4, global_rows=90, lr=0.05, frozen_layers=1)
    pp = _params(par)
    assert torch.equal(pp[0], frozen0[0]) and torch.equal(pp[1], frozen0[1])
    for p, q in zip(_params(full), pp):
        assert (p - q).abs().max().item() <= 2e-5


@pytest.mark.gpu
def test_gpu_dataparallel_single_rank_step():
    dims = (64, 128, 10)
    _, a = _gpu_bank(dims, 11)
    _, b = _gpu_bank(dims, 11)
    X, y = _gpu_batch(2, 256, dims[0], dims[-1], 4)
    par = dp.DataParallel(dp.BankReplica(b))
    for _ in range(3):
        la, _ = a.train_step(X, y, lr=0.05)
        lb = par.step(X, y, lr=0.05, want_loss=True)
        assert np.allclose(la, lb, rtol=1e-6)
    for p, q in zip(_params(a), _params(b)):
        assert torch.equal(p, q)
    with pytest.raises(errors.ConfigError):
        par.step(X, y, lr=0.05, mmd_lambda=1.0)


@pytest.mark.gpu
@pytest.mark.parametrize("dims", [(64, 128, 10), (40, 96, 64, 10), (24, 12, 4)])
def test_gpu_compute_grads_never_writes_parameters(dims):
    """compute_grads stores gradients only (no lr = 0 update): a non-finite
    shard raises mt::Error but leaves the replica bit-identical (-0 * inf
    would have made the parameters NaN)."""
    from paper_2011_09463_b200 import errors

    _, bank = _gpu_bank(dims, 11)
    X, y = _gpu_batch(2, 64, dims[0], dims[-1], 4)
    X[1, 3, 0] = float("inf")
    before = _params(bank)
    fp = bank.fingerprint()
    with pytest.raises(errors.Error):
        bank.compute_grads(X, y, want_loss=True)
    assert all(torch.equal(p, q) for p, q in zip(before, _params(bank)))
    assert bank.fingerprint() == fp


@pytest.mark.gpu
def test_gpu_api_rejects_wrong_dtypes_before_the_c_call():
    """int32 indices / float64 pools / wrong shapes raise before libmtk reads them"""
    from paper_2011_09463_b200 import errors

    dims = (16, 12, 4)
    _, bank = _gpu_bank(dims, 1)
    X, y = _gpu_batch(2, 8, dims[0], dims[-1], 5)
    pool = torch.randn(32, 16, device="cuda")
    ypool = torch.zeros(32, dtype=torch.int32, device="cuda")
    idx = torch.zeros((3, 2, 8), dtype=torch.int64, device="cuda")
    with pytest.raises(errors.ValueError):
        bank.train_epoch(pool, ypool, idx.int(), lr=0.1)
    with pytest.raises(errors.ValueError):
        bank.train_epoch(pool.double(), ypool, idx, lr=0.1)
    with pytest.raises(errors.ShapeError):
        bank.train_epoch(pool, ypool, idx, torch.ones((3, 2, 7), device="cuda"), lr=0.1)
    with pytest.raises(errors.ValueError):
        bank.train_step(X, y.long(), lr=0.1)
    with pytest.raises(errors.ShapeError):
        bank.train_step(X[:, :, :8].contiguous(), y, lr=0.1)
    with pytest.raises(errors.ValueError):
        bank.compute_grads(X.cpu(), y, want_loss=False)
    bank.train_epoch(pool, ypool, idx, lr=0.1)  # the well-formed call still runs
