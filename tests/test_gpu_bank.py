"""GPU parity of the grouped shadow-model bank against the CPU oracle.

Tolerance (north_star): per-kernel fp32 outputs within 1e-5 relative,
measured as max|gpu - oracle| / max|oracle| per tensor, on identical inputs
(the oracle is fed the exact fp32 values the GPU sees).  Oracle steps are
bit-identical to the reference Tape (tests/test_oracle.py).
"""
import numpy as np
import pytest
import torch

import pyoracle as po

pytestmark = pytest.mark.gpu

TOL = 1e-5


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def make_bank(ctx, G, dims, n_heads=1, seed=11):
    from paper_2011_09463_b200 import api

    bank = api.Bank(ctx, G, dims, n_heads=n_heads)
    rng = api.Rng(seed)
    for g in range(G):
        bank.init_params(g, rng)
    return bank


def inputs(G, B, d0, C, seed=5, shift=0.0):
    r = po.Rng(seed)
    X = r.normals(G * B * d0).reshape(G, B, d0).astype(np.float32)
    X[:, B // 2:, :] += np.float32(shift)
    y = np.array([[r.below(C) for _ in range(B)] for _ in range(G)], dtype=np.int32)
    return X, y


def to_dev(X, y):
    return torch.tensor(X, device="cuda"), torch.tensor(y, device="cuda")


def check_step(bank, X, y, *, n_heads=1, src=0, frozen=0, lam=0.0, lr=0.05, w=None, tol=TOL):
    dims = bank.dims
    G = bank.G
    before = [bank.get_params(g) for g in range(G)]
    bank.keep_grads(True)
    Xd, yd = to_dev(X, y)
    wd = None if w is None else torch.tensor(w, device="cuda")
    loss, mmd = bank.train_step(Xd, yd, wd, lr=lr, src_rows=src, frozen_layers=frozen,
                                mmd_lambda=lam)
    worst = 0.0
    for g in range(G):
        W, b = [x.copy() for x in before[g][0]], [x.copy() for x in before[g][1]]
        Xg = X[g].astype(np.float64)
        dH = None
        if lam > 0:
            _, H = po.mlp_forward(dims, W, b, Xg)
            v, _, gs, gt = po.mmd_gaussian(H[:src], H[src:])
            dH = lam * np.concatenate([gs, gt])
            assert rel(mmd[g], v) <= TOL, (g, mmd[g], v)
        lo, gW, gb = po.mlp_train_step(dims, W, b, Xg, y[g], n_heads=n_heads, frozen=frozen,
                                       src_rows=src, lr=lr, dH=dH,
                                       w=None if w is None else w[g].astype(np.float64),
                                       want_grads=True)
        assert rel(loss[g], lo) <= TOL, (g, loss[g], lo)
        dW, db = bank.get_grads(g)
        Wn, bn = bank.get_params(g)
        l_lo = 0
        for i in range(bank.n_mats):
            lay = i if i < bank.L else bank.L - 1
            if lay < frozen:
                # frozen parameters must be bit-unchanged (SPEC.md finetune post-condition)
                assert np.array_equal(Wn[i], before[g][0][i]) and np.array_equal(bn[i], before[g][1][i])
                continue
            e = max(rel(dW[i], gW[i]), rel(db[i], gb[i]) if np.abs(gb[i]).max() > 0 else 0.0)
            worst = max(worst, e)
            assert e <= tol, (g, i, e)
            assert rel(Wn[i], W[i]) <= tol
    return worst


def test_forward_matches_oracle(ctx):
    dims = [784, 256, 10]
    G, B = 5, 64
    bank = make_bank(ctx, G, dims)
    X, _ = inputs(G, B, dims[0], dims[-1])
    logits, hid = bank.forward(torch.tensor(X, device="cuda"), hidden=True)
    logits, hid = logits.cpu().numpy(), hid.cpu().numpy()
    for g in range(G):
        W, b = bank.get_params(g)
        lo, H = po.mlp_forward(dims, W, b, X[g].astype(np.float64))
        assert rel(logits[g], lo) <= TOL
        assert rel(hid[g], H) <= TOL


@pytest.mark.parametrize("dims", [[3, 64, 2], [4, 48, 2], [8, 200, 4]])
def test_forward_attack_model_shape(ctx, dims):
    """k -> H -> 2 forward (the attack model) runs as one fused kernel."""
    G, B = 3, 1000
    bank = make_bank(ctx, G, dims)
    r = po.Rng(9)
    X = r.normals(G * B * dims[0]).reshape(G, B, dims[0]).astype(np.float32)
    logits = bank.forward(torch.tensor(X, device="cuda")).cpu().numpy()
    for g in range(G):
        W, b = bank.get_params(g)
        lo, _ = po.mlp_forward(dims, W, b, X[g].astype(np.float64))
        assert rel(logits[g], lo) <= TOL


def test_step_c1_shape(ctx):
    """C1: 784-256-10, 1 target + 4 shadows, B=128."""
    dims = [784, 256, 10]
    bank = make_bank(ctx, 5, dims)
    X, y = inputs(5, 128, 784, 10)
    check_step(bank, X, y)


def test_step_c2_shape_with_mmd(ctx):
    """C2 architecture 1024-512-256-10, src+tgt batch, 5-bandwidth MMD injected."""
    dims = [1024, 512, 256, 10]
    bank = make_bank(ctx, 2, dims)
    X, y = inputs(2, 96, 1024, 10, shift=0.5)
    # this compares the whole chained step (fwd x3, CE, MMD, DX x2, DW x3) with
    # the f64 oracle's own intermediates, not one kernel on identical inputs:
    # the fp32 MMD gradient injected at layer 2 propagates into layer-1/2 dW.
    # Per-kernel 1e-5 parity is asserted in test_gpu_umma.py / test_gpu_mmd.py.
    check_step(bank, X, y, src=48, lam=1.0, tol=2e-5)


@pytest.mark.parametrize("B,src,dims", [(300, 140, [96, 64, 10]), (1024, 512, [1024, 512, 256, 10]),
                                        (260, 100, [64, 48, 7])])
def test_mmd_materialised_w_path_matches_fused(ctx, monkeypatch, B, src, dims):
    """The bank's MMD runs on the materialised-W path (each unordered tile
    pair once + a GEMM for V) unless MTK_MMD_FUSED=1; both must give the same
    step (ragged tiles: N = 300 / 260 is not a multiple of 128)."""
    X, y = inputs(3, B, dims[0], dims[-1], shift=0.4)
    Xd, yd = to_dev(X, y)
    res = []
    for fused in ("0", "1"):
        monkeypatch.setenv("MTK_MMD_FUSED", fused)
        bank = make_bank(ctx, 3, dims, seed=5)
        bank.keep_grads(True)
        loss, mmd = bank.train_step(Xd, yd, lr=0.05, src_rows=src, mmd_lambda=0.8)
        res.append((loss, mmd, bank.get_grads(2)[0]))
    (l0, m0, g0), (l1, m1, g1) = res
    assert rel(l0, l1) <= 1e-6 and rel(m0, m1) <= 1e-5, (m0, m1)
    for a, b in zip(g0, g1):
        assert rel(a, b) <= 2e-5


@pytest.mark.parametrize("B,src,dims,frozen,fused", [
    (320, 140, [96, 64, 10], 0, True), (1024, 512, [1024, 512, 256, 10], 0, True),
    (224, 90, [100, 64, 32, 10], 1, True), (96, 40, [64, 32, 2], 0, True), (256, 100, [64, 48, 20], 0, True),
    (300, 140, [96, 64, 10], 0, False)])  # B % 32 != 0: separate head DX launch
def test_head_dx_fused_into_mmd_gradient_gemm(ctx, monkeypatch, B, src, dims, frozen, fused):
    """With MMD on the materialised-W path and a skinny head, the head's DX
    ((lambda g + dlogits W_head^T) * (h > 0)) rides on the V = W.Z GEMM as an
    extra K block instead of a separate head_dx launch (MTK_NO_HEAD_FUSE=1):
    one launch fewer, same step to fp32 rounding (3xTF32 head product)."""
    G = 3
    X, y = inputs(G, B, dims[0], dims[-1], shift=0.4)
    Xd, yd = to_dev(X, y)
    res = []
    for off in ("0", "1"):
        monkeypatch.setenv("MTK_NO_HEAD_FUSE", off)
        bank = make_bank(ctx, G, dims, seed=9)
        bank.keep_grads(True)
        torch.cuda.synchronize()
        n0 = ctx.launches
        loss, mmd = bank.train_step(Xd, yd, lr=0.05, src_rows=src, mmd_lambda=0.7, frozen_layers=frozen)
        res.append((loss.copy(), mmd.copy(), [bank.get_grads(g) for g in range(G)],
                    [bank.get_params(g) for g in range(G)], ctx.launches - n0))
    (l0, m0, g0, p0, n0), (l1, m1, g1, p1, n1) = res
    assert n0 == n1 - (1 if fused else 0), (n0, n1)
    assert np.array_equal(l0, l1) and np.array_equal(m0, m1)
    L = len(dims) - 1
    for g in range(G):
        for i in range(frozen, L):
            for k in (0, 1):  # dW, db
                assert rel(g0[g][k][i], g1[g][k][i]) <= 2e-6, (g, i, k)
                assert rel(p0[g][k][i], p1[g][k][i]) <= 2e-6, (g, i, k)
            if i == L - 1 or not fused:
                assert np.array_equal(g0[g][0][i], g1[g][0][i]), (g, i)  # the head's own dW


@pytest.mark.parametrize("B,dims,lam,weighted", [
    (300, [96, 64, 10], 0.0, True), (77, [40, 3], 0.0, False), (130, [64, 48, 20], 0.5, True),
    (300, [96, 64, 10], 0.7, False), (1024, [1024, 512, 256, 10], 1.0, False), (96, [64, 32, 16], 0.6, True)])
def test_head_forward_with_fused_ce_is_bit_identical(ctx, monkeypatch, B, dims, lam, weighted):
    """The skinny head's forward kernel also runs the softmax-CE rows (same
    ce_row code as ce_kernel, same per-32-row partial order): the step must be
    bit-identical to the separate CE launch (MTK_NO_HEAD_CE=1), including
    ragged 64-row blocks and label weights; one launch fewer."""
    G = 3
    X, y = inputs(G, B, dims[0], dims[-1], shift=0.3)
    Xd, yd = to_dev(X, y)
    wd = None
    if weighted:
        wd = torch.tensor(np.linspace(0.0, 2.0, G * B, dtype=np.float32).reshape(G, B), device="cuda")
    res = []
    for off in ("0", "1"):
        monkeypatch.setenv("MTK_NO_HEAD_CE", off)
        bank = make_bank(ctx, G, dims, seed=4)
        torch.cuda.synchronize()
        n0 = ctx.launches
        loss, mmd = bank.train_step(Xd, yd, wd, lr=0.05, src_rows=B // 2 if lam else 0, mmd_lambda=lam)
        res.append((loss.copy(), mmd.copy(), [bank.get_params(g) for g in range(G)], ctx.launches - n0))
    (l0, m0, p0, n0), (l1, m1, p1, n1) = res
    assert n0 == n1 - 1, (n0, n1)
    assert np.array_equal(l0, l1) and np.array_equal(m0, m1)
    for g in range(G):
        for k in (0, 1):
            for a, b in zip(p0[g][k], p1[g][k]):
                assert np.array_equal(a, b), g


def test_step_two_heads_parameter_based(ctx):
    dims = [784, 256, 10]
    bank = make_bank(ctx, 3, dims, n_heads=2)
    X, y = inputs(3, 64, 784, 10)
    check_step(bank, X, y, n_heads=2, src=40)


def test_step_frozen_prefix_model_based(ctx):
    dims = [100, 64, 32, 10]
    bank = make_bank(ctx, 2, dims)
    X, y = inputs(2, 50, 100, 10)
    check_step(bank, X, y, frozen=1)


def test_step_ragged_shapes_and_weights(ctx):
    dims = [37, 19, 3]
    bank = make_bank(ctx, 4, dims)
    X, y = inputs(4, 5, 37, 3)
    w = np.array([[0.5, 0.0, 1.0, 2.0, 1.0]] * 4, dtype=np.float32)
    check_step(bank, X, y, w=w, lr=0.3)


@pytest.mark.parametrize("lam", [0.0, 0.7])
def test_step_staged_epilogue_ragged_chunks(ctx, lam):
    """tcgen05 layers whose widths are not multiples of 32 and row counts not
    multiples of the 128-row tile: the smem-staged epilogues (bias + ReLU,
    ReLU-mask DX without an addend, SGD) take the thread-per-row path for the
    last, ragged 32-column chunk and mask the rows past M; parity with the
    oracle at the per-kernel tolerance (with and without the MMD)."""
    dims = [100, 72, 44, 10]
    bank = make_bank(ctx, 3, dims, seed=21)
    assert bank.tc_layers()[:2] == [True, True], bank.tc_layers()
    X, y = inputs(3, 300, dims[0], dims[-1], shift=0.3)
    check_step(bank, X, y, src=140 if lam else 0, lam=lam, lr=0.1)


def test_step_narrow_input_layer(ctx):
    """fan_in <= 32 < fan_out (the attack model's k -> 64 layer): dW runs as the
    transposed skinny reduction."""
    dims = [5, 48, 3]
    bank = make_bank(ctx, 3, dims)
    X, y = inputs(3, 300, 5, 3)
    check_step(bank, X, y, lr=0.2)


def test_multi_step_trajectory(ctx):
    dims = [64, 32, 10]
    G = 3
    bank = make_bank(ctx, G, dims)
    X, y = inputs(G, 32, 64, 10)
    Xd, yd = to_dev(X, y)
    ref = [bank.get_params(g) for g in range(G)]
    for _ in range(8):
        bank.train_step(Xd, yd, lr=0.1, want_loss=False)
        for g in range(G):
            po.mlp_train_step(dims, ref[g][0], ref[g][1], X[g].astype(np.float64), y[g], lr=0.1)
    for g in range(G):
        W, b = bank.get_params(g)
        for i in range(len(W)):
            assert rel(W[i], ref[g][0][i]) <= 1e-4


@pytest.mark.parametrize("dims,n_heads,frozen", [([784, 256, 10], 1, 0), ([100, 64, 32, 10], 1, 1),
                                                 ([64, 48, 10], 2, 0), ([37, 19, 3], 1, 0),
                                                 ([3, 64, 2], 1, 0)])
def test_adam_steps_match_oracle_update(ctx, dims, n_heads, frozen):
    """Adam (optim.hpp:49-63) in the dW/db epilogues: three steps; each step's
    parameters must equal the oracle Adam update (f64, its own moments) applied
    to the step's GPU gradients (gradients themselves are pinned by the SGD
    tests above).  Moments persist across steps; reset_optimizer restarts."""
    G, B = 3, 40
    bank = make_bank(ctx, G, dims, n_heads=n_heads)
    X, y = inputs(G, B, dims[0], dims[-1])
    Xd, yd = to_dev(X, y)
    bank.keep_grads(True)
    lr, betas, eps = 0.01, (0.8, 0.99), 1e-6
    opts = None
    for step in range(3):
        before = [bank.get_params(g) for g in range(G)]
        bank.train_step(Xd, yd, lr=lr, src_rows=24, frozen_layers=frozen, optimizer="adam",
                        adam_betas=betas, adam_eps=eps, want_loss=False)
        if opts is None:
            opts = [po.Adam(before[g][0] + before[g][1], lr, betas[0], betas[1], eps) for g in range(G)]
        for g in range(G):
            W, b = [x.copy() for x in before[g][0]], [x.copy() for x in before[g][1]]
            dW, db = bank.get_grads(g)
            live = [i for i in range(bank.n_mats) if (i if i < bank.L else bank.L - 1) >= frozen]
            # the oracle state steps every parameter; frozen ones get zero grads
            # and are compared for bit-identity instead
            grads = [dW[i] if i in live else np.zeros_like(W[i]) for i in range(len(W))] + \
                    [db[i] if i in live else np.zeros_like(b[i]) for i in range(len(b))]
            opts[g].update(W + b, grads)
            Wn, bn = bank.get_params(g)
            for i in range(bank.n_mats):
                if i not in live:
                    assert np.array_equal(Wn[i], before[g][0][i])
                    continue
                assert rel(Wn[i], W[i]) <= TOL, (step, g, i, rel(Wn[i], W[i]))
                assert rel(bn[i], b[i]) <= TOL, (step, g, i)
    # a fresh state: the next step is a first step again
    bank.reset_optimizer()
    before = bank.get_params(0)
    bank.train_step(Xd, yd, lr=lr, src_rows=24, frozen_layers=frozen, optimizer="adam",
                    adam_betas=betas, adam_eps=eps, want_loss=False)
    dW, db = bank.get_grads(0)
    i = bank.n_mats - 1
    W = before[0][i].copy()
    po.Adam([W], lr, betas[0], betas[1], eps).update([W], [dW[i]])
    assert rel(bank.get_params(0)[0][i], W) <= TOL


def test_determinism(ctx):
    dims = [128, 64, 10]
    X, y = inputs(2, 40, 128, 10)
    Xd, yd = to_dev(X, y)
    outs = []
    for _ in range(2):
        bank = make_bank(ctx, 2, dims, seed=3)
        for _ in range(3):
            bank.train_step(Xd, yd, lr=0.1, src_rows=20, mmd_lambda=0.5, want_loss=False)
        outs.append(bank.get_params(1)[0])
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("env", [{"MTK_UMMA_SEPC_KF": "0"}, {"MTK_MMD_NO_WDIAG": "1"}, {"MTK_UMMA_PREFETCH": "1"},
                                 {"MTK_UMMA_SEPC_KF": "0", "MTK_MMD_NO_WDIAG": "1", "MTK_UMMA_PREFETCH": "1"}])
def test_ab_switches_keep_parity(ctx, monkeypatch, env):
    """The A/B switches that restore earlier schedules (corrections shared by no
    k-block, the z * Wsum MMD epilogue, the producer-side prefetch) stay
    correct: a step with the MMD on tcgen05 shapes (K >= 768: SEPC launches)
    against the oracle at the per-kernel tolerance."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    dims = [800, 256, 128, 10]
    bank = make_bank(ctx, 2, dims, seed=17)
    X, y = inputs(2, 512, dims[0], dims[-1], shift=0.3)
    check_step(bank, X, y, src=256, lam=0.8, lr=0.05)


def test_host_step_equals_device_step(ctx):
    dims = [64, 32, 10]
    X, y = inputs(2, 16, 64, 10)
    b1 = make_bank(ctx, 2, dims)
    b2 = make_bank(ctx, 2, dims)
    Xd, yd = to_dev(X, y)
    l1, _ = b1.train_step(Xd, yd, lr=0.1)
    l2, _ = b2.train_step_host(torch.tensor(X).pin_memory(), torch.tensor(y).pin_memory(), lr=0.1)
    assert np.array_equal(l1, l2)
    for a, b in zip(b1.get_params(1)[0], b2.get_params(1)[0]):
        assert np.array_equal(a, b)


def test_errors(ctx):
    from paper_2011_09463_b200 import api, errors

    with pytest.raises(errors.ShapeError):
        api.Bank(ctx, 2, [10, 0, 3])
    bank = make_bank(ctx, 1, [8, 4, 3])
    X, y = inputs(1, 4, 8, 3)
    y[0, 2] = 7
    Xd, yd = to_dev(X, y)
    with pytest.raises(errors.ValueError):
        bank.train_step(Xd, yd)
    y[0, 2] = 1
    Xd, yd = to_dev(X, y)
    with pytest.raises(errors.ValueError):
        bank.train_step(Xd, yd, denom=(-1.0, 0.0))  # tape.hpp:485
    # the context recovers: the next good call works
    bank.train_step(Xd, yd)
    with pytest.raises(errors.ConfigError):
        bank.train_step(Xd, yd, frozen_layers=5)


def test_tensor_core_layers_engaged(ctx):
    """the dense layers of the C1/C2 architectures run on the tcgen05 path"""
    from paper_2011_09463_b200 import api

    assert api.Bank(ctx, 2, [1024, 512, 256, 10]).tc_layers() == [True, True, False]
    assert api.Bank(ctx, 2, [784, 256, 10]).tc_layers() == [True, False]
    assert api.Bank(ctx, 1, [3, 64, 2]).tc_layers() == [False, False]


def test_tc_and_simt_paths_agree(ctx, monkeypatch):
    dims = [256, 128, 64, 10]
    X, y = inputs(2, 100, 256, 10, shift=0.3)
    Xd, yd = to_dev(X, y)
    res = []
    for off in ("0", "1"):
        monkeypatch.setenv("MTK_DISABLE_TC", off)
        bank = make_bank(ctx, 2, dims, seed=9)
        assert bank.tc_layers()[0] == (off == "0")
        for _ in range(2):
            loss, mmd = bank.train_step(Xd, yd, lr=0.05, src_rows=50, mmd_lambda=0.7)
        res.append((loss, mmd, bank.get_params(1)[0]))
    (l0, m0, W0), (l1, m1, W1) = res
    assert rel(l0, l1) <= 1e-5 and rel(m0, m1) <= 1e-5
    for a, b in zip(W0, W1):
        assert rel(a, b) <= 1e-5


def test_async_host_pipeline_matches_sync(ctx):
    dims = [128, 64, 10]
    X, y = inputs(2, 32, 128, 10)
    Xh, yh = torch.tensor(X).pin_memory(), torch.tensor(y).pin_memory()
    b1 = make_bank(ctx, 2, dims)
    b2 = make_bank(ctx, 2, dims)
    ref = [b1.train_step_host(Xh, yh, lr=0.1, src_rows=16, mmd_lambda=0.5) for _ in range(3)]
    got = []
    for k in range(3):
        b2.train_step_host_async(Xh, yh, lr=0.1, src_rows=16, mmd_lambda=0.5)
        if k > 0:
            got.append(b2.step_result(1))
    got.append(b2.step_result(0))
    for (l1, m1), (l2, m2) in zip(ref, got):
        assert np.array_equal(l1, l2) and np.array_equal(m1, m2)
    for a, b in zip(b1.get_params(0)[0], b2.get_params(0)[0]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("G,B,steps,weighted", [(1, 1024, 6, True), (2, 300, 5, False), (1, 77, 9, True)])
def test_attack_model_epoch_in_one_launch(ctx, monkeypatch, G, B, steps, weighted):
    """mtk_bank_train_epoch on the attack model (3 -> 64 -> 2, SGD) runs every
    step of the epoch in one launch (small2_epoch_kernel: parameters in shared
    memory, one thread per row).  Per row it follows the generic kernels;
    the gradient sums run in another fixed order, so the epoch agrees with the
    generic per-step path (MTK_NO_SMALL_EPOCH=1) to fp32 rounding, and it is
    deterministic."""
    from paper_2011_09463_b200 import api

    dims = [3, 64, 2]
    r = po.Rng(B + steps)
    pool = 2000
    X = r.normals(pool * 3).reshape(pool, 3).astype(np.float32)
    y = np.array([r.below(2) for _ in range(pool)], dtype=np.int32)
    idx = np.array([r.below(pool) for _ in range(steps * G * B)], dtype=np.int64).reshape(steps, G, B)
    w = None
    den = None
    if weighted:
        w = np.ones((steps, G, B), dtype=np.float32)
        w[-1, :, B // 2:] = 0.0  # a padded last batch
        den = w[:, 0, :].sum(axis=1).astype(np.float64)
    Xd, yd, idd = torch.tensor(X, device="cuda"), torch.tensor(y, device="cuda"), torch.tensor(idx, device="cuda")
    wd = None if w is None else torch.tensor(w, device="cuda")
    res = []
    for off in ("0", "0", "1", "1"):
        monkeypatch.setenv("MTK_NO_SMALL_EPOCH", off)
        bank = make_bank(ctx, G, dims, seed=3)
        torch.cuda.synchronize()
        n0 = ctx.launches
        bank.train_epoch(Xd, yd, idd, wd, den, lr=0.1)
        res.append(([bank.get_params(g) for g in range(G)], ctx.launches - n0))
    (p0, n0), (p1, n1), (p2, n2), (p3, n3) = res
    assert n0 == 1 and n2 > steps, (n0, n2)
    for g in range(G):
        for k in (0, 1):
            for a, b, c, d in zip(p0[g][k], p1[g][k], p2[g][k], p3[g][k]):
                assert np.array_equal(a, b)  # deterministic
                # the generic path too: its side-stream head dW and the main
                # stream's narrow-input dW have separate partial-sum scratch
                assert np.array_equal(c, d)
                assert rel(a, c) <= 1e-5, (g, k, rel(a, c))


def _f64_backward(X, H1, H2, logits, y, W1, W2, dH_mmd, lam):
    """TEST INFRASTRUCTURE: the reference backward of CE + lambda * MMD for a
    3-layer MLP (tape.hpp:475-520 CE gradient, :349 strict ReLU mask,
    :225-290 matmul backward, :153-171 injection) in numpy f64, evaluated on
    the GPU's OWN forward activations -- so every dW / db kernel is checked on
    identical inputs, ReLU masks included."""
    B = X.shape[0]
    z = logits - logits.max(1, keepdims=True)
    P = np.exp(z) / np.exp(z).sum(1, keepdims=True)
    dlog = P.copy()
    dlog[np.arange(B), y] -= 1.0
    dlog /= B
    dZ2 = (dlog @ W2.T + lam * dH_mmd) * (H2 > 0)
    dZ1 = (dZ2 @ W1.T) * (H1 > 0)
    return [X.T @ dZ1, H1.T @ dZ2, H2.T @ dlog], [dZ1.sum(0), dZ2.sum(0), dlog.sum(0)]


def test_step_bench_shape_c2_models_of_the_32_model_bank(ctx):
    """The bench's own step (bench.py: 1024-512-256-10, 512 src + 512 tgt,
    5-bandwidth MMD lambda = 1 on the 256-d hidden layer, SGD lr 0.01) on the
    bench's 32-model bank; models 0, 17 and 31 against f64.

    Per kernel on identical inputs (north_star: 1e-5, max|d| / max|ref|):
      * each forward GEMM on the GPU's own input activation: layer 0
        (K = 1024), layer 1 (K = 512), the head (K = 256);
      * MMD^2 value and gradient dH on the GPU's own h;
      * every dW / db of the step against the f64 backward evaluated on the
        GPU's own activations and injected MMD gradient.
    Chained (the f64 oracle's own forward from the same X, W): reported, and
    bounded looser, because the strict ReLU mask (tape.hpp:349) flips where
    |z| is below the fp32-vs-f64 forward difference (~1e-6): each flipped
    element moves one row's whole contribution to dW (the flip count is
    printed)."""
    from paper_2011_09463_b200 import api

    dims = [1024, 512, 256, 10]
    G, B, src = 32, 1024, 512
    bank = make_bank(ctx, G, dims, seed=20110946)
    X, y = inputs(G, B, dims[0], dims[-1], seed=1000, shift=0.5)
    Xd, yd = to_dev(X, y)
    logits, H = bank.forward(Xd, hidden=True)
    picks = (0, 17, 31)
    before = {g: bank.get_params(g) for g in picks}
    # the first two layers as their own bank: its hidden output is H1 and its
    # (linear) output is Z2, from the same tcgen05 GEMMs
    trunk = api.Bank(ctx, G, dims[:3])
    for g in range(G):
        W, b = bank.get_params(g)
        trunk.set_params(g, W[:2], b[:2])
    Z2, H1 = trunk.forward(Xd, hidden=True)
    bank.keep_grads(True)
    loss, mmd = bank.train_step(Xd, yd, lr=0.01, src_rows=src, mmd_lambda=1.0)
    worst, chained, flips = {}, {}, 0

    def put(d, k, v):
        d[k] = max(d.get(k, 0.0), v)

    for g, (W, b) in before.items():
        Xg = X[g].astype(np.float64)
        h1 = H1[g].double().cpu().numpy()
        z2 = Z2[g].double().cpu().numpy()
        h2 = H[g].double().cpu().numpy()
        lg = logits[g].double().cpu().numpy()
        put(worst, "fwd0 (K=1024)", rel(h1, np.maximum(Xg @ W[0] + b[0], 0.0)))
        put(worst, "fwd1 (K=512)", rel(z2, h1 @ W[1] + b[1]))
        put(worst, "fwd2 head (K=256)", rel(lg, h2 @ W[2] + b[2]))
        v, _, ogs, ogt = po.mmd_gaussian(h2[:src], h2[src:])
        gv, _, ggs, ggt = api.mmd_gaussian(ctx, H[g, :src].contiguous(), H[g, src:].contiguous())
        put(worst, "mmd value", max(rel(mmd[g], v), rel(gv, v)))
        dH_gpu = np.concatenate([ggs.cpu().numpy(), ggt.cpu().numpy()]).astype(np.float64)
        put(worst, "mmd dH", rel(dH_gpu, np.concatenate([ogs, ogt])))
        gW, gb = _f64_backward(Xg, h1, h2, lg, y[g], W[1], W[2], dH_gpu, 1.0)
        dW, db = bank.get_grads(g)
        for i in range(3):
            put(worst, f"dW{i}", rel(dW[i], gW[i]))
            put(worst, f"db{i}", rel(db[i], gb[i]))
        Wn, _ = bank.get_params(g)
        for i in range(3):  # the SGD update itself: W - lr * dW (fp32 FMA)
            put(worst, f"W{i} update", rel(Wn[i], W[i] - 0.01 * dW[i]))
        # chained: the f64 oracle's own forward / MMD / backward from X, W
        lo, Ho = po.mlp_forward(dims, W, b, Xg)
        put(chained, "logits", rel(lg, lo))
        put(chained, "h", rel(h2, Ho))
        _, _, cgs, cgt = po.mmd_gaussian(Ho[:src], Ho[src:])
        Wc, bc = [x.copy() for x in W], [x.copy() for x in b]
        lo_, cW, cb = po.mlp_train_step(dims, Wc, bc, Xg, y[g], src_rows=src, lr=0.01,
                                        dH=np.concatenate([cgs, cgt]), want_grads=True)
        put(chained, "loss", rel(loss[g], lo_))
        for i in range(3):
            put(chained, f"dW{i}", rel(dW[i], cW[i]))
            put(chained, f"db{i}", rel(db[i], cb[i]))
        h1o = np.maximum(Xg @ W[0] + b[0], 0.0)
        flips += int(((h1 > 0) != (h1o > 0)).sum() + ((h2 > 0) != (Ho > 0)).sum())
    print("bench-shape C2, per kernel on identical inputs:", {k: f"{v:.2e}" for k, v in worst.items()})
    print(f"bench-shape C2, chained vs the oracle's own forward ({flips} ReLU mask flips over "
          f"{len(picks)} models):", {k: f"{v:.2e}" for k, v in chained.items()})
    for k, v in worst.items():
        assert v <= TOL, (k, v, worst)
    assert chained["logits"] <= 2 * TOL and chained["h"] <= 2 * TOL and chained["loss"] <= TOL
    assert max(v for k, v in chained.items() if k.startswith(("dW", "db"))) <= 1e-2
