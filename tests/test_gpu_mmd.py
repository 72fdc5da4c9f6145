"""GPU parity of the multi-bandwidth Gaussian MMD kernels.

Small cases: value, beta and gradients against the f64 oracle at 1e-5
relative (max-abs / max-abs).  C4 size (65536 x 8192 x 512): size-independent
properties -- row-sharded sums add up to the full sums bit-for-bit, the
gradient sums to zero over all rows (antisymmetric pair terms), and a sampled
subset of gradient rows matches the oracle.
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


def sample(m, n, d, seed=3, shift=0.3):
    r = po.Rng(seed)
    Xs = r.normals(m * d).reshape(m, d).astype(np.float32)
    Xt = (r.normals(n * d).reshape(n, d) + shift).astype(np.float32)
    return Xs, Xt


@pytest.mark.parametrize("m,n,d", [(64, 48, 32), (100, 37, 256), (5, 3, 7), (200, 200, 512),
                                   (1, 1, 1)])
def test_mmd_matches_oracle(ctx, m, n, d):
    from paper_2011_09463_b200 import api

    Xs, Xt = sample(m, n, d)
    v, beta, gs, gt = api.mmd_gaussian(ctx, torch.tensor(Xs, device="cuda"),
                                       torch.tensor(Xt, device="cuda"))
    ov, ob, ogs, ogt = po.mmd_gaussian(Xs.astype(np.float64), Xt.astype(np.float64))
    assert rel(beta, ob) <= 1e-9
    assert rel(v, ov) <= TOL, (v, ov)
    g = np.concatenate([gs.cpu().numpy(), gt.cpu().numpy()])
    og = np.concatenate([ogs, ogt])
    assert rel(g, og) <= TOL


def test_mmd_explicit_beta_and_bandwidths(ctx):
    from paper_2011_09463_b200 import api

    Xs, Xt = sample(40, 30, 16)
    mult = [0.5, 3.0]
    v, beta, gs, gt = api.mmd_gaussian(ctx, torch.tensor(Xs, device="cuda"),
                                       torch.tensor(Xt, device="cuda"), mult=mult, beta=7.5)
    ov, _, ogs, ogt = po.mmd_gaussian(Xs.astype(np.float64), Xt.astype(np.float64),
                                      mult=np.array(mult), beta=7.5)
    assert beta == 7.5
    assert rel(v, ov) <= TOL
    assert rel(np.concatenate([gs.cpu(), gt.cpu()]), np.concatenate([ogs, ogt])) <= TOL


def test_mmd_identical_samples_is_zero(ctx):
    from paper_2011_09463_b200 import api

    Xs, _ = sample(32, 1, 8)
    t = torch.tensor(Xs, device="cuda")
    v, _, gs, gt = api.mmd_gaussian(ctx, t, t.clone())
    assert abs(v) < 1e-6
    assert float((gs + gt).abs().max()) < 1e-6


def test_mmd_translation_invariance(ctx):
    from paper_2011_09463_b200 import api

    Xs, Xt = sample(50, 40, 24)
    a = api.mmd_gaussian(ctx, torch.tensor(Xs, device="cuda"), torch.tensor(Xt, device="cuda"))[0]
    b = api.mmd_gaussian(ctx, torch.tensor(Xs + 2.0, device="cuda"),
                         torch.tensor(Xt + 2.0, device="cuda"))[0]
    assert rel(a, b) <= 1e-4


def test_mmd_errors(ctx):
    from paper_2011_09463_b200 import api, errors

    Xs, Xt = sample(4, 4, 601)  # tc path needs d % 4 == 0; SIMT path d <= 512
    with pytest.raises(errors.ShapeError):
        api.mmd_gaussian(ctx, torch.tensor(Xs, device="cuda"), torch.tensor(Xt, device="cuda"))
    Xs, Xt = sample(4, 4, 8)
    with pytest.raises(errors.ValueError):
        api.mmd_gaussian(ctx, torch.tensor(Xs, device="cuda"), torch.tensor(Xt, device="cuda"),
                         mult=[1.0, -2.0])


def test_mmd_c4_stress_properties(ctx):
    """C4: m=65536, n=8192, d=512 (2.7e9 unique pairs)."""
    from paper_2011_09463_b200 import api

    m, n, d = 65536, 8192, 512
    g = torch.Generator(device="cuda").manual_seed(0)
    Xs = torch.randn(m, d, device="cuda", generator=g)
    Xt = torch.randn(n, d, device="cuda", generator=g) + 0.1
    beta = api.mmd_beta(ctx, Xs, Xt)
    gs = torch.empty_like(Xs)
    gt = torch.empty_like(Xt)
    full = api.mmd_gaussian_rows(ctx, Xs, Xt, beta, 0, m + n, gXs=gs, gXt=gt)
    # two-way row shard (as two ranks would): partial sums add up exactly
    cut = 40000
    gs2 = torch.empty_like(Xs)
    gt2 = torch.empty_like(Xt)
    p0 = api.mmd_gaussian_rows(ctx, Xs, Xt, beta, 0, cut, gXs=gs2, gXt=gt2)
    p1 = api.mmd_gaussian_rows(ctx, Xs, Xt, beta, cut, m + n, gXs=gs2, gXt=gt2)
    assert np.allclose(p0 + p1, full, rtol=1e-12, atol=0)
    assert torch.equal(gs, gs2) and torch.equal(gt, gt2)
    v = api.mmd_value_from_sums(full, m, n)
    assert v > 0
    # sum of all gradient rows vanishes (antisymmetric pair terms)
    tot = torch.cat([gs, gt]).double().sum(0)
    scale = torch.cat([gs, gt]).double().abs().sum(0).max()
    assert float(tot.abs().max() / scale) < 1e-5
    # sampled rows against the oracle (rows vs all columns, f64)
    Xs_h = Xs.cpu().double().numpy()
    Xt_h = Xt.cpu().double().numpy()
    ob = po.mmd_beta(Xs_h, Xt_h)
    assert rel(beta, ob) <= 1e-9
    mult = np.array(api.MMD_MULT)
    Z = np.concatenate([Xs_h, Xt_h])
    rows = [0, 12345, m - 1, m, m + 4321, m + n - 1]
    G = torch.cat([gs, gt]).cpu().double().numpy()
    for i in rows:
        d2 = ((Z - Z[i]) ** 2).sum(1)
        A = sum(2.0 / (ob * q) * np.exp(-d2 / (ob * q)) for q in mult)
        same = np.arange(m + n) < m if i < m else np.arange(m + n) >= m
        c = np.where(same, -2.0 / (m * m) if i < m else -2.0 / (n * n), 2.0 / (m * n))
        c[i] = 0.0
        gi = ((c * A)[:, None] * (Z[i] - Z)).sum(0)
        assert rel(G[i], gi) <= TOL, i


@pytest.mark.parametrize("m,n,d", [(300, 200, 256), (1000, 24, 512), (64, 64, 36)])
def test_mmd_tensor_core_vs_simt(ctx, monkeypatch, m, n, d):
    """the tcgen05 path (default) and the SIMT path agree, both vs the oracle"""
    from paper_2011_09463_b200 import api

    Xs, Xt = sample(m, n, d, seed=m)
    out = []
    for off in ("0", "1"):
        monkeypatch.setenv("MTK_DISABLE_TC", off)
        v, beta, gs, gt = api.mmd_gaussian(ctx, torch.tensor(Xs, device="cuda"),
                                           torch.tensor(Xt, device="cuda"))
        out.append((v, np.concatenate([gs.cpu().numpy(), gt.cpu().numpy()])))
    ov, _, ogs, ogt = po.mmd_gaussian(Xs.astype(np.float64), Xt.astype(np.float64))
    og = np.concatenate([ogs, ogt])
    for v, g in out:
        assert rel(v, ov) <= TOL
        assert rel(g, og) <= TOL


@pytest.mark.parametrize("m,n,d", [(3000, 1000, 64), (700, 332, 96), (600, 400, 128)])
def test_mmd_api_materialised_w_path(ctx, monkeypatch, m, n, d):
    """Xs, Xt given as views of one [m + n, d] block: the C-ABI call takes the
    materialised-W path (each unordered 128x128 tile pair once, V = W.Z as a
    GEMM).  It must agree with the fused pair kernel (MTK_MMD_FUSED=1) and the
    f64 oracle.  N > 1024 runs V as 1024-deep GEMMs summed in fp64 (N = 4000,
    1032); N = 1000 is one GEMM with the fused gradient epilogue."""
    from paper_2011_09463_b200 import api

    rng = np.random.default_rng(m + d)
    Z = rng.standard_normal((m + n, d)).astype(np.float32)
    Z[m:] += 0.2
    Zd = torch.tensor(Z, device="cuda")
    res = []
    for fused in ("0", "1"):
        monkeypatch.setenv("MTK_MMD_FUSED", fused)
        torch.cuda.synchronize()
        n0 = ctx.launches
        v, beta, gs, gt = api.mmd_gaussian(ctx, Zd[:m], Zd[m:])
        res.append((v, beta, gs.cpu().numpy(), gt.cpu().numpy(), ctx.launches - n0))
    (v0, b0, gs0, gt0, n0), (v1, b1, gs1, gt1, n1) = res
    assert n0 != n1  # different kernels ran
    assert b0 == b1
    assert abs(v0 - v1) <= 1e-5 * abs(v1)
    assert rel(gs0, gs1) <= 2e-5 and rel(gt0, gt1) <= 2e-5
    ov, ob, ogs, ogt = po.mmd_gaussian(Z[:m].astype(np.float64), Z[m:].astype(np.float64))
    assert abs(v0 - ov) <= 1e-5 * abs(ov)
    assert rel(gs0, ogs) <= 1e-5 and rel(gt0, ogt) <= 1e-5


@pytest.mark.parametrize("m,n,d", [(512, 512, 256), (700, 324, 64)])
def test_mmd_w_diagonal_tiles_share_operands_bit_identically(ctx, monkeypatch, m, n, d):
    """mmd_w loads a diagonal tile pair's operand planes once and swaps the
    two accumulator blocks (B = [Z_I hi | Z_I lo]); the epilogue's sum is
    commutative, so value, bandwidth and gradients are bit-identical to
    loading Z_J separately (MTK_MMDW_NO_DIAG_SHARE=1)."""
    from paper_2011_09463_b200 import api

    rng = np.random.default_rng(m + 3 * d)
    Z = rng.standard_normal((m + n, d)).astype(np.float32)
    Z[m:] += 0.25
    Zd = torch.tensor(Z, device="cuda")
    res = []
    for off in ("0", "1"):
        monkeypatch.setenv("MTK_MMDW_NO_DIAG_SHARE", off)
        v, beta, gs, gt = api.mmd_gaussian(ctx, Zd[:m], Zd[m:])
        res.append((v, beta, gs.cpu().numpy(), gt.cpu().numpy()))
    (v0, b0, gs0, gt0), (v1, b1, gs1, gt1) = res
    assert v0 == v1 and b0 == b1
    assert np.array_equal(gs0, gs1) and np.array_equal(gt0, gt1)


def _f64_mmd_reference(Z, m, beta, rows, mult=(0.25, 0.5, 1.0, 2.0, 4.0), tile=4096):
    """Independent fp64 evaluation on the GPU (torch float64, tiled): the
    V-statistic MMD^2 over ALL pairs and the gradient of the given rows, in
    the difference form of SURVEY.md Appendix A (no shared code with libmtk)."""
    N = Z.shape[0]
    n = N - m
    Zd = Z.double()
    nrm = (Zd * Zd).sum(1)
    dom = torch.arange(N, device=Z.device) >= m
    tot = torch.zeros(3, dtype=torch.float64, device=Z.device)  # ss, tt, st (ordered double sums)
    for a0 in range(0, N, tile):
        a1 = min(N, a0 + tile)
        d2 = (nrm[a0:a1, None] + nrm[None, :] - 2.0 * (Zd[a0:a1] @ Zd.T)).clamp_min_(0.0)
        k = sum(torch.exp(-d2 / (beta * q)) for q in mult)
        di = dom[a0:a1, None]
        tot[0] += k[~di.expand_as(k) & ~dom[None, :]].sum()
        tot[1] += k[di.expand_as(k) & dom[None, :]].sum()
        tot[2] += k[~di.expand_as(k) & dom[None, :]].sum()
        del d2, k
    value = tot[0] / (m * m) + tot[1] / (n * n) - 2.0 * tot[2] / (m * n)
    G = []
    for i in rows:
        diff = Zd[i][None, :] - Zd
        d2 = (diff * diff).sum(1)
        A = sum(2.0 / (beta * q) * torch.exp(-d2 / (beta * q)) for q in mult)
        same = (dom == dom[i])
        c = torch.where(same, torch.tensor(-2.0 / (n * n) if i >= m else -2.0 / (m * m), dtype=torch.float64,
                                           device=Z.device),
                        torch.tensor(2.0 / (m * n), dtype=torch.float64, device=Z.device))
        c[i] = 0.0
        G.append(((c * A)[:, None] * diff).sum(0))
    return float(value), torch.stack(G).cpu().numpy()


def test_mmd_c4_materialised_w_path_vs_fp64(ctx, monkeypatch):
    """C4 at full scale on the path its 1-GPU number is measured on: Xs, Xt
    views of one [73728, 512] block -> the materialised-W path (21.7 GB of W,
    166,176 unique tile pairs, V as 72 1024-deep GEMMs summed in fp64).  The
    MMD^2 value and 16 sampled gradient rows (both domains, first / last /
    interior rows, tile edges) against an independent fp64 evaluation at 1e-5,
    and against the fused pair kernel (MTK_MMD_FUSED=1) on the same rows."""
    from paper_2011_09463_b200 import api

    m, n, d = 65536, 8192, 512
    g = torch.Generator(device="cuda").manual_seed(4)
    Z = torch.randn(m + n, d, device="cuda", generator=g)
    Z[m:] += 0.1
    Xs, Xt = Z[:m], Z[m:]
    rows = [0, 1, 127, 128, 4095, 12345, 40000, m - 129, m - 1, m, m + 1, m + 1023, m + 1024,
            m + 4321, m + n - 128, m + n - 1]
    monkeypatch.setenv("MTK_MMD_FUSED", "0")
    torch.cuda.synchronize()
    v, beta, gs, gt = api.mmd_gaussian(ctx, Xs, Xt)
    Gw = torch.cat([gs, gt])[rows].double().cpu().numpy()
    del gs, gt
    ref_v, ref_g = _f64_mmd_reference(Z, m, beta, rows)
    # beta: the fp64 closed form on the same fp32 inputs
    Zd = Z.double()
    N = m + n
    ob = float((2.0 * N * (Zd * Zd).sum() - 2.0 * (Zd.sum(0) ** 2).sum()) / (N * N - N))
    assert abs(beta - ob) <= 1e-9 * ob
    assert abs(v - ref_v) <= TOL * abs(ref_v), (v, ref_v)
    print(f"C4 W path: value {abs(v - ref_v) / abs(ref_v):.2e}, gradient rows {rel(Gw, ref_g):.2e} (bound {TOL})")
    assert rel(Gw, ref_g) <= TOL, rel(Gw, ref_g)
    for r, i in enumerate(rows):  # row by row too (each row's own scale)
        assert rel(Gw[r], ref_g[r]) <= 2 * TOL, (i, rel(Gw[r], ref_g[r]))
    monkeypatch.setenv("MTK_MMD_FUSED", "1")
    v1, b1, gs1, gt1 = api.mmd_gaussian(ctx, Xs, Xt)
    G1 = torch.cat([gs1, gt1])[rows].double().cpu().numpy()
    assert b1 == beta
    assert abs(v1 - v) <= TOL * abs(v)
    assert rel(Gw, G1) <= 2 * TOL


@pytest.mark.parametrize("m,n,d,world", [(700, 324, 64, 2), (3000, 1000, 96, 3), (1500, 600, 128, 4)])
def test_mmd_tile_sharding_is_bit_identical_to_one_rank(ctx, m, n, d, world):
    """SURVEY.md 8(e) on the materialised-W path: `world` ranks each own an
    equal range of 128-row tiles (simulated one after another on this GPU --
    the ranks never wait on each other); the gradients of each rank's rows and
    the MMD^2 value from the ascending-tile combination of the partials are
    bit-identical to the one-rank evaluation (ragged last tiles, chunked V
    for N > 1024)."""
    from paper_2011_09463_b200 import api

    rng = np.random.default_rng(m + world)
    Z = torch.tensor(rng.standard_normal((m + n, d)).astype(np.float32), device="cuda")
    Z[m:] += 0.2
    v1, beta, gs, gt = api.mmd_gaussian(ctx, Z[:m], Z[m:])
    g1 = torch.cat([gs, gt])
    gZ = torch.full_like(Z, float("nan"))
    tot = None
    for lo, hi in api.mmd_tile_ranges(m, n, world):
        part = api.mmd_gaussian_tiles(ctx, Z, m, beta, lo, hi, gZ)
        assert not part[:lo].any() and not part[hi:].any()
        tot = part if tot is None else tot + part  # one owner per tile row: exact
    assert torch.equal(gZ, g1)
    assert api.mmd_value_from_tiles(tot, m, n) == v1
