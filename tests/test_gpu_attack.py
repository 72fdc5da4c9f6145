"""GPU parity of the attack stage: posteriors, top-k features, AUC."""
import numpy as np
import pytest
import torch

import pyoracle as po

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def logits(rows, C, seed=1, scale=3.0):
    r = po.Rng(seed)
    return (scale * r.normals(rows * C)).reshape(rows, C).astype(np.float32)


def test_softmax_matches_reference_semantics(ctx):
    from paper_2011_09463_b200 import api

    x = logits(1000, 10)
    p = api.softmax(ctx, torch.tensor(x, device="cuda")).cpu().numpy()
    assert rel(p, po.softmax(x.astype(np.float64))) <= 1e-5
    assert np.abs(p.sum(1) - 1).max() < 1e-5
    # SPEC.md:70 known answer softmax([0, ln 3]) = [0.25, 0.75]
    kq = api.softmax(ctx, torch.tensor([[0.0, np.log(3.0)]], dtype=torch.float32, device="cuda"))
    assert np.allclose(kq.cpu().numpy(), [[0.25, 0.75]], atol=1e-7)


@pytest.mark.parametrize("k,with_labels", [(3, False), (3, True), (1, True), (10, False)])
def test_features(ctx, k, with_labels):
    from paper_2011_09463_b200 import api

    x = logits(777, 10, seed=k)
    lab = np.arange(777, dtype=np.int32) % 10 if with_labels else None
    f = api.posterior_features(ctx, torch.tensor(x, device="cuda"), k,
                               None if lab is None else torch.tensor(lab, device="cuda"))
    of = po.posterior_features(x.astype(np.float64), k, lab)
    assert rel(f.cpu().numpy(), of) <= 1e-5


def test_posterior_column(ctx):
    from paper_2011_09463_b200 import api

    x = logits(500, 2)
    c = api.posterior_column(ctx, torch.tensor(x, device="cuda"), 1).cpu().numpy()
    assert rel(c, po.softmax(x.astype(np.float64))[:, 1]) <= 1e-5


@pytest.mark.parametrize("n,ties", [(1000, False), (4096, True), (1 << 20, False), (7, True)])
def test_auc_matches_oracle(ctx, n, ties):
    from paper_2011_09463_b200 import api

    r = po.Rng(n)
    s = r.normals(n).astype(np.float32)
    if ties:
        s = np.round(s * 4) / 4
    lab = np.array([r.below(2) for _ in range(n)], dtype=np.uint8) if n < 100000 else \
        (r.normals(n) + 0.3 * s > 0).astype(np.uint8)
    lab[0], lab[-1] = 1, 0
    a, acc = api.auc(ctx, torch.tensor(s, device="cuda"), torch.tensor(lab, device="cuda"))
    oa = po.auc(s.astype(np.float64), lab)
    oacc = po.accuracy(s.astype(np.float64), lab, 0.5)
    assert abs(a - oa) <= 1e-12
    assert abs(acc - oacc) <= 1e-12


def test_auc_errors(ctx):
    from paper_2011_09463_b200 import api, errors

    with pytest.raises(errors.ValueError):
        api.auc(ctx, torch.zeros(10, device="cuda"), torch.ones(10, dtype=torch.uint8, device="cuda"))


def test_gather_rows_matches_indexing(ctx):
    """mtk_gather_rows: device batch assembly (bitwise copies, row offsets)."""
    from paper_2011_09463_b200 import api, errors

    g = torch.Generator().manual_seed(3)
    X = torch.randn(500, 37, generator=g).cuda()
    y = torch.randint(0, 10, (500,), generator=g, dtype=torch.int32).cuda()
    idx = torch.randint(0, 500, (4, 9), generator=g, dtype=torch.int64).cuda()
    out = torch.zeros(4, 20, 37, device="cuda")
    api.gather_rows(ctx, X, idx, out, row0=5)
    assert torch.equal(out[:, 5:14], X[idx])
    assert torch.equal(out[:, :5], torch.zeros_like(out[:, :5]))
    yo = torch.zeros(4, 9, 1, device="cuda", dtype=torch.int32)
    api.gather_rows(ctx, y, idx, yo)
    assert torch.equal(yo[..., 0], y[idx])
    bad = idx.clone()
    bad[1, 2] = 500
    api.gather_rows(ctx, X, bad, out, row0=5)
    with pytest.raises(errors.ValueError):
        ctx.synchronize()


@pytest.mark.parametrize("rows,C,dims,ties", [(65573, 10, [3, 64, 2], False), (4096, 10, [3, 64, 2], True),
                                              (3001, 16, [3, 64, 2], False), (2000, 7, [4, 32, 2], False)])
def test_attack_auc_in_one_call(ctx, rows, C, dims, ties):
    """mtk_attack_auc (features -> attack model -> member probability -> AUC in
    one call; the [3, 64, 2] model as one streaming kernel) must reproduce the
    four-call composition bit for bit: scores, AUC and accuracy; other attack
    shapes take the composition itself.  AUC and accuracy are also checked
    against the oracle on the GPU scores."""
    from paper_2011_09463_b200 import api

    x = logits(rows, C, seed=rows)
    if ties:
        x = np.round(x)
    r = po.Rng(rows + 1)
    lab = np.array([r.below(2) for _ in range(rows)], dtype=np.uint8)
    lab[0], lab[1] = 1, 0
    xd, ld = torch.tensor(x, device="cuda"), torch.tensor(lab, device="cuda")
    att = api.Bank(ctx, 1, dims)
    att.init_params(0, api.Rng(5))
    a1, acc1, s1 = api.attack_auc(att, xd, ld, scores=True)
    F = api.posterior_features(ctx, xd, dims[0])
    out = att.forward(F.reshape(1, rows, dims[0]))
    s2 = api.posterior_column(ctx, out, 1)
    a2, acc2 = api.auc(ctx, s2, ld)
    assert torch.equal(s1, s2)
    assert a1 == a2 and acc1 == acc2
    sc = s1.cpu().numpy().astype(np.float64)
    assert abs(a1 - po.auc(sc, lab)) <= 1e-12
    assert abs(acc1 - po.accuracy(sc, lab, 0.5)) <= 1e-12


def _u2_numpy(s, lab):
    """exact U2 = sum over members of 2 #{non-members below} + #{equal}
    (integers; numpy sort + searchsorted on float64 scores)"""
    neg = np.sort(s[lab == 0].astype(np.float64))
    pos = s[lab == 1].astype(np.float64)
    lo = np.searchsorted(neg, pos, side="left")
    hi = np.searchsorted(neg, pos, side="right")
    return int((2 * lo + (hi - lo)).sum()), int(lab.sum())


@pytest.mark.parametrize("case", ["spread", "few_values", "one_value", "signed_zero", "narrow", "huge_bucket",
                                  "tiny", "fast_edge", "general_edge", "fast_dense"])
def test_auc_histogram_paths_exact(ctx, case):
    """The sort-free AUC (auc.cuh) on both paths: the full-resolution key
    histogram (key range < 2^23: one_value, narrow, huge_bucket, fast_edge =
    a range of exactly 2^23 - 1 keys, fast_dense = 2^20 queries over a 2^20
    range) and the top-16-bit buckets (wider: spread, few_values,
    signed_zero, tiny, general_edge = a range of exactly 2^23): cross-bucket
    counts, small buckets (shared-memory sort), large buckets (65536-bin
    histogram), all-equal scores, -0.0 == +0.0, negative scores -- the AUC
    equals the exact integer U2 / 2 / (npos nneg) computed independently."""
    from paper_2011_09463_b200 import api

    rng = np.random.default_rng(hash(case) % 2**32)
    n = 300_000
    if case == "spread":
        s = rng.standard_normal(n).astype(np.float32) * 1e3
    elif case == "few_values":  # 37 distinct values: every bucket large, many ties
        s = (rng.integers(0, 37, n) / 37.0).astype(np.float32)
    elif case == "one_value":
        s = np.full(n, 0.3, dtype=np.float32)
    elif case == "signed_zero":
        s = np.where(rng.random(n) < 0.5, np.float32(0.0), np.float32(-0.0)).astype(np.float32)
        s[:1000] = rng.standard_normal(1000).astype(np.float32)
    elif case == "narrow":  # scores in [0.5, 0.5 + 2^-8): a handful of hi-16 buckets
        s = (0.5 + rng.random(n) / 256).astype(np.float32)
    elif case == "huge_bucket":  # one bucket with ~all queries, distinct low bits
        s = np.float32(0.75) + (rng.integers(0, 60000, n) * np.float32(2.0 ** -24)).astype(np.float32)
    elif case in ("fast_edge", "general_edge"):  # floats in [1, 2] have consecutive keys
        k = rng.integers(0, 1 << 23, n, dtype=np.int64)
        k[1] = 0
        k[2] = (1 << 23) - 1 if case == "fast_edge" else 1 << 23  # 2^23 - 1 / 2^23 keys of range
        s = (np.uint32(0x3F800000) + k.astype(np.uint32)).view(np.float32)
    elif case == "fast_dense":  # attack-score-like: 2^20 queries, ~2^20-key range, many ties
        n = 1 << 20
        s = np.float32(0.5) + (rng.integers(0, 1 << 20, n) * np.float32(2.0 ** -24)).astype(np.float32)
    else:
        n = 5
        s = np.array([0.1, 0.4, 0.35, 0.8, 0.4], dtype=np.float32)
    lab = (rng.random(n) < 0.4).astype(np.uint8)
    lab[0], lab[-1] = 1, 0
    a, acc = api.auc(ctx, torch.tensor(s, device="cuda"), torch.tensor(lab, device="cuda"))
    u2, npos = _u2_numpy(s, lab)
    nneg = n - npos
    assert a == (0.5 * u2) / (npos * nneg), (a, u2)
    assert abs(a - po.auc(s.astype(np.float64), lab)) <= 1e-12
    assert acc == float(((s > 0.5) == (lab == 1)).sum()) / n
