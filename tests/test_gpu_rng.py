"""Counter-based device data (k_rng.cu) against the
oracle restatement (oracle.c orc_philox4x64 / orc_synth_counter, itself
pinned to the Random123 known answer and numpy's Philox in test_oracle.py).

Contract: raw Philox words and labels bit-exact; normals (fp32 device
transform vs the oracle's f64 libm transform) within
|dz| <= 8 ulp_fp32(max(1, |z|)); X = mu[y] + z (+ shift) within the same
bound plus one rounding of the sums.
"""
import numpy as np
import pytest
import torch

import pyoracle as po

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_2011_09463_b200 import api

    return api.Context(0)


def _u64(t):
    return [int(x) & (2**64 - 1) for x in t.cpu().numpy().ravel().tolist()]


@pytest.mark.parametrize("seed,stream,ctr0,ctr1", [(0, 0, 0, 0), (20110946, 1, 0, 0),
                                                   (2**64 - 1, 2**63 + 5, 2**40, 1), (7, 3, 123, 0)])
def test_philox_words_bit_exact(ctx, seed, stream, ctr0, ctr1):
    from paper_2011_09463_b200 import api

    n = 1000
    got = _u64(api.philox4x64_fill(ctx, seed, stream, n, ctr0, ctr1))
    for i in list(range(0, n, 97)) + [n - 1]:
        assert got[4 * i:4 * i + 4] == po.philox4x64([ctr0 + i, ctr1, 0, 0], [seed, stream]), i
    if seed == stream == ctr0 == ctr1 == 0:
        assert got[:4] == [0x16554D9ECA36314C, 0xDB20FE9D672D0FDC, 0xD7E772CEE186176B,
                           0x7E68B68AEC7BA23B]


def _ulp_bound(z):
    return 8 * np.spacing(np.maximum(1.0, np.abs(z)).astype(np.float32)).astype(np.float64)


@pytest.mark.parametrize("first,count", [(0, 1 << 20), (3, 4097), (1 << 33, 1000)])
def test_counter_normals_match_oracle(ctx, first, count):
    from paper_2011_09463_b200 import api

    z = api.counter_normals(ctx, 99, 2, first, count).cpu().numpy().astype(np.float64)
    ref = po.counter_normals(99, 2, first, count)
    err = np.abs(z - ref)
    assert np.all(err <= _ulp_bound(ref)), (err.max(), np.argmax(err / _ulp_bound(ref)))


@pytest.mark.parametrize("C,d,n,shift", [(10, 784, 3000, True), (10, 33, 1001, False),
                                         (100, 512, 257, True), (2, 4, 5, False)])
def test_synth_counter_matches_oracle(ctx, C, d, n, shift):
    from paper_2011_09463_b200 import api

    rs = np.random.default_rng(C * d)
    mu = (0.3 * rs.standard_normal((C, d))).astype(np.float32)
    sh = (0.5 * rs.standard_normal(d)).astype(np.float32) if shift else None
    X, y = api.synth_counter(ctx, 20110946, 1, n, torch.from_numpy(mu),
                             None if sh is None else torch.from_numpy(sh))
    Xr, yr = po.synth_counter(20110946, 1, C, d, n, mu.astype(np.float64),
                              None if sh is None else sh.astype(np.float64))
    assert np.array_equal(y.cpu().numpy(), yr)
    Xg = X.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(Xg - Xr) <= _ulp_bound(Xr) + 2 * np.spacing(np.abs(Xr).astype(np.float32))), \
        np.abs(Xg - Xr).max()


def test_synth_counter_pool_scale(ctx):
    # one C5-scale pool (2^20 x 784) straight into HBM; labels / moments sane
    from paper_2011_09463_b200 import api

    mu = torch.zeros(10, 784)
    X, y = api.synth_counter(ctx, 5, 1, 1 << 20, mu)
    torch.cuda.synchronize()
    assert X.shape == (1 << 20, 784) and int(y.min()) >= 0 and int(y.max()) < 10
    cnt = torch.bincount(y.long(), minlength=10).cpu().numpy()
    assert cnt.min() > 0.98 * (1 << 20) / 10
    m, v = X.mean().item(), X.var().item()
    assert abs(m) < 1e-3 and abs(v - 1.0) < 1e-3
