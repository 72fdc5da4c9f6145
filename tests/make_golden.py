"""Mint the golden fixtures in tests/golden/ (run here, where /root/reference
is mounted; the fixtures travel, the reference does not).

  python tests/make_golden.py

Sources:
  * rng / mlp / softmax: oracle/_ref/libmtref.so -- the reference headers
    (/root/reference/proj/include/minitransfer) compiled unmodified;
  * mmd: an independent numpy f64 implementation written here (not the
    oracle), since the reference has no MMD;
  * auc: sklearn.metrics.roc_auc_score.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
import pyoracle as po  # noqa: E402

OUT = os.path.join(HERE, "golden")


def ref_rng_draws(seed):
    R = po.ref()
    h = R.ref_rng_create(seed)
    u64 = np.array([R.ref_rng_next(h) for _ in range(64)], dtype=np.uint64)
    nrm = np.array([R.ref_rng_normal(h) for _ in range(65)])
    uni = np.array([R.ref_rng_uniform_range(h, -0.3, 0.7) for _ in range(64)])
    bel = np.array([R.ref_rng_below(h, 10) for _ in range(64)], dtype=np.uint64)
    perm = np.empty(100, dtype=np.uint64)
    R.ref_rng_permutation(h, 100, perm.ctypes.data_as(po._u64p))
    c = R.ref_rng_split(h, 3)
    spl = np.array([R.ref_rng_next(c) for _ in range(8)], dtype=np.uint64)
    R.ref_rng_destroy(c)
    R.ref_rng_destroy(h)
    return dict(u64=u64, normal=nrm, uniform=uni, below=bel, perm=perm, split=spl)


def make_rng():
    out = {}
    for s in (0, 1, 42, 20110946):
        for k, v in ref_rng_draws(s).items():
            out[f"s{s}_{k}"] = v
    np.savez_compressed(os.path.join(OUT, "rng_ref.npz"), **out)


def init_ref(seed, dims, n_heads):
    """init through the reference Rng (uniform +-1/sqrt(fan_in))"""
    R = po.ref()
    h = R.ref_rng_create(seed)
    L = len(dims) - 1
    shapes = [(dims[l], dims[l + 1]) for l in range(L)]
    if n_heads == 2:
        shapes.append((dims[L - 1], dims[L]))
    W, b = [], []
    for (fi, fo) in shapes:
        lim = 1.0 / np.sqrt(fi)
        W.append(np.array([R.ref_rng_uniform_range(h, -lim, lim) for _ in range(fi * fo)]).reshape(fi, fo))
        b.append(np.zeros(fo))
    X = np.array([R.ref_rng_normal(h) for _ in range(9 * dims[0])]).reshape(9, dims[0])
    y = np.array([R.ref_rng_below(h, dims[-1]) for _ in range(9)], dtype=np.int32)
    R.ref_rng_destroy(h)
    return W, b, X, y


MLP_CASES = {
    "plain": dict(dims=[6, 5, 4, 3], n_heads=1, frozen=0, inject=False, src=0),
    "inject": dict(dims=[6, 5, 4, 3], n_heads=1, frozen=0, inject=True, src=4),
    "frozen": dict(dims=[6, 5, 4, 3], n_heads=1, frozen=1, inject=False, src=0),
    "two_heads": dict(dims=[6, 5, 4, 3], n_heads=2, frozen=0, inject=False, src=4),
    "weighted": dict(dims=[7, 3], n_heads=1, frozen=0, inject=False, src=0),
}


def make_mlp():
    out = {}
    for name, c in MLP_CASES.items():
        W, b, X, y = init_ref(7, c["dims"], c["n_heads"])
        out[f"{name}_W0"] = np.array(W, dtype=object)
        for i, (w, bb) in enumerate(zip(W, b)):
            out[f"{name}_W{i}_before"] = w.copy()
            out[f"{name}_b{i}_before"] = bb.copy()
        out[f"{name}_X"] = X
        out[f"{name}_y"] = y
        dH = None
        if c["inject"]:
            _, H = po.ref_mlp_forward(c["dims"], W, b, X)
            v, _, gs, gt = mmd_numpy(H[:c["src"]], H[c["src"]:], np.array(po.MMD_MULT))
            dH = np.concatenate([gs, gt])
            out[f"{name}_dH"] = dH
        w = None
        if name == "weighted":
            w = np.array([0.5, 0.0, 1.0, 2.0, 1.0, 1.0, 0.25, 3.0, 1.0])
            out[f"{name}_w"] = w
        loss, gW, gb = po.ref_mlp_train_step(c["dims"], W, b, X, y, n_heads=c["n_heads"],
                                             frozen=c["frozen"], src_rows=c["src"], lr=0.1, dH=dH,
                                             w=w, denoms=[4.5] if name == "weighted" else None,
                                             want_grads=True)
        out[f"{name}_loss"] = np.array([loss])
        for i in range(len(W)):
            out[f"{name}_W{i}_after"] = W[i].copy()
            out[f"{name}_b{i}_after"] = b[i]
            out[f"{name}_gW{i}"] = gW[i]
            out[f"{name}_gb{i}"] = gb[i]
    out = {k: v for k, v in out.items() if not k.endswith("_W0")}
    np.savez_compressed(os.path.join(OUT, "mlp_ref.npz"), **out)


def mmd_numpy(Xs, Xt, mult, beta=None):
    """Independent f64 implementation of SURVEY.md Appendix A (vectorised)."""
    Z = np.concatenate([Xs, Xt])
    m, n = len(Xs), len(Xt)
    N = m + n
    if beta is None:
        D = ((Z[:, None, :] - Z[None, :, :]) ** 2).sum(-1)
        beta = D.sum() / (N * N - N)
    D = ((Z[:, None, :] - Z[None, :, :]) ** 2).sum(-1)
    K = sum(np.exp(-D / (beta * q)) for q in mult)
    A = sum(2.0 / (beta * q) * np.exp(-D / (beta * q)) for q in mult)
    s = np.arange(N) < m
    val = K[np.ix_(s, s)].sum() / m**2 + K[np.ix_(~s, ~s)].sum() / n**2 - 2 * K[np.ix_(s, ~s)].sum() / (m * n)
    c = np.where(s[:, None] & s[None, :], -2.0 / m**2,
                 np.where(~s[:, None] & ~s[None, :], -2.0 / n**2, 2.0 / (m * n)))
    np.fill_diagonal(c, 0.0)
    W = c * A
    g = W.sum(1)[:, None] * Z - W @ Z
    return val, beta, g[:m], g[m:]


def make_mmd():
    out = {}
    rng = np.random.default_rng(0)
    for i, (m, n, d) in enumerate([(7, 5, 3), (16, 16, 8), (1, 2, 4), (30, 11, 20)]):
        Xs = rng.standard_normal((m, d))
        Xt = rng.standard_normal((n, d)) + 0.4
        v, beta, gs, gt = mmd_numpy(Xs, Xt, np.array(po.MMD_MULT))
        out.update({f"c{i}_Xs": Xs, f"c{i}_Xt": Xt, f"c{i}_value": np.array([v]),
                    f"c{i}_beta": np.array([beta]), f"c{i}_gXs": gs, f"c{i}_gXt": gt})
    np.savez_compressed(os.path.join(OUT, "mmd_numpy.npz"), **out)


def make_auc():
    from sklearn.metrics import roc_auc_score

    out = {}
    rng = np.random.default_rng(1)
    for i, (n, ties) in enumerate([(50, False), (200, True), (1000, True), (3, False)]):
        s = rng.standard_normal(n)
        if ties:
            s = np.round(s * 2) / 2
        lab = (rng.standard_normal(n) + s > 0).astype(np.uint8)
        lab[0], lab[-1] = 1, 0
        out.update({f"c{i}_s": s, f"c{i}_l": lab, f"c{i}_auc": np.array([roc_auc_score(lab, s)])})
    np.savez_compressed(os.path.join(OUT, "auc_sklearn.npz"), **out)


if __name__ == "__main__":
    assert po.ref() is not None, "oracle/_ref/libmtref.so missing: run make -C oracle here"
    os.makedirs(OUT, exist_ok=True)
    make_rng()
    make_mlp()
    make_mmd()
    make_auc()
    print("golden fixtures written to", OUT)
