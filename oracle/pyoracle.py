"""TEST INFRASTRUCTURE ONLY: numpy/ctypes front-end for the CPU oracle.

Loads ``oracle/liboracle.so`` (the C restatement, oracle.c) and, when present,
``oracle/_ref/libmtref_v{3,4}.so`` (the shim over the UNMODIFIED reference headers,
ref_shim.cpp).  Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU
legs import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORC = os.path.join(HERE, "liboracle.so")
_REF_V = {v: os.path.join(HERE, "_ref", f"libmtref_{v}.so") for v in ("v3", "v4")}


def host_isa() -> str:
    """x86-64 micro-architecture level of this host: "v4" with AVX-512
    (F/BW/CD/DQ/VL), else "v3" -- picks the libmtref build ("-march=native"
    resolved on the box that runs it)."""
    try:
        with open("/proc/cpuinfo") as f:
            flags = next((ln.split(":", 1)[1].split() for ln in f if ln.startswith("flags")), [])
    except OSError:
        flags = []
    return "v4" if {"avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"} <= set(flags) else "v3"


def ref_path():
    """the libmtref build for this host (None when never built)"""
    for v in (host_isa(), "v3"):
        if os.path.exists(_REF_V[v]):
            return _REF_V[v]
    return None


def cpu_info() -> dict:
    """CPU model / threads usable / ISA level, recorded beside CPU timings"""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), model)
    except OSError:
        pass
    try:
        threads = len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        threads = os.cpu_count() or 1
    return {"cpu_model": model, "nproc": os.cpu_count(), "threads_available": threads,
            "isa": "x86-64-" + host_isa()}

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_i32p = C.POINTER(C.c_int32)
_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _load(path):
    if not os.path.exists(path):
        return None
    return C.CDLL(path)


_orc = None
_ref = None


def orc():
    global _orc
    if _orc is None:
        if not os.path.exists(_ORC):
            build()
        _orc = C.CDLL(_ORC)
        _setup_orc(_orc)
    return _orc


def ref():
    """The reference-header shim, or None when it was never built here."""
    global _ref
    if _ref is None:
        p = ref_path()
        _ref = _load(p) if p else None
        if _ref is not None:
            _setup_ref(_ref)
    return _ref


def _setup_orc(L):
    L.orc_rng_sizeof.restype = C.c_size_t
    L.orc_rng_next.restype = C.c_uint64
    L.orc_rng_uniform.restype = C.c_double
    L.orc_rng_uniform_range.restype = C.c_double
    L.orc_rng_uniform_range.argtypes = [C.c_void_p, C.c_double, C.c_double]
    L.orc_rng_normal.restype = C.c_double
    L.orc_rng_below.restype = C.c_uint64
    L.orc_rng_below.argtypes = [C.c_void_p, C.c_uint64]
    L.orc_rng_seed.argtypes = [C.c_void_p, C.c_uint64]
    L.orc_rng_split.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p]
    L.orc_rng_permutation.argtypes = [C.c_void_p, C.c_size_t, _u64p]
    L.orc_rng_fill_normal.argtypes = [C.c_void_p, _dp, C.c_size_t]
    L.orc_rng_fill_uniform_range.argtypes = [C.c_void_p, _dp, C.c_size_t, C.c_double, C.c_double]
    L.orc_mmd_gaussian.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t, _dp, C.c_int,
                                   C.c_double, _dp, _dp, _dp, _dp]
    L.orc_mmd_beta.restype = C.c_double
    L.orc_mmd_beta.argtypes = [_dp, C.c_size_t, _dp, C.c_size_t, C.c_size_t]
    L.orc_softmax.argtypes = [_dp, C.c_size_t, C.c_int, _dp]
    L.orc_posterior_features.argtypes = [_dp, C.c_size_t, C.c_int, C.c_int, _i32p, _dp]
    L.orc_auc.argtypes = [_dp, _u8p, C.c_size_t, _dp]
    L.orc_accuracy.restype = C.c_double
    L.orc_accuracy.argtypes = [_dp, _u8p, C.c_size_t, C.c_double]
    L.orc_synth.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_size_t, _dp, _dp, _dp, _i32p]
    L.orc_philox4x64.argtypes = [C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
    L.orc_counter_normals.argtypes = [C.c_uint64, C.c_uint64, C.c_size_t, C.c_size_t, _dp]
    L.orc_synth_counter.argtypes = [C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_size_t, _dp, _dp,
                                    _dp, _i32p]
    step_args = [C.c_int, _ip, C.c_int, C.c_int, C.POINTER(_dp), C.POINTER(_dp), _dp, C.c_int,
                 C.c_int, _i32p, _dp, _dp, C.c_double, _dp, _dp, C.POINTER(_dp), C.POINTER(_dp)]
    L.orc_mlp_train_step.argtypes = step_args
    L.orc_mlp_forward.argtypes = [C.c_int, _ip, C.c_int, C.POINTER(_dp), C.POINTER(_dp), _dp,
                                  C.c_int, _dp, _dp]
    L.orc_mlp_init.argtypes = [C.c_void_p, C.c_int, _ip, _ip, C.POINTER(_dp), C.POINTER(_dp)]
    L.orc_adam_update.argtypes = [_dp, _dp, _dp, _dp, C.c_size_t, C.c_double, C.c_double,
                                  C.c_double, C.c_double, C.c_uint64]


def _setup_ref(L):
    L.ref_last_error.restype = C.c_char_p
    L.ref_rng_create.restype = C.c_void_p
    L.ref_rng_create.argtypes = [C.c_uint64]
    L.ref_rng_destroy.argtypes = [C.c_void_p]
    for n in ("ref_rng_next", "ref_rng_below"):
        getattr(L, n).restype = C.c_uint64
    L.ref_rng_next.argtypes = [C.c_void_p]
    L.ref_rng_below.argtypes = [C.c_void_p, C.c_uint64]
    for n in ("ref_rng_uniform", "ref_rng_normal"):
        getattr(L, n).restype = C.c_double
        getattr(L, n).argtypes = [C.c_void_p]
    L.ref_rng_uniform_range.restype = C.c_double
    L.ref_rng_uniform_range.argtypes = [C.c_void_p, C.c_double, C.c_double]
    L.ref_rng_permutation.argtypes = [C.c_void_p, C.c_size_t, _u64p]
    L.ref_rng_split.restype = C.c_void_p
    L.ref_rng_split.argtypes = [C.c_void_p, C.c_uint64]
    L.ref_mlp_train_step.argtypes = [C.c_int, _ip, C.c_int, C.c_int, C.POINTER(_dp),
                                     C.POINTER(_dp), _dp, C.c_int, C.c_int, _i32p, _dp, _dp,
                                     C.c_double, _dp, _dp, C.POINTER(_dp), C.POINTER(_dp)]
    L.ref_mlp_forward.argtypes = [C.c_int, _ip, C.c_int, C.POINTER(_dp), C.POINTER(_dp), _dp,
                                  C.c_int, _dp, _dp]
    L.ref_softmax.argtypes = [_dp, C.c_size_t, C.c_int, _dp]
    L.ref_grad_check_mmd.restype = C.c_double
    L.ref_grad_check_mmd.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _dp, C.c_int, _dp, _dp, _dp,
                                     C.c_int, C.c_double, C.c_double]
    L.ref_bench_mmd.restype = C.c_double
    L.ref_bench_mmd.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int, C.c_int64, C.c_uint64, _dp, _dp]
    L.ref_bench_attack.restype = C.c_double
    L.ref_bench_attack.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_uint64, _dp]
    L.ref_build_info.restype = C.c_char_p
    L.ref_bench_train_heads.restype = C.c_double
    L.ref_bench_train_heads.argtypes = [C.c_int, C.c_int, _ip, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_double, C.c_uint64]
    L.ref_bench_train.restype = C.c_double
    L.ref_bench_train.argtypes = [C.c_int, C.c_int, _ip, C.c_int, C.c_int, C.c_int, C.c_double,
                                  C.c_uint64]
    L.ref_adam_sequence.argtypes = [_dp, _dp, C.c_size_t, C.c_int, C.c_double, C.c_double,
                                    C.c_double, C.c_double]


def dp(a):
    return a.ctypes.data_as(_dp) if a is not None else None


def _ptrs(arrs):
    return (_dp * len(arrs))(*[dp(a) for a in arrs])


# ---------------------------------------------------------------- RNG
class Rng:
    """mt::Rng restated in C (oracle.c); same draws as rng.hpp."""

    def __init__(self, seed: int | None = None, _buf=None):
        L = orc()
        self._buf = _buf if _buf is not None else C.create_string_buffer(L.orc_rng_sizeof())
        if seed is not None:
            L.orc_rng_seed(self._buf, C.c_uint64(seed & (2**64 - 1)))

    @property
    def ptr(self):
        return C.cast(self._buf, C.c_void_p)

    def next_u64(self):
        return orc().orc_rng_next(self._buf)

    def uniform(self, lo=None, hi=None):
        if lo is None:
            return orc().orc_rng_uniform(self._buf)
        return orc().orc_rng_uniform_range(self._buf, lo, hi)

    def normal(self):
        return orc().orc_rng_normal(self._buf)

    def below(self, n):
        return orc().orc_rng_below(self._buf, n)

    def permutation(self, n):
        out = np.empty(n, dtype=np.uint64)
        orc().orc_rng_permutation(self._buf, n, out.ctypes.data_as(_u64p))
        return out

    def split(self, stream):
        child = Rng(None)
        orc().orc_rng_split(self._buf, stream, child._buf)
        return child

    def normals(self, n):
        out = np.empty(n, dtype=np.float64)
        orc().orc_rng_fill_normal(self._buf, dp(out), n)
        return out

    def uniforms(self, n, lo, hi):
        out = np.empty(n, dtype=np.float64)
        orc().orc_rng_fill_uniform_range(self._buf, dp(out), n, lo, hi)
        return out


# ---------------------------------------------------------------- MLP
def mlp_init(rng: Rng, dims, n_heads=1):
    """SPEC.md:182 init for one model: W uniform +-1/sqrt(fan_in), b = 0."""
    L = len(dims) - 1
    shapes = [(dims[l], dims[l + 1]) for l in range(L)]
    if n_heads == 2:
        shapes.append((dims[L - 1], dims[L]))
    W = [np.empty(s, dtype=np.float64) for s in shapes]
    b = [np.zeros(s[1], dtype=np.float64) for s in shapes]
    fi = (C.c_int * len(shapes))(*[s[0] for s in shapes])
    fo = (C.c_int * len(shapes))(*[s[1] for s in shapes])
    orc().orc_mlp_init(rng._buf, len(shapes), fi, fo, _ptrs(W), _ptrs(b))
    return W, b


def _train_step(fn, dims, W, b, X, y, *, n_heads=1, frozen=0, src_rows=0, w=None, denoms=None,
                lr=0.05, dH=None, want_grads=False):
    L = len(dims) - 1
    B = X.shape[0]
    X = np.ascontiguousarray(X, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.int32)
    if denoms is None:
        denoms = [float(B)] if n_heads == 1 else [float(src_rows), float(B - src_rows)]
    den = np.asarray(denoms, dtype=np.float64)
    dimsc = (C.c_int * (L + 1))(*dims)
    loss = C.c_double(0.0)
    gW = gb = None
    if want_grads:
        gW = [np.zeros_like(x) for x in W]
        gb = [np.zeros_like(x) for x in b]
    wv = None if w is None else np.ascontiguousarray(w, dtype=np.float64)
    dHv = None if dH is None else np.ascontiguousarray(dH, dtype=np.float64)
    st = fn(L, dimsc, n_heads, frozen, _ptrs(W), _ptrs(b), dp(X), B, src_rows,
            y.ctypes.data_as(_i32p), dp(wv), dp(den), lr, dp(dHv), C.byref(loss),
            _ptrs(gW) if gW else None, _ptrs(gb) if gb else None)
    if st != 0:
        raise RuntimeError(f"train step failed with status {st}")
    return (loss.value, gW, gb) if want_grads else loss.value


def mlp_train_step(dims, W, b, X, y, **kw):
    """Oracle (C restatement) SGD step; updates W/b in place."""
    return _train_step(orc().orc_mlp_train_step, dims, W, b, X, y, **kw)


class Adam:
    """Oracle Adam state over a list of parameter arrays (optim.hpp:13-26,
    49-63): moments aligned with the list order, one step counter."""

    def __init__(self, params, lr, beta1=0.9, beta2=0.999, eps=1e-8):
        self.lr, self.b1, self.b2, self.eps = lr, beta1, beta2, eps
        self.m = [np.zeros_like(p) for p in params]
        self.v = [np.zeros_like(p) for p in params]
        self.step = 0

    def update(self, params, grads):
        self.step += 1
        for p, g, m, v in zip(params, grads, self.m, self.v):
            g = np.ascontiguousarray(g, dtype=np.float64)
            orc().orc_adam_update(dp(p), dp(g), dp(m), dp(v), p.size, self.lr, self.b1, self.b2,
                                  self.eps, self.step)


def ref_adam_sequence(w, grads, lr, beta1=0.9, beta2=0.999, eps=1e-8):
    """mt::optimizer_step (Adam) applied len(grads) times to a copy of w."""
    w = np.array(w, dtype=np.float64).ravel()
    g = np.ascontiguousarray(np.stack([np.ravel(x) for x in grads]), dtype=np.float64)
    st = ref().ref_adam_sequence(dp(w), dp(g), w.size, len(grads), lr, beta1, beta2, eps)
    if st != 0:
        raise RuntimeError(ref().ref_last_error().decode())
    return w


def ref_mlp_train_step(dims, W, b, X, y, **kw):
    """Reference Tape SGD step (unmodified headers); updates W/b in place."""
    return _train_step(ref().ref_mlp_train_step, dims, W, b, X, y, **kw)


def _forward(fn, dims, W, b, X, head=0):
    L = len(dims) - 1
    B = X.shape[0]
    X = np.ascontiguousarray(X, dtype=np.float64)
    logits = np.empty((B, dims[-1]))
    hid = np.empty((B, dims[-2])) if L > 1 else None
    dimsc = (C.c_int * (L + 1))(*dims)
    st = fn(L, dimsc, head, _ptrs(W), _ptrs(b), dp(X), B, dp(logits), dp(hid))
    if st != 0:
        raise RuntimeError(f"forward failed with status {st}")
    return logits, hid


def mlp_forward(dims, W, b, X, head=0):
    return _forward(orc().orc_mlp_forward, dims, W, b, X, head)


def ref_mlp_forward(dims, W, b, X, head=0):
    return _forward(ref().ref_mlp_forward, dims, W, b, X, head)


# ---------------------------------------------------------------- MMD
MMD_MULT = np.array([0.25, 0.5, 1.0, 2.0, 4.0])


def mmd_gaussian(Xs, Xt, mult=MMD_MULT, beta=0.0, grads=True):
    Xs = np.ascontiguousarray(Xs, dtype=np.float64)
    Xt = np.ascontiguousarray(Xt, dtype=np.float64)
    mult = np.ascontiguousarray(mult, dtype=np.float64)
    m, d = Xs.shape
    n = Xt.shape[0]
    v = C.c_double()
    bo = C.c_double()
    gs = np.zeros_like(Xs) if grads else None
    gt = np.zeros_like(Xt) if grads else None
    st = orc().orc_mmd_gaussian(dp(Xs), m, dp(Xt), n, d, dp(mult), len(mult), beta, C.byref(v),
                                C.byref(bo), dp(gs), dp(gt))
    if st != 0:
        raise RuntimeError(f"mmd failed with status {st}")
    return v.value, bo.value, gs, gt


def mmd_beta(Xs, Xt):
    Xs = np.ascontiguousarray(Xs, dtype=np.float64)
    Xt = np.ascontiguousarray(Xt, dtype=np.float64)
    return orc().orc_mmd_beta(dp(Xs), Xs.shape[0], dp(Xt), Xt.shape[0], Xs.shape[1])


# ---------------------------------------------------------------- attack stage
def softmax(logits):
    logits = np.ascontiguousarray(logits, dtype=np.float64)
    out = np.empty_like(logits)
    orc().orc_softmax(dp(logits), logits.shape[0], logits.shape[1], dp(out))
    return out


def posterior_features(logits, k=3, labels=None):
    logits = np.ascontiguousarray(logits, dtype=np.float64)
    rows, Cn = logits.shape
    nf = k + (1 if labels is not None else 0)
    out = np.empty((rows, nf))
    lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
    st = orc().orc_posterior_features(dp(logits), rows, Cn, k,
                                      None if lab is None else lab.ctypes.data_as(_i32p), dp(out))
    if st != 0:
        raise RuntimeError(f"features failed with status {st}")
    return out


def auc(scores, labels):
    s = np.ascontiguousarray(scores, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint8)
    out = C.c_double()
    st = orc().orc_auc(dp(s), lab.ctypes.data_as(_u8p), len(s), C.byref(out))
    if st != 0:
        raise RuntimeError(f"auc failed with status {st}")
    return out.value


def accuracy(scores, labels, threshold=0.5):
    s = np.ascontiguousarray(scores, dtype=np.float64)
    lab = np.ascontiguousarray(labels, dtype=np.uint8)
    return orc().orc_accuracy(dp(s), lab.ctypes.data_as(_u8p), len(s), threshold)


def synth(rng: Rng, C_, d, n, mu, shift=None):
    X = np.empty((n, d))
    y = np.empty(n, dtype=np.int32)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    sh = None if shift is None else np.ascontiguousarray(shift, dtype=np.float64)
    orc().orc_synth(rng._buf, C_, d, n, dp(mu), dp(sh), dp(X), y.ctypes.data_as(_i32p))
    return X, y


def philox4x64(ctr, key):
    """Philox4x64-10 bijection (oracle.h): 4 counter words, 2 key words -> 4 words."""
    c = (C.c_uint64 * 4)(*[int(x) & (2**64 - 1) for x in ctr])
    k = (C.c_uint64 * 2)(*[int(x) & (2**64 - 1) for x in key])
    o = (C.c_uint64 * 4)()
    orc().orc_philox4x64(c, k, o)
    return [int(x) for x in o]


def counter_normals(seed, stream, first, count):
    z = np.empty(count)
    orc().orc_counter_normals(seed, stream, first, count, dp(z))
    return z


def synth_counter(seed, stream, C_, d, n, mu, shift=None):
    """Counter-based class-conditional Gaussians (oracle.h); f64 X, int32 y."""
    X = np.empty((n, d))
    y = np.empty(n, dtype=np.int32)
    mu = np.ascontiguousarray(mu, dtype=np.float64)
    sh = None if shift is None else np.ascontiguousarray(shift, dtype=np.float64)
    orc().orc_synth_counter(seed, stream, C_, d, n, dp(mu), dp(sh), dp(X), y.ctypes.data_as(_i32p))
    return X, y
