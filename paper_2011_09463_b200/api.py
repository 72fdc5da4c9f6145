"""Python host mirror of the reference interface for the shadow-training path.

Names and argument meaning follow the reference's C++ API where one exists
(``mt::Rng`` rng.hpp, the Tape ops composed by ``Bank.train_step``, SGD
``optimizer_step`` optim.hpp) and SURVEY.md section 8(b) for the entry points
the reference lacks (MMD, posterior features, AUC).  Every call goes through
libmtk.so (CUDA, sm_100a) via the C ABI; torch only provides device memory
and the stream.  Errors raise the classes in ``errors`` (error.hpp:10-51).
"""
from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np
import torch

from . import errors
from ._lib import MtkStep, MtkSweepConfig, MtkSweepResult, lib

_dp = C.POINTER(C.c_double)

MMD_MULT = (0.25, 0.5, 1.0, 2.0, 4.0)


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        if not t.is_contiguous():
            raise errors.ShapeError("tensor must be contiguous")
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(int(t))


def _need(t, name: str, dtype, shape=None, cuda=True, optional=False):
    """Argument check before a C call: a wrong dtype / device / shape would
    otherwise be read with the C side's element size and bounds (e.g. int32
    indices read as int64 run past the buffer)."""
    if t is None:
        if optional:
            return
        raise errors.ValueError(f"{name}: required")
    if not isinstance(t, torch.Tensor):
        raise errors.ValueError(f"{name}: expected a torch.Tensor, got {type(t).__name__}")
    if t.dtype != dtype:
        raise errors.ValueError(f"{name}: expected {dtype}, got {t.dtype}")
    if cuda and t.device.type != "cuda":
        raise errors.ValueError(f"{name}: expected a CUDA tensor, got {t.device}")
    if not cuda and t.device.type != "cpu":
        raise errors.ValueError(f"{name}: expected a host tensor, got {t.device}")
    if not t.is_contiguous():
        raise errors.ShapeError(f"{name}: tensor must be contiguous")
    if shape is not None:
        if t.dim() != len(shape) or any(s is not None and a != s for a, s in zip(t.shape, shape)):
            want = "[" + ", ".join("*" if s is None else str(s) for s in shape) + "]"
            raise errors.ShapeError(f"{name}: expected shape {want}, got {list(t.shape)}")


def _dvec(a):
    return (_dp * len(a))(*[x.ctypes.data_as(_dp) if x is not None else None for x in a])


class _CudaArray:
    def __init__(self, ptr, shape):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4",
                                         "data": (int(ptr), False), "version": 3}


def _device_view(ptr, shape, device):
    return torch.as_tensor(_CudaArray(ptr, shape), device=device)


class Context:
    """One per (thread, device); stream-ordered on torch's current stream."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None):
        self.device = device
        torch.cuda.set_device(device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        h = C.c_void_p()
        errors.check(lib.mtk_ctx_create(device, C.c_void_p(self.stream.cuda_stream), C.byref(h)),
                     "mtk_ctx_create")
        self.h = h

    def synchronize(self):
        errors.check(lib.mtk_ctx_synchronize(self.h), "synchronize")

    @property
    def launches(self) -> int:
        v = C.c_uint64()
        errors.check(lib.mtk_ctx_launch_count(self.h, C.byref(v)))
        return v.value

    # side_stream: wall time of the side-stream groups (MMD prep, bias updates,
    # head dW); they overlap the main-stream phases
    PHASES = ("fwd_gemm", "ce", "mmd_beta", "mmd_pairs", "dx_gemm", "dw_gemm", "bias_sgd", "other",
              "side_stream")

    def set_timing(self, on: bool = True):
        errors.check(lib.mtk_ctx_set_timing(self.h, 1 if on else 0))

    def phase_times(self):
        """{phase: (ms summed, launches)} since the last call (synchronizes)."""
        ms = np.zeros(len(self.PHASES))
        n = np.zeros(len(self.PHASES), dtype=np.uint64)
        errors.check(lib.mtk_ctx_phase_times(self.h, ms.ctypes.data_as(_dp),
                                             n.ctypes.data_as(C.POINTER(C.c_uint64))))
        return {p: (float(ms[i]), int(n[i])) for i, p in enumerate(self.PHASES)}

    def close(self):
        if getattr(self, "h", None):
            lib.mtk_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Rng:
    """mt::Rng (rng.hpp:13-75), host-side and bit-exact."""

    def __init__(self, seed: int | None = None, _h=None):
        if _h is not None:
            self.h = _h
        else:
            h = C.c_void_p()
            errors.check(lib.mtk_rng_create(C.c_uint64(seed & (2**64 - 1)), C.byref(h)))
            self.h = h

    def __del__(self):
        try:
            lib.mtk_rng_destroy(self.h)
        except Exception:
            pass

    def next_u64(self) -> int:
        return lib.mtk_rng_next_u64(self.h)

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        return lib.mtk_rng_uniform(self.h, lo, hi)

    def normal(self) -> float:
        return lib.mtk_rng_normal(self.h)

    def below(self, n: int) -> int:
        return lib.mtk_rng_below(self.h, n)

    def permutation(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.uint64)
        errors.check(lib.mtk_rng_permutation(self.h, n, out.ctypes.data_as(C.POINTER(C.c_uint64))))
        return out

    def split(self, stream: int) -> "Rng":
        h = C.c_void_p()
        errors.check(lib.mtk_rng_split(self.h, stream, C.byref(h)))
        return Rng(_h=h)

    def normals(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        errors.check(lib.mtk_rng_fill_normal(self.h, out.ctypes.data_as(_dp), n))
        return out

    def synth(self, n_classes: int, d: int, n: int, mu: np.ndarray, shift=None, f64=False):
        """Class-conditional Gaussians; returns (X float32 [n,d], y int32 [n]) (+X f64)."""
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        X32 = np.empty((n, d), dtype=np.float32)
        X64 = np.empty((n, d), dtype=np.float64) if f64 else None
        y = np.empty(n, dtype=np.int32)
        sh = None if shift is None else np.ascontiguousarray(shift, dtype=np.float64)
        errors.check(lib.mtk_synth(self.h, n_classes, d, n, mu.ctypes.data_as(_dp),
                                   None if sh is None else sh.ctypes.data_as(_dp),
                                   None if X64 is None else X64.ctypes.data_as(_dp),
                                   C.c_void_p(X32.ctypes.data), C.c_void_p(y.ctypes.data)),
                     "synth")
        return (X32, y, X64) if f64 else (X32, y)


class Bank:
    """G independent MLPs trained as one grouped step (see mtk_bank_* in mtk.h)."""

    def __init__(self, ctx: Context, G: int, dims: Sequence[int], n_heads: int = 1):
        self.ctx, self.G, self.dims, self.n_heads = ctx, G, list(dims), n_heads
        self.L = len(dims) - 1
        self.n_mats = self.L + n_heads - 1
        h = C.c_void_p()
        d = (C.c_int * len(dims))(*dims)
        errors.check(lib.mtk_bank_create(ctx.h, G, self.L, d, n_heads, C.byref(h)),
                     "mtk_bank_create")
        self.h = h
        self._loss = np.zeros(G)
        self._mmd = np.zeros(G)

    @classmethod
    def load(cls, ctx: Context, path: str) -> "Bank":
        """A bank restored from a checkpoint written by save() (bit-exact)."""
        h = C.c_void_p()
        errors.check(lib.mtk_bank_load(ctx.h, str(path).encode(), C.byref(h)), "load")
        G, L, heads = C.c_int(), C.c_int(), C.c_int()
        errors.check(lib.mtk_bank_info(h, C.byref(G), C.byref(L), None, C.byref(heads)))
        dims = (C.c_int * (L.value + 1))()
        errors.check(lib.mtk_bank_info(h, None, None, dims, None))
        self = cls.__new__(cls)
        self.ctx, self.G, self.dims, self.n_heads = ctx, G.value, list(dims), heads.value
        self.L = L.value
        self.n_mats = self.L + self.n_heads - 1
        self.h = h
        self._loss = np.zeros(self.G)
        self._mmd = np.zeros(self.G)
        return self

    def save(self, path: str):
        """Checkpoint parameters (and Adam state) to `path`."""
        errors.check(lib.mtk_bank_save(self.h, str(path).encode()), "save")

    def __del__(self):
        try:
            lib.mtk_bank_destroy(self.h)
        except Exception:
            pass

    def shapes(self):
        out = []
        for i in range(self.n_mats):
            l = i if i < self.L else self.L - 1
            out.append((self.dims[l], self.dims[l + 1]))
        return out

    def set_params(self, model: int, W, b):
        W = [np.ascontiguousarray(x, dtype=np.float64) for x in W]
        b = [np.ascontiguousarray(x, dtype=np.float64) for x in b]
        errors.check(lib.mtk_bank_set_params(self.h, model, _dvec(W), _dvec(b)), "set_params")

    def get_params(self, model: int):
        W = [np.empty(s) for s in self.shapes()]
        b = [np.empty(s[1]) for s in self.shapes()]
        errors.check(lib.mtk_bank_get_params(self.h, model, _dvec(W), _dvec(b)), "get_params")
        return W, b

    def init_params(self, model: int, rng: Rng):
        errors.check(lib.mtk_bank_init_params(self.h, model, rng.h), "init_params")

    def param_device(self, mat: int):
        w, b = C.c_void_p(), C.c_void_p()
        errors.check(lib.mtk_bank_param_device(self.h, mat, C.byref(w), C.byref(b)))
        return w.value, b.value

    def param_tensors(self):
        """zero-copy torch views [W_0, b_0, W_1, b_1, ...] of the device
        parameters (W_i [G, fan_in, fan_out], b_i [G, fan_out]); used to
        broadcast a replica's initial parameters (dp.DataParallel)."""
        dev = torch.device("cuda", self.ctx.device)
        out = []
        for i, (fi, fo) in enumerate(self.shapes()):
            w, b = self.param_device(i)
            out.append(_device_view(w, (self.G, fi, fo), dev))
            out.append(_device_view(b, (self.G, fo), dev))
        return out

    def forward(self, X: torch.Tensor, head: int = 0, hidden: bool = False):
        _need(X, "forward: X", torch.float32, (self.G, None, self.dims[0]))
        B = X.shape[1]
        logits = torch.empty((self.G, B, self.dims[-1]), device=X.device, dtype=torch.float32)
        hid = (torch.empty((self.G, B, self.dims[-2]), device=X.device, dtype=torch.float32)
               if hidden and self.L > 1 else None)
        errors.check(lib.mtk_bank_forward(self.h, _ptr(X), B, head, _ptr(logits), _ptr(hid)),
                     "forward")
        return (logits, hid) if hidden else logits

    @staticmethod
    def make_step(B, *, src_rows=0, denom=(0.0, 0.0), lr=0.05, frozen_layers=0, mmd_lambda=0.0,
                  mmd_mult=None, optimizer="sgd", adam_betas=(0.0, 0.0), adam_eps=0.0,
                  X=None, y=None, w=None) -> MtkStep:
        """optimizer: "sgd" (optim.hpp:46-48) or "adam" (optim.hpp:49-63; the
        bank keeps the moments, see reset_optimizer).  Zero betas / eps select
        the reference defaults 0.9 / 0.999 / 1e-8."""
        s = MtkStep()
        s.X, s.y, s.w = _ptr(X), _ptr(y), _ptr(w)
        s.B = B
        s.src_rows = src_rows
        s.denom[0], s.denom[1] = denom
        s.lr = lr
        if optimizer not in ("sgd", "adam"):
            raise errors.ConfigError(f"unknown optimizer {optimizer!r}")
        s.optimizer = 1 if optimizer == "adam" else 0
        s.adam_beta1, s.adam_beta2 = adam_betas
        s.adam_eps = adam_eps
        s.frozen_layers = frozen_layers
        s.mmd_lambda = mmd_lambda
        if mmd_mult is not None:
            s.mmd_nb = len(mmd_mult)
            for i, v in enumerate(mmd_mult):
                s.mmd_mult[i] = v
        return s

    def train_step(self, X, y, w=None, *, want_loss=True, **kw):
        """One SGD step of all G models; returns (loss[G], mmd[G]) or None."""
        self._check_batch("train_step", X, y, w)
        B = X.shape[1]
        s = self.make_step(B, X=X, y=y, w=w, **kw)
        lp = self._loss.ctypes.data_as(_dp) if want_loss else None
        mp = self._mmd.ctypes.data_as(_dp) if want_loss else None
        errors.check(lib.mtk_bank_train_step(self.h, C.byref(s), lp, mp), "train_step")
        return (self._loss.copy(), self._mmd.copy()) if want_loss else None

    def _check_batch(self, what, X, y, w, cuda=True):
        _need(X, f"{what}: X", torch.float32, (self.G, None, self.dims[0]), cuda=cuda)
        B = X.shape[1]
        _need(y, f"{what}: y", torch.int32, (self.G, B), cuda=cuda)
        _need(w, f"{what}: w", torch.float32, (self.G, B), cuda=cuda, optional=True)

    def train_step_host(self, X_host, y_host, w_host=None, *, want_loss=True, **kw):
        """Same step from host (ideally pinned) buffers; copies inside the call."""
        self._check_batch("train_step_host", X_host, y_host, w_host, cuda=False)
        B = X_host.shape[1]
        s = self.make_step(B, **kw)
        lp = self._loss.ctypes.data_as(_dp) if want_loss else None
        mp = self._mmd.ctypes.data_as(_dp) if want_loss else None
        errors.check(lib.mtk_bank_train_step_host(self.h, C.byref(s), _ptr(X_host), _ptr(y_host),
                                                  _ptr(w_host), lp, mp), "train_step_host")
        return (self._loss.copy(), self._mmd.copy()) if want_loss else None

    def tc_layers(self):
        """per layer: True if its GEMMs run on the tcgen05 3xTF32 path"""
        out = (C.c_int * self.L)()
        errors.check(lib.mtk_bank_tc_layers(self.h, out))
        return [bool(x) for x in out]

    def train_step_host_async(self, X_host, y_host, w_host=None, **kw):
        """Enqueue a step from pinned host buffers (copy overlaps the previous
        step's compute); collect results with step_result()."""
        self._check_batch("train_step_host_async", X_host, y_host, w_host, cuda=False)
        B = X_host.shape[1]
        s = self.make_step(B, **kw)
        errors.check(lib.mtk_bank_train_step_host_async(self.h, C.byref(s), _ptr(X_host),
                                                        _ptr(y_host), _ptr(w_host)),
                     "train_step_host_async")

    def step_result(self, which: int = 0):
        """(loss[G], mmd[G]) of the last (which=0) or previous (1) async step."""
        errors.check(lib.mtk_bank_step_result(self.h, which, self._loss.ctypes.data_as(_dp),
                                              self._mmd.ctypes.data_as(_dp)), "step_result")
        return self._loss.copy(), self._mmd.copy()

    def train_epoch(self, X_pool, y_pool, idx, w=None, denom0=None, **kw):
        """idx.shape[0] steps, each gathering X_pool[idx[s]] / y_pool[idx[s]] on
        the device (idx int64 [steps, G, B]); w [steps, G, B] or None; denom0
        per-step head-0 denominators (host) or None (kw's denom)."""
        _need(idx, "train_epoch: idx", torch.int64, (None, self.G, None))
        steps, G, B = idx.shape
        _need(X_pool, "train_epoch: X_pool", torch.float32, (None, self.dims[0]))
        _need(y_pool, "train_epoch: y_pool", torch.int32, (X_pool.shape[0],))
        _need(w, "train_epoch: w", torch.float32, (steps, G, B), optional=True)
        s = self.make_step(B, **kw)
        dn = None
        if denom0 is not None:
            dn = np.ascontiguousarray(denom0, dtype=np.float64)
            if dn.shape != (steps,):
                raise errors.ShapeError("train_epoch: denom0 needs one value per step")
        errors.check(lib.mtk_bank_train_epoch(self.h, C.byref(s), _ptr(X_pool), _ptr(y_pool),
                                              X_pool.shape[0], _ptr(idx), _ptr(w),
                                              dn.ctypes.data_as(_dp) if dn is not None else None,
                                              steps), "train_epoch")

    def reset_optimizer(self):
        """zero the Adam moments and step count (a fresh OptimizerState)"""
        errors.check(lib.mtk_bank_reset_optimizer(self.h), "reset_optimizer")

    # ---- data-parallel replicas (dp_step; see dp.py) ----
    def grad_size(self) -> int:
        """floats in the gradient arena (per matrix: dW [G,fi,fo] then db [G,fo])"""
        n = C.c_int64()
        errors.check(lib.mtk_bank_grad_size(self.h, C.byref(n)), "grad_size")
        return n.value

    def compute_grads(self, X, y, w=None, out: torch.Tensor = None, *, want_loss=True, **kw):
        """Forward + backward of this shard into a device gradient arena
        (parameters and optimizer state unchanged); returns (arena, loss, mmd)."""
        self._check_batch("compute_grads", X, y, w)
        n = self.grad_size()
        if out is None:
            out = torch.empty(n, dtype=torch.float32, device=X.device)
        if out.dtype != torch.float32 or not out.is_contiguous() or out.numel() < n:
            raise errors.ShapeError(f"compute_grads: out must be contiguous fp32 with >= {n} floats")
        s = self.make_step(X.shape[1], X=X, y=y, w=w, **kw)
        lp = self._loss.ctypes.data_as(_dp) if want_loss else None
        mp = self._mmd.ctypes.data_as(_dp) if want_loss else None
        errors.check(lib.mtk_bank_compute_grads(self.h, C.byref(s), _ptr(out), lp, mp),
                     "compute_grads")
        return out, (self._loss.copy() if want_loss else None), (self._mmd.copy() if want_loss else None)

    def dp_apply(self, parts: torch.Tensor, **kw):
        """parts [n_workers, >= grad_size] fp32 device: g = ordered mean over
        workers (ascending), then one optimizer step (make_step options)."""
        if parts.dim() != 2 or parts.dtype != torch.float32 or parts.stride(1) != 1:
            raise errors.ShapeError("dp_apply: parts must be [n_workers, arena] fp32, row-contiguous")
        if parts.shape[1] < self.grad_size():
            raise errors.ShapeError("dp_apply: parts rows are shorter than the gradient arena")
        s = self.make_step(1, **kw)
        errors.check(lib.mtk_bank_dp_apply(self.h, C.byref(s), _ptr(parts), parts.shape[0],
                                           parts.stride(0)), "dp_apply")

    def fingerprint(self) -> int:
        """order-independent 64-bit hash of all parameter bits"""
        v = C.c_uint64()
        errors.check(lib.mtk_bank_fingerprint(self.h, C.byref(v)), "fingerprint")
        return v.value

    def keep_grads(self, on: bool = True):
        errors.check(lib.mtk_bank_set_keep_grads(self.h, 1 if on else 0))

    def get_grads(self, model: int):
        W = [np.empty(s) for s in self.shapes()]
        b = [np.empty(s[1]) for s in self.shapes()]
        errors.check(lib.mtk_bank_get_grads(self.h, model, _dvec(W), _dvec(b)), "get_grads")
        return W, b


def _mult_arr(mult):
    mult = MMD_MULT if mult is None else mult
    return np.ascontiguousarray(mult, dtype=np.float64)


def mmd_gaussian(ctx: Context, Xs: torch.Tensor, Xt: torch.Tensor, mult=None, beta: float = 0.0,
                 grads: bool = True):
    """Multi-bandwidth Gaussian MMD^2 (biased V-statistic) and d/dX (device)."""
    m, d = Xs.shape
    n = Xt.shape[0]
    mu = _mult_arr(mult)
    v, bo = C.c_double(), C.c_double()
    gs = gt = None
    if grads:  # one [m + n, d] block: with Xs, Xt views of one block too, the
        # library can take its materialised-kernel-matrix path
        g = torch.empty((m + n, d), dtype=Xs.dtype, device=Xs.device)
        gs, gt = g[:m], g[m:]
    errors.check(lib.mtk_mmd_gaussian(ctx.h, _ptr(Xs), m, _ptr(Xt), n, d, mu.ctypes.data_as(_dp),
                                      len(mu), beta, C.byref(v), C.byref(bo), _ptr(gs), _ptr(gt)),
                 "mmd_gaussian")
    return v.value, bo.value, gs, gt


def mmd_gaussian_rows(ctx: Context, Xs, Xt, beta: float, row_begin: int, row_end: int, mult=None,
                      gXs=None, gXt=None):
    """Row-sharded MMD: raw kernel sums (ss, tt, st) over pair rows [begin, end)."""
    m, d = Xs.shape
    n = Xt.shape[0]
    mu = _mult_arr(mult)
    part = np.zeros(3)
    errors.check(lib.mtk_mmd_gaussian_rows(ctx.h, _ptr(Xs), m, _ptr(Xt), n, d,
                                           mu.ctypes.data_as(_dp), len(mu), beta, row_begin,
                                           row_end, part.ctypes.data_as(_dp), _ptr(gXs),
                                           _ptr(gXt)), "mmd_gaussian_rows")
    return part


MMD_TILE = 128


def mmd_tile_ranges(m: int, n: int, world: int):
    """Equal 128-row tile ranges over [Xs; Xt], one per rank: with the
    materialised-W sharding every rank then does s*T - s^2/2 tile pairs
    (mtk_mmd_gaussian_tiles), i.e. the same work."""
    T = -(-(m + n) // MMD_TILE)
    return [(r * T // world, (r + 1) * T // world) for r in range(world)]


def mmd_gaussian_tiles(ctx: Context, Z: torch.Tensor, m: int, beta: float, tile_begin: int, tile_end: int,
                       gZ: torch.Tensor, mult=None) -> np.ndarray:
    """This rank's share of the materialised-W MMD (mtk_mmd_gaussian_tiles):
    Z = [Xs; Xt] one [m + n, d] block, gZ its gradient block (rows of tiles
    [tile_begin, tile_end) written).  Returns the [T, 3] kernel-sum partials
    (zeros outside the range); combine the ranks' with mmd_value_from_tiles."""
    N, d = Z.shape
    n = N - m
    mu = _mult_arr(mult)
    T = -(-N // MMD_TILE)
    part = np.zeros((T, 3))
    errors.check(lib.mtk_mmd_gaussian_tiles(ctx.h, _ptr(Z), m, C.c_void_p(Z.data_ptr() + m * d * 4), n, d,
                                            mu.ctypes.data_as(_dp), len(mu), beta, tile_begin, tile_end,
                                            part.ctypes.data_as(_dp), _ptr(gZ),
                                            C.c_void_p(gZ.data_ptr() + m * d * 4)), "mmd_gaussian_tiles")
    return part


def mmd_value_from_tiles(partials: np.ndarray, m: int, n: int) -> float:
    """MMD^2 from [T, 3] tile-row kernel sums (the ranks' partials added
    elementwise: each tile row has one owner), in the one-rank finish order"""
    p = np.ascontiguousarray(partials, dtype=np.float64)
    v = C.c_double()
    errors.check(lib.mtk_mmd_value_from_tile_partials(p.ctypes.data_as(_dp), p.shape[0], m, n, C.byref(v)),
                 "mmd_value_from_tile_partials")
    return v.value


def mmd_beta(ctx: Context, Xs, Xt) -> float:
    m, d = Xs.shape
    out = C.c_double()
    errors.check(lib.mtk_mmd_beta(ctx.h, _ptr(Xs), m, _ptr(Xt), Xt.shape[0], d, C.byref(out)))
    return out.value


def mmd_value_from_sums(sums, m: int, n: int) -> float:
    ss, tt, st = sums
    return ss / (m * m) + tt / (n * n) - 2.0 * st / (m * n)


def sha256(data: bytes) -> bytes:
    """FIPS 180-4 SHA-256 (the checkpoint digest)."""
    out = (C.c_uint8 * 32)()
    buf = C.create_string_buffer(bytes(data), len(data))
    errors.check(lib.mtk_sha256(buf, len(data), out))
    return bytes(out)


def gather_rows(ctx: Context, src: torch.Tensor, idx: torch.Tensor, out: torch.Tensor = None,
                row0: int = 0) -> torch.Tensor:
    """out[g, row0 + r] = src[idx[g, r]] on the device (batch assembly).
    src [rows, d] (float32 or int32), idx int64 [G, nb]; out [G, out_rows, d]
    (allocated [G, nb, d] when None)."""
    if not isinstance(src, torch.Tensor) or src.dtype not in (torch.float32, torch.int32):
        raise errors.ValueError("gather_rows: src must be a float32 or int32 tensor")
    _need(src, "gather_rows: src", src.dtype)
    _need(idx, "gather_rows: idx", torch.int64, (None, None))
    src2 = src.reshape(src.shape[0], -1)
    G, nb = idx.shape
    d = src2.shape[1]
    if out is None:
        out = torch.empty((G, nb) + tuple(src.shape[1:]), device=src.device, dtype=src.dtype)
    _need(out, "gather_rows: out", src.dtype)
    if out.dim() < 2 or out.shape[0] != G or row0 < 0 or row0 + nb > out.shape[1] or \
            out[0, 0].numel() != d:
        raise errors.ShapeError(f"gather_rows: out must be [{G}, >= row0 + {nb}, {d}]")
    errors.check(lib.mtk_gather_rows(ctx.h, _ptr(src2), src2.shape[0], d, _ptr(idx), G, nb,
                                     _ptr(out), out.shape[1], row0), "gather_rows")
    return out


# ---- counter-based synthetic data on the device (mtk.h) ----
_U64 = 2**64 - 1


def philox4x64_fill(ctx: Context, seed: int, stream: int, nblocks: int, ctr0: int = 0,
                    ctr1: int = 0) -> torch.Tensor:
    """raw Philox4x64-10 words: out[i] = philox({ctr0 + i, ctr1, 0, 0}, {seed, stream}),
    as an int64 tensor [nblocks, 4] (bit pattern of the uint64 words)."""
    out = torch.empty((nblocks, 4), dtype=torch.int64, device=torch.device("cuda", ctx.device))
    errors.check(lib.mtk_philox4x64_fill(ctx.h, seed & _U64, stream & _U64, ctr0 & _U64,
                                         ctr1 & _U64, nblocks, _ptr(out)), "philox4x64_fill")
    return out


def counter_normals(ctx: Context, seed: int, stream: int, first: int, count: int) -> torch.Tensor:
    out = torch.empty(count, dtype=torch.float32, device=torch.device("cuda", ctx.device))
    errors.check(lib.mtk_counter_normals(ctx.h, seed & _U64, stream & _U64, first, count,
                                         _ptr(out)), "counter_normals")
    return out


def synth_counter(ctx: Context, seed: int, stream: int, n: int, mu: torch.Tensor,
                  shift: torch.Tensor = None):
    """X [n, d] fp32, y [n] int32 on the device: y from the label counter
    space, X = mu[y] + N(0, I) (+ shift) (mtk_synth_counter)."""
    C, d = mu.shape
    dev = torch.device("cuda", ctx.device)
    mu = mu.to(dev, torch.float32).contiguous()
    sh = None if shift is None else shift.to(dev, torch.float32).contiguous()
    X = torch.empty((n, d), dtype=torch.float32, device=dev)
    y = torch.empty(n, dtype=torch.int32, device=dev)
    errors.check(lib.mtk_synth_counter(ctx.h, seed & _U64, stream & _U64, C, d, n, _ptr(mu),
                                       _ptr(sh), _ptr(X), _ptr(y)), "synth_counter")
    return X, y


def softmax(ctx: Context, logits: torch.Tensor) -> torch.Tensor:
    logits2 = logits.reshape(-1, logits.shape[-1])
    out = torch.empty_like(logits2)
    errors.check(lib.mtk_softmax(ctx.h, _ptr(logits2), logits2.shape[0], logits2.shape[1],
                                 _ptr(out)), "softmax")
    return out.reshape(logits.shape)


def posterior_features(ctx: Context, logits: torch.Tensor, k: int = 3, labels=None):
    logits2 = logits.reshape(-1, logits.shape[-1])
    rows, Cn = logits2.shape
    nf = k + (1 if labels is not None else 0)
    out = torch.empty((rows, nf), device=logits.device, dtype=torch.float32)
    lab = None if labels is None else labels.reshape(-1)
    errors.check(lib.mtk_posterior_features(ctx.h, _ptr(logits2), rows, Cn, k, _ptr(lab),
                                            _ptr(out)), "posterior_features")
    return out


def posterior_column(ctx: Context, logits: torch.Tensor, col: int = 1):
    logits2 = logits.reshape(-1, logits.shape[-1])
    out = torch.empty(logits2.shape[0], device=logits.device, dtype=torch.float32)
    errors.check(lib.mtk_posterior_column(ctx.h, _ptr(logits2), logits2.shape[0],
                                          logits2.shape[1], col, _ptr(out)), "posterior_column")
    return out


def auc(ctx: Context, scores: torch.Tensor, labels: torch.Tensor):
    """(AUC with mid-ranks, accuracy at 0.5); labels uint8, 1 = member."""
    a, acc = C.c_double(), C.c_double()
    errors.check(lib.mtk_auc(ctx.h, _ptr(scores), _ptr(labels), scores.numel(), C.byref(a),
                             C.byref(acc)), "auc")
    return a.value, acc.value


def attack_auc(attack: "Bank", logits: torch.Tensor, labels: torch.Tensor, scores: bool = False):
    """The attack stage in one call: posteriors -> top-k features -> attack
    model (model 0 of `attack`) -> member probability -> (AUC, accuracy[, scores]).
    Same results as posterior_features + Bank.forward + posterior_column + auc."""
    logits2 = logits.reshape(-1, logits.shape[-1])
    a, acc = C.c_double(), C.c_double()
    out = torch.empty(logits2.shape[0], device=logits.device, dtype=torch.float32) if scores else None
    errors.check(lib.mtk_attack_auc(attack.h, _ptr(logits2), logits2.shape[0], logits2.shape[1],
                                    _ptr(labels), C.byref(a), C.byref(acc), _ptr(out)), "attack_auc")
    return (a.value, acc.value, out) if scores else (a.value, acc.value)


def diag_gemm_tf32x3(ctx: Context, A: torch.Tensor, B: torch.Tensor, a_mn: bool, b_mn: bool):
    """Diagnostics: C = A @ B on the tcgen05 3xTF32 path.  A is [G,M,K] (or
    [G,K,M] if a_mn), B is [G,K,N] (or [G,N,K] if not b_mn); returns [G,M,N]."""
    G = A.shape[0]
    M, K = (A.shape[2], A.shape[1]) if a_mn else (A.shape[1], A.shape[2])
    N = B.shape[2] if b_mn else B.shape[1]
    C_ = torch.empty((G, M, N), device=A.device, dtype=torch.float32)
    errors.check(lib.mtk_diag_gemm_tf32x3(ctx.h, int(a_mn), int(b_mn), G, M, N, K, _ptr(A),
                                          _ptr(B), _ptr(C_)), "diag_gemm_tf32x3")
    return C_


class Comm:
    """NCCL communicator for the path's one collective, the feature all-gather
    (mtk_comm_* / mtk_allgather).  The 128-byte NCCL id
    is created on rank 0 and broadcast over the given torch.distributed group
    (any backend); with no process group, a one-rank communicator."""

    def __init__(self, ctx: Context, group=None):
        import torch.distributed as dist

        self.ctx = ctx
        if dist.is_available() and dist.is_initialized():
            self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        else:
            self.rank, self.world = 0, 1
        uid = (C.c_uint8 * 128)()
        if self.rank == 0:
            errors.check(lib.mtk_comm_unique_id(uid), "comm_unique_id")
        if self.world > 1:
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                       group=group)
            uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        torch.cuda.set_device(ctx.device)
        h = C.c_void_p()
        errors.check(lib.mtk_comm_init(self.world, self.rank, uid, C.byref(h)), "comm_init")
        self.h = h

    def nccl_version(self) -> int:
        v = C.c_int()
        errors.check(lib.mtk_comm_info(self.h, None, None, None, C.byref(v)), "comm_info")
        return v.value

    def all_gather(self, t: torch.Tensor, out: torch.Tensor = None) -> torch.Tensor:
        """[world, *t.shape]: rank r's tensor at index r (stream-ordered on the ctx)."""
        if t.device.type != "cuda" or not t.is_contiguous():
            raise errors.ValueError("all_gather: a contiguous CUDA tensor is required")
        if out is None:
            out = torch.empty((self.world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        if out.numel() != self.world * t.numel() or out.dtype != t.dtype or not out.is_contiguous():
            raise errors.ShapeError("all_gather: out must hold world x the input")
        errors.check(lib.mtk_allgather(self.h, self.ctx.h, _ptr(t), _ptr(out),
                                       t.numel() * t.element_size()), "allgather")
        return out

    def close(self):
        if getattr(self, "h", None):
            lib.mtk_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass


def sweep_run(ctx: Context, cfg: dict | None = None, comm: "Comm" = None) -> dict:
    """The whole sweep (one paradigm) through the native driver, mtk_sweep_run:
    cfg keys are SweepConfig's (paradigm "model" | "mapping" | "parameter",
    optimizer "sgd" | "adam", data_rng "host" | "counter", dims a tuple);
    unspecified keys keep the C1 defaults."""
    c = MtkSweepConfig()
    lib.mtk_sweep_config_default(C.byref(c))
    enum = {"paradigm": {"model": 0, "mapping": 1, "parameter": 2}, "optimizer": {"sgd": 0, "adam": 1},
            "attack_optimizer": {"sgd": 0, "adam": 1}, "data_rng": {"host": 0, "counter": 1}}
    for key, v in (cfg or {}).items():
        if key == "dims":
            if not 2 <= len(v) <= 9:
                raise errors.ConfigError("sweep: 1 to 8 layers")
            c.n_layers = len(v) - 1
            for i, x in enumerate(v):
                c.dims[i] = int(x)
        elif key in enum:
            if v not in enum[key]:
                raise errors.ConfigError(f"sweep: unknown {key} {v!r}")
            setattr(c, key, enum[key][v])
        elif hasattr(c, key):
            setattr(c, key, v)
        else:
            raise errors.ConfigError(f"sweep: unknown key {key!r}")
    r = MtkSweepResult()
    errors.check(lib.mtk_sweep_run(ctx.h, C.byref(c), comm.h if comm is not None else None, C.byref(r)),
                 "sweep_run")
    return {"auc": r.auc, "accuracy": r.accuracy, "models": r.models,
            "rank_models": list(range(r.rank_model_begin, r.rank_model_end)),
            "n_queries": r.n_queries, "seconds": r.seconds}
