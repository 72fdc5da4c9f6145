"""TEST INFRASTRUCTURE: the sweep driver's backend interface implemented on the
CPU oracle (oracle/oracle.c via pyoracle), one f64 model at a time.  Used to
replay paper_2011_09463_b200.sweep on the CPU and compare attack AUC /
accuracy with the GPU path (north_star: within +-0.01)."""
import numpy as np

import pyoracle as po


class OracleRng(po.Rng):
    def synth(self, C, d, n, mu, shift=None):
        X, y = po.synth(self, C, d, n, mu, shift)
        # the GPU path trains on the fp32 rounding of the same draws
        return X.astype(np.float32), y

    def split(self, stream):
        child = OracleRng(None)
        po.orc().orc_rng_split(self._buf, stream, child._buf)
        return child


class OracleBank:
    def __init__(self, G, dims, n_heads):
        self.G, self.dims, self.n_heads = G, list(dims), n_heads
        self.params = [None] * G
        self.adam = [None] * G  # po.Adam per model, created on the first Adam step


def _pmap(fn, n):
    """fn(g) for g < n on host threads (ctypes releases the GIL, so the oracle's
    C loops run in parallel; each model's arithmetic is unchanged)"""
    import os
    from concurrent.futures import ThreadPoolExecutor

    workers = min(n, len(os.sched_getaffinity(0)))
    if workers <= 1:
        return [fn(g) for g in range(n)]
    with ThreadPoolExecutor(workers) as ex:
        return list(ex.map(fn, range(n)))


class OracleBackend:
    Rng = OracleRng

    def bank(self, G, dims, n_heads=1):
        return OracleBank(G, dims, n_heads)

    def init(self, bank, g, rng):
        bank.params[g] = po.mlp_init(rng, bank.dims, bank.n_heads)

    def synth_counter(self, seed, stream, n, mu, shift):
        # the device generator's contract (oracle.c orc_synth_counter); the GPU
        # path builds its pools from fp32 mu / shift, so round them the same way
        mu32 = np.asarray(mu, dtype=np.float32).astype(np.float64)
        sh32 = None if shift is None else np.asarray(shift, dtype=np.float32).astype(np.float64)
        X, y = po.synth_counter(seed, stream, mu32.shape[0], mu32.shape[1], n, mu32, sh32)
        return X.astype(np.float32), y

    def step(self, bank, X, y, w, *, lr, src_rows=0, frozen_layers=0, mmd_lambda=0.0,
             denom=(0.0, 0.0), optimizer="sgd"):
        X = np.asarray(X, dtype=np.float64)
        _pmap(lambda g: self._step_one(bank, g, X, y, w, lr, src_rows, frozen_layers, mmd_lambda,
                                       denom, optimizer), bank.G)

    def _step_one(self, bank, g, X, y, w, lr, src_rows, frozen_layers, mmd_lambda, denom, optimizer):
        W, b = bank.params[g]
        dH = None
        if mmd_lambda > 0:
            _, H = po.mlp_forward(bank.dims, W, b, X[g])
            _, _, gs, gt = po.mmd_gaussian(H[:src_rows], H[src_rows:])
            dH = mmd_lambda * np.concatenate([gs, gt])
        B = X.shape[1]
        if bank.n_heads == 2:
            den = [denom[0] or src_rows, denom[1] or B - src_rows]
        else:
            den = [denom[0] or B]
        if optimizer == "sgd":
            po.mlp_train_step(bank.dims, W, b, X[g], y[g], n_heads=bank.n_heads,
                              frozen=frozen_layers, src_rows=src_rows, w=w[g], denoms=den,
                              lr=lr, dH=dH)
            return
        # Adam: gradients of the same Tape composition (lr = 0), then
        # optimizer_step over every parameter (frozen ones get zero grads,
        # which leaves them and their moments unchanged)
        _, gW, gb = po.mlp_train_step(bank.dims, W, b, X[g], y[g], n_heads=bank.n_heads,
                                      frozen=frozen_layers, src_rows=src_rows, w=w[g],
                                      denoms=den, lr=0.0, dH=dH, want_grads=True)
        if bank.adam[g] is None:
            bank.adam[g] = po.Adam(W + b, lr)
        bank.adam[g].update(W + b, gW + gb)

    def features(self, bank, X, head, k):
        def one(g):
            W, b = bank.params[g]
            logits, _ = po.mlp_forward(bank.dims, W, b, np.asarray(X[g], dtype=np.float64), head)
            return po.posterior_features(logits, k)

        return np.stack(_pmap(one, bank.G))

    def attack_scores(self, bank, F):
        W, b = bank.params[0]
        logits, _ = po.mlp_forward(bank.dims, W, b, np.asarray(F, dtype=np.float64))
        return po.softmax(logits)[:, 1]

    def auc(self, scores, labels):
        return po.auc(scores, labels), po.accuracy(scores, labels, 0.5)


class OracleReplica:
    """TEST INFRASTRUCTURE: one f64 oracle model behind the replica interface
    paper_2011_09463_b200.dp.DataParallel drives (G = 1, single head), so the
    dp_step plumbing (sharding, gather, ascending-order mean, replica check)
    runs over gloo on the CPU against single-process full-batch training."""

    import torch as _torch

    grad_dtype = _torch.float64
    device = _torch.device("cpu")

    def __init__(self, dims, W, b):
        self.dims = list(dims)
        self.W = [np.array(x, dtype=np.float64) for x in W]
        self.b = [np.array(x, dtype=np.float64) for x in b]
        self.adam = None

    def grad_size(self):
        return sum(w.size + b.size for w, b in zip(self.W, self.b))

    def compute_grads(self, X, y, w, out, denom, *, lr=0.0, optimizer="sgd", frozen_layers=0,
                      **_):
        X = np.asarray(X, dtype=np.float64)[0]
        y = np.asarray(y)[0]
        wv = None if w is None else np.asarray(w, dtype=np.float64)[0]
        loss, gW, gb = po.mlp_train_step(self.dims, self.W, self.b, X, y, frozen=frozen_layers,
                                         w=wv, denoms=[denom[0]], lr=0.0, want_grads=True)
        flat = np.concatenate([np.concatenate([a.ravel(), c.ravel()]) for a, c in zip(gW, gb)])
        out.copy_(self._torch.from_numpy(flat))
        return np.array([loss])

    def apply(self, parts, *, lr=0.05, optimizer="sgd", frozen_layers=0, **_):
        P = parts.numpy()
        acc = P[0].copy()
        for r in range(1, P.shape[0]):  # ascending worker order
            acc = acc + P[r]
        g = acc / P.shape[0]
        off = 0
        gW, gb = [], []
        for Wi, bi in zip(self.W, self.b):
            gW.append(g[off:off + Wi.size].reshape(Wi.shape))
            off += Wi.size
            gb.append(g[off:off + bi.size])
            off += bi.size
        L = len(self.dims) - 1
        if optimizer == "adam":
            if self.adam is None:
                self.adam = po.Adam(self.W + self.b, lr)
            self.adam.update(self.W + self.b, gW + gb)
            return
        for i in range(L):
            if i < frozen_layers:
                continue
            self.W[i] -= lr * gW[i]
            self.b[i] -= lr * gb[i]

    def fingerprint(self):
        import hashlib

        h = hashlib.sha256()
        for a in self.W + self.b:
            h.update(a.tobytes())
        return int.from_bytes(h.digest()[:8], "little")

    def param_tensors(self):
        out = []
        for Wi, bi in zip(self.W, self.b):
            out += [self._torch.from_numpy(Wi), self._torch.from_numpy(bi)]
        return out


class TorchFeatureOracleBackend(OracleBackend):
    """TEST INFRASTRUCTURE: the oracle's arithmetic, but the posterior features
    travel the way the GPU backend's do -- as tensors, combined across ranks
    by an EQUAL-size tensor all-gather (dist.all_gather over the default
    group: gloo in the CPU tests, NCCL / mtk_allgather on GPUs) -- so the
    sweep's padding / trimming / rank-order logic runs without a GPU."""

    def features(self, bank, X, head, k):
        import torch

        return torch.from_numpy(super().features(bank, X, head, k))

    def all_gather(self, F):
        import torch
        import torch.distributed as dist

        parts = [torch.empty_like(F) for _ in range(dist.get_world_size())]
        dist.all_gather(parts, F.contiguous())
        return parts

    def attack_scores(self, bank, F):
        return super().attack_scores(bank, np.asarray(F))
