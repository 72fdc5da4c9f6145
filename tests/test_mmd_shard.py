"""The multi-GPU MMD plan of SURVEY.md 8(e) on the materialised kernel
matrix, host side (CPU, gloo world_size 2): ranks own equal ranges of
128-row tiles; a tile pair touching two ranks is evaluated by both, each
keeping its own rows; only the owner of tile row I counts the kernel sums of
pairs (I, J >= I); the [T, 3] tile-row partials are all-gathered and combined
in ascending tile order (mtk_mmd_value_from_tile_partials, the one-rank
finish's order).  The per-tile arithmetic is a numpy f64 restatement (test
infrastructure); world 2 must reproduce world 1 bit for bit.  The device
side (mtk_mmd_gaussian_tiles) is checked in tests/test_gpu_mmd.py."""
import os
import socket

import numpy as np
import pytest

TILE = 128
MULT = (0.25, 0.5, 1.0, 2.0, 4.0)


def tile_ranges(N, world):
    from paper_2011_09463_b200 import api

    T = -(-N // TILE)
    assert api.mmd_tile_ranges(N - 1, 1, world) == [(r * T // world, (r + 1) * T // world) for r in range(world)]
    return api.mmd_tile_ranges(N - 1, 1, world)


def rank_share(Z, m, beta, lo, hi):
    """f64 restatement of one rank's share: gradient rows of its tiles and the
    kernel sums of its tile rows, tile pair by tile pair in the kernel's order"""
    N, d = Z.shape
    n = N - m
    T = -(-N // TILE)
    coef = {(True, True): -2.0 / (m * m), (False, False): -2.0 / (n * n)}
    part = np.zeros((T, 3))
    g = np.zeros_like(Z)
    rows = lambda t: range(t * TILE, min(N, (t + 1) * TILE))  # noqa: E731
    pairs = [(I, J) for I in range(T) for J in range(I, T) if lo <= I < hi or lo <= J < hi]
    for I, J in pairs:
        own_i, own_j = lo <= I < hi, lo <= J < hi
        for i in rows(I):
            for j in rows(J):
                if I == J and j < i:
                    continue
                d2 = float(((Z[i] - Z[j]) ** 2).sum())
                k = sum(np.exp(-d2 / (beta * q)) for q in MULT)
                A = sum(2.0 / (beta * q) * np.exp(-d2 / (beta * q)) for q in MULT)
                si, sj = i < m, j < m
                f = coef.get((si, sj), 2.0 / (m * n)) * A
                if i != j:
                    if own_i:
                        g[i] += f * (Z[i] - Z[j])
                    if own_j:
                        g[j] += f * (Z[j] - Z[i])
                if own_i:
                    mult = 1.0 if i == j else 2.0
                    c = 0 if (si and sj) else 1 if (not si and not sj) else 2
                    part[I, c] += k if c == 2 else mult * k
    return g, part


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    Z, m, beta = _sample()
    lo, hi = tile_ranges(Z.shape[0], world)[rank]
    g, part = rank_share(Z, m, beta, lo, hi)
    parts = [torch.empty(part.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, torch.from_numpy(part))
    grads = [torch.empty(g.shape, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(grads, torch.from_numpy(g))
    tot = sum(p.numpy() for p in parts)
    G = np.zeros_like(g)
    for r, (a, b) in enumerate(tile_ranges(Z.shape[0], world)):
        G[a * TILE:b * TILE] = grads[r].numpy()[a * TILE:b * TILE]
    out[rank] = (tot.tobytes(), G.tobytes())
    dist.destroy_process_group()


def _sample():
    rng = np.random.default_rng(7)
    m, n, d = 300, 212, 6
    Z = rng.standard_normal((m + n, d))
    Z[m:] += 0.3
    N = m + n
    beta = (2 * N * (Z * Z).sum() - 2 * (Z.sum(0) ** 2).sum()) / (N * N - N)
    return Z, m, beta


@pytest.mark.timeout(600)
def test_tile_sharded_mmd_two_ranks_gloo_bit_identical_to_one():
    import torch.multiprocessing as mp

    from paper_2011_09463_b200 import api

    Z, m, beta = _sample()
    g1, p1 = rank_share(Z, m, beta, 0, -(-Z.shape[0] // TILE))
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    for r in range(2):
        assert out[r][0] == p1.tobytes()  # partials: one owner per tile row, exact
        assert out[r][1] == g1.tobytes()  # gradient rows: the owner's arithmetic
    n = Z.shape[0] - m
    v = api.mmd_value_from_tiles(p1, m, n)
    # the library's combination = ascending tile rows of the V-statistic
    s3 = [sum(p1[I, c] for I in range(p1.shape[0])) for c in range(3)]
    assert v == s3[0] / (m * m) + s3[1] / (n * n) - 2.0 * s3[2] / (m * n)
    # and it is the MMD^2 (independent all-pairs evaluation)
    d2 = ((Z[:, None, :] - Z[None, :, :]) ** 2).sum(-1)
    K = sum(np.exp(-d2 / (beta * q)) for q in MULT)
    ref = K[:m, :m].mean() + K[m:, m:].mean() - 2 * K[:m, m:].mean()
    assert abs(v - ref) <= 1e-12 * abs(ref)
    # ranks balanced: s*T - s^2/2 tile pairs each for equal ranges
    T = p1.shape[0]
    work = [sum(1 for I in range(T) for J in range(I, T) if a <= I < b or a <= J < b)
            for a, b in tile_ranges(Z.shape[0], 2)]
    assert work == [7, 7]  # T = 4: s T - s^2/2 + s/2 = 7 pairs each
