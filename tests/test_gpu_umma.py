"""GPU: the tcgen05 3xTF32 grouped GEMM (k_umma.cu) against an f64 product.

All four operand-major combinations the bank uses, aligned and ragged shapes,
both the 128x128 single-CTA kernel and the 256x256 CTA-pair kernel (M, N > 128)
(K not a multiple of 32, M/N not multiples of 128), G > 1.  Tolerance
1e-5 relative (max-abs / max-abs), the north_star per-kernel bound.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.mark.parametrize("a_mn,b_mn", [(0, 1), (0, 0), (1, 1), (1, 0)])
@pytest.mark.parametrize("G,M,N,K", [(1, 128, 128, 32), (2, 256, 128, 784), (3, 200, 96, 76), (2, 136, 40, 20),
                                     (2, 1024, 512, 1024), (1, 64, 256, 512),
                                     (2, 384, 320, 100), (3, 300, 260, 64)])
def test_umma_gemm(ctx, a_mn, b_mn, G, M, N, K):
    from paper_2011_09463_b200 import api

    g = torch.Generator().manual_seed(M + N + K)
    A = torch.randn((G, M, K), generator=g)
    B = torch.randn((G, K, N), generator=g)
    ref = torch.matmul(A.double(), B.double()).numpy()
    Ad = (A.transpose(1, 2) if a_mn else A).contiguous().cuda()
    Bd = (B if b_mn else B.transpose(1, 2)).contiguous().cuda()
    C = api.diag_gemm_tf32x3(ctx, Ad, Bd, bool(a_mn), bool(b_mn)).cpu().double().numpy()
    e = rel(C, ref)
    assert e <= 1e-5, e


@pytest.mark.parametrize("a_mn,b_mn", [(0, 1), (0, 0), (1, 1), (1, 0)])
@pytest.mark.parametrize("G,M,N,K", [(32, 1024, 512, 64), (20, 512, 392, 100), (40, 300, 300, 36)])
def test_umma_gemm_half_tiles(ctx, a_mn, b_mn, G, M, N, K):
    """Tile counts whose last partial wave is split into N halves (256 x 128
    pair tiles), including ragged M / N edges inside the halves."""
    from paper_2011_09463_b200 import api

    g = torch.Generator(device="cuda").manual_seed(G + M + N + K)
    A = torch.randn((G, M, K), device="cuda", generator=g)
    B = torch.randn((G, K, N), device="cuda", generator=g)
    ref = torch.matmul(A.double(), B.double())
    Ad = (A.transpose(1, 2) if a_mn else A).contiguous()
    Bd = (B if b_mn else B.transpose(1, 2)).contiguous()
    C = api.diag_gemm_tf32x3(ctx, Ad, Bd, bool(a_mn), bool(b_mn)).double()
    e = float((C - ref).abs().max() / ref.abs().max())
    assert e <= 1e-5, e
