"""Error of the tcgen05 3xTF32 GEMM vs fp64 as K grows (diagnostics):
max|C - C64| / max|C64| for zero-mean and for positive (same-sign running
sums) operands.  python tools/gemm_precision.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2011_09463_b200 import api  # noqa: E402

ctx = api.Context(0)
g = torch.Generator(device="cuda").manual_seed(0)
for sepc in ("0", "1"):
  os.environ["MTK_UMMA_SEPC"] = sepc
  print(f"MTK_UMMA_SEPC={sepc}")
  for kind in ("zero-mean", "positive"):
    for K in (256, 512, 1024, 2048, 4096):
        M, N = 512, 256
        A = torch.randn(1, M, K, device="cuda", generator=g)
        Bm = torch.randn(1, K, N, device="cuda", generator=g)
        if kind == "positive":
            A = A.abs()
            Bm = Bm.abs()
        C = api.diag_gemm_tf32x3(ctx, A, Bm, False, True)
        ref = A.double() @ Bm.double()
        err = ((C.double() - ref).abs().max() / ref.abs().max()).item()
        bias = ((C.double() - ref) / ref.abs().max()).mean().item()
        print(f"{kind:9s} K={K:5d}: rel err {err:.2e}  mean signed err {bias:+.2e}")
