"""Run the diagnostic grouped GEMM once (for ncu): python tools/diag_gemm.py G M N K a_mn b_mn"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_09463_b200 import api  # noqa: E402

G, M, N, K, a_mn, b_mn = [int(x) for x in sys.argv[1:7]]
ctx = api.Context(0)
A = torch.randn((G, K, M) if a_mn else (G, M, K), device="cuda")
B = torch.randn((G, K, N) if b_mn else (G, N, K), device="cuda")
for _ in range(2):
    api.diag_gemm_tf32x3(ctx, A, B, bool(a_mn), bool(b_mn))
torch.cuda.synchronize()
print("ok")
