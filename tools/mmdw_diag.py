"""mmd_w ablations (W path, one group, N = 8192 rows x d = 256: 2080 tile
pairs): MTK_MMDW_DIAG 0 normal, 1 epilogue only arrives, 2 no MMAs, 3 no W
stores.  Times the whole mtk_mmd_gaussian call by CUDA events."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_09463_b200 import api  # noqa: E402

ctx = api.Context(0)
N, d = 8192, 256
Z = torch.relu(torch.randn(N, d, device="cuda"))
Xs, Xt = Z[:4096], Z[4096:]
for mode in ("0", "1", "2", "3", "0"):
    os.environ["MTK_MMDW_DIAG"] = mode
    ts = []
    for it in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        try:
            api.mmd_gaussian(ctx, Xs, Xt)
        except Exception:
            pass
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1000)
    print("diag", mode, "us:", [round(t, 1) for t in ts[2:]])
