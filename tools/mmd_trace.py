"""Timeline of one MMD CTA (diagnostics): python tools/mmd_trace.py [N] [d] [G]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
tr = torch.zeros(12288, dtype=torch.int64, device="cuda")
os.environ["MTK_MMD_TRACE"] = str(tr.data_ptr())
from paper_2011_09463_b200 import api  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
d = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ctx = api.Context(0)
Xs = torch.randn(N // 2, d, device="cuda")
Xt = torch.randn(N - N // 2, d, device="cuda") + 0.3
for _ in range(2):
    tr.zero_()
    api.mmd_gaussian(ctx, Xs, Xt)
t = tr.cpu().numpy().astype(np.int64)
t0 = min(x for x in t if x > 0)
def show(name, arr):
    arr = arr[arr > 0] - t0
    print(name, len(arr), "events; first 40 (us):", np.round(arr[:40] / 1000, 2).tolist())
    if len(arr) > 1:
        print("   span", (arr.max() - arr.min()) / 1000, "us; mean gap", np.diff(arr).mean() / 1000, "us")
show("producer stage-issue", t[:4096])
show("mma stage-consume", t[4096:8192])
ep = t[8192:12288]
show("epilogue s_full seen / w arrived", ep)
