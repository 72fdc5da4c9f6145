"""Per-GEMM timelines of CTA 0 inside a C2 bank step (diagnostics):
  python tools/umma_bank_trace.py
For each tcgen05 GEMM of the step (selected by MTK_UMMA_TRACE_SHAPE) prints
the MMA stage pacing, each tile's epilogue span and its chunk stamps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
tr = torch.zeros(5000, dtype=torch.int64, device="cuda")
os.environ["MTK_UMMA_TRACE"] = str(tr.data_ptr())
from paper_2011_09463_b200 import api  # noqa: E402

DIMS = [1024, 512, 256, 10]
G, B = 32, 1024
ctx = api.Context(0)
bank = api.Bank(ctx, G, DIMS)
rng = api.Rng(1)
for g in range(G):
    bank.init_params(g, rng)
X = torch.randn((G, B, DIMS[0]), device="cuda")
y = torch.randint(0, 10, (G, B), device="cuda", dtype=torch.int32)
# (name, M, N, K, epi): kBias 0, kBiasRelu 1, kMask 2, kSgd 3, kStore 4, kMmdGrad 6
SHAPES = [("fwd0", B, 512, 1024, 1), ("fwd1", B, 256, 512, 1), ("vgemm", B, 256, B + 32, 7),
          ("dx1", B, 512, 256, 2), ("dw1", 512, 256, B, 3), ("dw0", 1024, 512, B, 3)]
for name, M, N, K, e in SHAPES:
    os.environ["MTK_UMMA_TRACE_SHAPE"] = f"{M},{N},{K},{e}"
    for _ in range(3):
        tr.zero_()
        bank.train_step(X, y, lr=0.01, src_rows=512, mmd_lambda=1.0, want_loss=False)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.int64)
    if not (t[:4000] > 0).any():
        print(name, "no trace (shape not launched?)")
        continue
    t0 = t[:4000][t[:4000] > 0].min()
    mma = (t[1000:2000][t[1000:2000] > 0] - t0) / 1000
    d = np.diff(mma)
    c = t[4000:4800].reshape(-1, 2)
    c = c[c[:, 0] > 0]
    en = (c[:, 1] - c[:, 0].min()) / 1000
    print(f"== {name} M{M} N{N} K{K} epi{e}: CTA end median {np.median(en):.1f} max {en.max():.1f} us; "
          f"mma stages {len(mma)} median {np.median(d):.3f} us mean {d.mean():.3f}")
    if os.environ.get("SHOW_STAGES") == name:
        prod = (t[:1000][t[:1000] > 0] - t0) / 1000
        cv = (t[3000:4000][t[3000:4000] > 0] - t0) / 1000
        print("  producer", np.round(prod[:40], 2).tolist())
        print("  conv    ", np.round(cv[:40], 2).tolist())
        print("  mma     ", np.round(mma[:40], 2).tolist())
    ep = t[2000:2032]
    for i in range(16):
        if ep[2 * i] > 0:
            row = t[2100 + 32 * i: 2100 + 32 * i + 32].reshape(8, 4) if i < 4 else None
            ch = ""
            if row is not None:
                ch = " chunks " + " ".join(f"[{(r[0]-t0)/1000:.1f} ld{(r[1]-r[0])/1000:.2f} +{(r[2]-r[1])/1000:.2f}]"
                                           for r in row if r[0] > 0)
            print(f"  tile {i} epi {(ep[2*i]-t0)/1000:.2f} -> {(ep[2*i+1]-t0)/1000:.2f}{ch}")
