"""Phase stamps of the attack-model epoch kernel (MTK_EPOCH_TRACE), CTA 0, steps 0-7."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
tr = torch.zeros(64, dtype=torch.int64, device="cuda")
os.environ["MTK_EPOCH_TRACE"] = str(tr.data_ptr())
from paper_2011_09463_b200 import api  # noqa: E402

ctx = api.Context(0)
n, B, steps = 1 << 20, 1024, 1024
X = torch.randn(n, 3, device="cuda")
y = torch.randint(0, 2, (n,), device="cuda", dtype=torch.int32)
idx = torch.randint(0, n, (steps, 1, B), device="cuda", dtype=torch.int64)
bank = api.Bank(ctx, 1, [3, 64, 2])
bank.init_params(0, api.Rng(3))
for _ in range(3):
    tr.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bank.train_epoch(X, y, idx, None, None, lr=0.1)
    e1.record()
    torch.cuda.synchronize()
print(f"epoch {e0.elapsed_time(e1):.2f} ms = {e0.elapsed_time(e1) * 1000 / steps:.2f} us/step")
t = tr.cpu().numpy().reshape(8, 8).astype(np.int64)
names = ["loads+fwd", "bwd", "butterflies", "sync1", "update", "sync2"]
for s in range(1, 8):
    d = np.diff(t[s, :7]) / 1000
    nxt = (t[s + 1, 0] - t[s, 6]) / 1000 if s < 7 else 0
    print(f"step {s}: " + " ".join(f"{nm} {v:.2f}" for nm, v in zip(names, d)) + f" | to next {nxt:.2f} us")
