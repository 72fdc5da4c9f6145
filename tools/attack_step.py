"""Attack-model training steps ([k, 64, 2], B = 1024) for ncu launch lists."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_09463_b200 import api  # noqa: E402

dims = [3, 64, 2]
ctx = api.Context(0)
bank = api.Bank(ctx, 1, dims)
bank.init_params(0, api.Rng(1))
X = torch.rand((1, 1024, 3), device="cuda")
y = torch.randint(0, 2, (1, 1024), device="cuda", dtype=torch.int32)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 5):
    bank.train_step(X, y, lr=0.1, want_loss=False)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(200):
    bank.train_step(X, y, lr=0.1, want_loss=False)
e1.record()
torch.cuda.synchronize()
print("us per step", e0.elapsed_time(e1) * 1000 / 200)
