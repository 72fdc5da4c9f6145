"""Run a few bank steps at the bench configuration (for ncu captures).

  python tools/profile_step.py [steps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_09463_b200 import api  # noqa: E402

DIMS = [1024, 512, 256, 10]
G, SRC, B = 32, 512, 1024
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
ctx = api.Context(0)
bank = api.Bank(ctx, G, DIMS)
rng = api.Rng(1)
for g in range(G):
    bank.init_params(g, rng)
gen = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn((G, B, DIMS[0]), device="cuda", generator=gen)
X[:, SRC:] += 0.5
y = torch.randint(0, 10, (G, B), device="cuda", dtype=torch.int32, generator=gen)
for _ in range(steps):
    bank.train_step(X, y, lr=0.01, src_rows=SRC, mmd_lambda=1.0, want_loss=False)
torch.cuda.synchronize()
print("ok", ctx.launches)
