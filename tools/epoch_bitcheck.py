"""Parameters after one attack-model epoch, dumped for a cross-build comparison."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_09463_b200 import api  # noqa: E402

ctx = api.Context(0)
g = torch.Generator(device="cuda").manual_seed(1)
n, B, steps = 1 << 16, 1024, 50
X = torch.randn(n, 3, device="cuda", generator=g)
y = torch.randint(0, 2, (n,), device="cuda", dtype=torch.int32, generator=g)
idx = torch.randint(0, n, (steps, 1, B), device="cuda", dtype=torch.int64, generator=g)
w = torch.ones(steps, 1, B, device="cuda")
den = np.full(steps, float(B))
bank = api.Bank(ctx, 1, [3, 64, 2])
bank.init_params(0, api.Rng(3))
bank.train_epoch(X, y, idx, w, den, lr=0.1)
W, b = bank.get_params(0)
np.savez(sys.argv[1], *W, *b)
print("saved", sys.argv[1])
