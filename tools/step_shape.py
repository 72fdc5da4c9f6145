"""Device time and phase split of one bank train_step at a given shape
(diagnostics for the sweep's shadow banks):
  python tools/step_shape.py G B d0,d1,...,dL [heads] [src_rows] [mmd_lambda]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_09463_b200 import api  # noqa: E402

G, B = int(sys.argv[1]), int(sys.argv[2])
dims = [int(x) for x in sys.argv[3].split(",")]
heads = int(sys.argv[4]) if len(sys.argv) > 4 else 1
src = int(sys.argv[5]) if len(sys.argv) > 5 else 0
lam = float(sys.argv[6]) if len(sys.argv) > 6 else 0.0
ctx = api.Context(0)
bank = api.Bank(ctx, G, dims, heads)
for g in range(G):
    bank.init_params(g, api.Rng(100 + g))
X = torch.randn(G, B, dims[0], device="cuda")
y = torch.randint(0, dims[-1], (G, B), device="cuda", dtype=torch.int32)
kw = dict(src_rows=src, mmd_lambda=lam, lr=0.01)
if heads == 2:
    kw["denom"] = (float(src), float(B - src))
for _ in range(5):
    bank.train_step(X, y, want_loss=False, **kw)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 50
n0 = ctx.launches
e0.record()
for _ in range(n):
    bank.train_step(X, y, want_loss=False, **kw)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
launches = (ctx.launches - n0) / n
ctx.set_timing(True)
for _ in range(n):
    bank.train_step(X, y, want_loss=False, **kw)
ph = ctx.phase_times()
ctx.set_timing(False)
flop = 6 * G * B * sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))
print(f"G={G} B={B} dims={dims} heads={heads} src={src} lam={lam}: {ms * 1000:.1f} us/step, "
      f"{launches:.0f} launches, {flop / ms / 1e9:.1f} TFLOP/s, tc={bank.tc_layers()}")
print("  phases us/step:", {k: round(v[0] * 1000 / n, 1) for k, v in ph.items() if v[0]})

# the same steps through train_epoch (device gather of a [pool] by indices):
# the host-side cost of one call beyond the steps
steps = 16
pool = torch.randn(8192, dims[0], device="cuda")
ypool = torch.randint(0, dims[-1], (8192,), device="cuda", dtype=torch.int32)
idx = torch.randint(0, 8192, (steps, G, B), device="cuda", dtype=torch.int64)
for _ in range(2):
    bank.train_epoch(pool, ypool, idx, **kw)
torch.cuda.synchronize()
import time  # noqa: E402
t = time.perf_counter()
for _ in range(5):
    bank.train_epoch(pool, ypool, idx, **kw)
torch.cuda.synchronize()
dt = (time.perf_counter() - t) / 5
print(f"  train_epoch of {steps} steps: {dt * 1000:.2f} ms host clock ({dt * 1e6 / steps:.1f} us/step)")
