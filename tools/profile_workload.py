"""One step of a bench workload between cudaProfilerStart/Stop, for ncu
captures with --profile-from-start off:

  ncu --profile-from-start off --set full ... python tools/profile_workload.py c2
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      ... python tools/profile_workload.py c4|attack|c3

The step is the bench's own (bench.py measure_* set-up), after 2 warm-up steps."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_09463_b200 import api  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "c2"
ctx = api.Context(0)
gen = torch.Generator(device="cuda").manual_seed(4)
if wl == "c2":
    import bench

    bank = api.Bank(ctx, bench.G, bench.DIMS)
    r = api.Rng(1)
    for g in range(bench.G):
        bank.init_params(g, r)
    X = torch.randn((bench.G, bench.B, bench.DIMS[0]), device="cuda", generator=gen)
    X[:, bench.SRC:] += 0.5
    y = torch.randint(0, 10, (bench.G, bench.B), device="cuda", dtype=torch.int32, generator=gen)

    def step():
        bank.train_step(X, y, lr=bench.LR, src_rows=bench.SRC, mmd_lambda=bench.LAMBDA, want_loss=False)
elif wl == "c4":
    m, n, d = 65536, 8192, 512
    Z = torch.randn(m + n, d, device="cuda", generator=gen)
    Z[m:] += 0.1
    beta = api.mmd_beta(ctx, Z[:m], Z[m:])

    def step():
        api.mmd_gaussian(ctx, Z[:m], Z[m:], beta=beta)
elif wl == "attack":
    Q = 1 << 20
    logits = torch.randn(Q, 10, device="cuda", generator=gen)
    labels = (torch.rand(Q, device="cuda", generator=gen) < 0.5).to(torch.uint8)
    logits[labels.bool(), 0] += 1.0
    att = api.Bank(ctx, 1, [3, 64, 2])
    att.init_params(0, api.Rng(77))

    def step():
        api.attack_auc(att, logits, labels)
else:
    raise SystemExit(f"unknown workload {wl}")
for _ in range(2):
    step()
torch.cuda.synchronize()
n0 = ctx.launches
torch.cuda.profiler.start()
step()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(f"profiled one {wl} step: {ctx.launches - n0} launches")
