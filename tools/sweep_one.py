"""One paradigm of the C5 sweep (for ncu launch lists): python tools/sweep_one.py mapping"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2011_09463_b200 import api  # noqa: E402

par = sys.argv[1] if len(sys.argv) > 1 else "mapping"
cfg = dict(paradigm=par, n_shadows=256)
if par == "mapping":
    cfg["dims"] = (1024, 512, 256, 10)
ctx = api.Context(0)
api.sweep_run(ctx, cfg, None)
torch.cuda.synchronize()
t = time.perf_counter()
api.sweep_run(ctx, cfg, None)
torch.cuda.synchronize()
print(f"{par}: {time.perf_counter() - t:.3f} s wall", flush=True)
