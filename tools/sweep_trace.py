"""Phase wall times of the native C5 sweep (MTK_SWEEP_TRACE), per paradigm."""
import os
import sys
import time

os.environ["MTK_SWEEP_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2011_09463_b200 import api  # noqa: E402

ctx = api.Context(0)
cfgs = [dict(paradigm="model", n_shadows=256), dict(paradigm="mapping", n_shadows=256, dims=(1024, 512, 256, 10)),
        dict(paradigm="parameter", n_shadows=256)]
for c in cfgs:
    api.sweep_run(ctx, c, None)  # warm
for c in cfgs:
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = api.sweep_run(ctx, c, None)
    torch.cuda.synchronize()
    print(f"== {c['paradigm']}: {time.perf_counter() - t:.3f} s  {r}", file=sys.stderr, flush=True)
