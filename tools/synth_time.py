"""Host-clock time of mtk_synth (the sweep's population draws) at the C5 pool sizes."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_09463_b200 import api  # noqa: E402

r = api.Rng(5)
mu = np.random.default_rng(0).standard_normal((10, 784))
for n in (8192, 16384):
    ts = []
    for _ in range(5):
        t = time.perf_counter()
        r.synth(10, 784, n, mu)
        ts.append(time.perf_counter() - t)
    print(f"synth {n} x 784: median {1000 * sorted(ts)[2]:.1f} ms (min {1000 * min(ts):.1f})")
