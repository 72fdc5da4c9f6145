"""Time one paradigm of the sweep on the GPU backend (per-phase wall clock):
python tools/time_sweep.py [paradigm] [n_shadows] [epochs] [attack_epochs] [data_rng] [pool]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2011_09463_b200 import sweep  # noqa: E402

par = sys.argv[1] if len(sys.argv) > 1 else "model"
ns = int(sys.argv[2]) if len(sys.argv) > 2 else 95
ep = int(sys.argv[3]) if len(sys.argv) > 3 else 10
aep = int(sys.argv[4]) if len(sys.argv) > 4 else 30
drng = sys.argv[5] if len(sys.argv) > 5 else "host"
pool = int(sys.argv[6]) if len(sys.argv) > 6 else 8192
cfg = sweep.SweepConfig(paradigm=par, n_shadows=ns, epochs=ep, attack_epochs=aep, data_rng=drng,
                        pool=pool, source_pool=max(16384, pool),
                        dims=(784, 256, 10) if par != "mapping" else (1024, 512, 256, 10))
be = sweep.GpuBackend()
t0 = time.perf_counter()
pop = sweep.Population(cfg, be.Rng, be.synth_counter)
M = 1 + cfg.n_shadows
streams = pop.model_streams(M + 1)
torch.cuda.synchronize()
t1 = time.perf_counter()
bank, mem, non = sweep.train_bank(be, cfg, pop, streams, list(range(M)))
torch.cuda.synchronize()
t2 = time.perf_counter()
F, lab = sweep.query_features(be, cfg, pop, bank, mem, non)
t3 = time.perf_counter()
import numpy as np  # noqa: E402
Ftr = F[1:].reshape(-1, cfg.k).float().contiguous()
ltr = np.tile(lab, cfg.n_shadows)
att = sweep.train_attack(be, cfg, Ftr, ltr, streams[M])
torch.cuda.synchronize()
t4 = time.perf_counter()
scores = be.attack_scores(att, F[0].float().contiguous())
auc, acc = be.auc(scores, lab)
t5 = time.perf_counter()
print(f"{par} [{drng}, pool {pool}]: models {M}: data {t1-t0:.2f}s train {t2-t1:.2f}s query {t3-t2:.2f}s "
      f"attack-train {t4-t3:.2f}s score+auc {t5-t4:.2f}s total {t5-t0:.2f}s; auc {auc:.4f} acc {acc:.4f}")
