"""A/B of the two MMD paths inside a C2 bank step (fused pair kernel vs the
materialised-W path): python tools/ab_mmd_path.py -> max |dParams| after one
step, and the MMD values.  Run once with MTK_MMD_FUSED=1 and once without;
the script runs both itself in subprocesses."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np
    import torch

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2011_09463_b200 import api

    DIMS = [1024, 512, 256, 10]
    G, SRC, B = int(sys.argv[2]), 512, int(sys.argv[3])
    ctx = api.Context(0)
    bank = api.Bank(ctx, G, DIMS)
    rng = api.Rng(1)
    for g in range(G):
        bank.init_params(g, rng)
    gen = torch.Generator(device="cuda").manual_seed(0)
    X = torch.randn((G, B, DIMS[0]), device="cuda", generator=gen)
    X[:, SRC:] += 0.5
    y = torch.randint(0, 10, (G, B), device="cuda", dtype=torch.int32, generator=gen)
    bank.keep_grads(True)
    loss, mmd = bank.train_step(X, y, lr=0.01, src_rows=SRC, mmd_lambda=1.0)
    W, b = bank.get_grads(0)
    np.savez(sys.argv[4], mmd=mmd, loss=loss, *W)
    sys.exit(0)

G = sys.argv[1] if len(sys.argv) > 1 else "4"
B = sys.argv[2] if len(sys.argv) > 2 else "1024"
env = dict(os.environ)
subprocess.run([sys.executable, __file__, "child", G, B, "/tmp/ab_w.npz"], check=True, env=env)
env["MTK_MMD_FUSED"] = "1"
subprocess.run([sys.executable, __file__, "child", G, B, "/tmp/ab_f.npz"], check=True, env=env)
import numpy as np  # noqa: E402

a, f = np.load("/tmp/ab_w.npz"), np.load("/tmp/ab_f.npz")
print("mmd W-path", a["mmd"][:4], "fused", f["mmd"][:4], "max rel", np.max(np.abs(a["mmd"] - f["mmd"]) / np.abs(f["mmd"])))
for k in a.files:
    if k.startswith("arr_"):
        d = np.abs(a[k] - f[k]).max() / max(np.abs(f[k]).max(), 1e-30)
        print(k, a[k].shape, "max|d|/max|ref| = %.3e" % d)
