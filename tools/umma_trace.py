"""Timeline of CTA 0 of the CTA-pair GEMM (diagnostics):
python tools/umma_trace.py G M N K a_mn b_mn"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
tr = torch.zeros(5000, dtype=torch.int64, device="cuda")
os.environ["MTK_UMMA_TRACE"] = str(tr.data_ptr())
from paper_2011_09463_b200 import api  # noqa: E402

ctx = api.Context(0)
if sys.argv[1] == "bank":  # the last tcgen05 GEMM of a C2 bank step (DW of layer 0)
    DIMS = [1024, 512, 256, 10]
    bank = api.Bank(ctx, 32, DIMS)
    rng = api.Rng(1)
    for g in range(32):
        bank.init_params(g, rng)
    X = torch.randn((32, 1024, 1024), device="cuda")
    y = torch.randint(0, 10, (32, 1024), device="cuda", dtype=torch.int32)
    for _ in range(3):
        tr.zero_()
        bank.train_step(X, y, lr=0.01, src_rows=512, mmd_lambda=1.0, want_loss=False)
    torch.cuda.synchronize()
    G, M, N, K, a_mn, b_mn = 32, 1024, 512, 1024, 1, 1
else:
    G, M, N, K, a_mn, b_mn = [int(x) for x in sys.argv[1:7]]
A = torch.randn((G, K, M) if a_mn else (G, M, K), device="cuda")
B = torch.randn((G, K, N) if b_mn else (G, N, K), device="cuda")
for _ in range(3 if sys.argv[1] != "bank" else 0):
    tr.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    api.diag_gemm_tf32x3(ctx, A, B, bool(a_mn), bool(b_mn))
    e1.record()
    torch.cuda.synchronize()
t = tr.cpu().numpy().astype(np.int64)
t0 = t[:4000][t[:4000] > 0].min()
prod = (t[:1000][t[:1000] > 0] - t0) / 1000
mma = (t[1000:2000][t[1000:2000] > 0] - t0) / 1000
cv0 = (t[3000:4000][t[3000:4000] > 0] - t0) / 1000
if sys.argv[1] != "bank":
    print(f"diag call {e0.elapsed_time(e1)*1000:.1f} us; flops {2*G*M*N*K*3/1e12:.3f} TF(tensor)")
print("producer stage issue (us):", np.round(prod[:40], 2).tolist(), "... n =", len(prod))
print("conv start (TMA landed):", np.round(cv0[:40], 2).tolist())
print("mma stage issue      (us):", np.round(mma[:40], 2).tolist(), "... last", np.round(mma[-1:], 2))
d = np.diff(mma)
print("mma per-stage median %.3f us, mean %.3f" % (np.median(d), d.mean()))
c = t[4000:4800].reshape(-1, 2)
c = c[c[:, 0] > 0]
st, en = (c[:, 0] - c[:, 0].min()) / 1000, (c[:, 1] - c[:, 0].min()) / 1000
print("CTAs %d: start max %.2f, end min %.2f median %.2f max %.2f us" % (len(c), st.max(), en.min(), np.median(en), en.max()))
print("CTA0 passes final barrier at %.2f us" % ((t[2040] - t0) / 1000))
ep = t[2000:2032]
for i in range(16):
    if ep[2 * i] > 0:
        print("tile %d epilogue %.2f -> %.2f us" % (i, (ep[2 * i] - t0) / 1000, (ep[2 * i + 1] - t0) / 1000))
for i in range(4):
    row = t[2100 + 32 * i: 2100 + 32 * i + 16].reshape(4, 4)
    if row[0, 0] > 0:
        print("tile %d chunks (pre-ld, post-ld, post-store) us:" % i,
              [[round((x - t0) / 1000, 2) for x in r[:3] if x > 0] for r in row])
