"""Timeline of one MMD CTA (diagnostics): python tools/mmd_trace.py [N] [d] [G]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
tr = torch.zeros(12288 + 3 * 4096, dtype=torch.int64, device="cuda")
os.environ["MTK_MMD_TRACE"] = str(tr.data_ptr())
from paper_2011_09463_b200 import api  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
d = int(sys.argv[2]) if len(sys.argv) > 2 else 256
ctx = api.Context(0)
Xs = torch.randn(N // 2, d, device="cuda")
Xt = torch.randn(N - N // 2, d, device="cuda") + 0.3
for _ in range(2):
    tr.zero_()
    api.mmd_gaussian(ctx, Xs, Xt)
t = tr.cpu().numpy().astype(np.int64)
t0 = min(x for x in t if x > 0)
def stage_types(njt, nkc=8, n2=4):
    ty = []
    for tt in range(njt + 1):
        if tt < njt:
            ty += ["G1"] * nkc
        if tt >= 1:
            ty += ["G2"] * n2
    return ty


def split_gaps(name, arr, njt, nkc):
    arr = arr[arr > 0]
    ty = stage_types(njt, nkc)[: len(arr)]
    dd = np.diff(arr) / 1000
    for kind in ("G1", "G2"):
        v = [dd[i] for i in range(len(dd)) if ty[i] == kind]
        if v:
            print(f"   {name} {kind}: {len(v)} stages, mean {np.mean(v):.3f} us, median {np.median(v):.3f}")


def show(name, arr):
    arr = arr[arr > 0] - t0
    print(name, len(arr), "events; first 40 (us):", np.round(arr[:40] / 1000, 2).tolist())
    if len(arr) > 1:
        print("   span", (arr.max() - arr.min()) / 1000, "us; mean gap", np.diff(arr).mean() / 1000, "us")
show("producer stage-issue", t[:4096])
show("mma stage-consume", t[4096:8192])
split_gaps("mma consume", t[4096:8192], (N + 63) // 64, (d + 31) // 32)
ep = t[8192:12288]
show("epilogue s_full seen / w arrived", ep)

if len(sys.argv) > 3:  # full bank step (G models) for CTA (0,0,0) under load
    G = int(sys.argv[3])
    DIMS = [1024, 512, d, 10]
    bank = api.Bank(ctx, G, DIMS)
    rng = api.Rng(1)
    for g in range(G):
        bank.init_params(g, rng)
    X = torch.randn((G, N, DIMS[0]), device="cuda")
    y = torch.randint(0, 10, (G, N), device="cuda", dtype=torch.int32)
    for _ in range(2):
        tr.zero_()
        bank.train_step(X, y, lr=0.01, src_rows=N // 2, mmd_lambda=1.0, want_loss=False)
    torch.cuda.synchronize()
    t = tr.cpu().numpy().astype(np.int64)
    t0 = min(x for x in t if x > 0)
    print(f"---- bank step, G={G}")
    show("producer stage-issue", t[:4096])
    show("mma stage-consume", t[4096:8192])
    split_gaps("mma consume", t[4096:8192], (N + 63) // 64, (d + 31) // 32)
    show("epilogue s_full seen / w arrived", t[8192:12288])
    c = t[12288:].reshape(-1, 3)
    c = c[c[:, 0] > 0]
    st, en, sm = (c[:, 0] - c[:, 0].min()) / 1000, (c[:, 1] - c[:, 0].min()) / 1000, c[:, 2]
    print("CTAs", len(c), "kernel span (us)", en.max(), "SMs used", len(set(sm.tolist())))
    dur = en - st
    print("CTA duration us: min %.1f median %.1f max %.1f" % (dur.min(), np.median(dur), dur.max()))
    print("start times sorted (us):", np.round(np.sort(st), 1)[::8].tolist())
    print("end times sorted (us):", np.round(np.sort(en), 1)[::8].tolist())
    base = c[:, 0].min()
    print("CTA0 warp1 loop done %.2f; epi: v_full %.2f zstage %.2f grad %.2f store %.2f red %.2f" % tuple((t[i] - base) / 1000 for i in (12282, 12283, 12284, 12285, 12286, 12287)))
    print("CTA0: warp1 after syncthreads %.2f, fence_after done %.2f, end %.2f, dealloc done %.2f (us)" % (
        (t[12281] - base) / 1000, (t[12280] - base) / 1000, en[0], (c[0, 2] - base) / 1000))
    dd = (c[:, 2] - c[:, 0].min()) / 1000 - en
    print("dealloc done - end (us): min %.2f median %.2f max %.2f" % (dd.min(), np.median(dd), dd.max()))
