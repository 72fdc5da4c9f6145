"""Host-clock cost per call of the attack / AUC entry points (diagnostics):
fixed per-call overhead (tiny inputs) vs the 2^20-query bench shape."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2011_09463_b200 import api  # noqa: E402

ctx = api.Context(0)
att = api.Bank(ctx, 1, [3, 64, 2])
att.init_params(0, api.Rng(77))
gen = torch.Generator(device="cuda").manual_seed(5)
for Q in (1024, 1 << 20):
    logits = torch.randn(Q, 10, device="cuda", generator=gen)
    labels = (torch.rand(Q, device="cuda", generator=gen) < 0.5).to(torch.uint8)
    logits[labels.bool(), 0] += 1.0
    scores = torch.rand(Q, device="cuda", generator=gen) * 0.05 + 0.48
    for name, fn in [("attack_auc", lambda: api.attack_auc(att, logits, labels)),
                     ("auc", lambda: api.auc(ctx, scores, labels))]:
        for _ in range(20):
            fn()
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(200):
            fn()
        dt = (time.perf_counter() - t) / 200 * 1e6
        print(f"Q={Q:8d} {name:10s} {dt:7.1f} us/call (host clock)")
# the raw C entry point (no Python argument handling)
import ctypes as C  # noqa: E402
from paper_2011_09463_b200._lib import lib  # noqa: E402
a, acc = C.c_double(), C.c_double()
for Q in (1024, 1 << 20):
    scores = torch.rand(Q, device="cuda", generator=gen) * 0.05 + 0.48
    labels = (torch.rand(Q, device="cuda", generator=gen) < 0.5).to(torch.uint8)
    ps, pl = C.c_void_p(scores.data_ptr()), C.c_void_p(labels.data_ptr())
    for _ in range(20):
        lib.mtk_auc(ctx.h, ps, pl, Q, C.byref(a), C.byref(acc))
    t = time.perf_counter()
    for _ in range(200):
        lib.mtk_auc(ctx.h, ps, pl, Q, C.byref(a), C.byref(acc))
    print(f"Q={Q:8d} raw mtk_auc {(time.perf_counter() - t) / 200 * 1e6:7.1f} us/call")
for Q in (1024, 1 << 20):
    logits = torch.randn(Q, 10, device="cuda", generator=gen)
    labels = (torch.rand(Q, device="cuda", generator=gen) < 0.5).to(torch.uint8)
    pl, pb = C.c_void_p(logits.data_ptr()), C.c_void_p(labels.data_ptr())
    for _ in range(20):
        lib.mtk_attack_auc(att.h, pl, Q, 10, pb, C.byref(a), C.byref(acc), None)
    t = time.perf_counter()
    for _ in range(200):
        lib.mtk_attack_auc(att.h, pl, Q, 10, pb, C.byref(a), C.byref(acc), None)
    print(f"Q={Q:8d} raw mtk_attack_auc {(time.perf_counter() - t) / 200 * 1e6:7.1f} us/call")
s = torch.cuda.current_stream()
x = torch.empty(16, device="cuda")
h = torch.empty(16, pin_memory=True)
t = time.perf_counter()
for _ in range(200):
    h.copy_(x, non_blocking=True)
    s.synchronize()
print(f"torch D2H 64 B + sync {(time.perf_counter() - t) / 200 * 1e6:7.1f} us")
