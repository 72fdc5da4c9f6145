import os, sys, torch, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2011_09463_b200 import api
ctx = api.Context(0)
gen = torch.Generator(device="cuda").manual_seed(5)
Q = 1 << 20
logits = torch.randn(Q, 10, device="cuda", generator=gen)
labels = (torch.rand(Q, device="cuda", generator=gen) < 0.5).to(torch.uint8)
logits[labels.bool(), 0] += 1.0
att = api.Bank(ctx, 1, [3, 64, 2]); att.init_params(0, api.Rng(77))
a, acc, s = api.attack_auc(att, logits, labels, scores=True)
s = s.cpu().numpy()
u = s.view(np.uint32).astype(np.uint64)
key = np.where(u & 0x80000000, (~u) & 0xffffffff, u | 0x80000000)
kmin, kmax = key.min(), key.max()
print("auc", a, "score range", s.min(), s.max(), "key range", int(kmax - kmin), "log2", np.log2(float(kmax - kmin) + 1))
print("distinct keys", len(np.unique(key)))
for bits in (14, 16, 18, 20):
    r = int(kmax - kmin); sh = max(0, r.bit_length() - bits)
    b = ((key - kmin) >> sh).astype(np.int64)
    c = np.bincount(b)
    lab = labels.cpu().numpy()
    cn = np.bincount(b, weights=(lab == 0))
    mixed = (cn > 0) & (cn < c)
    print(f"bins 2^{bits} shift {sh}: nonzero {np.count_nonzero(c)} max {c.max()} mean-nonzero {c[c>0].mean():.1f} "
          f"mixed bins {mixed.sum()} queries in mixed {c[mixed].sum()} p99 {np.percentile(c[c>0], 99):.0f} "
          f">512: {(c>512).sum()} >2048: {(c>2048).sum()}")
