import json, os, sys
sys.path.insert(0, "/root/repo")
import torch, gen, numpy as np
import paper_1407_3383_b200 as mm
import oracle as O
P = 998244353
dev = torch.device("cuda")
def t(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)
k = 13
B = 1 << (28 - k)
w = pow(3, (P - 1) >> k, P)
pl = mm.NttPlan(32, P, k, w, B)
print(pl.info())
x = gen.residues_torch(gen.config_seed(3), 5, 1 << 28, P, dev).view(torch.uint32)
y = torch.empty_like(x)
r = {"fwd": t(lambda: pl.forward(x, out=y, order=mm.BITREV)), "inv": t(lambda: pl.inverse(y, out=x, order=mm.BITREV)),
     "nat": t(lambda: pl.forward(x, out=y, order=mm.NATURAL))}
# correctness of row 0 and the last row vs the oracle
pl.forward(x, out=y, order=mm.NATURAL)
for row in (0, B - 1):
    xr = x.view(B, 1 << k)[row].cpu().numpy().astype(np.uint64)
    assert np.array_equal(y.view(B, 1 << k)[row].cpu().numpy().astype(np.uint64), O.ntt(xr, w, P)), row
d = 1 << 12
Bp = 1 << 15
a = x[:Bp * d].view(Bp, d); b = x[Bp * d:2 * Bp * d].view(Bp, d)
c = torch.empty((Bp, 2 * d), dtype=torch.uint32, device=dev)[:, :2 * d - 1]
r["pmul_la4096"] = t(lambda: mm.poly_mul(a, b, P, 3, out=c))
mm.poly_mul(a, b, P, 3, out=c)
for row in (0, Bp - 1):
    assert np.array_equal(c[row].cpu().numpy().astype(np.uint64), O.poly_mul_ntt(a[row].cpu().numpy(), b[row].cpu().numpy(), P, 3)), row
print(json.dumps(r))
