"""Small driver for compute-sanitizer runs over the TMA / bulk-copy kernels:
one 2^24 Goldilocks transform each way (column tiles, bulk-copied rows),
one 2^25-point integer product (16-bit limb super-tiles, fused product rows,
inverse columns, carries), one mm_run_jobs call.  Exits 0 when the results
round-trip / match a second path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1407_3383_b200 as mm

dev = torch.device("cuda")
PG = (1 << 64) - (1 << 32) + 1
x = gen.residues_torch(gen.config_seed(4), 31, 1 << 24, PG, dev).view(torch.uint64)
plan = mm.NttPlan(64, PG, 24, pow(7, (PG - 1) >> 24, PG), 1)
y = plan.forward(x, out=torch.empty_like(x), order=mm.BITREV)
z = plan.inverse(y, out=torch.empty_like(y), order=mm.BITREV)
assert torch.equal(z, x)
n = 1 << 24
a = gen.limbs16_torch(gen.config_seed(5), 31, n, dev).view(torch.uint16)
b = gen.limbs16_torch(gen.config_seed(5), 32, n, dev).view(torch.uint16)
c = mm.int_mul_u16(a, b)
torch.cuda.synchronize()
P30 = 998244353
w = pow(3, (P30 - 1) >> 10, P30)
p10 = mm.NttPlan(32, P30, 10, w, 4)
xs = gen.residues_torch(1, 33, 4 << 10, P30, dev).view(torch.uint32).view(4, 1024)
zs = torch.empty_like(xs)
jb = mm.Jobs()
for r in range(4):
    jb.roundtrip(p10, xs[r], zs[r])
jb.run()
torch.cuda.synchronize()
assert torch.equal(zs, xs)
print("sanitize driver ok")
