"""Per-kernel times of the C1 call (16 x 2^10 forward + inverse, 512 x 512 product)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1407_3383_b200 as mm

dev = torch.device("cuda")
p = 998244353
x = gen.residues_torch(gen.config_seed(1), 1, 16 << 10, p, dev).view(torch.uint32).reshape(16, 1 << 10)
a = gen.residues_torch(gen.config_seed(1), 2, 512, p, dev).view(torch.uint32).reshape(1, 512)
b = gen.residues_torch(gen.config_seed(1), 3, 512, p, dev).view(torch.uint32).reshape(1, 512)
plan = mm.NttPlan(32, p, 10, pow(3, (p - 1) >> 10, p), 16)
y = torch.empty_like(x)
c = torch.empty((1, 1023), dtype=torch.uint32, device=dev)


def c1():
    plan.forward(x, out=y, order=mm.NATURAL)
    plan.inverse(y, out=y, order=mm.NATURAL)
    mm.poly_mul(a, b, p, 3, out=c)


for _ in range(20):
    c1()
torch.cuda.synchronize()
mm.prof_enable(True)
for _ in range(50):
    c1()
torch.cuda.synchronize()
mm.prof_enable(False)
print({k: (v[0] // 50, round(v[1] / 50 * 1e3, 2)) for k, v in mm.prof_collect().items()}, "us")
