"""Experiment: per-kernel times of the C3 product for aligned vs unaligned
output rows (lc = 65535 vs 65536)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1407_3383_b200 as mm

dev = torch.device("cuda")
P = 998244353
B = 4096
for la, lb in [(1 << 15, 1 << 15), (1 << 15, (1 << 15) + 1), (1 << 15, (1 << 15) - 255)]:
    a = gen.residues_torch(3, 1, B * la, P, dev).view(torch.uint32).reshape(B, la)
    b = gen.residues_torch(3, 2, B * lb, P, dev).view(torch.uint32).reshape(B, lb)
    c = torch.empty((B, la + lb - 1), dtype=torch.uint32, device=dev)
    for _ in range(3):
        mm.poly_mul(a, b, P, 3, out=c)
    torch.cuda.synchronize()
    mm.prof_enable(True)
    for _ in range(5):
        mm.poly_mul(a, b, P, 3, out=c)
    torch.cuda.synchronize()
    mm.prof_enable(False)
    pr = mm.prof_collect()
    print(la, lb, {k: round(v[1] / v[0], 4) for k, v in pr.items()}, flush=True)
    del a, b, c
