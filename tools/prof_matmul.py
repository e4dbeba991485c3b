"""Per-kernel times of mm_poly_matmul at Table 15's n = 32, d < 2^15 shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1407_3383_b200 as mm

dev = torch.device("cuda")
N, d, p = 32, 1 << 15, 469762049
A = gen.residues_torch(15, 1, N * N * d, p, dev).view(torch.uint32).reshape(N, N, d)
B = gen.residues_torch(15, 2, N * N * d, p, dev).view(torch.uint32).reshape(N, N, d)
C = torch.empty((N, N, 2 * d - 1), dtype=torch.uint32, device=dev)
for _ in range(2):
    mm.poly_matmul(A, B, p, 3, out=C)
torch.cuda.synchronize()
mm.prof_enable(True)
for _ in range(3):
    mm.poly_matmul(A, B, p, 3, out=C)
torch.cuda.synchronize()
mm.prof_enable(False)
print({k: (v[0] // 3, round(v[1] / 3, 4)) for k, v in mm.prof_collect().items()})
