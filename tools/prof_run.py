"""Small driver for ncu captures: one warm-up + one measured call of the
C2 modmul, C3 poly_mul, C4 forward and C5 int_mul paths (select with argv[1])."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1407_3383_b200 as mm

which = sys.argv[1] if len(sys.argv) > 1 else "c3"
dev = torch.device("cuda")
P30, PG = 998244353, (1 << 64) - (1 << 32) + 1
if which == "c3":
    mm.set_product_streams(1)   # whole-batch launches, as bench.py's per-kernel roofline pass
    B, d = 4096, 1 << 15
    a = gen.residues_torch(gen.config_seed(3), 1, B * d, P30, dev).view(torch.uint32).reshape(B, d)
    b = gen.residues_torch(gen.config_seed(3), 2, B * d, P30, dev).view(torch.uint32).reshape(B, d)
    c = torch.empty((B, 1 << 16), dtype=torch.uint32, device=dev)[:, :2 * d - 1]   # bench.py's ldc
    for _ in range(2):
        mm.poly_mul(a, b, P30, 3, out=c)
elif which == "c4":
    x = gen.residues_torch(gen.config_seed(4), 1, 8 << 24, PG, dev).view(torch.uint64)
    plan = mm.NttPlan(64, PG, 24, pow(7, (PG - 1) >> 24, PG), 8)
    y = torch.empty_like(x)
    for _ in range(2):
        plan.forward(x, out=y, order=mm.BITREV)
elif which == "c2":
    n = 1 << 28
    x = gen.residues_torch(gen.config_seed(2), 1, n, 3221225473, dev).view(torch.uint32)
    y = gen.residues_torch(gen.config_seed(2), 2, n, 3221225473, dev).view(torch.uint32)
    z = torch.empty_like(x)
    M = mm.Mod32(3221225473)
    ys = M.shoup_precompute(y)
    for _ in range(2):
        M.mul(x, y, mm.MUL_MONTGOMERY, out=z)
        M.mul(x, y, mm.MUL_SHOUP, y_shoup=ys, out=z)
        M.mul(x, y, mm.MUL_BARRETT, out=z)
elif which == "c5":
    n = 1 << 24
    a = gen.limbs16_torch(gen.config_seed(5), 1, n, dev).view(torch.uint16)
    b = gen.limbs16_torch(gen.config_seed(5), 2, n, dev).view(torch.uint16)
    for _ in range(2):
        mm.int_mul_u16(a, b)
torch.cuda.synchronize()
print("ok", which)
