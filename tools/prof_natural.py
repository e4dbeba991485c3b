"""One NATURAL-order C4 forward (8 x 2^24 Goldilocks) for ncu captures of the
mirror permutation (k_bitrev_tiled)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1407_3383_b200 as mm
PG = (1 << 64) - (1 << 32) + 1
dev = torch.device("cuda")
pl = mm.NttPlan(64, PG, 24, pow(7, (PG - 1) >> 24, PG), 8)
x = gen.residues_torch(gen.config_seed(4), 1, 8 << 24, PG, dev).view(torch.uint64)
y = torch.empty_like(x)
for _ in range(2):
    pl.forward(x, out=y, order=mm.NATURAL)
torch.cuda.synchronize()
print("ok")
