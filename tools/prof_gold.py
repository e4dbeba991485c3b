"""ncu driver: one 2^12 x 32768 Goldilocks forward with the canonical root
(gold.cuh tile), then one with w^3 (generic tile)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1407_3383_b200 as mm
PG = (1 << 64) - (1 << 32) + 1
k = int(sys.argv[1]) if len(sys.argv) > 1 else 12
batch = (1 << 27) >> k
x = gen.residues_torch(gen.config_seed(4), 1, batch << k, PG, torch.device("cuda")).view(torch.uint64)
y = torch.empty_like(x)
w = pow(7, (PG - 1) >> k, PG)
for root in (w, pow(w, 3, PG)):
    plan = mm.NttPlan(64, PG, k, root, batch)
    plan.forward(x, out=y, order=mm.BITREV)
torch.cuda.synchronize()
print("ok")
