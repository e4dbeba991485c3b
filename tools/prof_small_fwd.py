import os, sys
sys.path.insert(0, "/root/repo")
import torch, gen
import paper_1407_3383_b200 as mm
P = 998244353
dev = torch.device("cuda")
k = int(sys.argv[1]) if len(sys.argv) > 1 else 10
B = 1 << (28 - k)
pl = mm.NttPlan(32, P, k, pow(3, (P - 1) >> k, P), B)
x = gen.residues_torch(gen.config_seed(3), 5, 1 << 28, P, dev).view(torch.uint32)
y = torch.empty_like(x)
for _ in range(2):
    pl.forward(x, out=y, order=mm.BITREV)
torch.cuda.synchronize()
print("ok")
