import sys, torch
sys.path.insert(0, ".")
import paper_1407_3383_b200 as mm, gen
P30=998244353
dev=torch.device("cuda:0")
la,bt=2049,2
a = gen.residues_torch(3, 5, bt * la, P30, dev).view(torch.uint32).reshape(bt, la)
b = gen.residues_torch(3, 6, bt * la, P30, dev).view(torch.uint32).reshape(bt, la)
c=mm.poly_mul(a,b,P30,3); d=mm.poly_mul_tft(a,b,P30,3)
torch.cuda.synchronize()
bad=(c!=d).nonzero()
print("bad", bad.shape[0], bad[:10].tolist())
