"""One padded and one truncated product (for an ncu launch list)."""
import sys, torch
sys.path.insert(0, ".")
import paper_1407_3383_b200 as mm, gen
P30, G30 = 998244353, 3
dev = torch.device("cuda:0")
la, bt = int(sys.argv[1]) if len(sys.argv) > 1 else 40000, int(sys.argv[2]) if len(sys.argv) > 2 else 512
a = gen.residues_torch(3, 5, bt * la, P30, dev).view(torch.uint32).reshape(bt, la)
b = gen.residues_torch(3, 6, bt * la, P30, dev).view(torch.uint32).reshape(bt, la)
c = torch.empty((bt, 2 * la - 1), dtype=torch.uint32, device=dev)
for _ in range(2):
    mm.poly_mul(a, b, P30, G30, out=c)
    mm.poly_mul_tft(a, b, P30, G30, out=c)
torch.cuda.synchronize()
