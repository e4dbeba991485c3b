"""32-bit four-step splits: forward ms per 2^28 elements for log2 n = argv[1]
under the split MMNTT_K2_32 selects (unset: the default)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1407_3383_b200 as mm
P = 998244353
dev = torch.device("cuda")
k = int(sys.argv[1])
B = 1 << (28 - k)
pl = mm.NttPlan(32, P, k, pow(3, (P - 1) >> k, P), B)
x = gen.residues_torch(gen.config_seed(3), 5, 1 << 28, P, dev).view(torch.uint32)
y = torch.empty_like(x)
def t(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)
inf = pl.info()
print(json.dumps({"k": k, "n2": inf["n2"], "n1": inf["n1"], "fwd": t(lambda: pl.forward(x, out=y, order=mm.BITREV)),
                  "inv": t(lambda: pl.inverse(y, out=x, order=mm.BITREV))}))
