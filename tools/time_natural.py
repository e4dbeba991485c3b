"""C3-fwd shape (4096 x 2^16, p = 998244353): forward / inverse in TFT (bit-
reversed) and natural order."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1407_3383_b200 as mm
P = 998244353
dev = torch.device("cuda")
pl = mm.NttPlan(32, P, 16, pow(3, (P - 1) >> 16, P), 4096)
x = gen.residues_torch(gen.config_seed(3), 3, 4096 << 16, P, dev).view(torch.uint32)
y = torch.empty_like(x)
def t(fn, reps=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)
print(json.dumps({"fwd_bitrev": t(lambda: pl.forward(x, out=y, order=mm.BITREV)),
                  "fwd_natural": t(lambda: pl.forward(x, out=y, order=mm.NATURAL)),
                  "inv_bitrev": t(lambda: pl.inverse(y, out=x, order=mm.BITREV)),
                  "inv_natural": t(lambda: pl.inverse(y, out=x, order=mm.NATURAL))}))
# other four-step sizes (permutation pass through a pool temporary): C4 and 64 x 2^20 32-bit
del x, y, pl
PG = (1 << 64) - (1 << 32) + 1
out = {}
for name, bits, p, g, k, B in (("C4_8x2^24_u64", 64, PG, 7, 24, 8), ("64x2^20_u32", 32, P, 3, 20, 64),
                               ("256x2^18_u64", 64, PG, 7, 18, 256)):
    pl = mm.NttPlan(bits, p, k, pow(g, (p - 1) >> k, p), B)
    x = gen.residues_torch(gen.config_seed(4), 1, B << k, p, dev).view(torch.uint64 if bits == 64 else torch.uint32)
    y = torch.empty_like(x)
    out[name] = {"fwd_bitrev": t(lambda: pl.forward(x, out=y, order=mm.BITREV), 5),
                 "fwd_natural": t(lambda: pl.forward(x, out=y, order=mm.NATURAL), 5),
                 "inv_natural": t(lambda: pl.inverse(y, out=x, order=mm.NATURAL), 5)}
    del pl, x, y
print(json.dumps(out))
