"""Forward / inverse transform and product throughput against the transform size:
32-bit (p = 998244353) k = 8..23 at 2^28 elements per call, Goldilocks k = 8..25
at 2^27 elements per call.  One JSON line per word size."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1407_3383_b200 as mm
P, PG = 998244353, (1 << 64) - (1 << 32) + 1
dev = torch.device("cuda")


def t(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for bits, p, g, total, ks in ((32, P, 3, 28, range(8, 24)), (64, PG, 7, 27, range(8, 26))):
    x = gen.residues_torch(gen.config_seed(3), 5, 1 << total, p, dev).view(torch.uint64 if bits == 64 else torch.uint32)
    y = torch.empty_like(x)
    out = {}
    for k in ks:
        B = 1 << (total - k)
        pl = mm.NttPlan(bits, p, k, pow(g, (p - 1) >> k, p), B)
        bf = B * (k << (k - 1)) / 1e9
        f = t(lambda: pl.forward(x, out=y, order=mm.BITREV))
        i = t(lambda: pl.inverse(y, out=x, order=mm.BITREV))
        n = t(lambda: pl.forward(x, out=y, order=mm.NATURAL))
        out[k] = {"fwd_ms": round(f, 3), "inv_ms": round(i, 3), "nat_ms": round(n, 3), "fwd_Gbfly": round(bf / f * 1e3, 0)}
        del pl
    print(json.dumps({"bits": bits, "elements": 1 << total, "by_log2n": out}))
    del x, y
    mm.release_cached() if hasattr(mm, "release_cached") else None
