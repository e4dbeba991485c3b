"""mm_poly_mul against the operand length (la = lb = 2^j, 2^27 coefficients
per operand per call): ms and Gbutterfly/s (three transforms of 2^(j+1))."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1407_3383_b200 as mm
dev = torch.device("cuda")
P, PG = 998244353, (1 << 64) - (1 << 32) + 1


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


for bits, p, g, tot in ((32, P, 3, 27), (64, PG, 7, 26)):
    dt = torch.uint32 if bits == 32 else torch.uint64
    A = gen.residues_torch(gen.config_seed(3), 1, 1 << tot, p, dev).view(dt)
    Bm = gen.residues_torch(gen.config_seed(3), 2, 1 << tot, p, dev).view(dt)
    C = torch.empty(2 << tot, dtype=dt, device=dev)
    out = {}
    for j in range(6, 22 if bits == 32 else 24):
        d, B = 1 << j, 1 << (tot - j)
        a, b = A.view(B, d), Bm.view(B, d)
        c = C.view(B, 2 * d)[:, :2 * d - 1]
        ms = t(lambda: mm.poly_mul(a, b, p, g, out=c))
        k = j + 1
        out[j] = {"ms": round(ms, 3), "Gbutterfly_per_s": round(3 * B * (k << (k - 1)) / ms / 1e6, 0)}
    print(json.dumps({"bits": bits, "coefficients_per_operand": 1 << tot, "by_log2_len": out}))
    del A, Bm, C
