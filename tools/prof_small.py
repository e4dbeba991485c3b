"""Per-kernel-family device times (library event profiler) of the small
configs: the Table-16 three-prime product (32 x 2^20-bit operands), the same
through the Goldilocks path, and BASELINE C1 (16 x 2^10 fwd+inv + a 512 x 512
product)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1407_3383_b200 as mm

dev = torch.device("cuda")


def kern(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    mm.prof_collect()
    mm.prof_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    r = mm.prof_collect()
    mm.prof_enable(False)
    tot = e0.elapsed_time(e1) / reps
    return {"total_ms_with_events": round(tot, 4), **{k: [v[0] // reps, round(v[1] / reps, 4)] for k, v in r.items()}}


def plain(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps, 4)


out = {}
n32 = 1 << 20
ja = gen.limbs16_torch(gen.config_seed(5), 3, 2 * n32, dev).view(torch.uint32)
jb = gen.limbs16_torch(gen.config_seed(5), 4, 2 * n32, dev).view(torch.uint32)
jc = torch.empty(2 * n32, dtype=torch.uint32, device=dev)
f3 = lambda: mm.int_mul_u32(ja, jb, out=jc)
out["three_prime_ms"] = plain(f3)
out["three_prime_kernels"] = kern(f3)
jc16 = torch.empty(4 * n32, dtype=torch.uint16, device=dev)
fg = lambda: mm.int_mul_u16(ja.view(torch.uint16), jb.view(torch.uint16), out=jc16)
out["goldilocks_ms"] = plain(fg)
out["goldilocks_kernels"] = kern(fg)
P, G = 998244353, 3
w10 = pow(G, (P - 1) >> 10, P)
plan = mm.NttPlan(32, P, 10, w10, 16)
xa = gen.residues_torch(gen.config_seed(1), 1, 16 << 10, P, dev).view(torch.uint32)
pa = gen.residues_torch(gen.config_seed(1), 2, 512, P, dev).view(torch.uint32)
pb = gen.residues_torch(gen.config_seed(1), 3, 512, P, dev).view(torch.uint32)
pc = torch.empty(1023, dtype=torch.uint32, device=dev)


def c1():
    plan.forward(xa, order=mm.NATURAL)
    plan.inverse(xa, order=mm.NATURAL)
    mm.poly_mul(pa, pb, P, G, out=pc)


out["c1_us"] = plain(c1, 200) * 1e3
out["c1_kernels"] = kern(c1, 50)
print(json.dumps(out, indent=1))
