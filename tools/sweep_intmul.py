"""mm_int_mul_u16 / mm_int_mul_u32 against the operand size: ms per product
and Gbit/s of operand bits (2 x 16 na)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1407_3383_b200 as mm
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


out = {"u16_goldilocks": {}, "u32_three_primes": {}}
for lg in range(10, 25):
    n = 1 << lg
    a = gen.limbs16_torch(gen.config_seed(5), 1, n, dev).view(torch.uint16)
    b = gen.limbs16_torch(gen.config_seed(5), 2, n, dev).view(torch.uint16)
    c = torch.empty(2 * n, dtype=torch.uint16, device=dev)
    ms = t(lambda: mm.int_mul_u16(a, b, out=c))
    out["u16_goldilocks"][lg] = {"ms": round(ms, 4), "Gbit_per_s": round(32 * n / ms / 1e6, 1)}
for lg in range(9, 21):
    n = 1 << lg
    a = gen.limbs16_torch(gen.config_seed(5), 1, 2 * n, dev).view(torch.uint32)
    b = gen.limbs16_torch(gen.config_seed(5), 2, 2 * n, dev).view(torch.uint32)
    c = torch.empty(2 * n, dtype=torch.uint32, device=dev)
    try:
        ms = t(lambda: mm.int_mul_u32(a, b, out=c))
        out["u32_three_primes"][lg] = {"ms": round(ms, 4), "Gbit_per_s": round(64 * n / ms / 1e6, 1)}
    except Exception as e:
        out["u32_three_primes"][lg] = {"error": str(e)[:80]}
print(json.dumps(out))
