"""Goldilocks forward transforms of 2^14 .. 2^23 points (2^27 elements per
call) and int products of 2^16 .. 2^22 limbs: ms per call."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import gen
import paper_1407_3383_b200 as mm
PG = (1 << 64) - (1 << 32) + 1
dev = torch.device("cuda")
def tloop(fn, reps=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
out = {}
for k in range(14, 24):
    batch = (1 << 27) >> k
    x = gen.residues_torch(gen.config_seed(4), k, batch << k, PG, dev).view(torch.uint64)
    y = torch.empty_like(x)
    plan = mm.NttPlan(64, PG, k, pow(7, (PG - 1) >> k, PG), batch)
    inf = plan.info()
    out[f"2^{k}"] = [round(tloop(lambda: plan.forward(x, out=y, order=mm.BITREV)), 4), inf["n2"], inf["n1"]]
for lg in (16, 18, 20, 22):
    a = gen.limbs16_torch(gen.config_seed(5), 1, 1 << lg, dev).view(torch.uint16)
    out[f"int_mul_2^{lg}_limbs"] = round(tloop(lambda: mm.int_mul_u16(a, a)), 4)
print(json.dumps(out))
