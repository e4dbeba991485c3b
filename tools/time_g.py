"""Goldilocks timing (C4 forward / inverse, C5 int product) with per-kernel
shares from the library's event profiler.  Prints one JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1407_3383_b200 as mm

dev = torch.device("cuda")
PG = (1 << 64) - (1 << 32) + 1


def tloop(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def kern(fn, reps=5):
    mm.set_product_streams(1)   # kernels serialised on one stream: their times add up
    fn()
    torch.cuda.synchronize()
    mm.prof_collect()
    mm.prof_enable(True)
    for _ in range(reps):
        fn()
    r = mm.prof_collect()
    mm.prof_enable(False)
    mm.set_product_streams(2)
    return {k: round(v[1] / reps, 4) for k, v in r.items()}


out = {}
x = gen.residues_torch(gen.config_seed(4), 1, 8 << 24, PG, dev).view(torch.uint64)
plan = mm.NttPlan(64, PG, 24, pow(7, (PG - 1) >> 24, PG), 8)
y = torch.empty_like(x)
z = torch.empty_like(x)
f = lambda: plan.forward(x, out=y, order=mm.BITREV)
g = lambda: plan.inverse(y, out=z, order=mm.BITREV)
out["C4_fwd_ms"] = round(tloop(f), 4)
out["C4_inv_ms"] = round(tloop(g), 4)
mm.set_product_streams(1)
out["C4_fwd_ms_one_stream"] = round(tloop(f), 4)
out["C4_inv_ms_one_stream"] = round(tloop(g), 4)
mm.set_product_streams(2)
out["C4_fwd_kernels"] = kern(f)
out["C4_inv_kernels"] = kern(g)
out["C4_roundtrip_ok"] = bool(torch.equal(z, x))
del x, y, z, plan
n = 1 << 24
a = gen.limbs16_torch(gen.config_seed(5), 1, n, dev).view(torch.uint16)
b = gen.limbs16_torch(gen.config_seed(5), 2, n, dev).view(torch.uint16)
h = lambda: mm.int_mul_u16(a, b)
out["C5_ms"] = round(tloop(h, 5), 4)
mm.set_product_streams(1)
out["C5_ms_one_stream"] = round(tloop(h, 5), 4)
mm.set_product_streams(2)
out["C5_kernels"] = kern(h, 3)
print(json.dumps(out))
