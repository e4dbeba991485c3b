"""64 x 2^20 forward NTTs by residue type (u32 p = 998244353, FP64 p = 63 2^44 + 1,
Goldilocks): ms per call and per-kernel times (one stream).  Prints one JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1407_3383_b200 as mm

dev = torch.device("cuda")


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


out = {}
for name, bits, p, g in (("u32", 32, 998244353, 3), ("f64", 52, 1108307720798209, 11), ("gold", 64, (1 << 64) - (1 << 32) + 1, 7)):
    if bits == 52:
        x = gen.residues_torch(9, 1, 64 << 20, p, dev).view(torch.int64).to(torch.float64)
    else:
        x = gen.residues_torch(9, 1, 64 << 20, p, dev)
        x = x.view(torch.uint32) if bits == 32 else x.view(torch.uint64)
    w = pow(g, (p - 1) >> 20, p)
    plan = mm.NttPlan(bits, p, 20, w, 64)
    y = torch.empty_like(x)
    f = lambda: plan.forward(x, out=y, order=mm.BITREV)
    ms = tloop(f)
    mm.set_product_streams(1)
    ms1 = tloop(f)
    f()
    torch.cuda.synchronize()
    mm.prof_collect()
    mm.prof_enable(True)
    for _ in range(5):
        f()
    r = mm.prof_collect()
    mm.prof_enable(False)
    mm.set_product_streams(2)
    out[name] = {"ms": round(ms, 4), "ms_one_stream": round(ms1, 4), "info": plan.info(),
                 "kernels_ms": {k: round(v[1] / 5, 4) for k, v in r.items()}}
    del x, y, plan
print(json.dumps(out))
