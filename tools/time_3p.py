"""Three-prime integer product (mm_int_mul_u32) at Table 16's
largest size (two 2^20-limb operands): time per call and per-kernel shares
from the library's event profiler.  Prints one JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1407_3383_b200 as mm

dev = torch.device("cuda")
n32 = 1 << 20
ja = gen.limbs16_torch(gen.config_seed(5), 3, 2 * n32, dev).view(torch.uint32)
jb = gen.limbs16_torch(gen.config_seed(5), 4, 2 * n32, dev).view(torch.uint32)
jc = torch.empty(2 * n32, dtype=torch.uint32, device=dev)
f = lambda: mm.int_mul_u32(ja, jb, out=jc)


def tloop(fn, reps=20, warm=3):
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


out = {"ms": round(tloop(f), 4)}
mm.prof_collect()
mm.prof_enable(True)
for _ in range(5):
    f()
r = mm.prof_collect()
mm.prof_enable(False)
out["kernels_ms"] = {k: round(v[1] / 5, 4) for k, v in r.items()}
out["launches_per_call"] = {k: v[0] / 5 for k, v in r.items()}
print(json.dumps(out))
