"""C2 elementwise timings (2^28 residues mod 3221225473): ms and fraction of
the measured HBM copy bandwidth per operation.  Prints one JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import gen
import paper_1407_3383_b200 as mm

dev = torch.device("cuda")
P, n = 3221225473, 1 << 28
x = gen.residues_torch(gen.config_seed(2), 1, n, P, dev).view(torch.uint32)
y = gen.residues_torch(gen.config_seed(2), 2, n, P, dev).view(torch.uint32)
z = torch.empty_like(x)
M = mm.Mod32(P)
ys = M.shoup_precompute(y)
hbm = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists("MEASURED_PEAKS.json") else 6534.5


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


ops = {"add": (lambda: M.add(x, y, out=z), 12), "sub": (lambda: M.sub(x, y, out=z), 12),
       "mont": (lambda: M.mul(x, y, mm.MUL_MONTGOMERY, out=z), 12),
       "barrett": (lambda: M.mul(x, y, mm.MUL_BARRETT, out=z), 12),
       "shoup": (lambda: M.mul(x, y, mm.MUL_SHOUP, y_shoup=ys, out=z), 16),
       "shoup_pre": (lambda: M.shoup_precompute(y, out=z), 8)}
out = {}
for k, (fn, bpe) in ops.items():
    ms = tloop(fn)
    out[k] = {"ms": round(ms, 4), "hbm_frac": round(n * bpe / (ms * 1e-3) / 1e9 / hbm, 3)}
print(json.dumps(out))
