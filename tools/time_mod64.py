"""Goldilocks elementwise operations (2^27 residues): ms and fraction of the
measured HBM copy bandwidth (24 bytes per element)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1407_3383_b200 as mm
PG, n = (1 << 64) - (1 << 32) + 1, 1 << 27
dev = torch.device("cuda")
x = gen.residues_torch(gen.config_seed(4), 1, n, PG, dev).view(torch.uint64)
y = gen.residues_torch(gen.config_seed(4), 2, n, PG, dev).view(torch.uint64)
z = torch.empty_like(x)
M = mm.Mod64(PG)
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
try:
    hbm = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    hbm = 6534.5
out = {}
for nm, fn in (("add", lambda: M.add(x, y, out=z)), ("sub", lambda: M.sub(x, y, out=z)), ("mul", lambda: M.mul(x, y, out=z))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    out[nm] = {"ms": round(ms, 4), "hbm_frac": round(24 * n / (ms * 1e-3) / 1e9 / hbm, 3)}
print(json.dumps(out))
