"""Fast (gold.cuh) vs generic Goldilocks tiles: same sizes, canonical root
(fast path) vs the root w^3 (generic path, same layout)."""
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
for k, batch in [(11, 1 << 16), (12, 1 << 15), (13, 1 << 14), (24, 8)]:
    x = gen.residues_torch(gen.config_seed(4), 1, batch << k, PG, dev).view(torch.uint64)
    y = torch.empty_like(x)
    w = pow(7, (PG - 1) >> k, PG)
    for name, root in [("fast", w), ("generic", pow(w, 3, PG))]:
        plan = mm.NttPlan(64, PG, k, root, batch)
        ms = tloop(lambda: plan.forward(x, out=y, order=mm.BITREV))
        msi = tloop(lambda: plan.inverse(x, out=y, order=mm.BITREV))
        out[f"2^{k}x{batch}_{name}"] = {"fwd_ms": round(ms, 4), "inv_ms": round(msi, 4),
                                         "Gbfly_s": round(batch * (1 << (k - 1)) * k / ms / 1e6, 1)}
print(json.dumps(out, indent=1))
