"""Experiment: C3 products in waves of W products through one per-stream
workspace (the column-pass output stays L2-resident between passes)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1407_3383_b200 as mm

P, G = 998244353, 3
B, d = 4096, 1 << 15
dev = torch.device("cuda")
a = gen.residues_torch(gen.config_seed(3), 1, B * d, P, dev).view(torch.uint32).reshape(B, d)
b = gen.residues_torch(gen.config_seed(3), 2, B * d, P, dev).view(torch.uint32).reshape(B, d)
cp = torch.empty((B, 1 << 16), dtype=torch.uint32, device=dev)
c = cp[:, :2 * d - 1]
ref = None
out = {}
for W in [4096, 1024, 512, 256, 128, 64, 32]:
    def step():
        for i in range(0, B, W):
            mm.poly_mul(a[i:i + W], b[i:i + W], P, G, out=c[i:i + W])
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    if ref is None:
        ref = cp.clone()
    ok = bool(torch.equal(cp.view(torch.int32)[:, :2 * d - 1], ref.view(torch.int32)[:, :2 * d - 1]))
    out[W] = {"ms": round(ms, 4), "ok": ok}
    print(W, out[W], flush=True)
print(json.dumps(out))
