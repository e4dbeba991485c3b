"""Experiment: C3 products split over S streams (S sub-batches issued
round-robin) so that one sub-batch's memory-bound column passes can overlap
another's ALU-bound product rows."""
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
mm.poly_mul(a, b, P, G, out=c)
ref = cp.clone()
out = {}
for S in [1, 2, 3, 4]:
    streams = [torch.cuda.Stream() for _ in range(S)]
    W = B // S
    def step():
        cur = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(cur)
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                mm.poly_mul(a[i * W:(i + 1) * W], b[i * W:(i + 1) * W], P, G, out=c[i * W:(i + 1) * W])
        for s in streams:
            cur.wait_stream(s)
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
    ok = bool(torch.equal(cp.view(torch.int32)[:, :2 * d - 1], ref.view(torch.int32)[:, :2 * d - 1]))
    out[S] = {"ms": round(ms, 4), "ok": ok}
    print(S, out[S], flush=True)
print(json.dumps(out))
