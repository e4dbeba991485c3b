"""Experiment: sub-batch fork streams for C4 (8 x 2^24 Goldilocks forward) and
C3-fwd (4096 x 2^16 forward): S streams of 8/S (4096/S) transforms each."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1407_3383_b200 as mm

dev = torch.device("cuda")
PG = (1 << 64) - (1 << 32) + 1
P30 = 998244353


def run(name, bits, p, g, k, B, dt, S):
    w = pow(g, (p - 1) >> k, p)
    x = gen.residues_torch(gen.config_seed(4), 1, B << k, p, dev)
    x = x.view(torch.uint64) if bits == 64 else x.view(torch.uint32)
    x = x.reshape(B, 1 << k)
    y = torch.empty_like(x)
    W = B // S
    plan = mm.NttPlan(bits, p, k, w, W)
    streams = [torch.cuda.Stream() for _ in range(S)]

    def step():
        cur = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(cur)
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                plan.forward(x[i * W:(i + 1) * W].reshape(-1), out=y[i * W:(i + 1) * W].reshape(-1), order=mm.BITREV)
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
    return round(e0.elapsed_time(e1) / 10, 4)


out = {}
for S in (1, 2, 4):
    out[f"C4_S{S}"] = run("c4", 64, PG, 7, 24, 8, None, S)
    print(S, out[f"C4_S{S}"], flush=True)
for S in (1, 2, 4):
    out[f"C3fwd_S{S}"] = run("c3f", 32, P30, 3, 16, 4096, None, S)
    print(S, out[f"C3fwd_S{S}"], flush=True)
print(json.dumps(out))
