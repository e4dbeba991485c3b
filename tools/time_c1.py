"""C1 (16 x 2^10 forward + inverse, NATURAL, and one 512 x 512 product) per
call in a CUDA graph: serial capture, and with the independent product on a
second branch of the graph; plus 64 x 2^20 forward (rows of 2^10)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen
import paper_1407_3383_b200 as mm
dev = torch.device("cuda")
p = 998244353
x = gen.residues_torch(gen.config_seed(1), 1, 16 << 10, p, dev).view(torch.uint32)
pa = gen.residues_torch(gen.config_seed(1), 2, 512, p, dev).view(torch.uint32)
pb = gen.residues_torch(gen.config_seed(1), 3, 512, p, dev).view(torch.uint32)
pc = torch.empty(1023, dtype=torch.uint32, device=dev)
plan = mm.NttPlan(32, p, 10, pow(3, (p - 1) >> 10, p), 16)
side = torch.cuda.Stream()
def serial():
    plan.forward(x, order=mm.NATURAL)
    plan.inverse(x, order=mm.NATURAL)
    mm.poly_mul(pa, pb, p, 3, out=pc)
def forked():
    cur = torch.cuda.current_stream()
    side.wait_stream(cur)
    with torch.cuda.stream(side):
        mm.poly_mul(pa, pb, p, 3, out=pc)
    plan.forward(x, order=mm.NATURAL)
    plan.inverse(x, order=mm.NATURAL)
    cur.wait_stream(side)
def graph_time(fn, reps=500):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        with torch.cuda.graph(g, stream=s):
            fn()
    torch.cuda.synchronize()
    for _ in range(20): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): g.replay()
    e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / reps * 1e3, 2)
out = {"c1_graph_serial_us": graph_time(serial), "c1_graph_forked_us": graph_time(forked)}
k = 20
p20 = mm.NttPlan(32, p, k, pow(3, (p - 1) >> k, p), 64)
xx = gen.residues_torch(10, 1, 64 << k, p, dev).view(torch.uint32)
yy = torch.empty_like(xx)
for _ in range(3): p20.forward(xx, out=yy, order=mm.BITREV)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): p20.forward(xx, out=yy, order=mm.BITREV)
e1.record(); torch.cuda.synchronize()
out["fwd_64x2^20_ms"] = round(e0.elapsed_time(e1) / 10, 4)
print(json.dumps(out))
