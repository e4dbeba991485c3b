"""Time mm_poly_mul_tft against the padded mm_poly_mul."""
import sys, torch
sys.path.insert(0, ".")
import paper_1407_3383_b200 as mm, gen
P30, G30 = 998244353, 3
dev = torch.device("cuda:0")


def tloop(fn, reps=5, warm=3):
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


for la, bt in [(33000, 512), (40000, 512), (49152, 512), (60000, 256), (2100, 8192), (5000, 4096), (300000, 64)]:
    a = gen.residues_torch(3, 5, bt * la, P30, dev).view(torch.uint32).reshape(bt, la)
    b = gen.residues_torch(3, 6, bt * la, P30, dev).view(torch.uint32).reshape(bt, la)
    c = torch.empty((bt, 2 * la - 1), dtype=torch.uint32, device=dev)
    c2 = torch.empty_like(c)
    msp = tloop(lambda: mm.poly_mul(a, b, P30, G30, out=c))
    mst = tloop(lambda: mm.poly_mul_tft(a, b, P30, G30, out=c2))
    assert torch.equal(c, c2)
    print(f"batch {bt} la=lb={la}: padded {msp:.3f} ms  tft {mst:.3f} ms  x{msp / mst:.2f}", flush=True)
