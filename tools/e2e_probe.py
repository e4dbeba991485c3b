"""Copy-only model of mm_poly_mul_host's pipeline (no kernels): C3's 1 GiB up
and 1 GiB down per step in chunks of `ch` products, three device slots, the
upload of chunk i waiting for the download of chunk i-3; then the same with a
kernel-sized delay (a device busy-wait) in place of the product.  Separates
the copy schedule from the compute interplay."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

B, d, lc = 4096, 1 << 15, (1 << 16) - 1
ah = torch.empty((B, d), dtype=torch.uint32, pin_memory=True)
bh = torch.empty((B, d), dtype=torch.uint32, pin_memory=True)
chh = torch.empty((B, lc), dtype=torch.uint32, pin_memory=True)
up, down, comp = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()


def schedule(ch, ramp):
    """chunk sizes: ramp = (first sizes, last sizes) around chunks of ch"""
    head, tail = ramp
    rest = B - sum(head) - sum(tail)
    mid = [ch] * (rest // ch) + ([rest % ch] if rest % ch else [])
    return list(head) + mid + list(tail)


def run(ch, slots=3, work=None, ramp=((), ())):
    sizes = schedule(ch, ramp)
    mx = max(sizes)
    da = [torch.empty((mx, d), dtype=torch.uint32, device="cuda") for _ in range(slots)]
    db = [torch.empty((mx, d), dtype=torch.uint32, device="cuda") for _ in range(slots)]
    dc = [torch.empty((mx, lc), dtype=torch.uint32, device="cuda") for _ in range(slots)]
    freed = [None] * slots
    nch = len(sizes)
    offs = [sum(sizes[:i]) for i in range(nch)]
    cur = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    up.wait_stream(cur)
    for i in range(nch):
        k = i % slots
        r0, r = offs[i], sizes[i]
        if freed[k] is not None:
            up.wait_event(freed[k])
        with torch.cuda.stream(up):
            da[k][:r].copy_(ah[r0:r0 + r], non_blocking=True)
            db[k][:r].copy_(bh[r0:r0 + r], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(up)
        comp.wait_event(ev)
        if work is not None:
            with torch.cuda.stream(comp):
                work(da[k], db[k], dc[k], r)
        ev2 = torch.cuda.Event()
        ev2.record(comp)
        down.wait_event(ev2)
        with torch.cuda.stream(down):
            chh[r0:r0 + r].copy_(dc[k][:r], non_blocking=True)
        freed[k] = torch.cuda.Event()
        freed[k].record(down)
    cur.wait_stream(down)
    e1.record(cur)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1)


if __name__ == "__main__":
    import paper_1407_3383_b200 as mm
    out = {}

    def prod(a, b, c, r):
        mm.poly_mul(a[:r], b[:r], 998244353, 3, out=c[:r])
    R1 = ((16, 32, 64, 128), (128, 64, 32, 16))
    R2 = ((8, 16, 32, 64, 128), (128, 64, 32, 16, 8))
    for nm, ch, rp in (("flat192", 192, ((), ())), ("ramp1_192", 192, R1), ("ramp2_192", 192, R2),
                       ("ramp1_256", 256, R1), ("ramp2_384", 384, R2)):
        for w in (None, prod):
            t = [run(ch, work=w, ramp=rp) for _ in range(4)]
            out[f"{'prod' if w else 'copy'}_{nm}"] = [round(x, 2) for x in t[1:]]
    print(json.dumps(out))
