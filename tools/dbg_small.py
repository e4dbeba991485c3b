import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_1407_3383_b200 as mm

def run(bits, p, g, k, batch, order, which):
    w = pow(g, (p - 1) >> k, p)
    x = gen.residues(5, k, batch << k, p).reshape(batch, 1 << k)
    plan = mm.NttPlan(bits, p, k, w, batch)
    xt = torch.from_numpy(x).cuda()
    if which == "fwd":
        y = plan.forward(xt, out=torch.empty_like(xt), order=order)
    else:
        y = plan.inverse(xt, out=torch.empty_like(xt), order=order)
    torch.cuda.synchronize()

cfg = sys.argv[1:]
bits, k, batch, order, which = int(cfg[0]), int(cfg[1]), int(cfg[2]), int(cfg[3]), cfg[4]
p, g = (998244353, 3) if bits == 32 else ((1 << 64) - (1 << 32) + 1, 7)
try:
    run(bits, p, g, k, batch, order, which)
    print(cfg, "ok")
except Exception as e:
    print(cfg, "FAIL", str(e)[:60])
