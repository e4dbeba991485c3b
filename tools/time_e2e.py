"""C3 through mm_poly_mul_host (pinned host buffers) at several chunk sizes."""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1:
    import torch, gen
    import paper_1407_3383_b200 as mm
    P, G, B, d = 998244353, 3, 4096, 1 << 15
    dev = torch.device("cuda")
    a = gen.residues_torch(gen.config_seed(3), 1, B * d, P, dev).view(torch.uint32).reshape(B, d)
    b = gen.residues_torch(gen.config_seed(3), 2, B * d, P, dev).view(torch.uint32).reshape(B, d)
    ah = torch.empty((B, d), dtype=torch.uint32, pin_memory=True); ah.copy_(a)
    bh = torch.empty((B, d), dtype=torch.uint32, pin_memory=True); bh.copy_(b)
    ch = torch.empty((B, 2 * d - 1), dtype=torch.uint32, pin_memory=True)
    for _ in range(2): mm.poly_mul_host(ah, bh, P, G, out=ch)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): mm.poly_mul_host(ah, bh, P, G, out=ch)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"chunk_mib": os.environ.get("MMNTT_HOST_CHUNK_MIB"), "packed": os.environ.get("MMNTT_HOST_PACKED"),
                      "ms": round(e0.elapsed_time(e1) / 5, 3)}))
else:
    for mib, pk in ((96, 0), (96, 1), (64, 0), (64, 1), (48, 1), (128, 1), (96, 0), (96, 1), (64, 1)):
        env = dict(os.environ, MMNTT_HOST_CHUNK_MIB=str(mib), MMNTT_HOST_PACKED=str(pk))
        print(subprocess.run([sys.executable, __file__, "x"], env=env, capture_output=True, text=True).stdout.strip(),
              flush=True)
