#!/usr/bin/env python
"""bench.py -- throughput of the B200 hot path of arXiv 1407.3383.

Contract (driver): python bench.py --gpus N --steps K --warmup W [--impl reference]
  N > 1 is launched by torchrun (one rank per GPU, NCCL); rank 0 prints ONE
  JSON line.

Headline workload (config.workload): BASELINE C3 -- 4096 independent
products of two polynomials of degree < 2^15 over p = 998244353 (generator 3),
i.e. per product two forward NTTs of length 2^16, the pointwise product and
one inverse NTT.  One step = one mm_poly_mul over the whole batch.
Metric: NTT Gbutterfly/s = 3 * (n/2) log2 n butterflies per product / time.
Weak scaling: every rank runs its own 4096 products (its own generator range).

Secondary measurements (C1, C2, C4, C5 and the ALU probe) go in "extra".
--impl reference times the CPU oracle (oracle/, test infrastructure) on the
same workload, a bounded sample per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

P30, G30 = 998244353, 3
P32 = 3221225473
PG = (1 << 64) - (1 << 32) + 1

C3_BATCH, C3_D = 4096, 1 << 15        # products per rank, coefficients per operand
C3_LOG = 16                           # transform length 2^16
C3_BFLY_PER_PROD = 3 * (1 << (C3_LOG - 1)) * C3_LOG
C3_LDC = 1 << C3_LOG                  # output row stride (words): 128-byte aligned rows


def c3_butterflies(batch: int) -> int:
    return batch * C3_BFLY_PER_PROD


# ----------------------------------------------------------------------------- helpers
def load_peaks() -> dict:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {}


HBM_FALLBACK_GBS = 6650.0


def root_of_unity(p: int, g: int, k: int) -> int:
    """w = g^((p-1)/2^k): a primitive 2^k-th root for a generator g (plan input)."""
    return pow(g, (p - 1) >> k, p)


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML
    (pynvml) polled every 2 ms from a thread, else nvidia-smi at 100 ms."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.samples = []          # (sm_mhz, max_mhz, reason bits) from NVML
        self.stop = threading.Event()
        self.nvml = None

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.nvml = (pynvml, h)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
        except Exception:
            self.nvml = None
        try:
            fields = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
                      "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
                      "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={','.join(fields)}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def mark(self, start: bool):
        """Bracket the timed region (samples outside it are dropped when any fall inside)."""
        n = len(self.samples)
        if start:
            self.i0 = n
        else:
            self.i1 = n

    def _poll(self):
        nv, h = self.nvml
        try:
            mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        except Exception:
            mx = 0
        reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            getattr(nv, "nvmlDeviceGetCurrentClocksThrottleReasons", None)
        while not self.stop.is_set():
            try:
                clk = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                bits = reasons(h) if reasons else 0
                self.samples.append((clk, mx, bits))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        i0, i1 = getattr(self, "i0", 0), getattr(self, "i1", None)
        if self.samples and i1 is not None and i1 > i0 + 2:
            self.samples = self.samples[i0:i1]
        for clk, m, bits in self.samples:
            sm.append(float(clk))
            mx = max(mx, float(m))
            for nm, bit in self.REASONS.items():
                if bits & bit:
                    reasons.add(nm)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml" if self.samples else "nvidia-smi"}


def dist_setup():
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(world, value: float) -> float:
    if world == 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def timed(fn, steps, warmup, world, stream=None, on_start=None, on_stop=None):
    """W untimed steps, then K steps bracketed by barrier + synchronize; CUDA
    events on the launching stream; returns max-over-ranks ms for K steps."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    if on_start:
        on_start()
    st = stream or torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(steps):
        fn()
    e1.record(st)
    if on_stop:
        on_stop()
    torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(world, e0.elapsed_time(e1))


# ----------------------------------------------------------------------------- CPU oracle (reference arm)
def oracle_c3_sample(nprod: int, seed_off: int = 0, budget_s: float | None = None) -> tuple[float, int]:
    """Time the oracle (as it stands) on nprod C3 products (or as many as fit in
    budget_s seconds); returns (s, butterflies)."""
    import gen
    import oracle as O
    O.build()
    t = 0.0
    done = 0
    for i in range(nprod if budget_s is None else 1 << 30):
        if budget_s is not None and t >= budget_s:
            break
        done += 1
        a = gen.residues(gen.config_seed(3), 1, C3_D, P30, start=(seed_off + i) * C3_D)
        b = gen.residues(gen.config_seed(3), 2, C3_D, P30, start=(seed_off + i) * C3_D)
        t0 = time.perf_counter()
        O.poly_mul_ntt(a, b, P30, G30)
        t += time.perf_counter() - t0
    return t, done * C3_BFLY_PER_PROD


def run_reference(args, world, rank):
    if rank != 0:
        return
    # size one step so that W + K steps take ~ a couple of minutes at most
    t1, _ = oracle_c3_sample(1)
    per_step = max(1, min(400, int(6.0 / max(t1, 1e-3))))
    for _ in range(args.warmup):
        oracle_c3_sample(per_step)
    tot_t, tot_b = 0.0, 0
    for s in range(args.steps):
        t, b = oracle_c3_sample(per_step, seed_off=s * per_step)
        tot_t += t
        tot_b += b
    val = tot_b / tot_t / 1e9
    line = {
        "impl": "reference", "metric": "NTT Gbutterfly/s", "value": round(val, 6), "unit": "Gbutterfly/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot_t / args.steps, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded SplitMix64, uniform in [0,p))",
        "config": {"workload": f"C3 poly_mul sample: {per_step} of the 4096 products per step "
                               f"(deg < 2^15, n = 2^16, p = 998244353)",
                   "sample_products_per_step": per_step, "parallelism": "single CPU thread"},
        "cpu_baseline": {"value": round(val, 6), "unit": "Gbutterfly/s", "cores": 1, "kind": "oracle",
                         "sample": f"{per_step} products x {args.steps} steps of the C3 workload"},
        "e2e": {"value": round(val, 6), "unit": "Gbutterfly/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def extras_run(mm, torch, dev, peaks):
    """Secondary configs on rank 0 / N = 1 (C1, C2, C4, C5, ALU probe)."""
    import gen
    out = {}
    hbm = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)

    def tloop(fn, reps, warm=3):
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

    # ALU probe (register-only butterflies) and per-class instruction issue rates
    b32 = mm.probe_butterfly(32, 4000)
    b64 = mm.probe_butterfly(64, 1000)
    bg8 = mm.probe_butterfly(65, 1000)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    clk = peaks.get("sm_max_mhz", 1965.0) * 1e6
    issue = {}
    for kind, nm in enumerate(["IMAD", "IMAD.HI", "IADD3", "VIADDMNMX", "IMAD.HI+2xIADD3", "DFMA"]):
        r = mm.probe_issue(kind, 4000)
        issue[nm] = round(r / (nsm * clk), 3)
    out["alu_probe"] = {"bfly32_G_per_s": round(b32 / 1e9, 1), "bfly64_G_per_s": round(b64 / 1e9, 1),
                        "gold8_G_per_s": round(bg8 / 1e9, 1),
                        "warp_inst_per_clk_per_SM": issue,
                        "note": "register-resident butterflies / single-class instruction chains, full grid, "
                                "no memory traffic; per-clk rates at the max SM clock"}

    # C2: elementwise over 2^28 uint32 pairs, p = 3221225473
    n = 1 << 28
    x = gen.residues_torch(gen.config_seed(2), 1, n, P32, dev).view(torch.uint32)
    y = gen.residues_torch(gen.config_seed(2), 2, n, P32, dev).view(torch.uint32)
    z = torch.empty_like(x)
    M = mm.Mod32(P32)
    ys = M.shoup_precompute(y)
    c2 = {}
    for name, fn, bytes_per in [
        ("modadd", lambda: M.add(x, y, out=z), 12),
        ("modsub", lambda: M.sub(x, y, out=z), 12),
        ("modmul_montgomery", lambda: M.mul(x, y, mm.MUL_MONTGOMERY, out=z), 12),
        ("modmul_barrett", lambda: M.mul(x, y, mm.MUL_BARRETT, out=z), 12),
        ("modmul_shoup", lambda: M.mul(x, y, mm.MUL_SHOUP, y_shoup=ys, out=z), 16),
        ("shoup_precompute", lambda: M.shoup_precompute(y, out=z), 8),
    ]:
        ms = tloop(fn, 10)
        gbs = n * bytes_per / (ms * 1e-3) / 1e9
        c2[name] = {"Gelem_per_s": round(n / (ms * 1e-3) / 1e9, 1), "ms": round(ms, 4),
                    "GB_per_s": round(gbs, 1), "hbm_frac": round(gbs / hbm, 3)}
    out["C2_elementwise_2^28_p3221225473"] = c2
    del x, y, z, ys

    # C1: 16 x (fwd + inv) NTT 2^10 + one 512 x 512 product, p = 998244353
    w10 = root_of_unity(P30, G30, 10)
    plan = mm.NttPlan(32, P30, 10, w10, 16)
    xa = gen.residues_torch(gen.config_seed(1), 1, 16 << 10, P30, dev).view(torch.uint32)
    pa = gen.residues_torch(gen.config_seed(1), 2, 512, P30, dev).view(torch.uint32)
    pb = gen.residues_torch(gen.config_seed(1), 3, 512, P30, dev).view(torch.uint32)
    pc = torch.empty(1023, dtype=torch.uint32, device=dev)

    def c1():
        plan.forward(xa, order=mm.NATURAL)
        plan.inverse(xa, order=mm.NATURAL)
        mm.poly_mul(pa, pb, P30, G30, out=pc)

    ms = tloop(c1, 200)
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        c1()
        with torch.cuda.graph(g, stream=s):
            c1()
    torch.cuda.synchronize()
    ms_graph = tloop(g.replay, 200)
    bf = 16 * 2 * 5 * 512 + 3 * 5 * 512
    out["C1_16x2^10_fwd_inv_plus_poly511"] = {"us_per_call": round(ms * 1e3, 2),
                                             "us_per_call_cuda_graph": round(ms_graph * 1e3, 2),
                                             "Gbutterfly_per_s_graph": round(bf / (ms_graph * 1e-3) / 1e9, 2)}

    # FP64 FMA reduction (Functions 16-18), 2^27 doubles, p = 63 2^44 + 1
    p50, nf = 1108307720798209, 1 << 27
    xf = (gen.residues_torch(9, 1, nf, p50, dev).view(torch.int64)).to(torch.float64)
    yf = (gen.residues_torch(9, 2, nf, p50, dev).view(torch.int64)).to(torch.float64)
    zf = torch.empty_like(xf)
    MF = mm.ModF64(p50)
    c3f = {}
    for name, fn in [("modadd_f64", lambda: MF.add(xf, yf, out=zf)), ("modmul_f64", lambda: MF.mul(xf, yf, out=zf))]:
        msf = tloop(fn, 10)
        c3f[name] = {"Gelem_per_s": round(nf / (msf * 1e-3) / 1e9, 1), "ms": round(msf, 4),
                     "hbm_frac": round(nf * 24 / (msf * 1e-3) / 1e9 / hbm, 3)}
    out["f64_elementwise_2^27_p63x2^44+1"] = c3f
    del xf, yf, zf

    # C3-fwd: 4096 forward NTTs of length 2^16 (TFT order), and the inverse
    pl16 = mm.NttPlan(32, P30, 16, root_of_unity(P30, G30, 16), 4096)
    x16 = gen.residues_torch(gen.config_seed(3), 3, 4096 << 16, P30, dev).view(torch.uint32)
    y16 = torch.empty_like(x16)
    msf = tloop(lambda: pl16.forward(x16, out=y16, order=mm.BITREV), 10)
    msi = tloop(lambda: pl16.inverse(y16, out=x16, order=mm.BITREV), 10)
    bf16 = 4096 * (1 << 15) * 16
    out["C3_fwd_4096x2^16"] = {"forward_ms": round(msf, 4), "forward_Gbutterfly_per_s": round(bf16 / (msf * 1e-3) / 1e9, 1),
                               "inverse_ms": round(msi, 4), "inverse_Gbutterfly_per_s": round(bf16 / (msi * 1e-3) / 1e9, 1),
                               "hbm_frac_2pass": round(4 * 4096 * (1 << 16) * 4 / (msf * 1e-3) / 1e9 / hbm, 3)}
    del x16, y16, pl16

    # the same batched forward NTT (64 x 2^20) over the three residue types:
    # 32-bit Shoup (p < 2^30), FP64 Function 16 (Table 12's 50-bit prime), Goldilocks
    cmp = {}
    kk20, bt = 20, 64
    for tag, bits, pp, g, dt in [("u32_p998244353", 32, P30, 3, None), ("f64_p63x2^44+1", 52, 1108307720798209, 11, "f"),
                                 ("u64_goldilocks", 64, PG, 7, None)]:
        xs = gen.residues_torch(10, 1, bt << kk20, pp, dev)
        if dt == "f":
            xs = xs.to(torch.float64)
        elif bits == 32:
            xs = xs.view(torch.uint32)
        else:
            xs = xs.view(torch.uint64)
        pl = mm.NttPlan(bits, pp, kk20, root_of_unity(pp, g, kk20), bt)
        ys = torch.empty_like(xs)
        msn = tloop(lambda: pl.forward(xs, out=ys, order=mm.BITREV), 10)
        cmp[tag] = {"ms": round(msn, 4), "Gbutterfly_per_s": round(bt * (1 << (kk20 - 1)) * kk20 / (msn * 1e-3) / 1e9, 1)}
        del xs, ys, pl
    out["ntt_fwd_64x2^20_by_residue_type"] = cmp

    # C3 with the packed output layout (ldc = 2^16 - 1: rows not 32-byte aligned)
    a3 = gen.residues_torch(gen.config_seed(3), 1, C3_BATCH * C3_D, P30, dev).view(torch.uint32).reshape(C3_BATCH, C3_D)
    b3 = gen.residues_torch(gen.config_seed(3), 2, C3_BATCH * C3_D, P30, dev).view(torch.uint32).reshape(C3_BATCH, C3_D)
    c3 = torch.empty((C3_BATCH, 2 * C3_D - 1), dtype=torch.uint32, device=dev)
    ms = tloop(lambda: mm.poly_mul(a3, b3, P30, G30, out=c3), 10)
    out["C3_packed_output"] = {"ms": round(ms, 4), "Gbutterfly_per_s": round(c3_butterflies(C3_BATCH) / (ms * 1e-3) / 1e9, 1),
                               "note": "same C3 products, c rows packed at 2^16 - 1 words"}
    del a3, b3, c3

    def kern_ms(fn, reps=5):
        # per-family kernel time per call (library event profiler, launching stream)
        fn()
        torch.cuda.synchronize()
        mm.prof_collect()
        mm.prof_enable(True)
        for _ in range(reps):
            fn()
        r = mm.prof_collect()
        mm.prof_enable(False)
        return {k: round(v[1] / reps, 4) for k, v in r.items()}

    # C4: 8 x 2^24 Goldilocks forward NTT (four-step 2^11 columns x 2^13 rows, gold.cuh tiles)
    w24 = root_of_unity(PG, 7, 24)
    plan4 = mm.NttPlan(64, PG, 24, w24, 8)
    x4 = gen.residues_torch(gen.config_seed(4), 1, 8 << 24, PG, dev).view(torch.uint64)
    y4 = torch.empty_like(x4)
    f4 = lambda: plan4.forward(x4, out=y4, order=mm.BITREV)
    ms = tloop(f4, 10)
    bfly = 8 * (1 << 23) * 24
    gbs2 = 8 * (1 << 24) * 32 / (ms * 1e-3) / 1e9
    inf4 = plan4.info()
    out["C4_8x2^24_goldilocks_fwd"] = {"ms": round(ms, 3), "Gbutterfly_per_s": round(bfly / (ms * 1e-3) / 1e9, 1),
                                       "GB_per_s_2pass": round(gbs2, 1), "hbm_frac_2pass": round(gbs2 / hbm, 3),
                                       "split": f"{inf4['n2']} cols x {inf4['n1']} rows", "kernels_ms": kern_ms(f4),
                                       "alu_frac_vs_gold8_probe": round(bfly / (ms * 1e-3) / bg8, 3),
                                       "alu_note": "achieved butterflies / register-resident gold.cuh 8-point rate "
                                                   "(the passes also carry the w_L and step-2 table products)"}
    del x4, y4, plan4

    # C5: 2^28-bit x 2^28-bit integer product (2^24 16-bit limbs each)
    na = 1 << 24
    ia = gen.limbs16_torch(gen.config_seed(5), 1, na, dev).view(torch.uint16)
    ib = gen.limbs16_torch(gen.config_seed(5), 2, na, dev).view(torch.uint16)
    ic = torch.empty(2 * na, dtype=torch.uint16, device=dev)
    f5 = lambda: mm.int_mul_u16(ia, ib, out=ic)
    ms = tloop(f5, 10)
    out["C5_int_mul_2^28bit"] = {"ms": round(ms, 3), "Mbit_per_s": round(2 * (1 << 28) / (ms * 1e-3) / 1e6, 1),
                                 "Gbutterfly_per_s": round(3 * (1 << 24) * 25 / (ms * 1e-3) / 1e9, 1),
                                 "kernels_ms": kern_ms(f5)}
    # polynomial matrix product (Table 15: n x n, d < 2^15 over 469762049)
    pm = {}
    for N in (8, 32):
        d, pp = 1 << 15, 469762049
        A = gen.residues_torch(15, 1, N * N * d, pp, dev).view(torch.uint32).reshape(N, N, d)
        B = gen.residues_torch(15, 2, N * N * d, pp, dev).view(torch.uint32).reshape(N, N, d)
        Cm = torch.empty((N, N, 2 * d - 1), dtype=torch.uint32, device=dev)
        msm = tloop(lambda: mm.poly_matmul(A, B, pp, 3, out=Cm), 5)
        pm[f"n{N}"] = {"ms": round(msm, 3),
                       "Gbutterfly_per_s": round((2 * N * N + N * N) * (1 << 15) * 16 / (msm * 1e-3) / 1e9, 1)}
        del A, B, Cm
    out["poly_matmul_d2^15_p469762049"] = dict(pm, note="paper Table 15 (one i7-4770 core, context only): "
                                                        "n = 8: 0.15 s, n = 32: 4.7 s")

    # truncated products (lc just above a power of two) vs the padded transform
    tf = {}
    for la, bt in ((33000, 512), (40000, 512), (49152, 512)):
        a3 = gen.residues_torch(gen.config_seed(3), 5, bt * la, P30, dev).view(torch.uint32).reshape(bt, la)
        b3 = gen.residues_torch(gen.config_seed(3), 6, bt * la, P30, dev).view(torch.uint32).reshape(bt, la)
        c3 = torch.empty((bt, 2 * la - 1), dtype=torch.uint32, device=dev)
        msp = tloop(lambda: mm.poly_mul(a3, b3, P30, G30, out=c3), 5)
        mst = tloop(lambda: mm.poly_mul_tft(a3, b3, P30, G30, out=c3), 5)
        tf[f"{bt}x(la=lb={la})"] = {"padded_ms": round(msp, 3), "tft_ms": round(mst, 3),
                                    "speedup": round(msp / mst, 3)}
        del a3, b3, c3
    out["tft_vs_padded_p998244353"] = tf

    # integer matrix product (Table 17: n x n, entries of 32 x 2^15 bits)
    im = {}
    for N in (8, 32):
        nl = 1 << 15
        A = gen.limbs16_torch(17, 1, 2 * N * N * nl, dev).view(torch.uint32).reshape(N, N, nl)
        B = gen.limbs16_torch(17, 2, 2 * N * N * nl, dev).view(torch.uint32).reshape(N, N, nl)
        Cm = torch.empty((N, N, 2 * nl + 1), dtype=torch.uint32, device=dev)
        msi = tloop(lambda: mm.int_matmul_u32(A, B, out=Cm), 3)
        im[f"n{N}"] = {"ms": round(msi, 3)}
        del A, B, Cm
    out["int_matmul_32x2^15bit"] = dict(im, note="paper Table 17 (one i7-4770 core, context only): "
                                                 "n = 8: 0.44 s, n = 32: 13 s")

    # the paper's three-prime integer product at
    # Table 16's largest size, 32 x 2^20-bit operands, beside the Goldilocks path
    n32 = 1 << 20
    ja = gen.limbs16_torch(gen.config_seed(5), 3, 2 * n32, dev).view(torch.uint32)
    jb = gen.limbs16_torch(gen.config_seed(5), 4, 2 * n32, dev).view(torch.uint32)
    jc = torch.empty(2 * n32, dtype=torch.uint32, device=dev)
    ms3 = tloop(lambda: mm.int_mul_u32(ja, jb, out=jc), 10)
    jc16 = torch.empty(4 * n32, dtype=torch.uint16, device=dev)
    ms1 = tloop(lambda: mm.int_mul_u16(ja.view(torch.uint16), jb.view(torch.uint16), out=jc16), 10)
    out["int_mul_32x2^20bit"] = {
        "three_prime_ms": round(ms3, 4), "three_prime_Mbit_per_s": round(2 * 32 * n32 / (ms3 * 1e-3) / 1e6, 1),
        "goldilocks_ms": round(ms1, 4), "goldilocks_Mbit_per_s": round(2 * 32 * n32 / (ms1 * 1e-3) / 1e6, 1),
        "note": "Table 16 size (paper: 200 ms MATHEMAGIX / 240 ms GMP on one i7-4770 core, context only)"}
    return out


def sharded_run(mm, torch, dev, world, rank):
    """N > 1: the partitioned configs -- C4's 2^24 Goldilocks
    transforms and C5's integer product, each split across all ranks by
    dist.py (column blocks, NCCL all-to-all, row blocks); strong scaling,
    device time max over ranks."""
    import gen
    from paper_1407_3383_b200.dist import ShardedIntMul, ShardedNtt
    out = {}
    # C4: 8 forward transforms of 2^24, each sharded over all ranks
    k = 24
    plan = mm.NttPlan(64, PG, k, root_of_unity(PG, 7, k), 1)
    sh = ShardedNtt(plan)
    idx = sh.column_block_indices().reshape(-1).to(dev)
    xs = []
    for t in range(8):
        full = gen.residues_torch(gen.config_seed(4), 1, 1 << k, PG, dev, start=t << k).view(torch.int64)
        xs.append(full[idx].reshape(sh.n2, sh.c1).view(torch.uint64).contiguous())
        del full

    def c4():
        for x in xs:
            sh.forward(x)

    ms = timed(c4, 3, 3, world)
    ms /= 3
    bfly = 8 * (1 << (k - 1)) * k
    out["C4_sharded_8x2^24_fwd"] = {"ms": round(ms, 3), "Gbutterfly_per_s": round(bfly / (ms * 1e-3) / 1e9, 1),
                                    "scaling": "strong", "ranks": world}
    # the same with the transpose fused into the column pass (CUDA IPC peer stores)
    try:
        from paper_1407_3383_b200.dist import peer_pointers
        import torch.distributed as dist
        recv = torch.empty(sh.n2 * sh.c1, dtype=torch.uint64, device=dev)
        ptrs = peer_pointers(recv)
        rows = torch.empty((sh.r2, sh.n1), dtype=torch.uint64, device=dev)

        def c4p():
            for x in xs:
                sh.forward_p2p(x, recv, ptrs)
                torch.cuda.synchronize()
                dist.barrier()
                sh.plan.fwd_rows_seg(recv, rows, sh.rank * sh.r2, sh.r2, sh.c1, sh.r2 * sh.c1)

        msp = timed(c4p, 3, 3, world) / 3
        out["C4_sharded_8x2^24_fwd_p2p"] = {"ms": round(msp, 3),
                                            "Gbutterfly_per_s": round(bfly / (msp * 1e-3) / 1e9, 1),
                                            "scaling": "strong", "ranks": world,
                                            "note": "column pass stores into peer receive buffers; host barrier"}
    except Exception as e:
        out["C4_sharded_p2p_error"] = repr(e)[:200]
    del xs
    # C5: one 2^28-bit x 2^28-bit product sharded over all ranks
    n = 1 << 24
    a = gen.limbs16_torch(gen.config_seed(5), 1, n, dev).view(torch.uint16)
    b = gen.limbs16_torch(gen.config_seed(5), 2, n, dev).view(torch.uint16)
    plan5 = mm.NttPlan(64, PG, 25, root_of_unity(PG, 7, 25), 1)
    im = ShardedIntMul(plan5, n, n)
    ms = timed(lambda: im(a, b), 3, 3, world) / 3
    out["C5_sharded_int_mul_2^28bit"] = {"ms": round(ms, 3), "Mbit_per_s": round(2 * (1 << 28) / (ms * 1e-3) / 1e6, 1),
                                         "scaling": "strong", "ranks": world}
    return out


def run_ours(args, world, rank, local):
    import torch
    import gen
    import paper_1407_3383_b200 as mm

    mm.lib()
    dev = torch.device("cuda", local)
    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json)" if hbm_peak else "fallback (B200_PROFILING.md)"
    hbm_peak = hbm_peak or HBM_FALLBACK_GBS

    B, d = C3_BATCH, C3_D
    lc = 2 * d - 1
    start = rank * B * d             # each rank draws its own products
    a = gen.residues_torch(gen.config_seed(3), 1, B * d, P30, dev, start=start).view(torch.uint32).reshape(B, d)
    b = gen.residues_torch(gen.config_seed(3), 2, B * d, P30, dev, start=start).view(torch.uint32).reshape(B, d)
    # output rows at a 128-byte leading dimension (ldc = 2^16 words; the row's
    # last word is padding, never written): packed rows of 2^16 - 1 words split
    # 32-byte sectors between neighbouring column tiles (the packed
    # layout is timed in extra.C3_packed_output)
    c_pad = torch.empty((B, C3_LDC), dtype=torch.uint32, device=dev)
    c = c_pad[:, :lc]

    def step():
        mm.poly_mul(a, b, P30, G30, out=c)

    step()   # plan + workspace creation outside the timed region
    torch.cuda.synchronize()
    cnt = {}
    clk = ClockSampler(local).__enter__()   # polls from here to the end of the run; the timed region is marked
    time.sleep(0.05)
    if True:
        ms_total = timed(step, args.steps, args.warmup, world,
                         on_start=lambda: (cnt.__setitem__("n0", mm.launch_count()), mm.prof_enable(True),
                                           clk.mark(True)),
                         on_stop=lambda: (mm.prof_enable(False), cnt.__setitem__("n1", mm.launch_count())))
        clk.mark(False)
    launches = cnt["n1"] - cnt["n0"]
    prof = mm.prof_collect()
    ms_step = ms_total / args.steps
    bfly_step = c3_butterflies(B)
    value = world * bfly_step / (ms_step * 1e-3) / 1e9

    # ---- per-kernel roofline (dominant kernel, measured live with CUDA events on the launch stream)
    n = 1 << C3_LOG
    kb = {   # algorithmic bytes and butterflies per launch, per kernel family
        "ntt_cols_fwd": (B * d * 4 + B * n * 4, B * (1 << 8) * (1 << 7) * 8),
        "pmul_rows_fourstep": (3 * B * n * 4, 3 * B * (1 << 8) * (1 << 7) * 8),
        "ntt_cols_inv": (B * n * 4 + B * lc * 4, B * (1 << 8) * (1 << 7) * 8),
    }
    fam = max(prof, key=lambda k: prof[k][1]) if prof else None
    # DRAM bytes per launch from the committed ncu --set full capture (profiles/)
    try:
        with open(os.path.join(ROOT, "profiles", "traffic_c3.json")) as fh:
            traffic = json.load(fh)
    except OSError:
        traffic = {}
    roof = None
    kernels = {}
    sm_mhz_max = peaks.get("sm_max_mhz", 1965.0)
    # ALU roofline: integer multiplies issue only to the fmaheavy pipe,
    # IMAD at 2 and IMAD.HI at 4 cycles per warp per SMSP (mm_probe_issue, ncu pipe
    # counters).  The lazy Shoup butterfly needs IMAD.HI + 2 IMAD = 8 heavy cycles per
    # warp (its 3 adds/mins go to the ALU pipe in parallel) -> 4 SMSP x 32 / 8 = 16
    # butterflies / clk / SM, at the max SM clock.
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_bfly_peak = nsm * 16 * sm_mhz_max * 1e6
    for k_, (cnt, tot) in prof.items():
        per = tot / cnt
        entry = {"launches": cnt, "avg_ms": round(per, 4), "share": round(tot / ms_total, 3)}
        if k_ in kb:
            by, bf = kb[k_]
            entry["GB_per_s"] = round(by / (per * 1e-3) / 1e9, 1)
            entry["hbm_frac"] = round(by / (per * 1e-3) / 1e9 / hbm_peak, 3)
            entry["Gbutterfly_per_s"] = round(bf / (per * 1e-3) / 1e9, 1)
            entry["alu_frac"] = round(bf / (per * 1e-3) / alu_bfly_peak, 3)
        kernels[k_] = entry
    if fam in kb:
        e = kernels[fam]
        if e["alu_frac"] >= e["hbm_frac"]:
            roof = {"bound": "alu", "kernel": fam, "achieved": e["Gbutterfly_per_s"],
                    "peak": round(alu_bfly_peak / 1e9, 1), "unit": "Gbutterfly/s", "frac": e["alu_frac"],
                    "traffic": traffic.get(fam), "algorithmic_bytes": kb[fam][0], "hbm_frac": e["hbm_frac"],
                    "peak_source": f"derived: {nsm} SMs x 16 butterflies/clk/SM (fmaheavy pipe: IMAD.HI 4 + "
                                   f"2 x IMAD 2 cycles per warp) x {sm_mhz_max:.0f} MHz"}
        else:
            roof = {"bound": "hbm", "kernel": fam, "achieved": e["GB_per_s"], "peak": hbm_peak, "unit": "GB/s",
                    "frac": e["hbm_frac"], "traffic": traffic.get(fam), "algorithmic_bytes": kb[fam][0],
                    "alu_frac": e["alu_frac"], "peak_source": peak_src}

    # ---- e2e: same step through the public API from pinned host buffers
    # (mm_poly_mul_host: chunked uploads / kernels / downloads, three-slot pipeline)
    e2e_steps = max(1, min(args.steps, 5))
    ah = torch.empty((B, d), dtype=torch.uint32, pin_memory=True)
    bh = torch.empty((B, d), dtype=torch.uint32, pin_memory=True)
    ch = torch.empty((B, lc), dtype=torch.uint32, pin_memory=True)
    ah.copy_(a)
    bh.copy_(b)

    def e2e_step():
        mm.poly_mul_host(ah, bh, P30, G30, out=ch)

    ms_e2e = timed(e2e_step, e2e_steps, 1, world) / e2e_steps
    e2e_val = world * bfly_step / (ms_e2e * 1e-3) / 1e9
    if world == 1:   # the host result must equal the device result
        ok = bool(torch.equal(ch[:4], c[:4].cpu())) and bool(torch.equal(ch[-4:], c[-4:].cpu()))
        if not ok:
            raise RuntimeError("poly_mul_host result differs from poly_mul")

    time.sleep(0.02)
    clk.__exit__(None, None, None)
    clk_summary = clk.summary()

    extra = {}
    if world == 1 and not args.no_extras:
        extra = extras_run(mm, torch, dev, peaks)
    if world > 1 and not args.no_extras:
        try:
            extra = sharded_run(mm, torch, dev, world, rank)
        except Exception as e:   # the headline line must survive a failing secondary measurement
            extra = {"sharded_error": repr(e)[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t, bf = oracle_c3_sample(0, budget_s=args.cpu_seconds)
        cpu = {"value": round(bf / t / 1e9, 6), "unit": "Gbutterfly/s", "cores": 1, "kind": "oracle",
               "sample": f"{bf // C3_BFLY_PER_PROD} of the 4096 C3 products (oracle: u128 %, textbook radix-2 NTT), "
                         f"{t:.1f} s on one host thread"}

    if rank != 0:
        return
    line = {
        "metric": "NTT Gbutterfly/s", "value": round(value, 2), "unit": "Gbutterfly/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (seeded counter-based SplitMix64, uniform in [0,p), generated in HBM)",
        "config": {"workload": "C3: 4096 poly products/GPU, deg < 2^15, n = 2^16, p = 998244353 (fwd NTT x2, "
                               "pointwise modmul, inverse NTT)",
                   "global_batch": B * world, "transform_len": n, "p": P30,
                   "butterflies_per_step_per_gpu": bfly_step,
                   "l2": "inputs 1 GiB + outputs 1 GiB per GPU > 126 MB L2 (no flush needed)",
                   "output_layout": f"c[{B}][{lc}] at row stride {C3_LDC} words (mm_poly_mul_ld)",
                   "parallelism": f"dp{world} (independent products, no collective)"},
        "e2e": {"value": round(e2e_val, 2), "unit": "Gbutterfly/s",
                "h2d_bytes_per_step": 2 * B * d * 4, "d2h_bytes_per_step": B * lc * 4,
                "ms_per_step": round(ms_e2e, 3)},
        "gpu_launches": int(launches),
        "roofline": roof,
        "kernels": kernels,
        "clocks": clk_summary,
        "cpu_baseline": cpu,
        "extra": extra,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        run_reference(args, world, rank)
        return
    world, rank, local = dist_setup()
    try:
        run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
