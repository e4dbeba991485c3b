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


# ----------------------------------------------------------------------------- CPU oracle (reference arm, cpu_baseline)
# The oracle (oracle/, test infrastructure: u128 %, textbook radix-2 NTT) as it
# stands, on the host cores of the box: one thread, and all cores (threads over
# independent units -- products, transforms, element chunks; ctypes releases
# the GIL inside every oracle call).  Bounded samples of each workload.
def cpu_info() -> dict:
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    return {"model": model, "cores": cores}


def _parallel(fn, nthreads: int, quota: int):
    """Run fn(thread, i) for i < quota on each of nthreads threads; wall seconds."""
    from concurrent.futures import ThreadPoolExecutor

    def work(t):
        for i in range(quota):
            fn(t, i)
    t0 = time.perf_counter()
    with ThreadPoolExecutor(nthreads) as ex:
        list(ex.map(work, range(nthreads)))
    return time.perf_counter() - t0


def oracle_c3(nthreads: int, budget_s: float, seed_off: int = 0) -> dict:
    """C3 products (two degree < 2^15 polynomials mod 998244353) by the oracle's
    NTT product; quota per thread sized from a one-product calibration."""
    import gen
    import oracle as O
    O.build()

    def inputs(i):
        a = gen.residues(gen.config_seed(3), 1, C3_D, P30, start=(seed_off + i) * C3_D)
        b = gen.residues(gen.config_seed(3), 2, C3_D, P30, start=(seed_off + i) * C3_D)
        return a, b
    a0, b0 = inputs(0)
    t0 = time.perf_counter()
    O.poly_mul_ntt(a0, b0, P30, G30)
    t1 = time.perf_counter() - t0
    quota = max(1, int(budget_s / max(t1, 1e-4)))
    pool = [[inputs(t * quota + i) for i in range(quota)] for t in range(nthreads)]   # drawn outside the timing
    wall = _parallel(lambda t, i: O.poly_mul_ntt(*pool[t][i], P30, G30), nthreads, quota)
    prods = nthreads * quota
    return {"value": round(prods * C3_BFLY_PER_PROD / wall / 1e9, 6), "unit": "Gbutterfly/s", "cores": nthreads,
            "products": prods, "wall_s": round(wall, 2)}


def oracle_c2(nthreads: int, n_per_thread: int = 1 << 22) -> dict:
    """C2 modmul over 2^28 uint32 pairs mod 3221225473: a sample of n_per_thread
    pairs per thread through the oracle's vector product."""
    import gen
    import oracle as O
    O.build()
    xs = [gen.residues(gen.config_seed(2), 1, n_per_thread, P32, start=t * n_per_thread) for t in range(nthreads)]
    ys = [gen.residues(gen.config_seed(2), 2, n_per_thread, P32, start=t * n_per_thread) for t in range(nthreads)]
    wall = _parallel(lambda t, i: O.vec_mulmod(xs[t], ys[t], P32), nthreads, 1)
    return {"value": round(nthreads * n_per_thread / wall / 1e9, 6), "unit": "Gelem/s", "cores": nthreads,
            "elements": nthreads * n_per_thread, "wall_s": round(wall, 2)}


def oracle_c4(nthreads: int, k: int = 24) -> dict:
    """C4: forward Goldilocks transforms of 2^k (one per thread) by the oracle's
    textbook NTT (k = 24 is the BASELINE size: ~10 s per transform per core)."""
    import gen
    import oracle as O
    O.build()
    w = O.root_of_unity(7, k, PG)
    xs = [gen.residues(gen.config_seed(4), 1, 1 << k, PG, start=t << k) for t in range(nthreads)]
    wall = _parallel(lambda t, i: O.ntt(xs[t], w, PG), nthreads, 1)
    bf = nthreads * (1 << (k - 1)) * k
    return {"value": round(bf / wall / 1e9, 6), "unit": "Gbutterfly/s", "cores": nthreads,
            "transforms": f"{nthreads} x 2^{k}", "wall_s": round(wall, 2)}


def oracle_c5(nthreads: int, limbs: int = 1 << 20) -> dict:
    """C5 shape at a bounded size: one or_int_mul_ntt_u16 product of two
    `limbs`-limb integers per thread (BASELINE: 2^24 limbs, ~1 min per core)."""
    import gen
    import oracle as O
    O.build()
    ab = [(gen.limbs16(gen.config_seed(5), 1, limbs, start=t * limbs), gen.limbs16(gen.config_seed(5), 2, limbs,
                                                                                    start=t * limbs))
          for t in range(nthreads)]
    wall = _parallel(lambda t, i: O.int_mul_ntt_u16(*ab[t]), nthreads, 1)
    return {"value": round(nthreads * 2 * 16 * limbs / wall / 1e6, 3), "unit": "Mbit/s", "cores": nthreads,
            "sample": f"{nthreads} products of {limbs} x {limbs} limbs", "wall_s": round(wall, 2)}


def cpu_baseline_run(budget_s: float, legs: str) -> dict:
    ci = cpu_info()
    allc = ci["cores"]
    one = oracle_c3(1, budget_s)
    many = oracle_c3(allc, budget_s, seed_off=1 << 12)
    out = {"value": many["value"], "unit": "Gbutterfly/s", "cores": allc, "kind": "oracle",
           "cpu_model": ci["model"],
           "sample": f"C3: {many['products']} of the 4096 products on {allc} threads ({many['wall_s']} s wall); "
                     f"single-thread leg {one['products']} products",
           "single_thread": one, "all_cores": many}
    extra = {}
    if "c2" in legs:
        extra["C2_modmul"] = {"single_thread": oracle_c2(1), "all_cores": oracle_c2(allc)}
    if "c4" in legs:
        extra["C4_ntt_2^24"] = {"single_thread": oracle_c4(1), "all_cores": oracle_c4(min(allc, 8))}
    if "c5" in legs:
        extra["C5_int_mul"] = {"single_thread": oracle_c5(1), "all_cores": oracle_c5(allc)}
    out["other_configs"] = extra
    return out


def run_reference(args, world, rank):
    if rank != 0:
        return
    ci = cpu_info()
    nth = ci["cores"]
    # size one step so that W + K steps take ~ a couple of minutes at most
    per = max(2.0, min(8.0, 100.0 / (args.warmup + args.steps)))
    for _ in range(args.warmup):
        oracle_c3(nth, per / 4)
    tot_p, tot_t = 0, 0.0
    for s_ in range(args.steps):
        r = oracle_c3(nth, per, seed_off=s_ << 10)
        tot_p += r["products"]
        tot_t += r["wall_s"]
    val = tot_p * C3_BFLY_PER_PROD / tot_t / 1e9
    line = {
        "impl": "reference", "metric": "NTT Gbutterfly/s", "value": round(val, 6), "unit": "Gbutterfly/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * tot_t / args.steps, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic (seeded SplitMix64, uniform in [0,p))",
        "config": {"workload": "C3 poly_mul sample: about %d of the 4096 products per step on %d host threads "
                               "(deg < 2^15, n = 2^16, p = 998244353)" % (tot_p // max(1, args.steps), nth),
                   "sample_products_per_step": tot_p // max(1, args.steps), "parallelism": f"{nth} CPU threads"},
        "cpu_baseline": {"value": round(val, 6), "unit": "Gbutterfly/s", "cores": nth, "kind": "oracle",
                         "cpu_model": ci["model"],
                         "sample": f"{tot_p} C3 products over {args.steps} steps, {nth} threads"},
        "e2e": {"value": round(val, 6), "unit": "Gbutterfly/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- GPU arm
def extras_run(mm, torch, dev, peaks):
    """Secondary configs on rank 0 / N = 1 (C1, C2, C4, C5, ALU probe)."""
    import gen
    out = {}
    hbm = peaks.get("hbm_gbs", HBM_FALLBACK_GBS)

    def with_clocks(fn):
        # the SM clock (median of NVML samples) and throttle reasons while fn runs
        cs = ClockSampler(dev.index or 0).__enter__()
        cs.mark(True)
        r = fn()
        cs.mark(False)
        cs.__exit__(None, None, None)
        sm = cs.summary()
        return r, {"sm_mhz": sm.get("sm_mhz"), "reasons": sm.get("reasons"), "samples": sm.get("samples")}

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

    side = torch.cuda.Stream()

    def c1_forked():
        # the product does not depend on the 16 transforms: a second graph branch
        cur = torch.cuda.current_stream()
        side.wait_stream(cur)
        with torch.cuda.stream(side):
            mm.poly_mul(pa, pb, P30, G30, out=pc)
        plan.forward(xa, order=mm.NATURAL)
        plan.inverse(xa, order=mm.NATURAL)
        cur.wait_stream(side)

    def graph_ms(fn):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
            with torch.cuda.graph(g, stream=s):
                fn()
        torch.cuda.synchronize()
        return tloop(g.replay, 500)

    # the same work as ONE launch (mm_run_jobs): 16 round trips + the product
    ya, za = torch.empty_like(xa).view(16, 1 << 10), torch.empty_like(xa).view(16, 1 << 10)
    jb = mm.Jobs()
    for r in range(16):
        jb.roundtrip(plan, xa.view(16, 1 << 10)[r], za[r], out=ya[r], order=mm.NATURAL)
    jb.poly_mul(pa, pb, P30, G30, pc)

    ms = tloop(c1, 200)
    ms_graph = graph_ms(c1)
    ms_fork = graph_ms(c1_forked)
    ms_jobs = tloop(jb.run, 500)
    ms_jobs_graph = graph_ms(jb.run)
    bf = 16 * 2 * 5 * 512 + 3 * 5 * 512
    out["C1_16x2^10_fwd_inv_plus_poly511"] = {"us_per_call": round(ms * 1e3, 2),
                                             "us_per_call_cuda_graph": round(ms_graph * 1e3, 2),
                                             "us_per_call_cuda_graph_2_branches": round(ms_fork * 1e3, 2),
                                             "us_per_call_one_launch": round(ms_jobs * 1e3, 2),
                                             "us_per_call_one_launch_cuda_graph": round(ms_jobs_graph * 1e3, 2),
                                             "Gbutterfly_per_s_one_launch": round(bf / (ms_jobs_graph * 1e-3) / 1e9, 2),
                                             "note": "separate calls: three dependent latency-bound launches (the "
                                                     "product on a second graph branch); one launch: mm_run_jobs, "
                                                     "17 CTAs (16 round trips + the product)"}

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

    # paper §3.2-3.3: Functions 14 / 15 / 16 and their toward-+inf forms (mm_mulmod_num),
    # doubles (2^27) and floats (2^28) at Table 10's bit sizes (context: P:748-755)
    num = {}
    for fbits, pn, nn, variants in ((64, 33554393, 1 << 27, (0, 1, 2, 3, 4, 5)), (64, 1125899906842597, 1 << 27, (4, 5)),
                                    (32, 2039, 1 << 28, (0, 1, 2, 3, 4, 5)), (32, 2097143, 1 << 28, (4, 5))):
        dt = torch.float64 if fbits == 64 else torch.float32
        xn = gen.residues_torch(11, 1, nn, pn, dev).to(torch.int64).to(dt)    # int32 (p < 2^32) or int64 words
        yn = gen.residues_torch(11, 2, nn, pn, dev).to(torch.int64).to(dt)
        assert xn.numel() == nn
        zn = torch.empty_like(xn)
        MN = mm.ModNum(fbits, pn)
        names = ["F14", "F14_up", "F15_up", "F15_near", "F16", "F16_up"]
        for v in variants:
            msn = tloop(lambda: MN.mul(xn, yn, variant=v, out=zn), 10)
            by = 3 * nn * (fbits // 8)
            num[f"{'f64' if fbits == 64 else 'f32'}_m{pn.bit_length()}_{names[v]}"] = {
                "Gelem_per_s": round(nn / (msn * 1e-3) / 1e9, 1), "ms": round(msn, 4),
                "hbm_frac": round(by / (msn * 1e-3) / 1e9 / hbm, 3)}
        del xn, yn, zn
    out["numeric_mulmod_functions_14_16"] = num

    # C3-fwd: 4096 forward NTTs of length 2^16 (TFT order), and the inverse
    pl16 = mm.NttPlan(32, P30, 16, root_of_unity(P30, G30, 16), 4096)
    x16 = gen.residues_torch(gen.config_seed(3), 3, 4096 << 16, P30, dev).view(torch.uint32)
    y16 = torch.empty_like(x16)
    msf = tloop(lambda: pl16.forward(x16, out=y16, order=mm.BITREV), 10)
    msi = tloop(lambda: pl16.inverse(y16, out=x16, order=mm.BITREV), 10)
    msn = tloop(lambda: pl16.forward(x16, out=y16, order=mm.NATURAL), 10)
    msni = tloop(lambda: pl16.inverse(y16, out=x16, order=mm.NATURAL), 10)
    bf16 = 4096 * (1 << 15) * 16
    out["C3_fwd_4096x2^16"] = {"forward_ms": round(msf, 4), "forward_Gbutterfly_per_s": round(bf16 / (msf * 1e-3) / 1e9, 1),
                               "inverse_ms": round(msi, 4), "inverse_Gbutterfly_per_s": round(bf16 / (msi * 1e-3) / 1e9, 1),
                               "hbm_frac_2pass": round(4 * 4096 * (1 << 16) * 4 / (msf * 1e-3) / 1e9 / hbm, 3),
                               "hbm_frac_1pass": round(2 * 4096 * (1 << 16) * 4 / (msf * 1e-3) / 1e9 / hbm, 3),
                               "forward_natural_ms": round(msn, 4), "inverse_natural_ms": round(msni, 4),
                               "alu_frac": round(bf16 / (msf * 1e-3) / (nsm * 16 * clk), 3),
                               "note": "SURVEY 8(d) C3-fwd: 1-pass = 8 B/elem (the contract), 2-pass = 16 B/elem"}
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
        # per-family kernel time per call (library event profiler, launching
        # stream), kernels serialised on one stream so their times add up
        mm.set_product_streams(1)
        fn()
        torch.cuda.synchronize()
        mm.prof_collect()
        mm.prof_enable(True)
        for _ in range(reps):
            fn()
        r = mm.prof_collect()
        mm.prof_enable(False)
        mm.set_product_streams(2)
        return {k: round(v[1] / reps, 4) for k, v in r.items()}

    # C4: 8 x 2^24 Goldilocks forward NTT (four-step 2^11 columns x 2^13 rows, gold.cuh tiles)
    w24 = root_of_unity(PG, 7, 24)
    plan4 = mm.NttPlan(64, PG, 24, w24, 8)
    x4 = gen.residues_torch(gen.config_seed(4), 1, 8 << 24, PG, dev).view(torch.uint64)
    y4 = torch.empty_like(x4)
    f4 = lambda: plan4.forward(x4, out=y4, order=mm.BITREV)
    ms, ck4 = with_clocks(lambda: tloop(f4, 10))
    bfly = 8 * (1 << 23) * 24
    gbs2 = 8 * (1 << 24) * 32 / (ms * 1e-3) / 1e9
    inf4 = plan4.info()
    out["C4_8x2^24_goldilocks_fwd"] = {"ms": round(ms, 3), "Gbutterfly_per_s": round(bfly / (ms * 1e-3) / 1e9, 1),
                                       "GB_per_s_2pass": round(gbs2, 1), "hbm_frac_2pass": round(gbs2 / hbm, 3),
                                       "split": f"{inf4['n2']} cols x {inf4['n1']} rows", "kernels_ms": kern_ms(f4),
                                       "alu_frac_vs_gold8_probe": round(bfly / (ms * 1e-3) / bg8, 3),
                                       "alu_note": "achieved butterflies / register-resident gold.cuh 8-point rate "
                                                   "(the passes also carry the w_L and step-2 table products)",
                                       "clocks": ck4}
    del x4, y4, plan4

    # C5: 2^28-bit x 2^28-bit integer product (2^24 16-bit limbs each)
    na = 1 << 24
    ia = gen.limbs16_torch(gen.config_seed(5), 1, na, dev).view(torch.uint16)
    ib = gen.limbs16_torch(gen.config_seed(5), 2, na, dev).view(torch.uint16)
    ic = torch.empty(2 * na, dtype=torch.uint16, device=dev)
    f5 = lambda: mm.int_mul_u16(ia, ib, out=ic)
    ms, ck5 = with_clocks(lambda: tloop(f5, 10))
    out["C5_int_mul_2^28bit"] = {"ms": round(ms, 3), "Mbit_per_s": round(2 * (1 << 28) / (ms * 1e-3) / 1e6, 1),
                                 "Gbutterfly_per_s": round(3 * (1 << 24) * 25 / (ms * 1e-3) / 1e9, 1),
                                 "kernels_ms": kern_ms(f5), "clocks": ck5}
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


def sharded_run(mm, torch, dev, world, rank, steps):
    """N > 1: the partitioned configs through the library's
    distributed C ABI (mm_dist_create over the NCCL torch loaded):
      * C4: 8 forward transforms of 2^24, each split across all ranks (column
        block in, row block out): NCCL transport on one stream, pipelined on
        two streams (transform t's all-to-all overlaps t+1's column pass), and
        the peer-memory transport (fused transpose, device-side flags);
      * C5: one 2^28-bit x 2^28-bit product (mm_int_mul_u16_dist).
    Strong scaling; device time, max over ranks; E(G) = T(1) / (G T(G)) with
    T(1) measured on this node's GPU in the same run; a standalone NCCL
    all-to-all probe of the same block size gives the achieved NVLink rate."""
    import gen
    import torch.distributed as dist
    from paper_1407_3383_b200.dist import ShardedNtt
    out = {"ranks": world}
    k = 24
    w24 = root_of_unity(PG, 7, k)
    # ---- T(1): the same work on one GPU (every rank runs it; rank 0's number is used)
    plan8 = mm.NttPlan(64, PG, k, w24, 8)
    x8 = gen.residues_torch(gen.config_seed(4), 1, 8 << k, PG, dev).view(torch.uint64)
    y8 = torch.empty_like(x8)
    t1_c4 = timed(lambda: plan8.forward(x8, out=y8, order=mm.BITREV), 3, 2, 1)
    t1_c4 /= 3
    del x8, y8, plan8
    n5 = 1 << 24
    a5 = gen.limbs16_torch(gen.config_seed(5), 1, n5, dev).view(torch.uint16)
    b5 = gen.limbs16_torch(gen.config_seed(5), 2, n5, dev).view(torch.uint16)
    c5 = torch.empty(2 * n5, dtype=torch.uint16, device=dev)
    t1_c5 = timed(lambda: mm.int_mul_u16(a5, b5, out=c5), 3, 2, 1) / 3
    t1 = torch.tensor([t1_c4, t1_c5], dtype=torch.float64, device=dev)
    dist.broadcast(t1, 0)
    t1_c4, t1_c5 = float(t1[0]), float(t1[1])
    # ---- C4 sharded
    plan = mm.NttPlan(64, PG, k, w24, 1)
    sh = ShardedNtt(plan, rank=rank, world=world)
    idx = sh.column_block_indices().reshape(-1).to(dev)
    xs, ys = [], []
    for t in range(8):
        full = gen.residues_torch(gen.config_seed(4), 1, 1 << k, PG, dev, start=t << k).view(torch.int64)
        xs.append(full[idx].reshape(sh.n2, sh.c1).view(torch.uint64).contiguous())
        ys.append(torch.empty((sh.r2, sh.n1), dtype=torch.uint64, device=dev))
        if t == 0:
            ref0 = plan.forward(full.view(torch.uint64), out=torch.empty_like(full).view(torch.uint64), order=mm.BITREV)
            ref0 = ref0.view(torch.int64)[rank * sh.r2 * sh.n1:(rank + 1) * sh.r2 * sh.n1].clone()
        del full
    D = mm.Dist()
    bfly = 8 * (1 << (k - 1)) * k
    blk = sh.n2 * sh.c1 * 8

    def c4_one():
        for t in range(8):
            D.ntt_forward(plan, xs[t], out=ys[t])

    s_a, s_b = torch.cuda.Stream(), torch.cuda.Stream()

    def c4_pipe():
        cur = torch.cuda.current_stream()
        s_a.wait_stream(cur)
        s_b.wait_stream(cur)
        for t in range(8):
            with torch.cuda.stream(s_a if t % 2 == 0 else s_b):
                D.ntt_forward(plan, xs[t], out=ys[t])
        cur.wait_stream(s_a)
        cur.wait_stream(s_b)

    def rec(ms, note):
        return {"ms": round(ms, 3), "Gbutterfly_per_s": round(bfly / (ms * 1e-3) / 1e9, 1),
                "E_G": round(t1_c4 / (world * ms), 3), "note": note}

    ms = timed(c4_one, steps, 3, world) / steps
    ok = bool(torch.equal(ys[0].view(torch.int64).reshape(-1), ref0))
    out["C4_sharded_8x2^24_fwd_nccl"] = dict(rec(ms, "mm_ntt_forward_dist, NCCL grouped send/recv, one stream"),
                                             verified_vs_single_gpu=ok)
    ms = timed(c4_pipe, steps, 3, world) / steps
    out["C4_sharded_8x2^24_fwd_nccl_2streams"] = rec(ms, "transforms alternate between two streams: all-to-all of t "
                                                         "overlaps the column pass of t + 1")
    try:
        D.enable_p2p(blk)
        ms = timed(c4_one, steps, 3, world) / steps
        ok = bool(torch.equal(ys[0].view(torch.int64).reshape(-1), ref0))
        out["C4_sharded_8x2^24_fwd_p2p"] = dict(rec(ms, "fused transpose: column pass stores into the peers' receive "
                                                        "buffers (CUDA IPC), device-side release/acquire flags"),
                                                verified_vs_single_gpu=ok, timeout_slot=D.p2p_status())
    except Exception as e:   # the headline must survive a failing secondary path
        out["C4_sharded_p2p_error"] = repr(e)[:200]
    out["C4_single_gpu_ms"] = round(t1_c4, 3)
    # ---- NCCL all-to-all probe at the C4 block size
    send = torch.empty(blk // 8, dtype=torch.int64, device=dev)
    recv = torch.empty_like(send)
    msa = timed(lambda: dist.all_to_all_single(recv, send), steps, 3, world) / steps
    sent = blk * (world - 1) / world
    out["nccl_all_to_all_probe"] = {"bytes_per_rank": blk, "ms": round(msa, 4),
                                    "GB_per_s_per_gpu_out": round(sent / (msa * 1e-3) / 1e9, 1),
                                    "note": "torch.distributed all_to_all_single, equal split, NCCL"}
    del xs, ys, send, recv
    # ---- C5 sharded
    ms = timed(lambda: D.int_mul_u16(a5, b5), steps, 3, world) / steps
    loc = D.int_mul_u16(a5, b5)
    lay = D.int_mul_layout(n5, n5)
    pos = (torch.arange(lay["n2"], device=dev).view(-1, 1) * lay["n1"] + rank * lay["c1"]
           + torch.arange(lay["c1"], device=dev).view(1, -1)).reshape(-1)
    mm.int_mul_u16(a5, b5, out=c5)
    ok = bool(torch.equal(loc.view(torch.int16).reshape(-1), c5.view(torch.int16)[pos.clamp(max=2 * n5 - 1)]))
    out["C5_sharded_int_mul_2^28bit"] = {"ms": round(ms, 3), "Mbit_per_s": round(2 * (1 << 28) / (ms * 1e-3) / 1e6, 1),
                                         "E_G": round(t1_c5 / (world * ms), 3), "single_gpu_ms": round(t1_c5, 3),
                                         "verified_vs_single_gpu": ok}
    D.close()
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
    # headline: the library's default sub-batch concurrency (two fork streams,
    # mm_set_product_streams), every kernel launched inside the timed region
    ms_total = timed(step, args.steps, args.warmup, world,
                     on_start=lambda: (cnt.__setitem__("n0", mm.launch_count()), clk.mark(True)),
                     on_stop=lambda: cnt.__setitem__("n1", mm.launch_count()))
    clk.mark(False)
    launches = cnt["n1"] - cnt["n0"]
    ms_step = ms_total / args.steps
    bfly_step = c3_butterflies(B)
    value = world * bfly_step / (ms_step * 1e-3) / 1e9
    # per-kernel roofline: the same step with every kernel on one stream (with
    # two sub-batches overlapping, a launch's event-bracketed duration includes
    # the other stream's work), timed the same way; CUDA events recorded around
    # each launch on its launching stream (mm_prof_*)
    mm.set_product_streams(1)
    ms_serial = timed(step, args.steps, args.warmup, world, on_start=lambda: mm.prof_enable(True),
                      on_stop=lambda: mm.prof_enable(False)) / args.steps
    mm.set_product_streams(2)
    prof = mm.prof_collect()

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
    # the issue rates the ALU peak is derived from, measured on this GPU (mm_probe_issue),
    # after the timed regions so that the clocks have ramped up
    clk_hz = sm_mhz_max * 1e6
    rates = {nm: round(mm.probe_issue(kind, 4000) / (nsm * clk_hz), 3) for kind, nm in ((0, "IMAD"), (1, "IMAD.HI"))}
    for k_, (cnt, tot) in prof.items():
        per = tot / cnt
        entry = {"launches": cnt, "avg_ms": round(per, 4), "share": round(tot / (ms_serial * args.steps), 3)}
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
                                   f"2 x IMAD 2 cycles per warp) x {sm_mhz_max:.0f} MHz",
                    "peak_inputs": {"sms": nsm, "sm_max_mhz": sm_mhz_max,
                                    "warp_inst_per_clk_per_sm_measured": rates,
                                    "heavy_cycles_per_butterfly": "IMAD.HI 4 + 2 x IMAD 2 = 8 per warp per SMSP",
                                    "butterflies_per_clk_per_sm": 16}}
        else:
            roof = {"bound": "hbm", "kernel": fam, "achieved": e["GB_per_s"], "peak": hbm_peak, "unit": "GB/s",
                    "frac": e["hbm_frac"], "traffic": traffic.get(fam), "algorithmic_bytes": kb[fam][0],
                    "alu_frac": e["alu_frac"], "peak_source": peak_src}

    # ---- the whole step against SURVEY 8(d)'s byte models and the ALU peak
    step_s = ms_step * 1e-3
    fused_bytes = B * (2 * d + (2 * d - 1)) * 4          # read a, b once, write c once (1 HBM pass)
    unfused_bytes = sum(v[0] for v in kb.values()) + kb["ntt_cols_fwd"][0]   # the 4 launches' algorithmic bytes
    contract = {"step_alu_frac": round(bfly_step / step_s / alu_bfly_peak, 3),
                "step_hbm_frac_fused_model": round(fused_bytes / step_s / 1e9 / hbm_peak, 3),
                "step_hbm_frac_unfused_model": round(unfused_bytes / step_s / 1e9 / hbm_peak, 3),
                "fused_bytes_per_step": fused_bytes, "unfused_bytes_per_step": unfused_bytes,
                "note": "SURVEY 8(d) C3-poly: fused = 512 KiB per product; unfused = 2 column passes + fused "
                        "rows + inverse columns as launched"}

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
            extra = sharded_run(mm, torch, dev, world, rank, args.steps)
        except Exception as e:   # the headline line must survive a failing secondary measurement
            extra = {"sharded_error": repr(e)[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_run(args.cpu_seconds, args.cpu_legs)

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
        "roofline": dict(roof or {}, measured_in="serialized pass of the same step (mm_set_product_streams(1)): "
                                                  f"{ms_serial:.4f} ms/step vs {ms_step:.4f} with two fork streams"),
        "roofline_contract": contract,
        "kernels": kernels,
        "clocks": clk_summary,
        "cpu_baseline": cpu,
        "extra": extra,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- other BASELINE configs (--config)
# `--config c1|c2|c4|c5` prints the contract line of that BASELINE config
# instead of C3's: the same timing rules (W >= 3 untimed steps, K steps on the
# device, max over ranks, clocks sampled during the timed region), an e2e leg
# through the public API with the step's inputs uploaded from pinned host
# memory and its result read back inside the timed region, the dominant
# kernel's roofline from a serialised per-launch pass, and the oracle on the
# host cores.  Weak scaling at N > 1: every rank runs its own copy of the
# config's work on its own generator range (the partitioned C4 / C5 forms are
# the N > 1 extras of the default run).
def timed_flush(fn, steps, warmup, world, flush, on_start=None, on_stop=None):
    """timed() for configs whose inputs fit in L2 (C1, C5): a write larger than
    L2 before every timed step, outside that step's event pair; the K
    per-step durations are summed."""
    import torch
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    evs = []
    if on_start:
        on_start()
    for _ in range(steps):
        flush.add_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        evs.append((e0, e1))
    if on_stop:
        on_stop()
    torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(world, sum(a.elapsed_time(b) for a, b in evs))


def oracle_c1(nthreads: int, budget_s: float = 3.0) -> dict:
    """C1 on the oracle: 16 forward + inverse NTTs of 2^10 and one product of two
    degree-511 polynomials per unit; units spread over the threads."""
    import gen
    import oracle as O
    O.build()
    w = O.root_of_unity(G30, 10, P30)
    x = gen.residues(gen.config_seed(1), 1, 16 << 10, P30).reshape(16, 1 << 10)
    a = gen.residues(gen.config_seed(1), 2, 512, P30)
    b = gen.residues(gen.config_seed(1), 3, 512, P30)

    def unit(t, i):
        O.intt_rows(O.ntt_rows(x, w, P30), w, P30)
        O.poly_mul_ntt(a, b, P30, G30)
    t0 = time.perf_counter()
    unit(0, 0)
    quota = max(1, int(budget_s / max(time.perf_counter() - t0, 1e-4)))
    wall = _parallel(unit, nthreads, quota)
    units = nthreads * quota
    return {"value": round(units * C1_BFLY / wall / 1e9, 6), "unit": "Gbutterfly/s", "cores": nthreads,
            "units": units, "wall_s": round(wall, 2)}


C1_BFLY = 16 * 2 * (1 << 9) * 10 + 3 * (1 << 9) * 10   # 16 round trips of 2^10 + one 1024-point product


def config_spec(which, mm, torch, dev, rank):
    """Device inputs, the step, its host-side (e2e) form and the per-launch
    algorithmic work of each kernel family for one BASELINE config."""
    import gen
    s = {}
    if which == "c1":
        w10 = root_of_unity(P30, G30, 10)
        plan = mm.NttPlan(32, P30, 10, w10, 16)
        x = gen.residues_torch(gen.config_seed(1), 1, 16 << 10, P30, dev, start=rank << 14).view(torch.uint32)
        x = x.reshape(16, 1 << 10)
        a = gen.residues_torch(gen.config_seed(1), 2, 512, P30, dev, start=rank << 9).view(torch.uint32)
        b = gen.residues_torch(gen.config_seed(1), 3, 512, P30, dev, start=rank << 9).view(torch.uint32)
        y, z = torch.empty_like(x), torch.empty_like(x)
        c = torch.empty(1023, dtype=torch.uint32, device=dev)
        jobs = mm.Jobs()
        for r in range(16):
            jobs.roundtrip(plan, x[r], z[r], out=y[r], order=mm.NATURAL)
        jobs.poly_mul(a, b, P30, G30, c)
        s.update(step=jobs.run, inputs=[x, a, b], outputs=[y, z, c], units=C1_BFLY, unit="Gbutterfly/s",
                 metric="NTT Gbutterfly/s", scale=1e9, dtype="u32", flush=True, keep=(plan, jobs),
                 workload="C1: 16 independent forward + inverse NTTs of 2^10 (NATURAL order) and one product of two "
                          "degree-511 polynomials, p = 998244353, ONE launch (mm_run_jobs)",
                 fam={"jobs": (4 * (3 * 16 * 1024 + 2 * 512 + 1023), C1_BFLY)}, peak="alu32")
    elif which == "c2":
        n = 1 << 28
        x = gen.residues_torch(gen.config_seed(2), 1, n, P32, dev, start=rank * n).view(torch.uint32)
        y = gen.residues_torch(gen.config_seed(2), 2, n, P32, dev, start=rank * n).view(torch.uint32)
        z = torch.empty_like(x)
        M = mm.Mod32(P32)
        s.update(step=lambda: M.mul(x, y, mm.MUL_MONTGOMERY, out=z), inputs=[x, y], outputs=[z], units=n,
                 unit="Gelem/s", metric="modmul Gelem/s", scale=1e9, dtype="u32", flush=False, keep=(M,),
                 workload="C2: Montgomery modmul over 2^28 uint32 pairs, p = 3221225473 (Shoup, Barrett, add, sub "
                          "in config.variants)",
                 fam={"modmul_montgomery": (12 * n, 0)}, peak="hbm",
                 traffic=("r12_traffic_c2.json", {"modmul_montgomery": "modmul_montgomery"}),
                 e2e_host=(lambda hin, hout: M.op_host("mul_montgomery", hin[0], hin[1], out=hout[0]),
                           "mm_modop_u32_host (chunked upload, REDC product, download pipelined)"))
        ys = M.shoup_precompute(y)
        s["variants"] = [("modadd", lambda: M.add(x, y, out=z), 12), ("modsub", lambda: M.sub(x, y, out=z), 12),
                         ("modmul_barrett", lambda: M.mul(x, y, mm.MUL_BARRETT, out=z), 12),
                         ("modmul_shoup", lambda: M.mul(x, y, mm.MUL_SHOUP, y_shoup=ys, out=z), 16),
                         ("shoup_precompute", lambda: M.shoup_precompute(y, out=z), 8)]
        s["keep"] = (M, ys)
    elif which == "c4":
        plan = mm.NttPlan(64, PG, 24, root_of_unity(PG, 7, 24), 8)
        x = gen.residues_torch(gen.config_seed(4), 1, 8 << 24, PG, dev, start=rank << 27).view(torch.uint64)
        y = torch.empty_like(x)
        bf = 8 * (1 << 23) * 24
        inf = plan.info()
        kc, kr = 11, 13          # 2^11-point column tiles, 2^13-point rows
        s.update(step=lambda: plan.forward(x, out=y, order=mm.BITREV), inputs=[x], outputs=[y], units=bf,
                 unit="Gbutterfly/s", metric="NTT Gbutterfly/s", scale=1e9, dtype="u64", flush=False, keep=(plan,),
                 workload=f"C4: 8 forward NTTs of 2^24 over p = 2^64 - 2^32 + 1 (generator 7), four-step "
                          f"({inf['n2']} cols x {inf['n1']} rows), BITREV output",
                 fam={"ntt_cols_fwd": (2 * 8 * 8 << 24, 8 * (1 << 23) * kc),
                      "ntt_rows_fwd": (2 * 8 * 8 << 24, 8 * (1 << 23) * kr)}, peak="gold8",
                 traffic=("r11_traffic_c4.json", {"ntt_cols_fwd": "k_gcols_fwd", "ntt_rows_fwd": "k_grows_fwd"}),
                 e2e_host=(lambda hin, hout: plan.forward_host(hin[0], out=hout[0], order=mm.BITREV),
                           "mm_ntt_forward_host (one transform per chunk: upload, four-step, download pipelined)"))
    elif which == "c5":
        n = 1 << 24
        a = gen.limbs16_torch(gen.config_seed(5), 1, n, dev, start=rank * n).view(torch.uint16)
        b = gen.limbs16_torch(gen.config_seed(5), 2, n, dev, start=rank * n).view(torch.uint16)
        c = torch.empty(2 * n, dtype=torch.uint16, device=dev)
        N = 1 << 25
        s.update(step=lambda: mm.int_mul_u16(a, b, out=c), inputs=[a, b], outputs=[c], units=2 * 16 * n,
                 unit="Mbit/s", metric="int_mul Mbit/s", scale=1e6, dtype="u64", flush=True, keep=(),
                 workload="C5: product of two 2^28-bit integers (2^24 16-bit limbs each), length-2^25 convolution "
                          "over p = 2^64 - 2^32 + 1 (four-step 2^13 x 2^12), carries to 16-bit limbs",
                 fam={"ntt_cols_fwd": (2 * (2 * n + 8 * N), 2 * (1 << 24) * 12),
                      "pmul_rows_fourstep": (3 * 8 * N, 3 * (1 << 24) * 13),
                      "ntt_cols_inv": (2 * 8 * N, (1 << 24) * 12)}, peak="gold8",
                 traffic=("r12_traffic_c5.json", {"ntt_cols_fwd": "k_gcols16_fwd", "pmul_rows_fourstep": "k_gpmul_rows",
                                                  "ntt_cols_inv": "k_gcols_inv"}))
    else:
        raise SystemExit(f"unknown --config {which}")
    return s


def run_config(args, world, rank, local):
    import torch
    import paper_1407_3383_b200 as mm

    which = args.config
    mm.lib()
    dev = torch.device("cuda", local)
    peaks = load_peaks()
    hbm_peak = peaks.get("hbm_gbs")
    peak_src = "measured (MEASURED_PEAKS.json)" if hbm_peak else "fallback (B200_PROFILING.md)"
    hbm_peak = hbm_peak or HBM_FALLBACK_GBS
    sm_mhz_max = peaks.get("sm_max_mhz", 1965.0)
    nsm = torch.cuda.get_device_properties(dev).multi_processor_count
    S = config_spec(which, mm, torch, dev, rank)
    step = S["step"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev) if S["flush"] else None
    step()
    torch.cuda.synchronize()
    cnt = {}
    clk = ClockSampler(local).__enter__()
    time.sleep(0.05)
    on_start = lambda: (cnt.__setitem__("n0", mm.launch_count()), clk.mark(True))
    on_stop = lambda: cnt.__setitem__("n1", mm.launch_count())
    if flush is not None:
        ms_total = timed_flush(step, args.steps, args.warmup, world, flush, on_start, on_stop)
    else:
        ms_total = timed(step, args.steps, args.warmup, world, on_start=on_start, on_stop=on_stop)
    clk.mark(False)
    ms_step = ms_total / args.steps
    value = world * S["units"] / (ms_step * 1e-3) / S["scale"]

    # serialised per-launch pass (one stream; events on the launching stream)
    mm.set_product_streams(1)
    mm.prof_collect()
    mm.prof_enable(True)
    for _ in range(args.steps):
        if flush is not None:
            flush.add_(1)
        step()
    torch.cuda.synchronize()
    mm.prof_enable(False)
    prof = mm.prof_collect()
    mm.set_product_streams(2)
    ms_serial = sum(v[1] for v in prof.values()) / args.steps
    alu32 = nsm * 16 * sm_mhz_max * 1e6
    gold8 = None
    if S["peak"] == "gold8":   # first call loads the probe module: warm up, keep the best of three
        mm.probe_butterfly(65, 200)
        gold8 = max(mm.probe_butterfly(65, 1000) for _ in range(3))
    kernels, roof = {}, None
    for k_, (n_, tot) in prof.items():
        per = tot / n_
        e = {"launches": n_, "avg_ms": round(per, 4), "share": round(tot / max(ms_serial * args.steps, 1e-9), 3)}
        if k_ in S["fam"]:
            by, bf = S["fam"][k_]
            lps = n_ / args.steps                     # launches per step
            by, bf = by / lps, bf / lps
            e["GB_per_s"] = round(by / (per * 1e-3) / 1e9, 1)
            e["hbm_frac"] = round(by / (per * 1e-3) / 1e9 / hbm_peak, 3)
            if bf:
                e["Gbutterfly_per_s"] = round(bf / (per * 1e-3) / 1e9, 1)
        kernels[k_] = e
    fam = max((k for k in prof if k in S["fam"]), key=lambda k: prof[k][1], default=None)
    traffic = None     # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture
    if fam is not None and S.get("traffic"):
        try:
            with open(os.path.join(ROOT, "profiles", S["traffic"][0])) as fh:
                traffic = json.load(fh).get(S["traffic"][1].get(fam))
        except OSError:
            traffic = None
    if fam is not None:
        e = kernels[fam]
        if S["peak"] == "hbm":
            roof = {"bound": "hbm", "kernel": fam, "achieved": e["GB_per_s"], "peak": hbm_peak, "unit": "GB/s",
                    "frac": e["hbm_frac"], "traffic": traffic, "peak_source": peak_src,
                    "algorithmic_bytes": int(S["fam"][fam][0] * args.steps / prof[fam][0])}
        else:
            pk = alu32 if S["peak"] == "alu32" else gold8
            src = (f"derived: {nsm} SMs x 16 butterflies/clk/SM (fmaheavy: IMAD.HI 4 + 2 x IMAD 2 cycles per warp) "
                   f"x {sm_mhz_max:.0f} MHz" if S["peak"] == "alu32" else
                   "measured on this GPU: register-resident gold.cuh 8-point Goldilocks DIF rate (mm_probe_butterfly "
                   "65; no loads, shift twiddles only: an upper bound the passes' table products cannot reach)")
            ach = e["Gbutterfly_per_s"] * 1e9
            roof = {"bound": "alu", "kernel": fam, "achieved": e["Gbutterfly_per_s"], "peak": round(pk / 1e9, 1),
                    "unit": "Gbutterfly/s", "frac": round(ach / pk, 3), "traffic": traffic, "hbm_frac": e["hbm_frac"],
                    "algorithmic_bytes": int(S["fam"][fam][0] * args.steps / prof[fam][0]),
                    "peak_source": src}

    # e2e: upload the step's inputs from pinned host memory, run, read the result back
    hin = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True).copy_(t) for t in S["inputs"]]
    hout = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in S["outputs"]]

    def e2e_step():
        for h, d in zip(hin, S["inputs"]):
            d.copy_(h, non_blocking=True)
        step()
        for h, d in zip(hout, S["outputs"]):
            h.copy_(d, non_blocking=True)
    e2e_api = "device call between explicit pinned-host copies"
    if "e2e_host" in S:   # the library's own host-buffer entry point
        host_fn, e2e_api = S["e2e_host"]

        def e2e_step():
            host_fn(hin, hout)
    e2e_steps = max(1, min(args.steps, 5))
    ms_e2e = timed(e2e_step, e2e_steps, 1, world) / e2e_steps
    if "e2e_host" in S and world == 1:   # the host result must equal the device result
        step()
        torch.cuda.synchronize()
        for h, d in zip(hout, S["outputs"]):
            if not torch.equal(h, d.cpu()):
                raise SystemExit("e2e: host-buffer result differs from the device result")
    h2d = sum(t.numel() * t.element_size() for t in S["inputs"])
    d2h = sum(t.numel() * t.element_size() for t in S["outputs"])
    variants = {}
    for nm, fn, bpe in S.get("variants", []):
        msv = timed(fn, args.steps, args.warmup, world) / args.steps
        gbs = S["units"] * bpe / (msv * 1e-3) / 1e9
        variants[nm] = {"Gelem_per_s": round(S["units"] / (msv * 1e-3) / 1e9, 1), "ms": round(msv, 4),
                        "hbm_frac": round(gbs / hbm_peak, 3)}
    time.sleep(0.02)
    clk.__exit__(None, None, None)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_config(which, args.cpu_seconds)
    if rank != 0:
        return
    cfg = {"workload": S["workload"], "config": which.upper(),
           "l2": "L2 flushed (256 MiB write) before every timed step, outside its events" if S["flush"]
           else "inputs > 126 MB L2 (no flush needed)",
           "parallelism": f"dp{world} (each rank its own copy of the config's work, no collective)"}
    if variants:
        cfg["variants"] = variants
    line = {
        "metric": S["metric"], "value": round(value, 2), "unit": S["unit"], "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": S["dtype"],
        "data": "synthetic (seeded counter-based SplitMix64, uniform, generated in HBM)", "config": cfg,
        "e2e": {"value": round(world * S["units"] / (ms_e2e * 1e-3) / S["scale"], 2), "unit": S["unit"],
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(ms_e2e, 4), "api": e2e_api},
        "gpu_launches": int(cnt["n1"] - cnt["n0"]), "roofline": roof, "kernels": kernels,
        "clocks": clk.summary(), "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def cpu_baseline_config(which: str, budget_s: float) -> dict:
    ci = cpu_info()
    allc = ci["cores"]
    fn = {"c1": lambda t: oracle_c1(t, budget_s / 2), "c2": oracle_c2,
          "c4": lambda t: oracle_c4(min(t, 8)), "c5": oracle_c5}[which]
    one, many = fn(1), fn(allc)
    return {"value": many["value"], "unit": many["unit"], "cores": many["cores"], "kind": "oracle",
            "cpu_model": ci["model"], "sample": {k: v for k, v in many.items() if k not in ("value", "unit")},
            "single_thread": one, "all_cores": many}


def run_reference_config(args, rank):
    """--impl reference --config cX: the oracle on the host cores, one bounded
    sample of the config's work per step."""
    if rank != 0:
        return
    ci = cpu_info()
    nth = ci["cores"]
    fn = {"c1": lambda: oracle_c1(nth, 2.0), "c2": lambda: oracle_c2(nth),
          "c4": lambda: oracle_c4(min(nth, 8), k=22), "c5": lambda: oracle_c5(nth, limbs=1 << 18)}[args.config]
    for _ in range(args.warmup):
        fn()
    vals, walls, samp = [], [], None
    for _ in range(args.steps):
        r = fn()
        vals.append(r["value"])
        walls.append(r["wall_s"])
        samp = {k: v for k, v in r.items() if k not in ("value", "unit")}
    val = statistics.mean(vals)
    unit = r["unit"]
    line = {
        "impl": "reference", "metric": {"c1": "NTT Gbutterfly/s", "c2": "modmul Gelem/s", "c4": "NTT Gbutterfly/s",
                                        "c5": "int_mul Mbit/s"}[args.config],
        "value": round(val, 6), "unit": unit, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * statistics.mean(walls), 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64" if args.config in ("c4", "c5") else "u32",
        "data": "synthetic (seeded SplitMix64)",
        "config": {"workload": f"{args.config.upper()} oracle sample per step: {samp}", "config": args.config.upper(),
                   "parallelism": f"{nth} CPU threads"},
        "cpu_baseline": {"value": round(val, 6), "unit": unit, "cores": samp.get("cores", nth), "kind": "oracle",
                         "cpu_model": ci["model"], "sample": samp},
        "e2e": {"value": round(val, 6), "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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
    ap.add_argument("--cpu-seconds", type=float, default=6.0)
    ap.add_argument("--cpu-legs", default="c2,c4,c5", help="other configs timed on the oracle beside C3")
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4", "c5"],
                    help="BASELINE config of the printed line (default: the C3 headline with the others in extra)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        if args.config != "c3":
            run_reference_config(args, rank)
        else:
            run_reference(args, world, rank)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # launched without torchrun: start N ranks ourselves (one per GPU)
        import socket
        import torch
        if torch.cuda.device_count() < args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus}: only {torch.cuda.device_count()} CUDA devices visible")
        so = socket.socket()
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
        so.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        raise SystemExit(subprocess.call(cmd))
    # NCCL INIT lines (rank count, transports) to stderr so the driver can check them
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    world, rank, local = dist_setup()
    if world != args.gpus:
        raise SystemExit(f"bench.py --gpus {args.gpus} but WORLD_SIZE = {world}")
    try:
        if args.config != "c3":
            run_config(args, world, rank, local)
        else:
            run_ours(args, world, rank, local)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
