"""Debug helper: exercise bench.ClockSampler for ~0.5 s under a GPU load."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench

x = torch.randn(8192, 8192, device="cuda")
with bench.ClockSampler(0) as clk:
    time.sleep(0.1)
    clk.mark(True)
    t0 = time.time()
    while time.time() - t0 < 0.5:
        y = x @ x
    torch.cuda.synchronize()
    clk.mark(False)
print("nvml", clk.nvml is not None, "samples", len(clk.samples), "lines", len(clk.lines), clk.lines[:2])
print(clk.summary())
try:
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(0)
    print("clock", pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
    print("reasons", pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
except Exception as e:
    print("nvml error", repr(e))
