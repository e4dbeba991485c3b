ls /sys/devices/system/node/ | grep node; for n in /sys/devices/system/node/node*; do echo $n $(cat $n/cpulist); done
python - <<'PY'
import os, torch
print("affinity", sorted(os.sched_getaffinity(0)))
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0),'pci_bus_id') else None
print("props", torch.cuda.get_device_properties(0))
import pynvml
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
pci = pynvml.nvmlDeviceGetPciInfo(h); print("bus", pci.busId)
try:
    print("cpu affinity mask", [hex(x) for x in pynvml.nvmlDeviceGetCpuAffinity(h, 8)])
except Exception as e: print("aff err", e)
b = pci.busId.decode() if isinstance(pci.busId, bytes) else pci.busId
b = b.lower()[4:] if len(b) > 12 else b.lower()
import glob
for p in glob.glob("/sys/bus/pci/devices/*"):
    if p.endswith(b[-7:]):
        print(p, open(p + "/numa_node").read().strip())
PY
