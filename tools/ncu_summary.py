"""Summarise ncu outputs into small text/JSON files under profiles/.

  python tools/ncu_summary.py launches <launches.csv> <out.txt>
      per-kernel-family launch counts, mean device time and share of the
      launch list (cold-cache, serialised: compare SHARES, not absolutes).
  python tools/ncu_summary.py full <report.ncu-rep> <out.txt> [traffic.json]
      key metrics of each profiled kernel (time, DRAM bytes, issue / pipe
      utilisation, bank conflicts, occupancy, top stall reasons); optionally
      writes {kernel family: dram bytes per launch} for bench.py's roofline.
"""
from __future__ import annotations

import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict


def family(name: str) -> str:
    m = re.search(r"(k_[a-z0-9_]+)", name)
    base = m.group(1) if m else name.split("(")[0][:60]
    inv = ""
    if base in ("k_rows", "k_cols"):
        t = re.search(r"<[^,]+,\s*(?:\(int\))?\s*(\d+),\s*(?:\(bool\))?\s*(\w+)", name)
        if t:
            inv = "_inv" if t.group(2) in ("1", "true") else "_fwd"
            inv += f"_L2^{t.group(1)}"
    elif base == "k_rows_pmul":
        t = re.search(r"<[^,]+,\s*(?:\(int\))?\s*(\d+)", name)
        if t:
            inv = f"_L2^{t.group(1)}"
    return base + inv


def scope_name(fam: str) -> str:
    """ncu family -> the LaunchScope name bench.py reports."""
    fast = {"k_col_fwd": "ntt_cols_fwd", "k_col_inv": "ntt_cols_inv", "k_row_pmul": "pmul_rows_fourstep"}
    if fam in fast:   # the specialised 2^16 = 256 x 256 kernels (ntt_fast32.cu)
        return fast[fam]
    if fam.startswith("k_cols_fwd"):
        return "ntt_cols_fwd"
    if fam.startswith("k_cols_inv"):
        return "ntt_cols_inv"
    if fam.startswith("k_rows_fwd"):
        return "ntt_rows_fwd"
    if fam.startswith("k_rows_inv"):
        return "ntt_rows_inv"
    if fam.startswith("k_rows_pmul"):
        return "pmul_rows"
    return fam


def scope_of(name: str) -> str:
    fam = scope_name(family(name))
    if fam == "pmul_rows":   # epilogue template argument: 1/2 = four-step twiddle, 8 = single pass
        m = re.search(r",\s*(\d+)>\(", name)
        fam = "pmul_rows_fourstep" if m and m.group(1) in ("1", "2") else "pmul_rows_single"
    return fam


def launches(path: str, out: str):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        v = float(r[vi].replace(",", ""))
        unit = r[h.index("Metric Unit")] if "Metric Unit" in h else "nsecond"
        ms = v / 1e6 if unit.startswith("ns") else (v / 1e3 if unit.startswith("us") else v)
        f = family(r[ki])
        agg[f][0] += 1
        agg[f][1] += ms
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list summary: {path}", "# family launches mean_ms total_ms share"]
    for f, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{f:45s} {n:6d} {ms / n:10.4f} {ms:10.4f} {ms / tot:7.3f}")
    # the list also holds the generator, probe, e2e-chunk and warm-up launches:
    # the shares to compare with bench.py's "kernels" are those within the C3 step
    step = [f for f in ("k_col_fwd", "k_row_pmul", "k_col_inv") if f in agg]
    if step:
        st = sum(agg[f][1] for f in step)
        lines.append("# shares within the C3 step kernels (compare bench.py kernels[*].share):")
        for f in step:
            lines.append(f"#   {f:20s} {agg[f][1] / st:7.3f}")
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_write.sum",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
]


def full(rep: str, out: str, traffic_json: str | None = None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, data = rows[0], rows[1], rows[2:]
    lines = [f"# ncu --set full summary: {rep}"]
    traffic = defaultdict(list)
    for r in data:
        name = r[h.index("Kernel Name")]
        lines.append(f"== {family(name)}   [{name[:110]}]")
        for w in WANT:
            if w in h:
                i = h.index(w)
                lines.append(f"   {w:60s} {r[i]:>18s} {units[i]}")
        stalls = []
        for i, k in enumerate(h):
            if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        lines.append("   top stalls: " + ", ".join(f"{k}={int(v)}" for v, k in stalls[:6]))
        try:
            rd = float(r[h.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[h.index("dram__bytes_write.sum")].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(units[h.index("dram__bytes_read.sum")], 1)
            wr *= scale.get(units[h.index("dram__bytes_write.sum")], 1)
            traffic[scope_of(name)].append(rd + wr)
        except (ValueError, KeyError):
            pass
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if traffic_json:
        avg = {k: sum(v) / len(v) for k, v in traffic.items()}
        json.dump(avg, open(traffic_json, "w"), indent=1)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
