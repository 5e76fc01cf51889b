"""Summarise an ncu --set full report: per-kernel duration, DRAM bytes, throughput,
IPC, smem wavefronts, issue-active %, MUFU (xu pipe) and FMA pipe utilisation.  Writes profiles/ncu_traffic.json (dram bytes per launch of
each kernel name, averaged) and prints a table."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out_json = sys.argv[2] if len(sys.argv) > 2 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
H = {h: i for i, h in enumerate(hdr)}
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
units = rows[1]
SCALE = {"": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1, "nsecond": 1,
         "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "s": 1e9, "second": 1e9, "%": 1,
         "inst": 1, "register/thread": 1, "cycle": 1}


def scale(w):
    u = units[H[w]].strip()
    return SCALE.get(u, 1.0)


agg = defaultdict(list)
for r in rows[2:]:
    name = r[H["Kernel Name"]]
    short = name.split("(")[0].replace("void ", "")
    if "k_fb<" in name:
        tmpl = name[name.index("<"):name.index(">") + 1]
        short = "k_fb" + tmpl
    vals = {}
    for w in want:
        if w in H:
            try:
                vals[w] = float(r[H[w]].replace(",", "")) * scale(w)  # bytes, ns
            except ValueError:
                vals[w] = None
    agg[short].append(vals)
summary = {}
for k, lst in agg.items():
    avg = {w: sum(v[w] for v in lst if v.get(w) is not None) / max(1, len(lst)) for w in want if w in H}
    summary[k] = avg
    dur_ms = avg["gpu__time_duration.sum"] / 1e6 if "gpu__time_duration.sum" in avg else None
    by = avg.get("dram__bytes_read.sum", 0) + avg.get("dram__bytes_write.sum", 0)
    print(f"{k:36s} n={len(lst)} dur={dur_ms:.3f}ms dram={by/1e9:.3f}GB ({by/1e9/(dur_ms/1e3):.0f} GB/s) "
          f"dram%={avg.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} "
          f"sm%={avg.get('sm__throughput.avg.pct_of_peak_sustained_elapsed', 0):.1f} "
          f"inst={avg.get('smsp__inst_executed.sum', 0)/1e6:.0f}M smem_wf={avg.get('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 0)/1e6:.0f}M "
          f"conf={avg.get('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 0)/1e6:.0f}M "
          f"issue%={avg.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.1f} "
          f"mufu%={avg.get('sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active', 0):.1f} "
          f"fma%={avg.get('sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 0):.1f} regs={avg.get('launch__registers_per_thread', 0):.0f}")
if out_json:
    names = {}
    for k in summary:
        if k.startswith("k_fb<") and k.endswith(", 1024>") and k.split(",")[1].strip() in ("0", "4"):
            names[k] = "k_fb_bwd[G=1]" if k.startswith("k_fb<1") else "k_fb_fwd[G=1]"
    traffic = {}
    for k, avg in summary.items():
        key = names.get(k, k)
        traffic[key] = avg.get("dram__bytes_read.sum", 0) + avg.get("dram__bytes_write.sum", 0)
    os.makedirs(os.path.dirname(out_json), exist_ok=True)
    with open(out_json, "w") as f:
        json.dump(traffic, f, indent=1)
