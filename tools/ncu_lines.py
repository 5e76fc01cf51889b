"""Per-source-line warp-instruction counts and stall samples from an ncu report
(--import-source on, -lineinfo build), deduplicated per SASS instruction: an
instruction inlined from a helper is charged to its outermost call-site line in
the kernel's own source file (the highest line number among the lines ncu lists
it under, helpers being defined above their callers).

    python tools/ncu_lines.py REPORT.ncu-rep LAUNCH_INDEX [top] [regions.json]
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

rep, idx = sys.argv[1], int(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--launch-skip", str(idx), "--launch-count", "1"], capture_output=True, text=True).stdout
by_addr = {}  # address -> (inst, samples, sass text)
lines_of = defaultdict(set)
src = {}
cur = None
fname = ""
main_file = None
for line in txt.splitlines():
    if line.startswith('"File Path"'):
        fname = line.split(",")[1].strip('"').split("/")[-1]
        if main_file is None:
            main_file = fname
        continue
    r = next(csv.reader(io.StringIO(line)))
    if len(r) < 9 or r[0] == "Line No":
        continue
    if r[0]:
        cur = (fname, int(r[0]))
        src[cur] = r[1][:100]
        continue
    if r[2].startswith("0x") and cur is not None:
        try:
            n = int(float(r[7])); s = int(float(r[4]))
        except ValueError:
            continue
        by_addr[r[2]] = (n, s, r[3].strip())
        lines_of[r[2]].add(cur)
inst = defaultdict(int)
samp = defaultdict(int)
for a, (n, s, _) in by_addr.items():
    ls = lines_of[a]
    own = [l for l in ls if l[0] == main_file]
    key = max(own) if own else max(ls)
    inst[key] += n
    samp[key] += s
total = sum(inst.values())
tsamp = sum(samp.values())
print(f"total warp-instructions {total:,}  stall samples {tsamp:,}")
for k, v in sorted(inst.items(), key=lambda x: -x[1])[:top]:
    print(f"{v / total * 100:5.1f}%  {v:>12,}  samp {samp[k] / max(tsamp, 1) * 100:5.1f}%  {k[0]}:{k[1]}  {src.get(k, '')}")
if len(sys.argv) > 4:
    regions = json.load(open(sys.argv[4]))  # {"name": [lo, hi], ...} line ranges of the main file
    for name, (lo, hi) in regions.items():
        v = sum(n for k, n in inst.items() if k[0] == main_file and lo <= k[1] <= hi)
        s = sum(n for k, n in samp.items() if k[0] == main_file and lo <= k[1] <= hi)
        print(f"region {name:24s} {v / total * 100:5.1f}% inst  {s / max(tsamp, 1) * 100:5.1f}% samples")
