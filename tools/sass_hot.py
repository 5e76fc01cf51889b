"""Hot SASS regions of one kernel from `ncu -i R --page source --csv --print-source sass`:
prints instructions with their executed warp-instruction counts, folding runs of
instructions whose count is below a threshold.   python tools/sass_hot.py FILE.csv [min_frac]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
H = {h: i for i, h in enumerate(hdr)}
tot = 0
ins = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    n = int(r[H["Instructions Executed"]] or 0)
    smp = int(r[H["Warp Stall Sampling (All Samples)"]] or 0)
    ins.append((r[H["Address"]][-5:], r[H["Source"]].strip(), n, smp))
    tot += n
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.002
print(f"total warp-instructions {tot:,}")
skipped = 0
for a, s, n, smp in ins:
    if n >= thr * tot / 100:
        if skipped:
            print(f"   ... {skipped} cold")
            skipped = 0
        print(f"{a} {n/tot*100:6.3f}% {n:>12,} smp {smp:>6}  {s}")
    else:
        skipped += 1
