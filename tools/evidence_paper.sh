#!/bin/bash
# Re-capture the N2 (paper shape) bench line and its ncu --set full summary.   TAG=r2 tools/evidence_paper.sh
cd "$(dirname "$0")/.."
T=${TAG:-r2}; O=gpurun_out
python bench.py --workload paper --no-cpu-baseline > $O/${T}_bench_paper.json 2> $O/${T}_bench_paper.err; echo "paper rc=$?"
ncu --set full --import-source on --clock-control none -k regex:^k_fb -c 3 -o /tmp/${T}_paper -f \
    python bench.py --ncu-child --workload paper > $O/ncu_paper.out 2>&1; echo "ncu paper rc=$?"
python tools/ncu_summary.py /tmp/${T}_paper.ncu-rep > $O/${T}_ncu_paper_summary.txt 2>&1
for i in 0 1 2; do python tools/ncu_lines.py /tmp/${T}_paper.ncu-rep $i 40 > $O/${T}_ncu_paper_lines$i.txt 2>&1; done
ncu -i /tmp/${T}_paper.ncu-rep --page raw --csv > $O/${T}_ncu_paper_raw.csv 2>/dev/null
