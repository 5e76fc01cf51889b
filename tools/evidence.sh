#!/bin/bash
# One GPU session that regenerates the round's committed evidence under gpurun_out/:
# bench lines for every workload, the reference arm, the ncu launch list of the
# default bench command, one `ncu --set full` capture per headline workload and
# the compute-sanitizer logs.   TAG=r2 tools/evidence.sh
cd "$(dirname "$0")/.."
T=${TAG:-r2}
O=gpurun_out
python bench.py > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err; echo "c4 rc=$?"
for w in c2 c3 paper c5-weak c5-strong viterbi viterbi-paper; do
  python bench.py --workload $w --no-cpu-baseline > $O/${T}_bench_$w.json 2> $O/${T}_bench_$w.err; echo "$w rc=$?"
done
python bench.py --impl reference > $O/${T}_bench_reference.json 2> $O/${T}_bench_reference.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/${T}_launches_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-ncu --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
# full captures stay on the box (/tmp: gpurun copies back at most 64 MiB); their summaries come back
for w in c4 paper; do
  ncu --set full --import-source on --clock-control none -k regex:^k_fb -c 3 -o /tmp/${T}_$w -f \
      python bench.py --ncu-child --workload $w > $O/ncu_$w.out 2>&1; echo "ncu $w rc=$?"
  python tools/ncu_summary.py /tmp/${T}_$w.ncu-rep > $O/${T}_ncu_${w}_summary.txt 2>&1
  for i in 0 1 2; do python tools/ncu_lines.py /tmp/${T}_$w.ncu-rep $i 40 > $O/${T}_ncu_${w}_lines$i.txt 2>&1; done
  ncu -i /tmp/${T}_$w.ncu-rep --page raw --csv > $O/${T}_ncu_${w}_raw.csv 2>/dev/null
done
python -m tests.parity_report > $O/${T}_parity_errors.txt 2>&1; echo "parity rc=$?"
# compute-sanitizer (closed on the GPU pool since round 2; SAN=1 to run it where it is available)
if [ -n "$SAN" ]; then
  for t in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $t --log-file $O/${T}_sanitizer_$t.log python tools/sanitize.py > $O/san_$t.out 2>&1
    echo "$t rc=$? $(tail -1 $O/${T}_sanitizer_$t.log)"
  done
fi
