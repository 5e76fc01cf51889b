T=r2; O=gpurun_out
timeout 800 python -m pytest tests -m gpu -q > $O/gputest_final.log 2>&1; echo "pytest rc=$?"; tail -1 $O/gputest_final.log
python bench.py > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err; echo "c4 rc=$?"
for w in c5-weak c5-strong; do python bench.py --workload $w --no-cpu-baseline > $O/${T}_bench_$w.json 2> $O/${T}_bench_$w.err; echo "$w rc=$?"; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file $O/${T}_launches_c4.csv python bench.py --steps 2 --warmup 3 --no-ncu --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
ncu --set full --import-source on --clock-control none -k regex:^k_fb -c 3 -o /tmp/${T}_c4 -f python bench.py --ncu-child --workload c4 > $O/ncu_c4.out 2>&1; echo "ncu c4 rc=$?"
python tools/ncu_summary.py /tmp/${T}_c4.ncu-rep > $O/${T}_ncu_c4_summary.txt 2>&1
for i in 0 1 2; do python tools/ncu_lines.py /tmp/${T}_c4.ncu-rep $i 40 > $O/${T}_ncu_c4_lines$i.txt 2>&1; done
ncu -i /tmp/${T}_c4.ncu-rep --page raw --csv > $O/${T}_ncu_c4_raw.csv 2>/dev/null
python -m tests.parity_report > $O/${T}_parity_errors.txt 2>&1; echo "parity rc=$?"
