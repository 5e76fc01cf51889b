#!/bin/bash
# Env-var sweeps of the schedule shape (slice length caps) on the N2 and C4 bench workloads:
#   W=paper bash tools/sweep_n2.sh "FBX_CLUSTER_LMAX=24" "FBX_CLUSTER_LMAX=32" …
run() { env "$@" python bench.py --workload $W --no-cpu-baseline --no-ncu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$W $*', round(d['ms_per_step'],3), {k:round(v['avg_ms'],3) for k,v in d['kernels'].items() if 'k_fb' in k})"; }
W=${W:-paper}
if [ $# -eq 0 ]; then set -- X=1; fi
for cfg in "$@"; do run $cfg; done
