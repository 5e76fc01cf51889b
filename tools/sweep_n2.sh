#!/bin/bash
# Env-var sweeps of the schedule shape (slice length caps) on the N2 and C4 bench workloads.
run() { env "$@" python bench.py --workload $W --no-cpu-baseline --no-ncu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$W $*', round(d['ms_per_step'],3), {k:round(v['avg_ms'],3) for k,v in d['kernels'].items() if 'k_fb' in k})"; }
W=paper
run FBX_CLUSTER_LMAX=32
run FBX_CLUSTER_LMAX=48
run FBX_CLUSTER_LMAX=64
run FBX_CLUSTER_LMAX=96
W=c4
run X=1
run FBX_LMAX=32
run FBX_LMAX=48
run FBX_LMAX=64
