#!/bin/bash
# A/B timing of the denominator kernels on C3 / C4: one CTA per utterance (default)
# vs cluster-batched configurations "C,S" or "C,S,1" (no-p), e.g.
#   EXTRA_CFGS="4,4,1 4,2" tools/ab_cluster.sh
cd "$(dirname "$0")/.."
for cfg in "default" "2,2" ${EXTRA_CFGS}; do
  if [ "$cfg" = "default" ]; then unset FBX_CLUSTER; else export FBX_CLUSTER=$cfg; fi
  echo "== $cfg"
  timeout 300 python tools/quick_time.py ${WHICH:-c3 c4} 2>&1 | grep -E "profile|C3|C4"
done
