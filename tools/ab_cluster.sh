#!/bin/bash
# A/B timing of the denominator kernels: legacy (one CTA per sequence) vs cluster configs.
cd "$(dirname "$0")/.."
for cfg in "legacy" "2,2:1024" "2,2:512" ${EXTRA_CFGS}; do
  if [ "$cfg" = "legacy" ]; then export FBX_NO_CLUSTER=1; unset FBX_CLUSTER FBX_CLUSTER_T
  else unset FBX_NO_CLUSTER; export FBX_CLUSTER=${cfg%%:*} FBX_CLUSTER_T=${cfg##*:}; fi
  echo "== $cfg"
  timeout 300 python tools/quick_time.py ${WHICH:-c3 c4} 2>&1 | grep -E "profile|C3|C4"
done
