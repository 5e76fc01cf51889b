#!/bin/bash
# A/B timing of alternative builds of libfb in one GPU session, interleaved:
#   LIBS="paper_2112_00709_b200/libfb.so paper_2112_00709_b200/libfb_x.so" REPS=3 tools/ab_libs.sh [c3] [c4]
cd "$(dirname "$0")/.."
for r in $(seq ${REPS:-2}); do
  for lib in ${LIBS}; do
    echo "== rep $r $lib"
    FBX_LIB=$lib timeout 300 python tools/quick_time.py "$@" 2>&1 | grep -E "profile|C3|C4"
  done
done
