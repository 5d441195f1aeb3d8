#!/bin/bash
# A/B of perspective builds: tools/ab_persp.sh lib1.so lib2.so ... (per-class timings + cfg3 1-LSB check)
for lib in "$@"; do
  echo "== $lib"
  FOVEA_B200_LIB=$lib timeout 300 python tools/persp_classes.py
  FOVEA_B200_LIB=$lib timeout 300 python tools/persp_perf.py --reps 10 | grep -v r01
done
