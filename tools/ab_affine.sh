#!/bin/bash
# A/B of affine builds: tools/ab_affine.sh lib1.so lib2.so ... (cfg2 f32 and u8 timing, bit-equality vs the dst-tiled kernel)
for lib in "$@"; do
  echo "== $lib"
  FOVEA_B200_LIB=$lib timeout 300 python tools/affine_perf.py --reps 20 | grep -v dst_tiles
done
