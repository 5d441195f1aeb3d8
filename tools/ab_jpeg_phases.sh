#!/bin/bash
# GPU phase times of the JPEG path for alternative builds: tools/ab_jpeg_phases.sh lib1.so lib2.so ...
for lib in "$@"; do
  echo "== $lib"
  FOVEA_B200_LIB=$lib FV_JPEG_TIMING=1 timeout 300 python bench.py --ops jpeg --no-cpu --no-e2e --steps 20 --warmup 5 \
    2> gpurun_out/phases.log > /dev/null
  python tools/jpeg_phase_avg.py gpurun_out/phases.log 6 | grep -e "gpu spec" -e "gpu round" -e "gpu scan" -e "changed"
  grep "changed per round" gpurun_out/phases.log | tail -1
done
