#!/bin/bash
# Round evidence refresh on one B200 (run under gpurun from the repo root):
#   GPU tests, the default bench line, the ncu launch list of a short bench,
#   and one `ncu --set full` capture per config's dominant kernel(s).
# Usage: tools/refresh_profiles.sh TAG   (outputs gpurun_out/TAG_*)
tag=${1:-rXX}
out=gpurun_out
python -m paper_2505_12425_b200._build > /dev/null
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $out/${tag}_pytest_gpu.log 2>&1
echo "pytest rc=$?"; tail -1 $out/${tag}_pytest_gpu.log
timeout 900 python bench.py > $out/${tag}_bench_full.json 2> $out/${tag}_bench_full.err
echo "bench rc=$?"
short="--steps 2 --warmup 1 --no-cpu --no-e2e --no-verify --soak 0"
timeout 600 python bench.py $short > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    -k "regex:resize_|warp_|gray_u8|k_|jpeg_" --log-file $out/${tag}_launches.csv \
    python bench.py $short > $out/${tag}_ncu_launch.log 2>&1
echo "launch list rc=$?"
for op in resize fused affine persp gray graybatch jpeg r720 r1080; do
  n=1; kre="regex:resize_|warp_|gray_u8"
  [ $op = resize ] && n=2
  [ $op = gray ] && n=4
  [ $op = jpeg ] && n=10 && kre="regex:k_spec|k_round|k_write|jpeg_idct_batch|jpeg_color_batch"
  timeout 300 python tools/profile_ops.py --op $op --reps 1 > /dev/null 2>&1 && \
    timeout 900 ncu --set full --clock-control none --import-source on -k "$kre" -c $n \
      -o $out/${tag}_$op python tools/profile_ops.py --op $op --reps 1 > $out/${tag}_ncu_$op.log 2>&1
  echo "ncu $op rc=$?"
done
