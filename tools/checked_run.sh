#!/bin/bash
# The bounds-checked build (device-side FV_CHECK asserts on every TMA copy's
# source / shared-memory destination and on the staged kernels' shared-memory
# reads) run over the small-shape driver and the GPU parity tests. This is the
# stand-in for compute-sanitizer, which is closed on the GPU pool.
# Usage (under gpurun, from the repo root): bash tools/checked_run.sh TAG
tag=${1:-checked}
out=gpurun_out
python -m paper_2505_12425_b200._build --checked > /dev/null || exit 1
lib=$PWD/paper_2505_12425_b200/lib/libfovea_b200_checked.so
export FOVEA_B200_LIB=$lib FOVEA_B200_KNOBS_LIB=$lib
timeout 600 python tools/sanitize_ops.py > $out/${tag}_ops.txt 2>&1
echo "ops rc=$?"; tail -1 $out/${tag}_ops.txt
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider \
  -k "not jpeg and not full_batch and not exhaustive" > $out/${tag}_pytest.txt 2>&1
echo "pytest rc=$?"; tail -2 $out/${tag}_pytest.txt
grep -c "FV_CHECK failed" $out/${tag}_ops.txt $out/${tag}_pytest.txt
