#!/bin/bash
# Round-end evidence on one B200 (under gpurun, from the repo root):
#   tools/refresh_profiles.sh TAG, then smoke(), the two fuzz sweeps and the
#   bounds-checked build's run. Usage: bash tools/final_evidence.sh TAG
tag=${1:-rXX}
out=gpurun_out
bash tools/refresh_profiles.sh $tag
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/${tag}_smoke.txt 2>&1
echo "smoke rc=$?"
( echo "\$ python tools/fuzz_warp.py --cases 20000 --seed 2026"; timeout 1500 python tools/fuzz_warp.py --cases 20000 --seed 2026; echo "rc=$?" ) > $out/${tag}_fuzz_warp.txt 2>&1
tail -2 $out/${tag}_fuzz_warp.txt
( echo "\$ python tools/fuzz_resize.py --cases 20000 --seed 2026"; timeout 1500 python tools/fuzz_resize.py --cases 20000 --seed 2026; echo "rc=$?" ) > $out/${tag}_fuzz_resize.txt 2>&1
tail -2 $out/${tag}_fuzz_resize.txt
bash tools/checked_run.sh ${tag}_checked
