#!/bin/bash
A=paper_2505_12425_b200/lib/ab
for v in "$@"; do
  echo "== $v"
  FOVEA_B200_LIB=$PWD/$A/$v.so FOVEA_B200_KNOBS_LIB=$PWD/$A/${v}_k.so timeout 300 python tools/generic_resize_perf.py
  FOVEA_B200_LIB=$PWD/$A/$v.so timeout 300 python bench.py --ops fused --no-cpu --no-e2e --steps 10 | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); [print(k, [(x['kernel'], x['ms'], x['frac']) for x in v['kernels']]) for k,v in d['ops'].items()]"
done
