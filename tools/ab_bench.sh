#!/bin/bash
# A/B timing of alternative builds of the same ABI: tools/ab_bench.sh OPS lib1.so lib2.so ...
ops=$1; shift
for lib in "$@"; do
  echo "== $lib"
  FOVEA_B200_LIB=$lib timeout 300 python bench.py --ops "$ops" --no-cpu --no-e2e --steps ${STEPS:-10} | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); [print(k, [(x['kernel'], x['ms'], x['frac']) for x in v['kernels']]) for k,v in d['ops'].items()]"
done
