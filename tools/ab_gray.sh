#!/bin/bash
for lib in "$@"; do echo "== $lib"; FOVEA_B200_LIB=$lib timeout 300 python bench.py --ops gray --no-cpu --no-e2e --steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); [print(k, [(x['kernel'][:30], x['ms'], x['frac']) for x in v['kernels']], v.get('verified')) for k,v in d['ops'].items()]"; done
