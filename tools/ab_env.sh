#!/bin/bash
# A/B of env-selected plan variants on one box: tools/ab_env.sh "" "VAR=1" ...
for v in "$@"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('[$v]', round(d['ms_per_step'],2), {k: round(v['ms'],2) for k,v in d['passes'].items() if v['ms']>0.5})"
done
