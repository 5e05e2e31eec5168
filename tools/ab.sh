#!/bin/bash
# A/B of two plan variants on the same box
for v in "" "DQMC_IB_E_NONE=1" "" "DQMC_IB_E_NONE=1"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k: round(v['ms'],2) for k,v in d['passes'].items() if v['ms']>1})"
done
