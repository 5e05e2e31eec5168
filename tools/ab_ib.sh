#!/bin/bash
# A/B of the in-block axis split between passes C and D (DQMC_IB_C mask)
for v in "X=1" "DQMC_NO_SPARSE=1" "DQMC_IB_C=3" "DQMC_IB_C=7" "DQMC_IB_C=31" "DQMC_IB_C=0"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), {k: round(v['ms'],2) for k,v in d['passes'].items() if v['ms']>1})"
done
