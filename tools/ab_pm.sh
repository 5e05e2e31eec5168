#!/bin/bash
# A/B: piece-major group 0 vs the contiguous-tile layout
for v in "X=1" "DQMC_NO_PM=1" "X=1" "DQMC_NO_PM=1"; do
  env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/ab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab.log').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), {k: round(v['ms'],2) for k,v in d['passes'].items() if v['ms']>0.1})" || tail -5 gpurun_out/ab.log
done
