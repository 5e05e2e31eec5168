#!/bin/bash
# one short bench run, one summary line: ms/step, e2e ms, per-pass ms
env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu > gpurun_out/bb.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bb.log').read().strip().splitlines()[-1]); print('$*', round(d['ms_per_step'],2), round(d['e2e']['ms_per_step'],2), {k: round(v['ms'],2) for k,v in d['passes'].items() if v['ms']>0.1})" || tail -5 gpurun_out/bb.log
