#!/bin/bash
# device-resident ms per call and cells/s by n (the DESIGN.md throughput table)
for n in 20 21 22 23 24 25; do
  timeout 600 python bench.py --nvars $n --steps 5 --warmup 3 --no-cpu > gpurun_out/bs.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/bs.log').read().strip().splitlines()[-1]); print($n, d['config']['plan']['r'][:d['config']['plan']['m']], round(d['ms_per_step'],2), '%.3g' % d['value'])" || tail -3 gpurun_out/bs.log
done
