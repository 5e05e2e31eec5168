#!/bin/bash
# Round evidence on one B200: bench line, reference arm, ncu launch list, ncu --set full of every kernel
# of one n=24 call, and of one sparse-engine call.
# usage (under gpurun): bash tools/evidence.sh TAG
T=${1:-rX}
set -x
timeout 600 python bench.py > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$T.json 2> gpurun_out/bench_ref_$T.err
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$T.csv \
    python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_launch_$T.log 2>&1
timeout 300 python tools/run_once.py 24 > /dev/null 2>&1 && \
  timeout 1500 ncu --set full --clock-control none --import-source on -c 12 -o gpurun_out/prof_$T \
    python tools/run_once.py 24 > gpurun_out/ncu_full_$T.log 2>&1
timeout 300 python tools/run_sparse_once.py 20 0.1 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sp_ -c 12 -o gpurun_out/prof_sparse_$T \
    python tools/run_sparse_once.py 20 0.1 > gpurun_out/ncu_sparse_$T.log 2>&1
tail -c 300 gpurun_out/bench_$T.json; tail -c 300 gpurun_out/bench_ref_$T.json; ls -la gpurun_out/prof_$T.ncu-rep
