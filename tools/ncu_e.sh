#!/bin/bash
# ncu --set full of one pass-E launch at n=24 (under gpurun): bash tools/ncu_e.sh TAG [LIB]
T=$1
timeout 300 python tools/run_once.py 24 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${2:-k_c0_final} -c 1 -o gpurun_out/prof_$T \
    python tools/run_once.py 24 > gpurun_out/ncu_$T.log 2>&1
tail -1 gpurun_out/ncu_$T.log
