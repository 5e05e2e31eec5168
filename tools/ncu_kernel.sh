#!/bin/bash
# ncu --set full of one launch of a kernel at n=24 (under gpurun):
#   bash tools/ncu_kernel.sh TAG KERNEL_REGEX [LIB.so]
T=$1
timeout 300 python tools/run_once.py 24 1 $3 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -c 1 -o gpurun_out/prof_$T \
    python tools/run_once.py 24 1 $3 > gpurun_out/ncu_$T.log 2>&1
tail -1 gpurun_out/ncu_$T.log
