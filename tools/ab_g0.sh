#!/bin/bash
# A/B of the gather finish (pass D replaced by group-0 parent reads in E) at n = 24
# usage: tools/ab_g0.sh "pon list" LIB...   (each LIB with DQMC_EXP_G0=1; the in-tree library also with 0)
PONS=${1:-0.75}; shift
L=paper_2302_10083_b200/libdqmc.so
for pon in $PONS; do
  echo "== P_ON=$pon"
  DC=$( [ $pon = 0.75 ] && echo 0.05 || echo 0 )
  P_ON=$pon P_DC=$DC DQMC_EXP_G0=0 python tools/ab_passes.py 24 $L 2>&1 | tail -1
  for V in $L "$@"; do
    P_ON=$pon P_DC=$DC DQMC_EXP_G0=1 python tools/ab_passes.py 24 $V 2>&1 | tail -1
  done
done
