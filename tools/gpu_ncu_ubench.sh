#!/bin/bash
# ncu --set full of one ubench_p2p launch (source-level stall sampling)
mkdir -p gpurun_out
BIN=${1:-scratch/ub/sw_li}; LV=${2:-l5}; SH=${3:-0.5}
timeout 300 $BIN $LV $SH 2 > gpurun_out/ncu_ub_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tasks -s 2 -c 1 -f -o gpurun_out/ub_p2p $BIN $LV $SH 2 > gpurun_out/ncu_ub.log 2>&1
echo "rc $?" >> gpurun_out/ncu_ub.log
