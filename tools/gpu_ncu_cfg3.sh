#!/bin/bash
# ncu evidence for the cfg-3 headline plan: one --set full capture of a whole
# matvec's GEMV/P2P launches, summarised ON the box (the report is > 64 MiB).
mkdir -p gpurun_out/ncu_cfg3
timeout 900 python tools/ncu_cfg3.py build /tmp/cfg3 > gpurun_out/ncu_build.log 2>&1 || exit 1
python tools/ncu_cfg3.py run /tmp/cfg3 > gpurun_out/ncu_plain.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"stream_gemv|p2p_tasks" -s 32 -c 31 -o /tmp/prof_cfg3 python tools/ncu_cfg3.py run /tmp/cfg3 > gpurun_out/ncu_full.log 2>&1
echo "ncu rc $?" >> gpurun_out/ncu_full.log
ncu -i /tmp/prof_cfg3.ncu-rep --page raw --csv > gpurun_out/ncu_cfg3/prof_cfg3_raw.csv 2>&1
python tools/ncu_cfg3.py summarize /tmp/prof_cfg3.ncu-rep gpurun_out/ncu_cfg3 > gpurun_out/ncu_cfg3/summary.log 2>&1
ncu -i /tmp/prof_cfg3.ncu-rep --page details --csv > gpurun_out/ncu_cfg3/prof_cfg3_details.csv 2>&1
ls -la /tmp/prof_cfg3.ncu-rep >> gpurun_out/ncu_full.log
