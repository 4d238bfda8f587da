#!/bin/bash
# Full ncu capture of the batched engine's two largest launches (cfg2, 16 RHS:
# down_l7 and leaf of the second pass) + raw-page CSV for reading here.
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stream_mma -s 28 -c 2 \
  -o gpurun_out/prof_mma16 -f python tools/ncu_mma.py > gpurun_out/ncu_mma_full.log 2>&1
ncu -i gpurun_out/prof_mma16.ncu-rep --page raw --csv > gpurun_out/prof_mma16_raw.csv 2>/dev/null
