#!/bin/bash
# Single-RHS per-phase timing of diagnostic builds (cfg2 H2* and (H2+H)*).
mkdir -p gpurun_out
for v in base "$@"; do
  if [ $v = base ]; then unset H2G_LIB_PATH; else export H2G_LIB_PATH=$PWD/paper_2309_14085_b200/lib/var/libh2g_$v.so; fi
  timeout 600 python tools/phases.py h2plusH-star > gpurun_out/ph_hplus_$v.json 2>&1
  timeout 600 python tools/phases.py h2star-bt > gpurun_out/ph_h2s_$v.json 2>&1
done
