#!/bin/bash
# Per-phase timing of the batched-RHS engine (base build and diagnostic variants).
mkdir -p gpurun_out
timeout 600 python tools/mma_phases.py > gpurun_out/mma_phases_base.json 2> gpurun_out/mma_phases_base.err
for v in "$@"; do
  H2G_LIB_PATH=$PWD/paper_2309_14085_b200/lib/var/libh2g_$v.so timeout 600 python tools/mma_phases.py > gpurun_out/mma_phases_$v.json 2> gpurun_out/mma_phases_$v.err
done
