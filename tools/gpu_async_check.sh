#!/bin/bash
# async (decoupled task pipeline) vs sync P2P kernels: ubench, then cfg 3 itself; launch list.
mkdir -p gpurun_out
LEVELS="l5r l4r" SHARES="1.0 0.7 0.6 0.5" bash tools/gpu_ubench_p2p.sh
SHARES="1.0 0.6" bash tools/gpu_variant_sweep.sh
timeout 280 python tools/ncu_cfg3.py run /tmp/cfg3 > gpurun_out/launches_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cfg3.csv python tools/ncu_cfg3.py run /tmp/cfg3 > gpurun_out/launches.log 2>&1
