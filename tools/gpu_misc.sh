#!/bin/bash
mkdir -p gpurun_out
LEVELS="l5c l5r l4r" SHARES="1.0" bash tools/gpu_ubench_p2p.sh
timeout 900 python bench.py --config cfg2 --variants h2plusH-star --steps 50 --warmup 5 --nrhs 1 --cpu-budget 1 > gpurun_out/bench_cfg2_h2plusH.json 2> gpurun_out/bench_cfg2_h2plusH.err; echo "rc $?" >> gpurun_out/bench_cfg2_h2plusH.err
