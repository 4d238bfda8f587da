#!/bin/bash
# cfg2 bench (multi-RHS engine with dual accumulators), then the cfg3 ncu evidence
mkdir -p gpurun_out
timeout 900 python bench.py --config cfg2 --steps 20 --warmup 5 --cpu-budget 5 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "rc $?" >> gpurun_out/bench_cfg2.err
bash tools/gpu_ncu_cfg3.sh
