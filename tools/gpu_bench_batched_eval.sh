#!/bin/bash
# Multi-RHS on evaluated plans (batched P2P engine): cfg3 headline plan and cfg5s.
mkdir -p gpurun_out
SECONDS=0
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc $? after ${SECONDS}s" >> gpurun_out/bench.err
timeout 1500 python bench.py --config cfg5s --steps 10 --warmup 5 > gpurun_out/bench_cfg5s.json 2> gpurun_out/bench_cfg5s.err; echo "rc $?" >> gpurun_out/bench_cfg5s.err
