#!/bin/bash
# Round-2 bench check: both arms as the driver runs them (cfg3 default).
mkdir -p gpurun_out
timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc $?" >> gpurun_out/bench_ref.err
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc $?" >> gpurun_out/bench.err
