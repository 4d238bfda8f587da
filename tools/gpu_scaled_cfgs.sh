#!/bin/bash
# Scaled configs 4 and 5 on the GPU box (bench.py --config cfg4s / cfg5s).
mkdir -p gpurun_out
timeout 1200 python bench.py --config cfg4s --variants h2star-bt --steps 50 > gpurun_out/bench_cfg4s.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg4s.log
timeout 2400 python bench.py --config cfg5s --variants h2star-bt --steps 10 --nrhs 1 > gpurun_out/bench_cfg5s.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg5s.log
