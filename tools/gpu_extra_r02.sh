#!/bin/bash
# Stress tests + the secondary bench configurations with the final round-2 build.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stress.py -x -q > gpurun_out/pytest_stress.log 2>&1; echo "exit $?" >> gpurun_out/pytest_stress.log
timeout 1200 python bench.py --config cfg2 --steps 100 --warmup 5 > gpurun_out/bench_cfg2.json 2> gpurun_out/bench_cfg2.err; echo "rc $?" >> gpurun_out/bench_cfg2.err
timeout 1500 python bench.py --config cfg5s --steps 20 --warmup 5 > gpurun_out/bench_cfg5s.json 2> gpurun_out/bench_cfg5s.err; echo "rc $?" >> gpurun_out/bench_cfg5s.err
timeout 900 python bench.py --config cfg4s --steps 20 --warmup 5 > gpurun_out/bench_cfg4s.json 2> gpurun_out/bench_cfg4s.err; echo "rc $?" >> gpurun_out/bench_cfg4s.err
