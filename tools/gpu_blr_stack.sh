#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_solver.py tests/test_gpu_stress.py -x -q > gpurun_out/pytest_blr_stack.log 2>&1; echo "exit $?" >> gpurun_out/pytest_blr_stack.log
timeout 900 python -m pytest tests/test_gpu_scale.py -x -q -k "parity_at_scale" > gpurun_out/pytest_blr_scale.log 2>&1; echo "exit $?" >> gpurun_out/pytest_blr_scale.log
timeout 900 python bench.py --config cfg2 --variants h2plusH-star --steps 50 --warmup 5 --cpu-budget 1 > gpurun_out/bench_cfg2_h2plusH.json 2> gpurun_out/bench_cfg2_h2plusH.err; echo "rc $?" >> gpurun_out/bench_cfg2_h2plusH.err
H2G_BLR_STACK=0 timeout 900 python bench.py --config cfg2 --variants h2plusH-star --steps 50 --warmup 5 --cpu-budget 1 --nrhs 1 > gpurun_out/bench_cfg2_h2plusH_nostack.json 2> gpurun_out/bench_cfg2_h2plusH_nostack.err
