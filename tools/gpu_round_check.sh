#!/bin/bash
# Round check on the GPU box: all GPU tests, smoke, default bench, launch list.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg2.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --variants h2star-bt --cpu-budget 1 --nrhs 1 > gpurun_out/launches.log 2>&1
