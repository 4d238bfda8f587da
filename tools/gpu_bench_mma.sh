#!/bin/bash
# Default bench (cfg2, incl. 16-RHS multi_rhs) + scaled cfg4 (Gaussian, 16-RHS GMRES(30)).
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg2.log
timeout 1200 python bench.py --config cfg4s --variants h2star-bt --steps 50 > gpurun_out/bench_cfg4s.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg4s.log
timeout 900 python tools/mma_phases.py 262144 3 > gpurun_out/mma_phases_3d.json 2>&1
