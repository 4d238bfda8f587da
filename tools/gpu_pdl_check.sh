#!/bin/bash
# PDL bring-up: full GPU tests, bench, and a PDL on/off A/B of cfg2 / 3D timings.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg2.log
H2G_PDL=0 timeout 600 python tools/recompute_sweep.py cfg2 stream > gpurun_out/sweep_cfg2_nopdl.log 2>&1
timeout 600 python tools/recompute_sweep.py cfg2 stream > gpurun_out/sweep_cfg2_pdl.log 2>&1
H2G_PDL=0 timeout 600 python tools/recompute_sweep.py 262144,3,lap3d,1e-6 stream m2l > gpurun_out/sweep_3d_nopdl.log 2>&1
timeout 600 python tools/recompute_sweep.py 262144,3,lap3d,1e-6 stream m2l > gpurun_out/sweep_3d_pdl.log 2>&1
