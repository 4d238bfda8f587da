#!/bin/bash
# P2P engine on the GPU box: parity tests, then timing sweeps.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_recompute.py -x -q > gpurun_out/p2p_pytest.log 2>&1; echo "exit $?" >> gpurun_out/p2p_pytest.log
timeout 900 python tools/recompute_sweep.py 262144,3,lap3d,1e-6 stream m2l near,m2l@0.7 near,m2l@0.55 near,m2l@0.4 > gpurun_out/sweep_base.log 2>&1; echo "exit $?" >> gpurun_out/sweep_base.log
timeout 1500 python tools/recompute_sweep.py cfg2 stream near,m2l@0.15 near,m2l@0.22 near,m2l@0.3 > gpurun_out/sweep_cfg3.log 2>&1; echo "exit $?" >> gpurun_out/sweep_cfg3.log
