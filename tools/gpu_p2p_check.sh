#!/bin/bash
# P2P engine bring-up on the GPU box: parity tests, then timing sweeps.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_recompute.py -x -q > gpurun_out/p2p_pytest.log 2>&1; echo "exit $?" >> gpurun_out/p2p_pytest.log
timeout 900 python tools/recompute_sweep.py 262144,3,lap3d,1e-6 stream near,m2l near,m2l@0.7 near,m2l@0.6 near,m2l@0.5 near,m2l@0.4 > gpurun_out/sweep_base.log 2>&1; echo "exit $?" >> gpurun_out/sweep_base.log
