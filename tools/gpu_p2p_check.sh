#!/bin/bash
# P2P engine bring-up on the GPU box: parity tests, then timing sweeps of variants.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_recompute.py -x -q > gpurun_out/p2p_pytest.log 2>&1; echo "exit $?" >> gpurun_out/p2p_pytest.log
for v in base j8 j8w8; do
  if [ $v = base ]; then unset H2G_LIB_PATH; M="stream near,m2l near,m2l@0.3 near,m2l@0.45 near,m2l@0.6"; else export H2G_LIB_PATH=$PWD/paper_2309_14085_b200/lib/var/libh2g_$v.so; M="near,m2l near,m2l@0.45"; fi
  timeout 900 python tools/recompute_sweep.py 262144,3,lap3d,1e-6 $M > gpurun_out/sweep_$v.log 2>&1; echo "exit $?" >> gpurun_out/sweep_$v.log
done
