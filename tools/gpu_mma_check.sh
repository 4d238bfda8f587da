#!/bin/bash
# Batched-RHS engine variants: parity, 16-RHS timing, smem wavefronts of the cfg2 leaf launch.
mkdir -p gpurun_out
for v in base pair0 pair2; do
  if [ $v = base ]; then unset H2G_LIB_PATH; else export H2G_LIB_PATH=$PWD/paper_2309_14085_b200/lib/var/libh2g_$v.so; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "batched or split_k or matmat" > gpurun_out/mma_pytest_$v.log 2>&1; echo "exit $?" >> gpurun_out/mma_pytest_$v.log
  timeout 600 python tools/multirhs_sweep.py 0 > gpurun_out/multirhs_$v.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,smsp__sass_inst_executed_op_shared_ld.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active --print-units base --clock-control none -k regex:stream_mma -s 29 -c 1 --csv --log-file gpurun_out/mma_ncu_$v.csv python tools/ncu_mma.py > /dev/null 2>&1
done
