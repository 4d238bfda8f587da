#!/bin/bash
# Batched engine group mode: parity (golden + scale), then per-phase timing of variants.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "batched or split_k" > gpurun_out/group_pytest.log 2>&1; echo "exit $?" >> gpurun_out/group_pytest.log
bash tools/gpu_mma_phases.sh "$@"
timeout 1200 python -m pytest tests/test_gpu_scale.py -x -q > gpurun_out/group_scale.log 2>&1; echo "exit $?" >> gpurun_out/group_scale.log
