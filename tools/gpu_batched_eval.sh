#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_recompute.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_batched_eval.log 2>&1; echo "exit $?" >> gpurun_out/pytest_batched_eval.log
LEVELS="l5c l5r" SHARES="1.0" bash tools/gpu_ubench_p2p.sh
