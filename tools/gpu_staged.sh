#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_recompute.py tests/test_gpu_sharded.py -x -q -k "recompute or evaluated or Evaluated or unstored" > gpurun_out/pytest_staged.log 2>&1; echo "exit $?" >> gpurun_out/pytest_staged.log
timeout 1700 python tools/hybrid_sweep.py cfg3 s1 s0.8 s0.7 s0.6 s0.5 s0.4 > gpurun_out/staged.jsonl 2> gpurun_out/staged.err; echo "rc $?" >> gpurun_out/staged.err
