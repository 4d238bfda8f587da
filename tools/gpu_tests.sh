#!/bin/bash
# GPU test suite + smoke on the box (durations of the slowest tests kept).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -s --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
