#!/bin/bash
# Round-2 check on the GPU box: GPU tests, smoke, both bench arms as the driver
# runs them, tools/sanitize_cases.py (plain), then the ncu evidence of the
# cfg-3 headline plan (tools/gpu_ncu_cfg3.sh).
mkdir -p gpurun_out
(nproc; free -g; nvidia-smi --query-gpu=name,memory.total --format=csv) > gpurun_out/box.txt 2>&1
SECONDS=0
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/pytest_gpu.log 2>&1; echo "exit $? after ${SECONDS}s" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "exit $?" >> gpurun_out/smoke.log
SECONDS=0
timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc $? after ${SECONDS}s" >> gpurun_out/bench_ref.err
SECONDS=0
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "rc $? after ${SECONDS}s" >> gpurun_out/bench.err
timeout 900 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1
# (compute-sanitizer is closed on this pool: profiles/sanitizer_r02.md)
bash tools/gpu_ncu_cfg3.sh
