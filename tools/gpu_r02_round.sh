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
if [ "${NCU_CFG3:-0}" = "1" ]; then bash tools/gpu_ncu_cfg3.sh; fi
# launch list of the bench command (kernel names and durations; cold-cache, serialised)
[ "${LAUNCH_LIST:-1}" = "1" ] && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --nrhs 1 --cpu-budget 1 --streamed-variant 0 > gpurun_out/launches.log 2>&1
timeout 1500 python bench.py --config cfg5s --steps 10 --warmup 5 > gpurun_out/bench_cfg5s.json 2> gpurun_out/bench_cfg5s.err; echo "rc $?" >> gpurun_out/bench_cfg5s.err
