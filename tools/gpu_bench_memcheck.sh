#!/bin/bash
# bench (cfg3 default) + compute-sanitizer memcheck over every engine on small operators
mkdir -p gpurun_out
(df -h /tmp /dev/shm; free -g) > gpurun_out/disk2.txt 2>&1
timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "rc $?" >> gpurun_out/bench2.err
timeout 900 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 &&
timeout 1800 compute-sanitizer --tool memcheck --leak-check full --print-limit 50 python tools/sanitize_cases.py > gpurun_out/memcheck.log 2>&1
echo "memcheck rc $?" >> gpurun_out/memcheck.log
