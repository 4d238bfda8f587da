#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python tools/hybrid_sweep.py cfg3 s1 s0.7 s0.6 > gpurun_out/staged2.jsonl 2> gpurun_out/staged2.err; echo "rc $?" >> gpurun_out/staged2.err
timeout 900 python tools/sanitize_cases.py > gpurun_out/sanitize_plain.log 2>&1 &&
timeout 1800 compute-sanitizer --tool memcheck --leak-check full --print-limit 50 python tools/sanitize_cases.py > gpurun_out/memcheck.log 2>&1
echo "memcheck rc $?" >> gpurun_out/memcheck.log
