#!/bin/bash
mkdir -p gpurun_out
(df -h /tmp /root . ; free -g) > gpurun_out/disk.txt 2>&1
timeout 1700 python tools/hybrid_sweep.py cfg3 0 0.15 0.25 0.35 0.45 > gpurun_out/hybrid.jsonl 2> gpurun_out/hybrid.err; echo "rc $?" >> gpurun_out/hybrid.err
