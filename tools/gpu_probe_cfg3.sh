#!/bin/bash
# Probe: box shape + the cfg-3 bench line (auto evaluation policy).
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -20; nvidia-smi) > gpurun_out/box.txt 2>&1
timeout 1500 python bench.py --config cfg3 --steps 20 --warmup 5 --variants h2star-bt --nrhs 1 --cpu-budget 5 > gpurun_out/cfg3_auto.json 2> gpurun_out/cfg3_auto.err
echo "rc $?" >> gpurun_out/cfg3_auto.err
