#!/bin/bash
# cfg-3 share sweep over the prebuilt libh2g variants in paper_2309_14085_b200/lib/variants/
mkdir -p gpurun_out
timeout 900 python tools/ncu_cfg3.py build /tmp/cfg3 > gpurun_out/variant_build.log 2>&1 || exit 1
: > gpurun_out/variants.jsonl
for lib in paper_2309_14085_b200/lib/variants/*.so; do
  H2G_LIB_PATH=$PWD/$lib SWEEP_CHECK=${SWEEP_CHECK:-1} timeout 600 python tools/variant_sweep.py /tmp/cfg3 ${SHARES:-0.7 0.6 0.5} >> gpurun_out/variants.jsonl 2>> gpurun_out/variants.err
done
