#!/bin/bash
# P2P engine microbenchmark variants (tools/ubench_p2p.cu, prebuilt under scratch/ub/ by tools/build_ubench_p2p.sh)
mkdir -p gpurun_out
out=gpurun_out/ubench_p2p.jsonl
: > $out
for b in $(ls scratch/ub); do
  for lv in ${LEVELS:-l5r l4r}; do
    for s in ${SHARES:-1.0 0.7 0.6 0.5}; do
      echo -n "{\"bin\": \"$b\"} " >> $out
      timeout 120 scratch/ub/$b $lv $s >> $out 2>&1 || echo "FAILED rc $?" >> $out
    done
  done
done
