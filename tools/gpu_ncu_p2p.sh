#!/bin/bash
# ncu of the P2P launches at a cfg3-like leaf structure (3D N=131072: 32 points
# per leaf on average, as cfg 3), all-evaluated vs 30 % of M2L TMA-staged.
# Reports are summarised on the box (gpurun brings back <= 64 MiB).
mkdir -p gpurun_out/ncu_p2p
for cfg in "1.0 s1" "0.7 s07"; do
  set -- $cfg
  python tools/ncu_p2p.py 131072 m2l $1 > gpurun_out/ncu_p2p/plain_$2.log 2>&1 &&
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:p2p_tasks -s 8 -c 4 -o /tmp/p2p_$2 python tools/ncu_p2p.py 131072 m2l $1 > gpurun_out/ncu_p2p/ncu_$2.log 2>&1
  ncu -i /tmp/p2p_$2.ncu-rep --page raw --csv > gpurun_out/ncu_p2p/raw_$2.csv 2>&1
  ncu -i /tmp/p2p_$2.ncu-rep --page source --csv --print-source sass > /tmp/src_$2.csv 2>&1
  python tools/ncu_source_top.py /tmp/src_$2.csv 60 > gpurun_out/ncu_p2p/src_top_$2.txt 2>&1
  ls -la /tmp/p2p_$2.ncu-rep /tmp/src_$2.csv >> gpurun_out/ncu_p2p/ncu_$2.log
done
gzip -f gpurun_out/ncu_p2p/raw_*.csv
du -sh gpurun_out/ncu_p2p
