#!/bin/bash
# Round measurements on the GPU box: default bench (cfg2), DRAM traffic of one
# cfg2 matvec, cfg3 bench with evaluated near/M2L.  Outputs under gpurun_out/.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg2.log
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --print-units base --clock-control none -k regex:"stream_gemv|p2p_tasks" --csv --log-file gpurun_out/traffic_cfg2.csv python tools/ncu_traffic.py cfg2 > gpurun_out/traffic_cfg2.log 2>&1
python tools/ncu_traffic.py --summarize gpurun_out/traffic_cfg2.csv cfg2 h2star-bt 15 >> gpurun_out/traffic_cfg2.log 2>&1
cp profiles/traffic_cfg2_h2star-bt.json gpurun_out/ 2>/dev/null
timeout 1800 python bench.py --config cfg3 --variants h2star-bt --steps 20 --nrhs 1 > gpurun_out/bench_cfg3.log 2>&1; echo "exit $?" >> gpurun_out/bench_cfg3.log
