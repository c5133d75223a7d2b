#!/bin/bash
# round-2 baseline: per-config device times, c5 launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
for c in 5 4; do timeout 300 python tools/run_config.py $c 2 > gpurun_out/cfg$c.log 2>&1; echo "cfg$c rc=$?"; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv \
    python tools/run_config.py 5 1 > gpurun_out/ncu_c5.log 2>&1; echo "ncu c5 rc=$?"
