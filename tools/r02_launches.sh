#!/bin/bash
# launch list (device time per kernel, DRAM bytes) of one config run
mkdir -p gpurun_out
C=${1:-5}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_c$C.csv \
    python tools/run_config.py $C 1 > gpurun_out/ncu_c$C.log 2>&1; echo "ncu c$C rc=$?"
