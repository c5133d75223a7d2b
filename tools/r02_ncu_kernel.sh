#!/bin/bash
# full ncu capture of one launch of a kernel: r02_ncu_kernel.sh <config> <regex> <skip> <tag>
mkdir -p gpurun_out
C=$1; K=$2; SKIP=${3:-0}; TAG=${4:-prof}
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" --launch-skip $SKIP --launch-count 1 \
   -o gpurun_out/$TAG -f python tools/run_config.py $C 1 > gpurun_out/$TAG.log 2>&1; echo "ncu rc=$?"
