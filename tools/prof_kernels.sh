#!/bin/bash
# full ncu captures of several kernels of one config-5 solve, summarised (run under gpurun):
#   prof_kernels.sh "regex,skip,tag" ...
for spec in "$@"; do
  IFS=, read K SKIP TAG <<< "$spec"
  bash tools/r02_ncu_kernel.sh ${CFG:-5} "$K" $SKIP $TAG
  python tools/ncu_summary.py gpurun_out/$TAG.ncu-rep > gpurun_out/${TAG}_summary.txt 2>&1
  ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip > gpurun_out/${TAG}_src.csv.gz
  rm -f gpurun_out/$TAG.ncu-rep
done
