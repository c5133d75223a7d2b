#!/bin/bash
# round-2 third session: A/B of the coarse-space second labelling pass (MCH_COARSE_ERODE: 0 off,
# 1 majority-cell threshold, 2 all-cells-high erosion) on config 5
mkdir -p gpurun_out
for e in ${MODES:-0 1}; do
  MCH_COARSE_ERODE=$e timeout 300 python tools/iters_level.py 5 2 > gpurun_out/it_c5_l2_e$e.log 2>&1; echo "iters e$e rc=$?"
  head -7 gpurun_out/it_c5_l2_e$e.log
  MCH_COARSE_ERODE=$e timeout 300 python tools/run_config.py ${CFG:-5} 2 > gpurun_out/cfg_e$e.log 2>&1; echo "cfg e$e rc=$?"
  grep "rep1" gpurun_out/cfg_e$e.log | cut -c1-330
done
