#!/bin/bash
# round-2 (second session) measurement recipe, run under gpurun from the repo root:
#   1. bench line (config 5 headline + other configs), 2. launch list of one config-5 solve (device
#   time + DRAM bytes per launch), 3. ncu --set full of the dominant launches.  Each ncu run only
#   after the same command exited 0 without ncu.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/run_config.py 5 1 > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c5.csv python tools/run_config.py 5 1 > gpurun_out/ncu_c5.log 2>&1; echo "launches rc=$?"
if [ -z "$SKIP_FULL" ]; then
  bash tools/prof_kernels.sh ${FULL_SPECS:-"k_fine3d_transport,2,fine3d_l4" "k_pcg3d_w7,0,w7_l4" "^k_pcg3d$,0,pcg3d13_l3" "k_pcg3dc,0,pcg3dc25_l2" "k_pcg3d_l1c,0,l1c_l1" "k_fine3d_combine,1,combine_l3"}
fi
