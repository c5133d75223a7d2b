#!/bin/bash
# GPU-side measurement recipe (run under gpurun from the repo root): launch list of one bench step
# and a full ncu capture of the level-1 and level-2 on-chip PCG launches of config 2.
mkdir -p gpurun_out
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
python tools/run_config.py 2 1 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pcg2d -c 2 -o gpurun_out/prof_pcg2d_c2 -f \
    python tools/run_config.py 2 1 > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
