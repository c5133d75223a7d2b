#!/bin/bash
# GPU-side measurement recipe (run under gpurun from the repo root).
set -x
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/bench_small0.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pcg -c 3 -o gpurun_out/prof_pcg \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
