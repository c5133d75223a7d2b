#!/bin/bash
# round-2 measurement recipe (run under gpurun from the repo root):
#   1. the GPU test suite, 2. the bench line, 3. the launch list of one config-5 run (device time +
#   DRAM bytes per launch), 4. ncu --set full of the dominant launches.  Each ncu run only after the
#   same command exited 0 without ncu.
mkdir -p gpurun_out
if [ -z "$SKIP_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/pytest_gpu.log)"
fi
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python tools/run_config.py 5 1 > gpurun_out/plain_c5.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/launches_c5.csv python tools/run_config.py 5 1 > gpurun_out/ncu_c5.log 2>&1; echo "launches rc=$?"
if [ -z "$SKIP_FULL" ]; then
  # (kernel regex, launches to skip, tag); reports exported to csv (raw + source) and removed: the
  # merged gpurun_out/ is capped at 64 MiB
  for spec in ${FULL_SPECS:-"k_pcg3d_l1c,0,l1c" "k_pcg3d_w7,0,w7" "k_fine3d_transport,2,fine3d_l4" "k_pcg3d<2,0,pcg3d25"}; do
    IFS=, read K SKIP TAG <<< "$spec"
    timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" --launch-skip $SKIP --launch-count 1 \
      -o gpurun_out/r02_$TAG -f python tools/run_config.py ${CFG:-5} 1 > gpurun_out/ncu_$TAG.log 2>&1; echo "ncu $TAG rc=$?"
    ncu -i gpurun_out/r02_$TAG.ncu-rep --page raw --csv > gpurun_out/r02_${TAG}_raw.csv 2>/dev/null
    ncu -i gpurun_out/r02_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r02_${TAG}_src.csv 2>/dev/null
    gzip -f gpurun_out/r02_${TAG}_src.csv
    rm -f gpurun_out/r02_$TAG.ncu-rep
  done
fi
