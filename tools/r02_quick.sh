#!/bin/bash
# quick GPU check: 3D parity subset + per-config device times
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny_all_points or config_sampled" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"
for c in ${CFGS:-5}; do timeout 300 python tools/run_config.py $c 2 > gpurun_out/cfg$c.log 2>&1; echo "cfg$c rc=$?"; done
