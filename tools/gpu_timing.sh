mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for c in 1 2; do MCH_LIB=paper_2503_01276_b200/lib/libmch_timing.so MCH_PCG_TIMING=1 timeout 300 python tools/run_config.py $c 1 > gpurun_out/tcfg$c.log 2>&1; echo "tcfg$c rc=$?"; done
for c in 1 2; do timeout 300 python tools/run_config.py $c 2 > gpurun_out/cfg$c.log 2>&1; echo "cfg$c rc=$?"; done
