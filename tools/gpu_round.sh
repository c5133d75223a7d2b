mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for c in 1 2 3; do timeout 300 python tools/run_config.py $c 2 > gpurun_out/cfg$c.log 2>&1; echo "cfg$c rc=$?"; done
MCH_PCG=gn timeout 300 python tools/run_config.py 1 2 > gpurun_out/cfg1_gn.log 2>&1; echo "cfg1gn rc=$?"
timeout 400 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
