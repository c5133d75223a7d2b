mkdir -p gpurun_out
for c in 2; do MCH_HOST_TIMING=1 timeout 300 python tools/run_config.py $c 3 > gpurun_out/hcfg$c.log 2>&1; echo "hcfg$c rc=$?"; done
timeout 400 python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
