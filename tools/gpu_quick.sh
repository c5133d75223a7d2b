# parity + per-level timings + one ncu capture of the level-1 on-chip PCG (config 1)
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
for c in ${CFGS:-1 2}; do timeout 300 python tools/run_config.py $c 2 > gpurun_out/cfg$c.log 2>&1; echo "cfg$c rc=$?"; done
if [ -n "$PROF" ]; then
python tools/run_config.py 1 1 > gpurun_out/plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pcg2d -c 1 -o gpurun_out/prof_pcg2d_c1 -f \
    python tools/run_config.py 1 1 > gpurun_out/ncu_c1.log 2>&1; echo "ncu rc=$?"
fi
