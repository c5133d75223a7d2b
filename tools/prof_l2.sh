mkdir -p gpurun_out
python tools/run_config.py 2 1 > gpurun_out/plain_c2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pcg2d -s 1 -c 1 -o gpurun_out/prof_pcg2d_c2L2 -f \
    python tools/run_config.py 2 1 > gpurun_out/ncu_c2.log 2>&1; echo "ncu rc=$?"
