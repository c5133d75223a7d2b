# ncu full capture of the level-1 on-chip PCG launch of config 1 (one launch, 486 CTAs)
mkdir -p gpurun_out
python tools/run_config.py 1 1 > gpurun_out/plain_c1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_pcg2d -c 1 -o gpurun_out/prof_pcg2d_c1 \
    python tools/run_config.py 1 1 > gpurun_out/ncu_c1.log 2>&1; echo "ncu rc=$?"
