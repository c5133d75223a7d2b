# A/B: run config ${CFG:-2} with each library given in LIBS
mkdir -p gpurun_out
for L in ${LIBS}; do MCH_LIB=paper_2503_01276_b200/lib/$L timeout 300 python tools/run_config.py ${CFG:-2} 3 > gpurun_out/ab_$L.log 2>&1; echo "$L rc=$?"; done
