#!/bin/bash
# A/B of the Jacobi tolerance of k_pinv on config 5 (launch list of the level-4 k_pinv)
for t in "" _pt30 _pt26; do
  L=paper_2503_01276_b200/lib/libmch$t.so
  MCH_LIB=$L ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_pinv --csv python tools/run_config.py 5 1 2>/dev/null | grep k_pinv | tail -2 | sed "s/^/$t /"
  MCH_LIB=$L python -m pytest tests/test_gpu_parity.py -q -x -k "rank_deficient or interior_3d and 5 or config_sampled and 5" 2>&1 | tail -1 | sed "s/^/$t /"
done
