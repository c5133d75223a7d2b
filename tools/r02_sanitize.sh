#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the tiny runs of every kernel variant
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  for v in 2d 3d_small 3d_13; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_small.py $v > gpurun_out/san_${tool}_$v.log 2>&1
    echo "$tool $v rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/san_${tool}_$v.log | tail -1)"
  done
done
