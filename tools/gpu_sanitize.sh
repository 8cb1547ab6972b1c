#!/bin/bash
# compute-sanitizer racecheck / synccheck / memcheck over the streaming and fused kernels
mkdir -p gpurun_out/sanitize
for m in ${MODES:-split fused codec small lane8}; do
  for t in racecheck synccheck memcheck; do
    extra=""
    [ $t = racecheck ] && extra="--racecheck-report all"
    timeout 900 compute-sanitizer --tool $t $extra --print-limit 50 python tools/sanitize_target.py $m \
      > gpurun_out/sanitize/${t}_${m}.log 2>&1
    echo "$t $m rc=$?" >> gpurun_out/sanitize/summary.txt
    tail -3 gpurun_out/sanitize/${t}_${m}.log >> gpurun_out/sanitize/summary.txt
  done
done
cat gpurun_out/sanitize/summary.txt
