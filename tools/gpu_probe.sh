#!/bin/bash
# Probe call: phase-time sweeps (tools/reduce_probe.py) + optional ncu of one kernel.
mkdir -p gpurun_out
for b in ${BITS:-4}; do
  SWEEP="${SWEEP}" timeout 600 python tools/reduce_probe.py $b >> gpurun_out/probe.txt 2>&1
done
cat gpurun_out/probe.txt
if [ -n "$NCUK" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCUK" -s ${NCUS:-3} -c ${NCUC:-1} \
      -o /tmp/prof_k -f python tools/ncu_target.py ${NCUMODE:-split} > gpurun_out/ncu_k.log 2>&1
  python tools/ncu_summary.py /tmp/prof_k.ncu-rep > gpurun_out/ncu_k_summary.txt 2>&1
  ncu -i /tmp/prof_k.ncu-rep --page source --csv --print-source sass > /tmp/src_k.csv 2>/dev/null
  gzip -c /tmp/src_k.csv > gpurun_out/src_k.csv.gz
  cp /tmp/prof_k.ncu-rep gpurun_out/ 2>/dev/null
  cat gpurun_out/ncu_k_summary.txt
fi
