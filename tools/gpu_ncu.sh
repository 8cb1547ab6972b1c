#!/bin/bash
# One gpurun call: ncu --set full captures of the flash phase kernels and the codec kernels.
# Reports stay in /tmp on the box; text summaries (and reports under 20 MB) come back in gpurun_out/.
mkdir -p gpurun_out /tmp/ncu
KS=${KS:-"k_scatter|k_reduce|k_gather|k_qstream|k_rstream|k_dstream"}
KC=${KC:-"k_quant_fast|k_dequant_fast|k_qstream|k_dstream"}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KS" -c 3 \
    -o /tmp/ncu/prof_split -f python tools/ncu_target.py split > gpurun_out/ncu_split.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"$KC" -c 2 \
    -o /tmp/ncu/prof_codec -f python tools/ncu_target.py codec > gpurun_out/ncu_codec.log 2>&1
for r in split codec; do
  python tools/ncu_summary.py /tmp/ncu/prof_$r.ncu-rep > gpurun_out/ncu_${r}_summary.txt 2>&1
  ncu -i /tmp/ncu/prof_$r.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src_$r.csv 2>/dev/null
  gzip -c /tmp/ncu/src_$r.csv > gpurun_out/src_$r.csv.gz
  sz=$(stat -c %s /tmp/ncu/prof_$r.ncu-rep 2>/dev/null || echo 0)
  if [ "$sz" -lt 20000000 ]; then cp /tmp/ncu/prof_$r.ncu-rep gpurun_out/; fi
done
python tools/make_traffic.py /tmp/ncu/prof_split.ncu-rep gpurun_out/ncu_traffic.json > /dev/null 2>&1
cat gpurun_out/ncu_split_summary.txt gpurun_out/ncu_codec_summary.txt
