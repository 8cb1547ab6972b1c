#!/bin/bash
# ncu --set full of the streaming reduce kernel only, with CUDA-line attribution.
mkdir -p gpurun_out /tmp/ncu
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_rstream" -c 1 \
    -o /tmp/ncu/prof_reduce -f python tools/ncu_target.py split > gpurun_out/ncu_reduce.log 2>&1
python tools/ncu_summary.py /tmp/ncu/prof_reduce.ncu-rep > gpurun_out/ncu_reduce_summary.txt 2>&1
ncu -i /tmp/ncu/prof_reduce.ncu-rep --page source --csv --print-source cuda,sass > /tmp/ncu/src_reduce.csv 2>/dev/null
gzip -c /tmp/ncu/src_reduce.csv > gpurun_out/src_reduce_cuda.csv.gz
ncu -i /tmp/ncu/prof_reduce.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src_reduce_sass.csv 2>/dev/null
gzip -c /tmp/ncu/src_reduce_sass.csv > gpurun_out/src_reduce.csv.gz
cat gpurun_out/ncu_reduce_summary.txt
