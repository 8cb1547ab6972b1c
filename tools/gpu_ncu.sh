#!/bin/bash
# One gpurun call: ncu --set full captures of the split flash kernels and the codec kernels.
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_reduce|k_gather" -c 3 \
    -o gpurun_out/prof_split -f python tools/ncu_target.py split > gpurun_out/ncu_split.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_quant_fast|k_dequant_fast" -c 2 \
    -o gpurun_out/prof_codec -f python tools/ncu_target.py codec > gpurun_out/ncu_codec.log 2>&1
tail -3 gpurun_out/ncu_split.log gpurun_out/ncu_codec.log
ls -la gpurun_out
