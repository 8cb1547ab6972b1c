#!/bin/bash
# Iteration call: GPU parity tests + kernel sweep + bench (+ optional ncu of the split kernels).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/kernel_bench.py codec flash --quick > gpurun_out/kernel_bench.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "$NCU" = "1" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter|k_reduce|k_gather|k_qstream|k_rstream|k_dstream" -c 3 \
      -o gpurun_out/prof_split -f python tools/ncu_target.py split > gpurun_out/ncu_split.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_quant_fast|k_dequant_fast|k_qstream|k_dstream" -c 2 \
      -o gpurun_out/prof_codec -f python tools/ncu_target.py codec > gpurun_out/ncu_codec.log 2>&1
fi
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/kernel_bench.log | cut -c1-200; cut -c1-400 gpurun_out/bench.json; tail -2 gpurun_out/bench.err
