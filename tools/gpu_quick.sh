#!/bin/bash
# Quick iteration: GPU parity tests (optionally a subset) + kernel sweep + ncu summaries.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q ${PYT:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python tools/kernel_bench.py codec flash ${KB:-} --quick > gpurun_out/kernel_bench.log 2>&1
if [ "${NCU:-1}" = "1" ]; then bash tools/gpu_ncu.sh > /dev/null 2>&1; fi
tail -n 3 gpurun_out/pytest_gpu.log; cut -c1-200 gpurun_out/kernel_bench.log; cat gpurun_out/ncu_split_summary.txt gpurun_out/ncu_codec_summary.txt 2>/dev/null
