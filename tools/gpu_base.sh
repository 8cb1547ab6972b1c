#!/bin/bash
# Baseline call: GPU tests, smoke, bench (ours + reference arm).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q ${PYT:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
if [ "${REF:-1}" = "1" ]; then timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; fi
tail -n 3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cut -c1-1500 gpurun_out/bench.json; tail -n 3 gpurun_out/bench.err; cut -c1-600 gpurun_out/bench_ref.json 2>/dev/null
