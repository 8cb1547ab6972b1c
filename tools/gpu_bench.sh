#!/bin/bash
# Round measurement: bench (ours + reference arm), ncu launch list of the bench
# command, ncu --set full of the phase and codec kernels, traffic json.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/ncu_target.py split > gpurun_out/bench_ncu.log 2>&1
bash tools/gpu_ncu.sh > /dev/null 2>&1
cat gpurun_out/bench.json gpurun_out/bench_ref.json; tail -n 3 gpurun_out/bench.err gpurun_out/bench_ref.err
cat gpurun_out/ncu_traffic.json
