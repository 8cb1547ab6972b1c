#!/bin/bash
# Round measurement: GPU tests + smoke, bench (ours + reference arm), the ncu launch list of the
# bench's C2 step, ncu --set full of the phase + codec kernels (summaries, traffic json), SASS
# evidence, compute-sanitizer over every kernel family.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 python bench.py --config c1 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
timeout 600 python bench.py --config c4 --no-cpu > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/ncu_target.py split > gpurun_out/bench_ncu.log 2>&1
python tools/launch_summary.py gpurun_out/launches.csv > gpurun_out/launches_summary.txt 2>&1
bash tools/gpu_ncu.sh > /dev/null 2>&1
timeout 600 python tools/decode_probe.py > gpurun_out/decode.txt 2>&1
timeout 300 python tools/small_probe.py > gpurun_out/small_probe.txt 2>&1
[ "${SAN:-1}" = "1" ] && bash tools/gpu_sanitize.sh > /dev/null 2>&1
tail -n 2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; cut -c1-600 gpurun_out/bench.json; cut -c1-300 gpurun_out/bench_ref.json
cat gpurun_out/launches_summary.txt | head -20; cat gpurun_out/ncu_split_summary.txt gpurun_out/ncu_codec_summary.txt 2>/dev/null | head -30
cat gpurun_out/sanitize/summary.txt 2>/dev/null
