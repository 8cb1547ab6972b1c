#!/bin/bash
# Quick perf check: parity subset + one bench run, printing the step and per-phase kernel times.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_flash.py -x -q ${PYT:-} 2>&1 | tail -2
python bench.py --steps 20 --warmup 5 ${BARGS:-} > gpurun_out/bench_phase.json 2> gpurun_out/bench_phase.err
python - <<'PY'
import json
d = json.loads(open("gpurun_out/bench_phase.json").read().strip().splitlines()[-1])
print("step ms", round(d["ms_per_step"], 4), "value", round(d["value"], 1), "frac", round(d["roofline"]["frac"], 3))
for k, v in d.get("phases", {}).items():
    print(f"  {k:8s} {v['kernel']:10s} {v['us']:7.1f} us  {v['gbs']:7.0f} GB/s  {v['frac'] * 100:5.1f}%")
print("e2e", round(d["e2e"]["ms_per_step"], 2), "ms")
PY
