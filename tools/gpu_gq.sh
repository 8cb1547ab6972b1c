mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_codec.py tests/test_gpu_bench.py -q -x > gpurun_out/pytest_codec.log 2>&1; echo rc=$? >> gpurun_out/pytest_codec.log
for k in lane gpl gq default; do FC_CODEC_QKERNEL=$k timeout 300 python tools/kernel_bench.py codec 2>&1 | grep '"quantize"' | sed "s/^/$k /"; done > gpurun_out/codec_ab.log
for cfg in "0 0 0" "0 2 0" "0 3 0" "0 4 4" "64 4 4"; do timeout 120 python tools/fused_profile.py $cfg; done > gpurun_out/fused_profile.log 2>&1
tail -3 gpurun_out/pytest_codec.log; cat gpurun_out/codec_ab.log gpurun_out/fused_profile.log
