mkdir -p gpurun_out
for d in 0 2048 2304 768; do timeout 120 python tools/fused_profile.py 0 0 0 $d; done > gpurun_out/fused_profile3.log 2>&1
cat gpurun_out/fused_profile3.log
