# ncu --set full of the fused kernel (C2, 8 logical ranks on one GPU) + source-level stalls;
# plus the phase profile with the current build
mkdir -p gpurun_out /tmp/ncu
for d in 0 768; do timeout 120 python tools/fused_profile.py 0 0 0 $d; done > gpurun_out/fused_profile4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fstream -c 1 \
    -o /tmp/ncu/prof_fused -f python tools/ncu_target.py fused > gpurun_out/ncu_fused.log 2>&1
python tools/ncu_summary.py /tmp/ncu/prof_fused.ncu-rep > gpurun_out/ncu_fused_summary.txt 2>&1
ncu -i /tmp/ncu/prof_fused.ncu-rep --page source --csv --print-source sass > /tmp/ncu/src_fused.csv 2>/dev/null
gzip -c /tmp/ncu/src_fused.csv > gpurun_out/src_fused.csv.gz
python tools/src_stalls.py /tmp/ncu/src_fused.csv k_fstream 60 > gpurun_out/src_fused_stalls.txt 2>&1
cat gpurun_out/fused_profile4.log gpurun_out/ncu_fused_summary.txt | head -80
