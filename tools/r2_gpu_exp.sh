#!/bin/bash
# Round-2 experiment batch (run on the GPU box): variant timings + ncu of the C1 default kernel + sanitizers.
mkdir -p gpurun_out
python tools/quick_time.py --kernels 42,43 C1-10k C1-1250 > gpurun_out/r2_k42_43.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_reg32b -s 1 -c 1 -o gpurun_out/r2_c1_k42 -f \
    python tools/quick_time.py C1-10k > gpurun_out/r2_c1_k42.log 2>&1
for t in memcheck racecheck synccheck initcheck; do
  timeout 600 compute-sanitizer --tool $t python tools/sanitize_smoke.py > gpurun_out/r2_san_$t.txt 2>&1
done
