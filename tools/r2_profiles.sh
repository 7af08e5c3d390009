#!/bin/bash
# Round-2 measurement evidence (run on the GPU box): bench lines for every BASELINE config, the reference
# arm, the C1 launch list, ncu --set full of the north-star kernel, per-config ncu metrics, sanitizers.
mkdir -p gpurun_out/r2
for c in c1-10k c1 c1r c2-full c2-vals c3-geo c3-rank c4 c4-blocked c4-qr c5; do
    timeout 900 python bench.py --config $c > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err || echo "$c failed"
done
python bench.py --config c1-10k --batch 1250 > gpurun_out/r2/bench_c1-slice1250.json 2> gpurun_out/r2/bench_slice.err
python bench.py --impl reference --config c1-10k > gpurun_out/r2/bench_c1-10k_reference.json 2> gpurun_out/r2/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2/launches_c1.csv \
    python bench.py --steps 2 --warmup 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_reg32b -s 1 -c 1 \
    -o gpurun_out/r2/c1_k42 -f python tools/quick_time.py C1-10k > /dev/null 2>&1
bash tools/ncu_configs.sh gpurun_out/r2/prof
for t in memcheck racecheck synccheck initcheck; do
  timeout 600 compute-sanitizer --tool $t python tools/sanitize_smoke.py > gpurun_out/r2/san_$t.txt 2>&1
done
echo r2 profiles done
