#!/bin/bash
# Every BASELINE config through bench.py (default K / W) plus the reference arm; JSON lines into
# gpurun_out/r2_bench_<config>.json (run on the GPU box: gpurun -- bash tools/bench_all.sh)
mkdir -p gpurun_out
for c in c1-10k c1 c1r c2-full c2-vals c3-geo c3-rank c4 c4-blocked c4-qr c5; do
    python bench.py --config $c > gpurun_out/r2_bench_$c.json 2> gpurun_out/r2_bench_$c.err || echo "$c failed"
done
python bench.py --impl reference --config c1-10k > gpurun_out/r2_bench_c1-10k_reference.json 2> gpurun_out/r2_bench_ref.err
echo done
