#!/bin/sh
# Build the W-iteration stage-latency probe (tools/microbench/wchain.cu).
R=$(cd "$(dirname "$0")/../.." && pwd)
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -std=c++17 --expt-relaxed-constexpr -I "$R/include" \
     -I "$R/paper_2601_17979_b200/csrc" "$R/tools/microbench/wchain.cu" "$R/paper_2601_17979_b200/csrc/finalize.cu" \
     -o "$R/tools/microbench/wchain"
