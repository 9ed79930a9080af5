#!/bin/bash
# Build tools/variant_bench.cu under several code-generation knob settings.
set -e
cd "$(dirname "$0")/.."
F="-gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -I paper_2403_16341_b200/csrc -Xptxas -v"
build() { nvcc $F $2 tools/variant_bench.cu -o tools/bin/vb_$1 > tools/bin/vb_$1.log 2>&1 & }
rm -f tools/bin/vb_*
build thread "-DNLK_COOP_MIN=99"
build coop8 "-DNLK_COOP_MIN=8"
build coop8_mb2 "-DNLK_COOP_MIN=8 -DNLK_MIN_BLOCKS=2"
build coop8_mb3 "-DNLK_COOP_MIN=8 -DNLK_MIN_BLOCKS=3"
wait
