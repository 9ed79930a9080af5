#!/bin/bash
# Build tools/variant_bench.cu under several code-generation knob settings.
set -e
cd "$(dirname "$0")/.."
F="-gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -std=c++17 -I paper_2403_16341_b200/csrc -Xptxas -v"
build() { nvcc $F $2 tools/variant_bench.cu -o tools/bin/vb_$1 > tools/bin/vb_$1.log 2>&1 & }
build v0_unroll_sw4_inl "-DNLK_COMPACT_MIN=99 -DNLK_SWEEP_MAX=4 -DNLK_INLINE_TRANS=1"
build v1_unroll_sw4_call "-DNLK_COMPACT_MIN=99 -DNLK_SWEEP_MAX=4 -DNLK_INLINE_TRANS=0"
build v2_unroll_sw16_call "-DNLK_COMPACT_MIN=99 -DNLK_SWEEP_MAX=16 -DNLK_INLINE_TRANS=0"
build v3_unroll_sw5_call "-DNLK_COMPACT_MIN=99 -DNLK_SWEEP_MAX=5 -DNLK_INLINE_TRANS=0"
build v4_compact "-DNLK_COMPACT_MIN=7 -DNLK_SWEEP_MAX=16 -DNLK_INLINE_TRANS=0"
build v5_unroll_sw4_call_mb2 "-DNLK_COMPACT_MIN=99 -DNLK_SWEEP_MAX=4 -DNLK_INLINE_TRANS=0 -DNLK_MIN_BLOCKS=2"
build v6_unroll_sw2_call "-DNLK_COMPACT_MIN=99 -DNLK_SWEEP_MAX=2 -DNLK_INLINE_TRANS=0"
wait
