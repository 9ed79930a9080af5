#!/bin/bash
# A/B of variant libraries: parity tests selected by -k on each variant, then
# per-launch times of chosen C2 jobs.
#   tools/gpu_ab.sh TAG ONLY PYTEST_K variant...
T=$1; ONLY=$2; K=$3; shift 3
mkdir -p gpurun_out
for lib in "$@"; do
  export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_$lib.so
  timeout 600 python -m pytest tests -m gpu -x -q -k "$K" > gpurun_out/${T}_${lib}_pytest.log 2>&1
  echo "$lib pytest rc=$? $(tail -1 gpurun_out/${T}_${lib}_pytest.log)"
done
unset NLK_LIB_PATH
bash tools/gpu_variants.sh "$T" "$ONLY" "$@"
