#!/bin/bash
# Per-launch times of chosen C2 jobs for the default and variant libraries.
#   tools/gpu_variants.sh TAG ONLY variant...
T=$1; ONLY=$2; shift 2
for lib in default "$@"; do
  if [ $lib = default ]; then unset NLK_LIB_PATH; else export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_$lib.so; fi
  timeout 600 python bench.py --config c2 --batch 1048576 --steps 3 --warmup 1 --e2e-steps 0 --no-cpu-baseline --only "$ONLY" --stats gpurun_out/${T}_${lib}_stats.json > /dev/null 2>gpurun_out/${T}_${lib}.err
  python -c "
import json; d=json.load(open('gpurun_out/${T}_${lib}_stats.json')); print('%-8s' % '$lib', {k[13:-1]: round(v, 2) for k, v in d['stats']['per_launch_ms'].items()})"
done
