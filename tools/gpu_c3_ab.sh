#!/bin/bash
# C3 per-launch A/B of variant libraries (+ quasi-Newton parity tests on the first variant).
T=$1; shift
export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_$1.so
timeout 600 python -m pytest tests -m gpu -q -x -k "klement or broyden or c3 or fp32" 2>&1 | tail -1
for lib in default "$@"; do
  if [ $lib = default ]; then unset NLK_LIB_PATH; else export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_$lib.so; fi
  python bench.py --config c3 --batch 10000000 --steps 5 --warmup 2 --e2e-steps 0 --no-cpu-baseline --stats gpurun_out/${T}_c3_${lib}_stats.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/${T}_c3_${lib}_stats.json')); print('$lib', round(d['result']['value']/1e6,1), {k[13:-1]: round(v,3) for k, v in d['stats']['per_launch_ms'].items()})"
done
