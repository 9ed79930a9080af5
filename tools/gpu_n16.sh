#!/bin/bash
# n = 16 Newton / trust region: parity tests + bench per library variant.
T=${1:-x}; shift
timeout 600 python -m pytest tests -m gpu -q -x -k "16 or c3_c4" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${T}_pytest.log
for lib in default "$@"; do
  if [ $lib = default ]; then unset NLK_LIB_PATH; else export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_$lib.so; fi
  timeout 600 python bench.py --config n16 --batch 1048576 --steps 3 --warmup 1 --e2e-steps 0 --no-cpu-baseline --stats gpurun_out/${T}_n16_${lib}_stats.json > gpurun_out/${T}_n16_$lib.json 2>gpurun_out/${T}_n16_$lib.err
  python -c "
import json; d=json.load(open('gpurun_out/${T}_n16_${lib}_stats.json')); print('$lib', {k[13:]: v for k, v in d['stats']['per_launch_ms'].items()})"
done
