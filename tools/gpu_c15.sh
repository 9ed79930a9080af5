#!/bin/bash
# C1/C5 full-size benches for the default library and variant libraries,
# plus the quadratic parity tests.   tools/gpu_c15.sh TAG [variant ...]
T=${1:-x}; shift
timeout 600 python -m pytest tests -m gpu -q -x -k "c1 or c5 or quadratic or poly or edges or fp32" > gpurun_out/${T}_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/${T}_pytest.log
for lib in default "$@"; do
  if [ $lib = default ]; then unset NLK_LIB_PATH; else export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_$lib.so; fi
  python bench.py --config c1 --batch 16777216 --steps 1000 --warmup 5 --e2e-steps 3 --no-cpu-baseline > gpurun_out/${T}_c1_$lib.json 2>gpurun_out/${T}_c1_$lib.err
  python bench.py --config c5 --batch 12500000 --steps 400 --warmup 5 --e2e-steps 3 --no-cpu-baseline --stats gpurun_out/${T}_c5_${lib}_stats.json > gpurun_out/${T}_c5_$lib.json 2>gpurun_out/${T}_c5_$lib.err
  python -c "
import json
for c in ['c1','c5']:
    d=json.load(open('gpurun_out/${T}_'+c+'_$lib.json')); print('$lib', c, round(d['value']/1e9,3),'G/s', round(d['ms_per_step'],3),'ms', d['roofline']['bound'], round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value']/1e9,3), d['clocks'])"
done
unset NLK_LIB_PATH
