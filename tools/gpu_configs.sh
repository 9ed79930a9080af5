#!/bin/bash
# Full-size single-GPU runs of the non-default configurations (clocks sampled:
# every timed region >= 0.7 s).   tools/gpu_configs.sh TAG [configs...]
T=${1:-x}; shift
CFGS=${@:-c1 c3 c4 c5 n16}
for c in $CFGS; do
  case $c in
    c1) a="--config c1 --batch 16777216 --steps 1000 --warmup 5";;
    c3) a="--config c3 --batch 10000000 --steps 5 --warmup 3";;
    c3f32) a="--config c3 --batch 10000000 --steps 10 --warmup 3 --dtype f32";;
    c4) a="--config c4 --batch 10000000 --steps 5 --warmup 3";;
    c5) a="--config c5 --batch 12500000 --steps 400 --warmup 5";;
    n16) a="--config n16 --batch 1048576 --steps 1 --warmup 1";;
  esac
  timeout 900 python bench.py $a --e2e-steps 3 --no-cpu-baseline --stats gpurun_out/${T}_${c}_stats.json > gpurun_out/${T}_${c}.json 2>gpurun_out/${T}_${c}.err
  python -c "
import json; d=json.load(open('gpurun_out/${T}_${c}_stats.json')); r=d['result']
print('$c', round(r['value']/1e6,2), 'M/s', round(r['ms_per_step'],3), 'ms e2e', round(r['e2e']['value']/1e6,2), r['roofline']['bound'], round(r['roofline']['frac'],4), r['clocks'])
print('   ', {k[13:-1]: v for k, v in d['stats']['per_launch_ms'].items()})"
done
