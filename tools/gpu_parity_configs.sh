#!/bin/bash
# The bench's parity leg (>= 20k stratified systems vs the unmodified reference on
# this host) for every configuration.   tools/gpu_parity_configs.sh TAG
T=${1:-x}
for c in c1 c3 c4 c5 c2s1; do
  case $c in
    c1) a="--config c1 --batch 16777216 --steps 20 --warmup 3";;
    c3) a="--config c3 --batch 10000000 --steps 2 --warmup 1";;
    c4) a="--config c4 --batch 10000000 --steps 2 --warmup 1";;
    c5) a="--config c5 --batch 12500000 --steps 20 --warmup 3";;
  esac
  [ $c = c2s1 ] && continue
  timeout 1800 python bench.py $a --e2e-steps 0 > gpurun_out/${T}_parity_${c}.json 2> gpurun_out/${T}_parity_${c}.err
  python -c "
import json; d=json.load(open('gpurun_out/${T}_parity_${c}.json')); p=d['parity']
print('$c', p['systems'], 'systems', p['mismatches'], 'mismatches', p['mismatches_by_field'], 'dfsane(unpinned)', p['systems_unpinned_dfsane'], 'cpu', round(d['cpu_baseline']['value']), d['cpu_baseline']['sample'][:60])"
done
