#!/bin/bash
# GPU tests + C2 bench with per-launch stats (+ optional configs):
#   tools/gpu_check_stats.sh TAG [configs...]
T=$1; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo "pytest rc=$? $(tail -1 gpurun_out/${T}_pytest_gpu.log)"
timeout 900 python bench.py --steps 5 --warmup 3 --e2e-steps 2 --stats gpurun_out/${T}_bench_stats.json > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.load(open('gpurun_out/${T}_bench_stats.json')); r=d['result']
print('C2', round(r['value']/1e6,2), 'M/s', round(r['ms_per_step'],2), 'ms parity', r.get('parity',{}).get('mismatches'), r['clocks'])
for k,v in sorted(d['stats']['per_launch_ms'].items(), key=lambda x:-x[1])[:10]: print('   %8.2f %s' % (v, k))"
[ $# -gt 0 ] && bash tools/gpu_configs.sh ${T} "$@"
