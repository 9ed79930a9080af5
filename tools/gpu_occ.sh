for x in 0 30000; do
  export NLK_EXTRA_SMEM=$x
  python bench.py --config c2 --batch 1048576 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --only "trigonometric:newton,matrix-sqrt-3x3:trust" --stats gpurun_out/occ_$x.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/occ_$x.json')); print('extra $x', {k[13:-1]: round(v,2) for k, v in d['stats']['per_launch_ms'].items()})"
done
