bash tools/gpu_check_stats.sh r02O
bash tools/gpu_ab.sh r02Og "trigonometric,matrix-sqrt,brown" "trigonometric or sqrt or brown" grs
for B in 1048576 2097152 4194304; do
  timeout 600 python bench.py --config c2 --batch $B --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --only "trigonometric:newton,matrix-sqrt-3x3:trust" --stats gpurun_out/r02O_tail_$B.json > /dev/null 2>&1
  python -c "
import json; d=json.load(open('gpurun_out/r02O_tail_$B.json')); print($B, {k[13:-1]: round(v*1048576/$B,2) for k, v in d['stats']['per_launch_ms'].items()}, '(ms per 1M systems)')"
done
