export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_$1.so
timeout 600 python -m pytest tests -m gpu -q -x -k "dfsane or c4 or c5 or quadratic" 2>&1 | tail -2
for lib in default "$@"; do
  if [ $lib = default ]; then unset NLK_LIB_PATH; else export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_$lib.so; fi
  for c in c4 c5; do
    if [ $c = c4 ]; then a="--config c4 --batch 10000000 --steps 5 --warmup 2"; else a="--config c5 --batch 12500000 --steps 200 --warmup 5"; fi
    python bench.py $a --e2e-steps 0 --no-cpu-baseline --stats gpurun_out/${T:-r02q}_${c}_${lib}_stats.json > /dev/null 2>&1
    python -c "
import json; d=json.load(open('gpurun_out/${T:-r02q}_${c}_${lib}_stats.json')); print('$lib $c', round(d['result']['value']/1e6,1), {k[13:-1]: round(v,3) for k, v in d['stats']['per_launch_ms'].items()})"
  done
done
