export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_nrall.so
timeout 900 python -m pytest tests -m gpu -q -k "c2 or edge or registry or defer or poly" > gpurun_out/r02AY_pytest.log 2>&1; echo "nrall pytest rc=$? $(tail -1 gpurun_out/r02AY_pytest.log)"
unset NLK_LIB_PATH
for lib in default nrall; do
  if [ $lib = default ]; then unset NLK_LIB_PATH; else export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_$lib.so; fi
  timeout 900 python bench.py --config c2 --steps 3 --warmup 1 --e2e-steps 0 --no-cpu-baseline --only "newton" --stats gpurun_out/r02AY_$lib.json > /dev/null 2>&1
done
python - <<'PY'
import json
a=json.load(open('gpurun_out/r02AY_default.json'))['stats']['per_launch_ms']; b=json.load(open('gpurun_out/r02AY_nrall.json'))['stats']['per_launch_ms']
print('total', round(sum(a.values()),2), round(sum(b.values()),2))
for k in sorted(a, key=lambda k: -a[k])[:12]: print('  %-60s %8.2f %8.2f' % (k[13:-1], a[k], b[k]))
PY
