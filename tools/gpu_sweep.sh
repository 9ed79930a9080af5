#!/bin/bash
# Per-launch times of every job of C2/C3/C4/C5 for the default and variant
# libraries (per-kernel compiler-option sweeps).   tools/gpu_sweep.sh TAG variant...
T=$1; shift
mkdir -p gpurun_out
for lib in default "$@"; do
  if [ $lib = default ]; then unset NLK_LIB_PATH; else export NLK_LIB_PATH=paper_2403_16341_b200/libnlk_b200_$lib.so; fi
  timeout 900 python bench.py --config c2 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --stats gpurun_out/${T}_${lib}_c2.json > /dev/null 2>&1
  timeout 600 python bench.py --config c3 --batch 10000000 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --stats gpurun_out/${T}_${lib}_c3.json > /dev/null 2>&1
  timeout 600 python bench.py --config c4 --batch 10000000 --steps 2 --warmup 1 --e2e-steps 0 --no-cpu-baseline --stats gpurun_out/${T}_${lib}_c4.json > /dev/null 2>&1
  timeout 600 python bench.py --config c5 --batch 12500000 --steps 20 --warmup 3 --e2e-steps 0 --no-cpu-baseline --stats gpurun_out/${T}_${lib}_c5.json > /dev/null 2>&1
  echo "$lib done"
done
python - "$T" default "$@" <<'PY'
import json, sys
T, libs = sys.argv[1], sys.argv[2:]
rows = {}
for lib in libs:
    for c in ("c2", "c3", "c4", "c5"):
        try:
            d = json.load(open(f"gpurun_out/{T}_{lib}_{c}.json"))
        except Exception:
            continue
        for k, v in d["stats"]["per_launch_ms"].items():
            rows.setdefault(f"{c}:{k[13:-1]}", {})[lib] = v
print("%-60s " % "job" + " ".join("%9s" % l for l in libs))
for k, r in sorted(rows.items(), key=lambda x: -x[1].get("default", 0)):
    if r.get("default", 0) < 0.5:
        continue
    print("%-60s " % k[:60] + " ".join("%9.2f" % r.get(l, float("nan")) for l in libs))
PY
