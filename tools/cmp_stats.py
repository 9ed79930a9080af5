"""Compare per-launch kernel times of several `bench.py --stats` JSON files.
    python tools/cmp_stats.py a.json b.json ... [--top 20]"""
import json
import sys

paths = [a for a in sys.argv[1:] if a.endswith(".json")]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 20
runs = [json.load(open(p)) for p in paths]
pls = [r["stats"]["per_launch_ms"] for r in runs]
keys = sorted(pls[0], key=lambda k: -max(pl.get(k, 0) for pl in pls))
print("  ".join(f"{p.split('/')[-1][:14]:>14}" for p in paths), " kernel")
print("  ".join(f"{sum(pl.values()):14.1f}" for pl in pls), " TOTAL ms")
for k in keys[:top]:
    print("  ".join(f"{pl.get(k, float('nan')):14.2f}" for pl in pls), "", k.replace("solve_kernel<", "")[:-1])
