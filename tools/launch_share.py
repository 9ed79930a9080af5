"""Per-kernel share of the step from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv python bench.py`),
next to the share measured live by bench.py (--stats JSON), to check that the
dominant kernel's share agrees (ncu times are serialised, cold-cache).
    python tools/launch_share.py launches.csv [bench_stats.json]"""
import csv
import json
import re
import sys
from collections import defaultdict


def main(path, stats=None):
    rows = [r for r in csv.DictReader(l for l in open(path) if l.startswith('"'))]
    per = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        per[r["Kernel Name"]].append(float(r["Metric Value"].replace(",", "")) / 1e6)
    tot = sum(sum(v) for v in per.values())
    print(f"ncu launch list: {len(rows)} launches, {tot:.1f} ms total kernel time")
    live = None
    if stats:
        live = json.load(open(stats))["stats"]["per_launch_ms"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1]))[:15]:
        print(f"  {100 * sum(v) / tot:5.1f}%  {len(v):4d} launches  mean {sum(v) / len(v):9.3f} ms  {k[:100]}")
    if live:
        lt = sum(live.values())
        print(f"bench.py live (CUDA events, one step): {lt:.1f} ms")
        for k, v in sorted(live.items(), key=lambda kv: -kv[1])[:8]:
            print(f"  {100 * v / lt:5.1f}%  {v:9.3f} ms  {k}")


if __name__ == "__main__":
    main(*sys.argv[1:])
