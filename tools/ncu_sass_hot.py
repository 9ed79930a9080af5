"""Summarise an ncu report's SASS source page: instruction mix and hot
instructions (samples), to read a kernel's bottleneck from the CLI.
    python tools/ncu_sass_hot.py REPORT.ncu-rep [top]"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out[1:]))
h = rows[0]
ix = {k: i for i, k in enumerate(h)}
data = []
for r in rows[1:]:
    if len(r) < len(h):
        continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    samp = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    ins = int(r[ix["Instructions Executed"]] or 0)
    data.append((r[ix["Address"]], src, op.split(".")[0], samp, ins))
tot_s = sum(d[3] for d in data) or 1
tot_i = sum(d[4] for d in data) or 1
mix = collections.Counter()
smix = collections.Counter()
for d in data:
    mix[d[2]] += d[4]
    smix[d[2]] += d[3]
print(f"{len(data)} SASS instructions, {tot_i} warp insts executed, {tot_s} samples")
print("opcode mix (executed %, samples %):")
for op, c in mix.most_common(25):
    print(f"  {op:10s} {100*c/tot_i:6.2f}%  {100*smix[op]/tot_s:6.2f}%")
print("hot instructions:")
for d in sorted(data, key=lambda d: -d[3])[:top]:
    print(f"  {100*d[3]/tot_s:5.2f}% {d[4]:>10d}  {d[0][-5:]}  {d[1][:90]}")
