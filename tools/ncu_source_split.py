"""Attribute warp-stall samples and executed instructions to source files and
lines from `ncu -i REP --page source --csv --print-source cuda,sass` output.
    python tools/ncu_source_split.py src.csv [top_lines]"""
import csv
import sys
from collections import defaultdict


def main(path, top=25):
    kern = None
    per_file = defaultdict(lambda: defaultdict(lambda: [0, 0]))
    per_line = defaultdict(lambda: defaultdict(lambda: [0, 0, "", 0]))
    fpath = None
    hdr = None
    for row in csv.reader(open(path)):
        if not row:
            continue
        if row[0] == "File Path":
            fpath = row[1].split("/")[-1]
            continue
        if row[0] == "Function Name":
            kern = row[1]
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or not row[0].isdigit():
            continue
        d = dict(zip(hdr, row))
        s = int(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
        ins = int(d.get("Instructions Executed", "0") or 0)
        thr = int(d.get("Thread Instructions Executed", "0") or 0)
        per_file[kern][fpath][0] += s
        per_file[kern][fpath][1] += ins
        pl = per_line[kern][(fpath, int(row[0]))]
        pl[0] += s
        pl[1] += ins
        pl[2] = row[1][:70]
        pl[3] += thr
    for k in per_file:
        tot_s = sum(v[0] for v in per_file[k].values()) or 1
        tot_i = sum(v[1] for v in per_file[k].values()) or 1
        print(f"== {k}\n   samples {tot_s}  warp insts {tot_i}")
        for f, (s, i) in sorted(per_file[k].items(), key=lambda x: -x[1][0]):
            print(f"   {100*s/tot_s:5.1f}% samples {100*i/tot_i:5.1f}% insts  {f}")
        print("   samples% insts% threads/inst  line")
        for (f, ln), (s, i, src, thr) in sorted(per_line[k].items(), key=lambda x: -x[1][0])[:top]:
            tpi = thr / i if i else 0.0
            print(f"   {100*s/tot_s:5.1f}% {100*i/tot_i:5.1f}% {tpi:5.1f}  {f}:{ln}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
