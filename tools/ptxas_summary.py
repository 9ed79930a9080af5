"""Summarise nvcc -Xptxas -v logs (paper_2403_16341_b200/_obj/*.ptxas.log):
registers, stack frame and spill bytes per solve-kernel instantiation."""
import glob
import os
import re
import sys

ALGS = ["NR", "TR", "Broyden", "Klement", "DFSane", "NR-LS"]


def parse(path):
    rows, cur = [], None
    for line in open(path):
        m = re.search(r"Compiling entry function '(\S+)'", line)
        if m:
            cur = {"sym": m.group(1)}
            rows.append(cur)
            continue
        if cur is None:
            continue
        m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            cur["stack"], cur["spill_st"], cur["spill_ld"] = map(int, m.groups())
        m = re.search(r"Used (\d+) registers", line)
        if m:
            cur["regs"] = int(m.group(1))
    return rows


def pretty(sym):
    m = re.match(r"_ZN3nlk12solve_kernelINS_(\d+)(\w+?)(ILi(\d+)EEE|E)Li(\d+)E([df])Li(\d)E", sym)
    if not m:
        return sym
    name = m.group(2)
    return f"{name}{'<'+m.group(4)+'>' if m.group(4) else ''} n={m.group(5)} {'f64' if m.group(6)=='d' else 'f32'} {ALGS[int(m.group(7))]}"


if __name__ == "__main__":
    logs = sorted(glob.glob(os.path.join(sys.argv[1] if len(sys.argv) > 1 else "paper_2403_16341_b200/_obj", "*.ptxas.log")))
    print(f"{'kernel':50s} {'regs':>5s} {'stack':>6s} {'spill_st':>9s} {'spill_ld':>9s}")
    for lg in logs:
        for r in parse(lg):
            print(f"{pretty(r['sym']):50s} {r.get('regs',0):5d} {r.get('stack',0):6d} {r.get('spill_st',0):9d} {r.get('spill_ld',0):9d}")
