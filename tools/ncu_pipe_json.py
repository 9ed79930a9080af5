"""Collect per-kernel ncu metrics into profiles/ncu_pipe.json (read by
bench.py's roofline "ncu" field) and profiles/ncu_traffic.json (roofline
"traffic").  Usage: python tools/ncu_pipe_json.py REPORT BENCH_NAME BATCH [REPORT ...]
(one report / bench kernel name / batch triple per kernel)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
        "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_warp_inst",
        "launch__registers_per_thread": "registers"}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return [dict(zip(rows[0], r)) for r in rows[2:]]


def main(args):
    out = os.environ.get("NCU_JSON_DIR", os.path.join(ROOT, "profiles"))
    pj = os.path.join(out, "ncu_pipe.json")
    tj = os.path.join(out, "ncu_traffic.json")
    pipe = json.load(open(pj)) if os.path.exists(pj) else {}
    traffic = json.load(open(tj)) if os.path.exists(tj) else {}
    for rep, name, batch, match in zip(args[0::4], args[1::4], args[2::4], args[3::4]):
        for d in raw(rep):
            # the solve kernel itself, not the one completing deferred systems
            if match not in d["Kernel Name"] or "deferred" in d["Kernel Name"]:
                continue
            e = {v: float(d[k]) for k, v in KEYS.items() if k in d}
            e["source"] = f"profiles/{os.path.basename(rep)} (ncu --set full, B = {batch})"
            pipe[name] = e
            rd, wr = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
            traffic[name] = {"dram_bytes": rd + wr, "batch": int(batch),
                             "source": e["source"]}
    json.dump(pipe, open(pj, "w"), indent=1)
    json.dump(traffic, open(tj, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:])
