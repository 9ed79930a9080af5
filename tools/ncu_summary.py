"""One-screen summary of an ncu --set full report (run here, no GPU):
duration, occupancy, pipe utilisation, issue stalls, local-memory traffic."""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe inst % of peak"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe cycles active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "lsu pipe %"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "xu pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__instruction_throughput.avg.pct_of_peak_sustained_active", "SM inst throughput %"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active threads / warp inst"),
    ("dram__bytes_read.sum", "dram read bytes"),
    ("dram__bytes_write.sum", "dram write bytes"),
    ("l1tex__t_sector_pipe_lsu_mem_local_op_ld_hit_rate.pct", "local ld L1 hit %"),
    ("sass__inst_executed_local_loads", "local load insts"),
    ("sass__inst_executed_local_stores", "local store insts"),
    ("smsp__inst_executed.sum", "warp insts executed"),
]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    units = dict(zip(hdr, rows[1]))  # ncu scales units per report (ns/us/ms, byte/Kbyte/...)
    for vals in rows[2:]:
        summarize(path, dict(zip(hdr, vals)), units)


def summarize(path, d, units):
    print(f"== {path}  kernel: {d.get('Kernel Name', '?')[:90]}")
    for k, label in KEYS:
        if k in d:
            u = units.get(k, "")
            lab = f"{label} ({u})" if u and u not in ("%",) else label
            print(f"  {lab:32s} {d[k]}")
    stalls = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(v), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    print("  top stalls (warps per issue):", ", ".join(f"{n} {v:.2f}" for v, n in stalls[:6]))

if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
