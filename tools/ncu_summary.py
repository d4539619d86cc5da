"""Summarize an ncu report: key SOL / occupancy / smem / stall metrics and
per-opcode shared-memory wavefronts (from the source page).

    python tools/ncu_summary.py report.ncu-rep [> profiles/<name>.txt]
"""
import csv
import io
import subprocess
import sys

KEYS = ("Duration", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy", "Issue Slots Busy",
        "Executed Instructions", "Eligible Warps Per Scheduler", "No Eligible", "DRAM Throughput",
        "L1/TEX Cache Throughput", "Memory Throughput", "Warp Cycles Per Issued Instruction", "Compute (SM) Throughput",
        "Achieved Active Warps Per SM", "Dynamic Shared Memory Per Block", "Block Limit Registers",
        "Block Limit Shared Mem", "SM Frequency", "Grid Size", "Block Size")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
       "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
       "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
       "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_tmem.avg.pct_of_peak_sustained_active",
       "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active")


def run(args):
    return subprocess.run(["ncu", "-i", *args], capture_output=True, text=True).stdout


def main(path):
    out = []
    rows = list(csv.reader(io.StringIO(run([path, "--page", "details", "--csv"]))))
    hdr = rows[0]
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in KEYS:
            out.append(f"{d['Metric Name']:45s} {d['Metric Value']:>16s} {d.get('Metric Unit', '')}")
    raw = list(csv.reader(io.StringIO(run([path, "--page", "raw", "--csv"]))))
    if len(raw) >= 3:
        d = dict(zip(raw[0], raw[2]))
        for k in RAW:
            if k in d:
                out.append(f"{k:80s} {d[k]}")
    src = list(csv.reader(io.StringIO(run([path, "--page", "source", "--csv", "--print-source", "sass"]))))
    if len(src) > 2:
        h = {n: i for i, n in enumerate(src[1])}
        tot = {}
        for r in src[2:]:
            try:
                s = r[h["Source"]].split()
                op = s[1] if s and s[0].startswith("@") else (s[0] if s else "")
                wf = float(r[h["L1 Wavefronts Shared"]] or 0)
                ex = float(r[h["Instructions Executed"]] or 0)
            except (KeyError, ValueError, IndexError):
                continue
            if wf > 0:
                t = tot.setdefault(op, [0.0, 0.0])
                t[0] += wf
                t[1] += ex
        out.append("shared-memory wavefronts by opcode (total, per instruction):")
        for op, (wf, ex) in sorted(tot.items(), key=lambda x: -x[1][0]):
            out.append(f"  {op:24s} {wf / 1e6:9.2f} M   {wf / max(ex, 1):.2f}/instr")
    print("\n".join(out))


if __name__ == "__main__":
    main(sys.argv[1])
