"""Key metrics of an `ncu --set full` report (read offline with `ncu -i`): duration, DMMA-pipe
activity, occupancy limits, waves, DRAM bytes, shared-memory bank conflicts and the stall
breakdown per issued instruction.  Usage: python tools/ncu_summary.py report.ncu-rep [...]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("launch__grid_size", "grid CTAs"),
    ("launch__registers_per_thread", "registers"),
    ("launch__shared_mem_per_block_dynamic", "smem/CTA"),
    ("launch__occupancy_limit_registers", "occ limit regs"),
    ("launch__occupancy_limit_shared_mem", "occ limit smem"),
    ("launch__waves_per_multiprocessor", "waves/SM"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active %"),
    ("sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active", "DMMA inst % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "smem ld bank conflicts"),
    ("smsp__inst_executed_op_shared_ld.sum", "smem ld instr"),
]
STALLS = ["wait", "math_pipe_throttle", "long_scoreboard", "short_scoreboard", "barrier", "not_selected", "selected",
          "no_instruction", "branch_resolving", "dispatch_stall", "drain", "mio_throttle"]


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    name_col = idx.get("Kernel Name")
    out = [f"# {path}"]
    for r in data:
        out.append(f"## {r[name_col][:110] if name_col is not None else '?'}")
        for k, label in KEYS:
            if k in idx:
                out.append(f"  {label:26s} {r[idx[k]]:>14s} {units[idx[k]]}")
        st = []
        for s in STALLS:
            k = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
            if k in idx:
                st.append(f"{s} {float(r[idx[k]]):.2f}")
        out.append("  stalls per issue: " + ", ".join(st))
    return "\n".join(out)


if __name__ == "__main__":
    print("\n\n".join(summarize(p) for p in sys.argv[1:]))
