"""Summarise ncu --set full captures into a markdown table (profiles/)."""
import csv, subprocess, sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active % of peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "smem wavefronts % of peak"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ("smsp__inst_executed.sum", "warp instructions"),
]


def summarize(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]
    m = {k: (x, un) for k, x, un in zip(h, v, u)}
    out = [f"### {m['Kernel Name'][0]}", "", f"capture: `{rep.split('/')[-1]}`", "",
           "| metric | value |", "|---|---|"]
    for k, name in KEYS:
        if k in m:
            x, un = m[k]
            out.append(f"| {name} | {x} {un} |")
    stalls = sorted(((float(x), k) for k, (x, un) in m.items()
                     if k.startswith("smsp__average_warps_issue_stalled_") and
                     k.endswith("_per_issue_active.ratio") and x not in ("", "n/a")),
                    reverse=True)[:6]
    out.append("| top stalls (warps per issue) | " + ", ".join(
        f"{k.split('stalled_')[1].split('_per_issue')[0]} {x:.2f}" for x, k in stalls) + " |")
    return "\n".join(out) + "\n"


if __name__ == "__main__":
    print("\n".join(summarize(r) for r in sys.argv[1:]))
