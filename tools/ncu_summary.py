"""Summarise an ncu --set full report into a small markdown file for profiles/.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/r01_x.md [algorithmic_bytes] [label]
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "sm__cycles_elapsed.avg.per_second",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep, dst = sys.argv[1], sys.argv[2]
    algo = float(sys.argv[3]) if len(sys.argv) > 3 else None
    label = sys.argv[4] if len(sys.argv) > 4 else rep
    hdr, units, data = raw(rep)
    lines = [f"# ncu --set full summary: {label}", "", f"source report: `{rep}` (not committed; 20 MB)", ""]
    for r in data:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        lines.append(f"## {name}")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        vals = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                vals[k] = r[i]
                lines.append(f"| {k} | {r[i]} | {units[i]} |")
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    v = float(r[i])
                except ValueError:
                    continue
                if v >= 0.05:
                    stalls.append((v, h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        lines.append("")
        lines.append("stall reasons (warps per issue-active cycle): " +
                     ", ".join(f"{n} {v:.2f}" for v, n in sorted(stalls, reverse=True)))
        try:
            rd = float(vals["dram__bytes_read.sum"]); wr = float(vals["dram__bytes_write.sum"])
            ur = units[hdr.index("dram__bytes_read.sum")]; uw = units[hdr.index("dram__bytes_write.sum")]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            traffic = rd * scale.get(ur, 1) + wr * scale.get(uw, 1)
            lines.append(f"\nDRAM traffic per launch: {traffic / 1e9:.4f} GB" +
                         (f" vs algorithmic {algo / 1e9:.4f} GB (ratio {traffic / algo:.3f})" if algo else ""))
        except Exception:
            pass
        lines.append("")
    open(dst, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
