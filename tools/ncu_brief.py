"""One line per kernel (largest launch) from a tools/ncu_summary.py markdown file."""
import re
import sys

txt = open(sys.argv[1]).read()
best = {}
for s in txt.split("\n## ")[1:]:
    name = s.split("(")[0].strip()
    m = re.search(r"gpu__time_duration.sum \| ([\d.]+) \| (\w+)", s)
    t = float(m.group(1)) * (1000 if m.group(2) == "ms" else 1)
    if name not in best or t > best[name][0]:
        best[name] = (t, s)
print("| kernel (largest launch) | us | warps/SM | issue % | fma % | alu % | DRAM GB | top stalls |")
print("|---|---|---|---|---|---|---|---|")
for name, (t, s) in sorted(best.items(), key=lambda kv: -kv[1][0]):
    def g(k):
        m = re.search(re.escape(k) + r" \| ([\d.]+) \| (\w*)", s)
        return (float(m.group(1)), m.group(2)) if m else (float("nan"), "")
    rd, ru = g("dram__bytes_read.sum")
    wr, wu = g("dram__bytes_write.sum")
    sc = {"Gbyte": 1, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9}
    dram = rd * sc.get(ru, 0) + wr * sc.get(wu, 0)
    st = re.search(r"stall reasons.*?: (.*)", s).group(1).split(", ")[:3]
    print(f"| `{name.replace('void ', '')}` | {t:.0f} | {g('sm__warps_active.avg.per_cycle_active')[0]:.1f} | "
          f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active')[0]:.0f} | "
          f"{g('sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active')[0]:.0f} | "
          f"{g('sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active')[0]:.0f} | {dram:.3f} | {'; '.join(st)} |")
