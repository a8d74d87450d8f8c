"""Markdown table (launches, total us, share) from an `ncu --metrics gpu__time_duration.sum --csv`
launch list:  python tools/launch_table.py launches.csv > table.md"""
import csv
import io
import sys
from collections import defaultdict

text = open(sys.argv[1]).read()
start = text.index('"ID"')
rows = list(csv.DictReader(io.StringIO(text[start:])))
tot = defaultdict(float)
cnt = defaultdict(int)
per = defaultdict(list)
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    us = v / 1e3 if r["Metric Unit"] in ("ns", "nsecond") else (v * 1e3 if r["Metric Unit"] in ("ms", "msecond") else v)
    name = r["Kernel Name"].split("(")[0]
    if len(name) > 110:
        name = name[:110] + "..."
    tot[name] += us
    cnt[name] += 1
    per[name].append(us)
all_us = sum(tot.values())
print("| kernel | launches | total us | share |")
print("|---|---|---|---|")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"| `{k}` | {cnt[k]} | {tot[k]:.1f} | {100 * tot[k] / all_us:.1f}% |")
big = [k for k in per if "k_cpmul" in k]
for k in big:
    print(f"\n`{k}` per-launch us: " + ", ".join(f"{u:.0f}" for u in per[k] if u > 500))
