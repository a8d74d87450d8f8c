"""Aggregate an `ncu --page source --csv` SASS dump (gzip or plain): executed warp instructions and
stall samples per opcode, plus the stall-reason totals.

    python tools/sass_profile.py gpurun_out/x_source.csv.gz [top]
"""
import collections
import csv
import gzip
import io
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = (gzip.open(path, "rt") if path.endswith(".gz") else open(path)).read()
rows = list(csv.reader(io.StringIO(txt)))
# several launches may be concatenated (one "Kernel Name" block each): keep the first
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"] + [len(rows)]
rows = rows[starts[0]:starts[1]]
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ex = collections.Counter()
samp = collections.Counter()
stall = collections.Counter()
for r in rows[2:]:
    if len(r) < len(hdr) or not r[ix["Source"]].strip():
        continue
    op = r[ix["Source"]].split()[0]
    if op.startswith("@"):
        op = r[ix["Source"]].split()[1]
    op = op.split(".")[0]
    ex[op] += int(r[ix["Instructions Executed"]] or 0)
    samp[op] += int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    for h, i in ix.items():
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                stall[h] += int(r[i] or 0)
            except ValueError:
                pass
tot_e, tot_s = sum(ex.values()), sum(samp.values())
print(f"{'opcode':12s} {'warp-inst':>14s} {'%inst':>6s} {'%samples':>8s}")
for op, n in ex.most_common(top):
    print(f"{op:12s} {n:14d} {100 * n / tot_e:6.2f} {100 * samp[op] / max(tot_s, 1):8.2f}")
print("stalls:", ", ".join(f"{k[6:]} {100 * v / max(sum(stall.values()), 1):.1f}%" for k, v in stall.most_common(10)))
