"""Executed-instruction mix and stall samples per opcode from an `ncu --page source --csv
--print-source sass` export:  python tools/sass_mix.py file.csv [file2.csv]"""
import csv
import sys
from collections import Counter


def mix(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    isrc, iex, ist = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    ex, st = Counter(), Counter()
    for r in rows[2:]:
        if len(r) <= iex:
            continue
        toks = r[isrc].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") else toks[0]
        op = op.rstrip(";")
        ex[op] += int(r[iex] or 0)
        st[op] += int(r[ist] or 0)
    return ex, st


res = [mix(p) for p in sys.argv[1:]]
ops = sorted(set().union(*[r[0] for r in res]), key=lambda o: -res[0][0].get(o, 0))
tot = [sum(r[0].values()) for r in res]
print(f"{'op':24s}" + "".join(f"{'exec(M)':>10s}{'stall%':>8s}" for _ in res))
for o in ops[:40]:
    print(f"{o:24s}" + "".join(f"{r[0].get(o, 0) / 1e6:10.2f}{100 * r[1].get(o, 0) / max(1, sum(r[1].values())):8.1f}" for r in res))
print(f"{'TOTAL':24s}" + "".join(f"{t / 1e6:10.2f}{'':8s}" for t in tot))
