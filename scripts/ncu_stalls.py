"""Summarise an ncu --page source --csv --print-source sass dump: top
instructions per stall reason (usage: python scripts/ncu_stalls.py dump.csv [reason...])."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
data = rows[2:]
isrc = h.index("Source")
reasons = sys.argv[2:] or ["stall_long_sb", "stall_barrier", "stall_short_sb", "stall_wait", "stall_mio", "stall_math"]
for rs in reasons:
    k = h.index(rs)
    tot = sum(int(r[k]) for r in data if r[k].isdigit())
    print(f"== {rs}: {tot}")
    top = sorted(range(len(data)), key=lambda i: -int(data[i][k]) if data[i][k].isdigit() else 0)[:6]
    for i in top:
        print("  ", data[i][k].rjust(6), data[i - 1][isrc][:60].ljust(60), "=>", data[i][isrc][:70])
