"""Executed-instruction mix by SASS opcode from an ncu source-page dump."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
isrc, iex = h.index("Source"), h.index("Instructions Executed")
mix = collections.Counter()
for r in rows[2:]:
    if not r[iex].isdigit():
        continue
    op = r[isrc].split()
    op = [o for o in op if not o.startswith("@")]
    mix[op[0].split(".")[0] if op else "?"] += int(r[iex])
tot = sum(mix.values())
print("total", tot)
for k, v in mix.most_common(30):
    print(f"{k:12s} {v:12d} {100*v/tot:5.1f}%")
