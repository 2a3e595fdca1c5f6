#!/usr/bin/env python
"""Per-opcode warp-stall breakdown from an ncu report's source page (SASS)."""
import collections
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[1]
isrc, iall, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
sc = [i for i, n in enumerate(h) if n.startswith("stall_") and "Not Issued" not in n]
data = [r for r in rows[2:] if len(r) == len(h)]
agg = collections.defaultdict(collections.Counter)
tot = collections.Counter()
for r in data:
    toks = r[isrc].split()
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    for i in sc:
        v = int(r[i] or 0)
        agg[op][h[i]] += v
        tot[h[i]] += v
print("total", sum(tot.values()), tot.most_common(8))
for op, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:14]:
    print(f"{op:10s} {sum(c.values()):7d}", c.most_common(4))
if len(sys.argv) > 2:
    for r in sorted(data, key=lambda r: -int(r[iall] or 0))[: int(sys.argv[2])]:
        print(r[iall].rjust(6), r[iex].rjust(10), r[isrc][:100])
