"""Print selected columns of a trace_fwd.py per-step table: python tools/trace_cols.py FILE 'col a' 'col b' ..."""
import sys
lines = open(sys.argv[1]).read().split("\n")
h = lines[0]
hdr = [h[4 + 14 * i: 4 + 14 * (i + 1)].strip() for i in range((len(h) - 4) // 14)]
rows = [l.split() for l in lines[1:] if l.strip() and l.split()[0].isdigit()]
want = sys.argv[2:] or hdr
idx = [hdr.index(w) for w in want]
print("step " + " ".join(f"{w:>13s}" for w in want))
for r in rows:
    print(f"{r[0]:>4s} " + " ".join(f"{r[1 + i]:>13s}" for i in idx))
