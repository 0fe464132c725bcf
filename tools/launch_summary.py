"""Print the last N launches of an ncu --csv launch list (duration, grid)."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
gi = h.index("Grid Size") if "Grid Size" in h else None
data = [(r[ki][:60], float(r[vi].replace(",", "")), r[gi] if gi is not None else "") for r in rows[1:]]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
tot = 0.0
for name, v, g in data[-n:]:
    tot += v
    print(f"{v / 1000:9.1f} us  {name}  {g}")
print(f"{len(data)} launches; last {n}: {tot / 1000:.1f} us")
