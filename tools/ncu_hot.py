"""Top SASS lines by warp-stall samples of one kernel in an ncu report."""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kre}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
i = next(j for j, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i]
data = []
for r in rows[i + 1:]:
    if not r or r[0] in ("Kernel Name", "Address"):
        break   # (first matching launch only)
    data.append(r)
si, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
tot = sum(int(r[si] or 0) for r in data if len(r) > si)
print("total samples", tot)
for r in sorted(data, key=lambda r: -int(r[si] or 0))[:n]:
    top = sorted(((int(r[h.index(c)] or 0), c) for c in cols), reverse=True)[:2]
    print(f"{int(r[si]):6d} {r[0][-5:]} {r[src].strip()[:60]:60s} {top}")
