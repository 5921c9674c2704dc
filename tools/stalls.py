"""Per-reason warp-stall totals from an ncu source CSV (--page source --csv --print-source sass),
optionally restricted to an address range (hex substrings of the epilogue loop)."""
import csv
import subprocess
import sys
import io

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
reasons = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in reasons}
iE = h.index("Instructions Executed")
iS = h.index("Source")
tot = {c: 0 for c in reasons}
ops = {}
for r in rows[2:]:
    if len(r) < len(h):
        continue
    for c in reasons:
        try:
            tot[c] += int(r[idx[c]] or 0)
        except ValueError:
            pass
    try:
        e = int(r[iE] or 0)
    except ValueError:
        e = 0
    op = r[iS].split()[0] if r[iS].split() else "?"
    if op.startswith("@"):
        op = r[iS].split()[1]
    op = op.split(".")[0]
    ops[op] = ops.get(op, 0) + e
T = sum(tot.values())
for c, v in sorted(tot.items(), key=lambda x: -x[1]):
    if v:
        print("%-28s %6.2f%%" % (c, 100.0 * v / T))
E = sum(ops.values())
print("--- executed instruction mix")
for op, v in sorted(ops.items(), key=lambda x: -x[1])[:25]:
    print("%-14s %6.2f%%" % (op, 100.0 * v / E))
