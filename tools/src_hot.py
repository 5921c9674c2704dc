"""Per-source-line executed instructions and stall samples from an ncu report (CUDA source view)."""
import csv, io, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = next(i for i, r in enumerate(rows) if "Source" in r)
h = rows[hi]
iE, iS, iL = h.index("Instructions Executed"), h.index("Source"), h.index("Line") if "Line" in h else 0
iW = h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[hi + 1:]:
    if len(r) < len(h): continue
    try:
        e = int(r[iE] or 0); w = int(r[iW] or 0)
    except ValueError:
        continue
    data.append((r[iL], r[iS].strip()[:90], e, w))
E = sum(d[2] for d in data) or 1; W = sum(d[3] for d in data) or 1
for l, s, e, w in sorted(data, key=lambda x: -x[2])[:top]:
    print("%5s %6.2f%% %6.2f%%  %s" % (l, 100.0 * e / E, 100.0 * w / W, s))
