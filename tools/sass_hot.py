"""Dump SASS lines of an ncu report with executed-instruction counts and stall samples:
python tools/sass_hot.py REP [min_exec_fraction]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.001
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
iE, iS, iA, iW = h.index("Instructions Executed"), h.index("Source"), h.index("Address"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) < len(h): continue
    e = int(r[iE] or 0); w = int(r[iW] or 0)
    data.append((r[iA][-5:], r[iS].strip(), e, w))
E = sum(d[2] for d in data); W = sum(d[3] for d in data)
print("total exec", E, "samples", W)
for a, s, e, w in data:
    if e >= thr * E or w >= thr * W:
        print("%s %8.3f%% %6.2f%%  %s" % (a, 100.0 * e / E, 100.0 * w / W, s))
