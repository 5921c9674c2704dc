"""Print per-kernel durations (us) from an ncu --metrics gpu__time_duration.sum CSV."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if 'Kernel Name' in r:
        h = r; start = i; break
ik = h.index('Kernel Name'); iv = h.index('Metric Value')
for r in rows[start + 1:]:
    name = r[ik].split('(')[0].replace('void ', '').replace('tod::<unnamed>::', '')
    print("%-40s %10.1f" % (name[:40], float(r[iv].replace(',', '')) / 1000))
