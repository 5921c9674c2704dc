"""Per-kernel share of a step from an ncu gpu__time_duration launch list (CSV)."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
i0 = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[i0]; ik = h.index('Kernel Name'); iv = h.index('Metric Value'); iu = h.index('Metric Unit')
tot = collections.OrderedDict()
for r in rows[i0 + 1:]:
    name = r[ik].split('(')[0].replace('void ', '').replace('tod::<unnamed>::', '').strip()
    if name.startswith('at::') or 'elementwise' in name:
        continue
    scale = {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3}.get(r[iu], 1e-3)
    tot[name] = tot.get(name, 0.0) + float(r[iv].replace(',', '')) * scale
T = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print("%-34s %9.1f us/step  %5.1f %%" % (k, v / steps, 100 * v / T))
