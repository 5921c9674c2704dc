"""Analyse the per-tile clock64 trace of CTA 0 (TOD_F_DEBUG_TRACE)."""
import sys
import numpy as np
t = np.fromfile(sys.argv[1], dtype=np.int64).reshape(-1, 8)
mma = t[(t[:, 0] > 0) & (t[:, 2] > 0)][:, :3]
epi = t[(t[:, 3] > 0) & (t[:, 5] > 0)][:, 3:6]
print("tiles traced: mma %d epi %d" % (len(mma), len(epi)))
def q(x): return "p10 %6.0f  p50 %6.0f  p90 %6.0f" % tuple(np.percentile(x, [10, 50, 90]))
print("MMA   wait full      ", q(mma[:, 1] - mma[:, 0]))
print("MMA   wait t_empty+issue", q(mma[:, 2] - mma[:, 1]))
print("MMA   tile period    ", q(np.diff(mma[:, 0])))
print("EPI   wait t_full    ", q(epi[:, 1] - epi[:, 0]))
print("EPI   process        ", q(epi[:, 2] - epi[:, 1]))
print("EPI   tile period    ", q(np.diff(epi[:, 0])))
n = min(len(mma), len(epi))
base = min(mma[0, 0], epi[0, 0])
print("first tiles (cycles rel.): mma_start mma_full mma_done | epi_start epi_gotfull epi_done")
for i in range(100, 112):
    print(i, mma[i] - base, "|", epi[i] - base)
m = t[(t[:, 3] > 0) & (t[:, 5] > 0)][:, 6:8]
if len(m):
    big = m[:, 0] > 500
    print("tile-boundary reserve: p50 %.0f cycles; merges (>500 cyc): %d of %d tiles, mean %.0f cycles; pending after p50 %.0f max %d"
          % (np.median(m[:, 0]), big.sum(), len(m), m[big, 0].mean() if big.any() else 0, np.median(m[:, 1]), m[:, 1].max()))
