"""Per-tile pipeline trace of the single-SM main pass (k_knn_tc3, CTA 0; TOD_F_DEBUG_TRACE):
python tools/trace_main.py --n 100000 --d 32 --k 20   (prints cycle percentiles per stage)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2110_14007_b200 as tod  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--d", type=int, default=32)
ap.add_argument("--k", type=int, default=20)
ap.add_argument("--fmt", default="fp16")
ap.add_argument("--out", default="/tmp/tod_trace.bin")
ap.add_argument("--lib", default=None, help="load this libtod.so instead of the in-tree one")
a = ap.parse_args()
os.environ["TOD_TRACE_FILE"] = a.out
if a.lib:
    import paper_2110_14007_b200.tod as T  # noqa: E402
    T.load_library(a.lib)
os.environ.setdefault("TOD_MAIN_PAIR", "0")
X = torch.from_numpy(datagen.gaussian_mixture(a.n, a.d, seed=0)).cuda()
with tod.Context(fmt=a.fmt, flags=tod.F_TIMING | (8 << 8)) as ctx:
    for _ in range(3):
        r = ctx.knn(X, a.k, want=("idx",))
        torch.cuda.synchronize()
print("pass 1 %.3f ms (main kernel %.3f ms)" % (r.stats["ms_main"], r.stats.get("ms_main_kernel", 0)))
t = np.fromfile(a.out, dtype=np.int64).reshape(-1, 16)
nacc = 3 if r.stats.get("main_kernel") == 5 else 2
ok = (t[:, 0] > 0) & (t[:, 2] > 0) & (t[:, 3] > 0) & (t[:, 6] > 0) & (t[:, 7] > 0) & (t[:, 8] > 0)
t = t[ok][50:]


def q(x):
    return "p10 %6.0f  p50 %6.0f  p90 %6.0f  mean %6.0f" % (*np.percentile(x, [10, 50, 90]), np.mean(x))


rel = np.maximum(t[:, 5], t[:, 10])  # accumulator free: the later of warp 2's and the last warp's release
print("tiles", len(t), "accumulators", nacc)
print("MMA  period               ", q(np.diff(t[:, 0])))
print("MMA  wait B tile          ", q(t[:, 1] - t[:, 0]))
print("MMA  wait accumulator     ", q(t[:, 2] - t[:, 1]))
print("MMA  issue (MMAs+commits) ", q(t[:, 8] - t[:, 2]))
print("FILT period               ", q(np.diff(t[:, 3])))
print("FILT wait t_full          ", q(t[:, 4] - t[:, 3]))
print("FILT ldtm (warp 2)        ", q(t[:, 9] - t[:, 4]))
print("FILT release (warp 2)     ", q(t[:, 5] - t[:, 4]))
print("FILT release skew last-w2 ", q(t[:, 10] - t[:, 5]))
print("FILT filter work          ", q(t[:, 6] - t[:, 5]))
print("MMA issued -> FILT full   ", q(t[:, 4] - t[:, 8]))
print("acc free(t) -> MMA acc ok(t+%d)" % nacc, q(t[nacc:, 2] - rel[:-nacc]))
print("PROD copy issue -> MMA got B", q(t[:, 1] - t[:, 7]))
