"""A/B a library build against the current one on the same box: python tools/ab_lib.py LIB --n .. --d .. --k .. --fmt .."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2110_14007_b200.tod as T  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("lib")
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--d", type=int, default=32)
ap.add_argument("--k", type=int, default=20)
ap.add_argument("--fmt", default="fp16")
ap.add_argument("--reps", type=int, default=4)
a = ap.parse_args()
T.load_library(a.lib)
X = torch.from_numpy(datagen.gaussian_mixture(a.n, a.d, seed=0)).cuda()
with T.Context(fmt=a.fmt, flags=T.F_TIMING) as ctx:
    for _ in range(a.reps):
        r = ctx.knn(X, a.k, want=("idx", "score_kth"))
        torch.cuda.synchronize()
    st = r.stats
    n = max(st["rows"], 1)
    print("%s: main %.3f (kernel %.3f, K%d) cert %.3f fb %.3f ms | per row: staged %.1f visited %.1f "
          "kept %.1f pre-skipped %.1f | certified %d/%d" % (os.path.basename(a.lib), st["ms_main"],
          st.get("ms_main_kernel", 0), st.get("main_kernel", 0), st["ms_certify"], st["ms_fallback"],
          st["cand_groups"] / n, st["visited_groups"] / n, st["cand_columns"] / n,
          st.get("prebound_skipped", 0) / n, st["certified"], n))
