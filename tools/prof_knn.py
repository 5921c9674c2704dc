"""Profiling driver: tod_knn calls on a seeded mixture (for ncu / phase timings)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2110_14007_b200 as tod  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=200_000)
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--k", type=int, default=10)
ap.add_argument("--fmt", default="fp16")
ap.add_argument("--chunks", type=int, default=0)
ap.add_argument("--kprime", type=int, default=0)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--flags", type=int, default=0)
ap.add_argument("--split", type=int, default=0)
a = ap.parse_args()
X = torch.from_numpy(datagen.gaussian_mixture(a.n, a.d, seed=0)).cuda()
with tod.Context(fmt=a.fmt, chunks=a.chunks, kprime=a.kprime, flags=tod.F_TIMING | a.flags, split=a.split) as ctx:
    for _ in range(a.reps):
        r = ctx.knn(X, a.k, want=("idx", "score_kth"))
        torch.cuda.synchronize()
        st = r.stats
        print("cert %d fb %d kp %d S %d | prep %.3f main %.3f cert %.3f fb %.3f ms | per row: groups %.1f visited %.1f cols %.1f"
              % (st["certified"], st["fallback_rows"], st["kprime"], st["chunks"], st["ms_prep"],
                 st["ms_main"], st["ms_certify"], st["ms_fallback"], st["cand_groups"] / a.n,
                 st["visited_groups"] / a.n, st["cand_columns"] / a.n))
