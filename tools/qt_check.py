"""A/B experiment knobs (TOD_<KEY>=v, e.g. MAIN_PAIR=0+RR_SPLIT=1): identical outputs, timings."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_2110_14007_b200 as tod  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=100_000)
ap.add_argument("--d", type=int, default=32)
ap.add_argument("--k", type=int, default=20)
ap.add_argument("--fmt", default="fp16")
ap.add_argument("--variants", default="MAIN_PAIR=1,MAIN_PAIR=0")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
X = torch.from_numpy(datagen.gaussian_mixture(a.n, a.d, seed=0)).cuda()
ref = None
for var in a.variants.split(","):
    env = dict(kv.split("=") for kv in var.split("+"))
    for key in ("MAIN_PAIR", "RR_GRID", "RR_SPLIT", "SAMPLE_V1", "SAMPLE_R"):
        os.environ.pop("TOD_" + key, None)
    for key, v in env.items():
        os.environ["TOD_" + key] = v
    with tod.Context(fmt=a.fmt, flags=tod.F_TIMING) as ctx:
        ts = []
        for _ in range(a.reps):
            r = ctx.knn(X, a.k, want=("idx", "dist"))
            torch.cuda.synchronize()
            ts.append((r.stats["ms_main_kernel"], r.stats["ms_main"], r.stats["ms_certify"], r.stats["ms_total"]))
        st = r.stats
        same = "ref" if ref is None else (bool(torch.equal(ref[0], r.idx)) and bool(torch.equal(ref[1], r.dist)))
        if ref is None:
            ref = (r.idx.clone(), r.dist.clone())
        mk, mm, mc, tt = ts[-1]
        print("%-14s main_kernel %.3f main %.3f cert %.3f total %.3f ms | kernel %d certified %d groups/row %.1f visited %.1f | identical %s"
              % (var, mk, mm, mc, tt, st["main_kernel"], st["certified"], st["cand_groups"] / a.n,
                 st["visited_groups"] / a.n, same), flush=True)
