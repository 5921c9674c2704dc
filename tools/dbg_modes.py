"""Main-pass decomposition (profiling aid): full pass vs. the pipeline without the
filter work (flags dbg 1: TMEM loads kept; dbg 2: no TMEM loads), per main kernel."""
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
a = ap.parse_args()
X = torch.from_numpy(datagen.gaussian_mixture(a.n, a.d, seed=0)).cuda()
for pair in ("0", "1"):
    os.environ["TOD_MAIN_PAIR"] = pair
    for dbg in (0, 1, 2):
        with tod.Context(fmt="fp16", flags=tod.F_TIMING | (dbg << 8)) as ctx:
            for _ in range(3):
                r = ctx.knn(X, a.k, want=("idx",))
                torch.cuda.synchronize()
            print("pair %s dbg %d: pass 1 (sample + main) %.3f ms" % (pair, dbg, r.stats["ms_main"]), flush=True)
