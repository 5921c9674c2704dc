import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import datagen, oracle
import paper_2110_14007_b200 as tod
n, d, k = 2500, 64, 10
X = datagen.gaussian_mixture(n, d, seed=n + d)
ri, rd = oracle.knn(X, k)
for fmt in ("bf16", "fp16"):
    for sp in (1, 2, 4):
        for chunks in (0, 1):
            with tod.Context(fmt=fmt, split=sp, chunks=chunks) as ctx:
                r = ctx.knn(torch.from_numpy(X).cuda(), k)
            gi = r.idx.cpu().numpy()
            bad = np.nonzero((gi != ri).any(1))[0]
            st = r.stats
            print(fmt, "split", sp, "chunks", st["chunks"], "kp", st["kprime"], "cert", st["certified"], "fb", st["fallback_rows"], "bad rows", len(bad), bad[:5])
            if len(bad):
                b = bad[0]
                print("  gpu", gi[b], "\n  ora", ri[b])
                print("  gpu d", r.dist64.cpu().numpy()[b][:4], "ora d", np.sqrt(rd[b][:4]))
