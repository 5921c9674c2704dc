import sys, os
sys.path.insert(0, os.getcwd())
import torch, numpy as np, datagen
import paper_2110_14007_b200 as tod
X = datagen.gaussian_mixture(9000, 16, seed=9000+48)
with tod.Context(fmt="fp16", chunks=2) as ctx:
    r = ctx.knn(torch.from_numpy(X).cuda(), 6)
    print(r.stats)
