"""Small invocations of every kernel family, for compute-sanitizer
(memcheck / racecheck / synccheck): two-pass kNN (key-only sample, single-SM
main pass), d=64 bf16 (list sample, CTA-pair main pass, second tier), d=128
(K-pipelined main pass), forced fallback tiers, LOF, NWR, ABOD, the loopback
ring.  Outputs are not checked here (the GPU tests do that)."""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import datagen
import paper_2110_14007_b200 as pkg

which = sys.argv[1] if len(sys.argv) > 1 else "all"


def X(n, d, seed=0):
    return torch.from_numpy(datagen.gaussian_mixture(n, d, seed=seed)).cuda()


if which in ("all", "knn"):
    with pkg.Context(device=0, fmt="fp16") as c:
        c.knn(X(9000, 32), 10)                       # k_knn_tc3 sample + main, re-rank
    with pkg.Context(device=0, fmt="bf16") as c:
        c.knn(X(9000, 64, 1), 10)                    # knn_tc list sample, k_knn_tc4, tier 2
    with pkg.Context(device=0, fmt="fp16") as c:
        c.knn(X(9000, 128, 2), 8)                    # K-pipelined tc3
if which in ("all", "fallback"):
    with pkg.Context(device=0, flags=pkg.F_NO_CERTIFY) as c:
        c.knn(X(5000, 32, 3), 10)                    # threshold + brute-force tiers
    with pkg.Context(device=0, fmt="fp32") as c:
        c.knn(X(5000, 12, 4), 6)                     # SIMT pass
if which in ("all", "lof"):
    with pkg.Context(device=0) as c:
        c.lof(X(9000, 32, 5), 10)
        c.abod(X(3000, 16, 6), 8)
if which in ("all", "nwr"):
    with pkg.Context(device=0) as c:
        c.nwr(X(9000, 32, 7), 12.0)
if which in ("all", "ring"):
    with pkg.Context(device=0, fmt="fp16") as c:
        c.comm_init_loopback(2)
        c.knn_sharded(X(9000, 32, 8), 9000, 0, 10)
torch.cuda.synchronize()
print("sanitize cases done:", which)
