"""tod_nwr phase timings on the C2 data at two radii (profiling aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, datagen
import paper_2110_14007_b200 as tod
X = torch.from_numpy(datagen.gaussian_mixture(100000, 32, seed=0)).cuda()
with tod.Context(flags=tod.F_TIMING) as ctx:
    for phi in (8.0, 12.0):
        for _ in range(2):
            c, p, l, st = ctx.nwr(X, phi)
        print(phi, {k: round(v, 3) if isinstance(v, float) else v for k, v in st.items() if k.startswith("ms") or k in ("fallback_rows", "kernel_launches")})
