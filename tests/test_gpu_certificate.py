"""The certificate's tensor-core error model (reading A9), checked on
the library's OWN main-pass kernels (k_knn_tc3 single-SM, k_knn_tc4 CTA pairs),
not on a library GEMM.  The verification step (iii) of provable quantization
(§5.1) bounds |w~ - w| with the accumulation model; its check
form is Eq. 4.  tod_debug_mainpass returns the raw fp32 accumulators
w~ of one 128-row query tile against every reference row, plus the 16-bit
operands exactly as multiplied, so the exact w = sum_c a_c b_c is known (every
product is exact in fp32; the fp64 sum below errs by < K 2^-53 sum|ab|).
Over >= 1e7 pairs per (dpad, format), including adversarial dynamic range
(one feature 2^12 larger than the rest, the bad case of alignment truncation),
no pair may exceed the model 17 ceil(K/16) 2^-23 sum_c |a_c b_c|."""
import numpy as np
import pytest

import datagen

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2110_14007_b200 import build
    build.build()
    import paper_2110_14007_b200 as p
    return p


def _datasets(n, d):
    yield "mixture", datagen.gaussian_mixture(n, d, seed=21)
    x = datagen.gaussian_mixture(n, d, seed=22)
    x[:, 0] *= 4096.0                     # one dominant feature: per-K-step dynamic range 2^12
    yield "dominant-feature", np.ascontiguousarray(x)
    u = datagen.uniform(n, d, seed=23)
    u[: n // 2] *= 1.0 / 1024             # half the rows 2^10 shorter: cancellation-heavy pairs
    yield "mixed-norms", np.ascontiguousarray(u)


@pytest.mark.parametrize("d", [16, 32, 64, 128, 512])
@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
def test_certificate_bound_on_product_kernel(pkg, d, fmt):
    n = 80_000 if d <= 128 else 40_000      # >= 1e7 pairs per (dpad, format) over the datasets
    K = d + 16
    gamma = 17 * ((K + 15) // 16) * 2.0 ** -23 * (1 + 1e-3)
    pairs, worst = 0, 0.0
    for name, X in _datasets(n, d):
        with pkg.Context(device=0, fmt=fmt) as ctx:
            w, a, b, kern = ctx.debug_mainpass(torch.from_numpy(X).cuda())
        A = a.double()
        B = b.double()
        exact = A @ B.t()                                   # [128, n]
        mag = A.abs() @ B.abs().t()
        err = (w.double() - exact).abs()
        slack = K * 2.0 ** -53 * mag                        # fp64 reference rounding
        ratio = ((err - slack).clamp_min(0) / (gamma * mag).clamp_min(1e-300)).max().item()
        worst = max(worst, ratio)
        pairs += w.numel()
        assert ratio <= 1.0, (name, fmt, d, ratio)
        # the kernel really is the production main pass
        assert kern == (4 if d >= 64 else 3)  # CTA pairs for dpad >= 64 (K-pipelined above 64)
    assert pairs >= 10_000_000
    print("dpad=%d %s: %d pairs, worst error / model = %.4f" % (K - 16, fmt, pairs, worst))
