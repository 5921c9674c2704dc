"""Empirical tcgen05 fp16/bf16 -> fp32 accumulation error on B200 (reading A9).

For A (M x K) and B (N x K) with 16-bit entries, compare the tensor-core product
C~ = A B^T (torch.matmul, fp32 accumulate; cuBLAS issues the same tcgen05 MMAs)
with the exact fp64 product, and report max |C~ - C| / (sum_k |A_ik B_jk| * 2^-24)
over all entries, i.e. the effective number of unit roundoffs of the sum.
"""
import sys
import torch

torch.backends.cuda.matmul.allow_fp16_reduced_precision_reduction = False
torch.backends.cuda.matmul.allow_bf16_reduced_precision_reduction = False
g = torch.Generator(device="cuda").manual_seed(0)
for dt in (torch.float16, torch.bfloat16):
    for K in (48, 80, 144, 272, 528, 1040):
        worst = 0.0
        for trial in range(6):
            M, N = 2048, 2048
            if trial % 3 == 0:      # gaussian
                A = torch.randn(M, K, generator=g, device="cuda")
                B = torch.randn(N, K, generator=g, device="cuda")
            elif trial % 3 == 1:    # mixture-like: shared large offset (cancellation)
                A = torch.randn(M, K, generator=g, device="cuda") + 30
                B = -(torch.randn(N, K, generator=g, device="cuda") + 30)
            else:                   # wide dynamic range
                A = torch.randn(M, K, generator=g, device="cuda") * torch.exp2(torch.randint(-8, 8, (M, K), generator=g, device="cuda").float())
                B = torch.randn(N, K, generator=g, device="cuda") * torch.exp2(torch.randint(-8, 8, (N, K), generator=g, device="cuda").float())
            A = A.to(dt); B = B.to(dt)
            C = torch.mm(A, B.t(), out_dtype=torch.float32)   # fp32 accumulate and output
            Ad, Bd = A.double(), B.double()
            Ce = Ad @ Bd.t()
            S = Ad.abs() @ Bd.abs().t()
            r = ((C.double() - Ce).abs() / (S * 2.0 ** -24)).max().item()
            worst = max(worst, r)
        print("%s K=%5d  max |err| / (sum|ab| 2^-24) = %8.3f   (A9 model m*4 = %d; K/16 = %d)"
              % (str(dt).split(".")[-1], K, worst, 2 * K * 4, K // 16))
        sys.stdout.flush()
