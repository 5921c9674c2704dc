// alu_bench.cu — microbenchmark: issue throughput of the filter's ALU instructions
// (FMNMX3 3-input min, FMNMX, FSETP, IMNMX) per SM sub-partition.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o alu_bench alu_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_alu(int iters, float seed, float* out, long long* cyc) {
  float a[8], b[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    a[i] = seed * (threadIdx.x + i);
    b[i] = seed * (threadIdx.x - i);
  }
  int cnt = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0) a[i] = fminf(fminf(a[i], b[i]), b[(i + 1) & 7]);  // FMNMX3
      if constexpr (OP == 1) a[i] = fminf(a[i], b[i]);                          // FMNMX
      if constexpr (OP == 2) cnt += a[i] < b[i];                                 // FSETP + add
      if constexpr (OP == 3) a[i] = __int_as_float(min(__float_as_int(a[i]), __float_as_int(b[i])));
      if constexpr (OP == 4) a[i] = a[i] * b[i] + b[(i + 1) & 7];               // FFMA
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) b[i] = b[i] + 1e-30f;  // keep b live (FADD, FMA pipe)
  }
  const long long t1 = clock64();
  float s = cnt;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int warps) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 20000;
  k_alu<OP><<<148, warps * 32>>>(iters, 1.0001f, out, cyc);
  cudaDeviceSynchronize();
  k_alu<OP><<<148, warps * 32>>>(iters, 1.0001f, out, cyc);
  cudaDeviceSynchronize();
  long long c;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  // per SMSP: warps/4 warps x iters x 8 ops (plus 8 FADDs per iteration on the FMA pipe)
  const double ops = (double)warps / 4 * iters * 8;
  printf("%-8s warps/SM=%2d  cycles per warp-instruction per SMSP = %.2f\n", name, warps, c / ops);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {4, 8, 16}) {
    run<0>("FMNMX3", w);
    run<1>("FMNMX", w);
    run<2>("FSETP", w);
    run<3>("IMNMX", w);
    run<4>("FFMA", w);
  }
  return 0;
}
