// tmem_bench.cu — microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bench tmem_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int NW, int X>
__global__ void __launch_bounds__(NW * 32, 1) k_ld(int iters, unsigned long long* cycles, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  float acc8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};  // independent sums: the
  // reduction must not be a dependent FADD chain (round 2's first numbers were)
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[32];
#pragma unroll
    for (int c = 0; c < X / 32; ++c) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
            "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
            "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
          : "r"(base + (uint32_t)(c * 32 + (it & 1) * 0)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int i = 0; i < 32; ++i) acc8[i & 7] += __uint_as_float(r[i]);
    }
  }
  unsigned long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += acc8[i];
  if ((threadIdx.x & 31) == 0) cycles[blockIdx.x * NW + warp] = t1 - t0;
  sink[blockIdx.x * NW * 32 + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

// same but loads without per-load wait (issue 4 then wait)
template <int NW>
__global__ void __launch_bounds__(NW * 32, 1) k_ld4(int iters, unsigned long long* cycles, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  float acc8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[4][16];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[c][0]), "=r"(r[c][1]), "=r"(r[c][2]), "=r"(r[c][3]), "=r"(r[c][4]), "=r"(r[c][5]),
            "=r"(r[c][6]), "=r"(r[c][7]), "=r"(r[c][8]), "=r"(r[c][9]), "=r"(r[c][10]),
            "=r"(r[c][11]), "=r"(r[c][12]), "=r"(r[c][13]), "=r"(r[c][14]), "=r"(r[c][15])
          : "r"(base + (uint32_t)(c * 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int i = 0; i < 16; ++i) acc8[i & 7] += __uint_as_float(r[c][i]);
  }
  unsigned long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) acc += acc8[i];
  if ((threadIdx.x & 31) == 0) cycles[blockIdx.x * NW + warp] = t1 - t0;
  sink[blockIdx.x * NW * 32 + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <class K>
void run(const char* name, K kern, int nw, int bytes_per_iter_per_warp, int iters) {
  unsigned long long* dc;
  float* ds;
  cudaMalloc(&dc, 148 * 16 * 8);
  cudaMalloc(&ds, 148 * 16 * 32 * 4);
  kern<<<148, nw * 32>>>(iters, dc, ds);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<148, nw * 32>>>(iters, dc, ds);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  unsigned long long h[16];
  cudaMemcpy(h, dc, nw * 8, cudaMemcpyDeviceToHost);
  double cyc = 0;
  for (int i = 0; i < nw; ++i) cyc = cyc > h[i] ? cyc : (double)h[i];
  const double bytes_sm = (double)bytes_per_iter_per_warp * nw * iters;
  printf("%-28s warps=%d  %s  cycles/iter/warp=%.1f  bytes/cycle/SM=%.1f  TB/s(chip)=%.2f\n", name, nw,
         cudaGetErrorString(e), cyc / iters, bytes_sm / cyc, bytes_sm * 148 / (ms * 1e-3) / 1e12);
  cudaFree(dc);
  cudaFree(ds);
}

int main() {
  const int it = 20000;
  run("ld x32 (+wait each)", k_ld<4, 32>, 4, 32 * 32 * 4, it);
  run("ld x32 (+wait each)", k_ld<8, 32>, 8, 32 * 32 * 4, it);
  run("ld 4x32 cols (+wait each)", k_ld<4, 128>, 4, 128 * 32 * 4, it);
  run("ld 4x32 cols (+wait each)", k_ld<8, 128>, 8, 128 * 32 * 4, it);
  run("ld 4 x16 then wait", k_ld4<4>, 4, 64 * 32 * 4, it);
  run("ld 4 x16 then wait", k_ld4<8>, 8, 64 * 32 * 4, it);
  run("ld 4 x16 then wait", k_ld4<16>, 16, 64 * 32 * 4, it);
  run("ld 4x32 cols (+wait each)", k_ld<16, 128>, 16, 128 * 32 * 4, it);
  return 0;
}
