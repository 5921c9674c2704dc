// mma_bench.cu — microbenchmark + layout check for the main-pass MMA shapes.
//
// (1) Layout check: D = A * B^T with A from shared memory (SS) vs A copied into
//     TMEM by tcgen05.cp 128x256b from the same swizzled shared tile (TS);
//     random fp16 A and B; prints the max |D_ss - D_ts|.
// (2) Throughput: back-to-back kind::f16 MMAs on one SM per CTA (148 CTAs),
//     M = 128, N = 256 / 160 / 128, K = 48 per "tile" (3 MMAs), SS or TS, with or
//     without a concurrent bulk-copy stream into shared memory (the B-tile traffic
//     of the real kernel).  Reports cycles per tile and per 256 columns.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2110_14007_b200/csrc -o build/mma_bench tools/mma_bench.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"

using namespace tod;

// A tile: 128 rows x 32 halves (SW64, one K region of 64 B per row) + a 16-wide
// extra block (SW32): K = 48 like dpad = 32.  B tile: N rows, same layout.
constexpr int KA = 32;
__host__ __device__ inline int sw_off(int row, int chunk16, int rb) {
  // 16-byte chunk index within the row XORed with (row % 8) bits (SW32: 2 chunks,
  // SW64: 4 chunks, SW128: 8 chunks per row); rows of 8-row atoms contiguous.
  const int nch = rb / 16;
  const int c = chunk16 ^ ((row % 8) / (8 / nch)) % nch;
  return row * rb + c * 16;
}

__device__ __forceinline__ void tc_mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_cp_128x256b(uint32_t taddr, uint64_t s_desc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(s_desc) : "memory");
}

// ---------------------------------------------------------------- layout check
__global__ void k_check(const uint8_t* gA, const uint8_t* gAx, const uint8_t* gB, const uint8_t* gBx,
                        float* out_ss, float* out_ts) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint8_t* sA = sm;                 // 128 x 64 B
  uint8_t* sAx = sm + 8192;         // 128 x 32 B
  uint8_t* sB = sm + 16384;         // 256 x 64 B
  uint8_t* sBx = sm + 32768;        // 256 x 32 B
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sA[i] = gA[i];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) sAx[i] = gAx[i];
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sB[i] = gB[i];
  for (int i = threadIdx.x; i < 8192; i += blockDim.x) sBx[i] = gBx[i];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  constexpr uint32_t IDESC = idesc_f16(128, 256, 0);
  uint32_t ph = 0;
  if (threadIdx.x == 0) {
    // SS into columns [0,256)
    for (int ks = 0; ks < 3; ++ks) {
      const uint64_t ad = ks < 2 ? smem_desc(smem_u32(sA) + ks * 32, 8 * 64, 4) : smem_desc(smem_u32(sAx), 8 * 32, 6);
      const uint64_t bd = ks < 2 ? smem_desc(smem_u32(sB) + ks * 32, 8 * 64, 4) : smem_desc(smem_u32(sBx), 8 * 32, 6);
      tc_mma_f16(tm, ad, bd, IDESC, ks > 0);
    }
    // A -> TMEM columns [256, 280) by tcgen05.cp (one 128x256b per K step = 8 columns)
    for (int ks = 0; ks < 3; ++ks) {
      const uint64_t ad = ks < 2 ? smem_desc(smem_u32(sA) + ks * 32, 8 * 64, 4) : smem_desc(smem_u32(sAx), 8 * 32, 6);
      tc_cp_128x256b(tm + 256 + ks * 8, ad);
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, ph);
  ph ^= 1;
  tc_fence_after();
  if (threadIdx.x == 0) {
    // TS: N = 128 (256 + 24 + 256 > 512 columns): columns [288, 416) from B rows 0..127
    constexpr uint32_t ID2 = idesc_f16(128, 128, 0);
    for (int ks = 0; ks < 3; ++ks) {
      const uint64_t bd = ks < 2 ? smem_desc(smem_u32(sB) + ks * 32, 8 * 64, 4) : smem_desc(smem_u32(sBx), 8 * 32, 6);
      tc_mma_ts(tm + 288, tm + 256 + ks * 8, bd, ID2, ks > 0);
    }
    tc_commit(&bar);
  }
  mbar_wait(&bar, ph);
  tc_fence_after();
  if (warp < 4) {
    float v[32];
    for (int c = 0; c < 256; c += 32) {
      tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + c, v);
      tmem_ld_wait();
      for (int e = 0; e < 32; ++e) out_ss[(warp * 32 + (threadIdx.x & 31)) * 256 + c + e] = v[e];
    }
    for (int c = 0; c < 128; c += 32) {
      tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + 288 + c, v);
      tmem_ld_wait();
      for (int e = 0; e < 32; ++e) out_ts[(warp * 32 + (threadIdx.x & 31)) * 128 + c + e] = v[e];
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

// ------------------------------------------------------------------ throughput
// TS: A resident in TMEM (copied once); SS: A read from shared memory per MMA.
// NB columns per accumulator, NACC accumulators in rotation.  COPY: warp 1 streams
// bulk copies of COPY_BYTES per tile into a scratch ring (throttled to the MMA).
template <bool TS, int NB, int NACC, int COPY>
__global__ void __launch_bounds__(64, 1) k_tp(int tiles, const uint8_t* gsrc, unsigned long long* cyc) {
  extern __shared__ uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (smem_u32(sm_raw) & 1023u)) & 1023u);
  uint8_t* sA = sm;
  uint8_t* sAx = sm + 8192;
  uint8_t* sB = sm + 16384;
  uint8_t* sBx = sm + 16384 + NB * 64;
  uint8_t* ring = sm + 65536;   // 3 x 32 KB scratch for the copy stream
  __shared__ uint64_t done[NACC], cfull[3], cempty[3];
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NACC; ++i) mbar_init(&done[i], 1);
    for (int i = 0; i < 3; ++i) {
      mbar_init(&cfull[i], 1);
      mbar_init(&cempty[i], 1);
    }
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = slot;
  constexpr uint32_t IDESC = idesc_f16(128, NB, 0);
  const uint32_t a_t = tm + NACC * NB;  // A columns in TMEM (24)
  unsigned long long t0 = clock64();
  if (warp == 0) {
    if (elect_one()) {
      if (TS) {
        for (int ks = 0; ks < 3; ++ks) {
          const uint64_t ad = ks < 2 ? smem_desc(smem_u32(sA) + ks * 32, 8 * 64, 4) : smem_desc(smem_u32(sAx), 8 * 32, 6);
          tc_cp_128x256b(a_t + ks * 8, ad);
        }
      }
      uint32_t ph[NACC] = {};
      for (int t = 0; t < tiles; ++t) {
        const int acc = t % NACC;
        if (t >= NACC) {  // the accumulator's previous tile must be complete (no reader here)
          mbar_wait(&done[acc], ph[acc]);
          ph[acc] ^= 1;
        }
        if (COPY && t >= 3) {  // consume one copied stage per tile
          const int s = t % 3;
          mbar_wait(&cfull[s], ((t / 3) - 1) & 1);
          mbar_arrive(&cempty[s]);
        }
        tc_fence_after();
        for (int ks = 0; ks < 3; ++ks) {
          const uint64_t bd = ks < 2 ? smem_desc(smem_u32(sB) + ks * 32, 8 * 64, 4) : smem_desc(smem_u32(sBx), 8 * 32, 6);
          if (TS) {
            tc_mma_ts(tm + acc * NB, a_t + ks * 8, bd, IDESC, ks > 0);
          } else {
            const uint64_t ad = ks < 2 ? smem_desc(smem_u32(sA) + ks * 32, 8 * 64, 4) : smem_desc(smem_u32(sAx), 8 * 32, 6);
            tc_mma_f16(tm + acc * NB, ad, bd, IDESC, ks > 0);
          }
        }
        tc_commit(&done[acc]);
      }
      for (int i = 0; i < NACC; ++i) {
        mbar_wait(&done[i], ph[i]);
      }
    }
    __syncwarp();
  } else if (COPY) {
    if (elect_one()) {
      for (int t = 0; t < tiles - 3; ++t) {
        const int s = t % 3;
        if (t >= 3) mbar_wait(&cempty[s], ((t / 3) - 1) & 1);
        mbar_arrive_expect_tx(&cfull[s], COPY);
        bulk_g2s(ring + s * 32768, gsrc + (size_t)(blockIdx.x * 7 + t) % 2048 * 32768, COPY, &cfull[s]);
      }
    }
    __syncwarp();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tm, 512);
}

template <bool TS, int NB, int NACC, int COPY>
void tp(const char* name, const uint8_t* gsrc, unsigned long long* dc) {
  auto k = k_tp<TS, NB, NACC, COPY>;
  const int smem = 65536 + 3 * 32768 + 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int tiles = 20000;
  k<<<148, 64, smem>>>(200, gsrc, dc);
  cudaDeviceSynchronize();
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<<<148, 64, smem>>>(tiles, gsrc, dc);
  cudaEventRecord(b);
  cudaError_t e = cudaDeviceSynchronize();
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  std::vector<unsigned long long> h(148);
  cudaMemcpy(h.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (auto x : h) mx = mx > x ? mx : (double)x;
  const double flops = 2.0 * 128 * NB * 48 * tiles * 148;
  printf("%-34s %s cycles/tile %.1f  per 256 cols %.1f  TFLOP/s(K=48) %.0f  ms %.3f\n", name,
         cudaGetErrorString(e), mx / tiles, mx / tiles * 256.0 / NB, flops / (ms * 1e-3) / 1e12, ms);
}

static uint16_t h16(float f) {
  __half h = __float2half_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}

int main() {
  // ---- layout check
  srand(1);
  std::vector<float> A(128 * 48), B(256 * 48);
  for (auto& x : A) x = (float)((rand() % 17) - 8) / 8.f;
  for (auto& x : B) x = (float)((rand() % 17) - 8) / 8.f;
  auto pack = [&](const std::vector<float>& M, int rows, std::vector<uint8_t>& main, std::vector<uint8_t>& ex) {
    main.assign(rows * 64, 0);
    ex.assign(rows * 32, 0);
    for (int r = 0; r < rows; ++r)
      for (int k = 0; k < 48; ++k) {
        const uint16_t v = h16(M[r * 48 + k]);
        uint8_t* dst;
        if (k < 32) dst = &main[sw_off(r, k / 8, 64) + (k % 8) * 2];
        else dst = &ex[sw_off(r, (k - 32) / 8, 32) + ((k - 32) % 8) * 2];
        dst[0] = v & 0xFF;
        dst[1] = v >> 8;
      }
  };
  std::vector<uint8_t> am, ax, bm, bx;
  pack(A, 128, am, ax);
  pack(B, 256, bm, bx);
  uint8_t *dA, *dAx, *dB, *dBx;
  float *dss, *dts;
  cudaMalloc(&dA, am.size()); cudaMalloc(&dAx, ax.size()); cudaMalloc(&dB, bm.size()); cudaMalloc(&dBx, bx.size());
  cudaMalloc(&dss, 128 * 256 * 4); cudaMalloc(&dts, 128 * 128 * 4);
  cudaMemcpy(dA, am.data(), am.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dAx, ax.data(), ax.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, bm.data(), bm.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dBx, bx.data(), bx.size(), cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, 49 * 1024);
  k_check<<<1, 128, 49 * 1024>>>(dA, dAx, dB, dBx, dss, dts);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> ss(128 * 256), ts(128 * 128);
  cudaMemcpy(ss.data(), dss, ss.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(ts.data(), dts, ts.size() * 4, cudaMemcpyDeviceToHost);
  double e_ss = 0, e_ts = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 256; ++j) {
      double ref = 0;
      for (int k = 0; k < 48; ++k) ref += (double)A[i * 48 + k] * B[j * 48 + k];
      e_ss = fmax(e_ss, fabs(ref - ss[i * 256 + j]));
      if (j < 128) e_ts = fmax(e_ts, fabs(ref - ts[i * 128 + j]));
    }
  printf("layout check: %s  max|SS - exact| %.3g  max|TS(cp) - exact| %.3g\n", cudaGetErrorString(e), e_ss, e_ts);

  // ---- throughput
  uint8_t* gsrc;
  cudaMalloc(&gsrc, (size_t)2048 * 32768);
  unsigned long long* dc;
  cudaMalloc(&dc, 148 * 8);
  tp<false, 256, 2, 0>("SS N=256 x2", gsrc, dc);
  tp<false, 256, 2, 24576>("SS N=256 x2 + 24KB copy", gsrc, dc);
  tp<false, 160, 3, 0>("SS N=160 x3", gsrc, dc);
  tp<false, 128, 3, 0>("SS N=128 x3", gsrc, dc);
  tp<false, 128, 3, 12288>("SS N=128 x3 + 12KB copy", gsrc, dc);
  tp<true, 240, 2, 0>("TS N=240 x2", gsrc, dc);
  tp<true, 240, 2, 23040>("TS N=240 x2 + 22.5KB copy", gsrc, dc);
  tp<true, 160, 3, 0>("TS N=160 x3", gsrc, dc);
  tp<true, 160, 3, 15360>("TS N=160 x3 + 15KB copy", gsrc, dc);
  tp<true, 128, 3, 0>("TS N=128 x3", gsrc, dc);
  tp<true, 128, 3, 12288>("TS N=128 x3 + 12KB copy", gsrc, dc);
  return 0;
}
