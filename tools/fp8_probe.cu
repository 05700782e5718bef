// fp8_probe.cu — does tcgen05.mma kind::f8f6f4 (e4m3 x e4m3, fp32 accumulate, A from TMEM)
// sum exactly, and how fast is it against kind::f16 on this B200?  (A measurement tool, not
// part of the product.)
//
// Exactness: one CTA, D[128 x 256] = A[128 x 128 bytes] * W[256 x 128 bytes]^T as 4 MMAs of
// K = 32, repeated `reps` times into the same accumulator, against the exact sum in double.
// Modes (A bytes / W codes): 0 {0, 1.0} x random finite e4m3; 1 {0, 2^-9 (0x01, subnormal)} x
// random; 2 {0, 1.0} x {+-448, +-2^-9} (the widest dynamic range); 3 {0, 2^-9} x powers of two.
// Throughput: one CTA per SM issuing back-to-back MMAs (M = 128, N = 256) of each kind.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Ipaper_2407_19987_b200/csrc \
//        tools/fp8_probe.cu -o /tmp/fp8_probe -lcuda && /tmp/fp8_probe
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace hobo;

// W[n][k] (256 x 128 bytes) -> SW128 K-major: atom of 8 rows x 128 B, 16-byte chunk c of row r
// at chunk c ^ (r & 7)
__global__ void __launch_bounds__(128, 1) exact_kernel(const uint8_t* __restrict__ A, const uint8_t* __restrict__ Wt,
                                                       int reps, float* __restrict__ D) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* g = smem_raw + (base - raw);
  const uint32_t sB = base, bar = base + 32768, tslot = bar + 8;
  for (int i = threadIdx.x; i < 256 * 128; i += 128) {
    const int n = i / 128, k = i % 128;
    g[(n / 8) * 1024 + (n % 8) * 128 + ((((k / 16) ^ (n % 8))) * 16) + (k % 16)] = Wt[i];
  }
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  fence_async_smem();
  if (threadIdx.x < 32) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(g + (tslot - base));
  const int w = threadIdx.x >> 5;
  {  // row m = threadIdx.x: 128 A bytes -> 32 columns at [256, 288)
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) r[c] = reinterpret_cast<const uint32_t*>(A + threadIdx.x * 128)[c];
    tmem_st32(tmem + ((uint32_t)(w * 32) << 16) + 256, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_e4m3_f32(128, 256);
    const uint64_t bd = sw128_kmajor_desc(sB);
    for (int it = 0; it < reps; ++it)
      for (int k = 0; k < 4; ++k) umma_f8_ts(tmem, tmem + 256 + 8 * k, bd + 2 * k, idesc, (it | k) != 0);
    umma_commit(bar);
    mbar_wait(bar, 0);
  }
  __syncthreads();
  tc_fence_after();
  for (int c0 = 0; c0 < 256; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(w * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int c = 0; c < 32; ++c) D[threadIdx.x * 256 + c0 + c] = __uint_as_float(r[c]);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int KIND>   // 0 f16 (bf16), 1 f8f6f4, 2 i8; 3/4: f8f6f4 with 1/2 commits per 4 MMAs (the
                      // e4m3 kernel's per-stage EMPTY + EMPTYA); 5: bf16 with 1 commit per 8 MMAs
__global__ void __launch_bounds__(128, 1) rate_kernel(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* g = smem_raw + (base - raw);
  const uint32_t sB = base, bar = base + 32768, tslot = bar + 8, bar2 = bar + 16, bar3 = bar + 24;
  for (int i = threadIdx.x; i < 32768 / 4; i += 128) reinterpret_cast<uint32_t*>(g)[i] = 0x38383838u & (i * 2654435761u);
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar2, 1); mbar_init(bar3, 1); fence_mbar_init(); }
  fence_async_smem();
  if (threadIdx.x < 32) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(g + (tslot - base));
  if (threadIdx.x == 0) {
    const uint64_t bd = sw128_kmajor_desc(sB);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (KIND == 0 || KIND == 5) umma_bf16_ts(tmem, tmem + 256 + 8 * k, bd + 2 * k, idesc_bf16_f32(128, 256), (it | k) != 0);
        else if (KIND == 2) umma_i8_ts(tmem, tmem + 256 + 8 * k, bd + 2 * k, idesc_i8_s32(128, 256, 1), (it | k) != 0);
        else umma_f8_ts(tmem, tmem + 256 + 8 * k, bd + 2 * k, idesc_e4m3_f32(128, 256), (it | k) != 0);
      }
      if (KIND == 3 || KIND == 4) umma_commit(bar2);
      if (KIND == 4) umma_commit(bar3);
      if (KIND == 5 && (it & 1)) umma_commit(bar2);
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    cycles[blockIdx.x] = clock64() - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

static double e4m3(uint8_t c) {
  const int s = c >> 7, e = (c >> 3) & 15, m = c & 7;
  const double v = e ? std::ldexp(1.0 + m / 8.0, e - 7) : std::ldexp(m / 8.0, -6);
  return s ? -v : v;
}

int main() {
  std::vector<uint8_t> A(128 * 128), Wt(256 * 128);
  uint8_t *dA, *dW;
  float* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dW, Wt.size());
  cudaMalloc(&dD, 128 * 256 * 4);
  const size_t smem = 32768 + 2048 + 1024;
  cudaFuncSetAttribute(exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  std::vector<float> D(128 * 256);
  srand(7);
  for (int mode = 0; mode < 4; ++mode)
    for (int reps : {1, 16}) {
      const uint8_t aone = (mode == 1 || mode == 3) ? 0x01 : 0x38;
      for (auto& a : A) a = (rand() & 1) ? aone : 0;
      for (auto& w : Wt) {
        uint8_t c;
        if (mode == 2) c = (rand() & 1) ? 0x7E : 0x01;              // 448 or 2^-9
        else if (mode == 3) c = (uint8_t)(((1 + rand() % 14) << 3));  // 2^(e-7), e = 1..14
        else do { c = (uint8_t)(rand() & 0x7F); } while (c == 0x7F);
        w = c | ((rand() & 1) ? 0x80 : 0);
      }
      cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
      cudaMemcpy(dW, Wt.data(), Wt.size(), cudaMemcpyHostToDevice);
      exact_kernel<<<1, 128, smem>>>(dA, dW, reps, dD);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      double maxrel = 0, maxabs = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 256; ++n) {
          double s = 0;
          for (int k = 0; k < 128; ++k) s += e4m3(A[m * 128 + k]) * e4m3(Wt[n * 128 + k]);
          s *= reps;
          const double f = (double)(float)s;   // the exactly-rounded fp32 of the exact sum
          if ((double)D[m * 256 + n] != f) {
            ++bad;
            maxabs = std::fmax(maxabs, std::fabs(D[m * 256 + n] - s));
            maxrel = std::fmax(maxrel, std::fabs(D[m * 256 + n] - s) / std::fmax(std::fabs(s), 1e-30));
          }
        }
      printf("exact mode %d reps %2d: %s, %d of 32768 differ from fp32(exact) (max abs %.3g, max rel %.3g)\n", mode, reps,
             cudaGetErrorString(e), bad, maxabs, maxrel);
    }
  unsigned long long* dc;
  cudaMalloc(&dc, 148 * 8);
  std::vector<unsigned long long> cyc(148);
  const int iters = 4096;
  auto rate = [&](auto kern, const char* name, double macs_per_mma) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<148, 128, smem>>>(iters, dc);
    cudaDeviceSynchronize();
    kern<<<148, 128, smem>>>(iters, dc);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(cyc.data(), dc, 148 * 8, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (auto c : cyc) mx = std::fmax(mx, (double)c);
    printf("%-8s %s: %.1f cycles per MMA, %.0f MAC/clk/SM\n", name, cudaGetErrorString(e), mx / (4.0 * iters),
           macs_per_mma * 4.0 * iters / mx);
  };
  rate(rate_kernel<0>, "bf16", 128.0 * 256 * 16);
  rate(rate_kernel<1>, "e4m3", 128.0 * 256 * 32);
  rate(rate_kernel<2>, "i8", 128.0 * 256 * 32);
  rate(rate_kernel<3>, "e4m3+1c", 128.0 * 256 * 32);
  rate(rate_kernel<4>, "e4m3+2c", 128.0 * 256 * 32);
  rate(rate_kernel<5>, "bf16+c/8", 128.0 * 256 * 16);
  return 0;
}
