// mma_i8.cu — tcgen05.mma kind::i8 vs kind::f16 issue ceiling on this B200 (measurement tool only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2407_19987_b200/csrc mma_i8.cu -o mma_i8
#include <cstdio>
#include <cuda_runtime.h>

#include <cuda.h>
#include "ptx.cuh"

using namespace hobo;

__device__ __forceinline__ void mma_i8_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__host__ __device__ constexpr uint32_t idesc_i8_s32(int M, int N) {   // A u8, B s8, D s32
  return (2u << 4) | (0u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, bool TS, bool I8>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* cycles, int* out) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + 16384, bar = base + 16384 + 32768, tslot = bar + 8;
  uint8_t* g = smem_raw + (base - raw);
  // A: all ones (u8 1 / bf16 1.0); B: all s8 3 / bf16 3.0  ->  D = K * 3 per element
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) {
    uint32_t v;
    if (I8) v = i < 16384 / 4 ? 0x01010101u : 0x03030303u;
    else v = i < 16384 / 4 ? 0x3F803F80u : 0x40404040u;
    reinterpret_cast<uint32_t*>(g)[i] = v;
  }
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  fence_async_smem();
  if (threadIdx.x < 32) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(g + (tslot - base));
  if (TS) {
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) r[c] = I8 ? 0x01010101u : 0x3F803F80u;
    tmem_st32(tmem + ((uint32_t)((threadIdx.x >> 5) * 32) << 16) + 256, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = I8 ? idesc_i8_s32(128, N) : idesc_bf16_f32(128, N);
    const uint64_t ad = sw128_kmajor_desc(sA), bd = sw128_kmajor_desc(sB);
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (I8) {
          if (TS) mma_i8_ts(tmem, tmem + 256 + 8 * k, bd + 2 * k, idesc, (it | k) != 0);
          else mma_i8_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
        } else {
          if (TS) umma_bf16_ts(tmem, tmem + 256 + 8 * k, bd + 2 * k, idesc, (it | k) != 0);
          else umma_bf16_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
        }
      }
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)((threadIdx.x >> 5) * 32) << 16), r);
    tmem_ld_wait();
    if (blockIdx.x == 0 && threadIdx.x == 0) { out[0] = (int)r[0]; out[1] = (int)r[31]; }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N, bool TS, bool I8>
void run(const char* name, int iters) {
  auto k = mma_loop<N, TS, I8>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  unsigned long long* d;
  int* o;
  cudaMalloc(&d, 8);
  cudaMalloc(&o, 8);
  k<<<148, 128, 64 * 1024>>>(10, d, o);
  int ov[2];
  cudaMemcpy(ov, o, 8, cudaMemcpyDeviceToHost);
  const float expect_small = I8 ? 10 * 4 * 32 * 3 : 10 * 4 * 16 * 3;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 128, 64 * 1024>>>(iters, d, o);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double macs = 148.0 * iters * 4 * 128.0 * N * (I8 ? 32 : 16);
  const double v0 = I8 ? (double)ov[0] : (double)*reinterpret_cast<float*>(&ov[0]);
  printf("%-26s %7.1f T(FL)OP/s  %6.1f MAC/clk/SM  (%.3f ms) check %.0f (expect %.0f) err=%s\n", name,
         2 * macs / (ms * 1e-3) / 1e12, macs / 148.0 / (double)cyc, ms, v0, expect_small,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
  cudaFree(o);
}

int main() {
  const int it = 20000;
  run<256, false, false>("bf16 SS M128 N256", it);
  run<256, true, false>("bf16 TS M128 N256", it);
  run<256, false, true>("i8 SS M128 N256", it);
  run<256, true, true>("i8 TS M128 N256", it);
  run<128, false, true>("i8 SS M128 N128", it);
  run<128, true, true>("i8 TS M128 N128", it);
  run<64, true, true>("i8 TS M128 N64", it);
  return 0;
}
