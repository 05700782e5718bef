// mma_ceiling.cu — measures the issue-bound ceiling of tcgen05.mma kind::f16 on this B200
// for the shapes the contraction kernel uses (not part of the product; a measurement tool).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2407_19987_b200/csrc mma_ceiling.cu -o mma_ceiling
#include <cstdio>
#include <cuda_runtime.h>

#include <cuda.h>
#include "ptx.cuh"

using namespace hobo;

template <int N, bool TS, int COMMIT_EVERY, bool RND = false>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sA = base, sB = base + 16384, bar = base + 16384 + 32768, tslot = bar + 8;
  uint8_t* g = smem_raw + (base - raw);
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x) {
    uint32_t v = 0;
    if (RND) {  // random bf16 pairs with exponent in [-8, 7] and random sign / mantissa
      uint32_t hsh = (uint32_t)(i * 2654435761u) ^ (blockIdx.x * 97u);
      hsh ^= hsh >> 13; hsh *= 0x5bd1e995u; hsh ^= hsh >> 15;
      const uint32_t lo = (hsh & 0x807Fu) | ((119u + ((hsh >> 7) & 15u)) << 7);
      const uint32_t hi = ((hsh >> 16) & 0x807Fu) | ((119u + ((hsh >> 23) & 15u)) << 7);
      v = lo | (hi << 16);
      if (i < 16384 / 4) v &= 0x3F803F80u;   // A operand: {0, 1.0} like the Khatri-Rao operand
    }
    reinterpret_cast<uint32_t*>(g)[i] = v;
  }
  if (threadIdx.x == 0) { mbar_init(bar, 1); fence_mbar_init(); }
  fence_async_smem();
  if (threadIdx.x < 32) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(g + (tslot - base));
  if (RND && TS) {  // random {0,1} A rows in TMEM columns [256, 288)
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) r[c] = reinterpret_cast<uint32_t*>(g)[(threadIdx.x * 32 + c) % 4096];
    tmem_st32(tmem + ((uint32_t)((threadIdx.x >> 5) * 32) << 16) + 256, r);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
    const uint64_t ad = sw128_kmajor_desc(sA), bd = sw128_kmajor_desc(sB);
    const long long t0 = clock64();
    uint32_t ph = 0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (TS) umma_bf16_ts(tmem, tmem + 256 + 8 * k, bd + 2 * k, idesc, (it | k) != 0);
        else umma_bf16_ss(tmem, ad + 2 * k, bd + 2 * k, idesc, (it | k) != 0);
      }
      if (COMMIT_EVERY && (it % COMMIT_EVERY) == COMMIT_EVERY - 1) {
        umma_commit(bar);
        mbar_wait(bar, ph);
        ph ^= 1;
      }
    }
    umma_commit(bar);
    mbar_wait(bar, ph);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N, bool TS, int CE, bool RND = false>
void run(const char* name, int iters) {
  auto k = mma_loop<N, TS, CE, RND>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  k<<<148, 128, 64 * 1024>>>(10, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<148, 128, 64 * 1024>>>(iters, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc;
  cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double macs = 148.0 * iters * 4 * 128.0 * N * 16;
  printf("%-34s %7.1f TFLOP/s  %6.1f MAC/clk/SM  (%.3f ms, err=%s)\n", name, 2 * macs / (ms * 1e-3) / 1e12,
         macs / 148.0 / (double)cyc, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}


// TMA-fed B ring (NB stages of N x 64 bf16), A fixed in TMEM: the real kernel minus the A generator
template <int N, int NB, int STW>
__global__ void __launch_bounds__(384, 1) mma_tma(const __grid_constant__ CUtensorMap tmap, int iters, int rows_total,
                                                  unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  constexpr uint32_t BST = N * 128;
  const uint32_t sB = base, bar = base + NB * BST, tslot = bar + 16 * NB;
  uint8_t* g = smem_raw + (base - raw);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NB; ++s) { mbar_init(bar + 8 * s, 1); mbar_init(bar + 8 * (NB + s), 1); }
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(tslot, 512);
  if (threadIdx.x == 0) *reinterpret_cast<volatile uint32_t*>(g + (tslot - base) + 4) = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(g + (tslot - base));
  const int warp = threadIdx.x >> 5;
  if (warp == 0 && threadIdx.x == 0) {
    int sb = 0; uint32_t ph = 0;
    const int row0 = (blockIdx.x % (rows_total / N)) * N;
    for (int it = 0; it < iters; ++it) {
      mbar_wait(bar + 8 * (NB + sb), ph ^ 1u);
      mbar_arrive_expect_tx(bar + 8 * sb, BST);
      tma_load_2d(sB + sb * BST, &tmap, bar + 8 * sb, (it % 2048) * 64, row0);
      if (++sb == NB) { sb = 0; ph ^= 1u; }
    }
  } else if (warp == 1 && threadIdx.x == 32) {
    constexpr uint32_t idesc = idesc_bf16_f32(128, N);
    int sb = 0; uint32_t ph = 0;
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      mbar_wait(bar + 8 * sb, ph);
      tc_fence_after();
      const uint64_t bd = sw128_kmajor_desc(sB + sb * BST);
#pragma unroll
      for (int k = 0; k < 4; ++k) umma_bf16_ts(tmem, tmem + 256 + 8 * k, bd + 2 * k, idesc, (it | k) != 0);
      umma_commit(bar + 8 * (NB + sb));
      if (++sb == NB) { sb = 0; ph ^= 1u; }
    }
    // drain: wait for the last commit
    const int last = (iters - 1) % NB;
    const uint32_t lph = ((iters - 1) / NB) & 1;
    mbar_wait(bar + 8 * (NB + last), lph);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
    *reinterpret_cast<volatile uint32_t*>(g + (tslot - base) + 4) = 1;   // stop flag
  } else if (warp >= 4 && warp < 4 + STW) {
    // TMEM store traffic like the A generator: 32 columns per K-block per warp, into [256, 512)
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = 0;
    const uint32_t lb = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    volatile uint32_t* stop = reinterpret_cast<volatile uint32_t*>(g + (tslot - base) + 4);
    int k = 0;
    while (!*stop) {
      tmem_st32(lb + 256 + 32 * (k & 7), r);
      tmem_st_wait();
      ++k;
      for (int d = 0; d < 8; ++d) __nanosleep(100);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int N, int NB, int STW = 0>
void run_tma(const char* name, int iters, int rows_total, int ctas) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  const long long cols = 2048 * 64;
  void* buf;
  cudaMalloc(&buf, (size_t)rows_total * cols * 2);
  cudaMemset(buf, 0, (size_t)rows_total * cols * 2);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows_total};
  cuuint64_t str[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)N};
  cuuint32_t es[2] = {1, 1};
  ((EncFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  auto k = mma_tma<N, NB, STW>;
  const int smem = NB * N * 128 + 4096;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  k<<<ctas, 384, smem>>>(m, 100, rows_total, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<ctas, 384, smem>>>(m, iters, rows_total, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double macs = (double)ctas * iters * 4 * 128.0 * N * 16;
  const double bytes = (double)ctas * iters * N * 128;
  printf("%-44s %7.1f TFLOP/s  %6.1f MAC/clk/SM  L2->smem %6.1f TB/s (%.3f ms, %s)\n", name, 2 * macs / (ms * 1e-3) / 1e12,
         macs / ctas / (double)cyc, bytes / (ms * 1e-3) / 1e12, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d); cudaFree(buf);
}

// the real kernel's synchronisation skeleton: TMA B ring + TMEM A ring handed over by 8
// "generator" warps (2 teams x 4 lane quarters) that compute nothing
__global__ void fill_random(uint32_t* p, size_t n, uint32_t salt) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ salt;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    const uint32_t lo = (h & 0x807Fu) | ((119u + ((h >> 7) & 15u)) << 7);
    const uint32_t hi = ((h >> 16) & 0x807Fu) | ((119u + ((h >> 23) & 15u)) << 7);
    p[i] = lo | (hi << 16);
  }
}

template <int NB, int NA, bool GEN, bool COMMIT_A, bool GEN_ST, bool RNDA = false>
__global__ void __launch_bounds__(320, 1) mma_pipe(const __grid_constant__ CUtensorMap tmap, int iters, int rows_total,
                                                   unsigned long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  constexpr uint32_t BST = 256 * 128;
  const uint32_t sB = base, bar = base + NB * BST, tslot = bar + 8 * (2 * NB + 2 * NA) + 8;
#define FB(s) (bar + 8u * (s))
#define EB(s) (bar + 8u * (NB + (s)))
#define FA(s) (bar + 8u * (2 * NB + (s)))
#define EA(s) (bar + 8u * (2 * NB + NA + (s)))
  uint8_t* g = smem_raw + (base - raw);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NB; ++s) { mbar_init(FB(s), 1); mbar_init(EB(s), 1); }
    for (int s = 0; s < NA; ++s) { mbar_init(FA(s), 4); mbar_init(EA(s), 1); }
    fence_mbar_init();
  }
  if (threadIdx.x < 32) tmem_alloc(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(g + (tslot - base));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      int sb = 0; uint32_t ph = 0;
      const int row0 = (blockIdx.x % (rows_total / 256)) * 256;
      for (int it = 0; it < iters; ++it) {
        mbar_wait(EB(sb), ph ^ 1u);
        mbar_arrive_expect_tx(FB(sb), BST);
        tma_load_2d(sB + sb * BST, &tmap, FB(sb), (it % 2048) * 64, row0);
        if (++sb == NB) { sb = 0; ph ^= 1u; }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, 256);
      int sb = 0, sa = 0; uint32_t ph = 0, pha = 0;
      const long long t0 = clock64();
      for (int it = 0; it < iters; ++it) {
        if (GEN) { mbar_wait(FA(sa), pha); tc_fence_after(); }
        mbar_wait(FB(sb), ph);
        tc_fence_after();
        const uint64_t bd = sw128_kmajor_desc(sB + sb * BST);
        const uint32_t at = tmem + 256 + 32 * sa;
#pragma unroll
        for (int k = 0; k < 4; ++k) umma_bf16_ts(tmem, at + 8 * k, bd + 2 * k, idesc, (it | k) != 0);
        umma_commit(EB(sb));
        if (++sb == NB) { sb = 0; ph ^= 1u; }
        if (GEN || COMMIT_A) umma_commit(EA(sa));
        if (++sa == NA) { sa = 0; pha ^= 1u; }
      }
      const int last = (iters - 1) % NB;
      mbar_wait(EB(last), ((iters - 1) / NB) & 1);
      const long long t1 = clock64();
      if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
    }
  } else if (GEN) {
    const int h = (warp - 2) >> 2, q = warp & 3;
    uint32_t r[32];
    for (int c = 0; c < 32; ++c) r[c] = 0;
    uint32_t st = (uint32_t)(threadIdx.x * 7919 + blockIdx.x);
    for (int pos = h; pos < iters; pos += 2) {
      const int sa = pos % NA;
      mbar_wait(EA(sa), (uint32_t)(((pos / NA) & 1) ^ 1));
      tc_fence_after();
      if (RNDA) {
#pragma unroll
        for (int c = 0; c < 32; ++c) { st = st * 1664525u + 1013904223u; r[c] = (st & 0x80008000u) ? (st & 0x3F803F80u) : 0u; }
      }
      if (GEN_ST) tmem_st32(tmem + ((uint32_t)(q * 32) << 16) + 256 + 32 * sa, r);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(FA(sa));
    }
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
#undef FB
#undef EB
#undef FA
#undef EA
}

template <int NB, int NA, bool GEN, bool CA, bool GST, bool RND = false>
void run_pipe(const char* name, int iters, int ctas = 148) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  const int rows_total = 512;
  const long long cols = 2048 * 64;
  void* buf;
  cudaMalloc(&buf, (size_t)rows_total * cols * 2);
  cudaMemset(buf, 0, (size_t)rows_total * cols * 2);
  if (RND) fill_random<<<1024, 256>>>((uint32_t*)buf, (size_t)rows_total * cols / 2, 12345u);
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows_total};
  cuuint64_t str[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, 256};
  cuuint32_t es[2] = {1, 1};
  ((EncFn)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  auto k = mma_pipe<NB, NA, GEN, CA, GST, RND>;
  const int smem = NB * 256 * 128 + 4096;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long* d;
  cudaMalloc(&d, 8);
  k<<<ctas, 320, smem>>>(m, 100, rows_total, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<<<ctas, 320, smem>>>(m, iters, rows_total, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc; cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
  const double macs = (double)ctas * iters * 4 * 128.0 * 256 * 16;
  printf("%-44s %7.1f TFLOP/s  %6.1f cyc/kblock (%.3f ms, %s)\n", name, 2 * macs / (ms * 1e-3) / 1e12,
         (double)cyc / iters, ms, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d); cudaFree(buf);
}

int main(int argc, char** argv) {
  const int it = 20000;
  if (argc > 1 && argv[1][0] == 'n') {   // the N sweep only (bf16, A in TMEM, no waits)
    run<256, true, 0>("TS M128 N256 no-wait", it);
    run<128, true, 0>("TS M128 N128 no-wait", it);
    run<64, true, 0>("TS M128 N64 no-wait", it);
    run<64, false, 0>("SS M128 N64 no-wait", it);
    return 0;
  }
  run<256, false, 0>("SS M128 N256 no-wait", it);
  run<256, true, 0>("TS M128 N256 no-wait", it);
  run<128, false, 0>("SS M128 N128 no-wait", it);
  run<128, true, 0>("TS M128 N128 no-wait", it);
  run<256, false, 0, true>("SS M128 N256 RANDOM data", it);
  run<256, true, 0, true>("TS M128 N256 RANDOM data", it);
  run<256, true, 1>("TS M128 N256 commit+wait/kblock", it);
  run<256, true, 8>("TS M128 N256 commit+wait/8 kblocks", it);
  run_pipe<6, 8, false, false, false>("pipe: TMA only", it);
  run_pipe<6, 8, false, false, false>("pipe: TMA only, 1024 CTAs x 2052", 2052, 1024);
  run_pipe<6, 8, true, true, true>("pipe: full handoff, 1024 CTAs x 2052", 2052, 1024);
  run_pipe<6, 8, false, true, false>("pipe: TMA + 2nd commit/kblock", it);
  run_pipe<6, 8, true, true, false>("pipe: TMA + A ring handoff (no st)", it);
  run_pipe<6, 8, true, true, true>("pipe: TMA + A ring handoff + tcgen05.st", it);
  run_pipe<6, 8, true, true, true, true>("pipe: + RANDOM B stream and random 0/1 A", it);
  run_pipe<6, 8, false, false, false, true>("pipe: TMA only, RANDOM B stream", it);
  run_tma<256, 6>("TMA-fed B NB=6, all CTAs same 256 rows", it, 256, 148);
  run_tma<256, 6, 4>("  + 4 warps tcgen05.st (light)", it, 512, 148);
  run_tma<256, 6, 8>("  + 8 warps tcgen05.st (light)", it, 512, 148);
  run_tma<256, 6>("TMA-fed B NB=6, 2 column tiles (512 rows)", it, 512, 148);
  run_tma<256, 6>("TMA-fed B NB=6, 148 distinct tiles (37888 rows)", 4000, 256 * 148, 148);
  run_tma<256, 4>("TMA-fed B NB=4, 2 column tiles", it, 512, 148);
  return 0;
}
