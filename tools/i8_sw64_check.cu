// i8_sw64_check.cu — checks the int8 operand path of the contraction kernel in isolation:
// TMA 3-D load of an NT x 64-byte box with SWIZZLE_64B, A {0,1} bytes in TMEM (tcgen05.st),
// two tcgen05.mma kind::i8 (K = 32) per box, u8 or s8 B, s32 accumulate; compared with the CPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_2407_19987_b200/csrc i8_sw64_check.cu -o i8_sw64_check -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#include "ptx.cuh"

using namespace hobo;

__device__ __forceinline__ uint64_t sw64_desc(uint32_t a) {
  uint64_t d = 0;
  d |= (uint64_t)((a >> 4) & 0x3FFF);
  d |= (uint64_t)(512 >> 4) << 32;   // SBO: 8 rows x 64 B
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;            // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ void mma_i8_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc)
               : "memory");
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, int bsigned) {
  return (2u << 4) | (0u << 7) | ((uint32_t)bsigned << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

constexpr int NT = 128, NBOX = 3;
__global__ void __launch_bounds__(128, 1) k_check(const __grid_constant__ CUtensorMap tm, const uint8_t* A, int* out,
                                                  int bsigned) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t sB = base, bar = base + NBOX * NT * 64, bar2 = bar + 8, tslot = bar + 16;
  uint8_t* g = smem_raw + (base - raw);
  if (threadIdx.x == 0) { mbar_init(bar, 1); mbar_init(bar2, 1); fence_mbar_init(); }
  if (threadIdx.x < 32) tmem_alloc(tslot, 256);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(g + (tslot - base));
  const int w = threadIdx.x >> 5, row = threadIdx.x;
  // A row: NBOX K-blocks x 64 bytes -> NBOX x 16 columns at [128, ...)
  for (int kb = 0; kb < NBOX; ++kb) {
    uint32_t r[16];
    for (int c = 0; c < 16; ++c) {
      uint32_t v = 0;
      for (int b = 0; b < 4; ++b) v |= (uint32_t)A[(size_t)row * NBOX * 64 + kb * 64 + 4 * c + b] << (8 * b);
      r[c] = v;
    }
    tmem_st16(tmem + ((uint32_t)(w * 32) << 16) + 128 + 16 * kb, r);
  }
  tmem_st_wait();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(bar, NBOX * NT * 64);
    for (int kb = 0; kb < NBOX; ++kb) tma_load_3d(sB + kb * NT * 64, &tm, bar, 0, 0, kb);
    mbar_wait(bar, 0);
    tc_fence_after();
    for (int kb = 0; kb < NBOX; ++kb) {
      const uint64_t bd = sw64_desc(sB + kb * NT * 64);
      for (int k = 0; k < 2; ++k)
        mma_i8_ts(tmem, tmem + 128 + 16 * kb + 8 * k, bd + 2 * k, idesc_i8(128, NT, bsigned), (kb | k) != 0);
    }
    umma_commit(bar2);
    mbar_wait(bar2, 0);
  }
  __syncthreads();
  tc_fence_after();
  for (int c0 = 0; c0 < NT; c0 += 32) {
    uint32_t r[32];
    tmem_ld32(tmem + ((uint32_t)(w * 32) << 16) + c0, r);
    tmem_ld_wait();
    for (int c = 0; c < 32; ++c) out[row * NT + c0 + c] = (int)r[c];
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tmem, 256);
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  srand(7);
  std::vector<uint8_t> A(128 * NBOX * 64), Bm(NBOX * NT * 64);   // B tile-blocked [box][row][64]
  for (auto& v : A) v = rand() & 1;
  for (auto& v : Bm) v = rand() & 255;
  uint8_t *dA, *dB;
  int* dO;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, Bm.size());
  cudaMalloc(&dO, 128 * NT * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, Bm.data(), Bm.size(), cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[3] = {64, NT, NBOX};
  cuuint64_t str[2] = {64, 64 * NT};
  cuuint32_t box[3] = {64, NT, 1}, es[3] = {1, 1, 1};
  CUresult cr = ((EncFn)fp)(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, dB, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)cr);
  const size_t smem = NBOX * NT * 64 + 2048;
  cudaFuncSetAttribute(k_check, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int bs = 0; bs < 2; ++bs) {
    k_check<<<1, 128, smem>>>(tm, dA, dO, bs);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<int> O(128 * NT);
    cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
    long bad = 0;
    for (int r = 0; r < 128; ++r)
      for (int c = 0; c < NT; ++c) {
        long s = 0;
        for (int kb = 0; kb < NBOX; ++kb)
          for (int t = 0; t < 64; ++t) {
            const uint8_t bv = Bm[((size_t)kb * NT + c) * 64 + t];
            s += (long)A[(size_t)r * NBOX * 64 + kb * 64 + t] * (bs ? (long)(int8_t)bv : (long)bv);
          }
        if (s != O[r * NT + c]) { if (bad < 5) printf("  mismatch r%d c%d: %ld vs %d\n", r, c, s, O[r * NT + c]); ++bad; }
      }
    printf("B %s: %s, mismatches %ld of %d\n", bs ? "s8" : "u8", cudaGetErrorString(e), bad, 128 * NT);
  }
  return 0;
}
