// eg_epilogue_probe.cu -- the epilogue that SURVEY 8(a) steps 3-5's "E + G with 2 nnz MMAs"
// would need at BASELINE config 4, timed on its own.
//
// GEMM-A gives, per (prefix row r = (i < j < l) of C(128, 3), candidate b), T[r, b] =
// sum_{m > l} c(i, j, l, m) x_bm.  The fields of the three prefix positions and the energy then
// need, per element: the bits x_i, x_j, x_l of the candidate, the products of the other two,
// three scattered adds into the candidate's field vector (shared memory, [field][candidate],
// conflict-free) and the energy update.  This kernel does exactly that arithmetic over the
// element count of one cfg4 launch (341,376 rows x 262,144 candidates) with T read from a
// register-resident synthetic value, i.e. a lower bound on that epilogue (no TMEM loads, no
// MMA).  If it alone takes longer than the MMA time the 2 nnz formulation saves, the
// formulation cannot win.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/eg_probe tools/eg_epilogue_probe.cu && /tmp/eg_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int N = 128;
constexpr int kBM = 64;    // candidates per block (the [field][candidate] vector: 32 KB of shared memory)

__global__ void __launch_bounds__(kBM) probe(const uint32_t* __restrict__ xbits, long long B, float* __restrict__ out,
                                             int rows_per_block_pass) {
  __shared__ float g[N][kBM];   // [field position][candidate]: lanes of a warp hit consecutive banks
  const int b_local = threadIdx.x;
  for (int i = 0; i < N; ++i) g[i][b_local] = 0.0f;
  __syncthreads();
  float E = 0.0f;
  long long cb = blockIdx.x;
  const long long b = cb * kBM + b_local;
  uint32_t xw[4];
  for (int w = 0; w < 4; ++w) xw[w] = b < B ? xbits[b * 4 + w] : 0u;
  auto bit = [&](int v) -> float { return (float)((xw[v >> 5] >> (v & 31)) & 1u); };
  float T = 1.0f + 1e-7f * (float)b_local;   // stands in for the TMEM value of the element
  // the C(128, 3) prefix rows, in colex order (l outermost), rows_per_block_pass of them
  int done = 0;
  for (int l = 2; l < N && done < rows_per_block_pass; ++l) {
    const float xl = bit(l);
    float Fl = 0.0f;
    for (int j = 1; j < l && done < rows_per_block_pass; ++j) {
      const float xj = bit(j);
      for (int i = 0; i < j && done < rows_per_block_pass; ++i, ++done) {
        const float xi = bit(i);
        const float t = T;
        T = T * 0.999999f + 1e-9f;            // a fresh value per element (keeps the FMAs live)
        const float s = xi * xj * t;           // the prefix mask times T
        Fl += s;                                // field of position l (the row's fixed index)
        E += xl * s;                            // energy
        g[i][b_local] += xl * xj * t;           // field of position i
        g[j][b_local] += xl * xi * t;           // field of position j
      }
    }
    g[l][b_local] += Fl;
  }
  __syncthreads();
  float acc = E;
  for (int i = 0; i < N; ++i) acc += g[i][b_local];
  if (b < B) out[b] = acc;
}

int main() {
  const long long B = 262144;              // cfg4's batch
  const long long rows = 341376;           // C(128, 3) prefix rows
  const long long nblocks = B / kBM;
  uint32_t* x;
  float* out;
  cudaMalloc(&x, B * 4 * sizeof(uint32_t));
  cudaMalloc(&out, B * sizeof(float));
  cudaMemset(x, 0x5A, B * 4 * sizeof(uint32_t));
  // time a 1/16 slice of the rows per block and scale (the loop body is uniform per element)
  const int slice = (int)(rows / 16);
  probe<<<(unsigned)nblocks, kBM>>>(x, B, out, 1000);
  cudaDeviceSynchronize();
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  probe<<<(unsigned)nblocks, kBM>>>(x, B, out, slice);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double full = ms * (double)rows / slice;
  printf("epilogue probe: %.3f ms for %d of %lld rows x %lld candidates -> %.1f ms for a full cfg4 launch "
         "(%.3g elements); cudaError=%s\n",
         ms, slice, rows, B, full, (double)rows * B, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
