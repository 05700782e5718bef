// hobo_api.cu — the C ABI of include/hobo.h: device layouts, launches, search loop.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/hobo.h"
#include "host_compile.h"
#include "tt.h"
#include "kernels.cuh"
#include "sa_kernel.cuh"
#include "persist.cuh"

using namespace hobo;

namespace {

thread_local std::string g_err;

hobo_status fail(hobo_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

// ---- multi-GPU: one NCCL communicator per process, resolved with dlopen so
// the library uses the NCCL already loaded in the process (torch's) or the system one ----
struct Dist {
  void* lib = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*destroy)(ncclComm_t) = nullptr;
  const char* (*err)(ncclResult_t) = nullptr;
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = -1;
};
Dist g_dist;

hobo_status nccl_load(std::string& msg) {
  if (g_dist.lib) return HOBO_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) { msg = std::string("libnccl.so.2 not loadable: ") + dlerror(); return HOBO_ENCCL; }
  g_dist.get_unique_id = (decltype(g_dist.get_unique_id))dlsym(h, "ncclGetUniqueId");
  g_dist.init_rank = (decltype(g_dist.init_rank))dlsym(h, "ncclCommInitRank");
  g_dist.all_reduce = (decltype(g_dist.all_reduce))dlsym(h, "ncclAllReduce");
  g_dist.broadcast = (decltype(g_dist.broadcast))dlsym(h, "ncclBroadcast");
  g_dist.destroy = (decltype(g_dist.destroy))dlsym(h, "ncclCommDestroy");
  g_dist.err = (decltype(g_dist.err))dlsym(h, "ncclGetErrorString");
  if (!g_dist.get_unique_id || !g_dist.init_rank || !g_dist.all_reduce || !g_dist.broadcast || !g_dist.destroy ||
      !g_dist.err) {
    msg = "libnccl.so.2 lacks a required symbol";
    return HOBO_ENCCL;
  }
  g_dist.lib = h;
  return HOBO_OK;
}

bool dist_active() { return g_dist.comm != nullptr; }   // world 1 runs the same path (identity collectives)

struct DevLayout {
  bool built = false;
  int NT = 256, n_ct = 0, Npad = 0;
  __nv_bfloat16* W = nullptr;          // bf16 limb planes, or (i8 > 0) int8 digit planes
  int i8 = 0;                          // int8 digit planes: their count; 0 = bf16 limbs
  double qscale = 1.0;                 // int8: cell = qscale * (digit integer)
  bool f8 = false;                     // the i8 1-byte planes hold e4m3 limbs (kind::f8f6f4)
  float fscale = 1.0f;                 // e4m3: F = fscale * accumulator (2^(s + 9))
  double f8_density = 0.0;             // e4m3: mean limb boxes per stage (MMA work vs one plane)
  uint32_t* d_nltab = nullptr;         // e4m3: [n_ct][nl_words] limb counts per K-block pair, 2 bits
  int nl_words = 0;
  int2* d_sched = nullptr;
  std::vector<int32_t> sched;
  alignas(64) CUtensorMap tmap;
  alignas(64) CUtensorMap tmap_half;   // CTA pairs: NT/2-row boxes (each CTA loads its half)
  double lcm = 1.0;
  double wdeg[8] = {1, 1, 1, 1, 1, 1, 1, 1};
  double wp = 1.0;
};

}  // namespace

struct hobo_tensor {
  HostTensor host;
  KLayout kl;
  int device = -1;         // bound on first device use (the then-current CUDA device)
  bool dev_init = false;
  bool poisoned = false;
  uint4* d_runs = nullptr;
  uint4* d_kdesc = nullptr;
  uint32_t* d_runoff = nullptr;
  uint4* d_srec = nullptr;  // int8 path: per K-block pair, a header + all its generator runs
  int srec_u4 = 0;          // uint4s per record (1 + the most runs of any pair)
  float* d_p1 = nullptr;   // padded to 256-multiples
  int W = 0;               // 32-bit words per candidate bit row
  DevLayout lay[6];        // 0 = energy (strict), 1 = field (open index), 2 = field with 128-column
                           // tiles for the real-valued path (p rows + a deeper W ring in smem),
                           // 3 = bf16 field layout for the real-valued path when 1 holds int8 digits,
                           // 4 = bf16 energy layout with 128-column tiles (the persistent kernel),
                           // 5 = int8 energy layout with 64-column tiles (the int8 persistent kernel)
  int* d_p1q = nullptr; int p1_int = -1;                // degree-1 cells on the digit grid (int8 persistent)
  int* d_items = nullptr; size_t items_cap = 0;          // persistent kernel: per-pair item ranges
  // stream-K schedule of CTA-pair field launches (sk_plan): units, split tiles, partials
  // stream-K plans, one per (batch, layout, column order), uploaded once and kept for the
  // handle's lifetime (captured graphs point at them); the partial buffers are shared
  struct SkPlan {
    long long B;
    const void* L;
    int ctdesc;
    int4* d_units;
    int4* d_sktiles;
    int nunits, ntiles;
  };
  std::vector<SkPlan> sk_plans;
  float* d_skG = nullptr; size_t skG_cap = 0;
  double* d_skQ = nullptr; size_t skQ_cap = 0;
  // the search loop as one CUDA graph per (chains, iterations, buffers); seed, chain0 and the
  // P_t table travel in d_sargs, so a replay needs one small copy and one graph launch
  unsigned long long* d_sargs = nullptr; size_t sargs_cap = 0;
  cudaGraphExec_t search_exec = nullptr;
  cudaStream_t gs = nullptr;                            // graph capture stream
  // energy / field calls: one CUDA graph (stage X, contraction, split-K reduce, argmin) per
  // (mode, input format, batch, buffers, kernel choice); replayed when the same call repeats
  cudaGraphExec_t call_exec[2] = {nullptr, nullptr};
  std::vector<uintptr_t> call_key[2];
  std::vector<uintptr_t> search_key;
  long long items_B = -1; int items_nct = 0;            // ... computed for this batch and tiling
  int dig = -1;            // int8 digit planes of slots 0/1 (0 = bf16 limbs; -1 = not decided yet)
  int f8 = -1;             // e4m3 limbs of slots 0/1 (0 = none; -1 = not decided yet)
  int f8_s = 0;            // their scale exponent: limbs of cell * 2^-f8_s
  bool f8_off[2] = {false, false};   // slot measured not worth it (too many second limbs)
  // scratch (grown on demand)
  uint32_t* d_bits = nullptr; size_t bits_cap = 0;
  double* d_Q = nullptr; size_t Q_cap = 0;
  unsigned long long* d_key = nullptr;
  unsigned long long* h_key = nullptr;                  // page-locked readback of the key
  float* d_G = nullptr; size_t G_cap = 0;
  uint32_t* d_xbest = nullptr; size_t xbest_cap = 0;
  float* d_ebest = nullptr; size_t ebest_cap = 0;
  float* d_Gpart = nullptr; size_t Gpart_cap = 0;      // split-K partials
  unsigned long long* d_k1 = nullptr; size_t k_cap = 0; // aggregation sort keys
  unsigned long long* d_k2 = nullptr; size_t k2_cap = 0;
  uint32_t* d_flag = nullptr; size_t flag_cap = 0;
  float* d_theta = nullptr; size_t theta_cap = 0;       // gradient descent state
  TTCores tt;                                           // Tensor-Train form (hobo_tt_build)
  double* d_tt = nullptr;
  int* d_tt_meta = nullptr;                             // [k] core offsets, [k+1] ranks
  uint16_t* d_P = nullptr; size_t P_cap = 0;
  uint32_t* d_starts = nullptr; size_t starts_cap = 0;
  double* d_Qpart = nullptr; size_t Qpart_cap = 0;
  uint8_t* d_xh[2] = {nullptr, nullptr}; size_t xh_cap = 0;   // host-input path: staged X chunks
  uint32_t* d_xbc = nullptr; size_t xbc_cap = 0;        // multi-GPU search: the winner's bits
  float* d_Eh = nullptr; size_t Eh_cap = 0;
  cudaStream_t cs = nullptr;                            // its input copy stream
  cudaStream_t cs_out = nullptr;                        // its field copy-out stream
  cudaEvent_t ev_in = nullptr, ev_copied[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
  cudaEvent_t ev_gdone[2] = {nullptr, nullptr}, ev_gfree[2] = {nullptr, nullptr};
  std::vector<hobo_tensor*> sa_child;                   // annealing: P_m = dE/dx_m per site m
  bool sa_borrowed = false;                             // a site tensor: its tables belong to the parent
  uint4* d_sa_runs = nullptr;                           // the site tensors' shared tables (same order, N)
  uint4* d_sa_kdesc = nullptr;
  uint32_t* d_sa_runoff = nullptr;
  int2* d_sa_sched = nullptr;
  // persistent annealer (Npad <= 512): every site's layout in one buffer, one TMA map
  bool sa_persistent = false;
  __nv_bfloat16* d_sa_W = nullptr;
  int* d_sa_L = nullptr;
  int* d_sa_base = nullptr;
  double* d_sa_T = nullptr; size_t sa_T_cap = 0;
  alignas(64) CUtensorMap sa_tmap;
  alignas(64) CUtensorMap sa_tmap2;   // CTA-pair kernel: half boxes (NT/2 rows)
  int sa_NT = 256, sa_nct = 1, sa_nkb1 = 1, sa_nseg = 0, sa_nq = 1;
  int sa_seg_kb0[8] = {0}, sa_seg_cnt[8] = {0};
  std::vector<int> sa_L;
  int8_t* d_sa_s = nullptr; size_t sa_s_cap = 0;        // decisions of the last two sites
  double* d_sa_E = nullptr; size_t sa_E_cap = 0;        // tracked energies
  int64_t last_launches = 0;
  double last_mma_macs = 0, last_algo_macs = 0;
  int last_i8 = 0;                                      // MMA kind of the last call: int8 digit planes (count) or 0 = bf16
  bool profile = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;   // around the contraction kernel(s) of the last call
  bool ev_valid = false;
};

namespace {

#define CK(call)                                                                                     \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) {                                                                         \
      t->poisoned = true;                                                                            \
      return fail(HOBO_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));                   \
    }                                                                                                \
  } while (0)

template <class T>
hobo_status grow(hobo_tensor* t, T*& p, size_t& cap, size_t n) {
  if (n <= cap) return HOBO_OK;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  CK(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  cap = n;
  return HOBO_OK;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device attribute of a kernel: set it
// once per (kernel, device), for the largest size requested so far
std::map<std::pair<const void*, int>, size_t>& smem_configured() {
  static std::map<std::pair<const void*, int>, size_t> m;
  return m;
}
template <class K>
cudaError_t set_smem(K* k, size_t smem) {
  static std::mutex mu;   // handles may live on different threads
  std::lock_guard<std::mutex> lock(mu);
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev)) return e;
  size_t& have = smem_configured()[{reinterpret_cast<const void*>(k), dev}];
  if (have >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e == cudaSuccess) have = smem;
  return e;
}

// profiling event around a contraction kernel; inside a stream capture it becomes an
// external event-record node of the graph, so the replayed graph still times the kernel
cudaError_t record_event(cudaEvent_t ev, cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaError_t e = cudaStreamIsCapturing(s, &cs)) return e;
  return cs == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal)
                                             : cudaEventRecord(ev, s);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  }
  return fn;
}

template <int NT, bool REAL, bool I8 = false, bool F8 = false>
cudaError_t launch_kr(const DevLayout& L, const KrParams& p, cudaStream_t s) {
  auto* k = kr_gemm_kernel<NT, REAL, false, false, I8, F8>;
  const size_t smem =
      REAL ? KrCfg<NT>::smem_bytes_real(p.ring_boxes, p.pstride) : KrCfg<NT, I8>::smem_bytes(p.W, p.srec_u4 * (F8 ? 2 : 1), F8 ? p.nl_words : 0, p.desc_lg);
  if (cudaError_t e = set_smem(k, smem)) return e;
  const int mb = (REAL || I8 || p.field_mode || p.n_split > 1 || p.cb_iters < 1) ? 1 : p.cb_iters;
  k<<<dim3((unsigned)(p.n_split * p.n_ct * ((p.n_cb + mb - 1) / mb))), dim3(kr_threads<F8>()), smem, s>>>(L.tmap, p);
  return cudaGetLastError();
}

template <int NT>
cudaError_t launch_kr_sa(const DevLayout& L, const KrParams& p, cudaStream_t s) {
  auto* k = kr_gemm_kernel<NT, false, true>;
  const size_t smem = KrCfg<NT>::smem_bytes(p.W);
  if (cudaError_t e = set_smem(k, smem)) return e;
  k<<<dim3((unsigned)(p.n_ct * p.n_cb)), dim3(kThreads), smem, s>>>(L.tmap, p);
  return cudaGetLastError();
}

// CTA pairs: clusters of 2 (adjacent candidate blocks of one column tile), cta_group::2 MMAs
template <int NT, bool REAL, bool I8 = false, bool F8 = false>
cudaError_t launch_kr_pair(const DevLayout& L, const KrParams& p, cudaStream_t s) {
  auto* k = kr_gemm_kernel<NT, REAL, false, true, I8, F8>;
  const size_t smem =
      REAL ? KrCfg<NT>::smem_bytes_real(p.ring_boxes, p.pstride) : KrCfg<NT, I8>::smem_bytes(p.W, p.srec_u4 * (F8 ? 2 : 1), F8 ? p.nl_words : 0, p.desc_lg);
  if (cudaError_t e = set_smem(k, smem)) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(p.units ? 2 * p.n_units : 2 * ((p.n_cb + 1) / 2) * p.n_ct * p.n_split));
  cfg.blockDim = dim3(kr_threads<F8>());
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, L.tmap_half, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// CTA pairs for long K loops (measured: cfg3-fp32 +19%, cfg5 +12%, cfg4 (128-column tiles)
// +21% at L = 3; cfg3 at L = 1 +2.3% since the ring counters and descriptor prefetch (it was
// 5% slower before); the real-valued cfg3 14.7 -> 13.6 ms).  Short K loops (cfg2's QUBO, 4-16
// K-blocks per CTA) do not amortise the pair's cluster synchronisation (-8%).
// HOBO_PAIR=1 / =0 forces the choice (A/B runs, tests of both paths).
bool use_pairs(const DevLayout& L, const KrParams& p) {
  if (p.n_split != 1) return false;
  if (const char* e = getenv("HOBO_PAIR")) return e[0] == '1';
  return p.n_kb >= 64;
}

cudaError_t launch_kr_any(const DevLayout& L, const KrParams& p, cudaStream_t s) {
  if (L.f8) {
    if (use_pairs(L, p))
      return L.NT == 128 ? launch_kr_pair<128, false, true, true>(L, p, s) : launch_kr_pair<256, false, true, true>(L, p, s);
    return L.NT == 128 ? launch_kr<128, false, true, true>(L, p, s) : launch_kr<256, false, true, true>(L, p, s);
  }
  if (L.i8) {
    if (use_pairs(L, p)) return L.NT == 128 ? launch_kr_pair<128, false, true>(L, p, s) : launch_kr_pair<256, false, true>(L, p, s);
    return L.NT == 128 ? launch_kr<128, false, true>(L, p, s) : launch_kr<256, false, true>(L, p, s);
  }
  if (use_pairs(L, p)) {
    if (p.preal) return L.NT == 128 ? launch_kr_pair<128, true>(L, p, s) : launch_kr_pair<256, true>(L, p, s);
    return L.NT == 128 ? launch_kr_pair<128, false>(L, p, s) : launch_kr_pair<256, false>(L, p, s);
  }
  if (L.NT == 128) return p.preal ? launch_kr<128, true>(L, p, s) : launch_kr<128, false>(L, p, s);
  return p.preal ? launch_kr<256, true>(L, p, s) : launch_kr<256, false>(L, p, s);
}

template <int NT>
int ring_boxes_for() { return KrCfg<NT>::RING_BOXES; }

constexpr size_t kMaxSmem = 232448 - 1024;   // 227 KB opt-in per block, minus static smem + margin

// real-valued path geometry: p rows in shared memory next to the W ring
template <int NT>
int real_ring(int pstride) {
  int ring = 0;
  while (ring < KrCfg<NT>::RING_BOXES && KrCfg<NT>::smem_bytes_real(ring + 1, pstride) <= kMaxSmem) ++ring;
  return ring;
}

bool real_geometry(hobo_tensor* t, int NT, int& pstride, int& ring, int& LA) {
  int words = (t->host.N + 1) / 2;
  if ((words & 1) == 0) ++words;            // odd word stride: conflict-free per-row reads
  pstride = 2 * words;
  ring = NT == 128 ? real_ring<128>(pstride) : real_ring<256>(pstride);
  LA = std::min(3, std::max(1, t->host.order - 1));
  return ring >= t->host.limbs;
}

hobo_status init_device(hobo_tensor* t);

// int8 digit planes for the binary energy / field layouts (slots 0 and 1): used when the degree
// >= 2 cells are a fixed-point grid of <= 3 bytes (exact), the int32 accumulators cannot
// overflow (255 x tuples < 2^31) and they take fewer tensor-core cycles than the bf16 limbs
// (an int8 MMA runs at twice the bf16 rate: d digits cost d/2 vs L limbs) over K loops of
// >= 64 K-blocks.  HOBO_I8=0 / =1 forces bf16 / int8 (when exact).
// the most generator runs of any K-block pair (the int8 path's stage records)
uint32_t pair_runs_max(const KLayout& kl) {
  const size_t nkb = kl.run_off.size() - 1;
  uint32_t rmax = 0;
  for (size_t a = 0; a < nkb; a += 2) rmax = std::max(rmax, kl.run_off[std::min(a + 2, nkb)] - kl.run_off[a]);
  return rmax;
}

int digit_planes(hobo_tensor* t) {
  if (t->dig >= 0) return t->dig;
  const HostTensor& H = t->host;
  int d = H.digits;
  if (d > 0 && 255.0 * (double)std::max<int64_t>(t->kl.Tpad, kBK) >= 2147483648.0) d = 0;
  // shared memory: W ring + 16 run-record slots + the candidates' bits must fit one CTA
  if (d > 0 && KrCfg<128, true>::smem_bytes(t->W, 1 + (int)pair_runs_max(t->kl), 0, 4) > kMaxSmem) d = 0;
  if (d > 0) {
    const char* e = getenv("HOBO_I8");
    if (e && e[0] == '0') d = 0;
    // default: only when it saves tensor-core cycles and the K loops are long enough (>= 64
    // K-blocks) to amortise the per-CTA cost of L accumulators (cfg2's 16-K-block QUBO: -12%)
    else if (!(e && e[0] == '1') && (d >= 2 * H.limbs || t->kl.Tpad / kBK < 64)) d = 0;
  }
  t->dig = d;
  return d;
}

// e4m3 limbs (kind::f8f6f4 at the int8 rate, one fp32 accumulator) for the binary energy /
// field layouts of INTEGER instances: every degree >= 2
// cell c, scaled by 2^-s so that max |c| 2^-s <= 448, must split exactly into <= 3 e4m3 limbs
// (greedy round-to-nearest, the layout kernel's split).  Binary-integer-encoded instances
// (cells = small integers x powers of two) need one limb for almost every cell, so a stage
// multiplies one limb box at the int8 rate, twice the bf16 rate; the limbs are exact and the
// accumulation is exact in fp32 under the bf16 path's own condition (integer cells,
// sum |H| < 2^24).  HOBO_F8=0 / =1: never / also for non-integer instances when the split is
// exact.  Returns the limb planes needed (0: not used).
double e4m3_rn(double v) {   // round to nearest even on the e4m3 grid (|v| <= 448 assumed)
  const double a = std::fabs(v);
  if (a == 0.0) return 0.0;
  int e = std::ilogb(a);
  const double q = std::ldexp(1.0, std::max(e, -6) - 3);   // the grid step (subnormals below 2^-6)
  const double r = std::nearbyint(a / q) * q;
  return v < 0 ? -r : r;
}

int e4m3_limbs(hobo_tensor* t) {
  if (t->f8 >= 0) return t->f8;
  t->f8 = 0;
  const HostTensor& H = t->host;
  const char* e = getenv("HOBO_F8");
  if (e && e[0] == '0') return 0;
  const char* ei = getenv("HOBO_I8");
  if (ei && ei[0] == '1') return 0;   // int8 digit planes forced
  if (H.order < 2 || t->kl.Tpad / kBK < 64) return 0;   // short K loops: the persistent / bf16 kernels
  if (!H.is_integer && !(e && e[0] == '1')) return 0;
  if (H.is_integer && !(H.sum_abs < 16777216.0)) return 0;
  if (KrCfg<256, true>::smem_bytes(t->W, 2 * (1 + (int)pair_runs_max(t->kl)), (int)((t->kl.Tpad / (2 * kBK) + 15) / 16), 4) >
      kMaxSmem)
    return 0;
  double amax = 0.0;
  for (int r = 2; r <= H.order; ++r)
    for (float c : H.strict[r]) amax = std::max(amax, (double)std::fabs(c));
  if (amax == 0.0) return 0;
  // s >= 0 on integer instances: every limb is then an integer in cell units (a cell >= 16 has
  // a grid step >= 1, a smaller one is a single exact limb), so each partial sum is an integer
  // multiple of 2^-(s+9) bounded by sum |H| < 2^24 of them: exact in fp32.  Otherwise the largest
  // cell is scaled into [224, 448] (the most headroom above the subnormal floor).
  int sexp = 0;
  while (std::ldexp(amax, -sexp) > 448.0) ++sexp;
  if (!H.is_integer)
    while (sexp > -60 && std::ldexp(amax, -(sexp - 1)) <= 448.0) --sexp;
  int need = 1;
  for (int r = 2; r <= H.order && need <= 3; ++r)
    for (float c : H.strict[r]) {
      double v = std::ldexp((double)c, -sexp);
      int l = 0;
      while (v != 0.0 && l < 4) {
        const double h = e4m3_rn(v);
        if (h == 0.0) { l = 4; break; }   // below the e4m3 grid: not representable
        v -= h;                            // exact (h is v rounded to 4 significant bits)
        ++l;
      }
      if (l > need) need = l;
      if (need > 3) break;
    }
  if (need > 3) return 0;
  t->f8_s = sexp;
  t->f8 = need;
  return need;
}

hobo_status check_device(hobo_tensor* t) {
  if (t->poisoned) return fail(HOBO_ESTATE, "handle poisoned by an earlier CUDA error");
  if (!t->dev_init) return init_device(t);
  int cur = -1;
  CK(cudaGetDevice(&cur));
  if (cur != t->device) CK(cudaSetDevice(t->device));
  return HOBO_OK;
}

hobo_status init_device(hobo_tensor* t) {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  if (prop.major != 10) return fail(HOBO_ECUDA, "sm_100 (B200) device required; found sm_" + std::to_string(prop.major) +
                                                    std::to_string(prop.minor));
  t->device = dev;
  const int N = t->host.N;
  t->W = (N + 31) / 32;
  std::string msg;
  if (build_klayout(t->host.order, N, t->kl, msg)) return fail(HOBO_ENOMEM, msg);
  CK(cudaMalloc(&t->d_runs, std::max<size_t>(t->kl.runs.size() / 4, 1) * sizeof(uint4)));
  if (!t->kl.runs.empty())
    CK(cudaMemcpy(t->d_runs, t->kl.runs.data(), t->kl.runs.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&t->d_kdesc, std::max<size_t>(t->kl.kdesc.size() / 4, 2) * sizeof(uint4)));
  if (!t->kl.kdesc.empty())
    CK(cudaMemcpy(t->d_kdesc, t->kl.kdesc.data(), t->kl.kdesc.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&t->d_runoff, t->kl.run_off.size() * 4));
  CK(cudaMemcpy(t->d_runoff, t->kl.run_off.data(), t->kl.run_off.size() * 4, cudaMemcpyHostToDevice));
  const int Npad = (N + 255) / 256 * 256;
  std::vector<float> p1(Npad, 0.0f);
  for (int m = 0; m < N; ++m) p1[m] = t->host.strict[1][m];
  CK(cudaMalloc(&t->d_p1, Npad * sizeof(float)));
  CK(cudaMemcpy(t->d_p1, p1.data(), Npad * sizeof(float), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&t->d_key, 2 * sizeof(unsigned long long)));   // [0] argmin key, [1] ~0 unless a NaN was seen
  t->dev_init = true;
  return HOBO_OK;
}

// builds W (bf16 limb planes) of one layout on the device, plus its TMA map and schedule
hobo_status ensure_layout(hobo_tensor* t, int slot) {
  DevLayout& L = t->lay[slot];
  if (L.built) return HOBO_OK;
  const int field = (slot == 0 || slot == 4 || slot == 5) ? 0 : 1;
  const HostTensor& H = t->host;
  const int N = H.N, k = H.order;
  L.i8 = slot <= 1 ? digit_planes(t) : slot == 5 ? H.digits : 0;
  L.f8 = false;
  if (slot <= 1 && !t->f8_off[slot] && e4m3_limbs(t) > 0) {   // tried first; kept if the scan says it pays
    L.i8 = e4m3_limbs(t);
    L.f8 = true;
    if (const char* ex = getenv("HOBO_KR_EXP"))   // MEASUREMENT ONLY: 4 = one limb plane (results wrong)
      if (atoi(ex) & 4) L.i8 = 1;
    L.fscale = (float)std::ldexp(1.0, t->f8_s + 9);   // A = e4m3 0x01 = 2^-9
  }
  L.NT = (N <= 128 || slot == 2 || slot == 4) ? 128 : 256;   // a 128-column tile when N fits (no padded columns)
  if (L.i8 >= 2 && !L.f8) L.NT = 128;           // TMEM: i8 accumulators of NT columns + the A stages
  if (slot == 5) {                              // the int8 persistent kernel's tiles: 64 columns, two
    const char* e = getenv("HOBO_PERSIST_I8_NT");   // accumulator sets (128: one set, measured slower)
    L.NT = (e && atoi(e) == 128) ? 128 : 64;
  }
  L.qscale = std::ldexp(1.0, H.qexp);
  const int planes = L.i8 ? L.i8 : H.limbs;
  if (N > 1024) return fail(HOBO_EINVAL, "the device path supports N <= 1024 (candidate bits are staged in shared memory)");
  L.n_ct = (N + L.NT - 1) / L.NT;
  L.Npad = L.n_ct * L.NT;
  const int64_t Tpad = std::max<int64_t>(t->kl.Tpad, 2 * kBK);   // (a multiple of 2 K-blocks)
  const double bytes = (double)planes * L.Npad * Tpad * (L.i8 ? 1.0 : 2.0);
  if (L.i8 && slot <= 1 && !t->d_srec) {
    // stage records: for K-block pair P, uint4 {runs of 2P, runs of 2P+1, nfix, 0} followed by
    // the pair's runs (contiguous in kl.runs), padded to the most runs of any pair; one TMA
    // bulk copy brings a stage's whole generator input (no dependent global loads)
    const KLayout& kl = t->kl;
    const int64_t npair = Tpad / (2 * kBK);
    t->srec_u4 = 1 + (int)pair_runs_max(kl);
    std::vector<uint32_t> rec((size_t)(npair + 1) * t->srec_u4 * 4, 0);   // + a zero record (e4m3 stages copy 2)
    for (int64_t P = 0; P < npair; ++P) {
      uint32_t* r = &rec[(size_t)P * t->srec_u4 * 4];
      const size_t nkb = kl.run_off.size() - 1;
      if ((size_t)(2 * P) >= nkb) continue;
      const uint32_t a = kl.run_off[2 * P], b = kl.run_off[2 * P + 1];
      const uint32_t c = (size_t)(2 * P + 2) <= nkb ? kl.run_off[2 * P + 2] : b;
      r[0] = b - a;
      r[1] = c - b;
      r[2] = kl.kdesc[(size_t)(2 * P) * 8 + 3] & 7u;   // nfix (a pair never spans two segments)
      for (uint32_t i = a; i < c; ++i) {
        // run (start, cnt, lo, fixed ids) -> the precomputed form run_bits8 reads (kernels.cuh):
        // output bits [start, start + cnt) of the K-block = x bits lo .. lo + cnt, i.e. the
        // 64-bit window at s = lo - start + 64 counted from two zero words in front of the row
        const uint32_t* q = &kl.runs[(size_t)i * 4];
        const uint32_t start = q[0] & 0xFFu, cnt = (q[0] >> 8) & 0xFFu, lo = q[0] >> 16;
        const uint64_t mask = (cnt >= 64 ? ~0ull : ((1ull << cnt) - 1ull)) << start;
        const uint32_t sw = lo + 64u - start;
        const uint32_t f0 = q[1] & 1023u, f1 = (q[1] >> 16) & 1023u, f2 = q[2] & 1023u, f3 = (q[2] >> 16) & 1023u;
        uint32_t* o = &r[4 * (1 + i - a)];
        o[0] = (uint32_t)mask;
        o[1] = (uint32_t)(mask >> 32);
        o[2] = (sw >> 5) | ((sw & 31u) << 6) | (f0 << 11) | (f1 << 21);
        o[3] = f2 | (f3 << 10);
      }
    }
    CK(cudaMalloc(&t->d_srec, rec.size() * 4));
    CK(cudaMemcpy(t->d_srec, rec.data(), rec.size() * 4, cudaMemcpyHostToDevice));
  }
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  if (bytes > 0.8 * (double)free_b)
    return fail(HOBO_ENOMEM, "device layout needs " + std::to_string(bytes / 1e9) + " GB (N=" + std::to_string(N) +
                                 ", order=" + std::to_string(k) + ", planes=" + std::to_string(planes) + ")");
  CK(cudaMalloc(&L.W, (size_t)bytes));
  if (t->kl.Tpad > 0) {
    // temporaries: per-degree cells, binomials, tuple list
    std::vector<float*> dstrict(7, nullptr);
    for (int r = 2; r <= k; ++r) {
      CK(cudaMalloc(&dstrict[r], std::max<size_t>(H.strict[r].size(), 1) * sizeof(float)));
      CK(cudaMemcpy(dstrict[r], H.strict[r].data(), H.strict[r].size() * sizeof(float), cudaMemcpyHostToDevice));
    }
    float** d_strict_ptrs = nullptr;
    CK(cudaMalloc(&d_strict_ptrs, 7 * sizeof(float*)));
    CK(cudaMemcpy(d_strict_ptrs, dstrict.data(), 7 * sizeof(float*), cudaMemcpyHostToDevice));
    std::vector<long long> bt((size_t)(N + 1) * 7);
    for (int n = 0; n <= N; ++n)
      for (int i = 0; i < 7; ++i) bt[(size_t)n * 7 + i] = binom(n, i);
    long long* d_bt = nullptr;
    CK(cudaMalloc(&d_bt, bt.size() * sizeof(long long)));
    CK(cudaMemcpy(d_bt, bt.data(), bt.size() * sizeof(long long), cudaMemcpyHostToDevice));
    uint16_t* d_tup = nullptr;
    CK(cudaMalloc(&d_tup, t->kl.tuples.size() * sizeof(uint16_t)));
    CK(cudaMemcpy(d_tup, t->kl.tuples.data(), t->kl.tuples.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    LayoutParams lp;
    lp.tuples = d_tup;
    lp.strict = d_strict_ptrs;
    lp.binomT = d_bt;
    lp.Wout = L.W;
    lp.Tpad = Tpad;
    lp.N = N;
    lp.Npad = L.Npad;
    lp.L = planes;
    lp.field_mode = field;
    lp.NT = L.NT;
    int* d_err = nullptr;
    if (L.i8) {
      lp.Wout8 = reinterpret_cast<uint8_t*>(L.W);
      lp.inv_qscale = std::ldexp(1.0, -H.qexp);
    }
    if (L.f8) {
      lp.f8_scale = std::ldexp(1.0, -t->f8_s);
      CK(cudaMalloc(&d_err, sizeof(int)));
      CK(cudaMemset(d_err, 0, sizeof(int)));
      lp.err = d_err;
    }
    layout_kernel<<<148 * 8, 256>>>(lp);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    if (L.f8) {
      // each K-block pair's limb count per column tile (the most limb planes a cell of its box
      // needs), packed 2 bits per pair into L.d_nltab [n_ct][nl_words] (KrParams::nltab)
      int err = 0;
      CK(cudaMemcpy(&err, d_err, sizeof(int), cudaMemcpyDeviceToHost));
      cudaFree(d_err);
      const char* ex = getenv("HOBO_KR_EXP");
      if (err && !(ex && (atoi(ex) & 4)))
        return fail(HOBO_ECUDA, "e4m3 limb split inexact on the device (host and device grids disagree)");
      const int64_t n_kbp = Tpad / (2 * kBK);
      std::vector<uint32_t> nl((size_t)L.n_ct * n_kbp, 1u);
      uint32_t* d_nl = nullptr;
      CK(cudaMalloc(&d_nl, nl.size() * 4));
      CK(cudaMemcpy(d_nl, nl.data(), nl.size() * 4, cudaMemcpyHostToDevice));
      f8_limbs_kernel<<<148 * 8, 256>>>(reinterpret_cast<const uint8_t*>(L.W), L.i8, L.n_ct, n_kbp, L.NT, d_nl);
      CK(cudaGetLastError());
      CK(cudaMemcpy(nl.data(), d_nl, nl.size() * 4, cudaMemcpyDeviceToHost));
      cudaFree(d_nl);
      double sum = 0;
      for (uint32_t v : nl) sum += v;
      L.f8_density = sum / (double)nl.size();
      L.nl_words = (int)((n_kbp + 15) / 16);
      std::vector<uint32_t> tab((size_t)L.n_ct * L.nl_words, 0u);
      for (int ct = 0; ct < L.n_ct; ++ct)
        for (int64_t P = 0; P < n_kbp; ++P)
          tab[(size_t)ct * L.nl_words + P / 16] |= nl[(size_t)ct * n_kbp + P] << (2 * (P % 16));
      CK(cudaMalloc(&L.d_nltab, tab.size() * 4));
      CK(cudaMemcpy(L.d_nltab, tab.data(), tab.size() * 4, cudaMemcpyHostToDevice));
      // a limb box costs half a bf16 limb box (as an int8 digit plane does): keep e4m3 only
      // when it saves >= 20% of the tensor-core cycles of the path chosen otherwise, else
      // rebuild this slot's layout with int8 digits / bf16 limbs
      const int dp = digit_planes(t);
      const double other = dp ? 0.5 * dp : (double)H.limbs;
      if (0.5 * L.f8_density > 0.8 * other) {
        for (int r = 2; r <= k; ++r) cudaFree(dstrict[r]);
        cudaFree(d_strict_ptrs);
        cudaFree(d_bt);
        cudaFree(d_tup);
        cudaFree(L.W);
        cudaFree(L.d_nltab);
        L = DevLayout();
        t->f8_off[slot] = true;
        return ensure_layout(t, slot);
      }
    }
    for (int r = 2; r <= k; ++r) cudaFree(dstrict[r]);
    cudaFree(d_strict_ptrs);
    cudaFree(d_bt);
    cudaFree(d_tup);
  } else {
    CK(cudaMemset(L.W, 0, (size_t)bytes));
  }
  // TMA map over the 2-D view [L * Npad rows][Tpad tuples], box 64 x NT, 128-byte swizzle
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(HOBO_ECUDA, "cuTensorMapEncodeTiled unavailable");
  // 3-D view of the tile-blocked planes: (64 tuples, NT rows, box index), box = one block
  // (int8 digit planes: 128-byte rows = K-block pairs, boxes (128 tuples, NT rows, pair index))
  const int64_t n_kb = Tpad / kBK;
  const int inner = L.i8 ? 2 * kBK : kBK;          // elements per 128-byte box row (e4m3 limbs: UINT8 too)
  const int64_t nbox = L.i8 ? n_kb / 2 : n_kb;
  const CUtensorMapDataType dt = L.i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B;
  cuuint64_t dims[3] = {(cuuint64_t)inner, (cuuint64_t)L.NT, (cuuint64_t)planes * L.n_ct * nbox};
  cuuint64_t strides[2] = {128, (cuuint64_t)128 * L.NT};
  cuuint32_t box[3] = {(cuuint32_t)inner, (cuuint32_t)L.NT, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = enc(&L.tmap, dt, 3, L.W, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(HOBO_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
  cuuint32_t box_half[3] = {(cuuint32_t)inner, (cuuint32_t)(L.NT / 2), 1};
  cr = enc(&L.tmap_half, dt, 3, L.W, dims, strides, box_half, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(HOBO_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
  L.sched = schedule(t->kl, L.NT, L.n_ct, field != 0);
  CK(cudaMalloc(&L.d_sched, L.sched.size() * sizeof(int32_t)));
  CK(cudaMemcpy(L.d_sched, L.sched.data(), L.sched.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  if (field) {
    double lcm = 1;
    for (int r = 2; r <= k; ++r) {
      double a = lcm, b = r;
      while (b) { double tmp = std::fmod(a, b); a = b; b = tmp; }
      lcm = lcm * r / a;
    }
    L.lcm = lcm;
    for (int r = 0; r < 8; ++r) L.wdeg[r] = (r >= 1 && r <= k) ? lcm / (double)r : 0.0;
    L.wp = lcm;
  }
  L.built = true;
  return HOBO_OK;
}

KrParams make_params(hobo_tensor* t, const DevLayout& L, const uint32_t* bits, long long B, float* G, double* Q) {
  KrParams p;
  p.xbits = bits;
  p.runs = t->d_runs;
  p.kdesc = t->d_kdesc;
  p.sched = L.d_sched;
  p.p1 = t->d_p1;
  p.G = G;
  p.Q = Q;
  p.B = B;
  p.N = t->host.N;
  p.W = t->W;
  p.Npad = L.Npad;
  p.n_ct = L.n_ct;
  p.n_cb = (int)((B + kBM - 1) / kBM);
  p.n_kb = (int)(std::max<int64_t>(t->kl.Tpad, 2 * kBK) / kBK);
  p.n_split = 1;
  p.cb_iters = 1;
  {
    // longest-first: the open index's last column tile has the most rows,
    // and issuing it first keeps the short tiles for the tail of the last wave
    auto kbs = [&](int ct) {
      long long kb = 0;
      for (int j = 0; j < t->kl.nseg; ++j) kb += L.sched[((size_t)ct * t->kl.nseg + j) * 2 + 1];
      return kb;
    };
    p.ct_desc = (L.n_ct > 1 && kbs(L.n_ct - 1) > kbs(0)) ? 1 : 0;
    if (const char* e = getenv("HOBO_CT_DESC")) p.ct_desc = e[0] == '1';
  }
  p.preal = nullptr;
  p.units = nullptr;
  p.n_units = 0;
  p.skG = nullptr;
  p.skQ = nullptr;
  p.LA = 1;
  p.ring_boxes = L.NT == 128 ? ring_boxes_for<128>() : ring_boxes_for<256>();
  p.pstride = 0;
  p.nseg = t->kl.nseg;
  p.L = L.i8 ? L.i8 : t->host.limbs;
  p.qscale = L.qscale;
  p.fscale = L.fscale;
  p.srec = t->d_srec;
  p.srec_u4 = L.i8 ? t->srec_u4 : 0;
  // 32 descriptor-ring slots when they fit next to the rest of the CTA's shared memory, else 16
  const int rslot = p.srec_u4 * (L.f8 ? 2 : 1);   // e4m3 stages carry two pairs' records
  const size_t sm32 = L.NT == 128 ? KrCfg<128, true>::smem_bytes(t->W, rslot, L.nl_words, 5)
                                  : KrCfg<256, true>::smem_bytes(t->W, rslot, L.nl_words, 5);
  p.desc_lg = (L.i8 && sm32 > kMaxSmem) ? 4 : 5;
  p.field_mode = (&L == &t->lay[0] || &L == &t->lay[4] || &L == &t->lay[5]) ? 0 : 1;
  p.nltab = L.d_nltab;
  p.nl_words = L.nl_words;
  p.exp = 0;
  if (const char* e = getenv("HOBO_KR_EXP")) p.exp = atoi(e);
  for (int r = 0; r < 8; ++r) p.wdeg[r] = L.wdeg[r];
  p.wp = L.wp;
  return p;
}

// split-K factor: only when the (candidate block x column tile) grid cannot fill the GPU;
// then about one wave of long-running CTAs (each streams its K chunk of W once)
int choose_split(hobo_tensor* t, const DevLayout& L, long long B) {
  const long long tiles = ((B + kBM - 1) / kBM) * L.n_ct;
  if (tiles >= 148) return 1;
  const int KPS = L.f8 ? 4 : L.i8 ? 2 : L.NT == 128 ? KrCfg<128>::kps(t->host.limbs) : KrCfg<256>::kps(t->host.limbs);
  int stages = 0;
  for (int ct = 0; ct < L.n_ct; ++ct) {
    int s = 0;
    for (int j = 0; j < t->kl.nseg; ++j) s += (L.sched[((size_t)ct * t->kl.nseg + j) * 2 + 1] + KPS - 1) / KPS;
    stages = std::max(stages, s);
  }
  const long long want = 148 / tiles;
  return (int)std::max<long long>(1, std::min<long long>({want, stages / 4, 148}));
}

double exec_macs(hobo_tensor* t, const DevLayout& L, long long B) {
  double kb = 0;
  for (int ct = 0; ct < L.n_ct; ++ct)
    for (int j = 0; j < t->kl.nseg; ++j) kb += L.sched[((size_t)ct * t->kl.nseg + j) * 2 + 1];
  return kb * kBK * (double)L.NT * kBM * (double)((B + kBM - 1) / kBM) *
         (L.f8 ? L.f8_density : L.i8 ? L.i8 : t->host.limbs);
}

// SURVEY 8(d)'s algorithmic work: nnz MACs (2 nnz flops) per candidate for the energy, 2 nnz
// MACs (4 nnz flops) for energy + field, nnz = sum_{r<=k} C(N, r) canonical cells.  (The
// open-index GEMM executes sum_r r C(N, r) MACs per candidate in field mode: exec_macs.)
double algo_macs(hobo_tensor* t, bool field, long long B) {
  double s = 0;
  for (int r = 1; r <= t->host.order; ++r) s += (double)binom(t->host.N, r);
  return (field ? 2.0 : 1.0) * s * (double)B;
}

// C1: the global lexicographic (E, idx) minimum over ranks, on the compute stream
hobo_status key_allreduce(hobo_tensor* t, cudaStream_t s) {
  if (!dist_active()) return HOBO_OK;
  ncclResult_t r = g_dist.all_reduce(t->d_key, t->d_key, 2, ncclUint64, ncclMin, g_dist.comm, s);
  if (r != ncclSuccess) return fail(HOBO_ENCCL, std::string("ncclAllReduce: ") + g_dist.err(r));
  return HOBO_OK;
}

// the 16-byte key to the host through a page-locked buffer (a pageable destination makes the
// driver stage the copy synchronously), then wait for the stream
cudaError_t read_key(hobo_tensor* t, unsigned long long (&key)[2], cudaStream_t s) {
  if (!t->h_key)
    if (cudaError_t e = cudaMallocHost(&t->h_key, 2 * sizeof(unsigned long long))) return e;
  if (cudaError_t e = cudaMemcpyAsync(t->h_key, t->d_key, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s))
    return e;
  if (cudaError_t e = cudaStreamSynchronize(s)) return e;
  key[0] = t->h_key[0];
  key[1] = t->h_key[1];
  return cudaSuccess;
}

// the argmin key (device) -> host best, after the multi-GPU combine when one is active
hobo_status finish_best(hobo_tensor* t, hobo_best* best, cudaStream_t s) {
  if (hobo_status st = key_allreduce(t, s)) return st;
  unsigned long long key[2] = {0, 0};
  CK(read_key(t, key, s));
  if (key[1] != ~0ull) return fail(HOBO_ERANGE, "a candidate's energy is NaN (the argmin rejects NaN)");
  return hobo_best_from_key(key[0], best);
}

// an empty local batch still takes part in the combine (the other ranks wait for it)
hobo_status empty_best(hobo_tensor* t, hobo_best* best, cudaStream_t s) {
  if (!best) return HOBO_OK;
  if (!dist_active()) {
    best->e = INFINITY;
    best->idx = -1;
    return HOBO_OK;
  }
  CK(cudaMemsetAsync(t->d_key, 0xFF, 2 * sizeof(unsigned long long), s));
  return finish_best(t, best, s);
}

// stage X: u8 B x N -> bit rows; whole-word rows from an aligned buffer
// take the vectorised kernel (cfg2: 65 -> ~12 us per 64 MB)
void launch_pack_x(const uint8_t* X, long long B, int N, int W, uint32_t* bits, cudaStream_t s) {
  if (N % 32 == 0 && ((uintptr_t)X & 15) == 0) {
    const long long nchunks = B * (long long)N / 16;
    pack_x16_kernel<<<(unsigned)std::max<long long>(1, std::min<long long>((nchunks + 255) / 256, 148 * 16)), 256, 0, s>>>(
        reinterpret_cast<const uint4*>(X), nchunks, bits);
  } else {
    const long long nw = B * W;
    pack_x_kernel<<<(unsigned)std::min<long long>((nw + 255) / 256, 148 * 16), 256, 0, s>>>(X, B, N, W, bits);
  }
}

// layout slot of the real-valued path: the field layout, or, when its p rows plus L limb
// boxes of 256 columns do not fit in shared memory (e.g. N = 512 at L = 3), the same layout
// with 128-column tiles (half-size boxes).  (128-column tiles everywhere measured 1.8x slower
// at cfg3: twice the CTAs generate A.)
int real_slot(hobo_tensor* t) {
  // the real-valued path needs bf16 limb planes: slot 1 holds 1-byte planes (int8 digits, or
  // e4m3 limbs unless its build measured them not worth it) -> a bf16 copy in slot 3 (or 2)
  const bool bytes = t->lay[1].built ? t->lay[1].i8 != 0 : (digit_planes(t) || (e4m3_limbs(t) > 0 && !t->f8_off[1]));
  const int full = bytes ? 3 : 1;
  if (t->host.N <= 128) return bytes ? 2 : 1;
  int ps = 0, ring = 0, la = 0;
  return real_geometry(t, 256, ps, ring, la) ? full : 2;
}

// the persistent energy kernel (persist.cuh) for short K loops: energy mode on bf16 limbs whose
// tiles have fewer than 64 K-blocks (QUBO-like, BASELINE config 2), with enough (candidate-block
// pair, column tile) items to keep every SM pair busy.  HOBO_PERSIST=1 / =0 forces it on / off.
// Returns 0 (per-tile kr_gemm_kernel), 1 (bf16 limbs, kr_persist_kernel) or 2 (int8 digit
// planes, kr_persist_i8_kernel: exact, half the MMA work and W bytes of 3 bf16 limbs -- but
// each plane has its own s32 accumulator, and reading 3 accumulators per tile through TMEM's
// 64 B/clk read port costs about as much as a short tile's MMAs: 0.176 ms (64-column tiles,
// two accumulator sets) / 0.197 ms (128-column tiles, one set) against 0.161 ms on bf16
// limbs at cfg2, so opt-in).  HOBO_PERSIST=1 / =0 forces a
// persistent kernel on / off, HOBO_PERSIST_I8=1 selects the int8 one when the cells allow.
int use_persist(hobo_tensor* t, long long B) {
  const HostTensor& H = t->host;
  const bool i8_ok = H.digits >= 1 && H.digits <= PersistI8Cfg<128>::MAXP && 255.0 * 32.0 * (double)t->kl.Tpad < 2147483648.0;
  const char* ei = getenv("HOBO_PERSIST_I8");
  const int kind = (i8_ok && ei && ei[0] == '1') ? 2 : (H.limbs <= PersistCfg::MAXL ? 1 : 0);
  if (kind == 0 || t->kl.nseg > 8) return 0;
  if (const char* e = getenv("HOBO_PERSIST")) return e[0] == '1' ? kind : 0;
  if (digit_planes(t) || t->kl.Tpad / kBK >= 64) return 0;
  const long long items = (B + 2 * kBM - 1) / (2 * kBM) * ((H.N + 127) / 128);
  return items >= 4 * 74 ? kind : 0;
}

// contiguous item ranges of the persistent kernel, balanced by MMA work: item = candidate-block
// pair x column tile (heaviest tile of a block first), weight = its K-blocks + one for the
// per-item handoffs; pair p takes the items whose cumulative weight starts in [p W/P, (p+1) W/P)
hobo_status persist_items(hobo_tensor* t, const DevLayout& L, long long B, int& npairs, cudaStream_t s) {
  const int n_cbp = (int)((B + 2 * kBM - 1) / (2 * kBM));
  const long long nitems = (long long)n_cbp * L.n_ct;
  npairs = (int)std::min<long long>(74, nitems);
  if (t->items_B == B && t->items_nct == L.n_ct) return HOBO_OK;
  std::vector<double> w(L.n_ct);
  double per_block = 0;
  for (int k = 0; k < L.n_ct; ++k) {
    const int ct = L.n_ct - 1 - k;
    double kb = 0;
    for (int j = 0; j < t->kl.nseg; ++j) kb += L.sched[((size_t)ct * t->kl.nseg + j) * 2 + 1];
    w[k] = kb + 1.0;
    per_block += w[k];
  }
  const double total = per_block * n_cbp;
  std::vector<int> items((size_t)npairs + 1, 0);
  double acc = 0;
  int p = 1;
  for (long long i = 0; i < nitems && p < npairs; ++i) {
    while (p < npairs && acc >= total * p / npairs) items[(size_t)p++] = (int)i;
    acc += w[(size_t)(i % L.n_ct)];
  }
  while (p <= npairs) items[(size_t)p++] = (int)nitems;
  items[(size_t)npairs] = (int)nitems;
  if (hobo_status st = grow(t, t->d_items, t->items_cap, items.size())) return st;
  // ordered on the call's stream: an earlier launch on it may still read the old ranges
  CK(cudaMemcpyAsync(t->d_items, items.data(), items.size() * sizeof(int), cudaMemcpyHostToDevice, s));
  t->items_B = B;
  t->items_nct = L.n_ct;
  return HOBO_OK;
}

template <class K, class Params>
cudaError_t launch_persist(K* k, size_t smem, const DevLayout& L, const Params& p, int npairs, cudaStream_t s) {
  if (cudaError_t e = set_smem(k, smem)) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(2 * npairs));
  cfg.blockDim = dim3(kPThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, L.tmap_half, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// Stream-K schedule for CTA-pair field launches (bf16 limbs).  A field-mode tile (candidate-
// block pair x column tile) is the same K loop for every tile, and one CTA pair per two SMs runs
// at a time (74 slots), so T tiles take ceil(T / 74) tile-times: cfg3's 512 tiles 6.92 -> 7, a
// GPU's 64 tiles at 8-GPU strong scaling 0.86 -> 1.  Whole waves stay data-parallel (each tile
// one CTA pair, written in place); the R < 74 tiles left over are cut into 74 equal K ranges of
// R/74 tile, each range one or two units (its pieces in one or two tiles).  Every unit of a
// split tile writes partial fields + energies to its own slot; sk_reduce_kernel sums them in K
// order.  Units are ordered whole tiles, then the ranges' first pieces, then their second pieces
// longest first: a slot whose first piece ends early takes a long second piece, so every slot
// does about R/74 of a tile after the data-parallel waves.  HOBO_SK=0 disables it.
hobo_status sk_plan(hobo_tensor* t, const DevLayout& L, const KrParams& p, long long B,
                    const hobo_tensor::SkPlan*& use, cudaStream_t s) {
  use = nullptr;
  if (const char* e = getenv("HOBO_SK"))
    if (e[0] == '0') return HOBO_OK;
  const int KPS = L.f8 ? 4 : L.i8 ? 2 : L.NT == 128 ? KrCfg<128>::kps(t->host.limbs) : KrCfg<256>::kps(t->host.limbs);
  std::vector<int> tot(L.n_ct, 0);
  for (int ct = 0; ct < L.n_ct; ++ct)
    for (int j = 0; j < t->kl.nseg; ++j) tot[ct] += (L.sched[((size_t)ct * t->kl.nseg + j) * 2 + 1] + KPS - 1) / KPS;
  for (int ct = 1; ct < L.n_ct; ++ct)
    if (tot[ct] != tot[0]) return HOBO_OK;   // (field mode: every tile has the same K loop)
  const int total = tot[0];
  const int slots = 74;
  const long long ncbp = (B + 2 * kBM - 1) / (2 * kBM);
  const long long tiles = ncbp * L.n_ct;
  const long long D = tiles / slots * slots, R = tiles - D;
  if (R == 0 || tiles < slots / 2 || total < 4 * slots || total >= (1 << 20)) return HOBO_OK;
  // a leftover wave this full behind whole waves gains less than the partial sums cost
  // (e4m3 cfg3, 68 of 74 slots: step 2.242 ms without, 2.257 ms with)
  if (D > 0 && 10 * R >= 9 * slots) return HOBO_OK;
  for (const auto& q : t->sk_plans)
    if (q.B == B && q.L == &L && q.ctdesc == p.ct_desc) {
      use = &q;
      return HOBO_OK;
    }
  if (t->sk_plans.size() >= 16) return HOBO_OK;   // a new batch size beyond the cache: data-parallel
  auto tile = [&](long long tau, int& cbp, int& ct) {
    const int ct_i = (int)(tau / ncbp);
    ct = p.ct_desc ? L.n_ct - 1 - ct_i : ct_i;
    cbp = (int)(tau % ncbp);
  };
  std::vector<int4> units, firsts, seconds, sktiles;
  for (long long tau = 0; tau < D; ++tau) {
    int cbp, ct;
    tile(tau, cbp, ct);
    units.push_back(make_int4(cbp, ct, 0, total));
  }
  const long long flat = R * total;
  const long long Lr = (flat + slots - 1) / slots;
  int part = 0;
  std::vector<int> first_part(R, -1), nparts(R, 0);
  for (long long i = 0; i < slots; ++i) {
    long long a = i * Lr, b = std::min(flat, a + Lr);
    for (int piece = 0; a < b; ++piece) {
      const long long r = a / total;
      const long long e = std::min(b, (r + 1) * total);
      int cbp, ct;
      tile(D + r, cbp, ct);
      if (first_part[r] < 0) first_part[r] = part;
      ++nparts[r];
      const int4 u = make_int4(cbp, ct, (int)(a - r * total), (int)(e - r * total) | ((part + 1) << 20));
      (piece == 0 ? firsts : seconds).push_back(u);
      ++part;
      a = e;
    }
  }
  if (part >= (1 << 11)) return HOBO_OK;
  std::stable_sort(seconds.begin(), seconds.end(), [](const int4& x, const int4& y) {
    return ((x.w & 0xFFFFF) - x.z) > ((y.w & 0xFFFFF) - y.z);
  });
  units.insert(units.end(), firsts.begin(), firsts.end());
  units.insert(units.end(), seconds.begin(), seconds.end());
  for (long long r = 0; r < R; ++r) {
    int cbp, ct;
    tile(D + r, cbp, ct);
    sktiles.push_back(make_int4(cbp, ct, first_part[r], nparts[r]));
  }
  if (hobo_status st = grow(t, t->d_skG, t->skG_cap, (size_t)part * 2 * kBM * L.NT)) return st;
  if (hobo_status st = grow(t, t->d_skQ, t->skQ_cap, (size_t)part * 2 * kBM)) return st;
  hobo_tensor::SkPlan q{B, &L, p.ct_desc, nullptr, nullptr, (int)units.size(), (int)sktiles.size()};
  CK(cudaMalloc(&q.d_units, units.size() * sizeof(int4)));
  if (cudaMalloc(&q.d_sktiles, sktiles.size() * sizeof(int4)) != cudaSuccess) {
    cudaFree(q.d_units);
    return fail(HOBO_ECUDA, "stream-K plan allocation");
  }
  t->sk_plans.push_back(q);   // freed with the handle
  CK(cudaMemcpyAsync(q.d_units, units.data(), units.size() * sizeof(int4), cudaMemcpyHostToDevice, s));
  CK(cudaMemcpyAsync(q.d_sktiles, sktiles.data(), sktiles.size() * sizeof(int4), cudaMemcpyHostToDevice, s));
  use = &t->sk_plans.back();
  return HOBO_OK;
}

hobo_status contract(hobo_tensor* t, int field, const uint8_t* X, long long B, float* G, cudaStream_t s,
                     const uint16_t* P = nullptr, bool packed = false, int* slot_used = nullptr) {
  const int pk = (!P && !field) ? use_persist(t, B) : 0;
  const bool persist = pk != 0;
  const int slot = P ? real_slot(t) : pk == 2 ? 5 : pk == 1 ? 4 : field;
  if (slot_used) *slot_used = slot;
  if (hobo_status st = ensure_layout(t, slot)) return st;
  const DevLayout& L = t->lay[slot];
  if (hobo_status st = grow(t, t->d_Q, t->Q_cap, (size_t)B * L.n_ct)) return st;
  if (!P) {
    if (hobo_status st = grow(t, t->d_bits, t->bits_cap, (size_t)B * t->W)) return st;
    const long long nw = B * t->W;
    if (packed)
      mask_bits_kernel<<<(unsigned)std::min<long long>((nw + 255) / 256, 148 * 16), 256, 0, s>>>(
          reinterpret_cast<const uint32_t*>(X), B, t->host.N, t->W, t->d_bits);
    else
      launch_pack_x(X, B, t->host.N, t->W, t->d_bits, s);
    CK(cudaGetLastError());
  }
  if (pk == 2) {
    int npairs = 0;
    if (hobo_status st = persist_items(t, L, B, npairs, s)) return st;
    if (t->p1_int < 0) {   // the degree-1 cells as integers on the digit grid, when they all are
      const int Npad = (t->host.N + 255) / 256 * 256;
      std::vector<int> q1(Npad, 0);
      int ok = 1;
      for (int m = 0; m < t->host.N && ok; ++m) {
        const double v = std::ldexp((double)t->host.strict[1][m], -t->host.qexp);
        if (v != std::floor(v) || std::fabs(v) >= 16777216.0) ok = 0;
        else q1[m] = (int)v;
      }
      if (ok) {
        CK(cudaMalloc(&t->d_p1q, Npad * sizeof(int)));
        CK(cudaMemcpy(t->d_p1q, q1.data(), Npad * sizeof(int), cudaMemcpyHostToDevice));
      }
      t->p1_int = ok;
    }
    PersistI8Params q;
    q.xbits = t->d_bits;
    q.runs = t->d_runs;
    q.kdesc = t->d_kdesc;
    q.sched = L.d_sched;
    q.p1 = t->d_p1;
    q.p1q = t->d_p1q;
    q.p1_int = t->p1_int;
    q.qscale = L.qscale;
    q.Q = t->d_Q;
    q.items = t->d_items;
    q.B = B;
    q.N = t->host.N;
    q.W = t->W;
    q.n_ct = L.n_ct;
    q.nseg = t->kl.nseg;
    q.P = L.i8;
    q.n_kb = (int)(std::max<int64_t>(t->kl.Tpad, 2 * kBK) / kBK);
    q.exp = 0;
    if (const char* e = getenv("HOBO_PERSIST_EXP")) q.exp = atoi(e);
    if (t->profile) CK(record_event(t->ev0, s));
    if (L.NT == 64) CK(launch_persist(kr_persist_i8_kernel<64>, PersistI8Cfg<64>::smem_bytes(q.W), L, q, npairs, s));
    else CK(launch_persist(kr_persist_i8_kernel<128>, PersistI8Cfg<128>::smem_bytes(q.W), L, q, npairs, s));
    if (t->profile) { CK(record_event(t->ev1, s)); t->ev_valid = true; }
    t->last_launches = 2;
    t->last_mma_macs = exec_macs(t, L, B);
    t->last_i8 = L.f8 ? -L.i8 : L.i8;
    t->last_algo_macs = algo_macs(t, false, B);
    return HOBO_OK;
  }
  if (persist) {
    int npairs = 0;
    if (hobo_status st = persist_items(t, L, B, npairs, s)) return st;
    PersistParams q;
    q.xbits = t->d_bits;
    q.runs = t->d_runs;
    q.kdesc = t->d_kdesc;
    q.sched = L.d_sched;
    q.p1 = t->d_p1;
    q.Q = t->d_Q;
    q.items = t->d_items;
    q.B = B;
    q.N = t->host.N;
    q.W = t->W;
    q.n_ct = L.n_ct;
    q.n_cbp = (int)((B + 2 * kBM - 1) / (2 * kBM));
    q.nseg = t->kl.nseg;
    q.L = t->host.limbs;
    q.n_kb = (int)(std::max<int64_t>(t->kl.Tpad, 2 * kBK) / kBK);
    q.exp = 0;
    if (const char* e = getenv("HOBO_PERSIST_EXP")) q.exp = atoi(e);
    if (t->profile) CK(record_event(t->ev0, s));
    const char* ek = getenv("HOBO_PERSIST_KPS");   // A/B of the stage size
    if (ek && ek[0] == '2') CK(launch_persist(kr_persist_kernel<2>, PersistCfgT<2>::smem_bytes(q.W), L, q, npairs, s));
    else CK(launch_persist(kr_persist_kernel<1>, PersistCfgT<1>::smem_bytes(q.W), L, q, npairs, s));
    if (t->profile) { CK(record_event(t->ev1, s)); t->ev_valid = true; }
    t->last_launches = 2;
    t->last_mma_macs = exec_macs(t, L, B);
    t->last_i8 = 0;
    t->last_algo_macs = algo_macs(t, false, B);
    return HOBO_OK;
  }
  KrParams p = make_params(t, L, t->d_bits, B, G, t->d_Q);
  if (P) {
    if (!real_geometry(t, L.NT, p.pstride, p.ring_boxes, p.LA))
      return fail(HOBO_EINVAL, "real-valued path: N=" + std::to_string(t->host.N) + " with " +
                                   std::to_string(t->host.limbs) + " limbs does not fit shared memory (N <= 512 at L=1)");
    p.preal = P;
  }
  p.n_split = choose_split(t, L, B);
  // energy-mode bf16 launches on single CTAs (short K loops, e.g. cfg2): each CTA loops over
  // cb_iters candidate blocks (HOBO_CB_ITERS overrides)
  if (!P && !field && !L.i8 && p.n_split == 1 && !use_pairs(L, p)) {
    // two blocks per CTA when that still leaves >= 4 waves (cfg2: 195 -> 199 M cand/s; 3-4
    // blocks lose more to the coarser tail than they save)
    p.cb_iters = (long long)L.n_ct * ((p.n_cb + 1) / 2) >= 4 * 148 ? 2 : 1;
    if (const char* e = getenv("HOBO_CB_ITERS")) p.cb_iters = std::max(1, atoi(e));
  }
  const hobo_tensor::SkPlan* sk = nullptr;
  if (field && !P && (!L.i8 || L.f8) && use_pairs(L, p) && slot == 1)
    if (hobo_status st = sk_plan(t, L, p, B, sk, s)) return st;
  if (sk) {
    p.n_split = 1;
    p.units = sk->d_units;
    p.n_units = sk->nunits;
    p.skG = t->d_skG;
    p.skQ = t->d_skQ;
  }
  if (p.n_split > 1) {
    if (field) {
      if (hobo_status st = grow(t, t->d_Gpart, t->Gpart_cap, (size_t)p.n_split * B * t->host.N * (L.i8 && !L.f8 ? 2 : 1)))
        return st;
      p.G = t->d_Gpart;
    }
    if (hobo_status st = grow(t, t->d_Qpart, t->Qpart_cap, (size_t)p.n_split * L.n_ct * B)) return st;
    p.Q = t->d_Qpart;
  }
  if (t->profile) CK(record_event(t->ev0, s));
  CK(launch_kr_any(L, p, s));
  if (t->profile) { CK(record_event(t->ev1, s)); t->ev_valid = true; }
  if (sk) {
    const long long n = (long long)sk->ntiles * 2 * kBM * (L.NT / 4);
    sk_reduce_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 8), 256, 0, s>>>(
        sk->d_sktiles, sk->ntiles, t->d_skG, t->d_skQ, G, t->d_Q, B, t->host.N, L.NT, 1);
    CK(cudaGetLastError());
  }
  t->last_launches = (P ? 1 : 2) + (sk ? 1 : 0);
  if (p.n_split > 1) {
    const long long nG = field ? B * t->host.N : 0, nQ = (long long)L.n_ct * B;
    splitk_reduce_kernel<<<(unsigned)std::min<long long>((std::max(nG, nQ) + 255) / 256, 148 * 8), 256, 0, s>>>(
        t->d_Gpart, G, nG, t->d_Qpart, t->d_Q, nQ, p.n_split, L.i8 && !L.f8 ? 1 : 0);
    CK(cudaGetLastError());
    t->last_launches += 1;
  }
  t->last_mma_macs = exec_macs(t, L, B) * p.LA;
  t->last_i8 = L.f8 ? -L.i8 : L.i8;
  t->last_algo_macs = algo_macs(t, field != 0, B);
  return HOBO_OK;
}

}  // namespace

extern "C" {

const char* hobo_last_error(void) { return g_err.c_str(); }

hobo_status hobo_tensor_build(int order, int N, const hobo_term* terms, size_t nterms, const hobo_factor* facs,
                              const hobo_lin* lins, hobo_tensor** out, double* offset_out) {
  if (!out) return fail(HOBO_EINVAL, "null output handle");
  std::unique_ptr<hobo_tensor> t(new hobo_tensor());
  std::string msg;
  TermView tv{terms, nterms, facs, lins};
  int st = compile_terms(order, N, tv, t->host, msg);
  if (st) return fail(st == 3 ? HOBO_ENOMEM : (hobo_status)st, msg);
  if (offset_out) *offset_out = t->host.offset;
  *out = t.release();
  return HOBO_OK;
}

hobo_status hobo_tensor_import_cells(int order, int N, int64_t ncells, const int32_t* idx, const float* val,
                                     hobo_tensor** out) {
  if (!out) return fail(HOBO_EINVAL, "null output handle");
  std::unique_ptr<hobo_tensor> t(new hobo_tensor());
  std::string msg;
  int st = compile_cells(order, N, ncells, idx, val, t->host, msg);
  if (st) return fail(st == 3 ? HOBO_ENOMEM : (hobo_status)st, msg);
  *out = t.release();
  return HOBO_OK;
}

hobo_status hobo_tensor_import_dense(int order, int N, const float* dense, hobo_tensor** out) {
  if (!out || !dense) return fail(HOBO_EINVAL, "null argument");
  if (order < 1 || order > 6 || N < 1) return fail(HOBO_EINVAL, "order must be in 1..6 and N >= 1");
  const double cells = std::pow((double)N, order);
  if (cells > (double)(1u << 28)) return fail(HOBO_ENOMEM, "dense import limited to N^order <= 2^28 cells");
  // every nonzero cell (row-major, last index fastest) goes to the canonical cell of its index SET
  std::vector<int32_t> idx;
  std::vector<float> val;
  std::vector<int32_t> ix(order, 0);
  for (int64_t lin = 0; lin < (int64_t)cells; ++lin) {
    if (dense[lin] != 0.0f) {
      idx.insert(idx.end(), ix.begin(), ix.end());
      val.push_back(dense[lin]);
    }
    for (int p = order - 1; p >= 0; --p) {   // odometer increment of the index tuple
      if (++ix[p] < N) break;
      ix[p] = 0;
    }
  }
  return hobo_tensor_import_cells(order, N, (int64_t)val.size(), idx.data(), val.data(), out);
}

hobo_status hobo_tensor_import_colex(int order, int N, const float* const* cells_by_degree, hobo_tensor** out) {
  if (!out) return fail(HOBO_EINVAL, "null output handle");
  std::unique_ptr<hobo_tensor> t(new hobo_tensor());
  std::string msg;
  int st = compile_colex(order, N, cells_by_degree, t->host, msg);
  if (st) return fail(st == 3 ? HOBO_ENOMEM : (hobo_status)st, msg);
  *out = t.release();
  return HOBO_OK;
}

hobo_status hobo_tensor_free(hobo_tensor* t) {
  if (!t) return HOBO_OK;
  if (t->dev_init) cudaSetDevice(t->device);
  if (t->sa_borrowed) {   // annealing site tensor: owns only its W planes and degree-1 cells
    for (auto& L : t->lay)
      if (L.W) cudaFree(L.W);
    if (t->d_p1) cudaFree(t->d_p1);
    delete t;
    return HOBO_OK;
  }
  void* sa_tabs[] = {t->d_sa_runs, t->d_sa_kdesc, t->d_sa_runoff, t->d_sa_sched, t->d_sa_W, t->d_sa_L, t->d_sa_base, t->d_sa_T};
  for (void* p : sa_tabs)
    if (p) cudaFree(p);
  for (auto& L : t->lay) {
    if (L.W) cudaFree(L.W);
    if (L.d_sched) cudaFree(L.d_sched);
    if (L.d_nltab) cudaFree(L.d_nltab);
  }
  if (t->ev0) { cudaEventDestroy(t->ev0); cudaEventDestroy(t->ev1); }
  for (hobo_tensor* c : t->sa_child) hobo_tensor_free(c);
  if (t->cs) {
    cudaStreamDestroy(t->cs);
    cudaStreamDestroy(t->cs_out);
    cudaEventDestroy(t->ev_in);
    for (int i = 0; i < 2; ++i) {
      cudaEventDestroy(t->ev_copied[i]);
      cudaEventDestroy(t->ev_free[i]);
      cudaEventDestroy(t->ev_gdone[i]);
      cudaEventDestroy(t->ev_gfree[i]);
    }
  }
  for (int i = 0; i < 2; ++i)
    if (t->d_xh[i]) cudaFree(t->d_xh[i]);
  if (t->d_Eh) cudaFree(t->d_Eh);
  if (t->d_xbc) cudaFree(t->d_xbc);
  if (t->d_sa_s) cudaFree(t->d_sa_s);
  if (t->d_sa_E) cudaFree(t->d_sa_E);
  if (t->d_srec) cudaFree(t->d_srec);
  if (t->d_items) cudaFree(t->d_items);
  for (const auto& q : t->sk_plans) {
    cudaFree(q.d_units);
    cudaFree(q.d_sktiles);
  }
  for (void* q : {(void*)t->d_skG, (void*)t->d_skQ})
    if (q) cudaFree(q);
  if (t->d_p1q) cudaFree(t->d_p1q);
  if (t->d_sargs) cudaFree(t->d_sargs);
  if (t->h_key) cudaFreeHost(t->h_key);
  if (t->search_exec) cudaGraphExecDestroy(t->search_exec);
  for (auto& e : t->call_exec)
    if (e) cudaGraphExecDestroy(e);
  if (t->gs) cudaStreamDestroy(t->gs);
  void* ptrs[] = {t->d_tt, t->d_tt_meta, t->d_theta, t->d_P, t->d_k1, t->d_k2, t->d_flag, t->d_starts, t->d_Gpart, t->d_Qpart, t->d_runs, t->d_kdesc, t->d_runoff, t->d_p1, t->d_bits, t->d_Q, t->d_key, t->d_G, t->d_xbest, t->d_ebest};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  delete t;
  return HOBO_OK;
}

hobo_status hobo_tensor_digits(const hobo_tensor* t, int* digits, int* qexp) {
  if (!t || !digits || !qexp) return fail(HOBO_EINVAL, "null argument");
  *digits = t->host.digits;
  *qexp = t->host.qexp;
  return HOBO_OK;
}

hobo_status hobo_tensor_info(const hobo_tensor* t, int* order, int* N, int64_t* ncells, int* is_integer,
                             double* sum_abs, int* limbs, double* offset) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (order) *order = t->host.order;
  if (N) *N = t->host.N;
  if (ncells) *ncells = t->host.nnz;
  if (is_integer) *is_integer = t->host.is_integer ? 1 : 0;
  if (sum_abs) *sum_abs = t->host.sum_abs;
  if (limbs) *limbs = t->host.limbs;
  if (offset) *offset = t->host.offset;
  return HOBO_OK;
}

hobo_status hobo_tensor_export_cells(const hobo_tensor* t, int32_t* idx, float* val) {
  if (!t || !idx || !val) return fail(HOBO_EINVAL, "null argument");
  export_cells(t->host, idx, val);
  return HOBO_OK;
}

hobo_status hobo_tensor_export_dense(const hobo_tensor* t, float* host_out) {
  if (!t || !host_out) return fail(HOBO_EINVAL, "null argument");
  if (export_dense(t->host, host_out)) return fail(HOBO_ENOMEM, "dense export limited to N^order <= 2^28 cells");
  return HOBO_OK;
}

}  // extern "C"

namespace {
// the device part of an energy (field = 0) or field (field = 1) call: stage X, contraction,
// split-K reduce, argmin; the multi-GPU combine and the readback follow in finish_best
hobo_status enqueue_call(hobo_tensor* t, int field, const uint8_t* X, bool packed, int64_t B, int64_t row0, float* G,
                         float* E, bool best, cudaStream_t s) {
  int slot = field;
  if (hobo_status st = contract(t, field, X, B, G, s, nullptr, packed, &slot)) return st;
  if (E || best) {
    const DevLayout& L = t->lay[slot];
    if (best) CK(cudaMemsetAsync(t->d_key, 0xFF, 2 * sizeof(unsigned long long), s));
    finalize_kernel<<<(unsigned)std::min<long long>((B + 255) / 256, 148 * 4), 256, 0, s>>>(
        t->d_Q, L.n_ct, B, L.lcm, row0, E, best ? t->d_key : nullptr);
    CK(cudaGetLastError());
    t->last_launches += 1;
  }
  return HOBO_OK;
}

// what a captured call depends on besides its arguments: the scratch buffers it wrote and the
// kernel choices read from the environment (a change re-captures)
std::vector<uintptr_t> call_key(hobo_tensor* t, int field, const uint8_t* X, bool packed, int64_t B, int64_t row0,
                                const float* G, const float* E, bool best) {
  std::vector<uintptr_t> k = {(uintptr_t)field, (uintptr_t)packed, (uintptr_t)B, (uintptr_t)row0, (uintptr_t)X,
                              (uintptr_t)G, (uintptr_t)E, (uintptr_t)best, (uintptr_t)t->profile,
                              (uintptr_t)t->d_bits, (uintptr_t)t->d_Q, (uintptr_t)t->d_Gpart, (uintptr_t)t->d_Qpart,
                              (uintptr_t)t->d_items, (uintptr_t)t->d_key, (uintptr_t)t->items_B, (uintptr_t)t->d_skG,
                              (uintptr_t)t->d_skQ};
  for (const char* v : {"HOBO_PAIR", "HOBO_I8", "HOBO_CT_DESC", "HOBO_CB_ITERS", "HOBO_PERSIST", "HOBO_PERSIST_I8",
                        "HOBO_PERSIST_KPS", "HOBO_PERSIST_EXP", "HOBO_SK"}) {
    const char* e = getenv(v);
    k.push_back(e ? (uintptr_t)(unsigned char)e[0] + 1 : 0);
  }
  for (auto& L : t->lay) k.push_back((uintptr_t)L.W);
  return k;
}

// energy / field call: replay the captured graph when the same call repeats (HOBO_GRAPH=0:
// launch directly every time); a new call runs directly, then is captured for the next time
hobo_status run_call(hobo_tensor* t, int field, const uint8_t* X, bool packed, int64_t B, int64_t row0, float* G,
                     float* E, hobo_best* best, cudaStream_t s) {
  const char* ge = getenv("HOBO_GRAPH");
  const bool graphs = !(ge && ge[0] == '0');
  std::vector<uintptr_t> key = call_key(t, field, X, packed, B, row0, G, E, best != nullptr);
  if (graphs && t->call_exec[field] && key == t->call_key[field]) {
    CK(cudaGraphLaunch(t->call_exec[field], s));
    if (t->profile) t->ev_valid = true;
  } else {
    if (hobo_status st = enqueue_call(t, field, X, packed, B, row0, G, E, best != nullptr, s)) return st;
    key = call_key(t, field, X, packed, B, row0, G, E, best != nullptr);   // the buffers it grew
    if (graphs) {
      if (!t->gs) CK(cudaStreamCreateWithFlags(&t->gs, cudaStreamNonBlocking));
      const int64_t launches = t->last_launches;
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(t->gs, cudaStreamCaptureModeRelaxed));
      hobo_status st = enqueue_call(t, field, X, packed, B, row0, G, E, best != nullptr, t->gs);
      cudaError_t ce = cudaStreamEndCapture(t->gs, &g);
      if (st) { if (g) cudaGraphDestroy(g); return st; }
      CK(ce);
      if (t->call_exec[field]) cudaGraphExecDestroy(t->call_exec[field]);
      t->call_exec[field] = nullptr;
      cudaError_t ie = cudaGraphInstantiate(&t->call_exec[field], g, 0);
      cudaGraphDestroy(g);
      CK(ie);
      t->call_key[field] = key;
      t->last_launches = launches;
    }
  }
  if (best)
    if (hobo_status st = finish_best(t, best, s)) return st;
  return HOBO_OK;
}

hobo_status energy_impl(hobo_tensor* t, const uint8_t* X, bool packed, int64_t B, int64_t row0, float* E,
                        hobo_best* best, void* stream) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (B < 0 || (B > 0 && !X) || row0 < 0 || row0 + B > (int64_t)0xFFFFFFFF)
    return fail(HOBO_EINVAL, "bad batch (B >= 0, X non-null, row0 + B < 2^32)");
  if (hobo_status st = check_device(t)) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (B == 0) return empty_best(t, best, s);
  return run_call(t, 0, X, packed, B, row0, nullptr, E, best, s);
}

hobo_status field_impl(hobo_tensor* t, const uint8_t* X, bool packed, int64_t B, int64_t row0, float* G, float* E,
                       hobo_best* best, void* stream) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (B < 0 || (B > 0 && (!X || !G)) || row0 < 0 || row0 + B > (int64_t)0xFFFFFFFF)
    return fail(HOBO_EINVAL, "bad batch (B >= 0, X and G non-null, row0 + B < 2^32)");
  if (hobo_status st = check_device(t)) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (B == 0) return empty_best(t, best, s);
  return run_call(t, 1, X, packed, B, row0, G, E, best, s);
}
}  // namespace

extern "C" {

hobo_status hobo_energy(hobo_tensor* t, const uint8_t* X, int64_t B, int64_t row0, float* E, hobo_best* best,
                        void* stream) {
  return energy_impl(t, X, false, B, row0, E, best, stream);
}

hobo_status hobo_local_field(hobo_tensor* t, const uint8_t* X, int64_t B, int64_t row0, float* G, float* E,
                             hobo_best* best, void* stream) {
  return field_impl(t, X, false, B, row0, G, E, best, stream);
}

hobo_status hobo_energy_bits(hobo_tensor* t, const uint32_t* Xbits, int64_t B, int64_t row0, float* E,
                             hobo_best* best, void* stream) {
  return energy_impl(t, reinterpret_cast<const uint8_t*>(Xbits), true, B, row0, E, best, stream);
}

hobo_status hobo_local_field_bits(hobo_tensor* t, const uint32_t* Xbits, int64_t B, int64_t row0, float* G, float* E,
                                  hobo_best* best, void* stream) {
  return field_impl(t, reinterpret_cast<const uint8_t*>(Xbits), true, B, row0, G, E, best, stream);
}

}  // extern "C"

namespace {
// host-input path of hobo_energy_host / hobo_local_field_host (whole-wave chunks, copy streams)
hobo_status run_host(hobo_tensor* t, int field, const uint8_t* X_host, int64_t B, int64_t row0, float* G_host,
                     float* E_host, hobo_best* best, void* stream, bool packed = false) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (B < 0 || (B > 0 && !X_host) || row0 < 0 || row0 + B > (int64_t)0xFFFFFFFF)
    return fail(HOBO_EINVAL, "bad batch (B >= 0, X non-null, row0 + B < 2^32)");
  if (hobo_status st = check_device(t)) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (B == 0) return empty_best(t, best, s);
  if (hobo_status st = ensure_layout(t, field)) return st;
  const DevLayout& L = t->lay[field];
  const int N = t->host.N;
  const bool gout = field && G_host;
  const size_t row_bytes = packed ? (size_t)t->W * 4 : (size_t)N;   // one candidate's input bytes
  // chunks of whole waves of (candidate block x column tile) CTAs (CTA pairs take candidate
  // blocks two by two).  Inputs only: a one-wave first chunk (its copy is the exposed one),
  // then chunks growing 6x, each copy (PCIe, ~10-20 ns per candidate) hidden behind the
  // previous chunk's contraction (>= 60 ns per candidate).  With the fields coming back
  // (4N bytes per candidate, about as long as the contraction at N = 512), chunk i's
  // device->host copy overlaps chunk i+1's contraction, so the chunks stay two waves long and
  // the ends are short (below).
  const long long per_wave = std::max<long long>(2, 148 / L.n_ct / 2 * 2) * kBM;
  std::vector<long long> sizes;
  if (!gout) {
    for (long long off = 0, n = per_wave; off < B; off += sizes.back(), n *= 6) sizes.push_back(std::min(n, B - off));
  } else {
    // one-wave first chunk, two-wave chunks, one-wave last chunk.  The e4m3 contraction
    // (2.2 ms at cfg3) is now faster than the 128 MiB copy-out (2.35 ms at 57 GB/s, less while
    // X streams the other way), so the call is copy-bound and fewer chunks mean fewer gaps:
    // cfg3 3.25 ms; a quarter-wave head 3.34, plus a half-wave tail 3.52, plus a quarter-wave
    // tail 3.65 ms.  (While the bf16 kernel, 4.2 ms, was the longer side, half-wave ends had
    // won: 4.89 -> 4.75 ms.)  HOBO_E2E_TAIL = halvings after the last whole wave,
    // HOBO_E2E_HEAD = first chunk in quarter waves (A/B knobs, tools/e2e_chunks.sh).
    int tail = 0;
    if (const char* e = getenv("HOBO_E2E_TAIL")) tail = atoi(e);
    long long head = per_wave;
    if (const char* e = getenv("HOBO_E2E_HEAD")) head = std::max<long long>(kBM, per_wave * atoi(e) / 4 / kBM * kBM);
    std::vector<long long> ends;   // the tail, smallest last
    long long rest = B - std::min<long long>(head, B);
    for (long long w = per_wave / 2, i = 0; i < tail && rest > 2 * w && w >= kBM; ++i, w /= 2) {
      ends.push_back(w / kBM * kBM);
      rest -= ends.back();
    }
    sizes.push_back(std::min<long long>(head, B));
    while (rest > 0) {
      if (rest <= per_wave) { sizes.push_back(rest); break; }
      if (rest <= 3 * per_wave) { sizes.push_back(rest - per_wave); sizes.push_back(per_wave); break; }
      sizes.push_back(2 * per_wave);
      rest -= 2 * per_wave;
    }
    sizes.insert(sizes.end(), ends.begin(), ends.end());
  }
  const long long chunk = *std::max_element(sizes.begin(), sizes.end());
  if (!t->cs) {
    CK(cudaStreamCreateWithFlags(&t->cs, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&t->cs_out, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&t->ev_in, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      CK(cudaEventCreateWithFlags(&t->ev_copied[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&t->ev_free[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&t->ev_gdone[i], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&t->ev_gfree[i], cudaEventDisableTiming));
    }
  }
  if ((size_t)chunk * row_bytes > t->xh_cap) {
    for (int i = 0; i < 2; ++i) {
      if (t->d_xh[i]) cudaFree(t->d_xh[i]);
      t->d_xh[i] = nullptr;
    }
    t->xh_cap = 0;
    for (int i = 0; i < 2; ++i) CK(cudaMalloc(&t->d_xh[i], (size_t)chunk * row_bytes));
    t->xh_cap = (size_t)chunk * row_bytes;
  }
  if (hobo_status st = grow(t, t->d_Eh, t->Eh_cap, (size_t)B)) return st;
  // field chunks: two buffers when they go back to the host (chunk i's copy-out runs while
  // chunk i+1 is computed into the other one), else one scratch buffer
  if (field)
    if (hobo_status st = grow(t, t->d_G, t->G_cap, (size_t)chunk * N * (gout ? 2 : 1))) return st;
  if (best) CK(cudaMemsetAsync(t->d_key, 0xFF, 2 * sizeof(unsigned long long), s));
  CK(cudaEventRecord(t->ev_in, s));             // the copies follow the caller's prior work
  CK(cudaStreamWaitEvent(t->cs, t->ev_in, 0));
  if (gout) CK(cudaStreamWaitEvent(t->cs_out, t->ev_in, 0));
  int64_t launches = 0;
  for (long long off = 0, i = 0, n = 0; off < B; off += n, ++i) {
    n = sizes[(size_t)i];
    const int slot = (int)(i & 1);
    if (i >= 2) CK(cudaStreamWaitEvent(t->cs, t->ev_free[slot], 0));   // its previous chunk is packed
    CK(cudaMemcpyAsync(t->d_xh[slot], X_host + (size_t)off * row_bytes, (size_t)n * row_bytes, cudaMemcpyHostToDevice,
                       t->cs));
    CK(cudaEventRecord(t->ev_copied[slot], t->cs));
    CK(cudaStreamWaitEvent(s, t->ev_copied[slot], 0));
    float* Gc = field ? t->d_G + (gout ? (size_t)slot * chunk * N : 0) : nullptr;
    if (gout && i >= 2) CK(cudaStreamWaitEvent(s, t->ev_gfree[slot], 0));   // chunk i-2's fields are on the host
    int cslot = field;
    if (hobo_status st = contract(t, field, t->d_xh[slot], n, Gc, s, nullptr, packed, &cslot)) return st;
    CK(cudaEventRecord(t->ev_free[slot], s));
    const DevLayout& Lc = t->lay[cslot];
    finalize_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 4), 256, 0, s>>>(
        t->d_Q, Lc.n_ct, n, Lc.lcm, row0 + off, t->d_Eh + off, best ? t->d_key : nullptr);
    CK(cudaGetLastError());
    launches += t->last_launches + 1;
    if (gout) {
      CK(cudaEventRecord(t->ev_gdone[slot], s));
      CK(cudaStreamWaitEvent(t->cs_out, t->ev_gdone[slot], 0));
      CK(cudaMemcpyAsync(G_host + (size_t)off * N, Gc, (size_t)n * N * sizeof(float), cudaMemcpyDeviceToHost, t->cs_out));
      CK(cudaEventRecord(t->ev_gfree[slot], t->cs_out));
    }
  }
  // energies: one copy of the whole batch at the end (a pageable E_host would otherwise make
  // every chunk's copy synchronous and stall the next chunk's input copy)
  if (E_host) CK(cudaMemcpyAsync(E_host, t->d_Eh, (size_t)B * sizeof(float), cudaMemcpyDeviceToHost, s));
  if (gout) {   // the caller's stream is ordered after the last field copy
    CK(cudaEventRecord(t->ev_gfree[0], t->cs_out));
    CK(cudaStreamWaitEvent(s, t->ev_gfree[0], 0));
  }
  if (best) {
    if (hobo_status st = finish_best(t, best, s)) return st;
  } else {
    CK(cudaStreamSynchronize(s));
  }
  t->last_launches = launches;
  t->last_mma_macs = exec_macs(t, L, B);
  t->last_i8 = L.f8 ? -L.i8 : L.i8;
  t->last_algo_macs = algo_macs(t, field != 0, B);
  return HOBO_OK;
}

}  // namespace

extern "C" {

hobo_status hobo_energy_host(hobo_tensor* t, const uint8_t* X_host, int64_t B, int64_t row0, float* E_host,
                             hobo_best* best, void* stream) {
  return run_host(t, 0, X_host, B, row0, nullptr, E_host, best, stream);
}

hobo_status hobo_local_field_host(hobo_tensor* t, const uint8_t* X_host, int64_t B, int64_t row0, float* G_host,
                                  float* E_host, hobo_best* best, void* stream) {
  return run_host(t, 1, X_host, B, row0, G_host, E_host, best, stream);
}

hobo_status hobo_energy_host_bits(hobo_tensor* t, const uint32_t* Xbits_host, int64_t B, int64_t row0, float* E_host,
                                  hobo_best* best, void* stream) {
  return run_host(t, 0, reinterpret_cast<const uint8_t*>(Xbits_host), B, row0, nullptr, E_host, best, stream, true);
}

hobo_status hobo_local_field_host_bits(hobo_tensor* t, const uint32_t* Xbits_host, int64_t B, int64_t row0,
                                       float* G_host, float* E_host, hobo_best* best, void* stream) {
  return run_host(t, 1, reinterpret_cast<const uint8_t*>(Xbits_host), B, row0, G_host, E_host, best, stream, true);
}

}  // extern "C"

namespace {
// the search loop (reading 14): leaves each chain's best state in d_xbest / d_ebest
hobo_status run_search(hobo_tensor* t, uint64_t seed, int64_t chain0, int64_t nchains, int64_t iters, double p0,
                       double p1, cudaStream_t s, int64_t& launches) {
  if (nchains < 1 || iters < 0 || chain0 < 0 || chain0 + nchains > (int64_t)0xFFFFFFFF || !(p0 > 0) || !(p1 > 0))
    return fail(HOBO_EINVAL, "bad search arguments");
  if (hobo_status st = check_device(t)) return st;
  if (hobo_status st = ensure_layout(t, 1)) return st;
  const DevLayout& L = t->lay[1];
  const int N = t->host.N, W = t->W;
  const long long B = nchains;
  if (hobo_status st = grow(t, t->d_bits, t->bits_cap, (size_t)B * W)) return st;
  if (hobo_status st = grow(t, t->d_Q, t->Q_cap, (size_t)B * L.n_ct)) return st;
  if (hobo_status st = grow(t, t->d_G, t->G_cap, (size_t)B * N)) return st;
  if (hobo_status st = grow(t, t->d_xbest, t->xbest_cap, (size_t)B * W)) return st;
  if (hobo_status st = grow(t, t->d_ebest, t->ebest_cap, (size_t)B)) return st;
  // exploration threshold P_t = floor(2^32 p0 (p1/p0)^(t / max(1, iters-1)))
  std::vector<uint32_t> P((size_t)std::max<int64_t>(iters, 1));
  for (int64_t it = 0; it < iters; ++it) {
    const double v = std::floor(4294967296.0 * p0 * std::pow(p1 / p0, (double)it / (double)std::max<int64_t>(1, iters - 1)));
    P[(size_t)it] = (uint32_t)std::min(4294967295.0, std::max(0.0, v));
  }
  // device-side arguments: seed, chain0, then the P_t table two per word
  std::vector<unsigned long long> args(2 + ((size_t)std::max<int64_t>(iters, 1) + 1) / 2, 0ull);
  args[0] = seed;
  args[1] = (unsigned long long)chain0;
  std::memcpy(args.data() + 2, P.data(), P.size() * sizeof(uint32_t));
  if (hobo_status st = grow(t, t->d_sargs, t->sargs_cap, args.size())) return st;
  CK(cudaMemcpyAsync(t->d_sargs, args.data(), args.size() * sizeof(unsigned long long), cudaMemcpyHostToDevice, s));
  launches = 0;
  const unsigned g1 = (unsigned)std::min<long long>((B * W + 255) / 256, 148 * 16);
  KrParams p = make_params(t, L, t->d_bits, B, t->d_G, t->d_Q);   // n_split = 1: per-chain results never
  const unsigned gs = (unsigned)((B * 32 + 255) / 256);             // depend on the shard size
  auto enqueue = [&](cudaStream_t q) -> hobo_status {
    search_init_kernel<<<g1, 256, 0, q>>>(0, 0, B, N, W, t->d_bits, t->d_ebest, t->d_sargs);
    CK(cudaGetLastError());
    for (int64_t it = 0; it <= iters; ++it) {
      CK(launch_kr_any(L, p, q));
      const int move = it < iters;
      search_step_kernel<<<gs, 256, 0, q>>>(t->d_Q, L.n_ct, L.lcm, t->d_G, t->d_bits, t->d_xbest, t->d_ebest, 0, B, N,
                                            W, 0, it, 0u, move, 0, t->d_sargs);
      CK(cudaGetLastError());
    }
    return HOBO_OK;
  };
  launches = 1 + 2 * (iters + 1);
  if (t->profile) CK(cudaEventRecord(t->ev0, s));
  const char* ge = getenv("HOBO_GRAPH");
  if (ge && ge[0] == '0') {
    if (hobo_status st = enqueue(s)) return st;
  } else {
    // one graph per (chains, iterations, buffers, kernel choice); HOBO_GRAPH=0 launches directly
    const std::vector<uintptr_t> key = {(uintptr_t)B, (uintptr_t)iters, (uintptr_t)t->d_bits, (uintptr_t)t->d_G,
                                        (uintptr_t)t->d_Q, (uintptr_t)t->d_xbest, (uintptr_t)t->d_ebest,
                                        (uintptr_t)t->d_sargs, (uintptr_t)use_pairs(L, p), (uintptr_t)L.W};
    if (!t->search_exec || key != t->search_key) {
      // captured on a private stream (the caller's may be the legacy default stream, which
      // cannot capture); nothing executes during capture, the launch below orders it on s
      if (!t->gs) CK(cudaStreamCreateWithFlags(&t->gs, cudaStreamNonBlocking));
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(t->gs, cudaStreamCaptureModeRelaxed));
      hobo_status st = enqueue(t->gs);
      cudaError_t ce = cudaStreamEndCapture(t->gs, &g);
      if (st) { if (g) cudaGraphDestroy(g); return st; }
      CK(ce);
      if (t->search_exec) cudaGraphExecDestroy(t->search_exec);
      t->search_exec = nullptr;
      cudaError_t ie = cudaGraphInstantiate(&t->search_exec, g, 0);
      cudaGraphDestroy(g);
      CK(ie);
      t->search_key = key;
    }
    CK(cudaGraphLaunch(t->search_exec, s));
  }
  if (t->profile) { CK(cudaEventRecord(t->ev1, s)); t->ev_valid = true; }
  t->last_mma_macs = exec_macs(t, L, B) * (double)(iters + 1);
  t->last_i8 = L.f8 ? -L.i8 : L.i8;
  t->last_algo_macs = algo_macs(t, true, B) * (double)(iters + 1);
  return HOBO_OK;
}
}  // namespace

extern "C" {

hobo_status hobo_multilinear_field(hobo_tensor* t, const uint16_t* P, int64_t B, float* G, float* E, void* stream) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (B < 0 || (B > 0 && (!P || !G))) return fail(HOBO_EINVAL, "bad batch or null P/G");
  if (hobo_status st = check_device(t)) return st;
  cudaStream_t s = (cudaStream_t)stream;
  if (B == 0) return HOBO_OK;
  if (hobo_status st = contract(t, 1, nullptr, B, G, s, P)) return st;
  if (E) {
    const DevLayout& L = t->lay[real_slot(t)];
    finalize_kernel<<<(unsigned)std::min<long long>((B + 255) / 256, 148 * 4), 256, 0, s>>>(t->d_Q, L.n_ct, B, L.lcm, 0,
                                                                                          E, nullptr);
    CK(cudaGetLastError());
    t->last_launches += 1;
  }
  return HOBO_OK;
}

hobo_status hobo_search_shard(hobo_tensor* t, uint64_t seed, int64_t chain0, int64_t nchains, int64_t iters,
                              double p0, double p1, uint8_t* x_best_host, float* e_best_host, int64_t* best_chain,
                              void* stream) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t launches = 0;
  if (hobo_status st = run_search(t, seed, chain0, nchains, iters, p0, p1, s, launches)) return st;
  const int N = t->host.N, W = t->W;
  const long long B = nchains;
  CK(cudaMemsetAsync(t->d_key, 0xFF, 2 * sizeof(unsigned long long), s));
  search_best_kernel<<<(unsigned)std::min<long long>((B + 255) / 256, 148 * 4), 256, 0, s>>>(t->d_ebest, B, chain0,
                                                                                             t->d_key);
  CK(cudaGetLastError());
  ++launches;
  unsigned long long key[2] = {0, 0};
  CK(read_key(t, key, s));
  if (key[1] != ~0ull) return fail(HOBO_ERANGE, "a chain's energy is NaN (the argmin rejects NaN)");
  hobo_best b;
  hobo_best_from_key(key[0], &b);
  const int64_t c = b.idx;
  std::vector<uint32_t> xb(W);
  CK(cudaMemcpyAsync(xb.data(), t->d_xbest + (size_t)(c - chain0) * W, W * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (x_best_host)
    for (int m = 0; m < N; ++m) x_best_host[m] = (uint8_t)((xb[m >> 5] >> (m & 31)) & 1u);
  if (e_best_host) *e_best_host = b.e;
  if (best_chain) *best_chain = c;
  t->last_launches = launches;
  return HOBO_OK;
}

}  // extern "C"

namespace {
// ---- simulated annealing (SPEC sa_run S:447-453) ---------
// The chains' local fields G (B x N) are computed once and then kept current: flipping x_m
// changes g_j by (x_m' - x_m) d^2E/dx_m dx_j, the field of the derivative tensor P_m at j.
// One launch per visited site runs the KR-GEMM of P_m with the decision of site m fused in
// front and the G update fused behind (kr_gemm_kernel<NT, false, true>).
hobo_status ensure_sa_sites(hobo_tensor* t) {
  if (!t->sa_child.empty()) return HOBO_OK;
  const int N = t->host.N, k = t->host.order, kc = std::max(1, k - 1);
  std::string msg;
  // tables shared by all site tensors (they have the same order k-1 and N)
  KLayout kl;
  if (build_klayout(kc, N, kl, msg)) return fail(HOBO_ENOMEM, msg);
  CK(cudaMalloc(&t->d_sa_runs, std::max<size_t>(kl.runs.size() / 4, 1) * sizeof(uint4)));
  if (!kl.runs.empty()) CK(cudaMemcpy(t->d_sa_runs, kl.runs.data(), kl.runs.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&t->d_sa_kdesc, std::max<size_t>(kl.kdesc.size() / 4, 2) * sizeof(uint4)));
  if (!kl.kdesc.empty()) CK(cudaMemcpy(t->d_sa_kdesc, kl.kdesc.data(), kl.kdesc.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&t->d_sa_runoff, kl.run_off.size() * 4));
  CK(cudaMemcpy(t->d_sa_runoff, kl.run_off.data(), kl.run_off.size() * 4, cudaMemcpyHostToDevice));
  const int NT = N <= 128 ? 128 : 256, n_ct = (N + NT - 1) / NT, Npad = n_ct * NT;
  const std::vector<int32_t> sched = schedule(kl, NT, n_ct, true);
  CK(cudaMalloc(&t->d_sa_sched, sched.size() * sizeof(int32_t)));
  CK(cudaMemcpy(t->d_sa_sched, sched.data(), sched.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  const int64_t Tpad = std::max<int64_t>(kl.Tpad, kBK);
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  const double need = (double)N * t->host.limbs * Npad * (double)Tpad * 2.0;   // site limbs <= the tensor's
  if (need > 0.8 * (double)free_b)
    return fail(HOBO_ENOMEM, "annealing site layouts need " + std::to_string(need / 1e9) + " GB (N=" +
                                 std::to_string(N) + ", order=" + std::to_string(k) + ")");
  // layout-kernel inputs shared by every site: binomials, tuple list, per-degree staging
  std::vector<long long> bt((size_t)(N + 1) * 7);
  for (int n = 0; n <= N; ++n)
    for (int i = 0; i < 7; ++i) bt[(size_t)n * 7 + i] = binom(n, i);
  long long* d_bt = nullptr;
  uint16_t* d_tup = nullptr;
  float** d_strict_ptrs = nullptr;
  std::vector<float*> dstage(7, nullptr);
  auto release = [&]() {
    for (float* p : dstage)
      if (p) cudaFree(p);
    if (d_bt) cudaFree(d_bt);
    if (d_tup) cudaFree(d_tup);
    if (d_strict_ptrs) cudaFree(d_strict_ptrs);
  };
  std::vector<hobo_tensor*> kids;
  auto drop = [&](hobo_status st) {
    cudaDeviceSynchronize();
    release();
    for (hobo_tensor* c : kids) hobo_tensor_free(c);
    void** tabs[] = {(void**)&t->d_sa_runs, (void**)&t->d_sa_kdesc, (void**)&t->d_sa_runoff, (void**)&t->d_sa_sched};
    for (void** p : tabs) {
      if (*p) cudaFree(*p);
      *p = nullptr;
    }
    return st;
  };
#define CKS(call)                                                                                    \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) return drop(fail(HOBO_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_))); \
  } while (0)
  if (kl.Tpad > 0) {
    CKS(cudaMalloc(&d_bt, bt.size() * sizeof(long long)));
    CKS(cudaMemcpy(d_bt, bt.data(), bt.size() * sizeof(long long), cudaMemcpyHostToDevice));
    CKS(cudaMalloc(&d_tup, kl.tuples.size() * sizeof(uint16_t)));
    CKS(cudaMemcpy(d_tup, kl.tuples.data(), kl.tuples.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    for (int r = 2; r <= kc; ++r) CKS(cudaMalloc(&dstage[r], std::max<int64_t>(binom(N, r), 1) * sizeof(float)));
    CKS(cudaMalloc(&d_strict_ptrs, 7 * sizeof(float*)));
    CKS(cudaMemcpy(d_strict_ptrs, dstage.data(), 7 * sizeof(float*), cudaMemcpyHostToDevice));
  }
  EncodeTiledFn enc = encode_fn();
  if (!enc) return drop(fail(HOBO_ECUDA, "cuTensorMapEncodeTiled unavailable"));
  std::vector<float> zeros((size_t)N, 0.0f);
  const float* zp = zeros.data();
  for (int m = 0; m < N; ++m) {
    hobo_tensor* c = new hobo_tensor();
    kids.push_back(c);
    c->sa_borrowed = true;
    c->dig = 0;               // site tensors keep bf16 limb layouts (built below)
    // order 1: the fields never change (P_m is a constant): an all-zero order-1 tensor
    const int st = k >= 2 ? derive(t->host, m, c->host, msg) : compile_colex(1, N, &zp, c->host, msg);
    if (st) return drop(fail(st == 3 ? HOBO_ENOMEM : HOBO_EINVAL, "annealing site tensor: " + msg));
    c->device = t->device;
    c->dev_init = true;
    c->W = t->W;
    c->kl.order = kc;
    c->kl.N = N;
    c->kl.nseg = kl.nseg;
    c->kl.Tpad = kl.Tpad;
    c->d_runs = t->d_sa_runs;
    c->d_kdesc = t->d_sa_kdesc;
    c->d_runoff = t->d_sa_runoff;
    std::vector<float> p1(Npad, 0.0f);
    for (int j = 0; j < N; ++j) p1[j] = c->host.strict[1][j];
    CKS(cudaMalloc(&c->d_p1, Npad * sizeof(float)));
    CKS(cudaMemcpy(c->d_p1, p1.data(), Npad * sizeof(float), cudaMemcpyHostToDevice));
    DevLayout& L = c->lay[1];
    L.NT = NT;
    L.n_ct = n_ct;
    L.Npad = Npad;
    const size_t bytes = (size_t)c->host.limbs * Npad * Tpad * 2;
    CKS(cudaMalloc(&L.W, bytes));
    if (kl.Tpad > 0) {
      // the staging buffers are reused: the copies below queue behind the previous site's
      // layout kernel on the legacy stream
      for (int r = 2; r <= kc; ++r)
        CKS(cudaMemcpy(dstage[r], c->host.strict[r].data(), c->host.strict[r].size() * sizeof(float),
                       cudaMemcpyHostToDevice));
      LayoutParams lp;
      lp.tuples = d_tup;
      lp.strict = d_strict_ptrs;
      lp.binomT = d_bt;
      lp.Wout = L.W;
      lp.Tpad = kl.Tpad;
      lp.N = N;
      lp.Npad = Npad;
      lp.L = c->host.limbs;
      lp.field_mode = 1;
      lp.NT = NT;
      layout_kernel<<<148 * 8, 256>>>(lp);
      CKS(cudaGetLastError());
    } else {
      CKS(cudaMemset(L.W, 0, bytes));
    }
    const int64_t n_kb = Tpad / kBK;
    cuuint64_t dims[3] = {(cuuint64_t)kBK, (cuuint64_t)NT, (cuuint64_t)c->host.limbs * n_ct * n_kb};
    cuuint64_t strides[2] = {(cuuint64_t)kBK * 2, (cuuint64_t)kBK * 2 * NT};
    cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)NT, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult cr = enc(&L.tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, L.W, dims, strides, box, estr,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return drop(fail(HOBO_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr)));
    L.sched = sched;
    L.d_sched = t->d_sa_sched;
    L.built = true;
    for (size_t r = 2; r < c->host.strict.size(); ++r) std::vector<float>().swap(c->host.strict[r]);
  }
  CKS(cudaDeviceSynchronize());
#undef CKS
  release();
  t->sa_child = kids;
  return HOBO_OK;
}

// the persistent annealer's layout: for every site m, the field layout of P_m over the site
// K-blocks plus one block holding the empty tuple (W[j, {}] = c({m, j})), all sites in one
// buffer addressed by one 3-D TMA map (box = NT rows x 64 tuples)
hobo_status ensure_sa_persistent(hobo_tensor* t) {
  if (t->sa_persistent) return HOBO_OK;
  const int N = t->host.N, k = t->host.order, kc = std::max(1, k - 1);
  std::string msg;
  KLayout kl;
  if (build_klayout(kc, N, kl, msg)) return fail(HOBO_ENOMEM, msg);
  const int NT = N <= 128 ? 128 : 256, n_ct = (N + NT - 1) / NT, Npad = n_ct * NT;
  const int64_t Tp = kl.Tpad + kBK;        // + the degree-1 block
  const int nkb1 = (int)(Tp / kBK);
  if (kl.nseg > 8) return fail(HOBO_EINVAL, "annealing: too many degree segments");
  std::vector<uint16_t> tup(kl.tuples);
  tup.resize((size_t)Tp * 6, 0);
  tup[(size_t)kl.Tpad * 6] = 1;            // r = 1: the empty tuple
  // pass 1: limbs per site
  std::vector<float> zeros((size_t)N, 0.0f);
  const float* zp = zeros.data();
  auto site = [&](int m, HostTensor& c) {
    return k >= 2 ? derive(t->host, m, c, msg) : compile_colex(1, N, &zp, c, msg);
  };
  std::vector<int> Ls(N), bases(N);
  int64_t boxes = 0;
  for (int m = 0; m < N; ++m) {
    HostTensor c;
    if (int st = site(m, c)) return fail(st == 3 ? HOBO_ENOMEM : HOBO_EINVAL, "annealing site tensor: " + msg);
    Ls[m] = c.limbs;
    bases[m] = (int)boxes;
    boxes += (int64_t)c.limbs * n_ct * nkb1;
  }
  if (boxes >= (1ll << 31)) return fail(HOBO_ENOMEM, "annealing layout too large");
  const double bytes = (double)boxes * NT * kBK * 2.0;
  size_t free_b = 0, total_b = 0;
  CK(cudaMemGetInfo(&free_b, &total_b));
  if (bytes > 0.8 * (double)free_b)
    return fail(HOBO_ENOMEM, "annealing site layouts need " + std::to_string(bytes / 1e9) + " GB");
  CK(cudaMalloc(&t->d_sa_W, (size_t)bytes));
  CK(cudaMalloc(&t->d_sa_runs, std::max<size_t>(kl.runs.size() / 4, 1) * sizeof(uint4)));
  if (!kl.runs.empty()) CK(cudaMemcpy(t->d_sa_runs, kl.runs.data(), kl.runs.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&t->d_sa_kdesc, std::max<size_t>(kl.kdesc.size() / 4, 2) * sizeof(uint4)));
  if (!kl.kdesc.empty()) CK(cudaMemcpy(t->d_sa_kdesc, kl.kdesc.data(), kl.kdesc.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&t->d_sa_L, N * sizeof(int)));
  CK(cudaMemcpy(t->d_sa_L, Ls.data(), N * sizeof(int), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&t->d_sa_base, N * sizeof(int)));
  CK(cudaMemcpy(t->d_sa_base, bases.data(), N * sizeof(int), cudaMemcpyHostToDevice));
  // layout-kernel inputs shared by every site
  std::vector<long long> bt((size_t)(N + 1) * 7);
  for (int n = 0; n <= N; ++n)
    for (int i = 0; i < 7; ++i) bt[(size_t)n * 7 + i] = binom(n, i);
  long long* d_bt = nullptr;
  uint16_t* d_tup = nullptr;
  float** d_ptrs = nullptr;
  std::vector<float*> dstage(7, nullptr);
  auto release = [&]() {
    for (float* p : dstage)
      if (p) cudaFree(p);
    if (d_bt) cudaFree(d_bt);
    if (d_tup) cudaFree(d_tup);
    if (d_ptrs) cudaFree(d_ptrs);
  };
#define CKP(call)                                                                                    \
  do {                                                                                               \
    cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) {                                                                         \
      cudaDeviceSynchronize();                                                                       \
      release();                                                                                     \
      t->poisoned = true;                                                                            \
      return fail(HOBO_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));                   \
    }                                                                                                \
  } while (0)
  CKP(cudaMalloc(&d_bt, bt.size() * sizeof(long long)));
  CKP(cudaMemcpy(d_bt, bt.data(), bt.size() * sizeof(long long), cudaMemcpyHostToDevice));
  CKP(cudaMalloc(&d_tup, tup.size() * sizeof(uint16_t)));
  CKP(cudaMemcpy(d_tup, tup.data(), tup.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
  for (int r = 1; r <= kc; ++r) CKP(cudaMalloc(&dstage[r], std::max<int64_t>(binom(N, r), 1) * sizeof(float)));
  CKP(cudaMalloc(&d_ptrs, 7 * sizeof(float*)));
  CKP(cudaMemcpy(d_ptrs, dstage.data(), 7 * sizeof(float*), cudaMemcpyHostToDevice));
  for (int m = 0; m < N; ++m) {   // pass 2: lay out each site (staging reused: legacy-stream order)
    HostTensor c;
    if (int st = site(m, c)) {
      cudaDeviceSynchronize();
      release();
      return fail(st == 3 ? HOBO_ENOMEM : HOBO_EINVAL, "annealing site tensor: " + msg);
    }
    for (int r = 1; r <= kc; ++r)
      CKP(cudaMemcpy(dstage[r], c.strict[r].data(), c.strict[r].size() * sizeof(float), cudaMemcpyHostToDevice));
    LayoutParams lp;
    lp.tuples = d_tup;
    lp.strict = d_ptrs;
    lp.binomT = d_bt;
    lp.Wout = t->d_sa_W + (size_t)bases[m] * NT * kBK;
    lp.Tpad = Tp;
    lp.N = N;
    lp.Npad = Npad;
    lp.L = Ls[m];
    lp.field_mode = 1;
    lp.NT = NT;
    layout_kernel<<<148 * 4, 256>>>(lp);
    CKP(cudaGetLastError());
  }
  CKP(cudaDeviceSynchronize());
#undef CKP
  release();
  EncodeTiledFn enc = encode_fn();
  if (!enc) return fail(HOBO_ECUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[3] = {(cuuint64_t)kBK, (cuuint64_t)NT, (cuuint64_t)boxes};
  cuuint64_t strides[2] = {(cuuint64_t)kBK * 2, (cuuint64_t)kBK * 2 * NT};
  cuuint32_t box[3] = {(cuuint32_t)kBK, (cuuint32_t)NT, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult cr = enc(&t->sa_tmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, t->d_sa_W, dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(HOBO_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
  cuuint32_t box2[3] = {(cuuint32_t)kBK, (cuuint32_t)(NT / 2), 1};
  cr = enc(&t->sa_tmap2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, t->d_sa_W, dims, strides, box2, estr,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (cr != CUDA_SUCCESS) return fail(HOBO_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string((int)cr));
  t->sa_NT = NT;
  t->sa_nct = n_ct;
  t->sa_nkb1 = nkb1;
  t->sa_nseg = kl.nseg;
  int nq = 1;
  for (int j = 0; j < kl.nseg; ++j) {
    t->sa_seg_kb0[j] = (int)(kl.seg_t0[j] / kBK);
    t->sa_seg_cnt[j] = (int)((kl.seg_len[j] + kBK - 1) / kBK);
    nq += t->sa_seg_cnt[j];
  }
  t->sa_nq = nq;
  t->sa_L = Ls;
  t->sa_persistent = true;
  return HOBO_OK;
}

bool sa_fits_persistent(int N) {
  const int NT = N <= 128 ? 128 : 256;
  return ((N + NT - 1) / NT) * NT <= 512;
}

hobo_status ensure_sa(hobo_tensor* t) {
  return sa_fits_persistent(t->host.N) ? ensure_sa_persistent(t) : ensure_sa_sites(t);
}

template <int NT>
cudaError_t launch_sa(const CUtensorMap& tmap, const SaParams& p, unsigned grid, cudaStream_t s) {
  auto* k = sa_kernel<NT>;
  const size_t smem = SaCfg<NT>::smem_bytes(p.W);
  if (cudaError_t e = set_smem(k, smem)) return e;
  k<<<grid, kThreads, smem, s>>>(tmap, p);
  return cudaGetLastError();
}

template <int NT>
cudaError_t launch_sa_stage(const CUtensorMap& tmap, const SaParams& p, int SB, unsigned grid, cudaStream_t s) {
  auto* k = sa_stage_kernel<NT>;
  const size_t smem = SaStCfg<NT>::smem_bytes(SB, p.W);
  if (cudaError_t e = set_smem(k, smem)) return e;
  k<<<grid, kThreads, smem, s>>>(tmap, p, SB, SaStCfg<NT>::nst(SB));
  return cudaGetLastError();
}

template <int NT>
cudaError_t launch_sa2(const CUtensorMap& tmap, const SaParams& p, unsigned grid, cudaStream_t s) {
  auto* k = sa2_kernel<NT>;
  const size_t smem = Sa2Cfg<NT>::smem_bytes(p.W);
  if (cudaError_t e = set_smem(k, smem)) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, tmap, p);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

hobo_status run_sa(hobo_tensor* t, uint64_t seed, int64_t chain0, int64_t nchains, int64_t sweeps, double t_start,
                   double t_end, cudaStream_t s, int64_t& launches) {
  if (nchains < 1 || sweeps < 0 || chain0 < 0 || chain0 + nchains > (int64_t)0xFFFFFFFF)
    return fail(HOBO_EINVAL, "bad annealing batch (nchains >= 1, sweeps >= 0, chain0 + nchains < 2^32)");
  if (!(t_start > 0) || !(t_end > 0) || !(t_end <= t_start) || !std::isfinite(t_start))
    return fail(HOBO_EINVAL, "annealing schedule needs 0 < t_end <= t_start < inf");
  if (hobo_status st = check_device(t)) return st;
  if (hobo_status st = ensure_layout(t, 1)) return st;
  if (hobo_status st = ensure_sa(t)) return st;
  const DevLayout& L = t->lay[1];
  const int N = t->host.N, W = t->W;
  const long long B = nchains;
  if (hobo_status st = grow(t, t->d_bits, t->bits_cap, (size_t)B * W)) return st;
  if (hobo_status st = grow(t, t->d_Q, t->Q_cap, (size_t)B * L.n_ct)) return st;
  if (hobo_status st = grow(t, t->d_G, t->G_cap, (size_t)B * N)) return st;
  if (hobo_status st = grow(t, t->d_ebest, t->ebest_cap, (size_t)B)) return st;
  if (hobo_status st = grow(t, t->d_sa_s, t->sa_s_cap, (size_t)2 * B)) return st;
  if (hobo_status st = grow(t, t->d_sa_E, t->sa_E_cap, (size_t)B)) return st;
  launches = 0;
  const unsigned g1 = (unsigned)std::min<long long>((B * W + 255) / 256, 148 * 16);
  search_init_kernel<<<g1, 256, 0, s>>>(seed, chain0, B, N, W, t->d_bits, t->d_ebest);
  CK(cudaGetLastError());
  KrParams p0 = make_params(t, L, t->d_bits, B, t->d_G, t->d_Q);   // the initial fields and energies
  CK(launch_kr_any(L, p0, s));
  const unsigned gb = (unsigned)std::min<long long>((B + 255) / 256, 148 * 8);
  sa_e_init_kernel<<<gb, 256, 0, s>>>(t->d_Q, L.n_ct, B, L.lcm, t->d_sa_E);
  CK(cudaGetLastError());
  launches += 3;
  // geometric schedule T_s = t_start (t_end / t_start)^(s / max(1, sweeps - 1))
  std::vector<double> T((size_t)std::max<int64_t>(sweeps, 1));
  for (int64_t sw = 0; sw < sweeps; ++sw)
    T[(size_t)sw] = t_start * std::pow(t_end / t_start, (double)sw / (double)std::max<int64_t>(1, sweeps - 1));
  if (t->sa_persistent) {
    if (sweeps == 0) return HOBO_OK;
    if (hobo_status st = grow(t, t->d_sa_T, t->sa_T_cap, (size_t)sweeps)) return st;
    CK(cudaMemcpyAsync(t->d_sa_T, T.data(), (size_t)sweeps * sizeof(double), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));   // T is a pageable host vector
    SaParams q;
    q.bits = t->d_bits;
    q.G0 = t->d_G;
    q.E = t->d_sa_E;
    q.runs = t->d_sa_runs;
    q.kdesc = t->d_sa_kdesc;
    q.site_L = t->d_sa_L;
    q.site_base = t->d_sa_base;
    q.temps = t->d_sa_T;
    q.seed = seed;
    q.chain0 = chain0;
    q.B = B;
    q.steps = sweeps * (long long)N;
    q.N = N;
    q.W = W;
    q.n_ct = t->sa_nct;
    q.nkb1 = t->sa_nkb1;
    q.nseg = t->sa_nseg;
    q.nq = t->sa_nq;
    for (int j = 0; j < 8; ++j) { q.seg_kb0[j] = t->sa_seg_kb0[j]; q.seg_cnt[j] = t->sa_seg_cnt[j]; }
    const long long n_cb = (B + kBM - 1) / kBM;
    if (t->profile) CK(cudaEventRecord(t->ev0, s));
    const unsigned grid = (unsigned)std::min<long long>(n_cb, 148);
    // one column tile (Npad <= 256): the staged kernel (one barrier pair per K-block); two
    // tiles: CTA pairs sharing every W box (the box ring is the single-block fallback).
    int Lmax = 1;
    for (int l : t->sa_L) Lmax = std::max(Lmax, l);
    const int SB = Lmax * t->sa_nct;
    char kind = t->sa_nct == 1 ? 's' : 'p';   // two 256-column tiles: CTA pairs (cfg3 15.3 -> 13.3 ms)
    if ((t->sa_NT == 128 ? SaStCfg<128>::nst(SB) : SaStCfg<256>::nst(SB)) < 2) kind = 'r';
    if (const char* e = getenv("HOBO_SA_KERNEL")) kind = e[0];   // kernel override (tests run each): ring|stage|pair
    if (kind == 's')
      CK((t->sa_NT == 128 ? launch_sa_stage<128>(t->sa_tmap, q, SB, grid, s)
                          : launch_sa_stage<256>(t->sa_tmap, q, SB, grid, s)));
    else if (kind == 'p' && n_cb >= 2) {
      const unsigned g2 = (unsigned)(2 * std::min<long long>((n_cb + 1) / 2, 74));
      CK(t->sa_NT == 128 ? launch_sa2<128>(t->sa_tmap2, q, g2, s) : launch_sa2<256>(t->sa_tmap2, q, g2, s));
    } else
      CK(t->sa_NT == 128 ? launch_sa<128>(t->sa_tmap, q, grid, s) : launch_sa<256>(t->sa_tmap, q, grid, s));
    if (t->profile) { CK(cudaEventRecord(t->ev1, s)); t->ev_valid = true; }
    launches += 1;
    double per_sweep = 0;
    for (int m = 0; m < N; ++m) per_sweep += (double)t->sa_L[m] * t->sa_nq * t->sa_nct * t->sa_NT * kBK * kBM;
    t->last_mma_macs = per_sweep * (double)n_cb * (double)sweeps;
    t->last_i8 = 0;
    t->last_algo_macs = 0;   // site tensors are not kept on the host in this layout
    return HOBO_OK;
  }
  double macs = 0;
  if (t->profile) CK(cudaEventRecord(t->ev0, s));
  int64_t step = 0;
  for (int64_t sw = 0; sw < sweeps; ++sw) {
    for (int m = 0; m < N; ++m, ++step) {
      hobo_tensor* c = t->sa_child[m];
      const DevLayout& Lc = c->lay[1];
      KrParams p = make_params(c, Lc, t->d_bits, B, t->d_G, nullptr);
      p.sa_bits = t->d_bits;
      p.sa_sprev = step > 0 ? t->d_sa_s + (size_t)((step - 1) & 1) * B : nullptr;
      p.sa_scur = t->d_sa_s + (size_t)(step & 1) * B;
      p.sa_E = t->d_sa_E;
      p.sa_T = T[(size_t)sw];
      p.sa_seed = seed;
      p.sa_chain0 = chain0;
      p.sa_step = step;
      p.sa_m = m;
      p.sa_prev = step > 0 ? (m + N - 1) % N : -1;
      CK(Lc.NT == 128 ? launch_kr_sa<128>(Lc, p, s) : launch_kr_sa<256>(Lc, p, s));
      if (sw == 0) macs += exec_macs(c, Lc, B);
    }
  }
  if (step > 0) {
    sa_flush_kernel<<<gb, 256, 0, s>>>(t->d_bits, t->d_sa_s + (size_t)((step - 1) & 1) * B, N - 1, B, W);
    CK(cudaGetLastError());
    ++launches;
  }
  if (t->profile) { CK(cudaEventRecord(t->ev1, s)); t->ev_valid = true; }
  launches += step;
  t->last_i8 = 0;
  t->last_mma_macs = macs * (double)sweeps;   // upper bound: blocks whose chains all reject skip the MMA
  t->last_algo_macs = 0;
  for (int m = 0; m < N; ++m) t->last_algo_macs += algo_macs(t->sa_child[m], true, B);
  t->last_algo_macs *= (double)sweeps;
  return HOBO_OK;
}

// fresh energies of the chains' current bits (field layout + finalize) into E (float)
hobo_status sa_energies(hobo_tensor* t, long long B, float* E, cudaStream_t s, int64_t& launches) {
  const DevLayout& L = t->lay[1];
  KrParams p = make_params(t, L, t->d_bits, B, t->d_G, t->d_Q);
  CK(launch_kr_any(L, p, s));
  finalize_kernel<<<(unsigned)std::min<long long>((B + 255) / 256, 148 * 4), 256, 0, s>>>(t->d_Q, L.n_ct, B, L.lcm, 0,
                                                                                        E, nullptr);
  CK(cudaGetLastError());
  launches += 2;
  return HOBO_OK;
}

// dedupe the chains' best states (d_xbest / d_ebest), count occurrences, return the top-k in
// the paper's listing order (energy ascending, occurrence descending, assignment lexicographic)
hobo_status aggregate_best(hobo_tensor* t, int64_t batch, int64_t topk, uint8_t* x_host, float* e_host,
                           int64_t* count_host, int64_t* n_out, cudaStream_t s, int64_t& launches) {
  const int N = t->host.N, W = t->W;
  const long long B = batch;
  long long n = 2048;
  while (n < B) n <<= 1;
  if (hobo_status st = grow(t, t->d_k1, t->k_cap, (size_t)n)) return st;
  if (hobo_status st = grow(t, t->d_k2, t->k2_cap, (size_t)n)) return st;
  if (hobo_status st = grow(t, t->d_flag, t->flag_cap, (size_t)B + 1)) return st;
  if (hobo_status st = grow(t, t->d_starts, t->starts_cap, (size_t)B + 1)) return st;
  const unsigned gb = (unsigned)std::min<long long>((n + 255) / 256, 148 * 16);
  agg_key_kernel<<<gb, 256, 0, s>>>(t->d_ebest, t->d_xbest, B, W, n, t->d_k1, t->d_k2);
  CK(cudaGetLastError());
  ++launches;
  for (long long k = 2; k <= n; k <<= 1) {   // bitonic sort of (k1, k2), ascending
    for (long long j = k >> 1; j >= 2048; j >>= 1) {
      bitonic_global_kernel<<<gb, 256, 0, s>>>(t->d_k1, t->d_k2, n, j, k);
      ++launches;
    }
    bitonic_shared_kernel<<<(unsigned)(n / 2048), 1024, 0, s>>>(t->d_k1, t->d_k2, k);
    ++launches;
  }
  CK(cudaGetLastError());
  agg_flag_kernel<<<(unsigned)std::min<long long>((B + 255) / 256, 148 * 16), 256, 0, s>>>(t->d_k1, t->d_k2, t->d_xbest,
                                                                                          B, W, t->d_flag);
  agg_scan_kernel<<<1, 1024, 0, s>>>(t->d_flag, B, t->d_starts, t->d_flag + B);
  CK(cudaGetLastError());
  launches += 2;
  uint32_t ng = 0;
  CK(cudaMemcpyAsync(&ng, t->d_flag + B, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // host: take leading groups (E ascending) until every group tied with the k-th is included
  struct Grp { float e; int64_t count; uint32_t chain; std::vector<uint8_t> x; };
  std::vector<Grp> gs;
  std::vector<uint32_t> starts;
  int64_t G = std::min<int64_t>(ng, std::max<int64_t>(4 * topk, 64));
  for (;;) {
    starts.resize((size_t)G + 1);
    CK(cudaMemcpyAsync(starts.data(), t->d_starts, (size_t)G * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    starts[(size_t)G] = G < (int64_t)ng ? 0u : (uint32_t)B;
    if (G < (int64_t)ng) CK(cudaMemcpy(&starts[(size_t)G], t->d_starts + G, 4, cudaMemcpyDeviceToHost));
    std::vector<unsigned long long> k1(G), k2(G);
    for (int64_t g = 0; g < G; ++g) {
      CK(cudaMemcpyAsync(&k1[g], t->d_k1 + starts[g], 8, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(&k2[g], t->d_k2 + starts[g], 8, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    const int64_t kth = std::min<int64_t>(topk, G) - 1;
    const bool need_more = G < (int64_t)ng && (k1[G - 1] >> 32) == (k1[kth] >> 32);
    if (need_more) { G = std::min<int64_t>(ng, 2 * G); continue; }
    gs.clear();
    for (int64_t g = 0; g < G; ++g) {
      if ((k1[g] >> 32) > (k1[kth] >> 32)) break;
      Grp r;
      {
        hobo_best bb;
        hobo_best_from_key((k1[g] & 0xFFFFFFFF00000000ull), &bb);   // the energy half of the sort key
        r.e = bb.e;
      }
      r.count = (int64_t)starts[g + 1] - starts[g];
      r.chain = (uint32_t)(k2[g] & 0xFFFFFFFFull);
      std::vector<uint32_t> row(W);
      CK(cudaMemcpy(row.data(), t->d_xbest + (size_t)r.chain * W, W * 4, cudaMemcpyDeviceToHost));
      r.x.resize(N);
      for (int m = 0; m < N; ++m) r.x[m] = (uint8_t)((row[m >> 5] >> (m & 31)) & 1u);
      gs.push_back(std::move(r));
    }
    break;
  }
  // the paper's listing order: energy ascending, occurrence descending, assignment lexicographic
  std::sort(gs.begin(), gs.end(), [](const Grp& a, const Grp& b) {
    if (a.e != b.e) return a.e < b.e;
    if (a.count != b.count) return a.count > b.count;
    return a.x < b.x;
  });
  const int64_t nk = std::min<int64_t>(topk, (int64_t)gs.size());
  for (int64_t i = 0; i < nk; ++i) {
    std::memcpy(x_host + i * N, gs[i].x.data(), N);
    e_host[i] = gs[i].e;
    count_host[i] = gs[i].count;
  }
  *n_out = nk;
  return HOBO_OK;
}
}  // namespace

extern "C" {

hobo_status hobo_search_samples(hobo_tensor* t, uint64_t seed, int64_t batch, int64_t iters, int64_t topk,
                                uint8_t* x_host, float* e_host, int64_t* count_host, int64_t* n_out, void* stream) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (topk < 1 || !x_host || !e_host || !count_host || !n_out) return fail(HOBO_EINVAL, "bad output arguments");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t launches = 0;
  if (hobo_status st = run_search(t, seed, 0, batch, iters, 0.5, 0.005, s, launches)) return st;
  if (hobo_status st = aggregate_best(t, batch, topk, x_host, e_host, count_host, n_out, s, launches)) return st;
  t->last_launches = launches;
  return HOBO_OK;
}

hobo_status hobo_gd_run(hobo_tensor* t, uint64_t seed, int64_t shots, int64_t steps, double step_size,
                        int64_t greedy_iters, int64_t topk, uint8_t* x_host, float* e_host, int64_t* count_host,
                        int64_t* n_out, void* stream) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (shots < 1 || steps < 0 || greedy_iters < 0 || !(step_size > 0) || topk < 1 || !x_host || !e_host ||
      !count_host || !n_out || shots > (int64_t)0xFFFFFFFF)
    return fail(HOBO_EINVAL, "bad gradient-descent arguments");
  if (hobo_status st = check_device(t)) return st;
  if (hobo_status st = ensure_layout(t, 1)) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const DevLayout& L = t->lay[1];
  const int N = t->host.N, W = t->W;
  const long long B = shots;
  if (hobo_status st = grow(t, t->d_theta, t->theta_cap, (size_t)B * N)) return st;
  if (hobo_status st = grow(t, t->d_P, t->P_cap, (size_t)B * N)) return st;
  if (hobo_status st = grow(t, t->d_G, t->G_cap, (size_t)B * N)) return st;
  if (hobo_status st = grow(t, t->d_bits, t->bits_cap, (size_t)B * W)) return st;
  if (hobo_status st = grow(t, t->d_Q, t->Q_cap, (size_t)B * L.n_ct)) return st;
  if (hobo_status st = grow(t, t->d_xbest, t->xbest_cap, (size_t)B * W)) return st;
  if (hobo_status st = grow(t, t->d_ebest, t->ebest_cap, (size_t)B)) return st;
  int64_t launches = 0;
  const unsigned ge = (unsigned)std::min<long long>((B * N + 255) / 256, 148 * 16);
  gd_init_kernel<<<ge, 256, 0, s>>>(seed, B, N, t->d_theta, reinterpret_cast<__nv_bfloat16*>(t->d_P));
  CK(cudaGetLastError());
  ++launches;
  if (t->profile) CK(cudaEventRecord(t->ev0, s));
  for (int64_t it = 0; it < steps; ++it) {   // descent on the relaxation
    if (hobo_status st = contract(t, 1, nullptr, B, t->d_G, s, t->d_P)) return st;
    launches += t->last_launches;
    gd_update_kernel<<<ge, 256, 0, s>>>(B * N, (float)step_size, t->d_G, t->d_theta,
                                          reinterpret_cast<__nv_bfloat16*>(t->d_P));
    CK(cudaGetLastError());
    ++launches;
  }
  if (t->profile) { CK(cudaEventRecord(t->ev1, s)); t->ev_valid = true; }
  // round at 0.5, then steepest single-flip descent on the binary problem
  gd_round_kernel<<<(unsigned)std::min<long long>((B * W + 255) / 256, 148 * 16), 256, 0, s>>>(B, N, W, reinterpret_cast<const __nv_bfloat16*>(t->d_P), t->d_bits,
                                                                                             t->d_ebest);
  CK(cudaGetLastError());
  ++launches;
  KrParams p = make_params(t, L, t->d_bits, B, t->d_G, t->d_Q);
  const unsigned gs = (unsigned)((B * 32 + 255) / 256);
  for (int64_t it = 0; it <= greedy_iters; ++it) {
    CK(launch_kr_any(L, p, s));
    search_step_kernel<<<gs, 256, 0, s>>>(t->d_Q, L.n_ct, L.lcm, t->d_G, t->d_bits, t->d_xbest, t->d_ebest, 0, B, N, W,
                                          seed, it, 0u, it < greedy_iters ? 1 : 0, 1);
    CK(cudaGetLastError());
    launches += 2;
  }
  if (hobo_status st = aggregate_best(t, B, topk, x_host, e_host, count_host, n_out, s, launches)) return st;
  t->last_launches = launches;
  return HOBO_OK;
}

hobo_status hobo_sa_shard(hobo_tensor* t, uint64_t seed, int64_t chain0, int64_t nchains, int64_t sweeps,
                          double t_start, double t_end, uint8_t* X_out, float* E_out, double* E_tracked, void* stream) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t launches = 0;
  if (hobo_status st = run_sa(t, seed, chain0, nchains, sweeps, t_start, t_end, s, launches)) return st;
  const long long B = nchains;
  if (E_tracked) CK(cudaMemcpyAsync(E_tracked, t->d_sa_E, (size_t)B * sizeof(double), cudaMemcpyDeviceToDevice, s));
  if (X_out) {
    unpack_bits_kernel<<<(unsigned)std::min<long long>((B * t->host.N + 255) / 256, 148 * 16), 256, 0, s>>>(
        t->d_bits, B, t->host.N, t->W, X_out);
    CK(cudaGetLastError());
    ++launches;
  }
  if (E_out)
    if (hobo_status st = sa_energies(t, B, E_out, s, launches)) return st;
  t->last_launches = launches;
  return HOBO_OK;
}

hobo_status hobo_sa_run(hobo_tensor* t, uint64_t seed, int64_t shots, int64_t sweeps, double t_start, double t_end,
                        int64_t topk, uint8_t* x_host, float* e_host, int64_t* count_host, int64_t* n_out,
                        void* stream) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (topk < 1 || !x_host || !e_host || !count_host || !n_out) return fail(HOBO_EINVAL, "bad output arguments");
  cudaStream_t s = (cudaStream_t)stream;
  int64_t launches = 0;
  if (hobo_status st = run_sa(t, seed, 0, shots, sweeps, t_start, t_end, s, launches)) return st;
  const long long B = shots;
  // the sample set holds the chains' final states with freshly evaluated energies
  if (hobo_status st = grow(t, t->d_xbest, t->xbest_cap, (size_t)B * t->W)) return st;
  CK(cudaMemcpyAsync(t->d_xbest, t->d_bits, (size_t)B * t->W * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
  if (hobo_status st = sa_energies(t, B, t->d_ebest, s, launches)) return st;
  if (hobo_status st = aggregate_best(t, B, topk, x_host, e_host, count_host, n_out, s, launches)) return st;
  t->last_launches = launches;
  return HOBO_OK;
}

hobo_status hobo_tt_build(hobo_tensor* t, double rel_tol, int32_t* ranks_out) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (!(rel_tol >= 0.0) || rel_tol >= 1.0) return fail(HOBO_EINVAL, "rel_tol must be in [0, 1)");
  const double cells = std::pow((double)t->host.N, t->host.order);
  if (cells > (double)(1 << 24)) return fail(HOBO_ENOMEM, "TT build needs the dense tensor: N^order <= 2^24 cells");
  std::vector<float> dense((size_t)cells);
  if (export_dense(t->host, dense.data())) return fail(HOBO_ENOMEM, "dense export failed");
  std::vector<double> dd(dense.begin(), dense.end());
  std::string msg;
  // rel_tol below 1e-12 means "without approximation": the double SVD's round-off floor
  if (int st = tt_decompose(t->host.order, t->host.N, dd, std::max(rel_tol, 1e-12), t->tt, msg))
    return fail(st == 3 ? HOBO_ENOMEM : HOBO_EINVAL, msg);
  if (ranks_out)
    for (int p = 0; p <= t->host.order; ++p) ranks_out[p] = t->tt.ranks[p];
  if (t->d_tt) { cudaFree(t->d_tt); t->d_tt = nullptr; }   // device copy rebuilt lazily
  return HOBO_OK;
}

hobo_status hobo_tt_energy(hobo_tensor* t, const uint8_t* X, int64_t B, int64_t row0, float* E, hobo_best* best,
                           void* stream) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (t->tt.cores.empty()) return fail(HOBO_ESTATE, "call hobo_tt_build first");
  if (B < 0 || (B > 0 && (!X || !E)) || row0 < 0 || row0 + B > (int64_t)0xFFFFFFFF) return fail(HOBO_EINVAL, "bad batch");
  if (hobo_status st = check_device(t)) return st;
  const int k = t->host.order, N = t->host.N, W = t->W;
  int rmax = 1;
  for (int r : t->tt.ranks) rmax = std::max(rmax, r);
  if (rmax > 32) return fail(HOBO_EINVAL, "TT rank " + std::to_string(rmax) + " > 32: use the dense contraction");
  cudaStream_t s = (cudaStream_t)stream;
  if (!t->d_tt) {
    std::vector<double> flat;
    std::vector<int> meta;
    for (int p = 0; p < k; ++p) {
      meta.push_back((int)flat.size());
      flat.insert(flat.end(), t->tt.cores[p].begin(), t->tt.cores[p].end());
    }
    for (int r : t->tt.ranks) meta.push_back(r);
    CK(cudaMalloc(&t->d_tt, flat.size() * sizeof(double)));
    CK(cudaMemcpy(t->d_tt, flat.data(), flat.size() * sizeof(double), cudaMemcpyHostToDevice));
    if (!t->d_tt_meta) CK(cudaMalloc(&t->d_tt_meta, 16 * sizeof(int)));
    CK(cudaMemcpy(t->d_tt_meta, meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice));
  }
  if (B == 0) return empty_best(t, best, (cudaStream_t)stream);
  if (hobo_status st = grow(t, t->d_bits, t->bits_cap, (size_t)B * W)) return st;
  launch_pack_x(X, B, N, W, t->d_bits, s);
  int ncores = 0;
  for (const auto& c : t->tt.cores) ncores += (int)c.size();
  const size_t smem = (size_t)ncores * sizeof(double);
  if (t->profile) CK(cudaEventRecord(t->ev0, s));
  if (smem <= 48 * 1024 && k <= 16) {   // cores staged in shared memory, 4 (rank <= 4) or 2 candidates per thread
    const int cpt = rmax <= 4 ? 4 : 2;
    const unsigned g = (unsigned)std::min<long long>((B + 128 * cpt - 1) / (128 * cpt), 148 * 16);
    if (rmax <= 4)
      tt_energy_smem_kernel<4, 4><<<g, 128, smem, s>>>(t->d_tt, ncores, t->d_tt_meta, t->d_tt_meta + k, k, N, W, t->d_bits, B, E);
    else if (rmax <= 8)
      tt_energy_smem_kernel<8, 2><<<g, 128, smem, s>>>(t->d_tt, ncores, t->d_tt_meta, t->d_tt_meta + k, k, N, W, t->d_bits, B, E);
    else if (rmax <= 16)
      tt_energy_smem_kernel<16, 1><<<(unsigned)std::min<long long>((B + 127) / 128, 148 * 16), 128, smem, s>>>(
          t->d_tt, ncores, t->d_tt_meta, t->d_tt_meta + k, k, N, W, t->d_bits, B, E);
    else
      tt_energy_smem_kernel<32, 1><<<(unsigned)std::min<long long>((B + 127) / 128, 148 * 16), 128, smem, s>>>(
          t->d_tt, ncores, t->d_tt_meta, t->d_tt_meta + k, k, N, W, t->d_bits, B, E);
  } else {
    const unsigned g = (unsigned)std::min<long long>((B + 127) / 128, 148 * 32);
    if (rmax <= 4) tt_energy_kernel<4><<<g, 128, 0, s>>>(t->d_tt, t->d_tt_meta, t->d_tt_meta + k, k, N, W, t->d_bits, B, E);
    else if (rmax <= 16) tt_energy_kernel<16><<<g, 128, 0, s>>>(t->d_tt, t->d_tt_meta, t->d_tt_meta + k, k, N, W, t->d_bits, B, E);
    else tt_energy_kernel<32><<<g, 128, 0, s>>>(t->d_tt, t->d_tt_meta, t->d_tt_meta + k, k, N, W, t->d_bits, B, E);
  }
  if (t->profile) { CK(cudaEventRecord(t->ev1, s)); t->ev_valid = true; }
  CK(cudaGetLastError());
  t->last_launches = 2;
  if (best) {
    CK(cudaMemsetAsync(t->d_key, 0xFF, 2 * sizeof(unsigned long long), s));
    search_best_kernel<<<(unsigned)std::min<long long>((B + 255) / 256, 148 * 4), 256, 0, s>>>(E, B, row0, t->d_key);
    CK(cudaGetLastError());
    t->last_launches += 1;
    if (hobo_status st = finish_best(t, best, s)) return st;
  }
  return HOBO_OK;
}

hobo_status hobo_search(hobo_tensor* t, uint64_t seed, int64_t batch, int64_t iters, uint8_t* x_best_host,
                        float* e_best_host, void* stream) {
  if (!dist_active())
    return hobo_search_shard(t, seed, 0, batch, iters, 0.5, 0.005, x_best_host, e_best_host, nullptr, stream);
  // multi-GPU: this rank's contiguous shard of the global chains (the first ranks take the
  // remainder), C1 all-reduce(MIN) of the packed (E_best, chain) key, C2 broadcast of the
  // winner's bits from the rank that owns its chain.  Per-chain RNG streams are keyed by the
  // global chain id, so the result equals the single-GPU search.
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (batch < 1 || batch > (int64_t)0xFFFFFFFF) return fail(HOBO_EINVAL, "bad search batch");
  if (hobo_status st = check_device(t)) return st;
  cudaStream_t s = (cudaStream_t)stream;
  const int R = g_dist.rank, P = g_dist.world;
  int64_t lo = 0, n = 0;
  if (hobo_status st = hobo_shard(batch, R, P, &lo, &n)) return st;
  const int N = t->host.N, W = t->W;
  int64_t launches = 0;
  if (n > 0) {
    if (hobo_status st = run_search(t, seed, lo, n, iters, 0.5, 0.005, s, launches)) return st;
  } else if (hobo_status st = check_device(t)) {
    return st;
  }
  CK(cudaMemsetAsync(t->d_key, 0xFF, 2 * sizeof(unsigned long long), s));
  if (n > 0) {
    search_best_kernel<<<(unsigned)std::min<long long>((n + 255) / 256, 148 * 4), 256, 0, s>>>(t->d_ebest, n, lo,
                                                                                               t->d_key);
    CK(cudaGetLastError());
    ++launches;
  }
  hobo_best b;
  if (hobo_status st = finish_best(t, &b, s)) return st;   // C1 (synchronises the stream)
  const int64_t c = b.idx;
  int owner = 0;
  if (hobo_status st = hobo_shard_owner(batch, P, c, &owner)) return st;   // every rank has >= 1 chain overall
  if (hobo_status st = grow(t, t->d_xbc, t->xbc_cap, (size_t)W)) return st;
  if (R == owner)
    CK(cudaMemcpyAsync(t->d_xbc, t->d_xbest + (size_t)(c - lo) * W, (size_t)W * 4, cudaMemcpyDeviceToDevice, s));
  ncclResult_t r = g_dist.broadcast(t->d_xbc, t->d_xbc, (size_t)W * 4, ncclUint8, owner, g_dist.comm, s);   // C2
  if (r != ncclSuccess) return fail(HOBO_ENCCL, std::string("ncclBroadcast: ") + g_dist.err(r));
  std::vector<uint32_t> xb(W);
  CK(cudaMemcpyAsync(xb.data(), t->d_xbc, (size_t)W * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (x_best_host)
    for (int m = 0; m < N; ++m) x_best_host[m] = (uint8_t)((xb[m >> 5] >> (m & 31)) & 1u);
  if (e_best_host) *e_best_host = b.e;
  t->last_launches = launches + 2;
  return HOBO_OK;
}

hobo_status hobo_shard(int64_t total, int rank, int world, int64_t* lo, int64_t* n) {
  if (total < 0 || world < 1 || rank < 0 || rank >= world || !lo || !n)
    return fail(HOBO_EINVAL, "hobo_shard: total >= 0, 0 <= rank < world, non-null outputs");
  auto lo_of = [&](int64_t r) { return r * (total / world) + std::min<int64_t>(r, total % world); };
  *lo = lo_of(rank);
  *n = lo_of(rank + 1) - *lo;
  return HOBO_OK;
}

hobo_status hobo_shard_owner(int64_t total, int world, int64_t index, int* owner) {
  if (world < 1 || !owner || index < 0 || index >= total)
    return fail(HOBO_EINVAL, "hobo_shard_owner: index outside [0, total) or world < 1");
  // the first total % world ranks hold base + 1 items, the rest base
  const int64_t base = total / world, rem = total % world, big = rem * (base + 1);
  *owner = (int)(index < big ? index / (base + 1) : rem + (index - big) / base);
  return HOBO_OK;
}

hobo_status hobo_best_key(float e, int64_t idx, uint64_t* key) {
  if (!key || e != e || idx < 0 || idx > (int64_t)0xFFFFFFFF)
    return fail(HOBO_EINVAL, "hobo_best_key: NaN energy or index outside [0, 2^32)");
  if (e == 0.0f) e = 0.0f;   // -0 -> +0
  int32_t i;
  std::memcpy(&i, &e, 4);
  if (i < 0) i ^= 0x7FFFFFFF;
  *key = ((uint64_t)((uint32_t)i ^ 0x80000000u) << 32) | (uint64_t)idx;
  return HOBO_OK;
}

hobo_status hobo_best_from_key(uint64_t key, hobo_best* best) {
  if (!best) return fail(HOBO_EINVAL, "null best");
  if (key == ~0ull) {
    best->e = INFINITY;
    best->idx = -1;
    return HOBO_OK;
  }
  int32_t i = (int32_t)((uint32_t)(key >> 32) ^ 0x80000000u);
  if (i < 0) i ^= 0x7FFFFFFF;
  std::memcpy(&best->e, &i, 4);
  best->idx = (int64_t)(key & 0xFFFFFFFFull);
  return HOBO_OK;
}

hobo_status hobo_dist_unique_id(void* id_out) {
  if (!id_out) return fail(HOBO_EINVAL, "null id buffer");
  std::string msg;
  if (hobo_status st = nccl_load(msg)) return fail(st, msg);
  ncclUniqueId id;
  ncclResult_t r = g_dist.get_unique_id(&id);
  if (r != ncclSuccess) return fail(HOBO_ENCCL, std::string("ncclGetUniqueId: ") + g_dist.err(r));
  std::memcpy(id_out, &id, sizeof(id));
  return HOBO_OK;
}

hobo_status hobo_dist_init(int rank, int world, const void* id, int device) {
  if (world < 1 || rank < 0 || rank >= world || !id || device < 0) return fail(HOBO_EINVAL, "bad rank / world / id / device");
  if (g_dist.comm) return fail(HOBO_ESTATE, "a communicator is already initialised (hobo_dist_finalize first)");
  std::string msg;
  if (hobo_status st = nccl_load(msg)) return fail(st, msg);
  if (cudaSetDevice(device) != cudaSuccess) return fail(HOBO_ECUDA, "cudaSetDevice failed");
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclComm_t comm = nullptr;
  ncclResult_t r = g_dist.init_rank(&comm, world, uid, rank);
  if (r != ncclSuccess) return fail(HOBO_ENCCL, std::string("ncclCommInitRank: ") + g_dist.err(r));
  g_dist.comm = comm;
  g_dist.rank = rank;
  g_dist.world = world;
  g_dist.device = device;
  return HOBO_OK;
}

hobo_status hobo_dist_finalize(void) {
  if (!g_dist.comm) return HOBO_OK;
  ncclResult_t r = g_dist.destroy(g_dist.comm);
  g_dist.comm = nullptr;
  g_dist.rank = 0;
  g_dist.world = 1;
  if (r != ncclSuccess) return fail(HOBO_ENCCL, std::string("ncclCommDestroy: ") + g_dist.err(r));
  return HOBO_OK;
}

hobo_status hobo_dist_info(int* rank, int* world) {
  if (rank) *rank = g_dist.comm ? g_dist.rank : 0;
  if (world) *world = g_dist.comm ? g_dist.world : 1;
  return HOBO_OK;
}

hobo_status hobo_last_launch_stats(hobo_tensor* t, int64_t* launches, double* mma_macs, double* algo,
                                   double* kernel_ms) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (launches) *launches = t->last_launches;
  if (mma_macs) *mma_macs = t->last_mma_macs;
  if (algo) *algo = t->last_algo_macs;
  if (kernel_ms) {
    *kernel_ms = -1.0;
    if (t->profile && t->ev_valid) {
      CK(cudaEventSynchronize(t->ev1));
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, t->ev0, t->ev1));
      *kernel_ms = ms;
    }
  }
  return HOBO_OK;
}

hobo_status hobo_last_launch_kind(const hobo_tensor* t, int* i8_planes) {
  if (!t || !i8_planes) return fail(HOBO_EINVAL, "null argument");
  *i8_planes = t->last_i8;
  return HOBO_OK;
}


hobo_status hobo_set_profiling(hobo_tensor* t, int enable) {
  if (!t) return fail(HOBO_EINVAL, "null handle");
  if (hobo_status st = check_device(t)) return st;
  if (enable && !t->ev0) {
    CK(cudaEventCreate(&t->ev0));
    CK(cudaEventCreate(&t->ev1));
  }
  t->profile = enable != 0;
  t->ev_valid = false;
  return HOBO_OK;
}

}  // extern "C"
