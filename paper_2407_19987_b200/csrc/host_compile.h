// host_compile.h — host side of hobo_tensor_build: polynomial expansion, canonical cells
// and the device-layout tables (tuple list, A-generator runs, K schedules).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace hobo {

// C(n, r) for the sizes used here (n <= 65536, r <= 6); saturates at INT64_MAX
int64_t binom(int64_t n, int r);

// The compiled problem.  strict[r][colex_rank(S)] holds the fp32 cell of every monomial S
// of degree r (1 <= r <= order); colex_rank({a1<...<ar}) = sum_i C(a_i, i).
struct HostTensor {
  int order = 0, N = 0;
  double offset = 0.0;
  std::vector<std::vector<float>> strict;  // index 0 unused
  int64_t nnz = 0;
  bool is_integer = true;
  double sum_abs = 0.0;
  int limbs = 1;
  // int8 digit planes: every cell of degree >= 2 is q * 2^qexp with q an integer of `digits`
  // two's-complement bytes (1..3); digits = 0 when no such q fits in 3 bytes
  int digits = 1, qexp = 0;
};

struct TermView {  // mirrors hobo_term / hobo_factor / hobo_lin
  const void* terms;
  size_t nterms;
  const void* facs;
  const void* lins;
};

// status: 0 ok, 1 EINVAL, 2 ERANGE, 3 ENOMEM; msg receives the reason
int compile_terms(int order, int N, const TermView& tv, HostTensor& out, std::string& msg);
int compile_cells(int order, int N, int64_t ncells, const int32_t* idx, const float* val, HostTensor& out,
                  std::string& msg);
// canonical cells given directly: by_degree[r-1][colex_rank(S)] = c(S), r = 1..order
int compile_colex(int order, int N, const float* const* by_degree, HostTensor& out, std::string& msg);
// derivative tensor P_m = dE/dx_m (order k-1): c_Pm(T) = c(T u {m}) for m not in T
int derive(const HostTensor& H, int m, HostTensor& out, std::string& msg);
void export_cells(const HostTensor& t, int32_t* idx, float* val);   // lexicographic by tuple
int export_dense(const HostTensor& t, float* out);                   // 0 ok, 3 too large

// K-dimension of the open-index contraction: segments of (r-1)-subsets (r = order..2), each
// in colex order and padded to a multiple of 2 KBLK tuples (so every segment starts at an
// even K-block: the int8 digit planes' 128-byte boxes hold K-block pairs).
constexpr int KBLK = 64;
struct KLayout {
  int order = 0, N = 0, nseg = 0;
  int64_t Tpad = 0;                   // total padded tuples (multiple of KBLK)
  std::vector<int64_t> seg_t0;        // first tuple of segment j (degree order - j)
  std::vector<int64_t> seg_len;       // C(N, r-1) real tuples
  std::vector<uint16_t> tuples;       // [Tpad][6]: r (0 = padding), then the r-1 elements
  std::vector<uint32_t> runs;         // [nruns][4] generator runs (see kernels.cuh)
  std::vector<uint32_t> run_off;      // [Tpad/KBLK + 1]
  // per K-block descriptor, directly indexed (no dependent loads): two inline runs
  // rec0, rec1; rec0.w = nfix | nruns << 3 | (index of the 3rd run in `runs`) << 10
  std::vector<uint32_t> kdesc;        // [Tpad/KBLK][8]
};
int build_klayout(int order, int N, KLayout& k, std::string& msg);

// per column tile, per segment: (first K-block, #K-blocks)
std::vector<int32_t> schedule(const KLayout& k, int NT, int n_ct, bool field_mode);

}  // namespace hobo
