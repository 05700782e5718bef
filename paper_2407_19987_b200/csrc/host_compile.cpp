// host_compile.cpp — hobo_tensor_build on the host (not timed; runs once per problem).
//
// Implements "Compile(H).get_hobo() -> hobo, offset": expand the terms
// with x^n = x, sum like monomials, and give every monomial its canonical
// cell (smallest subscript replicated).  Internally a cell is
// stored once, by degree r and colex rank of its variable set, which is all the device
// layout needs; the tuple form (s,..,s,v2..vr) is produced only by the export helpers.
#include "host_compile.h"

#include <climits>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <unordered_map>

#include "../../include/hobo.h"

namespace hobo {

int64_t binom(int64_t n, int r) {
  if (r < 0 || n < 0 || n < r) return 0;
  if (r > n - r) r = (int)(n - r);
  __int128 c = 1;
  for (int i = 1; i <= r; ++i) {
    c = c * (n - r + i) / i;
    if (c > (__int128)std::numeric_limits<int64_t>::max()) return std::numeric_limits<int64_t>::max();
  }
  return (int64_t)c;
}

namespace {

constexpr int MAXV = 15;  // distinct variables a monomial may carry during expansion

struct Mono {
  uint16_t n = 0;
  uint16_t v[MAXV] = {};
  bool operator==(const Mono& o) const { return n == o.n && std::memcmp(v, o.v, sizeof(uint16_t) * n) == 0; }
  bool operator<(const Mono& o) const {
    if (n != o.n) return n < o.n;
    for (int i = 0; i < n; ++i)
      if (v[i] != o.v[i]) return v[i] < o.v[i];
    return false;
  }
  // multiply by x_u (idempotent): insert u keeping the ids sorted; false on overflow
  bool times(uint16_t u) {
    int i = 0;
    while (i < n && v[i] < u) ++i;
    if (i < n && v[i] == u) return true;
    if (n == MAXV) return false;
    for (int j = n; j > i; --j) v[j] = v[j - 1];
    v[i] = u;
    ++n;
    return true;
  }
};
struct MonoHash {
  size_t operator()(const Mono& m) const {
    uint64_t h = 1469598103934665603ULL ^ m.n;
    for (int i = 0; i < m.n; ++i) h = (h ^ m.v[i]) * 1099511628211ULL;
    return (size_t)h;
  }
};

bool integral(double v) { return std::isfinite(v) && v == std::nearbyint(v) && std::fabs(v) < 4.0e18; }

int64_t colex_rank(const Mono& s) {
  int64_t r = 0;
  for (int i = 0; i < s.n; ++i) r += binom(s.v[i], i + 1);
  return r;
}

// bf16 round-to-nearest-even of an fp32 value (finite inputs)
float bf16_round(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  u += 0x7FFFu + ((u >> 16) & 1u);
  u &= 0xFFFF0000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}
int limbs_needed(float c) {
  float hi = bf16_round(c);
  float r1 = c - hi;
  if (r1 == 0.0f) return 1;
  float mid = bf16_round(r1);
  float r2 = r1 - mid;
  if (r2 == 0.0f) return 2;
  return 3;
}

void cell_stats(HostTensor& out) {
  out.nnz = 0;
  out.sum_abs = 0.0;
  out.is_integer = true;
  out.limbs = 1;
  for (int r = 1; r <= out.order; ++r)
    for (float f : out.strict[r]) {
      if (f == 0.0f) continue;
      ++out.nnz;
      out.sum_abs += std::fabs((double)f);
      if (f != std::nearbyint(f)) out.is_integer = false;
      out.limbs = std::max(out.limbs, limbs_needed(f));
    }
  // fixed-point quantum of the degree >= 2 cells: the smallest exponent of a cell's lowest set bit
  int qe = INT_MAX;
  for (int r = 2; r <= out.order; ++r)
    for (float f : out.strict[r]) {
      if (f == 0.0f) continue;
      int e = 0;
      const double m = std::frexp(std::fabs((double)f), &e);     // |f| = m 2^e, m in [0.5, 1)
      uint32_t M = (uint32_t)std::ldexp(m, 24);                 // the 24-bit significand
      qe = std::min(qe, e - 24 + __builtin_ctz(M));
    }
  out.qexp = qe == INT_MAX ? 0 : qe;
  out.digits = 1;
  double qmax = 0.0, qmin = 0.0;
  for (int r = 2; r <= out.order; ++r)
    for (float f : out.strict[r]) {
      const double q = std::ldexp((double)f, -out.qexp);
      qmax = std::max(qmax, q);
      qmin = std::min(qmin, q);
    }
  while (out.digits <= 3 && (qmax > std::ldexp(1.0, 8 * out.digits - 1) - 1.0 || qmin < -std::ldexp(1.0, 8 * out.digits - 1)))
    ++out.digits;
  if (out.digits > 3) out.digits = 0;
}

template <class Num>
int finish(int order, int N, const std::unordered_map<Mono, Num, MonoHash>& poly, HostTensor& out, std::string& msg) {
  out = HostTensor();
  out.order = order;
  out.N = N;
  out.strict.resize(order + 1);
  double total = 0;
  for (int r = 1; r <= order; ++r) total += (double)binom(N, r);
  if (total > 1.6e9) {
    msg = "canonical cell space sum_r C(N,r) = " + std::to_string(total) + " exceeds the 1.6e9-cell host budget (N=" +
          std::to_string(N) + ", order=" + std::to_string(order) + ")";
    return 3;
  }
  try {
    for (int r = 1; r <= order; ++r) out.strict[r].assign((size_t)binom(N, r), 0.0f);
  } catch (...) {
    msg = "host allocation of the canonical cells failed";
    return 3;
  }
  for (const auto& kv : poly) {
    const long double c = (long double)kv.second;
    if (kv.first.n == 0) {
      out.offset += (double)c;
      continue;
    }
    if (c == 0) continue;
    if (kv.first.n > order) {
      msg = "monomial of degree " + std::to_string(kv.first.n) + " exceeds tensor order " + std::to_string(order);
      return 1;
    }
    if (std::fabs(c) > (long double)std::numeric_limits<float>::max()) {
      msg = "a compiled cell exceeds FLT_MAX";
      return 2;
    }
    const float f = (float)c;  // the single RNE rounding to fp32
    if (f == 0.0f) continue;
    out.strict[kv.first.n][(size_t)colex_rank(kv.first)] = f;
  }
  cell_stats(out);
  return 0;
}

template <class Num>
int expand(int order, int N, const TermView& tv, HostTensor& out, std::string& msg) {
  const hobo_term* T = (const hobo_term*)tv.terms;
  const hobo_factor* F = (const hobo_factor*)tv.facs;
  const hobo_lin* Lv = (const hobo_lin*)tv.lins;
  std::unordered_map<Mono, Num, MonoHash> poly;
  std::vector<std::pair<Mono, Num>> cur, nxt;
  for (size_t t = 0; t < tv.nterms; ++t) {
    cur.assign(1, {Mono(), (Num)T[t].coeff});
    for (int f = 0; f < T[t].nfac; ++f) {
      const hobo_factor& fa = F[T[t].fac0 + f];
      nxt.clear();
      for (const auto& mc : cur) {
        if (fa.c0 != 0.0) nxt.push_back({mc.first, mc.second * (Num)fa.c0});
        for (int l = 0; l < fa.nlin; ++l) {
          const hobo_lin& li = Lv[fa.lin0 + l];
          Mono m = mc.first;
          if (!m.times((uint16_t)li.var)) {
            msg = "a term multiplies more than 15 distinct variables";
            return 1;
          }
          nxt.push_back({m, mc.second * (Num)li.w});
        }
      }
      // merge like monomials of the partial product
      std::sort(nxt.begin(), nxt.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      cur.clear();
      for (const auto& mc : nxt) {
        if (!cur.empty() && cur.back().first == mc.first) cur.back().second += mc.second;
        else cur.push_back(mc);
      }
    }
    for (const auto& mc : cur) poly[mc.first] += mc.second;
  }
  return finish<Num>(order, N, poly, out, msg);
}

}  // namespace

int compile_terms(int order, int N, const TermView& tv, HostTensor& out, std::string& msg) {
  if (order < 1 || order > 6) { msg = "order must be in 1..6"; return 1; }
  if (N < 1 || N > 65535 || (order > 3 && N > 1024)) { msg = "N out of range (1..65535, <=1024 for order>3)"; return 1; }
  if (tv.nterms && (!tv.terms)) { msg = "null terms array"; return 1; }
  const hobo_term* T = (const hobo_term*)tv.terms;
  const hobo_factor* F = (const hobo_factor*)tv.facs;
  const hobo_lin* Lv = (const hobo_lin*)tv.lins;
  bool exact = true;
  for (size_t t = 0; t < tv.nterms; ++t) {
    if (!std::isfinite(T[t].coeff) || T[t].nfac < 0) { msg = "term " + std::to_string(t) + ": bad coefficient or nfac"; return 1; }
    exact = exact && integral(T[t].coeff);
    if (T[t].nfac > 0 && !F) { msg = "null factor array"; return 1; }
    for (int f = 0; f < T[t].nfac; ++f) {
      const hobo_factor& fa = F[T[t].fac0 + f];
      if (!std::isfinite(fa.c0) || fa.nlin < 0) { msg = "term " + std::to_string(t) + ": bad factor"; return 1; }
      exact = exact && integral(fa.c0);
      if (fa.nlin > 0 && !Lv) { msg = "null lin array"; return 1; }
      for (int l = 0; l < fa.nlin; ++l) {
        const hobo_lin& li = Lv[fa.lin0 + l];
        if (li.var < 0 || li.var >= N) { msg = "variable id " + std::to_string(li.var) + " outside [0,N)"; return 1; }
        if (!std::isfinite(li.w)) { msg = "non-finite weight"; return 1; }
        exact = exact && integral(li.w);
      }
    }
  }
  return exact ? expand<__int128>(order, N, tv, out, msg) : expand<long double>(order, N, tv, out, msg);
}

int compile_cells(int order, int N, int64_t ncells, const int32_t* idx, const float* val, HostTensor& out,
                  std::string& msg) {
  if (order < 1 || order > 6) { msg = "order must be in 1..6"; return 1; }
  if (N < 1 || N > 65535 || (order > 3 && N > 1024)) { msg = "N out of range"; return 1; }
  if (ncells < 0 || (ncells && (!idx || !val))) { msg = "bad cell arrays"; return 1; }
  std::unordered_map<Mono, long double, MonoHash> poly;
  poly.reserve((size_t)std::min<int64_t>(ncells, 1 << 26));
  for (int64_t c = 0; c < ncells; ++c) {
    if (!std::isfinite(val[c])) { msg = "non-finite cell value"; return 1; }
    if (val[c] == 0.0f) continue;
    Mono m;
    for (int p = 0; p < order; ++p) {
      const int32_t v = idx[c * order + p];
      if (v < 0 || v >= N) { msg = "cell index outside [0,N)"; return 1; }
      m.times((uint16_t)v);
    }
    poly[m] += (long double)val[c];
  }
  return finish<long double>(order, N, poly, out, msg);
}

int compile_colex(int order, int N, const float* const* by_degree, HostTensor& out, std::string& msg) {
  if (order < 1 || order > 6) { msg = "order must be in 1..6"; return 1; }
  if (N < 1 || N > 65535 || (order > 3 && N > 1024)) { msg = "N out of range"; return 1; }
  if (!by_degree) { msg = "null cell arrays"; return 1; }
  double total = 0;
  for (int r = 1; r <= order; ++r) total += (double)binom(N, r);
  if (total > 1.6e9) { msg = "canonical cell space exceeds the 1.6e9-cell host budget"; return 3; }
  out = HostTensor();
  out.order = order;
  out.N = N;
  out.strict.resize(order + 1);
  for (int r = 1; r <= order; ++r) {
    const size_t n = (size_t)binom(N, r);
    if (n && !by_degree[r - 1]) { msg = "null cell array for degree " + std::to_string(r); return 1; }
    try {
      out.strict[r].assign(by_degree[r - 1], by_degree[r - 1] + n);
    } catch (...) {
      msg = "host allocation of the canonical cells failed";
      return 3;
    }
    for (float f : out.strict[r])
      if (!std::isfinite(f)) { msg = "non-finite cell value"; return 1; }
  }
  cell_stats(out);
  return 0;
}

namespace {
// successor of a sorted r-subset in colex order; false after the last subset of [0,N)
bool colex_next(std::vector<int32_t>& a, int N) {
  const int r = (int)a.size();
  for (int i = 0; i < r; ++i) {
    const int32_t lim = (i + 1 < r) ? a[i + 1] : N;
    if (a[i] + 1 < lim) {
      ++a[i];
      for (int j = 0; j < i; ++j) a[j] = j;
      return true;
    }
  }
  return false;
}
}  // namespace

// P_m = dE/dx_m as an order-(k-1) tensor: c_Pm(T) = c(T u {m}) for m not in T.  Its local
// field at j is the second difference d^2E / dx_m dx_j, the change of g_j when x_m flips
// (the incremental field update of the annealing sweep).
int derive(const HostTensor& H, int m, HostTensor& out, std::string& msg) {
  const int k = H.order, N = H.N;
  if (k < 2 || m < 0 || m >= N) { msg = "derive: order >= 2 and 0 <= m < N required"; return 1; }
  std::vector<std::vector<int64_t>> bt((size_t)N + 1, std::vector<int64_t>(8, 0));
  for (int n = 0; n <= N; ++n)
    for (int i = 0; i < 8; ++i) bt[n][i] = binom(n, i);
  std::vector<std::vector<float>> by(k - 1);
  for (int rp = 1; rp <= k - 1; ++rp) {
    std::vector<float>& a = by[rp - 1];
    a.assign((size_t)binom(N, rp), 0.0f);
    if (rp + 1 > N) continue;
    const std::vector<float>& src = H.strict[rp + 1];
    std::vector<int32_t> T(rp);
    for (int i = 0; i < rp; ++i) T[i] = i;
    int64_t rank = 0;
    do {
      // colex rank of T u {m} among (rp+1)-subsets: sum_i C(c_i, i), c sorted, i from 1
      bool has = false, placed = false;
      int pos = 1;
      int64_t r2 = 0;
      for (int i = 0; i < rp; ++i) {
        if (T[i] == m) { has = true; break; }
        if (!placed && m < T[i]) { r2 += bt[m][pos++]; placed = true; }
        r2 += bt[T[i]][pos++];
      }
      if (!has) {
        if (!placed) r2 += bt[m][pos];
        a[(size_t)rank] = src[(size_t)r2];
      }
      ++rank;
    } while (colex_next(T, N));
  }
  std::vector<const float*> ptrs(k - 1);
  for (int r = 0; r < k - 1; ++r) ptrs[r] = by[r].data();
  return compile_colex(k - 1, N, ptrs.data(), out, msg);
}

void export_cells(const HostTensor& t, int32_t* idx, float* val) {
  std::vector<std::pair<std::vector<int32_t>, float>> cells;
  for (int r = 1; r <= t.order; ++r) {
    std::vector<int32_t> a(r);
    for (int i = 0; i < r; ++i) a[i] = i;
    int64_t rank = 0;
    if (r > t.N) continue;
    do {
      const float f = t.strict[r][(size_t)rank];
      if (f != 0.0f) {
        std::vector<int32_t> tup(t.order - r + 1, a[0]);  // replicate the smallest subscript
        for (int i = 1; i < r; ++i) tup.push_back(a[i]);
        cells.push_back({tup, f});
      }
      ++rank;
    } while (colex_next(a, t.N));
  }
  std::sort(cells.begin(), cells.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
  for (size_t c = 0; c < cells.size(); ++c) {
    for (int p = 0; p < t.order; ++p) idx[c * t.order + p] = cells[c].first[p];
    val[c] = cells[c].second;
  }
}

int export_dense(const HostTensor& t, float* out) {
  const double cells = std::pow((double)t.N, t.order);
  if (cells > (double)(1u << 28)) return 3;
  std::memset(out, 0, sizeof(float) * (size_t)cells);
  std::vector<int32_t> idx((size_t)t.nnz * t.order);
  std::vector<float> val((size_t)t.nnz);
  export_cells(t, idx.data(), val.data());
  for (int64_t c = 0; c < t.nnz; ++c) {
    int64_t lin = 0;
    for (int p = 0; p < t.order; ++p) lin = lin * t.N + idx[c * t.order + p];
    out[lin] = val[c];
  }
  return 0;
}

int build_klayout(int order, int N, KLayout& k, std::string& msg) {
  k = KLayout();
  k.order = order;
  k.N = N;
  k.nseg = order - 1;
  int64_t T = 0;
  for (int j = 0; j < k.nseg; ++j) {
    const int r = order - j;
    const int64_t len = binom(N, r - 1);
    k.seg_t0.push_back(T);
    k.seg_len.push_back(len);
    T += (len + 2 * KBLK - 1) / (2 * KBLK) * (2 * KBLK);   // segments start at even K-blocks (int8
  }                                                       // boxes hold K-block pairs)
  k.Tpad = T;
  if ((double)T * 12.0 > 4.0e9) { msg = "K dimension too large"; return 3; }
  k.tuples.assign((size_t)T * 6, 0);
  const int64_t nkb = T / KBLK;
  std::vector<int64_t> run_t;  // first tuple of each run (for run_off)
  for (int j = 0; j < k.nseg; ++j) {
    const int r = order - j;
    int64_t t = k.seg_t0[j];
    const int nup = r - 2;  // size of the fixed ("upper") part; lowest element runs contiguously
    // upper parts (u_1 < ... ) in colex order; within one, the lowest element runs over
    // [0, u_1) — together this is the colex order of the (r-1)-subsets.  (u_1 = 0: no tuples.)
    std::vector<int32_t> up(nup);
    for (int i = 0; i < nup; ++i) up[i] = i;
    bool more = nup <= N;
    while (more) {
      const int32_t span = nup ? up[0] : N;  // lowest element ranges over [0, span)
      int32_t lo = 0;
      while (lo < span) {
        const int64_t blk_end = (t / KBLK + 1) * KBLK;
        const int32_t cnt = (int32_t)std::min<int64_t>(span - lo, blk_end - t);
        uint32_t rec[4];
        rec[0] = (uint32_t)(t % KBLK) | ((uint32_t)cnt << 8) | ((uint32_t)lo << 16);
        uint16_t f[4] = {0xFFFF, 0xFFFF, 0xFFFF, 0xFFFF};
        for (int i = 0; i < nup; ++i) f[i] = (uint16_t)up[i];
        rec[1] = f[0] | ((uint32_t)f[1] << 16);
        rec[2] = f[2] | ((uint32_t)f[3] << 16);
        rec[3] = 0;
        k.runs.insert(k.runs.end(), rec, rec + 4);
        run_t.push_back(t);
        for (int32_t q = 0; q < cnt; ++q) {
          uint16_t* tp = &k.tuples[(size_t)(t + q) * 6];
          tp[0] = (uint16_t)r;
          tp[1] = (uint16_t)(lo + q);
          for (int i = 0; i < nup; ++i) tp[2 + i] = (uint16_t)up[i];
        }
        t += cnt;
        lo += cnt;
      }
      if (nup == 0) break;
      more = colex_next(up, N);
    }
    if (t != k.seg_t0[j] + k.seg_len[j]) { msg = "internal: tuple count mismatch"; return 1; }
  }
  k.run_off.assign((size_t)nkb + 1, 0);
  size_t ri = 0;
  for (int64_t kb = 0; kb <= nkb; ++kb) {
    while (ri < run_t.size() && run_t[ri] < kb * KBLK) ++ri;
    k.run_off[(size_t)kb] = (uint32_t)ri;
  }
  k.kdesc.assign((size_t)nkb * 8, 0);
  if (k.runs.size() / 4 + 2 >= (1u << 22)) { msg = "too many generator runs"; return 3; }
  for (int64_t kb = 0; kb < nkb; ++kb) {
    int seg = 0;
    while (seg + 1 < k.nseg && k.seg_t0[seg + 1] <= kb * KBLK) ++seg;
    const uint32_t nfix = (uint32_t)std::max(0, order - seg - 2);
    const uint32_t r0 = k.run_off[(size_t)kb], n = k.run_off[(size_t)kb + 1] - r0;
    uint32_t* d = &k.kdesc[(size_t)kb * 8];
    for (uint32_t q = 0; q < std::min(n, 2u); ++q)
      for (int f = 0; f < 4; ++f) d[4 * q + f] = k.runs[(size_t)(r0 + q) * 4 + f];
    d[3] = nfix | (n << 3) | ((r0 + 2) << 10);
  }
  return 0;
}

std::vector<int32_t> schedule(const KLayout& k, int NT, int n_ct, bool field_mode) {
  std::vector<int32_t> s((size_t)n_ct * std::max(1, k.nseg) * 2, 0);
  for (int ct = 0; ct < n_ct; ++ct)
    for (int j = 0; j < k.nseg; ++j) {
      const int r = k.order - j;
      int64_t need = k.seg_len[j];
      if (!field_mode) {  // strict layout: column m needs tuples whose elements are all < m
        const int64_t m_max = std::min<int64_t>(k.N, (int64_t)(ct + 1) * NT) - 1;
        need = m_max > 0 ? binom(m_max, r - 1) : 0;
      }
      s[((size_t)ct * k.nseg + j) * 2 + 0] = (int32_t)(k.seg_t0[j] / KBLK);
      s[((size_t)ct * k.nseg + j) * 2 + 1] = (int32_t)((need + KBLK - 1) / KBLK);
    }
  return s;
}

}  // namespace hobo
