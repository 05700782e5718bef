// hobo_oracle.cpp — plain, slow, obviously-correct CPU oracle (TEST INFRASTRUCTURE).
//
// Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference)
// may load this.  It shares no code, header, table or constant with the product
// (paper_2407_19987_b200/), and never includes anything from it.
//
// Each function follows a passage of PAPER.md (/root/reference/PAPER.md, the
// HOBOTAN paper) or, where the paper is silent, the reading recorded in DESIGN.md
// ("Readings of the paper").  Citations are "P:<line>".
#include "hobo_oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <map>
#include <thread>
#include <vector>

namespace {

using Mono = std::vector<int32_t>;  // sorted, duplicate-free variable ids (x^n = x)

struct Poly {                       // the reduced multilinear polynomial of P:51
  bool exact = true;                // every input integral -> __int128 arithmetic
  std::map<Mono, __int128> ic;      // exact coefficients
  std::map<Mono, long double> fc;   // otherwise long double
};

struct Oracle {
  int order = 0, N = 0;
  double offset = 0.0;
  // canonical cells, lexicographic by index tuple (O3)
  std::vector<Mono> sets;           // the monomial S of each cell
  std::vector<std::vector<int32_t>> tuple;  // its canonical index tuple
  std::vector<float> val;           // fp32 cell value (one RNE rounding)
  bool integer_cells = true;
  double sum_abs = 0.0;
};

bool is_int(double v) { return std::isfinite(v) && std::floor(v) == v && std::fabs(v) < 9.0e15; }

Mono mono_with(const Mono& m, int32_t v) {
  Mono r = m;
  auto it = std::lower_bound(r.begin(), r.end(), v);
  if (it == r.end() || *it != v) r.insert(it, v);  // x_v * x_v = x_v  (P:46 binary)
  return r;
}

// O3: smallest subscript replicated (order - r + 1) times at the front
std::vector<int32_t> canonical_tuple(const Mono& s, int order) {
  std::vector<int32_t> t;
  int r = (int)s.size();
  for (int i = 0; i < order - r + 1; ++i) t.push_back(s[0]);
  for (int i = 1; i < r; ++i) t.push_back(s[i]);
  return t;
}

// shared tail of both constructors: canonical cells from the coefficient of each set
template <class Map>
int finish(Oracle* o, const Map& m) {
  std::vector<std::pair<std::vector<int32_t>, std::pair<Mono, float>>> cells;
  for (auto& kv : m) {
    if (kv.first.empty()) continue;                   // constant -> offset
    long double c = (long double)kv.second;
    if (c == 0) continue;                             // O1: exact zeros dropped (a cancelled monomial is gone)
    if ((int)kv.first.size() > o->order) return 3;    // O2, on what remains: order < degree is an error
    if (std::fabs(c) > (long double)std::numeric_limits<float>::max()) return 2;
    float f = (float)c;                               // one round-to-nearest-even
    if (f == 0.0f) continue;
    cells.push_back({canonical_tuple(kv.first, o->order), {kv.first, f}});
  }
  std::sort(cells.begin(), cells.end(),
            [](const auto& a, const auto& b) { return a.first < b.first; });
  for (auto& c : cells) {
    o->tuple.push_back(c.first);
    o->sets.push_back(c.second.first);
    o->val.push_back(c.second.second);
    if (std::floor(c.second.second) != c.second.second) o->integer_cells = false;
    o->sum_abs += std::fabs((double)c.second.second);
  }
  return 0;
}

inline bool all_set(const Mono& s, const uint8_t* x) {
  for (int32_t u : s)
    if (!x[u]) return false;
  return true;
}

// O4 for one candidate: sum over cells of val * prod_{u in S} x_u
double energy_one(const Oracle* o, const uint8_t* x) {
  if (o->integer_cells) {
    int64_t e = 0;
    for (size_t c = 0; c < o->val.size(); ++c)
      if (all_set(o->sets[c], x)) e += (int64_t)o->val[c];
    return (double)e;
  }
  long double e = 0;
  for (size_t c = 0; c < o->val.size(); ++c)
    if (all_set(o->sets[c], x)) e += (long double)o->val[c];
  return (double)e;
}

// O5 for one candidate: g_m = sum_{S contains m} val * prod_{u in S, u != m} x_u
void field_one(const Oracle* o, const uint8_t* x, double* g) {
  std::vector<long double> acc(o->N, 0.0L);
  for (size_t c = 0; c < o->val.size(); ++c) {
    const Mono& s = o->sets[c];
    for (int32_t m : s) {
      bool on = true;
      for (int32_t u : s)
        if (u != m && !x[u]) { on = false; break; }
      if (on) acc[m] += (long double)o->val[c];
    }
  }
  for (int m = 0; m < o->N; ++m) g[m] = (double)acc[m];
}

template <class F>
void parallel_for(int64_t n, int nthreads, F f) {
  if (nthreads <= 1 || n < 2) {
    for (int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::vector<std::thread> th;
  int64_t chunk = (n + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    int64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([=]() { for (int64_t i = lo; i < hi; ++i) f(i); });
  }
  for (auto& t : th) t.join();
}

}  // namespace

extern "C" {

uint64_t or_splitmix64(uint64_t z) {  // SURVEY 8(d) generator spec
  z += 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

uint64_t or_hash(uint64_t s, uint64_t a, uint64_t b, uint64_t c) {
  return or_splitmix64(or_splitmix64(or_splitmix64(s ^ a) ^ b) ^ c);
}

// O1: expand every term coeff * prod_f (c0_f + sum w x) with x^n = x
int or_build(int order, int N, const or_term* terms, int64_t nterms, const or_factor* facs,
             const or_lin* lins, void** handle, double* offset_out) {
  if (order < 1 || N < 1 || nterms < 0 || !handle) return 1;
  bool exact = true;
  for (int64_t t = 0; t < nterms; ++t) {
    if (!std::isfinite(terms[t].coeff) || terms[t].nfac < 0) return 1;
    exact = exact && is_int(terms[t].coeff);
    for (int f = 0; f < terms[t].nfac; ++f) {
      const or_factor& F = facs[terms[t].fac0 + f];
      if (!std::isfinite(F.c0) || F.nlin < 0) return 1;
      exact = exact && is_int(F.c0);
      for (int l = 0; l < F.nlin; ++l) {
        const or_lin& L = lins[F.lin0 + l];
        if (L.var < 0 || L.var >= N || !std::isfinite(L.w)) return 1;
        exact = exact && is_int(L.w);
      }
    }
  }
  Poly P;
  P.exact = exact;
  for (int64_t t = 0; t < nterms; ++t) {
    std::map<Mono, __int128> ip;
    std::map<Mono, long double> fp;
    if (exact) ip[Mono()] = (__int128)terms[t].coeff; else fp[Mono()] = terms[t].coeff;
    for (int f = 0; f < terms[t].nfac; ++f) {
      const or_factor& F = facs[terms[t].fac0 + f];
      if (exact) {
        std::map<Mono, __int128> nx;
        for (auto& kv : ip) {
          if (F.c0 != 0) nx[kv.first] += kv.second * (__int128)F.c0;
          for (int l = 0; l < F.nlin; ++l) {
            const or_lin& L = lins[F.lin0 + l];
            nx[mono_with(kv.first, L.var)] += kv.second * (__int128)L.w;
          }
        }
        ip.swap(nx);
      } else {
        std::map<Mono, long double> nx;
        for (auto& kv : fp) {
          if (F.c0 != 0) nx[kv.first] += kv.second * (long double)F.c0;
          for (int l = 0; l < F.nlin; ++l) {
            const or_lin& L = lins[F.lin0 + l];
            nx[mono_with(kv.first, L.var)] += kv.second * (long double)L.w;
          }
        }
        fp.swap(nx);
      }
    }
    for (auto& kv : ip) P.ic[kv.first] += kv.second;
    for (auto& kv : fp) P.fc[kv.first] += kv.second;
  }
  Oracle* o = new Oracle();
  o->order = order;
  o->N = N;
  int st;
  if (exact) {
    auto it = P.ic.find(Mono());
    o->offset = it == P.ic.end() ? 0.0 : (double)(long double)it->second;
    st = finish(o, P.ic);
  } else {
    auto it = P.fc.find(Mono());
    o->offset = it == P.fc.end() ? 0.0 : (double)it->second;
    st = finish(o, P.fc);
  }
  if (st) { delete o; return st; }
  if (offset_out) *offset_out = o->offset;
  *handle = o;
  return 0;
}

int or_from_cells(int order, int N, int64_t ncells, const int32_t* idx, const float* val, void** handle) {
  if (order < 1 || N < 1 || ncells < 0 || !handle) return 1;
  std::map<Mono, long double> m;
  for (int64_t c = 0; c < ncells; ++c) {
    if (!std::isfinite(val[c])) return 1;
    Mono s;
    for (int p = 0; p < order; ++p) {
      int32_t v = idx[c * order + p];
      if (v < 0 || v >= N) return 1;
      s = mono_with(s, v);
    }
    if (val[c] != 0.0f) m[s] += (long double)val[c];
  }
  Oracle* o = new Oracle();
  o->order = order;
  o->N = N;
  int st = finish(o, m);
  if (st) { delete o; return st; }
  *handle = o;
  return 0;
}

void or_free(void* h) { delete (Oracle*)h; }

int or_info(void* h, int* order, int* N, int64_t* ncells, int* is_integer, double* sum_abs) {
  Oracle* o = (Oracle*)h;
  if (!o) return 1;
  if (order) *order = o->order;
  if (N) *N = o->N;
  if (ncells) *ncells = (int64_t)o->val.size();
  if (is_integer) *is_integer = o->integer_cells ? 1 : 0;
  if (sum_abs) *sum_abs = o->sum_abs;
  return 0;
}

int or_cells(void* h, int32_t* idx, float* val) {
  Oracle* o = (Oracle*)h;
  for (size_t c = 0; c < o->val.size(); ++c) {
    for (int p = 0; p < o->order; ++p) idx[c * o->order + p] = o->tuple[c][p];
    val[c] = o->val[c];
  }
  return 0;
}

int or_monomials(void* h, int32_t* degree, int32_t* vars, float* val) {
  Oracle* o = (Oracle*)h;
  for (size_t c = 0; c < o->val.size(); ++c) {
    degree[c] = (int32_t)o->sets[c].size();
    for (int p = 0; p < o->order; ++p)
      vars[c * o->order + p] = p < (int)o->sets[c].size() ? o->sets[c][p] : -1;
    val[c] = o->val[c];
  }
  return 0;
}

int or_export_dense(void* h, float* out) {
  Oracle* o = (Oracle*)h;
  double cells = std::pow((double)o->N, o->order);
  if (cells > (double)(1u << 28)) return 2;
  std::memset(out, 0, sizeof(float) * (size_t)cells);
  for (size_t c = 0; c < o->val.size(); ++c) {
    int64_t lin = 0;
    for (int p = 0; p < o->order; ++p) lin = lin * o->N + o->tuple[c][p];  // last index fastest
    out[lin] = o->val[c];
  }
  return 0;
}

int or_energy(void* h, const uint8_t* X, int64_t B, double* E, int nthreads) {
  Oracle* o = (Oracle*)h;
  if (!o || B < 0) return 1;
  std::vector<uint8_t> dummy;
  parallel_for(B, nthreads, [&](int64_t b) {
    std::vector<uint8_t> x(o->N);
    for (int m = 0; m < o->N; ++m) x[m] = X[b * o->N + m] ? 1 : 0;
    E[b] = energy_one(o, x.data());
  });
  return 0;
}

// O4': H(x) = sum_{i,j,k,...} H_{ijk...} x_i x_j x_k ... over ALL N^k cells
int or_energy_tensor(void* h, const uint8_t* X, int64_t B, double* E) {
  Oracle* o = (Oracle*)h;
  double cells = std::pow((double)o->N, o->order);
  if (cells > (double)(1u << 24)) return 2;
  std::vector<float> H((size_t)cells);
  or_export_dense(h, H.data());
  std::vector<int32_t> c(o->order);
  for (int64_t b = 0; b < B; ++b) {
    const uint8_t* x = X + b * o->N;
    long double e = 0;
    for (int64_t lin = 0; lin < (int64_t)cells; ++lin) {
      int64_t r = lin;
      long double prod = H[lin];
      for (int p = o->order - 1; p >= 0; --p) { prod *= (x[r % o->N] ? 1 : 0); r /= o->N; }
      e += prod;
    }
    E[b] = (double)e;
  }
  return 0;
}

int or_field(void* h, const uint8_t* X, int64_t B, double* G, int nthreads) {
  Oracle* o = (Oracle*)h;
  parallel_for(B, nthreads, [&](int64_t b) {
    std::vector<uint8_t> x(o->N);
    for (int m = 0; m < o->N; ++m) x[m] = X[b * o->N + m] ? 1 : 0;
    field_one(o, x.data(), G + b * o->N);
  });
  return 0;
}

// O7: idx t in [0, 2^N), x_m = (t >> m) & 1 (SURVEY 8(c) reading 12)
int or_menergy(void* h, const double* P, int64_t B, double* E, int nthreads) {
  Oracle* o = (Oracle*)h;
  parallel_for(B, nthreads, [&](int64_t b) {
    const double* p = P + b * o->N;
    long double e = 0;
    for (size_t c = 0; c < o->val.size(); ++c) {
      long double t = o->val[c];
      for (int32_t u : o->sets[c]) t *= p[u];
      e += t;
    }
    E[b] = (double)e;
  });
  return 0;
}

int or_mfield(void* h, const double* P, int64_t B, double* G, int nthreads) {
  Oracle* o = (Oracle*)h;
  parallel_for(B, nthreads, [&](int64_t b) {
    const double* p = P + b * o->N;
    std::vector<long double> acc(o->N, 0.0L);
    for (size_t c = 0; c < o->val.size(); ++c) {
      const Mono& s = o->sets[c];
      for (int32_t m : s) {
        long double t = o->val[c];
        for (int32_t u : s)
          if (u != m) t *= p[u];
        acc[m] += t;
      }
    }
    for (int m = 0; m < o->N; ++m) G[b * o->N + m] = (double)acc[m];
  });
  return 0;
}

int or_brute(void* h, double* emin, int64_t* argmin, int64_t* n_ground, double* next_level,
             int64_t* ground, int64_t max_ground, int nthreads) {
  Oracle* o = (Oracle*)h;
  if (o->N > 26) return 2;
  const int64_t total = (int64_t)1 << o->N;
  // the cell's monomial as a bit mask: prod_{u in S} x_u = 1  <=>  (t & mask) == mask
  std::vector<uint32_t> mask(o->val.size());
  for (size_t c = 0; c < o->val.size(); ++c)
    for (int32_t u : o->sets[c]) mask[c] |= 1u << u;
  const int T = std::max(1, nthreads);
  std::vector<double> tmin(T, INFINITY);
  std::vector<int64_t> targ(T, -1);
  auto eval = [&](int64_t t) -> double {
    if (o->integer_cells) {
      int64_t e = 0;
      for (size_t c = 0; c < mask.size(); ++c)
        if ((t & mask[c]) == mask[c]) e += (int64_t)o->val[c];
      return (double)e;
    }
    long double e = 0;
    for (size_t c = 0; c < mask.size(); ++c)
      if ((t & mask[c]) == mask[c]) e += o->val[c];
    return (double)e;
  };
  std::vector<double> all((size_t)total);
  parallel_for(T, T, [&](int64_t w) {
    int64_t chunk = (total + T - 1) / T, lo = w * chunk, hi = std::min(total, lo + chunk);
    for (int64_t t = lo; t < hi; ++t) {
      double e = eval(t);
      all[t] = e;
      if (e < tmin[w]) { tmin[w] = e; targ[w] = t; }
    }
  });
  double best = INFINITY;
  int64_t barg = -1;
  for (int w = 0; w < T; ++w)
    if (targ[w] >= 0 && (tmin[w] < best || (tmin[w] == best && targ[w] < barg))) { best = tmin[w]; barg = targ[w]; }
  int64_t ng = 0;
  double nxt = NAN;
  for (int64_t t = 0; t < total; ++t) {
    if (all[t] == best) {
      if (ng < max_ground && ground) ground[ng] = t;
      ++ng;
    } else if (std::isnan(nxt) || all[t] < nxt) {
      nxt = all[t];
    }
  }
  *emin = best;
  *argmin = barg;
  *n_ground = ng;
  *next_level = nxt;
  return 0;
}

}  // extern "C"

// C(n, i) for the colex ranks (n <= 65536, i <= 6)
static long double binom_ld(int64_t n, int i) {
  if (i < 0 || n < i) return 0;
  long double c = 1;
  for (int t = 1; t <= i; ++t) c = c * (long double)(n - i + t) / t;
  return c;
}

// sum over all k-subsets of `v` (sorted) of f(subset)
template <class F>
static void for_subsets(const std::vector<int32_t>& v, int k, F f) {
  const int n = (int)v.size();
  if (k > n) return;
  std::vector<int> c(k);
  for (int i = 0; i < k; ++i) c[i] = i;
  std::vector<int32_t> s(k);
  while (true) {
    for (int i = 0; i < k; ++i) s[i] = v[c[i]];
    f(s);
    int i = k - 1;
    while (i >= 0 && c[i] == n - k + i) --i;
    if (i < 0) return;
    ++c[i];
    for (int j = i + 1; j < k; ++j) c[j] = c[j - 1] + 1;
  }
}

static int64_t colex_rank_of(const std::vector<int32_t>& s) {
  long double r = 0;
  for (size_t i = 0; i < s.size(); ++i) r += binom_ld(s[i], (int)i + 1);
  return (int64_t)r;
}

extern "C" {

int or_colex_energy(int order, int N, const float* const* by_degree, const uint8_t* X, int64_t B, double* E,
                    int nthreads) {
  if (order < 1 || N < 1 || !by_degree) return 1;
  parallel_for(B, nthreads, [&](int64_t b) {
    std::vector<int32_t> ones;
    for (int m = 0; m < N; ++m)
      if (X[b * N + m]) ones.push_back(m);
    long double e = 0;
    for (int r = 1; r <= order; ++r)
      for_subsets(ones, r, [&](const std::vector<int32_t>& s) { e += by_degree[r - 1][colex_rank_of(s)]; });
    E[b] = (double)e;
  });
  return 0;
}

int or_colex_field(int order, int N, const float* const* by_degree, const uint8_t* X, int64_t B, double* G,
                   int nthreads) {
  if (order < 1 || N < 1 || !by_degree) return 1;
  parallel_for(B, nthreads, [&](int64_t b) {
    std::vector<int32_t> ones;
    for (int m = 0; m < N; ++m)
      if (X[b * N + m]) ones.push_back(m);
    for (int m = 0; m < N; ++m) {
      std::vector<int32_t> rest;
      for (int32_t u : ones)
        if (u != m) rest.push_back(u);
      long double g = by_degree[0][m];  // T = {} : the degree-1 cell of {m}
      for (int r = 2; r <= order; ++r)
        for_subsets(rest, r - 1, [&](const std::vector<int32_t>& t) {
          std::vector<int32_t> s(t);
          s.insert(std::lower_bound(s.begin(), s.end(), m), m);
          g += by_degree[r - 1][colex_rank_of(s)];
        });
      G[b * N + m] = (double)g;
    }
  });
  return 0;
}

int or_search_thresholds(int64_t iters, double p0, double p1, uint32_t* out) {
  for (int64_t t = 0; t < iters; ++t) {
    double frac = (double)t / (double)std::max<int64_t>(1, iters - 1);
    double p = 4294967296.0 * p0 * std::pow(p1 / p0, frac);
    double f = std::floor(p);
    if (f < 0) f = 0;
    if (f > 4294967295.0) f = 4294967295.0;
    out[t] = (uint32_t)f;
  }
  return 0;
}

// O8: the hobo_search rule of SURVEY 8(c) (the paper's sampler is undisclosed, P:199;
// SA is described only qualitatively), replayed one chain at a time.
// x_trace (nullable): [nchains][iters+1][N], the state evaluated at t = 0..iters;
// m_trace (nullable): [nchains][iters], the flipped site m* of iteration t.
int or_search_trace(void* h, uint64_t seed, int64_t chain0, int64_t nchains, int64_t iters,
                    double p0, double p1, double* chain_ebest, uint8_t* chain_xbest,
                    double* e_best, int64_t* best_chain, int nthreads, uint8_t* x_trace, int32_t* m_trace) {
  Oracle* o = (Oracle*)h;
  if (!o || nchains < 1 || iters < 0) return 1;
  const int N = o->N;
  std::vector<uint32_t> P((size_t)std::max<int64_t>(iters, 1));
  or_search_thresholds(iters, p0, p1, P.data());
  parallel_for(nchains, nthreads, [&](int64_t i) {
    const uint64_t c = (uint64_t)(chain0 + i);
    std::vector<uint8_t> x(N), xb(N);
    for (int m = 0; m < N; ++m) x[m] = (or_hash(seed, 1, c, (uint64_t)(m >> 6)) >> (m & 63)) & 1;
    std::vector<double> g(N);
    float best = INFINITY;
    auto consider = [&]() {
      float e = (float)energy_one(o, x.data());    // the kernel decides in fp32
      if (e < best) { best = e; xb = x; }            // equal E: the earliest t is kept
    };
    auto record = [&](int64_t t) {
      if (x_trace)
        for (int m = 0; m < N; ++m) x_trace[((size_t)i * (size_t)(iters + 1) + (size_t)t) * N + m] = x[m];
    };
    for (int64_t t = 0; t < iters; ++t) {
      record(t);
      consider();
      field_one(o, x.data(), g.data());
      const uint64_t r = or_hash(seed, 2, c, (uint64_t)t);
      const int mrand = (int)(((r & 0xffffffffULL) * (uint64_t)N) >> 32);
      int ms;
      if ((uint32_t)(r >> 32) < P[t]) {
        ms = mrand;
      } else {
        ms = 0;
        float dmin = INFINITY;
        for (int m = 0; m < N; ++m) {
          float gm = (float)g[m];
          float d = x[m] ? -gm : gm;                 // (1 - 2 x_m) g_m
          if (d < dmin) { dmin = d; ms = m; }        // lowest m on ties
        }
        if (!(dmin < 0.0f)) ms = mrand;
      }
      if (m_trace) m_trace[(size_t)i * (size_t)iters + (size_t)t] = ms;
      x[ms] ^= 1;
    }
    record(iters);
    consider();
    chain_ebest[i] = best;
    for (int m = 0; m < N; ++m) chain_xbest[i * N + m] = xb[m];
  });
  double be = INFINITY;
  int64_t bc = -1;
  for (int64_t i = 0; i < nchains; ++i)
    if (chain_ebest[i] < be) { be = chain_ebest[i]; bc = chain0 + i; }
  *e_best = be;
  *best_chain = bc;
  return 0;
}

int or_search(void* h, uint64_t seed, int64_t chain0, int64_t nchains, int64_t iters,
              double p0, double p1, double* chain_ebest, uint8_t* chain_xbest,
              double* e_best, int64_t* best_chain, int nthreads) {
  return or_search_trace(h, seed, chain0, nchains, iters, p0, p1, chain_ebest, chain_xbest, e_best, best_chain,
                         nthreads, nullptr, nullptr);
}


// SPEC sa_run's geometric schedule: T_s = t_start (t_end/t_start)^(s/max(1,sweeps-1))
int or_sa_temps(int64_t sweeps, double t_start, double t_end, double* out) {
  if (sweeps < 1 || !(t_start > 0) || !(t_end > 0) || t_end > t_start) return 1;
  for (int64_t s = 0; s < sweeps; ++s)
    out[s] = t_start * std::pow(t_end / t_start, (double)s / (double)std::max<int64_t>(1, sweeps - 1));
  return 0;
}

// Metropolis acceptance of an energy change d at temperature T with the uniform u in [0, 1):
// accept with probability min(1, exp(-d/T)), i.e. iff d <= 0 or
// u < exp(-d/T) <=> d < -T ln u for u in (0, 1) (the log form, reading 22)
int or_sa_accept(double d, double T, double u) { return (d <= 0.0 || d < -T * std::log(u)) ? 1 : 0; }

// SPEC sa_run: Metropolis single-bit flips in index order, one chain at a time
int or_sa(void* h, uint64_t seed, int64_t chain0, int64_t nchains, int64_t sweeps, double t_start, double t_end,
          uint8_t* x_out, double* e_out, int nthreads) {
  Oracle* o = (Oracle*)h;
  if (!o || nchains < 1) return 1;
  std::vector<double> T((size_t)std::max<int64_t>(sweeps, 1));
  if (or_sa_temps(std::max<int64_t>(sweeps, 1), t_start, t_end, T.data())) return 1;
  const int N = o->N;
  // the cells whose monomial contains m (g_m sums exactly these, O5)
  std::vector<std::vector<size_t>> touching(N);
  for (size_t c = 0; c < o->val.size(); ++c)
    for (int32_t m : o->sets[c]) touching[m].push_back(c);
  parallel_for(nchains, nthreads, [&](int64_t i) {
    const uint64_t c = (uint64_t)(chain0 + i);
    std::vector<uint8_t> x(N);
    for (int m = 0; m < N; ++m) x[m] = (or_hash(seed, 1, c, (uint64_t)(m >> 6)) >> (m & 63)) & 1;
    double e = energy_one(o, x.data());
    for (int64_t s = 0; s < sweeps; ++s) {
      for (int m = 0; m < N; ++m) {
        long double g = 0;                            // g_m(x) = E(x|x_m=1) - E(x|x_m=0)
        for (size_t cc : touching[m]) {
          bool on = true;
          for (int32_t u : o->sets[cc])
            if (u != m && !x[u]) { on = false; break; }
          if (on) g += (long double)o->val[cc];
        }
        const double d = x[m] ? -(double)g : (double)g;   // energy change of flipping x_m
        // Metropolis: accept with probability min(1, exp(-d/T)), i.e. iff d <= 0 or
        // u < exp(-d/T) <=> d < -T ln u for u in (0,1)  (reading 22)
        const double u = (double)(or_hash(seed, 4, c, (uint64_t)(s * N + m)) >> 11) * 0x1.0p-53;
        const bool accept = or_sa_accept(d, T[(size_t)s], u) != 0;
        if (accept) {
          x[m] ^= 1;
          e += d;
        }
      }
    }
    for (int m = 0; m < N; ++m) x_out[i * N + m] = x[m];
    e_out[i] = e;
  });
  return 0;
}

}  // extern "C"
