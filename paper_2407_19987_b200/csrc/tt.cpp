// tt.cpp — Tensor-Train decomposition of the HOBO tensor on the host.
//
// "Reshape the high-dimensional tensor A into a matrix A_(1); apply SVD ...; incorporate
// Sigma V* into the next tensor and reshape it into A_(2); repeat".  The SVD is a
// one-sided (Hestenes) Jacobi iteration in double precision, applied to the transpose of
// each unfolding (few rows, many columns).  Build time only; not on the timed path.
#include "tt.h"

#include <algorithm>
#include <cmath>
#include <numeric>

namespace hobo {

namespace {

// thin SVD of an m x n row-major matrix C with m <= n via Jacobi on C^T:
// C = U diag(s) V^T, U: m x m (row-major), s: m, Vt: m x n (row-major rows = right vectors)
void jacobi_svd_wide(int m, int64_t n, const std::vector<double>& C, std::vector<double>& U, std::vector<double>& s,
                     std::vector<double>& Vt) {
  // Y = C^T (n x m) stored column-major as m columns of length n: col j = row j of C
  std::vector<double> Y(C);
  std::vector<double> W((size_t)m * m, 0.0);   // accumulated rotations, row-major
  for (int i = 0; i < m; ++i) W[(size_t)i * m + i] = 1.0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int i = 0; i < m; ++i)
      for (int j = i + 1; j < m; ++j) {
        const double* yi = &Y[(size_t)i * n];
        const double* yj = &Y[(size_t)j * n];
        double a = 0, b = 0, g = 0;
        for (int64_t k = 0; k < n; ++k) { a += yi[k] * yi[k]; b += yj[k] * yj[k]; g += yi[k] * yj[k]; }
        if (g == 0.0 || std::fabs(g) <= 1e-15 * std::sqrt(a * b)) continue;
        off = std::max(off, std::fabs(g) / std::sqrt(a * b));
        const double zeta = (b - a) / (2.0 * g);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
        double* wi = &Y[(size_t)i * n];
        double* wj = &Y[(size_t)j * n];
        for (int64_t k = 0; k < n; ++k) {
          const double x = wi[k], y = wj[k];
          wi[k] = c * x - sn * y;
          wj[k] = sn * x + c * y;
        }
        for (int r = 0; r < m; ++r) {   // W <- W * rotation (columns i, j)
          const double x = W[(size_t)r * m + i], y = W[(size_t)r * m + j];
          W[(size_t)r * m + i] = c * x - sn * y;
          W[(size_t)r * m + j] = sn * x + c * y;
        }
      }
    if (off < 1e-15) break;
  }
  // C^T W = Y (orthogonal columns) => C = W diag(s) Vt with s_j = |Y_j|, Vt_j = Y_j^T / s_j
  s.assign(m, 0.0);
  for (int j = 0; j < m; ++j) {
    double a = 0;
    for (int64_t k = 0; k < n; ++k) a += Y[(size_t)j * n + k] * Y[(size_t)j * n + k];
    s[j] = std::sqrt(a);
  }
  std::vector<int> ord(m);
  std::iota(ord.begin(), ord.end(), 0);
  std::sort(ord.begin(), ord.end(), [&](int x, int y) { return s[x] > s[y]; });
  U.assign((size_t)m * m, 0.0);
  Vt.assign((size_t)m * n, 0.0);
  std::vector<double> s2(m);
  for (int q = 0; q < m; ++q) {
    const int j = ord[q];
    s2[q] = s[j];
    for (int r = 0; r < m; ++r) U[(size_t)r * m + q] = W[(size_t)r * m + j];
    if (s[j] > 0)
      for (int64_t k = 0; k < n; ++k) Vt[(size_t)q * n + k] = Y[(size_t)j * n + k] / s[j];
  }
  s.swap(s2);
}

}  // namespace

int tt_decompose(int order, int N, const std::vector<double>& dense, double rel_tol, TTCores& out, std::string& msg) {
  out = TTCores();
  out.order = order;
  out.N = N;
  out.ranks.assign(order + 1, 1);
  std::vector<double> C(dense);
  int r_prev = 1;
  int64_t rest = (int64_t)dense.size();
  for (int p = 0; p < order - 1; ++p) {
    const int64_t m64 = (int64_t)r_prev * N;
    rest /= N;  // columns of this unfolding: N^(order-p-1)
    if (m64 > 4096) { msg = "TT unfolding too tall for the host Jacobi SVD"; return 3; }
    const int m = (int)m64;
    std::vector<double> U, s, Vt;
    if (m <= rest) {
      jacobi_svd_wide(m, rest, C, U, s, Vt);
    } else {  // tall unfolding: decompose the transpose, swap the factors
      std::vector<double> Ct((size_t)m * rest);
      for (int i = 0; i < m; ++i)
        for (int64_t k = 0; k < rest; ++k) Ct[(size_t)k * m + i] = C[(size_t)i * rest + k];
      std::vector<double> U2, Vt2;
      jacobi_svd_wide((int)rest, m, Ct, U2, s, Vt2);   // Ct = U2 s Vt2 => C = Vt2^T s U2^T
      const int q = (int)rest;
      U.assign((size_t)m * q, 0.0);
      Vt.assign((size_t)q * rest, 0.0);
      for (int i = 0; i < m; ++i)
        for (int j = 0; j < q; ++j) U[(size_t)i * q + j] = Vt2[(size_t)j * m + i];
      for (int j = 0; j < q; ++j)
        for (int64_t k = 0; k < rest; ++k) Vt[(size_t)j * rest + k] = U2[(size_t)k * q + j];
      // U is m x q here; keep the bookkeeping below generic in the number of singular values
    }
    const int nsv = (int)s.size();
    const int ucols = (int)(U.size() / (size_t)m);
    int r = 0;
    const double smax = nsv ? s[0] : 0.0;
    while (r < nsv && s[r] > rel_tol * smax && s[r] > 0.0) ++r;
    r = std::max(r, 1);
    // core p: (r_prev, N, r) from U's first r columns (rows of U are (a, i) pairs)
    std::vector<double> core((size_t)r_prev * N * r);
    for (int a = 0; a < r_prev; ++a)
      for (int i = 0; i < N; ++i)
        for (int c = 0; c < r; ++c) core[((size_t)a * N + i) * r + c] = U[((size_t)a * N + i) * ucols + c];
    out.cores.push_back(core);
    out.ranks[p + 1] = r;
    // next matrix: diag(s_:r) Vt_:r  -> (r x rest), reshaped (r*N) x (rest/N)
    std::vector<double> Cn((size_t)r * rest);
    for (int c = 0; c < r; ++c)
      for (int64_t k = 0; k < rest; ++k) Cn[(size_t)c * rest + k] = s[c] * Vt[(size_t)c * rest + k];
    C.swap(Cn);
    r_prev = r;
  }
  out.cores.push_back(C);  // last core: (r_prev, N, 1)
  return 0;
}

}  // namespace hobo
