// tt.h — Tensor-Train form of the HOBO tensor, host side.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace hobo {

struct TTCores {
  int order = 0, N = 0;
  std::vector<int> ranks;                    // r_0 .. r_k, r_0 = r_k = 1
  std::vector<std::vector<double>> cores;    // core p: r_{p} x N x r_{p+1}, row-major
};

// sequential SVD of the dense tensor (row-major, last index fastest); singular values
// <= rel_tol * sigma_max of an unfolding are dropped (rel_tol = 0: exact)
int tt_decompose(int order, int N, const std::vector<double>& dense, double rel_tol, TTCores& out, std::string& msg);

}  // namespace hobo
