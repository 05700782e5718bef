/*
 * hobo_oracle.h — CPU ORACLE for the HOBOTAN batched HOBO contraction (arXiv 2407.19987).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2407_19987_b200/) never includes, links or calls anything under oracle/,
 * and this file includes nothing from the product.
 *
 * What it computes (plain definitions, no blocking / fusion / reordering):
 *   O1 expand      terms -> multilinear polynomial with x^n = x
 *   O2 order check max degree <= order
 *   O3 canonical   smallest subscript replicated at the front
 *   O4 energy      E(x) = sum_cells val * prod_{u in S} x_u            PAPER.md:65, 146 (offset excluded)
 *   O4' tensor     literal sum over all N^k cells of H[c] * prod x_c
 *   O5 field       g_m = sum_{S contains m} val * prod_{S\m} x         (discrete local field; SURVEY 8(c) reading 13)
 *   O6 argmin      lexicographic min over (E, global index)
 *   O7 brute force idx = sum_m x_m 2^m over all 2^N assignments
 *   O8 search      the hobo_search move rule, replayed chain by chain
 *
 * Every function returns 0 on success, nonzero on error (1 = bad argument,
 * 2 = size/resource, 3 = degree > order).
 */
#pragma once
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { int32_t var; double w; } or_lin;             /* w * x_var                         */
typedef struct { double c0; int32_t nlin, lin0; } or_factor;  /* c0 + sum lins[lin0 .. lin0+nlin)   */
typedef struct { double coeff; int32_t nfac, fac0; } or_term; /* coeff * prod factors[fac0 .. +nfac)*/

/* O1-O3 from the term format.  *handle receives an opaque pointer. */
int or_build(int order, int N, const or_term* terms, int64_t nterms, const or_factor* facs,
             const or_lin* lins, void** handle, double* offset_out);
/* O3 from explicit tensor cells (any index order/repetition): each cell is added to the
 * canonical cell of its index SET (x binary => same energy).                           */
int or_from_cells(int order, int N, int64_t ncells, const int32_t* idx, const float* val, void** handle);
void or_free(void* handle);

/* order, N, number of canonical (nonzero) cells, whether every cell is an integer, sum |cell| */
int or_info(void* handle, int* order, int* N, int64_t* ncells, int* is_integer, double* sum_abs);
/* canonical cells in lexicographic order of their index tuples: idx[ncells*order], val[ncells] */
int or_cells(void* handle, int32_t* idx, float* val);
/* dense N^order fp32 export, row-major, last index fastest (N^order <= 2^28) */
int or_export_dense(void* handle, float* out);
/* sorted monomial view: degree[c], vars[c*order] (padded with -1), coefficient (the fp32 cell) */
int or_monomials(void* handle, int32_t* degree, int32_t* vars, float* val);

/* O4: E[b] term by term (long double, or exact int64 for integer cells), X u8 row-major B x N */
int or_energy(void* handle, const uint8_t* X, int64_t B, double* E, int nthreads);
/* O4': the literal N^k contraction of the dense canonical tensor (small N only) */
int or_energy_tensor(void* handle, const uint8_t* X, int64_t B, double* E);
/* multilinear relaxation at real p in [0,1]^N:
 *   E(p) = sum_cells val * prod_{u in S} p_u,  dE/dp_m = sum_{S contains m} val * prod_{S\m} p_u */
int or_menergy(void* handle, const double* P, int64_t B, double* E, int nthreads);
int or_mfield(void* handle, const double* P, int64_t B, double* G, int nthreads);
/* O5: G[b*N + m] */
int or_field(void* handle, const uint8_t* X, int64_t B, double* G, int nthreads);
/* O7: brute force over 2^N (N <= 26).  Returns min, lowest argmin, #ground states,
 * next distinct level (NaN if none), and up to max_ground ground-state indices.   */
int or_brute(void* handle, double* emin, int64_t* argmin, int64_t* n_ground, double* next_level,
             int64_t* ground, int64_t max_ground, int nthreads);
/* O8: replay of hobo_search on chains [chain0, chain0+nchains) of the global chain space.
 * Outputs the per-chain best energy (fp32 value, as double) and bits (nchains x N), and
 * the lexicographic (E_best, chain) winner.                                              */
int or_search(void* handle, uint64_t seed, int64_t chain0, int64_t nchains, int64_t iters,
              double p0, double p1, double* chain_ebest, uint8_t* chain_xbest,
              double* e_best, int64_t* best_chain, int nthreads);
/* or_search with its trajectory: x_trace (nullable) [nchains][iters+1][N] = the state
 * evaluated at t = 0..iters; m_trace (nullable) [nchains][iters] = the site flipped at t.  */
int or_search_trace(void* handle, uint64_t seed, int64_t chain0, int64_t nchains, int64_t iters,
                    double p0, double p1, double* chain_ebest, uint8_t* chain_xbest,
                    double* e_best, int64_t* best_chain, int nthreads, uint8_t* x_trace, int32_t* m_trace);
/* Metropolis acceptance of or_sa: 1 iff d <= 0 or d < -T ln u (= u < exp(-d/T), u in (0,1)) */
int or_sa_accept(double d, double T, double u);
/* Simulated annealing, SPEC sa_run ("starts at a high
 * temperature and gradually cools down"), replayed on chains [chain0, chain0+nchains):
 * chain c starts at x_m = bit (m & 63) of h(seed,1,c,m>>6); sweep s = 0..sweeps-1 at
 * T_s = t_start (t_end/t_start)^(s / max(1, sweeps-1)) visits m = 0..N-1 in index order,
 * d = (1 - 2 x_m) g_m(x) (O5, exact), accepts iff d <= 0 or d < -T_s ln u (that is
 * u < exp(-d/T_s)) with u = (h(seed,4,c,s*N+m) >> 11) 2^-53, and on acceptance flips x_m and adds d to the
 * chain's energy.  Outputs the final states (nchains x N) and their tracked energies.  */
int or_sa(void* handle, uint64_t seed, int64_t chain0, int64_t nchains, int64_t sweeps, double t_start,
          double t_end, uint8_t* x_out, double* e_out, int nthreads);
/* the temperature table T_s of or_sa */
int or_sa_temps(int64_t sweeps, double t_start, double t_end, double* out);
/* Large instances given as canonical cells per degree in colex order
 * (by_degree[r-1][colex_rank(S)] = c(S), colex_rank({a1<..<ar}) = sum_i C(a_i, i)):
 * E(x) = sum over subsets S of the candidate's ones, |S| <= order, of c(S)
 * g_m(x) = sum over subsets T of ones minus {m}, |T| <= order-1, of c(T u {m})
 * evaluated one candidate at a time by plain subset enumeration (long double).       */
int or_colex_energy(int order, int N, const float* const* by_degree, const uint8_t* X, int64_t B, double* E,
                    int nthreads);
int or_colex_field(int order, int N, const float* const* by_degree, const uint8_t* X, int64_t B, double* G,
                   int nthreads);

/* the counter-based hash of SURVEY 8(d): h(s,a,b,c) = sm(sm(sm(s^a)^b)^c) */
uint64_t or_hash(uint64_t s, uint64_t a, uint64_t b, uint64_t c);
uint64_t or_splitmix64(uint64_t z);
/* exploration threshold table of the search rule, P_t for t in [0, iters) */
int or_search_thresholds(int64_t iters, double p0, double p1, uint32_t* out);

#ifdef __cplusplus
}
#endif
