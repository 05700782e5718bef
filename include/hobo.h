/*
 * hobo.h — C ABI of the B200-native HOBOTAN hot path (arXiv 2407.19987).
 *
 * The library (paper_2407_19987_b200/_lib/libhobo.so) contracts a dense, upper-
 * triangular order-k HOBO tensor with a batch of binary candidates on sm_100a tensor
 * cores.  Citations "P:<n>" refer to lines of the paper's LaTeX.
 *
 * Conventions (all calls):
 *   - Every call returns hobo_status; nothing throws across the ABI.  On failure
 *     hobo_last_error() returns a thread-local message naming the problem.
 *   - "device" pointers live on the CUDA device that was current when the handle was
 *     built (the handle's device); they are caller-owned (e.g. torch tensors'
 *     data_ptr()).  "host" pointers are ordinary CPU memory.
 *   - Work is ordered on the caller's `stream` (a cudaStream_t passed as void*; NULL =
 *     legacy default stream).  Calls that fill host outputs synchronise that stream.
 *   - A handle must not be used from two threads at once.  A CUDA error poisons the
 *     handle (later calls return HOBO_ECUDA).
 *   - Energies EXCLUDE the compile offset, like the paper's printed "Energy"
 *     (Energy -30 reported together with offset 30).
 *   - Kernel choice is automatic; environment variables override it for A/B
 *     measurements and tests (read when the handle first uses the choice):
 *       HOBO_PAIR=1|0        CTA-pair (cta_group::2) contraction on / off
 *       HOBO_SA_KERNEL=ring|stage|pair   the persistent annealing kernel
 *       HOBO_I8=1|0          int8 digit planes (kind::i8) whenever exact / never
 *       HOBO_F8=1|0          e4m3 limbs (kind::f8f6f4) also on non-integer instances when
 *                            the split is exact / never (default: integer instances whose
 *                            limbs save >= 20% of the tensor-core cycles)
 *       HOBO_CT_DESC=1|0     column tiles longest-first (default when the last tile is the
 *                            heaviest) / in index order
 *       HOBO_PERSIST=1|0     the persistent energy kernel (short K loops, e.g. QUBO) on / off
 *       HOBO_PERSIST_I8=1    ... on int8 digit planes when the cells allow (exact; opt-in)
 *       HOBO_PERSIST_I8_NT=64|128, HOBO_PERSIST_KPS=1|2   its tile width / stage size
 *       HOBO_GRAPH=0         launch energy / field calls and the search loop directly instead
 *                            of replaying their captured CUDA graphs
 *       HOBO_SK=0            no stream-K schedule for CTA-pair field launches
 *       HOBO_E2E_TAIL=<n>, HOBO_E2E_HEAD=<q>   host-buffer field calls returning G: n
 *                            halvings after the last whole wave (default 0), first chunk q
 *                            quarter waves (default 4)
 *       HOBO_KR_EXP=<bits>   MEASUREMENT ONLY: switches parts of the 1-byte-plane contraction
 *                            off (1 run decode, 2 A store, 4 second e4m3 limb; tools/f8_check.sh);
 *                            results are wrong whenever it is set
 *       HOBO_PERSIST_EXP=<bits>  MEASUREMENT ONLY: switches parts of the persistent kernels off
 *                            (tools/persist_exp.sh); results are wrong whenever it is set
 *     Pairs, persistent kernels, graphs and annealing kernels give the same results (bit for
 *     bit on integer instances).  The int8 path computes the contraction exactly (integer
 *     accumulation), the bf16 path within the fp32 tolerance; both are exact on integer
 *     instances with sum|H| < 2^24, as is the e4m3-limb path (taken only for such instances
 *     unless HOBO_F8=1).
 */
#ifndef HOBO_H_
#define HOBO_H_
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HOBO_OK = 0,
  HOBO_EINVAL = 1,  /* bad order/N/ids/degree, non-finite coefficient, bad pointer/size  */
  HOBO_ERANGE = 2,  /* a compiled cell exceeds FLT_MAX                                     */
  HOBO_ENOMEM = 3,  /* host or device allocation failed / size budget exceeded             */
  HOBO_ECUDA = 4,   /* CUDA error (sticky per handle) or no sm_100 device                  */
  HOBO_ENCCL = 5,   /* NCCL error in the multi-GPU combine (hobo_dist_*)                   */
  HOBO_ESTATE = 6   /* handle poisoned, call out of order (e.g. TT energy before the TT
                       build), or a communicator already initialised                       */
} hobo_status;

typedef struct hobo_tensor hobo_tensor;   /* opaque; owns host cells + one device replica */

/* Term format: coeff * prod_f (c0_f + sum_l w_l * x_{var_l}).  It covers plain monomials,
 * the binary integer encoding y = sum_k 2^k x_k of P:133-139 (one factor with weights
 * 2^k, LSB- or MSB-first as in P:283-286 / P:371-373), (1 - q) factors and
 * powers (repeat a factor).  A term with nfac = 0 is a constant.        */
typedef struct { int32_t var; double w; } hobo_lin;
typedef struct { double c0; int32_t nlin, lin0; } hobo_factor;
typedef struct { double coeff; int32_t nfac, fac0; } hobo_term;
typedef struct { float e; int64_t idx; } hobo_best;

/* hobo_tensor_build — "Compile(H).get_hobo() -> hobo, offset".
 * Expands every term with x^n = x (binary variables), sums like monomials, drops
 * exact zeros, and stores each monomial S = {s1<...<sr} in the order-`order` tensor at
 * its canonical cell (s1 repeated order-r+1 times, s2..sr): the smallest-subscript
 * replication of P:111-117 / P:123-127.  Exact in integer arithmetic when all inputs are
 * integral, otherwise long double; one round-to-nearest-even to fp32 per cell.
 *   order   tensor order k, 1..6; must be >= the reduced degree (else HOBO_EINVAL)
 *   N       number of binary variables (axis extent), 1..65535 (N <= 1024 when order>3)
 *   terms/facs/lins  host arrays in the format above (copied; caller keeps ownership)
 *   out     receives the new handle (device = current CUDA device)
 *   offset_out (nullable) receives the constant term.                                  */
hobo_status hobo_tensor_build(int order, int N, const hobo_term* terms, size_t nterms,
                              const hobo_factor* facs, const hobo_lin* lins,
                              hobo_tensor** out, double* offset_out);

/* hobo_tensor_import_cells — explicit tensor cells (host).  Cell c has index tuple
 * idx[c*order .. c*order+order) (any order, any repetition) and value val[c]; it is added
 * to the canonical cell of its index SET, so energies on binary x are those of the raw
 * tensor.  This is how the dense random configs enter (BASELINE configs 2, 4, 5).       */
hobo_status hobo_tensor_import_cells(int order, int N, int64_t ncells, const int32_t* idx,
                                     const float* val, hobo_tensor** out);

/* hobo_tensor_import_dense — SURVEY 8(b) dense import: a host tensor of N^order fp32
 * cells, row-major with the last index fastest (the layout hobo_tensor_export_dense writes).
 * Every nonzero cell is added to the canonical cell of its index SET (as in
 * hobo_tensor_import_cells), so energies on binary x are unchanged.  N^order <= 2^28 cells
 * (HOBO_ENOMEM otherwise); other errors as hobo_tensor_import_cells.                      */
hobo_status hobo_tensor_import_dense(int order, int N, const float* dense_host, hobo_tensor** out);

/* hobo_tensor_import_colex — the canonical cells themselves (the upper-triangular tensor
 * without its replicated copies): cells_by_degree[r-1] is a host float array of
 * C(N, r) entries, entry colex_rank(S) = sum_i C(s_i, i) holding c(S) for the r-subset
 * S = {s1<...<sr}, r = 1..order.  Copied.  The efficient path for large dense instances
 * (BASELINE config 5: 178,957,824 cells).                                                 */
hobo_status hobo_tensor_import_colex(int order, int N, const float* const* cells_by_degree,
                                     hobo_tensor** out);

hobo_status hobo_tensor_free(hobo_tensor* t);

/* info: order, N, #nonzero canonical cells, all cells integral (0/1), sum |cell| (the
 * parity scale: tolerance = 1e-5 * sum_abs), bf16 limb count L used on the device (1..3,
 * the least L such that hi+mid+lo represents every fp32 cell exactly), offset.          */
hobo_status hobo_tensor_info(const hobo_tensor* t, int* order, int* N, int64_t* ncells,
                             int* is_integer, double* sum_abs, int* limbs, double* offset);
/* The fixed-point decomposition behind the int8 path, host
 * only: every cell of degree >= 2 equals q * 2^qexp with q an integer of `digits`
 * two's-complement bytes (1..3; 0 = no such q fits in 3 bytes).  Whether a call takes the
 * int8 path also depends on its cost (hobo_last_launch_kind reports the path taken).      */
hobo_status hobo_tensor_digits(const hobo_tensor* t, int* digits, int* qexp);

/* host export of the canonical cells (lexicographic by index tuple): idx[ncells*order],
 * val[ncells]; and of the dense N^order fp32 tensor (row-major, last index fastest;
 * refuses N^order > 2^28 with HOBO_ENOMEM).  Test/inspection helpers.                 */
hobo_status hobo_tensor_export_cells(const hobo_tensor* t, int32_t* idx, float* val);
hobo_status hobo_tensor_export_dense(const hobo_tensor* t, float* host_out);

/* hobo_energy — the tensor batch system: E_b = sum H_{ij..} X_bi X_bj ...
 *   X_dev   device u8, row-major B x N; any nonzero byte means 1
 *   B       number of candidates (>= 0)
 *   row0    global index of row 0 (0 on one GPU; the shard offset on a multi-GPU run)
 *   E_dev   device float[B] output (nullable if only `best` is wanted)
 *   best    host output (nullable): argmin over (E, row0+b), ties -> lowest index
 * Runs the energy-mode tensor-core contraction (strict, last-index-open layout).       */
hobo_status hobo_energy(hobo_tensor* t, const uint8_t* X_dev, int64_t B, int64_t row0,
                        float* E_dev, hobo_best* best, void* stream);

/* hobo_local_field — the same contraction with one index left open ("the gradient
 * is computed based on tensor contraction results"):
 *   G_dev[b*N+m] = E(x_b | x_m <- 1) - E(x_b | x_m <- 0)
 * (the discrete local field; flip gain (1 - 2 x_m) G).  E_dev (nullable) receives the
 * energies, computed from the per-degree fields in the same pass; best (host, nullable)
 * receives the argmin over (E, row0+b) as in hobo_energy.                               */
hobo_status hobo_local_field(hobo_tensor* t, const uint8_t* X_dev, int64_t B, int64_t row0,
                             float* G_dev, float* E_dev, hobo_best* best, void* stream);

/* hobo_local_field_host — hobo_local_field for candidates in HOST memory, end to end:
 * X_host [B*N] u8 in; host outputs (each nullable): G_host [B*N] f32 the local fields,
 * E_host [B] f32 the energies, best the argmin.  Page-locked X_host / G_host let the copies
 * overlap the contraction: the batch runs in chunks of whole waves, chunk i+1's host->device
 * copy (an internal copy stream ordered after the caller's stream) overlaps chunk i's
 * contraction, and chunk i's fields go back to the host (a second internal stream) while
 * chunk i+1 is contracted.  With G_host NULL the fields stay in device scratch.  E_host is
 * written by one copy after the last chunk.  Results equal hobo_local_field's.  Synchronises
 * the stream.                                                                              */
hobo_status hobo_local_field_host(hobo_tensor* t, const uint8_t* X_host, int64_t B, int64_t row0,
                                  float* G_host, float* E_host, hobo_best* best, void* stream);
/* hobo_energy_host — hobo_energy for candidates in host memory, the same pipeline (energy
 * layout; no fields).  Results equal hobo_energy's.  Synchronises the stream.            */
hobo_status hobo_energy_host(hobo_tensor* t, const uint8_t* X_host, int64_t B, int64_t row0,
                             float* E_host, hobo_best* best, void* stream);

/* Packed candidates — the same four calls with X given as bit rows instead of bytes
 * (the candidates are binary vectors; a byte per bit is 8x the bytes the
 * contraction needs, and through host buffers the host->device copy of X is the cost):
 *   Xbits    u32, row-major B x W with W = ceil(N / 32); bit (m mod 32) of word m / 32 of
 *            row b is x_bm (LSB first).  Bits at positions >= N are ignored (cleared on
 *            the device).  _bits: device pointer; _host_bits: host pointer (page-locked
 *            lets the copies overlap), B*W*4 bytes copied instead of B*N.
 * Everything else (outputs, row0, best, errors, streams) is as in the byte-input call;
 * results are identical to it for the same candidates.                                  */
hobo_status hobo_energy_bits(hobo_tensor* t, const uint32_t* Xbits_dev, int64_t B, int64_t row0,
                             float* E_dev, hobo_best* best, void* stream);
hobo_status hobo_local_field_bits(hobo_tensor* t, const uint32_t* Xbits_dev, int64_t B, int64_t row0,
                                  float* G_dev, float* E_dev, hobo_best* best, void* stream);
hobo_status hobo_energy_host_bits(hobo_tensor* t, const uint32_t* Xbits_host, int64_t B, int64_t row0,
                                  float* E_host, hobo_best* best, void* stream);
hobo_status hobo_local_field_host_bits(hobo_tensor* t, const uint32_t* Xbits_host, int64_t B, int64_t row0,
                                       float* G_host, float* E_host, hobo_best* best, void* stream);

/* hobo_multilinear_field — the same contraction on REAL candidates p in [0,1]^N, the
 * multilinear relaxation used by gradient descent ("the gradient is computed based
 * on tensor contraction results"):
 *   G_dev[b*N+m] = dE/dp_m = sum_{S contains m} c(S) prod_{u in S, u != m} p_bu,
 *   E_dev[b]     = E(p_b) = sum_S c(S) prod_{u in S} p_bu        (nullable)
 *   P_dev        device bf16 (raw 16-bit patterns), row-major B x N.  The products of up to
 *                three bf16 values are exact in fp32 and are split exactly into bf16 limbs,
 *                so the result is the gradient AT the bf16 p (fp32 accumulation).
 * The p rows are staged in shared memory next to the W ring: N up to ~800 (HOBO_EINVAL
 * beyond); when 256-column W boxes do not fit beside them (e.g. N = 512 at L = 3) the call
 * uses a copy of the field layout with 128-column tiles (one-time extra device memory).    */
hobo_status hobo_multilinear_field(hobo_tensor* t, const uint16_t* P_dev, int64_t B, float* G_dev,
                                   float* E_dev, void* stream);

/* hobo_gd_run — gradient descent on the multilinear relaxation:
 * `shots` independent restarts; each starts from p = U(0,1) (counter hash), takes `steps`
 * logit-parameterised steps theta <- theta - step_size * dE/dp * p(1-p) with p = sigmoid(theta)
 * carried in bf16 (gradient from hobo_multilinear_field's contraction), rounds at 0.5 and
 * runs `greedy_iters` steepest single-flip descent steps on the binary problem.  The final
 * states are aggregated like hobo_search_samples (top-k, energy / occurrence).           */
hobo_status hobo_gd_run(hobo_tensor* t, uint64_t seed, int64_t shots, int64_t steps, double step_size,
                        int64_t greedy_iters, int64_t topk, uint8_t* x_host, float* e_host,
                        int64_t* count_host, int64_t* n_out, void* stream);

/* hobo_tt_build — Tensor-Train decomposition of the canonical HOBO tensor by sequential SVD
 * (host, double precision, one-sided Jacobi).  Singular values <= rel_tol *
 * sigma_max of each unfolding are dropped; rel_tol < 1e-12 is raised to 1e-12, the
 * round-off floor of the double SVD ("without approximation").
 * ranks_out (nullable, order+1 ints) receives r_0..r_k (P:560 prints the TSP cores).
 * Needs the dense tensor: N^order <= 2^24 cells, else HOBO_ENOMEM.                       */
hobo_status hobo_tt_build(hobo_tensor* t, double rel_tol, int32_t* ranks_out);

/* hobo_tt_energy — energies from the TT cores: E_b = prod_p (sum_i x_bi G_p[:, i, :])
 * (the TT contraction of P:560-575, batched), fp64 arithmetic, ranks <= 32.  Same
 * X / E / best conventions as hobo_energy.                                                 */
hobo_status hobo_tt_energy(hobo_tensor* t, const uint8_t* X_dev, int64_t B, int64_t row0,
                           float* E_dev, hobo_best* best, void* stream);

/* hobo_search — batched heuristic search (P:81-83 simulated annealing is described only
 * qualitatively and the paper's sampler is undisclosed; the rule implemented is
 * DESIGN.md "Search rule").  `batch` chains start from counter-hash random x, run
 * `iters` field evaluations + single-flip moves, and the lexicographically smallest
 * (E_best, chain) is returned: x_best_host (u8[N]) and *e_best_host.  Deterministic in
 * (tensor, seed, batch, iters).  iters = 0 returns the best random initial candidate.   */
hobo_status hobo_search(hobo_tensor* t, uint64_t seed, int64_t batch, int64_t iters,
                        uint8_t* x_best_host, float* e_best_host, void* stream);

/* hobo_search_shard — the same rule on global chains [chain0, chain0+nchains) (one GPU's
 * shard); p0/p1 are the exploration-probability endpoints (defaults 0.5 / 0.005).  Also
 * returns the winning global chain id.  Results per chain do not depend on the shard.   */
hobo_status hobo_search_shard(hobo_tensor* t, uint64_t seed, int64_t chain0, int64_t nchains,
                              int64_t iters, double p0, double p1, uint8_t* x_best_host,
                              float* e_best_host, int64_t* best_chain, void* stream);

/* hobo_search_samples — the paper's result list ("Energy e, Occurrence n", P:202-206,
 * P:226-243): the same search as hobo_search over `batch` chains, then the chains' best
 * states are aggregated on the device (sorted by (E, assignment hash), duplicates grouped
 * and counted) and the first `topk` distinct assignments are returned in the order
 * energy ascending, occurrence descending, assignment lexicographic (x_0 first):
 *   x_host [topk*N] u8, e_host [topk] (offset excluded), count_host [topk], *n_out =
 *   min(topk, #distinct).  Host outputs; synchronises the stream.                        */
hobo_status hobo_search_samples(hobo_tensor* t, uint64_t seed, int64_t batch, int64_t iters,
                                int64_t topk, uint8_t* x_host, float* e_host, int64_t* count_host,
                                int64_t* n_out, void* stream);

/* hobo_sa_shard — simulated annealing, SPEC sa_run after PAPER.md:81-83 ("starts
 * at a high temperature and gradually cools down"), on global chains [chain0, chain0+nchains):
 * chain c starts at x_m = bit (m & 63) of h(seed,1,c,m>>6); sweep s = 0..sweeps-1 at
 * T_s = t_start (t_end/t_start)^(s / max(1, sweeps-1)) visits m = 0..N-1 in index order and
 * accepts the flip of x_m iff d = (1-2x_m) g_m <= 0 or d < -T_s ln u (i.e. u < exp(-d/T_s)),
 * u = (h(seed,4,c,s*N+m) >> 11) 2^-53 (reading 22).  Requires 0 < t_end <= t_start.  Outputs
 * (device, caller-owned, nullable): X_out [nchains*N] u8 final states, E_out [nchains]
 * their freshly evaluated energies (offset excluded), E_tracked [nchains] the energies
 * the sweep tracked incrementally (double).  Per-chain results do not depend on the shard;
 * on integer instances (sum|H| < 2^24) they equal the oracle's replay bit for bit.
 * Device memory: one order-(k-1) derivative tensor layout per site, built on first use. */
hobo_status hobo_sa_shard(hobo_tensor* t, uint64_t seed, int64_t chain0, int64_t nchains,
                          int64_t sweeps, double t_start, double t_end, uint8_t* X_out_dev,
                          float* E_out_dev, double* E_tracked_dev, void* stream);

/* hobo_sa_run — SPEC sa_run's SampleSet: `shots` chains annealed as above, their final
 * states aggregated like hobo_search_samples (energy ascending, occurrence descending,
 * assignment lexicographic; occurrences sum to shots over all distinct states).  Host
 * outputs as in hobo_search_samples; synchronises the stream.                           */
hobo_status hobo_sa_run(hobo_tensor* t, uint64_t seed, int64_t shots, int64_t sweeps,
                        double t_start, double t_end, int64_t topk, uint8_t* x_host,
                        float* e_host, int64_t* count_host, int64_t* n_out, void* stream);

/* ---- multi-GPU: one process per GPU, one NCCL communicator per
 * process.  H is replicated (each rank builds its own handle); candidates / chains are
 * sharded by the caller (row0) or, for hobo_search, by rank.  Once a communicator is
 * initialised (any world size), every call that returns a `best` combines it over the ranks on
 * the compute stream (C1: ncclAllReduce MIN of the packed 64-bit (E, global index) key)
 * before reading it back, and hobo_search runs chains [lo_r, lo_{r+1}) of the global batch
 * (lo_r = r*(batch/P) + min(r, batch%P)) and broadcasts the winner's bits from the rank that
 * owns its chain (C2: ncclBroadcast).  All ranks must make the same calls in the same order
 * (collectives).  Sample-set calls (hobo_*_samples, hobo_sa_run, hobo_gd_run) and the
 * *_shard calls stay per rank.  libnccl.so.2 is loaded on first use (the process's own
 * NCCL when one is already loaded).
 * hobo_dist_unique_id: 128 bytes to hand from rank 0 to every rank (e.g. via
 * torch.distributed.broadcast_object_list).  hobo_dist_init: makes `device` current and
 * joins the communicator; HOBO_ESTATE if one exists.  hobo_dist_finalize: destroys it.
 * hobo_dist_info: (rank, world), (0, 1) without a communicator.                            */
hobo_status hobo_dist_unique_id(void* id_out);
hobo_status hobo_dist_init(int rank, int world, const void* id, int device);
hobo_status hobo_dist_finalize(void);
hobo_status hobo_dist_info(int* rank, int* world);

/* ---- multi-GPU host logic (SURVEY 8(e) partition and C1 key).  Plain host
 * arithmetic: no device, no communicator (callable on a machine without a GPU).  The library's
 * own hobo_search and every best-combining call use exactly these functions.
 * hobo_shard: rank `rank` of `world` owns items [*lo, *lo + *n) of `total` (>= 0), with
 *   lo = rank*(total/world) + min(rank, total % world): contiguous, the first ranks take the
 *   remainder, *n may be 0 when total < world.  EINVAL for world < 1 or rank outside [0, world).
 * hobo_shard_owner: *owner = the rank whose shard holds `index`; EINVAL outside [0, total).
 * hobo_best_key: the 64-bit argmin key of (e, idx):
 *   key = (ord(e) << 32) | idx, ord(e) = the fp32 bits of e made monotone (i = bits(e); if i < 0
 *   then i ^= 0x7FFFFFFF; -0 is +0) with the sign bit flipped, so that the UNSIGNED minimum of
 *   keys is the lexicographic minimum of (e, idx) -- the ncclUint64 MIN of C1.  EINVAL for a NaN
 *   e or idx outside [0, 2^32).
 * hobo_best_from_key: its inverse into a hobo_best; key = ~0 (no candidate) gives (+inf, -1).   */
hobo_status hobo_shard(int64_t total, int rank, int world, int64_t* lo, int64_t* n);
hobo_status hobo_shard_owner(int64_t total, int world, int64_t index, int* owner);
hobo_status hobo_best_key(float e, int64_t idx, uint64_t* key);
hobo_status hobo_best_from_key(uint64_t key, hobo_best* best);

/* Launch statistics of the last call on this handle: number of kernel launches issued,
 * the executed tensor-core MACs of its contraction kernel(s), the algorithmic MACs (SURVEY
 * 8(d): nnz per candidate for energies, 2 nnz for energy + field, nnz = sum_{r<=k} C(N, r)),
 * and — when profiling is on — the CUDA-event time in ms of its contraction kernel(s),
 * recorded on the launch stream (this call synchronises on it).  */
hobo_status hobo_last_launch_stats(hobo_tensor* t, int64_t* launches, double* mma_macs,
                                   double* algo_macs, double* kernel_ms);
/* The MMA kind of the last call's contraction: *i8_planes = the number of int8 digit planes
 * (tcgen05.mma kind::i8), MINUS the number of e4m3 limb
 * planes (kind::f8f6f4; the stages multiply only the limbs they
 * need), or 0 for bf16 limbs (kind::f16).  mma_macs above counts 8-bit MACs in the first two
 * cases, bf16 MACs in the third.                                                           */
hobo_status hobo_last_launch_kind(const hobo_tensor* t, int* i8_planes);
/* profiling on/off: record CUDA events around every contraction-kernel launch.         */
hobo_status hobo_set_profiling(hobo_tensor* t, int enable);

const char* hobo_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* HOBO_H_ */
