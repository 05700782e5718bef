// kernels.cuh — sm_100a kernels of the HOBOTAN hot path.
//
// The contraction (batched as in PAPER.md:141-149) is evaluated as ONE
// tensor-core GEMM per (candidate block, column tile) with one tensor index left open:
//
//     F[b, m] = sum_t  A[b, t] * W[m, t]          (tcgen05.mma, fp32 accumulate in TMEM)
//
// t runs over the "tuples" = (r-1)-subsets T of the variables, grouped in segments by
// degree r = k..2, each segment in colex order.  A[b, t] = prod_{u in T} x_bu is the
// Khatri-Rao product of the candidate's bits — generated on chip from the bit-packed
// candidates, never stored in HBM.  W is the bf16 limb plane of one of two layouts:
//   field  mode: W[m, T] = c(T u {m}) for m not in T   -> F = per-degree local fields
//   energy mode: W[m, T] = c(T u {m}) for max T < m    -> F = last-index-open partials
// c(S) is the fp32 canonical cell of monomial S (PAPER.md:111-117 puts c(S) at the
// smallest-subscript-replicated cell; for binary x only the set S matters).
// The epilogue reduces F over m against x_bm (energy) and writes the fields.
#pragma once
#include <cstdint>
#include <cuda_bf16.h>

#include "ptx.cuh"

namespace hobo {

constexpr int kBM = 128;        // candidates per CTA (UMMA M, TMEM lanes)
constexpr int kBK = 64;         // tuples per K-block (one 128-byte SW128 row of bf16)
constexpr int kThreads = 320;   // warp 0 TMA, warp 1 MMA, warps 2-9 A-generator + epilogue (2 per lane quarter);
                                // e4m3 launches add warps 10-17 (generation only, kr_threads)

struct KrParams {
  const uint32_t* xbits;    // [B][W] bit-packed candidates (bit m of word m/32)
  const uint4* runs;        // A-generator runs (host_compile.cpp build_klayout)
  const uint4* kdesc;       // [n_kb][2] per-K-block descriptor (two inline runs)
  const int2* sched;        // [n_ct][nseg] (first K-block, #K-blocks)
  const float* p1;          // [Npad] degree-1 cells (the field of an order-1 term), 0 past N
  float* G;                 // field mode: [B][N] local fields; else nullptr
  double* Q;                // [n_ct][B] weighted partial energies (fixed-order, no atomics)
  long long B;
  int N, W, Npad, n_ct, n_cb, nseg, L, field_mode;
  int n_kb;                 // K-blocks per (limb, column tile): Tpad / 64
  // real-valued candidates (multilinear relaxation): p in bf16, B x N
  const uint16_t* preal;
  int LA;                   // bf16 limbs of the Khatri-Rao products of p (exact for <= 3 factors)
  int ring_boxes;           // W boxes that fit next to the p rows in shared memory
  int pstride;              // p row stride in shared memory (elements, odd word count)
  int cb_iters;             // > 1 (single-CTA bf16 binary launches only): each CTA loops over this many
                            // candidate blocks of one column tile, so a block's W fill and prologue
                            // overlap the previous block's epilogue (short K loops, e.g. cfg2)
  int ct_desc;              // 1: column tiles in descending order (the heaviest K schedules start
                            // first, so the light tiles fill the tail of the last wave)
  int n_split;              // split-K: CTAs of one (candidate block, column tile) split the K
                            // schedule; split s writes partials G + s*B*N, Q[(s*n_ct + ct)*B + b]
  double wdeg[8];           // field mode: weight lcm/r of the degree-r part of the energy
  double wp;                // weight of the degree-1 term
  double qscale;            // int8 digit planes (kr_gemm_kernel<..., I8>): cell = qscale * sum_l 256^l d_l
  float fscale;             // e4m3 limbs (kr_gemm_kernel<..., I8, F8>): F = fscale * accumulator
  int exp;                  // MEASUREMENT ONLY (HOBO_KR_EXP, 1-byte plane launches): 1 = the generator
                            // skips the run decode, 2 = skips the TMEM store (4: host side, one e4m3
                            // limb plane); results are wrong
  const uint32_t* nltab;    // e4m3 limbs: [n_ct][nl_words] limb counts of the K-block pairs, 2 bits each
  int nl_words;             // (16 pairs per word); copied to shared memory by every CTA
  const uint4* srec;        // int8: per K-block pair, {runs of 2P, runs of 2P+1, nfix, 0} + the runs
  int srec_u4;              // int8: uint4s per record (the descriptor ring's slot size)
  int desc_lg;              // int8: log2 of the descriptor ring's slots in use (4 or 5)
  // simulated annealing (kr_gemm_kernel<NT, false, true>): one launch per visited site m with
  // the layout of P_m = dE/dx_m; every CTA decides site m for its chains, column tile 0
  // commits the decisions, and the epilogue adds s_b * (field of P_m) to G
  uint32_t* sa_bits;        // the chains' state bits (== xbits); the flip of sa_prev lands here
  const int8_t* sa_sprev;   // decisions of the previous site (+1 set, -1 clear, 0 rejected)
  int8_t* sa_scur;          // decisions of this site
  double* sa_E;             // tracked energies
  double sa_T;              // temperature of the sweep
  unsigned long long sa_seed;
  long long sa_chain0;      // global id of chain 0 of this shard
  long long sa_step;        // s * N + m: counter of the acceptance uniform
  int sa_m, sa_prev;        // visited site, previous site (-1: none)
  // stream-K schedule (CTA-pair field launches; nullable): unit u of CTA pair u = {candidate-
  // block pair, column tile, first stage, last stage | (part + 1) << 20}; part -1 = the whole
  // tile, written in place; part >= 0 = a K range of a split tile, written to the partial
  // buffers skG [part][256 rows][NT] and skQ [part][256], summed by sk_reduce_kernel
  const int4* units;
  int n_units;              // CTA pairs of a stream-K launch
  float* skG;
  double* skQ;
};

// I8: W as int8 digit planes (one byte per tuple; a box row = 128 bytes = the K-block pair
// (2i, 2i+1), SW128) against A as {0,1} bytes, tcgen05.mma kind::i8 at twice the bf16 rate,
// one s32 accumulator per digit plane
template <int NT, bool I8 = false>
struct KrCfg {
  static constexpr int BOX = NT * 128;                   // one TMA box: NT rows x 64 bf16 tuples / 128 int8 tuples (SW128)
  static constexpr int RING_BOXES = 6 * 256 / NT;        // shared-memory budget for W (192 KB), in boxes
  static constexpr int MAXST = 8;                        // max W stages
  static constexpr int MAXA = 8;                         // binary energy/field launches: A stages, a ring of their
                                                         // own (TMEM-bound), decoupled from the W ring
  static constexpr int A_COLS = I8 ? kBK / 4 : kBK / 2;  // TMEM columns of one K-block of A (64 bf16 / 64 bytes per lane)
  static constexpr int TMEM_COLS = 512;                  // [0, NT): accumulator (I8: L of them), then the A stages
  static_assert(NT % 32 == 0 && NT >= 32 && NT <= 256, "UMMA N for M=128");
  static constexpr int MAXD = 32;                        // descriptor ring slots: 32 (records 16 stages ahead of
                                                         // W: e4m3 cfg3 2.94 -> 2.90 ms), or 16 (8 ahead) when
                                                         // 32 records do not fit shared memory (KrParams::desc_lg)
  static constexpr int NBAR = 2 * MAXST + 2 * MAXA + MAXD + 4;
  static constexpr int DESC_BYTES = 0;                   // (bf16 launches read their descriptors with __ldg)
  // I8: the descriptor ring holds the stages' run records (srec_u4 uint4s per slot)
  __host__ __device__ static size_t desc_bytes(int srec_u4, int desc_lg = 5) {
    return I8 ? ((size_t)1 << desc_lg) * srec_u4 * 16 : DESC_BYTES;
  }
  static size_t smem_bytes(int W, int srec_u4 = 0, int nl_words = 0, int desc_lg = 5) {
    return 1024 + (size_t)RING_BOXES * BOX + 8 * NBAR + 16 + 128 + kBM * 8 + desc_bytes(srec_u4, desc_lg) +
           (size_t)(W + (I8 ? 4 : 2)) * kBM * 4 + 128 +   // I8: two zero words in front (run_bits8)
           (size_t)nl_words * 4;                          // e4m3: the column tile's limb counts
  }
  // stage geometry for L limbs: KPS K-blocks x L limb boxes per stage, NST stages.  Two
  // K-blocks per stage halve the MMA thread's waits and commits per MMA; with 256-column
  // boxes that fits only at L = 1, with 128-column boxes at every L <= 3
  __host__ __device__ static constexpr int kps(int L) { return (I8 || L == 1 || NT <= 128) ? 2 : 1; }
  // decoupled rings (binary energy/field launches): W stages are bounded by shared memory
  // (pairs: twice the boxes) and MAXST, A stages by the TMEM left after the accumulator(s)
  // (I8: L of them).  A bf16 stage is KPS boxes per limb, an I8 stage one box per plane (the
  // box holds the K-block pair).
  __host__ __device__ static constexpr int nstw(int L, int ring) {
    return ring / ((I8 ? 1 : kps(L)) * L) < MAXST ? ring / ((I8 ? 1 : kps(L)) * L) : MAXST;
  }
  __host__ __device__ static constexpr int nsta(int L) {
    return (TMEM_COLS - (I8 ? L : 1) * NT) / (kps(L) * A_COLS) < MAXA ? (TMEM_COLS - (I8 ? L : 1) * NT) / (kps(L) * A_COLS) : MAXA;
  }
  __host__ __device__ static constexpr int nst(int L) { return nst_c(L, RING_BOXES); }
  // one ring (W boxes + A K-blocks per slot): bounded by shared memory, MAXST and TMEM
  __host__ __device__ static constexpr int nst_c(int L, int ring) {
    return ring / (kps(L) * L) < MAXST
               ? (ring / (kps(L) * L) < (TMEM_COLS - NT) / (kps(L) * A_COLS) ? ring / (kps(L) * L) : (TMEM_COLS - NT) / (kps(L) * A_COLS))
               : (MAXST < (TMEM_COLS - NT) / (kps(L) * A_COLS) ? MAXST : (TMEM_COLS - NT) / (kps(L) * A_COLS));
  }
  // real-valued A: one K-block per stage, LA limb tiles of A in TMEM, ring sized at run time
  __host__ __device__ static int nst_real(int L, int LA, int ring) {
    int n = ring / L;
    if (n > MAXST) n = MAXST;
    const int t = (TMEM_COLS - NT) / (LA * A_COLS);
    return n < t ? n : t;
  }
  static size_t smem_bytes_real(int ring, int pstride) {
    return 1024 + (size_t)ring * BOX + 8 * NBAR + 16 + 128 + kBM * 8 + DESC_BYTES + (size_t)kBM * pstride * 2 + 256;
  }
};

// A bits of one run for one candidate row: x[lo .. lo+cnt) AND the fixed elements' bits,
// placed at tuple offset `start` of the K-block (see host_compile.cpp build_klayout)
__device__ __forceinline__ uint64_t run_bits(const uint32_t* xs, int row, const uint4 rr, uint32_t nfix) {
  const uint32_t start = rr.x & 0xFFu, cnt = (rr.x >> 8) & 0xFFu, lo = rr.x >> 16;
  uint32_t on = 1;
  const uint32_t f[4] = {rr.y & 0xFFFFu, rr.y >> 16, rr.z & 0xFFFFu, rr.z >> 16};
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if ((uint32_t)q < nfix) on &= xs[(f[q] >> 5) * kBM + row] >> (f[q] & 31);
  // the 64-bit window x[lo .. lo+64) from three words, branch-free (funnel shifts)
  const uint32_t w = lo >> 5, sh = lo & 31;
  const uint32_t w0 = xs[w * kBM + row], w1 = xs[(w + 1) * kBM + row], w2 = xs[(w + 2) * kBM + row];
  const uint64_t v = ((uint64_t)__funnelshift_r(w1, w2, sh) << 32) | __funnelshift_r(w0, w1, sh);
  const uint64_t mask = cnt >= 64 ? ~0ull : ((1ull << cnt) - 1ull);
  return (v & mask & (0ull - (uint64_t)(on & 1u))) << start;
}

// the candidate row's 64 A bits of one K-block from its descriptor (d0, d1)
__device__ __forceinline__ uint64_t block_bits(const uint32_t* xs, int row, const uint4 d0, const uint4 d1,
                                               const uint4* __restrict__ runs) {
  const uint32_t nfix = d0.w & 7u, nruns = (d0.w >> 3) & 127u;
  uint64_t bits = 0;
  if (nruns > 0) bits |= run_bits(xs, row, d0, nfix);
  if (nruns > 1) bits |= run_bits(xs, row, d1, nfix);
#pragma unroll 1   // overflow runs are rare: keep the hot loop's code small
  for (uint32_t i = 2; i < nruns; ++i) bits |= run_bits(xs, row, __ldg(runs + (d0.w >> 10) + (i - 2)), nfix);
  return bits;
}

// 32 bits -> 16 words of two bf16 {0, 1.0}.  prmt with a selector-nibble msb replicates the
// picked byte's sign bit: after shifting by 7-2s (6-2s) bit 8k+2s (+1) is byte k's msb.
__device__ __forceinline__ void expand32(uint32_t half, uint32_t (&w)[16]) {
#pragma unroll
  for (int sh = 0; sh < 4; ++sh) {
    const uint32_t ev = half << (7 - 2 * sh), od = half << (6 - 2 * sh);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t sel = (0x8u | k) | ((0x8u | k) << 4) | ((0xCu | k) << 8) | ((0xCu | k) << 12);
      w[4 * k + sh] = prmt_b32(ev, od, sel) & 0x3F803F80u;
    }
  }
}

// int8 A bytes {0, 1} of a 64-tuple K-block from its 64 bits, 16 words.  The int8 planes store
// the K positions of each 32-tuple group permuted (layout_kernel: tuple 8i + k of the group at
// byte 4k + i), so word k of a group is bit k of each byte of the group's 32 bits: one shift
// and one AND per word (a natural order needs the 4-op nibble spread)
__device__ __forceinline__ void expand_bytes64(uint64_t bits, uint32_t (&w)[16]) {
  const uint32_t lo = (uint32_t)bits, hi = (uint32_t)(bits >> 32);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    w[k] = (lo >> k) & 0x01010101u;
    w[8 + k] = (hi >> k) & 0x01010101u;
  }
}

// the int8 path's generator runs, precomputed on the host (hobo_api.cu, the stage records):
// x, y = the 64-bit output mask ((1 << cnt) - 1) << start; z = window word | shift << 6 |
// fixed0 << 11 | fixed1 << 21; w = fixed2 | fixed3 << 10 (10-bit variable ids).  The 64 output
// bits are x bits [s, s + 64) of the row, s = 32 word + shift, counted from two zero words in
// front of the row (xs2 = xs - 2 kBM), so no per-run mask or 64-bit shift is computed here.
// NF >= 0: exactly NF fixed elements (no predicated loads for the absent ones: the stage's
// nfix is warp-uniform, so the caller dispatches on it); NF = -1: up to 4, nfix at run time
template <int NF = -1>
__device__ __forceinline__ void run_bits8(const uint32_t* xs, const uint32_t* xs2, int row, const uint4 rr,
                                          uint32_t nfix, uint32_t& lo, uint32_t& hi) {
  uint32_t on = 1;
  const uint32_t f[4] = {(rr.z >> 11) & 1023u, (rr.z >> 21) & 1023u, rr.w & 1023u, (rr.w >> 10) & 1023u};
#pragma unroll
  for (int q = 0; q < 4; ++q)
    if (NF >= 0 ? q < NF : (uint32_t)q < nfix) on &= xs[(f[q] >> 5) * kBM + row] >> (f[q] & 31);
  const uint32_t wi = rr.z & 63u, sh = (rr.z >> 6) & 31u;
  const uint32_t w0 = xs2[wi * kBM + row], w1 = xs2[(wi + 1) * kBM + row], w2 = xs2[(wi + 2) * kBM + row];
  const uint32_t m = 0u - (on & 1u);
  lo |= __funnelshift_r(w0, w1, sh) & rr.x & m;
  hi |= __funnelshift_r(w1, w2, sh) & rr.y & m;
}

// counter-based RNG of SURVEY 8(d): h(s,a,b,c) = sm(sm(sm(s^a)^b)^c)
__device__ __forceinline__ uint64_t d_splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t d_hash(uint64_t s, uint64_t a, uint64_t b, uint64_t c) {
  return d_splitmix64(d_splitmix64(d_splitmix64(s ^ a) ^ b) ^ c);
}

__device__ __forceinline__ float bf16_bits_to_float(uint16_t b) { return __uint_as_float((uint32_t)b << 16); }

// real-valued candidates: this thread's 32 Khatri-Rao entries (K-block half h) of one
// K-block, a[c] = prod_{u in T} p_u for the tuple T at position 32h + c (0 for padding)
__device__ __forceinline__ void real_block(const uint16_t* pr, const uint4 d0, const uint4 d1,
                                           const uint4* __restrict__ runs, int h, float (&a)[32]) {
  const uint32_t nfix = d0.w & 7u, nruns = (d0.w >> 3) & 127u;
  auto fixed_product = [&](const uint4 rr) {
    const uint32_t f[4] = {rr.y & 0xFFFFu, rr.y >> 16, rr.z & 0xFFFFu, rr.z >> 16};
    float pf = 1.0f;
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if ((uint32_t)q < nfix) pf *= bf16_bits_to_float(pr[f[q]]);
    return pf;
  };
  {
    // fast path: run 0 covers this whole half -> 32 consecutive p values
    const uint32_t start = d0.x & 0xFFu, cnt = (d0.x >> 8) & 0xFFu, lo = d0.x >> 16;
    if (nruns >= 1 && start <= (uint32_t)(32 * h) && start + cnt >= (uint32_t)(32 * h + 32)) {
      const float pf = fixed_product(d0);
      const uint32_t base = lo + 32 * h - start;
      const uint32_t* pw = reinterpret_cast<const uint32_t*>(pr) + (base >> 1);
      const bool odd = base & 1u;
      uint32_t wv[17];
#pragma unroll
      for (int i = 0; i < 17; ++i) wv[i] = pw[i];
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        const uint32_t pair = odd ? __funnelshift_r(wv[c], wv[c + 1], 16) : wv[c];
        a[2 * c] = pf * __uint_as_float(pair << 16);
        a[2 * c + 1] = pf * __uint_as_float(pair & 0xFFFF0000u);
      }
      return;
    }
  }
#pragma unroll
  for (int c = 0; c < 32; ++c) a[c] = 0.0f;
  auto apply = [&](const uint4 rr) {
    const uint32_t start = rr.x & 0xFFu, cnt = (rr.x >> 8) & 0xFFu, lo = rr.x >> 16;
    const float pf = fixed_product(rr);
#pragma unroll
    for (int c = 0; c < 32; ++c) {
      const uint32_t off = (uint32_t)(32 * h + c) - start;
      if (off < cnt) a[c] = pf * bf16_bits_to_float(pr[lo + off]);
    }
  };
  if (nruns > 0) apply(d0);
  if (nruns > 1) apply(d1);
  for (uint32_t i = 2; i < nruns; ++i) apply(__ldg(runs + (d0.w >> 10) + (i - 2)));
}

// int8 digit planes, the common stage (both K-blocks of the box pair) fully unrolled: L planes
// x 4 MMAs of K = 32, each plane into its own s32 accumulator (top digit signed); only the
// first MMA of a plane in the first stage starts the accumulator
template <int L, int NT, bool PAIR>
__device__ __forceinline__ void issue_i8_stage(uint32_t tmem, uint32_t a_t, uint32_t sbase, uint32_t boxb, uint32_t issued) {
  constexpr uint32_t id_u = idesc_i8_s32(PAIR ? 2 * kBM : kBM, NT, 0), id_s = idesc_i8_s32(PAIR ? 2 * kBM : kBM, NT, 1);
#pragma unroll
  for (int l = 0; l < L; ++l) {
    const uint64_t bd = sw128_kmajor_desc(sbase + (uint32_t)l * boxb);
    const uint32_t d = tmem + (uint32_t)(l * NT);
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const uint32_t acc = kk ? 1u : issued;
      if constexpr (PAIR) umma_i8_ts_pair(d, a_t + 8u * kk, bd + 2u * kk, l == L - 1 ? id_s : id_u, acc);
      else umma_i8_ts(d, a_t + 8u * kk, bd + 2u * kk, l == L - 1 ? id_s : id_u, acc);
    }
  }
}

// e4m3 limbs: np K-block pairs (1 or 2) x nl limb boxes of the stage, all into the ONE fp32
// accumulator (the limbs of a cell sum exactly: their products with A = 2^-9 are exact in
// fp32); only the stage's first MMA may start the accumulator.  Pair q's A is 32 TMEM columns
// at a_t + 32 q; box (limb l, pair q) sits at slot offset (2 l + q) boxes.
template <int NT, bool PAIR>
__device__ __forceinline__ void issue_f8_stage(uint32_t tmem, uint32_t a_t, uint32_t sbase, uint32_t boxb, uint32_t issued,
                                               int nl, int np) {
  constexpr uint32_t id = idesc_e4m3_f32(PAIR ? 2 * kBM : kBM, NT);
  if (np == 2 && nl == 1) {   // the common stage: 2 pairs x 4 MMAs of K = 32
    const uint64_t bd0 = sw128_kmajor_desc(sbase), bd1 = sw128_kmajor_desc(sbase + boxb);
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t at = a_t + 32u * q + 8u * kk;
        const uint64_t bd = (q ? bd1 : bd0) + 2u * kk;
        if constexpr (PAIR) umma_f8_ts_pair(tmem, at, bd, id, (q | kk) ? 1u : issued);
        else umma_f8_ts(tmem, at, bd, id, (q | kk) ? 1u : issued);
      }
    return;
  }
#pragma unroll 1
  for (int l = 0; l < nl; ++l)
#pragma unroll 1
    for (int q = 0; q < np; ++q) {
      const uint64_t bd = sw128_kmajor_desc(sbase + (uint32_t)(2 * l + q) * boxb);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t acc = (l | q | kk) ? 1u : issued;
        if constexpr (PAIR) umma_f8_ts_pair(tmem, a_t + 32u * q + 8u * kk, bd + 2u * kk, id, acc);
        else umma_f8_ts(tmem, a_t + 32u * q + 8u * kk, bd + 2u * kk, id, acc);
      }
    }
}

// One pipeline stage = KPS consecutive K-blocks of one segment (x L limb boxes of W).
// Ring slot s holds the stage's W boxes in shared memory and its A K-blocks in TMEM;
// FULL(s) completes when the 8 generator warps arrived and the TMA bytes landed, EMPTY(s)
// when the MMAs reading the slot completed (one tcgen05.commit).
// PAIR: the two CTAs of a cluster (launched with cluster dimension 2) take adjacent candidate
// blocks of one column tile and share every W box: each loads half of its NT rows, the
// leader issues cta_group::2 MMAs (M = 256: 128 rows of A in each CTA's TMEM), so one MMA
// instruction covers both SMs and each SM's shared memory carries half the W stream.
// F8 (with I8): the 1-byte planes hold e4m3 limbs of the cells scaled by 2^-s instead of int8
// digits; the generator's A bytes 0x01 are e4m3 2^-9, the MMAs are kind::f8f6f4 into one fp32
// accumulator, F = 2^(s+9) * accumulator; a stage loads and multiplies only the limb boxes its
// column tile needs (the stage record's limb count, 1 almost everywhere on integer-encoded
// instances)
// threads of a kr_gemm launch: F8 runs two more generator teams (warps 10-17, generation only,
// no epilogue): an e4m3 stage is half an int8 3-plane stage's MMA time (cfg3 kernel: 2 teams
// 2.80 ms, 3 teams 2.64 ms, 4 teams 2.60 ms)
template <bool F8>
__host__ __device__ constexpr int kr_threads() { return F8 ? kThreads + 256 : kThreads; }

template <int NT, bool REAL, bool SA = false, bool PAIR = false, bool I8 = false, bool F8 = false>
__global__ void __launch_bounds__(kr_threads<F8>(), 1) kr_gemm_kernel(const __grid_constant__ CUtensorMap tmap, const KrParams p) {
  constexpr int THREADS = kr_threads<F8>();
  constexpr int NTEAM = F8 ? 4 : 2;   // generator teams (the first two also run the epilogue)
  static_assert(!(PAIR && SA), "CTA pairs: not for the per-site annealing launch");
  static_assert(!F8 || I8, "e4m3 limbs run on the 1-byte plane path");
  static_assert(!(I8 && (REAL || SA)), "int8 digit planes: binary candidates, energy / field launches");
  using C = KrCfg<NT, I8>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // SW128 atoms need 1024-byte alignment
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sB = base;
  const int ring = REAL ? p.ring_boxes : C::RING_BOXES;
  const uint32_t sBar = sB + ring * C::BOX;
  const uint32_t acc_full = sBar + 8 * (2 * C::MAXST + 2 * C::MAXA + C::MAXD);
  const uint32_t snap_full = acc_full + 8, snap_empty = acc_full + 16;
  const uint32_t acc_empty = acc_full + 24;                      // cb_iters > 1: epilogue done with TMEM
  const uint32_t tslot = acc_full + 32;
  const uint32_t sQ = (tslot + 16 + 127u) & ~127u;              // 128 doubles: half-sum exchange
  const uint32_t sD = sQ + kBM * 8;                               // I8: descriptor ring (one slot per W stage)
  const uint32_t sX = sD + (uint32_t)C::desc_bytes(p.srec_u4 * (F8 ? 2 : 1), p.desc_lg) + (I8 ? 2u * kBM * 4u : 0u);
  const int MD = 1 << p.desc_lg;   // descriptor ring slots in use (16 or 32), records MD/2 stages ahead
  uint32_t* xs = reinterpret_cast<uint32_t*>(gbase + (sX - base));
  if constexpr (I8) {   // the two zero words in front of every row (run_bits8's window)
    for (int i = threadIdx.x; i < 2 * kBM; i += THREADS) xs[i - 2 * kBM] = 0u;
  }
  uint16_t* prow = reinterpret_cast<uint16_t*>(gbase + (sX - base));   // REAL: p rows [128][pstride]
  double* qpart = reinterpret_cast<double*>(gbase + (sQ - base));
  volatile uint32_t* tslot_g = reinterpret_cast<volatile uint32_t*>(gbase + (tslot - base));
#define FULL(s) (sBar + 8u * (s))
#define EMPTY(s) (sBar + 8u * (C::MAXST + (s)))
#define FULLA(s) (sBar + 8u * (2 * C::MAXST + (s)))
#define EMPTYA(s) (sBar + 8u * (2 * C::MAXST + C::MAXA + (s)))
#define DFULL(s) (sBar + 8u * (2 * C::MAXST + 2 * C::MAXA + (s)))

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // block order: candidate block fastest, then column tile, then K split (concurrent CTAs
  // share W tiles in L2); pairs: cluster c holds candidate blocks 2c', 2c'+1 of one tile
  const uint32_t prank = PAIR ? cluster_ctarank() : 0u;
  const bool leader = !PAIR || prank == 0;
  const int MB = (PAIR || SA || REAL || I8 || p.field_mode || p.n_split > 1 || p.cb_iters < 1) ? 1 : p.cb_iters;
  const int ncb_eff = PAIR ? (p.n_cb + 1) / 2 : (p.n_cb + MB - 1) / MB;
  const int bid = PAIR ? (int)(blockIdx.x / 2) : (int)blockIdx.x;
  const bool sk = PAIR && (!I8 || F8) && p.units != nullptr;   // stream-K unit (see KrParams::units)
  const int4 unit = sk ? __ldg(p.units + bid) : make_int4(0, 0, 0, 0);
  const int sk_part = sk ? (unit.w >> 20) - 1 : -1;
  const int ct_i = (bid / ncb_eff) % p.n_ct;
  const int cb = sk ? 2 * unit.x + (int)prank : PAIR ? 2 * (bid % ncb_eff) + (int)prank : bid % ncb_eff;
  const int ct = sk ? unit.y : (!SA && p.ct_desc) ? p.n_ct - 1 - ct_i : ct_i;
  const int split = sk ? 0 : bid / (ncb_eff * p.n_ct);
  const bool first_range = sk ? unit.z == 0 : split == 0;   // adds the degree-1 cells (counted once)
  const long long b0 = (long long)cb * kBM;
  // MB > 1: this CTA's candidate blocks are cb, cb + ncb_eff, ... (< n_cb)
  const int ntile = MB == 1 ? 1 : (p.n_cb - 1 - cb) / ncb_eff + 1;
  constexpr uint32_t BOXB = PAIR ? C::BOX / 2 : C::BOX;   // shared-memory bytes of one W box per CTA
  // F8: a stage is two K-block pairs (4 K-blocks): 1024 MMA cycles per stage like the bf16
  // kernel's, half the per-stage handshakes of one pair
  const int KPS = REAL ? 1 : F8 ? 4 : C::kps(p.L);
  constexpr int RPS = F8 ? 2 : 1;   // K-block pairs (run records, W boxes per limb) per stage
  // CTA pairs hold half boxes, so the same ring fits twice the stages (TMEM: 256 + 4 x 64 columns)
  // DEC: the int8 launches run decoupled W / A / descriptor rings (for bf16 limbs the single
  // ring measured faster: cfg3 15.2 vs 14.2 M cand/s)
  constexpr bool DEC = I8;
  const int NST = REAL ? C::nst_real(p.L, p.LA, PAIR ? 2 * ring : ring)
                 : F8 ? min(C::MAXST, (PAIR ? 2 * ring : ring) / (RPS * p.L))
                 : DEC ? C::nstw(p.L, PAIR ? 2 * ring : ring)
                       : C::nst_c(p.L, PAIR ? 2 * ring : ring);
  const int ACOLS = REAL ? p.LA * C::A_COLS : KPS * C::A_COLS;   // TMEM columns of A per stage
  const int NSTA = F8 ? ((C::TMEM_COLS - NT) / (KPS * C::A_COLS) >= 8   ? 8   // a power of two
                         : (C::TMEM_COLS - NT) / (KPS * C::A_COLS) >= 4 ? 4
                                                                          : 2)
                 : DEC ? C::nsta(p.L) : NST;                      // A stages (DEC: own ring)
  const int NACC = F8 ? 1 : I8 ? p.L : 1;                          // accumulators in TMEM [0, NACC * NT)
  // F8: the limb count of the stage at K-block kb0 (this column tile's table, in shared memory:
  // a dependent wait on the stage's record here cost 12% at cfg3)
  uint32_t* snl = reinterpret_cast<uint32_t*>(gbase + (sX - base) + (size_t)(p.W + 2) * kBM * 4);
  auto pair_nl = [&](int P) -> int { return (int)((snl[P >> 4] >> (P & 15) * 2) & 3u); };
  auto stage_nl = [&](int kb0, int np) -> int {   // the most limbs of the stage's np pairs
    const int v = np > 1 ? max(pair_nl(kb0 >> 1), pair_nl((kb0 >> 1) + 1)) : pair_nl(kb0 >> 1);
    return v ? v : 1;
  };
  if constexpr (F8)
    for (int i = threadIdx.x; i < p.nl_words; i += THREADS) snl[i] = __ldg(p.nltab + (size_t)ct * p.nl_words + i);
  __shared__ int2 sched[8];          // this CTA's (first K-block, #K-blocks) per segment
  __shared__ int ssa[SA ? kBM : 1];   // annealing: this CTA's decisions for site sa_m
  if (threadIdx.x == 0) {
    // stage range of this split over the tile's whole schedule (segments j = nseg-1 .. 0)
    const int2* gs = p.sched + (size_t)ct * p.nseg;
    int total = 0;
    for (int j = 0; j < p.nseg; ++j) total += (gs[j].y + KPS - 1) / KPS;
    const int per = (total + p.n_split - 1) / p.n_split;
    const int c0 = sk ? unit.z : split * per, c1 = sk ? (unit.w & 0xFFFFF) : min(total, c0 + per);
    int s0 = 0;
    for (int j = p.nseg - 1; j >= 0; --j) {
      const int ns = (gs[j].y + KPS - 1) / KPS;
      const int a = max(s0, c0) - s0, bb = min(s0 + ns, c1) - s0;
      if (bb > a) sched[j] = make_int2(gs[j].x + a * KPS, min(gs[j].y, bb * KPS) - a * KPS);
      else sched[j] = make_int2(gs[j].x, 0);
      s0 += ns;
    }
  }
  const uint32_t stage_bytes = (uint32_t)((I8 ? RPS : KPS) * p.L) * BOXB;
  // segments run in ascending degree order (j = nseg-1 .. 0); in field mode the single
  // accumulator is snapshot after each degree so the energy can weight degree r by 1/r
  const bool snaps = p.field_mode != 0 && !SA;

  if (threadIdx.x == 0) {
    // FULL: the TMA arrive + 8 generator warps (pairs: + the peer's 8, on the leader only)
    for (int s = 0; s < C::MAXST; ++s) { mbar_init(FULL(s), DEC ? 1 : PAIR ? 17 : 9); mbar_init(EMPTY(s), 1); }
    for (int s = 0; s < C::MAXA; ++s) { mbar_init(FULLA(s), (PAIR ? 2 : 1) * (I8 ? 4 : 8)); mbar_init(EMPTYA(s), 1); }
    for (int s = 0; s < C::MAXD; ++s) mbar_init(DFULL(s), 1);
    mbar_init(acc_full, 1);
    mbar_init(snap_full, 1);
    mbar_init(snap_empty, PAIR ? 16 : 8);
    mbar_init(acc_empty, 8);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch_desc(&tmap);
  if (warp == 1) {
    if constexpr (PAIR) tmem_alloc_pair(tslot, C::TMEM_COLS);
    else tmem_alloc(tslot, C::TMEM_COLS);
  }
  // this CTA's candidate bits, column-major xs[w][row] (+2 zero words for window reads).
  // Consecutive threads take consecutive rows of one word (conflict-free stores; the rows'
  // sectors are shared through L1), and XU loads are in flight before the first store, so
  // the staging costs ~1 global latency instead of one per 320 words
  auto stage_x = [&](long long bb0, int tid, int nthr) {
    const int Wp = p.W + 2;
    constexpr int XU = 16;
    for (int i0 = tid; i0 < Wp * kBM; i0 += nthr * XU) {
      uint32_t v[XU];
#pragma unroll
      for (int u = 0; u < XU; ++u) {
        const int i = i0 + u * nthr, r = i % kBM, w = i / kBM;
        v[u] = (w < p.W && bb0 + r < p.B) ? __ldg(p.xbits + (size_t)(bb0 + r) * p.W + w) : 0u;
      }
#pragma unroll
      for (int u = 0; u < XU; ++u) {
        const int i = i0 + u * nthr;
        if (i < Wp * kBM) xs[i] = v[u];   // i == w * kBM + r
      }
    }
  };
  if constexpr (REAL) {
    // this CTA's p rows (bf16), zero past N and past B; +64 slack for window over-reads
    for (int i = threadIdx.x; i < kBM * p.pstride + 64; i += kThreads) {
      const int r = i / p.pstride, c = i % p.pstride;
      uint16_t v = 0;
      if (r < kBM && c < p.N && b0 + r < p.B) v = __ldg(p.preal + (size_t)(b0 + r) * p.N + c);
      prow[i] = v;
    }
  } else {
    stage_x(b0, (int)threadIdx.x, THREADS);
  }
  tc_fence_before();
  if constexpr (PAIR) cluster_sync_all();   // both CTAs' barriers initialised, TMEM allocated
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot_g;
  bool sa_any = true;
  if constexpr (SA) {
    // the Metropolis step of site m for this CTA's chains (SPEC sa_run): apply the
    // previous site's decision to the staged bits, then d = (1 - 2 x_m) g_m, accept iff d <= 0
    // or d < -T ln u.  Every column tile decides identically; tile 0 commits.
    int sv = 0;
    if (threadIdx.x < kBM) {
      const int r = threadIdx.x;
      const long long b = b0 + r;
      if (b < p.B) {
        if (p.sa_prev >= 0) {
          const int sp = p.sa_sprev[b];
          if (sp != 0) {
            const int wi = p.sa_prev >> 5;
            const uint32_t bit = 1u << (p.sa_prev & 31);
            xs[wi * kBM + r] = sp > 0 ? (xs[wi * kBM + r] | bit) : (xs[wi * kBM + r] & ~bit);
            if (ct == 0) {
              if (sp > 0) atomicOr(p.sa_bits + b * p.W + wi, bit);
              else atomicAnd(p.sa_bits + b * p.W + wi, ~bit);
            }
          }
        }
        const int m = p.sa_m;
        const uint32_t xm = (xs[(m >> 5) * kBM + r] >> (m & 31)) & 1u;
        const float g = __ldcg(p.G + b * p.N + m);
        const float d = xm ? -g : g;
        bool acc = d <= 0.0f;
        if (!acc) {   // u < exp(-d/T)  <=>  d < -T ln u  (reading 22)
          const double u = (double)(d_hash(p.sa_seed, 4, (uint64_t)(p.sa_chain0 + b), (uint64_t)p.sa_step) >> 11) * 0x1.0p-53;
          acc = (double)d < -p.sa_T * log(u);
        }
        sv = acc ? (xm ? -1 : 1) : 0;
        if (ct == 0) {
          p.sa_scur[b] = (int8_t)sv;
          if (acc) p.sa_E[b] += (double)d;
        }
      }
      ssa[r] = sv;
    }
    sa_any = __syncthreads_or(sv != 0) != 0;   // no chain of this block moved: G is unchanged
  }

  if (SA && !sa_any) {
  } else if (warp == 0) {
    // ---------------- TMA producer: W limb boxes (NT rows x 64 tuples, SW128) ---------------
    if (lane == 0) {
      int st = 0;                    // ring slot and phase, advanced per stage (no divisions)
      uint32_t ph = 0;
      // I8: the A generator's K-block descriptors, bulk-copied DAHEAD stages ahead of the W
      // boxes into a ring of their own (slot m % MAXD is reused only after the generator is
      // done with stage m - MAXD <= the stage whose W slot was just freed)
      int dj = p.nseg - 1, dkb = 0, dslot = 0;
      auto dskip = [&]() {
        while (dj >= 0 && dkb >= sched[dj].x + sched[dj].y) { --dj; if (dj >= 0) dkb = sched[dj].x; }
      };
      auto dissue = [&]() {
        if (dj < 0) return;
        // the stage's run records (dkb even; RPS consecutive pairs, one bulk copy; the record
        // array carries a zero record past its end for a stage of one pair)
        const uint32_t rbytes = (uint32_t)p.srec_u4 * 16u * RPS;
        mbar_arrive_expect_tx(DFULL(dslot), rbytes);
        bulk_g2s(sD + (uint32_t)dslot * rbytes, p.srec + (size_t)(dkb >> 1) * p.srec_u4, rbytes, DFULL(dslot));
        if (++dslot == MD) dslot = 0;
        dkb += KPS;
        dskip();
      };
      if constexpr (DEC) {
        if (dj >= 0) dkb = sched[dj].x;
        dskip();
        for (int i = 0; i < MD / 2; ++i) dissue();
      }
      for (int it = 0; it < ntile; ++it)   // MB > 1: the same W sequence for every block
      for (int j = p.nseg - 1; j >= 0; --j) {
        const int2 s = sched[j];
        for (int kb0 = s.x; kb0 < s.x + s.y; kb0 += KPS) {
          const int nkb = min(KPS, s.x + s.y - kb0);
          mbar_wait(EMPTY(st), ph ^ 1u);
          if constexpr (DEC) dissue();
          if constexpr (I8) {   // one box per digit plane: the K-block pair (kb0, kb0 + 1), kb0 even
            // pairs in this stage (a segment's K-block count may be odd: its last pair then holds
            // one K-block of tuples and one of zero padding, multiplied whole)
            const int np = F8 ? ((nkb + 1) >> 1) : 1;
            const int nl = F8 ? stage_nl(kb0, np) : p.L;
            if (leader) mbar_arrive_expect_tx(FULL(st), (uint32_t)(nl * np) * C::BOX);
            for (int l = 0; l < nl; ++l)
              for (int q = 0; q < np; ++q) {   // box (limb l, pair q) at slot offset (l RPS + q)
                const int box = (l * p.n_ct + ct) * (p.n_kb >> 1) + (kb0 >> 1) + q;
                const uint32_t dst = sB + st * stage_bytes + (uint32_t)(l * RPS + q) * BOXB;
                if constexpr (PAIR) tma_load_3d_pair(dst, &tmap, mapa_shared(FULL(st), 0), 0, (int)prank * (NT / 2), box);
                else tma_load_3d(dst, &tmap, FULL(st), 0, 0, box);
              }
          } else {
            if (leader) mbar_arrive_expect_tx(FULL(st), (uint32_t)(nkb * p.L) * C::BOX);   // pairs: both halves
            for (int q = 0; q < nkb; ++q)
              for (int l = 0; l < p.L; ++l) {
                // W is tile-blocked: box (l, ct, kb) is one contiguous NT x 64 block
                const int box = (l * p.n_ct + ct) * p.n_kb + kb0 + q;
                const uint32_t dst = sB + st * stage_bytes + (uint32_t)(q * p.L + l) * BOXB;
                if constexpr (PAIR) tma_load_3d_pair(dst, &tmap, mapa_shared(FULL(st), 0), 0, (int)prank * (NT / 2), box);
                else tma_load_3d(dst, &tmap, FULL(st), 0, 0, box);
              }
          }
          if (++st == NST) { st = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: D[tmem] += A[tmem] * B[smem] -------------------------------
    // The whole warp runs the loop, so descriptors are warp-uniform and stay in uniform
    // registers; one elected lane issues the MMAs and commits.
    if (leader) {
      constexpr uint32_t idesc = idesc_bf16_f32(PAIR ? 2 * kBM : kBM, NT);
      int snap = 0;
      int st = 0, sa = 0;            // W and A ring slots and phases, advanced per stage
      uint32_t ph = 0, pha = 0;
      uint32_t issued = 0;
      for (int it = 0; it < ntile; ++it) {
      if (it > 0) {   // the previous block's epilogue has read the accumulator
        mbar_wait(acc_empty, (uint32_t)((it - 1) & 1));
        tc_fence_after();
        issued = 0;
      }
      for (int j = p.nseg - 1; j >= 0; --j) {
        const int2 s = sched[j];
        for (int kb0 = s.x; kb0 < s.x + s.y; kb0 += KPS) {
          const int nkb = min(KPS, s.x + s.y - kb0);
          const int nl = F8 ? stage_nl(kb0, (nkb + 1) >> 1) : 0;
          mbar_wait(FULL(st), ph);
          if (DEC) mbar_wait(FULLA(sa), pha);
          tc_fence_after();
          if (elect_one()) {
            if constexpr (F8) {
              issue_f8_stage<NT, PAIR>(tmem, tmem + (uint32_t)(NT + sa * KPS * C::A_COLS), sB + st * stage_bytes, BOXB,
                                       issued, nl, (nkb + 1) >> 1);
            } else if constexpr (I8) {   // KPS K-blocks x L digit planes, each into its own accumulator
              const uint32_t a_t = tmem + (uint32_t)(p.L * NT + sa * KPS * C::A_COLS);
              const uint32_t sbase = sB + st * stage_bytes;
              if (nkb == 2 && p.L == 3) issue_i8_stage<3, NT, PAIR>(tmem, a_t, sbase, BOXB, issued);
              else if (nkb == 2 && p.L == 2) issue_i8_stage<2, NT, PAIR>(tmem, a_t, sbase, BOXB, issued);
              else if (nkb == 2 && p.L == 1) issue_i8_stage<1, NT, PAIR>(tmem, a_t, sbase, BOXB, issued);
              else
              for (int l = 0; l < p.L; ++l) {
                const uint64_t bdesc = sw128_kmajor_desc(sbase + (uint32_t)l * BOXB);
                const uint32_t id = l == p.L - 1 ? idesc_i8_s32(PAIR ? 2 * kBM : kBM, NT, 1)    // top digit signed
                                                 : idesc_i8_s32(PAIR ? 2 * kBM : kBM, NT, 0);
                const uint32_t d = tmem + (uint32_t)(l * NT);
                for (int q = 0; q < nkb; ++q)
#pragma unroll
                  for (int k = 0; k < kBK / 32; ++k) {   // 32 bytes of K per MMA: 8 A columns, 2 descriptor units
                    const uint32_t kk = (uint32_t)(2 * q + k);
                    if constexpr (PAIR) umma_i8_ts_pair(d, a_t + 8u * kk, bdesc + 2u * kk, id, issued | kk);
                    else umma_i8_ts(d, a_t + 8u * kk, bdesc + 2u * kk, id, issued | kk);
                  }
              }
            } else if constexpr (REAL) {   // one K-block: LA limb tiles of A x L limb boxes of W
              for (int la = 0; la < p.LA; ++la) {
                const uint32_t a_t = tmem + (uint32_t)(NT + st * ACOLS + la * C::A_COLS);
                for (int l = 0; l < p.L; ++l) {
                  const uint64_t bdesc = sw128_kmajor_desc(sB + st * stage_bytes + (uint32_t)l * BOXB);
#pragma unroll
                  for (int k = 0; k < kBK / 16; ++k) {
                    if constexpr (PAIR) umma_bf16_ts_pair(tmem, a_t + 8u * k, bdesc + 2u * k, idesc, issued | (uint32_t)(la | l | k));
                    else umma_bf16_ts(tmem, a_t + 8u * k, bdesc + 2u * k, idesc, issued | (uint32_t)(la | l | k));
                  }
                }
              }
            } else if (p.L == 1 && nkb == 2 && KPS == 2) {   // the common stage, fully unrolled
              const uint32_t a_t = tmem + (uint32_t)(NT + (DEC ? sa : st) * 2 * C::A_COLS);
              const uint64_t bdesc = sw128_kmajor_desc(sB + st * stage_bytes);
#pragma unroll
              for (int q = 0; q < 2; ++q)
#pragma unroll
                for (int k = 0; k < kBK / 16; ++k) {
                  const uint32_t at = a_t + (uint32_t)(q * C::A_COLS) + 8u * k;
                  const uint64_t bd = bdesc + (uint64_t)((q * BOXB) >> 4) + 2u * k;
                  if constexpr (PAIR) umma_bf16_ts_pair(tmem, at, bd, idesc, issued | (uint32_t)(q | k));
                  else umma_bf16_ts(tmem, at, bd, idesc, issued | (uint32_t)(q | k));
                }
            } else {
              for (int q = 0; q < nkb; ++q) {
                const uint32_t a_t = tmem + (uint32_t)(NT + ((DEC ? sa : st) * KPS + q) * C::A_COLS);
                for (int l = 0; l < p.L; ++l) {
                  const uint64_t bdesc = sw128_kmajor_desc(sB + st * stage_bytes + (uint32_t)(q * p.L + l) * BOXB);
#pragma unroll
                  for (int k = 0; k < kBK / 16; ++k) {
                    if constexpr (PAIR) umma_bf16_ts_pair(tmem, a_t + 8u * k, bdesc + 2u * k, idesc, issued | (uint32_t)(q | l | k));
                    else umma_bf16_ts(tmem, a_t + 8u * k, bdesc + 2u * k, idesc, issued | (uint32_t)(q | l | k));
                  }
                }
              }
            }
            if constexpr (PAIR) umma_commit_pair(EMPTY(st), 3);
            else umma_commit(EMPTY(st));
            if constexpr (DEC) {
              if constexpr (PAIR) umma_commit_pair(EMPTYA(sa), 3);
              else umma_commit(EMPTYA(sa));
            }
          }
          __syncwarp();
          issued = 1;
          if (++st == NST) { st = 0; ph ^= 1u; }
          if (DEC && ++sa == NSTA) { sa = 0; pha ^= 1u; }
        }
        if (snaps && j > 0) {  // hand the degree-(k-j) partial sum to the epilogue warps
          if (elect_one()) {
            if constexpr (PAIR) {
              if (issued) umma_commit_pair(snap_full, 3);
              else { mbar_arrive(snap_full); mbar_arrive_remote(mapa_shared(snap_full, 1)); }
            } else {
              if (issued) umma_commit(snap_full);
              else mbar_arrive(snap_full);
            }
          }
          __syncwarp();
          mbar_wait(snap_empty, (uint32_t)(snap & 1));
          tc_fence_after();
          ++snap;
        }
      }
      if (elect_one()) {
        if constexpr (PAIR) {
          if (issued) umma_commit_pair(acc_full, 3);
          else { mbar_arrive(acc_full); mbar_arrive_remote(mapa_shared(acc_full, 1)); }
        } else {
          if (issued) umma_commit(acc_full);
          else mbar_arrive(acc_full);
        }
      }
      __syncwarp();
      }   // tiles
    }
  } else {
    // ---------------- A generator (warps 2..9), then epilogue --------------------------------
    // team h = (w-2)/4 builds K-block h of every stage; warp w of a team serves TMEM lane
    // quarter q = w % 4 (rows 32q..32q+31) and writes its rows of A with tcgen05.st.
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    const int row = q * 32 + lane;   // candidate row within the block == TMEM lane
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    const int c_lo = h * (NT / 2), c_hi = (h + 1) * (NT / 2);   // this warp's epilogue columns
    double S[8];                     // S[r]: sum_m x_m F_m over this warp's columns after degree r
    int nsnap = 0;
    int n = 0;                       // stage counter (same sequence as the MMA issuer)
    int gst = 0;                     // binary path: A slot and phase, advanced per stage
    uint32_t gph = 0;
    int gn = 0;                      // I8: stage counter (the teams alternate stages)
    bool any = false;                // has any MMA been issued yet (else F = 0)
    const uint16_t* prow_r = prow + (size_t)row * (REAL ? p.pstride : 0);
    // I8: F_m = qscale * sum_l 256^l acc_l[m], exact in int64
    auto load_i8 = [&](int c0, long long (&v)[32]) {
      uint32_t r[32];
      tmem_ld32(lane_base + (uint32_t)c0, r);
      tmem_ld_wait();
#pragma unroll
      for (int c = 0; c < 32; ++c) v[c] = (long long)(int32_t)r[c];
      for (int l = 1; l < p.L; ++l) {
        tmem_ld32(lane_base + (uint32_t)(l * NT + c0), r);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] += (long long)(int32_t)r[c] << (8 * l);
      }
    };
    auto xsum = [&](void) -> double {  // sum over this warp's columns of x_m * F_m (p_m * F_m)
      if constexpr (I8 && !F8) {
        long long acc = 0;
        for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
          const int mbase = ct * NT + c0;
          long long v[32];
          load_i8(c0, v);
          const uint32_t xw = (mbase >> 5) < p.W ? xs[(mbase >> 5) * kBM + row] : 0u;
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if ((xw >> c) & 1u) acc += v[c];
        }
        return (double)acc * p.qscale;
      }
      double acc = 0.0;
      for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
        const int mbase = ct * NT + c0;
        uint32_t r[32];
        tmem_ld32(lane_base + (uint32_t)c0, r);
        tmem_ld_wait();
        if constexpr (REAL) {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (mbase + c < p.N) acc += (double)bf16_bits_to_float(prow_r[mbase + c]) * (double)__uint_as_float(r[c]);
        } else {
          const uint32_t xw = (mbase >> 5) < p.W ? xs[(mbase >> 5) * kBM + row] : 0u;
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if ((xw >> c) & 1u) acc += (double)__uint_as_float(r[c]);
        }
      }
      if constexpr (F8) acc *= (double)p.fscale;
      return acc;
    };
    for (int it = 0; it < ntile; ++it) {
    const long long b0t = b0 + (long long)it * ncb_eff * kBM;   // this block's first candidate
    if (it > 0) {   // every warp is done with the previous block's bits: stage this block's
      named_bar_sync(1, 256);
      stage_x(b0t, (int)threadIdx.x - 64, 256);
      named_bar_sync(1, 256);
      any = false;
      nsnap = 0;
    }
    for (int j = p.nseg - 1; j >= 0; --j) {
      const int2 s = sched[j];
      if constexpr (REAL) {
        // one K-block per stage; both teams build it (team h: tuple positions 32h..32h+31)
        uint4 d0 = make_uint4(0, 0, 0, 0), d1 = d0;
        if (s.y > 0) { d0 = __ldg(p.kdesc + 2 * s.x); d1 = __ldg(p.kdesc + 2 * s.x + 1); }
        for (int kb = s.x; kb < s.x + s.y; ++kb, ++n) {
          uint4 n0 = d0, n1 = d1;
          if (kb + 1 < s.x + s.y) { n0 = __ldg(p.kdesc + 2 * (kb + 1)); n1 = __ldg(p.kdesc + 2 * (kb + 1) + 1); }
          const int st = n % NST;
          mbar_wait(EMPTY(st), (uint32_t)(((n / NST) & 1) ^ 1));
          tc_fence_after();
          float a[32];
          real_block(prow_r, d0, d1, p.runs, h, a);
          for (int la = 0; la < p.LA; ++la) {   // exact bf16 limb split of the fp32 products
            uint32_t w[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) {
              const __nv_bfloat162 hv = __floats2bfloat162_rn(a[2 * c], a[2 * c + 1]);   // one packed cvt
              const uint32_t u = *reinterpret_cast<const uint32_t*>(&hv);
              w[c] = u;
              a[2 * c] -= __uint_as_float(u << 16);
              a[2 * c + 1] -= __uint_as_float(u & 0xFFFF0000u);
            }
            tmem_st16(lane_base + (uint32_t)(NT + st * ACOLS + la * C::A_COLS + 16 * h), w);
          }
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR && !leader) mbar_arrive_remote(mapa_shared(FULL(st), 0));
            else mbar_arrive(FULL(st));
          }
          d0 = n0;
          d1 = n1;
        }
      } else if constexpr (DEC) {
        // 1-byte planes: the NTEAM teams take whole stages in turn (team h: stages n with
        // n % NTEAM == h; NTEAM = 2 for int8 digits, 4 for e4m3 limbs).  A team decodes the
        // K-blocks of its stage from the stage's run records (TMA bulk copy, MD/2 stages ahead,
        // DFULL ring) and writes each K-block pair with ONE tcgen05.st (32 columns), so one
        // store round trip (~400 cycles) covers two K-blocks and each team has NTEAM stage
        // times per stage.  FULLA counts the one team's 4 warps (pairs: 8).  The team visits
        // only its own stages: the absolute stage counter n gives the ring slots and phases
        // directly (MD and NSTA are powers of two), so the other teams' stages cost no loop
        // iterations.
        const uint4* dsm = reinterpret_cast<const uint4*>(gbase + (sD - base));
        const int nstages = (s.y + KPS - 1) / KPS;
        const int lg_a = NSTA == 8 ? 3 : NSTA == 4 ? 2 : NSTA == 2 ? 1 : 0;
        static_assert(C::MAXD == 32 && C::MAXST <= 8, "descriptor ring: 16 or 32 slots, >= MD / 2 + MAXST");
        for (int i = ((h - gn) % NTEAM + NTEAM) % NTEAM; i < nstages; i += NTEAM) {
          {
            const int n = gn + i;
            const int wst = n & (MD - 1), gst = n & (NSTA - 1);
            const uint32_t wph = (uint32_t)(n >> p.desc_lg) & 1u, gph = (uint32_t)(n >> lg_a) & 1u;
            mbar_wait(DFULL(wst), wph);
            // the K-block pair's A bits from its run record (two K-blocks: l0 h0 | l1 h1)
            auto decode = [&](const uint4* rec, uint32_t& l0, uint32_t& h0, uint32_t& l1, uint32_t& h1) {
              const uint4 hd = rec[0];
              if (p.exp & 1) { l0 = hd.x * (uint32_t)row; h0 = l0 ^ hd.y; l1 = h0 + 1; h1 = l1 * 3u; return; }
              if (hd.z == 1) {   // e.g. order 3's degree-3 part: one fixed element per run
#pragma unroll 1
                for (uint32_t i = 0; i < hd.x; ++i) run_bits8<1>(xs, xs - 2 * kBM, row, rec[1 + i], 1, l0, h0);
#pragma unroll 1
                for (uint32_t i = 0; i < hd.y; ++i) run_bits8<1>(xs, xs - 2 * kBM, row, rec[1 + hd.x + i], 1, l1, h1);
              } else if (hd.z == 2) {   // order 4's degree-4 part
#pragma unroll 1
                for (uint32_t i = 0; i < hd.x; ++i) run_bits8<2>(xs, xs - 2 * kBM, row, rec[1 + i], 2, l0, h0);
#pragma unroll 1
                for (uint32_t i = 0; i < hd.y; ++i) run_bits8<2>(xs, xs - 2 * kBM, row, rec[1 + hd.x + i], 2, l1, h1);
              } else if (hd.z == 0) {
#pragma unroll 1
                for (uint32_t i = 0; i < hd.x; ++i) run_bits8<0>(xs, xs - 2 * kBM, row, rec[1 + i], 0, l0, h0);
#pragma unroll 1
                for (uint32_t i = 0; i < hd.y; ++i) run_bits8<0>(xs, xs - 2 * kBM, row, rec[1 + hd.x + i], 0, l1, h1);
              } else {
#pragma unroll 1
                for (uint32_t i = 0; i < hd.x; ++i) run_bits8(xs, xs - 2 * kBM, row, rec[1 + i], hd.z, l0, h0);
#pragma unroll 1
                for (uint32_t i = 0; i < hd.y; ++i) run_bits8(xs, xs - 2 * kBM, row, rec[1 + hd.x + i], hd.z, l1, h1);
              }
            };
            const uint4* rec = dsm + (size_t)wst * p.srec_u4 * RPS;
            const int np = F8 ? ((min(KPS, s.y - i * KPS) + 1) >> 1) : 1;   // pairs in this stage
            uint32_t l0 = 0, h0 = 0, l1 = 0, h1 = 0;
            decode(rec, l0, h0, l1, h1);
            uint32_t w[32];   // the K-block pair's bytes in the planes' permuted K order
            expand_bytes64(((uint64_t)h0 << 32) | l0, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
            expand_bytes64(((uint64_t)h1 << 32) | l1, *reinterpret_cast<uint32_t(*)[16]>(&w[16]));
            mbar_wait(EMPTYA(gst), gph ^ 1u);
            tc_fence_after();
            const uint32_t a_col = lane_base + (uint32_t)(NACC * NT + gst * KPS * C::A_COLS);
            if (!(p.exp & 2)) tmem_st32(a_col, w);
            else {   // keep w live
              uint32_t x = 0;
#pragma unroll
              for (int c = 0; c < 32; ++c) x ^= w[c];
              if (x == 0x9E3779B9u) xs[0] = 0u;
            }
            if (F8 && np > 1) {   // the stage's second pair: 32 TMEM columns further
              tmem_st_wait();    // (w's registers are the source of the store above)
              l0 = h0 = l1 = h1 = 0;
              decode(rec + p.srec_u4, l0, h0, l1, h1);
              expand_bytes64(((uint64_t)h0 << 32) | l0, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
              expand_bytes64(((uint64_t)h1 << 32) | l1, *reinterpret_cast<uint32_t(*)[16]>(&w[16]));
              if (!(p.exp & 2)) tmem_st32(a_col + 32u, w);
            }
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (PAIR && !leader) mbar_arrive_remote(mapa_shared(FULLA(gst), 0));
              else mbar_arrive(FULLA(gst));
            }
          }
        }
        gn += nstages;
      } else {
      // this team's K-block descriptors, prefetched three stages ahead (d: this stage, e, f:
      // the next two)
      const int kend = s.x + s.y;
      auto ldk = [&](int kb, uint4& a, uint4& b) {
        if (kb < kend) { a = __ldg(p.kdesc + 2 * kb); b = __ldg(p.kdesc + 2 * kb + 1); }
      };
      uint4 d0 = make_uint4(0, 0, 0, 0), d1 = d0, e0 = d0, e1 = d0, f0 = d0, f1 = d0;
      ldk(s.x + h, d0, d1);
      ldk(s.x + h + KPS, e0, e1);
      ldk(s.x + h + 2 * KPS, f0, f1);
      for (int kb0 = s.x; kb0 < kend; kb0 += KPS) {
        const int kb = kb0 + h;                       // this team's K-block of the stage
        const bool mine = h < KPS && kb < kend;
        uint4 n0 = f0, n1 = f1;
        ldk(kb + 3 * KPS, n0, n1);
        const int st = gst;                           // A slot (== the W slot)
        // the A bits depend only on the candidates: computed before the slot frees up
        const uint64_t bits = mine ? block_bits(xs, row, d0, d1, p.runs) : 0ull;
        mbar_wait(EMPTY(st), gph ^ 1u);
        if (++gst == NSTA) { gst = 0; gph ^= 1u; }
        if (mine) {
          tc_fence_after();
          uint32_t w[32];
          expand32((uint32_t)bits, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
          expand32((uint32_t)(bits >> 32), *reinterpret_cast<uint32_t(*)[16]>(&w[16]));
          tmem_st32(lane_base + (uint32_t)(NT + (st * KPS + h) * C::A_COLS), w);
          tmem_st_wait();
          tc_fence_before();
        }
        __syncwarp();
        if (lane == 0) {
          if (PAIR && !leader) mbar_arrive_remote(mapa_shared(FULL(st), 0));
          else mbar_arrive(FULL(st));
        }
        d0 = e0;
        d1 = e1;
        e0 = f0;
        e1 = f1;
        f0 = n0;
        f1 = n1;
      }
      }
      any = any || s.y > 0;
      if (snaps && j > 0 && h < 2) {
        mbar_wait(snap_full, (uint32_t)(nsnap & 1));
        tc_fence_after();
        S[nsnap] = any ? xsum() : 0.0;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (PAIR && !leader) mbar_arrive_remote(mapa_shared(snap_empty, 0));
          else mbar_arrive(snap_empty);
        }
        ++nsnap;
      }
    }

    if (h >= 2) continue;   // generation-only team (F8)
    // ---------------- epilogue: fields, energy partial (this warp's column half) ---------------
    mbar_wait(acc_full, (uint32_t)(it & 1));
    tc_fence_after();
    const long long b = b0t + row;
    const bool live = b < p.B;
    double sfin = 0.0, sp = 0.0;
    for (int c0 = c_lo; c0 < c_hi; c0 += 32) {
      const int mbase = ct * NT + c0;
      const uint32_t xw = REAL ? 0u : ((mbase >> 5) < p.W ? xs[(mbase >> 5) * kBM + row] : 0u);
      // the chunk's degree-1 cells (counted once: split 0), 8 vector loads issued before the
      // accumulator is read (p1 is Npad floats, mbase a multiple of 32)
      float pmv[32];
#pragma unroll
      for (int c = 0; c < 32; c += 4) {
        const float4 v4 = first_range ? __ldg(reinterpret_cast<const float4*>(p.p1 + mbase + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
        pmv[c] = v4.x; pmv[c + 1] = v4.y; pmv[c + 2] = v4.z; pmv[c + 3] = v4.w;
      }
      float g[32];
      if constexpr (I8 && !F8) {   // exact integer field; one rounding to fp32 after adding the degree-1 cell
        long long v[32];
        if (any) load_i8(c0, v);
        else {
#pragma unroll
          for (int c = 0; c < 32; ++c) v[c] = 0;
        }
        // split-K partial fields stay exact: doubles, summed in a fixed order by splitk_reduce
        double* gdp = (p.field_mode && live && p.n_split > 1)
                          ? reinterpret_cast<double*>(p.G) + ((size_t)split * p.B + b) * p.N + mbase : nullptr;
#pragma unroll
        for (int c = 0; c < 32; ++c) {
          const double vd = (double)v[c] * p.qscale;
          const float pm = pmv[c];
          g[c] = (float)(vd + (double)pm);
          if (gdp && mbase + c < p.N) gdp[c] = vd + (double)pm;
          if ((xw >> c) & 1u) {
            sfin += vd;
            sp += (double)pm;
          }
        }
      }
      else {
      uint32_t r[32];
      if (any) {
        tmem_ld32(lane_base + (uint32_t)c0, r);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int c = 0; c < 32; ++c) r[c] = 0u;
      }
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const float v = F8 ? __uint_as_float(r[c]) * p.fscale : __uint_as_float(r[c]);
        const float pm = pmv[c];   // degree 1 counted once
        g[c] = v + pm;
        if constexpr (REAL) {
          const double pw = mbase + c < p.N ? (double)bf16_bits_to_float(prow_r[mbase + c]) : 0.0;
          sfin += pw * (double)v;
          sp += pw * (double)pm;
        } else if ((xw >> c) & 1u) {
          sfin += (double)v;
          sp += (double)pm;
        }
      }
      }
      if constexpr (SA) {   // G[b, j] += s_b * (field of P_m)[j]; column m is unchanged
        const int sv = ssa[row];
        if (live && sv != 0) {
          const float sf = (float)sv;
          float* gout = p.G + (size_t)b * p.N + mbase;
          const int nvalid = min(32, p.N - mbase);
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (mbase + c == p.sa_m) g[c] = 0.0f;
          if (nvalid == 32 && ((reinterpret_cast<uintptr_t>(gout) & 15) == 0)) {
#pragma unroll
            for (int c = 0; c < 32; c += 4) {
              float4 o = *reinterpret_cast<float4*>(gout + c);
              o.x += sf * g[c]; o.y += sf * g[c + 1]; o.z += sf * g[c + 2]; o.w += sf * g[c + 3];
              *reinterpret_cast<float4*>(gout + c) = o;
            }
          } else {
#pragma unroll
            for (int c = 0; c < 32; ++c)
              if (c < nvalid) gout[c] += sf * g[c];
          }
        }
      } else if (p.field_mode && live && !(I8 && !F8 && p.n_split > 1)) {
        float* gout = p.G + ((size_t)split * p.B + b) * p.N + mbase;
        int nvalid = min(32, p.N - mbase);
        if (sk_part >= 0) {   // a K range of a split tile: its partial fields, every column of the tile
          gout = p.skG + ((size_t)sk_part * 2 * kBM + prank * kBM + row) * NT + (mbase - ct * NT);
          nvalid = 32;
        }
        if (nvalid == 32 && ((reinterpret_cast<uintptr_t>(gout) & 15) == 0)) {
#pragma unroll
          for (int c = 0; c < 32; c += 4) *reinterpret_cast<float4*>(gout + c) = make_float4(g[c], g[c + 1], g[c + 2], g[c + 3]);
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if (c < nvalid) gout[c] = g[c];
        }
      }
    }
    if (MB > 1) {   // the accumulator is free for the next block's MMAs
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
    }
    if constexpr (!SA) {
    double qsum;
    if (snaps) {
      // S[0] = after degree 2, S[1] = after degree 3, ..., sfin = after degree k
      qsum = p.wp * sp;
      double prev = 0.0;
      for (int t = 0; t <= nsnap; ++t) {
        const double cur = t < nsnap ? S[t] : sfin;
        qsum += p.wdeg[t + 2] * (cur - prev);
        prev = cur;
      }
    } else {
      qsum = sfin + sp;
    }
    // combine the two column halves in a fixed order (deterministic, no atomics)
    if (h == 1) qpart[row] = qsum;
    named_bar_sync(1, 256);
    if (h == 0 && live) {
      if (sk_part >= 0) p.skQ[(size_t)sk_part * 2 * kBM + prank * kBM + row] = qsum + qpart[row];
      else p.Q[((size_t)split * p.n_ct + ct) * p.B + b] = qsum + qpart[row];
    }
    }
    }   // tiles
  }
#undef FULL
#undef EMPTY
#undef FULLA
#undef EMPTYA
#undef DFULL
  tc_fence_before();
  if constexpr (PAIR) {
    cluster_sync_all();   // the leader's last MMAs wrote both CTAs' TMEM
    if (warp == 1) tmem_dealloc_pair(tmem, C::TMEM_COLS);
  } else {
    __syncthreads();
    if (warp == 1) tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ------------------------------------------------------------------------------------------
// u8 candidates (row-major B x N, nonzero = 1) -> bit rows [B][W]
__global__ void pack_x_kernel(const uint8_t* __restrict__ X, long long B, int N, int W, uint32_t* __restrict__ bits) {
  const long long total = B * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / W;
    const int w = (int)(i % W);
    const uint8_t* src = X + b * N + (long long)w * 32;
    const int n = min(32, N - w * 32);
    uint32_t v = 0;
    for (int j = 0; j < n; ++j) v |= (uint32_t)(src[j] != 0) << j;
    bits[i] = v;
  }
}

// the same for N % 32 == 0 and a 16-byte aligned X: rows are whole words, so the batch is one
// flat stream of 16-byte chunks; lane l loads chunk l of its warp's 32 (coalesced 512 B per
// load), turns it into a 16-bit nonzero mask, and the even lane joins its odd neighbour's
// mask into one output word (flat word c/2 == row b, word w)
__global__ void pack_x16_kernel(const uint4* __restrict__ X, long long nchunks, uint32_t* __restrict__ bits) {
  const int lane = threadIdx.x & 31;
  const long long warp = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long base = warp * 32; base < nchunks; base += nwarps * 32) {
    const long long c = base + lane;
    uint32_t m = 0;
    if (c < nchunks) {
      const uint4 v = X[c];
      const uint32_t q[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        // 0xFF per nonzero byte -> byte k of (.. & 0x08040201) holds 2^k -> byte sum = the 4-bit mask
        const uint32_t ne = __vcmpne4(q[k], 0u) & 0x08040201u;
        m |= ((ne * 0x01010101u) >> 24) << (4 * k);
      }
    }
    const uint32_t hi = __shfl_down_sync(0xFFFFFFFFu, m, 1);
    if (!(lane & 1) && c < nchunks) bits[c >> 1] = m | (hi << 16);
  }
}

// packed candidates (hobo_*_bits): the caller's rows of W words, bit m of word m/32; the bits
// past N are cleared here, so the generator and the epilogue masks see the same rows as
// pack_x_kernel would produce
__global__ void mask_bits_kernel(const uint32_t* __restrict__ in, long long B, int N, int W, uint32_t* __restrict__ bits) {
  const long long total = B * W;
  const uint32_t last = (N & 31) ? ((1u << (N & 31)) - 1u) : 0xFFFFFFFFu;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const uint32_t v = in[i];
    bits[i] = ((int)(i % W) == W - 1) ? (v & last) : v;
  }
}

// split-K: sum the per-split partials in a fixed order (deterministic)
// (gp_double: the int8 path's exact partials, one rounding to fp32 after the sum)
__global__ void splitk_reduce_kernel(const float* __restrict__ Gp, float* __restrict__ G, long long nG,
                                     const double* __restrict__ Qp, double* __restrict__ Q, long long nQ, int n_split,
                                     int gp_double) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nG; i += stride) {
    if (gp_double) {
      double g = 0.0;
      for (int s = 0; s < n_split; ++s) g += reinterpret_cast<const double*>(Gp)[(size_t)s * nG + i];
      G[i] = (float)g;
      continue;
    }
    float g = 0.0f;
    for (int s = 0; s < n_split; ++s) g += Gp[(size_t)s * nG + i];
    G[i] = g;
  }
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nQ; i += stride) {
    double q = 0.0;
    for (int s = 0; s < n_split; ++s) q += Qp[(size_t)s * nQ + i];
    Q[i] = q;
  }
}

// stream-K: the split tiles' fields and energy partials, their K ranges summed in K order
// (deterministic).  tiles[s] = {candidate-block pair, column tile, first part, #parts}.
__global__ void sk_reduce_kernel(const int4* __restrict__ tiles, int ntiles, const float* __restrict__ skG,
                                 const double* __restrict__ skQ, float* __restrict__ G, double* __restrict__ Q,
                                 long long B, int N, int NT, int field) {
  const long long per_tile = 2LL * kBM * (NT / 4);   // float4 groups of one tile
  const long long total = (long long)ntiles * per_tile;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const int4 t = __ldg(tiles + i / per_tile);
    const long long e = i % per_tile;
    const int r = (int)(e / (NT / 4)), c4 = (int)(e % (NT / 4)) * 4;
    const long long b = 2LL * kBM * t.x + r;
    if (b >= B) continue;
    const int m = t.y * NT + c4;
    if (field && m < N) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int q = 0; q < t.w; ++q) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(skG + ((size_t)(t.z + q) * 2 * kBM + r) * NT + c4));
        a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
      }
      float* g = G + b * N + m;
      if (m + 3 < N && (reinterpret_cast<uintptr_t>(g) & 15) == 0) *reinterpret_cast<float4*>(g) = a;
      else {
        const float av[4] = {a.x, a.y, a.z, a.w};
        for (int c = 0; c < 4 && m + c < N; ++c) g[c] = av[c];
      }
    }
    if (c4 == 0) {
      double qs = 0.0;
      for (int q = 0; q < t.w; ++q) qs += skQ[(size_t)(t.z + q) * 2 * kBM + r];
      Q[(size_t)t.y * B + b] = qs;
    }
  }
}

// signed-orderable key of (E, global index): lexicographic min == min of the u64
__device__ __forceinline__ unsigned long long argmin_key(float e, unsigned long long idx) {
  if (e == 0.0f) e = 0.0f;  // -0 -> +0
  int i = __float_as_int(e);
  i ^= (i >> 31) & 0x7FFFFFFF;
  const uint32_t u = (uint32_t)i ^ 0x80000000u;
  return ((unsigned long long)u << 32) | (idx & 0xFFFFFFFFull);
}

// E_b = (sum_ct Q[ct][b]) / lcm in double (exact for integer instances), one rounding to fp32
__device__ __forceinline__ float combine_q(const double* __restrict__ Q, int n_ct, long long B, long long b, double lcm) {
  double s = 0.0;
  for (int c = 0; c < n_ct; ++c) s += Q[(size_t)c * B + b];
  return (float)(s / lcm);
}

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
    v = w < v ? w : v;
  }
  return v;
}

// block min of the keys -> one atomicMin on best_key[0]; a NaN energy clears best_key[1]
// (NaN is an error, reported by the host after the combine)
__device__ __forceinline__ void block_argmin(unsigned long long key, bool nan, unsigned long long* best_key) {
  __shared__ unsigned long long red[32];
  __shared__ int any_nan;
  if (threadIdx.x == 0) any_nan = 0;
  __syncthreads();
  if (nan) any_nan = 1;
  key = warp_min_u64(key);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = key;
  __syncthreads();
  if (threadIdx.x < 32) {
    key = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : ~0ull;
    key = warp_min_u64(key);
    if (threadIdx.x == 0) {
      atomicMin(best_key, key);
      if (any_nan) atomicAnd(best_key + 1, 0ull);
    }
  }
}

// E_b = (sum_ct Q[ct][b]) / lcm; argmin via warp shuffles -> smem block min -> one atomicMin
__global__ void finalize_kernel(const double* __restrict__ Q, int n_ct, long long B, double lcm, long long row0,
                                float* __restrict__ E, unsigned long long* __restrict__ best_key) {
  unsigned long long key = ~0ull;
  bool nan = false;
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < B; b += (long long)gridDim.x * blockDim.x) {
    const float e = combine_q(Q, n_ct, B, b, lcm);
    if (E) E[b] = e;
    nan |= e != e;
    const unsigned long long k = argmin_key(e, (unsigned long long)(row0 + b));
    key = k < key ? k : key;
  }
  if (best_key) block_argmin(key, nan, best_key);
}

// ------------------------------------------------------------------------------------------
// device layout: bf16 limb planes of W, tile-blocked so that every TMA box is one
// contiguous NT x 64 block: W[l][ct][kb][m % NT][t % 64]
struct LayoutParams {
  const uint16_t* tuples;        // [Tpad][6]
  const float* const* strict;    // strict[r] device pointers (r = 0..order)
  const long long* binomT;       // [(N+1) * 7]: C(n, i)
  __nv_bfloat16* Wout;           // [L][Npad][Tpad]
  uint8_t* Wout8 = nullptr;      // int8 digit planes instead (non-null): [L][n_ct][n_kb/2][NT][128] bytes
  double inv_qscale = 1.0;       // cell / qscale = the integer the digits encode
  double f8_scale = 0.0;         // > 0: the 1-byte planes hold e4m3 limbs of cell * f8_scale instead
  int* err = nullptr;            // e4m3: set when a cell does not split exactly into L limbs
  long long Tpad;
  int N, Npad, L, field_mode, NT;
};

__device__ __forceinline__ long long dbinom(const long long* t, int n, int i) { return (n < i || i < 0) ? 0 : t[n * 7 + i]; }

// the e4m3 grid: round to nearest even (|v| <= 448), and the byte of an exact e4m3 value
__device__ __forceinline__ double e4m3_rn_d(double v) {
  const double a = fabs(v);
  if (a == 0.0) return 0.0;
  const int e = ilogb(a);
  const double q = ldexp(1.0, max(e, -6) - 3);
  const double r = rint(a / q) * q;
  return v < 0 ? -r : r;
}
__device__ __forceinline__ uint8_t e4m3_byte(double h) {
  if (h == 0.0) return 0;
  const uint32_t sgn = h < 0 ? 0x80u : 0u;
  const double a = fabs(h);
  const int e = ilogb(a);
  if (e < -6) return (uint8_t)(sgn | (uint32_t)(a * 512.0));                      // subnormal: m 2^-9
  return (uint8_t)(sgn | ((uint32_t)(e + 7) << 3) | (uint32_t)((a * ldexp(1.0, -e) - 1.0) * 8.0));
}

// e4m3 limbs: nl[ct][P] = 1 + the highest limb plane with a nonzero byte in box (ct, P)
// (nl preset to 1 by the caller); one warp per (limb >= 1, ct, P) box of NT x 128 bytes
__global__ void f8_limbs_kernel(const uint8_t* __restrict__ W8, int L, int n_ct, long long n_kbp, int NT,
                                unsigned int* __restrict__ nl) {
  const long long nbox = (long long)(L - 1) * n_ct * n_kbp;
  const int lane = threadIdx.x & 31;
  for (long long wb = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; wb < nbox;
       wb += ((long long)gridDim.x * blockDim.x) >> 5) {
    const long long l = 1 + wb / (n_ct * n_kbp), rest = wb % (n_ct * n_kbp);
    const uint4* box = reinterpret_cast<const uint4*>(W8 + ((size_t)l * n_ct * n_kbp + rest) * NT * 128);
    uint32_t any = 0;
    for (int i = lane; i < NT * 8; i += 32) {
      const uint4 v = box[i];
      any |= v.x | v.y | v.z | v.w;
    }
    if (__any_sync(0xFFFFFFFFu, any != 0) && lane == 0) atomicMax(nl + rest, (unsigned int)(l + 1));
  }
}

__global__ void layout_kernel(const LayoutParams lp) {
  const long long total = (long long)lp.Npad * lp.Tpad;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total; e += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(e / lp.Tpad);
    const long long t = e % lp.Tpad;
    const uint16_t* tp = lp.tuples + t * 6;
    const int r = tp[0];
    float c = 0.0f;
    if (r >= 2 && m < lp.N) {
      int S[6];
      int n = 0;
      bool ok = true, placed = false;
      for (int i = 0; i < r - 1; ++i) {
        const int v = tp[1 + i];
        if (v == m) ok = false;
        if (!placed && m < v) { S[n++] = m; placed = true; }
        S[n++] = v;
      }
      if (!placed) S[n++] = m;
      if (!lp.field_mode && placed) ok = false;  // strict layout: m must be the largest index
      if (ok) {
        long long rank = 0;
        for (int i = 0; i < r; ++i) rank += dbinom(lp.binomT, S[i], i + 1);
        c = lp.strict[r][rank];
      }
    } else if (r == 1 && m < lp.N) {   // the empty tuple (annealing site layouts): W[m, {}] = c({m})
      c = lp.strict[1][m];
    }
    if (lp.Wout8) {
      // two's-complement base-256 digits of q = c / qscale: unsigned low digits, signed top digit
      const long long q = lp.f8_scale > 0.0 ? 0 : __double2ll_rn((double)c * lp.inv_qscale);
      const size_t plane = (size_t)lp.Npad * lp.Tpad;
      const long long n_kbp = lp.Tpad / 128;   // boxes of 128-byte rows: K-block pairs
      // K position of tuple t in its 128-byte row: within each 32-tuple group, tuple 8i + k at
      // byte 4k + i (the generator's one-shift expansion, expand_bytes64)
      const int tg = (int)(t % 128), j = tg % 32;
      const size_t off = ((size_t)((m / lp.NT) * n_kbp + t / 128) * lp.NT + (m % lp.NT)) * 128 + (tg - j) + 4 * (j % 8) + j / 8;
      if (lp.f8_scale > 0.0) {   // e4m3 limbs: greedy round-to-nearest-even (hobo_api.cu e4m3_rn)
        double v = (double)c * lp.f8_scale;
        for (int l = 0; l < lp.L; ++l) {
          const double h = e4m3_rn_d(v);
          lp.Wout8[(size_t)l * plane + off] = e4m3_byte(h);
          v -= h;
        }
        if (v != 0.0) atomicOr(lp.err, 1);
        continue;
      }
      for (int l = 0; l < lp.L; ++l) lp.Wout8[(size_t)l * plane + off] = (uint8_t)((q >> (8 * l)) & 0xFF);
      continue;
    }
    // exact split into bf16 limbs: hi + mid + lo
    const __nv_bfloat16 hi = __float2bfloat16_rn(c);
    const float r1 = c - __bfloat162float(hi);
    const __nv_bfloat16 mid = __float2bfloat16_rn(r1);
    const float r2 = r1 - __bfloat162float(mid);
    const __nv_bfloat16 lo = __float2bfloat16_rn(r2);
    const size_t plane = (size_t)lp.Npad * lp.Tpad;
    const long long n_kb = lp.Tpad / 64;
    const size_t off = ((size_t)((m / lp.NT) * n_kb + t / 64) * lp.NT + (m % lp.NT)) * 64 + (t % 64);
    lp.Wout[off] = hi;
    if (lp.L > 1) lp.Wout[plane + off] = mid;
    if (lp.L > 2) lp.Wout[2 * plane + off] = lo;
  }
}

// ------------------------------------------------------------------------------------------
// search: counter-hash RNG, integer decisions on fp32 values

// ---- simulated annealing helpers ---------------------------------------------------------
// E_b = sum_ct Q[ct][b] / lcm (double; the annealer tracks E in double)
__global__ void sa_e_init_kernel(const double* __restrict__ Q, int n_ct, long long B, double lcm, double* __restrict__ E) {
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < B; b += (long long)gridDim.x * blockDim.x) {
    double q = 0.0;
    for (int c = 0; c < n_ct; ++c) q += Q[(size_t)c * B + b];
    E[b] = q / lcm;
  }
}

// the last visited site's decisions, applied to the state bits after the final launch
__global__ void sa_flush_kernel(uint32_t* __restrict__ bits, const int8_t* __restrict__ s, int site, long long B, int W) {
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < B; b += (long long)gridDim.x * blockDim.x) {
    const int sv = s[b];
    const uint32_t bit = 1u << (site & 31);
    uint32_t& w = bits[b * W + (site >> 5)];
    if (sv > 0) w |= bit;
    else if (sv < 0) w &= ~bit;
  }
}

// bit rows [B][W] -> u8 rows [B][N]
__global__ void unpack_bits_kernel(const uint32_t* __restrict__ bits, long long B, int N, int W, uint8_t* __restrict__ X) {
  const long long total = B * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / N;
    const int m = (int)(i % N);
    X[i] = (uint8_t)((bits[b * W + (m >> 5)] >> (m & 31)) & 1u);
  }
}

// chain c's initial x: bit m = bit (m & 63) of h(seed, 1, c, m >> 6)
// dargs (nullable, a graph-replayable launch): {seed, chain0, P_0 | P_1 << 32, ...} in device
// memory override the scalar seed / chain0 / P_t
__global__ void search_init_kernel(uint64_t seed, long long chain0, long long nchains, int N, int W, uint32_t* bits,
                                   float* ebest, const unsigned long long* __restrict__ dargs = nullptr) {
  if (dargs) { seed = dargs[0]; chain0 = (long long)dargs[1]; }
  const long long total = nchains * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long c = i / W;
    const int w = (int)(i % W);
    const uint64_t hv = d_hash(seed, 1, (uint64_t)(chain0 + c), (uint64_t)(w >> 1));
    uint32_t v = (uint32_t)(hv >> ((w & 1) * 32));
    const int valid = N - w * 32;
    if (valid < 32) v &= (valid <= 0) ? 0u : ((1u << valid) - 1u);
    bits[i] = v;
    if (w == 0) ebest[c] = __int_as_float(0x7f800000);  // +inf
  }
}

// one warp per chain: best tracking, flip gain, move rule, flip
__global__ void search_step_kernel(const double* __restrict__ Q, int n_ct, double lcm, const float* __restrict__ G,
                                   uint32_t* bits, uint32_t* xbest, float* ebest, long long chain0, long long nchains,
                                   int N, int W, uint64_t seed, long long t, uint32_t P_t, int do_move, int greedy = 0,
                                   const unsigned long long* __restrict__ dargs = nullptr) {
  const long long c = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (c >= nchains) return;
  if (dargs) {
    seed = dargs[0];
    chain0 = (long long)dargs[1];
    if (do_move) P_t = reinterpret_cast<const uint32_t*>(dargs + 2)[t];
  }
  const float e = combine_q(Q, n_ct, nchains, c, lcm);
  uint32_t* xb = bits + c * W;
  if (e < ebest[c]) {  // strict: on equal E the earliest iteration is kept
    for (int w = lane; w < W; w += 32) xbest[c * W + w] = xb[w];
    __syncwarp();
    if (lane == 0) ebest[c] = e;
  }
  if (!do_move) return;
  // argmin over m of (1 - 2 x_m) g_m, lowest m on ties
  float dmin = __int_as_float(0x7f800000);
  int mmin = 0x7fffffff;
  for (int m = lane; m < N; m += 32) {
    const float g = G[(size_t)c * N + m];
    const float d = ((xb[m >> 5] >> (m & 31)) & 1u) ? -g : g;
    if (d < dmin) { dmin = d; mmin = m; }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float od = __shfl_xor_sync(0xffffffffu, dmin, o);
    const int om = __shfl_xor_sync(0xffffffffu, mmin, o);
    if (od < dmin || (od == dmin && om < mmin)) { dmin = od; mmin = om; }
  }
  if (lane == 0) {
    if (greedy) {            // steepest single-flip descent: flip only an improving site
      if (dmin < 0.0f) xb[mmin >> 5] ^= 1u << (mmin & 31);
    } else {
      const uint64_t r = d_hash(seed, 2, (uint64_t)(chain0 + c), (uint64_t)t);
      const int mrand = (int)(((r & 0xffffffffull) * (uint64_t)N) >> 32);
      int ms;
      if ((uint32_t)(r >> 32) < P_t) ms = mrand;
      else ms = (dmin < 0.0f) ? mmin : mrand;
      xb[ms >> 5] ^= 1u << (ms & 31);
    }
  }
}

__global__ void search_best_kernel(const float* __restrict__ ebest, long long nchains, long long chain0,
                                   unsigned long long* best_key) {
  unsigned long long key = ~0ull;
  bool nan = false;
  for (long long c = blockIdx.x * (long long)blockDim.x + threadIdx.x; c < nchains; c += (long long)gridDim.x * blockDim.x) {
    const float e = ebest[c];
    nan |= e != e;
    const unsigned long long k = argmin_key(e, (unsigned long long)(chain0 + c));
    key = k < key ? k : key;
  }
  block_argmin(key, nan, best_key);
}

}  // namespace hobo

namespace hobo {

// ------------------------------------------------------------------------------------------
// sample aggregation (the paper's result list): dedupe the chains' best states,
// count occurrences.  Sort key (k1, k2) = (ord(E) << 32 | hash_hi, hash_lo << 32 | chain):
// equal assignments are contiguous, the order is total and deterministic.
__device__ __forceinline__ uint64_t row_hash(const uint32_t* row, int W) {
  uint64_t h = 0x243F6A8885A308D3ull;
  for (int w = 0; w < W; ++w) h = d_splitmix64(h ^ row[w]);
  return h;
}

__global__ void agg_key_kernel(const float* __restrict__ ebest, const uint32_t* __restrict__ xbest, long long B, int W,
                               long long n, unsigned long long* k1, unsigned long long* k2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    if (i < B) {
      const uint64_t h = row_hash(xbest + i * W, W);
      k1[i] = (argmin_key(ebest[i], 0) & 0xFFFFFFFF00000000ull) | (h >> 32);
      k2[i] = (h << 32) | (unsigned long long)i;
    } else {
      k1[i] = ~0ull;
      k2[i] = ~0ull;
    }
  }
}

__device__ __forceinline__ bool key_gt(unsigned long long a1, unsigned long long a2, unsigned long long b1,
                                       unsigned long long b2) {
  return a1 > b1 || (a1 == b1 && a2 > b2);
}

// one bitonic pass with partner distance j >= 1024 (global memory)
__global__ void bitonic_global_kernel(unsigned long long* k1, unsigned long long* k2, long long n, long long j, long long k) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long l = i ^ j;
    if (l <= i) continue;
    const bool up = (i & k) == 0;
    const unsigned long long a1 = k1[i], a2 = k2[i], b1 = k1[l], b2 = k2[l];
    if (key_gt(a1, a2, b1, b2) == up) { k1[i] = b1; k2[i] = b2; k1[l] = a1; k2[l] = a2; }
  }
}

// all passes with j < 1024 of stage k, on 2048-element chunks in shared memory
__global__ void __launch_bounds__(1024) bitonic_shared_kernel(unsigned long long* k1, unsigned long long* k2, long long k) {
  __shared__ unsigned long long s1[2048], s2[2048];
  const long long base = (long long)blockIdx.x * 2048;
  for (int t = threadIdx.x; t < 2048; t += 1024) { s1[t] = k1[base + t]; s2[t] = k2[base + t]; }
  __syncthreads();
  for (long long j = (k >> 1) < 1024 ? (k >> 1) : 1024; j >= 1; j >>= 1) {
    for (int t = threadIdx.x; t < 2048; t += 1024) {
      const int l = t ^ (int)j;
      if (l > t) {
        const bool up = ((base + t) & k) == 0;
        const unsigned long long a1 = s1[t], a2 = s2[t], b1 = s1[l], b2 = s2[l];
        if (key_gt(a1, a2, b1, b2) == up) { s1[t] = b1; s2[t] = b2; s1[l] = a1; s2[l] = a2; }
      }
    }
    __syncthreads();
  }
  for (int t = threadIdx.x; t < 2048; t += 1024) { k1[base + t] = s1[t]; k2[base + t] = s2[t]; }
}

// group starts: element i opens a group unless it repeats the previous assignment
__global__ void agg_flag_kernel(const unsigned long long* __restrict__ k1, const unsigned long long* __restrict__ k2,
                                const uint32_t* __restrict__ xbest, long long B, int W, uint32_t* flag) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < B; i += (long long)gridDim.x * blockDim.x) {
    uint32_t f = 1;
    if (i > 0 && k1[i] == k1[i - 1] && (k2[i] >> 32) == (k2[i - 1] >> 32)) {
      const uint32_t* a = xbest + (k2[i] & 0xFFFFFFFFull) * W;
      const uint32_t* b = xbest + (k2[i - 1] & 0xFFFFFFFFull) * W;
      f = 0;
      for (int w = 0; w < W; ++w) f |= (a[w] != b[w]);   // a 64-bit hash collision stays a new group
    }
    flag[i] = f;
  }
}

// one block: exclusive scan of the flags -> starts[g] = sorted position of group g
__global__ void __launch_bounds__(1024) agg_scan_kernel(const uint32_t* __restrict__ flag, long long B, uint32_t* starts,
                                                        uint32_t* n_groups) {
  __shared__ uint32_t sums[1024];
  const long long per = (B + 1023) / 1024;
  const long long lo = threadIdx.x * per, hi = lo + per < B ? lo + per : B;
  uint32_t c = 0;
  for (long long i = lo; i < hi; ++i) c += flag[i];
  sums[threadIdx.x] = c;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {   // inclusive Hillis-Steele scan
    const uint32_t v = threadIdx.x >= o ? sums[threadIdx.x - o] : 0u;
    __syncthreads();
    sums[threadIdx.x] += v;
    __syncthreads();
  }
  uint32_t g = sums[threadIdx.x] - c;
  for (long long i = lo; i < hi; ++i)
    if (flag[i]) starts[g++] = (uint32_t)i;
  if (threadIdx.x == 1023) *n_groups = sums[1023];
}

}  // namespace hobo

namespace hobo {
// ------------------------------------------------------------------------------------------
// gradient descent on the multilinear relaxation:
// p = sigmoid(theta), theta <- theta - eta * dE/dp * p(1-p); p is carried in bf16.
__global__ void gd_init_kernel(uint64_t seed, long long B, int N, float* theta, __nv_bfloat16* P) {
  const long long total = B * N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / N;
    const int m = (int)(i % N);
    const double u = ((double)(d_hash(seed, 3, (uint64_t)b, (uint64_t)m) >> 40) + 0.5) * 0x1p-24;   // U(0,1)
    theta[i] = (float)log(u / (1.0 - u));
    P[i] = __float2bfloat16_rn((float)u);
  }
}

__global__ void gd_update_kernel(long long total, float eta, const float* __restrict__ G, float* theta,
                                 __nv_bfloat16* P) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const float p = 1.0f / (1.0f + __expf(-theta[i]));
    const float th = theta[i] - eta * G[i] * p * (1.0f - p);
    theta[i] = th;
    P[i] = __float2bfloat16_rn(1.0f / (1.0f + __expf(-th)));
  }
}

// round at 0.5 into candidate bit rows (and reset the per-chain best)
__global__ void gd_round_kernel(long long B, int N, int W, const __nv_bfloat16* __restrict__ P, uint32_t* bits,
                                float* ebest) {
  const long long total = B * W;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
    const long long b = i / W;
    const int w = (int)(i % W);
    uint32_t v = 0;
    for (int j = 0; j < 32 && w * 32 + j < N; ++j)
      v |= (uint32_t)(__bfloat162float(P[b * N + w * 32 + j]) >= 0.5f) << j;
    bits[i] = v;
    if (w == 0) ebest[b] = __int_as_float(0x7f800000);
  }
}
}  // namespace hobo

namespace hobo {
// ------------------------------------------------------------------------------------------
// Tensor-Train form: E_b = prod_p ( sum_{i: x_bi = 1} G_p[:, i, :] ), a
// chain of r x r matrices selected by the bits; fp64 (TT cores carry cancellations).
template <int RM>
__global__ void tt_energy_kernel(const double* __restrict__ cores, const int* __restrict__ off,
                                 const int* __restrict__ ranks, int k, int N, int W, const uint32_t* __restrict__ bits,
                                 long long B, float* __restrict__ E) {
  for (long long b = blockIdx.x * (long long)blockDim.x + threadIdx.x; b < B; b += (long long)gridDim.x * blockDim.x) {
    double v[RM];
#pragma unroll
    for (int a = 0; a < RM; ++a) v[a] = a == 0 ? 1.0 : 0.0;
    int rp = 1;
    for (int p = 0; p < k; ++p) {
      const int rn = __ldg(ranks + p + 1);
      const double* G = cores + __ldg(off + p);
      double nv[RM];
#pragma unroll
      for (int c = 0; c < RM; ++c) nv[c] = 0.0;
      for (int i = 0; i < N; ++i) {
        if (!((__ldg(bits + b * W + (i >> 5)) >> (i & 31)) & 1u)) continue;
#pragma unroll
        for (int a = 0; a < RM; ++a) {
          if (a >= rp) break;
#pragma unroll
          for (int c = 0; c < RM; ++c)
            if (c < rn) nv[c] = fma(v[a], __ldg(G + ((size_t)a * N + i) * rn + c), nv[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < RM; ++c) v[c] = nv[c];
      rp = rn;
    }
    E[b] = (float)v[0];
  }
}

// The same chain product with the cores staged in shared memory (warp-uniform reads are
// broadcasts) and CPT candidates per thread, so each core element loaded feeds CPT fp64
// FMAs; a candidate's bit word is loaded once per 32 indices.  Same summation order as
// tt_energy_kernel (x_i = 0 contributes an exact zero instead of being skipped).
template <int RM, int CPT>
__global__ void tt_energy_smem_kernel(const double* __restrict__ cores, int ncores, const int* __restrict__ off,
                                      const int* __restrict__ ranks, int k, int N, int W,
                                      const uint32_t* __restrict__ bits, long long B, float* __restrict__ E) {
  extern __shared__ double sc[];
  __shared__ int soff[16], sr[17];
  for (int i = threadIdx.x; i < ncores; i += blockDim.x) sc[i] = cores[i];
  if (threadIdx.x < k) soff[threadIdx.x] = off[threadIdx.x];
  if (threadIdx.x <= k) sr[threadIdx.x] = ranks[threadIdx.x];
  __syncthreads();
  const long long per_block = (long long)blockDim.x * CPT;
  for (long long base = blockIdx.x * per_block; base < B; base += (long long)gridDim.x * per_block) {
    long long bj[CPT];
    double v[CPT][RM];
#pragma unroll
    for (int j = 0; j < CPT; ++j) {
      bj[j] = base + (long long)j * blockDim.x + threadIdx.x;   // coalesced bits / E accesses
#pragma unroll
      for (int a = 0; a < RM; ++a) v[j][a] = a == 0 ? 1.0 : 0.0;
    }
    int rp = 1;
    for (int p = 0; p < k; ++p) {
      const int rn = sr[p + 1];
      const double* G = sc + soff[p];
      double nv[CPT][RM];
#pragma unroll
      for (int j = 0; j < CPT; ++j)
#pragma unroll
        for (int c = 0; c < RM; ++c) nv[j][c] = 0.0;
      uint32_t xw[CPT];
      for (int i = 0; i < N; ++i) {
        if ((i & 31) == 0) {
#pragma unroll
          for (int j = 0; j < CPT; ++j) xw[j] = bj[j] < B ? __ldg(bits + bj[j] * W + (i >> 5)) : 0u;
        }
#pragma unroll
        for (int a = 0; a < RM; ++a) {
          if (a >= rp) break;
          double va[CPT];
#pragma unroll
          for (int j = 0; j < CPT; ++j) va[j] = ((xw[j] >> (i & 31)) & 1u) ? v[j][a] : 0.0;
          const double* g = G + ((size_t)a * N + i) * rn;
#pragma unroll
          for (int c = 0; c < RM; ++c)
            if (c < rn) {
              const double gc = g[c];
#pragma unroll
              for (int j = 0; j < CPT; ++j) nv[j][c] = fma(va[j], gc, nv[j][c]);
            }
        }
      }
#pragma unroll
      for (int j = 0; j < CPT; ++j)
#pragma unroll
        for (int c = 0; c < RM; ++c) v[j][c] = nv[j][c];
      rp = rn;
    }
#pragma unroll
    for (int j = 0; j < CPT; ++j)
      if (bj[j] < B) E[bj[j]] = (float)v[j][0];
  }
}
}  // namespace hobo
