// sa_kernel.cuh — persistent simulated-annealing sweep (SPEC sa_run,
// S:447-453), one CTA per block of 128 chains for the whole run.
//
// The chains' local fields G (128 rows x Npad fp32) stay in tensor memory for all sweeps.
// Visiting site m: the decision warps read column m of G (tcgen05.ld), take the Metropolis
// decision d = (1 - 2 x_m) g_m, accept iff d <= 0 or d < -T ln u, and flip x_m in the
// staged bits (the threshold -T ln u of the uniform is computed before the field is
// ready, off the critical path).  The change of every other field is then the field of P_m = dE/dx_m:
//
//     G[b, j] += s_b * ( sum_T A[b, T] W_m[j, T] + c_m({j}) )        s_b = x_m' - x_m
//
// which is ONE accumulate-into-G GEMM: the generator writes the Khatri-Rao rows of A with
// the sign s_b folded in (s_b = 0 rows are zero), and the degree-1 part c_m({j}) rides as
// one extra K-block whose only tuple is the empty set (A = s_b, W[j, 0] = c({m, j})).
// W_m streams through a TMA ring independent of the decisions; the sites' layouts are
// concatenated in one buffer (site_base[m] = first box of site m).
#pragma once
#include <algorithm>

#include "kernels.cuh"

namespace hobo {

struct SaParams {
  uint32_t* bits;             // [B][W] chain bits: read at block start, written at block end
  const float* G0;            // [B][N] initial fields (the field contraction of the start states)
  double* E;                  // [B] tracked energies, in and out
  const uint4* runs;          // generator runs of the site layout (order k-1, N)
  const uint4* kdesc;         // [n_kb][2] per-K-block descriptors of the site layout
  const int* site_L;          // [N] bf16 limbs of site m's tensor
  const int* site_base;       // [N] first TMA box of site m
  const double* temps;        // [sweeps] temperature of each sweep
  unsigned long long seed;
  long long chain0;           // global id of chain 0 of this shard
  long long B;
  long long steps;            // sweeps * N site visits
  int N, W, n_ct, nkb1;       // nkb1 = K-blocks per (limb, column tile), the degree-1 block last
  int nseg, nq;               // nq = K-blocks per site (segments + the degree-1 block)
  int seg_kb0[8], seg_cnt[8]; // segment j: K-blocks [seg_kb0, seg_kb0 + seg_cnt), visited j = nseg-1..0
};

template <int NT>
struct SaCfg {
  static constexpr int BOX = NT * 128;        // one W box: NT rows x 64 bf16 (SW128)
  static constexpr int RW = NT == 256 ? 5 : 10; // W ring (boxes)
  static constexpr int ABOX = kBM * 128;      // one A tile: 128 rows x 64 bf16 (SW128, K-major)
  static constexpr int RA = 2;                // A ring (tiles)
  static constexpr int NBAR = 2 * RW + 2 * RA + 1;
  static size_t smem_bytes(int W) {
    return 1024 + (size_t)RW * BOX + (size_t)RA * ABOX + 8 * NBAR + 16 + (size_t)(W + 2) * kBM * 4 + kBM * 4 + 128;
  }
};

__device__ __forceinline__ uint32_t tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  return r;
}

// K-block of site-local index q (segments in ascending degree, then the degree-1 block)
__device__ __forceinline__ int sa_site_kb(const SaParams& p, int q) {
  for (int j = p.nseg - 1; j >= 0; --j) {
    if (q < p.seg_cnt[j]) return p.seg_kb0[j] + q;
    q -= p.seg_cnt[j];
  }
  return p.nkb1 - 1;
}

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) sa_kernel(const __grid_constant__ CUtensorMap tmap, const SaParams p) {
  using C = SaCfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sW = base;
  const uint32_t sA = sW + C::RW * C::BOX;
  const uint32_t sBar = sA + C::RA * C::ABOX;
#define FULLW(s) (sBar + 8u * (s))
#define EMPTYW(s) (sBar + 8u * (C::RW + (s)))
#define FULLA(s) (sBar + 8u * (2 * C::RW + (s)))
#define EMPTYA(s) (sBar + 8u * (2 * C::RW + C::RA + (s)))
  const uint32_t SITE = sBar + 8u * (2 * C::RW + 2 * C::RA);
  const uint32_t tslot = SITE + 8;
  const uint32_t sX = (tslot + 16 + 127u) & ~127u;
  uint32_t* xs = reinterpret_cast<uint32_t*>(gbase + (sX - base));
  int* sS = reinterpret_cast<int*>(gbase + (sX - base) + (size_t)(p.W + 2) * kBM * 4);
  volatile uint32_t* tslot_g = reinterpret_cast<volatile uint32_t*>(gbase + (tslot - base));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NPAD = NT * p.n_ct;     // TMEM columns of G (128, 256 or 512)
  const long long n_cb = (p.B + kBM - 1) / kBM;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::RW; ++s) { mbar_init(FULLW(s), 1); mbar_init(EMPTYW(s), 1); }
    for (int s = 0; s < C::RA; ++s) { mbar_init(FULLA(s), 4); mbar_init(EMPTYA(s), 1); }
    mbar_init(SITE, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch_desc(&tmap);
  if (warp == 1) tmem_alloc(tslot, (uint32_t)NPAD);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot_g;

  if (warp == 0) {
    // ---------------- TMA producer: the sites' W boxes, in visiting order, for every block ---------
    if (lane == 0) {
      uint32_t nw = 0;
      for (long long cb = blockIdx.x; cb < n_cb; cb += gridDim.x)
        for (long long step = 0; step < p.steps; ++step) {
          const int m = (int)(step % p.N);
          const int L = __ldg(p.site_L + m), sb = __ldg(p.site_base + m);
          for (int q = 0; q < p.nq; ++q) {
            const int kb = sa_site_kb(p, q);
            for (int l = 0; l < L; ++l)
              for (int h = 0; h < p.n_ct; ++h, ++nw) {
                const uint32_t s = nw % C::RW;
                mbar_wait(EMPTYW(s), ((nw / C::RW) & 1u) ^ 1u);
                mbar_arrive_expect_tx(FULLW(s), C::BOX);
                tma_load_3d(sW + s * C::BOX, &tmap, FULLW(s), 0, 0, sb + (l * p.n_ct + h) * p.nkb1 + kb);
              }
          }
        }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: G[:, tile h] += A_q * W_m,q (accumulate, never cleared) ---------
    // whole warp in the loop (uniform registers), one elected lane issues
    {
      constexpr uint32_t idesc = idesc_bf16_f32(kBM, NT);
      uint32_t nw = 0, na = 0;
      for (long long cb = blockIdx.x; cb < n_cb; cb += gridDim.x)
        for (long long step = 0; step < p.steps; ++step) {
          const int m = (int)(step % p.N);
          const int L = __ldg(p.site_L + m);
          for (int q = 0; q < p.nq; ++q, ++na) {
            const uint32_t a = na % C::RA;
            mbar_wait(FULLA(a), (na / C::RA) & 1u);
            tc_fence_after();
            const uint64_t adesc = sw128_kmajor_desc(sA + a * C::ABOX);
            for (int l = 0; l < L; ++l)
              for (int h = 0; h < p.n_ct; ++h, ++nw) {
                const uint32_t s = nw % C::RW;
                mbar_wait(FULLW(s), (nw / C::RW) & 1u);
                tc_fence_after();
                const uint64_t bdesc = sw128_kmajor_desc(sW + s * C::BOX);
                if (elect_one()) {
#pragma unroll
                  for (int k = 0; k < kBK / 16; ++k)
                    umma_bf16_ss(tmem + (uint32_t)(h * NT), adesc + 2u * k, bdesc + 2u * k, idesc, 1u);
                  umma_commit(EMPTYW(s));
                }
                __syncwarp();
              }
            if (elect_one()) umma_commit(EMPTYA(a));
            __syncwarp();
          }
          if (elect_one()) umma_commit(SITE);   // this site's G update is complete when this arrives
          __syncwarp();
        }
    }
  } else {
    // ---------------- decisions (team 0) + A generator (both teams), one row per thread -----------
    const int qd = warp & 3;                 // TMEM lane quarter
    const int h = (warp - 2) >> 2;           // team: K-blocks q with q % 2 == h; G columns half h
    const int row = qd * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(qd * 32) << 16);
    const int gtid = threadIdx.x - 64;       // 0..255
    uint32_t na = 0, nsite = 0;
    for (long long cb = blockIdx.x; cb < n_cb; cb += gridDim.x) {
      const long long b0 = cb * kBM, b = b0 + row;
      const bool live = b < p.B;
      // stage the block's bits column-major xs[w][row] (+2 zero words for window reads)
      const int Wp = p.W + 2;
      for (int i = gtid; i < Wp * kBM; i += 256) {
        const int r = i / Wp, w = i % Wp;
        xs[w * kBM + r] = (w < p.W && b0 + r < p.B) ? p.bits[(size_t)(b0 + r) * p.W + w] : 0u;
      }
      // this thread's half of the row's initial fields -> TMEM
      for (int c0 = h * (NPAD / 2); c0 < (h + 1) * (NPAD / 2); c0 += 32) {
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c)
          v[c] = (live && c0 + c < p.N) ? __float_as_uint(__ldg(p.G0 + (size_t)b * p.N + c0 + c)) : 0u;
        tmem_st32(lane_base + (uint32_t)c0, v);
      }
      tmem_st_wait();
      double E = (h == 0 && live) ? p.E[b] : 0.0;
      tc_fence_before();
      named_bar_sync(1, 256);
      tc_fence_after();
      for (long long step = 0; step < p.steps; ++step) {
        const int m = (int)(step % p.N);
        // the acceptance threshold -T ln u needs no field: computed while the site's MMAs run
        double thr = 0.0;
        if (h == 0 && live) {
          const double u = (double)(d_hash(p.seed, 4, (uint64_t)(p.chain0 + b), (uint64_t)step) >> 11) * 0x1.0p-53;
          thr = -__ldg(p.temps + step / p.N) * log(u);
        }
        if (step > 0) {
          mbar_wait(SITE, nsite & 1u);
          ++nsite;
          tc_fence_after();
        }
        if (h == 0) {
          const float g = __uint_as_float(tmem_ld1(lane_base + (uint32_t)m));
          tmem_ld_wait();
          int sv = 0;
          if (live) {
            const int wi = m >> 5;
            const uint32_t bit = 1u << (m & 31);
            const bool xm = (xs[wi * kBM + row] & bit) != 0u;
            const float d = xm ? -g : g;
            if (d <= 0.0f || (double)d < thr) {
              sv = xm ? -1 : 1;
              xs[wi * kBM + row] ^= bit;
              E += (double)d;
            }
          }
          sS[row] = sv;
          tc_fence_before();
        }
        named_bar_sync(1, 256);
        // A rows of site m: s_b * prod_{u in T} x_bu (x_m itself never occurs with W_m != 0)
        const int sv = sS[row];
        const uint32_t sgn = sv < 0 ? 0x80008000u : 0u;
        for (int q = 0; q < p.nq; ++q, ++na) {
          if ((q & 1) != h) continue;
          const uint32_t a = na % C::RA;
          mbar_wait(EMPTYA(a), ((na / C::RA) & 1u) ^ 1u);
          const int kb = sa_site_kb(p, q);
          uint64_t bits = 0;
          if (sv != 0) {
            if (kb == p.nkb1 - 1) bits = 1ull;   // the degree-1 block: the empty tuple only
            else bits = block_bits(xs, row, __ldg(p.kdesc + 2 * kb), __ldg(p.kdesc + 2 * kb + 1), p.runs);
          }
          uint32_t w[32];
          expand32((uint32_t)bits, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
          expand32((uint32_t)(bits >> 32), *reinterpret_cast<uint32_t(*)[16]>(&w[16]));
          const uint32_t rowaddr = sA + a * C::ABOX + (uint32_t)(row >> 3) * 1024u + (uint32_t)(row & 7) * 128u;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            st_shared_v4(rowaddr + (uint32_t)((c ^ (row & 7)) << 4), w[4 * c] ^ sgn, w[4 * c + 1] ^ sgn,
                         w[4 * c + 2] ^ sgn, w[4 * c + 3] ^ sgn);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) mbar_arrive(FULLA(a));
        }
      }
      if (p.steps > 0) {   // the last site's update: then the block's results are final
        mbar_wait(SITE, nsite & 1u);
        ++nsite;
        tc_fence_after();
      }
      if (h == 0 && live) {
        p.E[b] = E;
        for (int w = 0; w < p.W; ++w) p.bits[(size_t)b * p.W + w] = xs[w * kBM + row];
      }
      tc_fence_before();
      named_bar_sync(1, 256);   // xs and TMEM are reused by the next block
    }
  }
#undef FULLW
#undef EMPTYW
#undef FULLA
#undef EMPTYA
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, (uint32_t)NPAD);
}

// ---------------------------------------------------------------------------------------------
// Staged variant: one pipeline stage = one site K-block, i.e. all n_ct x L W boxes of that
// K-block plus its A tile, behind ONE full barrier (TMA bytes + 4 generator-warp arrivals)
// and ONE empty barrier (a single tcgen05.commit).  The box-ring kernel above pays a wait,
// a fence and a commit per W box and per A tile; with 128-column tiles (64-cycle MMAs) that
// bookkeeping is what the lone MMA-issuing thread cannot hide.  (A tiles in TMEM instead of
// shared memory were measured 4% slower at cfg4 and dropped.)
template <int NT>
struct SaStCfg {
  static constexpr int BOX = NT * 128;
  static constexpr int ABOX = kBM * 128;
  static constexpr int MAXST = 8;
  static constexpr int BUDGET = 232448 - 1024 - 1024 - 16 * 1024;   // ring bytes (bits, barriers after it)
  static int stage_bytes(int boxes) { return boxes * BOX + ABOX; }
  static int nst(int boxes) { return std::min(4, BUDGET / stage_bytes(boxes)); }
  static size_t smem_bytes(int boxes, int W) {
    return 1024 + (size_t)nst(boxes) * stage_bytes(boxes) + 8 * (2 * MAXST + 1) + 16 + (size_t)(W + 2) * kBM * 4 +
           kBM * 4 + 128;
  }
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) sa_stage_kernel(const __grid_constant__ CUtensorMap tmap, const SaParams p,
                                                               int SB, int NST) {
  using C = SaStCfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t SBYTES = (uint32_t)(SB * C::BOX + C::ABOX);
  const uint32_t sSt = base;                                  // stage s: SB W boxes, then the A tile
  const uint32_t sBar = sSt + (uint32_t)NST * SBYTES;
#define FULL(s) (sBar + 8u * (s))
#define EMPTY(s) (sBar + 8u * (C::MAXST + (s)))
  const uint32_t SITE = sBar + 8u * (2 * C::MAXST);
  const uint32_t tslot = SITE + 8;
  const uint32_t sX = (tslot + 16 + 127u) & ~127u;
  uint32_t* xs = reinterpret_cast<uint32_t*>(gbase + (sX - base));
  int* sS = reinterpret_cast<int*>(gbase + (sX - base) + (size_t)(p.W + 2) * kBM * 4);
  volatile uint32_t* tslot_g = reinterpret_cast<volatile uint32_t*>(gbase + (tslot - base));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NPAD = NT * p.n_ct;
  // TMEM: G in [0, NPAD)
  const uint32_t TCOLS = (uint32_t)NPAD;
  const long long n_cb = (p.B + kBM - 1) / kBM;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) { mbar_init(FULL(s), 5); mbar_init(EMPTY(s), 1); }
    mbar_init(SITE, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch_desc(&tmap);
  if (warp == 1) tmem_alloc(tslot, TCOLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot_g;

  if (warp == 0) {
    // ---------------- TMA producer: each stage gets one K-block's L x n_ct W boxes -------------
    if (lane == 0) {
      uint32_t n = 0;
      for (long long cb = blockIdx.x; cb < n_cb; cb += gridDim.x)
        for (long long step = 0; step < p.steps; ++step) {
          const int m = (int)(step % p.N);
          const int L = __ldg(p.site_L + m), sb = __ldg(p.site_base + m);
          for (int q = 0; q < p.nq; ++q, ++n) {
            const int kb = sa_site_kb(p, q);
            const uint32_t s = n % NST;
            mbar_wait(EMPTY(s), ((n / NST) & 1u) ^ 1u);
            mbar_arrive_expect_tx(FULL(s), (uint32_t)(L * p.n_ct) * C::BOX);
            for (int l = 0; l < L; ++l)
              for (int h = 0; h < p.n_ct; ++h)
                tma_load_3d(sSt + s * SBYTES + (uint32_t)(l * p.n_ct + h) * C::BOX, &tmap, FULL(s), 0, 0,
                            sb + (l * p.n_ct + h) * p.nkb1 + kb);
          }
        }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: one wait + one commit per K-block ----------------------------
    // The whole warp runs the loop (warp-uniform descriptors live in uniform registers) and one
    // elected lane issues; a single-lane loop pays register->uniform moves on every MMA.
    {
      constexpr uint32_t idesc = idesc_bf16_f32(kBM, NT);
      uint32_t n = 0;
      for (long long cb = blockIdx.x; cb < n_cb; cb += gridDim.x)
        for (long long step = 0; step < p.steps; ++step) {
          const int m = (int)(step % p.N);
          const int L = __ldg(p.site_L + m);
          for (int q = 0; q < p.nq; ++q, ++n) {
            const uint32_t s = n % NST;
            mbar_wait(FULL(s), (n / NST) & 1u);
            tc_fence_after();
            const uint32_t st = sSt + s * SBYTES;
            const uint64_t adesc = sw128_kmajor_desc(st + (uint32_t)SB * C::BOX);
            if (elect_one()) {
              for (int l = 0; l < L; ++l)
                for (int h = 0; h < p.n_ct; ++h) {
                  const uint64_t bdesc = sw128_kmajor_desc(st + (uint32_t)(l * p.n_ct + h) * C::BOX);
#pragma unroll
                  for (int k = 0; k < kBK / 16; ++k) {
                    umma_bf16_ss(tmem + (uint32_t)(h * NT), adesc + 2u * k, bdesc + 2u * k, idesc, 1u);
                  }
                }
              umma_commit(EMPTY(s));
            }
            __syncwarp();
          }
          if (elect_one()) umma_commit(SITE);
          __syncwarp();
        }
    }
  } else {
    // ---------------- decisions (team 0) + A generator (both teams), one row per thread -----------
    const int qd = warp & 3;
    const int h = (warp - 2) >> 2;
    const int row = qd * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(qd * 32) << 16);
    const int gtid = threadIdx.x - 64;
    uint32_t n = 0, nsite = 0;
    for (long long cb = blockIdx.x; cb < n_cb; cb += gridDim.x) {
      const long long b0 = cb * kBM, b = b0 + row;
      const bool live = b < p.B;
      const int Wp = p.W + 2;
      for (int i = gtid; i < Wp * kBM; i += 256) {
        const int r = i / Wp, w = i % Wp;
        xs[w * kBM + r] = (w < p.W && b0 + r < p.B) ? p.bits[(size_t)(b0 + r) * p.W + w] : 0u;
      }
      for (int c0 = h * (NPAD / 2); c0 < (h + 1) * (NPAD / 2); c0 += 32) {
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c)
          v[c] = (live && c0 + c < p.N) ? __float_as_uint(__ldg(p.G0 + (size_t)b * p.N + c0 + c)) : 0u;
        tmem_st32(lane_base + (uint32_t)c0, v);
      }
      tmem_st_wait();
      double E = (h == 0 && live) ? p.E[b] : 0.0;
      tc_fence_before();
      named_bar_sync(1, 256);
      tc_fence_after();
      for (long long step = 0; step < p.steps; ++step) {
        const int m = (int)(step % p.N);
        double thr = 0.0;   // -T ln u: no field needed, computed while the previous site's MMAs run
        if (h == 0 && live) {
          const double u = (double)(d_hash(p.seed, 4, (uint64_t)(p.chain0 + b), (uint64_t)step) >> 11) * 0x1.0p-53;
          thr = -__ldg(p.temps + step / p.N) * log(u);
        }
        if (step > 0) {
          mbar_wait(SITE, nsite & 1u);
          ++nsite;
          tc_fence_after();
        }
        if (h == 0) {
          const float g = __uint_as_float(tmem_ld1(lane_base + (uint32_t)m));
          tmem_ld_wait();
          int sv = 0;
          if (live) {
            const int wi = m >> 5;
            const uint32_t bit = 1u << (m & 31);
            const bool xm = (xs[wi * kBM + row] & bit) != 0u;
            const float d = xm ? -g : g;
            if (d <= 0.0f || (double)d < thr) {
              sv = xm ? -1 : 1;
              xs[wi * kBM + row] ^= bit;
              E += (double)d;
            }
          }
          sS[row] = sv;
          tc_fence_before();
        }
        named_bar_sync(1, 256);
        const int sv = sS[row];
        const uint32_t sgn = sv < 0 ? 0x80008000u : 0u;
        for (int q = 0; q < p.nq; ++q, ++n) {
          if ((q & 1) != h) continue;
          const uint32_t s = n % NST;
          mbar_wait(EMPTY(s), ((n / NST) & 1u) ^ 1u);
          const int kb = sa_site_kb(p, q);
          uint64_t bits = 0;
          if (sv != 0) {
            if (kb == p.nkb1 - 1) bits = 1ull;
            else bits = block_bits(xs, row, __ldg(p.kdesc + 2 * kb), __ldg(p.kdesc + 2 * kb + 1), p.runs);
          }
          uint32_t w[32];
          expand32((uint32_t)bits, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
          expand32((uint32_t)(bits >> 32), *reinterpret_cast<uint32_t(*)[16]>(&w[16]));
          {
            const uint32_t rowaddr = sSt + s * SBYTES + (uint32_t)SB * C::BOX + (uint32_t)(row >> 3) * 1024u +
                                     (uint32_t)(row & 7) * 128u;
#pragma unroll
            for (int c = 0; c < 8; ++c)
              st_shared_v4(rowaddr + (uint32_t)((c ^ (row & 7)) << 4), w[4 * c] ^ sgn, w[4 * c + 1] ^ sgn,
                           w[4 * c + 2] ^ sgn, w[4 * c + 3] ^ sgn);
            fence_async_smem();
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(FULL(s));
        }
      }
      if (p.steps > 0) {
        mbar_wait(SITE, nsite & 1u);
        ++nsite;
        tc_fence_after();
      }
      if (h == 0 && live) {
        p.E[b] = E;
        for (int w = 0; w < p.W; ++w) p.bits[(size_t)b * p.W + w] = xs[w * kBM + row];
      }
      tc_fence_before();
      named_bar_sync(1, 256);
    }
  }
#undef FULL
#undef EMPTY
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, TCOLS);
}

// ---------------------------------------------------------------------------------------------
// The same sweep on a CTA pair (cta_group::2): the two CTAs of a cluster own two 128-chain
// blocks and share every W box — each loads half of its NT rows, and the leader's MMAs
// (M = 256, 128 rows per CTA) read both halves.  Per SM this halves the W stream through
// shared memory and the MMA instructions per site.  The peer's A-tile arrivals on the
// leader's barriers are plain remote arrivals (see ptx.cuh: mbar_arrive_remote).
template <int NT>
struct Sa2Cfg {
  static constexpr int HBOX = (NT / 2) * 128;   // this CTA's half of a W box
  static constexpr int RW = 8;
  static constexpr int ABOX = kBM * 128;
  static constexpr int RA = 4;
  static constexpr int NBAR = 2 * RW + 2 * RA + 1;
  static size_t smem_bytes(int W) {
    return 1024 + (size_t)RW * HBOX + (size_t)RA * ABOX + 8 * NBAR + 16 + (size_t)(W + 2) * kBM * 4 + kBM * 4 + 128;
  }
};

template <int NT>
__global__ void __launch_bounds__(kThreads, 1) sa2_kernel(const __grid_constant__ CUtensorMap tmap, const SaParams p) {
  using C = Sa2Cfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sW = base;
  const uint32_t sA = sW + C::RW * C::HBOX;
  const uint32_t sBar = sA + C::RA * C::ABOX;
#define FULLW(s) (sBar + 8u * (s))
#define EMPTYW(s) (sBar + 8u * (C::RW + (s)))
#define FULLA(s) (sBar + 8u * (2 * C::RW + (s)))
#define EMPTYA(s) (sBar + 8u * (2 * C::RW + C::RA + (s)))
  const uint32_t SITE = sBar + 8u * (2 * C::RW + 2 * C::RA);
  const uint32_t tslot = SITE + 8;
  const uint32_t sX = (tslot + 16 + 127u) & ~127u;
  uint32_t* xs = reinterpret_cast<uint32_t*>(gbase + (sX - base));
  int* sS = reinterpret_cast<int*>(gbase + (sX - base) + (size_t)(p.W + 2) * kBM * 4);
  volatile uint32_t* tslot_g = reinterpret_cast<volatile uint32_t*>(gbase + (tslot - base));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int NPAD = NT * p.n_ct;
  const long long n_cb = (p.B + kBM - 1) / kBM;
  const long long n_pairs = (n_cb + 1) / 2;
  if (threadIdx.x == 0) {
    for (int s = 0; s < C::RW; ++s) { mbar_init(FULLW(s), 1); mbar_init(EMPTYW(s), 1); }
    for (int s = 0; s < C::RA; ++s) { mbar_init(FULLA(s), 8); mbar_init(EMPTYA(s), 1); }
    mbar_init(SITE, 1);
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch_desc(&tmap);
  if (warp == 1) tmem_alloc_pair(tslot, (uint32_t)NPAD);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tslot_g;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t nw = 0;
      for (long long pr = blockIdx.x / 2; pr < n_pairs; pr += gridDim.x / 2)
        for (long long step = 0; step < p.steps; ++step) {
          const int m = (int)(step % p.N);
          const int L = __ldg(p.site_L + m), sb = __ldg(p.site_base + m);
          for (int q = 0; q < p.nq; ++q) {
            const int kb = sa_site_kb(p, q);
            for (int l = 0; l < L; ++l)
              for (int h = 0; h < p.n_ct; ++h, ++nw) {
                const uint32_t s = nw % C::RW;
                mbar_wait(EMPTYW(s), ((nw / C::RW) & 1u) ^ 1u);
                if (leader) mbar_arrive_expect_tx(FULLW(s), 2 * C::HBOX);
                tma_load_3d_pair(sW + s * C::HBOX, &tmap, mapa_shared(FULLW(s), 0), 0, (int)rank * (NT / 2),
                                 sb + (l * p.n_ct + h) * p.nkb1 + kb);
              }
          }
        }
    }
  } else if (warp == 1) {
    if (leader) {   // whole warp in the loop, one elected lane issues
      constexpr uint32_t idesc = idesc_bf16_f32(2 * kBM, NT);
      uint32_t nw = 0, na = 0;
      for (long long pr = blockIdx.x / 2; pr < n_pairs; pr += gridDim.x / 2)
        for (long long step = 0; step < p.steps; ++step) {
          const int m = (int)(step % p.N);
          const int L = __ldg(p.site_L + m);
          for (int q = 0; q < p.nq; ++q, ++na) {
            const uint32_t a = na % C::RA;
            mbar_wait(FULLA(a), (na / C::RA) & 1u);
            tc_fence_after();
            const uint64_t adesc = sw128_kmajor_desc(sA + a * C::ABOX);
            for (int l = 0; l < L; ++l)
              for (int h = 0; h < p.n_ct; ++h, ++nw) {
                const uint32_t s = nw % C::RW;
                mbar_wait(FULLW(s), (nw / C::RW) & 1u);
                tc_fence_after();
                const uint64_t bdesc = sw128_kmajor_desc(sW + s * C::HBOX);
                if (elect_one()) {
#pragma unroll
                  for (int k = 0; k < kBK / 16; ++k)
                    umma_bf16_ss_pair(tmem + (uint32_t)(h * NT), adesc + 2u * k, bdesc + 2u * k, idesc, 1u);
                  umma_commit_pair(EMPTYW(s), 3);
                }
                __syncwarp();
              }
            if (elect_one()) umma_commit_pair(EMPTYA(a), 3);
            __syncwarp();
          }
          if (elect_one()) umma_commit_pair(SITE, 3);
          __syncwarp();
        }
    }
  } else {
    const int qd = warp & 3;
    const int h = (warp - 2) >> 2;
    const int row = qd * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(qd * 32) << 16);
    const int gtid = threadIdx.x - 64;
    uint32_t na = 0, nsite = 0;
    for (long long pr = blockIdx.x / 2; pr < n_pairs; pr += gridDim.x / 2) {
      const long long cb = 2 * pr + rank;
      const long long b0 = cb * kBM, b = b0 + row;
      const bool live = b < p.B;
      const int Wp = p.W + 2;
      for (int i = gtid; i < Wp * kBM; i += 256) {
        const int r = i / Wp, w = i % Wp;
        xs[w * kBM + r] = (w < p.W && b0 + r < p.B) ? p.bits[(size_t)(b0 + r) * p.W + w] : 0u;
      }
      for (int c0 = h * (NPAD / 2); c0 < (h + 1) * (NPAD / 2); c0 += 32) {
        uint32_t v[32];
#pragma unroll
        for (int c = 0; c < 32; ++c)
          v[c] = (live && c0 + c < p.N) ? __float_as_uint(__ldg(p.G0 + (size_t)b * p.N + c0 + c)) : 0u;
        tmem_st32(lane_base + (uint32_t)c0, v);
      }
      tmem_st_wait();
      double E = (h == 0 && live) ? p.E[b] : 0.0;
      tc_fence_before();
      named_bar_sync(1, 256);
      tc_fence_after();
      for (long long step = 0; step < p.steps; ++step) {
        const int m = (int)(step % p.N);
        double thr = 0.0;
        if (h == 0 && live) {
          const double u = (double)(d_hash(p.seed, 4, (uint64_t)(p.chain0 + b), (uint64_t)step) >> 11) * 0x1.0p-53;
          thr = -__ldg(p.temps + step / p.N) * log(u);
        }
        if (step > 0) {
          mbar_wait(SITE, nsite & 1u);
          ++nsite;
          tc_fence_after();
        }
        if (h == 0) {
          const float g = __uint_as_float(tmem_ld1(lane_base + (uint32_t)m));
          tmem_ld_wait();
          int sv = 0;
          if (live) {
            const int wi = m >> 5;
            const uint32_t bit = 1u << (m & 31);
            const bool xm = (xs[wi * kBM + row] & bit) != 0u;
            const float d = xm ? -g : g;
            if (d <= 0.0f || (double)d < thr) {
              sv = xm ? -1 : 1;
              xs[wi * kBM + row] ^= bit;
              E += (double)d;
            }
          }
          sS[row] = sv;
          tc_fence_before();
        }
        named_bar_sync(1, 256);
        const int sv = sS[row];
        const uint32_t sgn = sv < 0 ? 0x80008000u : 0u;
        for (int q = 0; q < p.nq; ++q, ++na) {
          if ((q & 1) != h) continue;
          const uint32_t a = na % C::RA;
          mbar_wait(EMPTYA(a), ((na / C::RA) & 1u) ^ 1u);
          const int kb = sa_site_kb(p, q);
          uint64_t bits = 0;
          if (sv != 0) {
            if (kb == p.nkb1 - 1) bits = 1ull;
            else bits = block_bits(xs, row, __ldg(p.kdesc + 2 * kb), __ldg(p.kdesc + 2 * kb + 1), p.runs);
          }
          uint32_t w[32];
          expand32((uint32_t)bits, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
          expand32((uint32_t)(bits >> 32), *reinterpret_cast<uint32_t(*)[16]>(&w[16]));
          const uint32_t rowaddr = sA + a * C::ABOX + (uint32_t)(row >> 3) * 1024u + (uint32_t)(row & 7) * 128u;
#pragma unroll
          for (int c = 0; c < 8; ++c)
            st_shared_v4(rowaddr + (uint32_t)((c ^ (row & 7)) << 4), w[4 * c] ^ sgn, w[4 * c + 1] ^ sgn,
                         w[4 * c + 2] ^ sgn, w[4 * c + 3] ^ sgn);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (leader) mbar_arrive(FULLA(a));
            else mbar_arrive_remote(mapa_shared(FULLA(a), 0));
          }
        }
      }
      if (p.steps > 0) {
        mbar_wait(SITE, nsite & 1u);
        ++nsite;
        tc_fence_after();
      }
      if (h == 0 && live) {
        p.E[b] = E;
        for (int w = 0; w < p.W; ++w) p.bits[(size_t)b * p.W + w] = xs[w * kBM + row];
      }
      tc_fence_before();
      named_bar_sync(1, 256);
    }
  }
#undef FULLW
#undef EMPTYW
#undef FULLA
#undef EMPTYA
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) tmem_dealloc_pair(tmem, (uint32_t)NPAD);
}

}  // namespace hobo
