// persist.cuh — the persistent energy-mode contraction for short K loops (sm_100a).
//
// Same computation as kr_gemm_kernel's energy mode (batched as in
// PAPER.md:141-149): per (candidate block, column tile)
// F[b, m] = sum_T A[b, T] W[m, T] over the strict last-index-open layout, and the tile's
// energy partial Q[ct][b] = sum_m x_bm (F[b, m] + c({m})).  What differs is the schedule.
// kr_gemm_kernel runs one CTA per tile, so a tile's pipeline fill, X staging and epilogue
// sit between its MMAs and the next tile's; with QUBO-like K loops of 2-16 K-blocks
// (BASELINE config 2) that fixed cost is larger than the MMA time.  Here:
//   * one CTA pair (cta_group::2, M = 256 candidates) per two SMs stays resident and walks a
//     contiguous range of (candidate-block pair, column tile) items, balanced by MMA work
//     on the host (hobo_api.cu: persist_items);
//   * the W ring, the A ring and the MMA issue run continuously across items;
//   * TWO accumulators (128-column tiles: 2 x 128 TMEM columns, the A stages in the other 256)
//     let item i+1's MMAs run while dedicated epilogue warps drain item i;
//   * the candidate bits are restaged only when the candidate block changes.
// Warps: 0 TMA producer, 1 MMA issuer, 2-9 A generator (two teams, one K-block of each
// 2-K-block stage), 10-13 epilogue (TMEM lane quarter = warp % 4).
#pragma once
#include "kernels.cuh"

namespace hobo {

constexpr int kPThreads = 448;

template <int KPS_>
struct PersistCfgT {
  static constexpr int NT = 128;                     // column tile (UMMA N)
  static constexpr int KPS = KPS_;                   // K-blocks per stage
  static constexpr int HBOX = (NT / 2) * 128;        // this CTA's half of one W box (64 rows x 64 bf16)
  static constexpr int MAXL = 3;                     // limb planes
  static constexpr int NST = 8 / KPS;                // ring stages (TMEM: 256 A columns)
  static constexpr int STAGE = KPS * MAXL * HBOX;    // 24 KB per K-block
  static constexpr int ACOLS = kBK / 2;              // TMEM columns of one bf16 K-block of A
  static constexpr int A0 = 2 * NT;                  // first A column (after the two accumulators)
  static constexpr int NBAR = 2 * NST + 4;
  static size_t smem_bytes(int W) { return 1024 + (size_t)NST * STAGE + 8 * NBAR + 16 + 128 + (size_t)(W + 2) * kBM * 4; }
};

struct PersistParams {
  const uint32_t* xbits;    // [B][W] bit-packed candidates
  const uint4* runs;        // A-generator runs (host_compile.cpp build_klayout)
  const uint4* kdesc;       // [n_kb][2] per-K-block descriptor
  const int2* sched;        // [n_ct][nseg] (first K-block, #K-blocks), energy layout, 128-column tiles
  const float* p1;          // [Npad] degree-1 cells
  double* Q;                // [n_ct][B] energy partials
  const int* items;         // [npairs + 1]: pair p walks items [items[p], items[p+1]); item = cbp * n_ct + (n_ct-1-ct)
  long long B;
  int N, W, n_ct, n_cbp, nseg, L, n_kb;
  int exp;                  // measurement switch (HOBO_PERSIST_EXP, wrong results): 1 no epilogue math, 2 no A
                            // decoding, 4 no bit restaging, 8 no MMAs, 16 every pair walks pair 0's items
};

using PersistCfg = PersistCfgT<1>;

// KPS = 2: both generator teams build one K-block of each stage; KPS = 1: the teams take whole
// stages in turn (twice the stages of half the size in the same ring)
template <int KPS>
__global__ void __launch_bounds__(kPThreads, 1) kr_persist_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                   const PersistParams p) {
  using C = PersistCfgT<KPS>;
  constexpr int NT = C::NT;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;  // SW128 atoms need 1024-byte alignment
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sB = base;
  const uint32_t sBar = sB + C::NST * C::STAGE;
#define FULL(s) (sBar + 8u * (s))
#define EMPTY(s) (sBar + 8u * (C::NST + (s)))
  const uint32_t ACC_FULL0 = sBar + 8u * (2 * C::NST);       // + 8 * buf
  const uint32_t ACC_EMPTY0 = ACC_FULL0 + 16;                  // + 8 * buf (leader: 8 epilogue warps of the pair)
  const uint32_t tslot = sBar + 8u * C::NBAR;
  const uint32_t sX = (tslot + 16 + 127u) & ~127u;
  uint32_t* xs = reinterpret_cast<uint32_t*>(gbase + (sX - base));
  volatile uint32_t* tslot_g = reinterpret_cast<volatile uint32_t*>(gbase + (tslot - base));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t prank = cluster_ctarank();
  const bool leader = prank == 0;
  const int pair = (int)(blockIdx.x >> 1);
  const int pr = (p.exp & 16) ? 0 : pair;   // exp 16: every pair walks pair 0's items (lockstep W stream)
  const int it0 = __ldg(p.items + pr), it1 = __ldg(p.items + pr + 1);
  auto item_ct = [&](int it) { return p.n_ct - 1 - it % p.n_ct; };   // heaviest tile of a block first
  auto item_cb = [&](int it) { return 2 * (it / p.n_ct) + (int)prank; };
  const uint32_t stage_bytes = (uint32_t)(C::KPS * p.L) * C::HBOX;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NST; ++s) { mbar_init(FULL(s), KPS == 2 ? 17 : 9); mbar_init(EMPTY(s), 1); }   // TMA + gen warps of both CTAs
    for (int b = 0; b < 2; ++b) { mbar_init(ACC_FULL0 + 8u * b, 1); mbar_init(ACC_EMPTY0 + 8u * b, 8); }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch_desc(&tmap);
  if (warp == 1) tmem_alloc_pair(tslot, 512);
  // candidate bits of a block, column-major xs[w][row] (+2 zero words for window reads)
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
        if (i < Wp * kBM) xs[i] = v[u];
      }
    }
  };
  if (it0 < it1) stage_x((long long)item_cb(it0) * kBM, (int)threadIdx.x, kPThreads);
  tc_fence_before();
  cluster_sync_all();   // both CTAs' barriers initialised, TMEM allocated, first bits staged
  tc_fence_after();
  const uint32_t tmem = *tslot_g;

  if (warp == 0) {
    // ---------------- TMA producer: this CTA's half of every W box, all items back to back ----
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int it = it0; it < it1; ++it) {
        const int ct = item_ct(it);
        for (int j = p.nseg - 1; j >= 0; --j) {
          const int2 s = __ldg(p.sched + (size_t)ct * p.nseg + j);
          for (int kb0 = s.x; kb0 < s.x + s.y; kb0 += C::KPS) {
            const int nkb = min(C::KPS, s.x + s.y - kb0);
            mbar_wait(EMPTY(st), ph ^ 1u);
            if (leader) mbar_arrive_expect_tx(FULL(st), (uint32_t)(nkb * p.L) * (2 * C::HBOX));   // both halves
            for (int q = 0; q < nkb; ++q)
              for (int l = 0; l < p.L; ++l) {
                const int box = (l * p.n_ct + ct) * p.n_kb + kb0 + q;
                const uint32_t dst = sB + st * stage_bytes + (uint32_t)(q * p.L + l) * C::HBOX;
                tma_load_3d_pair(dst, &tmap, mapa_shared(FULL(st), 0), 0, (int)prank * (NT / 2), box);
              }
            if (++st == C::NST) { st = 0; ph ^= 1u; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader): M = 256 over the pair, accumulator it & 1 ---------
    if (leader) {
      constexpr uint32_t idesc = idesc_bf16_f32(2 * kBM, NT);
      int st = 0;
      uint32_t ph = 0;
      for (int it = it0, n = 0; it < it1; ++it, ++n) {
        const int buf = n & 1;
        const uint32_t acc = tmem + (uint32_t)(buf * NT);
        mbar_wait(ACC_EMPTY0 + 8u * buf, (uint32_t)(((n >> 1) & 1) ^ 1));   // item n-2's epilogue is done
        tc_fence_after();
        const int ct = item_ct(it);
        uint32_t issued = 0;
        for (int j = p.nseg - 1; j >= 0; --j) {
          const int2 s = __ldg(p.sched + (size_t)ct * p.nseg + j);
          for (int kb0 = s.x; kb0 < s.x + s.y; kb0 += C::KPS) {
            const int nkb = min(C::KPS, s.x + s.y - kb0);
            mbar_wait(FULL(st), ph);
            tc_fence_after();
            if (elect_one()) {
              if (p.exp & 8) {
              } else if (nkb == KPS && p.L == 3) {   // the common stage, fully unrolled
#pragma unroll
                for (int q = 0; q < KPS; ++q)
#pragma unroll
                  for (int l = 0; l < 3; ++l) {
                    const uint32_t a_t = tmem + (uint32_t)(C::A0 + (st * C::KPS + q) * C::ACOLS);
                    const uint64_t bd = sw128_kmajor_desc(sB + st * stage_bytes + (uint32_t)(q * 3 + l) * C::HBOX);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                      umma_bf16_ts_pair(acc, a_t + 8u * k, bd + 2u * k, idesc, issued | (uint32_t)(q | l | k));
                  }
              } else {
                for (int q = 0; q < nkb; ++q)
                  for (int l = 0; l < p.L; ++l) {
                    const uint32_t a_t = tmem + (uint32_t)(C::A0 + (st * C::KPS + q) * C::ACOLS);
                    const uint64_t bd = sw128_kmajor_desc(sB + st * stage_bytes + (uint32_t)(q * p.L + l) * C::HBOX);
#pragma unroll
                    for (int k = 0; k < kBK / 16; ++k)
                      umma_bf16_ts_pair(acc, a_t + 8u * k, bd + 2u * k, idesc, issued | (uint32_t)(q | l | k));
                  }
              }
              umma_commit_pair(EMPTY(st), 3);
            }
            __syncwarp();
            issued = 1;
            if (++st == C::NST) { st = 0; ph ^= 1u; }
          }
        }
        if (elect_one()) {
          if (issued) umma_commit_pair(ACC_FULL0 + 8u * buf, 3);
          else { mbar_arrive(ACC_FULL0 + 8u * buf); mbar_arrive_remote(mapa_shared(ACC_FULL0 + 8u * buf, 1)); }
        }
        __syncwarp();
      }
    }
  } else if (warp < 10) {
    // ---------------- A generator: team h builds K-block h of every 2-K-block stage ----------
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    int gst = 0, gn = 0;
    uint32_t gph = 0;
    int cb_staged = it0 < it1 ? item_cb(it0) : -1;
    for (int it = it0; it < it1; ++it) {
      const int cb = item_cb(it);
      if (cb != cb_staged && !(p.exp & 4)) {   // every generator warp is done with the previous block's bits
        named_bar_sync(1, 256);
        stage_x((long long)cb * kBM, (int)threadIdx.x - 64, 256);
        named_bar_sync(1, 256);
        cb_staged = cb;
      }
      const int ct = item_ct(it);
      for (int j = p.nseg - 1; j >= 0; --j) {
        const int2 s = __ldg(p.sched + (size_t)ct * p.nseg + j);
        const int kend = s.x + s.y;
        for (int kb0 = s.x; kb0 < kend; kb0 += C::KPS, ++gn) {
          if (KPS == 1 && (gn & 1) != h) {   // the other team's stage
            if (++gst == C::NST) { gst = 0; gph ^= 1u; }
            continue;
          }
          const int kb = kb0 + (KPS == 2 ? h : 0);
          const bool mine = kb < kend;
          uint64_t bits = 0ull;
          if (mine && !(p.exp & 2)) bits = block_bits(xs, row, __ldg(p.kdesc + 2 * kb), __ldg(p.kdesc + 2 * kb + 1), p.runs);
          mbar_wait(EMPTY(gst), gph ^ 1u);
          if (mine) {
            tc_fence_after();
            uint32_t w[32];
            expand32((uint32_t)bits, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
            expand32((uint32_t)(bits >> 32), *reinterpret_cast<uint32_t(*)[16]>(&w[16]));
            tmem_st32(lane_base + (uint32_t)(C::A0 + (gst * C::KPS + (KPS == 2 ? h : 0)) * C::ACOLS), w);
            tmem_st_wait();
            tc_fence_before();
          }
          __syncwarp();
          if (lane == 0) {
            if (!leader) mbar_arrive_remote(mapa_shared(FULL(gst), 0));
            else mbar_arrive(FULL(gst));
          }
          if (++gst == C::NST) { gst = 0; gph ^= 1u; }
        }
      }
    }
  } else {
    // ---------------- epilogue: Q[ct][b] = sum_m x_bm (F[b, m] + c({m})) ----------------------
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    for (int it = it0, n = 0; it < it1; ++it, ++n) {
      const int buf = n & 1;
      const int ct = item_ct(it);
      const long long b = (long long)item_cb(it) * kBM + row;
      const bool live = b < p.B;
      // this tile's candidate bits and degree-1 cells, loaded before the accumulator is ready
      uint32_t xw[NT / 32];
#pragma unroll
      for (int c = 0; c < NT / 32; ++c) {
        const int w = ct * (NT / 32) + c;
        xw[c] = (live && w < p.W) ? __ldg(p.xbits + (size_t)b * p.W + w) : 0u;
      }
      mbar_wait(ACC_FULL0 + 8u * buf, (uint32_t)((n >> 1) & 1));
      tc_fence_after();
      // per 32-column chunk: v_c = x_c ? F_c + c({c}) : 0 summed by a fp32 tree, then one fp64
      // add.  Integer instances with sum|H| < 2^24 stay exact (every partial sum is an integer
      // below 2^24, reading 10); for fp32 cells the tree adds at most 31 u sum|v|
      // (u = 2^-24) per chunk, well inside tau = 1e-5 sum|H| (the per-element fp64 chain this
      // replaces held the FP64 pipe longer than the tile's MMAs took)
      double q = 0.0;
#pragma unroll
      for (int c0 = 0; c0 < (p.exp & 1 ? 0 : NT); c0 += 32) {
        const int mbase = ct * NT + c0;
        float v[32];
#pragma unroll
        for (int c = 0; c < 32; c += 4) {
          const float4 v4 = __ldg(reinterpret_cast<const float4*>(p.p1 + mbase + c));
          v[c] = v4.x; v[c + 1] = v4.y; v[c + 2] = v4.z; v[c + 3] = v4.w;
        }
        uint32_t r[32];
        tmem_ld32(lane_base + (uint32_t)(buf * NT + c0), r);
        tmem_ld_wait();
        const uint32_t x = xw[c0 / 32];
#pragma unroll
        for (int c = 0; c < 32; ++c) v[c] = ((x >> c) & 1u) ? __uint_as_float(r[c]) + v[c] : 0.0f;
#pragma unroll
        for (int w = 16; w >= 1; w >>= 1)
#pragma unroll
          for (int c = 0; c < w; ++c) v[c] += v[c + w];
        q += (double)v[0];
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {   // the accumulator is free for item n + 2 (the leader's MMA waits on both CTAs)
        if (!leader) mbar_arrive_remote(mapa_shared(ACC_EMPTY0 + 8u * buf, 0));
        else mbar_arrive(ACC_EMPTY0 + 8u * buf);
      }
      if (live) p.Q[(size_t)ct * p.B + b] = q;
    }
  }
#undef FULL
#undef EMPTY
  tc_fence_before();
  cluster_sync_all();   // the leader's last MMAs wrote both CTAs' TMEM
  if (warp == 1) tmem_dealloc_pair(tmem, 512);
}

// ------------------------------------------------------------------------------------------
// The same persistent schedule on int8 digit planes: every
// cell of degree >= 2 is q 2^e with q a d-byte integer (d <= 3); each plane accumulates into
// its own s32 accumulator, so the tile energy is an exact integer rounded once.  An int8 MMA
// runs at twice the bf16 rate on half the bytes, so for 3 digits against 3 bf16 limbs both the
// MMA time and the W stream from L2 halve.  TMEM: two accumulator sets of d x 64 columns
// (64-column tiles: 2 x 3 x 64 = 384) and the A stages (32 columns per K-block pair) in the
// rest; the W ring (smem) runs deeper than the A ring (TMEM), each with its own barriers.
template <int NT_>
struct PersistI8Cfg {
  static constexpr int NT = NT_;                     // column tile (UMMA N): 64 or 128
  static constexpr int HBOX = (NT / 2) * 128;        // this CTA's half of one plane box (NT/2 rows x 128 bytes)
  static constexpr int MAXP = 3;                     // digit planes
  static constexpr int WST = NT == 64 ? 12 : 6;      // W ring stages (one K-block pair each)
  static constexpr int MAXA = 8;                     // A ring stages (TMEM)
  static constexpr int ACOLS = 32;                   // TMEM columns of one K-block pair of A (128 bytes)
  static constexpr int NBAR = 2 * WST + 2 * MAXA + 4;
  // accumulator sets: two when 2 x d x NT columns leave room for A (64-column tiles), else one
  // (128-column tiles: the next item's MMAs wait for the epilogue's accumulator read)
  __host__ __device__ static int nbuf(int P) { return 2 * P * NT <= 384 ? 2 : 1; }
  __host__ __device__ static int nsta(int P) {
    return (512 - nbuf(P) * P * NT) / ACOLS < MAXA ? (512 - nbuf(P) * P * NT) / ACOLS : MAXA;
  }
  static size_t smem_bytes(int W) {
    return 1024 + (size_t)WST * MAXP * HBOX + 8 * NBAR + 16 + 128 + (size_t)(W + 2) * kBM * 4;
  }
};

struct PersistI8Params {
  const uint32_t* xbits;    // [B][W] bit-packed candidates
  const uint4* runs;        // A-generator runs
  const uint4* kdesc;       // [n_kb][2] per-K-block descriptor
  const int2* sched;        // [n_ct][nseg], energy layout, 64-column tiles
  const float* p1;          // [Npad] degree-1 cells (used when !p1_int)
  const int* p1q;           // [Npad] degree-1 cells / qscale when every one is on the digit grid
  int p1_int;
  double qscale;            // cell = qscale * q
  double* Q;                // [n_ct][B] energy partials (exact values rounded once to double)
  const int* items;         // per-pair item ranges (as PersistParams)
  long long B;
  int N, W, n_ct, nseg, P, n_kb;
  int exp;                  // measurement switch, as PersistParams::exp
};

template <int NT_>
__global__ void __launch_bounds__(kPThreads, 1) kr_persist_i8_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                      const PersistI8Params p) {
  using C = PersistI8Cfg<NT_>;
  constexpr int NT = C::NT;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* gbase = smem_raw + (base - raw);
  const uint32_t sB = base;
  const uint32_t stage_bytes = (uint32_t)p.P * C::HBOX;
  const uint32_t sBar = sB + C::WST * C::MAXP * C::HBOX;
#define FULL(s) (sBar + 8u * (s))
#define EMPTY(s) (sBar + 8u * (C::WST + (s)))
#define FULLA(s) (sBar + 8u * (2 * C::WST + (s)))
#define EMPTYA(s) (sBar + 8u * (2 * C::WST + C::MAXA + (s)))
  const uint32_t ACC_FULL0 = sBar + 8u * (2 * C::WST + 2 * C::MAXA);
  const uint32_t ACC_EMPTY0 = ACC_FULL0 + 16;
  const uint32_t tslot = sBar + 8u * C::NBAR;
  const uint32_t sX = (tslot + 16 + 127u) & ~127u;
  uint32_t* xs = reinterpret_cast<uint32_t*>(gbase + (sX - base));
  volatile uint32_t* tslot_g = reinterpret_cast<volatile uint32_t*>(gbase + (tslot - base));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t prank = cluster_ctarank();
  const bool leader = prank == 0;
  const int pair = (int)(blockIdx.x >> 1);
  const int it0 = __ldg(p.items + pair), it1 = __ldg(p.items + pair + 1);
  auto item_ct = [&](int it) { return p.n_ct - 1 - it % p.n_ct; };
  auto item_cb = [&](int it) { return 2 * (it / p.n_ct) + (int)prank; };
  const int NSTA = C::nsta(p.P);
  const int NBUF = C::nbuf(p.P);
  const uint32_t A0 = (uint32_t)(NBUF * p.P * NT);

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::WST; ++s) { mbar_init(FULL(s), 1); mbar_init(EMPTY(s), 1); }
    for (int s = 0; s < C::MAXA; ++s) { mbar_init(FULLA(s), 8); mbar_init(EMPTYA(s), 1); }   // one team x 2 CTAs
    for (int b = 0; b < 2; ++b) { mbar_init(ACC_FULL0 + 8u * b, 1); mbar_init(ACC_EMPTY0 + 8u * b, 8); }
    fence_mbar_init();
  }
  if (warp == 0 && lane == 0) tma_prefetch_desc(&tmap);
  if (warp == 1) tmem_alloc_pair(tslot, 512);
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
        if (i < Wp * kBM) xs[i] = v[u];
      }
    }
  };
  if (it0 < it1) stage_x((long long)item_cb(it0) * kBM, (int)threadIdx.x, kPThreads);
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = *tslot_g;

  if (warp == 0) {
    // ---------------- TMA producer: this CTA's half of each plane box, one K-block pair per stage
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int it = it0; it < it1; ++it) {
        const int ct = item_ct(it);
        for (int j = p.nseg - 1; j >= 0; --j) {
          const int2 s = __ldg(p.sched + (size_t)ct * p.nseg + j);
          for (int kb0 = s.x; kb0 < s.x + s.y; kb0 += 2) {
            mbar_wait(EMPTY(st), ph ^ 1u);
            if (leader) mbar_arrive_expect_tx(FULL(st), stage_bytes * 2u);   // both halves
            for (int l = 0; l < p.P; ++l) {
              const int box = (l * p.n_ct + ct) * (p.n_kb >> 1) + (kb0 >> 1);
              tma_load_3d_pair(sB + st * stage_bytes + (uint32_t)l * C::HBOX, &tmap, mapa_shared(FULL(st), 0), 0,
                               (int)prank * (NT / 2), box);
            }
            if (++st == C::WST) { st = 0; ph ^= 1u; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader): d planes x 4 MMAs (K = 32 bytes) per K-block pair ---
    if (leader) {
      constexpr uint32_t id_u = idesc_i8_s32(2 * kBM, NT, 0), id_s = idesc_i8_s32(2 * kBM, NT, 1);
      int st = 0, sa = 0;
      uint32_t ph = 0, pha = 0;
      for (int it = it0, n = 0; it < it1; ++it, ++n) {
        const int buf = NBUF == 2 ? (n & 1) : 0, use = NBUF == 2 ? (n >> 1) : n;
        const uint32_t acc = tmem + (uint32_t)(buf * p.P * NT);
        mbar_wait(ACC_EMPTY0 + 8u * buf, (uint32_t)((use & 1) ^ 1));   // the buffer's previous item is drained
        tc_fence_after();
        const int ct = item_ct(it);
        uint32_t issued = 0;
        for (int j = p.nseg - 1; j >= 0; --j) {
          const int2 s = __ldg(p.sched + (size_t)ct * p.nseg + j);
          for (int kb0 = s.x; kb0 < s.x + s.y; kb0 += 2) {
            mbar_wait(FULL(st), ph);
            mbar_wait(FULLA(sa), pha);
            tc_fence_after();
            if (elect_one()) {
              const uint32_t a_t = tmem + A0 + (uint32_t)(sa * C::ACOLS);
              const uint32_t sbase = sB + st * stage_bytes;
              if (p.exp & 8) {
              } else if (p.P == 3) {
#pragma unroll
                for (int l = 0; l < 3; ++l) {
                  const uint64_t bd = sw128_kmajor_desc(sbase + (uint32_t)l * C::HBOX);
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk)
                    umma_i8_ts_pair(acc + (uint32_t)(l * NT), a_t + 8u * kk, bd + 2u * kk, l == 2 ? id_s : id_u,
                                    kk ? 1u : issued);
                }
              } else {
                for (int l = 0; l < p.P; ++l) {
                  const uint64_t bd = sw128_kmajor_desc(sbase + (uint32_t)l * C::HBOX);
#pragma unroll
                  for (int kk = 0; kk < 4; ++kk)
                    umma_i8_ts_pair(acc + (uint32_t)(l * NT), a_t + 8u * kk, bd + 2u * kk, l == p.P - 1 ? id_s : id_u,
                                    kk ? 1u : issued);
                }
              }
              umma_commit_pair(EMPTY(st), 3);
              umma_commit_pair(EMPTYA(sa), 3);
            }
            __syncwarp();
            issued = 1;
            if (++st == C::WST) { st = 0; ph ^= 1u; }
            if (++sa == NSTA) { sa = 0; pha ^= 1u; }
          }
        }
        if (elect_one()) {
          if (issued) umma_commit_pair(ACC_FULL0 + 8u * buf, 3);
          else { mbar_arrive(ACC_FULL0 + 8u * buf); mbar_arrive_remote(mapa_shared(ACC_FULL0 + 8u * buf, 1)); }
        }
        __syncwarp();
      }
    }
  } else if (warp < 10) {
    // ---------------- A generator: the two teams take whole stages in turn; a stage is the
    // K-block pair (kb0, kb0 + 1) as bytes {0, 1}, written with one 32-column tcgen05.st
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    const int row = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    int gst = 0, gn = 0;
    uint32_t gph = 0;
    int cb_staged = it0 < it1 ? item_cb(it0) : -1;
    for (int it = it0; it < it1; ++it) {
      const int cb = item_cb(it);
      if (cb != cb_staged) {
        named_bar_sync(1, 256);
        stage_x((long long)cb * kBM, (int)threadIdx.x - 64, 256);
        named_bar_sync(1, 256);
        cb_staged = cb;
      }
      const int ct = item_ct(it);
      for (int j = p.nseg - 1; j >= 0; --j) {
        const int2 s = __ldg(p.sched + (size_t)ct * p.nseg + j);
        const int kend = s.x + s.y;
        for (int kb0 = s.x; kb0 < kend; kb0 += 2, ++gn) {
          if ((gn & 1) == h) {
            const uint64_t b0 = (p.exp & 2) ? 0ull : block_bits(xs, row, __ldg(p.kdesc + 2 * kb0), __ldg(p.kdesc + 2 * kb0 + 1), p.runs);
            const uint64_t b1 = (kb0 + 1 < kend && !(p.exp & 2))
                                    ? block_bits(xs, row, __ldg(p.kdesc + 2 * kb0 + 2), __ldg(p.kdesc + 2 * kb0 + 3), p.runs)
                                    : 0ull;
            uint32_t w[32];   // the K-block pair's bytes in the planes' permuted K order
            expand_bytes64(b0, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
            expand_bytes64(b1, *reinterpret_cast<uint32_t(*)[16]>(&w[16]));
            mbar_wait(EMPTYA(gst), gph ^ 1u);
            tc_fence_after();
            tmem_st32(lane_base + A0 + (uint32_t)(gst * C::ACOLS), w);
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
              if (!leader) mbar_arrive_remote(mapa_shared(FULLA(gst), 0));
              else mbar_arrive(FULLA(gst));
            }
          }
          if (++gst == NSTA) { gst = 0; gph ^= 1u; }
        }
      }
    }
  } else {
    // ---------------- epilogue: Q[ct][b] = qscale sum_m x_bm sum_l 256^l acc_l[m] + degree 1 ----
    // per plane a masked int32 sum (|acc| <= 255 x tuples, times 64 columns < 2^31), combined
    // in int64: the tile energy is exact; the degree-1 cells join as integers when they are on
    // the digit grid (else in double)
    const int q = warp & 3;
    const int row = q * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
    for (int it = it0, n = 0; it < it1; ++it, ++n) {
      const int buf = NBUF == 2 ? (n & 1) : 0, use = NBUF == 2 ? (n >> 1) : n;
      const int ct = item_ct(it);
      const long long b = (long long)item_cb(it) * kBM + row;
      const bool live = b < p.B;
      uint32_t xw[NT / 32];
#pragma unroll
      for (int c = 0; c < NT / 32; ++c) {
        const int w = ct * (NT / 32) + c;
        xw[c] = (live && w < p.W) ? __ldg(p.xbits + (size_t)b * p.W + w) : 0u;
      }
      mbar_wait(ACC_FULL0 + 8u * buf, (uint32_t)(use & 1));
      tc_fence_after();
      long long tot = 0;
      double d1 = 0.0;
#pragma unroll
      for (int c0 = 0; c0 < (p.exp & 1 ? 0 : NT); c0 += 32) {
        const uint32_t x = xw[c0 / 32];
        const int mbase = ct * NT + c0;
        // 16 columns of every plane loaded together, one wait (the loads' latency paid once)
#pragma unroll
        for (int hc = 0; hc < 32; hc += 16) {
          uint32_t r[C::MAXP][16];
#pragma unroll
          for (int l = 0; l < C::MAXP; ++l)
            if (l < p.P) tmem_ld16(lane_base + (uint32_t)(buf * p.P * NT + l * NT + c0 + hc), r[l]);
          tmem_ld_wait();
#pragma unroll
          for (int l = 0; l < C::MAXP; ++l) {
            if (l >= p.P) break;
            int v[16];
#pragma unroll
            for (int c = 0; c < 16; ++c) v[c] = ((x >> (hc + c)) & 1u) ? (int)r[l][c] : 0;
#pragma unroll
            for (int w = 8; w >= 1; w >>= 1)
#pragma unroll
              for (int c = 0; c < w; ++c) v[c] += v[c + w];
            tot += (long long)v[0] * (1ll << (8 * l));
          }
        }
        if (p.p1_int) {
          int v[32];
#pragma unroll
          for (int c = 0; c < 32; c += 4) {
            const int4 v4 = __ldg(reinterpret_cast<const int4*>(p.p1q + mbase + c));
            v[c] = ((x >> c) & 1u) ? v4.x : 0; v[c + 1] = ((x >> (c + 1)) & 1u) ? v4.y : 0;
            v[c + 2] = ((x >> (c + 2)) & 1u) ? v4.z : 0; v[c + 3] = ((x >> (c + 3)) & 1u) ? v4.w : 0;
          }
#pragma unroll
          for (int w = 16; w >= 1; w >>= 1)
#pragma unroll
            for (int c = 0; c < w; ++c) v[c] += v[c + w];   // |p1q| < 2^24, 32 of them: no overflow
          tot += v[0];
        } else {
#pragma unroll
          for (int c = 0; c < 32; ++c)
            if ((x >> c) & 1u) d1 += (double)__ldg(p.p1 + mbase + c);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (!leader) mbar_arrive_remote(mapa_shared(ACC_EMPTY0 + 8u * buf, 0));
        else mbar_arrive(ACC_EMPTY0 + 8u * buf);
      }
      if (live) p.Q[(size_t)ct * p.B + b] = (double)tot * p.qscale + d1;
    }
  }
#undef FULL
#undef EMPTY
#undef FULLA
#undef EMPTYA
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) tmem_dealloc_pair(tmem, 512);
}

}  // namespace hobo
