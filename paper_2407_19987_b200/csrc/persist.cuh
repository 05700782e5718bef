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

struct PersistCfg {
  static constexpr int NT = 128;                     // column tile (UMMA N)
  static constexpr int KPS = 2;                      // K-blocks per stage
  static constexpr int HBOX = (NT / 2) * 128;        // this CTA's half of one W box (64 rows x 64 bf16)
  static constexpr int MAXL = 3;                     // limb planes
  static constexpr int NST = 4;                      // ring stages (TMEM: 4 x 64 A columns)
  static constexpr int STAGE = KPS * MAXL * HBOX;    // 48 KB
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
                            // decoding, 4 no bit restaging, 8 no MMAs
};

__global__ void __launch_bounds__(kPThreads, 1) kr_persist_kernel(const __grid_constant__ CUtensorMap tmap,
                                                                   const PersistParams p) {
  using C = PersistCfg;
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
  const int it0 = __ldg(p.items + pair), it1 = __ldg(p.items + pair + 1);
  auto item_ct = [&](int it) { return p.n_ct - 1 - it % p.n_ct; };   // heaviest tile of a block first
  auto item_cb = [&](int it) { return 2 * (it / p.n_ct) + (int)prank; };
  const uint32_t stage_bytes = (uint32_t)(C::KPS * p.L) * C::HBOX;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::NST; ++s) { mbar_init(FULL(s), 17); mbar_init(EMPTY(s), 1); }   // TMA + 8 + 8 peer gen warps
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
              } else if (nkb == 2 && p.L == 3) {   // the common stage, fully unrolled
#pragma unroll
                for (int q = 0; q < 2; ++q)
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
    int gst = 0;
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
        for (int kb0 = s.x; kb0 < kend; kb0 += C::KPS) {
          const int kb = kb0 + h;
          const bool mine = kb < kend;
          uint64_t bits = 0ull;
          if (mine && !(p.exp & 2)) bits = block_bits(xs, row, __ldg(p.kdesc + 2 * kb), __ldg(p.kdesc + 2 * kb + 1), p.runs);
          mbar_wait(EMPTY(gst), gph ^ 1u);
          if (mine) {
            tc_fence_after();
            uint32_t w[32];
            expand32((uint32_t)bits, *reinterpret_cast<uint32_t(*)[16]>(&w[0]));
            expand32((uint32_t)(bits >> 32), *reinterpret_cast<uint32_t(*)[16]>(&w[16]));
            tmem_st32(lane_base + (uint32_t)(C::A0 + (gst * C::KPS + h) * C::ACOLS), w);
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

}  // namespace hobo
