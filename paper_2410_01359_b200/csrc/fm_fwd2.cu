// fm_fwd2.cu — K2b: FlashMask forward (Alg. 1) on a CTA pair (sm_100a,
// d = 128).
//
// A 2-CTA cluster owns the pair of 128-row query tiles (Q_2p, Q_2p+1) of one (batch, head) — the
// same rows as one K2a CTA (fm_fwd.cu) — but spreads them over two SMs: CTA r holds query tile
// 2p + r and the tensor cores of both SMs run every MMA together (tcgen05 cta_group::2, M = 256).
// Each SM holds only half of every K_j / V_j tile (keys [64r, 64r+64) of K_j as the B operand of
// S = Q K^T, columns [64r, 64r+64) of V_j as the B operand of O += P V), so the per-SM shared-memory
// operand traffic and the L2 -> SM traffic per visited tile are half of K2a's.  That frees TMEM:
// each SM keeps ONE query tile, with THREE S accumulators [0,128) [128,256) [256,384) and O
// [384,512).  S_{e+1} and S_{e+2} are computed while the softmax works on S_e, so the tensor core
// no longer waits for the softmax chain S -> softmax -> PV of one tile (that chain
// bounds K2a at ~2/3 of the tensor peak).
//
// Warp roles per CTA (576 threads):
//   warps 0-15  softmax, two warpsets: warpset W = warp / 8 processes the visited tiles e with
//               e % 2 == W; in a warpset, warp = (column half hh, TMEM lane quadrant wl), thread =
//               one query row, 64 of the 128 key columns of the tile
//   warp  16    TMA producer: own Q tile, own halves of K_j / V_j, mask slice of PARTIAL tiles
//   warp  17    TMEM allocator; in the leader CTA (rank 0) the MMA issuer of both SMs
// Online softmax across warpsets (Alg. 1 lines 22-26): the running row max of tile e is decided by
// the warpset of tile e from its tile maximum and the running max after tile e-1, which the other
// warpset publishes through shared memory (mbarrier `mchain`); the max moves only when it grows by
// more than 2^8 (exact, as in K2a), O in TMEM is rescaled then, and each thread keeps its row-sum
// share relative to the max it last saw (combined at the end).
// Skipping: the visit list is the union of the two tiles' non-SKIP column tiles (K1
// class map); a tile SKIP for one CTA's query tile is computed by the pair but that CTA writes
// P = 0 for it (the tile is fully masked: Eq. 4 soundness), so results are exact.
#include <cuda_bf16.h>
#include <cmath>

#include "fm_internal.h"
#include "fm_ptx.cuh"

#ifdef FM_TRACE
#ifndef FM_TRACE_BX
#define FM_TRACE_BX 64
#endif
namespace fm { __device__ long long g_fm_trace_fwd2[80 * 16]; __device__ long long g_fm_trace_fwd2_ev[16]; }
#define FT2(slot, e)                                                                                               \
  do {                                                                                                             \
    if (blockIdx.x == FM_TRACE_BX && blockIdx.y == 0 && blockIdx.z == 0 && (e) < 64) fm::g_fm_trace_fwd2[(e) * 16 + (slot)] = clock64(); \
  } while (0)
__device__ __forceinline__ long long fm_gtimer() { long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
#define FT2P(slot, e)                                                                                              \
  do {                                                                                                             \
    if (blockIdx.x == FM_TRACE_BX + 1 && blockIdx.y == 0 && blockIdx.z == 0 && (e) < 64) fm::g_fm_trace_fwd2[(e) * 16 + (slot)] = fm_gtimer(); \
  } while (0)
#define FT2G(slot, e)                                                                                              \
  do {                                                                                                             \
    if (blockIdx.x == FM_TRACE_BX && blockIdx.y == 0 && blockIdx.z == 0 && (e) < 64) fm::g_fm_trace_fwd2[(e) * 16 + (slot)] = fm_gtimer(); \
  } while (0)
#define FTE2(k)                                                                                                    \
  do {                                                                                                             \
    if (blockIdx.x == FM_TRACE_BX && blockIdx.y == 0 && blockIdx.z == 0) fm::g_fm_trace_fwd2_ev[k] = clock64();      \
  } while (0)
#else
#define FT2(slot, e) \
  do {               \
  } while (0)
#define FTE2(k) \
  do {          \
  } while (0)
#define FT2P(slot, e) \
  do {                \
  } while (0)
#define FT2G(slot, e) \
  do {                \
  } while (0)
#endif

namespace fm {

namespace fwd2 {

constexpr int NT = 576;
constexpr int KST = 4, VST = 4, MST = 4;  // ring depths (MST even: a mask stage belongs to one warpset)
// of every 8 column pairs, how many use the FMA-pipe exp2 (rest: MUFU): 1 measured best here —
// the pair kernel's softmax is issue-bound and a polynomial pair costs ~14 instructions against
// ~5 for a MUFU pair
constexpr int kPolyPairs = 1;
template <bool CAUSAL>
constexpr bool kRefine = CAUSAL;  // f3 words in the causal kernels only, as in K2a
constexpr int MMA_WARP = 17, PRODUCER_WARP = 16;
constexpr int D = 128;
constexpr uint32_t O_COL = 384;

struct Smem {
  static constexpr int QT = 128 * D * 2;       // own Q tile (A operand of S), later the O staging tile
  static constexpr int KH = 64 * D * 2;        // half K tile: 64 keys x D (B operand of S)
  static constexpr int VH = 128 * (D / 2) * 2;  // half V tile: 128 keys x D/2 (B operand of PV)
  uint8_t q[QT];
  uint8_t k[KST][KH];
  uint8_t v[VST][VH];
  int4 mask[MST][128];
  uint32_t cw[MST];  // f3 refinement word of the stage's tile for this CTA's query tile
  uint32_t list[kMaxTc];
  uint64_t bar_q;  // leader: both CTAs' Q tiles landed
  uint64_t k_full[KST], k_empty[KST], v_full[VST], v_empty[VST];
  uint64_t m_full[MST], m_empty[MST];
  uint64_t s_full[4], p_full[4], pv_done[4], o_full;  // indexed by tile e % 4
  uint64_t mchain[4][2];                              // [lane quadrant][tile parity], 64 arrivals
  float xmax[2][2][2][128];                           // [warpset][local tile parity][half][row]
  float mval[2][128];                                 // running max after tile e, by e parity
  float xl[2][2][128], xm[2][2][128];                 // final row-sum combine [warpset][half][row]
  uint32_t tmem_base;
  int n_entries;
  int warp_cnt[NT / 32];
  float warp_kmax[NT / 32];  // BND: largest key norm of the head, per warp's share of the column tiles
};

__device__ __forceinline__ int ent_cls(uint32_t ent, int q) { return (ent >> (24 + 2 * q)) & 3; }

}  // namespace fwd2

// BND (R33): the bounded single pass of K2a on the CTA pair — every P of a row against the fixed
// reference ||q_r|| max||k|| scale log2(e) - 96: no max pass, no max chain between the warpsets, no O
// rescale; rows whose sum ends below 2^-90 flag the unit for K2a's two-pass fixup launch.
template <bool CAUSAL, bool OUT_F32, bool F16, bool BND>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(fwd2::NT, 1)
    fm_fwd2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK64,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, const FwdArgs a) {
  using namespace fwd2;
  using S = Smem;
  extern __shared__ uint8_t smem_raw[];
  S& sm = *smem_align1024<S>(smem_raw);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int rank = static_cast<int>(cluster_ctarank());
  const bool leader = rank == 0;
  const int npairs = (a.Tr + 1) >> 1;
  const int pair = npairs - 1 - static_cast<int>(blockIdx.x >> 1);  // heaviest (last) row tiles first
  const int h = blockIdx.y, b = blockIdx.z;
  const int hk = h / a.G;
  const int hm = (a.Hm == 1) ? 0 : hk;
  const int i0 = 2 * pair, i1 = 2 * pair + 1;
  const int my_i = i0 + rank;  // this CTA's query tile (may be == Tr for an odd tile count: no rows)
  const size_t bhm = static_cast<size_t>(b) * a.Hm + hm;

  if (tid == 0) FTE2(0);
  if (warp == PRODUCER_WARP && lane == 0) {
    mbar_init(&sm.bar_q, 1);
    for (int s = 0; s < KST; ++s) { mbar_init(&sm.k_full[s], 1); mbar_init(&sm.k_empty[s], 1); }
    for (int s = 0; s < VST; ++s) { mbar_init(&sm.v_full[s], 1); mbar_init(&sm.v_empty[s], 1); }
    for (int s = 0; s < MST; ++s) { mbar_init(&sm.m_full[s], 1); mbar_init(&sm.m_empty[s], 8); }
    for (int x = 0; x < 4; ++x) {
      mbar_init(&sm.s_full[x], 1);
      mbar_init(&sm.p_full[x], 16);  // 8 softmax warps of each CTA
      mbar_init(&sm.pv_done[x], 1);
      for (int p = 0; p < 2; ++p) mbar_init(&sm.mchain[x][p], 64);  // every thread of the two warps
    }
    mbar_init(&sm.o_full, 1);
    fence_barrier_init();
  }
  if (warp == MMA_WARP) tmem_alloc_pair<512>(&sm.tmem_base);
  // barriers of both CTAs initialised before any cross-CTA signal
  cluster_sync_all();
  if (warp == PRODUCER_WARP && lane == 0) {
    // Q does not depend on the visit list: start its load before the list is built
    tma_prefetch_desc(&tmQ);
    if (leader) mbar_expect_tx(&sm.bar_q, 2 * S::QT);
    const uint32_t lq = mapa_shared(&sm.bar_q, 0);
#pragma unroll
    for (int c = 0; c < D / 64; ++c) tma_load_4d_pair(sm.q + c * 16384, &tmQ, lq, c * 64, h, my_i * 128, b);
  }
  pdl_wait();  // the class map (K1b) and refinement words (K1c) are complete
  pdl_launch();

  // ---- visit list: union of the non-SKIP column tiles of the pair's two query tiles ----
  {
    const uint8_t* row0 = a.fmap + (bhm * a.Tr + i0) * a.Tc;
    const uint8_t* row1 = row0 + a.Tc;
    const bool has_q1 = i1 < a.Tr;
    int base = 0;
    float kv = 0.f;  // BND: largest key norm of the kv head over all its column tiles
    const float* kmax_bh = BND ? a.kmax + (static_cast<size_t>(b) * (a.H / a.G) + hk) * a.Tc : nullptr;
    for (int j0 = 0; j0 < a.Tc; j0 += NT) {
      const int j = j0 + tid;
      uint32_t c0 = 0, c1 = 0;
      if (j < a.Tc) {
        c0 = row0[j];
        c1 = has_q1 ? row1[j] : 0u;
      }
      const bool vis = (c0 | c1) != 0u;
      const unsigned bal = __ballot_sync(0xffffffffu, vis);
      if (lane == 0) sm.warp_cnt[warp] = __popc(bal);
      __syncthreads();
      int off = base, tot = 0;
      for (int w = 0; w < NT / 32; ++w) {
        const int c = sm.warp_cnt[w];
        if (w < warp) off += c;
        tot += c;
      }
      off += __popc(bal & ((1u << lane) - 1u));
      if (vis) sm.list[off] = static_cast<uint32_t>(j) | (c0 << 24) | (c1 << 26);
      if (BND && j < a.Tc) kv = fmaxf(kv, __ldg(kmax_bh + j));
      base += tot;
      __syncthreads();
    }
    if (tid == 0) sm.n_entries = base;
    if constexpr (BND) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) kv = fmaxf(kv, __shfl_xor_sync(0xffffffffu, kv, o));
      if (lane == 0) sm.warp_kmax[warp] = kv;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int nE = sm.n_entries;
  const uint32_t tbase = sm.tmem_base;
  if (tid == 0) FTE2(1);
#ifdef FM_TRACE
  if (tid == 0 && blockIdx.x == FM_TRACE_BX && blockIdx.y == 0 && blockIdx.z == 0) g_fm_trace_fwd2_ev[9] = nE;
#endif

  if (warp == PRODUCER_WARP) {
    // ================================ TMA producer ================================
    if (lane == 0) {
      tma_prefetch_desc(&tmK64);
      tma_prefetch_desc(&tmV);
      const int4* vec_bh = a.vec4 + bhm * static_cast<size_t>(a.Tc) * 128;
      for (int e = 0; e < nE; ++e) {
        const uint32_t ent = sm.list[e];
        const int j = static_cast<int>(ent & 0xFFFFFFu);
        const int ks = e % KST, vs = e % VST, ms = e % MST;
        mbar_wait(&sm.k_empty[ks], ((e / KST) & 1) ^ 1);
        if (leader) mbar_expect_tx(&sm.k_full[ks], 2 * S::KH);
        const uint32_t lk = mapa_shared(&sm.k_full[ks], 0);
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          tma_load_4d_pair(sm.k[ks] + c * (64 * 128), &tmK64, lk, c * 64, hk, j * 128 + rank * 64, b);
        FT2(11, e);
        mbar_wait(&sm.m_empty[ms], ((e / MST) & 1) ^ 1);
        if (ent_cls(ent, rank) == 1) {
          uint32_t wq = 0xFFFFFFFFu;
          if (kRefine<CAUSAL> && a.cw != nullptr && !(j == a.Tc - 1 && (a.N & 127) != 0))
            wq = a.cw[(bhm * a.Tr + my_i) * a.Tc + j];
          sm.cw[ms] = wq;
          mbar_expect_tx(&sm.m_full[ms], 128 * 16);
          bulk_g2s(sm.mask[ms], vec_bh + static_cast<size_t>(j) * 128, 128 * 16, &sm.m_full[ms]);
        } else {
          mbar_arrive(&sm.m_full[ms]);
        }
        mbar_wait(&sm.v_empty[vs], ((e / VST) & 1) ^ 1);
        if (leader) mbar_expect_tx(&sm.v_full[vs], 2 * S::VH);
        tma_load_4d_pair(sm.v[vs], &tmV, mapa_shared(&sm.v_full[vs], 0), rank * (D / 2), hk, j * 128, b);
        FT2(12, e);
      }
    }
  } else if (warp == MMA_WARP) {
    // ============================ MMA issuer (leader CTA) ============================
    // Order: S_0, S_1, S_2, then PV_e, S_{e+3} for e = 0, 1, ...: S_{e+3} reuses the accumulator of
    // S_e (= P_e), so it follows PV_e in issue order (tcgen05.mma executes in issue order).
    if (leader) {
      if (nE > 0) {
        constexpr uint32_t ID_S = idesc16<F16>(256, 128, 0, 0);  // S = Q K^T, both K-major
        constexpr uint32_t ID_PV = idesc16<F16>(256, D, 0, 1);   // O += P V, V MN-major
        const uint32_t q_addr = smem_u32(sm.q);
        mbar_wait(&sm.bar_q, 0);
        tc_fence_after();
        if (lane == 0) FTE2(2);
        auto issue_s = [&](int e) {
          const int ks = e % KST;
          mbar_wait(&sm.k_full[ks], (e / KST) & 1);
          if (lane == 0) FT2(0, e);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sm.k[ks]);
          const uint32_t tS = tbase + (e % 3) * 128;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t qo = (kk >> 2) * 16384 + (kk & 3) * 32;
            const uint32_t ko = (kk >> 2) * (64 * 128) + (kk & 3) * 32;
            mma2_ss_w(tS, sdesc_sw128(q_addr + qo, 16, 1024), sdesc_sw128(k_addr + ko, 16, 1024), ID_S,
                      kk > 0 ? 1u : 0u);
          }
          mma2_commit_mc_w(&sm.s_full[e & 3]);
          mma2_commit_mc_w(&sm.k_empty[ks]);
          if (lane == 0) FT2(1, e);
        };
        auto issue_pv = [&](int e) {
          mbar_wait(&sm.p_full[e & 3], (e >> 2) & 1);
          if (lane == 0) FT2(2, e);
          if (lane == 0) FT2G(13, e);
          const int vs = e % VST;
          mbar_wait(&sm.v_full[vs], (e / VST) & 1);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(sm.v[vs]);
          const uint32_t tS = tbase + (e % 3) * 128;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            // P of keys [0,64) sits in S columns [0,32), of keys [64,128) in S columns [64,96)
            const uint32_t a_tm = tS + kk * 8 + (kk >= 4 ? 32u : 0u);
            mma2_ts_w(tbase + O_COL, a_tm, sdesc_sw128(v_addr + kk * 2048, 16384, 1024), ID_PV,
                      (e > 0 || kk > 0) ? 1u : 0u);
          }
          mma2_commit_mc_w(&sm.v_empty[vs]);
          mma2_commit_mc_w(&sm.pv_done[e & 3]);
          if (lane == 0) FT2(3, e);
        };
        for (int e = 0; e < 3 && e < nE; ++e) issue_s(e);
        for (int e = 0; e < nE; ++e) {
          issue_pv(e);
          if (e + 3 < nE) issue_s(e + 3);
        }
        mma2_commit_mc_w(&sm.o_full);
      } else {
        // no MMA: both Q tiles must have landed before either CTA reuses or releases its buffer
        mbar_wait(&sm.bar_q, 0);
        if (lane == 0) {
          mbar_arrive_cluster(mapa_shared(&sm.o_full, 0));
          mbar_arrive_cluster(mapa_shared(&sm.o_full, 1));
        }
      }
    }
  } else {
    // ================================ softmax warpsets ================================
    const int W = warp >> 3;
    const int hh = (warp >> 2) & 1;
    const int wl = warp & 3;
    const int row_t = wl * 32 + lane;
    const int row = my_i * 128 + row_t;
    const uint32_t lane_off = static_cast<uint32_t>(wl * 32) << 16;
    const float sl2 = a.scale_log2;
    const uint32_t bar_x = 1 + W * 4 + wl;  // this (warpset, quadrant)'s two column halves
    const uint32_t tO = tbase + lane_off + O_COL;
    const uint32_t p_full_lead = mapa_shared(&sm.p_full[0], 0);
    float m_ref = -INFINITY;  // the running max this thread's row-sum share is relative to
    float l = 0.f;
    if constexpr (BND) {
      // R33 fixed reference: ||q_r|| (this row of Q, read from global memory: L2-resident, once per
      // CTA) * the head's largest key norm * scale * log2(e) - 96
      float kvis = 0.f;
#pragma unroll
      for (int w = 0; w < NT / 32; ++w) kvis = fmaxf(kvis, sm.warp_kmax[w]);
      float ss = 0.f;
      if (row < a.N) {
        const uint4* qr = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(a.q) +
                                                         ((static_cast<size_t>(b) * a.N + row) * a.H + h) * D);
#pragma unroll 4
        for (int g = 0; g < D / 8; ++g) {
          const uint4 u4 = __ldg(qr + g);
          const uint32_t w4[4] = {u4.x, u4.y, u4.z, u4.w};
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            const float lo = __uint_as_float(w4[t] << 16), hi = __uint_as_float(w4[t] & 0xFFFF0000u);
            ss = fmaf(lo, lo, fmaf(hi, hi, ss));
          }
        }
      }
      m_ref = sqrtf(ss) * (1.0f + 1.0f / 65536.0f) * kvis * sl2 - kBndHeadroom;
    }
    for (int e = W, u = 0; e < nE; e += 2, ++u) {
      const uint32_t ent = sm.list[e];
      const int cls = ent_cls(ent, rank);
      const int ms = e % MST;
      const uint32_t tSh = tbase + lane_off + (e % 3) * 128 + hh * 64;  // this half's 64 S columns
      const bool tr0 = (hh == 0 && row_t == 0), tr1 = (hh == 1 && row_t == 96);
      mbar_wait(&sm.m_full[ms], (e / MST) & 1);
      mbar_wait(&sm.s_full[e & 3], (e >> 2) & 1);
      if (tr0) FT2(4, e);
      if (tr0) FT2P(14, e);
      if (tr0) FT2G(9, e);
      tc_fence_after();
      uint32_t sr[2][16];
      float m_cur = m_ref;
      if constexpr (!BND) {
      // Pass 1: max over this half's 64 columns (Alg. 1 line 22), element mask of lines 15-21 on
      // PARTIAL tiles written back to TMEM, 16 columns at a time
      float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
      if (cls != 0) {
        const int j = static_cast<int>(ent & 0xFFFFFFu);
        const uint32_t pm = (cls != 1) ? 0u : (kRefine<CAUSAL> ? (sm.cw[ms] >> (wl * 8 + hh * 4)) & 0xFu : 0xFu);
        tmem_ld16(tSh, sr[0]);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          tmem_wait_ld();
          if (c + 1 < 4) tmem_ld16(tSh + (c + 1) * 16, sr[(c + 1) & 1]);
          float* sv = reinterpret_cast<float*>(sr[c & 1]);
          if (pm & (1u << c)) {
            const int4* mk = sm.mask[ms] + hh * 64 + c * 16;
            const int rmy = row - (j * 128 + hh * 64 + c * 16);
            if (CAUSAL && j < my_i) {
#pragma unroll
              for (int t = 0; t < 16; ++t) {
                const int4 mv = mk[t];
                const bool msk = static_cast<unsigned>(row - mv.x) < static_cast<unsigned>(mv.y);
                sv[t] = msk ? -INFINITY : sv[t];
              }
            } else {
#pragma unroll
              for (int t = 0; t < 16; ++t) {
                const int4 mv = mk[t];
                bool msk = static_cast<unsigned>(row - mv.x) < static_cast<unsigned>(mv.y);
                if constexpr (CAUSAL)
                  msk |= rmy < t;
                else
                  msk |= static_cast<unsigned>(row - mv.z) < static_cast<unsigned>(mv.w);
                sv[t] = msk ? -INFINITY : sv[t];
              }
            }
            tmem_st16(tSh + c * 16, sr[c & 1]);
          }
#pragma unroll
          for (int t = 0; t < 16; t += 8) {
            mx0 = fmax3(mx0, sv[t], sv[t + 1]);
            mx1 = fmax3(mx1, sv[t + 2], sv[t + 3]);
            mx2 = fmax3(mx2, sv[t + 4], sv[t + 5]);
            mx3 = fmax3(mx3, sv[t + 6], sv[t + 7]);
          }
        }
        if (pm) tmem_wait_st();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.m_empty[ms]);
      const float mh = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
      if (tr0) FT2(5, e);
      sm.xmax[W][u & 1][hh][row_t] = mh;
      named_bar_sync(bar_x, 64);
      const float m_tile = fmaxf(mh, sm.xmax[W][u & 1][hh ^ 1][row_t]) * sl2;
      // running max after tile e-1 from the other warpset (Alg. 1 line 23)
      if (tr0) FT2(6, e);
      float m_prev = -INFINITY;
      if (e > 0) {
        mbar_wait(&sm.mchain[wl][(e - 1) & 1], ((e - 1) >> 1) & 1);
        m_prev = sm.mval[(e - 1) & 1][row_t];
      }
      if (tr0) FT2(7, e);
      const bool need = m_tile > m_prev + 8.0f;
      m_cur = need ? m_tile : m_prev;
      if (e + 1 < nE) {
        // each thread publishes (hh = 0) / releases (hh = 1) its own row: its arrive orders its own
        // accesses (also for compute-sanitizer racecheck, which does not follow warp-sync chains)
        if (hh == 0) sm.mval[e & 1][row_t] = m_cur;
        mbar_arrive(&sm.mchain[wl][e & 1]);
      }
      // O holds sum_{e' < e} P_e' V_e' relative to m_prev: rescale it between PV_{e-1} and PV_e
      // (PV_e cannot start before this warpset's P_e is released below)
      const bool resc = need && m_prev != -INFINITY;
      if (__any_sync(0xffffffffu, resc)) {
        mbar_wait(&sm.pv_done[(e - 1) & 3], ((e - 1) >> 2) & 1);
        tc_fence_after();
        const float alpha = resc ? ex2(m_prev - m_cur) : 1.0f;
#pragma unroll 1
        for (int c = 0; c < D / 64; ++c) {
          uint32_t ov[32];
          const uint32_t ta = tO + hh * (D / 2) + c * 32;
          tmem_ld32(ta, ov);
          tmem_wait_ld();
#pragma unroll
          for (int t = 0; t < 32; ++t) ov[t] = __float_as_uint(__uint_as_float(ov[t]) * alpha);
          tmem_st32(ta, ov);
        }
      }
      if (m_ref != m_cur) {
        l = (l == 0.f) ? 0.f : l * ex2(m_ref - m_cur);
        m_ref = m_cur;
      }
      }  // two-pass (!BND)
      // Pass 2: P = exp2(S*scale*log2e - m) (Alg. 1 line 24), packed into the first 32 of this
      // half's S columns; row-sum share (line 25)
      if (cls != 0) {
        const int j = static_cast<int>(ent & 0xFFFFFFu);
        const uint32_t pm =
            (!BND || cls != 1) ? 0u : (kRefine<CAUSAL> ? (sm.cw[ms] >> (wl * 8 + hh * 4)) & 0xFu : 0xFu);
        const float m_use = (m_cur == -INFINITY) ? 0.f : m_cur;
        const uint64_t sl2x2 = f2pack(sl2, sl2), negm2 = f2pack(-m_use, -m_use);
        uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
        tmem_ld16(tSh, sr[0]);
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          tmem_wait_ld();
          if (ch + 1 < 4) tmem_ld16(tSh + (ch + 1) * 16, sr[(ch + 1) & 1]);
          float* sv = reinterpret_cast<float*>(sr[ch & 1]);
          if (BND && (pm & (1u << ch))) {
            // element mask of Alg. 1 lines 15-21 in registers (no max pass to carry it to TMEM)
            const int4* mk = sm.mask[ms] + hh * 64 + ch * 16;
            const int rmy = row - (j * 128 + hh * 64 + ch * 16);
            if (CAUSAL && j < my_i) {
#pragma unroll
              for (int t = 0; t < 16; ++t) {
                const int4 mv = mk[t];
                sv[t] = static_cast<unsigned>(row - mv.x) < static_cast<unsigned>(mv.y) ? -INFINITY : sv[t];
              }
            } else {
#pragma unroll
              for (int t = 0; t < 16; ++t) {
                const int4 mv = mk[t];
                bool msk = static_cast<unsigned>(row - mv.x) < static_cast<unsigned>(mv.y);
                if constexpr (CAUSAL)
                  msk |= rmy < t;
                else
                  msk |= static_cast<unsigned>(row - mv.z) < static_cast<unsigned>(mv.w);
                sv[t] = msk ? -INFINITY : sv[t];
              }
            }
          }
          uint32_t pk[8];
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const int k = ch * 8 + kk;
            const uint64_t x2 = f2fma(f2pack(sv[2 * kk], sv[2 * kk + 1]), sl2x2, negm2);
            float p0, p1;
            if ((k & 7) >= 8 - (BND ? 2 : kPolyPairs)) {
              exp2_poly2(x2, p0, p1);
            } else {
              float x0, x1;
              f2unpack(x2, x0, x1);
              p0 = ex2(x0);
              p1 = ex2(x1);
            }
            acc[k & 3] = f2add(acc[k & 3], f2pack(p0, p1));
            pk[kk] = pack16<F16>(p0, p1);
          }
          tmem_st8(tSh + ch * 8, pk);
        }
        const uint64_t a01 = f2add(acc[0], acc[1]), a23 = f2add(acc[2], acc[3]);
        float u0, u1;
        f2unpack(f2add(a01, a23), u0, u1);
        l += u0 + u1;
      } else {
        // tile SKIP for this CTA's query tile but computed by the pair: contributes P = 0
        uint32_t z[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) z[t] = 0u;
        tmem_st16(tSh, z);
        tmem_st16(tSh + 16, z);
      }
      tmem_wait_st();
      if constexpr (BND) {  // the mask slice of stage ms was read by this pass
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.m_empty[ms]);
      }
      if (tr0) FT2(8, e);
      if (tr0) FT2P(15, e);
      if (tr0) FT2G(10, e);
#ifdef FM_TRACE
      if (lane == 0 && (e == 20 || e == 21) && blockIdx.y == 0 && blockIdx.z == 0 &&
          (blockIdx.x == FM_TRACE_BX || blockIdx.x == FM_TRACE_BX + 1))
        fm::g_fm_trace_fwd2[(64 + (e - 20)) * 16 + (blockIdx.x - FM_TRACE_BX) * 8 + (warp & 7)] = fm_gtimer();
#endif
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(p_full_lead + static_cast<uint32_t>((e & 3) * sizeof(uint64_t)));
    }
    // ---- epilogue: O = O / l, L = m + ln(l) (Alg. 1 lines 27-28) ----
    if (tid == 0) FTE2(3);
    sm.xl[W][hh][row_t] = l;
    sm.xm[W][hh][row_t] = m_ref;
    named_bar_sync(9, 512);
    float m_fin = -INFINITY;
    float lt = 0.f;
    if constexpr (BND) {  // one reference for the whole row
      m_fin = m_ref;
#pragma unroll
      for (int x = 0; x < 4; ++x) lt += sm.xl[x >> 1][x & 1][row_t];
    } else {
#pragma unroll
      for (int x = 0; x < 4; ++x) m_fin = fmaxf(m_fin, sm.xm[x >> 1][x & 1][row_t]);
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const float lx = sm.xl[x >> 1][x & 1][row_t];
        if (lx > 0.f) lt += lx * ex2(sm.xm[x >> 1][x & 1][row_t] - m_fin);
      }
    }
    // BND: a row whose sum ends below 2^-90 flags the unit for the two-pass fixup launch
    const bool live = BND ? (nE > 0 && lt >= kBndMinSum) : lt > 0.f;
    if (BND && row < a.N && !live) a.fix_out[(static_cast<size_t>(b) * a.H + h) * npairs + pair] = 1;
    const float inv = live ? 1.0f / lt : 0.f;
    mbar_wait(&sm.o_full, 0);  // every MMA of the pair done (or, with no MMA, both Q tiles landed)
    tc_fence_after();
    const int col0 = (W * 2 + hh) * 32;  // this warp's 32 of the D output columns
    uint32_t ov[32];
    if (nE > 0) {
      tmem_ld32(tO + col0, ov);
      tmem_wait_ld();
    }
    float f[32];
#pragma unroll
    for (int t = 0; t < 32; ++t) f[t] = live ? __uint_as_float(ov[t]) * inv : 0.f;
    if constexpr (!OUT_F32) {
      // staged in the own (now free) Q buffer, 128-B swizzled, stored by TMA (rows >= N clipped)
      uint8_t* blk = sm.q + (col0 / 64) * 16384 + row_t * 128;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int chunk = (col0 % 64) / 8 + t;
        *reinterpret_cast<uint4*>(blk + ((chunk ^ (row_t & 7)) << 4)) =
            make_uint4(pack16<F16>(f[8 * t], f[8 * t + 1]), pack16<F16>(f[8 * t + 2], f[8 * t + 3]),
                       pack16<F16>(f[8 * t + 4], f[8 * t + 5]), pack16<F16>(f[8 * t + 6], f[8 * t + 7]));
      }
      fence_proxy_async_smem();
      named_bar_sync(10, 512);
      if (warp == 0 && lane == 0 && my_i * 128 < a.N) {
#pragma unroll
        for (int c = 0; c < D / 64; ++c) tma_store_4d(&tmO, sm.q + c * 16384, c * 64, h, my_i * 128, b);
        bulk_commit();
        bulk_wait_read0();
      }
    } else if (row < a.N) {
      float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.o) +
                                              ((static_cast<size_t>(b) * a.N + row) * a.H + h) * D + col0);
#pragma unroll
      for (int t = 0; t < 8; ++t) dst[t] = make_float4(f[4 * t], f[4 * t + 1], f[4 * t + 2], f[4 * t + 3]);
    }
    if (row < a.N && W == 0 && hh == 0)
      a.lse[(static_cast<size_t>(b) * a.H + h) * a.N + row] =
          live ? (m_fin + __log2f(lt)) * 0.6931471805599453f : -INFINITY;
  }

  if (tid == 0) FTE2(4);
  // neither CTA leaves while the pair's MMAs or the peer's signals may still touch its memory
  tc_fence_before();
  cluster_sync_all();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc_pair<512>(tbase);
  }
  if (tid == 0) FTE2(5);
}

template <bool CAUSAL, bool OUT_F32, bool F16, bool BND>
static cudaError_t launch_fwd2_t(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk64, const CUtensorMap& tv,
                                 const CUtensorMap& to, const FwdArgs& a, cudaStream_t st) {
  auto kern = fm_fwd2_kernel<CAUSAL, OUT_F32, F16, BND>;
  const size_t smem = sizeof(fwd2::Smem) + 1024;
  static_assert(sizeof(fwd2::Smem) + 1024 <= 232448, "shared memory budget");
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(2 * ((d.Tr + 1) / 2), d.H, d.B);
  return launch_pdl(kern, grid, dim3(fwd2::NT), smem, st, tq, tk64, tv, to, a);
}

cudaError_t launch_fwd2(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk64, const CUtensorMap& tv,
                        const CUtensorMap& to, const FwdArgs& a, cudaStream_t st) {
  if (d.D != 128) return cudaErrorInvalidValue;
#define FM_F2(CC, FF)                                                                                    \
  do {                                                                                                   \
    if (a.kmax != nullptr && !d.in_f16) return launch_fwd2_t<CC, FF, false, true>(d, tq, tk64, tv, to, a, st); \
    return d.in_f16 ? launch_fwd2_t<CC, FF, true, false>(d, tq, tk64, tv, to, a, st)                       \
                    : launch_fwd2_t<CC, FF, false, false>(d, tq, tk64, tv, to, a, st);                     \
  } while (0)
  if (d.causal) {
    if (d.out_f32) FM_F2(true, true); else FM_F2(true, false);
  } else {
    if (d.out_f32) FM_F2(false, true); else FM_F2(false, false);
  }
#undef FM_F2
}

}  // namespace fm

#ifdef FM_TRACE
extern "C" __attribute__((visibility("default"))) int flashmask_debug_trace_fwd2(long long* host, long long* ev) {
  if (cudaMemcpyFromSymbol(host, fm::g_fm_trace_fwd2, sizeof(long long) * 80 * 16) != cudaSuccess) return 1;
  return cudaMemcpyFromSymbol(ev, fm::g_fm_trace_fwd2_ev, sizeof(long long) * 16) == cudaSuccess ? 0 : 1;
}
#endif
