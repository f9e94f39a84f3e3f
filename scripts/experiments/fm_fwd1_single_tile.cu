// fm_fwd1.cu — K2: FlashMask forward (Alg. 1) for sm_100a, one 128-row
// query tile per CTA with a double-buffered S accumulator.
//
// Warp roles (576 threads):
//   warps 0-15  softmax: warp w owns TMEM lane quadrant w % 4 (32 query rows, thread = row) and
//               key-column quarter w / 4 (32 of the 128 key columns of a tile)
//   warp  16    TMA producer: Q once, then K_j, V_j and (PARTIAL tiles only) the mask slice
//   warp  17    TMEM allocator + tcgen05 MMA issuer (converged warp, elect.sync)
// TMEM columns: S(0) [0,128)  S(1) [128,256)  O [256, 256+D)  Q [256+D, 256+3D/2).
//
// Why this shape: S_{e+1} = Q K_{e+1}^T is computed into the other S buffer
// while the softmax warps work on S_e, so the tensor core is not idle during the softmax; all 16
// softmax warps serve the one tile (32 columns each), halving its latency; and Q sits in TMEM as
// the A operand of S (TS MMA), so per visited tile the only shared-memory operand traffic is K
// (S), V (PV) and their TMA writes — 128 KiB per 1024 MMA clocks, inside the 128 B/clk budget.
// Issue order: S0, S1, PV0, S2, PV1, S3, ... (S_e reuses the buffer of S_{e-2} after PV_{e-2}
// has been issued by the same thread: tcgen05.mma executes in issue order).
// Fully masked tiles are never loaded (Alg. 1 lines 9-14): the visit list is built
// from the K1 class map.  PARTIAL tiles get the element-wise interval mask (lines 15-21).
#include <cuda_bf16.h>
#include <cmath>

#include "fm_internal.h"
#include "fm_ptx.cuh"

#ifndef FM_POLY_PAIRS1
#define FM_POLY_PAIRS1 3  // of every 8 column pairs, how many use the FMA-pipe exp2 (rest: MUFU)
#endif

namespace fm {

namespace fwd1 {

constexpr int NT = 576;
#ifndef FM_FWD1_KST
#define FM_FWD1_KST 3
#endif
#ifndef FM_FWD1_VST
#define FM_FWD1_VST 2
#endif
// K ring 3 deep: S_{e+2} is issued right after PV_e, so K_{e+2} must already be in flight while
// S_e is computed — with one query tile per CTA a K tile is consumed every ~1 K MMA clocks.
constexpr int KST = FM_FWD1_KST, VST = FM_FWD1_VST, MST = 4;
constexpr int PRODUCER_WARP = 16, MMA_WARP = 17;

template <int D>
struct Smem {
  static constexpr int TILE = 128 * D * 2;
  uint8_t q[TILE];  // Q (copied to TMEM at start), later the O staging tile of the TMA store
  uint8_t k[KST][TILE];
  uint8_t v[VST][TILE];
  int4 mask[MST][128];
  uint32_t list[kMaxTc];
  uint64_t bar_q, q_tmem;
  uint64_t k_full[KST], k_empty[KST], v_full[VST], v_empty[VST];
  uint64_t m_full[MST], m_empty[MST];
  uint64_t s_full[2], p_full[2], pv_done, o_full;
  float xmax[2][4][128];  // [parity][column quarter][row]
  float xsum[4][128];
  uint32_t tmem_base;
  int n_entries;
  int warp_cnt[NT / 32];
};

}  // namespace fwd1

template <int D, bool CAUSAL, bool OUT_F32>
__global__ void __launch_bounds__(fwd1::NT, 1)
    fm_fwd1_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                   const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
                   const FwdArgs a) {
  using namespace fwd1;
  using S = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  S& sm = *smem_align1024<S>(smem_raw);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i = a.Tr - 1 - static_cast<int>(blockIdx.x);  // heaviest (last) row tiles first
  const int h = blockIdx.y, b = blockIdx.z;
  const int hk = h / a.G;
  const int hm = (a.Hm == 1) ? 0 : hk;
  const size_t bhm = static_cast<size_t>(b) * a.Hm + hm;
  constexpr uint32_t S_COL0 = 0, O_COL = 256, Q_COL = 256 + D;

  if (warp == PRODUCER_WARP && lane == 0) {
    mbar_init(&sm.bar_q, 1);
    mbar_init(&sm.q_tmem, 16);
    for (int s = 0; s < KST; ++s) { mbar_init(&sm.k_full[s], 1); mbar_init(&sm.k_empty[s], 1); }
    for (int s = 0; s < VST; ++s) { mbar_init(&sm.v_full[s], 1); mbar_init(&sm.v_empty[s], 1); }
    for (int s = 0; s < MST; ++s) { mbar_init(&sm.m_full[s], 1); mbar_init(&sm.m_empty[s], 16); }
    for (int t = 0; t < 2; ++t) {
      mbar_init(&sm.s_full[t], 1);
      mbar_init(&sm.p_full[t], 512);
    }
    mbar_init(&sm.pv_done, 1);
    mbar_init(&sm.o_full, 1);
    fence_barrier_init();
    // Q does not depend on the visit list: start its load before the list is built
    tma_prefetch_desc(&tmQ);
    mbar_expect_tx(&sm.bar_q, S::TILE);
#pragma unroll
    for (int c = 0; c < D / 64; ++c) tma_load_4d(sm.q + c * 16384, &tmQ, &sm.bar_q, c * 64, h, i * 128, b);
  }
  if (warp == MMA_WARP) tmem_alloc<512>(&sm.tmem_base);

  // ---- visit list: the non-SKIP column tiles of row tile i (K1 class map), ascending j ----
  {
    const uint8_t* row = a.fmap + (bhm * a.Tr + i) * a.Tc;
    int base = 0;
    for (int j0 = 0; j0 < a.Tc; j0 += NT) {
      const int j = j0 + tid;
      const uint32_t c = (j < a.Tc) ? row[j] : 0u;
      const bool vis = c != 0u;
      const unsigned bal = __ballot_sync(0xffffffffu, vis);
      if (lane == 0) sm.warp_cnt[warp] = __popc(bal);
      __syncthreads();
      int off = base, tot = 0;
      for (int w = 0; w < NT / 32; ++w) {
        const int cw = sm.warp_cnt[w];
        if (w < warp) off += cw;
        tot += cw;
      }
      off += __popc(bal & ((1u << lane) - 1u));
      if (vis) sm.list[off] = static_cast<uint32_t>(j) | (c << 24);
      base += tot;
      __syncthreads();
    }
    if (tid == 0) sm.n_entries = base;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const int nE = sm.n_entries;
  const uint32_t tbase = sm.tmem_base;

  if (warp == PRODUCER_WARP) {
    // ================================ TMA producer ================================
    if (lane == 0) {
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      constexpr uint32_t TB = S::TILE;
      const int4* vec_bh = a.vec4 + bhm * static_cast<size_t>(a.Tc) * 128;
      for (int e = 0; e < nE; ++e) {
        const uint32_t ent = sm.list[e];
        const int j = static_cast<int>(ent & 0xFFFFFFu);
        const int ks = e % KST, vs = e % VST, ms = e % MST;
        mbar_wait(&sm.k_empty[ks], ((e / KST) & 1) ^ 1);
        mbar_expect_tx(&sm.k_full[ks], TB);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) tma_load_4d(sm.k[ks] + c * 16384, &tmK, &sm.k_full[ks], c * 64, hk, j * 128, b);
        mbar_wait(&sm.m_empty[ms], ((e / MST) & 1) ^ 1);
        if ((ent >> 24) == 1u) {
          mbar_expect_tx(&sm.m_full[ms], 128 * 16);
          bulk_g2s(sm.mask[ms], vec_bh + static_cast<size_t>(j) * 128, 128 * 16, &sm.m_full[ms]);
        } else {
          mbar_arrive(&sm.m_full[ms]);
        }
        mbar_wait(&sm.v_empty[vs], ((e / VST) & 1) ^ 1);
        mbar_expect_tx(&sm.v_full[vs], TB);
#pragma unroll
        for (int c = 0; c < D / 64; ++c) tma_load_4d(sm.v[vs] + c * 16384, &tmV, &sm.v_full[vs], c * 64, hk, j * 128, b);
      }
      if (nE == 0) mbar_wait(&sm.bar_q, 0);  // no MMA waits for Q: it must land before exit
    }
  } else if (warp == MMA_WARP) {
    // ================================ MMA issuer ================================
    if (nE > 0) {
      constexpr uint32_t ID_S = idesc_bf16(128, 128, 0, 0);  // S = Q K^T: A (TMEM) K-major, B K-major
      constexpr uint32_t ID_PV = idesc_bf16(128, D, 0, 1);   // O += P V: V is MN-major
      mbar_wait(&sm.q_tmem, 0);  // the softmax warps copied Q into TMEM
      tc_fence_after();
      for (int e = 0; e <= nE; ++e) {
        if (e < nE) {  // S_e into buffer e % 2 (its previous user PV_{e-2} was issued before)
          const int ks = e % KST;
          mbar_wait(&sm.k_full[ks], (e / KST) & 1);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sm.k[ks]);
          const uint32_t tS = tbase + S_COL0 + (e & 1) * 128;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            mma_ts_w(tS, tbase + Q_COL + kk * 8, sdesc_sw128(k_addr + off, 16, 1024), ID_S, kk > 0 ? 1u : 0u);
          }
          mma_commit_w(&sm.s_full[e & 1]);
          mma_commit_w(&sm.k_empty[ks]);
        }
        if (e >= 1) {  // O += P_{e-1} V_{e-1}
          const int pe = e - 1;
          mbar_wait(&sm.p_full[pe & 1], (pe >> 1) & 1);
          const int vs = pe % VST;
          mbar_wait(&sm.v_full[vs], (pe / VST) & 1);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(sm.v[vs]);
          const uint32_t tP = tbase + S_COL0 + (pe & 1) * 128;
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            // P of keys [32c, 32c+32) sits packed in S columns [32c, 32c+16) of its buffer
            mma_ts_w(tbase + O_COL, tP + (kk >> 1) * 32 + (kk & 1) * 8, sdesc_sw128(v_addr + kk * 2048, 16384, 1024),
                     ID_PV, (pe > 0 || kk > 0) ? 1u : 0u);
          }
          mma_commit_w(&sm.v_empty[vs]);
          mma_commit_w(&sm.pv_done);
        }
      }
    }
    mma_commit_w(&sm.o_full);
  } else {
    // ================================ softmax warps ================================
    const int wl = warp & 3, cq = warp >> 2;
    const int row_t = wl * 32 + lane;
    const int row = i * 128 + row_t;
    const uint32_t lane_off = static_cast<uint32_t>(wl * 32) << 16;
    const float sl2 = a.scale_log2;
    const uint32_t bar_id = 1 + wl;  // the four warps (column quarters) holding the same 32 rows
    // ---- Q -> TMEM (A operand of S): this warp copies D/4 of the row's columns ----
    if (nE > 0) {
      mbar_wait(&sm.bar_q, 0);
      constexpr int CPW = D / 32;  // 16-byte chunks per warp (of 2*D/16 per row)
      uint32_t qr[4 * CPW];
#pragma unroll
      for (int c = 0; c < CPW; ++c) {
        const int gc = cq * CPW + c;             // chunk index along the row (8 bf16 each)
        const int bx = gc >> 3, cc = gc & 7;     // 64-column block, chunk within the block
        const uint4 v4 = *reinterpret_cast<const uint4*>(sm.q + bx * 16384 + row_t * 128 + ((cc ^ (row_t & 7)) << 4));
        qr[4 * c] = v4.x;
        qr[4 * c + 1] = v4.y;
        qr[4 * c + 2] = v4.z;
        qr[4 * c + 3] = v4.w;
      }
      if constexpr (CPW == 4)
        tmem_st16(tbase + lane_off + Q_COL + cq * 16, qr);
      else
        tmem_st8(tbase + lane_off + Q_COL + cq * 8, qr);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.q_tmem);
    }
    float m_used = -INFINITY;  // running max of the scaled logits, log2 units (threshold-updated)
    float l = 0.f;             // this quarter's share of the row sum
    for (int e = 0; e < nE; ++e) {
      const uint32_t ent = sm.list[e];
      const int cls = static_cast<int>(ent >> 24);
      const int j = static_cast<int>(ent & 0xFFFFFFu);
      const int ms = e % MST;
      mbar_wait(&sm.m_full[ms], (e / MST) & 1);
      mbar_wait(&sm.s_full[e & 1], (e >> 1) & 1);
      tc_fence_after();
      const uint32_t tSq = tbase + lane_off + S_COL0 + (e & 1) * 128 + cq * 32;  // this quarter's S
      // Pass 1: max over this quarter's 32 columns (S stays in TMEM for pass 2).  PARTIAL tiles:
      // element mask of Alg. 1 lines 15-21 (row r masked for key y iff (unsigned)(r - start_y) <
      // len_y for either interval, or (causal) r < y), masked S written back to TMEM.
      uint32_t sr[2][16];
      tmem_ld16(tSq, sr[0]);
      tmem_ld16(tSq + 16, sr[1]);
      tmem_wait_ld();
      float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        float* sv = reinterpret_cast<float*>(sr[c]);
        if (cls == 1) {
          const int4* mk = sm.mask[ms] + cq * 32 + c * 16;
          const int rmy = row - (j * 128 + cq * 32 + c * 16);
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
#pragma unroll
        for (int t = 0; t < 16; t += 8) {
          mx0 = fmax3(mx0, sv[t], sv[t + 1]);
          mx1 = fmax3(mx1, sv[t + 2], sv[t + 3]);
          mx2 = fmax3(mx2, sv[t + 4], sv[t + 5]);
          mx3 = fmax3(mx3, sv[t + 6], sv[t + 7]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&sm.m_empty[ms]);
      const float mq = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
      sm.xmax[e & 1][cq][row_t] = mq;
      named_bar_sync(bar_id, 128);
      const float m_tile =
          fmaxf(fmaxf(sm.xmax[e & 1][0][row_t], sm.xmax[e & 1][1][row_t]),
                fmaxf(sm.xmax[e & 1][2][row_t], sm.xmax[e & 1][3][row_t])) * sl2;
      // Conditional rescale: the running max only moves when it grows by more than 2^8 (exact:
      // P is computed against the same m that scales l and O).  All four quarters see the same
      // m_tile and take the same decision.  O may still be accumulating PV_{e-1} (issued after
      // S_e), so a rescale first waits for it.
      const bool need = m_tile > m_used + 8.0f;
      float alpha = 1.0f;
      if (need) {
        alpha = ex2(m_used - m_tile);  // Alg. 1 line 25 factor e^{m_old - m_new}
        l *= alpha;
        m_used = m_tile;
      }
      if (__any_sync(0xffffffffu, need) && e > 0) {
        mbar_wait(&sm.pv_done, (e - 1) & 1);
        tc_fence_after();
        uint32_t ov[D / 4];
        if constexpr (D == 128) tmem_ld32(tbase + lane_off + O_COL + cq * 32, ov);
        else tmem_ld16(tbase + lane_off + O_COL + cq * 16, ov);
        tmem_wait_ld();
#pragma unroll
        for (int t = 0; t < D / 4; ++t) ov[t] = __float_as_uint(__uint_as_float(ov[t]) * alpha);
        if constexpr (D == 128) tmem_st32(tbase + lane_off + O_COL + cq * 32, ov);
        else tmem_st16(tbase + lane_off + O_COL + cq * 16, ov);
      }
      const float m_use = (m_used == -INFINITY) ? 0.f : m_used;
      // Pass 2: P = exp2(S*scale*log2e - m); packed FFMA2, MUFU ex2 for most pairs and the
      // FMA-pipe polynomial for FM_POLY_PAIRS1 of 8; packed bf16 P written over consumed S columns.
      const uint64_t sl2x2 = f2pack(sl2, sl2), negm2 = f2pack(-m_use, -m_use);
      uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        const float* sv = reinterpret_cast<const float*>(sr[ch]);
        uint32_t pk[8];
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const int k = ch * 8 + kk;
          const uint64_t x2 = f2fma(f2pack(sv[2 * kk], sv[2 * kk + 1]), sl2x2, negm2);
          float p0, p1;
          if ((k & 7) >= 8 - FM_POLY_PAIRS1) {
            exp2_poly2(x2, p0, p1);
          } else {
            float x0, x1;
            f2unpack(x2, x0, x1);
            p0 = ex2(x0);
            p1 = ex2(x1);
          }
          acc[k & 3] = f2add(acc[k & 3], f2pack(p0, p1));
          pk[kk] = pack_bf16(p0, p1);
        }
        tmem_st8(tSq + ch * 8, pk);
      }
      {
        const uint64_t a01 = f2add(acc[0], acc[1]), a23 = f2add(acc[2], acc[3]);
        float u0, u1;
        f2unpack(f2add(a01, a23), u0, u1);
        l += u0 + u1;
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&sm.p_full[e & 1]);
    }
    // ---- epilogue: O = O / l, L = m + ln(l) (Alg. 1 lines 27-28) ----
    sm.xsum[cq][row_t] = l;
    named_bar_sync(bar_id, 128);
    l = (sm.xsum[0][row_t] + sm.xsum[1][row_t]) + (sm.xsum[2][row_t] + sm.xsum[3][row_t]);
    const bool live = (nE > 0) && (l > 0.f);
    mbar_wait(&sm.o_full, 0);
    tc_fence_after();
    const float inv = live ? 1.0f / l : 0.f;
    constexpr int OC = D / 4;  // O columns of this warp
    uint32_t ov[OC];
    if (nE > 0) {
      if constexpr (D == 128) tmem_ld32(tbase + lane_off + O_COL + cq * OC, ov);
      else tmem_ld16(tbase + lane_off + O_COL + cq * OC, ov);
      tmem_wait_ld();
    }
    if constexpr (!OUT_F32) {
      // bf16 O through the (free) Q staging buffer, 128-B swizzled, and TMA tensor stores;
      // rows >= N are clipped by the TMA unit.
      mbar_wait(&sm.bar_q, 0);
      const int col = cq * OC;
      uint8_t* blk = sm.q + (col / 64) * 16384 + row_t * 128;
#pragma unroll
      for (int t = 0; t < OC / 8; ++t) {
        float f[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) f[u] = live ? __uint_as_float(ov[8 * t + u]) * inv : 0.f;
        const int chunk = (col % 64) / 8 + t;
        *reinterpret_cast<uint4*>(blk + ((chunk ^ (row_t & 7)) << 4)) =
            make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
      }
      fence_proxy_async_smem();
      named_bar_sync(9, 512);
      if (warp == 0 && lane == 0) {
#pragma unroll
        for (int c = 0; c < D / 64; ++c) tma_store_4d(&tmO, sm.q + c * 16384, c * 64, h, i * 128, b);
        bulk_commit();
        bulk_wait_read0();
      }
    } else if (row < a.N) {
      float* dst = static_cast<float*>(a.o) + ((static_cast<size_t>(b) * a.N + row) * a.H + h) * D + cq * OC;
#pragma unroll
      for (int t = 0; t < OC / 4; ++t)
        reinterpret_cast<float4*>(dst)[t] =
            live ? make_float4(__uint_as_float(ov[4 * t]) * inv, __uint_as_float(ov[4 * t + 1]) * inv,
                               __uint_as_float(ov[4 * t + 2]) * inv, __uint_as_float(ov[4 * t + 3]) * inv)
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (row < a.N && cq == 0)
      a.lse[(static_cast<size_t>(b) * a.H + h) * a.N + row] =
          live ? (m_used + __log2f(l)) * 0.6931471805599453f : -INFINITY;
  }

  tc_fence_before();
  __syncthreads();
  if (warp == MMA_WARP) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int D, bool CAUSAL, bool OUT_F32>
static cudaError_t launch_fwd1_t(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                                 const CUtensorMap& to, const FwdArgs& a, cudaStream_t st) {
  auto kern = fm_fwd1_kernel<D, CAUSAL, OUT_F32>;
  const size_t smem = sizeof(fwd1::Smem<D>) + 1024;
  static_assert(sizeof(fwd1::Smem<D>) + 1024 <= 232448, "shared memory budget");
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(d.Tr, d.H, d.B);
  kern<<<grid, fwd1::NT, smem, st>>>(tq, tk, tv, to, a);
  return cudaGetLastError();
}

cudaError_t launch_fwd1(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                        const CUtensorMap& to, const FwdArgs& a, cudaStream_t st) {
#define FM_F(DD, CC, FF) return launch_fwd1_t<DD, CC, FF>(d, tq, tk, tv, to, a, st)
  if (d.D == 128) {
    if (d.causal) { if (d.out_f32) FM_F(128, true, true); else FM_F(128, true, false); }
    else { if (d.out_f32) FM_F(128, false, true); else FM_F(128, false, false); }
  } else {
    if (d.causal) { if (d.out_f32) FM_F(64, true, true); else FM_F(64, true, false); }
    else { if (d.out_f32) FM_F(64, false, true); else FM_F(64, false, false); }
  }
#undef FM_F
}

}  // namespace fm
