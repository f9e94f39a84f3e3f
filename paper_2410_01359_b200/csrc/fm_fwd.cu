// fm_fwd.cu — K2: FlashMask forward (Alg. 1) for sm_100a.
//
// One CTA owns a pair of 128-row query tiles (Q0, Q1) of one (batch, head).  Warp roles:
//   warps 0-7   softmax of Q0: two warpgroups, each one half (64) of the key columns
//   warps 8-15  softmax of Q1  (thread = one row = one TMEM lane)
//   warp  16    TMA producer (lane 0): Q once, then K_j, V_j and the mask slice of tile j
//   warp  17    TMEM allocator + tcgen05 MMA issuer (lane 0)
// The visit list — the column tiles j that are not SKIP for Q0 or Q1 — is built from the
// K1 class map before the roles split, so fully masked tiles issue no load and no MMA
// (Alg. 1 lines 9-14).  S_q = Q_q K_j^T (tcgen05, fp32 in TMEM), softmax in
// registers with the element-wise interval mask applied only on PARTIAL tiles (Alg. 1
// lines 15-21), P_q written back to TMEM as bf16 (aliasing consumed S_q columns) and
// O_q += P_q V_j issued with P as the TMEM A operand.  The two query tiles ping-pong: while
// one WG runs its softmax the tensor core computes the other tile's S / PV.
// TMEM columns: S0 [0,128)  S1 [128,256)  O0 [256,256+D)  O1 [256+D, 256+2D).
#include <cuda_bf16.h>
#include <cmath>
#include <type_traits>

#include "fm_internal.h"
#include "fm_ptx.cuh"

#ifdef FM_TRACE
#ifndef FM_TRACE_BX
#define FM_TRACE_BX 64
#endif
#ifndef FM_TRACE_BY
#define FM_TRACE_BY 0
#endif
namespace fm { __device__ long long g_fm_trace_fwd[64 * 16]; __device__ long long g_fm_trace_fwd_ev[16];
__device__ long long g_fm_trace_fwd_w[8 * 32]; }
#define FT(slot, e)                                                                                   \
  do {                                                                                                 \
    if (blockIdx.x == FM_TRACE_BX && blockIdx.y == FM_TRACE_BY && blockIdx.z == 0 && (e) < 64) fm::g_fm_trace_fwd[(e) * 16 + (slot)] = clock64(); \
  } while (0)
#define FTE(k)                                                                                          \
  do {                                                                                                 \
    if (blockIdx.x == FM_TRACE_BX && blockIdx.y == FM_TRACE_BY && blockIdx.z == 0) fm::g_fm_trace_fwd_ev[k] = clock64(); \
  } while (0)
#define FM_TRACE_NE(n) (fm::g_fm_trace_fwd_ev[9] = (n))
#else
#define FT(slot, e) \
  do {              \
  } while (0)
#define FTE(k) \
  do {         \
  } while (0)
#define FM_TRACE_NE(n) ((void)0)
#endif

namespace fm {

namespace fwd {

constexpr int NT = 576;   // 16 softmax warps + TMA producer + MMA issuer
constexpr int MST = 4;
// of every 8 column pairs, how many take the FMA-pipe polynomial exp2 (the rest MUFU ex2):
// 1-3 of 8 change the forward by < 2 %
constexpr int kPolyPairs = 3;
// the bounded single pass (BND, R33) issues fewer instructions per tile: 2 of 8 measured best there
// (in-process A/B vs 3: C3 +0.2 %, 32K causal +1.1 %, random eviction +1.8 %, d = 64 +1.5..2 %)
constexpr int kPolyPairsBnd = 2;
// f3: mask only the dirty 32 x 16 sub-blocks of PARTIAL tiles (K1c words).  Compiled into the
// causal kernels only: in-process A/B measured +2..+6 % on causal families
// (+24 % QK-sparse) but -1.3 % on the non-causal C3 kernel (code generation) and +-1.5 % elsewhere.
template <bool CAUSAL>
constexpr bool kRefine = CAUSAL;
// K / V ring depths (d = 128: 2 each fills shared memory; d = 64 tiles are half the size:
// 3-deep rings, +1-3 % on the C5 d = 64 sweep)
template <int D>
struct Rings {
  static constexpr int KST = (D == 64) ? 3 : 2, VST = (D == 64) ? 3 : 2;
};

template <int D>
struct Smem {
  static constexpr int TILE = 128 * D * 2;
  uint8_t q[2][TILE];
  uint8_t k[Rings<D>::KST][TILE];
  uint8_t v[Rings<D>::VST][TILE];
  int4 mask[MST][128];
  uint32_t cw[MST][2];  // f3 refinement words of the stage's tile for Q0 / Q1 (PARTIAL only)
  uint32_t list[kMaxTc];
  uint64_t bar_q;
  uint64_t k_full[Rings<D>::KST], k_empty[Rings<D>::KST], v_full[Rings<D>::VST], v_empty[Rings<D>::VST];
  uint64_t m_full[MST], m_empty[MST];
  uint64_t s_full[2], p_full[2], o_full[2], s_read[2], pv_done[2];
  float xmax[2][2][2][128];  // [tile][parity][column half][row]: row-max exchange between halves
  float xsum[2][2][128];     // [tile][column half][row]: final row-sum exchange
  uint32_t tmem_base;
  int n_entries;
  int warp_cnt[NT / 32];
  float warp_kmax[NT / 32];  // BND: largest key norm over each warp's visited column tiles
  uint32_t fixbits[NT / 32];  // persistent fixup launch: this CTA's flagged units of a chunk
};

constexpr int PRODUCER_WARP = 16, MMA_WARP = 17;
// d=64 leaves 128 TMEM columns free (S0, S1 128 each, O0, O1 64 each): P gets its own buffers
// [384, 448) / [448, 512), so S_q(e+1) is issued as soon as the softmax has read S_q(e) — the S
// MMA then runs under the tail of the softmax instead of after it (d=128: P aliases S).
template <int D>
struct Layout {
  static constexpr bool SEP_P = (D == 64);
  static constexpr uint32_t P_COL = 384;
};

__device__ __forceinline__ int ent_cls(uint32_t ent, int q) { return (ent >> (24 + 2 * q)) & 3; }

}  // namespace fwd

// ROWW: row-wise representation (FM_FLAG_ROWWISE, R32) — a.vec4 holds each query
// ROW's masked key intervals; a softmax thread (= one row) keeps its own in registers and no mask
// slice is loaded per tile.
// BND: R33 bounded single pass (bf16 operands): P of every tile against the fixed per-row reference
// ||q_r|| max_y ||k_y|| scale log2(e) - 96, no max pass, no rescaling; unfinished rows flag the
// unit for the two-pass fixup launch (this kernel with BND = false and a.fix set).
// FIX: the persistent two-pass fixup launch over the units a bounded pass flagged (BND = false).
template <int D, bool CAUSAL, bool OUT_F32, bool F16, bool ROWW, bool BND, bool FIX>
__global__ void __launch_bounds__(fwd::NT, 1)
    fm_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, const FwdArgs a) {
  using namespace fwd;
  using S = Smem<D>;
  constexpr int KST = Rings<D>::KST, VST = Rings<D>::VST;
  extern __shared__ uint8_t smem_raw[];
  S& sm = *smem_align1024<S>(smem_raw);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int npairs = (a.Tr + 1) >> 1;
  // ---------------- one unit of work: the query-tile pair `pair` of head h, batch entry b ----------------
  // first: this CTA's first unit (TMEM allocation and the grid-dependency wait happen here)
  // reinit: an earlier unit of this CTA initialised the mbarriers (invalidate before re-initialising)
  auto unit_body = [&](const int b, const int h, const int pair, const bool first, const bool reinit) {
    const size_t unit = (static_cast<size_t>(b) * a.H + h) * npairs + pair;
    const int hk = h / a.G;                      // key/value head of this query head (GQA)
    const int hm = (a.Hm == 1) ? 0 : hk;
    const int i0 = 2 * pair, i1 = 2 * pair + 1;
    const bool has_q1 = i1 < a.Tr;
    const size_t bhm = static_cast<size_t>(b) * a.Hm + hm;

    if (tid == 0) FTE(0);
    // ---- setup: barriers (warp 8), TMEM (warp 9) ----
    if (warp == PRODUCER_WARP && lane == 0) {
      if (reinit) {  // persistent fixup: the previous unit's barriers are quiescent (end-of-unit sync)
        mbar_inval(&sm.bar_q);
        for (int s = 0; s < KST; ++s) { mbar_inval(&sm.k_full[s]); mbar_inval(&sm.k_empty[s]); }
        for (int s = 0; s < VST; ++s) { mbar_inval(&sm.v_full[s]); mbar_inval(&sm.v_empty[s]); }
        for (int s = 0; s < MST; ++s) { mbar_inval(&sm.m_full[s]); mbar_inval(&sm.m_empty[s]); }
        for (int q = 0; q < 2; ++q) {
          mbar_inval(&sm.s_full[q]); mbar_inval(&sm.p_full[q]); mbar_inval(&sm.o_full[q]);
          mbar_inval(&sm.s_read[q]); mbar_inval(&sm.pv_done[q]);
        }
      }
      mbar_init(&sm.bar_q, 1);
      for (int s = 0; s < KST; ++s) { mbar_init(&sm.k_full[s], 1); mbar_init(&sm.k_empty[s], 1); }
      for (int s = 0; s < VST; ++s) { mbar_init(&sm.v_full[s], 1); mbar_init(&sm.v_empty[s], 1); }
      for (int s = 0; s < MST; ++s) { mbar_init(&sm.m_full[s], 1); mbar_init(&sm.m_empty[s], 16); }
      for (int q = 0; q < 2; ++q) {
        mbar_init(&sm.s_full[q], 1);
        mbar_init(&sm.p_full[q], 256);
        mbar_init(&sm.o_full[q], 1);
        mbar_init(&sm.s_read[q], 256);
        mbar_init(&sm.pv_done[q], 1);
      }
      fence_barrier_init();
      // Q does not depend on the visit list: start its load before the list is built
      tma_prefetch_desc(&tmQ);
      mbar_expect_tx(&sm.bar_q, has_q1 ? 2 * S::TILE : S::TILE);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        tma_load_4d(sm.q[0] + c * 16384, &tmQ, &sm.bar_q, c * 64, h, i0 * 128, b);
        if (has_q1) tma_load_4d(sm.q[1] + c * 16384, &tmQ, &sm.bar_q, c * 64, h, i1 * 128, b);
      }
    }
    if (first) {
      if (warp == MMA_WARP) tmem_alloc<512>(&sm.tmem_base);
      pdl_wait();  // the class map (K1b) and refinement words (K1c, the stream predecessor) are complete
      pdl_launch();
    }

    // ---- visit list: union of the non-SKIP column tiles of Q0 and Q1 (K1 class map) ----
    {
      const uint8_t* row0 = a.fmap + (bhm * a.Tr + i0) * a.Tc;
      const uint8_t* row1 = row0 + a.Tc;
      int base = 0;
      // BND: largest key norm of the head over ALL its column tiles — independent of which tiles are
      // visited, so FM_FLAG_NO_SKIP (SKIP visited as PARTIAL) keeps the same reference bit for bit
      float kv = 0.f;
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
        int off = base;
        int tot = 0;
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
    if (tid == 0) FTE(1);

    if (warp == PRODUCER_WARP) {
      // ================================ TMA producer ================================
      if (lane == 0) {
        tma_prefetch_desc(&tmK);
        tma_prefetch_desc(&tmV);
        constexpr uint32_t TB = S::TILE;
        if (nE == 0) mbar_wait(&sm.bar_q, 0);  // no MMA will wait for Q: it must land before exit
        const int4* vec_bh = a.vec4 + bhm * static_cast<size_t>(a.Tc) * 128;
        for (int e = 0; e < nE; ++e) {
          const uint32_t ent = sm.list[e];
          const int j = static_cast<int>(ent & 0xFFFFFFu);
          const int ks = e % KST, vs = e % VST, ms = e % MST;
          mbar_wait(&sm.k_empty[ks], ((e / KST) & 1) ^ 1);
          mbar_expect_tx(&sm.k_full[ks], TB);
#pragma unroll
          for (int c = 0; c < D / 64; ++c) tma_load_4d(sm.k[ks] + c * 16384, &tmK, &sm.k_full[ks], c * 64, hk, j * 128, b);
          FT(11, e);
          mbar_wait(&sm.m_empty[ms], ((e / MST) & 1) ^ 1);
          if (!ROWW && (ent_cls(ent, 0) == 1 || ent_cls(ent, 1) == 1)) {
            // f3: which 32-row x 16-column sub-blocks hold a masked cell (K1c); the ragged last
            // column tile keeps every sub-block masked (its padded keys need the bounds mask)
#pragma unroll
            for (int qq = 0; qq < 2; ++qq) {
              uint32_t wq = 0xFFFFFFFFu;
              if (kRefine<CAUSAL> && a.cw != nullptr && ent_cls(ent, qq) == 1 && !(j == a.Tc - 1 && (a.N & 127) != 0))
                wq = a.cw[(bhm * a.Tr + (qq == 0 ? i0 : i1)) * a.Tc + j];
              sm.cw[ms][qq] = wq;
            }
            mbar_expect_tx(&sm.m_full[ms], 128 * 16);  // arrive (release): the words above are visible
            bulk_g2s(sm.mask[ms], vec_bh + static_cast<size_t>(j) * 128, 128 * 16, &sm.m_full[ms]);
          } else {
            mbar_arrive(&sm.m_full[ms]);
          }
          mbar_wait(&sm.v_empty[vs], ((e / VST) & 1) ^ 1);
          mbar_expect_tx(&sm.v_full[vs], TB);
#pragma unroll
          for (int c = 0; c < D / 64; ++c) tma_load_4d(sm.v[vs] + c * 16384, &tmV, &sm.v_full[vs], c * 64, hk, j * 128, b);
          FT(14, e);
        }
      }
    } else if (warp == MMA_WARP) {
      // ================================ MMA issuer ================================
      // One issuer for both tiles, in the order PV0(e-1), S0(e), PV1(e-1), S1(e): this keeps the
      // two tiles' softmax phases staggered (ping-pong).  Two independent issuers were measured
      // to fall into lock-step and lose ~30 %.
      {  // the whole warp runs the issue loop converged; one elected lane issues
        constexpr uint32_t ID_S = idesc16<F16>(128, 128, 0, 0);  // S = Q K^T, both K-major
        constexpr uint32_t ID_PV = idesc16<F16>(128, D, 0, 1);   // O += P V, V is MN-major
        const uint32_t tS[2] = {tbase + 0, tbase + 128};
        const uint32_t tO[2] = {tbase + 256, tbase + 256 + D};
        const uint32_t q_addr[2] = {smem_u32(sm.q[0]), smem_u32(sm.q[1])};
        int pend[2] = {-1, -1};
        uint32_t pv_cnt[2] = {0, 0};
        auto issue_pv = [&](int q) {
          const int pe = pend[q];
          mbar_wait(&sm.p_full[q], pv_cnt[q] & 1);
          if (lane == 0) FT(4 + q, pe);
          const int vs = pe % VST;
          mbar_wait(&sm.v_full[vs], (pe / VST) & 1);
          if (lane == 0 && q == 0) FT(15, pe);
          tc_fence_after();
          const uint32_t v_addr = smem_u32(sm.v[vs]);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint64_t bd = sdesc_sw128(v_addr + kk * 2048, 16384, 1024);
            // P of keys [0,64) sits in S columns [0,32), of keys [64,128) in S columns [64,96);
            // SEP_P: P of keys [16kk, 16kk+16) in columns P_COL + 64q + 8kk
            const uint32_t a_tm = Layout<D>::SEP_P ? tbase + Layout<D>::P_COL + q * 64 + kk * 8
                                                   : tS[q] + kk * 8 + (kk >= 4 ? 32u : 0u);
            mma_ts_w(tO[q], a_tm, bd, ID_PV, (pv_cnt[q] > 0 || kk > 0) ? 1u : 0u);
          }
          if constexpr (Layout<D>::SEP_P) mma_commit_w(&sm.pv_done[q]);
          pv_cnt[q]++;
          const uint32_t ent = sm.list[pe];
          const int last = (ent_cls(ent, 1) != 0) ? 1 : 0;
          if (q == last) mma_commit_w(&sm.v_empty[vs]);
          pend[q] = -1;
        };
        if (nE > 0) {
          mbar_wait(&sm.bar_q, 0);
          tc_fence_after();
        }
        if (lane == 0) FTE(2);
        for (int e = 0; e < nE; ++e) {
          const uint32_t ent = sm.list[e];
          const int ks = e % KST;
          mbar_wait(&sm.k_full[ks], (e / KST) & 1);
          if (lane == 0) FT(8, e);
          tc_fence_after();
          const uint32_t k_addr = smem_u32(sm.k[ks]);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            if (!Layout<D>::SEP_P && pend[q] >= 0) issue_pv(q);
            if (ent_cls(ent, q) != 0) {
              // SEP_P: S_q(e) overwrites S_q(pend) once the softmax has read it (s_read)
              if (Layout<D>::SEP_P && pend[q] >= 0) mbar_wait(&sm.s_read[q], pv_cnt[q] & 1);
              tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < D / 16; ++kk) {
                const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
                mma_ss_w(tS[q], sdesc_sw128(q_addr[q] + off, 16, 1024), sdesc_sw128(k_addr + off, 16, 1024), ID_S,
                       kk > 0 ? 1u : 0u);
              }
              mma_commit_w(&sm.s_full[q]);
              if (lane == 0) FT(6 + q, e);
            }
            if (Layout<D>::SEP_P && pend[q] >= 0) {
              // every s_read phase is observed, also when no S_q(e) follows (tile SKIP for q)
              if (ent_cls(ent, q) == 0) mbar_wait(&sm.s_read[q], pv_cnt[q] & 1);
              issue_pv(q);
            }
            if (ent_cls(ent, q) != 0) pend[q] = e;
          }
          mma_commit_w(&sm.k_empty[ks]);
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {  // O_q complete: its epilogue need not wait for the other tile
          // SEP_P: consume the last s_read phase too (already complete: P follows the read), so
          // every mbarrier phase is observed
          if (Layout<D>::SEP_P && pend[q] >= 0) mbar_wait(&sm.s_read[q], pv_cnt[q] & 1);
          if (pend[q] >= 0) issue_pv(q);
          mma_commit_w(&sm.o_full[q]);
        }
      }
    } else {
      // ================================ softmax WGs ================================
      // Four warpgroups: tile q = warp / 8, column half hh = (warp / 4) % 2.  The two halves of a
      // tile share TMEM lanes (rows) and split the 128 key columns, exchanging row maxima (and at
      // the end the row sums) through shared memory under a 64-thread named barrier per warp pair.
      const int q = warp >> 3;
      const int hh = (warp >> 2) & 1;
      const int wl = warp & 3;
      const int row_t = wl * 32 + lane;
      const int row = (q == 0 ? i0 : i1) * 128 + row_t;
      const uint32_t lane_off = static_cast<uint32_t>(wl * 32) << 16;
      const uint32_t tS = tbase + lane_off + (q == 0 ? 0u : 128u);
      const uint32_t tSh = tS + hh * 64;                      // this half's 64 S columns
      const uint32_t tPh = Layout<D>::SEP_P ? tbase + lane_off + Layout<D>::P_COL + q * 64 + hh * 32
                                            : tS + hh * 64;   // its packed P (32 columns) — see MMA
      const uint32_t tO = tbase + lane_off + 256u + (q == 0 ? 0u : static_cast<uint32_t>(D));
      const uint32_t tOh = tO + hh * (D / 2);                 // this half's O columns
      const float sl2 = a.scale_log2;
      // the two warps holding the same 32 rows (column halves 0/1) exchange through a 64-thread barrier
      const uint32_t bar_id = 1 + q * 4 + wl;
      float m_used = -INFINITY;  // running max of the scaled logits, log2 units (threshold-updated)
      float l = 0.f;             // this half's share of the row sum
      uint32_t cnt = 0;
      int4 rmv = make_int4(0, 0, 0, 0);  // row-wise: this row's (LTS, len, UTS, len) over key columns
      // (rows past N — the ragged last tile, or the absent second tile of an odd tile count — take
      // K1a's padding value: every key masked)
      if constexpr (ROWW)
        rmv = row < a.N ? a.vec4[bhm * static_cast<size_t>(a.Tc) * 128 + row] : make_int4(0, INT_MAX, 0, 0);
      // R33 (BND): the row's fixed reference, ||q_r|| * max key norm of the head * scale * log2(e) - 96,
      // so every P <= 2^96; set at the first visited tile (Q has landed once S has)
      float m_ref = 0.f;
      float kvis = 0.f;
      if constexpr (BND) {
#pragma unroll
        for (int w = 0; w < NT / 32; ++w) kvis = fmaxf(kvis, sm.warp_kmax[w]);
      }
      for (int e = 0; e < nE; ++e) {
        const uint32_t ent = sm.list[e];
        const int cls = ent_cls(ent, q);
        const int ms = e % MST;
        mbar_wait(&sm.m_full[ms], (e / MST) & 1);
        if (cls != 0) {
          const int j = static_cast<int>(ent & 0xFFFFFFu);
          mbar_wait(&sm.s_full[q], cnt & 1);
          if (row_t == 0 && hh == 0) FT(0 + q, e);
          tc_fence_after();
          uint32_t sr[2][16];
          // f3: the 16-column chunks of this warp's 32 rows x 64 columns that hold a masked cell
          const uint32_t pm =
              (cls != 1) ? 0u : ((kRefine<CAUSAL> && !ROWW) ? (sm.cw[ms][q] >> (wl * 8 + hh * 4)) & 0xFu : 0xFu);
          if constexpr (BND) {
            if (cnt == 0) {
              // ||q_r|| from the Q tile in shared memory: granule g ^ (row & 7) of the 128-byte
              // swizzled row, so the 8 rows of a bank group read 8 different 16-byte columns
              mbar_wait(&sm.bar_q, 0);  // observe the TMA write of Q (complete long since: S used it)
              float ss = 0.f;
#pragma unroll
              for (int c = 0; c < D / 64; ++c) {
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                  const uint4 u = *reinterpret_cast<const uint4*>(sm.q[q] + c * 16384 + row_t * 128 + ((g ^ (row_t & 7)) << 4));
                  const uint32_t w4[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
                  for (int t = 0; t < 4; ++t) {
                    const float lo = __uint_as_float(w4[t] << 16), hi = __uint_as_float(w4[t] & 0xFFFF0000u);
                    ss = fmaf(lo, lo, fmaf(hi, hi, ss));
                  }
                }
              }
              m_ref = sqrtf(ss) * (1.0f + 1.0f / 65536.0f) * kvis * sl2 - kBndHeadroom;
            }
            if (Layout<D>::SEP_P && cnt > 0) {  // PV_q(e-1) done with the P buffer
              mbar_wait(&sm.pv_done[q], (cnt - 1) & 1);
              tc_fence_after();
            }
          } else {
          // Pass 1: max over this half's 64 columns, 32 at a time (S stays in TMEM for pass 2).
          // On PARTIAL tiles the element mask (Alg. 1 lines 15-21) is applied here and the masked S
          // written back to TMEM, so pass 2 is identical for PARTIAL and UNMASKED tiles.
          float mx0 = -INFINITY, mx1 = -INFINITY, mx2 = -INFINITY, mx3 = -INFINITY;
          tmem_ld16(tSh, sr[0]);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            tmem_wait_ld();
            if (c + 1 < 4) tmem_ld16(tSh + (c + 1) * 16, sr[(c + 1) & 1]);
            float* sv = reinterpret_cast<float*>(sr[c & 1]);
            if (pm & (1u << c)) {
              // element mask of Alg. 1 lines 15-21: row r is masked for key y iff
              // (unsigned)(r - start_y) < len_y for either interval, or (causal) r < y
              const int4* mk = sm.mask[ms] + hh * 64 + c * 16;
              const int rmy = row - (j * 128 + hh * 64 + c * 16);
              if constexpr (ROWW) {
                // key y = row - rmy + t is masked for this row iff it lies in one of the row's key
                // intervals, after the row (causal), or past N (the ragged last column tile)
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                  const int y = row - rmy + t;
                  bool msk = (static_cast<unsigned>(y - rmv.x) < static_cast<unsigned>(rmv.y)) ||
                             (static_cast<unsigned>(y - rmv.z) < static_cast<unsigned>(rmv.w)) || y >= a.N;
                  if constexpr (CAUSAL) msk |= rmy < t;
                  sv[t] = msk ? -INFINITY : sv[t];
                }
              } else if (CAUSAL && j < (q == 0 ? i0 : i1)) {
                // causal: below the diagonal tile (j < i) no key of the tile lies after any of its
                // rows, so the r < y test is dropped there (warp-uniform choice)
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
              tmem_st16(tSh + c * 16, sr[c & 1]);  // masked S back to TMEM: pass 2 needs no mask work
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
          const float mh = fmaxf(fmaxf(mx0, mx1), fmaxf(mx2, mx3));
          if (row_t == 0 && q == 0 && hh == 0) FT(10, e);
          sm.xmax[q][cnt & 1][hh][row_t] = mh;
          named_bar_sync(bar_id, 64);
          const float m_tile = fmaxf(mh, sm.xmax[q][cnt & 1][hh ^ 1][row_t]) * sl2;
          if (row_t == 0 && q == 0 && hh == 0) FT(9, e);
          // Conditional rescale: the running max only moves when it grows by more than 2^8
          // (exact: P is computed against the same m that scales l and O).  Both halves see the
          // same m_tile and take the same decision; the TMEM accesses stay warp-collective.
          const bool need = m_tile > m_used + 8.0f;
          float alpha = 1.0f;
          if (need) {
            alpha = ex2(m_used - m_tile);  // Alg. 1 line 25 factor e^{m_old - m_new}
            l *= alpha;
            m_used = m_tile;
          }
          if (Layout<D>::SEP_P && cnt > 0) {  // PV_q(e-1) (issued after S_q(e)) done with O and P
            mbar_wait(&sm.pv_done[q], (cnt - 1) & 1);
            tc_fence_after();
          }
          if (__any_sync(0xffffffffu, need) && cnt > 0) {
#pragma unroll 1
            for (int c = 0; c < D / 64; ++c) {
              uint32_t ov[32];
              tmem_ld32(tOh + c * 32, ov);
              tmem_wait_ld();
#pragma unroll
              for (int t = 0; t < 32; ++t) ov[t] = __float_as_uint(__uint_as_float(ov[t]) * alpha);
              tmem_st32(tOh + c * 32, ov);
            }
          }
          }  // two-pass (!BND)
          const float m_use = BND ? m_ref : ((m_used == -INFINITY) ? 0.f : m_used);
          // Pass 2: P = exp2(S*scale*log2e - m) over this half's columns; packed FFMA2 for the
          // argument, MUFU ex2 for most pairs and the FMA-pipe polynomial for kPolyPairs of 8;
          // row sums with packed FADD2; packed bf16 P written back over consumed S columns.
          const uint64_t sl2x2 = f2pack(sl2, sl2), negm2 = f2pack(-m_use, -m_use);
          uint64_t acc[4] = {0ull, 0ull, 0ull, 0ull};
          tmem_ld16(tSh, sr[0]);
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            tmem_wait_ld();
            if (ch + 1 < 4) tmem_ld16(tSh + (ch + 1) * 16, sr[(ch + 1) & 1]);
            if (Layout<D>::SEP_P && ch == 3) {  // all of S_q(e) is in registers
              tc_fence_before();
              mbar_arrive(&sm.s_read[q]);
            }
            float* sv = reinterpret_cast<float*>(sr[ch & 1]);
            if (BND && (pm & (1u << ch))) {
              // element mask of Alg. 1 lines 15-21 in registers (no max pass to carry it to TMEM)
              const int4* mk = sm.mask[ms] + hh * 64 + ch * 16;
              const int rmy = row - (j * 128 + hh * 64 + ch * 16);
              if constexpr (ROWW) {
#pragma unroll
                for (int t = 0; t < 16; ++t) {
                  const int y = row - rmy + t;
                  bool msk = (static_cast<unsigned>(y - rmv.x) < static_cast<unsigned>(rmv.y)) ||
                             (static_cast<unsigned>(y - rmv.z) < static_cast<unsigned>(rmv.w)) || y >= a.N;
                  if constexpr (CAUSAL) msk |= rmy < t;
                  sv[t] = msk ? -INFINITY : sv[t];
                }
              } else if (CAUSAL && j < (q == 0 ? i0 : i1)) {
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
              if ((k & 7) >= 8 - (BND ? kPolyPairsBnd : kPolyPairs)) {
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
            tmem_st8(tPh + ch * 8, pk);
          }
          if (row_t == 0 && q == 0 && hh == 0) FT(12, e);
          {
            const uint64_t a01 = f2add(acc[0], acc[1]), a23 = f2add(acc[2], acc[3]);
            float u0, u1;
            f2unpack(f2add(a01, a23), u0, u1);
            l += u0 + u1;
          }
          tmem_wait_st();
          if (row_t == 0 && q == 0 && hh == 0) FT(13, e);
          tc_fence_before();
          mbar_arrive(&sm.p_full[q]);
          if (row_t == 0 && hh == 0) FT(2 + q, e);
  #ifdef FM_TRACE
          // per-warp P-ready time of visited entries 20..27 (all 16 softmax warps)
          if (lane == 0 && e >= 20 && e < 28 && blockIdx.x == FM_TRACE_BX && blockIdx.y == FM_TRACE_BY && blockIdx.z == 0)
            g_fm_trace_fwd_w[(e - 20) * 32 + warp] = clock64();
  #endif
          ++cnt;
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.m_empty[ms]);
      }
      // ---- epilogue: O = O / l, L = m + ln(l) (Alg. 1 lines 27-28) ----
      if (row_t == 0 && hh == 0) FTE(3 + q);
      sm.xsum[q][hh][row_t] = l;
      named_bar_sync(bar_id, 64);
      l += sm.xsum[q][hh ^ 1][row_t];
      // BND: a row whose sum ends below 2^-90 (its logits far below the Cauchy-Schwarz bound, or every
      // key masked) flags the unit; the two-pass fixup launch recomputes it (O and lse overwritten)
      const bool live = (cnt > 0) && (BND ? (l >= kBndMinSum) : (l > 0.f));
      if (BND && row < a.N && !live) a.fix_out[unit] = 1;
      if (cnt > 0) {
        mbar_wait(&sm.o_full[q], 0);
        tc_fence_after();
      }
      const float inv = live ? 1.0f / l : 0.f;
      const size_t orow = ((static_cast<size_t>(b) * a.N + row) * a.H + h) * D + hh * (D / 2);
      if constexpr (!OUT_F32) {
        // bf16 O goes out through shared memory and one TMA store per 64-column block: a thread
        // holds one row, so direct 16-byte stores would scatter every warp instruction over 32 rows
        // (measured ~6K clk of LSU time per CTA).  The Q tile buffer of this tile is free: all its
        // S MMAs completed before o_full.  Rows >= N are clipped by the TMA unit.
        uint8_t* stg = sm.q[q];
        mbar_wait(&sm.bar_q, 0);  // the Q load into this buffer has landed (even if no tile used it)
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          uint32_t ov[32];
          if (cnt > 0) {
            tmem_ld32(tOh + c * 32, ov);
            tmem_wait_ld();
          }
          const int col = hh * (D / 2) + c * 32;  // first of these 32 columns
          uint8_t* blk = stg + (col / 64) * 16384 + row_t * 128;
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            float f[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) f[u] = live ? __uint_as_float(ov[8 * t + u]) * inv : 0.f;
            const int chunk = (col % 64) / 8 + t;
            *reinterpret_cast<uint4*>(blk + ((chunk ^ (row_t & 7)) << 4)) =
                make_uint4(pack16<F16>(f[0], f[1]), pack16<F16>(f[2], f[3]), pack16<F16>(f[4], f[5]), pack16<F16>(f[6], f[7]));
          }
        }
        fence_proxy_async_smem();
        named_bar_sync(9 + q, 256);
        const int row0 = (q == 0 ? i0 : i1) * 128;
        if (warp == q * 8 && lane == 0 && row0 < a.N) {
#pragma unroll
          for (int c = 0; c < D / 64; ++c) tma_store_4d(&tmO, stg + c * 16384, c * 64, h, row0, b);
          bulk_commit();
          bulk_wait_read0();  // the staging buffer must outlive the TMA reads
        }
      }
#pragma unroll 1
      for (int c = 0; c < (OUT_F32 ? D / 64 : 0); ++c) {
        uint32_t ov[32];
        if (cnt > 0) {  // WG-uniform: the tcgen05.ld stays warp-collective
          tmem_ld32(tOh + c * 32, ov);
          tmem_wait_ld();
        }
        float f[32];
#pragma unroll
        for (int t = 0; t < 32; ++t) f[t] = live ? __uint_as_float(ov[t]) * inv : 0.f;
        if (row < a.N) {
          if constexpr (OUT_F32) {
            float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.o) + orow + c * 32);
#pragma unroll
            for (int t = 0; t < 8; ++t) dst[t] = make_float4(f[4 * t], f[4 * t + 1], f[4 * t + 2], f[4 * t + 3]);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(a.o) + orow + c * 32);
#pragma unroll
            for (int t = 0; t < 4; ++t)
              dst[t] = make_uint4(pack16<F16>(f[8 * t], f[8 * t + 1]), pack16<F16>(f[8 * t + 2], f[8 * t + 3]),
                                  pack16<F16>(f[8 * t + 4], f[8 * t + 5]), pack16<F16>(f[8 * t + 6], f[8 * t + 7]));
          }
        }
      }
      if (row < a.N && hh == 0)
        a.lse[(static_cast<size_t>(b) * a.H + h) * a.N + row] =
            live ? ((BND ? m_ref : m_used) + __log2f(l)) * 0.6931471805599453f : -INFINITY;
      if (row_t == 0 && hh == 0) FTE(5 + q);
    }


    tc_fence_before();
    __syncthreads();  // end of unit: every barrier phase complete, TMEM and shared memory free
  };

  if constexpr (FIX) {
    // Two-pass fixup launch (R33), persistent: one wave of CTAs; each CTA takes units
    // blockIdx.x + k * gridDim.x, reads their flags (written by the bounded pass, the stream
    // predecessor) NT at a time and runs the flagged ones one after another.
    if (warp == MMA_WARP) tmem_alloc<512>(&sm.tmem_base);
    pdl_wait();
    pdl_launch();
    const int nunits = a.B * a.H * npairs;
    bool any = false;
    for (int base = 0; static_cast<long>(base) * gridDim.x < nunits; base += NT) {
      const long u = blockIdx.x + static_cast<long>(gridDim.x) * (base + tid);
      const bool f = u < nunits && a.fix[u] != 0;
      const unsigned bal = __ballot_sync(0xffffffffu, f);
      if (lane == 0) sm.fixbits[warp] = bal;
      __syncthreads();
      for (int w = 0; w < NT / 32; ++w) {
        uint32_t bits = sm.fixbits[w];
        while (bits) {
          const int l = __ffs(bits) - 1;
          bits &= bits - 1;
          const int uu = static_cast<int>(blockIdx.x + static_cast<long>(gridDim.x) * (base + w * 32 + l));
          const int pr = uu % npairs, hb = uu / npairs;
          tc_fence_after();
          unit_body(hb / a.H, hb % a.H, pr, false, any);
          any = true;
        }
      }
      __syncthreads();  // fixbits is rewritten by the next chunk
    }
    tc_fence_after();
    if (warp == MMA_WARP) tmem_dealloc<512>(sm.tmem_base);
  } else {
    const int b = blockIdx.z;
    // unit of this CTA: without an LPT order, pair npairs-1-x of head y (last row tiles first: the
    // heaviest under causal-like masks); with one (K1d, small problems), the CTAs of a batch entry
    // take groups of a.hgrp heads, in each group the pairs by descending work, heads innermost
    int pair, h;
    // the order comes from the stream predecessor (K1d): wait for it before the (early) Q load
    if (a.order != nullptr) pdl_wait();
    if (a.order != nullptr && (a.Hm > 1 || a.order[static_cast<size_t>(a.B) * npairs + b] != 0)) {
      const int L = static_cast<int>(blockIdx.x) + npairs * static_cast<int>(blockIdx.y);
      const int per_g = npairs * a.hgrp;
      const int g = L / per_g, rem = L - g * per_g;
      const int prank = rem / a.hgrp;
      h = g * a.hgrp + (rem - prank * a.hgrp);
      const int hmo = (a.Hm == 1) ? 0 : h / a.G;
      pair = a.order[(static_cast<size_t>(b) * a.Hm + hmo) * npairs + prank];
    } else {
      pair = npairs - 1 - static_cast<int>(blockIdx.x);
      h = blockIdx.y;
    }
    unit_body(b, h, pair, true, false);
    if (warp == MMA_WARP) {
      tc_fence_after();
      tmem_dealloc<512>(sm.tmem_base);
    }
  }
#ifdef FM_TRACE
  if (tid == 0) {
    FTE(7);
  }
#endif
}

template <int D, bool CAUSAL, bool OUT_F32, bool F16, bool ROWW, bool BND, bool FIX = false>
static cudaError_t launch_fwd_t(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                                const CUtensorMap& to, const FwdArgs& a, cudaStream_t st) {
  auto kern = fm_fwd_kernel<D, CAUSAL, OUT_F32, F16, ROWW, BND, FIX>;
  const size_t smem = sizeof(fwd::Smem<D>) + 1024;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid((d.Tr + 1) / 2, d.H, d.B);
  if (FIX) {  // persistent fixup: one wave (one CTA per SM), each CTA walks its share of the units
    static int n_sm = 0;
    if (n_sm == 0 && cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0) != cudaSuccess) n_sm = 148;
    const long units = static_cast<long>(grid.x) * grid.y * grid.z;
    grid = dim3(static_cast<unsigned>(units < n_sm ? units : n_sm), 1, 1);
  }
  return launch_pdl(kern, grid, dim3(fwd::NT), smem, st, tq, tk, tv, to, a);
}

cudaError_t launch_fwd(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                       const CUtensorMap& to, const FwdArgs& a, cudaStream_t st) {
#define FM_F(DD, CC, FF)                                                                                    \
  do {                                                                                                      \
    if (a.fix != nullptr)  /* R33 two-pass fixup over the flagged units (bf16 operands) */                  \
      return d.rowwise ? launch_fwd_t<DD, CC, FF, false, true, false, true>(d, tq, tk, tv, to, a, st)       \
                       : launch_fwd_t<DD, CC, FF, false, false, false, true>(d, tq, tk, tv, to, a, st);     \
    if (a.kmax != nullptr && !d.in_f16)  /* R33 bounded single pass: bf16 operands */                       \
      return d.rowwise ? launch_fwd_t<DD, CC, FF, false, true, true>(d, tq, tk, tv, to, a, st)              \
                       : launch_fwd_t<DD, CC, FF, false, false, true>(d, tq, tk, tv, to, a, st);            \
    if (d.rowwise)                                                                                          \
      return d.in_f16 ? launch_fwd_t<DD, CC, FF, true, true, false>(d, tq, tk, tv, to, a, st)               \
                      : launch_fwd_t<DD, CC, FF, false, true, false>(d, tq, tk, tv, to, a, st);             \
    return d.in_f16 ? launch_fwd_t<DD, CC, FF, true, false, false>(d, tq, tk, tv, to, a, st)                \
                    : launch_fwd_t<DD, CC, FF, false, false, false>(d, tq, tk, tv, to, a, st);              \
  } while (0)
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

#ifdef FM_TRACE
extern "C" __attribute__((visibility("default"))) int flashmask_debug_trace_fwd(long long* host) {
  return cudaMemcpyFromSymbol(host, fm::g_fm_trace_fwd, sizeof(long long) * 64 * 16) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int flashmask_debug_trace_fwd_w(long long* host) {
  return cudaMemcpyFromSymbol(host, fm::g_fm_trace_fwd_w, sizeof(long long) * 8 * 32) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int flashmask_debug_trace_fwd_ev(long long* host) {
  return cudaMemcpyFromSymbol(host, fm::g_fm_trace_fwd_ev, sizeof(long long) * 16) == cudaSuccess ? 0 : 1;
}
#endif
