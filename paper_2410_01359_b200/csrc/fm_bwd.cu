// fm_bwd.cu — K4: FlashMask backward main kernel (Alg. 2) for sm_100a.
//
// Column-parallel: one CTA owns key tile j (128 keys) of one (batch, head),
// keeps dK_j and dV_j as fp32 accumulators in TMEM for the whole row loop and writes them
// once at the end (atomic-free).  The four mask values of its 128 keys are loaded once into
// registers — thread = key = TMEM lane in the transposed S^T layout (Alg. 2 lines 10-11,
// P:394-395).  Row tiles that are SKIP for this column tile are never loaded (Alg. 2 lines
// 13-18).
//
// Row tile Br = 64 (d = 128) or 128 (d = 64).  Per visited row tile i:
//   S^T  = K_j Q_i^T,  dP^T = V_j dO_i^T      (tcgen05, M = 128 keys)
//   P^T  = exp2(S^T*scale*log2e - L2_i), interval mask on PARTIAL tiles only
//   dS^T = P^T o (dP^T - D_i)
//   dV  += P^T dO_i,  dK += dS^T Q_i         (A operands bf16 from TMEM)
//   d=128: dQ_i^T = K_j^T dS^T (M = d);  d=64: dQ_i = dS K_j (M = queries)
// dQ tiles are added into the fp32 workspace by bulk / TMA reduce-adds from shared-memory stages
// (no read-modify-write).
//
// Pipelining: the compute WGs copy S^T/dP^T of row tile t into registers and release them at
// once, so the MMA warp issues S^T/dP^T of tile t+1 while P/dS of tile t are being computed;
// P and dS live in their own TMEM columns, which the dQ GEMM of the same tile then reuses.
// TMEM columns:
//   d=128: S [0,64) dP [64,128) P [128,160) dS [160,192) (dQ^T aliases [128,192)) K_j [192,256)
//          dV [256,384) dK [384,512)
//   d=64 : S [0,128) dP [128,256) P [256,320) dS [320,384) (dQ aliases [256,320))
//          dV [384,448) dK [448,512)
// Warp roles: 0-7 two compute WGs (query halves), 8-11 dQ WG (TMEM -> shared-memory stage ->
// bulk reduce-add), 12 TMA producer, 13 TMEM allocator + S/dP MMA issuer, 14 dV/dK/dQ issuer.
#include <cuda_bf16.h>
#include <cmath>

#include "fm_internal.h"
#include "fm_ptx.cuh"

#ifdef FM_TRACE
namespace fm { __device__ long long g_fm_trace[64 * 16]; __device__ long long g_fm_trace2[64 * 16]; }
#define FM_T(slot, t)                                                                        \
  do {                                                                                        \
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (t) < 64) fm::g_fm_trace[(t) * 16 + (slot)] = clock64(); \
  } while (0)
#else
#define FM_T(slot, t) \
  do {                \
  } while (0)
#endif

namespace fm {

namespace bwd {

constexpr int G_WARP = 14;  // warp issuing dV/dK/dQ (warp 13 issues S^T/dP^T)
constexpr int NT = (G_WARP + 1) * 32;
constexpr int DQ_NSTAGE = 2;  // dQ^T staging buffers (d=128), DQ_CROWS query rows each
constexpr int DQ_CROWS = 32;  // query rows per dQ^T staging chunk: two bulk reduce-adds per row tile
constexpr int kMaxTrb = 4096;  // d=128 (Br=64); d=64 (Br=128) uses half: the same max N
// d=64 dQ reduction: the dQ warpgroup stages the 128-row x 32-column fp32 half tiles (16 KiB,
// 128-byte swizzle) for one TMA tensor reduce-add each, DQ64_NBUF in flight — two operations per
// row tile (the cost of the reduction follows the number of operations).
constexpr int DQ64_NBUF = 3;
constexpr int DQ64_STAGES = DQ64_NBUF;
constexpr int DQ64_STAGE_FLOATS = kDq64BoxRows * 32;

template <int D>
struct Cfg {
  static constexpr int BR = (D == 128) ? 64 : 128;
  static constexpr bool DQT = (D == 128);          // dQ computed transposed (M = d)
  // K_j in TMEM as S^T's A operand: an SS MMA with N = 64 is bound by shared-memory operand
  // bandwidth (A 4 KiB + B 2 KiB per 48 clk), a TS one runs at the full 32 clk
  // (scripts/bwdmix_bench.cu).  Its 64 columns come from letting dQ^T share the P/dS columns.
  static constexpr bool KA_TMEM = (D == 128);
  // d=128: two P/dS column buffers, so the compute WGs write P/dS(t+1) while dV/dK/dQ(t) still
  // read buffer t; dQ^T(t) reuses the 64 columns of its own buffer (written after dV/dK(t)).
  static constexpr int NB = (D == 128 && !KA_TMEM) ? 2 : 1;
  static constexpr bool DQ_ALIAS = (D == 64) || KA_TMEM || NB == 2;  // dQ shares the P/dS columns
  static constexpr int KV_TILE = 128 * D * 2;      // bytes
  static constexpr int Q_TILE = BR * D * 2;
  static constexpr int DS_BYTES = 128 * BR * 2;
  static constexpr int CH_PER_WG = BR / 64;        // 32-query chunks per compute WG
  static constexpr int S_COL = 0, DP_COL = BR, P_COL = 2 * BR, DS_COL = 2 * BR + BR / 2;
  static constexpr int DQ_COL = DQ_ALIAS ? P_COL : 192;
  static constexpr int BUF_STRIDE = BR;  // column offset of P/dS/dQ buffer 1 (NB == 2)
  // (dK += dS^T Q with dS^T read from the dQ GEMM's shared-memory buffer (SS) instead of TMEM was
  // measured ~2 % slower: shared-memory bandwidth)
  static constexpr bool DK_SS = false;
  static constexpr int KA_COL = 192;
  static constexpr int DV_COL = (D == 128) ? 256 : 384;
  static constexpr int DK_COL = DV_COL + D;
  static constexpr int MAXTRB = (D == 128) ? kMaxTrb : kMaxTrb / 2;
  // per-head-dim ring depths: Q/dO stages and dS shared-memory buffers
  static constexpr int QST = 3;  // Q/dO ring (2 stages measured -6 %)
  static constexpr int NDS = 1;  // dS shared-memory buffers: one frees room for the dQ stages
};

template <int D, bool ROWW>
struct Smem {
  using C = Cfg<D>;
  uint8_t k[C::KV_TILE];
  uint8_t v[C::KV_TILE];
  uint8_t q[C::QST][C::Q_TILE];
  uint8_t dO[C::QST][C::Q_TILE];
  uint8_t ds[C::NDS][C::DS_BYTES];  // NDS = 1: dS(t+1) waits for dQ(t) to finish reading (frees room for dQ stages)
  // d=128: dQ^T staged 16 query rows (8 KiB, contiguous in dQacc) at a time for one bulk
  // reduce-add each, double-buffered
  float dq_stage[C::DQT ? DQ_NSTAGE : DQ64_STAGES][C::DQT ? DQ_CROWS * D : DQ64_STAGE_FLOATS];
  float lvec[C::QST][C::BR];
  float dvec[C::QST][C::BR];
  int4 rvec[C::QST][ROWW ? C::BR : 1];  // row-wise: the row tile's (LTS, len, UTS, len) per query row
  uint16_t list[C::MAXTRB];
  uint32_t part_bits[C::MAXTRB / 32];
  uint64_t kv_full;
  uint64_t q_full[C::QST], q_empty[C::QST];
  uint64_t s_full, sdp_free, p_full[2], pds_free[2], dq_full[2], dq_empty[2], ds_empty[2], done;
  uint32_t tmem_base;
  int n_entries;
  int warp_cnt[NT / 32];
};

// P^T / dS^T for one 32-query chunk of one key (Alg. 2 lines 20-25):
//   p = exp2(S*scale*log2e - L2_r) (masked to 0 on PARTIAL tiles), ds = p * (dP - D_r)
// Branch-free per template so the compiler can overlap the shared loads, FMAs and MUFU ops.
// Rows [r0, r0 + 32) masked for this thread's key, as a bit set (bit u = row r0 + u): the
// interval test of Alg. 2 lines 20-23 evaluated once per 32 rows instead of per element.
// lo in (-N, N], 0 <= len <= INT_MAX.  W32: 32-bit only — lo + len is formed only when it stays below
// 32 (at d = 64 the 64-bit form kept a sign word live across the compute loop, spilled to local
// memory: in-process A/B +4 % on PARTIAL-heavy d = 64 backwards; at d = 128 the 64-bit form measured
// 1-3 % faster, code generation)
template <bool W32>
__device__ __forceinline__ uint32_t range_bits(int lo, int len) {
  const int a = min(max(lo, 0), 32);
  if constexpr (W32) {
    const int b = (len >= 32 - lo) ? 32 : max(lo + len, 0);
    const uint32_t mb = (b >= 32) ? 0xFFFFFFFFu : ((1u << b) - 1u);
    const uint32_t ma = (a >= 32) ? 0xFFFFFFFFu : ((1u << a) - 1u);
    return mb & ~ma;  // bits [a, b); empty when b <= a
  } else {
    const int b = static_cast<int>(min(max(static_cast<long long>(lo) + len, 0ll), 32ll));
    return b > a ? static_cast<uint32_t>(((1ull << b) - 1ull) & ~((1ull << a) - 1ull)) : 0u;
  }
}
template <bool CAUSAL, bool W32>
__device__ __forceinline__ uint32_t row_mask_bits(int r0, int key, int4 mv) {
  uint32_t m = range_bits<W32>(mv.x - r0, mv.y);
  if constexpr (CAUSAL)
    m |= range_bits<W32>(0, key - r0);  // rows r < key
  else
    m |= range_bits<W32>(mv.z - r0, mv.w);
  return m;
}

// Row-wise representation (R32): bit u set iff query row r0 + u masks this thread's key — one of
// the row's key intervals holds it, it lies after the row (causal) or it is a padded key (>= N).
template <bool CAUSAL>
__device__ __forceinline__ uint32_t row_mask_bits_rw(int r0, int key, const int4* rv, int N) {
  uint32_t m = 0u;
#pragma unroll 8
  for (int u = 0; u < 32; ++u) {
    const int4 iv = rv[u];  // the same row for every thread of the warp: broadcast
    bool msk = (static_cast<unsigned>(key - iv.x) < static_cast<unsigned>(iv.y)) ||
               (static_cast<unsigned>(key - iv.z) < static_cast<unsigned>(iv.w));
    if constexpr (CAUSAL) msk |= r0 + u < key;
    m |= static_cast<uint32_t>(msk) << u;
  }
  return key >= N ? 0xFFFFFFFFu : m;
}

// lq = -l2 and dq = -D of the chunk's 32 queries (K3 stores them negated).  PACKED (d = 64, where
// the compute warpgroups are the critical resource): the argument
// S*scale*log2e - l2, dP - D and P*(dP - D) as packed FFMA2 / FADD2 / FMUL2 per query pair
// (backward +2..+5 % at d = 64; neutral within noise at d = 128, which keeps the scalar form).
template <bool PART, bool CAUSAL, bool F16, bool PACKED>
__device__ __forceinline__ void pds_chunk(const uint32_t* sr, const uint32_t* dr, const float* lq, const float* dq,
                                          float sl2, uint32_t mb, uint32_t* pp, uint32_t* dp) {
  if constexpr (!PACKED) {
#pragma unroll
    for (int c = 0; c < 32; c += 4) {
      const float4 L4 = *reinterpret_cast<const float4*>(lq + c);
      const float4 D4 = *reinterpret_cast<const float4*>(dq + c);
      const float l4[4] = {L4.x, L4.y, L4.z, L4.w};
      const float d4[4] = {D4.x, D4.y, D4.z, D4.w};
      float p[4], ds[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        p[u] = ex2(fmaf(__uint_as_float(sr[c + u]), sl2, l4[u]));
        if constexpr (PART) p[u] = ((mb >> (c + u)) & 1u) ? 0.f : p[u];
        ds[u] = p[u] * (__uint_as_float(dr[c + u]) + d4[u]);
      }
      pp[c / 2] = pack16<F16>(p[0], p[1]);
      pp[c / 2 + 1] = pack16<F16>(p[2], p[3]);
      dp[c / 2] = pack16<F16>(ds[0], ds[1]);
      dp[c / 2 + 1] = pack16<F16>(ds[2], ds[3]);
    }
    return;
  }
  const uint64_t sl2x2 = f2pack(sl2, sl2);
#pragma unroll
  for (int c = 0; c < 32; c += 4) {
    const float4 L4 = *reinterpret_cast<const float4*>(lq + c);
    const float4 D4 = *reinterpret_cast<const float4*>(dq + c);
    float x[4], p[4], ds[4];
    f2unpack(f2fma(f2pack(__uint_as_float(sr[c]), __uint_as_float(sr[c + 1])), sl2x2, f2pack(L4.x, L4.y)), x[0], x[1]);
    f2unpack(f2fma(f2pack(__uint_as_float(sr[c + 2]), __uint_as_float(sr[c + 3])), sl2x2, f2pack(L4.z, L4.w)), x[2],
             x[3]);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      p[u] = ex2(x[u]);
      if constexpr (PART) p[u] = ((mb >> (c + u)) & 1u) ? 0.f : p[u];
    }
    const uint64_t d01 = f2add(f2pack(__uint_as_float(dr[c]), __uint_as_float(dr[c + 1])), f2pack(D4.x, D4.y));
    const uint64_t d23 = f2add(f2pack(__uint_as_float(dr[c + 2]), __uint_as_float(dr[c + 3])), f2pack(D4.z, D4.w));
    f2unpack(f2mul(f2pack(p[0], p[1]), d01), ds[0], ds[1]);
    f2unpack(f2mul(f2pack(p[2], p[3]), d23), ds[2], ds[3]);
    pp[c / 2] = pack16<F16>(p[0], p[1]);
    pp[c / 2 + 1] = pack16<F16>(p[2], p[3]);
    dp[c / 2] = pack16<F16>(ds[0], ds[1]);
    dp[c / 2 + 1] = pack16<F16>(ds[2], ds[3]);
  }
}

}  // namespace bwd

// ROWW: row-wise representation (FM_FLAG_ROWWISE, R32): the producer loads each visited row tile's
// per-row key intervals next to L and D; the compute threads (= keys) test them per 32 rows.
template <int D, bool CAUSAL, bool OUT_F32, bool F16, bool ROWW>
__global__ void __launch_bounds__(bwd::NT, 1)
    fm_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                  const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO,
                  const __grid_constant__ CUtensorMap tmDQ, const __grid_constant__ CUtensorMap tmDK,
                  const __grid_constant__ CUtensorMap tmDV, const BwdArgs a) {
  using namespace bwd;
  using C = Cfg<D>;
  using S = Smem<D, ROWW>;
  constexpr int BR = C::BR;
  extern __shared__ uint8_t smem_raw[];
  S& sm = *smem_align1024<S>(smem_raw);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int b = blockIdx.z;
  // unit: key tile j of key/value head hk (its G query heads are looped over).  Split-G (MQA / GQA
  // grids under one wave): blockIdx.y = hk * gsplit + slice; the CTA takes the slice's G / gsplit
  // query heads of the group and writes fp32 dK / dV partials (K7 sums them).
  const int gsplit = a.gsplit > 1 ? a.gsplit : 1;
  const int slice = static_cast<int>(blockIdx.y) % gsplit;
  const int j = static_cast<int>(blockIdx.x);
  const int hk = static_cast<int>(blockIdx.y) / gsplit;
  const int hm = (a.Hm == 1) ? 0 : hk;
  const size_t bhm = static_cast<size_t>(b) * a.Hm + hm;
  const int Gs = a.G / (a.gsplit > 1 ? a.gsplit : 1);  // query heads of this CTA (all G unless split)

  if (warp == 12 && lane == 0) {
    mbar_init(&sm.kv_full, 1);
    for (int s = 0; s < C::QST; ++s) { mbar_init(&sm.q_full[s], 1); mbar_init(&sm.q_empty[s], 1); }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.sdp_free, 256);
    for (int bb = 0; bb < 2; ++bb) {
      mbar_init(&sm.p_full[bb], 256);
      mbar_init(&sm.pds_free[bb], 1);
      mbar_init(&sm.dq_full[bb], 1);
      mbar_init(&sm.dq_empty[bb], 128);
    }
    mbar_init(&sm.ds_empty[0], 1);
    mbar_init(&sm.ds_empty[1], 1);
    mbar_init(&sm.done, 1);
    fence_barrier_init();
    // K_j, V_j do not depend on the visit list: start their loads before it is built
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
    mbar_expect_tx(&sm.kv_full, 2 * C::KV_TILE);
#pragma unroll
    for (int c = 0; c < D / 64; ++c) {
      tma_load_4d(sm.k + c * 16384, &tmK, &sm.kv_full, c * 64, hk, j * 128, b);
      tma_load_4d(sm.v + c * 16384, &tmV, &sm.kv_full, c * 64, hk, j * 128, b);
    }
  }
  if (warp == 13) tmem_alloc<512>(&sm.tmem_base);

  // ---- visit list: row tiles i that are not SKIP for column tile j (K1 transposed map) ----
  {
    const uint8_t* col = a.bmap + (bhm * a.Tc + j) * a.Trb;
    int base = 0;
    // PARTIAL bit per visit-list entry: zeroed here, set below (ordered by the loop's first barrier)
    for (int w = tid; w < C::MAXTRB / 32; w += NT) sm.part_bits[w] = 0u;
    for (int i0 = 0; i0 < a.Trb; i0 += NT) {
      const int i = i0 + tid;
      const uint32_t c = (i < a.Trb) ? col[i] : 0u;
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
      if (vis) {
        sm.list[off] = static_cast<uint16_t>(i);
        if (c == 1u) atomicOr(&sm.part_bits[off >> 5], 1u << (off & 31));
      }
      base += tot;
      __syncthreads();
    }
    if (tid == 0) sm.n_entries = base;
  }
  // The class map came from K1b, two launches back (complete, see pdl_wait in fm_ptx.cuh);
  // D, L2 and the zeroed dQ accumulator come from K3, the stream predecessor.
  pdl_wait();
  pdl_launch();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // work items t = (query head of the group, visited row tile): t / nE1 selects the head
  const int nE1 = sm.n_entries;
  const int nE = nE1 * Gs;
  const int hq0 = hk * a.G + slice * Gs;  // first query head of this CTA
  const uint32_t tbase = sm.tmem_base;

  if (warp == 12) {
    // ================================ TMA producer ================================
    if (lane == 0 && nE == 0) mbar_wait(&sm.kv_full, 0);  // K/V must land before the CTA exits
    if (lane == 0 && nE > 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmdO);
      // t = g * nE1 + t1 walked with counters (a runtime division per item measured ~3 % of
      // the backward's stall samples)
      for (int t = 0, t1 = 0, g = 0; t < nE; ++t, (++t1 == nE1) ? (t1 = 0, ++g) : 0) {
        const int i = sm.list[t1];
        const int hq = hq0 + g;
        const size_t bh = static_cast<size_t>(b) * a.H + hq;
        const int st = t % C::QST;
        mbar_wait(&sm.q_empty[st], ((t / C::QST) & 1) ^ 1);
        mbar_expect_tx(&sm.q_full[st], 2 * C::Q_TILE + 2 * BR * 4 + (ROWW ? BR * 16 : 0));
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tma_load_4d(sm.q[st] + c * (BR * 128), &tmQ, &sm.q_full[st], c * 64, hq, i * BR, b);
          tma_load_4d(sm.dO[st] + c * (BR * 128), &tmdO, &sm.q_full[st], c * 64, hq, i * BR, b);
        }
        bulk_g2s(sm.lvec[st], a.l2 + bh * a.Npb + static_cast<size_t>(i) * BR, BR * 4, &sm.q_full[st]);
        bulk_g2s(sm.dvec[st], a.dvec + bh * a.Npb + static_cast<size_t>(i) * BR, BR * 4, &sm.q_full[st]);
        if constexpr (ROWW)
          bulk_g2s(sm.rvec[st], a.vec4 + bhm * static_cast<size_t>(a.Tc) * 128 + static_cast<size_t>(i) * BR,
                   BR * 16, &sm.q_full[st]);
      }
    }
  } else if (warp == 13 || warp == G_WARP) {
    // ============================ two MMA issuers ============================
    // The tensor core accepts only a few queued MMAs before an issuing thread blocks, so any
    // dependency wait in a single issuer starves it.  Warp 13 issues S^T/dP^T(t) as soon as the
    // compute WGs have released tile t-1; warp 14 issues dV/dK/dQ(t) once P/dS(t) are ready.
    // Each warp commits only to barriers that track its own MMAs.
    if (nE > 0) {  // the whole warp runs converged; one elected lane issues (fm_ptx.cuh)
      constexpr uint32_t ID_S = idesc16<F16>(128, BR, 0, 0);   // S^T, dP^T: A, B K-major
      constexpr uint32_t ID_G = idesc16<F16>(128, D, 0, 1);    // dV, dK: A in TMEM, B MN-major
      constexpr uint32_t ID_Q = idesc16<F16>(128, 64, 1, 1);   // dQ^T (d=128) / dQ (d=64), both MN-major
      const uint32_t k_addr = smem_u32(sm.k), v_addr = smem_u32(sm.v);
      mbar_wait_sleep(&sm.kv_full, 0);
      if (warp == 13) {
        if constexpr (C::KA_TMEM) {
          // K_j (SW128 K-major smem tile) -> TMEM columns [KA_COL, KA_COL + 64) by the tensor core:
          // k-step kk (16 d-values) of every key row lands in 8 columns, the A-operand layout of
          // the TS MMA below; ordered before it (same issuing thread).
          tc_fence_after();
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk)
            tmem_cp_128x256b_w(tbase + C::KA_COL + kk * 8,
                               sdesc_sw128(k_addr + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024));
        }
        for (int t = 0; t < nE; ++t) {
          const int st = t % C::QST;
          if (t > 0) mbar_wait_sleep(&sm.sdp_free, (t - 1) & 1);  // compute WGs hold S^T/dP^T(t-1) in registers          if (lane == 0) FM_T(1, t);
          mbar_wait_sleep(&sm.q_full[st], (t / C::QST) & 1);
          if (lane == 0) FM_T(14, t);
          tc_fence_after();
          const uint32_t q_addr = smem_u32(sm.q[st]), do_addr = smem_u32(sm.dO[st]);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t ao = (kk >> 2) * 16384 + (kk & 3) * 32;
            const uint32_t bo = (kk >> 2) * (BR * 128) + (kk & 3) * 32;
            if constexpr (C::KA_TMEM)
              mma_ts_w(tbase + C::S_COL, tbase + C::KA_COL + kk * 8, sdesc_sw128(q_addr + bo, 16, 1024), ID_S,
                     kk > 0 ? 1u : 0u);
            else
              mma_ss_w(tbase + C::S_COL, sdesc_sw128(k_addr + ao, 16, 1024), sdesc_sw128(q_addr + bo, 16, 1024), ID_S,
                     kk > 0 ? 1u : 0u);
            mma_ss_w(tbase + C::DP_COL, sdesc_sw128(v_addr + ao, 16, 1024), sdesc_sw128(do_addr + bo, 16, 1024), ID_S,
                   kk > 0 ? 1u : 0u);
          }
          mma_commit_w(&sm.s_full);
          if (lane == 0) FM_T(11, t);
        }
      } else {
        for (int t = 0; t < nE; ++t) {
          const int st = t % C::QST;
          if (lane == 0) FM_T(0, t);
          const int bi = t % C::NB;
          const uint32_t ph = (t / C::NB) & 1, boff = bi * C::BUF_STRIDE;
          mbar_wait_sleep(&sm.p_full[bi], ph);
          if (lane == 0) FM_T(2, t);
          tc_fence_after();
          const uint32_t q_addr = smem_u32(sm.q[st]), do_addr = smem_u32(sm.dO[st]);
#pragma unroll
          for (int kk = 0; kk < BR / 16; ++kk) {
            const uint32_t acc = (t > 0 || kk > 0) ? 1u : 0u;
            mma_ts_w(tbase + C::DV_COL, tbase + C::P_COL + boff + kk * 8,
                     sdesc_sw128(do_addr + kk * 2048, BR * 128, 1024), ID_G, acc);
            if constexpr (C::DK_SS)  // A = dS^T straight from the dQ operand buffer in smem
              mma_ss_w(tbase + C::DK_COL, sdesc_sw128(smem_u32(sm.ds[t % C::NDS]) + kk * 32, 16, 1024),
                       sdesc_sw128(q_addr + kk * 2048, BR * 128, 1024), ID_G, acc);
            else
              mma_ts_w(tbase + C::DK_COL, tbase + C::DS_COL + boff + kk * 8,
                       sdesc_sw128(q_addr + kk * 2048, BR * 128, 1024), ID_G, acc);
          }
          // S^T/dP^T(t) (warp 13) completed before the compute WGs produced P/dS(t)
          mma_commit_w(&sm.q_empty[st]);
          // pds_free is waited on only when dQ does not share the P/dS columns (else dq_empty
          // guards the buffer): commit it only then, so no mbarrier phase completes unobserved
          if (!(C::DQ_ALIAS && a.with_dq)) mma_commit_w(&sm.pds_free[bi]);
          if (lane == 0) FM_T(12, t);
          // dQ(t) overwrites the P/dS columns of buffer t % NB — issued after dV/dK(t) by this
          // thread (in order), and the compute WGs stored P/dS(t) there only after dQ(t-NB) was
          // read out (dq_empty[t % NB]).
          if (!a.with_dq) {
            if constexpr (C::DK_SS) mma_commit_w(&sm.ds_empty[t % C::NDS]);  // dK(t) read dS^T(t)
            continue;
          }
          if constexpr (!C::DQ_ALIAS) mbar_wait_sleep(&sm.dq_empty[0], (t & 1) ^ 1);          tc_fence_after();
          const uint32_t ds_addr = smem_u32(sm.ds[t % C::NDS]);
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            if constexpr (C::DQT)
              mma_ss_w(tbase + C::DQ_COL + boff, sdesc_sw128(k_addr + kk * 2048, 16384, 1024),
                     sdesc_sw128(ds_addr + kk * 2048, 16384, 1024), ID_Q, kk > 0 ? 1u : 0u);
            else
              mma_ss_w(tbase + C::DQ_COL + boff, sdesc_sw128(ds_addr + kk * 2048, 16384, 1024),
                     sdesc_sw128(k_addr + kk * 2048, 16384, 1024), ID_Q, kk > 0 ? 1u : 0u);
          }
          mma_commit_w(&sm.dq_full[bi]);
          mma_commit_w(&sm.ds_empty[t % C::NDS]);
          if (lane == 0) FM_T(13, t);
        }
        mma_commit_w(&sm.done);  // all S^T/dP^T completed earlier (they precede every p_full)
      }
    }
  } else if (warp < 8) {
    // ====================== compute WGs (thread = key, WG = query half) ======================
    const int wg = warp >> 2, wl = warp & 3;
    const int key_t = wl * 32 + lane;
    const int key = j * 128 + key_t;
    const uint32_t lane_off = static_cast<uint32_t>(wl * 32) << 16;
    // this key's (LTS, len, UTS, len), normalised (column-wise representation)
    const int4 mv = ROWW ? make_int4(0, 0, 0, 0) : a.vec4[(bhm * a.Tc) * 128 + key];
    const float sl2 = a.scale_log2;
    constexpr int CH = C::CH_PER_WG;
    for (int t = 0, t1 = 0; t < nE; ++t, t1 = (t1 + 1 == nE1) ? 0 : t1 + 1) {
      const int i = sm.list[t1];
      const bool partial = (sm.part_bits[t1 >> 5] >> (t1 & 31)) & 1u;
      const int st = t % C::QST;
      mbar_wait(&sm.q_full[st], (t / C::QST) & 1);
      mbar_wait(&sm.s_full, t & 1);
      if (tid == 0) FM_T(4, t);
#ifdef FM_TRACE
      if (lane == 0 && t >= 30 && t < 40 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        g_fm_trace2[(10 + t - 30) * 16 + warp] = clock64();
#endif
      tc_fence_after();
      const float* lv = sm.lvec[st];
      const float* dv = sm.dvec[st];
      uint32_t pp[CH][16], dp[CH][16];
#pragma unroll
      for (int ch = 0; ch < CH; ++ch) {
        const int q0 = (wg * CH + ch) * 32;  // first query of this chunk within the row tile
        uint32_t sr[32], dr[32];
        tmem_ld32(tbase + lane_off + C::S_COL + q0, sr);
        tmem_ld32(tbase + lane_off + C::DP_COL + q0, dr);
        tmem_wait_ld();
        if (ch == CH - 1) {
          tc_fence_before();
          mbar_arrive(&sm.sdp_free);
        }
        if (partial) {
          const uint32_t mb = ROWW ? row_mask_bits_rw<CAUSAL>(i * BR + q0, key, sm.rvec[st] + (ROWW ? q0 : 0), a.N)
                                   : row_mask_bits<CAUSAL, D == 64>(i * BR + q0, key, mv);
          pds_chunk<true, CAUSAL, F16, D == 64>(sr, dr, lv + q0, dv + q0, sl2, mb, pp[ch], dp[ch]);
        } else {
          pds_chunk<false, CAUSAL, F16, D == 64>(sr, dr, lv + q0, dv + q0, sl2, 0u, pp[ch], dp[ch]);
        }
      }
      if (tid == 0) FM_T(5, t);
#ifdef FM_TRACE
      if (lane == 0 && t >= 30 && t < 40 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        g_fm_trace2[(10 + t - 30) * 16 + 8 + warp] = clock64();
#endif
      // dS^T row of this key into the SW128 MN-major smem operand of the dQ GEMM
      // (first: it only needs dQ(t-1) to have finished reading the buffer)
      const bool ds_smem = a.with_dq || C::DK_SS;  // dS^T is a shared-memory operand (dQ, dK)
      if (ds_smem) mbar_wait(&sm.ds_empty[t % C::NDS], ((t / C::NDS) & 1) ^ 1);  // dK/dQ(t-2) have read this buffer
      if (tid == 0) FM_T(7, t);
#ifdef FM_TRACE
      if (lane == 0 && t >= 30 && t < 40 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        g_fm_trace2[(20 + t - 30) * 16 + 0 + warp] = clock64();
#endif
#pragma unroll
      for (int ch = 0; ch < (ds_smem ? CH : 0); ++ch) {
        const int q0 = (wg * CH + ch) * 32;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int g = (q0 >> 3) + u;  // 8-query group
          const int sub = g >> 3, gg = g & 7;
          uint8_t* dst = sm.ds[t % C::NDS] + sub * 16384 + key_t * 128 + ((gg ^ (key_t & 7)) << 4);
          *reinterpret_cast<uint4*>(dst) =
              make_uint4(dp[ch][4 * u], dp[ch][4 * u + 1], dp[ch][4 * u + 2], dp[ch][4 * u + 3]);
        }
      }
      if (tid == 0) FM_T(3, t);
#ifdef FM_TRACE
      if (lane == 0 && t >= 30 && t < 40 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        g_fm_trace2[(20 + t - 30) * 16 + 8 + warp] = clock64();
#endif
      // P / dS TMEM buffer t % NB free: dV/dK(t-NB) done, and dQ(t-NB), which reuses the
      // columns, read out
      const int bi = t % C::NB;
      const uint32_t ph = (t / C::NB) & 1, boff = bi * C::BUF_STRIDE;
      if (C::DQ_ALIAS && a.with_dq)
        mbar_wait(&sm.dq_empty[bi], ph ^ 1);
      else
        mbar_wait(&sm.pds_free[bi], ph ^ 1);
      if (tid == 0) FM_T(6, t);
#ifdef FM_TRACE
      if (lane == 0 && t >= 30 && t < 40 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        g_fm_trace2[(30 + t - 30) * 16 + 0 + warp] = clock64();
#endif
      tc_fence_after();
#pragma unroll
      for (int ch = 0; ch < CH; ++ch) {
        const int q0 = (wg * CH + ch) * 32;
        tmem_st16(tbase + lane_off + C::P_COL + boff + q0 / 2, pp[ch]);
        if constexpr (!C::DK_SS) tmem_st16(tbase + lane_off + C::DS_COL + boff + q0 / 2, dp[ch]);
      }
      fence_proxy_async_smem();
      tmem_wait_st();
      if (tid == 0) FM_T(15, t);
#ifdef FM_TRACE
      if (lane == 0 && t >= 30 && t < 40 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
        g_fm_trace2[(t - 30) * 16 + warp] = clock64();
#endif
      tc_fence_before();
      mbar_arrive(&sm.p_full[bi]);
      if (tid == 0) FM_T(8, t);
    }
    // ---- epilogue: dK_j = scale * dK, dV_j written once (Alg. 2 line 30) ----
    if (nE > 0) {
      mbar_wait(&sm.done, 0);
      tc_fence_after();
    }
    const size_t orow = ((static_cast<size_t>(b) * a.N + key) * a.Hkv + hk) * D;
    // WG0 writes dV, WG1 writes dK
    const uint32_t col = wg == 0 ? C::DV_COL : C::DK_COL;
    const float mul = wg == 0 ? 1.0f : a.scale;
    void* outp = wg == 0 ? a.dv : a.dk;
    if (gsplit > 1) {
      // split-G: this slice's unscaled fp32 partial, part[slice][dV | dK][b][key][hk][d]; K7 sums
      // the slices in order, scales dK and converts (deterministic, atomic-free)
      float* part = a.dkv_part + ((static_cast<size_t>(slice) * 2 + wg) * a.B * a.N) * a.Hkv * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        if (nE > 0) {
          tmem_ld32(tbase + lane_off + col + c * 32, r);
          tmem_wait_ld();
        }
        if (key < a.N) {
          float4* dst = reinterpret_cast<float4*>(part + orow + c * 32);
#pragma unroll
          for (int t = 0; t < 8; ++t)
            dst[t] = nE > 0 ? make_float4(__uint_as_float(r[4 * t]), __uint_as_float(r[4 * t + 1]),
                                          __uint_as_float(r[4 * t + 2]), __uint_as_float(r[4 * t + 3]))
                            : make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
    } else if constexpr (!OUT_F32) {
      // bf16 dV / dK go out through shared memory (the V / K tile buffers: every MMA that read
      // them completed before `done`) and TMA stores — a thread holds one key row, so direct
      // 16-byte stores would scatter each warp instruction over 32 rows.  Keys >= N are clipped.
      uint8_t* stg = wg == 0 ? sm.v : sm.k;
      mbar_wait(&sm.kv_full, 0);  // the K/V loads into these buffers have landed (even when nE == 0)
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t r[32];
        if (nE > 0) {
          tmem_ld32(tbase + lane_off + col + c * 32, r);
          tmem_wait_ld();
        }
        uint8_t* blk = stg + (c / 2) * (128 * 128) + key_t * 128;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          float f[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) f[u] = nE > 0 ? __uint_as_float(r[8 * t + u]) * mul : 0.f;
          const int chunk = (c % 2) * 4 + t;
          *reinterpret_cast<uint4*>(blk + ((chunk ^ (key_t & 7)) << 4)) =
              make_uint4(pack16<F16>(f[0], f[1]), pack16<F16>(f[2], f[3]), pack16<F16>(f[4], f[5]), pack16<F16>(f[6], f[7]));
        }
      }
      fence_proxy_async_smem();
      named_bar_sync(2 + wg, 128);
      if (wl == 0 && lane == 0) {
#pragma unroll
        for (int c = 0; c < D / 64; ++c)
          tma_store_4d(wg == 0 ? &tmDV : &tmDK, stg + c * (128 * 128), c * 64, hk, j * 128, b);
        bulk_commit();
        bulk_wait_read0();  // the staging buffer must outlive the TMA reads
      }
    }
#pragma unroll 1
    for (int c = 0; c < ((OUT_F32 && gsplit == 1) ? D / 32 : 0); ++c) {
      uint32_t r[32];
      if (nE > 0) {
        tmem_ld32(tbase + lane_off + col + c * 32, r);
        tmem_wait_ld();
      }
      float f[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) f[t] = nE > 0 ? __uint_as_float(r[t]) * mul : 0.f;
      if (key < a.N) {
        if constexpr (OUT_F32) {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(outp) + orow + c * 32);
#pragma unroll
          for (int t = 0; t < 8; ++t) dst[t] = make_float4(f[4 * t], f[4 * t + 1], f[4 * t + 2], f[4 * t + 3]);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(outp) + orow + c * 32);
#pragma unroll
          for (int t = 0; t < 4; ++t)
            dst[t] = make_uint4(pack16<F16>(f[8 * t], f[8 * t + 1]), pack16<F16>(f[8 * t + 2], f[8 * t + 3]),
                                pack16<F16>(f[8 * t + 4], f[8 * t + 5]), pack16<F16>(f[8 * t + 6], f[8 * t + 7]));
        }
      }
    }
  } else if (warp >= 8 && warp < 12) {
    // ================= dQ WG: TMEM -> registers -> red.global.add.f32 =================
    const int wl = warp - 8;
    const int t_id = wl * 32 + lane;  // TMEM lane: d index (d=128) or query (d=64)
    const uint32_t lane_off = static_cast<uint32_t>(wl * 32) << 16;
    uint32_t stage_n = 0;  // dQ staging chunks issued so far (DQT)
    for (int t = 0, t1 = 0, g = 0; t < (a.with_dq ? nE : 0); ++t, (++t1 == nE1) ? (t1 = 0, ++g) : 0) {
      const int i = sm.list[t1];
      const size_t bh = static_cast<size_t>(b) * a.H + hq0 + g;
      const int bi = C::DQ_ALIAS ? t % C::NB : 0;
      const uint32_t boff = bi * C::BUF_STRIDE;
      mbar_wait(&sm.dq_full[bi], (t / (C::DQ_ALIAS ? C::NB : 1)) & 1);
      if (t_id == 0) FM_T(9, t);
      tc_fence_after();
      uint32_t r[64];
      tmem_ld32(tbase + lane_off + C::DQ_COL + boff, r);
      tmem_ld32(tbase + lane_off + C::DQ_COL + boff + 32, r + 32);
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&sm.dq_empty[bi]);
      float* base = a.dqacc + (bh * a.Npb + static_cast<size_t>(i) * BR) * D;
      if constexpr (C::DQT) {
        // r[q] = dQ^T[d = t_id][q].  The 64 x 128 fp32 block is contiguous in dQacc: stage 16 rows
        // (8 KiB) in shared memory and add them with one bulk reduce (cp.reduce.async.bulk .add.f32)
        // — far fewer L2 transactions and LSU instructions than 64 scalar red.global per thread,
        // which were measured to starve the compute warps sharing the sub-partition.
#pragma unroll
        for (int c = 0; c < 64 / DQ_CROWS; ++c, ++stage_n) {
          float* stg = sm.dq_stage[stage_n % DQ_NSTAGE];
          if (stage_n >= DQ_NSTAGE) {  // the bulk reduce that read this buffer DQ_NSTAGE chunks ago is done
            if (t_id == 0) bulk_wait_read<DQ_NSTAGE - 1>();
            named_bar_sync(1, 128);
          }
#pragma unroll
          for (int q = 0; q < DQ_CROWS; ++q) stg[q * D + t_id] = __uint_as_float(r[c * DQ_CROWS + q]);
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (t_id == 0) {
            bulk_reduce_add_f32(base + c * DQ_CROWS * D, stg, DQ_CROWS * D * 4);
            bulk_commit();
          }
        }
      } else {
        // d=64: r[c] = dQ[query = t_id][c], t_id = 0..127 = the tile's rows.  Each 32-column half
        // of the 128 x 64 tile is written into a 128-byte-swizzled stage (16-B chunk c of row q at
        // c ^ (q & 7): conflict-free) and added by one TMA tensor reduce.
        const int row0 = static_cast<int>(bh * a.Npb) + i * BR;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch, ++stage_n) {
          float* stg = sm.dq_stage[stage_n % DQ64_NBUF];
          if (stage_n >= DQ64_NBUF) {  // the reduce that read this stage DQ64_NBUF operations ago is done
            if (t_id == 0) bulk_wait_read<DQ64_NBUF - 1>();
            named_bar_sync(1, 128);
          }
#pragma unroll
          for (int c = 0; c < 8; ++c)
            *reinterpret_cast<float4*>(reinterpret_cast<uint8_t*>(stg) + t_id * 128 + ((c ^ (t_id & 7)) << 4)) =
                make_float4(__uint_as_float(r[ch * 32 + 4 * c]), __uint_as_float(r[ch * 32 + 4 * c + 1]),
                            __uint_as_float(r[ch * 32 + 4 * c + 2]), __uint_as_float(r[ch * 32 + 4 * c + 3]));
          fence_proxy_async_smem();
          named_bar_sync(1, 128);
          if (t_id == 0) {
            tma_reduce_add_2d(&tmDQ, stg, ch * 32, row0);
            bulk_commit();
          }
        }
      }
      if (t_id == 0) FM_T(10, t);
    }
    if (t_id == 0) bulk_wait0();  // the staging buffers must outlive the bulk reads
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 13) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int D, bool CAUSAL, bool OUT_F32, bool F16, bool ROWW>
static cudaError_t launch_bwd_t(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                                const CUtensorMap& tdo, const CUtensorMap& tdq, const CUtensorMap& tdk,
                                const CUtensorMap& tdv, const BwdArgs& a, cudaStream_t st) {
  auto kern = fm_bwd_kernel<D, CAUSAL, OUT_F32, F16, ROWW>;
  const size_t smem = sizeof(bwd::Smem<D, ROWW>) + 1024;
  static_assert(sizeof(bwd::Smem<D, ROWW>) + 1024 <= 232448, "shared memory budget");
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(d.Tc, d.Hkv * (a.gsplit > 1 ? a.gsplit : 1), d.B);
  return launch_pdl(kern, grid, dim3(bwd::NT), smem, st, tq, tk, tv, tdo, tdq, tdk, tdv, a);
}

cudaError_t launch_bwd(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                       const CUtensorMap& tdo, const CUtensorMap& tdq, const CUtensorMap& tdk, const CUtensorMap& tdv,
                       const BwdArgs& a, cudaStream_t st) {
#define FM_B(DD, CC, FF)                                                                                     \
  do {                                                                                                       \
    if (d.rowwise)                                                                                           \
      return d.in_f16 ? launch_bwd_t<DD, CC, FF, true, true>(d, tq, tk, tv, tdo, tdq, tdk, tdv, a, st)       \
                      : launch_bwd_t<DD, CC, FF, false, true>(d, tq, tk, tv, tdo, tdq, tdk, tdv, a, st);     \
    return d.in_f16 ? launch_bwd_t<DD, CC, FF, true, false>(d, tq, tk, tv, tdo, tdq, tdk, tdv, a, st)        \
                    : launch_bwd_t<DD, CC, FF, false, false>(d, tq, tk, tv, tdo, tdq, tdk, tdv, a, st);      \
  } while (0)
  if (d.D == 128) {
    if (d.causal) { if (d.out_f32) FM_B(128, true, true); else FM_B(128, true, false); }
    else { if (d.out_f32) FM_B(128, false, true); else FM_B(128, false, false); }
  } else {
    if (d.causal) { if (d.out_f32) FM_B(64, true, true); else FM_B(64, true, false); }
    else { if (d.out_f32) FM_B(64, false, true); else FM_B(64, false, false); }
  }
#undef FM_B
}

}  // namespace fm

#ifdef FM_TRACE
extern "C" __attribute__((visibility("default"))) int flashmask_debug_trace(long long* host) {
  return cudaMemcpyFromSymbol(host, fm::g_fm_trace, sizeof(long long) * 64 * 16) == cudaSuccess ? 0 : 1;
}
extern "C" __attribute__((visibility("default"))) int flashmask_debug_trace2(long long* host) {
  return cudaMemcpyFromSymbol(host, fm::g_fm_trace2, sizeof(long long) * 64 * 16) == cudaSuccess ? 0 : 1;
}
#endif
