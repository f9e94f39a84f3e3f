// fm_dq.cu — K6: deterministic dQ (the "deterministic control" of P:300).
//
// Row-parallel recomputation: one CTA owns a 128-row query tile i of one (batch, query head)
// and walks the non-SKIP key tiles j of its row of the K1 class map in ascending j:
//   S  = Q_i K_j^T,  dP = dO_i V_j^T             (tcgen05, M = 128 queries, N = 128 keys)
//   P  = exp2(S*scale*log2e - L2_i)  (interval mask on PARTIAL tiles only, Alg. 2 l.15-21)
//   dS = P o (dP - D_i)                          (Alg. 2 line 25)
//   dQ += dS K_j                                 (A = bf16 dS from TMEM, fp32 accumulator in TMEM)
// dQ never leaves the CTA until the end, so its summation order is fixed and the result is
// bitwise reproducible; with FM_FLAG_DETERMINISTIC the backward kernel skips its dQ GEMM and
// fp32 reductions and this kernel writes dq = scale * dQ directly.  Costs two extra GEMMs
// (S, dP) per visited tile.
// Warps: 0-7 two compute WGs (column halves, thread = row), 8 TMA producer, 9 TMEM + MMA.
// TMEM: S [0,128) dP [128,256) dS [256,320) dQ [320, 320+d).
#include <cuda_bf16.h>
#include <cmath>

#include "fm_internal.h"
#include "fm_ptx.cuh"

namespace fm {

namespace dqk {

constexpr int NT = 320;
constexpr int KST = 2;

template <int D>
struct Smem {
  static constexpr int TILE = 128 * D * 2;
  uint8_t q[TILE];
  uint8_t dO[TILE];
  uint8_t k[KST][TILE];
  uint8_t v[KST][TILE];
  int4 mask[KST][128];
  uint16_t list[kMaxTc];
  uint32_t part_bits[kMaxTc / 32];
  uint64_t bar_q, kv_full[KST], kv_empty[KST], s_full, sdp_free, ds_full, ds_free, done;
  uint32_t tmem_base;
  int n_entries;
  int warp_cnt[NT / 32];
};

}  // namespace dqk

template <int D, bool CAUSAL, bool OUT_F32, bool F16>
__global__ void __launch_bounds__(dqk::NT, 1)
    fm_dq_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                 const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmdO, const DqArgs a) {
  using namespace dqk;
  using S = Smem<D>;
  extern __shared__ uint8_t smem_raw[];
  S& sm = *smem_align1024<S>(smem_raw);
  constexpr int S_COL = 0, DP_COL = 128, DS_COL = 256, DQ_COL = 320;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int i = static_cast<int>(a.Tr - 1 - blockIdx.x);  // heaviest row tiles first for causal masks
  const int h = blockIdx.y, b = blockIdx.z;
  const int hk = h / a.G;
  const int hm = (a.Hm == 1) ? 0 : hk;
  const size_t bhm = static_cast<size_t>(b) * a.Hm + hm;
  const size_t bh = static_cast<size_t>(b) * a.H + h;

  if (warp == 8 && lane == 0) {
    mbar_init(&sm.bar_q, 1);
    for (int s = 0; s < KST; ++s) { mbar_init(&sm.kv_full[s], 1); mbar_init(&sm.kv_empty[s], 1); }
    mbar_init(&sm.s_full, 1);
    mbar_init(&sm.sdp_free, 256);
    mbar_init(&sm.ds_full, 256);
    mbar_init(&sm.ds_free, 1);
    mbar_init(&sm.done, 1);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<512>(&sm.tmem_base);

  // ---- visit list: key tiles j that are not SKIP for row tile i (K1 forward map), ascending ----
  {
    const uint8_t* row = a.fmap + (bhm * a.Tr + i) * a.Tc;
    int base = 0;
    // PARTIAL bit per visit-list entry: zeroed here, set below (ordered by the loop's first barrier)
    for (int w = tid; w < kMaxTc / 32; w += NT) sm.part_bits[w] = 0u;
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
      if (vis) {
        sm.list[off] = static_cast<uint16_t>(j);
        if (c == 1u) atomicOr(&sm.part_bits[off >> 5], 1u << (off & 31));
      }
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

  if (warp == 8) {
    // ================================ TMA producer ================================
    if (lane == 0 && nE > 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmdO);
      mbar_expect_tx(&sm.bar_q, 2 * S::TILE);
#pragma unroll
      for (int c = 0; c < D / 64; ++c) {
        tma_load_4d(sm.q + c * 16384, &tmQ, &sm.bar_q, c * 64, h, i * 128, b);
        tma_load_4d(sm.dO + c * 16384, &tmdO, &sm.bar_q, c * 64, h, i * 128, b);
      }
      const int4* vec_bh = a.vec4 + bhm * static_cast<size_t>(a.Tc) * 128;
      for (int e = 0; e < nE; ++e) {
        const int j = sm.list[e];
        const int ks = e % KST;
        mbar_wait(&sm.kv_empty[ks], ((e / KST) & 1) ^ 1);
        const bool part = ((sm.part_bits[e >> 5] >> (e & 31)) & 1u) && !a.rowwise;  // row-wise: no column slice
        mbar_expect_tx(&sm.kv_full[ks], 2 * S::TILE + (part ? 128 * 16 : 0));
#pragma unroll
        for (int c = 0; c < D / 64; ++c) {
          tma_load_4d(sm.k[ks] + c * 16384, &tmK, &sm.kv_full[ks], c * 64, hk, j * 128, b);
          tma_load_4d(sm.v[ks] + c * 16384, &tmV, &sm.kv_full[ks], c * 64, hk, j * 128, b);
        }
        if (part) bulk_g2s(sm.mask[ks], vec_bh + static_cast<size_t>(j) * 128, 128 * 16, &sm.kv_full[ks]);
      }
    }
  } else if (warp == 9) {
    // ================================ MMA issuer ================================
    if (nE > 0) {  // converged warp, one elected lane issues
      constexpr uint32_t ID_S = idesc16<F16>(128, 128, 0, 0);  // S, dP: A, B K-major
      constexpr uint32_t ID_Q = idesc16<F16>(128, D, 0, 1);    // dQ: A = dS in TMEM, B = K MN-major
      const uint32_t q_addr = smem_u32(sm.q), do_addr = smem_u32(sm.dO);
      mbar_wait(&sm.bar_q, 0);
      for (int e = 0; e < nE; ++e) {
        const int ks = e % KST;
        mbar_wait(&sm.kv_full[ks], (e / KST) & 1);
        if (e > 0) mbar_wait(&sm.sdp_free, (e - 1) & 1);  // compute WGs hold S/dP(e-1) in registers
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sm.k[ks]), v_addr = smem_u32(sm.v[ks]);
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss_w(tbase + S_COL, sdesc_sw128(q_addr + off, 16, 1024), sdesc_sw128(k_addr + off, 16, 1024), ID_S,
                 kk > 0 ? 1u : 0u);
          mma_ss_w(tbase + DP_COL, sdesc_sw128(do_addr + off, 16, 1024), sdesc_sw128(v_addr + off, 16, 1024), ID_S,
                 kk > 0 ? 1u : 0u);
        }
        mma_commit_w(&sm.s_full);
        mbar_wait(&sm.ds_full, e & 1);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts_w(tbase + DQ_COL, tbase + DS_COL + kk * 8, sdesc_sw128(k_addr + kk * 2048, 16384, 1024), ID_Q,
                 (e > 0 || kk > 0) ? 1u : 0u);
        mma_commit_w(&sm.ds_free);
        mma_commit_w(&sm.kv_empty[ks]);
      }
      mma_commit_w(&sm.done);
    }
  } else {
    // ====================== compute WGs (thread = query row, WG = 64-key half) ======================
    const int hh = warp >> 2, wl = warp & 3;
    const int row_t = wl * 32 + lane;
    const int row = i * 128 + row_t;
    const uint32_t lane_off = static_cast<uint32_t>(wl * 32) << 16;
    const float sl2 = a.scale_log2;
    const size_t ri = bh * a.Npb + row;  // Npb >= Tr * 128 rows, so this index is in range
    const float nl2 = a.l2[ri], ndval = a.dvec[ri];  // -lse*log2e and -D (K3 stores them negated)
    // row-wise representation (R32): this row's (LTS, len, UTS, len) over key columns
    const int4 rmv = a.rowwise ? a.vec4[bhm * static_cast<size_t>(a.Tc) * 128 + row] : make_int4(0, 0, 0, 0);
    for (int e = 0; e < nE; ++e) {
      const int j = sm.list[e];
      const int ks = e % KST;
      const bool part = (sm.part_bits[e >> 5] >> (e & 31)) & 1u;
      mbar_wait(&sm.kv_full[ks], (e / KST) & 1);  // mask slice visibility
      mbar_wait(&sm.s_full, e & 1);
      tc_fence_after();
      uint32_t sr[2][32], dr[2][32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        tmem_ld32(tbase + lane_off + S_COL + hh * 64 + c * 32, sr[c]);
        tmem_ld32(tbase + lane_off + DP_COL + hh * 64 + c * 32, dr[c]);
      }
      tmem_wait_ld();
      tc_fence_before();
      mbar_arrive(&sm.sdp_free);
      uint32_t pk[32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
#pragma unroll
        for (int t = 0; t < 32; t += 2) {
          float ds2[2];
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            float p = ex2(fmaf(__uint_as_float(sr[c][t + u]), sl2, nl2));
            if (part) {
              const int col = hh * 64 + c * 32 + t + u;
              bool msk;
              if (a.rowwise) {  // this row's key intervals (R32); keys past N are padding
                const int y = j * 128 + col;
                msk = (static_cast<unsigned>(y - rmv.x) < static_cast<unsigned>(rmv.y)) ||
                      (static_cast<unsigned>(y - rmv.z) < static_cast<unsigned>(rmv.w)) || y >= a.N;
                if constexpr (CAUSAL) msk |= row < y;
              } else {
                const int4 mv = sm.mask[ks][col];
                msk = static_cast<unsigned>(row - mv.x) < static_cast<unsigned>(mv.y);
                if constexpr (CAUSAL)
                  msk |= row < j * 128 + col;
                else
                  msk |= static_cast<unsigned>(row - mv.z) < static_cast<unsigned>(mv.w);
              }
              p = msk ? 0.f : p;
            }
            ds2[u] = p * (__uint_as_float(dr[c][t + u]) + ndval);
          }
          pk[c * 16 + t / 2] = pack16<F16>(ds2[0], ds2[1]);
        }
      }
      mbar_wait(&sm.ds_free, (e & 1) ^ 1);  // dQ(e-1) has read the dS columns
      tc_fence_after();
      tmem_st32(tbase + lane_off + DS_COL + hh * 32, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&sm.ds_full);
    }
    // ---- epilogue: dq = scale * dQ, this half's d/2 columns ----
    if (nE > 0) {
      mbar_wait(&sm.done, 0);
      tc_fence_after();
    }
    const size_t orow = ((static_cast<size_t>(b) * a.N + row) * a.H + h) * D + hh * (D / 2);
#pragma unroll 1
    for (int c = 0; c < D / 64; ++c) {
      uint32_t r[32];
      if (nE > 0) {
        tmem_ld32(tbase + lane_off + DQ_COL + hh * (D / 2) + c * 32, r);
        tmem_wait_ld();
      }
      float f[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) f[t] = nE > 0 ? __uint_as_float(r[t]) * a.scale : 0.f;
      if (row < a.N) {
        if constexpr (OUT_F32) {
          float4* dst = reinterpret_cast<float4*>(static_cast<float*>(a.dq) + orow + c * 32);
#pragma unroll
          for (int t = 0; t < 8; ++t) dst[t] = make_float4(f[4 * t], f[4 * t + 1], f[4 * t + 2], f[4 * t + 3]);
        } else {
          uint4* dst = reinterpret_cast<uint4*>(static_cast<uint16_t*>(a.dq) + orow + c * 32);
#pragma unroll
          for (int t = 0; t < 4; ++t)
            dst[t] = make_uint4(pack16<F16>(f[8 * t], f[8 * t + 1]), pack16<F16>(f[8 * t + 2], f[8 * t + 3]),
                                pack16<F16>(f[8 * t + 4], f[8 * t + 5]), pack16<F16>(f[8 * t + 6], f[8 * t + 7]));
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) {
    tc_fence_after();
    tmem_dealloc<512>(tbase);
  }
}

template <int D, bool CAUSAL, bool OUT_F32, bool F16>
static cudaError_t launch_dq_t(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                               const CUtensorMap& tdo, const DqArgs& a, cudaStream_t st) {
  auto kern = fm_dq_kernel<D, CAUSAL, OUT_F32, F16>;
  const size_t smem = sizeof(dqk::Smem<D>) + 1024;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  if (e != cudaSuccess) return e;
  dim3 grid(d.Tr, d.H, d.B);
  kern<<<grid, dqk::NT, smem, st>>>(tq, tk, tv, tdo, a);
  return cudaGetLastError();
}

cudaError_t launch_dq(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                      const CUtensorMap& tdo, const DqArgs& a, cudaStream_t st) {
#define FM_Q(DD, CC, FF) \
  return d.in_f16 ? launch_dq_t<DD, CC, FF, true>(d, tq, tk, tv, tdo, a, st) \
                  : launch_dq_t<DD, CC, FF, false>(d, tq, tk, tv, tdo, a, st)
  if (d.D == 128) {
    if (d.causal) { if (d.out_f32) FM_Q(128, true, true); else FM_Q(128, true, false); }
    else { if (d.out_f32) FM_Q(128, false, true); else FM_Q(128, false, false); }
  } else {
    if (d.causal) { if (d.out_f32) FM_Q(64, true, true); else FM_Q(64, true, false); }
    else { if (d.out_f32) FM_Q(64, false, true); else FM_Q(64, false, false); }
  }
#undef FM_Q
}

}  // namespace fm
