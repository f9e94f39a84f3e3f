// fm_prep.cu — K1 (preprocessing + tile classification), K3 (backward preprocess) and
// K5 (dQ convert).  All three are integer / HBM-bound passes.
#include <cuda_bf16.h>
#include <climits>

#include "fm_internal.h"
#include "fm_ptx.cuh"

namespace fm {

// ---------------------------------------------------------------------------------------
// K1a: expand startend_row_indices with the C-table defaults (flashmask.h) and reduce the
// per-column-tile min/max of LTS, LTE, UTS, UTE (Alg. 1 lines 3-4).  Optionally
// also writes the per-column normalised interval vector used by the attention kernels:
// (LTS, LTE - LTS, UTS, UTE - UTS) after clamping to [0, N], empty intervals as (0, 0), so a
// row r is masked iff (unsigned)(r - start) < length for either interval; padded columns
// y >= N get the lower interval (0, INT_MAX) so that they are masked for every row.
// Grid (Tc, B*Hm), 128 threads; one CTA reduces one column tile.
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ void expand_col(const int32_t* s, int C, int causal, int N, int& lts, int& lte, int& uts,
                                           int& ute, int rowwise) {
  if (rowwise) {
    // row-wise C-table (R32): an implicit end extends to the far edge of its triangle
    if (causal) {
      lts = (C >= 2) ? s[0] : 0;
      lte = (C >= 2) ? s[1] : s[0];
      uts = 0;
      ute = 0;
    } else if (C == 2) {
      lts = 0;
      lte = s[0];
      uts = s[1];
      ute = N;
    } else {
      lts = s[0];
      lte = s[1];
      uts = s[2];
      ute = s[3];
    }
    return;
  }
  if (causal) {
    lts = s[0];
    lte = (C >= 2) ? s[1] : N;
    uts = 0;
    ute = 0;
  } else if (C == 2) {
    lts = s[0];
    lte = N;
    uts = 0;
    ute = s[1];
  } else {
    lts = s[0];
    lte = s[1];
    uts = s[2];
    ute = s[3];
  }
}

__device__ __forceinline__ int clampi(int x, int lo, int hi) { return x < lo ? lo : (x > hi ? hi : x); }

// C is a template parameter (1, 2, 4) so that a column's C values come in one 4/8/16-byte load and
// the column loop unrolls (several loads in flight per lane)
template <int C>
__global__ void __launch_bounds__(128) k1_expand(const int32_t* __restrict__ sri, int N, int causal, int bc,
                                                 int Tc, int32_t* __restrict__ ext8, int4* __restrict__ vec4,
                                                 int rowwise) {
  pdl_wait();
  pdl_launch();
  // one warp per column tile (4 per CTA): lanes stride over the tile's columns, the extrema
  // are reduced with warp shuffles only
  // (grid-stride over column tiles; the launch sizes the grid at one warp per column tile)
  const int lane = threadIdx.x & 31;
  const int bh = blockIdx.y;
  const int32_t* base = sri + static_cast<size_t>(bh) * N * C;
  for (int j = blockIdx.x * 4 + (threadIdx.x >> 5); j < Tc; j += gridDim.x * 4) {
    int mn[4] = {INT_MAX, INT_MAX, INT_MAX, INT_MAX};
    int mx[4] = {INT_MIN, INT_MIN, INT_MIN, INT_MIN};
    // four columns per lane per round, all four loads issued before any is used
    for (int cb = lane; cb < bc; cb += 128) {
      int raw[4][4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const long y = static_cast<long>(j) * bc + cb + 32 * k;
        raw[k][0] = raw[k][1] = raw[k][2] = raw[k][3] = 0;
        if (cb + 32 * k < bc && y < N) {
          if constexpr (C == 4) {
            const int4 t = __ldg(reinterpret_cast<const int4*>(base + y * 4));
            raw[k][0] = t.x; raw[k][1] = t.y; raw[k][2] = t.z; raw[k][3] = t.w;
          } else if constexpr (C == 2) {
            const int2 t = __ldg(reinterpret_cast<const int2*>(base + y * 2));
            raw[k][0] = t.x; raw[k][1] = t.y;
          } else {
            raw[k][0] = __ldg(base + y);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if (cb + 32 * k >= bc) break;
        const long y = static_cast<long>(j) * bc + cb + 32 * k;
        int4 nv;
        if (y < N) {
          int v[4];
          expand_col(raw[k], C, causal, N, v[0], v[1], v[2], v[3], rowwise);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            mn[t] = min(mn[t], v[t]);
            mx[t] = max(mx[t], v[t]);
          }
          int a = clampi(v[0], 0, N), b = clampi(v[1], 0, N), u = clampi(v[2], 0, N), w = clampi(v[3], 0, N);
          if (a >= b) a = b = 0;
          if (u >= w) u = w = 0;
          nv = make_int4(a, b - a, u, w - u);  // (start, length) per interval
        } else {
          nv = make_int4(0, INT_MAX, 0, 0);
        }
        if (vec4) vec4[static_cast<size_t>(bh) * Tc * bc + y] = nv;
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        mn[t] = min(mn[t], __shfl_xor_sync(0xffffffffu, mn[t], o));
        mx[t] = max(mx[t], __shfl_xor_sync(0xffffffffu, mx[t], o));
      }
    }
    if (lane < 8) {
      const int t = lane >> 1;
      int r = (lane & 1) ? mx[0] : mn[0];
#pragma unroll
      for (int k = 1; k < 4; ++k)
        if (t == k) r = (lane & 1) ? mx[k] : mn[k];
      ext8[(static_cast<size_t>(bh) * Tc + j) * 8 + lane] = r;
    }
  }
}

// ---------------------------------------------------------------------------------------
// K1b: Eq. 4 per tile with Alg. 1's tests, 0-based, real extents,
// causal region as a third triangle:
//   SKIP     iff (r0>=LTSmax && r1<=LTEmin) || (r0>=UTSmax && r1<=UTEmin) || (causal && r1-1<c0)
//   PARTIAL  iff (r1>LTSmin && r0<LTEmax)   || (r1>UTSmin && r0<UTEmax)   || (causal && r0<c1-1)
//   UNMASKED otherwise.
// kernel_map = 1 writes the map the attention kernels consume: SKIP -> PARTIAL under
// FM_FLAG_NO_SKIP, and a non-SKIP ragged last column tile -> PARTIAL (bounds mask).
// Counts always use the true classes: per (b, hm) the three class counts, and the
// number of non-SKIP tiles of every row tile and of every column tile — the per-unit work
// O((1-rho) T_r T_c) of P:262 that orders the attention kernels' units.
// Thread = JPT consecutive column tiles (extrema loaded once), looping over rows_per_cta row
// tiles; row map: one JPT-byte store per row; transposed map (JPT = 1): 16 consecutive row tiles
// of one column tile per 16-byte store.  Grid (ceil(Tc / (128 JPT)), ceil(Tr / rows_per_cta), B*Hm).
// ---------------------------------------------------------------------------------------
// 32-bit arithmetic: N <= 2^30 and br, bc are clamped to [1, N] on the host, so r0 < N + br
// and c0 < N + bc never overflow.
__device__ __forceinline__ int tile_class(const int4& a, const int4& b, int r0, int r1, int c0, int c1, int causal) {
  // branch-free (predicate logic only): the per-row loop of K1b is latency-bound on branches
  const bool s = ((r0 >= a.y) & (r1 <= a.z)) | ((r0 >= b.y) & (r1 <= b.z)) | ((causal != 0) & (r1 - 1 < c0));
  const bool p = ((r1 > a.x) & (r0 < a.w)) | ((r1 > b.x) & (r0 < b.w)) | ((causal != 0) & (r0 < c1 - 1));
  return s ? 0 : (p ? 1 : 2);
}

// Row-wise representation (R32): Eq. 4 on the transposed problem — the extrema are those of row
// tile i (key intervals of its rows), compared with the column range [c0, c1) of tile j; the
// causal triangle is unchanged.
__device__ __forceinline__ int tile_class_rw(const int4& a, const int4& b, int r0, int r1, int c0, int c1, int causal) {
  if ((c0 >= a.y && c1 <= a.z) || (c0 >= b.y && c1 <= b.z) || (causal && r1 - 1 < c0)) return 0;
  if ((c1 > a.x && c0 < a.w) || (c1 > b.x && c0 < b.w) || (causal && r0 < c1 - 1)) return 1;
  return 2;
}

// Compile-time variants: TRANS = the backward's transposed map (JPT = 1, 16-row runs per 16-byte
// store); API = flashmask_classify (true classes, counts; NS adds the a2 per-row / per-column
// non-SKIP counts) — otherwise the attention kernels' map (FM_FLAG_NO_SKIP, ragged last column
// tile PARTIAL) without counts.  Keeping every choice out of the row loop, four column tiles per
// thread and one 32-bit store per row took the Hm = 64 microbenchmark from 165 to 85 us.
#ifndef FM_K1_THREADS
#define FM_K1_THREADS 32
#endif
#ifndef FM_K1_MINB
#define FM_K1_MINB 24
#endif
#ifndef FM_K1_KB
#define FM_K1_KB 16
#endif
template <int JPT, bool ROWW, bool TRANS, bool API, bool NS>
__global__ void __launch_bounds__(FM_K1_THREADS, FM_K1_MINB) k1_classify(const int32_t* __restrict__ ext8, int N, int causal, int br, int bc,
                                                   int Tr, int Tc, uint8_t* __restrict__ map, int kernel_map,
                                                   int no_skip, unsigned long long* __restrict__ counts,
                                                   int* __restrict__ row_cnt, int* __restrict__ col_cnt,
                                                   int rows_per_cta) {
  static_assert(!TRANS || JPT == 1, "transposed map: one column tile per thread");
  pdl_wait();
  pdl_launch();
  __shared__ unsigned int cnt[2];
  __shared__ int row_acc[64];
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * JPT;
  const int ib = blockIdx.y * rows_per_cta;
  const int iend = min(Tr, ib + rows_per_cta);
  const int bh = blockIdx.z;
  if (API) {
    if (threadIdx.x < 2) cnt[threadIdx.x] = 0;
    if (NS)
      for (int t = threadIdx.x; t < 64; t += blockDim.x) row_acc[t] = 0;
    __syncthreads();
  }
  int4 ea[JPT], eb[JPT];
  int c0[JPT], c1[JPT];
  bool valid[JPT];
  int nvalid = 0;
  uint32_t force1 = 0u;  // kernel map: per column-tile byte, class 2 -> 1 (ragged last column tile)
#pragma unroll
  for (int u = 0; u < JPT; ++u) {
    const int j = j0 + u;
    valid[u] = j < Tc;
    nvalid += valid[u];
    if (valid[u] && !ROWW) {
      const int4* e = reinterpret_cast<const int4*>(ext8 + (static_cast<size_t>(bh) * Tc + j) * 8);
      ea[u] = e[0];  // (LTSmin, LTSmax, LTEmin, LTEmax)
      eb[u] = e[1];  // (UTSmin, UTSmax, UTEmin, UTEmax)
    } else {
      ea[u] = eb[u] = make_int4(0, 0, 0, 0);  // row-wise: the extrema come per row tile
    }
    c0[u] = valid[u] ? j * bc : N;
    c1[u] = c0[u] + min(bc, N - c0[u]);
    if (!API && kernel_map == 2 && j == Tc - 1) force1 |= 1u << (8 * u);  // N is not a multiple of bc
  }
  // extrema of every lane of the warp, for the rows of non-uniform lanes (see the block loop)
  __shared__ int4 ext_s[ROWW || TRANS ? 1 : FM_K1_THREADS / 32][ROWW || TRANS ? 1 : 32][ROWW || TRANS ? 1 : JPT][2];
  if constexpr (!ROWW && !TRANS) {
#pragma unroll
    for (int u = 0; u < JPT; ++u) {
      ext_s[threadIdx.x >> 5][threadIdx.x & 31][u][0] = ea[u];
      ext_s[threadIdx.x >> 5][threadIdx.x & 31][u][1] = eb[u];
    }
  }
  const bool skip_to_partial = !API && no_skip;
  uint32_t vmask = 0u;  // byte mask of the valid column tiles of this thread
#pragma unroll
  for (int u = 0; u < JPT; ++u) vmask |= valid[u] ? (0xFFu << (8 * u)) : 0u;
  unsigned int n0 = 0, n1 = 0;
  int colns[JPT];
#pragma unroll
  for (int u = 0; u < JPT; ++u) colns[u] = 0;
  const bool row_counts = NS && row_cnt != nullptr && rows_per_cta <= 64;
  const bool any = valid[0] && map != nullptr;
  constexpr int KB = (TRANS || ROWW) ? 16 : FM_K1_KB;  // rows per block
  for (int i16 = ib; i16 < iend; i16 += KB) {
    // Uniform block: every comparison of Eq. 4 / the causal test is between r0 or r1 (both in
    // [lo, hi] for the 16 row tiles, hi = min((i16+16) br, N)) and a column-tile value v; when no v
    // lies in [lo, hi] all 16 rows have the class of the first one (evaluated once, stored 16x).
    if constexpr (!ROWW) {
      if (i16 + KB <= iend) {
        const int lo = i16 * br;
        const unsigned span = static_cast<unsigned>(min(static_cast<long long>(i16 + KB) * br, static_cast<long long>(N)) - lo);
        bool ok = true;
#pragma unroll
        for (int u = 0; u < JPT; ++u) {
          const int vs[10] = {ea[u].x, ea[u].y, ea[u].z, ea[u].w, eb[u].x, eb[u].y, eb[u].z, eb[u].w, c0[u], c1[u] - 1};
#pragma unroll
          for (int k = 0; k < 10; ++k)
            ok = ok && (!valid[u] || (k >= 8 && !causal) || static_cast<unsigned>(vs[k]) - static_cast<unsigned>(lo) > span);
        }
        const uint32_t rest0 = __ballot_sync(0xffffffffu, !ok);
        if constexpr (!TRANS) {
         if (__popc(rest0) <= 16) {
          // Row map: the uniform lanes store their class word 16x; the 16 rows of each non-uniform
          // lane are spread over a half-warp (two lanes per round), which reloads that lane's
          // extrema and evaluates one row each — the band of a mask edge costs ~k/2 rounds
          // instead of 16 full-warp row evaluations.
          const int lane = threadIdx.x & 31;
          const int r0 = lo, r1 = r0 + min(br, N - r0);
          uint32_t word = 0u;
          int ns = 0, cz[JPT];
#pragma unroll
          for (int u = 0; u < JPT; ++u) {
            const int cls = tile_class(ea[u], eb[u], r0, r1, c0[u], c1[u], causal);
            cz[u] = cls != 0;
            ns += valid[u] && cls != 0;
            word |= static_cast<uint32_t>(cls) << (8 * u);
          }
          if (ok) {
            if (API) {
              n1 += KB * __popc(word & vmask & 0x01010101u);
              n0 += KB * __popc(word & vmask & 0x02020202u);
            }
            if (NS) {
#pragma unroll
              for (int u = 0; u < JPT; ++u) colns[u] += KB * cz[u];
            }
          }
          if (!API) {
            if (skip_to_partial) word |= (~word & (~word >> 1)) & 0x01010101u;
            word ^= (word & (force1 << 1)) | ((word & (force1 << 1)) >> 1);
          }
          if (row_counts) {
            const int wsum = __reduce_add_sync(0xffffffffu, ok ? ns : 0);
            if (lane < KB && wsum) atomicAdd(&row_acc[i16 - ib + lane], wsum);
          }
          if (ok && any) {
            uint8_t* dst = map + (static_cast<size_t>(bh) * Tr + i16) * Tc + j0;
            if (JPT == 4 && valid[JPT - 1]) {
#pragma unroll 4
              for (int v = 0; v < KB; ++v, dst += Tc) *reinterpret_cast<uint32_t*>(dst) = word;
            } else {
              for (int v = 0; v < KB; ++v, dst += Tc) {
#pragma unroll
                for (int u = 0; u < JPT; ++u)
                  if (valid[u]) dst[u] = static_cast<uint8_t>(word >> (8 * u));
              }
            }
          }
          uint32_t rest = rest0;
          __syncwarp();  // ext_s of this warp (written at the start) visible to every lane
          while (rest) {  // warp-uniform
            const int la = __ffs(rest) - 1;
            rest &= rest - 1;
            int lb = -1;
            if (KB == 16) {  // two lanes per round (a half-warp each); KB = 32: one lane per round
              lb = rest ? __ffs(rest) - 1 : -1;
              rest &= rest ? rest - 1 : 0u;
            }
            const int src = (KB == 32 || lane < 16) ? la : lb;
            int pk = 0;  // NS: per-u non-SKIP flags of this row (8-bit fields)
            if (src >= 0) {
              const int i = i16 + (lane & (KB - 1));
              const int js = (blockIdx.x * blockDim.x + (threadIdx.x & ~31) + src) * JPT;
              const int q0 = i * br, q1 = q0 + min(br, N - q0);
              uint32_t w = 0u, vm = 0u, f1 = 0u;
              int nsr = 0;
#pragma unroll
              for (int u = 0; u < JPT; ++u) {
                const int j = js + u;
                const bool vld = j < Tc;
                const int4 a4 = ext_s[threadIdx.x >> 5][src][u][0], b4 = ext_s[threadIdx.x >> 5][src][u][1];
                const int cc0 = vld ? j * bc : N;
                const int cls = tile_class(a4, b4, q0, q1, cc0, cc0 + min(bc, N - cc0), causal);
                w |= static_cast<uint32_t>(cls) << (8 * u);
                vm |= vld ? (0xFFu << (8 * u)) : 0u;
                if (!API && kernel_map == 2 && j == Tc - 1) f1 |= 1u << (8 * u);
                if (NS) {
                  nsr += vld && cls != 0;
                  pk += (cls != 0 ? 1 : 0) << (8 * u);
                }
              }
              if (API) {
                n1 += __popc(w & vm & 0x01010101u);
                n0 += __popc(w & vm & 0x02020202u);
              }
              if (!API) {
                if (skip_to_partial) w |= (~w & (~w >> 1)) & 0x01010101u;
                w ^= (w & (f1 << 1)) | ((w & (f1 << 1)) >> 1);
              }
              if (row_counts && nsr) atomicAdd(&row_acc[i - ib], nsr);
              if (map != nullptr && js < Tc) {
                uint8_t* dst = map + (static_cast<size_t>(bh) * Tr + i) * Tc + js;
                if (JPT == 4 && js + JPT <= Tc) {
                  *reinterpret_cast<uint32_t*>(dst) = w;
                } else {
#pragma unroll
                  for (int u = 0; u < JPT; ++u)
                    if (js + u < Tc) dst[u] = static_cast<uint8_t>(w >> (8 * u));
                }
              }
            }
            if (NS) {  // column counts of lanes la / lb: sums over their half-warp
#pragma unroll
              for (int o = KB / 2; o; o >>= 1) pk += __shfl_xor_sync(0xffffffffu, pk, o);
              const int pa = __shfl_sync(0xffffffffu, pk, 0), pb = KB == 16 ? __shfl_sync(0xffffffffu, pk, 16) : 0;
              const int mine = lane == la ? pa : (lane == lb ? pb : 0);
#pragma unroll
              for (int u = 0; u < JPT; ++u) colns[u] += (mine >> (8 * u)) & 0xFF;
            }
          }
          continue;
         }
        }
        if (__all_sync(0xffffffffu, ok)) {
          const int r0 = lo, r1 = r0 + min(br, N - r0);
          uint32_t word = 0u;
          int ns = 0;
#pragma unroll
          for (int u = 0; u < JPT; ++u) {
            const int cls = tile_class(ea[u], eb[u], r0, r1, c0[u], c1[u], causal);
            if (NS) {
              ns += valid[u] && cls != 0;
              colns[u] += cls != 0 ? 16 : 0;
            }
            word |= static_cast<uint32_t>(cls) << (8 * u);
          }
          if (API) {
            n1 += 16 * __popc(word & vmask & 0x01010101u);
            n0 += 16 * __popc(word & vmask & 0x02020202u);
          }
          if (!API) {
            if (skip_to_partial) word |= (~word & (~word >> 1)) & 0x01010101u;
            word ^= (word & (force1 << 1)) | ((word & (force1 << 1)) >> 1);
          }
          if (row_counts) {
            const int wsum = __reduce_add_sync(0xffffffffu, ns);
            if ((threadIdx.x & 31) < 16 && wsum) atomicAdd(&row_acc[i16 - ib + (threadIdx.x & 31)], wsum);
          }
          if (any) {
            if constexpr (TRANS) {
              uint8_t* dst = map + (static_cast<size_t>(bh) * Tc + j0) * Tr + i16;
              const uint32_t w4 = (word & 0xffu) * 0x01010101u;
              if ((Tr & 15) == 0) {
                *reinterpret_cast<uint4*>(dst) = make_uint4(w4, w4, w4, w4);
              } else {
                for (int v = 0; v < 16; ++v) dst[v] = static_cast<uint8_t>(w4);
              }
            } else {
              uint8_t* dst = map + (static_cast<size_t>(bh) * Tr + i16) * Tc + j0;
#pragma unroll 4
              for (int v = 0; v < 16; ++v, dst += Tc) {
                if (JPT == 4 && valid[JPT - 1]) {
                  *reinterpret_cast<uint32_t*>(dst) = word;
                } else {
#pragma unroll
                  for (int u = 0; u < JPT; ++u)
                    if (valid[u]) dst[u] = static_cast<uint8_t>(word >> (8 * u));
                }
              }
            }
          }
          continue;
        }
      }
    }
    uint32_t packed[4] = {0u, 0u, 0u, 0u};
#pragma unroll (TRANS ? 16 : 2)
    for (int v = 0; v < KB; ++v) {
      const int i = i16 + v;
      if (i16 + KB > iend && i >= iend) break;
      uint32_t word = 0u;
      int ns = 0;
      const int r0 = i * br, r1 = r0 + min(br, N - r0);
      int4 ra, rb;
      if constexpr (ROWW) {  // the same row tile for the whole warp: broadcast loads
        const int4* e = reinterpret_cast<const int4*>(ext8 + (static_cast<size_t>(bh) * Tr + i) * 8);
        ra = e[0];
        rb = e[1];
      }
#pragma unroll
      for (int u = 0; u < JPT; ++u) {
        const int cls = ROWW ? tile_class_rw(ra, rb, r0, r1, c0[u], c1[u], causal)
                             : tile_class(ea[u], eb[u], r0, r1, c0[u], c1[u], causal);
        if (NS) {
          ns += valid[u] && cls != 0;
          colns[u] += cls != 0;
        }
        word |= static_cast<uint32_t>(cls) << (8 * u);
      }
      if (API) {  // class bytes 0 / 1 / 2: PARTIAL = bit 0, UNMASKED = bit 1 of a valid byte
        n1 += __popc(word & vmask & 0x01010101u);
        n0 += __popc(word & vmask & 0x02020202u);  // (UNMASKED here; SKIP = tiles - the two)
      }
      if (!API) {
        // SKIP (0) -> PARTIAL (1) under FM_FLAG_NO_SKIP; UNMASKED (2) -> PARTIAL on the ragged tile
        if (skip_to_partial) word |= (~word & (~word >> 1)) & 0x01010101u;
        word ^= (word & (force1 << 1)) | ((word & (force1 << 1)) >> 1);
      }
      if (row_counts) {
        const int wsum = __reduce_add_sync(0xffffffffu, ns);
        if ((threadIdx.x & 31) == 0 && wsum) atomicAdd(&row_acc[i - ib], wsum);
      }
      if (any) {
        if constexpr (TRANS) {
          packed[v >> 2] |= (word & 0xffu) << (8 * (v & 3));
        } else {
          uint8_t* dst = map + (static_cast<size_t>(bh) * Tr + i) * Tc + j0;
          if (JPT == 4 && valid[JPT - 1]) {
            *reinterpret_cast<uint32_t*>(dst) = word;  // Tc % 4 == 0 when JPT == 4 (host)
          } else {
#pragma unroll
            for (int u = 0; u < JPT; ++u)
              if (valid[u]) dst[u] = static_cast<uint8_t>(word >> (8 * u));
          }
        }
      }
    }
    if (TRANS && any) {
      uint8_t* dst = map + (static_cast<size_t>(bh) * Tc + j0) * Tr + i16;
      if (i16 + 16 <= iend && (Tr & 15) == 0) {
        *reinterpret_cast<uint4*>(dst) = make_uint4(packed[0], packed[1], packed[2], packed[3]);
      } else {
        for (int v = 0; v < 16 && i16 + v < iend; ++v) dst[v] = static_cast<uint8_t>(packed[v >> 2] >> (8 * (v & 3)));
      }
    }
  }
  if (!API) return;
  if (NS && col_cnt) {
#pragma unroll
    for (int u = 0; u < JPT; ++u)
      if (valid[u] && colns[u]) atomicAdd(&col_cnt[static_cast<size_t>(bh) * Tc + j0 + u], colns[u]);
  }
  if (counts) {
    n0 = __reduce_add_sync(0xffffffffu, n0);
    n1 = __reduce_add_sync(0xffffffffu, n1);
    if ((threadIdx.x & 31) == 0) {
      atomicAdd(&cnt[0], n0);
      atomicAdd(&cnt[1], n1);
    }
  }
  __syncthreads();
  if (counts && threadIdx.x < 3) {
    const int cols = max(0, min(Tc - static_cast<int>(blockIdx.x * blockDim.x * JPT), static_cast<int>(blockDim.x) * JPT));
    const unsigned long long tiles = static_cast<unsigned long long>(cols) * static_cast<unsigned>(max(0, iend - ib));
    // cnt[0] = UNMASKED, cnt[1] = PARTIAL; SKIP = the CTA's valid tiles minus both
    const unsigned long long v = threadIdx.x == 0 ? tiles - cnt[0] - cnt[1] : (threadIdx.x == 1 ? cnt[1] : cnt[0]);
    if (v) atomicAdd(&counts[static_cast<size_t>(bh) * 3 + threadIdx.x], v);
  }
  if (row_counts)
    for (int t = threadIdx.x; t < iend - ib; t += blockDim.x)
      if (row_acc[t]) atomicAdd(&row_cnt[static_cast<size_t>(bh) * Tr + ib + t], row_acc[t]);
}


// ---------------------------------------------------------------------------------------
// K1c: f3 refinement (R31, oracle refine_chunks): for every PARTIAL 128 x 128 tile
// the 32-bit word whose bit (8 g + c) says whether the 32-row group g x 16-column chunk c holds
// a masked cell (real rows and columns only).  UNMASKED tiles get 0 and SKIP tiles every real
// sub-block (rule R is sound: no / every cell masked).  One warp per (b, hm, column tile j);
// lane = 4 consecutive columns whose expanded intervals stay in registers while the warp walks
// the column's row tiles; one ballot per row group turns the per-column tests into chunk bits.
// Optional counts per (b, hm): PARTIAL tiles whose word is 0 (no masked cell at all), and dirty
// sub-blocks over all PARTIAL tiles.  Grid (ceil(Tc / 4), B*Hm, ceil(Tr / rows)), 128 threads: a
// warp walks `rows` (8 or 32) row tiles, so small maps still spread over the SMs (one warp over all
// 64 row tiles of an 8K map was 14.6 us, latency-bound).
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ bool ivl_hits(int s, int e, int a, int b) { return s < e && s < b && e > a; }

__global__ void __launch_bounds__(128) k1_refine(const int32_t* __restrict__ sri, const uint8_t* __restrict__ cmap,
                                                 int N, int C, int causal, int Tr, int Tc, uint32_t* __restrict__ words,
                                                 unsigned long long* __restrict__ rcounts, int rows) {
  pdl_wait();
  pdl_launch();
  const int lane = threadIdx.x & 31;
  const int j = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int bh = blockIdx.y;
  if (j >= Tc) return;
  const int32_t* base = sri + static_cast<size_t>(bh) * N * C;
  int ls[4], le[4], us[4], ue[4], yy[4];
  bool ok[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    yy[u] = j * 128 + lane * 4 + u;
    ok[u] = yy[u] < N;
    if (ok[u]) {
      expand_col(base + static_cast<size_t>(yy[u]) * C, C, causal, N, ls[u], le[u], us[u], ue[u], 0);
    } else {
      ls[u] = le[u] = us[u] = ue[u] = 0;
    }
  }
  // real sub-blocks of this column tile (a SKIP tile has all of them dirty)
  uint32_t colbits = 0u;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (j * 128 + c * 16 < N) colbits |= 1u << c;
  unsigned long long n_clean = 0, n_dirty = 0;
  // classes of this warp's row tiles [i0, i0 + rows), rows <= 32: lane l holds row i0 + l — one
  // strided load per lane instead of a dependent load per row tile
  // (grid-stride over row chunks: gridDim.z is capped at 65535 on the host)
  for (int i0 = blockIdx.z * rows; i0 < Tr; i0 += gridDim.z * rows) {
  const int i1 = min(Tr, i0 + rows);
  const uint32_t cls32 = (lane < rows && i0 + lane < Tr) ? cmap[(static_cast<size_t>(bh) * Tr + i0 + lane) * Tc + j] : 0u;
  for (int i = i0; i < i1; ++i) {
    const uint32_t cls = __shfl_sync(0xffffffffu, cls32, i - i0);
    uint32_t w = 0u;
    if (cls == 0u) {
#pragma unroll
      for (int g = 0; g < 4; ++g)
        if (i * 128 + g * 32 < N) w |= colbits << (8 * g);
    } else if (cls == 1u) {
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        const int a = i * 128 + g * 32;
        const int b = min(a + 32, N);
        bool d = false;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          d |= ok[u] && a < N && (ivl_hits(ls[u], le[u], a, b) || ivl_hits(us[u], ue[u], a, b) || (causal && a < yy[u]));
        const uint32_t bal = __ballot_sync(0xffffffffu, d);
        uint32_t byte = 0u;
#pragma unroll
        for (int c = 0; c < 8; ++c) byte |= ((bal >> (4 * c)) & 0xFu) ? (1u << c) : 0u;
        w |= byte << (8 * g);
      }
      n_clean += (w == 0u);
      n_dirty += __popc(w);
    }
    if (lane == 0) words[(static_cast<size_t>(bh) * Tr + i) * Tc + j] = w;
  }
  }
  if (rcounts && lane == 0) {
    if (n_clean) atomicAdd(&rcounts[static_cast<size_t>(bh) * 2], n_clean);
    if (n_dirty) atomicAdd(&rcounts[static_cast<size_t>(bh) * 2 + 1], n_dirty);
  }
}

cudaError_t launch_refine(const int32_t* sri, const uint8_t* cmap, const Dims& d, uint32_t* words, int64_t* rcounts,
                          cudaStream_t st) {
  if (rcounts) {
    cudaError_t e = cudaMemsetAsync(rcounts, 0, sizeof(int64_t) * 2 * d.B * d.Hm, st);
    if (e != cudaSuccess) return e;
  }
  // row tiles per warp: 8 for maps up to 2^20 tiles (several CTAs per SM), else 32 (fewer
  // re-expansions of the column vectors)
  const long tiles = static_cast<long>(d.Tr) * d.Tc * d.B * d.Hm;
  const int rows = tiles <= (1L << 20) ? 8 : 32;
  const long chunks = (d.Tr + rows - 1) / rows;
  dim3 grid((d.Tc + 3) / 4, d.B * d.Hm, static_cast<unsigned>(chunks < 65535 ? chunks : 65535));
  return launch_pdl(k1_refine, grid, dim3(128), 0, st, sri, cmap, d.N, d.C, d.causal, d.Tr, d.Tc, words,
                    reinterpret_cast<unsigned long long*>(rcounts), rows);
}

// Sliding-window startend_row_indices (flashmask_sliding_window_indices): one thread per key.
__global__ void __launch_bounds__(256) k0_sliding_window(int B, int N, int w, int causal, int32_t* __restrict__ sri) {
  pdl_wait();
  pdl_launch();
  const long idx = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= static_cast<long>(B) * N) return;
  const int y = static_cast<int>(idx % N);
  const int lts = static_cast<int>(min(static_cast<long>(y) + w, static_cast<long>(N)));
  if (causal) {
    sri[idx] = lts;
  } else {
    sri[2 * idx] = lts;
    sri[2 * idx + 1] = max(y - w + 1, 0);
  }
}

cudaError_t launch_sliding_window(int B, int N, int w, int causal, int32_t* sri, cudaStream_t st) {
  const long n = static_cast<long>(B) * N;
  return launch_pdl(k0_sliding_window, dim3(static_cast<unsigned>((n + 255) / 256)), dim3(256), 0, st, B, N, w, causal,
                    sri);
}

cudaError_t launch_expand(const int32_t* sri, const Dims& d, int bc, int32_t* ext8, int4* vec4, cudaStream_t st) {
  const int Tc = (d.N + bc - 1) / bc;
  dim3 grid((Tc + 3) / 4, d.B * d.Hm);
  auto kern = d.C == 4 ? k1_expand<4> : (d.C == 2 ? k1_expand<2> : k1_expand<1>);
  return launch_pdl(kern, grid, dim3(128), 0, st, sri, d.N, d.causal, bc, Tc, ext8, vec4, d.rowwise);
}

cudaError_t launch_classify(const int32_t* ext8, const Dims& d, int br, int bc, uint8_t* map, int transposed,
                            int kernel_map, int64_t* counts, cudaStream_t st, int32_t* row_cnt, int32_t* col_cnt) {
  // the kernels' maps mark a ragged last column tile PARTIAL (bounds mask): decided on the tile size
  const int km = kernel_map ? ((d.N % bc) != 0 ? 2 : 1) : 0;
  br = br < d.N ? br : d.N;  // a tile taller / wider than N is the whole extent (same classes)
  bc = bc < d.N ? bc : d.N;
  const int Tr = (d.N + br - 1) / br, Tc = (d.N + bc - 1) / bc;
  const long bhm = static_cast<long>(d.B) * d.Hm;
  cudaError_t e;
  if (counts && (e = cudaMemsetAsync(counts, 0, sizeof(int64_t) * 3 * bhm, st)) != cudaSuccess) return e;
  if (row_cnt && (e = cudaMemsetAsync(row_cnt, 0, sizeof(int32_t) * Tr * bhm, st)) != cudaSuccess) return e;
  if (col_cnt && (e = cudaMemsetAsync(col_cnt, 0, sizeof(int32_t) * Tc * bhm, st)) != cudaSuccess) return e;
  // Row tiles per CTA: enough CTAs for ~8 per SM (148 SMs), at most 64 row tiles each (the
  // counts leave each CTA as a few atomics; the transposed map is written in 16-row runs)
  // (wide non-transposed maps: 4 column tiles per thread and one 32-bit store per row, see the kernel)
  const long gx = (Tc + FM_K1_THREADS - 1) / FM_K1_THREADS;
  long rpc = (gx * Tr * bhm * FM_K1_THREADS / 128 + 1183) / 1184;
  rpc = rpc < 1 ? 1 : (rpc > 64 ? 64 : rpc);
  if (rpc > 8) rpc = (rpc + 15) / 16 * 16;  // 16-row blocks (uniform-block fast path, 16-row runs)
  const int ns = (d.flags & 1) ? 1 : 0;
  auto cnt64 = reinterpret_cast<unsigned long long*>(counts);
  const bool api = !kernel_map;
  const bool nsc = row_cnt != nullptr || col_cnt != nullptr;
  const int jpt = (!transposed && (Tc % 4) == 0 && Tc >= 512) ? 4 : 1;  // wide maps: 4 column tiles per thread
  const long gxj = (Tc + static_cast<long>(FM_K1_THREADS) * jpt - 1) / (static_cast<long>(FM_K1_THREADS) * jpt);
  dim3 grid(static_cast<unsigned>(gxj), static_cast<unsigned>((Tr + rpc - 1) / rpc), static_cast<unsigned>(bhm));
  // (row-wise: ext8 holds the extrema of the br-row tiles)
  auto pick = [&](auto kern) {
    return launch_pdl(kern, grid, dim3(FM_K1_THREADS), 0, st, ext8, d.N, d.causal, br, bc, Tr, Tc, map, km, ns, cnt64, row_cnt,
                      col_cnt, static_cast<int>(rpc));
  };
#define FM_K1B(RW)                                                                          \
  if (transposed) return api ? pick(k1_classify<1, RW, true, true, false>) : pick(k1_classify<1, RW, true, false, false>); \
  if (api) {                                                                                \
    if (nsc) return jpt == 4 ? pick(k1_classify<4, RW, false, true, true>) : pick(k1_classify<1, RW, false, true, true>); \
    return jpt == 4 ? pick(k1_classify<4, RW, false, true, false>) : pick(k1_classify<1, RW, false, true, false>); \
  }                                                                                         \
  return jpt == 4 ? pick(k1_classify<4, RW, false, false, false>) : pick(k1_classify<1, RW, false, false, false>)
  if (d.rowwise) {
    FM_K1B(true);
  } else {
    FM_K1B(false);
  }
#undef FM_K1B
}

// ---------------------------------------------------------------------------------------
// K1d: longest-processing-time-first order of the forward's units (the work of a unit
// is its number of non-SKIP tiles, O((1-rho) T_r T_c) overall).  One CTA per (b, hm): a
// unit is a pair of 128-row query tiles (work = non-SKIP column tiles of their union, as K2a
// visits); a bitonic sort in shared memory orders them by descending work (ties: lower index
// first).  Used for small problems only (the forward's grid a few waves).  (The FWD = false
// variant orders key tiles by non-SKIP row tiles; measured neutral for the backward — its
// default order is already heaviest-first under causal-like masks — so flashmask_bwd does not
// launch it.)
// ---------------------------------------------------------------------------------------
template <bool FWD>
__global__ void __launch_bounds__(1024) k1_order(const uint8_t* __restrict__ map, int Tr, int Tc, int Trb,
                                                 uint16_t* __restrict__ order) {
  pdl_wait();
  pdl_launch();
  __shared__ uint32_t key[2048];
  const int bh = blockIdx.x;
  const int units = FWD ? (Tr + 1) / 2 : Tc;
  int p2 = 1;
  while (p2 < units) p2 <<= 1;
  // one warp per unit: lanes read the unit's class bytes coalesced, a warp reduction sums them
  const int lane = threadIdx.x & 31;
  for (int u = threadIdx.x >> 5; u < p2; u += blockDim.x >> 5) {
    uint32_t w = 0;
    if (u < units) {
      if (FWD) {
        const uint8_t* r0 = map + (static_cast<size_t>(bh) * Tr + 2 * u) * Tc;
        const uint8_t* r1 = (2 * u + 1 < Tr) ? r0 + Tc : r0;
        for (int j = lane; j < Tc; j += 32) w += (r0[j] | r1[j]) != 0;
      } else {
        const uint8_t* c = map + (static_cast<size_t>(bh) * Tc + u) * Trb;
        for (int i = lane; i < Trb; i += 32) w += c[i] != 0;
      }
      w = __reduce_add_sync(0xffffffffu, w);
    }
    if (lane == 0) key[u] = u < units ? (w << 16) | (0xFFFFu - static_cast<uint32_t>(u)) : 0u;
  }
  __syncthreads();
  for (int k = 2; k <= p2; k <<= 1) {
    for (int jj = k >> 1; jj > 0; jj >>= 1) {
      for (int t = threadIdx.x; t < p2; t += blockDim.x) {
        const int o = t ^ jj;
        if (o > t) {
          const uint32_t a = key[t], b = key[o];
          const bool desc = (t & k) == 0;  // descending runs first: the whole array ends descending
          if (desc ? (a < b) : (a > b)) {
            key[t] = b;
            key[o] = a;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int t = threadIdx.x; t < units; t += blockDim.x)
    order[static_cast<size_t>(bh) * units + t] = static_cast<uint16_t>(0xFFFFu - (key[t] & 0xFFFFu));
  // flag (after the B*Hm orders): 0 when the heavy end is thin — the unit at the 90th percentile of
  // work is within 25 % of the median — where the default order (head-major, better L2 reuse, no
  // early wait) measured ~3 % faster (C2 sliding window: a few light units at the sequence start)
  if (threadIdx.x == 0) {
    const uint32_t w10 = key[units / 10] >> 16, w50 = key[units / 2] >> 16;
    order[static_cast<size_t>(gridDim.x) * units + bh] = (w10 * 4u > w50 * 5u) ? 1 : 0;
  }
}

cudaError_t launch_order(const uint8_t* map, const Dims& d, int fwd, uint16_t* order, cudaStream_t st) {
  const unsigned bhm = static_cast<unsigned>(d.B * d.Hm);
  if (fwd) return launch_pdl(k1_order<true>, dim3(bhm), dim3(1024), 0, st, map, d.Tr, d.Tc, d.Trb, order);
  return launch_pdl(k1_order<false>, dim3(bhm), dim3(1024), 0, st, map, d.Tr, d.Tc, d.Trb, order);
}

// ---------------------------------------------------------------------------------------
// K3: backward preprocess (Alg. 2 line 4, D per row — DESIGN.md R5).  A group of D/8
// threads per (b, h, r), r < Npb, each owning 8 consecutive columns (16-byte loads):
// D = sum_c dO[r,c] * O[r,c]; l2 = lse * log2(e), or +inf when the row is empty (lse = -inf)
// (both written NEGATED — -D and -l2, -l2 = -inf for empty / padded rows — so K4 and K6 form
// scale*S*log2e - l2 and dP - D as one packed fma / add)
// or padded (r >= N) so that exp2(S - l2) = 0 exactly; zero the row of dQacc.
// ---------------------------------------------------------------------------------------
template <int D, bool OUT_F32, bool F16>
__global__ void __launch_bounds__(256) k3_bwd_pre(const void* __restrict__ o, const uint16_t* __restrict__ dout,
                                                  const float* __restrict__ lse, int B, int N, int H, int Npb,
                                                  float* __restrict__ dvec, float* __restrict__ l2,
                                                  float* __restrict__ dqacc) {
  pdl_wait();
  pdl_launch();
  constexpr int G = D / 8;  // threads per row
  const long gt = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long row = gt / G;
  const int part = static_cast<int>(gt % G);
  const long total = static_cast<long>(B) * H * Npb;
  const bool active = row < total;
  const long rr = active ? row : 0;
  const int r = static_cast<int>(rr % Npb);
  const long bh = rr / Npb;
  const int h = static_cast<int>(bh % H), b = static_cast<int>(bh / H);
  float acc = 0.f;
  if (active && r < N) {
    const size_t off = ((static_cast<size_t>(b) * N + r) * H + h) * D + part * 8;
    float ov[8], dv[8];
    unpack16x8<F16>(*reinterpret_cast<const uint4*>(dout + off), dv);
    if constexpr (OUT_F32) {
      const float4 a = *reinterpret_cast<const float4*>(static_cast<const float*>(o) + off);
      const float4 c = *reinterpret_cast<const float4*>(static_cast<const float*>(o) + off + 4);
      ov[0] = a.x; ov[1] = a.y; ov[2] = a.z; ov[3] = a.w; ov[4] = c.x; ov[5] = c.y; ov[6] = c.z; ov[7] = c.w;
    } else {
      unpack16x8<F16>(*reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(o) + off), ov);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) acc = fmaf(ov[t], dv[t], acc);
  }
#pragma unroll
  for (int s = G / 2; s > 0; s >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, s);
  if (!active) return;
  if (part == 0) {
    const size_t ri = static_cast<size_t>(bh) * Npb + r;
    dvec[ri] = (r < N) ? -acc : 0.f;  // stored negated: the consumers add it (packed FFMA2 / FADD2)
    const float lv = (r < N) ? lse[static_cast<size_t>(bh) * N + r] : -INFINITY;
    l2[ri] = (lv == -INFINITY) ? -INFINITY : -lv * 1.4426950408889634f;  // negated, as D
  }
  float4* dq = reinterpret_cast<float4*>(dqacc + (static_cast<size_t>(bh) * Npb + r) * D + part * 8);
  dq[0] = make_float4(0.f, 0.f, 0.f, 0.f);
  dq[1] = make_float4(0.f, 0.f, 0.f, 0.f);
}

cudaError_t launch_bwd_pre(const Dims& d, const void* o, const void* dout, const float* lse, float* dvec, float* l2,
                           float* dqacc, cudaStream_t st) {
  const long threads = static_cast<long>(d.B) * d.H * d.Npb * (d.D / 8);
  const long blocks = (threads + 255) / 256;
  const uint16_t* dob = static_cast<const uint16_t*>(dout);
  cudaError_t e;
#define FM_PRE(DD, F32)                                                                                        \
  e = d.in_f16 ? launch_pdl(k3_bwd_pre<DD, F32, true>, dim3(blocks), dim3(256), 0, st, o, dob, lse, d.B, d.N, d.H, \
                            d.Npb, dvec, l2, dqacc)                                                              \
               : launch_pdl(k3_bwd_pre<DD, F32, false>, dim3(blocks), dim3(256), 0, st, o, dob, lse, d.B, d.N,   \
                            d.H, d.Npb, dvec, l2, dqacc)
  if (d.D == 128) {
    if (d.out_f32) FM_PRE(128, true); else FM_PRE(128, false);
  } else {
    if (d.out_f32) FM_PRE(64, true); else FM_PRE(64, false);
  }
#undef FM_PRE
  return e;
}

// ---------------------------------------------------------------------------------------
// K5: dQ = scale * dQacc (the scale of Eq. 1 carried into dQ, R4) -> out dtype,
// [B,H,Npb,D] -> [B,N,H,D].  One thread per 8 elements (two 16-byte loads).
// ---------------------------------------------------------------------------------------
template <int D, bool OUT_F32, bool F16>
__global__ void __launch_bounds__(256) k5_dq_convert(const float* __restrict__ dqacc, int B, int N, int H, int Npb,
                                                     float scale, void* __restrict__ dq) {
  pdl_wait();
  pdl_launch();
  const long idx8 = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  const long total8 = static_cast<long>(B) * N * H * D / 8;
  if (idx8 >= total8) return;
  const long e = idx8 * 8;
  const int c = static_cast<int>(e % D);
  const long row = e / D;  // (b, r, h)
  const int h = static_cast<int>(row % H);
  const long br = row / H;
  const int r = static_cast<int>(br % N), b = static_cast<int>(br / N);
  const float4* src = reinterpret_cast<const float4*>(dqacc + ((static_cast<size_t>(b) * H + h) * Npb + r) * D + c);
  const float4 v0 = src[0], v1 = src[1];
  if constexpr (OUT_F32) {
    float4* dst = reinterpret_cast<float4*>(dq) + idx8 * 2;
    dst[0] = make_float4(v0.x * scale, v0.y * scale, v0.z * scale, v0.w * scale);
    dst[1] = make_float4(v1.x * scale, v1.y * scale, v1.z * scale, v1.w * scale);
  } else {
    reinterpret_cast<uint4*>(dq)[idx8] =
        make_uint4(pack16<F16>(v0.x * scale, v0.y * scale), pack16<F16>(v0.z * scale, v0.w * scale),
                   pack16<F16>(v1.x * scale, v1.y * scale), pack16<F16>(v1.z * scale, v1.w * scale));
  }
}

// ---------------------------------------------------------------------------------------
// K7 (split-G backward, MQA / GQA with fewer key-tile units than SMs): dV = sum_s dV_s and
// dK = scale * sum_s dK_s over the slices' fp32 partials, in slice order (deterministic), to the
// out dtype.  One thread per 8 elements of [B, N, Hkv, d] (both tensors).
// ---------------------------------------------------------------------------------------
template <bool OUT_F32, bool F16>
__global__ void __launch_bounds__(256) k7_dkv_reduce(const float* __restrict__ part, int gsplit, long total8,
                                                     float scale, void* __restrict__ dk, void* __restrict__ dv) {
  pdl_wait();
  pdl_launch();
  const long idx8 = static_cast<long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx8 >= 2 * total8) return;
  const int kind = idx8 >= total8 ? 1 : 0;  // 0: dV, 1: dK
  const long e8 = idx8 - kind * total8;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int s = 0; s < gsplit; ++s) {
    const float4* src = reinterpret_cast<const float4*>(part + ((static_cast<size_t>(s) * 2 + kind) * total8 + e8) * 8);
    const float4 a = src[0], b = src[1];
    acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
    acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
  }
  const float mul = kind ? scale : 1.0f;
  void* out = kind ? dk : dv;
  if constexpr (OUT_F32) {
    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(out) + e8 * 8);
    dst[0] = make_float4(acc[0] * mul, acc[1] * mul, acc[2] * mul, acc[3] * mul);
    dst[1] = make_float4(acc[4] * mul, acc[5] * mul, acc[6] * mul, acc[7] * mul);
  } else {
    *reinterpret_cast<uint4*>(static_cast<uint16_t*>(out) + e8 * 8) =
        make_uint4(pack16<F16>(acc[0] * mul, acc[1] * mul), pack16<F16>(acc[2] * mul, acc[3] * mul),
                   pack16<F16>(acc[4] * mul, acc[5] * mul), pack16<F16>(acc[6] * mul, acc[7] * mul));
  }
}

cudaError_t launch_dkv_reduce(const Dims& d, int gsplit, const float* part, void* dk, void* dv, cudaStream_t st) {
  const long total8 = static_cast<long>(d.B) * d.N * d.Hkv * d.D / 8;
  const unsigned blocks = static_cast<unsigned>((2 * total8 + 255) / 256);
  if (d.out_f32) return launch_pdl(k7_dkv_reduce<true, false>, dim3(blocks), dim3(256), 0, st, part, gsplit, total8, d.scale, dk, dv);
  if (d.in_f16) return launch_pdl(k7_dkv_reduce<false, true>, dim3(blocks), dim3(256), 0, st, part, gsplit, total8, d.scale, dk, dv);
  return launch_pdl(k7_dkv_reduce<false, false>, dim3(blocks), dim3(256), 0, st, part, gsplit, total8, d.scale, dk, dv);
}

// ---------------------------------------------------------------------------------------
// K1e (bounded single-pass forward, R33): largest key norm of every 128-key tile,
// kmax[b, hk, j] = max_y ||k_y||_2 in fp32, rounded up by a relative 2^-16 for the bf16 -> fp32
// sums; by Cauchy-Schwarz |q_r . k_y| <= ||q_r|| kmax.  Also zeroes the forward's fixup flags
// (n_fix bytes).  One warp per 32 keys, D/8 lanes per key row (16-byte loads, coalesced).
// Grid (Tc, Hkv, B), 128 threads.
// ---------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(128) k1e_key_norms(const uint16_t* __restrict__ k, int N, int Hkv, int Tc,
                                                     float* __restrict__ kmax, uint8_t* __restrict__ fix,
                                                     long n_fix) {
  pdl_wait();  // kmax / fix may still be read by an earlier forward sharing the workspace
  pdl_launch();
  constexpr int G = D / 8;     // 16-byte granules per key row
  constexpr int KPI = 32 / G;  // keys per warp iteration
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x, hk = blockIdx.y, b = blockIdx.z;
  const long cta = (static_cast<long>(b) * Hkv + hk) * Tc + j;
  for (long t = cta * 128 + threadIdx.x; t < n_fix; t += static_cast<long>(gridDim.x) * gridDim.y * gridDim.z * 128)
    fix[t] = 0;
  float best = 0.f;
#pragma unroll 4
  for (int it = 0; it < 32 / KPI; ++it) {
    const int y = j * 128 + warp * 32 + it * KPI + lane / G;
    float ss = 0.f;
    if (y < N) {
      const uint4 u = reinterpret_cast<const uint4*>(k + ((static_cast<size_t>(b) * N + y) * Hkv + hk) * D)[lane % G];
      const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float lo = __uint_as_float(w[t] << 16), hi = __uint_as_float(w[t] & 0xFFFF0000u);
        ss = fmaf(lo, lo, fmaf(hi, hi, ss));
      }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
    best = fmaxf(best, ss);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
  __shared__ float wmax[4];
  if (lane == 0) wmax[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0)
    kmax[cta] = sqrtf(fmaxf(fmaxf(wmax[0], wmax[1]), fmaxf(wmax[2], wmax[3]))) * (1.0f + 1.0f / 65536.0f);
}

cudaError_t launch_key_norms(const Dims& d, const void* k, float* kmax, uint8_t* fix, cudaStream_t st) {
  dim3 grid(d.Tc, d.Hkv, d.B);
  const long n_fix = static_cast<long>(d.B) * d.H * ((d.Tr + 1) / 2);
  const uint16_t* kp = static_cast<const uint16_t*>(k);
  if (d.D == 128) return launch_pdl(k1e_key_norms<128>, grid, dim3(128), 0, st, kp, d.N, d.Hkv, d.Tc, kmax, fix, n_fix);
  return launch_pdl(k1e_key_norms<64>, grid, dim3(128), 0, st, kp, d.N, d.Hkv, d.Tc, kmax, fix, n_fix);
}

cudaError_t launch_dq_convert(const Dims& d, const float* dqacc, void* dq, cudaStream_t st) {
  const long total8 = static_cast<long>(d.B) * d.N * d.H * d.D / 8;
  const long blocks = (total8 + 255) / 256;
  cudaError_t e;
#define FM_CV(DD, F32)                                                                                      \
  e = d.in_f16 ? launch_pdl(k5_dq_convert<DD, F32, true>, dim3(blocks), dim3(256), 0, st, dqacc, d.B, d.N, d.H, \
                            d.Npb, d.scale, dq)                                                               \
               : launch_pdl(k5_dq_convert<DD, F32, false>, dim3(blocks), dim3(256), 0, st, dqacc, d.B, d.N,   \
                            d.H, d.Npb, d.scale, dq)
  if (d.D == 128) {
    if (d.out_f32) FM_CV(128, true); else FM_CV(128, false);
  } else {
    if (d.out_f32) FM_CV(64, true); else FM_CV(64, false);
  }
#undef FM_CV
  return e;
}

}  // namespace fm
