// fm_f32.cu — the FP32-input path (in_dtype = FM_FP32; BASELINE configs[0] = C1, reading R26).
//
// C1 is a parity-only configuration (one 128x128 tile), so the fp32 path is written for exact
// fp32 arithmetic, not for throughput: one warp per query row (forward, dQ) or per key
// (dK/dV), the head dimension spread over the 32 lanes, dot products reduced with shuffles,
// expf/logf in fp32.  It follows the same method as the bf16 tensor-core path: the K1 class
// map decides per 128x128 tile (Alg. 1 lines 9-14) — SKIP tiles are not visited,
// UNMASKED tiles take no per-element mask work, PARTIAL tiles apply the column-interval
// predicate of Eq. 3 — and the backward is Alg. 2's recompute-from-L scheme
// (P:413-434).  It accumulates in fixed order (no atomics), so it is deterministic.
#include <cuda_bf16.h>
#include <cmath>

#include "fm_internal.h"

namespace fm {

namespace {

__device__ __forceinline__ float warp_sum(float x) {
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) x += __shfl_xor_sync(0xffffffffu, x, s);
  return x;
}

// masked(r, y) of Eq. 3 from the normalised column vector (LTS, LTE-LTS, UTS, UTE-UTS)
__device__ __forceinline__ bool cell_masked(const int4 mv, int r, int y, bool causal) {
  if (static_cast<unsigned>(r - mv.x) < static_cast<unsigned>(mv.y)) return true;
  return causal ? (r < y) : (static_cast<unsigned>(r - mv.z) < static_cast<unsigned>(mv.w));
}
// row-wise representation (R32): rv = query row r's (LTS, len, UTS, len) over key columns
__device__ __forceinline__ bool cell_masked_rw(const int4 rv, int r, int y, bool causal, int N) {
  if (static_cast<unsigned>(y - rv.x) < static_cast<unsigned>(rv.y)) return true;
  if (static_cast<unsigned>(y - rv.z) < static_cast<unsigned>(rv.w)) return true;
  return (causal && r < y) || y >= N;
}

template <bool F32>
__device__ __forceinline__ void store_out(void* base, size_t idx, float v) {
  if constexpr (F32)
    static_cast<float*>(base)[idx] = v;
  else
    static_cast<__nv_bfloat16*>(base)[idx] = __float2bfloat16_rn(v);
}

template <bool F32>
__device__ __forceinline__ float load_out(const void* base, size_t idx) {
  if constexpr (F32)
    return static_cast<const float*>(base)[idx];
  else
    return __bfloat162float(static_cast<const __nv_bfloat16*>(base)[idx]);
}

}  // namespace

// Forward (Alg. 1 with one row per warp): online softmax over the visited keys in fp32.
template <int D, bool OUT_F32>
__global__ void __launch_bounds__(128) f32_fwd_kernel(F32Args a) {
  constexpr int E = D / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 4 + warp;
  const int h = blockIdx.y, b = blockIdx.z;
  if (r >= a.N) return;
  const int hk = h / a.G, hm = (a.Hm == 1) ? 0 : hk;
  const size_t bhm = static_cast<size_t>(b) * a.Hm + hm;
  const int4* vec = a.vec4 + bhm * static_cast<size_t>(a.Tc) * 128;
  const uint8_t* cls_row = a.fmap + (bhm * a.Tr + r / 128) * a.Tc;
  float qv[E], acc[E];
  const float* qp = a.q + ((static_cast<size_t>(b) * a.N + r) * a.H + h) * D;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    qv[e] = qp[lane + 32 * e];
    acc[e] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int j = 0; j < a.Tc; ++j) {
    const int cls = cls_row[j];
    if (cls == 0) continue;  // SKIP: no load, no compute
    const int y1 = min(j * 128 + 128, a.N);
    for (int y = j * 128; y < y1; ++y) {
      if (cls == 1 && (a.rowwise ? cell_masked_rw(vec[r], r, y, a.causal, a.N) : cell_masked(vec[y], r, y, a.causal)))
        continue;
      const float* kp = a.k + ((static_cast<size_t>(b) * a.N + y) * a.Hkv + hk) * D;
      const float* vp = a.v + ((static_cast<size_t>(b) * a.N + y) * a.Hkv + hk) * D;
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) s = fmaf(qv[e], kp[lane + 32 * e], s);
      s = warp_sum(s) * a.scale;
      const float mn = fmaxf(m, s);
      const float alpha = (m == -INFINITY) ? 0.f : expf(m - mn);
      const float p = expf(s - mn);
      l = l * alpha + p;
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = fmaf(p, vp[lane + 32 * e], acc[e] * alpha);
      m = mn;
    }
  }
  const bool live = l > 0.f;
  const float inv = live ? 1.f / l : 0.f;
  const size_t orow = ((static_cast<size_t>(b) * a.N + r) * a.H + h) * D;
#pragma unroll
  for (int e = 0; e < E; ++e) store_out<OUT_F32>(a.o, orow + lane + 32 * e, acc[e] * inv);
  if (lane == 0) a.lse[(static_cast<size_t>(b) * a.H + h) * a.N + r] = live ? m + logf(l) : -INFINITY;
}

// dQ row (Alg. 2 lines 15-21 restated per row) and D_r = rowsum(dO o O).
template <int D, bool OUT_F32>
__global__ void __launch_bounds__(128) f32_dq_kernel(F32Args a) {
  constexpr int E = D / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 4 + warp;
  const int h = blockIdx.y, b = blockIdx.z;
  if (r >= a.N) return;
  const int hk = h / a.G, hm = (a.Hm == 1) ? 0 : hk;
  const size_t bhm = static_cast<size_t>(b) * a.Hm + hm;
  const int4* vec = a.vec4 + bhm * static_cast<size_t>(a.Tc) * 128;
  const uint8_t* cls_row = a.fmap + (bhm * a.Tr + r / 128) * a.Tc;
  const size_t row = (static_cast<size_t>(b) * a.N + r) * a.H + h;
  float qv[E], dov[E], dq[E];
  float dsum = 0.f;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    qv[e] = a.q[row * D + lane + 32 * e];
    dov[e] = a.dout[row * D + lane + 32 * e];
    dsum = fmaf(dov[e], load_out<OUT_F32>(a.o, row * D + lane + 32 * e), dsum);
    dq[e] = 0.f;
  }
  const float Dr = warp_sum(dsum);
  const float L = a.lse[(static_cast<size_t>(b) * a.H + h) * a.N + r];
  if (lane == 0) a.dvec[(static_cast<size_t>(b) * a.H + h) * a.Npb + r] = Dr;
  if (L != -INFINITY) {  // an empty row (L = -inf, reading R7) contributes nothing
    for (int j = 0; j < a.Tc; ++j) {
      const int cls = cls_row[j];
      if (cls == 0) continue;
      const int y1 = min(j * 128 + 128, a.N);
      for (int y = j * 128; y < y1; ++y) {
        if (cls == 1 && (a.rowwise ? cell_masked_rw(vec[r], r, y, a.causal, a.N) : cell_masked(vec[y], r, y, a.causal)))
          continue;
        const float* kp = a.k + ((static_cast<size_t>(b) * a.N + y) * a.Hkv + hk) * D;
        const float* vp = a.v + ((static_cast<size_t>(b) * a.N + y) * a.Hkv + hk) * D;
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          s = fmaf(qv[e], kp[lane + 32 * e], s);
          dp = fmaf(dov[e], vp[lane + 32 * e], dp);
        }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const float p = expf(s * a.scale - L);
        const float ds = p * (dp - Dr);
#pragma unroll
        for (int e = 0; e < E; ++e) dq[e] = fmaf(ds, kp[lane + 32 * e], dq[e]);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) store_out<OUT_F32>(a.dq, row * D + lane + 32 * e, dq[e] * a.scale);
}

// dK, dV of one key y of one key/value head: sums over the visible rows of all G query heads
// of the group (Alg. 2 lines 12-22 restated per key; dK/dV written once, no atomics).
template <int D, bool OUT_F32>
__global__ void __launch_bounds__(128) f32_dkdv_kernel(F32Args a) {
  constexpr int E = D / 32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int y = blockIdx.x * 4 + warp;
  const int hk = blockIdx.y, b = blockIdx.z;
  if (y >= a.N) return;
  const int hm = (a.Hm == 1) ? 0 : hk;
  const size_t bhm = static_cast<size_t>(b) * a.Hm + hm;
  const int4 mv = a.rowwise ? make_int4(0, 0, 0, 0) : a.vec4[bhm * static_cast<size_t>(a.Tc) * 128 + y];
  const int j = y / 128;
  const size_t krow = (static_cast<size_t>(b) * a.N + y) * a.Hkv + hk;
  float kv[E], vv[E], dk[E], dv[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    kv[e] = a.k[krow * D + lane + 32 * e];
    vv[e] = a.v[krow * D + lane + 32 * e];
    dk[e] = dv[e] = 0.f;
  }
  for (int g = 0; g < a.G; ++g) {
    const int h = hk * a.G + g;
    const float* Lh = a.lse + (static_cast<size_t>(b) * a.H + h) * a.N;
    const float* Dh = a.dvec + (static_cast<size_t>(b) * a.H + h) * a.Npb;
    for (int i = 0; i < a.Tr; ++i) {
      const int cls = a.fmap[(bhm * a.Tr + i) * a.Tc + j];
      if (cls == 0) continue;
      const int r1 = min(i * 128 + 128, a.N);
      for (int r = i * 128; r < r1; ++r) {
        if (cls == 1 && (a.rowwise ? cell_masked_rw(a.vec4[bhm * static_cast<size_t>(a.Tc) * 128 + r], r, y, a.causal, a.N)
                                   : cell_masked(mv, r, y, a.causal)))
          continue;
        const float L = Lh[r];
        if (L == -INFINITY) continue;
        const size_t row = (static_cast<size_t>(b) * a.N + r) * a.H + h;
        float s = 0.f, dp = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          s = fmaf(a.q[row * D + lane + 32 * e], kv[e], s);
          dp = fmaf(a.dout[row * D + lane + 32 * e], vv[e], dp);
        }
        s = warp_sum(s);
        dp = warp_sum(dp);
        const float p = expf(s * a.scale - L);
        const float ds = p * (dp - Dh[r]);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          dv[e] = fmaf(p, a.dout[row * D + lane + 32 * e], dv[e]);
          dk[e] = fmaf(ds, a.q[row * D + lane + 32 * e], dk[e]);
        }
      }
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) {
    store_out<OUT_F32>(a.dk, krow * D + lane + 32 * e, dk[e] * a.scale);
    store_out<OUT_F32>(a.dv, krow * D + lane + 32 * e, dv[e]);
  }
}

#define FM_F32_DISPATCH(KERNEL, GRID)                                                      \
  do {                                                                                     \
    if (d.D == 128) {                                                                      \
      if (d.out_f32) KERNEL<128, true><<<GRID, 128, 0, st>>>(a);                           \
      else KERNEL<128, false><<<GRID, 128, 0, st>>>(a);                                    \
    } else {                                                                               \
      if (d.out_f32) KERNEL<64, true><<<GRID, 128, 0, st>>>(a);                            \
      else KERNEL<64, false><<<GRID, 128, 0, st>>>(a);                                     \
    }                                                                                      \
  } while (0)

cudaError_t launch_f32_fwd(const Dims& d, const F32Args& a, cudaStream_t st) {
  const dim3 grid((d.N + 3) / 4, d.H, d.B);
  FM_F32_DISPATCH(f32_fwd_kernel, grid);
  return cudaGetLastError();
}

cudaError_t launch_f32_dq(const Dims& d, const F32Args& a, cudaStream_t st) {
  const dim3 grid((d.N + 3) / 4, d.H, d.B);
  FM_F32_DISPATCH(f32_dq_kernel, grid);
  return cudaGetLastError();
}

cudaError_t launch_f32_dkdv(const Dims& d, const F32Args& a, cudaStream_t st) {
  const dim3 grid((d.N + 3) / 4, d.Hkv, d.B);
  FM_F32_DISPATCH(f32_dkdv_kernel, grid);
  return cudaGetLastError();
}

#undef FM_F32_DISPATCH

}  // namespace fm
