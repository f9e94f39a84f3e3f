// fm_api.cu — the C ABI of include/flashmask.h: argument validation, workspace layout,
// TMA descriptor encoding and the launch sequence K1 -> K2 (forward) and
// K1 -> K3 -> K4 -> K5 (backward).
#include <cudaTypedefs.h>
#include <cuda.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/flashmask.h"
#include "fm_internal.h"

namespace {

thread_local std::string g_last_error;

fm_status fail(fm_status s, const std::string& msg) {
  g_last_error = msg;
  return s;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_once;
cudaError_t g_encode_err = cudaSuccess;

PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  std::call_once(g_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    g_encode_err = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    if (g_encode_err == cudaSuccess && q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode;
}

// [B, N, heads, D] bf16 tensor viewed as the 4-D box grid (D, heads, N, B); box = 64 x 1 x rows
// x 1, 128-byte swizzle, out-of-bounds rows zero-filled.
bool make_map(CUtensorMap* m, const void* ptr, const fm::Dims& d, int heads, int box_rows, std::string* err) {
  auto enc = get_encode();
  if (!enc) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(d.D), static_cast<cuuint64_t>(heads), static_cast<cuuint64_t>(d.N),
                        static_cast<cuuint64_t>(d.B)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(d.D) * 2, static_cast<cuuint64_t>(heads) * d.D * 2,
                           static_cast<cuuint64_t>(d.N) * heads * d.D * 2};
  cuuint32_t box[4] = {64, 1, static_cast<cuuint32_t>(box_rows), 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(m, d.in_f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4,
                   const_cast<void*>(ptr), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled failed with CUresult " + std::to_string(static_cast<int>(r));
    return false;
  }
  return true;
}

// fp32 dQ accumulator [B*H*Npb, D] viewed 2-D for TMA tensor reduce-adds: box = kDq64BoxRows x 32
// columns (128 B), 128-byte swizzle (d=64 backward, fm_bwd.cu).
bool make_dq_map(CUtensorMap* m, float* dqacc, const fm::Dims& d, std::string* err) {
  auto enc = get_encode();
  if (!enc) {
    *err = "cuTensorMapEncodeTiled unavailable";
    return false;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(d.D), static_cast<cuuint64_t>(d.B) * d.H * d.Npb};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(d.D) * 4};
  cuuint32_t box[2] = {32, static_cast<cuuint32_t>(fm::kDq64BoxRows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dqacc, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    *err = "cuTensorMapEncodeTiled (dQ accumulator) failed with CUresult " + std::to_string(static_cast<int>(r));
    return false;
  }
  return true;
}

fm_status check_params(const fm_params* p, fm::Dims* d, bool need_attention) {
  if (!p) return fail(FM_ERR_INVALID_ARGUMENT, "params is NULL");
  if (p->batch < 1 || p->seqlen < 1 || p->num_heads < 1)
    return fail(FM_ERR_INVALID_ARGUMENT, "batch, seqlen and num_heads must be >= 1");
  if (p->batch > 65535 || p->num_heads > 65535 || p->seqlen > (1LL << 30))
    return fail(FM_ERR_UNSUPPORTED, "batch/num_heads > 65535 or seqlen > 2^30");
  const int64_t hkv = p->num_kv_heads > 0 ? p->num_kv_heads : p->num_heads;
  if (p->num_kv_heads < 0 || p->num_heads % hkv != 0)
    return fail(FM_ERR_INVALID_ARGUMENT, "num_kv_heads must divide num_heads");
  if (p->mask_heads != 1 && p->mask_heads != hkv)
    return fail(FM_ERR_INVALID_ARGUMENT, "mask_heads must be 1 or num_kv_heads");
  // K1 puts (batch, mask head) pairs in one grid dimension (limit 65535)
  if (p->batch * p->mask_heads > 65535)
    return fail(FM_ERR_UNSUPPORTED, "batch * mask_heads > 65535");
  const int C = static_cast<int>(p->mask_cols);
  const bool ok_c = p->causal ? (C == 1 || C == 2) : (C == 2 || C == 4);
  if ((p->causal != 0 && p->causal != 1) || !ok_c)
    return fail(FM_ERR_INVALID_ARGUMENT, "invalid (causal, mask_cols) combination; see the C-table in flashmask.h");
  if (p->in_dtype != FM_BF16 && p->in_dtype != FM_FP32 && p->in_dtype != FM_FP16)
    return fail(FM_ERR_INVALID_ARGUMENT, "bad in_dtype");
  // 16-bit outputs have the 16-bit type of the inputs (fp32 inputs: bf16 outputs)
  const int out16 = p->in_dtype == FM_FP16 ? FM_FP16 : FM_BF16;
  if (p->out_dtype != out16 && p->out_dtype != FM_FP32)
    return fail(FM_ERR_INVALID_ARGUMENT, "out_dtype must be FM_FP32 or the 16-bit type of in_dtype");
  if (need_attention) {
    if (p->head_dim != 64 && p->head_dim != 128) return fail(FM_ERR_INVALID_ARGUMENT, "head_dim must be 64 or 128");
  }
  d->B = static_cast<int>(p->batch);
  d->N = static_cast<int>(p->seqlen);
  d->H = static_cast<int>(p->num_heads);
  d->D = static_cast<int>(p->head_dim);
  d->Hm = static_cast<int>(p->mask_heads);
  d->Hkv = static_cast<int>(hkv);
  d->G = d->H / d->Hkv;
  d->C = C;
  d->causal = p->causal;
  d->Tr = (d->N + fm::kTile - 1) / fm::kTile;
  d->Tc = d->Tr;
  d->Brb = (d->D == 128) ? 64 : 128;
  d->Trb = (d->N + d->Brb - 1) / d->Brb;
  d->Npb = d->Tr * fm::kTile;  // covers both the 64/128-row backward tiles and K6's 128-row tiles
  d->scale = (p->scale > 0.f) ? p->scale : 1.0f / std::sqrt(static_cast<float>(p->head_dim > 0 ? p->head_dim : 1));
  d->out_f32 = p->out_dtype == FM_FP32;
  d->in_f16 = p->in_dtype == FM_FP16;
  d->flags = p->flags;
  d->rowwise = (p->flags & FM_FLAG_ROWWISE) ? 1 : 0;
  if (need_attention && d->Tc > fm::kMaxTc) return fail(FM_ERR_UNSUPPORTED, "seqlen > 262144");
  return FM_OK;
}

// Split-G backward: when the key-tile units (Tc * Hkv * B) do not fill the 148 SMs and each CTA
// would loop over G > 1 query heads (MQA / GQA), the G heads are split over gsplit CTAs (the
// largest divisor of G up to two waves' worth), whose fp32 dK / dV partials K7 sums.
int gsplit_for(const fm::Dims& d) {
  const long units = static_cast<long>(d.Tc) * d.Hkv * d.B;
  if (d.G < 2 || units >= 148) return 1;
  const long target = (296 + units - 1) / units;
  int s = 1;
  for (int c = 2; c <= d.G; ++c)
    if (d.G % c == 0 && c <= target) s = c;
  return s;
}

// Carve the workspace.  Returns the total size; pointers valid only when base != nullptr.
// Every buffer starts on a 4 KiB boundary of the device address space (the caller's base is
// first rounded up to 64 KiB; the size bound includes that slack): the backward's 8 KiB bulk
// reduce-adds into dqacc measured ~10 % slower when the accumulator was only 256-B aligned.
size_t carve(const fm::Dims& d, int pass, void* base, fm::Workspace* w) {
  constexpr size_t kBaseAlign = 65536, kBufAlign = 4096;
  size_t off = base ? (kBaseAlign - reinterpret_cast<uintptr_t>(base) % kBaseAlign) % kBaseAlign : kBaseAlign;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes, kBufAlign);
    return base ? static_cast<uint8_t*>(base) + o : nullptr;
  };
  const size_t bhm = static_cast<size_t>(d.B) * d.Hm;
  const size_t bh = static_cast<size_t>(d.B) * d.H;
  w->ext8 = reinterpret_cast<int32_t*>(take(bhm * d.Tc * 8 * sizeof(int32_t)));
  // row-wise backward: extrema of the Brb-row tiles of the backward map (Trb >= Tc)
  w->ext8b = (pass == FM_PASS_BWD) ? reinterpret_cast<int32_t*>(take(bhm * d.Trb * 8 * sizeof(int32_t))) : nullptr;
  w->vec4 = reinterpret_cast<int4*>(take(bhm * d.Tc * 128 * sizeof(int4)));
  w->fmap = nullptr;
  w->bmap = nullptr;
  w->dvec = w->l2 = w->dqacc = w->dkv_part = nullptr;
  w->cw = nullptr;
  if (pass == FM_PASS_FWD) {
    w->fmap = take(bhm * d.Tr * d.Tc);
    w->cw = reinterpret_cast<uint32_t*>(take(bhm * d.Tr * d.Tc * sizeof(uint32_t)));
  } else {
    w->fmap = take(bhm * d.Tr * d.Tc);  // used by the deterministic dQ kernel (K6)
    w->bmap = take(bhm * d.Tc * d.Trb);
    w->dvec = reinterpret_cast<float*>(take(bh * d.Npb * sizeof(float)));
    w->l2 = reinterpret_cast<float*>(take(bh * d.Npb * sizeof(float)));
    w->dqacc = reinterpret_cast<float*>(take(bh * d.Npb * d.D * sizeof(float)));
    const int gs = gsplit_for(d);
    w->dkv_part = gs > 1 ? reinterpret_cast<float*>(take(static_cast<size_t>(2) * gs * d.B * d.N * d.Hkv * d.D *
                                                         sizeof(float)))
                         : nullptr;
  }
  // LPT orders (>= ceil(Tr/2) pairs or Tc key tiles per (b, hm)) followed by one flag per (b, hm)
  w->order = reinterpret_cast<uint16_t*>(take(bhm * (d.Tc + 1) * sizeof(uint16_t)));
  w->kmax = nullptr;
  w->fix = nullptr;
  if (pass == FM_PASS_FWD) {
    w->kmax = reinterpret_cast<float*>(take(static_cast<size_t>(d.B) * d.Hkv * d.Tc * sizeof(float)));
    w->fix = take(bh * ((d.Tr + 1) / 2));
  }
  w->bytes = off;
  return off;
}

// LPT scheduling (K1d) for small problems: the attention kernels' grid spans only a few waves of
// 148 SMs, so unequal unit costs leave SMs idle at the end (a list-scheduling simulation of C2
// put the default order at 0.87-0.90 of ideal, LPT by groups of heads at 0.95-0.97).  Returns the
// heads per group (a divisor of `heads`) sized so that the group's K/V (and for the backward
// Q/dO) stay in L2 while its units run, or 0 when LPT is not used.
int lpt_group(const fm::Dims& d, long units, int heads, size_t bytes_per_head) {
  if (units > 16L * 148 || units < 148) return 0;
  constexpr size_t kBudget = size_t(40) << 20;
  int g = 1;
  for (int c = heads; c >= 1; --c)
    if (heads % c == 0 && static_cast<size_t>(c) * bytes_per_head <= kBudget) {
      g = c;
      break;
    }
  return g;
}

fm::F32Args f32_args(const fm::Dims& d, const fm::Workspace& w) {
  fm::F32Args a{};
  a.B = d.B; a.N = d.N; a.H = d.H; a.Hm = d.Hm; a.Hkv = d.Hkv; a.G = d.G; a.Tr = d.Tr; a.Tc = d.Tc;
  a.Npb = d.Npb; a.causal = d.causal; a.rowwise = d.rowwise;
  a.scale = d.scale;
  a.fmap = w.fmap;
  a.vec4 = w.vec4;
  a.dvec = w.dvec;
  return a;
}

fm_status cuda_fail(cudaError_t e, const char* where) {
  return fail(FM_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

// ---- optional per-launch timing (flashmask_timing_enable / _collect) ----
struct TimingRec {
  int kid;
  cudaEvent_t a, b;
};
struct Timing {
  bool on = false;
  uint32_t mask = 0xFFFFFFFFu;  // kernel ids to bracket
  std::vector<TimingRec> recs;
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};
thread_local Timing g_timing;

// Launch `fn` (returns cudaError_t) bracketed by events when timing is on.
template <class F>
cudaError_t timed(int kid, cudaStream_t st, F&& fn) {
  if (!g_timing.on || !((g_timing.mask >> kid) & 1u)) return fn();
  TimingRec r{kid, g_timing.get(), g_timing.get()};
  cudaEventRecord(r.a, st);
  cudaError_t e = fn();
  cudaEventRecord(r.b, st);
  g_timing.recs.push_back(r);
  return e;
}

}  // namespace

extern "C" {

const char* flashmask_status_string(fm_status s) {
  switch (s) {
    case FM_OK: return "FM_OK";
    case FM_ERR_INVALID_ARGUMENT: return "FM_ERR_INVALID_ARGUMENT";
    case FM_ERR_UNSUPPORTED: return "FM_ERR_UNSUPPORTED";
    case FM_ERR_WORKSPACE_TOO_SMALL: return "FM_ERR_WORKSPACE_TOO_SMALL";
    case FM_ERR_CUDA: return "FM_ERR_CUDA";
  }
  return "FM_UNKNOWN_STATUS";
}

const char* flashmask_last_error(void) { return g_last_error.c_str(); }

size_t flashmask_workspace_size(const fm_params* p, int pass) {
  fm::Dims d{};
  if (check_params(p, &d, true) != FM_OK) return 0;
  if (pass != FM_PASS_FWD && pass != FM_PASS_BWD) {
    fail(FM_ERR_INVALID_ARGUMENT, "pass must be FM_PASS_FWD or FM_PASS_BWD");
    return 0;
  }
  fm::Workspace w{};
  return carve(d, pass, nullptr, &w);
}

fm_status flashmask_classify(const fm_params* p, const int32_t* sri, int32_t br, int32_t bc, int32_t* minmax,
                             uint8_t* class_map, int64_t* counts, int32_t* row_nonskip, int32_t* col_nonskip,
                             void* stream) {
  g_last_error.clear();
  fm::Dims d{};
  fm_status s = check_params(p, &d, false);
  if (s != FM_OK) return s;
  if (!sri || !minmax) return fail(FM_ERR_INVALID_ARGUMENT, "startend_row_indices and minmax are required");
  if (!aligned16(sri)) return fail(FM_ERR_INVALID_ARGUMENT, "startend_row_indices must be 16-byte aligned");
  if (br < 1 || bc < 1) return fail(FM_ERR_INVALID_ARGUMENT, "br and bc must be >= 1");
  // K1b: at most 64 row tiles per CTA and 65535 CTAs along the row-tile grid dimension
  if ((p->seqlen + std::min<int64_t>(br, p->seqlen) - 1) / std::min<int64_t>(br, p->seqlen) > 65535LL * 64)
    return fail(FM_ERR_UNSUPPORTED, "ceil(seqlen / br) > 4194240 row tiles");
  if (!aligned16(minmax)) return fail(FM_ERR_INVALID_ARGUMENT, "minmax must be 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // column-wise: extrema per bc-column tile; row-wise (R32): per br-row tile
  cudaError_t e = timed(FM_KERNEL_EXPAND, st, [&] { return fm::launch_expand(sri, d, d.rowwise ? br : bc, minmax, nullptr, st); });
  if (e != cudaSuccess) return cuda_fail(e, "expand");
  if (class_map || counts || row_nonskip || col_nonskip) {
    fm::Dims d0 = d;
    d0.flags = 0;  // true classes (FM_FLAG_NO_SKIP does not apply); d0.rowwise is kept
    e = timed(FM_KERNEL_CLASSIFY, st, [&] {
      return fm::launch_classify(minmax, d0, br, bc, class_map, 0, 0, counts, st, row_nonskip, col_nonskip);
    });
    if (e != cudaSuccess) return cuda_fail(e, "classify");
  }
  return FM_OK;
}

fm_status flashmask_refine(const fm_params* p, const int32_t* sri, const uint8_t* class_map, uint32_t* words,
                           int64_t* counts, void* stream) {
  g_last_error.clear();
  fm::Dims d{};
  fm_status s = check_params(p, &d, false);
  if (s != FM_OK) return s;
  if (!sri || !class_map || !words) return fail(FM_ERR_INVALID_ARGUMENT, "startend_row_indices, class_map, words required");
  if (d.rowwise) return fail(FM_ERR_UNSUPPORTED, "flashmask_refine: column-wise representation only (R31)");
  if (!aligned16(sri)) return fail(FM_ERR_INVALID_ARGUMENT, "startend_row_indices must be 16-byte aligned");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaError_t e = timed(FM_KERNEL_REFINE, st, [&] { return fm::launch_refine(sri, class_map, d, words, counts, st); });
  if (e != cudaSuccess) return cuda_fail(e, "refine");
  return FM_OK;
}

fm_status flashmask_fwd(const fm_params* p, const void* q, const void* k, const void* v, const int32_t* sri, void* o,
                        float* lse, void* workspace, size_t workspace_bytes, void* stream) {
  g_last_error.clear();
  fm::Dims d{};
  fm_status s = check_params(p, &d, true);
  if (s != FM_OK) return s;
  if (!q || !k || !v || !sri || !o || !lse || !workspace) return fail(FM_ERR_INVALID_ARGUMENT, "NULL pointer argument");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || !aligned16(sri) || !aligned16(workspace))
    return fail(FM_ERR_INVALID_ARGUMENT, "q, k, v, o, startend_row_indices and workspace must be 16-byte aligned");
  fm::Workspace w{};
  if (carve(d, FM_PASS_FWD, nullptr, &w) > workspace_bytes)
    return fail(FM_ERR_WORKSPACE_TOO_SMALL, "workspace smaller than flashmask_workspace_size(FM_PASS_FWD)");
  carve(d, FM_PASS_FWD, workspace, &w);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->in_dtype == FM_FP32) {  // fp32 inputs: fm_f32.cu (reading R26)
    cudaError_t e = timed(FM_KERNEL_EXPAND, st, [&] { return fm::launch_expand(sri, d, fm::kTile, w.ext8, w.vec4, st); });
    if (e != cudaSuccess) return cuda_fail(e, "expand");
    e = timed(FM_KERNEL_CLASSIFY, st, [&] { return fm::launch_classify(w.ext8, d, fm::kTile, fm::kTile, w.fmap, 0, 1, nullptr, st); });
    if (e != cudaSuccess) return cuda_fail(e, "classify");
    fm::F32Args a = f32_args(d, w);
    a.q = static_cast<const float*>(q);
    a.k = static_cast<const float*>(k);
    a.v = static_cast<const float*>(v);
    a.o = o;
    a.lse = lse;
    e = timed(FM_KERNEL_FWD, st, [&] { return fm::launch_f32_fwd(d, a, st); });
    if (e != cudaSuccess) return cuda_fail(e, "fp32 forward kernel");
    return FM_OK;
  }
  std::string err;
  CUtensorMap tq, tk, tv, to;
  if (!make_map(&tq, q, d, d.H, 128, &err) || !make_map(&tk, k, d, d.Hkv, 128, &err) ||
      !make_map(&tv, v, d, d.Hkv, 128, &err))
    return fail(FM_ERR_CUDA, err);
  if (d.out_f32)
    to = tq;  // fp32 O is stored directly by the kernel (the map is not used)
  else if (!make_map(&to, o, d, d.H, 128, &err))
    return fail(FM_ERR_CUDA, err);
  cudaError_t e = timed(FM_KERNEL_EXPAND, st, [&] { return fm::launch_expand(sri, d, fm::kTile, w.ext8, w.vec4, st); });
  if (e != cudaSuccess) return cuda_fail(e, "expand");
  e = timed(FM_KERNEL_CLASSIFY, st, [&] { return fm::launch_classify(w.ext8, d, fm::kTile, fm::kTile, w.fmap, 0, 1, nullptr, st); });
  if (e != cudaSuccess) return cuda_fail(e, "classify");
  // f3 refinement: consumed by the causal forward kernels (fm_fwd.cu FM_FWD_REFINE)
  const bool refine = d.causal && !d.rowwise && (p->flags & FM_FLAG_NO_REFINE) == 0;
  if (refine) {
    e = timed(FM_KERNEL_REFINE, st, [&] { return fm::launch_refine(sri, w.fmap, d, w.cw, nullptr, st); });
    if (e != cudaSuccess) return cuda_fail(e, "refine");
  }
  fm::FwdArgs a{};
  a.B = d.B; a.N = d.N; a.H = d.H; a.Hm = d.Hm; a.Tr = d.Tr; a.Tc = d.Tc; a.G = d.G;
  // LPT order of (head, pair) units for small grids (K1d); K/V bytes per query head ~ 2 N d 2 / G
  a.hgrp = lpt_group(d, static_cast<long>((d.Tr + 1) / 2) * d.H * d.B, d.H,
                     static_cast<size_t>(4) * d.N * d.D / static_cast<size_t>(d.G));
  a.order = nullptr;
  if (a.hgrp > 0 && !((p->flags & FM_FLAG_FWD_PAIR) && d.D == 128 && !d.rowwise)) {
    e = timed(FM_KERNEL_CLASSIFY, st, [&] { return fm::launch_order(w.fmap, d, 1, w.order, st); });
    if (e != cudaSuccess) return cuda_fail(e, "order");
    a.order = w.order;
  }
  a.scale_log2 = d.scale * 1.4426950408889634f;
  a.fmap = w.fmap;
  a.cw = refine ? w.cw : nullptr;
  a.vec4 = w.vec4;
  a.o = o;
  a.lse = lse;
  a.kmax = nullptr;
  a.fix_out = nullptr;
  a.fix = nullptr;
  a.q = q;
  // R33 bounded single pass (bf16 operands): key norms per tile (K1e), the single-pass forward, then
  // the persistent two-pass fixup over the units it flagged.  Used from N = 16K: on the few tiles of
  // a short unit its per-CTA bound set-up does not pay (C2 -4..-6 % when forced)
  // (column-wise masks only by default: row-wise ones keep the two-pass forward unless forced, see R33
  // on the precision of rows dominated by one key)
  const bool bounded = !d.in_f16 && (p->flags & FM_FLAG_NO_MAX_BOUND) == 0 &&
                       ((d.N >= 16384 && !d.rowwise) || (p->flags & FM_FLAG_MAX_BOUND) != 0);
  if (bounded) {
    e = timed(FM_KERNEL_KEYNORM, st, [&] { return fm::launch_key_norms(d, k, w.kmax, w.fix, st); });
    if (e != cudaSuccess) return cuda_fail(e, "key norms");
    a.kmax = w.kmax;
    a.fix_out = w.fix;
  }
  if ((p->flags & FM_FLAG_FWD_PAIR) && d.D == 128 && !d.rowwise) {
    CUtensorMap tk64;
    if (!make_map(&tk64, k, d, d.Hkv, 64, &err)) return fail(FM_ERR_CUDA, err);
    e = timed(FM_KERNEL_FWD, st, [&] { return fm::launch_fwd2(d, tq, tk64, tv, to, a, st); });
  } else {
    e = timed(FM_KERNEL_FWD, st, [&] { return fm::launch_fwd(d, tq, tk, tv, to, a, st); });
  }
  if (e != cudaSuccess) return cuda_fail(e, "forward kernel");
  if (bounded) {
    fm::FwdArgs f = a;
    f.kmax = nullptr;
    f.fix_out = nullptr;
    f.fix = w.fix;
    f.order = nullptr;
    e = timed(FM_KERNEL_FWD, st, [&] { return fm::launch_fwd(d, tq, tk, tv, to, f, st); });
    if (e != cudaSuccess) return cuda_fail(e, "forward fixup kernel");
  }
  return FM_OK;
}

fm_status flashmask_bwd(const fm_params* p, const void* q, const void* k, const void* v, const void* o,
                        const void* dout, const float* lse, const int32_t* sri, void* dq, void* dk, void* dv,
                        void* workspace, size_t workspace_bytes, void* stream) {
  g_last_error.clear();
  fm::Dims d{};
  fm_status s = check_params(p, &d, true);
  if (s != FM_OK) return s;
  if (!q || !k || !v || !o || !dout || !lse || !sri || !dq || !dk || !dv || !workspace)
    return fail(FM_ERR_INVALID_ARGUMENT, "NULL pointer argument");
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || !aligned16(dout) || !aligned16(sri) ||
      !aligned16(dq) || !aligned16(dk) || !aligned16(dv) || !aligned16(workspace))
    return fail(FM_ERR_INVALID_ARGUMENT, "tensor pointers and workspace must be 16-byte aligned");
  if (d.Trb > 4096) return fail(FM_ERR_UNSUPPORTED, "seqlen too large for the backward visit list");
  fm::Workspace w{};
  if (carve(d, FM_PASS_BWD, nullptr, &w) > workspace_bytes)
    return fail(FM_ERR_WORKSPACE_TOO_SMALL, "workspace smaller than flashmask_workspace_size(FM_PASS_BWD)");
  carve(d, FM_PASS_BWD, workspace, &w);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (p->in_dtype == FM_FP32) {  // fp32 inputs: fm_f32.cu (reading R26); deterministic by construction
    cudaError_t e = timed(FM_KERNEL_EXPAND, st, [&] { return fm::launch_expand(sri, d, fm::kTile, w.ext8, w.vec4, st); });
    if (e != cudaSuccess) return cuda_fail(e, "expand");
    e = timed(FM_KERNEL_CLASSIFY, st, [&] { return fm::launch_classify(w.ext8, d, fm::kTile, fm::kTile, w.fmap, 0, 1, nullptr, st); });
    if (e != cudaSuccess) return cuda_fail(e, "classify");
    fm::F32Args a = f32_args(d, w);
    a.q = static_cast<const float*>(q);
    a.k = static_cast<const float*>(k);
    a.v = static_cast<const float*>(v);
    a.dout = static_cast<const float*>(dout);
    a.o = const_cast<void*>(o);
    a.lse = const_cast<float*>(lse);
    a.dq = dq;
    a.dk = dk;
    a.dv = dv;
    e = timed(FM_KERNEL_DQ, st, [&] { return fm::launch_f32_dq(d, a, st); });
    if (e != cudaSuccess) return cuda_fail(e, "fp32 dq kernel");
    e = timed(FM_KERNEL_BWD, st, [&] { return fm::launch_f32_dkdv(d, a, st); });
    if (e != cudaSuccess) return cuda_fail(e, "fp32 dk/dv kernel");
    return FM_OK;
  }
  std::string err;
  CUtensorMap tq, tk, tv, tdo;
  if (!make_map(&tq, q, d, d.H, d.Brb, &err) || !make_map(&tk, k, d, d.Hkv, 128, &err) ||
      !make_map(&tv, v, d, d.Hkv, 128, &err) || !make_map(&tdo, dout, d, d.H, d.Brb, &err))
    return fail(FM_ERR_CUDA, err);
  cudaError_t e = timed(FM_KERNEL_EXPAND, st, [&] { return fm::launch_expand(sri, d, fm::kTile, w.ext8, w.vec4, st); });
  if (e != cudaSuccess) return cuda_fail(e, "expand");
  // row-wise: the backward map's rows are Brb-row tiles, whose extrema K1a computes separately
  const int32_t* ext_b = w.ext8;
  if (d.rowwise && d.Brb != fm::kTile) {
    e = timed(FM_KERNEL_EXPAND, st, [&] { return fm::launch_expand(sri, d, d.Brb, w.ext8b, nullptr, st); });
    if (e != cudaSuccess) return cuda_fail(e, "expand");
    ext_b = w.ext8b;
  }
  e = timed(FM_KERNEL_CLASSIFY, st, [&] { return fm::launch_classify(ext_b, d, d.Brb, fm::kTile, w.bmap, 1, 1, nullptr, st); });
  if (e != cudaSuccess) return cuda_fail(e, "classify");
  const int gsplit = gsplit_for(d);
  e = timed(FM_KERNEL_BWD_PRE, st, [&] { return fm::launch_bwd_pre(d, o, dout, lse, w.dvec, w.l2, w.dqacc, st); });
  if (e != cudaSuccess) return cuda_fail(e, "bwd preprocess");
  fm::BwdArgs a{};
  a.B = d.B; a.N = d.N; a.H = d.H; a.Hm = d.Hm; a.Tc = d.Tc; a.Trb = d.Trb; a.Npb = d.Npb;
  a.Hkv = d.Hkv; a.G = d.G;
  a.scale_log2 = d.scale * 1.4426950408889634f;
  a.scale = d.scale;
  a.bmap = w.bmap;
  a.vec4 = w.vec4;
  a.dvec = w.dvec;
  a.l2 = w.l2;
  a.dqacc = w.dqacc;
  a.dk = dk;
  a.dv = dv;
  a.gsplit = gsplit;
  a.dkv_part = w.dkv_part;
  const bool deterministic = (p->flags & FM_FLAG_DETERMINISTIC) != 0;
  a.with_dq = deterministic ? 0 : 1;
  CUtensorMap tdq, tdk, tdv;
  if (!make_dq_map(&tdq, w.dqacc, d, &err)) return fail(FM_ERR_CUDA, err);
  if (d.out_f32) {  // fp32 dK / dV are stored directly by the kernel (the maps are not used)
    tdk = tk;
    tdv = tv;
  } else if (!make_map(&tdk, dk, d, d.Hkv, 128, &err) || !make_map(&tdv, dv, d, d.Hkv, 128, &err)) {
    return fail(FM_ERR_CUDA, err);
  }
  e = timed(FM_KERNEL_BWD, st, [&] { return fm::launch_bwd(d, tq, tk, tv, tdo, tdq, tdk, tdv, a, st); });
  if (e != cudaSuccess) return cuda_fail(e, "backward kernel");
  if (gsplit > 1) {
    e = timed(FM_KERNEL_BWD, st, [&] { return fm::launch_dkv_reduce(d, gsplit, w.dkv_part, dk, dv, st); });
    if (e != cudaSuccess) return cuda_fail(e, "dk/dv reduce");
  }
  if (!deterministic) {
    e = timed(FM_KERNEL_DQ_CONVERT, st, [&] { return fm::launch_dq_convert(d, w.dqacc, dq, st); });
    if (e != cudaSuccess) return cuda_fail(e, "dq convert");
    return FM_OK;
  }
  // deterministic dQ: row-parallel recomputation (K6) over the forward class map
  CUtensorMap tq128, tdo128;
  if (!make_map(&tq128, q, d, d.H, 128, &err) || !make_map(&tdo128, dout, d, d.H, 128, &err))
    return fail(FM_ERR_CUDA, err);
  e = timed(FM_KERNEL_CLASSIFY, st, [&] { return fm::launch_classify(w.ext8, d, fm::kTile, fm::kTile, w.fmap, 0, 1, nullptr, st); });
  if (e != cudaSuccess) return cuda_fail(e, "classify");
  fm::DqArgs qa{};
  qa.B = d.B; qa.N = d.N; qa.H = d.H; qa.Hm = d.Hm; qa.G = d.G; qa.Tr = d.Tr; qa.Tc = d.Tc; qa.Npb = d.Npb;
  qa.rowwise = d.rowwise;
  qa.scale_log2 = a.scale_log2;
  qa.scale = d.scale;
  qa.fmap = w.fmap;
  qa.vec4 = w.vec4;
  qa.dvec = w.dvec;
  qa.l2 = w.l2;
  qa.dq = dq;
  e = timed(FM_KERNEL_DQ, st, [&] { return fm::launch_dq(d, tq128, tk, tv, tdo128, qa, st); });
  if (e != cudaSuccess) return cuda_fail(e, "deterministic dq kernel");
  return FM_OK;
}

fm_status flashmask_sliding_window_indices(int64_t batch, int64_t seqlen, int64_t window, int32_t causal,
                                          int32_t* sri, void* stream) {
  g_last_error.clear();
  if (!sri) return fail(FM_ERR_INVALID_ARGUMENT, "startend_row_indices is NULL");
  if (!aligned16(sri)) return fail(FM_ERR_INVALID_ARGUMENT, "startend_row_indices must be 16-byte aligned");
  if (batch < 1 || batch > 65535 || seqlen < 1 || seqlen > (1LL << 30) || window < 1 || (causal != 0 && causal != 1))
    return fail(FM_ERR_INVALID_ARGUMENT, "need batch in [1, 65535], seqlen in [1, 2^30], window >= 1, causal 0/1");
  const int w = static_cast<int>(window > seqlen ? seqlen : window);
  cudaError_t e = fm::launch_sliding_window(static_cast<int>(batch), static_cast<int>(seqlen), w, causal, sri,
                                            static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "sliding window indices");
  return FM_OK;
}

fm_status flashmask_timing_enable(int enable) {
  g_timing.on = enable != 0;
  g_timing.mask = (enable & FM_TIMING_SELECT) ? static_cast<uint32_t>(enable & 0xFFFF) : 0xFFFFFFFFu;
  return FM_OK;
}

fm_status flashmask_timing_collect(double* ms, int64_t* launches) {
  g_last_error.clear();
  if (!ms || !launches) return fail(FM_ERR_INVALID_ARGUMENT, "ms and launches are required");
  fm_status s = FM_OK;
  for (TimingRec& r : g_timing.recs) {
    float t = 0.f;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e == cudaSuccess) e = cudaEventElapsedTime(&t, r.a, r.b);
    if (e != cudaSuccess && s == FM_OK) s = cuda_fail(e, "timing");
    if (r.kid >= 0 && r.kid < FM_NUM_KERNELS) {
      ms[r.kid] += t;
      launches[r.kid] += 1;
    }
    g_timing.pool.push_back(r.a);
    g_timing.pool.push_back(r.b);
  }
  g_timing.recs.clear();
  return s;
}

}  // extern "C"

