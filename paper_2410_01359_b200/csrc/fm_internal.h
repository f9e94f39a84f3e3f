// fm_internal.h — host/device structures shared by the FlashMask kernels and the C-ABI layer.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include <utility>

namespace fm {

// Launch with programmatic stream serialization (PDL): the kernel may start while its stream
// predecessor drains; it must call pdl_wait() (fm_ptx.cuh) before touching dependent memory.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

constexpr int kTile = 128;      // column (key) tile Bc, forward row (query) tile Br
constexpr int kMaxTc = 2048;    // forward visit-list capacity -> N <= 262144
// rows of one d=64 dQ TMA reduce box (x 32 fp32 columns, 128-B swizzle; fm_bwd.cu)
constexpr int kDq64BoxRows = 128;

// Workspace layout (buffers 4 KiB-aligned in the device address space), produced by flashmask_fwd/bwd.
struct Workspace {
  int32_t* ext8;    // [B, Hm, Tc, 8] raw extrema (Alg. 1 line 4); row-wise: per 128-row tile
  int32_t* ext8b;   // row-wise backward: [B, Hm, Trb, 8] extrema per Brb-row tile
  int4* vec4;       // [B, Hm, Tc*128] normalised (LTS, LTE, UTS, UTE) per column, padded columns masked
  uint8_t* fmap;    // [B, Hm, Tr, Tc] forward kernel map (128 x 128)
  uint32_t* cw;     // [B, Hm, Tr, Tc] f3 refinement words of the forward map (K1c; PARTIAL tiles)
  uint8_t* bmap;    // [B, Hm, Tc, Trb] backward kernel map, transposed (Brb x 128)
  float* dvec;      // [B, H, Npb] -D, D = rowsum(dO o O) (negated: consumers add it)
  float* l2;        // [B, H, Npb] -lse * log2(e) (-inf for empty / padded rows)
  float* dqacc;     // [B, H, Npb, d] fp32 dQ accumulator
  float* dkv_part;  // split-G backward: [gsplit][2][B, N, Hkv, d] fp32 dV / dK partials
  uint16_t* order;  // LPT unit order (K1d): forward [B, Hm, ceil(Tr/2)] pairs, backward [B, Hm, Tc] key
                    // tiles, then one flag per (b, hm) (0: near-uniform work, keep the default order)
  float* kmax;      // forward: [B, Hkv, Tc] largest key norm per 128-key tile (K1e, R33)
  uint8_t* fix;     // forward: [B, H, ceil(Tr/2)] units the bounded single pass could not finish (R33)
  size_t bytes;
};

struct Dims {
  int B, N, H, D, Hm, C, causal;
  int Hkv, G;       // key/value heads, query heads per key/value head
  int Tr, Tc;       // 128-row / 128-column tile counts
  int Brb, Trb, Npb;  // backward row tile, its count, padded rows (a multiple of 128)
  float scale;
  int out_f32;
  int in_f16;       // 16-bit operands (and 16-bit outputs) are fp16 instead of bf16
  int flags;
  int rowwise;      // FM_FLAG_ROWWISE: vectors indexed by query row, values = key intervals (R32)
};

// R33 bounded single pass: the fixed reference sits kBndHeadroom (log2 units) below the
// Cauchy-Schwarz bound, so every P <= 2^96 (bf16 / fp32 sums of <= 2^18 terms of |v| < 2^13 stay
// finite); a row whose sum ends below kBndMinSum (its largest P < 2^-90, still 2^36 above the fp32
// normal range) is recomputed by the two-pass fixup.  A row fails only when the bound exceeds its
// true maximum by more than ~186 log2 units.
constexpr float kBndHeadroom = 96.0f;
constexpr float kBndMinSum = 0x1p-90f;

struct FwdArgs {
  int B, N, H, Hm, Tr, Tc, G;
  float scale_log2;
  const uint8_t* fmap;
  const uint32_t* cw;  // f3 refinement words (nullptr: every sub-block of a PARTIAL tile is masked)
  const int4* vec4;    // normalised (start, len, start, len) per key column, or per query row (row-wise)
  void* o;
  float* lse;
  // LPT schedule (small problems): query-tile pairs of each (b, hm) by descending work (K1d), the
  // CTA -> (head, pair) map taking `hgrp` heads at a time; nullptr: last pairs first per head
  const uint16_t* order;
  int hgrp;
  // R33 bounded single pass: [B, Hkv, Tc] largest key norm per key tile (K1e) and the per-unit
  // flags it raises for rows it cannot finish (fix_out); the two-pass fixup launch runs only the
  // flagged units (fix != nullptr)
  const float* kmax;
  uint8_t* fix_out;
  const uint8_t* fix;
  const void* q;  // Q itself (K2b's bounded pass reads ||q_r|| from it)
};

struct BwdArgs {
  int B, N, H, Hm, Tc, Trb, Npb, Hkv, G;
  float scale_log2;
  float scale;
  const uint8_t* bmap;
  const int4* vec4;
  const float* dvec;
  const float* l2;
  float* dqacc;
  void* dk;
  void* dv;
  int with_dq;  // 0 under FM_FLAG_DETERMINISTIC: dQ comes from K6 instead
  int gsplit;             // > 1: query heads of a group split over gsplit CTAs (fp32 partials, K7)
  float* dkv_part;        // [gsplit][2 (dV, dK)][B, N, Hkv, d] fp32 partials when gsplit > 1
};

struct DqArgs {
  int B, N, H, Hm, G, Tr, Tc, Npb, rowwise;
  float scale_log2;
  float scale;
  const uint8_t* fmap;
  const int4* vec4;
  const float* dvec;
  const float* l2;
  void* dq;
};

// FP32-input path (fm_f32.cu): plain fp32 tensors, same layouts as the bf16 path
struct F32Args {
  int B, N, H, Hm, Hkv, G, Tr, Tc, Npb, causal, rowwise;
  float scale;
  const uint8_t* fmap;  // [B, Hm, Tr, Tc] 128 x 128 kernel map
  const int4* vec4;
  const float *q, *k, *v, *dout;
  void* o;        // forward output (out dtype): written by the forward, read by the backward
  float* lse;
  float* dvec;    // [B, H, Npb] D_r, written by f32_dq_kernel, read by f32_dkdv_kernel
  void *dq, *dk, *dv;
};

// launchers (return cudaError_t of the launch)
// K1a: C-table -> normalised vec4 (when non-null) and min/max per tile of `bc` vector entries
// (key columns; query rows under Dims::rowwise)
cudaError_t launch_expand(const int32_t* sri, const Dims& d, int bc, int32_t* ext8, int4* vec4, cudaStream_t st);
cudaError_t launch_sliding_window(int B, int N, int w, int causal, int32_t* sri, cudaStream_t st);
cudaError_t launch_classify(const int32_t* ext8, const Dims& d, int br, int bc, uint8_t* map, int transposed,
                            int kernel_map, int64_t* counts, cudaStream_t st, int32_t* row_cnt = nullptr,
                            int32_t* col_cnt = nullptr);
cudaError_t launch_refine(const int32_t* sri, const uint8_t* cmap, const Dims& d, uint32_t* words, int64_t* rcounts,
                          cudaStream_t st);
// K1d: LPT order of the forward's units (pairs of row tiles) from its class map
cudaError_t launch_order(const uint8_t* map, const Dims& d, int fwd, uint16_t* order, cudaStream_t st);
cudaError_t launch_fwd(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                       const CUtensorMap& to, const FwdArgs& a, cudaStream_t st);
cudaError_t launch_fwd2(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk64, const CUtensorMap& tv,
                        const CUtensorMap& to, const FwdArgs& a, cudaStream_t st);
cudaError_t launch_bwd_pre(const Dims& d, const void* o, const void* dout, const float* lse, float* dvec, float* l2,
                           float* dqacc, cudaStream_t st);
cudaError_t launch_bwd(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                       const CUtensorMap& tdo, const CUtensorMap& tdq, const CUtensorMap& tdk, const CUtensorMap& tdv,
                       const BwdArgs& a, cudaStream_t st);
cudaError_t launch_dq_convert(const Dims& d, const float* dqacc, void* dq, cudaStream_t st);
cudaError_t launch_key_norms(const Dims& d, const void* k, float* kmax, uint8_t* fix, cudaStream_t st);
// K7: dK = scale * sum_s dK_s, dV = sum_s dV_s over the split-G partials, converted to the out dtype
cudaError_t launch_dkv_reduce(const Dims& d, int gsplit, const float* part, void* dk, void* dv, cudaStream_t st);
cudaError_t launch_dq(const Dims& d, const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                      const CUtensorMap& tdo, const DqArgs& a, cudaStream_t st);

cudaError_t launch_f32_fwd(const Dims& d, const F32Args& a, cudaStream_t st);
cudaError_t launch_f32_dq(const Dims& d, const F32Args& a, cudaStream_t st);
cudaError_t launch_f32_dkdv(const Dims& d, const F32Args& a, cudaStream_t st);

}  // namespace fm
