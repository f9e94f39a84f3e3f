/*
 * flashmask.h — C ABI of the B200 (sm_100a) FlashMask hot path.
 *
 * FlashMask (arXiv 2410.01359, /root/reference/PAPER.md) computes exact masked
 * attention  O = Softmax(scale * Q K^T + M) V  (Eq. 1, Eq. 2) and its
 * gradients, where M is never materialised: every key column y carries at most two
 * masked row intervals [LTS_y, LTE_y) and [UTS_y, UTE_y) (Eq. 3, §4.1
 * P:118-127).  A per-column-tile min/max preprocessing (Alg. 1 lines 3-4)
 * classifies every tile as fully masked (skipped before any load), partially masked
 * (masked element-wise) or unmasked (Eq. 4, Alg. 1).
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - All tensor pointers are DEVICE pointers owned by the caller; nothing is
 *    allocated inside the library.  `stream` is a cudaStream_t passed as void*
 *    (NULL = legacy default stream).  Every call is asynchronous on `stream`;
 *    no device synchronisation happens inside; asynchronous faults surface at the
 *    caller's next synchronisation.
 *  - Argument errors are detected on the host before anything is launched and are
 *    returned as FM_ERR_INVALID_ARGUMENT / FM_ERR_UNSUPPORTED /
 *    FM_ERR_WORKSPACE_TOO_SMALL; launch failures return FM_ERR_CUDA.  The detail
 *    of the last non-OK status of the calling thread is in flashmask_last_error().
 *    No C++ exception crosses the ABI.  There is no fallback path.
 *  - The library is stateless and re-entrant (a call_once device-attribute and
 *    driver-entry-point cache is its only global state).
 *  - Kernels are launched with programmatic dependent launch: each may begin while
 *    its stream predecessor drains, but touches no memory an earlier kernel on the
 *    stream writes or reads before that kernel has completed (griddepcontrol.wait),
 *    so stream order semantics are unchanged for the caller.
 *  - q, o, dout, dq: [batch, seqlen, num_heads, head_dim]; k, v, dk, dv: [batch, seqlen,
 *    num_kv_heads, head_dim] (grouped-query attention: query head h reads key/value head
 *    h / (num_heads / num_kv_heads)); all contiguous and 16-byte aligned.
 *    lse: [batch, num_heads, seqlen] fp32, natural log of the scaled logits (Alg. 1 line 28); -inf for a row masked in every column
 *    (then its O row is 0 and it contributes nothing to the gradients; R7).
 *  - startend_row_indices: int32 [batch, mask_heads, seqlen, C], 16-byte aligned.
 *    Column y = key token y.  Columns by (causal, C), missing vectors defaulted:
 *
 *        causal  C   col0  col1  col2  col3   implicit
 *        1       1   LTS   -     -     -      LTE = N, plus the r < y triangle
 *        1       2   LTS   LTE   -     -      plus the r < y triangle
 *        0       2   LTS   UTE   -     -      LTE = N, UTS = 0
 *        0       4   LTS   LTE   UTS   UTE    -
 *
 *    masked(r, y) = LTS_y <= r < LTE_y  or  UTS_y <= r < UTE_y  or  (causal and r < y).
 *    Any int32 value is accepted (start >= end is an empty interval); values are only
 *    compared, never used as addresses.  Self-attention only (query length = key
 *    length = seqlen).
 */
#ifndef FLASHMASK_H_
#define FLASHMASK_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define FM_API __attribute__((visibility("default")))
#else
#define FM_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FM_OK = 0,
  FM_ERR_INVALID_ARGUMENT = 1,   /* null / misaligned pointer, bad shape or combination */
  FM_ERR_UNSUPPORTED = 2,        /* valid request this build does not implement          */
  FM_ERR_WORKSPACE_TOO_SMALL = 3,
  FM_ERR_CUDA = 4                /* a CUDA runtime/driver call or launch failed          */
} fm_status;

typedef enum { FM_BF16 = 0, FM_FP32 = 1, FM_FP16 = 2 } fm_dtype;

/* Tile classes of Eq. 4, as written to class maps. */
typedef enum { FM_TILE_SKIP = 0, FM_TILE_PARTIAL = 1, FM_TILE_UNMASKED = 2 } fm_tile_class;

/* fm_params.flags bits. */
enum {
  /* Debug: visit SKIP tiles as PARTIAL (masked element-wise).  The outputs must be
   * bitwise identical to the default run — the exactness claim of §4.4. */
  FM_FLAG_NO_SKIP = 1,
  /* flashmask_bwd: compute dQ row-parallel in a separate kernel that accumulates over the key
   * tiles in ascending order on chip (no fp32 atomics), so dq is bitwise reproducible run to
   * run ("deterministic control").  Costs two extra GEMMs per visited tile. */
  FM_FLAG_DETERMINISTIC = 2,
  /* flashmask_fwd: do not run the f3 refinement (K1c, flashmask_refine below); every element of
   * a PARTIAL tile is then masked element-wise as in Alg. 1 lines 15-21.  Outputs are bitwise
   * identical either way (masking a sub-block with no masked cell changes nothing). */
  FM_FLAG_NO_REFINE = 4,
  /* flashmask_fwd, head_dim 128: run the forward on CTA pairs (K2b, tcgen05 cta_group::2: each
   * SM holds one query tile and half of every K/V tile, three S accumulators in TMEM) instead of
   * the single-SM kernel K2a.  Same results to rounding order (every output within the parity
   * tolerances of the single-SM kernel); with bf16 operands it takes the bounded single pass of
   * FM_FLAG_NO_MAX_BOUND's description under the same conditions as K2a. */
  FM_FLAG_FWD_PAIR = 8,
  /* Row-wise representation ("by transposing the attention matrix, we can obtain a row-wise
   * representation using column index intervals"; R32): startend_row_indices[b, hm, r, .]
   * holds the masked KEY column intervals of query row r, masked(r, y) = LTS_r <= y < LTE_r or
   * UTS_r <= y < UTE_r or (causal and r < y), with the mirrored (causal, C) table
   *     causal C=1: (LTE; LTS=0)   causal C=2: (LTS, LTE)
   *     non-causal C=2: (LTE, UTS; LTS=0, UTE=N)   non-causal C=4: (LTS, LTE, UTS, UTE).
   * Tiles are classified by Eq. 4 on the transposed problem (per-row-tile extrema against the
   * column range).  flashmask_classify then returns minmax per ROW tile ([B, Hm, Tr, 8], tile br).
   * Accepted by every entry point; FM_FLAG_FWD_PAIR is ignored with it (single-SM forward). */
  FM_FLAG_ROWWISE = 16,
  /* flashmask_fwd: always take each visited tile's row maximum before its exponentials (Alg. 1
   * line 242).  By default, with bf16 operands, column-wise masks and seqlen >= 16384, the single-SM
   * forward instead computes every P of a row against one fixed reference
   * m_r = ||q_r|| max_y ||k_y|| scale log2(e) - 96 (Cauchy-Schwarz bound of the row's logits; key
   * norms from one extra pass over K): no row maximum, no rescaling, one pass per tile; rows whose sum ends below
   * 2^-90 (bound too loose, or every key masked) are recomputed by the two-pass kernel
   * (R33).  Same outputs to rounding (parity tolerances). */
  FM_FLAG_NO_MAX_BOUND = 32,
  /* Testing: use the bounded single pass of FM_FLAG_NO_MAX_BOUND's description at any seqlen (bf16
   * operands).  Ignored together with FM_FLAG_NO_MAX_BOUND. */
  FM_FLAG_MAX_BOUND = 64
};

typedef struct {
  int64_t batch;       /* B >= 1                                                    */
  int64_t seqlen;      /* 1 <= N (queries = keys): N <= 262144 for the attention calls,
                        * N <= 2^30 and ceil(N / br) <= 4194240 for flashmask_classify;
                        * larger: FM_ERR_UNSUPPORTED                                 */
  int64_t num_heads;   /* H >= 1                                                    */
  int64_t head_dim;    /* d in {64, 128}                                            */
  int64_t mask_heads;  /* 1 (one mask per batch entry, broadcast) or num_kv_heads;
                        * batch * mask_heads <= 65535, else FM_ERR_UNSUPPORTED    */
  int64_t mask_cols;   /* C in {1, 2, 4}; must match `causal` per the table above   */
  int32_t causal;      /* 0 or 1                                                    */
  float   scale;       /* softmax scale; <= 0 means 1/sqrt(head_dim) (Eq. 1)        */
  int32_t in_dtype;    /* fm_dtype of q, k, v, dout: FM_BF16 or FM_FP16 (tcgen05 path) or
                        * FM_FP32 (exact-fp32 CUDA-core path for the parity config C1, reading R26) */
  int32_t out_dtype;   /* fm_dtype of o, dq, dk, dv: FM_FP32 or the 16-bit type of in_dtype
                        * (FM_BF16 for FM_BF16 / FM_FP32 inputs, FM_FP16 for FM_FP16 inputs) */
  int32_t flags;       /* FM_FLAG_*                                                 */
  int64_t num_kv_heads;/* key/value heads; 0 means num_heads; must divide num_heads   */
} fm_params;

enum { FM_PASS_FWD = 0, FM_PASS_BWD = 1 };

/* Bytes of device workspace flashmask_fwd (pass = FM_PASS_FWD) or flashmask_bwd
 * (FM_PASS_BWD) needs for these params: the expanded mask vectors and their per-tile
 * extrema (Alg. 1 line 4), the kernels' tile-class maps, and for the backward the
 * per-row D = rowsum(dO o O) (Alg. 2 line 4), a log2-scaled copy of lse and the
 * fp32 dQ accumulator (Alg. 2 line 3).  O(N * (1 + H * d) + T_r * T_c) per batch
 * entry.  Returns 0 for invalid params (see flashmask_last_error()). */
FM_API size_t flashmask_workspace_size(const fm_params* p, int pass);

/* Preprocessing + tile classification (Alg. 1 lines 3-4 P:210-211; Eq. 4 P:143-150 with
 * Alg. 1's skip tests P:220-226 and partial tests P:232-240, 0-based, causal region as a
 * third triangle).  Tiles are br x bc (br, bc >= 1); ragged last tiles use their real
 * extents.  Outputs (device pointers):
 *   minmax     int32 [B, Hm, Tc, 8], required: per column tile the min and max over its
 *              real columns of LTS, LTE, UTS, UTE (order LTSmin, LTSmax, LTEmin, LTEmax,
 *              UTSmin, UTSmax, UTEmin, UTEmax), with the table's defaults filled in.
 *   class_map  uint8 [B, Hm, Tr, Tc] fm_tile_class, or NULL.
 *   counts     int64 [B, Hm, 3] = (#SKIP, #PARTIAL, #UNMASKED), or NULL.
 *   row_nonskip int32 [B, Hm, Tr]: per row tile the number of non-SKIP tiles in that row, or NULL.
 *   col_nonskip int32 [B, Hm, Tc]: per column tile the number of non-SKIP tiles in that column,
 *              or NULL.  These are the per-unit work figures O((1-rho) T_r T_c) of P:262 that
 *              order the forward's row units and the backward's column units.
 * Tr = ceil(N / br), Tc = ceil(N / bc).  The class map and all counts use the true Eq. 4
 * classes (they ignore FM_FLAG_NO_SKIP).  Every output is written in full (no accumulation
 * into caller data). */
FM_API fm_status flashmask_classify(const fm_params* p, const int32_t* startend_row_indices, int32_t br, int32_t bc,
                             int32_t* minmax, uint8_t* class_map, int64_t* counts, int32_t* row_nonskip,
                             int32_t* col_nonskip, void* stream);

/* Tighter-than-Eq.-4 refinement (R31).  Eq. 4 classifies a tile from
 * the hulls of its columns' intervals, so a PARTIAL tile may contain large regions without any
 * masked cell.  For every 128 x 128 tile, the 32-bit word whose bit (8 g + c) is 1 iff the
 * sub-block of rows [128 i + 32 g, +32) x columns [128 j + 16 c, +16) (real rows / columns
 * only) holds a masked cell (masked(r, y) as in the header comment).  Inputs:
 *   startend_row_indices  as for flashmask_classify;
 *   class_map  uint8 [B, Hm, Tr, Tc] at 128 x 128 from flashmask_classify (br = bc = 128).
 * Outputs (device pointers):
 *   words      uint32 [B, Hm, Tr, Tc], required.
 *   counts     int64 [B, Hm, 2] = (#PARTIAL tiles without any masked cell, #dirty sub-blocks
 *              of PARTIAL tiles), or NULL.
 * flashmask_fwd runs the same refinement internally (unless FM_FLAG_NO_REFINE) and applies the
 * element mask only on the dirty sub-blocks of PARTIAL tiles. */
FM_API fm_status flashmask_refine(const fm_params* p, const int32_t* startend_row_indices, const uint8_t* class_map,
                                  uint32_t* words, int64_t* counts, void* stream);

/* Forward pass (Alg. 1): o = Softmax(scale*q k^T + M) v, lse = logsumexp.
 *   q, k, v  [B, N, H, d] in_dtype;  o [B, N, H, d] out_dtype;  lse fp32 [B, H, N].
 * in_dtype FM_BF16 / FM_FP16 runs the tcgen05 kernels (16-bit operands, fp32 accumulation);
 * FM_FP32 runs fp32 CUDA-core kernels with the same tile skipping (no tensor cores: it
 * serves the fp32 parity configuration, not throughput).
 * Fully masked tiles issue no load and no MMA; partially masked tiles are masked
 * element-wise; unmasked tiles do no mask work. */
FM_API fm_status flashmask_fwd(const fm_params* p, const void* q, const void* k, const void* v,
                        const int32_t* startend_row_indices, void* o, float* lse,
                        void* workspace, size_t workspace_bytes, void* stream);

/* Backward pass (Alg. 2): given dout = dL/do, writes dq, dk, dv
 * ([B, N, H, d], out_dtype).  o and lse must come from flashmask_fwd on the same inputs
 * (o in out_dtype).  dK/dV are accumulated per key tile on chip and written once
 * (column-parallel); dQ is reduced in fp32 in the workspace and
 * converted at the end.  Skipping and masking rules are those of the forward.
 * Determinism: by DEFAULT the dQ partial sums of the key tiles are added by fp32 hardware
 * reduce-adds in completion order, so dq may differ in the last bits from run to run (dk, dv
 * are always bitwise reproducible).  This deviates from SPEC S:305's ascending-j order on
 * purpose (speed; R25); set FM_FLAG_DETERMINISTIC for bitwise-reproducible dq. */
FM_API fm_status flashmask_bwd(const fm_params* p, const void* q, const void* k, const void* v, const void* o,
                        const void* dout, const float* lse, const int32_t* startend_row_indices,
                        void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes, void* stream);

/* Kernel ids of the optional per-launch timing below. */
enum {
  FM_KERNEL_EXPAND = 0,      /* K1a  preprocessing: expand + per-tile min/max (Alg. 1 l.3-4) */
  FM_KERNEL_CLASSIFY = 1,    /* K1b  tile classification (Eq. 4)                             */
  FM_KERNEL_FWD = 2,         /* K2   forward (Alg. 1)                                        */
  FM_KERNEL_BWD_PRE = 3,     /* K3   D = rowsum(dO o O), zero dQ accumulator (Alg. 2 l.3-4)  */
  FM_KERNEL_BWD = 4,         /* K4   backward main loop (Alg. 2); + K7 under split-G         */
  FM_KERNEL_DQ_CONVERT = 5,  /* K5   dQ = scale * dQacc -> out dtype                         */
  FM_KERNEL_DQ = 6,          /* K6   deterministic dQ (FM_FLAG_DETERMINISTIC)                */
  FM_KERNEL_REFINE = 7,      /* K1c  f3 refinement words of PARTIAL tiles                    */
  FM_KERNEL_KEYNORM = 8,     /* K1e  key norms per key tile for the bounded forward (R33)    */
  FM_NUM_KERNELS = 9
};

/* Optional per-kernel timing for roofline reporting (off by default).  enable = 0: off;
 * 1: every kernel this thread launches through the calls above is bracketed by two CUDA
 * events recorded on the caller's stream (no extra synchronisation, same stream order);
 * FM_TIMING_SELECT | mask: only kernels whose id bit (1 << FM_KERNEL_*) is in mask.
 * All kernels are launched with programmatic dependent launch (each may start while its
 * stream predecessor drains); an event between two kernels removes that overlap, so time
 * only the kernels you need when the step time matters.
 * flashmask_timing_collect() waits for the recorded events, ADDS the elapsed
 * milliseconds and the launch counts per kernel id into ms[FM_NUM_KERNELS] and
 * launches[FM_NUM_KERNELS] (caller-owned host arrays), and clears the record. */
#define FM_TIMING_SELECT 0x10000
FM_API fm_status flashmask_timing_enable(int enable);
FM_API fm_status flashmask_timing_collect(double* ms, int64_t* launches);

/* Sliding-window shortcut (the sliding-window family of Fig. 1 / §2.1):
 * writes startend_row_indices for a window of `window` keys without the caller building
 * the vectors.  causal = 1: int32 [batch, 1, seqlen, 1], LTS_y = min(y + window, seqlen)
 * (row r sees keys r-window+1 .. r); causal = 0: int32 [batch, 1, seqlen, 2],
 * (LTS_y, UTE_y) = (min(y + window, seqlen), max(y - window + 1, 0)) (row r sees keys with
 * |r - y| < window).  window >= 1, seqlen >= 1; out is a 16-byte-aligned device buffer
 * owned by the caller.  Asynchronous on `stream`; FM_ERR_INVALID_ARGUMENT otherwise. */
FM_API fm_status flashmask_sliding_window_indices(int64_t batch, int64_t seqlen, int64_t window, int32_t causal,
                                                  int32_t* startend_row_indices, void* stream);

/* Static description of a status code. */
FM_API const char* flashmask_status_string(fm_status s);

/* Thread-local detail message for the calling thread's last non-OK status ("" if none). */
FM_API const char* flashmask_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* FLASHMASK_H_ */
