/* tatn_b200.h — C ABI of the B200 (sm_100a) FlashAttention hot path.
 *
 * This is the drop-in boundary for the reference's tiled engine
 * (reference proj/core/include/tatn/flash.hpp:43-73):
 *
 *   tatn_fwd  replaces the body of  tatn::flash_forward      (flash.hpp:49-51)
 *                              and  tatn::blocksparse_forward (flash.hpp:64-67)
 *   tatn_bwd  replaces the body of  tatn::flash_backward      (flash.hpp:58-59)
 *                              and  tatn::blocksparse_backward(flash.hpp:71-73)
 *
 * The reference computes one head per call on row-major n x d fp64 matrices
 * (SPEC.md:185). This ABI batches B x H independent heads per call on 16-bit
 * device buffers (row-major in d, arbitrary b/h/n strides), which is how the
 * C++ wrapper (tatn::flash_forward in csrc/dropin) and the bench call it.
 *
 * Conventions (mirroring the reference's exception classes, flash.hpp:47-48):
 *   - every entry point returns a tatn_status; no exceptions cross the ABI;
 *   - no allocation and no host synchronisation on the hot path; the caller
 *     provides device buffers and (for the backward) a workspace;
 *   - stream-ordered on the caller's stream (a cudaStream_t passed as void*);
 *   - there is no CPU fallback: without an sm_100 device every compute entry
 *     point returns TATN_E_CUDA.
 */
#ifndef TATN_B200_H_
#define TATN_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TATN_B200_ABI_VERSION 4

typedef enum {
  TATN_OK = 0,
  TATN_E_ARG = 1,          /* null pointer / malformed descriptor        (std::invalid_argument) */
  TATN_E_SHAPE = 2,        /* B,H,N,d or stride mismatch                 (std::invalid_argument) */
  TATN_E_MASK = 3,         /* block-mask size / plan mismatch            (std::invalid_argument) */
  TATN_E_UNSUPPORTED = 4,  /* valid for the reference, not on this path  (e.g. Custom masks)     */
  TATN_E_CUDA = 5,         /* CUDA runtime / launch failure or no sm_100 device                 */
  TATN_E_WORKSPACE = 6     /* workspace too small                                                */
} tatn_status;

/* Input types. BF16 / FP16: the throughput path (kind::f16 MMAs, fp32 accumulate).
 * FP32 (ABI v4): the fp32-input check mode — q, k, v, dO are read as fp32 by TMA and
 * multiplied on the tensor cores as tf32 (kind::tf32, fp32 accumulate; P and dS rounded to
 * tf32 on chip); every output (o, dq, dk, dv) is fp32 and the backward reads o as fp32.
 * One CTA per tile, no pipelining: a precision mode for the reference's fp32 oracle shape
 * (BASELINE configs[0]), not a throughput path. FP32 is also an output type of
 * tatn_merge_partials. */
typedef enum { TATN_DTYPE_BF16 = 0, TATN_DTYPE_FP16 = 1, TATN_DTYPE_FP32 = 2 } tatn_dtype;

/* Output precision of 16-bit inputs: O (forward) and dQ/dK/dV (backward) are written either in
 * the 16-bit input dtype or in fp32 (no output rounding; the backward then also reads O as
 * fp32). The MMAs take the 16-bit inputs and accumulate in fp32. Ignored for FP32 inputs
 * (outputs are fp32). */
typedef enum { TATN_OUT_INPUT_DTYPE = 0, TATN_OUT_FP32 = 1 } tatn_out_dtype;

/* tatn::MaskKind (attn_config.hpp:12). Causal masks key j > query i;
 * KeyPadding masks key j >= valid_len[b]; Custom masks (i, j) where the additive
 * pattern is -inf (attn_config.cpp:20-32), given as the bit-packed custom_mask below. */
typedef enum {
  TATN_MASK_NONE = 0,
  TATN_MASK_CAUSAL = 1,
  TATN_MASK_KEY_PADDING = 2,
  TATN_MASK_CUSTOM = 3
} tatn_mask_kind;

typedef struct {
  int32_t B, H;      /* independent (batch, head) slices, each 1..65535           */
  int32_t Nq, Nk;    /* query rows, key rows (Nk <= Nq: key prefix, reference.hpp:43-46) */
  int32_t d;         /* head dimension: 64 or 128                                 */
  int32_t dtype;     /* tatn_dtype of q, k, v, dO (BF16, FP16 or FP32)            */
  int32_t out_dtype; /* tatn_out_dtype of o, dq, dk, dv                           */
  /* element strides of the b, h, n dimensions; d is contiguous (stride 1).
   * dO uses o_str; dQ/dK/dV use q_str/k_str/v_str. Strides must be multiples of 8. */
  int64_t q_str[3], k_str[3], v_str[3], o_str[3];
  float tau;               /* softmax scale, finite and > 0 (attn_config.cpp:52)        */
  int32_t mask_kind;       /* tatn_mask_kind                                            */
  const int32_t* valid_len;/* device [B] for KEY_PADDING, else NULL                    */
  /* Block-sparse mode (tatn::BlockMask, block_mask.hpp:14-24): row-major u8 tr x tc
   * grid in DEVICE memory, or NULL for dense. br, bc must both be 128 and
   * tr = ceil(Nq/128), tc = ceil(Nk/128). In dense mode tr/tc may be 0. */
  const uint8_t* block_grid;
  int32_t br, bc, tr, tc;
  /* optional device bitmap of tr*tc bits (bit = i*tc + j), OR-ed with the tiles
   * the kernels actually computed; must be zeroed by the caller. NULL = off. */
  uint32_t* visited_bitmap;
  /* Dropout (tatn::dropout_scale, dropout.cpp:7-27): element (i, j) of slice (b, h) is
   * kept iff the top 53 bits of mix64(mix64(mix64(seed + b*H + h) ^ (i+1)) ^ ((j+1) << 1))
   * * 2^-53 >= p_drop, and then scaled by 1/(1 - p_drop); slice 0 uses `seed` itself,
   * so a one-head call reproduces the reference's mask bit for bit. p_drop in [0, 1). */
  double p_drop;
  uint64_t seed;
  /* Custom mask (MaskSpec::custom_additive, attn_config.hpp:27; ABI v3): bit-packed keep
   * matrix in DEVICE memory, row-major [Nq][custom_words] uint32 per batch element: bit
   * (j & 31) of word (j >> 5) of row i is 1 iff custom(i, j) == 0 (keep), 0 iff -inf.
   * custom_words >= 4 * ceil((k_offset + Nk) / 128) (the kernels read word (k_offset + j) / 32,
   * 16 bytes per 128-key tile) and a multiple of 4; custom_bstride = words between batch
   * elements (0: one mask shared by every slice). NULL unless mask_kind == CUSTOM. */
  const uint32_t* custom_mask;
  int32_t custom_words;
  int64_t custom_bstride;
  /* Sequence-parallel key shard (ABI v3): key j of this call is global key
   * k_offset + j of an Nq-long sequence, for the causal / key-padding / custom predicates and
   * the dropout hash. 0 for ordinary calls; else a multiple of 128 with k_offset + Nk <= Nq and
   * no block grid. Partial (o, lse) pairs of the shards combine with tatn_merge_partials. */
  int32_t k_offset;
  /* Deterministic dQ (ABI v4): 0 = dQ partials of the key tiles are added into one fp32
   * accumulator with atomic reductions (fastest; the summation order, and so the last bits of
   * dQ, vary run to run); 1 = each key tile stores its partial in its own workspace slot and K4
   * sums them in key-tile order, so dQ is bit-reproducible and an all-true block grid gives
   * exactly the dense dQ (flash.hpp:62-63). The backward workspace grows by
   * ceil(Nk/128) x B x H x Nq_pad x d x 4 bytes (practical for N <= 8K). O, LSE, dK, dV are
   * deterministic in both modes. */
  int32_t deterministic;
} tatn_attn_desc;

/* Merge R partial attention results over disjoint key shards (merge_stats, softmax.hpp:48-59,
 * softmax.cpp:62-83, in log form): per row m = max_r lse_r, w_r = exp(lse_r - m),
 * o = sum_r w_r o_r / sum_r w_r, lse = m + ln(sum_r w_r); rows with every lse_r = -inf give
 * o = 0, lse = -inf. o_parts: fp32 [R][B][H][Nq][d] contiguous (each shard's tatn_fwd output in
 * TATN_OUT_FP32 mode); lse_parts: fp32 [R][B][H][Nq]. o: o_dtype with element strides o_str of
 * b, h, n (d contiguous); lse: fp32 [B][H][Nq]. The exchange that brings the partials together
 * (NCCL all-gather) is the caller's. */
int tatn_merge_partials(int32_t R, int32_t B, int32_t H, int32_t Nq, int32_t d, const float* o_parts,
                        const float* lse_parts, void* o, int32_t o_dtype, const int64_t o_str[3], float* lse,
                        void* stream);

/* Host-only descriptor check (no device access); same codes as the compute calls. */
int tatn_validate(const tatn_attn_desc* desc);

/* Workspace of tatn_fwd (ABI v4): 16 bytes, 16-byte aligned — the persistent kernels' work-item
 * counter. It must be zero before its first use (e.g. cudaMemset once); every tatn_fwd leaves it
 * zero again when its kernel completes, so a workspace is reused without re-zeroing. Calls
 * that may run concurrently (different streams, graphs replayed side by side) need distinct
 * workspaces; there is no global state in the library. */
size_t tatn_fwd_workspace_bytes(const tatn_attn_desc* desc);

/* Forward: o = softmax(mask(tau q k^T)) v, lse = natural-log logsumexp per row
 * ([B, H, Nq] contiguous fp32; -inf and o = 0 for fully masked rows). */
int tatn_fwd(const tatn_attn_desc* desc, const void* q, const void* k, const void* v, void* o,
             float* lse, void* workspace, size_t workspace_bytes, void* stream);

/* Workspace for tatn_bwd: fp32 dQ accumulator [B,H,Nq_pad,d] + lse2 and D vectors
 * [B,H,Nq_pad], Nq_pad = Nq rounded up to 128, + 16 bytes (persistent scheduler counter)
 * + for CUSTOM masks the transposed bit mask [B or 1][Nk][Nq_pad/32] uint32. */
size_t tatn_bwd_workspace_bytes(const tatn_attn_desc* desc);

/* Backward with recomputation from lse (Algorithm 4).
 * Writes dq, dk, dv (same dtype/strides as q, k, v). Keys covered by no
 * visited tile get exactly zero dK/dV (flash.hpp:70). */
int tatn_bwd(const tatn_attn_desc* desc, const void* q, const void* k, const void* v,
             const void* o, const void* dO, const float* lse, void* dq, void* dk, void* dv,
             void* workspace, size_t workspace_bytes, void* stream);

const char* tatn_strerror(int status);
int tatn_abi_version(void);

/* Number of device kernels the last tatn_fwd / tatn_bwd call on this thread launched. */
int tatn_last_launch_count(void);

/* Optional measurement hook, off by default. While enabled, tatn_fwd and tatn_bwd
 * record CUDA events on the caller's stream around their main kernel (K1 forward,
 * K3 backward). tatn_profile_read synchronises on the recorded events and returns
 * the summed device milliseconds and launch count for `which` (0 = K1, 1 = K3)
 * since the previous read, then resets that counter. */
int tatn_profile_enable(int on);
int tatn_profile_read(int which, double* total_ms, int* launches);

#ifdef __cplusplus
}
#endif

#endif /* TATN_B200_H_ */
