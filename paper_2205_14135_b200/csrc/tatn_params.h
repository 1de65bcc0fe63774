// tatn_params.h — kernel parameter blocks shared by the host launcher
// (tatn_capi.cu) and the device kernels. Plain-old-data only.
#pragma once
#include <cstdint>

namespace tatn_dev {

// Mirrors tatn::MaskKind (reference attn_config.hpp:12).
enum MaskKindDev : int { kMaskNone = 0, kMaskCausal = 1, kMaskKeyPadding = 2, kMaskCustom = 3 };

struct FwdParams {
  int B, H, Nq, Nk;
  float scale_log2;          // tau * log2(e): scores are kept in the log2 domain
  int mask_kind;             // MaskKindDev
  const int32_t* valid_len;  // [B] (KeyPadding) or nullptr
  const uint8_t* grid;       // block-sparse grid tr x tc at 128x128 tiles, or nullptr (dense)
  int tr, tc;                // tile counts (always set; grid dims when grid != nullptr)
  uint32_t* visited;         // optional tr*tc bitmap of tiles the kernel computed
  float* lse;                // [B, H, Nq] natural-log logsumexp (fp32)
  int n_pairs;               // ceil(Nq / 256): CTAs per (b, h)
  int n_items;               // persistent d = 64 kernel: B * H * ceil(Nq / 128) work items
  int group;                 // heads per scheduling group (CTA order, see tatn_fwd_kernel)
  uint64_t drop_seed;        // dropout: slice (b, h) uses mix64 chains from drop_seed + b*H + h
  uint64_t drop_thresh;      // keep iff hash >= drop_thresh  (= ceil(p * 2^53) << 11)
  float drop_scale;          // 1 / (1 - p)
  float* o_f32;              // fp32 output mode: O written here directly (strides below)
  void* o16;                 // 16-bit O (the persistent d = 128 kernel stores rows directly; strides below)
  int64_t o_sb, o_sh, o_sn;
  const uint32_t* custom;    // Custom mask: keep bits [Nq][custom_words] per batch element (or shared)
  int custom_words;
  int64_t custom_bstride;
  int k_off;                 // global index of key 0 (sequence-parallel key shards; multiple of 128)
};

struct BwdParams {
  int B, H, Nq, Nk;
  float scale_log2;  // tau * log2(e)
  float tau;
  int mask_kind;
  const int32_t* valid_len;
  const uint8_t* grid;
  int tr, tc;
  uint32_t* visited;
  const float* lse;  // [B, H, Nq]
  float* delta;      // [B, H, Nq] workspace: D_i = rowsum(dO_i * O_i)
  float* dq_acc;     // [B, H, Nq, d] fp32 workspace
  int n_ktiles;      // ceil(Nk / 128)
  int n_items;       // B * H * n_ktiles work items (one 128-key tile of one head each)
  int* item_counter; // persistent schedule: next unclaimed item (zeroed by K2 every launch)
  int group;         // heads per scheduling group (CTA order, see tatn_bwd_kernel)
  uint64_t drop_seed;   // dropout (see FwdParams)
  uint64_t drop_thresh;
  float drop_scale;
  float* dk_f32;     // fp32 output mode: dK / dV written directly (strides below)
  float* dv_f32;
  int64_t k_sb, k_sh, k_sn, v_sb, v_sh, v_sn;
  const uint32_t* custom_t;  // Custom mask transposed by K2b: keep bits [Bc][Nk][Nq_pad/32]
  int custom_t_words;        // Nq_pad / 32
  int custom_t_b;            // 1: one mask per batch element (b), 0: shared
  int k_off;                 // global index of key 0 (sequence-parallel key shards; multiple of 128)
  float* dq_part;            // deterministic dQ: per-key-tile partials [tc][B*H][Nq_pad][d] (else nullptr)
  const uint32_t* custom;    // Custom mask as given (tf32 check mode reads it untransposed)
  int custom_words;
  int64_t custom_bstride;
};

}  // namespace tatn_dev
