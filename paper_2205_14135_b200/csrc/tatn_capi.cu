// tatn_capi.cu — C-ABI entry points (include/tatn_b200.h): descriptor
// validation, TMA tensor-map construction and kernel launches.
//
// Error behaviour mirrors the reference's exceptions (flash.hpp:47-48,
// attn_config.cpp:42-58): shape / plan / mask mismatches and invalid tau or
// p_drop are reported as status codes instead of std::invalid_argument.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <utility>
#include <vector>

#include "../../include/tatn_b200.h"
#include "tatn_bwd.cuh"
#include "tatn_fwd.cuh"
#include "tatn_fwd1.cuh"
#include "tatn_fwd2.cuh"
#include "tatn_tf32.cuh"

namespace tatn_host {
int schedule_group(int heads, int tiles_per_head, double l2_bytes_per_head, int ctas_per_sm = 1);
int sm_count();
}  // namespace tatn_host
using tatn_host::set_dropout;
using tatn_host::schedule_group;

namespace {

thread_local int g_last_launches = 0;

// every tensor base pointer must be 16-byte aligned: TMA tiles and the kernels' 16-byte vector
// loads / stores (rows are 16-byte multiples by the stride rule) assume it
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
// forward workspace: the persistent kernels' self-resetting item counter {next item, finished
// CTAs}; zero before first use, left zero by every completed launch
constexpr size_t kFwdWorkspaceBytes = 16;

// ---- optional event timing of the main kernels (tatn_profile_*)
struct Profiler {
  std::mutex mu;
  bool on = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending[2];
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
Profiler& prof() {
  static Profiler p;
  return p;
}
// returns the stop event to record after the kernel (nullptr when profiling is off)
cudaEvent_t prof_begin(int which, cudaStream_t s) {
  Profiler& P = prof();
  std::lock_guard<std::mutex> lk(P.mu);
  if (!P.on) return nullptr;
  cudaEvent_t a = P.get(), b = P.get();
  cudaEventRecord(a, s);
  P.pending[which].emplace_back(a, b);
  return b;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult qres;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qres) == cudaSuccess &&
        qres == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  });
  return fn;
}

// 4-D map over (d, n, h, b) with a 64 x rows box and 128B swizzle.
bool make_map_4d(CUtensorMap* map, CUtensorMapDataType dt, uint32_t elem_bytes, const void* base, int d, int n,
                 int H, int B, const int64_t str[3], int box_rows, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B,
                 int box_cols = 64) {
  auto fn = get_encode_fn();
  if (!fn) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(B)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(str[2]) * elem_bytes, static_cast<cuuint64_t>(str[1]) * elem_bytes,
                           static_cast<cuuint64_t>(str[0]) * elem_bytes};
  cuuint32_t box[4] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows), 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, dt, 4, const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool strides_ok(const int64_t s[3], int H, int N, int d) {
  for (int i = 0; i < 3; ++i)
    if (s[i] <= 0 || (s[i] % 8) != 0) return false;
  (void)H;
  (void)N;
  (void)d;
  return true;
}

int validate(const tatn_attn_desc* d) {
  if (d == nullptr) return TATN_E_ARG;
  if (d->B < 1 || d->H < 1 || d->Nq < 1 || d->Nk < 1) return TATN_E_SHAPE;
  if (d->B > 65535 || d->H > 65535) return TATN_E_SHAPE;  // K2 / K4 grid (rows, H, B)
  if (d->Nk > d->Nq) return TATN_E_SHAPE;  // more keys than n (reference.cpp:25-26)
  if (d->d != 64 && d->d != 128) return TATN_E_UNSUPPORTED;
  // bf16 / fp16 inputs (the throughput path) or fp32 inputs (the tf32 check mode, tatn_tf32.cuh)
  if (d->dtype != TATN_DTYPE_BF16 && d->dtype != TATN_DTYPE_FP16 && d->dtype != TATN_DTYPE_FP32)
    return TATN_E_UNSUPPORTED;
  if (d->out_dtype != TATN_OUT_INPUT_DTYPE && d->out_dtype != TATN_OUT_FP32) return TATN_E_UNSUPPORTED;
  if (!(d->tau > 0.f) || !std::isfinite(d->tau)) return TATN_E_ARG;  // attn_config.cpp:52
  if (!(d->p_drop >= 0.0 && d->p_drop < 1.0)) return TATN_E_ARG;      // attn_config.cpp:54
  if (d->mask_kind != TATN_MASK_NONE && d->mask_kind != TATN_MASK_CAUSAL && d->mask_kind != TATN_MASK_KEY_PADDING &&
      d->mask_kind != TATN_MASK_CUSTOM)
    return TATN_E_ARG;  // not a tatn::MaskKind
  if (d->mask_kind == TATN_MASK_KEY_PADDING && d->valid_len == nullptr) return TATN_E_ARG;
  if (d->mask_kind == TATN_MASK_CUSTOM) {
    // custom mask must cover Nq x Nk (attn_config.cpp:50-52: "custom mask must be n x n")
    if (d->custom_mask == nullptr) return TATN_E_ARG;
    // the kernels read word (k_offset + j) / 32 of each row, 16 bytes per 128-key tile
    if (d->k_offset < 0) return TATN_E_SHAPE;
    const int64_t need_words = 4 * ((static_cast<int64_t>(d->k_offset) + d->Nk + 127) / 128);
    if (d->custom_words < need_words || (d->custom_words % 4) != 0) return TATN_E_MASK;
    if (d->custom_bstride != 0 && d->custom_bstride < static_cast<int64_t>(d->Nq) * d->custom_words) return TATN_E_MASK;
    if ((reinterpret_cast<uintptr_t>(d->custom_mask) & 15u) != 0) return TATN_E_ARG;  // 16-byte row loads
  }
  if (!strides_ok(d->q_str, d->H, d->Nq, d->d) || !strides_ok(d->k_str, d->H, d->Nk, d->d) ||
      !strides_ok(d->v_str, d->H, d->Nk, d->d) || !strides_ok(d->o_str, d->H, d->Nq, d->d))
    return TATN_E_SHAPE;
  const int tr = (d->Nq + 127) / 128, tc = (d->Nk + 127) / 128;
  if (d->block_grid != nullptr) {
    if (d->br != 128 || d->bc != 128) return TATN_E_MASK;  // bmask block sizes must equal the plan's
    if (d->tr != tr || d->tc != tc) return TATN_E_MASK;
    if (tc > 2048 || 2 * tr > 4096) return TATN_E_UNSUPPORTED;  // block-sparse bitmask capacity (N <= 256K)
  }
  if (d->visited_bitmap != nullptr && (d->tr != tr || d->tc != tc)) return TATN_E_MASK;
  // sequence-parallel key shard: keys are global keys [k_offset, k_offset + Nk) of an Nq-long sequence
  if (d->k_offset < 0 || (d->k_offset % 128) != 0 || static_cast<int64_t>(d->k_offset) + d->Nk > d->Nq)
    return TATN_E_SHAPE;
  if (d->k_offset != 0 && d->block_grid != nullptr) return TATN_E_UNSUPPORTED;
  if (d->Nq > (1 << 24) || static_cast<int64_t>(d->B) * d->H * ((d->Nq + 127) / 128) > (1ll << 31) - 1)
    return TATN_E_SHAPE;
  if (d->deterministic != 0 && d->deterministic != 1) return TATN_E_ARG;
  return TATN_OK;
}

CUtensorMapDataType tma_dtype(int dtype) {
  return dtype == TATN_DTYPE_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
}

template <bool BF16, bool OUT_F32, bool DROP>
cudaError_t launch_fwd1(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v, const CUtensorMap& o,
                        const tatn_dev::FwdParams& p, int* ctr, cudaStream_t stream) {
  using Cfg = tatn_dev::Fwd1Cfg;
  auto kern = tatn_dev::tatn_fwd1_kernel<BF16, OUT_F32, DROP>;
  cudaError_t e = tatn_host::ensure_smem_attr(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  tatn_dev::FwdParams pp = p;
  pp.n_pairs = (p.Nq + 127) / 128;  // Q tiles per (b, h)
  pp.n_items = p.B * p.H * pp.n_pairs;
  // persistent + dynamic claims: one head group (global longest-first order) unless the heads'
  // K/V would not stay L2-resident, so no group boundary brings heavy items back into the tail
  pp.group = schedule_group(p.B * p.H, 1, static_cast<double>(p.Nk) * 64 * 4.0, 2);
  // persistent: two CTAs per SM
  const int grid = std::min(pp.n_items, 2 * tatn_host::sm_count());
  return tatn_host::launch(kern, dim3(grid), dim3(tatn_dev::kFwd1Threads), Cfg::kSmemBytes, stream, q, k, v, o, pp,
                           ctr);
}

template <int D, bool BF16, bool OUT_F32, bool DROP>
cudaError_t launch_fwd2(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                        const tatn_dev::FwdParams& p, int* ctr, cudaStream_t stream) {
  using Cfg = tatn_dev::Fwd2Cfg<D>;
  auto kern = tatn_dev::tatn_fwd2_kernel<D, BF16, OUT_F32, DROP>;
  cudaError_t e = tatn_host::ensure_smem_attr(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  tatn_dev::FwdParams pp = p;
  pp.n_pairs = (p.Nq + 255) / 256;  // Q-tile pairs per (b, h)
  pp.n_items = p.B * p.H * pp.n_pairs;
  pp.group = schedule_group(p.B * p.H, 1, static_cast<double>(p.Nk) * D * 4.0, 1);
  const int grid = std::min(pp.n_items, tatn_host::sm_count());  // persistent, one CTA per SM
  return tatn_host::launch(kern, dim3(grid), dim3(384), Cfg::kSmemBytes, stream, q, k, v, pp, ctr);
}

// d = 64: tatn_fwd1 (persistent, one Q tile per item, 2 CTAs/SM); d = 128: tatn_fwd2 (persistent,
// Q-tile pairs, 1 CTA/SM). Both claim items from the caller's workspace counter.
template <int D, bool BF16, bool OUT_F32, bool DROP>
cudaError_t launch_fwd(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v, const CUtensorMap& o,
                       const tatn_dev::FwdParams& p, int* ctr, cudaStream_t stream) {
  if constexpr (D == 64) return launch_fwd1<BF16, OUT_F32, DROP>(q, k, v, o, p, ctr, stream);
  else return launch_fwd2<128, BF16, OUT_F32, DROP>(q, k, v, p, ctr, stream);
}

// fp32 inputs: the tf32 check-mode forward, one CTA per (Q tile, h, b)
template <int D, bool DROP>
cudaError_t launch_fwd_tf32(const CUtensorMap& q, const CUtensorMap& k, const CUtensorMap& v,
                            const tatn_dev::FwdParams& p, cudaStream_t stream) {
  using Cfg = tatn_dev::Tf32FwdCfg<D>;
  auto kern = tatn_dev::tatn_fwd_tf32_kernel<D, DROP>;
  cudaError_t e = tatn_host::ensure_smem_attr(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  const dim3 grid(static_cast<unsigned>((p.Nq + 127) / 128), p.H, p.B);
  return tatn_host::launch(kern, grid, dim3(tatn_dev::kTf32Threads), Cfg::kSmemBytes, stream, q, k, v, p);
}

// fp32 inputs: K2 (fp32 O, dO) -> the tf32 check-mode backward, one CTA per (key tile, h, b) -> K4
template <int D, bool DROP>
cudaError_t launch_bwd_tf32(const tatn_attn_desc& d, const void* q, const void* k, const void* v, const void* o,
                            const void* dO, const float* lse, void* dq, void* dk, void* dv, void* ws,
                            cudaStream_t stream, int* launches) {
  using Cfg = tatn_dev::Tf32BwdCfg<D>;
  const int Nq_pad = (d.Nq + 127) / 128 * 128;
  const size_t rows = static_cast<size_t>(d.B) * d.H * Nq_pad;
  float* dq_acc = static_cast<float*>(ws);
  float* lse2 = dq_acc + rows * D;
  float* delta = lse2 + rows;
  int* item_counter = reinterpret_cast<int*>(delta + rows);
  const dim3 rblocks(static_cast<unsigned>((Nq_pad + 256 / (D / 8) - 1) / (256 / (D / 8))), d.H, d.B);
  cudaError_t e = tatn_host::launch(tatn_dev::tatn_bwd_pre<D, false, true, true>, rblocks, dim3(256), 0, stream, o, dO,
                                    lse, d.o_str[0], d.o_str[1], d.o_str[2], d.B, d.H, d.Nq, Nq_pad, lse2, delta,
                                    dq_acc, item_counter);
  if (e != cudaSuccess) return e;
  CUtensorMap mq, mk, mkmn, mdo;
  if (!tatn_host::make_map_4d_ext(&mq, TATN_DTYPE_FP32, q, D, d.Nq, d.H, d.B, d.q_str, Cfg::QT) ||
      !tatn_host::make_map_4d_ext(&mk, TATN_DTYPE_FP32, k, D, d.Nk, d.H, d.B, d.k_str, 128) ||
      !tatn_host::make_map_4d_ext(&mkmn, TATN_DTYPE_FP32, k, D, d.Nk, d.H, d.B, d.k_str, 128, /*mn_major=*/true) ||
      !tatn_host::make_map_4d_ext(&mdo, TATN_DTYPE_FP32, dO, D, d.Nq, d.H, d.B, d.o_str, Cfg::QT))
    return cudaErrorInvalidValue;
  tatn_dev::BwdParams p{};
  p.B = d.B;
  p.H = d.H;
  p.Nq = d.Nq;
  p.Nk = d.Nk;
  p.scale_log2 = d.tau * 1.4426950408889634f;
  p.tau = d.tau;
  p.mask_kind = d.mask_kind;
  p.valid_len = d.valid_len;
  p.grid = d.block_grid;
  p.tr = (d.Nq + 127) / 128;
  p.tc = (d.Nk + 127) / 128;
  p.visited = d.visited_bitmap;
  p.lse = lse;
  p.delta = delta;
  p.dq_acc = dq_acc;
  p.dk_f32 = static_cast<float*>(dk);
  p.dv_f32 = static_cast<float*>(dv);
  p.k_sb = d.k_str[0];
  p.k_sh = d.k_str[1];
  p.k_sn = d.k_str[2];
  p.v_sb = d.v_str[0];
  p.v_sh = d.v_str[1];
  p.v_sn = d.v_str[2];
  p.k_off = d.k_offset;
  p.custom = d.mask_kind == TATN_MASK_CUSTOM ? d.custom_mask : nullptr;
  p.custom_words = d.custom_words;
  p.custom_bstride = d.custom_bstride;
  p.dq_part = d.deterministic ? tatn_host::dq_part_ptr(d, ws) : nullptr;
  set_dropout(d, &p.drop_seed, &p.drop_thresh, &p.drop_scale);
  auto kern = tatn_dev::tatn_bwd_tf32_kernel<D, DROP>;
  e = tatn_host::ensure_smem_attr(reinterpret_cast<const void*>(kern), Cfg::kSmemBytes);
  if (e != cudaSuccess) return e;
  cudaEvent_t prof_stop = prof_begin(1, stream);
  e = tatn_host::launch(kern, dim3(static_cast<unsigned>(p.tc), d.H, d.B), dim3(tatn_dev::kTf32Threads),
                        Cfg::kSmemBytes, stream, mq, mk, mkmn, mdo, static_cast<const float*>(v), p,
                        static_cast<const float*>(lse2), Nq_pad);
  if (prof_stop) cudaEventRecord(prof_stop, stream);
  if (e != cudaSuccess) return e;
  const dim3 qblocks(static_cast<unsigned>((d.Nq + 256 / (D / 8) - 1) / (256 / (D / 8))), d.H, d.B);
  if (p.dq_part != nullptr)
    e = tatn_host::launch_post_det<D, false, true>(d, p.dq_part, dq, Nq_pad, Cfg::QT, stream);
  else
    e = tatn_host::launch(tatn_dev::tatn_bwd_post<D, false, true>, qblocks, dim3(256), 0, stream,
                          static_cast<const float*>(dq_acc), dq, d.q_str[0], d.q_str[1], d.q_str[2], d.B, d.H, d.Nq,
                          Nq_pad);
  if (e != cudaSuccess) return e;
  *launches = 3;
  return cudaSuccess;
}

}  // namespace

namespace tatn_host {
cudaEvent_t profile_begin(int which, cudaStream_t s) { return prof_begin(which, s); }
// Heads per scheduling group: enough CTAs for ~2 waves on 148 SMs (so the
// longest-first order inside a group balances the tail) while the group's
// per-head working set stays well inside the 126 MB L2.
int schedule_group(int heads, int tiles_per_head, double l2_bytes_per_head, int ctas_per_sm) {
  int g = (2 * 148 * ctas_per_sm + tiles_per_head - 1) / tiles_per_head;
  const int l2_cap = static_cast<int>(64.0e6 / (l2_bytes_per_head > 1.0 ? l2_bytes_per_head : 1.0));
  g = std::min(g, std::max(1, l2_cap));
  return std::max(1, std::min(g, heads));
}
// SM count of the current device (cached per device: one process may drive several GPUs)
int sm_count() {
  static std::atomic<int> cache[kMaxDevices] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev < 0 || dev >= kMaxDevices) dev = 0;
  int n = cache[dev].load(std::memory_order_relaxed);
  if (n == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0) n = v;
    else n = 148;
    cache[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}
// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device setting: set it once per (kernel,
// device) the first time the kernel launches on that device
cudaError_t ensure_smem_attr(const void* kern, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& pr : done)
    if (pr.first == kern && pr.second == dev) return cudaSuccess;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.emplace_back(kern, dev);
  return e;
}
bool make_map_4d_ext(CUtensorMap* map, int dtype, const void* base, int d, int n, int H, int B, const int64_t str[3],
                     int box_rows, bool mn_major) {
  // fp32 tiles: 32 columns (128 bytes) per box; an MN-major tf32 operand needs the 128-byte
  // swizzle with 32-byte atoms (the only shared-memory layout the tf32 MMA reads MN-major)
  if (dtype == TATN_DTYPE_FP32)
    return make_map_4d(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, d, n, H, B, str, box_rows,
                       mn_major ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, 32);
  return make_map_4d(map, tma_dtype(dtype), 2, base, d, n, H, B, str, box_rows);
}
}  // namespace tatn_host

extern "C" {

int tatn_validate(const tatn_attn_desc* desc) { return validate(desc); }

int tatn_abi_version(void) { return TATN_B200_ABI_VERSION; }

int tatn_merge_partials(int32_t R, int32_t B, int32_t H, int32_t Nq, int32_t d, const float* o_parts,
                        const float* lse_parts, void* o, int32_t o_dtype, const int64_t o_str[3], float* lse,
                        void* stream) {
  g_last_launches = 0;
  if (R < 1 || B < 1 || H < 1 || Nq < 1 || (d != 64 && d != 128)) return TATN_E_SHAPE;
  if (!o_parts || !lse_parts || !o || !lse || !o_str) return TATN_E_ARG;
  if (o_dtype != TATN_DTYPE_BF16 && o_dtype != TATN_DTYPE_FP16 && o_dtype != TATN_DTYPE_FP32) return TATN_E_ARG;
  for (int i = 0; i < 3; ++i)
    if (o_str[i] <= 0 || (o_str[i] % 8) != 0) return TATN_E_SHAPE;
  if (B > 65535 || H > 65535) return TATN_E_SHAPE;
  const long long rows = static_cast<long long>(B) * H * Nq;
  const int rows_per_block = 256 / (d / 8);
  const dim3 blocks(static_cast<unsigned>((Nq + rows_per_block - 1) / rows_per_block), H, B);
  if (tatn_host::launch(tatn_dev::tatn_merge_kernel, blocks, dim3(256), 0, static_cast<cudaStream_t>(stream), R,
                        rows, d, H, Nq, o_parts, lse_parts, o, o_dtype, o_str[0], o_str[1], o_str[2],
                        lse) != cudaSuccess)
    return TATN_E_CUDA;
  g_last_launches = 1;
  return TATN_OK;
}

int tatn_last_launch_count(void) { return g_last_launches; }

#ifdef TATN_WAIT_DEBUG
// debug builds only: where a deadlocked mbarrier wait was stuck (scripts/repro_tiny.py)
int tatn_debug_set_wait_dbg(void* dev_buf) {
  unsigned long long* p = static_cast<unsigned long long*>(dev_buf);
  return cudaMemcpyToSymbol(tatn_dev::g_tatn_wait_dbg, &p, sizeof(p)) == cudaSuccess ? TATN_OK : TATN_E_CUDA;
}
#endif

#ifdef TATN_TRACE
// debug builds only: per-CTA globaltimer trace of the forward kernel (scripts/trace_fwd.py)
int tatn_debug_set_trace(void* dev_buf) {
  unsigned long long* p = static_cast<unsigned long long*>(dev_buf);
  return cudaMemcpyToSymbol(tatn_dev::g_tatn_trace, &p, sizeof(p)) == cudaSuccess ? TATN_OK : TATN_E_CUDA;
}
#endif

int tatn_profile_enable(int on) {
  Profiler& P = prof();
  std::lock_guard<std::mutex> lk(P.mu);
  P.on = on != 0;
  return TATN_OK;
}

int tatn_profile_read(int which, double* total_ms, int* launches) {
  if (which < 0 || which > 1 || !total_ms || !launches) return TATN_E_ARG;
  Profiler& P = prof();
  std::lock_guard<std::mutex> lk(P.mu);
  double sum = 0.0;
  int n = 0;
  for (auto& pr : P.pending[which]) {
    if (cudaEventSynchronize(pr.second) != cudaSuccess) return TATN_E_CUDA;
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, pr.first, pr.second) != cudaSuccess) return TATN_E_CUDA;
    sum += ms;
    ++n;
    P.pool.push_back(pr.first);
    P.pool.push_back(pr.second);
  }
  P.pending[which].clear();
  *total_ms = sum;
  *launches = n;
  return TATN_OK;
}

const char* tatn_strerror(int status) {
  switch (status) {
    case TATN_OK: return "ok";
    case TATN_E_ARG: return "invalid argument";
    case TATN_E_SHAPE: return "shape or stride mismatch";
    case TATN_E_MASK: return "block mask / plan mismatch";
    case TATN_E_UNSUPPORTED: return "unsupported on the sm_100a path";
    case TATN_E_CUDA: return "CUDA error or no sm_100 device";
    case TATN_E_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

size_t tatn_fwd_workspace_bytes(const tatn_attn_desc* desc) {
  if (validate(desc) != TATN_OK) return 0;
  return kFwdWorkspaceBytes;
}

int tatn_fwd(const tatn_attn_desc* desc, const void* q, const void* k, const void* v, void* o, float* lse,
             void* workspace, size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  int st = validate(desc);
  if (st != TATN_OK) return st;
  if (!q || !k || !v || !o || !lse || !workspace) return TATN_E_ARG;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o)) return TATN_E_ARG;
  if (workspace_bytes < kFwdWorkspaceBytes) return TATN_E_WORKSPACE;
  if ((reinterpret_cast<uintptr_t>(workspace) & 15u) != 0) return TATN_E_ARG;
  const tatn_attn_desc& d = *desc;
  const bool in_f32 = d.dtype == TATN_DTYPE_FP32;
  const bool f32 = in_f32 || d.out_dtype == TATN_OUT_FP32;  // fp32 inputs always give fp32 outputs
  CUtensorMap mq, mk, mv, mo;
  if (!tatn_host::make_map_4d_ext(&mq, d.dtype, q, d.d, d.Nq, d.H, d.B, d.q_str, 128) ||
      !tatn_host::make_map_4d_ext(&mk, d.dtype, k, d.d, d.Nk, d.H, d.B, d.k_str, 128) ||
      !tatn_host::make_map_4d_ext(&mv, d.dtype, v, d.d, d.Nk, d.H, d.B, d.v_str, 128, /*mn_major=*/in_f32))
    return TATN_E_CUDA;
  // 16-bit O is stored by TMA (d = 64); the fp32 modes write O from registers (map unused)
  if (!in_f32 && !tatn_host::make_map_4d_ext(&mo, d.dtype, f32 ? q : o, d.d, d.Nq, d.H, d.B, f32 ? d.q_str : d.o_str, 128))
    return TATN_E_CUDA;
  tatn_dev::FwdParams p{};
  p.B = d.B;
  p.H = d.H;
  p.Nq = d.Nq;
  p.Nk = d.Nk;
  p.scale_log2 = d.tau * 1.4426950408889634f;
  p.mask_kind = d.mask_kind;
  p.valid_len = d.valid_len;
  p.grid = d.block_grid;
  p.tr = (d.Nq + 127) / 128;
  p.tc = (d.Nk + 127) / 128;
  p.visited = d.visited_bitmap;
  p.lse = lse;
  p.n_pairs = 0;  // set per variant in launch_fwd
  p.group = 1;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  p.o_f32 = f32 ? static_cast<float*>(o) : nullptr;
  p.o16 = f32 ? nullptr : o;
  p.o_sb = d.o_str[0];
  p.o_sh = d.o_str[1];
  p.o_sn = d.o_str[2];
  p.custom = d.mask_kind == TATN_MASK_CUSTOM ? d.custom_mask : nullptr;
  p.custom_words = d.custom_words;
  p.custom_bstride = d.custom_bstride;
  p.k_off = d.k_offset;
  const bool drop = d.p_drop > 0.0;
  set_dropout(d, &p.drop_seed, &p.drop_thresh, &p.drop_scale);
  int* ctr = static_cast<int*>(workspace);
  e = cudaErrorInvalidValue;
  cudaEvent_t prof_stop = prof_begin(0, s);
  if (in_f32) {
    const int sel = (d.d == 128 ? 2 : 0) + (drop ? 1 : 0);
    switch (sel) {
      case 0: e = launch_fwd_tf32<64, false>(mq, mk, mv, p, s); break;
      case 1: e = launch_fwd_tf32<64, true>(mq, mk, mv, p, s); break;
      case 2: e = launch_fwd_tf32<128, false>(mq, mk, mv, p, s); break;
      case 3: e = launch_fwd_tf32<128, true>(mq, mk, mv, p, s); break;
    }
  } else {
    const int sel = (d.d == 128 ? 8 : 0) + (d.dtype == TATN_DTYPE_BF16 ? 4 : 0) + (f32 ? 2 : 0) + (drop ? 1 : 0);
#define TATN_FWD_CASE(i, DD, B16, F32, DR) \
  case i: e = launch_fwd<DD, B16, F32, DR>(mq, mk, mv, mo, p, ctr, s); break;
    switch (sel) {
      TATN_FWD_CASE(0, 64, false, false, false)
      TATN_FWD_CASE(1, 64, false, false, true)
      TATN_FWD_CASE(2, 64, false, true, false)
      TATN_FWD_CASE(3, 64, false, true, true)
      TATN_FWD_CASE(4, 64, true, false, false)
      TATN_FWD_CASE(5, 64, true, false, true)
      TATN_FWD_CASE(6, 64, true, true, false)
      TATN_FWD_CASE(7, 64, true, true, true)
      TATN_FWD_CASE(8, 128, false, false, false)
      TATN_FWD_CASE(9, 128, false, false, true)
      TATN_FWD_CASE(10, 128, false, true, false)
      TATN_FWD_CASE(11, 128, false, true, true)
      TATN_FWD_CASE(12, 128, true, false, false)
      TATN_FWD_CASE(13, 128, true, false, true)
      TATN_FWD_CASE(14, 128, true, true, false)
      TATN_FWD_CASE(15, 128, true, true, true)
    }
#undef TATN_FWD_CASE
  }
  if (prof_stop) cudaEventRecord(prof_stop, s);
  if (e != cudaSuccess) return TATN_E_CUDA;
  g_last_launches = 1;
  return TATN_OK;
}

size_t tatn_bwd_workspace_bytes(const tatn_attn_desc* desc) {
  if (validate(desc) != TATN_OK) return 0;
  // dQ accumulator [B,H,Nq_pad,d] fp32 + lse2 [B,H,Nq_pad] + D [B,H,Nq_pad], Nq_pad = roundup(Nq, 128),
  // + the persistent backward's item counter
  const size_t rows = static_cast<size_t>(desc->B) * desc->H * ((desc->Nq + 127) / 128 * 128);
  size_t bytes = rows * desc->d * sizeof(float) + 2 * rows * sizeof(float) + 16;  // + K3 item counter
  if (desc->mask_kind == TATN_MASK_CUSTOM) {  // + the custom mask transposed for K3 (K2b)
    const size_t nb = desc->custom_bstride != 0 ? static_cast<size_t>(desc->B) : 1;
    bytes += nb * static_cast<size_t>(desc->Nk) * ((desc->Nq + 127) / 128 * 4) * sizeof(uint32_t);
  }
  if (desc->deterministic)  // + per-key-tile dQ partials [tc][B*H][Nq_pad][d]
    bytes += static_cast<size_t>((desc->Nk + 127) / 128) * rows * desc->d * sizeof(float);
  return bytes;
}

int tatn_bwd(const tatn_attn_desc* desc, const void* q, const void* k, const void* v, const void* o, const void* dO,
             const float* lse, void* dq, void* dk, void* dv, void* workspace, size_t workspace_bytes, void* stream) {
  g_last_launches = 0;
  int st = validate(desc);
  if (st != TATN_OK) return st;
  if (!q || !k || !v || !o || !dO || !lse || !dq || !dk || !dv || !workspace) return TATN_E_ARG;
  if (!aligned16(q) || !aligned16(k) || !aligned16(v) || !aligned16(o) || !aligned16(dO) || !aligned16(dq) ||
      !aligned16(dk) || !aligned16(dv) || !aligned16(workspace))
    return TATN_E_ARG;
  if (workspace_bytes < tatn_bwd_workspace_bytes(desc)) return TATN_E_WORKSPACE;
  if (desc->dtype == TATN_DTYPE_FP32) {
    const int sel = (desc->d == 128 ? 2 : 0) + (desc->p_drop > 0.0 ? 1 : 0);
    cudaError_t e = cudaErrorInvalidValue;
    const cudaStream_t s = static_cast<cudaStream_t>(stream);
    int n = 0;
    switch (sel) {
      case 0: e = launch_bwd_tf32<64, false>(*desc, q, k, v, o, dO, lse, dq, dk, dv, workspace, s, &n); break;
      case 1: e = launch_bwd_tf32<64, true>(*desc, q, k, v, o, dO, lse, dq, dk, dv, workspace, s, &n); break;
      case 2: e = launch_bwd_tf32<128, false>(*desc, q, k, v, o, dO, lse, dq, dk, dv, workspace, s, &n); break;
      case 3: e = launch_bwd_tf32<128, true>(*desc, q, k, v, o, dO, lse, dq, dk, dv, workspace, s, &n); break;
    }
    if (e != cudaSuccess) return TATN_E_CUDA;
    g_last_launches = n;
    return TATN_OK;
  }
  return tatn_bwd_launch(*desc, q, k, v, o, dO, lse, dq, dk, dv, workspace, static_cast<cudaStream_t>(stream),
                         &g_last_launches);
}

}  // extern "C"
