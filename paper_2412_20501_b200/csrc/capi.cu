// extern "C" boundary of libtokenring.so (see include/tokenring.h).
// Validation mirrors the reference's Python-side checks
// (core.py:96-119 DimensionError, partition.py:59-62 ConfigError) so the
// Python wrapper can map status codes onto the same exception classes.
#include <cuda_runtime.h>
#include <algorithm>
#include <cmath>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

#include "tr_internal.h"

namespace tr {

static thread_local std::string g_last_error;
static thread_local int32_t g_launch_overlap = 0;   // tr_set_launch_overlap

void set_error(const std::string& msg) { g_last_error = msg; }
bool launch_overlap() { return (g_launch_overlap & TR_LAUNCH_AFTER_PREV) != 0; }
bool launch_release_next() { return (g_launch_overlap & TR_LAUNCH_RELEASE_NEXT) != 0; }
int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return TR_OK;
  // the failure is reported here: reset the runtime's (non-sticky) last-error
  // slot so a later launch check does not report it a second time
  cudaGetLastError();
  return fail(TR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

int set_smem_attr_once(const void* func, int bytes, const char* what) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  int rc = cuda_status(cudaGetDevice(&dev), "cudaGetDevice");
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(mu);
  if (done.count({func, dev})) return TR_OK;
  if ((rc = cuda_status(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes),
                        what)))
    return rc;
  done.insert({func, dev});
  return TR_OK;
}

int launch_merge(float* acc_out, float* acc_lse, const void* blk_out, int blk_dtype,
                 const float* blk_lse, int64_t T, int H, int D, int64_t als, int64_t bls,
                 void* fin, cudaStream_t s);
int launch_merge_n(float* acc_out, float* acc_lse, int64_t als, const void* const* blk,
                   int blk_dtype, const float* const* blk_lse, const int64_t* bls, int n,
                   int64_t T, int H, int D, void* fin, cudaStream_t s);
int launch_partial_init(float* acc_out, float* acc_lse, int64_t T, int H, int D, cudaStream_t s);
int launch_fill(float* p, int64_t n, float v, cudaStream_t s);
int launch_splitmix(uint64_t seed, int64_t first, int64_t count, double low, double high,
                    void* dst, cudaStream_t s);

static int check_segments(const tr_segment* segs, int n, int64_t total, const char* what) {
  if (n < 0 || n > TR_MAX_SEGMENTS)
    return fail(TR_ERR_CONFIG, std::string(what) + ": segment count must be in [0, 4]");
  for (int i = 0; i < n; ++i) {
    if (segs[i].rows < 0 || segs[i].row0 < 0 || segs[i].row0 + segs[i].rows > total)
      return fail(TR_ERR_DIMENSION, std::string(what) + ": segment outside the buffer");
  }
  return TR_OK;
}

// Longest-processing-time-first CTA order for a causal launch with several q
// segments (a TokenRing step: the rows of a light and a heavy chunk in one
// grid).  Head-major order would run each head's heavy tiles after its light
// ones, leaving the heaviest CTAs of the last head as the grid's tail; instead
// every (segment, tile) class is ranked by its kv-tile count and the grid walks
// the classes heaviest first, heads innermost, in head groups small enough
// that a group's K/V stays resident in L2.
static void order_ctas(AttnPlan& plan, int head_dim) {
  plan.n_order = 0;
#ifdef TR_NO_ORDER
  return;   // A/B switch: the plain head-major order
#endif
  const int64_t nt = plan.tile_prefix[plan.nq];
  if (!plan.causal || plan.nq < 2 || nt > TR_ORDER_MAX) return;
  std::vector<std::pair<int64_t, int>> work;
  work.reserve(nt);
  for (int sg = 0; sg < plan.nq; ++sg) {
    const tr_segment& Q = plan.q[sg];
    for (int64_t t = 0; t < plan.tile_prefix[sg + 1] - plan.tile_prefix[sg]; ++t) {
      const int64_t qmax = Q.pos0 + std::min<int64_t>(t * 256 + 255, Q.rows - 1);
      int64_t n = 0;
      for (int g = 0; g < plan.nkv; ++g) {
        const tr_segment& K = plan.kv[g];
        if (qmax < K.pos0) continue;
        n += std::min<int64_t>((K.rows + 127) / 128, (qmax - K.pos0) / 128 + 1);
      }
      work.emplace_back(-n, static_cast<int>(plan.tile_prefix[sg] + t));
    }
  }
  std::stable_sort(work.begin(), work.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  for (int64_t i = 0; i < nt; ++i) plan.order[i] = static_cast<uint16_t>(work[i].second);
  int64_t kv_rows = 0;
  for (int g = 0; g < plan.nkv; ++g) kv_rows += plan.kv[g].rows;
  const int64_t kv_bytes_per_head = std::max<int64_t>(1, kv_rows * head_dim * 2 * 2);
  const int64_t budget = 48ll << 20;     // of the 126 MB L2
  plan.head_group = static_cast<int32_t>(
      std::max<int64_t>(1, std::min<int64_t>(plan.heads, budget / kv_bytes_per_head)));
  plan.n_order = static_cast<int32_t>(nt);
}

// Push options of tr_attention_segments_push (all zero for a local launch).
struct PushOpts {
  int64_t row_shift = 0;           // out/lse row r lands at row r - row_shift
  int64_t lse_stride = -1;         // row stride of lse (-1: tq_total)
  unsigned int* done_count = nullptr;
  unsigned long long* done_flag = nullptr;
  unsigned long long done_value = 0;
  const long long* done_epoch = nullptr;
};

static int run_segments(const void* q, const void* k, const void* v, void* out, float* lse,
                        int64_t tq_total, int64_t tk_total, int heads, int head_dim,
                        const tr_segment* qs, int nq, const tr_segment* ks, int nk, int causal,
                        int out_dtype, cudaStream_t s, const PushOpts& push = PushOpts()) {
  if (out_dtype != TR_DTYPE_BF16 && out_dtype != TR_DTYPE_F32)
    return fail(TR_ERR_CONFIG, "out_dtype must be TR_DTYPE_BF16 or TR_DTYPE_F32");
  if (heads < 1 || head_dim < 1 || tq_total < 0 || tk_total < 0)
    return fail(TR_ERR_DIMENSION, "heads, head_dim must be >= 1 and token counts >= 0");
  int rc;
  if ((rc = check_segments(qs, nq, tq_total, "q"))) return rc;
  if ((rc = check_segments(ks, nk, tk_total, "kv"))) return rc;
  AttnPlan plan{};
  plan.nq = 0;
  for (int i = 0; i < nq; ++i)
    if (qs[i].rows > 0) plan.q[plan.nq++] = qs[i];
  plan.nkv = 0;
  for (int i = 0; i < nk; ++i)
    if (ks[i].rows > 0) plan.kv[plan.nkv++] = ks[i];
  // a pushing launch with nothing to compute still owes its receiver the flag
  auto flag_only = [&]() {
    return push.done_flag ? launch_flag_set(push.done_flag, push.done_value, s, push.done_epoch)
                          : TR_OK;
  };
  if (plan.nq == 0) return flag_only();
  plan.causal = causal ? 1 : 0;
  plan.heads = heads;
  plan.lse_stride = push.lse_stride >= 0 ? push.lse_stride : tq_total;
  plan.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(head_dim)));
  plan.scale_log2 = static_cast<float>(1.4426950408889634 / std::sqrt(static_cast<double>(head_dim)));
  plan.out_f32 = out_dtype == TR_DTYPE_F32 ? 1 : 0;
  // shifted bases: the kernels index rows of q's local buffer; row r of out /
  // lse is written at r - row_shift (a receive buffer holding only the rows
  // of one message).  Only rows >= row_shift are ever written.
  const int64_t esz = plan.out_f32 ? 4 : 2;
  plan.out = reinterpret_cast<void*>(reinterpret_cast<uintptr_t>(out) -
                                     static_cast<uintptr_t>(push.row_shift * heads * head_dim * esz));
  plan.lse = reinterpret_cast<float*>(reinterpret_cast<uintptr_t>(lse) -
                                      static_cast<uintptr_t>(push.row_shift * 4));
  plan.done_count = push.done_count;
  plan.done_flag = push.done_flag;
  plan.done_value = push.done_value;
  plan.done_epoch = push.done_epoch;
  plan.overlap_prev = launch_overlap() ? 1 : 0;
  plan.release_next = launch_release_next() ? 1 : 0;
  plan.tile_prefix[0] = 0;
  for (int i = 0; i < plan.nq; ++i)
    plan.tile_prefix[i + 1] = plan.tile_prefix[i] + (plan.q[i].rows + 255) / 256;
  order_ctas(plan, head_dim);
  const bool tc = head_dim == 64 || head_dim == 128;   // the tcgen05 kernels' head dims
  if (tc && !sm100_supports(head_dim, heads, q, k, v, out))
    return fail(TR_ERR_UNSUPPORTED,
                "head_dim " + std::to_string(head_dim) + " runs on the tcgen05 kernels, which need "
                "16-byte aligned q/k/v/out base pointers (TMA); got a misaligned tensor "
                "(e.g. a view starting at an odd element) -- pass a contiguous copy");
  if (tc && plan.nkv > 0) {
    // the kernel raises done_flag itself (last CTA); an empty grid does not run
    if ((rc = launch_attn_sm100(q, k, v, tq_total, tk_total, head_dim, plan, s))) return rc;
    return plan.tile_prefix[plan.nq] * heads == 0 ? flag_only() : TR_OK;
  }
  plan.done_flag = nullptr;          // the generic kernel signals with a trailing launch
  if ((rc = launch_attn_simt(q, k, v, head_dim, plan, s))) return rc;
  return flag_only();
}

}  // namespace tr

using namespace tr;

extern "C" {

int tr_attention_block(const void* q, const void* k, const void* v, void* out, float* lse,
                       int64_t tq, int64_t tk, int32_t heads, int32_t head_dim, int32_t mask_kind,
                       int64_t q_offset, int64_t k_offset, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (mask_kind != TR_MASK_NONE && mask_kind != TR_MASK_FULL && mask_kind != TR_MASK_CAUSAL)
    return fail(TR_ERR_CONFIG, "mask_kind must be 0 (none), 1 (full) or 2 (causal)");
  if (heads < 1 || head_dim < 1 || tq < 0 || tk < 0)
    return fail(TR_ERR_DIMENSION, "tq, tk >= 0 and heads, head_dim >= 1 required");
  if (mask_kind == TR_MASK_FULL || tk == 0) {
    // identity rows without reading the inputs (ref _kernels_ref.py:37-38)
    int rc = cuda_status(cudaMemsetAsync(out, 0, size_t(tq) * heads * head_dim * 2, s), "memset out");
    if (rc) return rc;
    return launch_fill(lse, tq * heads, -INFINITY, s);
  }
  tr_segment qs{0, tq, q_offset};
  tr_segment ks{0, tk, k_offset};
  return run_segments(q, k, v, out, lse, tq, tk, heads, head_dim, &qs, 1, &ks, 1,
                      mask_kind == TR_MASK_CAUSAL, TR_DTYPE_BF16, s);
}

int tr_attention_segments(const void* q, const void* k, const void* v, void* out, float* lse,
                          int64_t tq_total, int64_t tk_total, int32_t heads, int32_t head_dim,
                          const tr_segment* q_segs, int32_t n_q, const tr_segment* kv_segs,
                          int32_t n_kv, int32_t causal, int32_t out_dtype, void* stream) {
  return run_segments(q, k, v, out, lse, tq_total, tk_total, heads, head_dim, q_segs, n_q, kv_segs,
                      n_kv, causal, out_dtype, static_cast<cudaStream_t>(stream));
}

static int segments_push(const void* q, const void* k, const void* v, void* out, float* lse,
                               int64_t tq_total, int64_t tk_total, int32_t heads, int32_t head_dim,
                               const tr_segment* q_segs, int32_t n_q, const tr_segment* kv_segs,
                               int32_t n_kv, int32_t causal, int64_t row_shift, int64_t lse_stride,
                               uint32_t* done_count, uint64_t* done_flag, uint64_t done_value,
                               const int64_t* done_epoch, void* stream) {
  if (!out || !lse) return fail(TR_ERR_INPUT, "null out/lse");
  if (row_shift < 0 || lse_stride < 1) return fail(TR_ERR_DIMENSION, "row_shift >= 0, lse_stride >= 1 required");
  if ((done_flag == nullptr) != (done_count == nullptr))
    return fail(TR_ERR_INPUT, "done_flag and done_count go together");
  for (int i = 0; i < n_q && i < TR_MAX_SEGMENTS; ++i)
    if (q_segs[i].rows > 0 && (q_segs[i].row0 < row_shift || q_segs[i].row0 + q_segs[i].rows - row_shift > lse_stride))
      return fail(TR_ERR_DIMENSION, "q segment rows fall outside the receive buffer");
  PushOpts push;
  push.row_shift = row_shift;
  push.lse_stride = lse_stride;
  push.done_count = done_count;
  push.done_flag = reinterpret_cast<unsigned long long*>(done_flag);
  push.done_value = done_value;
  push.done_epoch = reinterpret_cast<const long long*>(done_epoch);
  return run_segments(q, k, v, out, lse, tq_total, tk_total, heads, head_dim, q_segs, n_q, kv_segs,
                      n_kv, causal, TR_DTYPE_BF16, static_cast<cudaStream_t>(stream), push);
}

int tr_attention_segments_push(const void* q, const void* k, const void* v, void* out, float* lse,
                               int64_t tq_total, int64_t tk_total, int32_t heads, int32_t head_dim,
                               const tr_segment* q_segs, int32_t n_q, const tr_segment* kv_segs,
                               int32_t n_kv, int32_t causal, int64_t row_shift, int64_t lse_stride,
                               uint32_t* done_count, uint64_t* done_flag, uint64_t done_value,
                               void* stream) {
  return segments_push(q, k, v, out, lse, tq_total, tk_total, heads, head_dim, q_segs, n_q, kv_segs,
                       n_kv, causal, row_shift, lse_stride, done_count, done_flag, done_value,
                       nullptr, stream);
}

int tr_attention_segments_push_rel(const void* q, const void* k, const void* v, void* out,
                                   float* lse, int64_t tq_total, int64_t tk_total, int32_t heads,
                                   int32_t head_dim, const tr_segment* q_segs, int32_t n_q,
                                   const tr_segment* kv_segs, int32_t n_kv, int32_t causal,
                                   int64_t row_shift, int64_t lse_stride, uint32_t* done_count,
                                   uint64_t* done_flag, const int64_t* done_epoch,
                                   int64_t done_offset, void* stream) {
  if (!done_epoch) return fail(TR_ERR_INPUT, "null epoch");
  return segments_push(q, k, v, out, lse, tq_total, tk_total, heads, head_dim, q_segs, n_q, kv_segs,
                       n_kv, causal, row_shift, lse_stride, done_count, done_flag,
                       static_cast<uint64_t>(done_offset), done_epoch, stream);
}

int tr_merge_state(float* acc_out, float* acc_lse, const void* blk_out, int32_t blk_dtype,
                   const float* blk_lse, int64_t tokens, int32_t heads, int32_t head_dim,
                   int64_t acc_lse_stride, int64_t blk_lse_stride, void* final_out, void* stream) {
  if (tokens < 0 || heads < 1 || head_dim < 1)
    return fail(TR_ERR_DIMENSION, "tokens >= 0, heads >= 1, head_dim >= 1 required");
  if (acc_lse_stride < tokens || blk_lse_stride < tokens)
    return fail(TR_ERR_DIMENSION, "lse row stride smaller than the token count");
  return launch_merge(acc_out, acc_lse, blk_out, blk_dtype, blk_lse, tokens, heads, head_dim,
                      acc_lse_stride, blk_lse_stride, final_out, static_cast<cudaStream_t>(stream));
}

int tr_merge_n(float* acc_out, float* acc_lse, int64_t acc_lse_stride, const void* const* blk_out,
               int32_t blk_dtype, const float* const* blk_lse, const int64_t* blk_lse_stride,
               int32_t n_blk, int64_t tokens, int32_t heads, int32_t head_dim, void* final_out,
               void* stream) {
  if (tokens < 0 || heads < 1 || head_dim < 1)
    return fail(TR_ERR_DIMENSION, "tokens >= 0, heads >= 1, head_dim >= 1 required");
  if (acc_lse_stride < tokens) return fail(TR_ERR_DIMENSION, "lse row stride smaller than the token count");
  if (n_blk > 0 && (!blk_out || !blk_lse || !blk_lse_stride))
    return fail(TR_ERR_INPUT, "null block arrays");
  return launch_merge_n(acc_out, acc_lse, acc_lse_stride, blk_out, blk_dtype, blk_lse,
                        blk_lse_stride, n_blk, tokens, heads, head_dim, final_out,
                        static_cast<cudaStream_t>(stream));
}

int tr_partial_init(float* acc_out, float* acc_lse, int64_t tokens, int32_t heads,
                    int32_t head_dim, void* stream) {
  if (tokens < 0 || heads < 1 || head_dim < 1)
    return fail(TR_ERR_DIMENSION, "tokens >= 0, heads >= 1, head_dim >= 1 required");
  return launch_partial_init(acc_out, acc_lse, tokens, heads, head_dim,
                             static_cast<cudaStream_t>(stream));
}

int tr_splitmix_bf16(uint64_t seed, int64_t first, int64_t count, double low, double high,
                     void* dst, void* stream) {
  if (first < 0 || count < 0) return fail(TR_ERR_CONFIG, "first and count must be >= 0");
  return launch_splitmix(seed, first, count, low, high, dst, static_cast<cudaStream_t>(stream));
}

int tr_flag_set(uint64_t* flag, uint64_t value, void* stream) {
  if (!flag) return fail(TR_ERR_INPUT, "null flag");
  return launch_flag_set(reinterpret_cast<unsigned long long*>(flag), value,
                         static_cast<cudaStream_t>(stream));
}

int tr_flag_wait(const uint64_t* flag, uint64_t value, void* stream) {
  if (!flag) return fail(TR_ERR_INPUT, "null flag");
  return launch_flag_wait(reinterpret_cast<const unsigned long long*>(flag), value,
                          static_cast<cudaStream_t>(stream));
}

int tr_flag_set_rel(uint64_t* flag, const int64_t* epoch, int64_t offset, void* stream) {
  if (!flag || !epoch) return fail(TR_ERR_INPUT, "null flag or epoch");
  return launch_flag_set(reinterpret_cast<unsigned long long*>(flag),
                         static_cast<unsigned long long>(offset), static_cast<cudaStream_t>(stream),
                         reinterpret_cast<const long long*>(epoch));
}

int tr_flag_wait_rel(const uint64_t* flag, const int64_t* epoch, int64_t offset, void* stream) {
  if (!flag || !epoch) return fail(TR_ERR_INPUT, "null flag or epoch");
  return launch_flag_wait(reinterpret_cast<const unsigned long long*>(flag),
                          static_cast<unsigned long long>(offset), static_cast<cudaStream_t>(stream),
                          reinterpret_cast<const long long*>(epoch));
}

int tr_epoch_add(int64_t* epoch, int64_t delta, void* stream) {
  if (!epoch) return fail(TR_ERR_INPUT, "null epoch");
  return launch_epoch_add(reinterpret_cast<long long*>(epoch), delta,
                          static_cast<cudaStream_t>(stream));
}

int tr_copy_async(void* dst, const void* src, uint64_t bytes, void* stream) {
  if (bytes == 0) return TR_OK;
  if (!dst || !src) return fail(TR_ERR_INPUT, "null pointer");
  return cuda_status(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault,
                                     static_cast<cudaStream_t>(stream)),
                     "tr_copy_async");
}

int tr_enable_peer_access(int32_t peer_device) {
  int cur = 0;
  int rc = cuda_status(cudaGetDevice(&cur), "cudaGetDevice");
  if (rc) return rc;
  if (peer_device == cur) return TR_OK;
  int can = 0;
  if ((rc = cuda_status(cudaDeviceCanAccessPeer(&can, cur, peer_device), "cudaDeviceCanAccessPeer")))
    return rc;
  if (!can)
    return fail(TR_ERR_UNSUPPORTED, "device " + std::to_string(cur) + " cannot access device " +
                                        std::to_string(peer_device) + " (no P2P path)");
  cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) {
    cudaGetLastError();   // clear the sticky-free status
    return TR_OK;
  }
  return cuda_status(e, "cudaDeviceEnablePeerAccess");
}

int tr_poll_error(void) { return poll_flag_error(); }

int32_t tr_set_launch_overlap(int32_t flags) {
  const int32_t prev = g_launch_overlap;
  g_launch_overlap = flags & (TR_LAUNCH_AFTER_PREV | TR_LAUNCH_RELEASE_NEXT);
  return prev;
}
void tr_clear_error(void) { clear_flag_error(); }
void tr_set_flag_timeout_ms(uint64_t ms) { set_flag_timeout_ns(ms * 1000000ull); }

// every __global__ kernel of the product library (templates once);
// tests/test_abi.py checks this list against the cubin's symbol table
static const char* const kKernels[] = {
    "attn_fwd_pair2_kernel",  "attn_fwd_sm100_kernel", "attn_simt_kernel",
    "merge_vec8_kernel",      "merge_scalar_kernel",   "merge_scalar_lse_kernel",
    "merge_n_vec8_kernel",    "merge_n_bf16_kernel",   "merge_n_scalar_kernel",
    "merge_n_lse_kernel",     "fill_kernel",
    "flag_set_kernel",        "flag_wait_kernel",      "epoch_add_kernel",
    "splitmix_bf16_kernel"};

const char* tr_version(void) { return "tokenring-b200 0.2 (sm_100a)"; }
int32_t tr_kernel_count(void) { return int32_t(sizeof(kKernels) / sizeof(kKernels[0])); }
const char* tr_kernel_name(int32_t i) {
  return i >= 0 && i < tr_kernel_count() ? kKernels[i] : nullptr;
}
const char* tr_last_error(void) { return g_last_error.c_str(); }

}  // extern "C"
