/*
 * tokenring.h -- C ABI of libtokenring.so, the B200 (sm_100a) TokenRing
 * attention path.
 *
 * Every entry point takes plain device pointers, sizes and a cudaStream_t
 * passed as void*; none of them synchronises the device.  The only state kept
 * across calls is per process: the kernels' shared-memory attribute (set once
 * per device), the pinned status block of the flag waits (tr_poll_error) and
 * the calling thread's last error message.
 * All return TR_OK (0) or a negative status; the message of the last failure
 * on the calling thread is available from tr_last_error().
 *
 * Tensor conventions (same as the reference, pkg/src/ringsim/core.py:5-7):
 *   q, k, v, out : token-major (T, H, D), contiguous, bf16 unless stated
 *   lse          : head-major  (H, T) float32, natural log, -inf = empty row
 *
 * Reference interfaces replaced (all paths relative to /root/reference):
 *   tr_attention_block  <- kernels.attention_block   pkg/src/ringsim/kernels.py:39
 *                          (_kernels_ref.py:34-54, _kernels.pyx:15-65)
 *   tr_merge_state      <- kernels.merge_state       pkg/src/ringsim/kernels.py:40
 *                          (_kernels_ref.py:66-73, _kernels.pyx:68-102)
 *   tr_attention_segments  the per-step block computations of
 *                          engine.execute pkg/src/ringsim/engine.py:558-593
 *                          (several ComputePlans of one step in one launch)
 *   tr_splitmix_bf16    <- rng.uniform / attention_inputs pkg/src/ringsim/rng.py:34-53
 */
#ifndef TOKENRING_H_
#define TOKENRING_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python layer maps them onto ringsim's exception types
 * (pkg/src/ringsim/errors.py:4-25). */
#define TR_OK 0
#define TR_ERR_DIMENSION -1   /* DimensionError */
#define TR_ERR_INPUT -2       /* InputError */
#define TR_ERR_CONFIG -3      /* ConfigError */
#define TR_ERR_CUDA -4        /* CUDA runtime / driver failure */
#define TR_ERR_UNSUPPORTED -5 /* shape the sm_100a kernels do not cover */
#define TR_ERR_TIMEOUT -6     /* ScheduleError: a message never arrived (tr_poll_error) */

/* mask kinds, identical to ringsim.kernels.MASK_* (pkg/src/ringsim/kernels.py:33-35) */
#define TR_MASK_NONE 0
#define TR_MASK_FULL 1
#define TR_MASK_CAUSAL 2

/* dtypes for merge operands */
#define TR_DTYPE_F32 0
#define TR_DTYPE_BF16 1

/* One contiguous run of tokens inside a local (T, H, D) buffer:
 * local rows [row0, row0 + rows) sit at global sequence positions
 * [pos0, pos0 + rows).  Causal visibility is decided on positions:
 * key j is visible to query i iff pos(i) >= pos(j)  (ref _kernels_ref.py:42-44). */
typedef struct tr_segment {
  int64_t row0;
  int64_t rows;
  int64_t pos0;
} tr_segment;

#define TR_MAX_SEGMENTS 4

/* kernels.attention_block: out (tq,H,D) bf16, lse (H,tq) f32 for one q block
 * against one kv block.  mask_kind FULL writes the identity (0 / -inf)
 * without reading q/k/v.  CAUSAL uses q_offset/k_offset as global positions. */
int tr_attention_block(const void* q, const void* k, const void* v, void* out, float* lse,
                       int64_t tq, int64_t tk, int32_t heads, int32_t head_dim,
                       int32_t mask_kind, int64_t q_offset, int64_t k_offset, void* stream);

/* Several q segments of one local q buffer against several kv segments of one
 * local k/v buffer, in one launch.  Every q segment attends to the union of the
 * kv segments (causal: by position).  out/lse rows follow q's local rows;
 * lse has row stride tq_total.  Rows of q not covered by a segment are left
 * untouched.  out_dtype TR_DTYPE_BF16 writes a bf16 block result;
 * TR_DTYPE_F32 writes float32 rows, so a block that is the first contribution
 * to a float32 accumulator (engine.py:585-589 merging into Partial.empty)
 * lands in it directly, with no bf16 round trip, init or merge pass. */
int tr_attention_segments(const void* q, const void* k, const void* v, void* out, float* lse,
                          int64_t tq_total, int64_t tk_total, int32_t heads, int32_t head_dim,
                          const tr_segment* q_segs, int32_t n_q, const tr_segment* kv_segs,
                          int32_t n_kv, int32_t causal, int32_t out_dtype, void* stream);

/* tr_attention_segments fused with the OUT_LSE message of the next step
 * (engine.py:346-353 sends the rows computed at step i to their home at step
 * i+1, where MergePlan folds them in, engine.py:187-200): the epilogue stores
 * the bf16 rows and their lse straight into the HOME rank's receive buffer --
 * `out`/`lse` may be CUDA-IPC-mapped peer memory, so the transfer rides
 * NVLink/NVSwitch tile by tile while the rest of the grid still computes.
 * Row r of q's local buffer lands at row r - row_shift of out (and of each
 * lse head row, stride lse_stride).  If done_flag != NULL the last CTA to
 * finish raises *done_flag to done_value with a system-scope release (after
 * every CTA's stores are fenced); done_count is a zeroed device counter the
 * launch uses and leaves zeroed. */
int tr_attention_segments_push(const void* q, const void* k, const void* v, void* out, float* lse,
                               int64_t tq_total, int64_t tk_total, int32_t heads, int32_t head_dim,
                               const tr_segment* q_segs, int32_t n_q, const tr_segment* kv_segs,
                               int32_t n_kv, int32_t causal, int64_t row_shift, int64_t lse_stride,
                               uint32_t* done_count, uint64_t* done_flag, uint64_t done_value,
                               void* stream);
int tr_attention_segments_push_rel(const void* q, const void* k, const void* v, void* out,
                                   float* lse, int64_t tq_total, int64_t tk_total, int32_t heads,
                                   int32_t head_dim, const tr_segment* q_segs, int32_t n_q,
                                   const tr_segment* kv_segs, int32_t n_kv, int32_t causal,
                                   int64_t row_shift, int64_t lse_stride, uint32_t* done_count,
                                   uint64_t* done_flag, const int64_t* done_epoch,
                                   int64_t done_offset, void* stream);

/* Launch options of the calling thread's later D=64/128 attention launches
 * (tr_attention_block / _segments / _segments_push*), flag-wait and flag-set
 * launches; flags, 0 (the default) = plain stream-ordered launches:
 *   TR_LAUNCH_AFTER_PREV   the launch is a programmatic dependent of the
 *                          previous kernel on its stream: its CTAs start on
 *                          the SMs the previous grid's last wave frees instead
 *                          of after the whole grid.  It does not wait for the
 *                          previous kernel's results -- only for a TokenRing
 *                          step every message of which was waited for by an
 *                          earlier kernel.
 *   TR_LAUNCH_RELEASE_NEXT an attention launch releases its programmatic
 *                          dependent as soon as all of its CTAs are resident
 *                          (griddepcontrol.launch_dependents; without it the
 *                          dependent starts when the grid ends).
 * Returns the previous flags.  No counterpart in the reference, whose steps
 * run one after another on the host (engine.py:468-638). */
#define TR_LAUNCH_AFTER_PREV 1
#define TR_LAUNCH_RELEASE_NEXT 2
int32_t tr_set_launch_overlap(int32_t flags);

/* kernels.merge_state, in place on a float32 accumulator:
 *   acc <- merge(acc, blk)     (ref _kernels.pyx:68-102)
 * blk_out is bf16 or f32 (blk_dtype); -inf rows are exact identities.
 * If final_out != NULL the merged output is also written there as bf16. */
int tr_merge_state(float* acc_out, float* acc_lse, const void* blk_out, int32_t blk_dtype,
                   const float* blk_lse, int64_t tokens, int32_t heads, int32_t head_dim,
                   int64_t acc_lse_stride, int64_t blk_lse_stride, void* final_out,
                   void* stream);

/* N-way form of tr_merge_state: acc <- merge(acc, blk_0, ..., blk_{n-1}) in one
 * pass (every MergePlan a chunk receives over the schedule, engine.py:187-200
 * and 620-628, folded at once -- the merge is associative and commutative).
 * blk_out[i] points at `tokens` rows (T, H, D) of dtype blk_dtype;
 * blk_lse[i] at an (H, .) float32 array with row stride blk_lse_stride[i].
 * The pointer arrays are host memory; n_blk <= TR_MERGE_MAX.  If final_out !=
 * NULL the merged output is also written there as bf16. */
#define TR_MERGE_MAX 16
int tr_merge_n(float* acc_out, float* acc_lse, int64_t acc_lse_stride, const void* const* blk_out,
               int32_t blk_dtype, const float* const* blk_lse, const int64_t* blk_lse_stride,
               int32_t n_blk, int64_t tokens, int32_t heads, int32_t head_dim, void* final_out,
               void* stream);

/* Identity accumulator (Partial.empty, ref core.py:75-78): out = 0, lse = -inf. */
int tr_partial_init(float* acc_out, float* acc_lse, int64_t tokens, int32_t heads,
                    int32_t head_dim, void* stream);

/* SplitMix64 draws [first, first+count) of `seed` mapped to uniform
 * [low, high) in float64 exactly as rng.uniform, then rounded
 * fp64 -> fp32 -> bf16 (RNE).  dst receives `count` bf16 values. */
int tr_splitmix_bf16(uint64_t seed, int64_t first, int64_t count, double low, double high,
                     void* dst, void* stream);

/* Copy-engine transport support (CUDA IPC / NVLink peer memory).  A sender
 * cudaMemcpyAsync's a block into the peer's mapped receive buffer and then
 * raises the peer's 64-bit sequence flag with a system-scope release store;
 * the receiver's stream spins (one thread, acquire loads) until its flag
 * reaches the expected value.  Replaces the in-process message delivery of
 * engine.execute (pkg/src/ringsim/engine.py:515-518, 595-619). */
int tr_flag_set(uint64_t* flag, uint64_t value, void* stream);
int tr_flag_wait(const uint64_t* flag, uint64_t value, void* stream);
/* Epoch-relative forms for CUDA-graph replay: the value is *epoch + offset,
 * read on the device when the operation runs (epoch: a device int64 of the
 * caller), and tr_epoch_add(epoch, delta) advances it at the end of a
 * captured forward -- a replayed graph then uses fresh sequence values without
 * any host work.  tr_attention_segments_push_rel raises done_flag to
 * *done_epoch + done_offset. */
int tr_flag_set_rel(uint64_t* flag, const int64_t* epoch, int64_t offset, void* stream);
int tr_flag_wait_rel(const uint64_t* flag, const int64_t* epoch, int64_t offset, void* stream);
int tr_epoch_add(int64_t* epoch, int64_t delta, void* stream);
int tr_copy_async(void* dst, const void* src, uint64_t bytes, void* stream);
/* Let kernels of the calling thread's current device load/store memory of
 * peer_device (flags, receive slots mapped over CUDA IPC): wraps
 * cudaDeviceEnablePeerAccess; TR_OK if already enabled or the same device,
 * TR_ERR_UNSUPPORTED if the two devices have no P2P path. */
int tr_enable_peer_access(int32_t peer_device);

/* A tr_flag_wait that times out (a lost or never-sent message; default 30 s)
 * does not trap -- that would kill the CUDA context -- but records the flag,
 * the expected and the observed value in a pinned host-mapped block and lets
 * the stream go on (its results are then invalid).  tr_poll_error() reads that
 * block without touching the device: TR_OK, or TR_ERR_TIMEOUT with the record
 * in tr_last_error() (the reference raises ScheduleError for an undelivered
 * message, engine.py:532-537).  tr_clear_error() re-arms it;
 * tr_set_flag_timeout_ms() changes the timeout of later waits (tests). */
int tr_poll_error(void);
void tr_clear_error(void);
void tr_set_flag_timeout_ms(uint64_t ms);

/* Version / capability probes (no GPU work).  tr_kernel_count() is the number
 * of __global__ kernels (templates counted once) in the library and
 * tr_kernel_name(i) their names, i in [0, count) (NULL outside). */
const char* tr_version(void);
int32_t tr_kernel_count(void);
const char* tr_kernel_name(int32_t i);
const char* tr_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* TOKENRING_H_ */
