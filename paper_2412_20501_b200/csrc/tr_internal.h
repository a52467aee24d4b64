// Internal declarations shared by the CUDA translation units of libtokenring.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/tokenring.h"

namespace tr {

constexpr int TR_ORDER_MAX = 2048;   // (segment, tile) classes an explicit CTA order can hold

// thread-local last error (tr_last_error)
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* what);
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device):
// the attribute is per device, so a process driving several GPUs sets it on each
int set_smem_attr_once(const void* func, int bytes, const char* what);

struct AttnPlan {
  tr_segment q[TR_MAX_SEGMENTS];
  tr_segment kv[TR_MAX_SEGMENTS];
  int64_t tile_prefix[TR_MAX_SEGMENTS + 1];  // cumulative 256-row q tiles per q segment
  int64_t lse_stride;                        // row stride of lse (= tq_total)
  int32_t nq, nkv;
  int32_t causal;
  int32_t heads;
  float scale;       // 1/sqrt(D)
  float scale_log2;  // log2(e)/sqrt(D)
  int32_t out_f32;   // out is float32 (an empty accumulator) instead of bf16
  void* out;
  float* lse;
  // Fused OUT push (tr_attention_segments_push): out/lse may be a peer GPU's
  // receive buffer (NVLink stores from the epilogue).  When done_flag is set,
  // the last CTA to finish raises it to done_value (system-scope release)
  // and resets done_count for the next launch on the stream.
  unsigned int* done_count;
  unsigned long long* done_flag;
  unsigned long long done_value;
  // epoch-relative done value (CUDA-graph replays): when set, the flag is
  // raised to *done_epoch + (signed) done_value, read when the kernel ends
  const long long* done_epoch;
  // Longest-first CTA order for multi-segment causal launches (n_order > 0):
  // heads in groups of `head_group` (so a group's K/V stays in L2); inside a
  // group the (segment, tile) classes run in order[] -- sorted by decreasing
  // kv-tile count -- with the group's heads innermost.  n_order == 0: the
  // plain order (head-major, each causal segment heaviest tile first).
  int32_t n_order;
  int32_t head_group;
  // tr_set_launch_overlap: launch as a programmatic dependent of the previous
  // kernel on the stream (host side; the kernel never waits on it), and let
  // the next launch start once every CTA of this one is resident (device:
  // griddepcontrol.launch_dependents -- only when asked, it is not free:
  // -0.5..0.9 % sustained when executed by every plain launch)
  int32_t overlap_prev;
  int32_t release_next;
  uint16_t order[TR_ORDER_MAX];
};

// last-CTA completion signal of a pushing launch (see AttnPlan::done_flag);
// call from one thread per CTA after every thread of the CTA has executed
// __threadfence_system() behind its out/lse stores and a __syncthreads().
__device__ __forceinline__ void signal_done(const AttnPlan& p) {
  const unsigned int prev = atomicAdd(p.done_count, 1u);
  if (prev == gridDim.x - 1) {
    *p.done_count = 0u;
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    const unsigned long long v =
        p.done_epoch ? static_cast<unsigned long long>(*p.done_epoch + static_cast<long long>(p.done_value))
                     : p.done_value;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p.done_flag), "l"(v) : "memory");
  }
}

// tcgen05 kernel (D in {64,128}); returns TR_OK or an error status
int launch_attn_sm100(const void* q, const void* k, const void* v, int64_t tq_total,
                      int64_t tk_total, int head_dim, AttnPlan& plan, cudaStream_t s);
// generic CUDA-core kernel for any head_dim <= 256 (small shapes, odd dims)
int launch_flag_set(unsigned long long* flag, unsigned long long value, cudaStream_t s,
                    const long long* epoch = nullptr);
int launch_flag_wait(const unsigned long long* flag, unsigned long long value, cudaStream_t s,
                     const long long* epoch = nullptr);
int launch_epoch_add(long long* epoch, long long delta, cudaStream_t s);
// host-mapped record of a timed-out flag wait (p2p_flags.cu)
int poll_flag_error();
void clear_flag_error();
void set_flag_timeout_ns(unsigned long long ns);
// thread-local launch option (tr_set_launch_overlap): attention, flag-wait
// and flag-set launches become programmatic dependents of the previous
// kernel on their stream
bool launch_overlap();
bool launch_release_next();

// kernel<<<grid, block, smem, s>>>(args...), or the same as a programmatic
// dependent launch when `overlap` (cudaLaunchAttributeProgrammaticStreamSerialization)
template <typename... KArgs, typename... Args>
cudaError_t launch_kernel(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t s, bool overlap, Args... args) {
  if (!overlap) {
    kernel<<<grid, block, smem, s>>>(args...);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}
int launch_attn_simt(const void* q, const void* k, const void* v, int head_dim, AttnPlan& plan,
                     cudaStream_t s);
bool sm100_supports(int head_dim, int heads, const void* q, const void* k, const void* v,
                    const void* out);

}  // namespace tr
