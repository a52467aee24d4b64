// Internal declarations shared by the CUDA translation units of libtokenring.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../include/tokenring.h"

namespace tr {

// thread-local last error (tr_last_error)
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_status(cudaError_t e, const char* what);

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
};

// tcgen05 kernel (D in {64,128}); returns TR_OK or an error status
int launch_attn_sm100(const void* q, const void* k, const void* v, int64_t tq_total,
                      int64_t tk_total, int head_dim, AttnPlan& plan, cudaStream_t s);
// generic CUDA-core kernel for any head_dim <= 256 (small shapes, odd dims)
int launch_attn_simt(const void* q, const void* k, const void* v, int head_dim, AttnPlan& plan,
                     cudaStream_t s);
bool sm100_supports(int head_dim, int heads, const void* q, const void* k, const void* v,
                    const void* out);

}  // namespace tr
