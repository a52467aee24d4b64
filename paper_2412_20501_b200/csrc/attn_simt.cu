// Generic CUDA-core block attention for head dims the tcgen05 kernel does not
// cover (any D <= 256, any alignment).  Same contract as attn_fwd_sm100.cu
// (ref _kernels_ref.py:34-54): one warp per (query row, head), exact online
// softmax in fp32 over the visible keys of every kv segment.
#include <cuda_bf16.h>
#include <cmath>

#include "tr_internal.h"
#include "tr_ptx.cuh"

namespace tr {

constexpr int kSimtMaxD = 256;

__global__ void __launch_bounds__(256) attn_simt_kernel(const __nv_bfloat16* __restrict__ q,
                                                        const __nv_bfloat16* __restrict__ k,
                                                        const __nv_bfloat16* __restrict__ v,
                                                        int D, const AttnPlan p) {
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  const int64_t total_rows = p.tile_prefix[p.nq];  // here: rows, not tiles
  if (warp_global >= total_rows * p.heads) return;
  const int head = warp_global % p.heads;
  int64_t lin = warp_global / p.heads;
  int seg = 0;
  while (seg + 1 < p.nq && lin >= p.tile_prefix[seg + 1]) ++seg;
  const int64_t r = lin - p.tile_prefix[seg];
  const int64_t row = p.q[seg].row0 + r;
  const int64_t pos = p.q[seg].pos0 + r;
  const int64_t ld = int64_t(p.heads) * D;

  constexpr int PER = kSimtMaxD / 32;
  float qv[PER], acc[PER];
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int d = lane + 32 * i;
    qv[i] = d < D ? __bfloat162float(q[row * ld + head * D + d]) : 0.f;
    acc[i] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int g = 0; g < p.nkv; ++g) {
    int64_t n = p.kv[g].rows;
    if (p.causal) n = imax64(0, imin64(n, pos - p.kv[g].pos0 + 1));
    for (int64_t j = 0; j < n; ++j) {
      const int64_t kr = (p.kv[g].row0 + j) * ld + head * D;
      float dot = 0.f;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int d = lane + 32 * i;
        if (d < D) dot += qv[i] * __bfloat162float(k[kr + d]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
      const float s = dot * p.scale;
      const float mn = fmaxf(m, s);
      const float alpha = (m == -INFINITY) ? 0.f : expf(m - mn);
      const float w = expf(s - mn);
      l = l * alpha + w;
#pragma unroll
      for (int i = 0; i < PER; ++i) {
        const int d = lane + 32 * i;
        const float vv = d < D ? __bfloat162float(v[kr + d]) : 0.f;
        acc[i] = acc[i] * alpha + w * vv;
      }
      m = mn;
    }
  }
  const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int d = lane + 32 * i;
    if (d >= D) continue;
    if (p.out_f32)
      reinterpret_cast<float*>(p.out)[row * ld + head * D + d] = acc[i] * inv;
    else
      reinterpret_cast<__nv_bfloat16*>(p.out)[row * ld + head * D + d] =
          __float2bfloat16_rn(acc[i] * inv);
  }
  if (lane == 0) p.lse[head * p.lse_stride + row] = l > 0.f ? m + logf(l) : -INFINITY;
}

int launch_attn_simt(const void* q, const void* k, const void* v, int head_dim, AttnPlan& plan,
                     cudaStream_t s) {
  if (head_dim > kSimtMaxD) return fail(TR_ERR_UNSUPPORTED, "head_dim > 256 not supported");
  // reuse tile_prefix as a row prefix for this kernel
  plan.tile_prefix[0] = 0;
  for (int i = 0; i < plan.nq; ++i) plan.tile_prefix[i + 1] = plan.tile_prefix[i] + plan.q[i].rows;
  const int64_t warps = plan.tile_prefix[plan.nq] * plan.heads;
  if (warps == 0) return TR_OK;
  const int64_t blocks = (warps * 32 + 255) / 256;
  attn_simt_kernel<<<static_cast<unsigned>(blocks), 256, 0, s>>>(
      static_cast<const __nv_bfloat16*>(q), static_cast<const __nv_bfloat16*>(k),
      static_cast<const __nv_bfloat16*>(v), head_dim, plan);
  return cuda_status(cudaGetLastError(), "attn_simt launch");
}

}  // namespace tr
