// Log-sum-exp merge of a block partial into a float32 accumulator, in place
// (paper Update; ref _kernels.pyx:68-102):
//   b == -inf            -> acc unchanged (exact identity)
//   a == -inf            -> acc = blk, lse = b
//   else  d = b - a, e = exp(-|d|), w = sigmoid(d) via the sign branch,
//         lse = max(a,b) + log1p(e),  out = acc + w * (blk - acc)
// HBM-bound: rows are walked head-major (h, t) so lse reads/writes coalesce
// and every row's D contiguous values go through 16-byte vector accesses.
#include <cuda_bf16.h>
#include <cmath>
#include <type_traits>

#include "tr_internal.h"

namespace tr {

template <typename BT>
struct Vec8;
template <>
struct Vec8<__nv_bfloat16> {
  __device__ static void load(const __nv_bfloat16* p, float (&x)[8]) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[2 * i] = __uint_as_float(w[i] << 16);
      x[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
};
template <>
struct Vec8<float> {
  __device__ static void load(const float* p, float (&x)[8]) {
    const float4 a = __ldg(reinterpret_cast<const float4*>(p));
    const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
    x[0] = a.x; x[1] = a.y; x[2] = a.z; x[3] = a.w;
    x[4] = b.x; x[5] = b.y; x[6] = b.z; x[7] = b.w;
  }
};

__device__ __forceinline__ uint32_t bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// One thread = 8 consecutive values of one (t, h) row; D % 8 == 0.  The lse
// update runs as a second (tiny) kernel so no thread can observe a row's new
// lse before reading the old one.
template <typename BT>
__global__ void __launch_bounds__(256) merge_vec8_kernel(float* __restrict__ acc_out,
                                                         float* __restrict__ acc_lse,
                                                         const BT* __restrict__ blk_out,
                                                         const float* __restrict__ blk_lse,
                                                         int64_t T, int H, int D,
                                                         int64_t acc_ls, int64_t blk_ls,
                                                         __nv_bfloat16* __restrict__ final_out) {
  const int per_row = D / 8;
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t row = gid / per_row;  // head-major row index
  if (row >= T * H) return;
  const int part = static_cast<int>(gid % per_row);
  const int h = static_cast<int>(row / T);
  const int64_t t = row % T;
  const float a = acc_lse[h * acc_ls + t];
  const float b = blk_lse[h * blk_ls + t];
  const int64_t off = (t * H + h) * D + part * 8;
  float* ap = acc_out + off;
  float o[8];
  if (b == -INFINITY) {
    if (!final_out) return;
    const float4 x0 = *reinterpret_cast<const float4*>(ap);
    const float4 x1 = *(reinterpret_cast<const float4*>(ap) + 1);
    o[0] = x0.x; o[1] = x0.y; o[2] = x0.z; o[3] = x0.w;
    o[4] = x1.x; o[5] = x1.y; o[6] = x1.z; o[7] = x1.w;
  } else {
    float blk[8];
    Vec8<BT>::load(blk_out + off, blk);
    if (a == -INFINITY) {
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = blk[i];
    } else {
      const float d = b - a;
      const float e = expf(-fabsf(d));
      const float w = d >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
      const float4 x0 = *reinterpret_cast<const float4*>(ap);
      const float4 x1 = *(reinterpret_cast<const float4*>(ap) + 1);
      const float x[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i] = fmaf(w, blk[i] - x[i], x[i]);
    }
    reinterpret_cast<float4*>(ap)[0] = make_float4(o[0], o[1], o[2], o[3]);
    reinterpret_cast<float4*>(ap)[1] = make_float4(o[4], o[5], o[6], o[7]);
  }
  if (final_out)
    *reinterpret_cast<uint4*>(final_out + off) =
        make_uint4(bf16x2(o[0], o[1]), bf16x2(o[2], o[3]), bf16x2(o[4], o[5]), bf16x2(o[6], o[7]));
}

// Scalar fallback for D % 8 != 0 or unaligned buffers: one thread per value.
template <typename BT>
__global__ void merge_scalar_kernel(float* acc_out, float* acc_lse, const BT* blk_out,
                                    const float* blk_lse, int64_t T, int H, int D, int64_t acc_ls,
                                    int64_t blk_ls, __nv_bfloat16* final_out) {
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= T * H * D) return;
  const int64_t row = gid / D;
  const int d = static_cast<int>(gid % D);
  const int h = static_cast<int>(row / T);
  const int64_t t = row % T;
  const float a = acc_lse[h * acc_ls + t];
  const float b = blk_lse[h * blk_ls + t];
  const int64_t off = (t * H + h) * D + d;
  float o = acc_out[off];
  if (b != -INFINITY) {
    const float blk = static_cast<float>(blk_out[off]);
    if (a == -INFINITY) {
      o = blk;
    } else {
      const float dd = b - a;
      const float e = expf(-fabsf(dd));
      const float w = dd >= 0.f ? 1.f / (1.f + e) : e / (1.f + e);
      o = fmaf(w, blk - o, o);
    }
    acc_out[off] = o;
  }
  if (final_out) final_out[off] = __float2bfloat16_rn(o);
}

__global__ void merge_scalar_lse_kernel(float* acc_lse, const float* blk_lse, int64_t T, int H,
                                        int64_t acc_ls, int64_t blk_ls) {
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= T * H) return;
  const int h = static_cast<int>(gid / T);
  const int64_t t = gid % T;
  const float a = acc_lse[h * acc_ls + t];
  const float b = blk_lse[h * blk_ls + t];
  if (b == -INFINITY) return;
  if (a == -INFINITY) { acc_lse[h * acc_ls + t] = b; return; }
  const float e = expf(-fabsf(b - a));
  acc_lse[h * acc_ls + t] = fmaxf(a, b) + log1pf(e);
}

// ---------------------------------------------------------------- N-way merge
// acc <- merge(acc, blk_0, ..., blk_{n-1}) in one pass: the reference folds
// returned partials one MergePlan at a time (engine.py:187-200, 620-628);
// the merge is associative and commutative (ref tests/test_core.py:151-173),
// so all of a row's partials are combined with one set of weights:
//   m = max(a, b_i),  w = exp(a - m), w_i = exp(b_i - m),  L = w + sum w_i
//   out = (w acc + sum w_i blk_i) / L,   lse = m + log L
// (-inf partials get weight 0; a row with every lse -inf stays 0 / -inf).
// HBM traffic per value: 4 (acc read) + n * sizeof(blk) + 4 (acc write),
// against n * (4 + sizeof(blk) + 4) for n pairwise merges.
struct MergeN {
  const void* blk[TR_MERGE_MAX];
  const float* lse[TR_MERGE_MAX];
  int64_t ls[TR_MERGE_MAX];
  int n;
};

template <typename BT>
__global__ void __launch_bounds__(256) merge_n_vec8_kernel(float* __restrict__ acc_out,
                                                           const float* __restrict__ acc_lse,
                                                           const __grid_constant__ MergeN m,
                                                           int64_t T, int H, int D, int64_t acc_ls,
                                                           __nv_bfloat16* __restrict__ final_out) {
  const int per_row = D / 8;
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t row = gid / per_row;  // head-major row index
  if (row >= T * H) return;
  const int part = static_cast<int>(gid % per_row);
  const int h = static_cast<int>(row / T);
  const int64_t t = row % T;
  const float a = acc_lse[h * acc_ls + t];
  float mx = a;
  float b[TR_MERGE_MAX];
#pragma unroll
  for (int i = 0; i < TR_MERGE_MAX; ++i) {
    b[i] = i < m.n ? __ldg(m.lse[i] + h * m.ls[i] + t) : -INFINITY;
    mx = fmaxf(mx, b[i]);
  }
  const int64_t off = (t * H + h) * D + part * 8;
  float* ap = acc_out + off;
  if (mx == -INFINITY) {          // nothing anywhere: the identity stays
    if (final_out) *reinterpret_cast<uint4*>(final_out + off) = make_uint4(0u, 0u, 0u, 0u);
    return;
  }
  float o[8];
  const float w0 = (a == -INFINITY) ? 0.f : __expf(a - mx);
  float L = w0;
  if (w0 != 0.f) {
    const float4 x0 = *reinterpret_cast<const float4*>(ap);
    const float4 x1 = *(reinterpret_cast<const float4*>(ap) + 1);
    o[0] = w0 * x0.x; o[1] = w0 * x0.y; o[2] = w0 * x0.z; o[3] = w0 * x0.w;
    o[4] = w0 * x1.x; o[5] = w0 * x1.y; o[6] = w0 * x1.z; o[7] = w0 * x1.w;
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = 0.f;
  }
  // (batching the block loads ahead of the math measured slower: 72 vs 42
  // registers, 0.241 vs 0.200 ms for c=8192, H=32, n=7)
#pragma unroll
  for (int i = 0; i < TR_MERGE_MAX; ++i) {
    if (i >= m.n) break;
    if (b[i] == -INFINITY) continue;      // exact identity: its values are never read
    const float w = __expf(b[i] - mx);
    L += w;
    float x[8];
    Vec8<BT>::load(static_cast<const BT*>(m.blk[i]) + off, x);
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = fmaf(w, x[k], o[k]);
  }
  const float inv = 1.f / L;
#pragma unroll
  for (int k = 0; k < 8; ++k) o[k] *= inv;
  reinterpret_cast<float4*>(ap)[0] = make_float4(o[0], o[1], o[2], o[3]);
  reinterpret_cast<float4*>(ap)[1] = make_float4(o[4], o[5], o[6], o[7]);
  if (final_out)
    *reinterpret_cast<uint4*>(final_out + off) =
        make_uint4(bf16x2(o[0], o[1]), bf16x2(o[2], o[3]), bf16x2(o[4], o[5]), bf16x2(o[6], o[7]));
}

// Compile-time block count (bf16 partials, N <= 8), 16 values per thread:
// each partial contributes two 16-byte loads per thread that ptxas issues
// together, so twice the bytes are in flight per thread than in the generic
// 8-value loop above (whose -inf test in front of every load also keeps a
// single load outstanding).  A partial whose lse is -inf contributes weight
// 0 and its values are never read.
template <int N>
__global__ void __launch_bounds__(256) merge_n_bf16_kernel(float* __restrict__ acc_out,
                                                           const float* __restrict__ acc_lse,
                                                           const __grid_constant__ MergeN m,
                                                           int64_t T, int H, int D, int64_t acc_ls,
                                                           __nv_bfloat16* __restrict__ final_out) {
  const int per_row = D / 16;
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t row = gid / per_row;
  if (row >= T * H) return;
  const int part = static_cast<int>(gid % per_row);
  const int h = static_cast<int>(row / T);
  const int64_t t = row % T;
  const int64_t off = (t * H + h) * D + part * 16;
  float* ap = acc_out + off;
  const float a = acc_lse[h * acc_ls + t];
  float b[N];
  float mx = a;
  #pragma unroll
  for (int i = 0; i < N; ++i) {
    b[i] = __ldg(m.lse[i] + h * m.ls[i] + t);
    mx = fmaxf(mx, b[i]);
  }
  if (mx == -INFINITY) {
    if (final_out) {
      reinterpret_cast<uint4*>(final_out + off)[0] = make_uint4(0u, 0u, 0u, 0u);
      reinterpret_cast<uint4*>(final_out + off)[1] = make_uint4(0u, 0u, 0u, 0u);
    }
    return;
  }
  float o[16];
  const float w0 = (a == -INFINITY) ? 0.f : __expf(a - mx);
  float L = w0;
  if (w0 != 0.f) {
    #pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 x = reinterpret_cast<const float4*>(ap)[q];
      o[4 * q] = w0 * x.x; o[4 * q + 1] = w0 * x.y; o[4 * q + 2] = w0 * x.z; o[4 * q + 3] = w0 * x.w;
    }
  } else {
    #pragma unroll
    for (int k = 0; k < 16; ++k) o[k] = 0.f;
  }
  #pragma unroll
  for (int i = 0; i < N; ++i) {
    if (b[i] == -INFINITY) continue;
    const float w = __expf(b[i] - mx);
    L += w;
    const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(m.blk[i]) + off);
    const uint4 r0 = __ldg(src), r1 = __ldg(src + 1);
    const uint32_t wd[8] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z, r1.w};
    #pragma unroll
    for (int q = 0; q < 8; ++q) {
      o[2 * q] = fmaf(w, __uint_as_float(wd[q] << 16), o[2 * q]);
      o[2 * q + 1] = fmaf(w, __uint_as_float(wd[q] & 0xFFFF0000u), o[2 * q + 1]);
    }
  }
  const float inv = 1.f / L;
  #pragma unroll
  for (int k = 0; k < 16; ++k) o[k] *= inv;
  #pragma unroll
  for (int q = 0; q < 4; ++q)
    reinterpret_cast<float4*>(ap)[q] = make_float4(o[4 * q], o[4 * q + 1], o[4 * q + 2], o[4 * q + 3]);
  if (final_out) {
    uint4* f = reinterpret_cast<uint4*>(final_out + off);
    f[0] = make_uint4(bf16x2(o[0], o[1]), bf16x2(o[2], o[3]), bf16x2(o[4], o[5]), bf16x2(o[6], o[7]));
    f[1] = make_uint4(bf16x2(o[8], o[9]), bf16x2(o[10], o[11]), bf16x2(o[12], o[13]),
                      bf16x2(o[14], o[15]));
  }
}

// scalar form (any D, any alignment): one thread per value
template <typename BT>
__global__ void merge_n_scalar_kernel(float* acc_out, const float* acc_lse, const __grid_constant__ MergeN m,
                                      int64_t T, int H, int D, int64_t acc_ls,
                                      __nv_bfloat16* final_out) {
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= T * H * D) return;
  const int64_t row = gid / D;
  const int d = static_cast<int>(gid % D);
  const int h = static_cast<int>(row / T);
  const int64_t t = row % T;
  const int64_t off = (t * H + h) * D + d;
  const float a = acc_lse[h * acc_ls + t];
  float mx = a;
  for (int i = 0; i < m.n; ++i) mx = fmaxf(mx, m.lse[i][h * m.ls[i] + t]);
  float o = 0.f;
  if (mx != -INFINITY) {
    float L = 0.f;
    if (a != -INFINITY) {
      L = __expf(a - mx);
      o = L * acc_out[off];
    }
    for (int i = 0; i < m.n; ++i) {
      const float bi = m.lse[i][h * m.ls[i] + t];
      if (bi == -INFINITY) continue;
      const float w = __expf(bi - mx);
      L += w;
      o = fmaf(w, static_cast<float>(static_cast<const BT*>(m.blk[i])[off]), o);
    }
    o /= L;
    acc_out[off] = o;
  }
  if (final_out) final_out[off] = __float2bfloat16_rn(o);
}

// the lse update, after the values (they read the old lse)
__global__ void merge_n_lse_kernel(float* acc_lse, const __grid_constant__ MergeN m, int64_t T, int H,
                                   int64_t acc_ls) {
  const int64_t gid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (gid >= T * H) return;
  const int h = static_cast<int>(gid / T);
  const int64_t t = gid % T;
  const float a = acc_lse[h * acc_ls + t];
  float mx = a;
  for (int i = 0; i < m.n; ++i) mx = fmaxf(mx, m.lse[i][h * m.ls[i] + t]);
  if (mx == -INFINITY) return;
  float L = (a == -INFINITY) ? 0.f : __expf(a - mx);
  for (int i = 0; i < m.n; ++i) {
    const float bi = m.lse[i][h * m.ls[i] + t];
    if (bi != -INFINITY) L += __expf(bi - mx);
  }
  acc_lse[h * acc_ls + t] = mx + logf(L);
}

template <typename BT>
static int merge_n_t(float* acc_out, float* acc_lse, const MergeN& m, int64_t T, int H, int D,
                     int64_t als, __nv_bfloat16* fin, cudaStream_t s) {
  bool vec = (D % 8 == 0) && (reinterpret_cast<uintptr_t>(acc_out) % 16 == 0) &&
             (!fin || reinterpret_cast<uintptr_t>(fin) % 16 == 0);
  for (int i = 0; i < m.n; ++i) vec = vec && (reinterpret_cast<uintptr_t>(m.blk[i]) % 16 == 0);
  if (vec) {
    const int64_t threads = T * H * (D / 8);
    const unsigned grid = static_cast<unsigned>((threads + 255) / 256);
    bool done = false;
    if constexpr (std::is_same<BT, __nv_bfloat16>::value) {
      done = (D % 16 == 0);
      const unsigned grid16 = static_cast<unsigned>((T * H * (D / 16) + 255) / 256);
      if (done) switch (m.n) {
        case 1: merge_n_bf16_kernel<1><<<grid16, 256, 0, s>>>(acc_out, acc_lse, m, T, H, D, als, fin); break;
        case 2: merge_n_bf16_kernel<2><<<grid16, 256, 0, s>>>(acc_out, acc_lse, m, T, H, D, als, fin); break;
        case 3: merge_n_bf16_kernel<3><<<grid16, 256, 0, s>>>(acc_out, acc_lse, m, T, H, D, als, fin); break;
        case 4: merge_n_bf16_kernel<4><<<grid16, 256, 0, s>>>(acc_out, acc_lse, m, T, H, D, als, fin); break;
        case 5: merge_n_bf16_kernel<5><<<grid16, 256, 0, s>>>(acc_out, acc_lse, m, T, H, D, als, fin); break;
        case 6: merge_n_bf16_kernel<6><<<grid16, 256, 0, s>>>(acc_out, acc_lse, m, T, H, D, als, fin); break;
        case 7: merge_n_bf16_kernel<7><<<grid16, 256, 0, s>>>(acc_out, acc_lse, m, T, H, D, als, fin); break;
        case 8: merge_n_bf16_kernel<8><<<grid16, 256, 0, s>>>(acc_out, acc_lse, m, T, H, D, als, fin); break;
        default: done = false;
      }
    }
    if (!done)
      merge_n_vec8_kernel<BT><<<grid, 256, 0, s>>>(acc_out, acc_lse, m, T, H, D, als, fin);
  } else {
    const int64_t n = T * H * D;
    merge_n_scalar_kernel<BT><<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
        acc_out, acc_lse, m, T, H, D, als, fin);
  }
  merge_n_lse_kernel<<<static_cast<unsigned>((T * H + 255) / 256), 256, 0, s>>>(acc_lse, m, T, H, als);
  return cuda_status(cudaGetLastError(), "merge_n launch");
}

int launch_merge_n(float* acc_out, float* acc_lse, int64_t als, const void* const* blk,
                   int blk_dtype, const float* const* blk_lse, const int64_t* bls, int n,
                   int64_t T, int H, int D, void* fin, cudaStream_t s) {
  if (n < 0 || n > TR_MERGE_MAX) return fail(TR_ERR_CONFIG, "merge_n: 0..16 blocks per call");
  if (T * H * D == 0 || (n == 0 && !fin)) return TR_OK;
  MergeN m{};
  m.n = n;
  for (int i = 0; i < n; ++i) {
    if (!blk[i] || !blk_lse[i]) return fail(TR_ERR_INPUT, "merge_n: null block");
    if (bls[i] < T) return fail(TR_ERR_DIMENSION, "merge_n: lse row stride smaller than T");
    m.blk[i] = blk[i];
    m.lse[i] = blk_lse[i];
    m.ls[i] = bls[i];
  }
  auto* f = static_cast<__nv_bfloat16*>(fin);
  if (blk_dtype == TR_DTYPE_BF16) return merge_n_t<__nv_bfloat16>(acc_out, acc_lse, m, T, H, D, als, f, s);
  if (blk_dtype == TR_DTYPE_F32) return merge_n_t<float>(acc_out, acc_lse, m, T, H, D, als, f, s);
  return fail(TR_ERR_INPUT, "unknown blk dtype");
}

__global__ void fill_kernel(float* p, int64_t n, float v) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

template <typename BT>
static int merge_t(float* acc_out, float* acc_lse, const BT* blk_out, const float* blk_lse,
                   int64_t T, int H, int D, int64_t als, int64_t bls, __nv_bfloat16* fin,
                   cudaStream_t s) {
  const bool vec = (D % 8 == 0) && (reinterpret_cast<uintptr_t>(acc_out) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(blk_out) % 16 == 0) &&
                   (!fin || reinterpret_cast<uintptr_t>(fin) % 16 == 0);
  if (vec) {
    const int64_t threads = T * H * (D / 8);
    merge_vec8_kernel<BT><<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(
        acc_out, acc_lse, blk_out, blk_lse, T, H, D, als, bls, fin);
  } else {
    const int64_t n = T * H * D;
    merge_scalar_kernel<BT><<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(
        acc_out, acc_lse, blk_out, blk_lse, T, H, D, als, bls, fin);
  }
  merge_scalar_lse_kernel<<<static_cast<unsigned>((T * H + 255) / 256), 256, 0, s>>>(
      acc_lse, blk_lse, T, H, als, bls);
  return cuda_status(cudaGetLastError(), "lse_merge launch");
}

int launch_merge(float* acc_out, float* acc_lse, const void* blk_out, int blk_dtype,
                 const float* blk_lse, int64_t T, int H, int D, int64_t als, int64_t bls,
                 void* fin, cudaStream_t s) {
  if (T * H * D == 0) return TR_OK;
  auto* f = static_cast<__nv_bfloat16*>(fin);
  if (blk_dtype == TR_DTYPE_BF16)
    return merge_t(acc_out, acc_lse, static_cast<const __nv_bfloat16*>(blk_out), blk_lse, T, H, D,
                   als, bls, f, s);
  if (blk_dtype == TR_DTYPE_F32)
    return merge_t(acc_out, acc_lse, static_cast<const float*>(blk_out), blk_lse, T, H, D, als,
                   bls, f, s);
  return fail(TR_ERR_INPUT, "unknown blk dtype");
}

int launch_fill(float* p, int64_t n, float v, cudaStream_t s) {
  if (n <= 0) return TR_OK;
  fill_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(p, n, v);
  return cuda_status(cudaGetLastError(), "fill");
}

int launch_partial_init(float* acc_out, float* acc_lse, int64_t T, int H, int D, cudaStream_t s) {
  if (T * H * D == 0) return TR_OK;
  cudaError_t e = cudaMemsetAsync(acc_out, 0, sizeof(float) * T * H * D, s);
  if (e != cudaSuccess) return cuda_status(e, "partial_init memset");
  const int64_t n = T * H;
  fill_kernel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, s>>>(acc_lse, n, -INFINITY);
  return cuda_status(cudaGetLastError(), "partial_init fill");
}

}  // namespace tr
