// Microbenchmark (diagnostic, not product): per-SM-sub-partition issue rate of
// MUFU.EX2 and of the product kernel's exp2 -> bf16 P inner loop, with W warps
// per sub-partition, timed with clock64 inside one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_probe scripts/mufu_probe.cu && ./mufu_probe
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

#include "../paper_2412_20501_b200/csrc/tr_ptx.cuh"

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// pure MUFU: 16 independent chains
__global__ void k_mufu(float* out, int iters, long long* cyc) {
  float a[16];
  for (int i = 0; i < 16; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    #pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = ex2(a[i]) - 1.0f;
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// the product kernel's per-pair work: FFMA2 scale/shift, 2 MUFU, FADD2 sum, F2FP pack
__global__ void k_softmax_like(uint32_t* out, int iters, long long* cyc) {
  float s[128];
  for (int i = 0; i < 128; ++i) s[i] = 0.01f * ((threadIdx.x * 7 + i * 13) % 97) - 0.5f;
  float2 sum0 = make_float2(0, 0), sum1 = make_float2(0, 0);
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float c = 1.4427f, m = -0.25f * it;
    #pragma unroll
    for (int i = 0; i < 64; ++i) {
      float a = fmaf(s[2 * i], c, m), b = fmaf(s[2 * i + 1], c, m);
      a = ex2(a);
      b = ex2(b);
      if (i & 1) { sum1.x += a; sum1.y += b; } else { sum0.x += a; sum0.y += b; }
      __nv_bfloat162 p = __floats2bfloat162_rn(a, b);
      acc ^= *reinterpret_cast<uint32_t*>(&p);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + __float_as_uint(sum0.x + sum0.y + sum1.x + sum1.y);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}


// the product kernel's emit_p loop (attn_common.cuh) minus the TMEM store:
// FFMA2 scale/shift, MUFU pairs with one pair in POLY on the FMA pipe,
// FADD2 row sums, cvt.rn.bf16x2
template <int POLY_MOD>
__global__ void k_emit_p(uint32_t* out, int iters, long long* cyc) {
  uint32_t s[128];
  for (int i = 0; i < 128; ++i) s[i] = __float_as_uint(0.01f * ((threadIdx.x * 7 + i * 13) % 97) - 0.5f);
  uint64_t lsum2[2] = {0ull, 0ull};
  uint32_t acc = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const uint64_t c2 = tr::f2pack(1.4427f, 1.4427f), nmc2 = tr::f2pack(-0.25f * it, -0.25f * it);
    #pragma unroll
    for (int i = 0; i < 64; ++i) {
      const uint64_t x2 = tr::ffma2(tr::f2pack(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), c2, nmc2);
      float a, b;
      tr::f2unpack(x2, a, b);
      uint64_t p2;
      if (POLY_MOD > 0 && (i % (POLY_MOD > 0 ? POLY_MOD : 1)) == POLY_MOD - 1)
        p2 = tr::exp2_poly2(tr::f2pack(fmaxf(a, -126.f), fmaxf(b, -126.f)));
      else
        p2 = tr::f2pack(tr::ex2_approx(a), tr::ex2_approx(b));
      lsum2[i & 1] = tr::fadd2(lsum2[i & 1], p2);
      float pa, pb;
      tr::f2unpack(p2, pa, pb);
      acc ^= tr::pack_bf16x2(pa, pb);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + static_cast<uint32_t>(lsum2[0] ^ lsum2[1]);
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int POLY_MOD>
void run_emit(int sms, uint32_t* ou, long long* cyc, int iters) {
  long long h[1];
  for (int wps = 1; wps <= 2; ++wps) {
    const int threads = 128 * wps;
    k_emit_p<POLY_MOD><<<sms, threads>>>(ou, iters, cyc);
    cudaDeviceSynchronize();
    k_emit_p<POLY_MOD><<<sms, threads>>>(ou, iters, cyc);
    cudaMemcpy(h, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
    printf("emit_p POLY_MOD=%d %d warp(s)/SMSP: %.0f cycles per 128-element row per warp (MUFU bound %d)\n",
           POLY_MOD, wps, double(h[0]) / iters / wps,
           POLY_MOD > 0 ? 8 * 2 * (64 - 64 / POLY_MOD) : 1024);
  }
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* of;
  uint32_t* ou;
  long long* cyc;
  cudaMalloc(&of, sizeof(float) * sms * 1024);
  cudaMalloc(&ou, sizeof(uint32_t) * sms * 1024);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  long long h[1024];
  const int iters = 2000;
  run_emit<6>(sms, ou, cyc, 200);
  run_emit<0>(sms, ou, cyc, 200);
  run_emit<4>(sms, ou, cyc, 200);
  for (int wps = 1; wps <= 2; wps *= 2) {
    const int threads = 128 * wps;   // wps warps per sub-partition
    k_mufu<<<sms, threads>>>(of, iters, cyc);
    cudaDeviceSynchronize();
    k_mufu<<<sms, threads>>>(of, iters, cyc);
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double ops = double(iters) * 16 * threads;   // ex2 per SM
    printf("MUFU.EX2  %d warp(s)/SMSP: %.2f ex2/clk/SM  (%.1f cycles per warp-instr per SMSP)\n", wps,
           ops / h[0], 4.0 * 32.0 * h[0] / ops);
    k_softmax_like<<<sms, threads>>>(ou, iters / 10, cyc);
    cudaDeviceSynchronize();
    k_softmax_like<<<sms, threads>>>(ou, iters / 10, cyc);
    cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double el = double(iters / 10) * 128 * threads;
    printf("exp->P loop %d warp(s)/SMSP: %.2f elements/clk/SM, %.0f cycles per 128-element row per warp\n",
           wps, el / h[0], double(h[0]) / (iters / 10) / wps);
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
