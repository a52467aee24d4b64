// Device-side sequence flags for the copy-engine (CUDA IPC) transport of the
// TokenRing runner.  A sender pushes a block into the peer's mapped receive
// buffer with cudaMemcpyAsync (copy engines, no SMs), then bumps the peer's
// flag with a system-scope release store; the consumer's stream runs a
// one-thread acquire-spin until the flag reaches the expected sequence
// number.  Flags only grow, so they never need resetting between steps.
#include <cuda_runtime.h>

#include "tr_internal.h"

namespace tr {

__global__ void flag_set_kernel(unsigned long long* flag, unsigned long long value) {
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

__global__ void flag_wait_kernel(const unsigned long long* flag, unsigned long long value,
                                 unsigned long long timeout_ns) {
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long x;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(flag) : "memory");
    if (x >= value) break;
    __nanosleep(256);
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) __trap();   // a lost message must not wedge the GPU
  }
}

int launch_flag_set(unsigned long long* flag, unsigned long long value, cudaStream_t s) {
  flag_set_kernel<<<1, 1, 0, s>>>(flag, value);
  return cuda_status(cudaGetLastError(), "flag_set");
}

int launch_flag_wait(const unsigned long long* flag, unsigned long long value, cudaStream_t s) {
  flag_wait_kernel<<<1, 1, 0, s>>>(flag, value, 30ull * 1000000000ull);
  return cuda_status(cudaGetLastError(), "flag_wait");
}

}  // namespace tr
