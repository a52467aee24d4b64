// Device-side sequence flags for the copy-engine (CUDA IPC) transport of the
// TokenRing runner.  A sender pushes a block into the peer's mapped receive
// buffer with cudaMemcpyAsync (copy engines, no SMs), then bumps the peer's
// flag with a system-scope release store; the consumer's stream runs a
// one-thread acquire-spin until the flag reaches the expected sequence
// number.  Flags only grow, so they never need resetting between steps.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "tr_internal.h"

namespace tr {

// `epoch` (optional, a device int64 of the caller): the value is relative,
// *epoch + (signed) value, read when the kernel runs -- so a captured CUDA
// graph replays with the epoch its previous replay advanced (epoch_add_kernel)
__device__ __forceinline__ unsigned long long flag_value(unsigned long long value,
                                                         const long long* epoch) {
  return epoch ? static_cast<unsigned long long>(*epoch + static_cast<long long>(value)) : value;
}

__global__ void epoch_add_kernel(long long* epoch, long long delta) { *epoch += delta; }

__global__ void flag_set_kernel(unsigned long long* flag, unsigned long long value,
                                const long long* epoch) {
  value = flag_value(value, epoch);
  asm volatile("fence.acq_rel.sys;" ::: "memory");
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

// A wait that times out does not trap (that would kill the CUDA context and
// every peer's view of it): it records what it waited for in a host-mapped
// status block and returns, and the host turns the record into a
// ScheduleError (tr_poll_error) -- the reference's "message never delivered"
// failure (engine.py:532-537).  The first timeout of the process wins.
struct FlagError {
  unsigned long long code;       // 0 = none, 1 = flag wait timed out
  unsigned long long flag;       // address waited on
  unsigned long long expected;
  unsigned long long observed;
};

static FlagError* g_err_host = nullptr;   // pinned, mapped into every device (UVA)
static std::once_flag g_err_once;
static cudaError_t g_err_alloc = cudaSuccess;

static FlagError* error_block() {
  std::call_once(g_err_once, [] {
    void* p = nullptr;
    g_err_alloc = cudaHostAlloc(&p, sizeof(FlagError), cudaHostAllocMapped | cudaHostAllocPortable);
    if (g_err_alloc == cudaSuccess) {
      memset(p, 0, sizeof(FlagError));
      g_err_host = static_cast<FlagError*>(p);
    }
  });
  return g_err_host;
}

__global__ void flag_wait_kernel(const unsigned long long* flag, unsigned long long value,
                                 unsigned long long timeout_ns, FlagError* err,
                                 const long long* epoch) {
  value = flag_value(value, epoch);
  unsigned long long t0;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long x;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(x) : "l"(flag) : "memory");
    if (x >= value) break;
    __nanosleep(256);
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) {
      if (atomicCAS_system(&err->code, 0ull, 1ull) == 0ull) {
        err->flag = reinterpret_cast<unsigned long long>(flag);
        err->expected = value;
        err->observed = x;
        __threadfence_system();
      }
      return;
    }
  }
}

int launch_flag_set(unsigned long long* flag, unsigned long long value, cudaStream_t s,
                    const long long* epoch) {
  return cuda_status(launch_kernel(flag_set_kernel, dim3(1), dim3(1), 0, s, launch_overlap(), flag,
                                   value, epoch),
                     "flag_set");
}

static unsigned long long g_timeout_ns = 30ull * 1000000000ull;

int launch_flag_wait(const unsigned long long* flag, unsigned long long value, cudaStream_t s,
                     const long long* epoch) {
  FlagError* err = error_block();
  if (!err) return cuda_status(g_err_alloc, "cudaHostAlloc(flag error block)");
  // (overlap: the wait may start while the previous kernel still runs; its
  // dependents start only once it has returned -- it never triggers early)
  return cuda_status(launch_kernel(flag_wait_kernel, dim3(1), dim3(1), 0, s, launch_overlap(),
                                   flag, value, g_timeout_ns, err, epoch),
                     "flag_wait");
}

int launch_epoch_add(long long* epoch, long long delta, cudaStream_t s) {
  epoch_add_kernel<<<1, 1, 0, s>>>(epoch, delta);
  return cuda_status(cudaGetLastError(), "epoch_add");
}

int poll_flag_error() {
  FlagError* err = error_block();
  if (!err) return cuda_status(g_err_alloc, "cudaHostAlloc(flag error block)");
  volatile FlagError* e = err;
  if (e->code == 0) return TR_OK;
  char buf[256];
  snprintf(buf, sizeof(buf),
           "message not delivered: a flag wait timed out after %.1f s (flag %#llx expected >= %llu, "
           "saw %llu); the device results of that forward are invalid",
           g_timeout_ns * 1e-9, e->flag, e->expected, e->observed);
  return fail(TR_ERR_TIMEOUT, buf);
}

void clear_flag_error() {
  if (FlagError* err = error_block()) memset(err, 0, sizeof(FlagError));
}

void set_flag_timeout_ns(unsigned long long ns) { g_timeout_ns = ns; }

}  // namespace tr
