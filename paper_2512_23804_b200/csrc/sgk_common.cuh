// Shared helpers for the sm_100a kernels of libsgkkt_b200.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <atomic>
#include <string>

#include "sgkkt_b200.h"

namespace sgk {

// Set by every entry point that fails; read through sgk_last_error().
void set_error(const std::string& msg);
// Launch bookkeeping for bench.py's "gpu_launches" claim.
void count_launch(int64_t n = 1);
// SM count of the current device (cached).
int sm_count();

inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(what) + ": " + cudaGetErrorString(e));
    return SGK_ECUDA;
  }
  count_launch();
  return SGK_OK;
}

// Acquire/release flag accesses for the sync-free triangular solves.
__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

}  // namespace sgk

#define SGK_REQUIRE(cond, msg)        \
  do {                                \
    if (!(cond)) {                    \
      ::sgk::set_error(msg);          \
      return SGK_EINVAL;              \
    }                                 \
  } while (0)
