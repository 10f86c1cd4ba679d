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
__device__ __forceinline__ int ld_relaxed(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_relaxed(int32_t* p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct ViewSet {
  sgk_view v[SGK_MAX_IO];
};
struct ScalarSet {
  double s[SGK_MAX_IO];
};

__device__ __forceinline__ const sgk_view& pick(const ViewSet& vs, int s) {
  // constant-index selection keeps the views in the parameter bank (a
  // dynamic index would spill the whole struct to local memory)
  switch (s) {
    case 0: return vs.v[0];
    case 1: return vs.v[1];
    case 2: return vs.v[2];
    default: return vs.v[3];
  }
}
__device__ __forceinline__ double pick_s(const ScalarSet& ss, int s) {
  switch (s) {
    case 0: return ss.s[0];
    case 1: return ss.s[1];
    case 2: return ss.s[2];
    default: return ss.s[3];
  }
}

}  // namespace sgk

#define SGK_REQUIRE(cond, msg)        \
  do {                                \
    if (!(cond)) {                    \
      ::sgk::set_error(msg);          \
      return SGK_EINVAL;              \
    }                                 \
  } while (0)
