// LSU cost model probe (one 512-thread CTA per SM): SM-wide cycles per warp
// instruction for the shared/global access shapes the matvec kernels use.
#include <cstdio>
#include <cuda_runtime.h>

enum Mode { LDS32, LDS64, LDS64_BCAST, LDS64_PERM, LDS64_4ADDR, LDS128, LDS128_BCAST, STS64, STS128, LDG64, LDG128, LDG64_L2, LDS128_PERM, LDS128_VARY, LDS64_VARY };

template <int MODE>
__global__ void __launch_bounds__(512, 1) probe(double* out, const double* g, int iters, long long* cyc) {
  extern __shared__ __align__(16) unsigned char sm[];
  double* sd = reinterpret_cast<double*>(sm);
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) sd[i] = 1e-3 * i;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  unsigned ia = 0;
  // per-lane byte offset inside a 256/512-byte warp tile
  int off;
  if (MODE == LDS64_BCAST || MODE == LDS128_BCAST) off = 0;
  else if (MODE == LDS64_PERM) off = ((lane * 5 + 3) & 15) * 8 + (lane >> 4) * 128 + 0;  // conflict-free permutation per half-warp
  else if (MODE == LDS64_4ADDR) off = (lane & 3) * 8;
  else if (MODE == LDS128_PERM) off = ((lane * 13 + 5) & 31) * 16 + ((lane * 7) & 3) * 1024;  // scattered 16-byte chunks
  else if (MODE == LDS128 || MODE == STS128 || MODE == LDG128 || MODE == LDS128_VARY) off = lane * 16;
  else if (MODE == LDS32) off = lane * 4;
  else off = lane * 8;
  const unsigned char* base = sm + warp * 4096 + off;
  const unsigned char* gb = reinterpret_cast<const unsigned char*>(g) + (size_t)blockIdx.x * 65536 + warp * 4096 + off;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int o = k * 512;
      if (MODE == LDS32) ia += *reinterpret_cast<const volatile unsigned*>(base + o);
      else if (MODE == LDS64 || MODE == LDS64_BCAST || MODE == LDS64_PERM || MODE == LDS64_4ADDR || MODE == LDS64_VARY) {
        const int vo = MODE == LDS64_VARY ? ((i * 1032) & 0x3ff8) : 0;
        const double x = *reinterpret_cast<const volatile double*>(base + o + vo);
        if (k & 1) acc1 += x; else acc0 += x;
      } else if (MODE == LDS128 || MODE == LDS128_BCAST || MODE == LDS128_PERM || MODE == LDS128_VARY) {
        double2 x;
        const int vo = MODE == LDS128_VARY ? ((i * 1040) & 0x3ff0) : 0;
        asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(x.x), "=d"(x.y) : "r"((unsigned)__cvta_generic_to_shared(base + o + vo)));
        if (k & 1) { acc1 += x.x; acc3 += x.y; } else { acc0 += x.x; acc2 += x.y; }
      } else if (MODE == STS64) {
        *reinterpret_cast<volatile double*>(const_cast<unsigned char*>(base + o)) = acc0;
      } else if (MODE == STS128) {
        asm volatile("st.shared.v2.f64 [%0], {%1,%2};" ::"r"((unsigned)__cvta_generic_to_shared(base + o)), "d"(acc0), "d"(acc1));
      } else if (MODE == LDG64) {
        double x;
        asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(x) : "l"(gb + o));
        if (k & 1) acc1 += x; else acc0 += x;
      } else if (MODE == LDG128) {
        double2 x;
        asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(x.x), "=d"(x.y) : "l"(gb + o));
        if (k & 1) { acc1 += x.x; acc3 += x.y; } else { acc0 += x.x; acc2 += x.y; }
      } else if (MODE == LDG64_L2) {
        double x;  // stream 4 MB per CTA: misses L1, hits L2
        asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(x) : "l"(gb + o + (size_t)((i * 8 + k) & 63) * 65536 * 148));
        if (k & 1) acc1 += x; else acc0 += x;
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3 + ia;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int MODE>
void run(const char* name, double* out, const double* g, long long* cyc, int sms) {
  const int iters = 4096;
  cudaFuncSetAttribute(probe<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  probe<MODE><<<sms, 512, 131072>>>(out, g, iters, cyc);
  cudaEventRecord(e0);
  probe<MODE><<<sms, 512, 131072>>>(out, g, iters, cyc);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  long long h = 0;
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  const double per = (double)h / (iters * 8.0 * 16);  // 16 warps issue each instruction
  printf("%-14s %6.2f SM-cycles per warp instruction (clock64)  kernel %.1f us = %.2f clk/instr incl. setup (%s)\n", name, per, ms * 1e3,
         ms * 1e-3 * 1.965e9 / (iters * 8.0 * 16), cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *out, *g;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * 148 * 512);
  cudaMalloc(&g, (size_t)65536 * 148 * 65);
  cudaMemset(g, 0, (size_t)65536 * 148 * 65);
  cudaMalloc(&cyc, 8);
  run<LDS32>("LDS.32", out, g, cyc, sms);
  run<LDS64>("LDS.64", out, g, cyc, sms);
  run<LDS64_BCAST>("LDS.64 bcast", out, g, cyc, sms);
  run<LDS64_4ADDR>("LDS.64 4addr", out, g, cyc, sms);
  run<LDS64_PERM>("LDS.64 perm", out, g, cyc, sms);
  run<LDS128>("LDS.128", out, g, cyc, sms);
  run<LDS128_BCAST>("LDS.128 bcast", out, g, cyc, sms);
  run<STS64>("STS.64", out, g, cyc, sms);
  run<STS128>("STS.128", out, g, cyc, sms);
  run<LDG64>("LDG.64 L1", out, g, cyc, sms);
  run<LDG128>("LDG.128 L1", out, g, cyc, sms);
  run<LDG64_L2>("LDG.64 L2", out, g, cyc, sms);
  run<LDS128_PERM>("LDS.128 perm", out, g, cyc, sms);
  run<LDS128_VARY>("LDS.128 vary", out, g, cyc, sms);
  run<LDS64_VARY>("LDS.64 vary", out, g, cyc, sms);
  return 0;
}
