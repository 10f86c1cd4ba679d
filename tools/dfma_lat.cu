// DFMA latency / ILP probe: one warp per SMSP (4 warps/CTA, 1 CTA/SM) runs
// C independent dependent-chains; reports cycles per DFMA per warp.
#include <cstdio>
#include <cuda_runtime.h>
template <int C>
__global__ void k(double* out, int iters, long long* cyc) {
  double a[C];
#pragma unroll
  for (int c = 0; c < C; ++c) a[c] = threadIdx.x * 1e-3 + c;
  const double m = 1.0000001, b = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < C; ++c) a[c] = fma(a[c], m, b);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) s += a[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
template <int C> void run(int warps) {
  double* o; long long* c; cudaMalloc(&o, 1 << 20); cudaMalloc(&c, 8);
  int iters = 4096;
  k<C><<<1, 32 * warps>>>(o, iters, c);
  k<C><<<1, 32 * warps>>>(o, iters, c);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("chains=%2d warps/CTA=%2d: %.2f cycles per chain-step (per-warp DFMA issue interval %.2f)\n", C, warps,
         (double)h / iters, (double)h / iters / C);
  cudaFree(o); cudaFree(c);
}
int main() {
  run<1>(1); run<2>(1); run<4>(1); run<8>(1); run<16>(1);
  run<1>(4); run<4>(4); run<8>(4); run<4>(8); run<4>(16); run<8>(16);
  return 0;
}
