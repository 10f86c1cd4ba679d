// Latency of the in-group chain of trsv_group (warp 0, g rows) in isolation.
#include <cstdio>
#include <cuda_runtime.h>
template <int GCW>
__global__ void k(int g, int reps, long long* out, double* sink) {
  __shared__ double part[32][GCW], ys[32][GCW], lg[32][33];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 32 * 33; i += blockDim.x) lg[i / 33][i % 33] = 1e-3 * (i % 7);
  for (int i = tid; i < 32 * GCW; i += blockDim.x) part[i / GCW][i % GCW] = 1.0 + i;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (warp == 0) {
      double pr[GCW];
      const bool mine = lane < g;
#pragma unroll
      for (int c = 0; c < GCW; ++c) pr[c] = mine ? part[lane][c] : 0.0;
      const double d = 1.0;
      for (int j = 0; j < g; ++j) {
        const double l = (lane > j && mine) ? lg[lane][j] : 0.0;
#pragma unroll
        for (int c = 0; c < GCW; ++c) {
          const double yj = __shfl_sync(0xffffffffu, pr[c] * d, j);
          if (lane == j) ys[j][c] = yj;
          pr[c] = fma(-l, yj, pr[c]);
        }
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) out[0] = (t1 - t0) / reps;
  if (tid < 32) sink[tid] = ys[tid][0];
}
int main() {
  long long* o; double* s; cudaMalloc(&o, 8); cudaMalloc(&s, 256 * 8);
  for (int g : {8, 16, 32}) {
    long long h;
    k<1><<<1, 512>>>(g, 1000, o, s); cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("GCW=1 g=%d: %lld cycles per chain (+barrier)\n", g, h);
    k<4><<<1, 512>>>(g, 1000, o, s); cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost);
    printf("GCW=4 g=%d: %lld cycles per chain (+barrier)\n", g, h);
  }
  return 0;
}
