// LDS broadcast vs DFMA balance probe: each LDS.64 (uniform address) feeds C DFMAs
// into C independent accumulators.
#include <cstdio>
#include <cuda_runtime.h>

template <int C, int W>  // W: 1 = LDS.64, 2 = LDS.128
__global__ void probe(double* out, int iters, int uniform) {
  __shared__ double coef[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) coef[i] = 1e-3 * i;
  __syncthreads();
  double v[C], acc[C][W];
#pragma unroll
  for (int c = 0; c < C; ++c) { v[c] = threadIdx.x + c; for (int w = 0; w < W; ++w) acc[c][w] = 0; }
  int base = uniform ? 0 : (threadIdx.x & 31) * 18;  // per-lane: 11 distinct-ish words pattern
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int idx = ((base + 2 * k + 16 * (i & 15)) & 1023) * 2;
      if (W == 1) {
        double cc = coef[idx];
#pragma unroll
        for (int c = 0; c < C; ++c) acc[c][0] = fma(cc, v[c], acc[c][0]);
      } else {
        double2 cc = *reinterpret_cast<const double2*>(&coef[idx]);
#pragma unroll
        for (int c = 0; c < C; ++c) { acc[c][0] = fma(cc.x, v[c], acc[c][0]); acc[c][1] = fma(cc.y, v[c], acc[c][1]); }
      }
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) for (int w = 0; w < W; ++w) s += acc[c][w];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int C, int W>
void run(const char* name, double* out, int sms, int uniform) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 2048, threads = 256, bps = 8;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    probe<C, W><<<sms * bps, threads>>>(out, iters, uniform);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double nthr = (double)sms * bps * threads;
    double dfma = nthr * iters * 8 * C * W;
    double lds = nthr / 32 * iters * 8;
    if (rep) printf("%-8s C=%d W=%d uniform=%d: %.3f ms  %.1f TFLOP/s  lds/clk/SM=%.3f  dfma-warp/clk/SM=%.3f\n", name, C, W, uniform, ms,
                    2 * dfma / ms / 1e9, lds / (ms * 1e-3) / sms / 1.965e9, dfma / 32 / (ms * 1e-3) / sms / 1.965e9);
  }
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
  for (int u = 1; u >= 0; --u) {
    run<1, 1>("lds64", out, sms, u); run<2, 1>("lds64", out, sms, u); run<4, 1>("lds64", out, sms, u); run<8, 1>("lds64", out, sms, u);
    run<1, 2>("lds128", out, sms, u); run<2, 2>("lds128", out, sms, u); run<4, 2>("lds128", out, sms, u);
  }
  return 0;
}
