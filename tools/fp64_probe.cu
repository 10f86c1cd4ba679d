// Micro-probe: FP64 vector (DFMA) vs FP64 tensor (DMMA mma.sync) throughput on B200.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_kernel(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double b = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a0 = fma(a0, b, c); a1 = fma(a1, b, c); a2 = fma(a2, b, c); a3 = fma(a3, b, c);
      a4 = fma(a4, b, c); a5 = fma(a5, b, c); a6 = fma(a6, b, c); a7 = fma(a7, b, c);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
}

__global__ void dmma884_kernel(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double d[8][2];
  for (int k = 0; k < 8; ++k) { d[k][0] = 0; d[k][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(d[k][0]), "+d"(d[k][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void dmma16816_kernel(double* out, int iters) {
  double a[8], b[4];
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x * 1e-3 + k;
  for (int k = 0; k < 4; ++k) b[k] = 1.0 + k * 1e-3;
  double d[4][4];
  for (int k = 0; k < 4; ++k) for (int j = 0; j < 4; ++j) d[k][j] = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, {%12,%13,%14,%15}, {%0,%1,%2,%3};"
                   : "+d"(d[k][0]), "+d"(d[k][1]), "+d"(d[k][2]), "+d"(d[k][3])
                   : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                     "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
  }
  double s = 0;
  for (int k = 0; k < 4; ++k) for (int j = 0; j < 4; ++j) s += d[k][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// DFMA fed by broadcast LDS (uniform address) — models coefficient delivery.
__global__ void lds_bcast_kernel(double* out, int iters) {
  __shared__ double coef[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) coef[i] = 1e-3 * i;
  __syncthreads();
  double v0 = threadIdx.x, v1 = v0 + 1, acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  int base = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double c = coef[(base + k) & 1023];
      acc0 = fma(c, v0, acc0); acc1 = fma(c, v1, acc1);
    }
    base += 8;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

// LDS.128 broadcast of 2 coefficients, each used by C=2 columns
__global__ void lds128_bcast_kernel(double* out, int iters) {
  __shared__ double2 coef[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) coef[i] = make_double2(1e-3 * i, 2e-3 * i);
  __syncthreads();
  double v0 = threadIdx.x, v1 = v0 + 1, acc0 = 0, acc1 = 0, acc2 = 0, acc3 = 0;
  int base = 0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      double2 c = coef[(base + k) & 511];
      acc0 = fma(c.x, v0, acc0); acc1 = fma(c.x, v1, acc1);
      acc2 = fma(c.y, v0, acc2); acc3 = fma(c.y, v1, acc3);
    }
    base += 4;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
}

int main() {
  int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out; cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d MHz\n", sms, clk / 1000);
  struct { const char* name; int kind; } ks[] = {{"dfma", 0}, {"dmma884", 1}, {"dmma16816", 2}, {"lds64_bcast+2dfma", 3}, {"lds128_bcast+4dfma", 4}};
  for (auto& k : ks) {
    for (int blocks_per_sm : {4, 8}) {
      int threads = 256, iters = 4096;
      dim3 grid(sms * blocks_per_sm);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (k.kind == 0) dfma_kernel<<<grid, threads>>>(out, iters);
        if (k.kind == 1) dmma884_kernel<<<grid, threads>>>(out, iters);
        if (k.kind == 2) dmma16816_kernel<<<grid, threads>>>(out, iters);
        if (k.kind == 3) lds_bcast_kernel<<<grid, threads>>>(out, iters);
        if (k.kind == 4) lds128_bcast_kernel<<<grid, threads>>>(out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double flops = 0;
        double nthr = (double)grid.x * threads;
        if (k.kind == 0) flops = nthr * iters * 64 * 2;
        if (k.kind == 1) flops = nthr / 32 * iters * 8 * (8 * 8 * 4) * 2;
        if (k.kind == 2) flops = nthr / 32 * iters * 4 * (16 * 8 * 16) * 2;
        if (k.kind == 3) flops = nthr * iters * 8 * 2 * 2;
        if (k.kind == 4) flops = nthr * iters * 4 * 4 * 2;
        cudaError_t err = cudaGetLastError();
        if (rep == 1) printf("%-20s blocks/SM %d: %.3f ms  %.2f TFLOP/s %s\n", k.name, blocks_per_sm, ms, flops / ms / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
      }
    }
  }
  return 0;
}
