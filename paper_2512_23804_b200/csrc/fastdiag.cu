// Depth-free lead solves by fast diagonalisation.
//
// On a tensor grid with a constant-coefficient lead the reference's sparse
// LU (linalg.py:103-120) factors a Kronecker sum:
//   A = K1 (x) M1 + M1 (x) K1,   M = M1 (x) M1     (node p = iy*n + ix),
// and with the generalised eigenpairs K1 S = M1 S diag(mu), S^T M1 S = I:
//   (S (x) S)^T A (S (x) S) = diag(mu_a + mu_b),  (S (x) S)^T M (S (x) S) = I.
// So A^-1 = T diag(1/lam) T^T and the hGSoc block
//   P~ = [M 0 -A; 0 beta M M; -A M 0]   (preconditioners.py:437-448)
// becomes one 3x3 system per mode:  P~^-1 = T' B(lam)^-1 T'^T with
//   B^-1 = d [[1, lam, -beta lam], [lam, lam^2, 1], [-beta lam, 1, -beta]],
//   d = 1 / (1 + beta lam^2).
//
// A solve is three hand-written sm_100a kernels, all fp64 on the tensor
// cores (mma.sync m8n8k4 f64 — tcgen05 has no fp64 kind) with S (n x n,
// zero-padded to np x np, np = n rounded up to 8) read through L1/L2:
//   fd_line<false>  pass 1:  T[s][iy][b][k] = sum_ix S[ix,b] X_s[iy*n+ix][k]
//   fd_mid          pass 2 + modal + pass 3 fused per (b, column chunk):
//                   Z_s = S^T T[s][:, b, :],  modal solve across the
//                   segments in registers,  T[s][:, b, :] = S Z_s
//                   (the transformed block never goes back to HBM)
//   fd_line<true>   pass 4:  X_s[iy*n+ix][k] = sum_b S[ix,b] T[s][iy][b][k]
// Each CTA stages its right-hand slab (np rows x chunk columns) in shared
// memory with a bank-conflict-free pitch; warps own row tiles of the output,
// lanes hold the m8n8k4 fragments.  No dependency chain: 24 n^3 flops per
// right-hand-side column (x segments/3) instead of the factor's level depth.
#include "sgk_common.cuh"

namespace sgk {

// D += A(8x4) * B(4x8), fp64 tensor cores.  Fragments (PTX m8n8k4 .f64):
//   a = A[lane/4][lane%4], b = B[lane%4][lane/4],
//   d[i] = D[lane/4][2*(lane%4)+i]
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

constexpr int FD_NC = 32;   // slab columns of a line-pass CTA (4 column tiles)
constexpr int FD_NCM = 16;  // columns per segment of a mid-pass CTA (2 column tiles)
__host__ __device__ constexpr int fd_pitch(int cols) { return cols + 4; }  // == 4 mod 16 doubles: conflict-free

// acc[rt][ct] += Amat(row tile rows) * slab(ct) over k in [0, np); Amat is
// S (TRANS=false: A[r][k] = S[r*np+k]) or S^T (TRANS=true: A[r][k] = S[k*np+r]).
// Row tiles of warp w: w, w+8, ... (RT of them).
template <int RT, int CT, bool TRANS>
__device__ __forceinline__ void fd_gemm(const double* __restrict__ S, int np, const double* __restrict__ slab,
                                        int pitch, int warp, int lane, double (&acc)[RT][CT][2]) {
  const int ar = lane >> 2, ak = lane & 3;
#pragma unroll 2
  for (int k0 = 0; k0 < np; k0 += 4) {
    double a[RT], b[CT];
#pragma unroll
    for (int i = 0; i < RT; ++i) {
      const int r = (warp + 8 * i) * 8 + ar;
      a[i] = r < np ? (TRANS ? __ldg(S + (int64_t)(k0 + ak) * np + r) : __ldg(S + (int64_t)r * np + k0 + ak)) : 0.0;
    }
#pragma unroll
    for (int j = 0; j < CT; ++j) b[j] = slab[(k0 + ak) * pitch + j * 8 + ar];
#pragma unroll
    for (int i = 0; i < RT; ++i)
#pragma unroll
      for (int j = 0; j < CT; ++j) dmma(acc[i][j], a[i], b[j]);
  }
}

// Passes 1 (BACK=false: slab = X_s rows of grid line iy, output T rows b,
// A = S^T) and 4 (BACK=true: slab = T rows b, A = S, output X_s rows).
// grid.x = n_seg * n lines, grid.y = column chunks of FD_NC.
template <int RT, bool BACK>
__global__ void __launch_bounds__(256) fd_line(sgk_fastdiag fd, sgk_segview xv, double* __restrict__ T, int width,
                                               int wpad) {
  constexpr int CT = FD_NC / 8;
  constexpr int P = fd_pitch(FD_NC);
  extern __shared__ __align__(16) double slab[];
  const int n = fd.n, np = fd.np;
  const int line = blockIdx.x;
  const int seg = line / n, iy = line - seg * n;
  const int c0 = blockIdx.y * FD_NC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* xs = seg == 0 ? xv.ptr[0] : (seg == 1 ? xv.ptr[1] : xv.ptr[2]);
  double* tl = T + ((int64_t)seg * n + iy) * n * wpad;  // [b][k] block of this line
  // stage the slab: np rows x FD_NC columns (zero beyond n rows / width columns)
  for (int i = tid; i < np * FD_NC; i += blockDim.x) {
    const int r = i / FD_NC, c = i - r * FD_NC;
    double v = 0.0;
    if (r < n && c0 + c < width)
      v = BACK ? __ldcg(tl + (int64_t)r * wpad + c0 + c) : xs[((int64_t)iy * n + r) * xv.ld + xv.col0 + c0 + c];
    slab[r * P + c] = v;
  }
  __syncthreads();
  double acc[RT][CT][2];
#pragma unroll
  for (int i = 0; i < RT; ++i)
#pragma unroll
    for (int j = 0; j < CT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  fd_gemm<RT, CT, !BACK>(fd.s, np, slab, P, warp, lane, acc);
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int r = (warp + 8 * i) * 8 + (lane >> 2);
    if (r >= n) continue;
#pragma unroll
    for (int j = 0; j < CT; ++j) {
      const int c = c0 + j * 8 + 2 * (lane & 3);
      if (BACK) {
        double* dst = xs + ((int64_t)iy * n + r) * xv.ld + xv.col0 + c;
        if (c < width) dst[0] = acc[i][j][0];
        if (c + 1 < width) dst[1] = acc[i][j][1];
      } else {
        // T rows are padded to wpad (a multiple of FD_NC): always in bounds
        __stcg(reinterpret_cast<double2*>(tl + (int64_t)r * wpad + c), make_double2(acc[i][j][0], acc[i][j][1]));
      }
    }
  }
}

// Pass 2 + modal + pass 3 for one mode column b and FD_NCM columns of every
// segment: slab[iy][s*FD_NCM + c] = T[s][iy][b][c0 + c].
template <int RT, int NSEG>
__global__ void __launch_bounds__(256) fd_mid(sgk_fastdiag fd, double* __restrict__ T, int width, int wpad) {
  constexpr int CPS = FD_NCM / 8;  // column tiles per segment
  constexpr int CT = NSEG * CPS;
  constexpr int W = NSEG * FD_NCM;
  constexpr int P = fd_pitch(W);
  extern __shared__ __align__(16) double slab[];
  const int n = fd.n, np = fd.np;
  const int b = blockIdx.x;
  const int c0 = blockIdx.y * FD_NCM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto tptr = [&](int s, int iy, int c) { return T + (((int64_t)s * n + iy) * n + b) * wpad + c0 + c; };
  for (int i = tid; i < np * W; i += blockDim.x) {
    const int r = i / W, sc = i - r * W;
    const int s = sc / FD_NCM, c = sc - s * FD_NCM;
    slab[r * P + sc] = r < n ? __ldcg(tptr(s, r, c)) : 0.0;
  }
  __syncthreads();
  double acc[RT][CT][2];
#pragma unroll
  for (int i = 0; i < RT; ++i)
#pragma unroll
    for (int j = 0; j < CT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  fd_gemm<RT, CT, true>(fd.s, np, slab, P, warp, lane, acc);
  // modal solve: row a of the tile is mode (a, b); segment s of column c is
  // column tile s*CPS + c/8 of the same thread
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int a = (warp + 8 * i) * 8 + (lane >> 2);
    const double l = a < n ? __ldg(fd.lam + (int64_t)a * n + b) : 1.0;
#pragma unroll
    for (int j = 0; j < CPS; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if constexpr (NSEG == 1) {
          acc[i][j][e] = acc[i][j][e] / l;
        } else {
          const double r1 = acc[i][j][e], r2 = acc[i][CPS + j][e], r3 = acc[i][2 * CPS + j][e];
          const double d = 1.0 / fma(fd.beta * l, l, 1.0);
          acc[i][j][e] = d * (r1 + l * (r2 - fd.beta * r3));
          acc[i][CPS + j][e] = d * (l * (r1 + l * r2) + r3);
          acc[i][2 * CPS + j][e] = d * (r2 - fd.beta * (l * r1 + r3));
        }
      }
  }
  __syncthreads();  // every warp is done reading the slab
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int a = (warp + 8 * i) * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < CT; ++j) {
      const int c = j * 8 + 2 * (lane & 3);
      if (a < np) {
        slab[a * P + c] = a < n ? acc[i][j][0] : 0.0;
        slab[a * P + c + 1] = a < n ? acc[i][j][1] : 0.0;
      }
      acc[i][j][0] = acc[i][j][1] = 0.0;
    }
  }
  __syncthreads();
  fd_gemm<RT, CT, false>(fd.s, np, slab, P, warp, lane, acc);
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int iy = (warp + 8 * i) * 8 + (lane >> 2);
    if (iy >= n) continue;
#pragma unroll
    for (int j = 0; j < CT; ++j) {
      const int s = j / CPS, c = (j - s * CPS) * 8 + 2 * (lane & 3);
      __stcg(reinterpret_cast<double2*>(tptr(s, iy, c)), make_double2(acc[i][j][0], acc[i][j][1]));
    }
  }
}

// ---------------------------------------------------------------------------
// Centrosymmetric ("half") form.  A uniform-grid Q1 lead has symmetric
// tridiagonal Toeplitz K1, M1, so every 1-D mode is symmetric or
// antisymmetric: S[n-1-i, j] = +-S[i, j].  With the modes ordered symmetric
// first (ne of them; host-permuted, lam permuted alike) a transform splits
// into two half-size GEMMs around a butterfly:
//   forward  C[0:ne]  = S_E^T E,  E[i] = X[i] + X[n-1-i] (i < h), E[h] = X[h] (n odd)
//            C[ne:n]  = S_O^T O,  O[i] = X[i] - X[n-1-i] (i < h)
//   inverse  X[i] = P_E[i] + P_O[i],  X[n-1-i] = P_E[i] - P_O[i],  X[h] = P_E[h]
//            P_E = S_E C[0:ne],  P_O = S_O C[ne:n]
// with h = n/2, S_E = S[0:h+odd, 0:ne], S_O = S[0:h, ne:n] (each zero-padded
// to hp x hp in fd.sh: S_E then S_O).  Half the flops of the full passes.
template <int RT, bool BACK>
__global__ void __launch_bounds__(256) fdh_line(sgk_fastdiag fd, sgk_segview xv, double* __restrict__ T, int width,
                                                int wpad) {
  constexpr int CT = FD_NC / 8;
  constexpr int P = fd_pitch(FD_NC);
  extern __shared__ __align__(16) double slab[];
  const int n = fd.n, hp = fd.hp, ne = fd.ne, h = n / 2, odd = n & 1;
  double* sE = slab;
  double* sO = slab + hp * P;
  const int line = blockIdx.x;
  const int seg = line / n, iy = line - seg * n;
  const int c0 = blockIdx.y * FD_NC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* xs = seg == 0 ? xv.ptr[0] : (seg == 1 ? xv.ptr[1] : xv.ptr[2]);
  double* tl = T + ((int64_t)seg * n + iy) * n * wpad;
  const double* SE = fd.sh;
  const double* SO = fd.sh + (int64_t)hp * hp;
  for (int i = tid; i < hp * FD_NC; i += blockDim.x) {
    const int r = i / FD_NC, c = i - r * FD_NC;
    double e = 0.0, o = 0.0;
    if (c0 + c < width) {
      if (BACK) {
        if (r < ne) e = __ldcg(tl + (int64_t)r * wpad + c0 + c);
        if (r < n - ne) o = __ldcg(tl + (int64_t)(ne + r) * wpad + c0 + c);
      } else {
        const double* xr = xs + (int64_t)iy * n * xv.ld + xv.col0 + c0 + c;
        if (r < h) {
          const double a = xr[(int64_t)r * xv.ld], b = xr[(int64_t)(n - 1 - r) * xv.ld];
          e = a + b;
          o = a - b;
        } else if (r == h && odd) {
          e = xr[(int64_t)r * xv.ld];
        }
      }
    }
    sE[r * P + c] = e;
    sO[r * P + c] = o;
  }
  __syncthreads();
  double aE[RT][CT][2], aO[RT][CT][2];
#pragma unroll
  for (int i = 0; i < RT; ++i)
#pragma unroll
    for (int j = 0; j < CT; ++j) aE[i][j][0] = aE[i][j][1] = aO[i][j][0] = aO[i][j][1] = 0.0;
  fd_gemm<RT, CT, !BACK>(SE, hp, sE, P, warp, lane, aE);
  fd_gemm<RT, CT, !BACK>(SO, hp, sO, P, warp, lane, aO);
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int r = (warp + 8 * i) * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < CT; ++j) {
      const int c = c0 + j * 8 + 2 * (lane & 3);
      if (BACK) {
        double* base = xs + (int64_t)iy * n * xv.ld + xv.col0 + c;
        if (r < h) {
          double* lo = base + (int64_t)r * xv.ld;
          double* hi = base + (int64_t)(n - 1 - r) * xv.ld;
          if (c < width) {
            lo[0] = aE[i][j][0] + aO[i][j][0];
            hi[0] = aE[i][j][0] - aO[i][j][0];
          }
          if (c + 1 < width) {
            lo[1] = aE[i][j][1] + aO[i][j][1];
            hi[1] = aE[i][j][1] - aO[i][j][1];
          }
        } else if (r == h && odd) {
          double* mid = base + (int64_t)r * xv.ld;
          if (c < width) mid[0] = aE[i][j][0];
          if (c + 1 < width) mid[1] = aE[i][j][1];
        }
      } else {
        if (r < ne)
          __stcg(reinterpret_cast<double2*>(tl + (int64_t)r * wpad + c), make_double2(aE[i][j][0], aE[i][j][1]));
        if (r < n - ne)
          __stcg(reinterpret_cast<double2*>(tl + (int64_t)(ne + r) * wpad + c), make_double2(aO[i][j][0], aO[i][j][1]));
      }
    }
  }
}

template <int RT, int NSEG>
__global__ void __launch_bounds__(256) fdh_mid(sgk_fastdiag fd, double* __restrict__ T, int width, int wpad) {
  constexpr int CPS = FD_NCM / 8;
  constexpr int CT = NSEG * CPS;
  constexpr int W = NSEG * FD_NCM;
  constexpr int P = fd_pitch(W);
  extern __shared__ __align__(16) double slab[];
  const int n = fd.n, hp = fd.hp, ne = fd.ne, h = n / 2, odd = n & 1;
  double* sE = slab;
  double* sO = slab + hp * P;
  const int b = blockIdx.x;
  const int c0 = blockIdx.y * FD_NCM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const double* SE = fd.sh;
  const double* SO = fd.sh + (int64_t)hp * hp;
  auto tptr = [&](int s, int iy, int c) { return T + (((int64_t)s * n + iy) * n + b) * wpad + c0 + c; };
  for (int i = tid; i < hp * W; i += blockDim.x) {
    const int r = i / W, sc = i - r * W;
    const int s = sc / FD_NCM, c = sc - s * FD_NCM;
    double e = 0.0, o = 0.0;
    if (r < h) {
      const double a = __ldcg(tptr(s, r, c)), bb = __ldcg(tptr(s, n - 1 - r, c));
      e = a + bb;
      o = a - bb;
    } else if (r == h && odd) {
      e = __ldcg(tptr(s, r, c));
    }
    sE[r * P + sc] = e;
    sO[r * P + sc] = o;
  }
  __syncthreads();
  double aE[RT][CT][2], aO[RT][CT][2];
#pragma unroll
  for (int i = 0; i < RT; ++i)
#pragma unroll
    for (int j = 0; j < CT; ++j) aE[i][j][0] = aE[i][j][1] = aO[i][j][0] = aO[i][j][1] = 0.0;
  fd_gemm<RT, CT, true>(SE, hp, sE, P, warp, lane, aE);
  fd_gemm<RT, CT, true>(SO, hp, sO, P, warp, lane, aO);
  // modal solve: row r of aE is mode a = r, of aO mode a = ne + r
  auto modal = [&](double (&acc)[RT][CT][2], int i, int a) {
    const double l = a < n ? __ldg(fd.lam + (int64_t)a * n + b) : 1.0;
#pragma unroll
    for (int j = 0; j < CPS; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        if constexpr (NSEG == 1) {
          acc[i][j][e] = acc[i][j][e] / l;
        } else {
          const double r1 = acc[i][j][e], r2 = acc[i][CPS + j][e], r3 = acc[i][2 * CPS + j][e];
          const double d = 1.0 / fma(fd.beta * l, l, 1.0);
          acc[i][j][e] = d * (r1 + l * (r2 - fd.beta * r3));
          acc[i][CPS + j][e] = d * (l * (r1 + l * r2) + r3);
          acc[i][2 * CPS + j][e] = d * (r2 - fd.beta * (l * r1 + r3));
        }
      }
  };
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int r = (warp + 8 * i) * 8 + (lane >> 2);
    modal(aE, i, r < ne ? r : n);
    modal(aO, i, r < n - ne ? ne + r : n);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int r = (warp + 8 * i) * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < CT; ++j) {
      const int c = j * 8 + 2 * (lane & 3);
      if (r < hp) {
        sE[r * P + c] = r < ne ? aE[i][j][0] : 0.0;
        sE[r * P + c + 1] = r < ne ? aE[i][j][1] : 0.0;
        sO[r * P + c] = r < n - ne ? aO[i][j][0] : 0.0;
        sO[r * P + c + 1] = r < n - ne ? aO[i][j][1] : 0.0;
      }
      aE[i][j][0] = aE[i][j][1] = aO[i][j][0] = aO[i][j][1] = 0.0;
    }
  }
  __syncthreads();
  fd_gemm<RT, CT, false>(SE, hp, sE, P, warp, lane, aE);
  fd_gemm<RT, CT, false>(SO, hp, sO, P, warp, lane, aO);
#pragma unroll
  for (int i = 0; i < RT; ++i) {
    const int r = (warp + 8 * i) * 8 + (lane >> 2);
#pragma unroll
    for (int j = 0; j < CT; ++j) {
      const int s = j / CPS, c = (j - s * CPS) * 8 + 2 * (lane & 3);
      if (r < h) {
        __stcg(reinterpret_cast<double2*>(tptr(s, r, c)),
               make_double2(aE[i][j][0] + aO[i][j][0], aE[i][j][1] + aO[i][j][1]));
        __stcg(reinterpret_cast<double2*>(tptr(s, n - 1 - r, c)),
               make_double2(aE[i][j][0] - aO[i][j][0], aE[i][j][1] - aO[i][j][1]));
      } else if (r == h && odd) {
        __stcg(reinterpret_cast<double2*>(tptr(s, r, c)), make_double2(aE[i][j][0], aE[i][j][1]));
      }
    }
  }
}

template <int RT>
static int fdh_launch(const sgk_fastdiag& fd, const sgk_segview& b, const sgk_segview& x, double* T, int width,
                      cudaStream_t st) {
  const int n = fd.n;
  const int wpad = (width + FD_NC - 1) / FD_NC * FD_NC;
  const size_t sm_line = 2 * sizeof(double) * (size_t)fd.hp * fd_pitch(FD_NC);
  const size_t sm_mid = 2 * sizeof(double) * (size_t)fd.hp * fd_pitch(fd.n_seg * FD_NCM);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fdh_line<RT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(fdh_line<RT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(fdh_mid<RT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(fdh_mid<RT, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaGetLastError();
    attr = true;
  }
  const dim3 gl(fd.n_seg * n, wpad / FD_NC);
  fdh_line<RT, false><<<gl, 256, sm_line, st>>>(fd, b, T, width, wpad);
  if (int rc = check_launch("fdh_line<pass1>")) return rc;
  const dim3 gm(n, (width + FD_NCM - 1) / FD_NCM);
  if (fd.n_seg == 1)
    fdh_mid<RT, 1><<<gm, 256, sm_mid, st>>>(fd, T, width, wpad);
  else
    fdh_mid<RT, 3><<<gm, 256, sm_mid, st>>>(fd, T, width, wpad);
  if (int rc = check_launch("fdh_mid")) return rc;
  fdh_line<RT, true><<<gl, 256, sm_line, st>>>(fd, x, T, width, wpad);
  return check_launch("fdh_line<pass4>");
}

template <int RT>
static int fd_launch(const sgk_fastdiag& fd, const sgk_segview& b, const sgk_segview& x, double* T, int width,
                     cudaStream_t st) {
  const int n = fd.n;
  const int wpad = (width + FD_NC - 1) / FD_NC * FD_NC;
  const size_t sm_line = sizeof(double) * (size_t)fd.np * fd_pitch(FD_NC);
  const size_t sm_mid = sizeof(double) * (size_t)fd.np * fd_pitch(fd.n_seg * FD_NCM);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fd_line<RT, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(fd_line<RT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(fd_mid<RT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaFuncSetAttribute(fd_mid<RT, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    cudaGetLastError();
    attr = true;
  }
  const dim3 gl(fd.n_seg * n, wpad / FD_NC);
  fd_line<RT, false><<<gl, 256, sm_line, st>>>(fd, b, T, width, wpad);
  if (int rc = check_launch("fd_line<pass1>")) return rc;
  const dim3 gm(n, (width + FD_NCM - 1) / FD_NCM);
  if (fd.n_seg == 1)
    fd_mid<RT, 1><<<gm, 256, sm_mid, st>>>(fd, T, width, wpad);
  else
    fd_mid<RT, 3><<<gm, 256, sm_mid, st>>>(fd, T, width, wpad);
  if (int rc = check_launch("fd_mid")) return rc;
  fd_line<RT, true><<<gl, 256, sm_line, st>>>(fd, x, T, width, wpad);
  return check_launch("fd_line<pass4>");
}

}  // namespace sgk

extern "C" int64_t sgk_fastdiag_work_doubles(const sgk_fastdiag* fd, int32_t width) {
  if (!fd || fd->n <= 0 || width < 0) return -1;
  const int64_t wpad = (width + sgk::FD_NC - 1) / sgk::FD_NC * sgk::FD_NC;
  return (int64_t)fd->n_seg * fd->n * fd->n * wpad;
}

extern "C" int sgk_fastdiag_solve(const sgk_fastdiag* fd, const sgk_segview* b, const sgk_segview* x, double* work,
                                  int32_t width, void* stream) {
  using namespace sgk;
  SGK_REQUIRE(fd && b && x && fd->s && fd->lam, "sgk_fastdiag_solve: null argument");
  SGK_REQUIRE(fd->n > 0 && (fd->n_seg == 1 || fd->n_seg == 3), "sgk_fastdiag_solve: bad factor (n, n_seg)");
  SGK_REQUIRE(fd->np >= fd->n && fd->np % 8 == 0 && fd->np <= 256, "sgk_fastdiag_solve: np must be n rounded up to 8, <= 256");
  SGK_REQUIRE(width >= 0, "sgk_fastdiag_solve: negative width");
  if (width == 0) return SGK_OK;
  const int64_t n2 = (int64_t)fd->n * fd->n;
  SGK_REQUIRE(b->seg_rows == n2 && x->seg_rows == n2, "sgk_fastdiag_solve: segment rows != n*n");
  SGK_REQUIRE(b->ld >= b->col0 + width && x->ld >= x->col0 + width, "sgk_fastdiag_solve: view narrower than width");
  SGK_REQUIRE(work != nullptr, "sgk_fastdiag_solve: null workspace");
  for (int s = 0; s < fd->n_seg; ++s)
    SGK_REQUIRE(b->ptr[s] && x->ptr[s], "sgk_fastdiag_solve: null segment");
  cudaStream_t st = (cudaStream_t)stream;
  if (fd->sh != nullptr) {
    SGK_REQUIRE(fd->hp % 8 == 0 && fd->hp <= 128 && 2 * fd->hp >= fd->n && fd->ne >= 0 && fd->ne <= fd->n,
                "sgk_fastdiag_solve: bad half form (hp, ne)");
    const int ht = fd->hp / 8;
    if (ht <= 8) return fdh_launch<1>(*fd, *b, *x, work, width, st);
    return fdh_launch<2>(*fd, *b, *x, work, width, st);
  }
  const int tiles = fd->np / 8;
  if (tiles <= 8) return fd_launch<1>(*fd, *b, *x, work, width, st);
  if (tiles <= 16) return fd_launch<2>(*fd, *b, *x, work, width, st);
  return fd_launch<4>(*fd, *b, *x, work, width, st);
}
