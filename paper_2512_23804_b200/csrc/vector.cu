// K5 (Chebyshev step), column scaling, K6 (deterministic Krylov vector ops)
// and K7 (F-order <-> node-major layout) kernels.
#include "sgk_common.cuh"

namespace sgk {

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 148 * 8;  // fixed => reduction order is fixed

// ---------------------------------------------------------------------------
// K5: one step of chebyshev_mass_solve (preconditioners.py:89-97) over all
// columns at once: one warp per mesh row (grid-stride), lanes along the
// columns (coalesced x/b rows), two columns per lane per iteration so both
// columns' neighbour loads are in flight together (the per-element kernel
// was latency-bound at 1.7 TB/s).  x == nullptr / xp == nullptr stand for the zero
// iterate (the first two steps start from x0 = 0: no reads of zero buffers).
// The FMA order (row entries ascending from 0.0) is the per-element kernel's.
constexpr int kChebRegs = 9;

__device__ __forceinline__ double cheb_update(double omega, double si, double bv, double mx, double xv,
                                              double xpv) {
  return omega * (si * (bv - mx) + xv - xpv) + xpv;
}

__global__ void __launch_bounds__(256, 4) cheb_step_kernel(sgk_pattern pat, int slice, const double* __restrict__ scale,
                                 int64_t n_batch, int64_t n_cols, const double* __restrict__ b_all,
                                 const double* __restrict__ x_all, const double* __restrict__ xp_all,
                                 double* __restrict__ xn_all, double omega) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool small = (int64_t)pat.n_rows * n_cols < ((int64_t)1 << 31);
  const int64_t n_items = n_batch * pat.n_rows;
  for (int64_t gi = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; gi < n_items; gi += nw) {
    // batch bi: an independent (n_rows x n_cols) block at offset bi*n_rows*n_cols
    const int64_t bi = gi / pat.n_rows, i = gi - bi * pat.n_rows;
    const int64_t base = bi * pat.n_rows * n_cols;
    const double* b = b_all + base;
    const double* x = x_all ? x_all + base : nullptr;
    const double* xp = xp_all ? xp_all + base : nullptr;
    double* xn = xn_all + base;
    const int rs = __ldg(pat.rowptr + i), len = __ldg(pat.rowptr + i + 1) - rs;
    const double* a = pat.vals + (int64_t)rs * pat.n_slices + (int64_t)slice * len;
    const double si = __ldg(scale + i);
    const int64_t row0 = i * n_cols;
    if (len <= kChebRegs && small) {
      // column indices and coefficients are warp-uniform L1 loads (registers
      // go to the two columns' x values; 64 registers -> 4 CTAs per SM);
      // element offsets fit in 32 bits here
      const int32_t* ci = pat.colind + rs;
      // two columns per lane per iteration: both columns' loads in flight
      for (int64_t k = lane; k < n_cols; k += 64) {
        const bool two = k + 32 < n_cols;
        double m0 = 0.0, m1 = 0.0;
        if (x != nullptr) {
          double x0[kChebRegs], x1[kChebRegs];
#pragma unroll
          for (int jj = 0; jj < kChebRegs; ++jj) {
            x0[jj] = jj < len ? __ldg(x + __ldg(ci + jj) * (int)n_cols + k) : 0.0;
            x1[jj] = (jj < len && two) ? __ldg(x + __ldg(ci + jj) * (int)n_cols + k + 32) : 0.0;
          }
#pragma unroll
          for (int jj = 0; jj < kChebRegs; ++jj)
            if (jj < len) {
              const double aj = __ldg(a + jj);
              m0 = fma(aj, x0[jj], m0);
              m1 = fma(aj, x1[jj], m1);
            }
        }
        const int64_t e = row0 + k;
        const double b0 = __ldg(b + e), b1 = two ? __ldg(b + e + 32) : 0.0;
        const double xv0 = x ? __ldg(x + e) : 0.0, xv1 = (x && two) ? __ldg(x + e + 32) : 0.0;
        const double xp0 = xp ? __ldg(xp + e) : 0.0, xp1 = (xp && two) ? __ldg(xp + e + 32) : 0.0;
        xn[e] = cheb_update(omega, si, b0, m0, xv0, xp0);
        if (two) xn[e + 32] = cheb_update(omega, si, b1, m1, xv1, xp1);
      }
    } else {
      for (int64_t k = lane; k < n_cols; k += 32) {
        double mx = 0.0;
        if (x != nullptr)
          for (int jj = 0; jj < len; ++jj)
            mx = fma(__ldg(a + jj), __ldg(x + (int64_t)__ldg(pat.colind + rs + jj) * n_cols + k), mx);
        const double xv = x ? __ldg(x + row0 + k) : 0.0;
        const double xpv = xp ? __ldg(xp + row0 + k) : 0.0;
        xn[row0 + k] = cheb_update(omega, si, __ldg(b + row0 + k), mx, xv, xpv);
      }
    }
  }
}

// Batched column scaling: block b of n_batch back-to-back (n_rows x n_cols)
// blocks is scaled by the device scalar s[b] (the N_t steps of the PINT
// preconditioner: one launch instead of one per step); per element the same
// arithmetic as colscale_kernel.
__global__ void colscale_batched_kernel(int64_t n_batch, int64_t n_rows, int64_t n_cols,
                                        const double* __restrict__ x, const double* __restrict__ w, int invert,
                                        const double* __restrict__ s, double* y) {
  const int64_t blk = n_rows * n_cols;
  const int64_t total = n_batch * blk;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double v = x[idx];
    if (w) {
      const double wk = __ldg(w + idx % n_cols);
      v = invert ? v / wk : v * wk;
    }
    y[idx] = __ldg(s + idx / blk) * v;
  }
}

__global__ void colscale_kernel(int64_t n_rows, int64_t n_cols, const double* __restrict__ x,
                                const double* __restrict__ w, int invert, double s, double* y) {
  const int64_t total = n_rows * n_cols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    double v = x[idx];
    if (w) {
      const double wk = __ldg(w + idx % n_cols);
      v = invert ? v / wk : v * wk;
    }
    y[idx] = s * v;
  }
}

// ---------------------------------------------------------------------------
// K6: deterministic reductions.  Block b always covers the same index set
// (grid-stride with a fixed grid) and reduces it in a fixed tree, so the
// result does not depend on scheduling.
template <int K>
__device__ __forceinline__ void block_reduce_store(double (&v)[K], double* part, int nb) {
  __shared__ double sh[K][kRedThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    double s = v[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) sh[j][warp] = s;
  }
  __syncthreads();
  if (threadIdx.x < K) {
    double s = 0.0;
    for (int w = 0; w < kRedThreads / 32; ++w) s += sh[threadIdx.x][w];
    part[(int64_t)threadIdx.x * nb + blockIdx.x] = s;
  }
}

template <int K>
__global__ void __launch_bounds__(kRedThreads) mdot_kernel(int64_t n, const double* __restrict__ x,
                                                           const double* __restrict__ y, int64_t ys,
                                                           double* part) {
  double v[K];
#pragma unroll
  for (int j = 0; j < K; ++j) v[j] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)kRedThreads + threadIdx.x; i < n;
       i += (int64_t)kRedBlocks * kRedThreads) {
    const double xi = __ldg(x + i);
#pragma unroll
    for (int j = 0; j < K; ++j) v[j] = fma(xi, __ldg(y + j * ys + i), v[j]);
  }
  block_reduce_store<K>(v, part, kRedBlocks);
}

__global__ void __launch_bounds__(1024) reduce_partials_kernel(const double* __restrict__ part, double* out,
                                                               int take_sqrt) {
  __shared__ double sh[32];
  const int j = blockIdx.x;
  const double* p = part + (int64_t)j * kRedBlocks;
  double s = 0.0;
  for (int b = threadIdx.x; b < kRedBlocks; b += 1024) s += p[b];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) sh[warp] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 32; ++w) t += sh[w];
    out[j] = take_sqrt ? sqrt(t) : t;
  }
}

__global__ void axpby_kernel(int64_t n, double sa, const double* da, int inv_a, const double* __restrict__ x,
                             double sb, const double* db, double* y) {
  double a = sa, b = sb;
  if (da) a = inv_a ? sa / *da : sa * *da;
  if (db) b = sb * *db;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double yi = (b == 0.0) ? 0.0 : b * y[i];
    y[i] = (a == 0.0) ? yi : fma(a, x[i], yi);
  }
}

// out = s * ((x0 + c1 x1) + c2 x2), each step rounded exactly as the axpby
// chain it replaces (y <- a x + b y with b = 1, then a final scale): one pass
// instead of a copy + three axpby passes (the MINRES three-term recurrences).
__device__ __forceinline__ double axpby_op(double a, double x, double b, double y) {
  const double yi = (b == 0.0) ? 0.0 : b * y;
  return (a == 0.0) ? yi : fma(a, x, yi);
}

__global__ void lincomb3_kernel(int64_t n, const double* x0, double c1, const double* __restrict__ x1, double c2,
                                const double* __restrict__ x2, double s, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double t = x0[i];
    if (x1) t = axpby_op(c1, __ldg(x1 + i), 1.0, t);
    if (x2) t = axpby_op(c2, __ldg(x2 + i), 1.0, t);
    if (s != 1.0) t = axpby_op(0.0, 0.0, s, t);
    out[i] = t;
  }
}

// Modified Gram–Schmidt step (krylov.py:81-84) fused with the partial dot
// product of the next basis vector against the updated w.
__global__ void __launch_bounds__(kRedThreads) mgs_step_kernel(int64_t n, const double* dh,
                                                               const double* __restrict__ q,
                                                               double* w,
                                                               const double* __restrict__ qn,
                                                               double* part) {
  const double h = *dh;
  double v[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)kRedThreads + threadIdx.x; i < n;
       i += (int64_t)kRedBlocks * kRedThreads) {
    const double wi = w[i] - h * q[i];
    w[i] = wi;
    if (qn) v[0] = fma(__ldg(qn + i), wi, v[0]);
  }
  if (qn) block_reduce_store<1>(v, part, kRedBlocks);
}

// ---------------------------------------------------------------------------
// K7: layout transposes (32x32 tiles through shared memory).
__global__ void transpose_kernel(int64_t rows, int64_t cols, const double* __restrict__ in,
                                 double* __restrict__ out) {
  // in: rows x cols row-major ; out: cols x rows row-major
  __shared__ double tile[32][33];
  const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t r = r0 + dy, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[dy][threadIdx.x] = in[r * cols + c];
  }
  __syncthreads();
  for (int dy = threadIdx.y; dy < 32; dy += blockDim.y) {
    const int64_t c = c0 + dy, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[c * rows + r] = tile[threadIdx.x][dy];
  }
}

static int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)sm_count() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

static int transpose(int64_t rows, int64_t cols, const double* in, double* out, cudaStream_t st) {
  if (rows == 0 || cols == 0) return SGK_OK;
  SGK_REQUIRE((cols + 31) / 32 < (1ll << 31) && (rows + 31) / 32 < 65536, "transpose: too large");
  dim3 grid((unsigned)((cols + 31) / 32), (unsigned)((rows + 31) / 32));
  transpose_kernel<<<grid, dim3(32, 8), 0, st>>>(rows, cols, in, out);
  return check_launch("transpose_kernel");
}

}  // namespace sgk

using namespace sgk;

extern "C" int sgk_cheb_step_batched(const sgk_pattern* pat, int32_t slice, const double* scale, int64_t n_batch,
                                     int64_t n_cols, const double* b, const double* x, const double* x_prev,
                                     double* x_new, double omega, void* stream) {
  SGK_REQUIRE(pat && scale && b && x_new, "sgk_cheb_step: null argument");
  SGK_REQUIRE(slice >= 0 && slice < pat->n_slices, "sgk_cheb_step: slice out of range");
  SGK_REQUIRE(n_batch >= 0 && n_cols >= 0, "sgk_cheb_step: negative size");
  SGK_REQUIRE(x_new != x && x_new != x_prev, "sgk_cheb_step: x_new must not alias x/x_prev");
  const int64_t rows = n_batch * pat->n_rows;
  if (rows == 0 || n_cols == 0) return SGK_OK;
  // one warp per row, 8 rows per CTA, grid = the resident CTAs (4 per SM)
  int64_t blocks = (rows + 7) / 8;
  if (blocks > (int64_t)sm_count() * 4) blocks = (int64_t)sm_count() * 4;
  cheb_step_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(*pat, slice, scale, n_batch, n_cols, b, x,
                                                                   x_prev, x_new, omega);
  return check_launch("cheb_step_kernel");
}

extern "C" int sgk_cheb_step(const sgk_pattern* pat, int32_t slice, const double* scale,
                             int64_t n_cols, const double* b, const double* x, const double* x_prev,
                             double* x_new, double omega, void* stream) {
  return sgk_cheb_step_batched(pat, slice, scale, 1, n_cols, b, x, x_prev, x_new, omega, stream);
}

extern "C" int sgk_colscale_batched(int64_t n_batch, int64_t n_rows, int64_t n_cols, const double* x,
                                    const double* w, int32_t invert_w, const double* s, double* y, void* stream) {
  SGK_REQUIRE(x && y && s, "sgk_colscale_batched: null argument");
  SGK_REQUIRE(n_batch >= 0 && n_rows >= 0 && n_cols >= 0, "sgk_colscale_batched: negative size");
  const int64_t total = n_batch * n_rows * n_cols;
  if (total == 0) return SGK_OK;
  colscale_batched_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(n_batch, n_rows, n_cols, x, w,
                                                                                 invert_w, s, y);
  return check_launch("colscale_batched_kernel");
}

extern "C" int sgk_colscale(int64_t n_rows, int64_t n_cols, const double* x, const double* w,
                            int32_t invert_w, double s, double* y, void* stream) {
  SGK_REQUIRE(x && y, "sgk_colscale: null argument");
  const int64_t total = n_rows * n_cols;
  if (total == 0) return SGK_OK;
  colscale_kernel<<<grid_for(total, 256), 256, 0, (cudaStream_t)stream>>>(n_rows, n_cols, x, w, invert_w, s, y);
  return check_launch("colscale_kernel");
}

extern "C" int32_t sgk_reduce_blocks(void) { return kRedBlocks; }

extern "C" int sgk_dot_partial(int64_t n, const double* x, const double* y, int64_t ystride, int32_t k,
                               double* part, void* stream) {
  SGK_REQUIRE(x && y && part, "sgk_dot_partial: null argument");
  SGK_REQUIRE(k >= 1 && k <= SGK_MAX_MDOT, "sgk_dot_partial: k out of range");
  cudaStream_t st = (cudaStream_t)stream;
  switch (k) {
#define SGK_MDOT_CASE(K) \
  case K:                \
    mdot_kernel<K><<<kRedBlocks, kRedThreads, 0, st>>>(n, x, y, ystride, part); break;
    SGK_MDOT_CASE(1) SGK_MDOT_CASE(2) SGK_MDOT_CASE(3) SGK_MDOT_CASE(4)
    SGK_MDOT_CASE(5) SGK_MDOT_CASE(6) SGK_MDOT_CASE(7) SGK_MDOT_CASE(8)
#undef SGK_MDOT_CASE
  }
  return check_launch("mdot_kernel");
}

extern "C" int sgk_reduce_partials(const double* part, int32_t k, double* out, int32_t take_sqrt,
                                   void* stream) {
  SGK_REQUIRE(part && out && k >= 1, "sgk_reduce_partials: bad argument");
  reduce_partials_kernel<<<k, 1024, 0, (cudaStream_t)stream>>>(part, out, take_sqrt);
  return check_launch("reduce_partials_kernel");
}

extern "C" int sgk_axpby_dev(int64_t n, double sa, const double* da, int32_t inv_a, const double* x,
                             double sb, const double* db, double* y, void* stream) {
  SGK_REQUIRE(y && (x || (sa == 0.0 && !da)), "sgk_axpby_dev: null argument");
  if (n == 0) return SGK_OK;
  axpby_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, sa, da, inv_a, x, sb, db, y);
  return check_launch("axpby_kernel");
}

extern "C" int sgk_lincomb3(int64_t n, const double* x0, double c1, const double* x1, double c2,
                            const double* x2, double s, double* out, void* stream) {
  SGK_REQUIRE(x0 && out, "sgk_lincomb3: null argument");
  SGK_REQUIRE(out == x0 || (out != x1 && out != x2), "sgk_lincomb3: out may alias x0 only");
  if (n == 0) return SGK_OK;
  lincomb3_kernel<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(n, x0, c1, x1, c2, x2, s, out);
  return check_launch("lincomb3_kernel");
}

extern "C" int sgk_mgs_step(int64_t n, const double* dh, const double* q_i, double* w,
                            const double* q_next, double* part_next, void* stream) {
  SGK_REQUIRE(dh && q_i && w && (!q_next || part_next), "sgk_mgs_step: null argument");
  mgs_step_kernel<<<kRedBlocks, kRedThreads, 0, (cudaStream_t)stream>>>(n, dh, q_i, w, q_next, part_next);
  return check_launch("mgs_step_kernel");
}

extern "C" int sgk_f2n(int64_t n_rows, int64_t n_cols, const double* f, double* nm, void* stream) {
  SGK_REQUIRE(f && nm && f != nm, "sgk_f2n: bad argument");
  // F-order (n_rows x n_cols) is row-major (n_cols x n_rows).
  return transpose(n_cols, n_rows, f, nm, (cudaStream_t)stream);
}

extern "C" int sgk_n2f(int64_t n_rows, int64_t n_cols, const double* nm, double* f, void* stream) {
  SGK_REQUIRE(f && nm && f != nm, "sgk_n2f: bad argument");
  return transpose(n_rows, n_cols, nm, f, (cudaStream_t)stream);
}
