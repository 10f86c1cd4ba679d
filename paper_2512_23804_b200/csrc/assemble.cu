// GPU setup pipeline: the t-stacked Q1 operator values
// and the lognormal chaos coefficient fields built on the device.
//
// sgk_q1_assemble — reference fem.py:171-206 (`_accumulate`, `assemble_mass`,
// `assemble_stiffness`) for every coefficient field at once: the element
// matrix of field t on element e is sum_q f_t[e,q] K_q (K_q the reference
// gradient products at Gauss point q; the (2/h)^2 gradient scaling cancels
// the (h/2)^2 weight in 2-D), the mass element matrix is w M_ref, and the
// global entry (i, j) sums the element entries of the (up to four) elements
// holding both nodes in ascending element order — the duplicate order of
// the reference's COO -> CSR scatter.  Boundary rows/columns are eliminated
// (interior nodes only).  One thread per (interior row, slice) writes the
// row's <= 9 values into both device layouts of DevicePattern: the general
// t-stacked CSR (vals[rowptr[i]*S + s*len_i + jj]) and the padded 9-point
// block (coef10[(i*S + s)*10 + jj], colind9[i*9 + jj], padding = last
// column with coefficient 0).
//
// sgk_lognormal_fields — reference random_field.py:130-151: the gPC
// coefficient of multi-index alpha at a Gauss point is
// mean * prod_i g_i^alpha_i / sqrt(alpha_i!).
#include <math.h>

#include "sgk_common.cuh"

namespace sgk {

__constant__ double c_stiff_q[4][4][4];  // [q][a][b]
__constant__ double c_mass_ref[4][4];

__global__ void q1_assemble_kernel(int n, int n_fields, int with_mass, double mass_w,
                                   const double* __restrict__ fields, const int32_t* __restrict__ rowptr,
                                   double* __restrict__ vals, double* __restrict__ coef10,
                                   int32_t* __restrict__ colind9) {
  const int m = n - 1;  // interior nodes per side
  const int n_rows = m * m;
  const int S = n_fields + with_mass;
  const int64_t total = (int64_t)n_rows * S;
  const int64_t n_el = (int64_t)n * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(idx / S);
    const int s = (int)(idx - (int64_t)row * S);
    const int X = row % m + 1, Y = row / m + 1;  // full-grid node coordinates
    double v[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) v[a][b] = 0.0;
    // elements (ex, ey) around the node, ascending element index ey*n + ex
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int ex = X - 1 + (k & 1), ey = Y - 1 + (k >> 1);
      const int64_t e = (int64_t)ey * n + ex;
      // local corners: 0 (ex,ey), 1 (ex+1,ey), 2 (ex+1,ey+1), 3 (ex,ey+1)
      const int dxi = X - ex, dyi = Y - ey;
      const int ai = dyi == 0 ? dxi : 3 - dxi;
      double fq[4];
      if (s < n_fields) {
#pragma unroll
        for (int q = 0; q < 4; ++q) fq[q] = __ldg(fields + ((int64_t)s * n_el + e) * 4 + q);
      }
#pragma unroll
      for (int aj = 0; aj < 4; ++aj) {
        const int cx = ex + (aj == 1 || aj == 2), cy = ey + (aj >= 2);
        double val;
        if (s < n_fields) {
          val = fq[0] * c_stiff_q[0][ai][aj];
#pragma unroll
          for (int q = 1; q < 4; ++q) val = fma(fq[q], c_stiff_q[q][ai][aj], val);
        } else {
          val = mass_w * c_mass_ref[ai][aj];
        }
        v[cy - Y + 1][cx - X + 1] += val;
      }
    }
    // interior neighbours in ascending column order (dy-major, dx-minor)
    const int rs = __ldg(rowptr + row), len = __ldg(rowptr + row + 1) - rs;
    double* out = vals + (int64_t)rs * S + (int64_t)s * len;
    double* c10 = coef10 ? coef10 + ((int64_t)row * S + s) * 10 : nullptr;
    int jj = 0, last = row;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        const int cx = X + dx, cy = Y + dy;
        if (cx < 1 || cx > m || cy < 1 || cy > m) continue;
        const int col = (cy - 1) * m + (cx - 1);
        out[jj] = v[dy + 1][dx + 1];
        if (c10) c10[jj] = v[dy + 1][dx + 1];
        if (colind9 && s == 0) colind9[(int64_t)row * 9 + jj] = col;
        last = col;
        ++jj;
      }
    if (c10) {
      for (int k = jj; k < 10; ++k) c10[k] = 0.0;
    }
    if (colind9 && s == 0) {
      for (int k = jj; k < 9; ++k) colind9[(int64_t)row * 9 + k] = last;
    }
  }
}

__global__ void lognormal_fields_kernel(int64_t n_points, int m, int n_terms, const double* __restrict__ mean,
                                        const double* __restrict__ g, const int32_t* __restrict__ idx,
                                        double* __restrict__ out) {
  const int64_t total = n_points * n_terms;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int t = (int)(i / n_points);
    const int64_t p = i - (int64_t)t * n_points;
    double c = __ldg(mean + p);
    for (int v = 0; v < m; ++v) {
      const int k = __ldg(idx + (int64_t)t * m + v);
      if (k) {
        const double gv = __ldg(g + (int64_t)v * n_points + p);
        double pw = gv;
        double fact = 1.0;
        for (int j = 2; j <= k; ++j) {
          pw *= gv;
          fact *= j;
        }
        c = c * pw / sqrt(fact);
      }
    }
    out[i] = c;
  }
}

}  // namespace sgk

extern "C" int sgk_q1_assemble(int32_t n_cells, int32_t n_fields, const double* fields, const double* stiff_q,
                               int32_t with_mass, double mass_weight, const double* mass_ref,
                               const int32_t* rowptr, double* vals, double* coef10, int32_t* colind9,
                               void* stream) {
  using namespace sgk;
  SGK_REQUIRE(n_cells >= 2, "sgk_q1_assemble: need at least 2 cells per side");
  SGK_REQUIRE(n_fields >= 0 && (n_fields > 0 || with_mass), "sgk_q1_assemble: nothing to assemble");
  SGK_REQUIRE(stiff_q && mass_ref && rowptr && vals && (n_fields == 0 || fields),
              "sgk_q1_assemble: null argument");
  cudaStream_t st = (cudaStream_t)stream;
  cudaMemcpyToSymbolAsync(c_stiff_q, stiff_q, sizeof(double) * 64, 0, cudaMemcpyHostToDevice, st);
  cudaMemcpyToSymbolAsync(c_mass_ref, mass_ref, sizeof(double) * 16, 0, cudaMemcpyHostToDevice, st);
  const int64_t total = (int64_t)(n_cells - 1) * (n_cells - 1) * (n_fields + (with_mass ? 1 : 0));
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)sm_count() * 32) blocks = (int64_t)sm_count() * 32;
  q1_assemble_kernel<<<(int)blocks, 256, 0, st>>>(n_cells, n_fields, with_mass ? 1 : 0, mass_weight, fields, rowptr,
                                                  vals, coef10, colind9);
  return check_launch("q1_assemble_kernel");
}

extern "C" int sgk_lognormal_fields(int64_t n_points, int32_t m, int32_t n_terms, const double* mean,
                                    const double* g, const int32_t* idx, double* out, void* stream) {
  using namespace sgk;
  SGK_REQUIRE(n_points >= 0 && m >= 0 && n_terms >= 0, "sgk_lognormal_fields: negative size");
  SGK_REQUIRE(mean && out && idx && (m == 0 || g), "sgk_lognormal_fields: null argument");
  const int64_t total = n_points * n_terms;
  if (total == 0) return SGK_OK;
  int64_t blocks = (total + 255) / 256;
  if (blocks > (int64_t)sm_count() * 32) blocks = (int64_t)sm_count() * 32;
  lognormal_fields_kernel<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(n_points, m, n_terms, mean, g, idx, out);
  return check_launch("lognormal_fields_kernel");
}
