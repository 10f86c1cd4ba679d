// K3 — sync-free, level-ordered, multi-RHS sparse triangular solves on the
// host-computed SuperLU factors (linalg.py:76-120: splu(diag_pivot_thresh=1)
// gives Pr A Pc = L U; LUFactors.solve = Pc U^-1 L^-1 Pr b).
//
// One warp per factor row; rows are claimed through an atomic ticket in
// level (topological) order, so a warp only ever waits on rows whose tickets
// were issued earlier — those warps are resident and finish, hence no
// deadlock without a grid-wide barrier.  Readiness is an epoch-stamped flag
// per row (st.release / ld.acquire at gpu scope); the solution rows are read
// through L2 (ld.cg) because other SMs write them during the same kernel.
// All RHS columns of a degree level ride along one row visit (lanes cover
// columns), so the factor is streamed once per level instead of once per
// column.
#include "sgk_common.cuh"

namespace sgk {

__device__ __forceinline__ double seg_load(const sgk_segview& s, int r, int c) {
  const int seg = r / s.seg_rows;
  const int rr = r - seg * s.seg_rows;
  return s.ptr[seg][(int64_t)rr * s.ld + s.col0 + c];
}
__device__ __forceinline__ void seg_store(const sgk_segview& s, int r, int c, double v) {
  const int seg = r / s.seg_rows;
  const int rr = r - seg * s.seg_rows;
  s.ptr[seg][(int64_t)rr * s.ld + s.col0 + c] = v;
}

// FWD: z[k] = b[in_perm[k]] - sum_{c} L[k,c] z[c]      (unit diagonal)
// BWD: y[k] = (z[k] - sum_{c} U[k,c] y[c]) * dinv[k];  x[out_perm[k]] = y[k]
template <int CPL, bool FWD>
__global__ void __launch_bounds__(256) trsv_kernel(sgk_trifactor f, const int32_t* __restrict__ perm,
                                                   sgk_segview io, double* __restrict__ work,
                                                   int width, int epoch) {
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  for (;;) {
    int ticket = 0;
    if (lane == 0) ticket = atomicAdd(f.ticket, 1);
    ticket = __shfl_sync(FULL, ticket, 0);
    if (ticket >= f.n) return;
    const int k = __ldg(f.order + ticket);
    const int e0 = __ldg(f.rowptr + k), e1 = __ldg(f.rowptr + k + 1);

    // Wait until every dependency row is published (lanes poll in parallel).
    for (int base = e0; base < e1; base += 32) {
      const int e = base + lane;
      if (e < e1) {
        const int32_t* fl = f.flags + __ldg(f.colind + e);
        while (ld_acquire(fl) != epoch) __nanosleep(32);
      }
    }
    __syncwarp();

    const int src = FWD ? __ldg(perm + k) : k;
    const double dinv = (!FWD && f.diag_inv) ? __ldg(f.diag_inv + k) : 1.0;
    for (int cb = 0; cb < width; cb += 32 * CPL) {
      double acc[CPL];
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int col = cb + lane + 32 * c;
        acc[c] = 0.0;
        if (col < width) acc[c] = FWD ? seg_load(io, src, col) : __ldcg(work + (int64_t)k * width + col);
      }
      for (int base = e0; base < e1; base += 32) {
        const int e = base + lane;
        int myc = 0;
        double myv = 0.0;
        if (e < e1) {
          myc = __ldg(f.colind + e);
          myv = __ldg(f.vals + e);
        }
        const int cnt = min(32, e1 - base);
        for (int j = 0; j < cnt; ++j) {
          const int cj = __shfl_sync(FULL, myc, j);
          const double vj = __shfl_sync(FULL, myv, j);
          const double* zr = work + (int64_t)cj * width;
#pragma unroll
          for (int c = 0; c < CPL; ++c) {
            const int col = cb + lane + 32 * c;
            if (col < width) acc[c] = fma(-vj, __ldcg(zr + col), acc[c]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < CPL; ++c) {
        const int col = cb + lane + 32 * c;
        if (col < width) {
          const double y = FWD ? acc[c] : acc[c] * dinv;
          __stcg(work + (int64_t)k * width + col, y);
          if (!FWD) seg_store(io, __ldg(perm + k), col, y);
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      __threadfence();
      st_release(f.flags + k, epoch);
    }
  }
}

template <int CPL>
static int launch_pair(const sgk_trifactor& L, const sgk_trifactor& U, const int32_t* in_perm,
                       const int32_t* out_perm, const sgk_segview& b, const sgk_segview& x,
                       double* work, int width, int epoch, cudaStream_t st) {
  const int threads = 256;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, trsv_kernel<CPL, true>, threads, 0);
  if (occ < 1) occ = 1;
  int64_t warps_needed = (L.n + 0);
  int64_t grid = (int64_t)sm_count() * occ;
  const int64_t max_grid = (warps_needed + 7) / 8;
  if (grid > max_grid) grid = max_grid;
  if (grid < 1) grid = 1;
  cudaMemsetAsync(L.ticket, 0, sizeof(int32_t), st);
  cudaMemsetAsync(U.ticket, 0, sizeof(int32_t), st);
  trsv_kernel<CPL, true><<<(int)grid, threads, 0, st>>>(L, in_perm, b, work, width, epoch);
  int rc = check_launch("trsv_kernel<fwd>");
  if (rc) return rc;
  trsv_kernel<CPL, false><<<(int)grid, threads, 0, st>>>(U, out_perm, x, work, width, epoch);
  return check_launch("trsv_kernel<bwd>");
}

}  // namespace sgk

extern "C" int sgk_trisolve(const sgk_trifactor* L, const sgk_trifactor* U, const int32_t* in_perm,
                            const int32_t* out_perm, const sgk_segview* b, const sgk_segview* x,
                            double* work, int32_t width, int32_t epoch, void* stream) {
  using namespace sgk;
  SGK_REQUIRE(L && U && in_perm && out_perm && b && x && work, "sgk_trisolve: null argument");
  SGK_REQUIRE(L->n == U->n && L->n >= 0, "sgk_trisolve: factor sizes differ");
  SGK_REQUIRE(L->lower == 1 && U->lower == 0, "sgk_trisolve: expected (lower, upper) factors");
  SGK_REQUIRE(U->diag_inv != nullptr, "sgk_trisolve: upper factor needs its inverse diagonal");
  SGK_REQUIRE(width >= 0, "sgk_trisolve: negative width");
  SGK_REQUIRE(epoch > 0, "sgk_trisolve: epoch must be positive");
  SGK_REQUIRE(b->seg_rows > 0 && x->seg_rows > 0, "sgk_trisolve: seg_rows must be positive");
  if (L->n == 0 || width == 0) return SGK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (width <= 32) return launch_pair<1>(*L, *U, in_perm, out_perm, *b, *x, work, width, epoch, st);
  if (width <= 64) return launch_pair<2>(*L, *U, in_perm, out_perm, *b, *x, work, width, epoch, st);
  if (width <= 128) return launch_pair<4>(*L, *U, in_perm, out_perm, *b, *x, work, width, epoch, st);
  return launch_pair<8>(*L, *U, in_perm, out_perm, *b, *x, work, width, epoch, st);
}
