// K3 — sync-free, level-ordered, multi-RHS sparse triangular solves on the
// host-computed SuperLU factors (linalg.py:76-120: splu(diag_pivot_thresh=1)
// gives Pr A Pc = L U; LUFactors.solve = Pc U^-1 L^-1 Pr b).
//
// One warp per factor row; rows are claimed through an atomic ticket in
// level (topological) order, so a warp only ever waits on rows whose tickets
// were issued earlier — those warps are resident and finish, hence no
// deadlock without a grid-wide barrier.  Readiness is an epoch-stamped flag
// per row (st.release / ld.acquire at gpu scope, polled with exponential
// back-off so idle warps do not flood L2); solution rows are read through L2
// (ld.cg) because other SMs write them during the same kernel.  All RHS
// columns of a degree level ride along one row visit.
//
// The critical path is the dependency depth (thousands of levels for the
// COLAMD-ordered KKT factor), so a row visit must cost about one L2 round
// trip: every load of the row is issued before any is consumed.
//   narrow (width <= 8): lanes split the row's entries, each lane keeps W
//     partial sums, then a butterfly reduction over the warp;
//   wide: lanes split the columns, entries processed 8 at a time with all 8
//     loads in flight.
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

__device__ __forceinline__ void wait_flag(const int32_t* fl, int epoch) {
  if (ld_acquire(fl) == epoch) return;
  unsigned ns = 32;
  while (ld_acquire(fl) != epoch) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
  }
}

// Column-chunked row visit.  A task is (factor row k, chunk of CW RHS
// columns); chunks of one row are independent, so wide degree levels spread
// over many SMs.  Lanes split the row's entries (EPL per lane per batch); the
// batch's flags are polled together and then all its loads are issued before
// any FMA, so a task costs ~2 L2 round trips per batch.  Partial sums are
// reduced across the warp with butterflies.
constexpr int CW = 16;
constexpr int EPL = 4;

template <bool FWD>
__global__ void __launch_bounds__(256) trsv_chunk(sgk_trifactor f, const int32_t* __restrict__ perm,
                                                  sgk_segview io, double* __restrict__ work, int width,
                                                  int n_chunks, int epoch) {
  const int lane = threadIdx.x & 31;
  const unsigned FULL = 0xffffffffu;
  const int64_t n_tasks = (int64_t)f.n * n_chunks;
  for (;;) {
    int ticket = 0;
    if (lane == 0) ticket = atomicAdd(f.ticket, 1);
    ticket = __shfl_sync(FULL, ticket, 0);
    if (ticket >= n_tasks) return;
    const int k = __ldg(f.order + ticket / n_chunks);
    const int chunk = ticket - (ticket / n_chunks) * n_chunks;
    const int c0 = chunk * CW;
    const int w = min(CW, width - c0);
    const int e0 = __ldg(f.rowptr + k), e1 = __ldg(f.rowptr + k + 1);
    double acc[CW];
#pragma unroll
    for (int c = 0; c < CW; ++c) acc[c] = 0.0;
    for (int base = e0; base < e1; base += 32 * EPL) {
      int cj[EPL];
      double vj[EPL];
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const int e = base + lane + 32 * u;
        cj[u] = e < e1 ? __ldg(f.colind + e) : -1;
        vj[u] = e < e1 ? __ldg(f.vals + e) : 0.0;
      }
      // poll this batch's flags together (relaxed), then one acquire fence
      for (;;) {
        bool ready = true;
#pragma unroll
        for (int u = 0; u < EPL; ++u)
          if (cj[u] >= 0) ready &= ld_relaxed(f.flags + (int64_t)cj[u] * n_chunks + chunk) == epoch;
        if (__all_sync(FULL, ready)) break;
        __nanosleep(64);
      }
      fence_acq_rel();  // acquire: the rows published under these flags are visible
      double xv[EPL][CW];
#pragma unroll
      for (int u = 0; u < EPL; ++u) {
        const double* zr = work + (int64_t)max(cj[u], 0) * width + c0;
#pragma unroll
        for (int c = 0; c < CW; ++c) xv[u][c] = (cj[u] >= 0 && c < w) ? __ldcg(zr + c) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < EPL; ++u)
#pragma unroll
        for (int c = 0; c < CW; ++c) acc[c] = fma(-vj[u], xv[u][c], acc[c]);
    }
#pragma unroll
    for (int c = 0; c < CW; ++c) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(FULL, acc[c], o);
    }
    if (lane < w) {
      double s = acc[0];
#pragma unroll
      for (int c = 1; c < CW; ++c)
        if (lane == c) s = acc[c];
      const int col = c0 + lane;
      double y;
      if (FWD) {
        y = seg_load(io, __ldg(perm + k), col) + s;
      } else {
        y = (__ldcg(work + (int64_t)k * width + col) + s) * __ldg(f.diag_inv + k);
        seg_store(io, __ldg(perm + k), col, y);
      }
      __stcg(work + (int64_t)k * width + col, y);
      fence_acq_rel();  // release this lane's results before the flag
    }
    __syncwarp();
    if (lane == 0) st_relaxed(f.flags + (int64_t)k * n_chunks + chunk, epoch);
  }
}

static int launch_chunked(const sgk_trifactor& L, const sgk_trifactor& U, const int32_t* in_perm,
                          const int32_t* out_perm, const sgk_segview& b, const sgk_segview& x, double* work,
                          int width, int n_chunks, int epoch, cudaStream_t st) {
  const int threads = 256;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, trsv_chunk<true>, threads, 0);
  if (occ < 1) occ = 1;
  if (occ > 4) occ = 4;  // enough warps to cover a level; fewer pollers on L2
  int64_t grid = (int64_t)sm_count() * occ;
  const int64_t max_grid = ((int64_t)L.n * n_chunks + 7) / 8;
  if (grid > max_grid) grid = max_grid;
  if (grid < 1) grid = 1;
  cudaMemsetAsync(L.ticket, 0, sizeof(int32_t), st);
  cudaMemsetAsync(U.ticket, 0, sizeof(int32_t), st);
  trsv_chunk<true><<<(int)grid, threads, 0, st>>>(L, in_perm, b, work, width, n_chunks, epoch);
  int rc = check_launch("trsv_chunk<fwd>");
  if (rc) return rc;
  trsv_chunk<false><<<(int)grid, threads, 0, st>>>(U, out_perm, x, work, width, n_chunks, epoch);
  return check_launch("trsv_chunk<bwd>");
}

}  // namespace sgk

extern "C" int32_t sgk_trisolve_chunk_cols(void) { return sgk::CW; }

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
  const int n_chunks = (width + CW - 1) / CW;
  return launch_chunked(*L, *U, in_perm, out_perm, *b, *x, work, width, n_chunks, epoch, (cudaStream_t)stream);
}
