// K3 for wide right-hand sides — the multi-RHS triangular solves of one
// degree level (widths 36..715: LUFactors.solve, linalg.py:83-87, applied to
// all columns of a level at once, preconditioners.py:411-434).
//
// Same factors, chain groups, dense in-group inverses and sync-free ticket
// order as trsv_group (trisolve.cu), re-tiled for width:
//   * a task is (tile, 32*CPL-column chunk); lane L holds CPL consecutive
//     columns, so every solution-row load is one coalesced 256*CPL-byte read
//     and a factor entry (column, value) is fetched once per warp (coalesced
//     batch of 32, then broadcast with shuffles) instead of once per
//     1..4-column chunk;
//   * a group's outside entries are cut into SEGMENTS of <= 32 entries (one
//     warp, <= 4 batches of 8 loads in flight) and segments into TILES of
//     <= 32 segments / 256 entries, so a heavy group (the separator rows:
//     tens of thousands of outside entries) spreads over many CTAs instead
//     of serialising the critical path on one SM;
//   * a tile's per-row partial sums go to shared memory (one-tile groups:
//     finalised in place) or to a `part` slot per (tile, row); the tile that
//     completes a group's counter last finalises it: P = B - sum of the
//     row's slots in tile order (fixed order: deterministic), X = inv(D+B_g) P
//     with the host-computed dense inverse, write, fence, publish the flag.
// Deadlock freedom is the ticket argument of trsv_group: tiles are ordered
// by group level, so a tile only waits for groups finalised by tiles with
// earlier tickets, which are resident or done.
#include <cstdlib>

#include "sgk_common.cuh"

namespace sgk {

constexpr int WG = 32;     // rows per group (= GMAX of trisolve.cu, linalg.GROUP_MAX)
constexpr int WSMAX = 32;  // segments per tile

template <int CPL>
__device__ __forceinline__ void ld_cpl(const double* __restrict__ p, double (&x)[CPL]) {
  if constexpr (CPL == 1) {
    x[0] = __ldcg(p);
  } else {
#pragma unroll
    for (int k = 0; k < CPL; k += 2) {
      const double2 v = __ldcg(reinterpret_cast<const double2*>(p + k));
      x[k] = v.x;
      x[k + 1] = v.y;
    }
  }
}

__device__ __forceinline__ double* wseg_ptr(const sgk_segview& s, int r, int c) {
  const int seg = r / s.seg_rows;
  const int rr = r - seg * s.seg_rows;
  double* base = seg == 0 ? s.ptr[0] : (seg == 1 ? s.ptr[1] : s.ptr[2]);
  return base + (int64_t)rr * s.ld + s.col0 + c;
}

template <bool FWD, int CPL>
__global__ void __launch_bounds__(256, 2) trsv_wide(sgk_triwide t, sgk_segview io, double* __restrict__ work,
                                                  double* __restrict__ part, int width, int ldw, int n_chunks,
                                                  int epoch) {
  constexpr int CH = 32 * CPL;
  extern __shared__ __align__(16) double wsm[];
  double (*sp)[CH] = reinterpret_cast<double (*)[CH]>(wsm);               // [WSMAX][CH] segment partials
  double (*pr)[CH] = reinterpret_cast<double (*)[CH]>(wsm + WSMAX * CH);  // [WG][CH] P rows of the group
  __shared__ double lg[WG][WG + 1];               // dense inverse of the in-group block
  __shared__ int task_s, last_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned FULL = 0xffffffffu;
  const int64_t n_tasks = (int64_t)t.n_tiles * n_chunks;
  for (;;) {
    if (tid == 0) task_s = atomicAdd(t.ticket, 1);
    __syncthreads();
    const int ticket = task_s;
    __syncthreads();
    if (ticket >= n_tasks) return;
    const int tile = ticket / n_chunks;
    const int chunk = ticket - tile * n_chunks;
    const int c0 = chunk * CH;
    const int gi = __ldg(t.tile_group + tile);
    const int s0 = __ldg(t.tile_seg + tile), s1 = __ldg(t.tile_seg + tile + 1);
    const int nt = __ldg(t.group_ntiles + gi);
    const int r0 = __ldg(t.group_ptr + gi), g = __ldg(t.group_ptr + gi + 1) - r0;

    // 0: wait for the groups this tile's entries read (relaxed polls, one fence)
    {
      const int da = __ldg(t.tile_dep_ptr + tile), db = __ldg(t.tile_dep_ptr + tile + 1);
      for (int d = da + tid; d < db; d += blockDim.x) {
        const int32_t* fl = t.flags + (int64_t)__ldg(t.tile_dep + d) * n_chunks + chunk;
        while (ld_relaxed(fl) != epoch) __nanosleep(64);
      }
      fence_acq_rel();
    }
    __syncthreads();

    // 1: segment partial sums, warps over segments, lanes over columns
    for (int s = s0 + warp; s < s1; s += 8) {
      const int e0 = __ldg(t.seg_e0 + s), e1 = __ldg(t.seg_e1 + s);
      double acc[CPL];
#pragma unroll
      for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
      // padding entries re-read the segment's first entry (a finished
      // dependency: final, finite) with weight 0
      const int e = e0 + lane;
      const int cj = __ldg(t.colind + (e < e1 ? e : e0));
      const double vj = e < e1 ? __ldg(t.vals + e) : 0.0;
      const int cnt = e1 - e0;
      for (int j = 0; j < cnt; j += 8) {
        double xv[8][CPL];
        double vv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int c = __shfl_sync(FULL, cj, j + u);
          vv[u] = __shfl_sync(FULL, vj, j + u);
          const int wr = t.reversed ? t.n - 1 - c : c;
          ld_cpl<CPL>(work + (int64_t)wr * ldw + c0 + CPL * lane, xv[u]);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int k = 0; k < CPL; ++k) acc[k] = fma(vv[u], xv[u][k], acc[k]);
      }
#pragma unroll
      for (int k = 0; k < CPL; ++k) sp[s - s0][CPL * lane + k] = acc[k];
    }
    __syncthreads();

    const int w = min(CH, width - c0);
    if (nt > 1) {
      // 2a: per (tile, row) sums in segment order -> part slots; count in
      for (int col = tid; col < CH; col += blockDim.x) {
        double a = 0.0;
        for (int s = s0; s < s1; ++s) {
          a += sp[s - s0][col];
          const int slot = __ldg(t.seg_slot + s);
          if (s + 1 == s1 || __ldg(t.seg_slot + s + 1) != slot) {
            __stcg(part + (int64_t)slot * ldw + c0 + col, a);
            a = 0.0;
          }
        }
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) last_s = atomicAdd(t.counters + (int64_t)gi * n_chunks + chunk, 1) == nt - 1;
      __syncthreads();
      if (!last_s) continue;
      __threadfence();
      // 2b: P = B - sum of the row's slots (tile order)
      for (int i = tid; i < g * CH; i += blockDim.x) {
        const int r = i / CH, col = i - r * CH;
        const int p = r0 + r;
        double b = 0.0;
        if (col < w)
          b = FWD ? *wseg_ptr(io, __ldg(t.io_row + p), c0 + col)
                  : __ldcg(work + (int64_t)__ldg(t.work_row + p) * ldw + c0 + col);
        const int qa = __ldg(t.row_slot_ptr + p), qb = __ldg(t.row_slot_ptr + p + 1);
        double sum = 0.0;
        for (int q = qa; q < qb; ++q) sum += __ldcg(part + (int64_t)__ldg(t.row_slot + q) * ldw + c0 + col);
        pr[r][col] = b - sum;
      }
    } else {
      // 2: one-tile group: P = B - segment sums of each row (segment order)
      for (int i = tid; i < g * CH; i += blockDim.x) {
        const int r = i / CH, col = i - r * CH;
        const int p = r0 + r;
        pr[r][col] = col >= w ? 0.0
                              : FWD ? *wseg_ptr(io, __ldg(t.io_row + p), c0 + col)
                                    : __ldcg(work + (int64_t)__ldg(t.work_row + p) * ldw + c0 + col);
      }
      __syncthreads();
      for (int col = tid; col < CH; col += blockDim.x)
        for (int s = s0; s < s1; ++s) pr[__ldg(t.seg_row + s) - r0][col] -= sp[s - s0][col];
    }
    {
      const int64_t mo = __ldg(t.minv_ptr + gi);
      for (int i = tid; i < g * g; i += blockDim.x) {
        const int r = i / g, k = i - r * g;
        lg[r][k] = __ldg(t.minv + mo + i);
      }
    }
    __syncthreads();

    // 3: X = inv(D + B_g) P (lower triangular), rows over warps; write,
    //    fence, publish
    for (int r = warp; r < g; r += 8) {
      double acc[CPL];
#pragma unroll
      for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
      for (int j = 0; j <= r; ++j) {
        const double m = lg[r][j];
#pragma unroll
        for (int k = 0; k < CPL; ++k) acc[k] = fma(m, pr[j][CPL * lane + k], acc[k]);
      }
      const int p = r0 + r;
      double* wrow = work + (int64_t)__ldg(t.work_row + p) * ldw + c0 + CPL * lane;
#pragma unroll
      for (int k = 0; k < CPL; ++k) {
        const int col = CPL * lane + k;
        __stcg(wrow + k, col < w ? acc[k] : 0.0);
        if (!FWD && col < w) *wseg_ptr(io, __ldg(t.io_row + p), c0 + col) = acc[k];
      }
    }
    fence_acq_rel();
    __syncthreads();
    if (tid == 0) st_relaxed(t.flags + (int64_t)gi * n_chunks + chunk, epoch);
  }
}

template <int CPL>
static int launch_wide_t(const sgk_triwide& L, const sgk_triwide& U, const sgk_segview& b, const sgk_segview& x,
                         double* work, double* part, int width, int epoch, cudaStream_t st) {
  constexpr int CH = 32 * CPL;
  const int n_chunks = (width + CH - 1) / CH;
  const int ldw = n_chunks * CH;
  const size_t dyn = sizeof(double) * (size_t)(WSMAX + WG) * CH;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(trsv_wide<true, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    cudaFuncSetAttribute(trsv_wide<false, CPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    cudaGetLastError();
    attr_set = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, trsv_wide<true, CPL>, 256, dyn);
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)sm_count() * occ;
  const int64_t tasks = (int64_t)std::max(L.n_tiles, U.n_tiles) * n_chunks;
  if (grid > tasks) grid = tasks;
  if (grid < 1) grid = 1;
  cudaMemsetAsync(L.ticket, 0, sizeof(int32_t), st);
  cudaMemsetAsync(U.ticket, 0, sizeof(int32_t), st);
  cudaMemsetAsync(L.counters, 0, sizeof(int32_t) * (size_t)L.n_groups * n_chunks, st);
  cudaMemsetAsync(U.counters, 0, sizeof(int32_t) * (size_t)U.n_groups * n_chunks, st);
  trsv_wide<true, CPL><<<(int)grid, 256, dyn, st>>>(L, b, work, part, width, ldw, n_chunks, epoch);
  int rc = check_launch("trsv_wide<fwd>");
  if (rc) return rc;
  trsv_wide<false, CPL><<<(int)grid, 256, dyn, st>>>(U, x, work, part, width, ldw, n_chunks, epoch);
  return check_launch("trsv_wide<bwd>");
}

}  // namespace sgk

extern "C" int32_t sgk_trisolve_wide_chunk_cols(int32_t width) { return width > 64 ? 128 : (width > 32 ? 64 : 32); }

extern "C" int sgk_trisolve_wide(const sgk_triwide* L, const sgk_triwide* U, const sgk_segview* b,
                                 const sgk_segview* x, double* work, double* part, int32_t width, int32_t epoch,
                                 void* stream) {
  using namespace sgk;
  SGK_REQUIRE(L && U && b && x && work && part, "sgk_trisolve_wide: null argument");
  SGK_REQUIRE(L->n == U->n && L->n >= 0, "sgk_trisolve_wide: factor sizes differ");
  SGK_REQUIRE(width >= 0 && epoch > 0, "sgk_trisolve_wide: bad width/epoch");
  SGK_REQUIRE(b->seg_rows > 0 && x->seg_rows > 0, "sgk_trisolve_wide: seg_rows must be positive");
  SGK_REQUIRE(L->flags && U->flags && L->counters && U->counters && L->ticket && U->ticket,
              "sgk_trisolve_wide: flags/counters/tickets not set");
  if (L->n == 0 || width == 0) return SGK_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int ch = sgk_trisolve_wide_chunk_cols(width);
  if (ch == 128) return launch_wide_t<4>(*L, *U, *b, *x, work, part, width, epoch, st);
  if (ch == 64) return launch_wide_t<2>(*L, *U, *b, *x, work, part, width, epoch, st);
  return launch_wide_t<1>(*L, *U, *b, *x, work, part, width, epoch, st);
}
