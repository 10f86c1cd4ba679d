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
#include <algorithm>
#include <cstdlib>

#include "sgk_common.cuh"

namespace sgk {

// segment pointer by select, not by a dynamic index into the parameter array
// (that copies the view to local memory: LDL round trips on the solve's
// critical path)
__device__ __forceinline__ double* seg_ptr(const sgk_segview& s, int r, int c) {
  const int seg = r / s.seg_rows;
  const int rr = r - seg * s.seg_rows;
  double* base = seg == 0 ? s.ptr[0] : (seg == 1 ? s.ptr[1] : s.ptr[2]);
  return base + (int64_t)rr * s.ld + s.col0 + c;
}
__device__ __forceinline__ double seg_load(const sgk_segview& s, int r, int c) { return *seg_ptr(s, r, c); }
__device__ __forceinline__ void seg_store(const sgk_segview& s, int r, int c, double v) { *seg_ptr(s, r, c) = v; }

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

// ---------------------------------------------------------------------------
// Grouped (chain-supernodal) solve.  Consecutive factor rows where each row
// depends on the previous one form a group (<= 32 rows); a task is (group,
// 16-column chunk) and is run by one CTA:
//   0. wait for every dependency outside the group (flags polled relaxed in
//      batches, one acquire fence);
//   1. outside contributions of all rows of the group in parallel (warps over
//      rows, lanes over entries, all loads of a batch in flight);
//   2. the in-group chain solved by one warp from shared memory (no global
//      round trip per row — the reason for grouping: the COLAMD factors'
//      critical path is mostly such chains);
//   3. results written, fenced, group flags published.
// The triangle is given in "processing space" (rows in dependency order,
// strictly lower); the U factor is passed reversed.
constexpr int GMAX = 32;
#ifndef SGK_TRI_EPL_NARROW
#define SGK_TRI_EPL_NARROW 16  // entries per lane per batch for 1-2 column chunks
#endif
constexpr int GCW_MIN = 1;  // narrowest grouped chunk (sizes the flag array)

template <int GCW>
__device__ __forceinline__ void load_cols(const double* __restrict__ p, double (&x)[GCW]) {
  // p is GCW-aligned inside a row padded to a multiple of GCW columns
  if constexpr (GCW == 1) {
    x[0] = __ldcg(p);
  } else {
#pragma unroll
    for (int c = 0; c < GCW; c += 2) {
      const double2 v = __ldcg(reinterpret_cast<const double2*>(p + c));
      x[c] = v.x;
      x[c + 1] = v.y;
    }
  }
}

#ifdef SGK_TRI_TRACE
__device__ unsigned long long sgk_tri_trace[2][1 << 20][8];
__device__ int sgk_tri_bad[2];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRI_TR(k) do { if (tid == 0 && ticket < (1 << 20)) sgk_tri_trace[FWD ? 0 : 1][ticket][k] = gtimer(); } while (0)
#else
#define TRI_TR(k) do {} while (0)
#endif

template <bool FWD, int GCW, int GEPL>
__global__ void __launch_bounds__(512, 2) trsv_group(sgk_trigroups t, sgk_segview io, double* __restrict__ work,
                                                  int width, int ldw, int n_chunks, int epoch) {
  __shared__ double part[GMAX][GCW];
  __shared__ double ys[GMAX][GCW];
  __shared__ double lg[GMAX][GMAX + 1];  // dense inverse of the in-group block
  __shared__ int task_s;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const unsigned FULL = 0xffffffffu;
  const int64_t n_tasks = (int64_t)t.n_groups * n_chunks;
  for (;;) {
    if (tid == 0) task_s = atomicAdd(t.ticket, 1);
    __syncthreads();
    const int ticket = task_s;
    __syncthreads();
    if (ticket >= n_tasks) return;
    TRI_TR(0);
    const int gi = __ldg(t.group_order + ticket / n_chunks);
    const int chunk = ticket - (ticket / n_chunks) * n_chunks;
    const int r0 = __ldg(t.group_ptr + gi), r1 = __ldg(t.group_ptr + gi + 1);
    const int g = r1 - r0;
    const int c0 = chunk * GCW;
    const int w = min(GCW, width - c0);

    // static data first (it does not depend on other groups, so its latency
    // overlaps the wait): the group's dense inverse block and the right-hand
    // side rows (b for L; for U the forward pass result, final at launch)
    const int64_t mo = __ldg(t.minv_ptr + gi);
    for (int i = tid; i < g * g; i += blockDim.x) {
      const int r = i / g, k = i - r * g;
      lg[r][k] = __ldg(t.minv + mo + i);
    }
    for (int i = tid; i < g * GCW; i += blockDim.x) {
      const int r = i / GCW, c = i - r * GCW;
      const int p = r0 + r;
      part[r][c] = c >= w ? 0.0
                          : FWD ? seg_load(io, __ldg(t.io_row + p), c0 + c)
                                : __ldcg(work + (int64_t)__ldg(t.work_row + p) * ldw + c0 + c);
    }

    // 0: wait for the groups this group depends on (host-computed distinct
    //    dependency groups; one flag per (group, chunk))
    {
      const int da = __ldg(t.gdep_ptr + gi), db = __ldg(t.gdep_ptr + gi + 1);
      for (int d = da + tid; d < db; d += blockDim.x) {
        const int32_t* fl = t.flags + (int64_t)__ldg(t.gdep + d) * n_chunks + chunk;
        while (ld_relaxed(fl) != epoch) __nanosleep(64);
      }
      fence_acq_rel();
    }
    __syncthreads();
    TRI_TR(1);
#ifdef SGK_TRI_TRACE
    if (tid == 0) {
      const int da = __ldg(t.gdep_ptr + gi), db = __ldg(t.gdep_ptr + gi + 1);
      int bad = 0;
      for (int d = da; d < db; ++d)
        bad += ld_relaxed(t.flags + (int64_t)__ldg(t.gdep + d) * n_chunks + chunk) != epoch;
      if (bad) atomicAdd(&sgk_tri_bad[FWD ? 0 : 1], 1);
    }
#endif

    // 1: outside contributions, rows over warps, lanes over entries
    for (int r = warp; r < g; r += nwarps) {
      const int p = r0 + r;
      const int e0 = __ldg(t.rowptr + p);
      const int e1 = __ldg(t.split + p);  // first in-group entry (host-computed)
      double acc[GCW];
#pragma unroll
      for (int c = 0; c < GCW; ++c) acc[c] = 0.0;
      for (int base = e0; base < e1; base += 32 * GEPL) {
        int cj[GEPL];
        double vj[GEPL];
#pragma unroll
        for (int u = 0; u < GEPL; ++u) {
          const int e = base + lane + 32 * u;
          // past the end: re-read the last outside entry (a finished
          // dependency, so its value is final and finite) with weight 0
          const int ec = min(e, e1 - 1);
          cj[u] = __ldg(t.colind + ec);
          vj[u] = e < e1 ? __ldg(t.vals + ec) : 0.0;
        }
        double xv[GEPL][GCW];
#pragma unroll
        for (int u = 0; u < GEPL; ++u) {
          const int wr = t.reversed ? t.n - 1 - cj[u] : cj[u];
          load_cols<GCW>(work + (int64_t)wr * ldw + c0, xv[u]);
        }
#pragma unroll
        for (int u = 0; u < GEPL; ++u)
#pragma unroll
          for (int c = 0; c < GCW; ++c) acc[c] = fma(-vj[u], xv[u][c], acc[c]);
      }
#pragma unroll
      for (int c = 0; c < GCW; ++c) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(FULL, acc[c], o);
      }
      if (lane < w) {
        double s = acc[0];
#pragma unroll
        for (int c = 1; c < GCW; ++c)
          if (lane == c) s = acc[c];
        part[r][lane] += s;
      }
    }

    // 1b: dense region block: stream the earlier region blocks as they finish
    //     (lane k polls block j+k; every ready prefix is consumed at once), a
    //     warp per row, lanes over the 32 columns of a block; the per-lane
    //     partial sums are reduced once at the end
    if ((unsigned)(gi - t.dense_g0) < (unsigned)t.dense_nb) {
      const int bi = gi - t.dense_g0;
      const int ldd = GMAX * bi;
      const double* D = t.dense + (int64_t)GMAX * GMAX * bi * (bi - 1) / 2;
      constexpr int RPW = 2;  // rows per warp and pass (one pass with 16 warps)
      for (int rb = 0; rb < g; rb += RPW * nwarps) {
        double dacc[RPW][GCW];
#pragma unroll
        for (int q = 0; q < RPW; ++q)
#pragma unroll
          for (int c = 0; c < GCW; ++c) dacc[q][c] = 0.0;
        int j = 0;
        while (j < bi) {
          const bool mine = lane < bi - j;
          const int v = mine ? ld_relaxed(t.flags + (int64_t)(t.dense_g0 + j + lane) * n_chunks + chunk) : epoch;
          const unsigned notready = __ballot_sync(FULL, v != epoch);
          const int ready = notready ? __ffs(notready) - 1 : min(32, bi - j);
          if (ready == 0) {
            __nanosleep(64);
            continue;
          }
          fence_acq_rel();
          __syncwarp();
          for (int jj = j; jj < j + ready; ++jj) {
            const int src = t.dense_r0 + GMAX * jj + lane;  // processing row of this lane's column
            const int wr = t.reversed ? t.n - 1 - src : src;
            double xv[GCW];
            load_cols<GCW>(work + (int64_t)wr * ldw + c0, xv);
#pragma unroll
            for (int q = 0; q < RPW; ++q) {
              const int r = rb + warp + q * nwarps;
              if (r < g) {
                const double d = __ldg(D + (int64_t)r * ldd + GMAX * jj + lane);
#pragma unroll
                for (int c = 0; c < GCW; ++c) dacc[q][c] = fma(d, xv[c], dacc[q][c]);
              }
            }
          }
          j += ready;
        }
#pragma unroll
        for (int q = 0; q < RPW; ++q) {
          const int r = rb + warp + q * nwarps;
#pragma unroll
          for (int c = 0; c < GCW; ++c) {
            double a = dacc[q][c];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(FULL, a, o);
            if (r < g && lane == c) part[r][c] -= a;
          }
        }
      }
    }
    __syncthreads();
    TRI_TR(2);

    // 2: the in-group block, y = (D + B)^-1 part: rows over warps, lanes over
    //    the row's columns k <= r, one warp reduction per column
    for (int r = warp; r < g; r += nwarps) {
      const double m = lane <= r ? lg[r][lane] : 0.0;
#pragma unroll
      for (int c = 0; c < GCW; ++c) {
        double v = lane <= r ? m * part[lane][c] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
        if (lane == 0) ys[r][c] = v;
      }
    }
    __syncthreads();
    TRI_TR(3);

    // 3: write back (padded columns too: keeps the loads above unconditional),
    //    fence, publish the group flag for this chunk
    for (int i = tid; i < g * GCW; i += blockDim.x) {
      const int r = i / GCW, c = i - r * GCW;
      const int p = r0 + r;
      __stcg(work + (int64_t)__ldg(t.work_row + p) * ldw + c0 + c, c < w ? ys[r][c] : 0.0);
      if (!FWD && c < w) seg_store(io, __ldg(t.io_row + p), c0 + c, ys[r][c]);
    }
    fence_acq_rel();
    __syncthreads();
    if (tid == 0) st_relaxed(t.flags + (int64_t)gi * n_chunks + chunk, epoch);
    TRI_TR(4);
  }
}

template <int GCW, int GEPL>
static int launch_grouped_t(const sgk_trigroups& L, const sgk_trigroups& U, const sgk_segview& b,
                            const sgk_segview& x, double* work, int width, int epoch, int threads, int occ_cap,
                            cudaStream_t st) {
  const int n_chunks = (width + GCW - 1) / GCW;
  const int ldw = n_chunks * GCW;  // work rows padded to whole chunks
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, trsv_group<true, GCW, GEPL>, threads, 0);
  if (occ < 1) occ = 1;
  if (occ > occ_cap) occ = occ_cap;
  int64_t grid = (int64_t)sm_count() * occ;
  const int64_t tasks = (int64_t)std::max(L.n_groups, U.n_groups) * n_chunks;
  if (grid > tasks) grid = tasks;
  if (grid < 1) grid = 1;
  cudaMemsetAsync(L.ticket, 0, sizeof(int32_t), st);
  cudaMemsetAsync(U.ticket, 0, sizeof(int32_t), st);
  trsv_group<true, GCW, GEPL><<<(int)grid, threads, 0, st>>>(L, b, work, width, ldw, n_chunks, epoch);
  int rc = check_launch("trsv_group<fwd>");
  if (rc) return rc;
  trsv_group<false, GCW, GEPL><<<(int)grid, threads, 0, st>>>(U, x, work, width, ldw, n_chunks, epoch);
  return check_launch("trsv_group<bwd>");
}

static int env_int(const char* name, int dflt) {
  const char* v = getenv(name);
  return v ? atoi(v) : dflt;
}

static int launch_grouped(const sgk_trigroups& L, const sgk_trigroups& U, const sgk_segview& b,
                          const sgk_segview& x, double* work, int width, int epoch, cudaStream_t st) {
  // chunk width by RHS width (env overrides for tuning experiments)
  // measured on B200 (tools/tri_sweep.py, profiles/r01_trisolve_sweep.txt):
  // narrow chunks win up to ~40 columns, 4-column chunks above; 16 warps per
  // task, 8 for very wide blocks (more tasks in flight: cfg5 w330 31 -> 26 ms)
  int cw = env_int("SGKKT_TRI_CW", width <= 8 ? 1 : (width <= 40 ? 2 : 4));
  const int threads = env_int("SGKKT_TRI_THREADS", width > 200 ? 256 : 512);
  const int occ_cap = env_int("SGKKT_TRI_OCC", width > 200 ? 4 : 2);
  const int epl = env_int("SGKKT_TRI_EPL", 8);
  if (cw <= 1) return launch_grouped_t<1, SGK_TRI_EPL_NARROW>(L, U, b, x, work, width, epoch, threads, occ_cap, st);
  if (cw <= 2) return launch_grouped_t<2, SGK_TRI_EPL_NARROW>(L, U, b, x, work, width, epoch, threads, occ_cap, st);
  if (cw <= 4 && epl >= 16) return launch_grouped_t<4, 16>(L, U, b, x, work, width, epoch, threads, occ_cap, st);
  if (cw <= 4) return launch_grouped_t<4, 8>(L, U, b, x, work, width, epoch, threads, occ_cap, st);
  if (cw <= 8) return launch_grouped_t<8, 4>(L, U, b, x, work, width, epoch, threads, occ_cap, st);
  return launch_grouped_t<16, 2>(L, U, b, x, work, width, epoch, threads, occ_cap, st);
}

}  // namespace sgk

extern "C" int sgk_trisolve_grouped(const sgk_trigroups* L, const sgk_trigroups* U, const sgk_segview* b,
                                    const sgk_segview* x, double* work, int32_t width, int32_t epoch,
                                    void* stream) {
  using namespace sgk;
  SGK_REQUIRE(L && U && b && x && work, "sgk_trisolve_grouped: null argument");
  SGK_REQUIRE(L->n == U->n && L->n >= 0, "sgk_trisolve_grouped: factor sizes differ");
  SGK_REQUIRE(U->diag_inv != nullptr && L->diag_inv == nullptr, "sgk_trisolve_grouped: expected unit L, U with diag");
  SGK_REQUIRE(width >= 0 && epoch > 0, "sgk_trisolve_grouped: bad width/epoch");
  SGK_REQUIRE(b->seg_rows > 0 && x->seg_rows > 0, "sgk_trisolve_grouped: seg_rows must be positive");
  if (L->n == 0 || width == 0) return SGK_OK;
  return launch_grouped(*L, *U, *b, *x, work, width, epoch, (cudaStream_t)stream);
}

#ifdef SGK_TRI_TRACE
extern "C" int sgk_tri_bad_read(int* out) { return (int)cudaMemcpyFromSymbol(out, sgk::sgk_tri_bad, 2 * sizeof(int)); }
extern "C" int sgk_tri_trace_read(unsigned long long* out, int fwd, int n) {
  return (int)cudaMemcpyFromSymbol(out, sgk::sgk_tri_trace, sizeof(unsigned long long) * 8 * (size_t)n,
                                   fwd ? 0 : sizeof(unsigned long long) * 8 * (1 << 20));
}
#endif

extern "C" int32_t sgk_trisolve_chunk_cols(void) { return sgk::CW; }
extern "C" int32_t sgk_trisolve_grouped_chunk_cols(void) { return sgk::GCW_MIN; }

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
