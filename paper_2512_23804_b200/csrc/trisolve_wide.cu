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
#include <algorithm>
#include <cstdlib>

#include "sgk_common.cuh"

namespace sgk {

constexpr int WG = 32;     // rows per group (= GMAX of trisolve.cu, linalg.GROUP_MAX)
constexpr int WSMAX = 32;  // segments per tile
constexpr int WW = 16;     // warps per CTA
constexpr int WB = 16;     // entries per batch (loads in flight per warp)

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

#ifdef SGK_TRIW_TRACE
__device__ unsigned long long sgk_triw_trace[2][1 << 19][6];
__device__ __forceinline__ unsigned long long triw_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRIW_TR(k) do { if (tid == 0 && ticket < (1 << 19)) sgk_triw_trace[FWD ? 0 : 1][ticket][k] = triw_timer(); } while (0)
#else
#define TRIW_TR(k) do {} while (0)
#endif

template <bool FWD, int CPL, bool PANEL>
__global__ void __launch_bounds__(512, 1) trsv_wide(sgk_triwide t, sgk_segview io, double* __restrict__ work,
                                                  double* __restrict__ part, int width, int ldw, int n_chunks,
                                                  int epoch) {
  constexpr int CH = 32 * CPL;
  extern __shared__ __align__(16) double wsm[];
  double (*sp)[CH] = reinterpret_cast<double (*)[CH]>(wsm);               // [WSMAX][CH] segment partials
  double (*pr)[CH] = reinterpret_cast<double (*)[CH]>(wsm + WSMAX * CH);  // [WG][CH] P rows of the group
  __shared__ double lg[WG][WG + 1];               // dense-region coefficient block (dense task)
  __shared__ double mv[WG][WG + 1];               // dense inverse of the in-group block
  __shared__ int task_s;
  // the tile's segment records and the group's part-slot lists, staged once
  // per task (a dependent global load inside the per-column loops below costs
  // an L2 round trip per iteration on the critical path)
  __shared__ int s_row[WSMAX], s_e0[WSMAX], s_e1[WSMAX], s_slot[WSMAX];
  constexpr int SLOTMAX = 1024;
  __shared__ int q_ptr[WG + 1];
  __shared__ int q_slot[SLOTMAX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned FULL = 0xffffffffu;
  const int64_t n_tasks = (int64_t)t.n_tiles * n_chunks;
  for (;;) {
    if (tid == 0) task_s = atomicAdd(t.ticket, 1);
    __syncthreads();
    const int ticket = task_s;
    __syncthreads();
    if (ticket >= n_tasks) return;
    TRIW_TR(0);
#ifdef SGK_TRIW_TRACE
    if (tid == 0 && ticket < (1 << 19)) sgk_triw_trace[FWD ? 0 : 1][ticket][4] = 0;  // set by the finaliser
#endif
    const int tile = ticket / n_chunks;
    const int chunk = ticket - tile * n_chunks;
    const int c0 = chunk * CH;
    const int gi = __ldg(t.tile_group + tile);
    const int kind = __ldg(t.tile_kind + tile);
    if (kind == 1 && t.region_inv != nullptr) continue;  // the region is solved by region_gemm
    const int s0 = __ldg(t.tile_seg + tile), s1 = __ldg(t.tile_seg + tile + 1);
    const int nt = __ldg(t.group_ntiles + gi);
    const int r0 = __ldg(t.group_ptr + gi), g = __ldg(t.group_ptr + gi + 1) - r0;
    const bool dgrp = (unsigned)(gi - t.dense_g0) < (unsigned)t.dense_nb;
    const int w = min(CH, width - c0);
    // the group's dense inverse is static: tasks that always finalise load it
    // up front (its latency overlaps the dependency wait / the streaming)
    auto load_minv = [&]() {
      const int64_t mo = __ldg(t.minv_ptr + gi);
      for (int i = tid; i < g * g; i += blockDim.x) {
        const int r = i / g, k = i - r * g;
        mv[r][k] = __ldg(t.minv + mo + i);
      }
    };
    const bool minv_early = kind != 0 || (nt == 1 && !dgrp);
    if (minv_early) load_minv();

    // P rows = B - (sum of the row's part slots, tile order) - extra(r, col)
    auto p_from_slots = [&](auto extra) {
      const int qa0 = __ldg(t.row_slot_ptr + r0);
      const int nq = __ldg(t.row_slot_ptr + r0 + g) - qa0;
      const bool staged = nq <= SLOTMAX;
      if (tid <= g) q_ptr[tid] = __ldg(t.row_slot_ptr + r0 + tid) - qa0;
      if (staged)
        for (int i = tid; i < nq; i += blockDim.x) q_slot[i] = __ldg(t.row_slot + qa0 + i);
      __syncthreads();
      for (int i = tid; i < g * CH; i += blockDim.x) {
        const int r = i / CH, col = i - r * CH;
        const int p = r0 + r;
        double b = 0.0;
        if (col < w)
          b = FWD ? *wseg_ptr(io, __ldg(t.io_row + p), c0 + col)
                  : __ldcg(work + (int64_t)__ldg(t.work_row + p) * ldw + c0 + col);
        const int qa = q_ptr[r], qb = q_ptr[r + 1];
        double sum = 0.0;
        if (staged) {
          int q = qa;
          for (; q + 4 <= qb; q += 4) {  // four independent loads in flight, summed in slot order
            const double v0 = __ldcg(part + (int64_t)q_slot[q] * ldw + c0 + col);
            const double v1 = __ldcg(part + (int64_t)q_slot[q + 1] * ldw + c0 + col);
            const double v2 = __ldcg(part + (int64_t)q_slot[q + 2] * ldw + c0 + col);
            const double v3 = __ldcg(part + (int64_t)q_slot[q + 3] * ldw + c0 + col);
            sum += v0;
            sum += v1;
            sum += v2;
            sum += v3;
          }
          for (; q < qb; ++q) sum += __ldcg(part + (int64_t)q_slot[q] * ldw + c0 + col);
        } else {
          for (int q = qa; q < qb; ++q) sum += __ldcg(part + (int64_t)__ldg(t.row_slot + qa0 + q) * ldw + c0 + col);
        }
        pr[r][col] = b - sum - extra(r, col);
      }
    };

    // P rows -= sum of the row's part slots (tile order)
    auto sub_slots = [&]() {
      const int qa0 = __ldg(t.row_slot_ptr + r0);
      const int nq = __ldg(t.row_slot_ptr + r0 + g) - qa0;
      const bool staged = nq <= SLOTMAX;
      if (tid <= g) q_ptr[tid] = __ldg(t.row_slot_ptr + r0 + tid) - qa0;
      if (staged)
        for (int i = tid; i < nq; i += blockDim.x) q_slot[i] = __ldg(t.row_slot + qa0 + i);
      __syncthreads();
      for (int i = tid; i < g * CH; i += blockDim.x) {
        const int r = i / CH, col = i - r * CH;
        const int qa = q_ptr[r], qb = q_ptr[r + 1];
        double sum = 0.0;
        int q = qa;
        for (; q + 4 <= qb; q += 4) {
          const int sa = staged ? q_slot[q] : __ldg(t.row_slot + qa0 + q);
          const int sb = staged ? q_slot[q + 1] : __ldg(t.row_slot + qa0 + q + 1);
          const int sc = staged ? q_slot[q + 2] : __ldg(t.row_slot + qa0 + q + 2);
          const int sd = staged ? q_slot[q + 3] : __ldg(t.row_slot + qa0 + q + 3);
          const double v0 = __ldcg(part + (int64_t)sa * ldw + c0 + col);
          const double v1 = __ldcg(part + (int64_t)sb * ldw + c0 + col);
          const double v2 = __ldcg(part + (int64_t)sc * ldw + c0 + col);
          const double v3 = __ldcg(part + (int64_t)sd * ldw + c0 + col);
          sum += v0;
          sum += v1;
          sum += v2;
          sum += v3;
        }
        for (; q < qb; ++q)
          sum += __ldcg(part + (int64_t)(staged ? q_slot[q] : __ldg(t.row_slot + qa0 + q)) * ldw + c0 + col);
        pr[r][col] -= sum;
      }
    };
    // pr[row] -= the tile's segment sums of that row, one thread per (run of
    // one row's consecutive segments, column), segment order within a run
    auto sub_runs = [&]() {
      const int ns = s1 - s0;
      for (int it = tid; it < ns * CH; it += blockDim.x) {
        const int i0 = it / CH, col = it - i0 * CH;
        if (i0 > 0 && s_row[i0 - 1] == s_row[i0]) continue;  // not a run start
        double a = sp[i0][col];
        for (int i = i0 + 1; i < ns && s_row[i] == s_row[i0]; ++i) a += sp[i][col];
        pr[s_row[i0] - r0][col] -= a;
      }
    };
    // P rows = B (the right-hand side rows of the group; static)
    auto init_b = [&]() {
      for (int i = tid; i < g * CH; i += blockDim.x) {
        const int r = i / CH, col = i - r * CH;
        const int p = r0 + r;
        pr[r][col] = col >= w ? 0.0
                              : FWD ? *wseg_ptr(io, __ldg(t.io_row + p), c0 + col)
                                    : __ldcg(work + (int64_t)__ldg(t.work_row + p) * ldw + c0 + col);
      }
    };
    if (kind == 1) {
      // dense-region task: stream the region's earlier blocks as they are
      // published (warp 0 polls 32 block flags at a time, every ready prefix
      // is applied at once: X block and the 32x32 coefficient block staged in
      // shared memory), then wait for the group's entry tiles and finalise.
      // Warp w accumulates rows 2w, 2w+1, lanes CPL columns each.
      __shared__ int ready_s;
      const int bi = gi - t.dense_g0;
      const double* D = t.dense + (int64_t)WG * WG * bi * (bi - 1) / 2;
      const int ldd = WG * bi;
      double dacc[2][CPL];
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int k = 0; k < CPL; ++k) dacc[q][k] = 0.0;
      TRIW_TR(1);
      init_b();  // static: off the critical path (the streaming below waits anyway)
      int j = 0, d_pref = -1;
      while (j < bi) {
        if (warp == 0) {
          const int v = lane < bi - j ? ld_relaxed(t.flags + (int64_t)(t.dense_g0 + j + lane) * n_chunks + chunk) : epoch;
          const unsigned notready = __ballot_sync(FULL, v != epoch);
          if (lane == 0) ready_s = notready ? __ffs(notready) - 1 : min(32, bi - j);
        }
        __syncthreads();
        const int ready = ready_s;
        __syncthreads();
        if (ready == 0) {
          if (d_pref != j) {  // the awaited block's coefficients are static: stage them while waiting
            for (int i = tid; i < WG * WG; i += blockDim.x) {
              const int r = i / WG, k = i - r * WG;
              lg[r][k] = __ldg(D + (int64_t)r * ldd + WG * j + k);
            }
            d_pref = j;
          }
          // the critical chain of the solve runs through these blocks: the
          // task awaiting the block right before its own spins on that flag;
          // tasks further down the chain back off (fewer L2 polls from the
          // CTAs that cannot make progress anyway)
          if (warp == 0) {
            if (bi - j > 2) {
              __nanosleep(1000);
            } else {
              const int32_t* fl = t.flags + (int64_t)(t.dense_g0 + j) * n_chunks + chunk;
              for (int spin = 0; spin < 256 && ld_relaxed(fl) != epoch; ++spin) {
              }
            }
          }
          continue;
        }
        fence_acq_rel();
        if (j + ready == bi) TRIW_TR(1);  // dense task: the awaited last block detected
        for (int jj = j; jj < j + ready; ++jj) {
          for (int i = tid; i < WG * CH; i += blockDim.x) {
            const int k = i / CH, c = i - k * CH;
            const int src = t.dense_r0 + WG * jj + k;
            const int wr = t.reversed ? t.n - 1 - src : src;
            sp[k][c] = __ldcg(work + (int64_t)wr * ldw + c0 + c);
          }
          if (d_pref != jj)
            for (int i = tid; i < WG * WG; i += blockDim.x) {
              const int r = i / WG, k = i - r * WG;
              lg[r][k] = __ldg(D + (int64_t)r * ldd + WG * jj + k);
            }
          d_pref = -1;
          __syncthreads();
#pragma unroll 4
          for (int k = 0; k < WG; ++k) {
            double xk[CPL];
#pragma unroll
            for (int kk = 0; kk < CPL; ++kk) xk[kk] = sp[k][CPL * lane + kk];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const double d = lg[2 * warp + q][k];
#pragma unroll
              for (int kk = 0; kk < CPL; ++kk) dacc[q][kk] = fma(d, xk[kk], dacc[q][kk]);
            }
          }
          __syncthreads();
        }
        j += ready;
      }
      TRIW_TR(2);
      if (nt > 0) {
        if (tid == 0) {
          const int32_t* cnt = t.counters + (int64_t)gi * n_chunks + chunk;
          while (ld_relaxed(cnt) != nt) __nanosleep(32);
        }
        __syncthreads();
        fence_acq_rel();
        TRIW_TR(3);
        // region contributions into pr via shared memory (sp is free again)
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int kk = 0; kk < CPL; ++kk) sp[2 * warp + q][CPL * lane + kk] = dacc[q][kk];
        __syncthreads();
        p_from_slots([&](int r, int col) { return sp[r][col]; });
      } else {
        // no entries left of the region: P = B (prefetched) - region sum
        __syncthreads();  // init_b's writes (bi == 0 has no streaming barrier)
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int kk = 0; kk < CPL; ++kk) pr[2 * warp + q][CPL * lane + kk] -= dacc[q][kk];
      }
    } else {
      // tasks that always finalise load their group's B rows up front (static)
      const bool b_early = kind == 2 || (nt == 1 && !dgrp);
      if (b_early) init_b();
      if constexpr (PANEL) {
        // column-panel tile: per panel the 32 distinct solution rows and the
        // dense 32 x 32 coefficient block are staged in shared memory once and
        // every warp accumulates two group rows (rows 2w, 2w+1; lanes CPL
        // columns each): a solution row is read once per (group, panel)
        auto stage_vals = [&](int pi) {
          const double* pv = t.pval + (int64_t)WG * WG * pi;
          for (int i = tid; i < WG * WG; i += blockDim.x) lg[i / WG][i % WG] = __ldg(pv + i);
        };
        if (s0 < s1) stage_vals(s0);  // static: before the dependency wait
        if (warp == 0) {
          const int da = __ldg(t.tile_dep_ptr + tile), db = __ldg(t.tile_dep_ptr + tile + 1);
          for (int d = da + lane; d < db; d += 32) {
            const int32_t* fl = t.flags + (int64_t)__ldg(t.tile_dep + d) * n_chunks + chunk;
            while (ld_relaxed(fl) != epoch) __nanosleep(32);
          }
          fence_acq_rel();
        }
        __syncthreads();
        TRIW_TR(1);
        double dacc[2][CPL];
#pragma unroll
        for (int q = 0; q < 2; ++q)
#pragma unroll
          for (int k = 0; k < CPL; ++k) dacc[q][k] = 0.0;
        for (int pi = s0; pi < s1; ++pi) {
          for (int i = tid; i < WG * CH; i += blockDim.x) {
            const int k = i / CH, c = i - k * CH;
            const int src = __ldg(t.pcol + WG * pi + k);
            const int wr = t.reversed ? t.n - 1 - src : src;
            sp[k][c] = __ldcg(work + (int64_t)wr * ldw + c0 + c);
          }
          if (pi > s0) stage_vals(pi);
          __syncthreads();
#pragma unroll 4
          for (int k = 0; k < WG; ++k) {
            double xk[CPL];
#pragma unroll
            for (int kk = 0; kk < CPL; ++kk) xk[kk] = sp[k][CPL * lane + kk];
#pragma unroll
            for (int q = 0; q < 2; ++q) {
              const double d = lg[2 * warp + q][k];
#pragma unroll
              for (int kk = 0; kk < CPL; ++kk) dacc[q][kk] = fma(d, xk[kk], dacc[q][kk]);
            }
          }
          __syncthreads();
        }
        TRIW_TR(2);
        if (kind == 2 || (nt == 1 && !dgrp)) {
          // finalising tile: P = B (prefetched) - own sums (- the other tiles' slots)
#pragma unroll
          for (int q = 0; q < 2; ++q)
#pragma unroll
            for (int kk = 0; kk < CPL; ++kk) pr[2 * warp + q][CPL * lane + kk] -= dacc[q][kk];
          if (kind == 2) {
            if (tid == 0) {
              const int32_t* cnt = t.counters + (int64_t)gi * n_chunks + chunk;
              while (ld_relaxed(cnt) != nt - 1) __nanosleep(32);
            }
            __syncthreads();
            fence_acq_rel();
            TRIW_TR(3);
            sub_slots();
          }
        } else {
          // slotted tile: the sums of every group row -> part slots; count in
          const int slot0 = __ldg(t.tile_slot + tile);
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int r = 2 * warp + q;
            if (r < g) {
              double* ps = part + (int64_t)(slot0 + r) * ldw + c0 + CPL * lane;
#pragma unroll
              for (int kk = 0; kk < CPL; ++kk) __stcg(ps + kk, dacc[q][kk]);
            }
          }
          __threadfence();
          __syncthreads();
          if (tid == 0) atomicAdd(t.counters + (int64_t)gi * n_chunks + chunk, 1);
          TRIW_TR(3);
          continue;
        }
      } else {
      for (int i = tid; i < s1 - s0; i += blockDim.x) {
        s_row[i] = __ldg(t.seg_row + s0 + i);
        s_e0[i] = __ldg(t.seg_e0 + s0 + i);
        s_e1[i] = __ldg(t.seg_e1 + s0 + i);
        s_slot[i] = __ldg(t.seg_slot + s0 + i);
      }
      // the first segment's entries are static: every warp fetches its
      // (column, value) batch before the dependency wait
      int pcj = 0;
      double pvj = 0.0;
      {
        const int sf = s0 + warp;
        if (sf < s1) {
          const int e0 = __ldg(t.seg_e0 + sf), e1 = __ldg(t.seg_e1 + sf);
          const int e = e0 + lane;
          pcj = __ldg(t.colind + (e < e1 ? e : e0));
          pvj = e < e1 ? __ldg(t.vals + e) : 0.0;
        }
      }
      // 0: wait for the groups this tile's entries read (warp 0 polls, one fence)
      if (warp == 0) {
        const int da = __ldg(t.tile_dep_ptr + tile), db = __ldg(t.tile_dep_ptr + tile + 1);
        for (int d = da + lane; d < db; d += 32) {
          const int32_t* fl = t.flags + (int64_t)__ldg(t.tile_dep + d) * n_chunks + chunk;
          while (ld_relaxed(fl) != epoch) __nanosleep(32);
        }
        fence_acq_rel();
      }
      __syncthreads();
      TRIW_TR(1);

      // 1: segment partial sums, warps over segments, lanes over columns
      for (int s = s0 + warp; s < s1; s += WW) {
        const int e0 = s_e0[s - s0], e1 = s_e1[s - s0];
        double acc[CPL];
#pragma unroll
        for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
        // padding entries re-read the segment's first entry (a finished
        // dependency: final, finite) with weight 0
        const int e = e0 + lane;
        const bool first = s == s0 + warp;
        const int cj = first ? pcj : __ldg(t.colind + (e < e1 ? e : e0));
        const double vj = first ? pvj : (e < e1 ? __ldg(t.vals + e) : 0.0);
        const int cnt = e1 - e0;
        for (int jb = 0; jb < cnt; jb += WB) {
          double xv[WB][CPL];
          double vv[WB];
#pragma unroll
          for (int u = 0; u < WB; ++u) {
            const int c = __shfl_sync(FULL, cj, jb + u);
            vv[u] = __shfl_sync(FULL, vj, jb + u);
            const int wr = t.reversed ? t.n - 1 - c : c;
            ld_cpl<CPL>(work + (int64_t)wr * ldw + c0 + CPL * lane, xv[u]);
          }
#pragma unroll
          for (int u = 0; u < WB; ++u)
#pragma unroll
            for (int k = 0; k < CPL; ++k) acc[k] = fma(vv[u], xv[u][k], acc[k]);
        }
#pragma unroll
        for (int k = 0; k < CPL; ++k) sp[s - s0][CPL * lane + k] = acc[k];
      }
      __syncthreads();
      TRIW_TR(2);

      if (kind == 2) {
        // designated finaliser of a multi-tile group: own segment sums from
        // shared memory, then the other tiles' part slots once they are in
        sub_runs();
        if (tid == 0) {
          const int32_t* cnt = t.counters + (int64_t)gi * n_chunks + chunk;
          while (ld_relaxed(cnt) != nt - 1) __nanosleep(32);
        }
        __syncthreads();
        fence_acq_rel();
        TRIW_TR(3);
        sub_slots();
      } else if (nt > 1 || dgrp) {
        // 2a: per (tile, row) sums in segment order -> part slots; count in;
        // a sparse group is finalised by its designated last tile (kind 2),
        // a dense-region group by its dense task (kind 1)
        // one thread per (run of one row's consecutive segments, column):
        // the run's segment sums in order -> its slot
        const int ns = s1 - s0;
        for (int it = tid; it < ns * CH; it += blockDim.x) {
          const int i0 = it / CH, col = it - i0 * CH;
          if (i0 > 0 && s_slot[i0 - 1] == s_slot[i0]) continue;  // not a run start
          double a = sp[i0][col];
          int i = i0 + 1;
          for (; i < ns && s_slot[i] == s_slot[i0]; ++i) a += sp[i][col];
          __stcg(part + (int64_t)s_slot[i0] * ldw + c0 + col, a);
        }
        __threadfence();
        __syncthreads();
        if (tid == 0) atomicAdd(t.counters + (int64_t)gi * n_chunks + chunk, 1);
        TRIW_TR(3);
        continue;
      } else {
        // 2: one-tile group: P = B (prefetched) - segment sums of each row
        sub_runs();
      }
      }  // !PANEL
    }
    if (!minv_early) load_minv();
    __syncthreads();

    // 3: X = inv(D + B_g) P (lower triangular), rows over warps; write,
    //    fence, publish
    for (int r = warp; r < g; r += WW) {
      double acc[CPL];
#pragma unroll
      for (int k = 0; k < CPL; ++k) acc[k] = 0.0;
      for (int j = 0; j <= r; ++j) {
        const double m = mv[r][j];
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
#ifndef SGK_TRIW_ONE_FENCE
#define SGK_TRIW_ONE_FENCE 1
#endif
#if SGK_TRIW_ONE_FENCE
    // release: the barrier orders every thread's stores before thread 0's
    // gpu-scope fence (cumulativity), so one fence publishes the group
    __syncthreads();
    if (tid == 0) {
      fence_acq_rel();
      st_relaxed(t.flags + (int64_t)gi * n_chunks + chunk, epoch);
    }
#else
    fence_acq_rel();
    __syncthreads();
    if (tid == 0) st_relaxed(t.flags + (int64_t)gi * n_chunks + chunk, epoch);
#endif
    TRIW_TR(4);
    TRIW_TR(5);
  }
}

// ---------------------------------------------------------------------------
// Dense region by explicit inverse (sgk_triwide.region_inv): the region's
// triangle T (2560 / 3072 rows at config 5: the separator rows COLAMD orders
// last) is inverted once on the host, so its solve is P = B - (part slots of
// the entries left of the region), X = inv(T) P — one blocked lower-triangular
// product with no dependency chain (the streamed form runs 80-96 sequential
// 32-row block solves, ~11.7 us each).  A trailing region (L) runs after the
// sync-free kernel, a leading one (reversed U) before it and publishes the
// region groups' flags for the tiles that read them.
template <bool FWD>
__global__ void region_prep(sgk_triwide t, sgk_segview io, const double* __restrict__ work, double* __restrict__ part,
                            int width, int ldw) {
  const int64_t total = (int64_t)WG * t.dense_nb * ldw;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / ldw), col = (int)(i - (int64_t)r * ldw);
    const int p = t.dense_r0 + r;
    double v = 0.0;
    if (col < width) {
      const double b = FWD ? *wseg_ptr(io, __ldg(t.io_row + p), col)
                           : __ldcg(work + (int64_t)__ldg(t.work_row + p) * ldw + col);
      double sum = 0.0;  // the row's part slots in tile order, as the streamed finaliser sums them
      for (int q = __ldg(t.row_slot_ptr + p); q < __ldg(t.row_slot_ptr + p + 1); ++q)
        sum += __ldcg(part + (int64_t)__ldg(t.row_slot + q) * ldw + col);
      v = b - sum;
    }
    part[((int64_t)t.part_rows + r) * ldw + col] = v;
  }
}

// CTA = RT (64) region rows x CH columns, 256 threads of (64 / TY) rows x 4
// columns each; 32-wide k tiles of inv(T) and P go through shared memory, the
// next tile's global loads are issued before the current tile's products
// (register prefetch), lower-triangular: k tiles up to the row tile's last row
constexpr int RT = 64;
template <bool FWD, int CH>
__global__ void __launch_bounds__(256) region_gemm(sgk_triwide t, sgk_segview io, double* __restrict__ work,
                                                  const double* __restrict__ part, int width, int ldw, int n_chunks,
                                                  int epoch) {
  constexpr int TX = CH / 4, TY = 256 / TX, RPT = RT / TY;  // CH 64: 16 x 16 threads, 4 rows; CH 32: 8 x 32, 2 rows
  constexpr int NA = RT * WG / 256, NP = WG * CH / 2 / 256;  // prefetch registers: doubles of A, double2 of P
  __shared__ double as[RT][WG + 1];
  __shared__ __align__(16) double ps[WG][CH];
  const int tid = threadIdx.x, tx = tid % TX, ty = tid / TX;
  const int m = WG * t.dense_nb;
  const int n_rt = (m + RT - 1) / RT;
  const int bi = n_rt - 1 - blockIdx.x;  // longest products first
  const int chunk = blockIdx.y, c0 = chunk * CH;
  const int row0 = RT * bi;
  const int rows = min(RT, m - row0);
  const int n_kb = (row0 + rows + WG - 1) / WG;
  const double* pd = part + (int64_t)t.part_rows * ldw + c0;
  double acc[RPT][4];
#pragma unroll
  for (int j = 0; j < RPT; ++j)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[j][c] = 0.0;
  double ra[NA];
  double2 rp[NP];
  auto fetch = [&](int kb) {
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      const int i = tid + 256 * u, r = i / WG, k = i - r * WG;
      ra[u] = r < rows ? __ldg(t.region_inv + (int64_t)(row0 + r) * m + WG * kb + k) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < NP; ++u) {
      const int i = tid + 256 * u, k = i / (CH / 2), c = 2 * (i - k * (CH / 2));
      rp[u] = __ldcg(reinterpret_cast<const double2*>(pd + (int64_t)(WG * kb + k) * ldw + c));
    }
  };
  fetch(0);
  for (int kb = 0; kb < n_kb; ++kb) {
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      const int i = tid + 256 * u, r = i / WG, k = i - r * WG;
      as[r][k] = ra[u];
    }
#pragma unroll
    for (int u = 0; u < NP; ++u) {
      const int i = tid + 256 * u, k = i / (CH / 2), c = 2 * (i - k * (CH / 2));
      *reinterpret_cast<double2*>(&ps[k][c]) = rp[u];
    }
    __syncthreads();
    if (kb + 1 < n_kb) fetch(kb + 1);
#pragma unroll 8
    for (int k = 0; k < WG; ++k) {
      const double2 p01 = *reinterpret_cast<const double2*>(&ps[k][4 * tx]);
      const double2 p23 = *reinterpret_cast<const double2*>(&ps[k][4 * tx + 2]);
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        const double a = as[ty + TY * j][k];
        acc[j][0] = fma(a, p01.x, acc[j][0]);
        acc[j][1] = fma(a, p01.y, acc[j][1]);
        acc[j][2] = fma(a, p23.x, acc[j][2]);
        acc[j][3] = fma(a, p23.y, acc[j][3]);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < RPT; ++j) {
    const int r = ty + TY * j;
    if (r < rows) {
      const int p = t.dense_r0 + row0 + r;
      double* wrow = work + (int64_t)__ldg(t.work_row + p) * ldw + c0 + 4 * tx;
      const int iorow = __ldg(t.io_row + p);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int col = c0 + 4 * tx + c;
        __stcg(wrow + c, col < width ? acc[j][c] : 0.0);
        if (!FWD && col < width) *wseg_ptr(io, iorow, col) = acc[j][c];
      }
    }
  }
  __syncthreads();
  if (tid < RT / WG && WG * tid < rows) {  // the row tile covers RT / WG region groups
    fence_acq_rel();
    st_relaxed(t.flags + (int64_t)(t.dense_g0 + (RT / WG) * bi + tid) * n_chunks + chunk, epoch);
  }
}

template <bool FWD, int CH>
static int launch_region(const sgk_triwide& t, const sgk_segview& io, double* work, double* part, int width, int ldw,
                         int n_chunks, int epoch, cudaStream_t st) {
  if constexpr (CH > 64) {  // 128-column chunks are not dispatched (sgk_trisolve_wide_chunk_cols)
    set_error("region_gemm: chunk width above 64 columns");
    return SGK_EINVAL;
  } else {
  const int64_t total = (int64_t)WG * t.dense_nb * ldw;
  const int pgrid = (int)std::min<int64_t>((total + 255) / 256, (int64_t)sm_count() * 8);
  region_prep<FWD><<<pgrid, 256, 0, st>>>(t, io, work, part, width, ldw);
  int rc = check_launch("region_prep");
  if (rc) return rc;
  region_gemm<FWD, CH><<<dim3((WG * t.dense_nb + RT - 1) / RT, n_chunks), 256, 0, st>>>(t, io, work, part, width, ldw, n_chunks, epoch);
  return check_launch("region_gemm");
  }
}

template <int CPL, bool PANEL>
static int launch_wide_t(const sgk_triwide& L, const sgk_triwide& U, const sgk_segview& b, const sgk_segview& x,
                         double* work, double* part, int width, int epoch, cudaStream_t st) {
  constexpr int CH = 32 * CPL;
  const int n_chunks = (width + CH - 1) / CH;
  const int ldw = n_chunks * CH;
  const size_t dyn = sizeof(double) * (size_t)(WSMAX + WG) * CH;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(trsv_wide<true, CPL, PANEL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    cudaFuncSetAttribute(trsv_wide<false, CPL, PANEL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    cudaGetLastError();
    attr_set = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, trsv_wide<true, CPL, PANEL>, 32 * WW, dyn);
  if (occ < 1) occ = 1;
  int64_t grid = (int64_t)sm_count() * occ;
  const int64_t tasks = (int64_t)std::max(L.n_tiles, U.n_tiles) * n_chunks;
  if (grid > tasks) grid = tasks;
  if (grid < 1) grid = 1;
  cudaMemsetAsync(L.ticket, 0, sizeof(int32_t), st);
  cudaMemsetAsync(U.ticket, 0, sizeof(int32_t), st);
  cudaMemsetAsync(L.counters, 0, sizeof(int32_t) * (size_t)L.n_groups * n_chunks, st);
  cudaMemsetAsync(U.counters, 0, sizeof(int32_t) * (size_t)U.n_groups * n_chunks, st);
  // an inverted dense region: before the sync-free kernel when it leads the triangle, after it when it trails
  const bool l_reg = L.region_inv != nullptr && L.dense_nb > 0, u_reg = U.region_inv != nullptr && U.dense_nb > 0;
  int rc = SGK_OK;
  if (l_reg && L.dense_r0 == 0 && (rc = launch_region<true, CH>(L, b, work, part, width, ldw, n_chunks, epoch, st))) return rc;
  trsv_wide<true, CPL, PANEL><<<(int)grid, 32 * WW, dyn, st>>>(L, b, work, part, width, ldw, n_chunks, epoch);
  rc = check_launch("trsv_wide<fwd>");
  if (rc) return rc;
  if (l_reg && L.dense_r0 != 0 && (rc = launch_region<true, CH>(L, b, work, part, width, ldw, n_chunks, epoch, st))) return rc;
  if (u_reg && U.dense_r0 == 0 && (rc = launch_region<false, CH>(U, x, work, part, width, ldw, n_chunks, epoch, st))) return rc;
  trsv_wide<false, CPL, PANEL><<<(int)grid, 32 * WW, dyn, st>>>(U, x, work, part, width, ldw, n_chunks, epoch);
  rc = check_launch("trsv_wide<bwd>");
  if (rc) return rc;
  if (u_reg && U.dense_r0 != 0) return launch_region<false, CH>(U, x, work, part, width, ldw, n_chunks, epoch, st);
  return SGK_OK;
}

}  // namespace sgk

extern "C" int32_t sgk_trisolve_wide_chunk_cols(int32_t width) {
  // 32-column chunks: every entry's solution-row load is one 256-byte read,
  // and a level's group finalisations spread over width/32 CTAs; above 128
  // columns 64-column chunks halve the task count (measured, cfg5 P~)
  return width > 128 ? 64 : 32;
}

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
  const bool panel = L->pcol != nullptr;
  SGK_REQUIRE(panel == (U->pcol != nullptr), "sgk_trisolve_wide: L and U must use the same tile form");
  SGK_REQUIRE(!panel || (L->pval && U->pval && L->tile_slot && U->tile_slot), "sgk_trisolve_wide: panel arrays not set");
  if (panel) {
    if (ch == 64) return launch_wide_t<2, true>(*L, *U, *b, *x, work, part, width, epoch, st);
    return launch_wide_t<1, true>(*L, *U, *b, *x, work, part, width, epoch, st);
  }
  if (ch == 128) return launch_wide_t<4, false>(*L, *U, *b, *x, work, part, width, epoch, st);
  if (ch == 64) return launch_wide_t<2, false>(*L, *U, *b, *x, work, part, width, epoch, st);
  return launch_wide_t<1, false>(*L, *U, *b, *x, work, part, width, epoch, st);
}

#ifdef SGK_TRIW_TRACE
extern "C" int sgk_triw_trace_read(unsigned long long* out, int fwd, int n) {
  return (int)cudaMemcpyFromSymbol(out, sgk::sgk_triw_trace, sizeof(unsigned long long) * 6 * (size_t)n,
                                   fwd ? 0 : sizeof(unsigned long long) * 6 * (1 << 19));
}
#endif
