// K1/K2/K4 fast path — the coupling program on a padded 9-point stencil.
//
// Same contract as program_kernel (galerkin.cu), specialised for the Q1
// pattern every BASELINE configuration uses (<= 9 entries per row):
//   * each warp owns a group of 128 CONSECUTIVE chaos columns (lane L holds
//     columns col0+L, +32, +64, +96), so the V loads of the 9 neighbour rows
//     are 256-byte coalesced and the values stay in registers (36 doubles)
//     while every term t of the group's step list is evaluated;
//   * a step evaluates one term t for all four column slots that have any
//     active (t, l) product: the 9 coefficients of A_t's row are read as 5
//     warp-broadcast LDS.128 from the row's staged block and each feeds 4
//     DFMAs (coefficient delivery, not DFMA, limits a 1-column-per-lane
//     layout on B200: ~0.5 broadcast LDS/clk/SM vs 2 warp-DFMA/clk/SM);
//   * the sparse H_t gather reads packed (slot, coefficient-index) entries
//     that live in shared memory for the whole kernel (loaded once per CTA),
//     so per row only the U values move through shared memory.
// Rows are processed grid-stride by persistent CTAs; the row's coefficient
// block (n_slices x 10 doubles) is staged with 16-byte loads.
#include <cstdio>
#include <cstdlib>

#include "sgk_common.cuh"

namespace sgk {

#ifndef SGK_S9_KC
#define SGK_S9_KC 4
#endif
constexpr int kCols = SGK_S9_KC;       // column slots per lane
constexpr int kGroupCols = 32 * kCols;  // columns of one group (one warp)
#ifndef SGK_VLD
#define SGK_VLD __ldg
#endif
#ifndef SGK_ALT_LDC_UNROLL
#define SGK_ALT_LDC_UNROLL 2
#endif
constexpr int kAltLdcUnroll = SGK_ALT_LDC_UNROLL;  // gather unroll of stencil9_kernel's parameter-bank path

// Shared-memory map.  ubuf holds n_ubuf U slots + 32 trash slots (inactive
// (step, column-slot) pairs store there) + 32 zero slots (gather padding).
struct Smem9 {
  size_t coef, cols, ubuf, ctab, steps, groups, ccnt, coff, gent, total;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

__host__ __device__ inline Smem9 smem9_layout(int n_slices, const sgk_program9& p) {
  Smem9 s;
  size_t off = 0;
  s.ctab = off;   off = align16(off + sizeof(double) * (size_t)p.n_coef);  // first: 14-bit offsets
  s.coef = off;   off = align16(off + 2 * sizeof(double) * (size_t)n_slices * 10);  // double buffer
  s.cols = off;   off = align16(off + 2 * 16 * sizeof(int32_t));
  s.ubuf = off;   off = align16(off + sizeof(double) * ((size_t)p.n_ubuf + 64));
  s.steps = off;  off = align16(off + sizeof(int32_t) * (size_t)p.n_steps);
  s.groups = off; off = align16(off + sizeof(int32_t) * 4 * (size_t)(p.n_groups + 1));
  const size_t n_chunks = (size_t)p.n_chunks;
  s.ccnt = off;   off = align16(off + sizeof(int32_t) * n_chunks);
  s.coff = off;   off = align16(off + sizeof(int32_t) * n_chunks);
  s.gent = off;   off = align16(off + sizeof(uint32_t) * (size_t)p.n_gather);
  s.total = off;
  return s;
}

template <typename T>
__device__ __forceinline__ T sel4(T a, T b, T c, T d, int i) {
  return i == 0 ? a : (i == 1 ? b : (i == 2 ? c : d));
}

// single accumulation chain: 1 DMUL + 8 DFMA, no extra adds on the FP64 pipe
__device__ __forceinline__ double dot9(const double (&a)[10], const double (&v)[9]) {
  double u = a[0] * v[0];
#pragma unroll
  for (int j = 1; j < 9; ++j) u = fma(a[j], v[j], u);
  return u;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// Gather layout (SELL-32): output positions are permuted on the host so that
// 32 consecutive positions (a chunk, one warp) have similar entry counts;
// chunk j has ccnt[j] entries per lane stored at gent[coff[j] + e*32 + lane];
// out_col[position] maps back to (output, column) (-1 = padding lane).
#ifndef SGK_S9_MINB
#define SGK_S9_MINB 2
#endif
// BIG: 9..16 column groups, one CTA of up to 16 warps per SM so every group
// stays resident (V prefetched) instead of warps looping over two groups
template <int MAXOUT, bool RESIDENT, bool ONEOUT, bool BIG>
__global__ void __launch_bounds__(BIG ? 512 : 256, BIG ? 1 : SGK_S9_MINB) stencil9_kernel(sgk_pattern9 pat, const __grid_constant__ sgk_program9 prog, ViewSet in,
                                                          ViewSet out, ViewSet init, ScalarSet alpha,
                                                          ScalarSet beta) {
  extern __shared__ __align__(16) unsigned char sm[];
  const Smem9 L = smem9_layout(pat.n_slices, prog);
  double* coef_s = reinterpret_cast<double*>(sm + L.coef);
  int32_t* cols_s = reinterpret_cast<int32_t*>(sm + L.cols);
  double* ubuf = reinterpret_cast<double*>(sm + L.ubuf);
  double* ctab = reinterpret_cast<double*>(sm + L.ctab);
  int32_t* steps = reinterpret_cast<int32_t*>(sm + L.steps);
  int32_t* groups = reinterpret_cast<int32_t*>(sm + L.groups);
  int32_t* ccnt = reinterpret_cast<int32_t*>(sm + L.ccnt);
  int32_t* coff = reinterpret_cast<int32_t*>(sm + L.coff);
  uint32_t* gent = reinterpret_cast<uint32_t*>(sm + L.gent);

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const int n_chunks = prog.n_chunks;
  __shared__ const double* in_ptr[SGK_MAX_IO];
  __shared__ int64_t in_ld[SGK_MAX_IO];
  if (tid < SGK_MAX_IO) {
    const sgk_view& vv = pick(in, tid);
    in_ptr[tid] = vv.ptr + vv.col0;
    in_ld[tid] = vv.ld;
  }
  const int ncoef = pat.n_slices * 10;

  // program tables -> shared memory, once per CTA
  for (int i = tid; i < prog.n_coef; i += blockDim.x) ctab[i] = prog.coef_tab[i];
  for (int i = tid; i < prog.n_steps; i += blockDim.x) steps[i] = prog.step_rec[i];
  for (int i = tid; i < 4 * (prog.n_groups + 1); i += blockDim.x) groups[i] = prog.group_info[i];
  for (int i = tid; i < n_chunks; i += blockDim.x) {
    ccnt[i] = prog.gather_ptr[2 * i];
    coff[i] = prog.gather_ptr[2 * i + 1];
  }
  for (int i = tid; i < prog.n_gather; i += blockDim.x) gent[i] = prog.gather_ent[i];

  for (int i = tid; i < 64; i += blockDim.x) ubuf[prog.n_ubuf + i] = 0.0;

  int ocol[MAXOUT];
  // a chunk never spans two outputs (program.py: positions are padded to whole
  // chunks per output), so the output index of a chunk is warp-uniform: two
  // bits per chunk, found once; the multi-output epilogue then branches on it
  // and reads the views straight from the parameter bank instead of running
  // select chains per element
  uint32_t opack = 0;
#pragma unroll
  for (int r = 0; r < MAXOUT; ++r) {
    const int chunk = warp + r * nwarps;
    ocol[r] = chunk < n_chunks ? __ldg(prog.out_col + chunk * 32 + lane) : -1;
    if constexpr (!ONEOUT) opack |= (uint32_t)max(__reduce_max_sync(0xffffffffu, ocol[r] >> 24), 0) << (2 * r);
  }

  auto stage = [&](int row, int buf) {
    const double* src = pat.coef10 + (int64_t)row * ncoef;
    double* dst = coef_s + buf * ncoef;
    for (int i = tid; i < ncoef / 2; i += blockDim.x) cp_async16(dst + 2 * i, src + 2 * i);
    if (tid < 9) cp_async4(cols_s + 16 * buf + tid, pat.colind9 + (int64_t)row * 9 + tid);
  };

  __syncthreads();  // tables and input views visible
  // row-invariant gather bookkeeping of this warp's chunks in registers (as in
  // stencil9_grid_kernel) when the warp has at most four chunks
  constexpr bool kHoist = MAXOUT <= 4;
  int npair_r[kHoist ? MAXOUT : 1];
  const uint2* gp_r[kHoist ? MAXOUT : 1];
  if constexpr (kHoist) {
#pragma unroll
    for (int r = 0; r < MAXOUT; ++r) {
      const int chunk = warp + r * nwarps;
      npair_r[r] = chunk < n_chunks ? ccnt[chunk] >> 1 : 0;
      gp_r[r] = reinterpret_cast<const uint2*>(gent + (chunk < n_chunks ? coff[chunk] : 0)) + lane;
    }
  }

  // resident mode: every warp owns at most one group for the whole kernel, so
  // its 36 V values of the next row can be prefetched during the gather phase
  int rbase = 0, rq0 = 0, rq1 = 0;
  const double* rvb = nullptr;
  int64_t rld = 0;
  int rncols = kGroupCols;
  double rv[kCols][9];
  if (RESIDENT && warp < prog.n_groups) {
    for (int g = 0; g < warp; ++g) rbase += kGroupCols * (groups[4 * (g + 1) + 3] - groups[4 * g + 3]);
    const int4 gi = *reinterpret_cast<const int4*>(groups + 4 * warp);
    rq0 = gi.w;
    rq1 = groups[4 * (warp + 1) + 3];
    rvb = in_ptr[gi.x] + gi.y;
    rld = in_ld[gi.x];
    rncols = gi.z;
  }
  auto load_v = [&](int r, double (&v)[kCols][9]) {
    const int32_t* cg = pat.colind9 + (int64_t)r * 9;
    if (rncols == kGroupCols) {  // common case: immediate offsets 0/256/... bytes
      const double* b = rvb + lane;
#pragma unroll
      for (int jj = 0; jj < 9; ++jj) {
        const double* vr = b + (int64_t)__ldg(cg + jj) * rld;
#pragma unroll
        for (int c = 0; c < kCols; ++c) v[c][jj] = SGK_VLD(vr + 32 * c);
      }
    } else {
#pragma unroll
      for (int jj = 0; jj < 9; ++jj) {
        const double* vr = rvb + (int64_t)__ldg(cg + jj) * rld;
#pragma unroll
        for (int c = 0; c < kCols; ++c) v[c][jj] = SGK_VLD(vr + min(32 * c + lane, rncols - 1));
      }
    }
  };

  // Row order.  Resident mode: every CTA walks a CONTIGUOUS chunk of rows, so
  // consecutive rows of a grid line share 6 of their 9 neighbours and the V
  // registers slide (3 new loads instead of 9); all CTAs advance in step, so
  // the 3-grid-line neighbourhood each one touches is shared through L2 with
  // the CTAs working on the adjacent lines.  Otherwise grid-stride.
#ifndef SGK_S9_CONTIG
#define SGK_S9_CONTIG 0  // measured: grid-stride 1.50 ms vs contiguous 1.58 ms (+slide 1.84 ms)
#endif
#ifndef SGK_S9_SLIDE
#define SGK_S9_SLIDE 0
#endif
  int r_begin, r_end, r_step;
  if (RESIDENT && SGK_S9_CONTIG) {
    const int per = (pat.n_rows + gridDim.x - 1) / gridDim.x;
    r_begin = min(pat.n_rows, (int)blockIdx.x * per);
    r_end = min(pat.n_rows, r_begin + per);
    r_step = 1;
  } else {
    r_begin = blockIdx.x;
    r_end = pat.n_rows;
    r_step = gridDim.x;
  }
  int row = r_begin;
  if (row < r_end) stage(row, 0);
  cp_async_commit();
  if (RESIDENT && warp < prog.n_groups && row < r_end) load_v(row, rv);
  for (int it = 0; row < r_end; row += r_step, ++it) {
    const int buf = it & 1;
    const int next = row + r_step;
    if (next < r_end) stage(next, buf ^ 1);
    cp_async_commit();
    cp_async_wait1();
    __syncthreads();  // (A) this row's block visible; previous gather done with ubuf

    const double* crow = coef_s + buf * ncoef;
    const int32_t* cr = cols_s + 16 * buf;
    if constexpr (RESIDENT) {
      // one group per warp for the whole kernel: V of this row was loaded
      // during the previous row's gather phase
      if (warp < prog.n_groups) {
        double* ubq = ubuf + rbase;
        // software pipeline: the step record and the first 4 coefficients of
        // step q+1 are loaded during step q, so each step's first 16 DFMAs
        // start without waiting on shared memory
        int recn = rq0 < rq1 ? steps[rq0] : 0;
        double2 p01 = make_double2(0.0, 0.0), p23 = p01;
        if (rq0 < rq1) {
          const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (recn & 0xFFFF));
          p01 = a2[0];
          p23 = a2[1];
        }
        for (int q = rq0; q < rq1; ++q, ubq += kGroupCols) {
          const int rec = recn;
          double* ub = ubq + (lane ^ (rec >> 16));  // swizzled slot, conflict-free STS
          double a[10];
          a[0] = p01.x; a[1] = p01.y; a[2] = p23.x; a[3] = p23.y;
          {
            const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (rec & 0xFFFF));
#pragma unroll
            for (int k = 2; k < 5; ++k) {
              const double2 p = a2[k];
              a[2 * k] = p.x;
              a[2 * k + 1] = p.y;
            }
          }
          recn = steps[q + 1 < rq1 ? q + 1 : q];
          {
            const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (recn & 0xFFFF));
            p01 = a2[0];
            p23 = a2[1];
          }
          // slot (q, c, lane) = base + 128 q + 32 c + (lane ^ sw_q)
#pragma unroll
          for (int c = 0; c < kCols; ++c) ub[32 * c] = dot9(a, rv[c]);
        }
        if (next < r_end) {  // prefetch: overlaps barrier + gather
          const int32_t* cn = pat.colind9 + (int64_t)next * 9;
          int nc[9];
#pragma unroll
          for (int jj = 0; jj < 9; ++jj) nc[jj] = __ldg(cn + jj);
          const bool slide = SGK_S9_SLIDE && SGK_S9_CONTIG && nc[0] == cr[1] && nc[1] == cr[2] && nc[3] == cr[4] && nc[4] == cr[5] &&
                             nc[6] == cr[7] && nc[7] == cr[8];
          if (slide) {
            const double* b = rvb + lane;
#pragma unroll
            for (int line = 0; line < 3; ++line) {
              const double* vr = b + (int64_t)nc[3 * line + 2] * rld;
#pragma unroll
              for (int c = 0; c < kCols; ++c) {
                rv[c][3 * line] = rv[c][3 * line + 1];
                rv[c][3 * line + 1] = rv[c][3 * line + 2];
                rv[c][3 * line + 2] = __ldg(vr + (rncols == kGroupCols ? 32 * c : min(32 * c, rncols - 1 - lane)));
              }
            }
          } else {
            load_v(next, rv);
          }
        }
      }
    } else {
    int ubase = 0;  // slot base of group g: 128 slots per step, groups in order
    for (int g = 0; g < warp && g < prog.n_groups; ++g)
      ubase += kGroupCols * (groups[4 * (g + 1) + 3] - groups[4 * g + 3]);
    for (int g = warp; g < prog.n_groups; g += nwarps) {
      const int4 gi = *reinterpret_cast<const int4*>(groups + 4 * g);
      const int q1 = groups[4 * (g + 1) + 3];
      const double* vbase = in_ptr[gi.x] + gi.y;
      const int64_t vld = in_ld[gi.x];
      double v[kCols][9];
      if (gi.z == kGroupCols) {
        const double* base = vbase + lane;
#pragma unroll
        for (int jj = 0; jj < 9; ++jj) {
          const double* vr = base + cr[jj] * vld;
#pragma unroll
          for (int c = 0; c < kCols; ++c) v[c][jj] = SGK_VLD(vr + 32 * c);
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < 9; ++jj) {
          const double* vr = vbase + cr[jj] * vld;
#pragma unroll
          for (int c = 0; c < kCols; ++c) v[c][jj] = SGK_VLD(vr + min(32 * c + lane, gi.z - 1));
        }
      }
      double* ubq = ubuf + ubase;
      for (int q = gi.w; q < q1; ++q, ubq += kGroupCols) {
        const int rec = steps[q];
        double* ub = ubq + (lane ^ (rec >> 16));
        const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (rec & 0xFFFF));
        double a[10];
#pragma unroll
        for (int k = 0; k < 5; ++k) {
          const double2 p = a2[k];
          a[2 * k] = p.x;
          a[2 * k + 1] = p.y;
        }
#pragma unroll
        for (int c = 0; c < kCols; ++c) ub[32 * c] = dot9(a, v[c]);
      }
      // skip the slots of the groups owned by the other warps
      for (int g2 = g; g2 < g + nwarps && g2 < prog.n_groups; ++g2)
        ubase += kGroupCols * (groups[4 * (g2 + 1) + 3] - groups[4 * g2 + 3]);
    }
    }

    __syncthreads();  // (B) all U of this row in ubuf

    // gather: the warp's chunk slots (chunk = warp + r*nwarps); a chunk has
    // an even number of entry rows (host-padded with zero entries) stored as
    // per-lane pairs, so one 8-byte load fetches the entries of two rows;
    // entry = (ubuf byte offset << 14) | ctab byte offset relative to the
    // dynamic shared memory; the host orders every lane's entries so the
    // rows' U loads repeat few bank pairs per half-warp
    // single-output programs: this row's output / init rows resolved once
    // (the per-column epilogue is then one multiply-add and one store)
    double* orow = nullptr;
    const double* irow = nullptr;
    if constexpr (ONEOUT) {
      orow = out.v[0].ptr + (int64_t)row * out.v[0].ld + out.v[0].col0;
      if (init.v[0].ptr != nullptr) irow = init.v[0].ptr + (int64_t)row * init.v[0].ld + init.v[0].col0;
    }
#pragma unroll
    for (int rb = 0; rb < MAXOUT; ++rb) {
      const int chunk = warp + rb * nwarps;
      if (chunk >= n_chunks) break;
      const int npair = kHoist ? npair_r[kHoist ? rb : 0] : ccnt[chunk] >> 1;
      const uint2* gp = kHoist ? gp_r[kHoist ? rb : 0] : reinterpret_cast<const uint2*>(gent + coff[chunk]) + lane;
      double acc0 = 0.0, acc1 = 0.0;
#ifndef SGK_NO_COEF_LDC
      if (prog.n_coef <= 8) {  // coefficients from the kernel parameter bank (see stencil9_grid_kernel;
                               // config-5 KKT matvec 0.455 -> 0.434 ms)
#pragma unroll kAltLdcUnroll
        for (int e = 0; e < npair; ++e, gp += 32) {
          const uint2 w = *gp;
          acc0 = fma(prog.coef8[(w.x >> 3) & 7], *reinterpret_cast<const double*>(sm + (w.x >> 14)), acc0);
          acc1 = fma(prog.coef8[(w.y >> 3) & 7], *reinterpret_cast<const double*>(sm + (w.y >> 14)), acc1);
        }
      } else
#endif
#pragma unroll 2
      for (int e = 0; e < npair; ++e, gp += 32) {
        const uint2 w = *gp;
        acc0 = fma(*reinterpret_cast<const double*>(sm + (w.x & 0x3FFF)),
                   *reinterpret_cast<const double*>(sm + (w.x >> 14)), acc0);
        acc1 = fma(*reinterpret_cast<const double*>(sm + (w.y & 0x3FFF)),
                   *reinterpret_cast<const double*>(sm + (w.y >> 14)), acc1);
      }
      const int oc = ocol[rb];
      if (oc >= 0) {
        const double acc = acc0 + acc1;
        if constexpr (ONEOUT) {
          double y = alpha.s[0] * acc;
          if (irow != nullptr) y = fma(beta.s[0], irow[oc], y);
          orow[oc] = y;
        } else {
          // per-lane output index: select the view fields by value (a
          // reference into the parameter views with a per-lane index makes
          // the compiler copy them to local memory on every output)
          const int k = oc & 0xFFFFFF;
          auto emit = [&](const sgk_view& ov, const sgk_view& iv, double al, double be) {
            double y = al * acc;
            if (iv.ptr != nullptr) y += be * iv.ptr[(int64_t)row * iv.ld + iv.col0 + k];
            ov.ptr[(int64_t)row * ov.ld + ov.col0 + k] = y;
          };
          switch ((opack >> (2 * rb)) & 3u) {  // warp-uniform
            case 0: emit(out.v[0], init.v[0], alpha.s[0], beta.s[0]); break;
            case 1: emit(out.v[1], init.v[1], alpha.s[1], beta.s[1]); break;
            case 2: emit(out.v[2], init.v[2], alpha.s[2], beta.s[2]); break;
            default: emit(out.v[3], init.v[3], alpha.s[3], beta.s[3]); break;
          }
        }
      }
    }
  }
  cp_async_wait1();
}

// ---------------------------------------------------------------------------
// Warp-specialised variant (resident programs with <= 8 column groups, e.g.
// the config-4 matvec): warps 0..7 produce the U values of row n into U
// buffer n&1 while warps 8..15 gather row n-1 from the other buffer.  Named
// barriers replace the two block-wide barriers per row:
//   FULL[b]  (ids 1,2): producers arrive after writing buffer b, consumers sync;
//   EMPTY[b] (ids 3,4): consumers arrive after reading buffer b, producers sync
//                       before overwriting it two rows later;
//   PROD     (id 5)   : producers only (coefficient staging hand-over).
// The products of one row and the gather of the previous one overlap instead
// of alternating.  Same arithmetic as stencil9_kernel (bit-identical).
__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive_n(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

__host__ __device__ inline Smem9 smem9_ws_layout(int n_slices, const sgk_program9& p) {
  Smem9 s = smem9_layout(n_slices, p);
  const size_t extra = align16(sizeof(double) * ((size_t)p.n_ubuf + 64));  // second U buffer
  s.steps += extra;
  s.groups += extra;
  s.ccnt += extra;
  s.coff += extra;
  s.gent += extra;
  s.total += extra;
  return s;
}

// speed-of-light probes (debug builds only, results wrong): SGK_DBG_QEND
// truncates the producers' step loop, SGK_DBG_NPAIR the consumers' gather
#ifndef SGK_GATHER_UNROLL
#define SGK_GATHER_UNROLL 2
#endif
constexpr int kGatherUnroll = SGK_GATHER_UNROLL;
#ifndef SGK_DBG_QEND
#define SGK_DBG_QEND rq1
#endif
#ifndef SGK_DBG_NPAIR
#define SGK_DBG_NPAIR (ccnt[chunk] >> 1)
#endif
// trace build (-DSGK_S9_TRACE, tools/s9_trace.py): CTA 0 stamps clock64() at
// the phase boundaries of its first 256 rows (producer warps 0 and 7,
// consumer warp 8); the producers additionally wait for the V registers
// before the products so the exposed load latency shows up as its own phase
#ifdef SGK_S9_TRACE
__device__ long long sgk_s9_trace[3][256][8];
#define S9_STAMP(w, k) do { if (blockIdx.x == 0 && lane == 0 && it < 256) sgk_s9_trace[w][it][k] = clock64(); } while (0)
#else
#define S9_STAMP(w, k) do {} while (0)
#endif
template <int MAXOUT, bool ONEOUT>
__global__ void __launch_bounds__(512, 1) stencil9_ws_kernel(sgk_pattern9 pat, sgk_program9 prog, ViewSet in,
                                                            ViewSet out, ViewSet init, ScalarSet alpha,
                                                            ScalarSet beta) {
  extern __shared__ __align__(16) unsigned char sm[];
  const Smem9 L = smem9_ws_layout(pat.n_slices, prog);
  double* coef_s = reinterpret_cast<double*>(sm + L.coef);
  double* ubuf = reinterpret_cast<double*>(sm + L.ubuf);
  double* ctab = reinterpret_cast<double*>(sm + L.ctab);
  int32_t* steps = reinterpret_cast<int32_t*>(sm + L.steps);
  int32_t* groups = reinterpret_cast<int32_t*>(sm + L.groups);
  int32_t* ccnt = reinterpret_cast<int32_t*>(sm + L.ccnt);
  int32_t* coff = reinterpret_cast<int32_t*>(sm + L.coff);
  uint32_t* gent = reinterpret_cast<uint32_t*>(sm + L.gent);
  const int ustride = (int)(align16(sizeof(double) * ((size_t)prog.n_ubuf + 64)));  // bytes between U buffers

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const bool producer = warp < 8;
  const int n_chunks = prog.n_chunks;
  __shared__ const double* in_ptr[SGK_MAX_IO];
  __shared__ int64_t in_ld[SGK_MAX_IO];
  if (tid < SGK_MAX_IO) {
    const sgk_view& vv = pick(in, tid);
    in_ptr[tid] = vv.ptr + vv.col0;
    in_ld[tid] = vv.ld;
  }
  const int ncoef = pat.n_slices * 10;
  for (int i = tid; i < prog.n_coef; i += blockDim.x) ctab[i] = prog.coef_tab[i];
  for (int i = tid; i < prog.n_steps; i += blockDim.x) steps[i] = prog.step_rec[i];
  for (int i = tid; i < 4 * (prog.n_groups + 1); i += blockDim.x) groups[i] = prog.group_info[i];
  for (int i = tid; i < n_chunks; i += blockDim.x) {
    ccnt[i] = prog.gather_ptr[2 * i];
    coff[i] = prog.gather_ptr[2 * i + 1];
  }
  for (int i = tid; i < prog.n_gather; i += blockDim.x) gent[i] = prog.gather_ent[i];
  for (int i = tid; i < 64; i += blockDim.x) {
    ubuf[prog.n_ubuf + i] = 0.0;
    reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(ubuf) + ustride)[prog.n_ubuf + i] = 0.0;
  }
  __syncthreads();

  const int r_begin = blockIdx.x, r_end = pat.n_rows, r_step = gridDim.x;
  if (producer) {
    const int pt = tid;  // 0..255
    auto stage = [&](int row, int buf) {
      const double* src = pat.coef10 + (int64_t)row * ncoef;
      double* dst = coef_s + buf * ncoef;
      for (int i = pt; i < ncoef / 2; i += 256) cp_async16(dst + 2 * i, src + 2 * i);
    };
    int rbase = 0, rq0 = 0, rq1 = 0;
    const double* rvb = nullptr;
    int64_t rld = 0;
    int rncols = kGroupCols;
    double rv[kCols][9];
    const bool active = warp < prog.n_groups;
    if (active) {
      for (int g = 0; g < warp; ++g) rbase += kGroupCols * (groups[4 * (g + 1) + 3] - groups[4 * g + 3]);
      const int4 gi = *reinterpret_cast<const int4*>(groups + 4 * warp);
      rq0 = gi.w;
      rq1 = groups[4 * (warp + 1) + 3];
      rvb = in_ptr[gi.x] + gi.y;
      rld = in_ld[gi.x];
      rncols = gi.z;
    }
    auto load_v = [&](int r) {
      const int32_t* cg = pat.colind9 + (int64_t)r * 9;
      if (rncols == kGroupCols) {  // common case: immediate column offsets
        const double* b = rvb + lane;
#pragma unroll
        for (int jj = 0; jj < 9; ++jj) {
          const double* vr = b + (int64_t)__ldg(cg + jj) * rld;
#pragma unroll
          for (int c = 0; c < kCols; ++c) rv[c][jj] = SGK_VLD(vr + 32 * c);
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < 9; ++jj) {
          const double* vr = rvb + (int64_t)__ldg(cg + jj) * rld;
#pragma unroll
          for (int c = 0; c < kCols; ++c) rv[c][jj] = SGK_VLD(vr + min(32 * c + lane, rncols - 1));
        }
      }
    };
    int row = r_begin;
    if (row < r_end) stage(row, 0);
    cp_async_commit();
    if (active && row < r_end) load_v(row);
    int it = 0;
    for (; row < r_end; row += r_step, ++it) {
      const int cb = it & 1;
      const int next = row + r_step;
      const int tw = warp == 0 ? 0 : 1;
      (void)tw;
      if (warp == 0 || warp == 7) S9_STAMP(tw, 0);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      bar_sync_n(5, 256);  // this row's coefficients visible; every producer is done with row it-1
      if (warp == 0 || warp == 7) S9_STAMP(tw, 1);
      if (next < r_end) stage(next, cb ^ 1);
      cp_async_commit();
      if (it >= 2) bar_sync_n(3 + cb, 512);  // consumers are done with U buffer cb (row it-2)
      if (warp == 0 || warp == 7) S9_STAMP(tw, 2);
#ifdef SGK_S9_TRACE
      if (active) {  // consume the last-issued V loads: the scoreboard wait lands here
        const double chk = rv[kCols - 1][8] + rv[0][8] + rv[kCols - 1][0];
        if (chk == 1.2345e-300) ubuf[prog.n_ubuf] = chk;
      }
      if (warp == 0 || warp == 7) S9_STAMP(tw, 3);
#endif
      if (active) {
        const double* crow = coef_s + cb * ncoef;
        double* ubq = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(ubuf) + cb * ustride) + rbase;
        int recn = rq0 < rq1 ? steps[rq0] : 0;
        double2 p01 = make_double2(0.0, 0.0), p23 = p01;
        if (rq0 < rq1) {
          const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (recn & 0xFFFF));
          p01 = a2[0];
          p23 = a2[1];
        }
        for (int q = rq0; q < SGK_DBG_QEND; ++q, ubq += kGroupCols) {
          const int rec = recn;
          double* ub = ubq + (lane ^ (rec >> 16));
          double a[10];
          a[0] = p01.x; a[1] = p01.y; a[2] = p23.x; a[3] = p23.y;
          {
            const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (rec & 0xFFFF));
#pragma unroll
            for (int k = 2; k < 5; ++k) {
              const double2 p = a2[k];
              a[2 * k] = p.x;
              a[2 * k + 1] = p.y;
            }
          }
          recn = steps[q + 1 < rq1 ? q + 1 : q];
          {
            const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (recn & 0xFFFF));
            p01 = a2[0];
            p23 = a2[1];
          }
#pragma unroll
          for (int c = 0; c < kCols; ++c) ub[32 * c] = dot9(a, rv[c]);
        }
      }
      if (warp == 0 || warp == 7) S9_STAMP(tw, 4);
      bar_arrive_n(1 + cb, 512);  // U buffer cb holds row it
      if (active && next < r_end) load_v(next);  // prefetch: overlaps the next waits
      if (warp == 0 || warp == 7) S9_STAMP(tw, 5);
    }
    // match the consumers' last EMPTY arrivals
    for (int k = (it >= 2 ? it - 2 : 0); k < it; ++k) bar_sync_n(3 + (k & 1), 512);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    const int cw = warp - 8;
    int ocol[MAXOUT];
#pragma unroll
    for (int r = 0; r < MAXOUT; ++r) {
      const int chunk = cw + r * 8;
      ocol[r] = chunk < n_chunks ? __ldg(prog.out_col + chunk * 32 + lane) : -1;
    }
    int it = 0;
    for (int row = r_begin; row < r_end; row += r_step, ++it) {
      const int cb = it & 1;
      if (cw == 0) S9_STAMP(2, 0);
      bar_sync_n(1 + cb, 512);  // products of this row are in U buffer cb
      if (cw == 0) S9_STAMP(2, 1);
      const unsigned char* smb = sm + cb * ustride;  // U addresses of buffer cb
      double* orow = nullptr;
      const double* irow = nullptr;
      if constexpr (ONEOUT) {
        orow = out.v[0].ptr + (int64_t)row * out.v[0].ld + out.v[0].col0;
        if (init.v[0].ptr != nullptr) irow = init.v[0].ptr + (int64_t)row * init.v[0].ld + init.v[0].col0;
      }
#pragma unroll
      for (int rb = 0; rb < MAXOUT; ++rb) {
        const int chunk = cw + rb * 8;
        if (chunk >= n_chunks) break;
        const int npair = SGK_DBG_NPAIR;
        const uint2* gp = reinterpret_cast<const uint2*>(gent + coff[chunk]) + lane;
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll kGatherUnroll
        for (int e = 0; e < npair; ++e, gp += 32) {
          const uint2 w = *gp;
          acc0 = fma(*reinterpret_cast<const double*>(sm + (w.x & 0x3FFF)),
                     *reinterpret_cast<const double*>(smb + (w.x >> 14)), acc0);
          acc1 = fma(*reinterpret_cast<const double*>(sm + (w.y & 0x3FFF)),
                     *reinterpret_cast<const double*>(smb + (w.y >> 14)), acc1);
        }
        const int oc = ocol[rb];
        if (oc >= 0) {
          const double acc = acc0 + acc1;
          if constexpr (ONEOUT) {
            double y = alpha.s[0] * acc;
            if (irow != nullptr) y = fma(beta.s[0], irow[oc], y);
            orow[oc] = y;
          } else {
            const int o = oc >> 24, k = oc & 0xFFFFFF;
            const double al = sel4(alpha.s[0], alpha.s[1], alpha.s[2], alpha.s[3], o);
            const double be = sel4(beta.s[0], beta.s[1], beta.s[2], beta.s[3], o);
            const double* ip = sel4(init.v[0].ptr, init.v[1].ptr, init.v[2].ptr, init.v[3].ptr, o);
            const int64_t il = sel4(init.v[0].ld, init.v[1].ld, init.v[2].ld, init.v[3].ld, o);
            const int ic = sel4(init.v[0].col0, init.v[1].col0, init.v[2].col0, init.v[3].col0, o);
            double* op = sel4(out.v[0].ptr, out.v[1].ptr, out.v[2].ptr, out.v[3].ptr, o);
            const int64_t ol = sel4(out.v[0].ld, out.v[1].ld, out.v[2].ld, out.v[3].ld, o);
            const int occ = sel4(out.v[0].col0, out.v[1].col0, out.v[2].col0, out.v[3].col0, o);
            double y = al * acc;
            if (ip != nullptr) y += be * ip[(int64_t)row * il + ic + k];
            op[(int64_t)row * ol + occ + k] = y;
          }
        }
      }
      if (cw == 0) S9_STAMP(2, 2);
      bar_arrive_n(3 + cb, 512);  // done reading U buffer cb
    }
  }
}

// ---------------------------------------------------------------------------
// TMA / mbarrier pipeline of the warp-specialised kernel (sm_100a).  Same
// roles, tables and arithmetic as stencil9_ws_kernel (bit-identical results);
// what changes is the hand-over:
//   * a row's coefficient block and its 9 column indices arrive by two bulk
//     copies (cp.async.bulk, complete_tx on an mbarrier) into a 4-slot ring,
//     issued four rows ahead by one consumer thread — the producers no
//     longer stage coefficients themselves, so the producer-wide barrier and
//     the dependent global colind load in front of the V loads are gone;
//   * FULL/EMPTY are mbarriers (one arrival per warp): a producer warp waits
//     only for the consumers, never for the other producer warps, so the
//     warps' non-product phases (V latency, waits) overlap other warps'
//     products instead of lining up behind a named barrier;
//   * NPW = 12 (programs with 9..12 column groups, e.g. the 3-input KKT
//     matvec): 12 producer + 8 consumer warps; the 640-thread CTA starts at 96
//     registers per thread and setmaxnreg moves the producers to 128 and the
//     consumers to 48 (the CTA's register total is unchanged).
// Measured and dropped (config 4, gpurun_out/g40..g43): V registers of two
// rows (setmaxnreg 200/56; 1.088 ms), two steps = 8 DFMA chains per producer
// iteration with coefficients a pair ahead (1.145 ms), coefficient selection
// from registers in the gather (1.130 ms) against 1.070 ms for this form.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
#define SGK_STR2(x) #x
#define SGK_STR(x) SGK_STR2(x)
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
#ifdef SGK_MBAR_HINT
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
#else
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
#endif
      "@P1 bra DONE;\n"
#ifdef SGK_MBAR_SLEEP
      "nanosleep.u32 " SGK_STR(SGK_MBAR_SLEEP) ";\n"
#endif
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}" ::"r"(smem_u32(b)),
      "r"(parity)
#ifdef SGK_MBAR_HINT
      , "r"(SGK_MBAR_HINT)
#endif
      : "memory");
}
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(b))
               : "memory");
}

constexpr int kRing = 4;  // coefficient ring depth (rows in flight)
// ring slot: the row's n_slices x 10 coefficients, then a 64-byte window of
// colind9 that starts at the 16-byte boundary below the row's 9 indices
__host__ __device__ inline size_t tma_slot_bytes(int n_slices) { return align16(sizeof(double) * 10 * (size_t)n_slices) + 64; }
__host__ __device__ inline size_t smem9_tma_total(int n_slices, const sgk_program9& p) {
  return smem9_ws_layout(n_slices, p).total + kRing * tma_slot_bytes(n_slices);
}

template <int MAXOUT, bool ONEOUT, int NPW>
__global__ void __launch_bounds__((NPW + 8) * 32, 1) stencil9_tma_kernel(sgk_pattern9 pat, sgk_program9 prog, ViewSet in,
                                                             ViewSet out, ViewSet init, ScalarSet alpha,
                                                             ScalarSet beta) {
  extern __shared__ __align__(16) unsigned char sm[];
  const Smem9 L = smem9_ws_layout(pat.n_slices, prog);
  double* ubuf = reinterpret_cast<double*>(sm + L.ubuf);
  double* ctab = reinterpret_cast<double*>(sm + L.ctab);
  int32_t* steps = reinterpret_cast<int32_t*>(sm + L.steps);
  int32_t* groups = reinterpret_cast<int32_t*>(sm + L.groups);
  int32_t* ccnt = reinterpret_cast<int32_t*>(sm + L.ccnt);
  int32_t* coff = reinterpret_cast<int32_t*>(sm + L.coff);
  uint32_t* gent = reinterpret_cast<uint32_t*>(sm + L.gent);
  unsigned char* ring = sm + L.total;
  const int ustride = (int)(align16(sizeof(double) * ((size_t)prog.n_ubuf + 64)));  // bytes between U buffers
  const int ncoef = pat.n_slices * 10;
  const int coef_bytes = ncoef * (int)sizeof(double);
  const int slot_bytes = (int)tma_slot_bytes(pat.n_slices);
  constexpr bool REGS = NPW > 8;  // 640 threads start at 96 registers: producers 128, consumers 48 (12*128 + 8*48 = 20*96)
  constexpr int kIssuer = NPW * 32;  // first consumer thread: issues the bulk copies
  __shared__ __align__(8) uint64_t bar_full[2], bar_empty[2], bar_coef[kRing];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const bool producer = warp < NPW;
  const int n_chunks = prog.n_chunks;
  __shared__ const double* in_ptr[SGK_MAX_IO];
  __shared__ int64_t in_ld[SGK_MAX_IO];
  if (tid < SGK_MAX_IO) {
    const sgk_view& vv = pick(in, tid);
    in_ptr[tid] = vv.ptr + vv.col0;
    in_ld[tid] = vv.ld;
  }
  if (tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_full[b], NPW);
      mbar_init(&bar_empty[b], 8);
    }
    for (int b = 0; b < kRing; ++b) mbar_init(&bar_coef[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < prog.n_coef; i += blockDim.x) ctab[i] = prog.coef_tab[i];
  for (int i = tid; i < prog.n_steps; i += blockDim.x) steps[i] = prog.step_rec[i];
  for (int i = tid; i < 4 * (prog.n_groups + 1); i += blockDim.x) groups[i] = prog.group_info[i];
  for (int i = tid; i < n_chunks; i += blockDim.x) {
    ccnt[i] = prog.gather_ptr[2 * i];
    coff[i] = prog.gather_ptr[2 * i + 1];
  }
  for (int i = tid; i < prog.n_gather; i += blockDim.x) gent[i] = prog.gather_ent[i];
  for (int i = tid; i < 64; i += blockDim.x) {
    ubuf[prog.n_ubuf + i] = 0.0;
    reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(ubuf) + ustride)[prog.n_ubuf + i] = 0.0;
  }
  __syncthreads();

  const int r_begin = blockIdx.x, r_step = gridDim.x;
  const int n_it = r_begin < pat.n_rows ? (pat.n_rows - r_begin + r_step - 1) / r_step : 0;
  // one thread: the two bulk copies of iteration itx's row into ring slot itx % kRing
  auto issue_row = [&](int itx) {
    const int64_t row = r_begin + (int64_t)itx * r_step;
    uint64_t* bar = &bar_coef[itx & (kRing - 1)];
    unsigned char* dst = ring + (itx & (kRing - 1)) * slot_bytes;
    // 16-byte window around the row's 9 indices (a row-range launch shifts colind9 by 36-byte rows)
    const uintptr_t ci = reinterpret_cast<uintptr_t>(pat.colind9) + (uintptr_t)row * 36;
    const uintptr_t ci0 = ci & ~uintptr_t(15);
    const uintptr_t ci_end = (reinterpret_cast<uintptr_t>(pat.colind9) + (uintptr_t)pat.n_rows * 36 + 15) &
                             ~uintptr_t(15);  // allocation granularity covers the round-up
    const uint32_t ci_bytes = (uint32_t)(ci_end - ci0 < 64 ? ci_end - ci0 : 64);
    mbar_expect_tx(bar, (uint32_t)coef_bytes + ci_bytes);
    bulk_load(dst, pat.coef10 + row * ncoef, (uint32_t)coef_bytes, bar);
    bulk_load(dst + slot_bytes - 64, reinterpret_cast<const void*>(ci0), ci_bytes, bar);
  };
  if (producer) {
    if constexpr (REGS) asm volatile("setmaxnreg.inc.sync.aligned.u32 128;");
    int rbase = 0, rq0 = 0, rq1 = 0;
    const double* rvb = nullptr;
    int64_t rld = 0;
    int rncols = kGroupCols;
    const bool active = warp < prog.n_groups;
    if (active) {
      for (int g = 0; g < warp; ++g) rbase += kGroupCols * (groups[4 * (g + 1) + 3] - groups[4 * g + 3]);
      const int4 gi = *reinterpret_cast<const int4*>(groups + 4 * warp);
      rq0 = gi.w;
      rq1 = groups[4 * (warp + 1) + 3];
      rvb = in_ptr[gi.x] + gi.y;
      rld = in_ld[gi.x];
      rncols = gi.z;
    }
    // V values of iteration itx's row; the column indices come from the ring
    auto load_v = [&](int itx, double (&v)[kCols][9]) {
#ifdef SGK_P_NOV
      if (itx > 0) return;
#endif
      mbar_wait(&bar_coef[itx & (kRing - 1)], (itx >> 2) & 1);
      const int64_t row = r_begin + (int64_t)itx * r_step;
      const int32_t* cg = reinterpret_cast<const int32_t*>(ring + (itx & (kRing - 1)) * slot_bytes + slot_bytes - 64) +
                          (int)(((reinterpret_cast<uintptr_t>(pat.colind9) + (uintptr_t)row * 36) & 15) >> 2);
      if (rncols == kGroupCols) {  // common case: immediate column offsets
        const double* b = rvb + lane;
#ifndef SGK_P_VN
#define SGK_P_VN 9  // probe builds load fewer neighbour rows (sliding-window upper bound; results wrong)
#endif
#pragma unroll
        for (int jj = 0; jj < SGK_P_VN; ++jj) {
          const double* vr = b + (int64_t)cg[jj] * rld;
#pragma unroll
          for (int c = 0; c < kCols; ++c) v[c][jj] = SGK_VLD(vr + 32 * c);
        }
      } else {
#pragma unroll
        for (int jj = 0; jj < 9; ++jj) {
          const double* vr = rvb + (int64_t)cg[jj] * rld;
#pragma unroll
          for (int c = 0; c < kCols; ++c) v[c][jj] = SGK_VLD(vr + min(32 * c + lane, rncols - 1));
        }
      }
    };
    // products of iteration it from the V registers v, handed to the consumers
    auto body = [&](int it, const double (&v)[kCols][9]) {
      const int cb = it & 1;
      if (it >= 2) mbar_wait(&bar_empty[cb], ((it >> 1) & 1) ^ 1);  // consumers are done with U buffer cb (row it-2)
      if (active) {
        mbar_wait(&bar_coef[it & (kRing - 1)], (it >> 2) & 1);
        const double* crow = reinterpret_cast<const double*>(ring + (it & (kRing - 1)) * slot_bytes);
        double* ubq = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(ubuf) + cb * ustride) + rbase;
        int recn = rq0 < rq1 ? steps[rq0] : 0;
        double2 p01 = make_double2(0.0, 0.0), p23 = p01;
        if (rq0 < rq1) {
          const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (recn & 0xFFFF));
          p01 = a2[0];
          p23 = a2[1];
        }
        for (int q = rq0; q < rq1; ++q, ubq += kGroupCols) {
          const int rec = recn;
          double* ub = ubq + (lane ^ (rec >> 16));
          double a[10];
          a[0] = p01.x; a[1] = p01.y; a[2] = p23.x; a[3] = p23.y;
          {
            const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (rec & 0xFFFF));
#pragma unroll
            for (int k = 2; k < 5; ++k) {
              const double2 p = a2[k];
              a[2 * k] = p.x;
              a[2 * k + 1] = p.y;
            }
          }
          recn = steps[q + 1 < rq1 ? q + 1 : q];
          {
            const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (recn & 0xFFFF));
            p01 = a2[0];
            p23 = a2[1];
          }
#ifdef SGK_P_NOSTS
#pragma unroll
          for (int c = 0; c < kCols; ++c) {
            const double u = dot9(a, v[c]);
            if (u == 1.2345e-300) ub[32 * c] = u;
          }
#else
#pragma unroll
          for (int c = 0; c < kCols; ++c) ub[32 * c] = dot9(a, v[c]);
#endif
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_full[cb]);  // U buffer cb holds row it
    };
    double rv[kCols][9];
    if (active && n_it > 0) load_v(0, rv);
    for (int it = 0; it < n_it; ++it) {
      body(it, rv);
      if (active && it + 1 < n_it) load_v(it + 1, rv);  // prefetch: overlaps the next waits
    }
  } else {
    if constexpr (REGS) asm volatile("setmaxnreg.dec.sync.aligned.u32 48;");
    const int cw = warp - NPW;
    if (tid == kIssuer)
      for (int itx = 0; itx < kRing && itx < n_it; ++itx) issue_row(itx);
    int ocol[MAXOUT];
#pragma unroll
    for (int r = 0; r < MAXOUT; ++r) {
      const int chunk = cw + r * 8;
      ocol[r] = chunk < n_chunks ? __ldg(prog.out_col + chunk * 32 + lane) : -1;
    }
    for (int it = 0; it < n_it; ++it) {
      const int cb = it & 1;
      const int64_t row = r_begin + (int64_t)it * r_step;
      mbar_wait(&bar_full[cb], (it >> 1) & 1);  // products of this row are in U buffer cb
      // every producer is past row it: its ring slot is free for row it + kRing
      if (tid == kIssuer && it + kRing < n_it) issue_row(it + kRing);
      const unsigned char* smb = sm + cb * ustride;  // U addresses of buffer cb
      double* orow = nullptr;
      const double* irow = nullptr;
      if constexpr (ONEOUT) {
        orow = out.v[0].ptr + row * out.v[0].ld + out.v[0].col0;
        if (init.v[0].ptr != nullptr) irow = init.v[0].ptr + row * init.v[0].ld + init.v[0].col0;
      }
#pragma unroll
      for (int rb = 0; rb < MAXOUT; ++rb) {
        const int chunk = cw + rb * 8;
        if (chunk >= n_chunks) break;
        const int npair = ccnt[chunk] >> 1;
        const uint2* gp = reinterpret_cast<const uint2*>(gent + coff[chunk]) + lane;
        double acc0 = 0.0, acc1 = 0.0;
#pragma unroll kGatherUnroll
        for (int e = 0; e < npair; ++e, gp += 32) {
          const uint2 w = *gp;
#ifdef SGK_P_NOCOEF
          acc0 += *reinterpret_cast<const double*>(smb + (w.x >> 14));
          acc1 += *reinterpret_cast<const double*>(smb + (w.y >> 14));
#else
          acc0 = fma(*reinterpret_cast<const double*>(sm + (w.x & 0x3FFF)),
                     *reinterpret_cast<const double*>(smb + (w.x >> 14)), acc0);
          acc1 = fma(*reinterpret_cast<const double*>(sm + (w.y & 0x3FFF)),
                     *reinterpret_cast<const double*>(smb + (w.y >> 14)), acc1);
#endif
        }
        const int oc = ocol[rb];
        if (oc >= 0) {
          const double acc = acc0 + acc1;
          if constexpr (ONEOUT) {
            double y = alpha.s[0] * acc;
            if (irow != nullptr) y = fma(beta.s[0], irow[oc], y);
            orow[oc] = y;
          } else {
            const int o = oc >> 24, k = oc & 0xFFFFFF;
            const double al = sel4(alpha.s[0], alpha.s[1], alpha.s[2], alpha.s[3], o);
            const double be = sel4(beta.s[0], beta.s[1], beta.s[2], beta.s[3], o);
            const double* ip = sel4(init.v[0].ptr, init.v[1].ptr, init.v[2].ptr, init.v[3].ptr, o);
            const int64_t il = sel4(init.v[0].ld, init.v[1].ld, init.v[2].ld, init.v[3].ld, o);
            const int ic = sel4(init.v[0].col0, init.v[1].col0, init.v[2].col0, init.v[3].col0, o);
            double* op = sel4(out.v[0].ptr, out.v[1].ptr, out.v[2].ptr, out.v[3].ptr, o);
            const int64_t ol = sel4(out.v[0].ld, out.v[1].ld, out.v[2].ld, out.v[3].ld, o);
            const int occ = sel4(out.v[0].col0, out.v[1].col0, out.v[2].col0, out.v[3].col0, o);
            double y = al * acc;
            if (ip != nullptr) y += be * ip[row * il + ic + k];
            op[row * ol + occ + k] = y;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar_empty[cb]);  // done reading U buffer cb
    }
  }
}

// ---------------------------------------------------------------------------
// Grid variant of the warp-specialised kernel (config-4 matvec): the pattern
// is the Q1 9-point stencil of an nx x ny grid in natural order, so the
// neighbours of node p = iy*nx + ix are p + dy*nx + dx and the producers
// address V geometrically.  Every CTA walks a CONTIGUOUS range of rows, so
// consecutive rows of a grid line share 6 of their 9 neighbours: the V
// window (3 lines x 3 columns x 4 slots in registers) slides, and each row
// loads only the new column (12 doubles per lane instead of 36; no colind
// loads).  Coefficients come from coefg, the t-stacked values in stencil
// position order (dy+1)*3 + (dx+1) with zeros for missing neighbours; a
// missing neighbour's V load is redirected to the row's own node (finite
// value times a zero coefficient).  Gather and barriers as stencil9_ws_kernel.
// V staging of the grid kernel: per producer warp 3 nodes x 4 slots x 32
// lanes doubles (the next row's new window column, cp.async'ed one row ahead)
constexpr int kVStage = 8 * 3 * kCols * 32;
__host__ __device__ inline Smem9 smem9_grid_layout(int n_slices, const sgk_program9& p) {
  Smem9 s = smem9_ws_layout(n_slices, p);
  s.total = align16(s.total) + sizeof(double) * kVStage;
  return s;
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem) : "memory");
}

// TMA: the hand-over of stencil9_tma_kernel (bulk-copied coefficient ring issued by one consumer thread,
// FULL/EMPTY mbarriers with one arrival per warp) instead of cp.async staging and named barriers
// (measured and dropped: the next row's window column loaded straight into registers a product phase
// ahead, with setmaxnreg 168 / 88 — 1.441 ms against 1.043 ms, gpurun_out/g59_ab.log)
template <int MAXOUT, bool ONEOUT, int TMODE>
__global__ void __launch_bounds__(512, 1) stencil9_grid_kernel(sgk_grid9 gp, const __grid_constant__ sgk_program9 prog, ViewSet in,
                                                              ViewSet out, ViewSet init, ScalarSet alpha,
                                                              ScalarSet beta) {
  extern __shared__ __align__(16) unsigned char sm[];
  const Smem9 L = smem9_grid_layout(gp.n_slices, prog);
  double* coef_s = reinterpret_cast<double*>(sm + L.coef);
  double* ubuf = reinterpret_cast<double*>(sm + L.ubuf);
  double* ctab = reinterpret_cast<double*>(sm + L.ctab);
  int32_t* steps = reinterpret_cast<int32_t*>(sm + L.steps);
  int32_t* groups = reinterpret_cast<int32_t*>(sm + L.groups);
  int32_t* ccnt = reinterpret_cast<int32_t*>(sm + L.ccnt);
  int32_t* coff = reinterpret_cast<int32_t*>(sm + L.coff);
  uint32_t* gent = reinterpret_cast<uint32_t*>(sm + L.gent);
  const int ustride = (int)(align16(sizeof(double) * ((size_t)prog.n_ubuf + 64)));
  constexpr bool TMA = TMODE != 0;
  unsigned char* ring = sm + L.total;  // TMA: kRing slots of the row's coefficient block
  const int slot_bytes = (int)align16(sizeof(double) * 10 * (size_t)gp.n_slices);
  __shared__ __align__(8) uint64_t bar_full[2], bar_empty[2], bar_coef[kRing];

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  const bool producer = warp < 8;
  const int n_chunks = prog.n_chunks;
  __shared__ const double* in_ptr[SGK_MAX_IO];
  __shared__ int64_t in_ld[SGK_MAX_IO];
  if (tid < SGK_MAX_IO) {
    const sgk_view& vv = pick(in, tid);
    in_ptr[tid] = vv.ptr + vv.col0;
    in_ld[tid] = vv.ld;
  }
  if (TMA && tid == 0) {
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bar_full[b], 8);
      mbar_init(&bar_empty[b], 8);
    }
    for (int b = 0; b < kRing; ++b) mbar_init(&bar_coef[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int ncoef = gp.n_slices * 10;
  for (int i = tid; i < prog.n_coef; i += blockDim.x) ctab[i] = prog.coef_tab[i];
  for (int i = tid; i < prog.n_steps; i += blockDim.x) steps[i] = prog.step_rec[i];
  for (int i = tid; i < 4 * (prog.n_groups + 1); i += blockDim.x) groups[i] = prog.group_info[i];
  for (int i = tid; i < n_chunks; i += blockDim.x) {
    ccnt[i] = prog.gather_ptr[2 * i];
    coff[i] = prog.gather_ptr[2 * i + 1];
  }
  for (int i = tid; i < prog.n_gather; i += blockDim.x) gent[i] = prog.gather_ent[i];
  for (int i = tid; i < 64; i += blockDim.x) {
    ubuf[prog.n_ubuf + i] = 0.0;
    reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(ubuf) + ustride)[prog.n_ubuf + i] = 0.0;
  }
  __syncthreads();

  // Rows are walked in grid-line SEGMENTS of seg_len nodes (segment s =
  // line s / nq, part s % nq); CTA b takes segments b, b + G, ... so at any
  // time the CTAs work on vertically adjacent segments at the same x: the
  // neighbour lines a CTA reads are the lines its neighbour CTAs are
  // streaming at that moment (L2 hits), while consecutive rows of a segment
  // slide the V window.  Segments are clipped to the launch's node range.
  const int nx = gp.nx, ny = gp.ny;
  const int A = gp.row0, B = gp.row0 + gp.n_rows;
  const int SL = gp.seg_len, nq = (nx + SL - 1) / SL;
  auto seg_of = [&](int node) { const int y = node / nx; return y * nq + (node - y * nx) / SL; };
  auto seg_range = [&](int sg, int& a, int& b) {
    const int y = sg / nq, q = sg - y * nq;
    a = max(A, y * nx + q * SL);
    b = min(B, y * nx + min(nx, (q + 1) * SL));
  };
  const int s_last = gp.n_rows > 0 ? seg_of(B - 1) : -1;
  const int s_first = gp.n_rows > 0 ? seg_of(A) : 0;
  // next row after `node` of segment sg ending at nend: same segment, or the
  // first row of this CTA's next segment (restart = true), or none
  auto advance = [&](int& sg, int& node, int& nend, bool& restart) -> bool {
    ++node;
    restart = false;
    if (node < nend) return true;
    sg += gridDim.x;
    if (sg > s_last) return false;
    seg_range(sg, node, nend);
    restart = true;
    return true;
  };
  if (producer) {
    const int pt = tid;  // 0..255
    auto stage = [&](int row, int buf) {
      const double* src = gp.coefg + (int64_t)(gp.row0 + row) * ncoef;
      double* dst = coef_s + buf * ncoef;
      for (int i = pt; i < ncoef / 2; i += 256) cp_async16(dst + 2 * i, src + 2 * i);
    };
    int rbase = 0, rq0 = 0, rq1 = 0;
    const double* rvb = nullptr;
    int64_t rld = 0;
    int rncols = kGroupCols;
    double rv[kCols][9];
    const bool active = warp < prog.n_groups;
    if (active) {
      for (int g = 0; g < warp; ++g) rbase += kGroupCols * (groups[4 * (g + 1) + 3] - groups[4 * g + 3]);
      const int4 gi = *reinterpret_cast<const int4*>(groups + 4 * warp);
      rq0 = gi.w;
      rq1 = groups[4 * (warp + 1) + 3];
      rvb = in_ptr[gi.x] + gi.y;
      rld = in_ld[gi.x];
      rncols = gi.z;
    }
    // every group is a full 128-column group here (host-checked), so a
    // neighbour's 4 slot loads are immediate offsets of one base address
    const double* vlane = rvb + lane;
    auto nbase = [&](int p, bool ok, int d) -> const double* { return vlane + (int64_t)(ok ? p + d : p) * rld; };
    // window of node p: shift the columns left and load column dxn into
    // the right one.  Sliding from p-1 is one call (dxn = 1); a line start or
    // the range start is three calls (dxn = -1, 0, 1) through the SAME code
    // (a second load path made ptxas spill the window at 128 registers).
    // L2 prefetch of the window column node p will need SGK_GRID_PF rows
    // later (lines y-1..y+1 at x + 1 + SGK_GRID_PF): lane l < 24 fetches one
    // 128-byte line of the warp's 1 KB slice of one node, so the next rows'
    // first-touch V loads hit L2 instead of waiting on HBM
#ifndef SGK_GRID_PF
#define SGK_GRID_PF 2
#endif
    auto prefetch_col = [&](int p) {
      if (SGK_GRID_PF <= 0) return;
      const int iy = p / nx, ix = p - iy * nx + 1 + SGK_GRID_PF;
      const int dy = lane / 8 - 1, ln = lane & 7;
      if (lane < 24 && ix < nx && iy + dy >= 0 && iy + dy < ny) {
        const double* a = rvb + (int64_t)(p + dy * nx + 1 + SGK_GRID_PF) * rld + 16 * ln;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
      }
    };
    auto window = [&](int p, bool restart) {
      prefetch_col(p);
      const int iy = p / nx, ix = p - iy * nx;
      const bool yl = iy > 0, yh = iy + 1 < ny;
#pragma unroll 1
      for (int dxn = restart ? -1 : 1; dxn <= 1; ++dxn) {
        const bool xok = ix + dxn >= 0 && ix + dxn < nx;
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
          const bool ok = (dy < 0 ? yl : (dy > 0 ? yh : true)) && xok;
          const double* b = nbase(p, ok, dy * nx + dxn);
#pragma unroll
          for (int c = 0; c < kCols; ++c) {
            rv[c][(dy + 1) * 3 + 0] = rv[c][(dy + 1) * 3 + 1];
            rv[c][(dy + 1) * 3 + 1] = rv[c][(dy + 1) * 3 + 2];
            rv[c][(dy + 1) * 3 + 2] = SGK_VLD(b + 32 * c);
          }
        }
      }
    };
    // the new window column of (non-restart) node p, cp.async'ed into this
    // warp's staging slots: lane L copies exactly the 12 doubles it will
    // read back (node k, slot c at [(k*kCols + c)*32 + L]), so no warp sync
    // (recomputed at each use: keeping it live across the product loop
    // costs the registers the window needs)
#define SGK_VST (reinterpret_cast<double*>(sm + L.total) - kVStage + (tid >> 5) * (3 * kCols * 32) + (tid & 31))
    auto stage_v = [&](int p, int dxn) {
      double* vst = SGK_VST;
      const int iy = p / nx, ix = p - iy * nx;
      const bool yl = iy > 0, yh = iy + 1 < ny, xok = ix + dxn >= 0 && ix + dxn < nx;
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy) {
        const bool ok = (dy < 0 ? yl : (dy > 0 ? yh : true)) && xok;
        const double* b = nbase(p, ok, dy * nx + dxn);
#pragma unroll
        for (int c = 0; c < kCols; ++c) cp_async8(vst + ((dy + 1) * kCols + c) * 32, b + 32 * c);
      }
    };
    // shift reads the last loaded column: it also retires that column's LDS
    // before the staging slots are overwritten
    auto window_shift = [&]() {
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int c = 0; c < kCols; ++c) {
          rv[c][k * 3 + 0] = rv[c][k * 3 + 1];
          rv[c][k * 3 + 1] = rv[c][k * 3 + 2];
        }
    };
    auto window_load = [&]() {
      const double* vst = SGK_VST;
#pragma unroll
      for (int k = 0; k < 3; ++k)
#pragma unroll
        for (int c = 0; c < kCols; ++c) rv[c][k * 3 + 2] = vst[(k * kCols + c) * 32];
    };
    // the ONE code path that writes the window registers (two paths made
    // ptxas spill at 128 registers): a slide consumes the column staged a
    // product phase earlier; a restart stages and consumes its three columns
    // synchronously (once per grid-line segment)
    auto window_unified = [&](int p, bool restart) {
#pragma unroll 1
      for (int k = restart ? 0 : 2; k < 3; ++k) {
        window_shift();
        if (restart) {
          stage_v(p, k - 1);
          cp_async_commit();
        }
        asm volatile("cp.async.wait_group 0;" ::: "memory");
        window_load();
      }
    };
    (void)window;
    int sg = s_first + blockIdx.x, node = 0, nend = 0;
    bool have = sg <= s_last;
    if (have) seg_range(sg, node, nend);
    if (!TMA && have) stage(node - A, 0);
    cp_async_commit();
    if (active && have) window_unified(node, true);
    int it = 0;
    for (; have; ++it) {
      const int cb = it & 1;
      int sg_n = sg, node_n = node, nend_n = nend;
      bool restart_n = false;
      const bool have_n = advance(sg_n, node_n, nend_n, restart_n);
      if constexpr (TMA) {
        if (active) {
          // the window registers are in (the last staged column's LDS have returned) before the
          // staging slots are overwritten
          const double chk = rv[0][2] + rv[kCols - 1][5] + rv[kCols - 1][8];
          if (chk == 1.2345e-300) ubuf[prog.n_ubuf] = chk;
          if (have_n && !restart_n) stage_v(node_n, 1);  // a whole product phase ahead of its use
          cp_async_commit();
          mbar_wait(&bar_coef[it & (kRing - 1)], (it >> 2) & 1);
        }
        if (it >= 2) mbar_wait(&bar_empty[cb], ((it >> 1) & 1) ^ 1);  // consumers are done with U buffer cb
      } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      bar_sync_n(5, 256);  // this row's coefficients visible; every producer is done with row it-1
      if (have_n) stage(node_n - A, cb ^ 1);
      // the barrier has retired the last staged column's LDS: stage the next
      // row's column now, a whole product phase ahead of its use
      if (active && have_n && !restart_n) stage_v(node_n, 1);
      cp_async_commit();
      if (it >= 2) bar_sync_n(3 + cb, 512);  // consumers are done with U buffer cb (row it-2)
      }
      if (active) {
        const double* crow = TMA ? reinterpret_cast<const double*>(ring + (it & (kRing - 1)) * slot_bytes)
                                 : coef_s + cb * ncoef;
        double* ubq = reinterpret_cast<double*>(reinterpret_cast<unsigned char*>(ubuf) + cb * ustride) + rbase;
        int recn = rq0 < rq1 ? steps[rq0] : 0;
        double2 p01 = make_double2(0.0, 0.0), p23 = p01;
        if (rq0 < rq1) {
          const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (recn & 0xFFFF));
          p01 = a2[0];
          p23 = a2[1];
        }
        for (int q = rq0; q < SGK_DBG_QEND; ++q, ubq += kGroupCols) {
          const int rec = recn;
          double* ub = ubq + (lane ^ (rec >> 16));
          double a[10];
          a[0] = p01.x; a[1] = p01.y; a[2] = p23.x; a[3] = p23.y;
          {
            const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (rec & 0xFFFF));
#pragma unroll
            for (int k = 2; k < 5; ++k) {
              const double2 p = a2[k];
              a[2 * k] = p.x;
              a[2 * k + 1] = p.y;
            }
          }
          recn = steps[q + 1 < rq1 ? q + 1 : q];
          {
            const double2* a2 = reinterpret_cast<const double2*>(crow + 10 * (recn & 0xFFFF));
            p01 = a2[0];
            p23 = a2[1];
          }
#pragma unroll
          for (int c = 0; c < kCols; ++c) ub[32 * c] = dot9(a, rv[c]);
        }
      }
      if constexpr (TMA) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_full[cb]);
      } else {
        bar_arrive_n(1 + cb, 512);  // U buffer cb holds row it
      }
      if (active && have_n) window_unified(node_n, restart_n);  // next row's window
      sg = sg_n;
      node = node_n;
      nend = nend_n;
      have = have_n;
    }
    if constexpr (!TMA)
      for (int k = (it >= 2 ? it - 2 : 0); k < it; ++k) bar_sync_n(3 + (k & 1), 512);
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  } else {
    const int cw = warp - 8;
    // TMA: thread 256 runs kRing rows ahead of the consumers and bulk-copies each row's coefficient block
    int isg = s_first + blockIdx.x, inode = 0, inend = 0, iit = 0;
    bool ihave = TMA && tid == 256 && isg <= s_last;
    auto issue_next = [&]() {
      uint64_t* bar = &bar_coef[iit & (kRing - 1)];
      mbar_expect_tx(bar, (uint32_t)(ncoef * sizeof(double)));
      bulk_load(ring + (iit & (kRing - 1)) * slot_bytes, gp.coefg + (int64_t)inode * ncoef,
                (uint32_t)(ncoef * sizeof(double)), bar);
      ++iit;
      bool r;
      ihave = advance(isg, inode, inend, r);
    };
    if (ihave) seg_range(isg, inode, inend);
    for (int q = 0; q < kRing && ihave; ++q) issue_next();
    int ocol[MAXOUT];
    // row-invariant gather bookkeeping of this warp's chunks, kept in registers
    // (a shared-memory read per chunk and row sat in front of every entry load)
    int npair_r[MAXOUT];
    const uint2* gpe_r[MAXOUT];
#pragma unroll
    for (int r = 0; r < MAXOUT; ++r) {
      const int chunk = cw + r * 8;
      ocol[r] = chunk < n_chunks ? __ldg(prog.out_col + chunk * 32 + lane) : -1;
      npair_r[r] = chunk < n_chunks ? ccnt[chunk] >> 1 : 0;
      gpe_r[r] = reinterpret_cast<const uint2*>(gent + (chunk < n_chunks ? coff[chunk] : 0)) + lane;
    }
    // (measured and dropped: the first 1..4 entry pairs of every chunk in registers, so their U loads
    // issue with no entry load in front: 0.995 / 1.024 / 1.014 / 1.017 ms against 0.990, g63/g64_ab.log)
    int sg = s_first + blockIdx.x, node = 0, nend = 0;
    bool have = sg <= s_last;
    if (have) seg_range(sg, node, nend);
    for (int it = 0; have; ++it) {
      const int row = node - A;  // local output row
      const int cb = it & 1;
      if constexpr (TMA) {
        mbar_wait(&bar_full[cb], (it >> 1) & 1);  // products of this row are in U buffer cb
        if (ihave) issue_next();  // every producer is past row it: its ring slot is free
      } else {
        bar_sync_n(1 + cb, 512);  // products of this row are in U buffer cb
      }
      const unsigned char* smb = sm + cb * ustride;
      double* orow = nullptr;
      const double* irow = nullptr;
      if constexpr (ONEOUT) {
        orow = out.v[0].ptr + (int64_t)row * out.v[0].ld + out.v[0].col0;
        if (init.v[0].ptr != nullptr) irow = init.v[0].ptr + (int64_t)row * init.v[0].ld + init.v[0].col0;
      }
#pragma unroll
      for (int rb = 0; rb < MAXOUT; ++rb) {
        const int chunk = cw + rb * 8;
        if (chunk >= n_chunks) break;
        const int npair = npair_r[rb];
        const uint2* gpe = gpe_r[rb];
        double acc0 = 0.0, acc1 = 0.0;
#ifndef SGK_NO_COEF_LDC
        if (TMA && prog.n_coef <= 8) {
          // <= 8 distinct coefficients: read from the kernel parameter bank (constant
          // cache, its own pipe) by index instead of from shared memory (1.044 -> 1.019 ms; unrolled 4x: 1.008)
#pragma unroll 4
          for (int e = 0; e < npair; ++e, gpe += 32) {
            const uint2 w = *gpe;
            acc0 = fma(prog.coef8[(w.x >> 3) & 7], *reinterpret_cast<const double*>(smb + (w.x >> 14)), acc0);
            acc1 = fma(prog.coef8[(w.y >> 3) & 7], *reinterpret_cast<const double*>(smb + (w.y >> 14)), acc1);
          }
        } else
#endif
#pragma unroll 2
        for (int e = 0; e < npair; ++e, gpe += 32) {
          const uint2 w = *gpe;
          acc0 = fma(*reinterpret_cast<const double*>(sm + (w.x & 0x3FFF)),
                     *reinterpret_cast<const double*>(smb + (w.x >> 14)), acc0);
          acc1 = fma(*reinterpret_cast<const double*>(sm + (w.y & 0x3FFF)),
                     *reinterpret_cast<const double*>(smb + (w.y >> 14)), acc1);
        }
        const int oc = ocol[rb];
        if (oc >= 0) {
          const double acc = acc0 + acc1;
          if constexpr (ONEOUT) {
            double y = alpha.s[0] * acc;
            if (irow != nullptr) y = fma(beta.s[0], irow[oc], y);
            orow[oc] = y;
          } else {
            const int o = oc >> 24, k = oc & 0xFFFFFF;
            const double al = sel4(alpha.s[0], alpha.s[1], alpha.s[2], alpha.s[3], o);
            const double be = sel4(beta.s[0], beta.s[1], beta.s[2], beta.s[3], o);
            const double* ip = sel4(init.v[0].ptr, init.v[1].ptr, init.v[2].ptr, init.v[3].ptr, o);
            const int64_t il = sel4(init.v[0].ld, init.v[1].ld, init.v[2].ld, init.v[3].ld, o);
            const int ic = sel4(init.v[0].col0, init.v[1].col0, init.v[2].col0, init.v[3].col0, o);
            double* op = sel4(out.v[0].ptr, out.v[1].ptr, out.v[2].ptr, out.v[3].ptr, o);
            const int64_t ol = sel4(out.v[0].ld, out.v[1].ld, out.v[2].ld, out.v[3].ld, o);
            const int occ = sel4(out.v[0].col0, out.v[1].col0, out.v[2].col0, out.v[3].col0, o);
            double y = al * acc;
            if (ip != nullptr) y += be * ip[(int64_t)row * il + ic + k];
            op[(int64_t)row * ol + occ + k] = y;
          }
        }
      }
      if constexpr (TMA) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&bar_empty[cb]);
      } else {
        bar_arrive_n(3 + cb, 512);  // done reading U buffer cb
      }
      bool restart;
      have = advance(sg, node, nend, restart);
    }
  }
}

template <int MAXOUT, bool ONEOUT, int TMA>
static int launch9grid_t(const sgk_grid9& gp, const sgk_program9& prog, const ViewSet& in, const ViewSet& out,
                       const ViewSet& init, const ScalarSet& a, const ScalarSet& b, cudaStream_t st) {
  const Smem9 L = smem9_grid_layout(gp.n_slices, prog);
  const size_t total = L.total + (TMA ? kRing * align16(sizeof(double) * 10 * (size_t)gp.n_slices) : 0);
  static bool attr_set = false;
  if (!attr_set) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, stencil9_grid_kernel<MAXOUT, ONEOUT, TMA>);
    cudaFuncSetAttribute(stencil9_grid_kernel<MAXOUT, ONEOUT, TMA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         optin - (int)fa.sharedSizeBytes);
    cudaGetLastError();
    attr_set = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stencil9_grid_kernel<MAXOUT, ONEOUT, TMA>, 512, total);
  if (occ < 1) {
    set_error("stencil9_grid_kernel: program does not fit in shared memory (" + std::to_string(total) + " B)");
    return SGK_ELIMIT;
  }
  int64_t grid = (int64_t)sm_count() * occ;
  if (grid < 1) return SGK_OK;
  stencil9_grid_kernel<MAXOUT, ONEOUT, TMA><<<(int)grid, 512, total, st>>>(gp, prog, in, out, init, a, b);
  return check_launch("stencil9_grid_kernel");
}

// SGKKT_GRID_TMA=0: the named-barrier hand-over of the grid kernel (A/B)
template <int MAXOUT, bool ONEOUT>
static int launch9grid(const sgk_grid9& gp, const sgk_program9& prog, const ViewSet& in, const ViewSet& out,
                       const ViewSet& init, const ScalarSet& a, const ScalarSet& b, cudaStream_t st) {
  static const int tma_env = [] {
    const char* v = getenv("SGKKT_GRID_TMA");
    return v ? atoi(v) : 1;
  }();
  if (tma_env) {
    const int rc = launch9grid_t<MAXOUT, ONEOUT, 1>(gp, prog, in, out, init, a, b, st);
    if (rc != SGK_ELIMIT) return rc;
  }
  return launch9grid_t<MAXOUT, ONEOUT, 0>(gp, prog, in, out, init, a, b, st);
}

template <int MAXOUT, bool ONEOUT>
static int launch9ws(const sgk_pattern9& pat, const sgk_program9& prog, const ViewSet& in, const ViewSet& out,
                     const ViewSet& init, const ScalarSet& a, const ScalarSet& b, cudaStream_t st) {
  const Smem9 L = smem9_ws_layout(pat.n_slices, prog);
  static bool attr_set = false;
  if (!attr_set) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, stencil9_ws_kernel<MAXOUT, ONEOUT>);
    cudaFuncSetAttribute(stencil9_ws_kernel<MAXOUT, ONEOUT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         optin - (int)fa.sharedSizeBytes);
    cudaGetLastError();
    attr_set = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stencil9_ws_kernel<MAXOUT, ONEOUT>, 512, L.total);
  if (occ < 1) return SGK_ELIMIT;
  int64_t grid = (int64_t)sm_count() * occ;
  if (grid > pat.n_rows) grid = pat.n_rows;
  if (grid < 1) return SGK_OK;
  stencil9_ws_kernel<MAXOUT, ONEOUT><<<(int)grid, 512, L.total, st>>>(pat, prog, in, out, init, a, b);
  return check_launch("stencil9_ws_kernel");
}

template <int MAXOUT, bool ONEOUT, int NPW>
static int launch9tma(const sgk_pattern9& pat, const sgk_program9& prog, const ViewSet& in, const ViewSet& out,
                      const ViewSet& init, const ScalarSet& a, const ScalarSet& b, cudaStream_t st) {
  const size_t total = smem9_tma_total(pat.n_slices, prog);
  constexpr int threads = (NPW + 8) * 32;
  static bool attr_set = false;
  if (!attr_set) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, stencil9_tma_kernel<MAXOUT, ONEOUT, NPW>);
    cudaFuncSetAttribute(stencil9_tma_kernel<MAXOUT, ONEOUT, NPW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         optin - (int)fa.sharedSizeBytes);
    cudaGetLastError();
    attr_set = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stencil9_tma_kernel<MAXOUT, ONEOUT, NPW>, threads, total);
  if (occ < 1) return SGK_ELIMIT;
  int64_t grid = (int64_t)sm_count() * occ;
  if (grid > pat.n_rows) grid = pat.n_rows;
  if (grid < 1) return SGK_OK;
  static const bool dbg = getenv("SGKKT_S9_DEBUG") != nullptr;
  if (dbg)
    fprintf(stderr, "stencil9_tma_kernel<%d,%d,%d>: smem %zu B, grid %d, rows %d, groups %d, chunks %d\n", MAXOUT,
            (int)ONEOUT, NPW, total, (int)grid, pat.n_rows, prog.n_groups, prog.n_chunks);
  stencil9_tma_kernel<MAXOUT, ONEOUT, NPW><<<(int)grid, threads, total, st>>>(pat, prog, in, out, init, a, b);
  return check_launch("stencil9_tma_kernel");
}

// TMA/mbarrier pipeline for resident product-heavy programs: 6..8 column
// groups (8 producer warps) or 9..12 (12 producer warps); 8 consumer warps
// share the output chunks.  SGK_ELIMIT when it does not apply or fit.
template <int NPW>
static int launch9tma_any(const sgk_pattern9& pat, const sgk_program9& prog, const ViewSet& in, const ViewSet& out,
                          const ViewSet& init, const ScalarSet& a, const ScalarSet& b, int n_out, cudaStream_t st) {
  const int per = (prog.n_chunks + 7) / 8;
#define SGK_TMA_CASE(M)                                                                         \
  if (per <= M)                                                                                 \
    return n_out == 1 ? launch9tma<M, true, NPW>(pat, prog, in, out, init, a, b, st)            \
                      : launch9tma<M, false, NPW>(pat, prog, in, out, init, a, b, st);
  SGK_TMA_CASE(1)
  SGK_TMA_CASE(2)
  SGK_TMA_CASE(4)
  SGK_TMA_CASE(8)
  SGK_TMA_CASE(16)
#undef SGK_TMA_CASE
  return SGK_ELIMIT;
}

template <int MAXOUT, bool RESIDENT, bool ONEOUT, bool BIG>
static int launch9r(const sgk_pattern9& pat, const sgk_program9& prog, const ViewSet& in, const ViewSet& out,
                    const ViewSet& init, const ScalarSet& a, const ScalarSet& b, int threads, cudaStream_t st) {
  const Smem9 L = smem9_layout(pat.n_slices, prog);
  static bool attr_set = false;
  if (!attr_set) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, stencil9_kernel<MAXOUT, RESIDENT, ONEOUT, BIG>);
    cudaFuncSetAttribute(stencil9_kernel<MAXOUT, RESIDENT, ONEOUT, BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         optin - (int)fa.sharedSizeBytes);
    cudaGetLastError();  // an attribute failure must not poison the launch check
    attr_set = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, stencil9_kernel<MAXOUT, RESIDENT, ONEOUT, BIG>, threads, L.total);
  if (occ < 1) {
    set_error("stencil9_kernel: program does not fit in shared memory (" + std::to_string(L.total) + " B)");
    return SGK_ELIMIT;
  }
  int64_t grid = (int64_t)sm_count() * occ;
  if (grid > pat.n_rows) grid = pat.n_rows;
  if (grid < 1) return SGK_OK;
  stencil9_kernel<MAXOUT, RESIDENT, ONEOUT, BIG><<<(int)grid, threads, L.total, st>>>(pat, prog, in, out, init, a, b);
  return check_launch("stencil9_kernel");
}

template <int MAXOUT>
static int launch9(const sgk_pattern9& pat, const sgk_program9& prog, const ViewSet& in, const ViewSet& out,
                   const ViewSet& init, const ScalarSet& a, const ScalarSet& b, int n_out, int threads,
                   cudaStream_t st) {
  const bool res = prog.n_groups <= threads / 32;
  // warp-specialised variant for product-heavy resident programs (6..8
  // column groups: the config-4 matvec 1.34 -> 1.10 ms); programs with few
  // groups keep the alternating kernel (their producers would idle: the
  // config-5 level couplings measured 1.14 -> 1.22 ms).  SGKKT_S9_WS=0 / 1
  // forces it off / on for every resident 8-warp program.
  static const int ws_env = [] {
    const char* v = getenv("SGKKT_S9_WS");
    return v ? atoi(v) : -1;
  }();
  const bool ws = ws_env < 0 ? prog.n_groups >= 6 : ws_env != 0;
  // SGKKT_S9_TMA=0 falls back to the named-barrier / alternating kernels; 2 also sends programs with
  // 9..12 column groups (the 3-input KKT matvec) to the 12-producer form (measured 0.454 vs 0.447 ms)
  static const int tma_env = [] {
    const char* v = getenv("SGKKT_S9_TMA");
    return v ? atoi(v) : 1;
  }();
  if (tma_env && ws && res) {
    int rc = SGK_ELIMIT;
    if (threads == 256 && prog.n_groups <= 8) rc = launch9tma_any<8>(pat, prog, in, out, init, a, b, n_out, st);
    else if (tma_env >= 2 && threads > 256 && prog.n_groups > 8 && prog.n_groups <= 12)
      rc = launch9tma_any<12>(pat, prog, in, out, init, a, b, n_out, st);  // A/B only: neutral on the KKT matvec
    if (rc != SGK_ELIMIT) return rc;
  }
  if (ws && res && threads == 256 && prog.n_groups <= 8) {
    const int rc = n_out == 1 ? launch9ws<MAXOUT, true>(pat, prog, in, out, init, a, b, st)
                              : launch9ws<MAXOUT, false>(pat, prog, in, out, init, a, b, st);
    if (rc != SGK_ELIMIT) return rc;  // does not fit: the alternating kernel below
  }
  if (threads > 256) {
    if (!res) {
      set_error("stencil9_kernel: more than 16 column groups need the 256-thread kernel");
      return SGK_EINVAL;
    }
    return n_out == 1 ? launch9r<MAXOUT, true, true, true>(pat, prog, in, out, init, a, b, threads, st)
                      : launch9r<MAXOUT, true, false, true>(pat, prog, in, out, init, a, b, threads, st);
  }
  if (n_out == 1)
    return res ? launch9r<MAXOUT, true, true, false>(pat, prog, in, out, init, a, b, threads, st)
               : launch9r<MAXOUT, false, true, false>(pat, prog, in, out, init, a, b, threads, st);
  return res ? launch9r<MAXOUT, true, false, false>(pat, prog, in, out, init, a, b, threads, st)
             : launch9r<MAXOUT, false, false, false>(pat, prog, in, out, init, a, b, threads, st);
}

}  // namespace sgk

extern "C" int64_t sgk_stencil9_smem_bytes(const sgk_pattern9* pat, const sgk_program9* prog) {
  if (!pat || !prog) return -1;
  return (int64_t)sgk::smem9_layout(pat->n_slices, *prog).total;
}

extern "C" int sgk_stencil9_apply(const sgk_pattern9* pat, const sgk_program9* prog, int32_t n_in,
                                  const sgk_view* in, int32_t n_out, const sgk_view* out, const sgk_view* init,
                                  const double* alpha, const double* beta, int32_t block_threads,
                                  void* stream) {
  using namespace sgk;
  SGK_REQUIRE(pat && prog && out && alpha && beta, "sgk_stencil9_apply: null argument");
  SGK_REQUIRE(n_in >= 0 && n_in <= SGK_MAX_IO && n_out >= 1 && n_out <= SGK_MAX_IO,
              "sgk_stencil9_apply: input/output count out of range");
  SGK_REQUIRE(prog->n_groups == 0 || n_in >= 1, "sgk_stencil9_apply: program needs inputs");
  SGK_REQUIRE((int64_t)prog->n_coef * 8 <= (1 << 14), "sgk_stencil9_apply: too many distinct coefficients");
  SGK_REQUIRE(prog->n_slices == pat->n_slices, "sgk_stencil9_apply: program compiled for another slice count");
  const int threads = block_threads > 0 ? block_threads : 256;
  SGK_REQUIRE(threads % 32 == 0 && threads <= 512, "sgk_stencil9_apply: block_threads must be a multiple of 32, <=512");
  ViewSet vin{}, vout{}, vinit{};
  ScalarSet a{}, b{};
  for (int i = 0; i < n_in; ++i) vin.v[i] = in[i];
  for (int i = 0; i < n_out; ++i) {
    SGK_REQUIRE(out[i].ptr != nullptr, "sgk_stencil9_apply: null output");
    vout.v[i] = out[i];
    if (init) vinit.v[i] = init[i];
    a.s[i] = alpha[i];
    b.s[i] = beta[i];
  }
  if (pat->n_rows == 0 || prog->n_out_cols == 0) return SGK_OK;
  SGK_REQUIRE(prog->n_chunks * 32 >= prog->n_out_cols, "sgk_stencil9_apply: n_chunks too small");
  const int per = (prog->n_chunks + threads / 32 - 1) / (threads / 32);
  cudaStream_t st = (cudaStream_t)stream;
  if (per <= 1) return launch9<1>(*pat, *prog, vin, vout, vinit, a, b, n_out, threads, st);
  if (per <= 2) return launch9<2>(*pat, *prog, vin, vout, vinit, a, b, n_out, threads, st);
  if (per <= 4) return launch9<4>(*pat, *prog, vin, vout, vinit, a, b, n_out, threads, st);
  if (per <= 8) return launch9<8>(*pat, *prog, vin, vout, vinit, a, b, n_out, threads, st);
  if (per <= 16) return launch9<16>(*pat, *prog, vin, vout, vinit, a, b, n_out, threads, st);
  set_error("sgk_stencil9_apply: too many output columns for one CTA");
  return SGK_ELIMIT;
}

extern "C" int sgk_stencil9_grid_apply(const sgk_grid9* gp, const sgk_program9* prog, int32_t n_in,
                                       const sgk_view* in, int32_t n_out, const sgk_view* out,
                                       const sgk_view* init, const double* alpha, const double* beta,
                                       void* stream) {
  using namespace sgk;
  SGK_REQUIRE(gp && prog && out && alpha && beta, "sgk_stencil9_grid_apply: null argument");
  SGK_REQUIRE(n_in >= 1 && n_in <= SGK_MAX_IO && n_out >= 1 && n_out <= SGK_MAX_IO,
              "sgk_stencil9_grid_apply: input/output count out of range");
  SGK_REQUIRE(gp->nx >= 3 && gp->ny >= 1 && gp->coefg != nullptr && gp->seg_len >= 1,
              "sgk_stencil9_grid_apply: bad grid");
  SGK_REQUIRE(gp->row0 >= 0 && gp->n_rows >= 0 && (int64_t)gp->row0 + gp->n_rows <= (int64_t)gp->nx * gp->ny,
              "sgk_stencil9_grid_apply: row range outside the grid");
  SGK_REQUIRE((int64_t)prog->n_coef * 8 <= (1 << 14), "sgk_stencil9_grid_apply: too many distinct coefficients");
  SGK_REQUIRE(prog->n_slices == gp->n_slices, "sgk_stencil9_grid_apply: program compiled for another slice count");
  SGK_REQUIRE(prog->n_groups >= 1 && prog->n_groups <= 8, "sgk_stencil9_grid_apply: needs 1..8 column groups");
  ViewSet vin{}, vout{}, vinit{};
  ScalarSet a{}, b{};
  for (int i = 0; i < n_in; ++i) vin.v[i] = in[i];
  for (int i = 0; i < n_out; ++i) {
    SGK_REQUIRE(out[i].ptr != nullptr, "sgk_stencil9_grid_apply: null output");
    vout.v[i] = out[i];
    if (init) vinit.v[i] = init[i];
    a.s[i] = alpha[i];
    b.s[i] = beta[i];
  }
  if (gp->n_rows == 0 || prog->n_out_cols == 0) return SGK_OK;
  SGK_REQUIRE(prog->n_chunks * 32 >= prog->n_out_cols, "sgk_stencil9_grid_apply: n_chunks too small");
  const int per = (prog->n_chunks + 7) / 8;
  cudaStream_t st = (cudaStream_t)stream;
  if (n_out == 1) {
    if (per <= 1) return launch9grid<1, true>(*gp, *prog, vin, vout, vinit, a, b, st);
    if (per <= 2) return launch9grid<2, true>(*gp, *prog, vin, vout, vinit, a, b, st);
    if (per <= 4) return launch9grid<4, true>(*gp, *prog, vin, vout, vinit, a, b, st);
    if (per <= 8) return launch9grid<8, true>(*gp, *prog, vin, vout, vinit, a, b, st);
  } else {
    if (per <= 1) return launch9grid<1, false>(*gp, *prog, vin, vout, vinit, a, b, st);
    if (per <= 2) return launch9grid<2, false>(*gp, *prog, vin, vout, vinit, a, b, st);
    if (per <= 4) return launch9grid<4, false>(*gp, *prog, vin, vout, vinit, a, b, st);
    if (per <= 8) return launch9grid<8, false>(*gp, *prog, vin, vout, vinit, a, b, st);
  }
  set_error("sgk_stencil9_grid_apply: too many output columns for one CTA");
  return SGK_ELIMIT;
}

namespace sgk {
// coefg[p][t][(dy+1)*3+dx+1] = sum of the padded coef10 entries of row p at
// that stencil position (padding entries carry zero values)
__global__ void grid9_coef_kernel(int32_t n_rows, int32_t n_slices, int32_t nx, const int32_t* colind9,
                                  const double* coef10, double* coefg) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)n_rows * n_slices) return;
  const int p = (int)(i / n_slices);
  double acc[10];
#pragma unroll
  for (int k = 0; k < 10; ++k) acc[k] = 0.0;
  for (int jj = 0; jj < 9; ++jj) {
    const int d = colind9[(int64_t)p * 9 + jj] - p;
    const int dx = (d == -nx - 1 || d == -1 || d == nx - 1) ? -1 : ((d == -nx + 1 || d == 1 || d == nx + 1) ? 1 : 0);
    const int dy = (d - dx) / nx;
    const int pos = (dy + 1) * 3 + dx + 1;
    const double v = coef10[i * 10 + jj];
#pragma unroll
    for (int k = 0; k < 9; ++k)
      if (k == pos) acc[k] += v;
  }
#pragma unroll
  for (int k = 0; k < 10; ++k) coefg[i * 10 + k] = acc[k];
}
}  // namespace sgk

#ifdef SGK_S9_TRACE
extern "C" int sgk_s9_trace_read(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, sgk::sgk_s9_trace, sizeof(long long) * 3 * 256 * 8);
}
#endif

extern "C" int sgk_grid9_coef(int32_t n_rows, int32_t n_slices, int32_t nx, const int32_t* colind9,
                              const double* coef10, double* coefg, void* stream) {
  using namespace sgk;
  SGK_REQUIRE(n_rows >= 0 && n_slices >= 1 && nx >= 3, "sgk_grid9_coef: bad sizes");
  SGK_REQUIRE(colind9 && coef10 && coefg, "sgk_grid9_coef: null argument");
  const int64_t n = (int64_t)n_rows * n_slices;
  if (n == 0) return SGK_OK;
  grid9_coef_kernel<<<(unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(n_rows, n_slices, nx, colind9,
                                                                                 coef10, coefg);
  return check_launch("grid9_coef_kernel");
}
