// K1/K2/K4 — fused shared-pattern Galerkin "coupling program" kernel.
//
// Computes, for every mesh row i,
//     out_o[i,k] = alpha_o * sum_{(p,h) in G(o,k)} h * U_p[i] + beta_o * init_o[i,k]
//     U_p[i]     = sum_j A_{t_p}[i,j] * V_{s_p}[j, l_p]
// where all A_t (and M) share one CSR pattern (t-stacked values) and the
// list of (t,s,l) products plus the sparse gather G are compiled on the host
// (program.py).  This single kernel covers
//   kron_apply          operators.py:88-96   (W = sum_t A_t V H_t)
//   kron_apply_sliced   operators.py:99-126  (column-range restricted)
//   HierarchicalGaussSeidel._cross_product  preconditioners.py:132-144
//   CoupledSweepPreconditioner._level_rhs   preconditioners.py:386-409
//   steady_kkt_apply    operators.py:181-194 (three block rows in one pass).
//
// Work decomposition (B200): one CTA per mesh row at a time (grid-stride over
// rows, CTAs ordered so rows in flight are adjacent and the 3 grid lines of V
// they touch stay L2-resident).  Inside a row, each warp owns "groups": 32
// chaos columns l (one per lane, V rows of the 9 neighbours held in registers)
// and a list of steps; at a step every lane forms one 9-term stencil dot
// U_(t,l) with the t the host scheduled for that lane (uniform t across the
// warp turns the coefficient loads into broadcasts).  U values land in shared
// memory; after a barrier each thread gathers the sparse H coupling for its
// output columns from shared memory, accumulating in registers.  Programs
// larger than the shared-memory budget are split into phases.
#include "sgk_common.cuh"

namespace sgk {

template <typename T>
__device__ __forceinline__ T sel4v(T a, T b, T c, T d, int i) {
  return i == 0 ? a : (i == 1 ? b : (i == 2 ? c : d));
}

constexpr int kChunk = 9;          // stencil entries held in registers per pass
// the row's t-stacked coefficients are staged in shared memory when they fit
// next to the U slots (many-term programs: config 3 has 924 slices x 9
// entries = 66.5 KB per row; read from global memory they are 9 scattered
// loads per product)
constexpr size_t kSmemBudget = 200 * 1024;

// STAGED: the row's t-stacked coefficients (n_slices*len doubles) are copied
// to shared memory once per row and read back from there (broadcasts when the
// warp's lanes evaluate the same term).
template <int MAXOUT, bool STAGED>
__global__ void __launch_bounds__(256) program_kernel(sgk_pattern pat, sgk_program prog,
                                                      ViewSet in, ViewSet out, ViewSet init,
                                                      ScalarSet alpha, ScalarSet beta, int stage_n) {
  extern __shared__ double smem[];
  double* coef_s = smem;                          // [stage_n] when STAGED
  double* ubuf = smem + (STAGED ? stage_n : 0);    // U slots of one phase
  // compact gather: the small coefficient table is read through L1 (it
  // stays resident; no shared memory next to the staged block)
  const bool compact = prog.gather_word != nullptr;
  const double* __restrict__ ctab = prog.coef_tab;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const int n_slices = pat.n_slices;
  // single-chunk gather split (MAXOUT == 1): `parts` threads share a column;
  // row-invariant, computed once (an integer division per phase otherwise)
  const int parts = MAXOUT == 1 ? max(1, (int)blockDim.x / max(prog.n_out_cols, 1)) : 1;
  const int part_col = threadIdx.x / parts, part_r = threadIdx.x - part_col * parts;

  for (int row = blockIdx.x; row < pat.n_rows; row += gridDim.x) {
    const int rs = __ldg(pat.rowptr + row);
    const int len = __ldg(pat.rowptr + row + 1) - rs;
    const double* arow = pat.vals + (int64_t)rs * n_slices;
    const int32_t* crow = pat.colind + rs;
    if (STAGED) {
      const int nco = n_slices * len;
      __syncthreads();  // the previous row's products are done with coef_s
      // asynchronous 8-byte copies: every load of the block in flight at once
      // (a load -> store loop serialises one memory latency per iteration)
      for (int i = threadIdx.x; i < nco; i += blockDim.x) {
        const unsigned sa = (unsigned)__cvta_generic_to_shared(coef_s + i);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(arow + i) : "memory");
      }
      asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
      __syncthreads();
    }
    const double* abase = STAGED ? coef_s : arow;

    double acc[MAXOUT];
#pragma unroll
    for (int r = 0; r < MAXOUT; ++r) acc[r] = 0.0;

    for (int p = 0; p < prog.n_phases; ++p) {
      const int g0 = __ldg(prog.phase_group0 + p);
      const int g1 = __ldg(prog.phase_group0 + p + 1);
      const int qbase = __ldg(prog.group_step0 + g0);
      for (int g = g0 + warp; g < g1; g += nwarps) {
        const int item = __ldg(prog.lane_item + g * 32 + lane);
        const int q0 = __ldg(prog.group_step0 + g);
        const int q1 = __ldg(prog.group_step0 + g + 1);
        const double* vb = nullptr;
        int64_t ldv = 0;
        if (item >= 0) {
          const sgk_view& vv = pick(in, item >> 24);
          vb = vv.ptr + vv.col0 + (item & 0xFFFFFF);
          ldv = vv.ld;
        }
        const int passes = len > 0 ? len : 1;
        for (int c0 = 0; c0 < passes; c0 += kChunk) {
          const int cl = min(kChunk, len - c0);
          double v[kChunk];
#pragma unroll
          for (int jj = 0; jj < kChunk; ++jj)
            v[jj] = (vb != nullptr && jj < cl) ? __ldg(vb + (int64_t)__ldg(crow + c0 + jj) * ldv) : 0.0;
          int q = q0;
          // two independent steps per iteration (ILP across stencil dots);
          // the next pair's term indices are loaded one iteration ahead (the
          // step table is an L2 read when the staged block fills the SM)
          int ta_n = q + 1 < q1 ? __ldg(prog.step_term + q * 32 + lane) : 0;
          int tb_n = q + 1 < q1 ? __ldg(prog.step_term + (q + 1) * 32 + lane) : 0;
          for (; q + 1 < q1; q += 2) {
            const int ta = ta_n;
            const int tb = tb_n;
            if (q + 3 < q1) {
              ta_n = __ldg(prog.step_term + (q + 2) * 32 + lane);
              tb_n = __ldg(prog.step_term + (q + 3) * 32 + lane);
            }
            const double* aa = abase + max(ta, 0) * len + c0;
            const double* ab = abase + max(tb, 0) * len + c0;
            double ua0 = 0.0, ua1 = 0.0, ub0 = 0.0, ub1 = 0.0;
            if (cl == kChunk) {  // interior rows: no per-entry predicates (warp-uniform branch)
#pragma unroll
              for (int jj = 0; jj < kChunk; jj += 2) {
                ua0 = fma(aa[jj], v[jj], ua0);
                ub0 = fma(ab[jj], v[jj], ub0);
                if (jj + 1 < kChunk) {
                  ua1 = fma(aa[jj + 1], v[jj + 1], ua1);
                  ub1 = fma(ab[jj + 1], v[jj + 1], ub1);
                }
              }
            } else {
#pragma unroll
              for (int jj = 0; jj < kChunk; jj += 2) {
                if (jj < cl) {
                  ua0 = fma(aa[jj], v[jj], ua0);
                  ub0 = fma(ab[jj], v[jj], ub0);
                }
                if (jj + 1 < cl) {
                  ua1 = fma(aa[jj + 1], v[jj + 1], ua1);
                  ub1 = fma(ab[jj + 1], v[jj + 1], ub1);
                }
              }
            }
            const int sa = (q - qbase) * 32 + lane;
            if (ta >= 0) ubuf[sa] = (c0 == 0) ? ua0 + ua1 : ubuf[sa] + (ua0 + ua1);
            if (tb >= 0) ubuf[sa + 32] = (c0 == 0) ? ub0 + ub1 : ubuf[sa + 32] + (ub0 + ub1);
          }
          if (q < q1) {
            const int t = __ldg(prog.step_term + q * 32 + lane);
            if (t >= 0) {
              const double* at = abase + t * len + c0;
              double u0 = 0.0, u1 = 0.0;
#pragma unroll
              for (int jj = 0; jj < kChunk; jj += 2) {
                if (jj < cl) u0 = fma(at[jj], v[jj], u0);
                if (jj + 1 < cl) u1 = fma(at[jj + 1], v[jj + 1], u1);
              }
              const int slot = (q - qbase) * 32 + lane;
              ubuf[slot] = (c0 == 0) ? u0 + u1 : ubuf[slot] + (u0 + u1);
            }
          }
        }
      }
      __syncthreads();
      const int32_t* gp = prog.gather_ptr + (int64_t)p * prog.n_out_cols;
      if constexpr (MAXOUT == 1) {
        // fewer output columns than threads: `parts` threads share a column,
        // thread part r takes entries r, r+parts, ... (coalesced table loads),
        // four independent accumulation chains per thread
        const int c = part_col, r = part_r;
        if (c < prog.n_out_cols) {
          const int e0 = __ldg(gp + c), e1 = __ldg(gp + c + 1);
          double a0 = acc[0], a1 = 0.0, a2 = 0.0, a3 = 0.0;
          int e = e0 + r;
          if (compact) {
            for (; e + 3 * parts < e1; e += 4 * parts) {
              const uint32_t w0 = __ldg(prog.gather_word + e), w1 = __ldg(prog.gather_word + e + parts);
              const uint32_t w2 = __ldg(prog.gather_word + e + 2 * parts);
              const uint32_t w3 = __ldg(prog.gather_word + e + 3 * parts);
              a0 = fma(__ldg(ctab + (w0 >> 16)), ubuf[w0 & 0xFFFF], a0);
              a1 = fma(__ldg(ctab + (w1 >> 16)), ubuf[w1 & 0xFFFF], a1);
              a2 = fma(__ldg(ctab + (w2 >> 16)), ubuf[w2 & 0xFFFF], a2);
              a3 = fma(__ldg(ctab + (w3 >> 16)), ubuf[w3 & 0xFFFF], a3);
            }
            for (; e < e1; e += parts) {
              const uint32_t w0 = __ldg(prog.gather_word + e);
              a0 = fma(__ldg(ctab + (w0 >> 16)), ubuf[w0 & 0xFFFF], a0);
            }
          } else {
            for (; e + 3 * parts < e1; e += 4 * parts) {
              const int s0 = __ldg(prog.gather_slot + e), s1 = __ldg(prog.gather_slot + e + parts);
              const int s2 = __ldg(prog.gather_slot + e + 2 * parts), s3 = __ldg(prog.gather_slot + e + 3 * parts);
              const double h0 = __ldg(prog.gather_coef + e), h1 = __ldg(prog.gather_coef + e + parts);
              const double h2 = __ldg(prog.gather_coef + e + 2 * parts), h3 = __ldg(prog.gather_coef + e + 3 * parts);
              a0 = fma(h0, ubuf[s0], a0);
              a1 = fma(h1, ubuf[s1], a1);
              a2 = fma(h2, ubuf[s2], a2);
              a3 = fma(h3, ubuf[s3], a3);
            }
            for (; e < e1; e += parts) a0 = fma(__ldg(prog.gather_coef + e), ubuf[__ldg(prog.gather_slot + e)], a0);
          }
          acc[0] = (a0 + a1) + (a2 + a3);
        }
      } else {
#pragma unroll
        for (int r = 0; r < MAXOUT; ++r) {
          const int c = threadIdx.x + r * blockDim.x;
          if (c < prog.n_out_cols) {
            const int e0 = __ldg(gp + c), e1 = __ldg(gp + c + 1);
            double a = acc[r];
            for (int e = e0; e < e1; ++e)
              a = fma(__ldg(prog.gather_coef + e), ubuf[__ldg(prog.gather_slot + e)], a);
            acc[r] = a;
          }
        }
      }
      __syncthreads();
    }
    if constexpr (MAXOUT == 1) {
      // combine the parts of each column in a fixed order (deterministic)
      if (parts > 1) {
        ubuf[threadIdx.x] = acc[0];
        __syncthreads();
        const int c = threadIdx.x;
        if (c < prog.n_out_cols) {
          double a = ubuf[c * parts];
          for (int r = 1; r < parts; ++r) a += ubuf[c * parts + r];
          acc[0] = a;
        }
        __syncthreads();
      }
    }

#pragma unroll
    for (int r = 0; r < MAXOUT; ++r) {
      const int c = threadIdx.x + r * blockDim.x;
      if (c < prog.n_out_cols) {
        const int oc = __ldg(prog.out_col + c);
        const int o = oc >> 24, k = oc & 0xFFFFFF;
        // view fields selected by value (a per-thread index into the
        // parameter views would copy them to local memory)
        const double* ip = sel4v(init.v[0].ptr, init.v[1].ptr, init.v[2].ptr, init.v[3].ptr, o);
        double* op = sel4v(out.v[0].ptr, out.v[1].ptr, out.v[2].ptr, out.v[3].ptr, o);
        double y = sel4v(alpha.s[0], alpha.s[1], alpha.s[2], alpha.s[3], o) * acc[r];
        if (ip != nullptr)
          y += sel4v(beta.s[0], beta.s[1], beta.s[2], beta.s[3], o) *
               ip[(int64_t)row * sel4v(init.v[0].ld, init.v[1].ld, init.v[2].ld, init.v[3].ld, o) +
                  sel4v(init.v[0].col0, init.v[1].col0, init.v[2].col0, init.v[3].col0, o) + k];
        op[(int64_t)row * sel4v(out.v[0].ld, out.v[1].ld, out.v[2].ld, out.v[3].ld, o) +
           sel4v(out.v[0].col0, out.v[1].col0, out.v[2].col0, out.v[3].col0, o) + k] = y;
      }
    }
  }
}

template <int MAXOUT, bool STAGED>
static int launch_program_t(const sgk_pattern& pat, const sgk_program& prog, const ViewSet& in,
                            const ViewSet& out, const ViewSet& init, const ScalarSet& alpha,
                            const ScalarSet& beta, int threads, cudaStream_t st, int stage_n) {
  // U slots of a phase; at least one double per thread (the column-parts
  // reduction of single-chunk programs reuses the slots)
  const int slots = prog.max_phase_slots > threads ? prog.max_phase_slots : threads;
  const size_t smem = (size_t)(slots + (STAGED ? stage_n : 0)) * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(program_kernel<MAXOUT, STAGED>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaGetLastError();
    attr_set = true;
  }
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, program_kernel<MAXOUT, STAGED>, threads, smem);
  if (occ < 1) {
    set_error("program_kernel: zero occupancy (shared memory " + std::to_string(smem) + " B)");
    return SGK_ELIMIT;
  }
  int64_t grid = (int64_t)sm_count() * occ;
  if (grid > pat.n_rows) grid = pat.n_rows;
  if (grid < 1) return SGK_OK;
  program_kernel<MAXOUT, STAGED><<<(int)grid, threads, smem, st>>>(pat, prog, in, out, init, alpha, beta, stage_n);
  return check_launch("program_kernel");
}

template <int MAXOUT>
static int launch_program(const sgk_pattern& pat, const sgk_program& prog, const ViewSet& in,
                          const ViewSet& out, const ViewSet& init, const ScalarSet& alpha,
                          const ScalarSet& beta, int threads, cudaStream_t st, int max_row_nnz) {
  const int64_t stage_n = (int64_t)pat.n_slices * max_row_nnz;
  if ((size_t)(stage_n + prog.max_phase_slots + threads) * sizeof(double) <= kSmemBudget)
    return launch_program_t<MAXOUT, true>(pat, prog, in, out, init, alpha, beta, threads, st, (int)stage_n);
  return launch_program_t<MAXOUT, false>(pat, prog, in, out, init, alpha, beta, threads, st, 0);
}

}  // namespace sgk

extern "C" int sgk_program_apply(const sgk_pattern* pat, const sgk_program* prog, int32_t n_in,
                                 const sgk_view* in, int32_t n_out, const sgk_view* out,
                                 const sgk_view* init, const double* alpha, const double* beta,
                                 int32_t block_threads, void* stream) {
  using namespace sgk;
  SGK_REQUIRE(pat && prog && out && alpha && beta, "sgk_program_apply: null argument");
  SGK_REQUIRE(n_in >= 0 && n_in <= SGK_MAX_IO && n_out >= 1 && n_out <= SGK_MAX_IO,
              "sgk_program_apply: input/output count out of range");
  SGK_REQUIRE(pat->n_rows >= 0 && pat->n_slices >= 1, "sgk_program_apply: bad pattern");
  SGK_REQUIRE(prog->n_groups == 0 || n_in >= 1, "sgk_program_apply: program needs inputs");
  int threads = block_threads > 0 ? block_threads : 256;
  SGK_REQUIRE(threads % 32 == 0 && threads <= 256, "sgk_program_apply: block_threads must be a multiple of 32, <=256");
  ViewSet vin{}, vout{}, vinit{};
  ScalarSet a{}, b{};
  for (int i = 0; i < n_in; ++i) vin.v[i] = in[i];
  for (int i = 0; i < n_out; ++i) {
    vout.v[i] = out[i];
    SGK_REQUIRE(out[i].ptr != nullptr, "sgk_program_apply: null output");
    if (init) vinit.v[i] = init[i];
    a.s[i] = alpha[i];
    b.s[i] = beta[i];
  }
  if (pat->n_rows == 0 || prog->n_out_cols == 0) return SGK_OK;
  const int per = (prog->n_out_cols + threads - 1) / threads;
  const int max_nnz = pat->max_row_nnz;
  cudaStream_t st = (cudaStream_t)stream;
  if (per <= 1) return launch_program<1>(*pat, *prog, vin, vout, vinit, a, b, threads, st, max_nnz);
  if (per <= 2) return launch_program<2>(*pat, *prog, vin, vout, vinit, a, b, threads, st, max_nnz);
  if (per <= 4) return launch_program<4>(*pat, *prog, vin, vout, vinit, a, b, threads, st, max_nnz);
  if (per <= 8) return launch_program<8>(*pat, *prog, vin, vout, vinit, a, b, threads, st, max_nnz);
  if (per <= 16) return launch_program<16>(*pat, *prog, vin, vout, vinit, a, b, threads, st, max_nnz);
  set_error("sgk_program_apply: too many output columns for one CTA (max 16*block_threads)");
  return SGK_ELIMIT;
}
