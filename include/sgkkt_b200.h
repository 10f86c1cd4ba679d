/*
 * sgkkt_b200.h — C ABI of libsgkkt_b200.so, the sm_100a hot path of the
 * stochastic-Galerkin KKT solver (arXiv 2512.23804, reference package
 * `sgkkt`).
 *
 * Every entry point takes plain device pointers (owned by the caller, e.g.
 * PyTorch), sizes and a cudaStream_t passed as void*.  Nothing here
 * allocates device memory, nothing synchronises the host, and every call
 * returns 0 on success or a negative SGK_E* code (see sgk_last_error()).
 *
 * Which reference interface each entry point replaces (paths relative to
 * /root/reference/pkg/src/sgkkt/):
 *
 *   sgk_program_apply      operators.py:88-96   kron_apply
 *                          operators.py:99-126  kron_apply_sliced
 *                          preconditioners.py:132-144 HierarchicalGaussSeidel._cross_product
 *                          preconditioners.py:359-409 CoupledSweepPreconditioner._stiffness_coupling,
 *                                                     _mass_coupling, _level_rhs
 *                          operators.py:181-194 steady_kkt_apply
 *   sgk_trisolve           linalg.py:76-87      LUFactors.solve (SuperLU gstrs),
 *                          applied to all columns of one degree level at once
 *                          (preconditioners.py:155-164, 422-433)
 *   sgk_fastdiag_solve     linalg.py:76-87      LUFactors.solve for a Kronecker-sum lead
 *                          (A_1, A_1 + c M, and the P~ block of preconditioners.py:437-448)
 *   sgk_q1_assemble        fem.py:171-206       assemble_stiffness / assemble_mass (all slices at once)
 *   sgk_lognormal_fields   random_field.py:130-151 lognormal gPC coefficient fields
 *   sgk_cheb_step          preconditioners.py:70-98  chebyshev_mass_solve (one step)
 *   sgk_colscale           preconditioners.py:248-255 (column weights h^gamma, 1/beta)
 *   sgk_dot_partial,
 *   sgk_reduce_partials,
 *   sgk_axpy_dev, ...      krylov.py:78-99,129  fgmres inner products / updates
 *                          (deterministic two-stage fp64 reductions)
 *   sgk_f2n / sgk_n2f      operators.py:41-50   matricize / vectorize (layout)
 */
#ifndef SGKKT_B200_H
#define SGKKT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* error codes */
#define SGK_OK 0
#define SGK_EINVAL -1   /* bad argument (shape, range, null pointer) */
#define SGK_ECUDA -2    /* CUDA launch / runtime error */
#define SGK_ELIMIT -3   /* size beyond a compiled limit */

/* Shared CSR pattern of all spatial matrices (A_t and M share one mesh).
 * vals holds n_slices value slices in row-block, slice-major order: the
 * values of row i for slice t are vals[rowptr[i]*n_slices + t*len_i + jj],
 * len_i = rowptr[i+1]-rowptr[i], jj in [0,len_i).                         */
typedef struct {
  int32_t n_rows;
  int32_t n_slices;
  int32_t max_row_nnz;   /* longest row (selects the staged kernel)      */
  int32_t pad;
  const int32_t* rowptr; /* [n_rows+1] */
  const int32_t* colind; /* [nnz] sorted per row */
  const double* vals;    /* [nnz*n_slices] */
} sgk_pattern;

/* Compiled coupling program: out_o[i,k] = alpha_o * sum_e coef_e * U_e[i]
 * + beta_o * init_o[i,k],  U_(s,l,t)[i] = sum_j A_t[i,j] V_s[j,l].
 * Built on the host (paper_2512_23804_b200/program.py).                   */
typedef struct {
  int32_t n_groups;        /* warp groups of 32 lane items                  */
  int32_t n_phases;        /* shared-memory phases                           */
  int32_t n_out_cols;      /* gather targets over all outputs               */
  int32_t max_phase_slots; /* doubles of shared memory one phase needs      */
  const int32_t* lane_item;   /* [n_groups*32] (input<<24)|column, -1 idle   */
  const int32_t* group_step0; /* [n_groups+1] first global step of group    */
  const int32_t* step_term;   /* [n_steps*32] slice per (step,lane), -1 idle */
  const int32_t* phase_group0;/* [n_phases+1] first group of phase          */
  const int32_t* gather_ptr;  /* [n_phases*n_out_cols+1]                    */
  const int32_t* gather_slot; /* phase-local slot (step-step0)*32+lane      */
  const double* gather_coef;
  const int32_t* out_col;     /* [n_out_cols] (output<<24)|column           */
  /* compact gather (optional, NULL = use gather_slot/gather_coef): word e =
   * gather_slot[e] | (index of gather_coef[e] in coef_tab) << 16           */
  int32_t n_coef;             /* <= 2048 distinct coefficients              */
  int32_t pad;
  const uint32_t* gather_word;
  const double* coef_tab;
} sgk_program;

/* Strided view of a node-major (n_rows x ld) fp64 block, columns
 * [col0, col0+width).                                                       */
typedef struct {
  double* ptr;
  int64_t ld;
  int32_t col0;
  int32_t pad;
} sgk_view;

#define SGK_MAX_IO 4

int sgk_program_apply(const sgk_pattern* pat, const sgk_program* prog,
                      int32_t n_in, const sgk_view* in,
                      int32_t n_out, const sgk_view* out,
                      const sgk_view* init, /* ptr may be NULL per output  */
                      const double* alpha, const double* beta,
                      int32_t block_threads, void* stream);

/* Fast path for patterns with at most 9 entries per row (the Q1 stencil):
 * every row padded to exactly 9 columns (padding entries carry a valid
 * column and zero values); coefficients per row as n_slices blocks of 10
 * doubles (16-byte aligned pairs, the 10th is zero).                        */
typedef struct {
  int32_t n_rows;
  int32_t n_slices;
  const int32_t* colind9; /* [n_rows*9]                                     */
  const double* coef10;   /* [n_rows*n_slices*10]                           */
} sgk_pattern9;

/* Contiguous-group uniform schedule: group g covers input columns
 * [col0, col0+ncols) (ncols <= 128) of input s; lane L of the owning warp
 * holds columns col0 + 32c + L (c < 4).  group_info[g] = {s, col0, ncols, q0}
 * (steps q0 .. group_info[g+1].q0).  Step q evaluates term t_q for the four
 * column slots: step_rec[q] = t_q | (sw_q << 16), sw_q < 16, and the product
 * of lane L, slot c lands in ubuf slot gbase + 128(q-q0) + 32c + (L ^ sw_q)
 * (gbase = slots of the groups before; 32 trash and 32 zero slots follow the
 * n_ubuf product slots).  Gather, SELL-32 (32 output positions per chunk,
 * a chunk never spans two outputs): gather_ptr[2j], [2j+1] = row count and
 * offset of chunk j; entries at off + e*32 + lane, packed (ubuf byte
 * offset << 14) | coef_tab byte offset, both relative to the kernel's dynamic
 * shared memory (layout: coef_tab, 2 coefficient blocks, 2 column blocks,
 * ubuf — so the program is compiled for the pattern's n_slices); padding
 * reads the zero slots.  Chunk j is gathered by warp j % (CTA warps); out_col[position]
 * = (output<<24)|column or -1.                                              */
typedef struct {
  int32_t n_groups;
  int32_t n_steps;
  int32_t n_ubuf;
  int32_t n_out_cols;
  int32_t n_coef;
  int32_t n_gather;
  int32_t n_slices;          /* pattern slices the entry offsets assume      */
  int32_t n_chunks;          /* >= ceil(n_out_cols/32)                      */
  const int32_t* group_info; /* [(n_groups+1)*4]                            */
  const int32_t* step_rec;   /* [n_steps]                                   */
  const double* coef_tab;    /* [n_coef]                                    */
  const int32_t* gather_ptr; /* [2*n_chunks]                                */
  const uint32_t* gather_ent;/* [n_gather]                                  */
  const int32_t* out_col;    /* [32*n_chunks]                               */
  double coef8[8];           /* host copy of coef_tab[0..8) (n_coef <= 8: the
                              * grid kernel's gather reads the coefficients from
                              * the kernel parameter bank, not shared memory) */
} sgk_program9;

/* Same contract as sgk_program_apply for a padded 9-point pattern.  Returns
 * SGK_ELIMIT when the program does not fit in shared memory (use the
 * general kernel then).                                                     */
int sgk_stencil9_apply(const sgk_pattern9* pat, const sgk_program9* prog,
                       int32_t n_in, const sgk_view* in,
                       int32_t n_out, const sgk_view* out,
                       const sgk_view* init, const double* alpha,
                       const double* beta, int32_t block_threads, void* stream);
/* Grid form of the 9-point pattern: the Q1 stencil of an nx x ny grid in
 * natural node order (p = iy*nx + ix; the neighbours of p are p+dy*nx+dx).
 * coefg[p][t][(dy+1)*3 + dx+1] holds the t-stacked values in stencil
 * position order, zero where a neighbour lies outside the grid (10 doubles
 * per (p, t), the 10th zero).  A launch covers nodes [row0, row0+n_rows);
 * output/init views start at node row0, input views at node 0.              */
typedef struct {
  int32_t n_rows;
  int32_t n_slices;
  int32_t nx;
  int32_t ny;
  int32_t row0;
  int32_t seg_len;        /* rows per grid-line segment of the CTA walk     */
  const double* coefg;    /* [nx*ny*n_slices*10]                            */
} sgk_grid9;

/* Warp-specialised 9-point program on the grid form (contiguous row ranges
 * per CTA, sliding V window).  Programs with 1..8 column groups.            */
int sgk_stencil9_grid_apply(const sgk_grid9* grid, const sgk_program9* prog,
                            int32_t n_in, const sgk_view* in,
                            int32_t n_out, const sgk_view* out,
                            const sgk_view* init, const double* alpha,
                            const double* beta, void* stream);
/* coefg from the padded layout (colind9, coef10) of the same grid pattern.  */
int sgk_grid9_coef(int32_t n_rows, int32_t n_slices, int32_t nx,
                   const int32_t* colind9, const double* coef10, double* coefg,
                   void* stream);
/* Shared-memory bytes the fast path needs for (pattern, program).          */
int64_t sgk_stencil9_smem_bytes(const sgk_pattern9* pat, const sgk_program9* prog);

/* Sparse triangular factor (CSR, off-diagonal entries only) with a
 * dependency-respecting row order (level order).  diag_inv==NULL means
 * unit diagonal (SuperLU's L).                                              */
typedef struct {
  int32_t n;
  int32_t lower;          /* 1: rows depend on smaller columns (L)         */
  const int32_t* rowptr;
  const int32_t* colind;
  const double* vals;
  const double* diag_inv; /* [n] or NULL                                   */
  const int32_t* order;   /* [n] topological (level) order                */
  int32_t* flags;         /* [n * ceil(width/CW)] scratch, zeroed once     */
  int32_t* ticket;        /* [1] scratch                                   */
} sgk_trifactor;

/* Grouped (chain-supernodal) triangle in "processing space": rows in
 * dependency order, strictly lower CSR; consecutive rows that each depend on
 * the previous one form a group of <= 32 rows solved by one CTA without a
 * global round trip per row.  L is passed as is (work_row[p] = p, io_row[p] =
 * source row of b, diag_inv = NULL); U is passed reversed (p = n-1-k,
 * work_row[p] = k, io_row[p] = destination row of x, diag_inv[p] = 1/U_kk).
 * The in-group block of every group is applied as a dense inverse:
 * minv[minv_ptr[g] + r*gs + k] = ((D + B_g)^-1)[r][k] (gs = group size, B_g
 * the strictly lower in-group entries, D = I for L and diag(U_kk) for U), so a
 * group's rows are finished in parallel instead of by a sequential chain.    */
typedef struct {
  int32_t n;
  int32_t n_groups;
  int32_t reversed;           /* 0: work_row[p] == p, 1: == n-1-p          */
  int32_t pad;
  const int32_t* rowptr;      /* [n+1]                                     */
  const int32_t* split;       /* [n] first entry of row p inside its group */
  const int32_t* colind;      /* processing-space columns, sorted          */
  const double* vals;
  const int32_t* group_ptr;   /* [n_groups+1] row ranges                   */
  const int32_t* group_order; /* [n_groups] topological (level) order      */
  const int32_t* gdep_ptr;    /* [n_groups+1] distinct dependency groups   */
  const int32_t* gdep;        /* of each group (CSR)                       */
  const int32_t* work_row;    /* [n]                                       */
  const int32_t* io_row;      /* [n]                                       */
  const double* diag_inv;     /* [n] or NULL                               */
  int32_t* flags;             /* [n_groups * chunks] scratch               */
  int32_t* ticket;            /* [1] scratch                               */
  const int64_t* minv_ptr;    /* [n_groups] offsets into minv              */
  const double* minv;         /* dense in-group inverses, row-major gs x gs */
  /* dense region: groups [dense_g0, dense_g0+dense_nb) are 32-row blocks of
   * rows dense_r0.. whose off-diagonal blocks against earlier region rows are
   * stored densely (block i: 32 x 32i row-major at dense + 1024*i*(i-1)/2)
   * and streamed block by block as the earlier blocks finish             */
  int32_t dense_g0;
  int32_t dense_nb;
  int32_t dense_r0;
  int32_t dense_pad;
  const double* dense;
} sgk_trigroups;

/* Segmented row view: global row r lives in segment r / seg_rows.          */
typedef struct {
  double* ptr[3];
  int64_t ld;
  int32_t col0;
  int32_t seg_rows;
} sgk_segview;

/* X = Pc U^-1 L^-1 Pr B for `width` columns (linalg.py:83-87).
 * in_perm[k]  = source row of B for factor row k   (inverse of perm_r)
 * out_perm[k] = destination row of X for factor row k (inverse of perm_c)
 * work: n x width contiguous scratch.  B and X may alias.                   */
/* CW: RHS columns per solve task (flags are per (row, CW-column chunk)).   */
int32_t sgk_trisolve_chunk_cols(void);
int sgk_trisolve(const sgk_trifactor* L, const sgk_trifactor* U,
                 const int32_t* in_perm, const int32_t* out_perm,
                 const sgk_segview* b, const sgk_segview* x, double* work,
                 int32_t width, int32_t epoch, void* stream);

/* Same result as sgk_trisolve, grouped task granularity (one readiness flag
 * per (group, chunk) with chunks of 1..16 columns; `work` must hold
 * n x (width rounded up to a multiple of 16) doubles).                       */
int32_t sgk_trisolve_grouped_chunk_cols(void);
int sgk_trisolve_grouped(const sgk_trigroups* L, const sgk_trigroups* U,
                         const sgk_segview* b, const sgk_segview* x,
                         double* work, int32_t width, int32_t epoch, void* stream);

/* Wide-RHS form of the grouped solve (csrc/trisolve_wide.cu): the same
 * processing-space triangle and chain groups, the groups' outside entries cut
 * into segments (<= 32 entries, one row each) and tiles (<= 32 segments) in
 * topological group order; a group with several tiles gathers its per-(tile,
 * row) partial sums in `part` slots and is finalised by its last tile.     */
typedef struct {
  int32_t n;
  int32_t n_groups;
  int32_t n_tiles;
  int32_t reversed;           /* U passed reversed: work row of p = n-1-p    */
  const int32_t* rowptr;      /* [n+1] strict triangle (processing space)   */
  const int32_t* colind;
  const double* vals;
  const int32_t* group_ptr;   /* [n_groups+1]                               */
  const int32_t* tile_group;  /* [n_tiles]                                  */
  const int32_t* tile_seg;    /* [n_tiles+1] segment range of each tile      */
  const int32_t* tile_dep_ptr;/* [n_tiles+1]                                */
  const int32_t* tile_dep;    /* groups each tile's entries read            */
  const int32_t* group_ntiles;/* [n_groups]                                 */
  const int32_t* seg_row;     /* [n_seg] processing row                     */
  const int32_t* seg_e0;      /* [n_seg] entry range [e0, e1), <= 32 entries */
  const int32_t* seg_e1;
  const int32_t* seg_slot;    /* [n_seg] part slot (multi-tile groups)      */
  const int32_t* row_slot_ptr;/* [n+1] part slots of each row, tile order   */
  const int32_t* row_slot;
  const int32_t* work_row;    /* [n]                                        */
  const int32_t* io_row;      /* [n]                                        */
  const int64_t* minv_ptr;    /* [n_groups]                                 */
  const double* minv;         /* dense inverse of each group's diagonal block */
  int32_t* flags;             /* [n_groups * chunks] epoch flags             */
  int32_t* counters;          /* [n_groups * chunks] tile counters (zeroed per solve) */
  int32_t* ticket;
  const int32_t* tile_kind;   /* [n_tiles] 0: entry tile, 1: dense-region task */
  int32_t dense_g0;           /* dense-region groups [dense_g0, +dense_nb)  */
  int32_t dense_nb;
  int32_t dense_r0;           /* first row of the dense region              */
  int32_t dense_pad;
  const double* dense;        /* off-diagonal region blocks (sgk_trigroups) */
  /* column-panel form (pcol != NULL; linalg.wide_panels): tile_seg holds the
   * panel range of each tile; a panel is 32 distinct solution rows (pcol)
   * against a dense zero-filled 32 x 32 block pval[panel][group row][column];
   * a slotted tile writes the partial sums of all group rows to part slots
   * tile_slot[tile] + row-in-group (-1: not slotted).  The seg_* arrays are
   * unused in this form.                                                    */
  const int32_t* pcol;        /* [32 * n_panels] processing-space columns    */
  const double* pval;         /* [1024 * n_panels]                           */
  const int32_t* tile_slot;   /* [n_tiles]                                   */
  /* explicit inverse of the dense region's triangle (NULL: the region's
   * blocks are streamed by the dense tasks): (32 dense_nb)^2 doubles,
   * row-major, inv(strict + diagonal) of rows/columns [dense_r0, +32 dense_nb).
   * The region is then solved by one blocked product around the sync-free
   * kernel (before it for a leading region, after it for a trailing one);
   * `part` needs 32 dense_nb extra rows after the part slots.               */
  const double* region_inv;
  int32_t part_rows;          /* part slots in use: the region's P rows start here */
  int32_t region_pad;
} sgk_triwide;

/* Chunk width (columns per task) the wide solve uses for `width`.          */
int32_t sgk_trisolve_wide_chunk_cols(int32_t width);
/* Same result as sgk_trisolve_grouped.  work and part: n x ldw doubles with
 * ldw = width rounded up to the chunk width (part: n_slots rows).           */
int sgk_trisolve_wide(const sgk_triwide* L, const sgk_triwide* U,
                      const sgk_segview* b, const sgk_segview* x,
                      double* work, double* part, int32_t width, int32_t epoch,
                      void* stream);

/* Fast-diagonalisation factor of a Kronecker-sum lead (
 * replaces LUFactors.solve, linalg.py:76-87, when the lead is
 * A = K1(x)M1 + M1(x)K1 on an n x n tensor grid and M = M1(x)M1):
 * s = S zero-padded to np x np (row-major, np = n rounded up to 8, <= 256;
 * K1 S = M1 S diag(mu), S^T M1 S = I), lam[a*n+b] = mu_a + mu_b.
 * n_seg == 1: X = A^-1 B.  n_seg == 3: the hGSoc block
 * P~ = [M 0 -A; 0 beta M M; -A M 0] (preconditioners.py:437-448) on the
 * (y, u, lambda) segments.  Three sm_100a kernels (fp64 mma.sync): pass 1,
 * passes 2 + modal solve + 3 fused, pass 4.  work:
 * sgk_fastdiag_work_doubles() doubles.  B and X may alias.                  */
typedef struct {
  int32_t n;
  int32_t n_seg;
  int32_t np;
  int32_t pad;
  const double* s;
  const double* lam;
  double beta;
  /* centrosymmetric form (NULL sh: full passes): modes ordered symmetric
   * first (ne of them, lam and s permuted alike); sh = S_E = S[0:h+n%2, 0:ne]
   * then S_O = S[0:h, ne:n], each zero-padded to hp x hp (h = n/2, hp = a
   * multiple of 8 >= h+1, <= 128): half-size GEMMs around a butterfly.    */
  int32_t ne;
  int32_t hp;
  const double* sh;
} sgk_fastdiag;
int64_t sgk_fastdiag_work_doubles(const sgk_fastdiag* fd, int32_t width);
int sgk_fastdiag_solve(const sgk_fastdiag* fd, const sgk_segview* b,
                       const sgk_segview* x, double* work, int32_t width,
                       void* stream);

/* GPU setup pipeline.
 * sgk_q1_assemble: the Q1 stiffness matrices of n_fields coefficient fields
 * (fields: n_fields x n_elements x 4 Gauss-point samples, x fastest) and,
 * with with_mass, the mass matrix as the last slice, assembled on the
 * uniform n_cells^2 grid with boundary elimination (fem.py:171-206) into
 * the pattern's t-stacked values (rowptr: the shared 9-point structure) and
 * the padded 9-point layout (coef10: rows x S x 10, colind9: rows x 9; both
 * may be NULL).  stiff_q: 4x4x4 reference gradient products per Gauss point
 * [q][a][b]; mass_ref: 4x4, scaled by mass_weight.  Host pointers for
 * stiff_q / mass_ref, device pointers for the rest.
 * sgk_lognormal_fields: out[t][p] = mean[p] * prod_v g[v][p]^idx[t][v] /
 * sqrt(idx[t][v]!)  (random_field.py:130-151).                              */
int sgk_q1_assemble(int32_t n_cells, int32_t n_fields, const double* fields,
                    const double* stiff_q, int32_t with_mass, double mass_weight,
                    const double* mass_ref, const int32_t* rowptr, double* vals,
                    double* coef10, int32_t* colind9, void* stream);
int sgk_lognormal_fields(int64_t n_points, int32_t m, int32_t n_terms,
                         const double* mean, const double* g, const int32_t* idx,
                         double* out, void* stream);

/* One Chebyshev semi-iteration step on all columns (preconditioners.py:89-97):
 * x_new = omega*(scale .* (b - M x) + x - x_prev) + x_prev,
 * scale[i] = 1/(alpha*M_ii).  slice selects M inside the shared pattern.
 * x and x_prev may be NULL: the zero iterate (first two steps from x0 = 0). */
int sgk_cheb_step(const sgk_pattern* pat, int32_t slice, const double* scale,
                  int64_t n_cols, const double* b, const double* x,
                  const double* x_prev, double* x_new, double omega,
                  void* stream);
/* The same step on n_batch independent blocks stored back to back
 * (block bi at offset bi*n_rows*n_cols of b/x/x_prev/x_new): the N_t mass
 * solves of the time-dependent preconditioner (preconditioners.py:278-312)
 * in one launch per step. */
int sgk_cheb_step_batched(const sgk_pattern* pat, int32_t slice, const double* scale,
                          int64_t n_batch, int64_t n_cols, const double* b,
                          const double* x, const double* x_prev, double* x_new,
                          double omega, void* stream);

/* y[i,k] = s * x[i,k] * w[k]  (w may be NULL: y = s*x).                   */
int sgk_colscale(int64_t n_rows, int64_t n_cols, const double* x,
                 const double* w, int32_t invert_w, double s, double* y,
                 void* stream);
/* n_batch back-to-back (n_rows x n_cols) blocks, block b scaled by the
 * device scalar s[b]: y = s[b] * (x / w or x * w) — the N_t steps of the
 * PINT preconditioner's y/u blocks (preconditioners.py:278-312) at once.   */
int sgk_colscale_batched(int64_t n_batch, int64_t n_rows, int64_t n_cols,
                         const double* x, const double* w, int32_t invert_w,
                         const double* s, double* y, void* stream);

/* y = beta*y + mass-stencil(x)*w  etc. are expressed as programs.          */

/* Deterministic fp64 reductions: partials of n-length dot products of x
 * with each of k vectors y_j = y + j*ystride (k<=SGK_MAX_MDOT), written to
 * part[j*n_blocks + b]; n_blocks fixed by sgk_reduce_blocks().             */
#define SGK_MAX_MDOT 8
int32_t sgk_reduce_blocks(void);
int sgk_dot_partial(int64_t n, const double* x, const double* y,
                    int64_t ystride, int32_t k, double* part, void* stream);
/* out[j] = sum_b part[j*n_blocks+b] in a fixed tree order (+ optional
 * sqrt when take_sqrt).                                                     */
int sgk_reduce_partials(const double* part, int32_t k, double* out,
                        int32_t take_sqrt, void* stream);
/* y = a*x + b*y with a = sa * (*da if da) and b likewise.                   */
int sgk_axpby_dev(int64_t n, double sa, const double* da, int32_t inv_a,
                  const double* x, double sb, const double* db, double* y,
                  void* stream);
/* out = s*((x0 + c1*x1) + c2*x2) in one pass, rounded exactly like the
 * sgk_axpby_dev chain y=x0; y+=c1*x1; y+=c2*x2; y*=s (x1/x2 may be NULL;
 * out may alias x0, not x1/x2).  MINRES three-term recurrences. */
int sgk_lincomb3(int64_t n, const double* x0, double c1, const double* x1,
                 double c2, const double* x2, double s, double* out, void* stream);
/* Modified Gram–Schmidt step fused with the next inner product:
 * w -= h * q_i  (h = *dh), then partial dot of q_next with the new w.        */
int sgk_mgs_step(int64_t n, const double* dh, const double* q_i, double* w,
                 const double* q_next, double* part_next, void* stream);
/* max_j |out[j]| etc. are done on the host from the reduced values.        */

/* Layout: F-order (column k = chaos mode, matricize) <-> node-major.       */
int sgk_f2n(int64_t n_rows, int64_t n_cols, const double* f, double* nm,
            void* stream);
int sgk_n2f(int64_t n_rows, int64_t n_cols, const double* nm, double* f,
            void* stream);

/* Diagnostics.                                                              */
const char* sgk_last_error(void);
int32_t sgk_version(void);
/* number of kernel launches issued by this library since load (all
 * entry points; used by bench.py for "gpu_launches").                       */
int64_t sgk_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif
