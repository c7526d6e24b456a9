/* c0ip.h -- C ABI of the B200 vertex-patch Schwarz smoother for the C0 interior penalty (C0IP)
 * biharmonic discretisation on Cartesian meshes (arXiv 2412.05082).
 *
 * Citations are PAPER.md line numbers (section / equation / algorithm) of the paper text
 * shipped with the reference; "reading Qn" refers to the ambiguity ledger in DESIGN.md
 * (SURVEY.md §8c).
 *
 * General conventions
 *  - Every call returns c0ip_status.  Nothing aborts or throws across the ABI.  On a non-OK
 *    status, c0ip_last_error() returns a thread-local message.
 *  - Argument errors (null pointers, level/colour/variant out of range, dim not 2/3, degree
 *    not in [2,7], unsupported dtype) are detected synchronously and return C0IP_ERR_ARG
 *    without side effects.
 *  - Device vectors: caller-owned device pointers (e.g. torch tensors' data_ptr), contiguous,
 *    length n_dofs(level) = (k N - 1)^d, lexicographic with x fastest (reading C1), element
 *    type given by the dtype argument (C0IP_F64 -> double, C0IP_F32 -> float).  Host vectors
 *    are only used where the signature says "host".
 *  - Streams: device ops are enqueued on the given cudaStream_t (passed as void*, NULL = legacy
 *    default stream) and do not synchronise.  c0ip_pcg synchronises once per iteration.
 *  - Asynchronous CUDA faults are reported as C0IP_ERR_CUDA by the call that detects them.
 *  - Ownership: the context owns every table (1D operators, FDM factors, transfer bands,
 *    colour lists) and all workspaces; it never retains a caller pointer after return.
 *  - Concurrency: one context per host thread / stream at a time.
 *  - Levels: level l has N = 2^l cells per axis, l = 1..finest_level (reading Q9; level 1 is the
 *    2^d-cell mesh with one vertex patch).  If cells_override > 0 the context
 *    has the single level `finest_level` with N = cells_override (throughput runs; no MG).
 */
#ifndef C0IP_H
#define C0IP_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct c0ip_ctx_s* c0ip_ctx;

typedef enum {
  C0IP_OK = 0,
  C0IP_ERR_ARG = 1,
  C0IP_ERR_STATE = 2,
  C0IP_ERR_COERCIVITY = 3,
  C0IP_ERR_OOM = 4,
  C0IP_ERR_CUDA = 5,
  C0IP_ERR_NCCL = 6
} c0ip_status;

typedef enum { C0IP_F64 = 0, C0IP_F32 = 1 } c0ip_dtype;

/* Smoother realisations:
 *  AVS_ATOMIC        additive, x += w sum_v R_v^T A~_v^{-1} R_v r with global atomics (paper's "atomic AVS")
 *  AVS_DETERMINISTIC additive, gather formulation: every DoF sums its <= 2^d patch corrections in a
 *                    fixed order (no atomics; run-to-run bitwise reproducible)
 *  AVS_COLORED       additive, writes serialised over the 2^d non-overlapping parity classes ("colored AVS")
 *  MVS               coloured multiplicative, residual recomputed per colour        */
typedef enum {
  C0IP_AVS_ATOMIC = 0,
  C0IP_AVS_DETERMINISTIC = 1,
  C0IP_AVS_COLORED = 2,
  C0IP_MVS = 3
} c0ip_smoother;

/* Kernel path selection (testing): AUTO picks the fused tile kernels when the level supports
 * them and the generic per-axis kernels otherwise (coarse levels); GENERIC forces the latter. */
typedef enum { C0IP_PATH_AUTO = 0, C0IP_PATH_GENERIC = 1 } c0ip_path;

typedef struct {
  int32_t dim;             /* 2 | 3                                             */
  int32_t degree;          /* k in [2,7] (Q_k)                                    */
  int32_t finest_level;    /* L >= 1: levels 1..L, N_l = 2^l (reading Q9)                      */
  int64_t cells_override;  /* 0, or N for one non-nested level (throughput runs)              */
  double penalty_scale;    /* sigma = penalty_scale * k (k+1) (reading Q4); 0 -> 1;
                              boundary facets use 2 sigma (h_e = h/2, reading Q27)                */
  int32_t device;          /* CUDA device ordinal                                              */
} c0ip_config;

/* Build maps, 1D operators, FDM factors per level and axis variant in FP64
 * and FP32, transfer bands and workspaces.
 * Errors: ARG (bad config), COERCIVITY (1D B or a patch block not SPD: sigma too small,
 * PAPER.md:134-142), OOM, CUDA.  *out is set only on success. */
c0ip_status c0ip_create(const c0ip_config* cfg, c0ip_ctx* out);
c0ip_status c0ip_destroy(c0ip_ctx ctx);

/* As c0ip_create on a graded / anisotropic Cartesian mesh ("the discretization
 * only requires shape regular, locally uniform cells"): nodes[a] (host, a < dim) holds the N+1 cell boundaries
 * 0 = x_0 < ... < x_N = 1 of axis a on the finest level (N = 2^finest_level, or cells_override), NULL = uniform;
 * level l uses every 2^(L-l)-th boundary (nested refinement).  Every cell has its own widths, an
 * interior facet h_e = harmonic mean of the adjacent widths, a boundary facet h_e = h/2 (Q27); the
 * FDM factors are per vertex (no translation invariance) and all operations use the generic per-axis kernels.
 * c0ip_get_fdm and the exact local solver return STATE, the slab calls STATE (no fused level).  ARG for nodes that
 * do not start at 0, end at 1 or increase strictly; the arrays are copied (not retained). */
c0ip_status c0ip_create_graded(const c0ip_config* cfg, const double* const* nodes, c0ip_ctx* out);

/* The comparison workload of PAPER.md:752-816 (Fig. 5): Poisson -Delta u = f, u = 0 weakly,
 * discontinuous Q_k with the symmetric interior penalty method (reading Q30: sigma_P = penalty_scale k(k+1) on
 * interior facets, twice that on boundary facets, h_e = h).  DoFs: N(k+1) Gauss-Lobatto nodes per axis (cell c
 * owns c(k+1)..c(k+1)+k), x fastest, n_dofs = (N(k+1))^d; a vertex patch holds the (2k+2)^d DoFs of its 2^d cells
 * and its operator is exactly L_v (x) M_v + M_v (x) L_v, so the FDM local solve is exact.  Supported: c0ip_apply,
 * c0ip_residual, c0ip_smooth (all smoothers), c0ip_restrict / c0ip_prolongate_add (DG embedding), c0ip_vcycle,
 * c0ip_pcg, c0ip_gmres, c0ip_rhs (f = d pi^2 prod sin(pi x_a)), c0ip_get_fdm (S is (2k+2)^2), c0ip_patch_dofs
 * ((2k+2)^d entries), c0ip_get_matrices_1d (M, L; B = L).  Generic per-axis kernels only; the slab calls and the
 * exact local solver return STATE. */
c0ip_status c0ip_create_sipg(const c0ip_config* cfg, c0ip_ctx* out);
const char* c0ip_last_error(void);
c0ip_status c0ip_set_path(c0ip_ctx ctx, c0ip_path path);

/* Local solver of the vertex-patch smoothers (applies to c0ip_smooth, c0ip_vcycle, c0ip_pcg, c0ip_gmres):
 *  FDM    the separable surrogate A~_v = sum_a B_a (x) M_others solved by fast diagonalisation
 *         (Eq. localsolverbila; the default, Table 2/3);
 *  EXACT  the exact patch matrix A_v = R_v A R_v^T (Table 1), built per
 *         patch variant tuple from the 1D blocks (Eqs. c0iptensorvp(3D)), inverted densely in FP64 on the host
 *         on first use (C0IP_ERR_COERCIVITY if an A_v is not SPD) and applied as a fused gather / DMMA GEMM /
 *         scatter-add (device memory: n_tuples (2k-1)^(2d) doubles per level, owned by the ctx).
 * ARG for an unknown value. */
typedef enum { C0IP_LOCAL_FDM = 0, C0IP_LOCAL_EXACT = 1 } c0ip_local_solver;
c0ip_status c0ip_set_local_solver(c0ip_ctx ctx, c0ip_local_solver solver);

/* Level geometry.  n_dofs = (kN-1)^d, n_1d = kN-1, cells = N, n_patches = (N-1)^d,
 * n_colors = 2^(d+1).  Any output pointer may be NULL. */
c0ip_status c0ip_level_info(c0ip_ctx ctx, int32_t level, int64_t* n_dofs, int64_t* n_1d,
                            int64_t* cells, int64_t* n_patches, int32_t* n_colors);

/* R_v of PAPER.md:206: global DoF ids (host int64 array of length (2k-1)^d, patch-local x fastest)
 * of patch `patch` (id = sum_a (v_a-1)(N-1)^a, reading C2). */
c0ip_status c0ip_patch_dofs(c0ip_ctx ctx, int32_t level, int64_t patch, int64_t* out);

/* Patches of colour `color` (0..2^(d+1)-1, reading C3: 2 * parity class + red-black key,
 * PAPER.md:226-227), ascending patch id, into host array out[cap]; *count = colour size.
 * out may be NULL to query the count.  ARG if cap < count and out != NULL. */
c0ip_status c0ip_color_patches(c0ip_ctx ctx, int32_t level, int32_t color, int64_t* out,
                               int64_t cap, int64_t* count);

/* FDM factors of axis variant (0 left v=1, 1 interior, 2 right v=N-1, 3 both N=2) on `level`:
 * S (host, (2k-1)^2 row-major, column i = i-th generalized eigenvector, S^T M_v S = I) and
 * lambda (host, 2k-1, ascending) of B_v S = M_v S Lambda (reading Q6).
 * STATE if the variant does not exist on this level. */
c0ip_status c0ip_get_fdm(c0ip_ctx ctx, int32_t level, int32_t variant, double* S, double* lambda);

/* Global 1D matrices M, L, B of `level` as dense host arrays n_1d x n_1d
 * (row-major; any pointer may be NULL).  ARG if n_1d > 4096. */
c0ip_status c0ip_get_matrices_1d(c0ip_ctx ctx, int32_t level, double* M, double* L, double* B);

/* F of the paper's solve experiments (readings Q1, Q8b): b_i = int f phi_i with
 * f = Delta^2 u* = d^2 pi^4 prod sin(pi x_a), plus the Nitsche boundary data of u* = prod sin(pi x_a)
 * (u* = 0 on the boundary, d_n u* = g != 0):  sum_{boundary facets} int g ((sigma_b/h) d_n phi_i - d_n^2 phi_i)
 * with sigma_b = 2 sigma (reading Q27), so that the discrete solution converges to u*.  Gauss
 * quadrature with k+3 points per cell and axis.  b: device FP64, length n_dofs. */
c0ip_status c0ip_rhs(c0ip_ctx ctx, int32_t level, double* b, void* stream);

/* y = A x with the matrix-free C0IP operator (Eqs. c0iptensorvp(3D)). */
c0ip_status c0ip_apply(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, const void* x, void* y,
                       void* stream);
/* r = b - A x. */
c0ip_status c0ip_residual(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, const void* b,
                          const void* x, void* r, void* stream);

/* `steps` applications of the smoother with the separable FDM local solver
 * A~_v^{-1} (Eq. localsolverbila) and damping omega; x is updated in place.
 * reverse_colors = 1 processes MVS colours in descending order (symmetric post-smoother,
 * reading Q11); ignored for AVS.  ARG for steps < 0 or bad smoother. */
c0ip_status c0ip_smooth(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, c0ip_smoother sm,
                        int32_t steps, double omega, int32_t reverse_colors, const void* b,
                        void* x, void* stream);

/* coarse = P^T fine (restriction), fine_level >= 2.  coarse has n_dofs(fine_level-1). */
c0ip_status c0ip_restrict(c0ip_ctx ctx, int32_t fine_level, c0ip_dtype dt, const void* fine,
                          void* coarse, void* stream);
/* fine += P coarse (prolongation = natural embedding). */
c0ip_status c0ip_prolongate_add(c0ip_ctx ctx, int32_t fine_level, c0ip_dtype dt,
                                const void* coarse, void* fine, void* stream);

typedef struct {
  c0ip_smoother smoother;
  int32_t steps;           /* pre- and post-smoothing steps                    */
  double omega;            /* damping                             */
  int32_t symmetric;       /* MVS: post-smoothing in reversed colour order (reading Q11)        */
  c0ip_dtype cycle_dtype;  /* F32: V-cycle entirely in single precision          */
} c0ip_mg_config;

/* z = MG_L(0, r) (Algorithm 1, PAPER.md:158-176 with readings Q12, Q13): r, z device FP64 of the
 * finest level; with cycle_dtype F32, r is converted at entry and z at exit.
 * STATE if the context has a single (override) level. */
c0ip_status c0ip_vcycle(c0ip_ctx ctx, const c0ip_mg_config* mg, const double* r, double* z,
                        void* stream);

typedef struct {
  int32_t iterations, converged;
  double r0, rn, nu, seconds;
} c0ip_report;

/* MG-preconditioned CG in FP64: x (device FP64, in: x0, out: solution),
 * b device FP64.  Stops when ||r_n|| <= rtol ||r_0|| (recursively updated residual) or after
 * max_iter iterations (not an error: converged = 0).  nu = -8/log10((r_n/r_0)^(1/n)) (reading Q7).
 * res_history: optional host array of max_iter+1 doubles (||r_0||..||r_n||). */
c0ip_status c0ip_pcg(c0ip_ctx ctx, const c0ip_mg_config* mg, const double* b, double* x,
                     double rtol, int32_t max_iter, c0ip_report* rep, double* res_history,
                     void* stream);

/* MG-preconditioned flexible GMRES(m) in FP64 (GMRES is the paper's
 * outer solver for the multiplicative smoother, whose same-order V-cycle (mg->symmetric = 0) is not
 * symmetric).  Right preconditioning z_j = MG(v_j) (c0ip_vcycle), Arnoldi by classical Gram-Schmidt with one
 * re-orthogonalisation (CGS2: batched projections, three host round trips per step),
 * Givens rotations, restart after `restart` steps (the device holds restart+1 Krylov vectors and
 * restart preconditioned vectors of the finest level: (2 restart + 2) * 8 n bytes, owned by the ctx).
 * x (device FP64, in: x0, out: solution), b device FP64.  Stops when the least-squares residual
 * |g_{j+1}| <= rtol ||r_0|| (the least-squares residual, as PCG uses its recursive residual) or
 * after max_iter Arnoldi steps (not an error: converged = 0).
 * rep->rn is the true residual norm ||b - A x|| at exit; res_history (optional host array of
 * max_iter+1 doubles) holds ||r_0||, |g_1|, ..., |g_n|.  ARG for restart < 1, max_iter < 0, rtol < 0. */
c0ip_status c0ip_gmres(c0ip_ctx ctx, const c0ip_mg_config* mg, const double* b, double* x,
                       double rtol, int32_t max_iter, int32_t restart, c0ip_report* rep,
                       double* res_history, void* stream);

/* ---- Slab (multi-GPU) entry points, SURVEY.md §8e -------------------------------------------------
 * The mesh is split into slabs along the slowest axis (y in 2D, z in 3D); each rank (one process per
 * GPU) holds a window of global interior rows [row0, row0 + lrows) of that axis in a contiguous array
 * (a "row" is n_1d^(d-1) values, x fastest) and owns the node rows [out_lo, out_hi) (node row
 * j = interior row + 1).  The caller fills the ghost rows of x_ext before each call (halo exchange, e.g.
 * NCCL send/recv through torch.distributed; paper_2412_05082_b200/dist.py).  Results are bitwise equal
 * to the single-domain call on the owned rows.  STATE if the level has no slab-capable kernel (2D levels
 * with N >= 8, 3D levels with N >= 8 and k <= 5 in this release). */

/* Ghost rows a slab call needs on each side of [out_lo, out_hi) (clipped at the domain boundary):
 * AVS step: 4k-2 (residual on the owned rows +- (2k-2), each needing x +- 2k); apply: 2k. */
c0ip_status c0ip_slab_ghosts(c0ip_ctx ctx, int32_t* ghost_avs, int32_t* ghost_apply);

/* One additive smoothing step on the owned rows: r_ext (scratch, same window) gets
 * b - A x on the owned rows +- (2k-2), then x_ext is updated in place on the owned rows.  b_ext may be
 * NULL-free only; ARG if the window does not hold the required ghost rows. */
c0ip_status c0ip_slab_avs_step(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, double omega, int64_t row0,
                               int64_t lrows, int64_t out_lo, int64_t out_hi, const void* b_ext,
                               void* x_ext, void* r_ext, void* stream);

/* The update half of c0ip_slab_avs_step: x_ext += omega sum_v R_v^T A~_v^{-1} R_v r on the owned rows [out_lo,
 * out_hi), reading r_ext on the owned rows +- (2k-2) (which the caller computed with c0ip_slab_apply).  Splitting
 * the step as residual(interior rows) | halo exchange | residual(boundary rows) | c0ip_slab_fdm overlaps the
 * exchange with the interior residual and gives the same owned rows as c0ip_slab_avs_step, bitwise. */
c0ip_status c0ip_slab_fdm(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, double omega, int64_t row0, int64_t lrows,
                          int64_t out_lo, int64_t out_hi, const void* r_ext, void* x_ext, void* stream);

/* y = A x (b_ext == NULL) or r = b - A x on the owned rows of a slab window (ghosts of width 2k). */
c0ip_status c0ip_slab_apply(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, int64_t row0, int64_t lrows,
                            int64_t out_lo, int64_t out_hi, const void* b_ext, const void* x_ext,
                            void* y_ext, void* stream);

/* One colour of the multiplicative smoother on a slab (SURVEY.md §8e "colours are processed in
 * lockstep across ranks"): every patch of `color` whose DoF rows meet the owned node rows [out_lo, out_hi) is
 * solved (residual on its footprint, FDM, update of its DoFs).  Patches straddling a slab boundary are solved
 * redundantly by both neighbours from identical inputs, so after the call the owned rows equal the single-domain
 * colour step bitwise; rows outside the owned range are ghost copies (refresh them by the next exchange).  The
 * caller exchanges the 4k-2 ghost rows of x_ext before every colour.  r_ext: scratch of the window's size.
 * ARG: bad colour / window; STATE with the exact local solver. */
c0ip_status c0ip_slab_mvs_color(c0ip_ctx ctx, int32_t level, c0ip_dtype dt, double omega, int32_t color,
                                int64_t row0, int64_t lrows, int64_t out_lo, int64_t out_hi, const void* b_ext,
                                void* x_ext, void* r_ext, void* stream);

/* Windowed transfers between a nested level pair: coarse node rows [c_out_lo, c_out_hi) of
 * P^T fine from a fine window (restrict), and fine node rows [f_out_lo, f_out_hi) += P coarse from a coarse
 * window (prolongate_add).  Windows as above (row0 = global interior row of local row 0, lrows rows).
 * c0ip_slab_transfer_rows reports the node-row ranges [need[0], need[1]) each call reads (fine rows for the
 * restriction of the coarse owned rows, coarse rows for the prolongation onto the fine owned rows).
 * ARG if a window misses rows it needs; STATE without a coarser nested level. */
c0ip_status c0ip_slab_restrict(c0ip_ctx ctx, int32_t fine_level, c0ip_dtype dt, int64_t f_row0, int64_t f_lrows,
                               const void* fine_ext, int64_t c_row0, int64_t c_lrows, int64_t c_out_lo,
                               int64_t c_out_hi, void* coarse_ext, void* stream);
c0ip_status c0ip_slab_prolongate_add(c0ip_ctx ctx, int32_t fine_level, c0ip_dtype dt, int64_t c_row0,
                                     int64_t c_lrows, const void* coarse_ext, int64_t f_row0, int64_t f_lrows,
                                     int64_t f_out_lo, int64_t f_out_hi, void* fine_ext, void* stream);
c0ip_status c0ip_slab_transfer_rows(c0ip_ctx ctx, int32_t fine_level, int64_t c_out_lo, int64_t c_out_hi,
                                    int64_t f_out_lo, int64_t f_out_hi, int64_t* fine_need, int64_t* coarse_need);

/* z = MG_level(0, r) (Algorithm 1 from an inner level): the replicated coarse part of the
 * distributed V-cycle (every rank runs it on the gathered coarse residual).  r, z: device FP64 of n_dofs(level);
 * the cycle dtype conversion as in c0ip_vcycle.  Not graph-captured. */
c0ip_status c0ip_vcycle_level(c0ip_ctx ctx, const c0ip_mg_config* mg, int32_t level, const double* r, double* z,
                              void* stream);

/* Vector kernels of the distributed Krylov drivers (the solver arithmetic stays in this library):
 * y = alpha x + beta y (n elements, device, dtype dt; beta = 0 does not read y), and up to two FP64 dot
 * products <x0,y0>, <x1,y1> over n elements (deterministic two-pass reduction; out: host array of ndots,
 * the call synchronises the stream).  The cross-rank sum is the caller's all-reduce. */
c0ip_status c0ip_vec_axpby(c0ip_ctx ctx, c0ip_dtype dt, int64_t n, double alpha, const void* x, double beta,
                          void* y, void* stream);
c0ip_status c0ip_vec_dots(c0ip_ctx ctx, int64_t n, int32_t ndots, const double* x0, const double* y0,
                          const double* x1, const double* y1, double* out, void* stream);

/* Number of kernels this context has launched since creation (for the bench's gpu_launches). */
c0ip_status c0ip_launch_count(c0ip_ctx ctx, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* C0IP_H */
