/* rhosolve-b200 C ABI.
 *
 * The drop-in boundary for the steady-state hot path of the reference
 * `rhosolve` package (arXiv 1504.06768).  The reference's own native seam is
 * its kernel module (pkg/src/rhosolve/kernels/__init__.py:19-36), four
 * functions bound from Cython: csr_matvec, lower_solve, upper_solve and
 * factorize (_ckernels.pyx:34,53,70,144).  This library exports device
 * equivalents of those four plus the other stages of the path
 * (liouville.py assembly/shift/modify, ordering.rcm, sparse.permute,
 * factor.solve_lu, the krylov / steady drivers and _postprocess), each citing
 * the reference interface it replaces.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers (cudaMalloc / torch tensors),
 *     except where a parameter is documented as host.
 *   - complex128 is rs_complex {double re, im;}: the numpy complex128 layout.
 *   - Indices are int32 (every configuration has nnz < 2^31).
 *   - Batches: `nsys` independent systems of equal order n are stored
 *     block-diagonally.  row_ptr spans nsys*n rows with absolute positions,
 *     column indices are local (0..n-1), vectors are nsys*n long.  A single
 *     system is nsys = 1.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).
 *   - Every function returns 0 (RS_OK) or a negative RS_ERR_* code and never
 *     throws; rs_last_error() describes the last failure of this thread.
 *     Numerical outcomes the reference reports as values (zero pivot step,
 *     Krylov breakdown, ...) are returned through output arguments, exactly
 *     as the reference returns them (fail_col, IterResult flags).
 *   - No function falls back to a CPU implementation.
 */
#ifndef RHOSOLVE_B200_H
#define RHOSOLVE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RS_ABI_VERSION 2

#define RS_OK 0
#define RS_ERR_ARG -1
#define RS_ERR_CUDA -2
#define RS_ERR_ALLOC -3
#define RS_ERR_BREAKDOWN -4
#define RS_ERR_NONFINITE -5
#define RS_ERR_OVERFLOW -6
#define RS_ERR_UNSUPPORTED -7
#define RS_ERR_STRUCT_SINGULAR -8

typedef struct rs_complex {
  double re;
  double im;
} rs_complex;

int rs_abi_version(void);
const char* rs_last_error(void);
/* Number of kernels this library has launched in the process (bench
 * bookkeeping: gpu_launches). */
long long rs_launch_count(void);
/* ---- 'cmd' ordering (host-native; steady._prepare, steady.py:95-107) -----
 * Both take HOST arrays: the CSR of a square matrix (int64 row_ptr[n+1] /
 * col_idx, complex128 values), as the reference's SparseComplexMatrix holds
 * it.  The algorithms are greedy and sequential, so they run on the host
 * once per structure; the elimination they order runs on the GPU. */

/* Replaces ordering.weighted_mbm (ordering.py:121-218): forward[r] = the
 * position row r moves to (a zero-free structural diagonal); weight-guided
 * column BFS from the largest |a_ij| (numpy complex abs = hypot), greedy
 * largest-|value| matching, completed by BFS augmenting paths.  Returns
 * RS_ERR_STRUCT_SINGULAR (StructurallySingularError) when no perfect
 * matching exists. */
int rs_weighted_mbm_host(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                         const rs_complex* values, int64_t* forward);

/* Replaces ordering.col_min_degree (ordering.py:221-282): exact greedy
 * minimum degree on the column-intersection graph (quotient form), ties to
 * the lowest column; order[k] = the k-th eliminated column
 * (Permutation.from_order(order)). */
int rs_col_min_degree_host(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                           int64_t* order);

/* Number of systems the last rs_factorize call factored with the
 * right-looking frontal kernel (complete LU whose front fits shared memory;
 * batches of <= 3 waves by default, RHOSOLVE_FRONTAL=1/0 forces it on/off;
 * diagnostics and tests). */
int rs_debug_frontal_taken(void);

/* ---- kernel seam (kernels/__init__.py:19-36) ---------------------------- */

/* y = A x.  Replaces csr_matvec (_ckernels.pyx:34-50): row-sequential sum,
 * plain complex products, empty rows give 0 -- bit-identical. */
int rs_csr_matvec(int32_t nsys, int32_t n, const int32_t* row_ptr,
                  const int32_t* col_idx, const rs_complex* values,
                  const rs_complex* x, rs_complex* y, void* stream);

/* Left-looking LU / ILUTP.  Replaces factorize (_ckernels.pyx:144-385) as
 * called by factor._factor (factor.py:70-112).
 *   A is given column-major: Ap/Ai/Ax = CSR of A^T (sparse.transpose(a)),
 *   q (nullable) = elimination column order, drop_tol, fill_cap (-1 = none)
 *   or fill_caps (nullable device int32[nsys], one cap per system: batches
 *   whose systems differ in nnz, e.g. block-Jacobi blocks),
 *   row_norms (nullable unless drop_tol > 0) = max |re|+|im| per row.
 * Outputs per system b (raw CSC exactly as the reference returns them):
 *   Lp/Up [nsys*(n+1)], Li/Lx at b*capL, Ui/Ux at b*capU, pinv [nsys*n].
 * state (device, int32 [3*nsys]) must be zeroed before the first call:
 *   state[3b] = 1 done, 2 zero pivot (state[3b+1] = fail_col, the
 *   reference's return value), 3 out of capacity (state[3b+1] = column to
 *   resume from: grow the buffers, copy, call again with the same state).
 * L row indices are remapped to pivotal order on completion, as in the
 * reference. */
int rs_factorize(int32_t nsys, int32_t n, const int32_t* Ap, const int32_t* Ai,
                 const rs_complex* Ax, const int32_t* q, double drop_tol,
                 int32_t fill_cap, const int32_t* fill_caps, const double* row_norms,
                 int32_t* Lp,
                 int32_t* Li, rs_complex* Lx, int64_t capL, int32_t* Up,
                 int32_t* Ui, rs_complex* Ux, int64_t capU, int32_t* pinv,
                 int32_t* state, void* stream);

/* rs_factorize with two opt-in extensions that the reference does NOT have
 * (used only by the block-Jacobi preconditioner of config 5; both off is
 * rs_factorize exactly):
 *   pivot_floor > 0: a diagonal block of the RCM-ordered matrix can reach a
 *     column with no usable pivot although the whole matrix factors; such a
 *     column takes the real value pivot_floor as its pivot, on the lowest
 *     non-pivotal row of its pattern, or, when the pattern has none, on the
 *     lowest row not yet pivotal.  state[3b+2] counts the substitutions.
 *   early_drop != 0: a U entry below the drop threshold (|x| < drop_tol *
 *     rownorm when its column is reached) is discarded BEFORE it eliminates
 *     (Saad's ILUT rule); the reference eliminates with it and drops it at
 *     the end of the column.  Cuts the pre-drop fill cascade of wide bands. */
int rs_factorize_opts(int32_t nsys, int32_t n, const int32_t* Ap, const int32_t* Ai,
                       const rs_complex* Ax, const int32_t* q, double drop_tol,
                       int32_t fill_cap, const int32_t* fill_caps, const double* row_norms,
                       int32_t* Lp, int32_t* Li, rs_complex* Lx, int64_t capL, int32_t* Up,
                       int32_t* Ui, rs_complex* Ux, int64_t capU, int32_t* pinv,
                       int32_t* state, double pivot_floor, int32_t early_drop, void* stream);

/* Row-oriented triangular factors for the solves.  From the raw CSC of
 * rs_factorize, builds the strictly-lower L and strictly-upper U in CSR
 * (ascending columns) plus rdiag = recipc(U_kk).  Call with L_ci == NULL to
 * get only the row pointers and *L_nnz / *U_nnz (host) for allocation. */
int rs_factor_rows(int32_t nsys, int32_t n, const int32_t* Lp, const int32_t* Li,
                   const rs_complex* Lx, int64_t capL, const int32_t* Up,
                   const int32_t* Ui, const rs_complex* Ux, int64_t capU,
                   int32_t* L_rp, int32_t* L_ci, rs_complex* L_v, int64_t* L_nnz,
                   int32_t* U_rp, int32_t* U_ci, rs_complex* U_v,
                   rs_complex* rdiag, int64_t* U_nnz, void* stream);

/* SELL-32 copy of a row-oriented triangular factor from rs_factor_rows for
 * the lane-per-row sweeps: sweep order q (L: row q; U: row n-1-q), slice s =
 * positions 32s..32s+31, entry k of lane l at sptr[s] + 32k + l, terms in the
 * reference fold order (L ascending, U descending column; _ckernels.pyx:
 * 53-85), padding column -1.  sptr has nsys*ceil(n/32)+1 entries (absolute).
 * Call with sci == NULL to fill sptr and *total (host), then again to fill. */
int rs_sell_build(int32_t nsys, int32_t n, int32_t upper, const int32_t* rp,
                  const int32_t* ci, const rs_complex* v, int32_t* sptr, int32_t* sci,
                  rs_complex* sv, int64_t* total, void* stream);

/* rdiag[b*n + k] = recipc(U_kk) (_ckernels.pyx:25-31, 70-85) from the raw
 * CSC U of rs_factorize (pivot = last entry of each column). */
int rs_pivot_recip(int32_t nsys, int32_t n, const int32_t* Up, const rs_complex* Ux,
                   int64_t capU, rs_complex* rdiag, void* stream);

/* 1 when systems of order n run the column-oriented sweeps (the factor
 * staging ring fits one CTA's shared memory; the sweep vector is kept there
 * too when it fits, else in global memory), else 0. */
int rs_col_sweep_supported(int32_t n);

/* Column stream of one triangle of the raw CSC factors (rs_factorize) for
 * the column-oriented sweeps: columns in sweep order j (L: column j; U:
 * column n-1-j), each column's off-diagonal entries padded to whole 64-entry
 * rows (index -1 = padding; idx/val hold 64 * rows entries); meta[row] = 1 when the row continues the
 * previous column; for U, rrd[first row of column c] = rdiag[c].  rowoff
 * (nsys*n+1, absolute) gives each column's first row.  Call with idx ==
 * NULL to fill rowoff and *total_rows (host), then again to fill. */
int rs_col_stream_build(int32_t nsys, int32_t n, int32_t upper, const int32_t* cp,
                        const int32_t* ci, const rs_complex* cv, int64_t cap,
                        const rs_complex* rdiag, int32_t* rowoff, int32_t* idx,
                        rs_complex* val, int32_t* meta, rs_complex* rrd, int64_t* total_rows,
                        void* stream);

/* x = M^{-1} b through the column streams: y[pinv] = b, then the reference
 * lower_solve / upper_solve column loops (_ckernels.pyx:53-85) verbatim on
 * shared memory; bit-identical.  Requires rs_col_sweep_supported(n). */
int rs_lu_solve_cols(int32_t nsys, int32_t n, const int32_t* pinv, const int32_t* Ls_rowoff,
                     const int32_t* Ls_idx, const rs_complex* Ls_val, const int32_t* Ls_meta,
                     const int32_t* Us_rowoff, const int32_t* Us_idx, const rs_complex* Us_val,
                     const int32_t* Us_meta, const rs_complex* Us_rd, const rs_complex* b,
                     rs_complex* x, void* stream);

/* rs_lu_solve_cols with the factors' reach (max |row - column| over the entries
 * of L and U; see rs_solver_args.col_reach) so that a system too large for
 * shared memory sweeps through the sliding window.  reach = 0: rs_lu_solve_cols. */
int rs_lu_solve_cols_reach(int32_t nsys, int32_t n, const int32_t* pinv,
                           const int32_t* Ls_rowoff, const int32_t* Ls_idx,
                           const rs_complex* Ls_val, const int32_t* Ls_meta,
                           const int32_t* Us_rowoff, const int32_t* Us_idx,
                           const rs_complex* Us_val, const int32_t* Us_meta,
                           const rs_complex* Us_rd, const rs_complex* b, rs_complex* x,
                           int32_t reach, void* stream);

/* x = M^{-1} b through the factors: y[pinv] = b; lower_solve; upper_solve;
 * x = y.  Replaces factor.solve_lu (factor.py:137-149) with
 * lower_solve/upper_solve (_ckernels.pyx:53-85); bit-identical. */
int rs_lu_solve(int32_t nsys, int32_t n, const int32_t* pinv, const int32_t* L_rp,
                const int32_t* L_ci, const rs_complex* L_v, const int32_t* U_rp,
                const int32_t* U_ci, const rs_complex* U_v, const rs_complex* rdiag,
                const rs_complex* b, rs_complex* x, void* stream);

/* In-place y <- L^{-1} y on the raw CSC L of rs_factorize (unit diagonal
 * first, pivotal row indices).  Replaces lower_solve (_ckernels.pyx:53-67),
 * the third function of the kernel seam; bit-identical.  cap = entries
 * between consecutive systems' Li/Lx (any value when nsys == 1).  Stream-
 * ordered: no allocation, no synchronisation. */
int rs_lower_solve(int32_t nsys, int32_t n, const int32_t* Lp, const int32_t* Li,
                   const rs_complex* Lx, int64_t cap, rs_complex* y, void* stream);

/* In-place y <- U^{-1} y on the raw CSC U (pivot last in each column):
 * x_c = y_c * recipc(U_cc), then the column scatter.  Replaces upper_solve
 * (_ckernels.pyx:70-85), the fourth function of the kernel seam;
 * bit-identical. */
int rs_upper_solve(int32_t nsys, int32_t n, const int32_t* Up, const int32_t* Ui,
                   const rs_complex* Ux, int64_t cap, rs_complex* y, void* stream);

/* ---- superoperator (liouville.py) ---------------------------------------- */

/* build_liouvillian (liouville.py:54-77), bit-identical structure and values.
 * H and the K collapse operators are D x D CSR on the device; C_rp/C_ci/C_v/
 * C_nnz are HOST arrays of K device pointers / sizes.  *herm_dev (host)
 * receives max|H - H^dag| (the reference rejects H above 1e-12).
 * Two passes: with out_ci == NULL fills out_rp and *nnz (host); then call
 * again with out_ci/out_v allocated for *nnz entries. */
int rs_liouvillian(int32_t D, const int32_t* H_rp, const int32_t* H_ci,
                   const rs_complex* H_v, int64_t H_nnz, int32_t K,
                   const int32_t* const* C_rp, const int32_t* const* C_ci,
                   const rs_complex* const* C_v, const int64_t* C_nnz,
                   double* herm_dev, int32_t* out_rp, int32_t* out_ci,
                   rs_complex* out_v, int64_t* nnz, void* stream);

/* build_liouvillian for nsys systems of equal dimension and operator count in
 * ONE launch set (the config-4 sweep: 512 instances): H and every C_k are
 * block-diagonal batches (row pointers over nsys*D rows with absolute
 * positions, local column indices; H_nnz / C_nnz = entries of the whole
 * batch).  out_rp spans nsys*D*D rows -- the batch layout of every other entry
 * point.  *herm_dev = max over the batch.  Two passes as rs_liouvillian;
 * bit-identical per system. */
int rs_liouvillian_batch(int32_t nsys, int32_t D, const int32_t* H_rp, const int32_t* H_ci,
                         const rs_complex* H_v, int64_t H_nnz, int32_t K,
                         const int32_t* const* C_rp, const int32_t* const* C_ci,
                         const rs_complex* const* C_v, const int64_t* C_nnz, double* herm_dev,
                         int32_t* out_rp, int32_t* out_ci, rs_complex* out_v, int64_t* nnz,
                         void* stream);

/* shift (liouville.py:80-96): L - sigma I, every diagonal stored.  Two passes
 * as above (out_ci == NULL: row pointers and *nnz only). */
int rs_shift(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci,
             const rs_complex* v, double sigma, int32_t* out_rp, int32_t* out_ci,
             rs_complex* out_v, int64_t* nnz, void* stream);

/* default_weight (liouville.py:99-111), one weight per system into w (device).
 * mode 0 = "abs", 1 = "signed". */
int rs_default_weight(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci,
                      const rs_complex* v, int32_t mode, double* w, void* stream);

/* build_modified (liouville.py:114-138): row 0 += w at columns k(D+1).
 * w is a device array of nsys weights.  Two passes as above. */
int rs_trace_modify(int32_t nsys, int32_t n, int32_t D, const int32_t* rp,
                    const int32_t* ci, const rs_complex* v, const double* w,
                    int32_t* out_rp, int32_t* out_ci, rs_complex* out_v,
                    int64_t* nnz, void* stream);

/* ---- ordering and permutation -------------------------------------------- */

/* ordering.rcm (ordering.py:82-118), bit-identical: forward/inverse int32
 * [nsys*n], local indices (Permutation.forward / .inverse). */
int rs_rcm(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci,
           int32_t* forward, int32_t* inverse, void* stream);

/* Batch helper (no reference counterpart: the reference orders one matrix at
 * a time, ordering.py:82-118).  *same (device int32) becomes 1 when every
 * system of the block-diagonal batch stores exactly system 0's pattern (row
 * extents and column indices; values may differ), else 0 -- the config-4
 * sweep, which is then ordered once (`rs_rcm` on system 0) and the
 * permutation replicated.  nnz = entries of the whole batch. */
int rs_same_pattern(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci, int64_t nnz,
                    int32_t* same, void* stream);

/* sparse.permute(a, p, p) (sparse.py:276-282): B[f[i], f[j]] = A[i, j]. */
int rs_permute(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci,
               const rs_complex* v, const int32_t* forward, const int32_t* inverse,
               int32_t* out_rp, int32_t* out_ci, rs_complex* out_v, void* stream);

/* sparse.permute(a, row_perm, col_perm) with distinct permutations
 * (sparse.py:276-282): B[rf[i], cf[j]] = A[i, j], given rf^-1 (row_inverse)
 * and cf (col_forward), per system.  The 'cmd' path uses it for the MBM row
 * permutation and the minimum-degree column order. */
int rs_permute_rows_cols(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci,
                         const rs_complex* v, const int32_t* row_inverse,
                         const int32_t* col_forward, int32_t* out_rp, int32_t* out_ci,
                         rs_complex* out_v, void* stream);

/* gather != 0: out[i] = x[forward[i]] (solution unpermute, steady.py:249-250);
 * gather == 0: out[forward[i]] = x[i] (rhs permute, steady.py:89-94). */
int rs_permute_vector(int32_t nsys, int32_t n, const rs_complex* x,
                      const int32_t* forward, rs_complex* out, int32_t gather,
                      void* stream);

/* CSR transpose (sparse.transpose, sparse.py:216-219); values nullable. */
int rs_transpose(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci,
                 const rs_complex* v, int32_t* out_rp, int32_t* out_ci,
                 rs_complex* out_v, void* stream);

/* factor.py:84-88: row_norms[r] = max |re|+|im| over row r. */
int rs_row_norms(int32_t nsys, int32_t n, const int32_t* rp, const rs_complex* v,
                 double* row_norms, void* stream);

/* ---- steady-state drivers (steady.py / krylov.py) ------------------------- */

enum rs_solve_mode {
  RS_INV_DIRECT = 0,   /* inverse_power(inner="direct")          steady.py:203-208 */
  RS_INV_BICGSTAB = 1, /* inverse_power(inner="iterative", "bicgstab") */
  RS_INV_GMRES = 2,    /* inverse_power(inner="iterative", "gmres")    */
  RS_LIN_DIRECT = 3,   /* solve_direct: one solve_lu                steady.py:116-134 */
  RS_LIN_BICGSTAB = 4, /* solve_iterative(solver="bicgstab")       steady.py:137-168 */
  RS_LIN_GMRES = 5     /* solve_iterative(solver="gmres")          */
};

/* status codes written to rs_solve_stats.status */
enum rs_solve_status {
  RS_SOLVE_OK = 0,
  RS_SOLVE_INNER_BREAKDOWN = 1,   /* InnerSolverError, steady.py:218-222 */
  RS_SOLVE_INNER_NONFINITE = 2,   /* InnerSolverError, steady.py:218-222 */
  RS_SOLVE_INNER_NO_PROGRESS = 3, /* InnerSolverError, steady.py:223-224 */
  RS_SOLVE_UNUSABLE_VECTOR = 4,   /* InnerSolverError, steady.py:234-235 */
  RS_SOLVE_POWER_NOT_CONVERGED = 5, /* PowerIterationError, steady.py:246-248 */
  RS_SOLVE_SKIPPED = 6              /* masked out by rs_solver_args.skip */
};

typedef struct rs_solve_stats {
  int32_t status;
  int32_t outer;       /* inverse-power outer iterations */
  int32_t inner_last;  /* Krylov iterations of the last inner solve */
  int32_t inner_total;
  int32_t converged;   /* IterResult.converged (linear modes) */
  int32_t breakdown;   /* IterResult.breakdown (linear modes) */
  double final_residual;
  double condest;      /* factor.condest (factor.py:152-157) when requested */
} rs_solve_stats;

typedef struct rs_solver_args {
  int32_t n;
  int32_t nsys;
  int32_t mode;    /* rs_solve_mode */
  int32_t threads; /* CTA size, multiple of 32, <= 512 (0 = 512; the Python layer
                      passes 128 for batches of more than 148 systems, else 256) */
  /* solver-ready (shifted or modified), ordered system matrix */
  const int32_t* A_rp;
  const int32_t* A_ci;
  const rs_complex* A_v;
  /* plain ordered matrix, for the inverse-power residual test */
  const int32_t* P_rp;
  const int32_t* P_ci;
  const rs_complex* P_v;
  /* preconditioner from rs_factor_rows (all NULL: no preconditioner) */
  const int32_t* L_rp;
  const int32_t* L_ci;
  const rs_complex* L_v;
  const int32_t* U_rp;
  const int32_t* U_ci;
  const rs_complex* U_v;
  const rs_complex* rdiag;
  const int32_t* pinv;
  const rs_complex* rhs; /* rhs (linear) or un-normalised start vector (inverse power) */
  rs_complex* x;         /* solution in the ordered coordinates */
  rs_solve_stats* stats; /* device, nsys entries */
  double tol;
  int32_t max_iter;
  int32_t restart_m;
  int32_t max_outer;
  int32_t want_condest;
  /* optional column streams of L and U from rs_col_stream_build.  When set
   * and rs_col_sweep_supported(n), the preconditioner apply runs the
   * reference's column-oriented lower/upper solves on shared memory and
   * L_rp..U_v may be NULL (rdiag is still required); otherwise the
   * row-oriented factors above are required. */
  const int32_t* Ls_rowoff;
  const int32_t* Ls_idx;
  const rs_complex* Ls_val;
  const int32_t* Ls_meta;
  const int32_t* Us_rowoff;
  const int32_t* Us_idx;
  const rs_complex* Us_val;
  const int32_t* Us_meta;
  const rs_complex* Us_rd;
  /* optional column pre-ordering of the preconditioner (factor.py:76-78,
   * 147-148): the factors are those of A[:, q] and every apply ends with
   * x[q] = y, i.e. x[j] = y[colp[j]] with colp = col_perm.forward (device
   * int32 [nsys*n], local indices).  NULL: identity.  A, P, rhs and x stay in
   * the caller's (unpermuted) column coordinates, exactly as in the
   * reference's krylov / steady drivers. */
  const int32_t* colp;
  /* optional per-system mask (device int32 [nsys]): systems with skip[b] != 0
   * (e.g. a zero pivot in their factorization) are not solved; their stats
   * report RS_SOLVE_SKIPPED and x is zeroed.  NULL: solve every system. */
  const int32_t* skip;
  /* optional residual history of system 0 in the linear modes -- the rows the
   * reference's gmres/bicgstab write to their `trace` stream (krylov.py:62-64,
   * 152, 228): trace[2k] = iteration, trace[2k+1] = monitored residual,
   * k < min(*trace_count, trace_cap).  Device pointers; NULL: not recorded. */
  double* trace;
  int32_t* trace_count;
  int32_t trace_cap;
  /* optional: max |row - column| over the entries of both factors (their
   * bandwidth in pivotal coordinates; 0 = unknown).  A lone system too large
   * for shared memory then sweeps through a sliding shared-memory window with
   * several consumer warps instead of through global memory. */
  int32_t col_reach;
} rs_solver_args;

/* One launch runs the whole solve of every system on the device. */
int rs_steady_solve(const rs_solver_args* args, void* stream);

/* steady._postprocess (steady.py:62-71) with the optional unpermute:
 * rho (D x D row-major per system), residual (device, nsys doubles),
 * trace (device, nullable).  forward == NULL on the natural ordering. */
int rs_postprocess(int32_t nsys, int32_t D, const rs_complex* x,
                   const int32_t* forward, const int32_t* plain_rp,
                   const int32_t* plain_ci, const rs_complex* plain_v,
                   rs_complex* rho, double* residual, rs_complex* trace,
                   void* stream);

/* ---- grid-wide solver for large systems (config 3, config 5) --------------
 * One cooperative launch runs the whole solve on every SM: SpMV, the
 * preconditioner apply as sync-free level-ordered triangular sweeps
 * (bit-identical to lower_solve / upper_solve, _ckernels.pyx:53-85),
 * deterministic grid-wide reductions and the reference's BiCGStab / GMRES /
 * inverse-power control flow (krylov.py:67-291, steady.py:177-260). */

/* Dependency levels of a triangular factor (upper = 0: L, 1: U): level[b*n +
 * i] = 1 + the largest level among the rows that row i's off-diagonal columns
 * name (0 when it has none); *nlevels (host) = number of levels.  rp = row
 * pointers of the row-oriented factor (rs_factor_rows: the dependency counts);
 * cp / ri / cap = column pointers, row indices and per-system stride of the
 * raw CSC factor of rs_factorize (column c lists the rows depending on c). */
int rs_tri_levels(int32_t nsys, int32_t n, int32_t upper, const int32_t* rp, const int32_t* cp,
                  const int32_t* ri, int64_t cap, int32_t* level, int64_t* nlevels,
                  void* stream);

/* Rows sorted by (level, longest row first, row) with every level padded to a
 * multiple of H rows (H = 32 / lanes-per-row: 32, 16, 8 or 1): order[pos] = global
 * row b*n + i, or -1 for padding.  rp = the row-oriented factor's row
 * pointers.  order must hold nsys*n + H*nlevels entries; *npos (host) =
 * positions used (a multiple of H). */
int rs_tri_order(int32_t nsys, int32_t n, const int32_t* level, const int32_t* rp,
                 int64_t nlevels, int32_t H, int32_t* order, int64_t* npos, void* stream);

/* Level-ordered SELL copy of the factor: slice s = positions H*s..H*s+H-1;
 * lane r*G + j (G = 32/H) holds entries j, j+G, ... of the slice's r-th row in
 * the reference fold order (L ascending, U descending column), entry (k, lane)
 * at sptr[s] + 32k + lane, global column indices, -1 = padding; skey holds, for
 * every chunk of 8 steps of every slice, the chunk's dependency of the highest
 * level (the one the slice's warp watches), -1 when it has none.  Two passes:
 * sci == NULL fills sptr[npos/H + 1] and *total (host); the second (with
 * *total as returned) fills sci / sv / skey[rs_tri_sell_keys(total, npos/H)]. */
int rs_tri_sell(int32_t nsys, int32_t n, int32_t upper, const int32_t* rp, const int32_t* ci,
                const rs_complex* v, const int32_t* order, int64_t npos, int32_t H,
                const int32_t* level, int32_t* sptr, int32_t* sci, rs_complex* sv,
                int32_t* skey, int64_t* total, void* stream);

/* Entries of rs_tri_sell's skey array. */
int64_t rs_tri_sell_keys(int64_t total, int64_t nslices);

typedef struct rs_tri_factor {
  const int32_t* order;
  const int32_t* sptr;
  const int32_t* sci;
  const rs_complex* sv;
  const int32_t* skey;
  int32_t nslices;       /* npos / H */
  int32_t lanes_per_row; /* G = 32 / H: 1, 2, 4 or 32 */
  int32_t active_warps;  /* warps per CTA that sweep (0 = all): the window of slices
                            in flight; narrow DAGs want few (fewer pollers) */
  int32_t reserved;
} rs_tri_factor;

typedef struct rs_grid_args {
  int32_t n;    /* order of the whole system */
  int32_t nb;   /* order of one preconditioner block (block-Jacobi: n = blocks * nb;
                   a single factorization: nb = n) */
  int32_t mode; /* rs_solve_mode */
  int32_t want_condest;
  /* solver-ready ordered system matrix and (inverse power) the plain one: n x n CSR */
  const int32_t* A_rp;
  const int32_t* A_ci;
  const rs_complex* A_v;
  const int32_t* P_rp;
  const int32_t* P_ci;
  const rs_complex* P_v;
  /* preconditioner (L.order == NULL: none) */
  rs_tri_factor L;
  rs_tri_factor U;
  const rs_complex* rdiag; /* recipc(U_cc), rs_pivot_recip */
  const int32_t* pinv;     /* row permutation of the factors, local to each block */
  const int32_t* colp;     /* column pre-ordering, single block only; NULL: identity */
  const rs_complex* rhs;   /* rhs (linear modes) / un-normalised start vector */
  rs_complex* x;
  rs_solve_stats* stats;   /* device, one entry */
  double tol;
  int32_t max_iter;
  int32_t restart_m;
  int32_t max_outer;
  int32_t reserved;
} rs_grid_args;

int rs_grid_solve(const rs_grid_args* args, void* stream);
/* x = M^{-1} rhs only (factor.solve_lu, factor.py:137-149) through the same
 * level-ordered sweeps; A / P / stats are ignored. */
int rs_grid_apply(const rs_grid_args* args, void* stream);

/* ---- grid-wide vector operations (large-system / sharded path) ---------- */

/* out[2k], out[2k+1] = re, im of vdot(xs[k], ys[k]) = sum conj(x) y, k < npairs
 * (<= 4); xs/ys are HOST arrays of device pointers; out is device.
 * Deterministic: fixed grid, fixed reduction order (krylov.py np.vdot /
 * np.linalg.norm**2 up to summation order). */
int rs_vdots(int64_t n, int32_t npairs, const rs_complex* const* xs,
             const rs_complex* const* ys, double* out, void* stream);

/* out[0] = max_i |x_i| (steady.py:532 np.max(np.abs(.))); out is device. */
int rs_amax(int64_t n, const rs_complex* x, double* out, void* stream);

/* out = sum_{k < nv} (coef_re[k] + i coef_im[k]) * vs[k], nv <= 4; vs, coef_*
 * are HOST arrays; out may alias an input (the BiCGStab updates). */
int rs_lincomb(int64_t n, int32_t nv, const rs_complex* const* vs, const double* coef_re,
               const double* coef_im, rs_complex* out, void* stream);

/* Block-Jacobi blocks: rows [g*block, (g+1)*block) of an nrows-row CSR whose
 * column indices are offset by col0, keeping entries whose (col - col0) lies
 * in the same block, as a block-diagonal batch with local indices.  Two
 * passes (out_ci == NULL: row pointers + *nnz). */
int rs_block_extract(int64_t nrows, int32_t block, int32_t col0, const int32_t* rp,
                     const int32_t* ci, const rs_complex* v, int32_t* out_rp,
                     int32_t* out_ci, rs_complex* out_v, int64_t* nnz, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* RHOSOLVE_B200_H */
