// Arguments of the device-resident steady-state solver (solver.cu).
#pragma once
#include "common.cuh"

namespace rs {

enum SolveMode {
  MODE_INV_DIRECT = 0,
  MODE_INV_BICGSTAB = 1,
  MODE_INV_GMRES = 2,
  MODE_LIN_DIRECT = 3,
  MODE_LIN_BICGSTAB = 4,
  MODE_LIN_GMRES = 5,
};

enum SolveStatus {
  SOLVE_OK = 0,
  SOLVE_INNER_BREAKDOWN = 1,    // steady.py:218-222
  SOLVE_INNER_NONFINITE = 2,    // steady.py:218-222
  SOLVE_INNER_NO_PROGRESS = 3,  // steady.py:223-224
  SOLVE_UNUSABLE_VECTOR = 4,    // steady.py:234-235
  SOLVE_POWER_NOT_CONVERGED = 5,  // steady.py:246-248
  SOLVE_SKIPPED = 6,            // masked out (SolverArgs::skip)
};

// Must match include/rhosolve_b200.h rs_solve_stats.
struct SolveStats {
  int32_t status;
  int32_t outer;
  int32_t inner_last;
  int32_t inner_total;
  int32_t converged;
  int32_t breakdown;
  double final_residual;
  double condest;
};

struct SolverArgs {
  int32_t n;
  int32_t B;
  int32_t mode;
  int32_t threads;
  // system matrix (shifted or modified, ordered), block-diagonal CSR
  const int32_t* Arp;
  const int32_t* Aci;
  const double2* Av;
  // plain ordered matrix (inverse power outer residual), block-diagonal CSR
  const int32_t* Prp;
  const int32_t* Pci;
  const double2* Pv;
  // preconditioner: strictly-lower L, strictly-upper U (block-diagonal CSR,
  // pivotal coordinates), reciprocal pivots, row permutation pinv (local)
  const int32_t* Lrp;
  const int32_t* Lci;
  const double2* Lv;
  const int32_t* Urp;
  const int32_t* Uci;
  const double2* Uv;
  const double2* rU;
  const int32_t* pinv;
  const double2* rhs;  // rhs (linear modes) or start vector (inverse power)
  double2* xout;
  SolveStats* stats;
  double2* work;
  int64_t work_stride;  // complex entries per system
  double tol;
  int32_t max_iter;
  int32_t restart_m;
  int32_t max_outer;
  int32_t want_condest;
  int32_t y_in_smem;
  // column streams for the column-oriented sweeps (colsweep.cuh)
  const int32_t* Lso;
  const int32_t* Lsi;
  const double2* Lsv;
  const int32_t* Lsm;
  const int32_t* Uso;
  const int32_t* Usi;
  const double2* Usv;
  const int32_t* Usm;
  const double2* Usr;
  int32_t ring_R;  // > 0: column sweeps with a ring of ring_R 64-entry slots
  int32_t col_reach;       // max |row - column| over both factors (0: unknown)
  int32_t col_win;         // > 0: sliding shared-memory window of this many rows over a global y
  int32_t col_consumers;   // consumer warps of the column sweeps (> 1: long columns, lone systems)
  int32_t col_y_global;    // column sweeps with the sweep vector in global memory
  double2* ywork;          // global sweep vectors (set by the launcher)
  int64_t ywork_stride;
  const SolverArgs* self;  // device copy of these arguments (set by the launcher)
  const int32_t* colp;     // column pre-ordering: apply ends with x[j] = y[colp[j]] (null: identity)
  const int32_t* skip;     // per-system mask: != 0 -> not solved (SOLVE_SKIPPED)
  double* trace;           // (iteration, residual) pairs of system 0 (krylov.py:62-64)
  int32_t* trace_count;
  int32_t trace_cap;
};

// Ring size for the column sweeps of systems of order n in a launch of B
// CTAs (0 = not supported: the sweep vector and ring do not fit).
int col_ring_size(int32_t n, int B);
// ring slots for the column sweeps; *y_global = 1 when the sweep vector
// must stay in global memory (it does not fit next to the ring)
int col_plan(int32_t n, int B, int* y_global);
// column streams of one triangle (pass 1: idx == null -> rowoff + *total)
int col_stream_build(int B, int32_t n, int upper, const int32_t* cp, const int32_t* ci,
                     const double2* cv, int64_t cap, const double2* rdiag, int32_t* rowoff,
                     int32_t* idx, double2* val, int32_t* meta, double2* rrd, int64_t* total,
                     cudaStream_t st);
// rd[b*n+k] = recipc(last entry of U column k) from the raw CSC factor
int pivot_recip(int B, int32_t n, const int32_t* Up, const double2* Ux, int64_t capU,
                double2* rd, cudaStream_t st);

int64_t solver_work_stride(int32_t n, int restart_m);
int launch_steady_solver(const SolverArgs& a, cudaStream_t st);

}  // namespace rs

namespace rs {
int launch_lu_solve(const SolverArgs& a, cudaStream_t st);
}
