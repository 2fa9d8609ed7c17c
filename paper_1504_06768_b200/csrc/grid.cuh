// Arguments of the grid-wide solver (grid.cu) and the level-ordered factor
// layout it consumes (levels.cu, trisell.cuh).
#pragma once
#include "common.cuh"
#include "solver.cuh"
#include "trisell.cuh"

namespace rs {

struct GridArgs {
  int32_t n;     // order of the whole system (all block-Jacobi blocks together)
  int32_t nb;    // order of one preconditioner block (nb == n: a single factorization)
  int32_t mode;  // SolveMode
  // system matrix (shifted or modified, ordered), one n x n CSR
  const int32_t* Arp;
  const int32_t* Aci;
  const double2* Av;
  // plain ordered matrix (inverse power outer residual)
  const int32_t* Prp;
  const int32_t* Pci;
  const double2* Pv;
  // preconditioner: level-ordered L and U (global row / column indices),
  // recipc(U_cc) per row, the factors' row permutation (local to each block)
  TriSell L, U;
  const double2* rd;
  const int32_t* pinv;
  const int32_t* colp;  // column pre-ordering (null: identity; single block only)
  int32_t have_M;
  const double2* rhs;  // rhs (linear modes) or start vector (inverse power)
  double2* xout;
  SolveStats* stats;
  double2* work;  // grid_work_len(n, restart_m) entries
  double* part;   // 2 * blocks * 8 doubles: reduction partials
  double tol;
  int32_t max_iter;
  int32_t restart_m;
  int32_t max_outer;
  int32_t want_condest;
};

int64_t grid_work_len(int32_t n, int restart_m);
int grid_blocks();
int launch_grid_solver(const GridArgs& a, cudaStream_t st);
int launch_grid_apply(const GridArgs& a, cudaStream_t st);

// levels.cu
int tri_levels(int B, int32_t n, int upper, const int32_t* rp, const int32_t* cp,
               const int32_t* ri, int64_t cap, int32_t* level, int64_t* nlev_host,
               cudaStream_t st);
int tri_order(int B, int32_t n, const int32_t* level, const int32_t* rp, int64_t nlev, int32_t H,
              int32_t* order, int64_t* npos_host, cudaStream_t st);
int64_t tri_sell_keys(int64_t total, int64_t nslices);
int tri_sell(int B, int32_t n, int upper, const int32_t* rp, const int32_t* ci, const double2* v,
             const int32_t* order, int64_t npos, int32_t H, const int32_t* level, int32_t* sptr,
             int32_t* sci, double2* sv, int32_t* skey, int64_t* total, cudaStream_t st);

}  // namespace rs
