// Internal launcher declarations shared by the .cu translation units.
#pragma once
#include "common.cuh"

namespace rs {

// ---- spmv.cu -------------------------------------------------------------
int launch_spmv(int64_t nrows, int32_t n, const int32_t* rp, const int32_t* ci,
                const double2* v, const double2* x, double2* y, cudaStream_t st);

// ---- csr.cu (structure utilities) -----------------------------------------
// Exclusive scan of int32 counts into int32 offsets (n+1 outputs); returns
// the total through *total_host when non-null (synchronises the stream).
int scan_counts(const int32_t* counts, int32_t* offsets, int64_t n,
                int64_t* total_host, cudaStream_t st);
// Transpose of a block-diagonal batch of B n-by-n CSR matrices.  Output
// rows hold their entries in ascending column order (counting sort that is
// stable in the input row order), matching sparse.transpose / from_coo.
int csr_transpose(int B, int32_t n, const int32_t* rp, const int32_t* ci,
                  const double2* v, int32_t* out_rp, int32_t* out_ci,
                  double2* out_v, cudaStream_t st);

// ---- sell.cu: SELL-32 layout of the triangular factors -------------------
// Pass 1 (sci == null): sptr[B*nsl+1] and *total padded entries; pass 2 fills.
int sell_build(int B, int32_t n, int upper, const int32_t* rp, const int32_t* ci,
               const double2* v, int32_t* sptr, int32_t* sci, double2* sv, int64_t* total,
               cudaStream_t st);

// ---- factorization (ilu.cu) -----------------------------------------------
struct FactorArgs {
  int32_t n;
  int32_t B;
  const int32_t* Ap;  // CSC column pointers, block-diagonal, [B*n+1]
  const int32_t* Ai;  // local row indices (ascending within a column)
  const double2* Ax;
  const int32_t* q;   // optional elimination order (local), [B*n] or null
  const double* rn;   // row norms [B*n] (required when drop_tol > 0)
  double drop_tol;
  int32_t fill_cap;   // -1: no cap
  const int32_t* fill_caps;  // optional per-system caps (overrides fill_cap)
  double pivot_floor;  // > 0: substitute this value for a missing / zero pivot (opt-in)
  int early_drop;      // 1: drop a U entry before eliminating with it (opt-in, Saad ILUT)
  // outputs per system b; pointers are relative to b*cap
  int32_t* Lp;  // [B*(n+1)]
  int32_t* Li;
  double2* Lx;
  int64_t capL;
  int32_t* Up;  // [B*(n+1)]
  int32_t* Ui;
  double2* Ux;
  int64_t capU;
  int32_t* pinv;  // [B*n]
  int32_t* prow;  // [B*n]
  int32_t* state;  // [B*3]: status, fail/next col, substituted pivots
  // per-warp private scratch: (B*warps) slices of n
  double2* wx;
  int32_t* wflag;
  uint32_t* wbits;  // [B*warps*nwords] when !bits_in_smem
  int32_t* wpat;
  int32_t* wurow;
  double2* wuval;
  int32_t* wlrow;
  uint8_t* wukeep;
  uint8_t* wlkeep;
  uint64_t* wkey;  // cap-selection keys
  int smem_mode;     // 1: pinv / prow / Lp shadow live in shared memory
  int bits_in_smem;  // 1: per-warp pending bitmaps in shared memory
  int warps;         // warps (columns in flight) per system
  int hist;          // 1: per-warp cap-selection histograms in shared memory (0 only for complete LU)
  int b0;            // first system of this launch (single-CTA mode; the grid covers b0 .. b0 + grid - 1)
  int hot_nap;       // ns the next column's owner naps between frontier polls
  unsigned nap_step; // ns per column of distance for the other warps' naps
  int cps;           // CTAs per system (> 1: multi-CTA mode for large systems)
  int32_t* gctl;     // [B*2] global control words in multi-CTA mode
  unsigned long long* probe;  // optional per-column phase clocks [n*6] (tuning)
};
// state[3b+0] codes
enum { FAC_RUNNING = 0, FAC_DONE = 1, FAC_ZERO_PIVOT = 2, FAC_OVERFLOW = 3 };
int launch_ilutp(const FactorArgs& a, cudaStream_t st);
__host__ __device__ size_t ilutp_smem_bytes(int32_t n, int warps, int shared_in_smem,
                                            int bits_in_smem, int hist);
int ilutp_plan(int32_t n, int warps, int* smem_mode, int* bits_in_smem);
// ilu_compact.cu: complete LU with the working column compact in shared
// memory (batches); systems it leaves in FAC_RUNNING go to launch_ilutp.
int launch_lu_compact(const FactorArgs& a, cudaStream_t st, int* launched);

// ---- halfsolve.cu: in-place lower / upper solves on the raw CSC factors ----
int half_solve(int upper, int B, int32_t n, const int32_t* cp, const int32_t* ci,
               const double2* cx, int64_t cap, double2* y, cudaStream_t st);

// ---- cmd_order.cu: host-native 'cmd' ordering ---------------------------
int weighted_mbm_host(int64_t n, const int64_t* rp, const int64_t* ci, const double2* v,
                      int64_t* forward);
void col_min_degree_host(int64_t n, const int64_t* rp, const int64_t* ci, int64_t* order);

// ---- frontal.cu: right-looking frontal complete LU ------------------------
// Factors (complete LU, q == null) every system whose structural front fits
// shared memory and marks it FAC_DONE; the rest keep their state for
// launch_ilutp.  RHOSOLVE_FRONTAL=1/0 forces it on/off (auto: <= 3 waves).
bool frontal_enabled(int nsys);
// share_sm: the 64-register build, so column-pipeline CTAs fit beside it.
int frontal_factor(const FactorArgs& a, cudaStream_t st, bool share_sm = false);
int frontal_last_taken();
int frontal_probe(int enable, double* out4);

}  // namespace rs
