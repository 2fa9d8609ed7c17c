// extern "C" entry points declared in include/rhosolve_b200.h.  Thin
// argument validation + dispatch to the launchers; no compute on the host and
// no fallback path.
#include <stdarg.h>
#include <stdlib.h>
#include <algorithm>
#include <atomic>
#include <mutex>
#include <stdio.h>
#include <string.h>

#include "../../include/rhosolve_b200.h"
#include "common.cuh"
#include "kernels.cuh"
#include "solver.cuh"
#include "grid.cuh"

namespace rs {

static thread_local char g_err[1024] = "";
static std::atomic<long long> g_launches{0};

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
static unsigned long long* g_factor_probe = nullptr;  // tuning hook
static std::atomic<int> g_compact_taken{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// defined in the other translation units
int csr_permute(int B, int32_t n, const int32_t* rp, const int32_t* ci, const double2* v,
                const int32_t* fwd, const int32_t* inv, int32_t* out_rp, int32_t* out_ci,
                double2* out_v, cudaStream_t st);
int csr_shift(int B, int32_t n, const int32_t* rp, const int32_t* ci, const double2* v,
              double sigma, int32_t* out_rp, int32_t* out_ci, double2* out_v,
              int64_t* nnz_out, cudaStream_t st);
int csr_modify(int B, int32_t n, int32_t D, const int32_t* rp, const int32_t* ci,
               const double2* v, const double* w, int32_t* out_rp, int32_t* out_ci,
               double2* out_v, int64_t* nnz_out, cudaStream_t st);
int csr_default_weight(int B, int32_t n, const int32_t* rp, const int32_t* ci,
                       const double2* v, int signed_mode, double* w, cudaStream_t st);
int csr_row_norms(int64_t nrows, const int32_t* rp, const double2* v, double* rn,
                  cudaStream_t st);
int factor_to_csr(int B, int32_t n, const int32_t* cp, const int32_t* ri, const double2* rv,
                  int64_t cap, int lower, int32_t* out_rp, int32_t* out_ci, double2* out_v,
                  double2* rU, int64_t* nnz_out, cudaStream_t st);
int liouvillian_assemble(int32_t B, int32_t D, const int32_t* Hrp, const int32_t* Hci,
                         const double2* Hv, int64_t Hnnz, int32_t K, const int32_t* const* Crp,
                         const int32_t* const* Cci, const double2* const* Cv,
                         const int64_t* Cnnz, double* herm_dev, int32_t* out_rp,
                         int32_t* out_ci, double2* out_v, int64_t* nnz_out, cudaStream_t st);
int same_pattern(int32_t B, int32_t n, const int32_t* rp, const int32_t* ci, int64_t nnz,
                 int32_t* same, cudaStream_t st);
int rcm_order(int B, int32_t n, const int32_t* rp, const int32_t* ci, int32_t* fwd,
              int32_t* inv, cudaStream_t st);
int postprocess(int B, int32_t D, const double2* x, const int32_t* fwd, const int32_t* Lrp,
                const int32_t* Lci, const double2* Lv, double2* rho, double* residual,
                double2* trace_out, cudaStream_t st);
int permute_vector(int B, int32_t n, const double2* x, const int32_t* fwd, double2* out,
                   int gather, cudaStream_t st);
int vec_vdots(int64_t n, int np, const double2* const* xs, const double2* const* ys, double* out,
              double* scratch, cudaStream_t st);
int vec_amax(int64_t n, const double2* x, double* out, double* scratch, cudaStream_t st);
int vec_lincomb(int64_t n, int nv, const double2* const* vs, const double* coef_re,
                const double* coef_im, double2* out, cudaStream_t st);
int block_extract(int64_t nrows, int32_t m, int32_t col0, const int32_t* rp, const int32_t* ci,
                  const double2* v, int32_t* out_rp, int32_t* out_ci, double2* out_v,
                  int64_t* nnz_out, cudaStream_t st);

}  // namespace rs

using namespace rs;

#define S(stream) reinterpret_cast<cudaStream_t>(stream)
#define C2(p) reinterpret_cast<const double2*>(p)
#define M2(p) reinterpret_cast<double2*>(p)

extern "C" {

int rs_abi_version(void) { return RS_ABI_VERSION; }

// Keep freed stream-ordered allocations in the device pool instead of
// returning them to the OS at every synchronisation: the solve path
// allocates and frees its scratch every call.
static int keep_pool_memory() {
  static std::atomic<unsigned long long> done{0};  // one bit per device
  int dev;
  RS_CUDA_TRY(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (done.load(std::memory_order_relaxed) & bit) return RS_OK;
  cudaMemPool_t pool;
  RS_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
  unsigned long long thr = ~0ull;
  RS_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  done.fetch_or(bit, std::memory_order_relaxed);
  return RS_OK;
}
// One non-blocking side stream per device (hybrid batch factorization).
static int side_stream(cudaStream_t* out) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  int dev;
  RS_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  cudaStream_t& s = streams[dev & 63];
  if (!s) RS_CUDA_TRY(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  *out = s;
  return RS_OK;
}
// How many leading systems of a complete-LU batch take the frontal kernel
// while the rest run through pipeline CTAs beside it (0: no hybrid).
// RHOSOLVE_HYBRID_F overrides (0 disables).
static int hybrid_frontal_count(int nsys, int n) {
  if (const char* e = getenv("RHOSOLVE_HYBRID_F")) return std::min(std::max(0, atoi(e)), nsys);
  (void)n;
  return 0;
}
// Complete LU: the compact shared-memory kernel (ilu_compact.cu) takes every
// batch size (measured against the frontal kernel and the general pipeline in
// tools/lu_policy.py); RHOSOLVE_COMPACT=0 turns it off.
static bool compact_enabled(int nsys) {
  (void)nsys;
  if (const char* e = getenv("RHOSOLVE_COMPACT")) return e[0] == '1';
  return true;
}
const char* rs_last_error(void) { return g_err; }
long long rs_launch_count(void) { return g_launches.load(); }
// Tuning hook (not part of the documented ABI): when set, the next
// factorizations record per-column phase clocks of system 0 into buf[n*6].
int rs_debug_frontal_taken(void) { return rs::frontal_last_taken(); }
// 1 when the last rs_factorize ran the compact complete-LU kernel (ilu_compact.cu)
int rs_debug_compact_taken(void) { return g_compact_taken.load(std::memory_order_relaxed); }

int rs_weighted_mbm_host(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                         const rs_complex* values, int64_t* forward) {
  RS_CHECK_ARG(n >= 0, "negative size");
  RS_CHECK_ARG(!n || (row_ptr && col_idx && values && forward), "null array");
  if (rs::weighted_mbm_host(n, row_ptr, col_idx, reinterpret_cast<const double2*>(values),
                            forward)) {
    rs::set_error("matrix is structurally singular: no zero-free diagonal");
    return RS_ERR_STRUCT_SINGULAR;
  }
  return RS_OK;
}

int rs_col_min_degree_host(int64_t n, const int64_t* row_ptr, const int64_t* col_idx,
                           int64_t* order) {
  RS_CHECK_ARG(n >= 0, "negative size");
  RS_CHECK_ARG(!n || (row_ptr && col_idx && order), "null array");
  rs::col_min_degree_host(n, row_ptr, col_idx, order);
  return RS_OK;
}
int rs_debug_frontal_probe(int enable, double* out4) { return rs::frontal_probe(enable, out4); }

int rs_debug_factor_probe(void* buf) {
  g_factor_probe = reinterpret_cast<unsigned long long*>(buf);
  return 0;
}

int rs_tri_levels(int32_t nsys, int32_t n, int32_t upper, const int32_t* rp, const int32_t* cp,
                  const int32_t* ri, int64_t cap, int32_t* level, int64_t* nlevels,
                  void* stream) {
  RS_CHECK_ARG(nsys >= 0 && n >= 0 && cap >= 0, "negative size");
  RS_CHECK_ARG(nlevels != nullptr, "null nlevels");
  RS_CHECK_ARG(!(nsys && n) || (rp && cp && ri && level), "null pointer");
  return tri_levels(nsys, n, upper, rp, cp, ri, cap, level, nlevels, S(stream));
}

int rs_tri_order(int32_t nsys, int32_t n, const int32_t* level, const int32_t* rp,
                 int64_t nlevels, int32_t H, int32_t* order, int64_t* npos, void* stream) {
  RS_CHECK_ARG(nsys >= 0 && n >= 0 && nlevels >= 0, "negative size");
  RS_CHECK_ARG(H >= 1 && H <= 32 && (H & (H - 1)) == 0, "H must be a power of two <= 32");
  RS_CHECK_ARG(npos != nullptr, "null npos");
  return tri_order(nsys, n, level, rp, nlevels, H, order, npos, S(stream));
}

int rs_tri_sell(int32_t nsys, int32_t n, int32_t upper, const int32_t* rp, const int32_t* ci,
                const rs_complex* v, const int32_t* order, int64_t npos, int32_t H,
                const int32_t* level, int32_t* sptr, int32_t* sci, rs_complex* sv, int32_t* skey,
                int64_t* total, void* stream) {
  RS_CHECK_ARG(nsys >= 0 && n >= 0 && npos >= 0, "negative size");
  RS_CHECK_ARG(H >= 1 && H <= 32 && (H & (H - 1)) == 0 && npos % H == 0, "bad slice height");
  return tri_sell(nsys, n, upper, rp, ci, C2(v), order, npos, H, level, sptr, sci, M2(sv), skey,
                  total, S(stream));
}

static int grid_args(const rs_grid_args* p, GridArgs* a) {
  RS_CHECK_ARG(p != nullptr, "null args");
  RS_CHECK_ARG(p->n >= 0 && p->nb > 0 && p->n % p->nb == 0, "n must be a multiple of nb");
  a->n = p->n;
  a->nb = p->nb;
  a->mode = p->mode;
  a->Arp = p->A_rp;
  a->Aci = p->A_ci;
  a->Av = C2(p->A_v);
  a->Prp = p->P_rp;
  a->Pci = p->P_ci;
  a->Pv = C2(p->P_v);
  auto tf = [](const rs_tri_factor& f) {
    TriSell t;
    t.order = f.order;
    t.sptr = f.sptr;
    t.sci = f.sci;
    t.sv = C2(f.sv);
    t.skey = f.skey;
    t.nslices = f.nslices;
    t.G = f.lanes_per_row;
    t.apw = f.active_warps;
    t.mode = f.reserved;
    return t;
  };
  a->L = tf(p->L);
  a->U = tf(p->U);
  a->have_M = p->L.order != nullptr;
  if (a->have_M) {
    RS_CHECK_ARG(p->U.order && p->rdiag && p->pinv && p->L.skey && p->U.skey,
                 "incomplete preconditioner");
    for (int g : {a->L.G, a->U.G})
      RS_CHECK_ARG(g == 1 || g == 2 || g == 4 || g == 32, "lanes_per_row must be 1, 2, 4 or 32");
    RS_CHECK_ARG(!p->colp || p->nb == p->n, "column pre-ordering needs a single block");
  }
  a->rd = C2(p->rdiag);
  a->pinv = p->pinv;
  a->colp = p->colp;
  a->rhs = C2(p->rhs);
  a->xout = M2(p->x);
  a->stats = reinterpret_cast<SolveStats*>(p->stats);
  a->tol = p->tol;
  a->max_iter = p->max_iter;
  a->restart_m = p->restart_m;
  a->max_outer = p->max_outer > 0 ? p->max_outer : 50;
  a->want_condest = p->want_condest;
  return RS_OK;
}

int rs_grid_solve(const rs_grid_args* p, void* stream) {
  RS_TRY(keep_pool_memory());
  GridArgs a{};
  RS_TRY(grid_args(p, &a));
  RS_CHECK_ARG(p->mode >= RS_INV_DIRECT && p->mode <= RS_LIN_GMRES, "unknown mode");
  RS_CHECK_ARG(p->tol > 0.0 && p->max_iter >= 1 && p->restart_m >= 1, "bad iteration options");
  RS_CHECK_ARG(p->mode >= RS_LIN_DIRECT || p->P_rp != nullptr,
               "inverse power needs the plain matrix");
  if (!a.n) return RS_OK;
  RS_CHECK_ARG(a.Arp && a.rhs && a.xout && a.stats, "null pointer");
  cudaStream_t st = S(stream);
  const int64_t wl = grid_work_len(a.n, a.restart_m);
  const size_t pbytes = sizeof(double) * 2 * 8 * (size_t)std::max(grid_blocks(), 1);
  char* buf = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&buf, sizeof(double2) * wl + pbytes, st));
  a.work = reinterpret_cast<double2*>(buf);
  a.part = reinterpret_cast<double*>(buf + sizeof(double2) * wl);
  const int rc = launch_grid_solver(a, st);
  cudaFreeAsync(buf, st);
  return rc;
}

int rs_grid_apply(const rs_grid_args* p, void* stream) {
  RS_TRY(keep_pool_memory());
  GridArgs a{};
  RS_TRY(grid_args(p, &a));
  if (!a.n) return RS_OK;
  RS_CHECK_ARG(a.have_M && a.rhs && a.xout, "null pointer");
  cudaStream_t st = S(stream);
  char* buf = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&buf, sizeof(double2) * 3 * (size_t)a.n + 256, st));
  a.work = reinterpret_cast<double2*>(buf);
  a.part = reinterpret_cast<double*>(buf + sizeof(double2) * 3 * (size_t)a.n);
  const int rc = launch_grid_apply(a, st);
  cudaFreeAsync(buf, st);
  return rc;
}

int64_t rs_tri_sell_keys(int64_t total, int64_t nslices) { return tri_sell_keys(total, nslices); }

int rs_lower_solve(int32_t nsys, int32_t n, const int32_t* Lp, const int32_t* Li,
                   const rs_complex* Lx, int64_t cap, rs_complex* y, void* stream) {
  RS_CHECK_ARG(nsys >= 0 && n >= 0 && cap >= 0, "negative size");
  if (!nsys || !n) return RS_OK;
  RS_CHECK_ARG(Lp && Li && Lx && y, "null pointer");
  return half_solve(0, nsys, n, Lp, Li, C2(Lx), cap, M2(y), S(stream));
}

int rs_upper_solve(int32_t nsys, int32_t n, const int32_t* Up, const int32_t* Ui,
                   const rs_complex* Ux, int64_t cap, rs_complex* y, void* stream) {
  RS_CHECK_ARG(nsys >= 0 && n >= 0 && cap >= 0, "negative size");
  if (!nsys || !n) return RS_OK;
  RS_CHECK_ARG(Up && Ui && Ux && y, "null pointer");
  return half_solve(1, nsys, n, Up, Ui, C2(Ux), cap, M2(y), S(stream));
}

int rs_csr_matvec(int32_t nsys, int32_t n, const int32_t* row_ptr, const int32_t* col_idx,
                  const rs_complex* values, const rs_complex* x, rs_complex* y, void* stream) {
  RS_CHECK_ARG(nsys >= 0 && n >= 0, "negative size");
  if (!nsys || !n) return RS_OK;
  RS_CHECK_ARG(row_ptr && x && y, "null pointer");
  return launch_spmv((int64_t)nsys * n, n, row_ptr, col_idx, C2(values), C2(x), M2(y), S(stream));
}

int rs_factorize(int32_t nsys, int32_t n, const int32_t* Ap, const int32_t* Ai,
                 const rs_complex* Ax, const int32_t* q, double drop_tol, int32_t fill_cap,
                 const int32_t* fill_caps, const double* row_norms, int32_t* Lp, int32_t* Li, rs_complex* Lx,
                 int64_t capL, int32_t* Up, int32_t* Ui, rs_complex* Ux, int64_t capU,
                 int32_t* pinv, int32_t* state, void* stream) {
  return rs_factorize_opts(nsys, n, Ap, Ai, Ax, q, drop_tol, fill_cap, fill_caps, row_norms, Lp,
                            Li, Lx, capL, Up, Ui, Ux, capU, pinv, state, 0.0, 0, stream);
}

int rs_factorize_opts(int32_t nsys, int32_t n, const int32_t* Ap, const int32_t* Ai,
                       const rs_complex* Ax, const int32_t* q, double drop_tol, int32_t fill_cap,
                       const int32_t* fill_caps, const double* row_norms, int32_t* Lp,
                       int32_t* Li, rs_complex* Lx, int64_t capL, int32_t* Up, int32_t* Ui,
                       rs_complex* Ux, int64_t capU, int32_t* pinv, int32_t* state,
                       double pivot_floor, int32_t early_drop, void* stream) {
  RS_TRY(keep_pool_memory());
  RS_CHECK_ARG(pivot_floor >= 0.0, "pivot_floor must be >= 0");
  RS_CHECK_ARG(nsys >= 0 && n >= 0, "negative size");
  RS_CHECK_ARG(drop_tol >= 0.0, "drop tolerance must be >= 0");
  RS_CHECK_ARG(!(drop_tol > 0.0) || row_norms, "row_norms required when drop_tol > 0");
  RS_CHECK_ARG(capL >= n && capU >= n, "factor capacity below n");
  if (!nsys || !n) return RS_OK;
  cudaStream_t st = S(stream);
  const int64_t N = (int64_t)nsys * n;
  FactorArgs a{};
  a.n = n;
  a.B = nsys;
  a.Ap = Ap;
  a.Ai = Ai;
  a.Ax = C2(Ax);
  a.q = q;
  a.rn = row_norms;
  a.drop_tol = drop_tol;
  a.fill_cap = fill_cap;
  a.fill_caps = fill_caps;
  a.pivot_floor = pivot_floor;
  a.early_drop = early_drop ? 1 : 0;
  a.Lp = Lp;
  a.Li = Li;
  a.Lx = M2(Lx);
  a.capL = capL;
  a.Up = Up;
  a.Ui = Ui;
  a.Ux = M2(Ux);
  a.capU = capU;
  a.pinv = pinv;
  a.state = state;
  a.warps = nsys >= 148 ? 8 : 16;
  // complete-LU batches of up to two systems per SM run 16 warps per system
  // in the compact kernel (ilu_compact.cu)
  if (!(drop_tol > 0.0) && fill_cap < 0 && !fill_caps && !q && nsys <= 2 * 148) a.warps = 16;
  a.hist = 1;
  a.b0 = 0;
  if (const char* e = getenv("RHOSOLVE_ILU_WARPS")) a.warps = atoi(e);  // tuning knob
  // the critical column's owner polls the frontier hot (naps measured: no
  // gain at 16-128 ns on the 512-system batch)
  a.hot_nap = 0;
  if (const char* e = getenv("RHOSOLVE_ILU_HOTNAP")) a.hot_nap = atoi(e);  // tuning knob
  a.nap_step = 64;
  if (const char* e = getenv("RHOSOLVE_ILU_NAPSTEP")) a.nap_step = atoi(e);  // tuning knob
  // large systems: one system spans several CTAs (columns in flight across
  // SMs; the per-column work of c3 / the c5 blocks dwarfs the cross-SM
  // hand-off)
  a.cps = 1;
  // (c3: 13.3 s at 1 CTA, 1.70 s at 16, 1.44 s at 32, flat beyond)
  // ... but only when a column carries enough work to pay for the cross-SM
  // hand-off: the sparse block-Jacobi factors of config 5 (fill cap ~30) run
  // faster with one CTA per block (16 blocks of 160k columns: 1.86 s vs 2.59 s
  // at 9 CTAs per block)
  const bool heavy_columns = fill_cap < 0 || fill_cap >= 64;  // fill_cap = the largest cap
  if (n >= 8192 && nsys < 148 && heavy_columns) a.cps = std::min(32, std::max(1, 148 / nsys));
  if (const char* e = getenv("RHOSOLVE_ILU_CPS")) a.cps = std::max(1, atoi(e));  // tuning knob
  if (a.cps > 1) a.warps = 16;
  RS_TRY(ilutp_plan(n, a.warps, &a.smem_mode, &a.bits_in_smem));
  if (a.cps > 1) a.smem_mode = 0;  // pinv / prow / Lp are shared across CTAs
  const int nwords = (n + 31) / 32;
  const int64_t NW = N * a.warps * a.cps;  // per-warp slices
  size_t bytes = 0;
  auto take = [&](size_t b) {
    size_t o = bytes;
    bytes += (b + 255) & ~(size_t)255;
    return o;
  };
  const size_t o_x = take(16 * NW);
  const size_t o_flag = take(4 * NW);
  const bool maybe_hybrid = hybrid_frontal_count(nsys, n) > 0;  // (its pipeline CTAs keep the bitmaps in global memory)
  const size_t o_bits = (a.bits_in_smem && !maybe_hybrid)
                            ? 0
                            : take(4 * (size_t)nwords * nsys * a.warps * a.cps);
  const size_t o_ctl = take(8 * (size_t)nsys);
  const size_t o_prow = take(4 * N);
  const size_t o_pat = take(4 * NW);
  const size_t o_urow = take(4 * NW);
  const size_t o_uval = take(16 * NW);
  const size_t o_lrow = take(4 * NW);
  const size_t o_uk = take(NW);
  const size_t o_lk = take(NW);
  const size_t o_key = take(8 * NW);
  unsigned char* ws = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&ws, bytes, st));
  a.wx = reinterpret_cast<double2*>(ws + o_x);
  a.wflag = reinterpret_cast<int32_t*>(ws + o_flag);
  a.wbits = (a.bits_in_smem && !maybe_hybrid) ? nullptr : reinterpret_cast<uint32_t*>(ws + o_bits);
  a.prow = reinterpret_cast<int32_t*>(ws + o_prow);
  a.wpat = reinterpret_cast<int32_t*>(ws + o_pat);
  a.wurow = reinterpret_cast<int32_t*>(ws + o_urow);
  a.wuval = reinterpret_cast<double2*>(ws + o_uval);
  a.wlrow = reinterpret_cast<int32_t*>(ws + o_lrow);
  a.wukeep = ws + o_uk;
  a.wlkeep = ws + o_lk;
  a.wkey = reinterpret_cast<uint64_t*>(ws + o_key);
  a.gctl = reinterpret_cast<int32_t*>(ws + o_ctl);
  a.probe = g_factor_probe;
  const bool complete_lu = !(drop_tol > 0.0) && fill_cap < 0 && !fill_caps && !q &&
                           !g_factor_probe && a.cps == 1;
  // Large batches of complete LUs (the 512-system c4 sweep): hybrid.  The
  // frontal kernel is bound by shared memory (one system per SM) and latency,
  // the column pipeline by instruction issue, so they share the SMs: the
  // first F systems go to the 64-register frontal build on `st`, the others to
  // pipeline CTAs without shared-memory state (two fit beside a front) on a
  // side stream, concurrently.  Both produce the reference's factors, so the
  // split is invisible in the output.
  const int hybrid_f = complete_lu ? hybrid_frontal_count(nsys, n) : 0;
  int compact = 0;
  g_compact_taken.store(0, std::memory_order_relaxed);
  const bool frontal_auto = frontal_enabled(nsys);  // (also resets its "taken" counter)
  const char* fenv = getenv("RHOSOLVE_FRONTAL");
  const bool frontal_forced = fenv && fenv[0] == '1';
  if (complete_lu && hybrid_f == 0 && !frontal_forced && compact_enabled(nsys)) {
    const int crc = launch_lu_compact(a, st, &compact);
    if (crc) {
      cudaFreeAsync(ws, st);
      return crc;
    }
  }
  if (compact) {
    // (whatever it left in FAC_RUNNING runs through the general kernel below)
    g_compact_taken.store(1, std::memory_order_relaxed);
  } else if (hybrid_f > 0) {
    cudaStream_t side = nullptr;
    RS_TRY(side_stream(&side));
    cudaEvent_t fork = nullptr, join = nullptr;
    RS_CUDA_TRY(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    RS_CUDA_TRY(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
    RS_CUDA_TRY(cudaEventRecord(fork, st));
    RS_CUDA_TRY(cudaStreamWaitEvent(side, fork, 0));
    FactorArgs fa = a;
    fa.B = hybrid_f;
    int rc = frontal_factor(fa, st, true);  // (launched first: the fronts claim their SMs)
    if (!rc) {
      FactorArgs pa = a;
      pa.b0 = hybrid_f;
      pa.B = nsys - hybrid_f;
      pa.smem_mode = 0;
      pa.bits_in_smem = 0;
      pa.hist = 0;
      rc = launch_ilutp(pa, side);
    }
    cudaEventRecord(join, side);
    cudaStreamWaitEvent(st, join, 0);
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
    if (rc) {
      cudaFreeAsync(ws, st);
      return rc;
    }
  } else if (frontal_auto && complete_lu) {
    // complete LU of small systems: right-looking frontal elimination in
    // shared memory; whatever it does not take (front too large, zero pivot)
    // runs through the column pipeline below
    const int frc = frontal_factor(a, st);
    if (frc) {
      cudaFreeAsync(ws, st);
      return frc;
    }
  }
  // prow is scratch: a resumed launch rebuilds it as the inverse of pinv.
  const int rc = launch_ilutp(a, st);
  cudaFreeAsync(ws, st);
  return rc;
}

int rs_factor_rows(int32_t nsys, int32_t n, const int32_t* Lp, const int32_t* Li,
                   const rs_complex* Lx, int64_t capL, const int32_t* Up, const int32_t* Ui,
                   const rs_complex* Ux, int64_t capU, int32_t* L_rp, int32_t* L_ci,
                   rs_complex* L_v, int64_t* L_nnz, int32_t* U_rp, int32_t* U_ci,
                   rs_complex* U_v, rs_complex* rdiag, int64_t* U_nnz, void* stream) {
  RS_TRY(keep_pool_memory());
  RS_CHECK_ARG(nsys >= 0 && n >= 0, "negative size");
  cudaStream_t st = S(stream);
  RS_TRY(factor_to_csr(nsys, n, Lp, Li, C2(Lx), capL, 1, L_rp, L_ci, M2(L_v), nullptr, L_nnz,
                       st));
  RS_TRY(factor_to_csr(nsys, n, Up, Ui, C2(Ux), capU, 0, U_rp, U_ci, M2(U_v), M2(rdiag), U_nnz,
                       st));
  return RS_OK;
}

int rs_sell_build(int32_t nsys, int32_t n, int32_t upper, const int32_t* rp,
                  const int32_t* ci, const rs_complex* v, int32_t* sptr, int32_t* sci,
                  rs_complex* sv, int64_t* total, void* stream) {
  RS_TRY(keep_pool_memory());
  RS_CHECK_ARG(nsys >= 0 && n >= 0, "negative size");
  RS_CHECK_ARG(sptr != nullptr, "sptr is required");
  return sell_build(nsys, n, upper ? 1 : 0, rp, ci, C2(v), sptr, sci, M2(sv), total, S(stream));
}

int rs_col_sweep_supported(int32_t n) {
  int yg = 0;
  return (n > 0 && rs::col_plan(n, 1, &yg) > 0) ? 1 : 0;
}

int rs_pivot_recip(int32_t nsys, int32_t n, const int32_t* Up, const rs_complex* Ux,
                   int64_t capU, rs_complex* rdiag, void* stream) {
  RS_CHECK_ARG(nsys >= 0 && n >= 0, "negative size");
  return pivot_recip(nsys, n, Up, C2(Ux), capU, M2(rdiag), S(stream));
}

int rs_col_stream_build(int32_t nsys, int32_t n, int32_t upper, const int32_t* cp,
                        const int32_t* ci, const rs_complex* cv, int64_t cap,
                        const rs_complex* rdiag, int32_t* rowoff, int32_t* idx,
                        rs_complex* val, int32_t* meta, rs_complex* rrd, int64_t* total_rows,
                        void* stream) {
  RS_TRY(keep_pool_memory());
  RS_CHECK_ARG(nsys >= 0 && n >= 0, "negative size");
  RS_CHECK_ARG(rowoff != nullptr, "rowoff is required");
  RS_CHECK_ARG(!upper || !idx || (rdiag && rrd), "U streams need rdiag and rrd");
  return col_stream_build(nsys, n, upper ? 1 : 0, cp, ci, C2(cv), cap, C2(rdiag), rowoff, idx,
                          M2(val), meta, M2(rrd), total_rows, S(stream));
}

int rs_lu_solve_cols(int32_t nsys, int32_t n, const int32_t* pinv, const int32_t* Ls_rowoff,
                     const int32_t* Ls_idx, const rs_complex* Ls_val, const int32_t* Ls_meta,
                     const int32_t* Us_rowoff, const int32_t* Us_idx, const rs_complex* Us_val,
                     const int32_t* Us_meta, const rs_complex* Us_rd, const rs_complex* b,
                     rs_complex* x, void* stream) {
  return rs_lu_solve_cols_reach(nsys, n, pinv, Ls_rowoff, Ls_idx, Ls_val, Ls_meta, Us_rowoff,
                                Us_idx, Us_val, Us_meta, Us_rd, b, x, 0, stream);
}

int rs_lu_solve_cols_reach(int32_t nsys, int32_t n, const int32_t* pinv,
                           const int32_t* Ls_rowoff, const int32_t* Ls_idx,
                           const rs_complex* Ls_val, const int32_t* Ls_meta,
                           const int32_t* Us_rowoff, const int32_t* Us_idx,
                           const rs_complex* Us_val, const int32_t* Us_meta,
                           const rs_complex* Us_rd, const rs_complex* b, rs_complex* x,
                           int32_t reach, void* stream) {
  RS_CHECK_ARG(nsys >= 0 && n >= 0 && reach >= 0, "negative size");
  if (!nsys || !n) return RS_OK;
  SolverArgs a{};
  a.col_reach = reach;
  a.n = n;
  a.B = nsys;
  a.Lso = Ls_rowoff;
  a.Lsi = Ls_idx;
  a.Lsv = C2(Ls_val);
  a.Lsm = Ls_meta;
  a.Uso = Us_rowoff;
  a.Usi = Us_idx;
  a.Usv = C2(Us_val);
  a.Usm = Us_meta;
  a.Usr = C2(Us_rd);
  a.pinv = pinv;
  a.rhs = C2(b);
  a.xout = M2(x);
  a.ring_R = col_plan(n, nsys, &a.col_y_global);
  cudaStream_t st = S(stream);
  double2* work = nullptr;
  if (a.col_y_global) {  // sweep vectors (+ dummy slot) in global memory
    RS_CUDA_TRY(cudaMallocAsync(&work, sizeof(double2) * 2 * (size_t)n * nsys, st));
    a.work = work;
  }
  const int rc = launch_lu_solve(a, st);
  if (work) cudaFreeAsync(work, st);
  return rc;
}

int rs_lu_solve(int32_t nsys, int32_t n, const int32_t* pinv, const int32_t* L_rp,
                const int32_t* L_ci, const rs_complex* L_v, const int32_t* U_rp,
                const int32_t* U_ci, const rs_complex* U_v, const rs_complex* rdiag,
                const rs_complex* b, rs_complex* x, void* stream) {
  RS_CHECK_ARG(nsys >= 0 && n >= 0, "negative size");
  SolverArgs a{};
  a.n = n;
  a.B = nsys;
  a.Lrp = L_rp;
  a.Lci = L_ci;
  a.Lv = C2(L_v);
  a.Urp = U_rp;
  a.Uci = U_ci;
  a.Uv = C2(U_v);
  a.rU = C2(rdiag);
  a.pinv = pinv;
  a.rhs = C2(b);
  a.xout = M2(x);
  cudaStream_t st = S(stream);
  int dev, max_smem;
  RS_CUDA_TRY(cudaGetDevice(&dev));
  RS_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  double2* work = nullptr;
  if (32 * (size_t)n + 2048 > (size_t)max_smem) {
    RS_CUDA_TRY(cudaMallocAsync(&work, sizeof(double2) * 2 * (size_t)n * nsys, st));
    a.work = work;
  }
  const int rc = launch_lu_solve(a, st);
  if (work) cudaFreeAsync(work, st);
  return rc;
}

int rs_liouvillian(int32_t D, const int32_t* H_rp, const int32_t* H_ci, const rs_complex* H_v,
                   int64_t H_nnz, int32_t K, const int32_t* const* C_rp,
                   const int32_t* const* C_ci, const rs_complex* const* C_v,
                   const int64_t* C_nnz, double* herm_dev, int32_t* out_rp, int32_t* out_ci,
                   rs_complex* out_v, int64_t* nnz, void* stream) {
  RS_TRY(keep_pool_memory());
  RS_CHECK_ARG(D >= 1, "hilbert dimension must be >= 1");
  RS_CHECK_ARG(K >= 0, "negative collapse operator count");
  RS_CHECK_ARG((int64_t)D * D < ((int64_t)1 << 31), "D*D exceeds int32 indexing");
  return liouvillian_assemble(1, D, H_rp, H_ci, C2(H_v), H_nnz, K, C_rp, C_ci,
                              reinterpret_cast<const double2* const*>(C_v), C_nnz, herm_dev,
                              out_rp, out_ci, M2(out_v), nnz, S(stream));
}

int rs_liouvillian_batch(int32_t nsys, int32_t D, const int32_t* H_rp, const int32_t* H_ci,
                         const rs_complex* H_v, int64_t H_nnz, int32_t K,
                         const int32_t* const* C_rp, const int32_t* const* C_ci,
                         const rs_complex* const* C_v, const int64_t* C_nnz, double* herm_dev,
                         int32_t* out_rp, int32_t* out_ci, rs_complex* out_v, int64_t* nnz,
                         void* stream) {
  RS_TRY(keep_pool_memory());
  RS_CHECK_ARG(nsys >= 1 && D >= 1, "sizes must be >= 1");
  RS_CHECK_ARG(K >= 0, "negative collapse operator count");
  RS_CHECK_ARG((int64_t)nsys * D * D < ((int64_t)1 << 31), "nsys*D*D exceeds int32 indexing");
  return liouvillian_assemble(nsys, D, H_rp, H_ci, C2(H_v), H_nnz, K, C_rp, C_ci,
                              reinterpret_cast<const double2* const*>(C_v), C_nnz, herm_dev,
                              out_rp, out_ci, M2(out_v), nnz, S(stream));
}

int rs_shift(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci, const rs_complex* v,
             double sigma, int32_t* out_rp, int32_t* out_ci, rs_complex* out_v, int64_t* nnz,
             void* stream) {
  RS_CHECK_ARG(sigma != 0.0, "sigma must be nonzero");
  return csr_shift(nsys, n, rp, ci, C2(v), sigma, out_rp, out_ci, M2(out_v), nnz, S(stream));
}

int rs_default_weight(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci,
                      const rs_complex* v, int32_t mode, double* w, void* stream) {
  RS_CHECK_ARG(mode == 0 || mode == 1, "unknown weight mode");
  return csr_default_weight(nsys, n, rp, ci, C2(v), mode, w, S(stream));
}

int rs_trace_modify(int32_t nsys, int32_t n, int32_t D, const int32_t* rp, const int32_t* ci,
                    const rs_complex* v, const double* w, int32_t* out_rp, int32_t* out_ci,
                    rs_complex* out_v, int64_t* nnz, void* stream) {
  RS_CHECK_ARG((int64_t)D * D == n, "n must equal D*D");
  return csr_modify(nsys, n, D, rp, ci, C2(v), w, out_rp, out_ci, M2(out_v), nnz, S(stream));
}

int rs_rcm(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci, int32_t* forward,
           int32_t* inverse, void* stream) {
  RS_TRY(keep_pool_memory());
  RS_CHECK_ARG(nsys >= 0 && n >= 0, "negative size");
  if (!nsys || !n) return RS_OK;
  return rcm_order(nsys, n, rp, ci, forward, inverse, S(stream));
}

int rs_same_pattern(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci, int64_t nnz,
                    int32_t* same, void* stream) {
  RS_CHECK_ARG(nsys >= 0 && n >= 0 && nnz >= 0, "negative size");
  RS_CHECK_ARG(same != nullptr, "same is required");
  return same_pattern(nsys, n, rp, ci, nnz, same, S(stream));
}

int rs_permute(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci, const rs_complex* v,
               const int32_t* forward, const int32_t* inverse, int32_t* out_rp, int32_t* out_ci,
               rs_complex* out_v, void* stream) {
  if (!nsys || !n) return RS_OK;
  return csr_permute(nsys, n, rp, ci, C2(v), forward, inverse, out_rp, out_ci, M2(out_v),
                     S(stream));
}

int rs_permute_rows_cols(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci,
                         const rs_complex* v, const int32_t* row_inverse,
                         const int32_t* col_forward, int32_t* out_rp, int32_t* out_ci,
                         rs_complex* out_v, void* stream) {
  if (!nsys || !n) return RS_OK;
  return csr_permute(nsys, n, rp, ci, C2(v), col_forward, row_inverse, out_rp, out_ci,
                     M2(out_v), S(stream));
}

int rs_permute_vector(int32_t nsys, int32_t n, const rs_complex* x, const int32_t* forward,
                      rs_complex* out, int32_t gather, void* stream) {
  RS_CHECK_ARG(x != out, "permute_vector cannot run in place");
  return permute_vector(nsys, n, C2(x), forward, M2(out), gather, S(stream));
}

int rs_transpose(int32_t nsys, int32_t n, const int32_t* rp, const int32_t* ci,
                 const rs_complex* v, int32_t* out_rp, int32_t* out_ci, rs_complex* out_v,
                 void* stream) {
  if (!nsys || !n) return RS_OK;
  return csr_transpose(nsys, n, rp, ci, C2(v), out_rp, out_ci, M2(out_v), S(stream));
}

int rs_row_norms(int32_t nsys, int32_t n, const int32_t* rp, const rs_complex* v,
                 double* row_norms, void* stream) {
  return csr_row_norms((int64_t)nsys * n, rp, C2(v), row_norms, S(stream));
}

int rs_steady_solve(const rs_solver_args* p, void* stream) {
  RS_TRY(keep_pool_memory());
  RS_CHECK_ARG(p != nullptr, "null args");
  RS_CHECK_ARG(p->n >= 0 && p->nsys >= 0, "negative size");
  RS_CHECK_ARG(p->mode >= RS_INV_DIRECT && p->mode <= RS_LIN_GMRES, "unknown mode");
  RS_CHECK_ARG(p->tol > 0.0, "tol must be > 0");
  RS_CHECK_ARG(p->max_iter >= 1, "max_iter must be >= 1");
  RS_CHECK_ARG(p->restart_m >= 1, "restart_m must be >= 1");
  RS_CHECK_ARG(p->mode < RS_INV_DIRECT + 3 ? p->P_rp != nullptr : true,
               "inverse power needs the plain matrix");
  if (!p->nsys || !p->n) return RS_OK;
  cudaStream_t st = S(stream);
  SolverArgs a{};
  a.n = p->n;
  a.B = p->nsys;
  a.mode = p->mode;
  a.threads = p->threads > 0 ? p->threads : 512;
  RS_CHECK_ARG(a.threads % 32 == 0 && a.threads <= 512, "threads must be a multiple of 32, <= 512");
  a.Arp = p->A_rp;
  a.Aci = p->A_ci;
  a.Av = C2(p->A_v);
  a.Prp = p->P_rp;
  a.Pci = p->P_ci;
  a.Pv = C2(p->P_v);
  a.Lrp = p->L_rp;
  a.Lci = p->L_ci;
  a.Lv = C2(p->L_v);
  a.Urp = p->U_rp;
  a.Uci = p->U_ci;
  a.Uv = C2(p->U_v);
  a.rU = C2(p->rdiag);
  a.pinv = p->pinv;
  a.rhs = C2(p->rhs);
  a.xout = M2(p->x);
  a.stats = reinterpret_cast<SolveStats*>(p->stats);
  a.tol = p->tol;
  a.max_iter = p->max_iter;
  a.restart_m = p->restart_m;
  a.max_outer = p->max_outer > 0 ? p->max_outer : 50;
  a.want_condest = p->want_condest;
  a.colp = p->colp;
  a.skip = p->skip;
  a.col_reach = p->col_reach;
  a.trace = p->trace;
  a.trace_count = p->trace_count;
  a.trace_cap = p->trace_cap;
  int dev, max_smem;
  RS_CUDA_TRY(cudaGetDevice(&dev));
  RS_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  a.y_in_smem = (32 * (size_t)a.n + 4096 <= (size_t)max_smem) ? 1 : 0;
  if (p->Ls_rowoff && p->Us_rowoff) {
    a.Lso = p->Ls_rowoff;
    a.Lsi = p->Ls_idx;
    a.Lsv = C2(p->Ls_val);
    a.Lsm = p->Ls_meta;
    a.Uso = p->Us_rowoff;
    a.Usi = p->Us_idx;
    a.Usv = C2(p->Us_val);
    a.Usm = p->Us_meta;
    a.Usr = C2(p->Us_rd);
    a.ring_R = col_plan(a.n, a.B, &a.col_y_global);
  }
  RS_CHECK_ARG(a.ring_R > 0 || a.Lrp != nullptr || p->Ls_rowoff == nullptr,
               "row-oriented factors required: n too large for the column sweeps");
  a.work_stride = solver_work_stride(a.n, a.restart_m);
  double2* work = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&work, sizeof(double2) * a.work_stride * a.B, st));
  a.work = work;
  int rc = launch_steady_solver(a, st);
  cudaFreeAsync(work, st);
  return rc;
}

int rs_postprocess(int32_t nsys, int32_t D, const rs_complex* x, const int32_t* forward,
                   const int32_t* plain_rp, const int32_t* plain_ci, const rs_complex* plain_v,
                   rs_complex* rho, double* residual, rs_complex* trace, void* stream) {
  RS_TRY(keep_pool_memory());
  RS_CHECK_ARG(nsys >= 0 && D >= 1, "bad size");
  if (!nsys) return RS_OK;
  return postprocess(nsys, D, C2(x), forward, plain_rp, plain_ci, C2(plain_v), M2(rho),
                     residual, M2(trace), S(stream));
}

int rs_vdots(int64_t n, int32_t npairs, const rs_complex* const* xs, const rs_complex* const* ys,
             double* out, void* stream) {
  RS_CHECK_ARG(n >= 0, "negative length");
  cudaStream_t st = S(stream);
  double* scratch = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&scratch, sizeof(double) * 592 * 8, st));
  const int rc = vec_vdots(n, npairs, reinterpret_cast<const double2* const*>(xs),
                           reinterpret_cast<const double2* const*>(ys), out, scratch, st);
  cudaFreeAsync(scratch, st);
  return rc;
}

int rs_amax(int64_t n, const rs_complex* x, double* out, void* stream) {
  RS_CHECK_ARG(n >= 0, "negative length");
  cudaStream_t st = S(stream);
  double* scratch = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&scratch, sizeof(double) * 592, st));
  const int rc = vec_amax(n, C2(x), out, scratch, st);
  cudaFreeAsync(scratch, st);
  return rc;
}

int rs_lincomb(int64_t n, int32_t nv, const rs_complex* const* vs, const double* coef_re,
               const double* coef_im, rs_complex* out, void* stream) {
  RS_CHECK_ARG(n >= 0, "negative length");
  return vec_lincomb(n, nv, reinterpret_cast<const double2* const*>(vs), coef_re, coef_im, M2(out),
                     S(stream));
}

int rs_block_extract(int64_t nrows, int32_t block, int32_t col0, const int32_t* rp,
                     const int32_t* ci, const rs_complex* v, int32_t* out_rp, int32_t* out_ci,
                     rs_complex* out_v, int64_t* nnz, void* stream) {
  RS_CHECK_ARG(block >= 1, "block size must be >= 1");
  return block_extract(nrows, block, col0, rp, ci, C2(v), out_rp, out_ci, M2(out_v), nnz,
                       S(stream));
}

}  // extern "C"
