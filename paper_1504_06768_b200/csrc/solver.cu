// Device-resident steady-state solver: one CTA per system runs a whole
//   * inverse_power (steady.py:177-260) with inner = direct LU apply,
//     BiCGStab (krylov.py:181-291) or GMRES(m) (krylov.py:67-178), or
//   * solve_iterative / solve_direct on the trace-modified system
//     (steady.py:137-168, 116-134),
// with the reference control flow reproduced branch for branch: monitor on the
// preconditioned residual, true-residual confirmation, target *= 0.1
// tightening, the 0.5*prev stall exit, breakdown tests, BiCGStab's half-step
// restart, GMRES happy breakdown and zero-diagonal breakdown, the outer
// phase-aligned difference and the infinity-norm plain residual test.
//
// Everything a step needs (matrix, factors, vectors) stays in L2 / shared
// memory and no scalar crosses to the host until the solve ends, so a solve
// costs one launch.  A batch of B independent systems (config-4 sweep) is a
// grid of B CTAs.
#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "colsweep.cuh"
#include "kernels.cuh"
#include "cta_ops.cuh"
#include "solver.cuh"

namespace rs {

namespace {

__device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
  // Smith's algorithm (scaled), as CPython/numpy complex division.
  if (fabs(b.x) >= fabs(b.y)) {
    if (b.x == 0.0 && b.y == 0.0) return make_double2(a.x / b.x, a.y / b.x);
    const double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  }
  const double r = b.x / b.y, d = b.x * r + b.y;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double cabs(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ bool finite2(double2 a) {
  return isfinite(a.x) && isfinite(a.y);
}

struct Ctx {
  int n;
  // system matrix
  const int32_t *Arp, *Aci;
  const double2* Av;
  // preconditioner
  const int32_t *Lrp, *Lci, *Urp, *Uci, *pinv, *colp;
  const double2 *Lv, *Uv, *rU;
  bool have_M;
  // column sweeps on the raw CSC factors (colsweep.cuh): the launch's
  // arguments, read in place from the grid-constant parameter space
  bool csc;
  const SolverArgs* sa;
  // scratch
  double2* y;   // triangular-solve scratch P (smem or global)
  double2* y2;  // triangular-solve scratch Q
  double* red;
  double2* small;  // GMRES H/g/sn (global, per system)
  double* cs;
  // residual history (krylov._trace_write, krylov.py:62-64); null: off
  double* trace;
  int32_t* trace_count;
  int32_t trace_cap;
};

__device__ __forceinline__ void trace_write(const Ctx& C, int iteration, double residual) {
  if (C.trace && threadIdx.x == 0) {
    const int k = *C.trace_count;
    if (k < C.trace_cap) {
      C.trace[2 * k] = (double)iteration;
      C.trace[2 * k + 1] = residual;
    }
    *C.trace_count = k + 1;
  }
}

// out = M^{-1} in  (factor.solve_lu, factor.py:137-149: y[pinv] = b; L; U;
// x[q] = y with q = identity on the natural/RCM path).  out may alias in.
// Two scratch vectors P, Q (shared memory when they fit): P = permuted rhs,
// Q = lower-solve output, then P is reused as the upper-solve output.
// M^{-1} through the reference column loops on shared memory: one
// out-of-line copy shared by every call site (the sweep code is large).
// Shared memory: [y: 16 n][factor staging ring].
__device__ __noinline__ void csc_psolve(const SolverArgs* a, const double2* in, double2* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a->n;
  const int64_t b = blockIdx.x;
  const bool yg = a->col_y_global != 0;  // sweep vector in global memory (large n)
  double2* P = yg ? a->ywork + b * a->ywork_stride : reinterpret_cast<double2*>(smem);
  const int32_t* pinv = a->pinv + b * n;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) P[pinv[i]] = in[i];
  __syncthreads();
  cta::ColStream Ls, Us;
  const int32_t l0 = a->Lso[b * n], u0 = a->Uso[b * n];
  Ls.idx = a->Lsi + cta::CW * (int64_t)l0;
  Ls.val = a->Lsv + cta::CW * (int64_t)l0;
  Ls.meta = a->Lsm + l0;
  Ls.rd = nullptr;
  Ls.rows = a->Lso[b * n + n] - l0;
  Us.idx = a->Usi + cta::CW * (int64_t)u0;
  Us.val = a->Usv + cta::CW * (int64_t)u0;
  Us.meta = a->Usm + u0;
  Us.rd = a->Usr + u0;
  Us.rows = a->Uso[b * n + n] - u0;
  const int win = yg ? a->col_win : 0;
  const size_t ybytes = win ? 16 * ((size_t)win + 1) : (yg ? 0 : cta::col_y_bytes(n));
  const cta::ColRing ring = cta::col_ring_at(smem + ybytes, a->ring_R);
  if (win) {
    cta::YWindow w;
    w.s = reinterpret_cast<double2*>(smem);
    w.g = P;
    w.mask = win - 1;
    w.panel = win - a->col_reach - 1;
    cta::col_lu_sweeps<unsigned long long>(n, Ls, Us, ring, P, a->col_consumers, &w);
  } else if (yg) {
    cta::col_lu_sweeps<unsigned long long>(n, Ls, Us, ring, P, a->col_consumers);
  } else {
    cta::col_lu_sweeps<unsigned>(n, Ls, Us, ring, P, a->col_consumers);
  }
  // x[q] = y (factor.py:147-148) when the factors are column pre-ordered
  const int32_t* colp = a->colp ? a->colp + b * n : nullptr;
  if (colp)
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = P[colp[i]];
  else
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = P[i];
  __syncthreads();
}

// tuning hook: [0] cycles in psolve, [1] psolve calls, [2] cycles in apply_op SpMV
__device__ unsigned long long* g_solver_prof = nullptr;

__device__ void psolve_body(const Ctx& C, const double2* in, double2* out);
__device__ void psolve(const Ctx& C, const double2* in, double2* out) {
  unsigned long long* const pf = (blockIdx.x == 0 && threadIdx.x == 0) ? g_solver_prof : nullptr;
  const long long t0 = pf ? clock64() : 0;
  psolve_body(C, in, out);
  if (pf) {
    pf[0] += clock64() - t0;
    pf[1] += 1;
  }
}

typedef void (*psolve_fn_t)(const SolverArgs*, const double2*, double2*);
__device__ psolve_fn_t g_csc_psolve = csc_psolve;

__device__ void psolve_body(const Ctx& C, const double2* in, double2* out) {
  const int n = C.n;
  if (!C.have_M) {
    if (in != out)
      for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = in[i];
    __syncthreads();
    return;
  }
  double2* P = C.y;
  double2* Q = C.y2;
  if (C.csc) {  // reference column loops on shared memory (colsweep.cuh)
    // reached by an indirect call: the standard ABI gives the sweeps their
    // own register allocation instead of what the Krylov code leaves free
    // (see trisell.cuh: the same direct call cost the grid solver 1.9x)
    psolve_fn_t fn = *(volatile psolve_fn_t*)&g_csc_psolve;
    fn(C.sa, in, out);
    return;
  }
  const double2 s = cta::sentinel2();
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    P[C.pinv[i]] = in[i];
    Q[i] = s;
  }
  __syncthreads();
  cta::lower_solve(n, C.Lrp, C.Lci, C.Lv, P, Q);
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) P[i] = s;
  __syncthreads();
  cta::upper_solve(n, C.Urp, C.Uci, C.Uv, C.rU, Q, P);
  __syncthreads();
  if (C.colp) {  // x[q] = y (factor.py:147-148); P is scratch, never the output
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = P[C.colp[i]];
  } else if (out != P) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = P[i];
  }
  __syncthreads();
}

// out = M^{-1} (A v)
__device__ void apply_op(const Ctx& C, const double2* v, double2* tmp, double2* out) {
  unsigned long long* const pf = (blockIdx.x == 0 && threadIdx.x == 0) ? g_solver_prof : nullptr;
  const long long t0 = pf ? clock64() : 0;
  cta::spmv(C.n, C.Arp, C.Aci, C.Av, v, tmp);
  __syncthreads();
  if (pf) pf[2] += clock64() - t0;
  psolve(C, tmp, out);
}

struct IterOut {
  int iterations;
  double final_residual;
  bool converged, breakdown;
};

// Workspace vectors, each n complex128.
struct Vecs {
  double2 *x, *r, *rhat, *p, *v, *s, *t, *pb, *tmp;
  double2* V;  // (m+1) x n for GMRES
};

__device__ void zero(int n, double2* a) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = make_double2(0.0, 0.0);
}

// krylov.bicgstab, krylov.py:181-291
__device__ IterOut bicgstab(const Ctx& C, const double2* b, const Vecs& W, double tol,
                            int max_iter) {
  const int n = C.n;
  IterOut out{0, 0.0, false, false};
  const double bnorm = cta::nrm2(n, b, C.red);
  if (bnorm == 0.0) {
    zero(n, W.x);
    __syncthreads();
    out.converged = true;
    return out;
  }
  psolve(C, b, W.pb);
  const double pbnorm = cta::nrm2(n, W.pb, C.red);
  if (pbnorm == 0.0 || !isfinite(pbnorm)) {
    zero(n, W.x);
    __syncthreads();
    out.final_residual = bnorm;
    out.breakdown = true;
    return out;
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    W.x[i] = make_double2(0.0, 0.0);
    W.r[i] = W.pb[i];
    W.rhat[i] = W.pb[i];
    W.v[i] = make_double2(0.0, 0.0);
    W.p[i] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  double rhat_norm = cta::nrm2(n, W.rhat, C.red);
  double2 rho_prev = make_double2(1.0, 0.0), alpha = make_double2(1.0, 0.0),
          omega = make_double2(1.0, 0.0);
  double target = tol * pbnorm;
  double prev_true = INFINITY;
  int it = 0;
  while (it < max_iter) {
    const double rnorm = cta::nrm2(n, W.r, C.red);
    trace_write(C, it, rnorm);
    if (rnorm <= target) {
      const double true_res = cta::resid_nrm2(n, C.Arp, C.Aci, C.Av, W.x, b, C.red);
      if (true_res <= tol * bnorm) {
        out.converged = true;
        break;
      }
      if (true_res >= 0.5 * prev_true) break;
      prev_true = true_res;
      target *= 0.1;
    }
    const double2 rho = cta::vdot(n, W.rhat, W.r, C.red);
    const double arho = cabs(rho);
    if (arho < 1e-30 || arho < 1e-16 * rhat_norm * rnorm) {
      out.breakdown = true;
      break;
    }
    if (it == 0) {
      for (int i = threadIdx.x; i < n; i += blockDim.x) W.p[i] = W.r[i];
    } else {
      const double2 beta = cmul(cdiv(rho, rho_prev), cdiv(alpha, omega));
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double2 d = csub(W.p[i], cmul(omega, W.v[i]));
        W.p[i] = cadd(W.r[i], cmul(beta, d));
      }
    }
    __syncthreads();
    apply_op(C, W.p, W.tmp, W.v);
    const double2 denom = cta::vdot(n, W.rhat, W.v, C.red);
    if (denom.x == 0.0 && denom.y == 0.0) {
      out.breakdown = true;
      break;
    }
    alpha = cdiv(rho, denom);
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      W.s[i] = csub(W.r[i], cmul(alpha, W.v[i]));
    __syncthreads();
    ++it;
    const double snorm = cta::nrm2(n, W.s, C.red);
    if (snorm <= target) {
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        W.x[i] = cadd(W.x[i], cmul(alpha, W.p[i]));
      __syncthreads();
      const double true_res = cta::resid_nrm2(n, C.Arp, C.Aci, C.Av, W.x, b, C.red);
      if (true_res <= tol * bnorm) {
        out.converged = true;
        break;
      }
      if (true_res >= 0.5 * prev_true) break;
      prev_true = true_res;
      target *= 0.1;
      for (int i = threadIdx.x; i < n; i += blockDim.x) {
        W.r[i] = W.s[i];
        W.rhat[i] = W.s[i];
        W.v[i] = make_double2(0.0, 0.0);
        W.p[i] = make_double2(0.0, 0.0);
      }
      __syncthreads();
      rhat_norm = cta::nrm2(n, W.rhat, C.red);
      rho_prev = alpha = omega = make_double2(1.0, 0.0);
      continue;
    }
    apply_op(C, W.s, W.tmp, W.t);
    const double2 tt = cta::vdot(n, W.t, W.t, C.red);
    if (tt.x == 0.0 && tt.y == 0.0) {
      out.breakdown = true;
      break;
    }
    omega = cdiv(cta::vdot(n, W.t, W.s, C.red), tt);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double2 xa = cadd(W.x[i], cmul(alpha, W.p[i]));
      W.x[i] = cadd(xa, cmul(omega, W.s[i]));
      W.r[i] = csub(W.s[i], cmul(omega, W.t[i]));
    }
    __syncthreads();
    rho_prev = rho;
    if (omega.x == 0.0 && omega.y == 0.0) {
      out.breakdown = true;
      break;
    }
  }
  out.iterations = it;
  out.final_residual = cta::resid_nrm2(n, C.Arp, C.Aci, C.Av, W.x, b, C.red);
  return out;
}

// krylov.gmres, krylov.py:67-178.  H is (m+1) x m row-major in C.small,
// followed by g (m+1) and sn (m); cs (m) in C.cs.  Scalar Givens work is done
// by thread 0 and published through global memory + a barrier.
__device__ IterOut gmres(const Ctx& C, const double2* b, const Vecs& W, double tol,
                         int max_iter, int m) {
  const int n = C.n;
  IterOut out{0, 0.0, false, false};
  double2* H = C.small;
  double2* g = H + (m + 1) * m;
  double2* sn = g + (m + 1);
  double2* yv = sn + m;
  double* cs = C.cs;
  const double bnorm = cta::nrm2(n, b, C.red);
  if (bnorm == 0.0) {
    zero(n, W.x);
    __syncthreads();
    out.converged = true;
    return out;
  }
  psolve(C, b, W.pb);
  const double pbnorm = cta::nrm2(n, W.pb, C.red);
  if (pbnorm == 0.0 || !isfinite(pbnorm)) {
    zero(n, W.x);
    __syncthreads();
    out.final_residual = bnorm;
    out.breakdown = true;
    return out;
  }
  zero(n, W.x);
  __syncthreads();
  double target = tol * pbnorm;
  int total = 0;
  bool converged = false, breakdown = false, invariant = false;
  double prev_true = INFINITY;
  __shared__ double s_res;
  __shared__ int s_flag;
  while (total < max_iter && !converged && !invariant) {
    double2* r = W.r;
    if (total) {
      apply_op(C, W.x, W.tmp, r);
      for (int i = threadIdx.x; i < n; i += blockDim.x) r[i] = csub(W.pb[i], r[i]);
    } else {
      for (int i = threadIdx.x; i < n; i += blockDim.x) r[i] = W.pb[i];
    }
    __syncthreads();
    const double beta = cta::nrm2(n, r, C.red);
    bool monitor_hit = beta <= target;
    double res = beta;
    if (!monitor_hit) {
      double2* V0 = W.V;
      for (int i = threadIdx.x; i < n; i += blockDim.x)
        V0[i] = make_double2(r[i].x / beta, r[i].y / beta);
      if (threadIdx.x == 0) {
        for (int i = 0; i < (m + 1) * m; ++i) H[i] = make_double2(0.0, 0.0);
        for (int i = 0; i <= m; ++i) g[i] = make_double2(0.0, 0.0);
        g[0] = make_double2(beta, 0.0);
      }
      __syncthreads();
      int j = 0;
      while (j < m && total < max_iter) {
        double2* Vj = W.V + (size_t)j * n;
        double2* w = W.r;  // reuse r as the Arnoldi vector
        apply_op(C, Vj, W.tmp, w);
        ++total;
        for (int i = 0; i <= j; ++i) {
          const double2* Vi = W.V + (size_t)i * n;
          const double2 hij = cta::vdot(n, Vi, w, C.red);
          for (int e = threadIdx.x; e < n; e += blockDim.x) w[e] = csub(w[e], cmul(hij, Vi[e]));
          if (threadIdx.x == 0) H[i * m + j] = hij;
          __syncthreads();
        }
        const double hnext = cta::nrm2(n, w, C.red);
        if (hnext > 0.0) {
          double2* Vn = W.V + (size_t)(j + 1) * n;
          for (int e = threadIdx.x; e < n; e += blockDim.x)
            Vn[e] = make_double2(w[e].x / hnext, w[e].y / hnext);
        }
        if (threadIdx.x == 0) {
          for (int i = 0; i < j; ++i) {
            const double2 hi = H[i * m + j], hi1 = H[(i + 1) * m + j];
            const double2 t = cadd(make_double2(cs[i] * hi.x, cs[i] * hi.y), cmul(sn[i], hi1));
            const double2 csn = make_double2(-sn[i].x, sn[i].y);  // -conj(sn)
            H[(i + 1) * m + j] = cadd(cmul(csn, hi), make_double2(cs[i] * hi1.x, cs[i] * hi1.y));
            H[i * m + j] = t;
          }
          const double2 al = H[j * m + j];
          const double aal = cabs(al);
          const double denom = hypot(aal, hnext);
          if (denom == 0.0) {
            cs[j] = 1.0;
            sn[j] = make_double2(0.0, 0.0);
          } else if (al.x == 0.0 && al.y == 0.0) {
            cs[j] = 0.0;
            sn[j] = make_double2(1.0, 0.0);
          } else {
            cs[j] = aal / denom;
            const double2 ph = make_double2(al.x / aal, al.y / aal);
            sn[j] = make_double2(ph.x * (hnext / denom), ph.y * (hnext / denom));
          }
          H[j * m + j] = cadd(make_double2(cs[j] * al.x, cs[j] * al.y),
                              make_double2(sn[j].x * hnext, sn[j].y * hnext));
          const double2 gj = g[j];
          g[j + 1] = cmul(make_double2(-sn[j].x, sn[j].y), gj);
          g[j] = make_double2(cs[j] * gj.x, cs[j] * gj.y);
          s_res = cabs(g[j + 1]);
        }
        __syncthreads();
        res = s_res;
        ++j;
        trace_write(C, total, res);
        if (hnext == 0.0) {
          invariant = true;
          break;
        }
        if (res <= target) break;
      }
      // zero diagonal -> breakdown; else back-substitute and update x
      if (threadIdx.x == 0) {
        int bad = 0;
        for (int i = 0; i < j; ++i) {
          const double2 d = H[i * m + i];
          if (d.x == 0.0 && d.y == 0.0) bad = 1;
        }
        if (!bad) {
          for (int i = j - 1; i >= 0; --i) {
            double2 acc = make_double2(0.0, 0.0);
            for (int k = i + 1; k < j; ++k) acc = cadd(acc, cmul(H[i * m + k], yv[k]));
            yv[i] = cdiv(csub(g[i], acc), H[i * m + i]);
          }
        }
        s_flag = bad;
      }
      __syncthreads();
      if (s_flag) {
        breakdown = true;
        break;
      }
      for (int e = threadIdx.x; e < n; e += blockDim.x) {
        double2 acc = make_double2(0.0, 0.0);
        for (int k = 0; k < j; ++k) acc = cadd(acc, cmul(yv[k], W.V[(size_t)k * n + e]));
        W.x[e] = cadd(W.x[e], acc);
      }
      __syncthreads();
      monitor_hit = res <= target || invariant;
    }
    if (monitor_hit) {
      const double true_res = cta::resid_nrm2(n, C.Arp, C.Aci, C.Av, W.x, b, C.red);
      if (true_res <= tol * bnorm) {
        converged = true;
      } else if (invariant || true_res >= 0.5 * prev_true) {
        break;
      } else {
        prev_true = true_res;
        target *= 0.1;
      }
    }
  }
  out.iterations = total;
  out.converged = converged;
  out.breakdown = breakdown;
  out.final_residual = cta::resid_nrm2(n, C.Arp, C.Aci, C.Av, W.x, b, C.red);
  return out;
}

}  // namespace

// MAXT = 512: batches (128-thread CTAs, four per SM, 128 registers);
// MAXT = 256: a lone system -- 255 registers, so the out-of-line
// column-sweep consumer runs without spills (it spilled in the loop at 128).
template <int MAXT>
__global__ void __launch_bounds__(MAXT, 1) steady_solver_kernel(SolverArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[32 * 4];
  const int b = blockIdx.x;
  const int n = a.n;
  const int64_t bn = (int64_t)b * n;
  SolveStats* st = a.stats + b;
  if (a.skip && a.skip[b]) {  // e.g. this system's factorization hit a zero pivot
    for (int i = threadIdx.x; i < n; i += blockDim.x) a.xout[bn + i] = make_double2(0.0, 0.0);
    if (threadIdx.x == 0) {
      *st = SolveStats{};
      st->status = SOLVE_SKIPPED;
    }
    return;
  }

  Ctx C;
  C.n = n;
  C.Arp = a.Arp + bn;  // local-offset views: rows of system b
  C.Aci = a.Aci;
  C.Av = a.Av;
  C.have_M = a.Lrp != nullptr || a.ring_R > 0;
  C.Lrp = a.Lrp ? a.Lrp + bn : nullptr;
  C.Lci = a.Lci;
  C.Lv = a.Lv;
  C.Urp = a.Urp ? a.Urp + bn : nullptr;
  C.Uci = a.Uci;
  C.Uv = a.Uv;
  C.rU = a.rU ? a.rU + bn : nullptr;
  C.pinv = a.pinv ? a.pinv + bn : nullptr;
  C.colp = a.colp ? a.colp + bn : nullptr;
  const bool tr = a.trace && b == 0 && a.mode >= MODE_LIN_DIRECT;
  C.trace = tr ? a.trace : nullptr;
  C.trace_count = a.trace_count;
  C.trace_cap = a.trace_cap;
  if (tr && threadIdx.x == 0) *a.trace_count = 0;
  C.red = red;
  double2* ws = a.work + (int64_t)b * a.work_stride;
  C.csc = a.ring_R > 0;
  C.sa = a.self;  // device copy of the launch arguments
  if (C.csc) {
    C.y = reinterpret_cast<double2*>(smem);
    C.y2 = nullptr;
  } else if (a.y_in_smem) {
    C.y = reinterpret_cast<double2*>(smem);
    C.y2 = C.y + n;
  } else {
    C.y = ws;  // slots 0 and 1
    C.y2 = ws + n;
  }
  const int m = a.restart_m;
  C.small = ws + 2 * (int64_t)n;  // (m+1)*m + (m+1) + m + m complex
  C.cs = reinterpret_cast<double*>(C.small + (m + 1) * m + (m + 1) + 2 * m);
  const int64_t small_slots = ((m + 1) * m + (m + 1) + 3 * m + n - 1) / n + 1;
  double2* vb = ws + (int64_t)n * (2 + small_slots);
  Vecs W;
  W.x = vb + 0 * (int64_t)n;
  W.r = vb + 1 * (int64_t)n;
  W.rhat = vb + 2 * (int64_t)n;
  W.p = vb + 3 * (int64_t)n;
  W.v = vb + 4 * (int64_t)n;
  W.s = vb + 5 * (int64_t)n;
  W.t = vb + 6 * (int64_t)n;
  W.pb = vb + 7 * (int64_t)n;
  W.tmp = vb + 8 * (int64_t)n;
  W.V = vb + 9 * (int64_t)n;  // (m+1) vectors; BiCGStab does not use them
  double2* xo = vb + (9 + (int64_t)m + 1) * n;      // outer iterate
  double2* yo = vb + (10 + (int64_t)m + 1) * n;     // inner result / aligned
  const double2* in = a.rhs + bn;
  double2* out = a.xout + bn;

  // local-index adjustment: CSR arrays are global block-diagonal; the row
  // pointers above are offset by b*n, entries are absolute positions.
  if (threadIdx.x == 0) {
    st->status = 0;
    st->outer = 0;
    st->inner_last = 0;
    st->inner_total = 0;
    st->converged = 0;
    st->breakdown = 0;
    st->final_residual = 0.0;
    st->condest = 0.0;
  }

  if (a.want_condest && C.have_M) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) W.tmp[i] = make_double2(1.0, 0.0);
    __syncthreads();
    psolve(C, W.tmp, W.pb);
    double mx = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) mx = fmax(mx, cabs(W.pb[i]));
    mx = cta::block_max(mx, red);
    if (threadIdx.x == 0) st->condest = mx;
  }

  const int mode = a.mode;
  if (mode == MODE_LIN_DIRECT || mode == MODE_LIN_BICGSTAB || mode == MODE_LIN_GMRES) {
    IterOut io{0, 0.0, true, false};
    if (mode == MODE_LIN_DIRECT) {
      psolve(C, in, W.x);
    } else if (mode == MODE_LIN_BICGSTAB) {
      io = bicgstab(C, in, W, a.tol, a.max_iter);
    } else {
      io = gmres(C, in, W, a.tol, a.max_iter, m);
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = W.x[i];
    if (threadIdx.x == 0) {
      st->inner_last = io.iterations;
      st->inner_total = io.iterations;
      st->converged = io.converged;
      st->breakdown = io.breakdown;
      st->final_residual = io.final_residual;
    }
    return;
  }

  // ---- inverse power, steady.py:211-245 -----------------------------------
  // start vector (drawn on the host, steady.py:171-174) normalised here
  {
    const double nx = cta::nrm2(n, in, red);
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      xo[i] = make_double2(in[i].x / nx, in[i].y / nx);
    __syncthreads();
  }
  const double tol = a.tol;
  int outer = 0, inner_total = 0, inner_last = 0;
  bool converged = false;
  int status = 0;
  while (outer < a.max_outer) {
    double2* y = yo;
    if (mode == MODE_INV_DIRECT) {
      psolve(C, xo, y);
    } else {
      IterOut io = (mode == MODE_INV_BICGSTAB)
                       ? bicgstab(C, xo, W, tol / 10.0, a.max_iter)
                       : gmres(C, xo, W, tol / 10.0, a.max_iter, m);
      inner_last = io.iterations;
      inner_total += io.iterations;
      int nonfin = 0;
      for (int i = threadIdx.x; i < n; i += blockDim.x) nonfin |= !finite2(W.x[i]);
      nonfin = __syncthreads_or(nonfin);
      if (io.breakdown || nonfin) {
        status = io.breakdown ? SOLVE_INNER_BREAKDOWN : SOLVE_INNER_NONFINITE;
        break;
      }
      if (cta::nrm2(n, W.x, red) == 0.0) {
        status = SOLVE_INNER_NO_PROGRESS;
        break;
      }
      for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = W.x[i];
      __syncthreads();
    }
    const double ny = cta::nrm2(n, y, red);
    if (ny == 0.0 || !isfinite(ny)) {
      status = SOLVE_UNUSABLE_VECTOR;
      break;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      y[i] = make_double2(y[i].x / ny, y[i].y / ny);
    __syncthreads();
    ++outer;
    const double2 ov = cta::vdot(n, y, xo, red);
    double2 ph = make_double2(1.0, 0.0);
    const bool ovnz = !(ov.x == 0.0 && ov.y == 0.0);
    if (ovnz) {
      const double aov = cabs(ov);
      ph = make_double2(ov.x / aov, ov.y / aov);
    }
    double acc[1];
    cta::vsum<1>(
        n,
        [&](int i, double (&s)[1]) {
          const double2 al = ovnz ? cmul(y[i], ph) : y[i];
          const double2 d = csub(al, xo[i]);
          s[0] = __fma_rn(d.x, d.x, __fma_rn(d.y, d.y, s[0]));
        },
        acc, red);
    const double diff = sqrt(acc[0]);
    // resid_inf = max |L_plain,perm y|
    double mx = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int p0 = a.Prp[bn + i], p1 = a.Prp[bn + i + 1];
      double2 s = make_double2(0.0, 0.0);
      if (p0 < p1) {
        s = cmul_plain(a.Pv[p0], y[a.Pci[p0]]);
        for (int p = p0 + 1; p < p1; ++p) s = cadd(s, cmul_plain(a.Pv[p], y[a.Pci[p]]));
      }
      mx = fmax(mx, cabs(s));
    }
    const double resid_inf = cta::block_max(mx, red);
    for (int i = threadIdx.x; i < n; i += blockDim.x) xo[i] = y[i];
    __syncthreads();
    if (diff <= tol || resid_inf <= tol) {
      converged = true;
      break;
    }
  }
  if (status == 0 && !converged) status = SOLVE_POWER_NOT_CONVERGED;
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = xo[i];
  if (threadIdx.x == 0) {
    st->status = status;
    st->outer = outer;
    st->inner_last = inner_last;
    st->inner_total = inner_total;
    st->converged = converged;
  }
}

int64_t solver_work_stride(int32_t n, int restart_m) {
  const int m = restart_m;
  const int64_t small_slots = ((int64_t)(m + 1) * m + (m + 1) + 3 * m + n - 1) / n + 1;
  return (int64_t)n * (2 + small_slots + 9 + (m + 1) + 2);
}

// Consumer warps of the column sweeps: several for a lone large system whose
// columns span several 64-entry stream rows (config 3: ~175 entries per
// column), one otherwise (a batch is bound by systems per SM, and short
// columns have nothing to share).  RHOSOLVE_COL_CONSUMERS overrides.
// Sliding window for a lone system whose sweep vector lives in global memory:
// the largest power of two that fits next to the ring, provided it leaves a
// panel of at least 64 columns beyond the factors' reach.  0 = no window.
static int col_window_for(const SolverArgs& a, int max_smem) {
  if (getenv("RHOSOLVE_COL_WINDOW") && atoi(getenv("RHOSOLVE_COL_WINDOW")) == 0) return 0;
  if (!a.col_y_global || a.col_reach <= 0 || a.B > 148 || a.ring_R <= 0) return 0;
  for (int win = 16384; win >= 256; win >>= 1) {
    if (16 * ((size_t)win + 1) + cta::col_ring_bytes(a.ring_R) + 4096 > (size_t)max_smem) continue;
    return win - a.col_reach - 1 >= 64 ? win : 0;
  }
  return 0;
}

static int col_consumers_for(const SolverArgs& a) {
  if (const char* e = getenv("RHOSOLVE_COL_CONSUMERS")) return std::max(1, atoi(e));
  if (a.ring_R <= 0 || a.B > 148 || !a.Lso || !a.Uso) return 1;
  // measured on config 3 (apply, ms): global y 81 / 75 / 68 for 1 / 4 / 6 consumers,
  // sliding window 101 / 67 / 51 / 46 for 1 / 2 / 4 / 6
  return a.col_y_global ? 6 : 1;
}

int launch_steady_solver(const SolverArgs& a, cudaStream_t st) {
  if (a.B == 0) return RS_OK;
  int dev, max_smem;
  RS_CUDA_TRY(cudaGetDevice(&dev));
  RS_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int win = col_window_for(a, max_smem);
  size_t smem = a.ring_R > 0
                    ? (win ? 16 * ((size_t)win + 1) : (a.col_y_global ? 0 : cta::col_y_bytes(a.n))) +
                          cta::col_ring_bytes(a.ring_R)
                    : (a.y_in_smem ? 32 * (size_t)a.n : 0);
  if (smem + 2048 > (size_t)max_smem) {
    set_error("steady solver: n=%d needs %zu B of shared memory", a.n, smem);
    return RS_ERR_UNSUPPORTED;
  }
  const bool lone = a.threads <= 256 && a.B <= 148;
  auto kern = lone ? steady_solver_kernel<256> : steady_solver_kernel<512>;
  RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  SolverArgs la = a;
  la.ywork = a.work;  // slot 0 of each system's workspace (y, then y2 = dummy)
  la.ywork_stride = a.work_stride;
  la.col_consumers = col_consumers_for(a);
  la.col_win = win;
  SolverArgs* dev_args = nullptr;
  if (la.ring_R > 0) {  // the out-of-line column sweeps read the arguments from here
    RS_CUDA_TRY(cudaMallocAsync(&dev_args, sizeof(SolverArgs), st));
    RS_CUDA_TRY(cudaMemcpyAsync(dev_args, &la, sizeof(SolverArgs), cudaMemcpyHostToDevice, st));
    la.self = dev_args;
  }
  kern<<<a.B, a.threads, smem, st>>>(la); ::rs::count_launch();
  if (dev_args) cudaFreeAsync(dev_args, st);
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

}  // namespace rs

namespace rs {

// Standalone preconditioner apply (factor.solve_lu), one CTA per system.
__global__ void __launch_bounds__(512) lu_solve_kernel(SolverArgs a, int y_in_smem) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int b = blockIdx.x;
  const int n = a.n;
  const int64_t bn = (int64_t)b * n;
  Ctx C;
  C.n = n;
  C.have_M = true;
  C.Lrp = a.Lrp + bn;
  C.Lci = a.Lci;
  C.Lv = a.Lv;
  C.Urp = a.Urp + bn;
  C.Uci = a.Uci;
  C.Uv = a.Uv;
  C.rU = a.rU + bn;
  C.pinv = a.pinv + bn;
  C.colp = a.colp ? a.colp + bn : nullptr;
  C.trace = nullptr;
  C.csc = a.ring_R > 0;
  C.sa = a.self;  // device copy of the launch arguments
  if (C.csc) {
    C.y = reinterpret_cast<double2*>(smem);
    C.y2 = nullptr;
  } else if (y_in_smem) {
    C.y = reinterpret_cast<double2*>(smem);
    C.y2 = C.y + n;
  } else {
    C.y = a.work + 2 * bn;
    C.y2 = C.y + n;
  }
  psolve(C, a.rhs + bn, a.xout + bn);
}

__global__ void pivot_recip_kernel(int B, int32_t n, const int32_t* __restrict__ Up,
                                   const double2* __restrict__ Ux, int64_t capU,
                                   double2* __restrict__ rd) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * n) return;
  const int64_t b = t / n, k = t % n;
  const int32_t e = Up[b * (n + 1) + k + 1];
  // a system whose factorization stopped early has no column k: leave 0
  rd[t] = e > Up[b * (n + 1) + k] ? recipc(Ux[b * capU + e - 1]) : make_double2(0.0, 0.0);
}

int pivot_recip(int B, int32_t n, const int32_t* Up, const double2* Ux, int64_t capU,
                double2* rd, cudaStream_t st) {
  if (!B || !n) return RS_OK;
  const int64_t N = (int64_t)B * n;
  pivot_recip_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(B, n, Up, Ux, capU, rd);
  ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

// ---- column streams (colsweep.cuh) ---------------------------------------
__global__ void col_stream_count_kernel(int B, int32_t n, int upper, const int32_t* __restrict__ cp,
                                        int32_t* __restrict__ rows) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * n) return;
  const int64_t b = t / n;
  const int32_t j = (int32_t)(t % n);
  const int32_t c = upper ? n - 1 - j : j;
  const int32_t* p = cp + b * (n + 1);
  const int32_t len = p[c + 1] - p[c] - 1;  // off-diagonal entries
  rows[t] = len > 0 ? (len + cta::CW - 1) / cta::CW : 1;
}

// one warp per column: coalesced copy into its padded rows
__global__ void col_stream_fill_kernel(int B, int32_t n, int upper, const int32_t* __restrict__ cp,
                                       const int32_t* __restrict__ ci,
                                       const double2* __restrict__ cv, int64_t cap,
                                       const double2* __restrict__ rdiag,
                                       const int32_t* __restrict__ rowoff,
                                       int32_t* __restrict__ idx, double2* __restrict__ val,
                                       int32_t* __restrict__ meta, double2* __restrict__ rrd) {
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= (int64_t)B * n) return;
  const int64_t b = t / n;
  const int32_t j = (int32_t)(t % n);
  const int32_t c = upper ? n - 1 - j : j;
  const int32_t* p = cp + b * (n + 1);
  const int32_t s = upper ? p[c] : p[c] + 1;
  const int32_t len = p[c + 1] - p[c] - 1;
  const int32_t r0 = rowoff[t], nr = rowoff[t + 1] - r0;
  const int32_t* I = ci + b * cap;
  const double2* X = cv + b * cap;
  for (int32_t k = lane; k < cta::CW * nr; k += 32) {
    const int64_t o = cta::CW * (int64_t)r0 + k;
    if (k < len) {
      idx[o] = I[s + k];
      val[o] = X[s + k];
    } else {
      idx[o] = -1;
      val[o] = make_double2(0.0, 0.0);
    }
  }
  for (int32_t q = lane; q < nr; q += 32) {
    meta[r0 + q] = q > 0 ? 1 : 0;
    if (upper) rrd[r0 + q] = q == 0 ? rdiag[b * n + c] : make_double2(0.0, 0.0);
  }
}

int col_stream_build(int B, int32_t n, int upper, const int32_t* cp, const int32_t* ci,
                     const double2* cv, int64_t cap, const double2* rdiag, int32_t* rowoff,
                     int32_t* idx, double2* val, int32_t* meta, double2* rrd, int64_t* total,
                     cudaStream_t st) {
  const int64_t N = (int64_t)B * n;
  if (!idx) {
    int32_t* rows = nullptr;
    RS_CUDA_TRY(cudaMallocAsync(&rows, sizeof(int32_t) * (N + 1), st));
    if (N > 0) {
      col_stream_count_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(B, n, upper, cp, rows);
      ::rs::count_launch();
      RS_CUDA_TRY(cudaGetLastError());
    }
    int64_t tot = 0;
    const int rc = scan_counts(rows, rowoff, N, &tot, st);
    cudaFreeAsync(rows, st);
    if (rc) return rc;
    if (tot < 0 || tot >= ((int64_t)1 << 25)) {
      set_error("col_stream_build: %lld rows exceed 32-bit entry indexing", (long long)tot);
      return RS_ERR_OVERFLOW;
    }
    if (total) *total = tot;
    return RS_OK;
  }
  if (N > 0) {
    col_stream_fill_kernel<<<(unsigned)((N * 32 + 255) / 256), 256, 0, st>>>(
        B, n, upper, cp, ci, cv, cap, rdiag, rowoff, idx, val, meta, rrd);
    ::rs::count_launch();
    RS_CUDA_TRY(cudaGetLastError());
  }
  return RS_OK;
}

int col_ring_size(int32_t n, int B) {
  int dev = 0, max_smem = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) !=
      cudaSuccess)
    return 0;
  // batches keep four CTAs per SM resident: a 16-slot ring (21 KB); a lone
  // system takes a deeper ring
  for (int S = (B > 148 ? 16 : 64); S >= 8; S >>= 1)
    if (cta::col_y_bytes(n) + cta::col_ring_bytes(S) + 4096 <= (size_t)max_smem) return S;
  return 0;
}

int col_plan(int32_t n, int B, int* y_global) {
  const int S = col_ring_size(n, B);
  if (S > 0) {
    *y_global = 0;
    return S;
  }
  // the sweep vector stays in global memory; the ring alone in shared
  *y_global = 1;
  return B > 148 ? 16 : 64;
}

int launch_lu_solve(const SolverArgs& a, cudaStream_t st) {
  if (a.B == 0 || a.n == 0) return RS_OK;
  int dev, max_smem;
  RS_CUDA_TRY(cudaGetDevice(&dev));
  RS_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const int y_smem = 32 * (size_t)a.n + 2048 <= (size_t)max_smem;
  const int win = col_window_for(a, max_smem);
  size_t smem = a.ring_R > 0
                    ? (win ? 16 * ((size_t)win + 1) : (a.col_y_global ? 0 : cta::col_y_bytes(a.n))) +
                          cta::col_ring_bytes(a.ring_R)
                    : (y_smem ? 32 * (size_t)a.n : 0);
  if (a.ring_R <= 0 && !y_smem && !a.work) {
    set_error("lu_solve: n=%d needs global scratch", a.n);
    return RS_ERR_UNSUPPORTED;
  }
  RS_CUDA_TRY(cudaFuncSetAttribute(lu_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)smem));
  // column sweeps: 1 consumer + 4 producer warps; row sweeps: 16 warps
  SolverArgs la = a;
  la.ywork = a.work;  // 2 n per system: y, then the dummy slot
  la.ywork_stride = 2 * (int64_t)a.n;
  la.col_consumers = col_consumers_for(a);
  la.col_win = win;
  SolverArgs* dev_args = nullptr;
  if (la.ring_R > 0) {
    RS_CUDA_TRY(cudaMallocAsync(&dev_args, sizeof(SolverArgs), st));
    RS_CUDA_TRY(cudaMemcpyAsync(dev_args, &la, sizeof(SolverArgs), cudaMemcpyHostToDevice, st));
    la.self = dev_args;
  }
  lu_solve_kernel<<<a.B, a.ring_R > 0 ? (a.B > 148 ? 128 : 288) : 512, smem, st>>>(la, y_smem);
  ::rs::count_launch();
  if (dev_args) cudaFreeAsync(dev_args, st);
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

}  // namespace rs

namespace rs {

// Debug / tuning: time one triangular sweep variant in isolation.
// which: 0 = lower, 1 = upper; variant: 0 = thread-per-row, 1 = warp-per-row.
__global__ void __launch_bounds__(1024) tri_probe_kernel(int n, const int32_t* rp,
                                                         const int32_t* ci, const double2* v,
                                                         const double2* rU, const double2* in,
                                                         double2* gout, int which, int variant,
                                                         int smem_buf) {
  extern __shared__ __align__(16) unsigned char smem[];
  cta::FoldBuf* fb = reinterpret_cast<cta::FoldBuf*>(smem);
  double2* out = smem_buf ? reinterpret_cast<double2*>(smem + sizeof(cta::FoldBuf) * 32) : gout;
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = cta::sentinel2();
  __syncthreads();
  if (which == 0) {
    if (variant == 0) cta::tri_sweep<false>(n, rp, ci, v, rU, in, out);
    else if (variant == 1) cta::tri_sweep_warp<false>(n, rp, ci, v, rU, in, out);
    else cta::tri_sweep_fold<false>(n, rp, ci, v, rU, in, out, fb);
  } else {
    if (variant == 0) cta::tri_sweep<true>(n, rp, ci, v, rU, in, out);
    else if (variant == 1) cta::tri_sweep_warp<true>(n, rp, ci, v, rU, in, out);
    else cta::tri_sweep_fold<true>(n, rp, ci, v, rU, in, out, fb);
  }
  __syncthreads();
  if (smem_buf)
    for (int i = threadIdx.x; i < n; i += blockDim.x) gout[i] = out[i];
}

// SELL lane-per-row sweep in isolation (rp/ci/v = sptr/sci/sv of one system)
template <int G>
__global__ void __launch_bounds__(512) sell_probe_kernel(int n, const int32_t* sptr,
                                                         const int32_t* sci, const double2* sv,
                                                         const double2* rU, const double2* in,
                                                         double2* gout, int which,
                                                         int smem_buf) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* out = smem_buf ? reinterpret_cast<double2*>(smem) : gout;
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = cta::sentinel2();
  __syncthreads();
  if (which == 0) cta::tri_sweep_sell<false, G>(n, sptr, sci, sv, rU, in, out);
  else cta::tri_sweep_sell<true, G>(n, sptr, sci, sv, rU, in, out);
  __syncthreads();
  if (smem_buf)
    for (int i = threadIdx.x; i < n; i += blockDim.x) gout[i] = out[i];
}

}  // namespace rs

extern "C" int rs_debug_tri_probe(int n, const int32_t* rp, const int32_t* ci, const void* v,
                                  const void* rU, const void* in, void* out, int which,
                                  int variant, int smem_buf, int threads, void* stream) {
  if (variant >= 3) {  // 3: SELL G=4, 4: SELL G=2, 5: SELL G=8
    const size_t sm = smem_buf ? 16 * (size_t)n : 0;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    auto go = [&](auto kern) -> int {
      RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
      kern<<<1, threads, sm, s>>>(n, rp, ci, reinterpret_cast<const double2*>(v),
                                  reinterpret_cast<const double2*>(rU),
                                  reinterpret_cast<const double2*>(in),
                                  reinterpret_cast<double2*>(out), which, smem_buf);
      RS_CUDA_TRY(cudaGetLastError());
      return 0;
    };
    if (variant == 3) return go(rs::sell_probe_kernel<4>);
    if (variant == 4) return go(rs::sell_probe_kernel<2>);
    return go(rs::sell_probe_kernel<8>);
  }
  const size_t smem = (smem_buf ? 16 * (size_t)n : 0) + sizeof(rs::cta::FoldBuf) * 32;
  RS_CUDA_TRY(cudaFuncSetAttribute(rs::tri_probe_kernel,
                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  rs::tri_probe_kernel<<<1, threads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      n, rp, ci, reinterpret_cast<const double2*>(v), reinterpret_cast<const double2*>(rU),
      reinterpret_cast<const double2*>(in), reinterpret_cast<double2*>(out), which, variant,
      smem_buf);
  RS_CUDA_TRY(cudaGetLastError());
  return 0;
}

extern "C" int rs_debug_tri_backoff(unsigned nap_min, unsigned nap_max) {
  RS_CUDA_TRY(cudaMemcpyToSymbol(rs::cta::g_tri_nap_min, &nap_min, sizeof(unsigned)));
  RS_CUDA_TRY(cudaMemcpyToSymbol(rs::cta::g_tri_nap_max, &nap_max, sizeof(unsigned)));
  return 0;
}

extern "C" int rs_debug_solver_prof(void* buf) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(buf);
  RS_CUDA_TRY(cudaMemcpyToSymbol(rs::g_solver_prof, &p, sizeof(p)));
  return 0;
}

extern "C" int rs_debug_col_times(void* buf) {
  long long* p = reinterpret_cast<long long*>(buf);
  RS_CUDA_TRY(cudaMemcpyToSymbol(rs::cta::g_col_times, &p, sizeof(p)));
  return 0;
}

extern "C" int rs_debug_tri_times(void* buf) {
  long long* p = reinterpret_cast<long long*>(buf);
  RS_CUDA_TRY(cudaMemcpyToSymbol(rs::cta::g_tri_times, &p, sizeof(p)));
  return 0;
}
