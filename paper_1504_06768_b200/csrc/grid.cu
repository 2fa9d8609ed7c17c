// Grid-wide device-resident steady-state solver: ONE cooperative launch runs a
// whole inverse_power (steady.py:177-260) / solve_iterative / solve_direct
// (steady.py:137-168, 116-134) of a system too large for a single CTA, on
// every SM of the GPU:
//   * config 3 (n = 57,600, factors of ~20M entries),
//   * config 5 on one GPU (n = 2,560,000 with a block-Jacobi ILUTP whose
//     blocks are the row shards -- the factors are simply block diagonal).
// The control flow is the reference's, branch for branch, as in the one-CTA
// solver (solver.cu): BiCGStab krylov.py:181-291, GMRES(m) krylov.py:67-178.
//
// Building blocks
//   * SpMV: the bit-exact warp-per-32-rows kernel of spmv.cu as a grid-stride
//     device function (element-parallel products, row-sequential folds).
//   * Preconditioner apply: sync-free level-ordered triangular sweeps
//     (trisell.cuh), bit-identical to the reference column loops.
//   * Reductions: fixed element -> thread map, fixed shuffle tree, per-CTA
//     partials in global memory, ONE grid barrier, then every CTA folds the
//     partials in the same fixed order: all threads of the grid hold the same
//     bits, so every branch of the Krylov control flow is grid-uniform and no
//     scalar ever crosses to the host.  Partials alternate between two
//     buffers, so a reduction costs exactly one grid barrier.
//   * GMRES's Hessenberg / Givens scalars are recomputed redundantly by every
//     CTA in shared memory (identical inputs, identical results): no barrier.
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"
#include "cta_ops.cuh"
#include "solver.cuh"
#include "trisell.cuh"
#include "grid.cuh"

namespace cg = cooperative_groups;

namespace rs {

namespace {

constexpr int GT = 256;      // threads per CTA: 255 registers per thread, so the sweeps
                              // keep a whole chunk in registers (at 512 threads / 128
                              // registers sweep_slice spilled ~1 KB per call and a
                              // dependency hop cost 4,460 cycles after the sources
                              // were loaded)
constexpr int SP_UNROLL = 8;  // SpMV: chunks of 8 x 32 products per warp pass (two chunks in flight)
constexpr int SP_CH = 32 * SP_UNROLL;
constexpr int SP_SLOTS = SP_CH + SP_CH / 8;

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
__device__ __forceinline__ bool finite2(double2 a) { return isfinite(a.x) && isfinite(a.y); }

struct Q {
  cg::grid_group g;
  int tid, nth;   // global thread index / count
  int gw, ngw;    // global warp index / count
  double* red;    // shared, 32 * 8 doubles
  double* part;   // global, [2][gridDim.x][8]
  int flip;
  double2* stage;  // shared, warp-private SpMV staging (SP_SLOTS entries)
};

// Grid-wide deterministic sum of K values per element; every thread of the
// grid receives the same bits.  One grid barrier.
template <int K, class F>
__device__ __forceinline__ void gsum(Q& q, int n, F f, double (&out)[K]) {
  double acc[K];
#pragma unroll
  for (int k = 0; k < K; ++k) acc[k] = 0.0;
  for (int i = q.tid; i < n; i += q.nth) f(i, acc);
  cta::block_sum<K>(acc, q.red);
  double* all = q.part + (size_t)q.flip * gridDim.x * 8;
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) all[(size_t)blockIdx.x * 8 + k] = acc[k];
  }
  q.g.sync();
  double t[K];
#pragma unroll
  for (int k = 0; k < K; ++k) t[k] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x) {
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = __dadd_rn(t[k], __ldcg(all + (size_t)b * 8 + k));
  }
  cta::block_sum<K>(t, q.red);
#pragma unroll
  for (int k = 0; k < K; ++k) out[k] = t[k];
  q.flip ^= 1;
}

template <class F>
__device__ __forceinline__ double gmax(Q& q, int n, F f) {
  double m = 0.0;
  for (int i = q.tid; i < n; i += q.nth) m = fmax(m, f(i));
  m = cta::block_max(m, q.red);
  double* all = q.part + (size_t)q.flip * gridDim.x * 8;
  if (threadIdx.x == 0) all[(size_t)blockIdx.x * 8] = m;
  q.g.sync();
  double t = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += blockDim.x)
    t = fmax(t, __ldcg(all + (size_t)b * 8));
  t = cta::block_max(t, q.red);
  q.flip ^= 1;
  return t;
}

__device__ __forceinline__ double gnrm2(Q& q, int n, const double2* a) {
  double o[1];
  gsum<1>(q, n, [&](int i, double (&s)[1]) {
    const double2 x = a[i];
    s[0] = __fma_rn(x.x, x.x, __fma_rn(x.y, x.y, s[0]));
  }, o);
  return sqrt(o[0]);
}

// vdot(a, b) = sum conj(a_i) b_i (numpy.vdot)
__device__ __forceinline__ double2 gvdot(Q& q, int n, const double2* a, const double2* b) {
  double o[2];
  gsum<2>(q, n, [&](int i, double (&s)[2]) {
    const double2 x = a[i], y = b[i];
    s[0] = __fma_rn(x.x, y.x, __fma_rn(x.y, y.y, s[0]));
    s[1] = __fma_rn(x.x, y.y, __fma_rn(-x.y, y.x, s[1]));
  }, o);
  return make_double2(o[0], o[1]);
}

// y = A x, bit-exact with csr_matvec (_ckernels.pyx:34-50); the arithmetic of
// spmv_warp_kernel (spmv.cu) for one system, warps striding over 32-row
// groups.  Only 8 warps per SM run here (the sweeps need the registers), so
// every warp keeps the NEXT chunk's CSR entries in flight -- of this group or
// of its next group, whose row pointers were fetched a group earlier -- while
// it gathers x, stages the products and folds the current chunk (in-solver
// SpMV on config 5: 0.96 ms with 4 chunks of 32 in flight per warp, 0.73 ms
// with 12, then this software pipeline).  Barriers: x complete before, y
// complete after.
__device__ __noinline__ void g_spmv_body(Q& q, int n, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ ci, const double2* __restrict__ v,
                            const double2* x, double2* y) {
  q.g.sync();
  const int lane = threadIdx.x & 31;
  double2* s_p = q.stage;
  const int ngroups = (n + 31) >> 5;
  int grp = q.gw;
  if (grp < ngroups) {
    // header of a group: entry range of its 32 rows and of this lane's row
    auto header = [&](int g, int32_t& b, int32_t& e, int32_t& a0, int32_t& a1) {
      const int r0 = g << 5, r1 = min(r0 + 32, n), row = r0 + lane;
      b = __ldg(rp + r0);
      e = __ldg(rp + r1);
      a0 = row < r1 ? __ldg(rp + row) : 0;
      a1 = row < r1 ? __ldg(rp + row + 1) : 0;
    };
    int32_t base, end, p0, p1, nb = 0, ne = 0, np0 = 0, np1 = 0;
    header(grp, base, end, p0, p1);
    if (grp + q.ngw < ngroups) header(grp + q.ngw, nb, ne, np0, np1);
    int c[SP_UNROLL], nc[SP_UNROLL];
    double2 a[SP_UNROLL], na[SP_UNROLL];
    int32_t cb = base;
#pragma unroll
    for (int u = 0; u < SP_UNROLL; ++u) {
      const int32_t e = cb + 32 * u + lane;
      if (e < min(cb + SP_CH, end)) {
        c[u] = __ldg(ci + e);
        a[u] = ldg2(v + e);
      }
    }
    double2 acc = make_double2(0.0, 0.0);
    while (true) {
      const int32_t ce = min(cb + SP_CH, end);
      // the chunk after this one: same group, or the first of the next group
      const bool same = cb + SP_CH < end;
      const bool more = same || grp + q.ngw < ngroups;
      const int32_t ncb = same ? cb + SP_CH : nb;
      const int32_t nce = min(ncb + SP_CH, same ? end : ne);
      if (more) {
#pragma unroll
        for (int u = 0; u < SP_UNROLL; ++u) {
          const int32_t e = ncb + 32 * u + lane;
          if (e < nce) {
            nc[u] = __ldg(ci + e);
            na[u] = ldg2(v + e);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < SP_UNROLL; ++u) {
        const int32_t e = cb + 32 * u + lane;
        if (e < ce) {
          const int k = e - cb;
          s_p[k + (k >> 3)] = cmul_plain(a[u], __ldcg(x + c[u]));
        }
      }
      __syncwarp();
      const int32_t qa = max(p0, cb), qb = min(p1, ce);
      for (int32_t t = qa; t < qb; ++t) {
        const int k = t - cb;
        const double2 pq = s_p[k + (k >> 3)];
        acc = (t == p0) ? pq : cadd(acc, pq);
      }
      __syncwarp();
      if (!same) {  // last chunk of the group: its rows are complete
        const int row = (grp << 5) + lane;
        if (row < n) y[row] = acc;
        if (!more) break;
        grp += q.ngw;
        base = nb;
        end = ne;
        p0 = np0;
        p1 = np1;
        acc = make_double2(0.0, 0.0);
        if (grp + q.ngw < ngroups) header(grp + q.ngw, nb, ne, np0, np1);
      }
      cb = ncb;
#pragma unroll
      for (int u = 0; u < SP_UNROLL; ++u) {
        c[u] = nc[u];
        a[u] = na[u];
      }
    }
  }
  q.g.sync();
}

// (reached by an indirect call, like the sweeps: its own register allocation)
typedef void (*spmv_fn_t)(Q&, int, const int32_t*, const int32_t*, const double2*, const double2*,
                          double2*);
__device__ spmv_fn_t g_spmv_ptr = g_spmv_body;
__device__ __forceinline__ void g_spmv(Q& q, int n, const int32_t* rp, const int32_t* ci,
                                       const double2* v, const double2* x, double2* y) {
  spmv_fn_t fn = *(volatile spmv_fn_t*)&g_spmv_ptr;
  fn(q, n, rp, ci, v, x, y);
}

struct Ctx {
  int n;
  const GridArgs* a;
  double2 *P, *Y, *X;  // apply scratch: permuted rhs, L output, U output
  double2* small;      // shared: GMRES H / g / sn / y
  double* cs;          // shared
};

// out = M^{-1} in (factor.solve_lu, factor.py:137-149); out may alias in.
// Element loops use the grid's fixed element map, so a vector produced by an
// element loop can be consumed by the next without a barrier.
__device__ __noinline__ void psolve(Q& q, const Ctx& C, const double2* in, double2* out) {
  const GridArgs& a = *C.a;
  const int n = C.n;
  if (!a.have_M) {
    if (in != out)
      for (int i = q.tid; i < n; i += q.nth) out[i] = in[i];
    return;
  }
  const double2 S = cta::sentinel2();
  for (int i = q.tid; i < n; i += q.nth) {
    C.P[a.nb == n ? a.pinv[i] : (i / a.nb) * a.nb + a.pinv[i]] = in[i];
    C.Y[i] = S;
    C.X[i] = S;
  }
  q.g.sync();
  tri::sweep_grid<false>(a.L, C.P, C.Y, nullptr);
  q.g.sync();
  tri::sweep_grid<true>(a.U, C.Y, C.X, a.rd);
  q.g.sync();
  if (a.colp) {  // x[q] = y (factor.py:147-148)
    for (int i = q.tid; i < n; i += q.nth) out[i] = __ldcg(C.X + a.colp[i]);
  } else {
    for (int i = q.tid; i < n; i += q.nth) out[i] = __ldcg(C.X + i);
  }
}

// out = M^{-1} (A v)
__device__ void apply_op(Q& q, const Ctx& C, const double2* v, double2* tmp, double2* out) {
  const GridArgs& a = *C.a;
  g_spmv(q, C.n, a.Arp, a.Aci, a.Av, v, tmp);
  psolve(q, C, tmp, out);
}

// || b - A x ||_2
__device__ double resid_nrm2(Q& q, const Ctx& C, const double2* x, const double2* b,
                             double2* tmp) {
  const GridArgs& a = *C.a;
  g_spmv(q, C.n, a.Arp, a.Aci, a.Av, x, tmp);
  double o[1];
  gsum<1>(q, C.n, [&](int i, double (&s)[1]) {
    const double2 d = csub(b[i], tmp[i]);
    s[0] = __fma_rn(d.x, d.x, __fma_rn(d.y, d.y, s[0]));
  }, o);
  return sqrt(o[0]);
}

struct IterOut {
  int iterations;
  double final_residual;
  bool converged, breakdown;
};

struct Vecs {
  double2 *x, *r, *rhat, *p, *v, *s, *t, *pb, *tmp, *V;
};

#define EACH(i) for (int i = q.tid; i < n; i += q.nth)

// krylov.bicgstab, krylov.py:181-291
__device__ __noinline__ IterOut bicgstab(Q& q, const Ctx& C, const double2* b, const Vecs& W, double tol,
                            int max_iter) {
  const int n = C.n;
  IterOut out{0, 0.0, false, false};
  const double2 Z = make_double2(0.0, 0.0);
  const double bnorm = gnrm2(q, n, b);
  if (bnorm == 0.0) {
    EACH(i) W.x[i] = Z;
    out.converged = true;
    return out;
  }
  psolve(q, C, b, W.pb);
  const double pbnorm = gnrm2(q, n, W.pb);
  if (pbnorm == 0.0 || !isfinite(pbnorm)) {
    EACH(i) W.x[i] = Z;
    out.final_residual = bnorm;
    out.breakdown = true;
    return out;
  }
  EACH(i) {
    W.x[i] = Z;
    W.r[i] = W.pb[i];
    W.rhat[i] = W.pb[i];
    W.v[i] = Z;
    W.p[i] = Z;
  }
  double rhat_norm = gnrm2(q, n, W.rhat);
  double2 rho_prev = make_double2(1.0, 0.0), alpha = rho_prev, omega = rho_prev;
  double target = tol * pbnorm;
  double prev_true = INFINITY;
  int it = 0;
  while (it < max_iter) {
    // ||r||^2 and rhat^H r in one pass
    double o3[3];
    gsum<3>(q, n, [&](int i, double (&s)[3]) {
      const double2 r = W.r[i], h = W.rhat[i];
      s[0] = __fma_rn(r.x, r.x, __fma_rn(r.y, r.y, s[0]));
      s[1] = __fma_rn(h.x, r.x, __fma_rn(h.y, r.y, s[1]));
      s[2] = __fma_rn(h.x, r.y, __fma_rn(-h.y, r.x, s[2]));
    }, o3);
    const double rnorm = sqrt(o3[0]);
    if (rnorm <= target) {
      const double true_res = resid_nrm2(q, C, W.x, b, W.tmp);
      if (true_res <= tol * bnorm) {
        out.converged = true;
        break;
      }
      if (true_res >= 0.5 * prev_true) break;
      prev_true = true_res;
      target *= 0.1;
    }
    const double2 rho = make_double2(o3[1], o3[2]);
    const double arho = cabs(rho);
    if (arho < 1e-30 || arho < 1e-16 * rhat_norm * rnorm) {
      out.breakdown = true;
      break;
    }
    if (it == 0) {
      EACH(i) W.p[i] = W.r[i];
    } else {
      const double2 beta = cmul(cdiv(rho, rho_prev), cdiv(alpha, omega));
      EACH(i) {
        const double2 d = csub(W.p[i], cmul(omega, W.v[i]));
        W.p[i] = cadd(W.r[i], cmul(beta, d));
      }
    }
    apply_op(q, C, W.p, W.tmp, W.v);
    const double2 denom = gvdot(q, n, W.rhat, W.v);
    if (denom.x == 0.0 && denom.y == 0.0) {
      out.breakdown = true;
      break;
    }
    alpha = cdiv(rho, denom);
    // s = r - alpha v and ||s||^2 in one pass
    double o1[1];
    gsum<1>(q, n, [&](int i, double (&s)[1]) {
      const double2 sv = csub(W.r[i], cmul(alpha, W.v[i]));
      W.s[i] = sv;
      s[0] = __fma_rn(sv.x, sv.x, __fma_rn(sv.y, sv.y, s[0]));
    }, o1);
    ++it;
    const double snorm = sqrt(o1[0]);
    if (snorm <= target) {
      EACH(i) W.x[i] = cadd(W.x[i], cmul(alpha, W.p[i]));
      const double true_res = resid_nrm2(q, C, W.x, b, W.tmp);
      if (true_res <= tol * bnorm) {
        out.converged = true;
        break;
      }
      if (true_res >= 0.5 * prev_true) break;
      prev_true = true_res;
      target *= 0.1;
      EACH(i) {
        W.r[i] = W.s[i];
        W.rhat[i] = W.s[i];
        W.v[i] = Z;
        W.p[i] = Z;
      }
      rhat_norm = gnrm2(q, n, W.rhat);
      rho_prev = alpha = omega = make_double2(1.0, 0.0);
      continue;
    }
    apply_op(q, C, W.s, W.tmp, W.t);
    double o4[3];
    gsum<3>(q, n, [&](int i, double (&s)[3]) {
      const double2 t = W.t[i], sv = W.s[i];
      s[0] = __fma_rn(t.x, t.x, __fma_rn(t.y, t.y, s[0]));
      s[1] = __fma_rn(t.x, sv.x, __fma_rn(t.y, sv.y, s[1]));
      s[2] = __fma_rn(t.x, sv.y, __fma_rn(-t.y, sv.x, s[2]));
    }, o4);
    // t^H t is real: the reference's np.vdot(t, t) has a zero imaginary part
    if (o4[0] == 0.0) {
      out.breakdown = true;
      break;
    }
    omega = cdiv(make_double2(o4[1], o4[2]), make_double2(o4[0], 0.0));
    EACH(i) {
      const double2 xa = cadd(W.x[i], cmul(alpha, W.p[i]));
      W.x[i] = cadd(xa, cmul(omega, W.s[i]));
      W.r[i] = csub(W.s[i], cmul(omega, W.t[i]));
    }
    rho_prev = rho;
    if (omega.x == 0.0 && omega.y == 0.0) {
      out.breakdown = true;
      break;
    }
  }
  out.iterations = it;
  out.final_residual = resid_nrm2(q, C, W.x, b, W.tmp);
  return out;
}

// krylov.gmres, krylov.py:67-178.  H is (m+1) x m row-major in shared memory
// (every CTA keeps its own, identical copy), then g (m+1), sn (m), y (m).
__device__ __noinline__ IterOut gmres(Q& q, const Ctx& C, const double2* b, const Vecs& W, double tol,
                         int max_iter, int m) {
  const int n = C.n;
  IterOut out{0, 0.0, false, false};
  const double2 Z = make_double2(0.0, 0.0);
  double2* H = C.small;
  double2* g = H + (m + 1) * m;
  double2* sn = g + (m + 1);
  double2* yv = sn + m;
  double* cs = C.cs;
  __shared__ double s_res;
  __shared__ int s_flag;
  const double bnorm = gnrm2(q, n, b);
  if (bnorm == 0.0) {
    EACH(i) W.x[i] = Z;
    out.converged = true;
    return out;
  }
  psolve(q, C, b, W.pb);
  const double pbnorm = gnrm2(q, n, W.pb);
  if (pbnorm == 0.0 || !isfinite(pbnorm)) {
    EACH(i) W.x[i] = Z;
    out.final_residual = bnorm;
    out.breakdown = true;
    return out;
  }
  EACH(i) W.x[i] = Z;
  double target = tol * pbnorm;
  int total = 0;
  bool converged = false, breakdown = false, invariant = false;
  double prev_true = INFINITY;
  while (total < max_iter && !converged && !invariant) {
    double2* r = W.r;
    if (total) {
      apply_op(q, C, W.x, W.tmp, r);
      EACH(i) r[i] = csub(W.pb[i], r[i]);
    } else {
      EACH(i) r[i] = W.pb[i];
    }
    const double beta = gnrm2(q, n, r);
    bool monitor_hit = beta <= target;
    double res = beta;
    if (!monitor_hit) {
      EACH(i) W.V[i] = make_double2(r[i].x / beta, r[i].y / beta);
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int i = 0; i < (m + 1) * m; ++i) H[i] = Z;
        for (int i = 0; i <= m; ++i) g[i] = Z;
        g[0] = make_double2(beta, 0.0);
      }
      __syncthreads();
      int j = 0;
      while (j < m && total < max_iter) {
        double2* Vj = W.V + (size_t)j * n;
        double2* w = W.r;  // reuse r as the Arnoldi vector
        apply_op(q, C, Vj, W.tmp, w);
        ++total;
        for (int i = 0; i <= j; ++i) {  // modified Gram-Schmidt
          const double2* Vi = W.V + (size_t)i * n;
          const double2 hij = gvdot(q, n, Vi, w);
          EACH(e) w[e] = csub(w[e], cmul(hij, Vi[e]));
          if (threadIdx.x == 0) H[i * m + j] = hij;
        }
        const double hnext = gnrm2(q, n, w);
        if (hnext > 0.0) {
          double2* Vn = W.V + (size_t)(j + 1) * n;
          EACH(e) Vn[e] = make_double2(w[e].x / hnext, w[e].y / hnext);
        }
        __syncthreads();
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
            sn[j] = Z;
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
        if (hnext == 0.0) {
          invariant = true;
          break;
        }
        if (res <= target) break;
      }
      // zero diagonal -> breakdown; else back-substitute and update x
      __syncthreads();
      if (threadIdx.x == 0) {
        int bad = 0;
        for (int i = 0; i < j; ++i) {
          const double2 d = H[i * m + i];
          if (d.x == 0.0 && d.y == 0.0) bad = 1;
        }
        if (!bad) {
          for (int i = j - 1; i >= 0; --i) {
            double2 acc = Z;
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
      EACH(e) {
        double2 acc = Z;
        for (int k = 0; k < j; ++k) acc = cadd(acc, cmul(yv[k], W.V[(size_t)k * n + e]));
        W.x[e] = cadd(W.x[e], acc);
      }
      monitor_hit = res <= target || invariant;
    }
    if (monitor_hit) {
      const double true_res = resid_nrm2(q, C, W.x, b, W.tmp);
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
  out.final_residual = resid_nrm2(q, C, W.x, b, W.tmp);
  return out;
}

}  // namespace

size_t grid_small_bytes(int m) {
  return sizeof(double2) * ((size_t)(m + 1) * m + (m + 1) + 2 * (size_t)m) + sizeof(double) * m;
}

int64_t grid_work_len(int32_t n, int restart_m) {
  // P, Y, X, 9 Krylov vectors, (m+1) Arnoldi vectors, outer iterate, inner result
  return (int64_t)n * (3 + 9 + (restart_m + 1) + 2);
}

__global__ void __launch_bounds__(GT, 1) grid_solver_kernel(GridArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double red[32 * 8];
  Q q{cg::this_grid()};
  q.tid = blockIdx.x * blockDim.x + threadIdx.x;
  q.nth = gridDim.x * blockDim.x;
  q.gw = q.tid >> 5;
  q.ngw = q.nth >> 5;
  q.red = red;
  q.part = a.part;
  q.flip = 0;
  q.stage = reinterpret_cast<double2*>(smem) + (size_t)(threadIdx.x >> 5) * SP_SLOTS;
  const int n = a.n;
  const int m = a.restart_m;
  Ctx C;
  C.n = n;
  C.a = &a;
  C.small = reinterpret_cast<double2*>(smem) + (size_t)(GT / 32) * SP_SLOTS;
  C.cs = reinterpret_cast<double*>(C.small + (m + 1) * m + (m + 1) + 2 * m);
  double2* ws = a.work;
  C.P = ws;
  C.Y = ws + (int64_t)n;
  C.X = ws + 2 * (int64_t)n;
  double2* vb = ws + 3 * (int64_t)n;
  Vecs W;
  W.x = vb;
  W.r = vb + 1 * (int64_t)n;
  W.rhat = vb + 2 * (int64_t)n;
  W.p = vb + 3 * (int64_t)n;
  W.v = vb + 4 * (int64_t)n;
  W.s = vb + 5 * (int64_t)n;
  W.t = vb + 6 * (int64_t)n;
  W.pb = vb + 7 * (int64_t)n;
  W.tmp = vb + 8 * (int64_t)n;
  W.V = vb + 9 * (int64_t)n;
  double2* xo = vb + (9 + (int64_t)m + 1) * n;
  double2* yo = vb + (10 + (int64_t)m + 1) * n;
  const double2* in = a.rhs;
  double2* out = a.xout;
  SolveStats* st = a.stats;
  const bool lead = q.tid == 0;
  if (lead) *st = SolveStats{};

  if (a.want_condest && a.have_M) {  // factor.condest, factor.py:152-157
    EACH(i) W.tmp[i] = make_double2(1.0, 0.0);
    psolve(q, C, W.tmp, W.pb);
    const double mx = gmax(q, n, [&](int i) { return cabs(W.pb[i]); });
    if (lead) st->condest = mx;
  }

  const int mode = a.mode;
  if (mode == MODE_LIN_DIRECT || mode == MODE_LIN_BICGSTAB || mode == MODE_LIN_GMRES) {
    IterOut io{0, 0.0, true, false};
    if (mode == MODE_LIN_DIRECT) psolve(q, C, in, W.x);
    else if (mode == MODE_LIN_BICGSTAB) io = bicgstab(q, C, in, W, a.tol, a.max_iter);
    else io = gmres(q, C, in, W, a.tol, a.max_iter, m);
    EACH(i) out[i] = W.x[i];
    if (lead) {
      st->inner_last = io.iterations;
      st->inner_total = io.iterations;
      st->converged = io.converged;
      st->breakdown = io.breakdown;
      st->final_residual = io.final_residual;
    }
    return;
  }

  // ---- inverse power, steady.py:211-245 -------------------------------------
  {
    const double nx = gnrm2(q, n, in);
    EACH(i) xo[i] = make_double2(in[i].x / nx, in[i].y / nx);
  }
  const double tol = a.tol;
  int outer = 0, inner_total = 0, inner_last = 0;
  bool converged = false;
  int status = 0;
  while (outer < a.max_outer) {
    double2* y = yo;
    if (mode == MODE_INV_DIRECT) {
      psolve(q, C, xo, y);
    } else {
      IterOut io = (mode == MODE_INV_BICGSTAB) ? bicgstab(q, C, xo, W, tol / 10.0, a.max_iter)
                                               : gmres(q, C, xo, W, tol / 10.0, a.max_iter, m);
      inner_last = io.iterations;
      inner_total += io.iterations;
      const double bad = gmax(q, n, [&](int i) { return finite2(W.x[i]) ? 0.0 : 1.0; });
      if (io.breakdown || bad != 0.0) {
        status = io.breakdown ? SOLVE_INNER_BREAKDOWN : SOLVE_INNER_NONFINITE;
        break;
      }
      if (gnrm2(q, n, W.x) == 0.0) {
        status = SOLVE_INNER_NO_PROGRESS;
        break;
      }
      EACH(i) y[i] = W.x[i];
    }
    const double ny = gnrm2(q, n, y);
    if (ny == 0.0 || !isfinite(ny)) {
      status = SOLVE_UNUSABLE_VECTOR;
      break;
    }
    EACH(i) y[i] = make_double2(y[i].x / ny, y[i].y / ny);
    ++outer;
    const double2 ov = gvdot(q, n, y, xo);
    double2 ph = make_double2(1.0, 0.0);
    const bool ovnz = !(ov.x == 0.0 && ov.y == 0.0);
    if (ovnz) {
      const double aov = cabs(ov);
      ph = make_double2(ov.x / aov, ov.y / aov);
    }
    double o1[1];
    gsum<1>(q, n, [&](int i, double (&s)[1]) {
      const double2 al = ovnz ? cmul(y[i], ph) : y[i];
      const double2 d = csub(al, xo[i]);
      s[0] = __fma_rn(d.x, d.x, __fma_rn(d.y, d.y, s[0]));
    }, o1);
    const double diff = sqrt(o1[0]);
    // resid_inf = max |L_plain,perm y|
    g_spmv(q, n, a.Prp, a.Pci, a.Pv, y, W.tmp);
    const double resid_inf = gmax(q, n, [&](int i) { return cabs(W.tmp[i]); });
    EACH(i) xo[i] = y[i];
    if (diff <= tol || resid_inf <= tol) {
      converged = true;
      break;
    }
  }
  if (status == 0 && !converged) status = SOLVE_POWER_NOT_CONVERGED;
  EACH(i) out[i] = xo[i];
  if (lead) {
    st->status = status;
    st->outer = outer;
    st->inner_last = inner_last;
    st->inner_total = inner_total;
    st->converged = converged;
  }
}

// Standalone x = M^{-1} b over the level-ordered factors (factor.solve_lu).
__global__ void __launch_bounds__(GT, 1) grid_apply_kernel(GridArgs a) {
  __shared__ double red[32 * 8];
  Q q{cg::this_grid()};
  q.tid = blockIdx.x * blockDim.x + threadIdx.x;
  q.nth = gridDim.x * blockDim.x;
  q.gw = q.tid >> 5;
  q.ngw = q.nth >> 5;
  q.red = red;
  q.part = a.part;
  q.flip = 0;
  q.stage = nullptr;
  Ctx C;
  C.n = a.n;
  C.a = &a;
  C.P = a.work;
  C.Y = a.work + (int64_t)a.n;
  C.X = a.work + 2 * (int64_t)a.n;
  C.small = nullptr;
  C.cs = nullptr;
  psolve(q, C, a.rhs, a.xout);
}

#undef EACH

static int coop_grid(const void* kern, size_t smem, int* blocks_out) {
  int dev = 0, sms = 0, per_sm = 0, coop = 0;
  RS_CUDA_TRY(cudaGetDevice(&dev));
  RS_CUDA_TRY(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev));
  if (!coop) {
    set_error("device does not support cooperative launches");
    return RS_ERR_UNSUPPORTED;
  }
  RS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, GT, smem));
  if (per_sm < 1) {
    set_error("grid solver: kernel does not fit an SM (%zu B shared)", smem);
    return RS_ERR_UNSUPPORTED;
  }
  *blocks_out = sms;  // one CTA per SM: the persistent-kernel shape
  return RS_OK;
}

int launch_grid_solver(const GridArgs& a, cudaStream_t st) {
  if (a.n == 0) return RS_OK;
  const size_t smem = sizeof(double2) * (size_t)(GT / 32) * SP_SLOTS + grid_small_bytes(a.restart_m);
  int blocks = 0;
  RS_TRY(coop_grid((const void*)grid_solver_kernel, smem, &blocks));
  GridArgs la = a;
  void* params[] = {&la};
  RS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)grid_solver_kernel, dim3(blocks), dim3(GT),
                                          params, smem, st));
  count_launch();
  return RS_OK;
}

int launch_grid_apply(const GridArgs& a, cudaStream_t st) {
  if (a.n == 0) return RS_OK;
  int blocks = 0;
  RS_TRY(coop_grid((const void*)grid_apply_kernel, 0, &blocks));
  GridArgs la = a;
  void* params[] = {&la};
  RS_CUDA_TRY(cudaLaunchCooperativeKernel((const void*)grid_apply_kernel, dim3(blocks), dim3(GT),
                                          params, 0, st));
  count_launch();
  return RS_OK;
}

}  // namespace rs

extern "C" int rs_debug_slice_clock_mode(int on) {
  RS_CUDA_TRY(cudaMemcpyToSymbol(rs::tri::g_slice_clock_mode, &on, sizeof(on)));
  return 0;
}

extern "C" int rs_debug_slice_times(void* buf) {
  unsigned long long* p = reinterpret_cast<unsigned long long*>(buf);
  RS_CUDA_TRY(cudaMemcpyToSymbol(rs::tri::g_slice_times, &p, sizeof(p)));
  return 0;
}

namespace rs {

int grid_blocks() {
  int dev = 0, sms = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
  return sms;
}

}  // namespace rs
