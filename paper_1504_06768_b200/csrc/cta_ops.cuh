// CTA-scope building blocks for the device-resident solver: one CTA owns one
// system and runs SpMV, the preconditioner apply (two sparse triangular
// solves), deterministic reductions and BLAS-1 updates without leaving the
// SM, so an entire Krylov solve is one kernel with no host round trips.
//
// Bit-exactness contracts (vs the reference Cython kernels):
//   spmv        == csr_matvec   _ckernels.pyx:34-50
//   lower_solve == lower_solve  _ckernels.pyx:53-67   (row-oriented form)
//   upper_solve == upper_solve  _ckernels.pyx:70-85   (row-oriented form)
// The reference triangular solves scatter column by column; row i of the
// result receives its subtractions in ascending column order (L) or
// descending column order (U).  The row-oriented solves below perform the
// same subtractions in the same order, so results are identical.
//
// Reductions are deterministic (fixed thread->element map, fixed shuffle
// tree, fixed cross-warp order) but use a different summation order than
// numpy/BLAS, so Krylov iterates agree with the reference to rounding only.
#pragma once
#include "common.cuh"

namespace rs {
namespace cta {

constexpr unsigned FULL = 0xffffffffu;

// Sum K doubles over the CTA; every thread receives the totals.
// red must hold 32*K doubles of shared memory.
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < K; ++k)
    for (int o = 16; o; o >>= 1) v[k] = __dadd_rn(v[k], __shfl_xor_sync(FULL, v[k], o));
  __syncthreads();  // protect red from a previous use
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < K; ++k) red[k * 32 + wid] = v[k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = red[k * 32];
    for (int w = 1; w < nw; ++w) s = __dadd_rn(s, red[k * 32 + w]);
    v[k] = s;
  }
}

__device__ __forceinline__ double block_max(double v, double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  double s = red[0];
  for (int w = 1; w < nw; ++w) s = fmax(s, red[w]);
  return s;
}

// vdot(a, b) = sum conj(a_i) b_i  (numpy.vdot convention)
__device__ __forceinline__ double2 vdot(int n, const double2* a, const double2* b,
                                        double* red) {
  double acc[2] = {0.0, 0.0};
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 x = a[i], y = b[i];
    acc[0] = __fma_rn(x.x, y.x, __fma_rn(x.y, y.y, acc[0]));
    acc[1] = __fma_rn(x.x, y.y, __fma_rn(-x.y, y.x, acc[1]));
  }
  block_sum<2>(acc, red);
  return make_double2(acc[0], acc[1]);
}

__device__ __forceinline__ double nrm2(int n, const double2* a, double* red) {
  double acc[1] = {0.0};
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const double2 x = a[i];
    acc[0] = __fma_rn(x.x, x.x, __fma_rn(x.y, x.y, acc[0]));
  }
  block_sum<1>(acc, red);
  return sqrt(acc[0]);
}

// ||b - A x||_2 without materialising the residual.
__device__ __forceinline__ double resid_nrm2(int n, const int32_t* rp, const int32_t* ci,
                                             const double2* v, const double2* x,
                                             const double2* b, double* red) {
  double acc[1] = {0.0};
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int p0 = rp[i], p1 = rp[i + 1];
    double2 s = make_double2(0.0, 0.0);
    if (p0 < p1) {
      s = cmul_plain(v[p0], x[ci[p0]]);
      for (int p = p0 + 1; p < p1; ++p) s = cadd(s, cmul_plain(v[p], x[ci[p]]));
    }
    const double2 r = csub(b[i], s);
    acc[0] = __fma_rn(r.x, r.x, __fma_rn(r.y, r.y, acc[0]));
  }
  block_sum<1>(acc, red);
  return sqrt(acc[0]);
}

// y = A x, row-sequential (bit-exact with csr_matvec).  rp/ci local.
__device__ __forceinline__ void spmv(int n, const int32_t* __restrict__ rp,
                                     const int32_t* __restrict__ ci,
                                     const double2* __restrict__ v,
                                     const double2* x, double2* y) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int p0 = rp[i], p1 = rp[i + 1];
    double2 s = make_double2(0.0, 0.0);
    if (p0 < p1) {
      s = cmul_plain(v[p0], x[ci[p0]]);
      for (int p = p0 + 1; p < p1; ++p) s = cadd(s, cmul_plain(v[p], x[ci[p]]));
    }
    y[i] = s;
  }
}

__device__ __forceinline__ double2 vld(const double2* p) {
  const volatile double* q = reinterpret_cast<const volatile double*>(p);
  return make_double2(q[0], q[1]);
}

// In-place unit-lower solve on y (strictly-lower CSR, ascending columns).
// Warp-per-row, rows dealt round-robin to warps in increasing order, so the
// oldest unfinished row always has its dependencies done (deadlock-free).
// Each chunk of 32 entries waits only for the lanes whose source rows are
// not ready yet; the ordered subtraction chain advances over the ready
// prefix, so early terms are folded in while late ones are still pending.
__device__ __noinline__ static void lower_solve(int n, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ ci,
                            const double2* __restrict__ v, double2* y,
                            volatile uint8_t* ready) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  for (int i = wid; i < n; i += nw) {
    const int p0 = rp[i], p1 = rp[i + 1];
    double2 acc = vld(y + i);
    for (int base = p0; base < p1; base += 32) {
      const int p = base + lane;
      const bool act = p < p1;
      int c = 0;
      double2 lv = make_double2(0.0, 0.0);
      if (act) {
        c = __ldg(ci + p);
        lv = __ldg(v + p);
      }
      const int cnt = min(32, p1 - base);
      bool have = !act;
      double2 prod = make_double2(0.0, 0.0);
      int done = 0;
      while (done < cnt) {
        if (!have && ready[c]) {
          __threadfence_block();
          prod = cmul_plain(lv, vld(y + c));
          have = true;
        }
        const unsigned m = __ballot_sync(FULL, have);
        const unsigned pend = ~m;
        int upto = pend ? (__ffs(pend) - 1) : 32;
        if (upto > cnt) upto = cnt;
        for (int e = done; e < upto; ++e) {
          const double px = __shfl_sync(FULL, prod.x, e);
          const double py = __shfl_sync(FULL, prod.y, e);
          acc = csub(acc, make_double2(px, py));
        }
        done = upto;
      }
    }
    if (lane == 0) {
      volatile double* yy = reinterpret_cast<volatile double*>(y + i);
      yy[0] = acc.x;
      yy[1] = acc.y;
      __threadfence_block();
      ready[i] = 1;
    }
    __syncwarp();
  }
}

// In-place upper solve on y: strictly-upper CSR (ascending columns) plus the
// reciprocal pivots rU = recipc(U_ii).  Rows in decreasing order; row i
// subtracts its terms in DEScending column order, then multiplies by rU[i]
// (reference: xc = y[c] * recipc(Ux[p1]), then scatter).
__device__ __noinline__ static void upper_solve(int n, const int32_t* __restrict__ rp,
                            const int32_t* __restrict__ ci,
                            const double2* __restrict__ v,
                            const double2* __restrict__ rU, double2* y,
                            volatile uint8_t* ready) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  for (int r = wid; r < n; r += nw) {
    const int i = n - 1 - r;
    const int p0 = rp[i], p1 = rp[i + 1];
    double2 acc = vld(y + i);
    for (int top = p1; top > p0; top -= 32) {
      const int p = top - 1 - lane;
      const bool act = p >= p0;
      int c = 0;
      double2 uv = make_double2(0.0, 0.0);
      if (act) {
        c = __ldg(ci + p);
        uv = __ldg(v + p);
      }
      const int cnt = min(32, top - p0);
      bool have = !act;
      double2 prod = make_double2(0.0, 0.0);
      int done = 0;
      while (done < cnt) {
        if (!have && ready[c]) {
          __threadfence_block();
          prod = cmul_plain(uv, vld(y + c));
          have = true;
        }
        const unsigned m = __ballot_sync(FULL, have);
        const unsigned pend = ~m;
        int upto = pend ? (__ffs(pend) - 1) : 32;
        if (upto > cnt) upto = cnt;
        for (int e = done; e < upto; ++e) {
          const double px = __shfl_sync(FULL, prod.x, e);
          const double py = __shfl_sync(FULL, prod.y, e);
          acc = csub(acc, make_double2(px, py));
        }
        done = upto;
      }
    }
    if (lane == 0) {
      const double2 xi = cmul_plain(acc, __ldg(rU + i));
      volatile double* yy = reinterpret_cast<volatile double*>(y + i);
      yy[0] = xi.x;
      yy[1] = xi.y;
      __threadfence_block();
      ready[i] = 1;
    }
    __syncwarp();
  }
}

}  // namespace cta
}  // namespace rs
