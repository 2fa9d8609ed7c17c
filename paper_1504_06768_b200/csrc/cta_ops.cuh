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

// Deterministic CTA sums whose rounding does not depend on the CTA size:
// elements are accumulated in the order of a 512-thread CTA (virtual thread
// v takes i = v, v+512, ...; shuffle tree per virtual warp; virtual warps
// summed 0..15 in order), each physical thread of a 128/256/512-thread CTA
// playing 4/2/1 virtual threads.  A lone-system solve (256 threads) and a
// batch (128 threads) therefore run the same arithmetic as a 512-thread CTA.
constexpr int RED_T = 512;

template <int K, int V, class F>
__device__ __forceinline__ void vsum_impl(int n, F f, double (&out)[K], double* red) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  double acc[V][K];
#pragma unroll
  for (int j = 0; j < V; ++j) {
#pragma unroll
    for (int k = 0; k < K; ++k) acc[j][k] = 0.0;
    for (int i = threadIdx.x + j * blockDim.x; i < n; i += RED_T) f(i, acc[j]);
#pragma unroll
    for (int k = 0; k < K; ++k)
      for (int o = 16; o; o >>= 1) acc[j][k] = __dadd_rn(acc[j][k], __shfl_xor_sync(FULL, acc[j][k], o));
  }
  __syncthreads();  // protect red from a previous use
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < V; ++j)
#pragma unroll
      for (int k = 0; k < K; ++k) red[k * 32 + wid + j * nw] = acc[j][k];
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < K; ++k) {
    double s = red[k * 32];
    for (int w = 1; w < RED_T / 32; ++w) s = __dadd_rn(s, red[k * 32 + w]);
    out[k] = s;
  }
}

template <int K, class F>
__device__ __forceinline__ void vsum(int n, F f, double (&out)[K], double* red) {
  if (blockDim.x >= RED_T) vsum_impl<K, 1>(n, f, out, red);
  else if (blockDim.x * 2 >= RED_T) vsum_impl<K, 2>(n, f, out, red);
  else vsum_impl<K, 4>(n, f, out, red);
}

// vdot(a, b) = sum conj(a_i) b_i  (numpy.vdot convention)
__device__ __forceinline__ double2 vdot(int n, const double2* a, const double2* b,
                                        double* red) {
  double out[2];
  vsum<2>(
      n,
      [&](int i, double (&acc)[2]) {
        const double2 x = a[i], y = b[i];
        acc[0] = __fma_rn(x.x, y.x, __fma_rn(x.y, y.y, acc[0]));
        acc[1] = __fma_rn(x.x, y.y, __fma_rn(-x.y, y.x, acc[1]));
      },
      out, red);
  return make_double2(out[0], out[1]);
}

__device__ __forceinline__ double nrm2(int n, const double2* a, double* red) {
  double out[1];
  vsum<1>(
      n,
      [&](int i, double (&acc)[1]) {
        const double2 x = a[i];
        acc[0] = __fma_rn(x.x, x.x, __fma_rn(x.y, x.y, acc[0]));
      },
      out, red);
  return sqrt(out[0]);
}

// ||b - A x||_2 without materialising the residual.
__device__ __forceinline__ double resid_nrm2(int n, const int32_t* rp, const int32_t* ci,
                                             const double2* v, const double2* x,
                                             const double2* b, double* red) {
  double out[1];
  vsum<1>(
      n,
      [&](int i, double (&acc)[1]) {
        const int p0 = rp[i], p1 = rp[i + 1];
        double2 s = make_double2(0.0, 0.0);
        if (p0 < p1) {
          s = cmul_plain(v[p0], x[ci[p0]]);
          for (int p = p0 + 1; p < p1; ++p) s = cadd(s, cmul_plain(v[p], x[ci[p]]));
        }
        const double2 r = csub(b[i], s);
        acc[0] = __fma_rn(r.x, r.x, __fma_rn(r.y, r.y, acc[0]));
      },
      out, red);
  return sqrt(out[0]);
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

// Readiness travels with the value: solve outputs start as a sentinel NaN
// (a payload no arithmetic produces from finite inputs) and a row publishes
// its result with one 16-byte store, so a single volatile 16-byte load both
// detects that a source row is final and delivers it.  A torn read shows a
// sentinel half and is simply polled again.
constexpr unsigned long long SENTINEL = 0x7ff4dead5eedbeefull;

// Poll backoff of the triangular sweeps (ns): first / maximum nap after a
// poll that made no progress.  Tunable through rs_debug_tri_backoff.
__device__ unsigned g_tri_nap_min = 0;
__device__ unsigned g_tri_nap_max = 0;
// tuning hook: per-row (start, publish) clocks of a sweep, [2*n]
__device__ long long* g_tri_times = nullptr;

__device__ __forceinline__ double sentinel_d() { return __longlong_as_double(SENTINEL); }
__device__ __forceinline__ double2 sentinel2() {
  return make_double2(sentinel_d(), sentinel_d());
}

__device__ __forceinline__ double2 vld2(const double2* p) {
  double2 v;
  if (__isShared(p)) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  } else {
    asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
  }
  return v;
}
__device__ __forceinline__ void vst2(double2* p, double2 v) {
  if (__isShared(p)) {
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("st.volatile.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y)
                 : "memory");
  } else {
    asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y)
                 : "memory");
  }
}
__device__ __forceinline__ bool is_ready(double2 v) {
  return __double_as_longlong(v.x) != (long long)SENTINEL &&
         __double_as_longlong(v.y) != (long long)SENTINEL;
}

// Thread-per-row sparse triangular sweep in lock-step.  Thread t owns rows
// t, t+T, t+2T, ... of the sweep order; each warp loops while any lane still
// has work, and in every iteration a lane either consumes its next entry
// (source final -> acc -= L * y_src, the reference's rounding order) or polls
// again.  No lane ever blocks another lane of its warp, and the per-step
// critical path is one 16-byte poll plus one complex multiply-subtract.
// Row entries stream through two register groups of G: the group being
// consumed and the next one, whose loads were issued G consumptions earlier
// -- registers of an in-flight load are never touched on the hot path (a
// read would stall the whole warp for a memory latency).  Deadlock-free: the
// oldest unfinished row has all of its sources final and its lane polls it.
template <int G>
struct EntryGroup {
  int c[G];
  double2 l[G];
};

template <int G>
__device__ __forceinline__ void load_group(EntryGroup<G>& g, const int32_t* __restrict__ ci,
                                           const double2* __restrict__ v, int p, int step,
                                           int avail) {
#pragma unroll
  for (int k = 0; k < G; ++k) {
    if (k < avail) {
      g.c[k] = __ldg(ci + p + k * step);
      g.l[k] = __ldg(v + p + k * step);
    }
  }
}

template <int G>
__device__ __forceinline__ void pick(const EntryGroup<G>& g, int i, int& c, double2& l) {
  c = g.c[0];
  l = g.l[0];
#pragma unroll
  for (int k = 1; k < G; ++k)
    if (i == k) {
      c = g.c[k];
      l = g.l[k];
    }
}

template <bool UPPER>
__device__ __forceinline__ void tri_sweep(int n, const int32_t* __restrict__ rp,
                                          const int32_t* __restrict__ ci,
                                          const double2* __restrict__ v,
                                          const double2* __restrict__ rU, const double2* in,
                                          double2* out) {
  constexpr int G = 4;
  const int T = blockDim.x;
  const int step = UPPER ? -1 : 1;
  for (int base = 0; base < n; base += T) {
    const int q = base + threadIdx.x;
    const bool act = q < n;
    const int r = UPPER ? n - 1 - q : q;
    int left = 0, pnext = 0;
    double2 acc = make_double2(0.0, 0.0);
    EntryGroup<G> A, B;
    if (act) {
      const int p0 = rp[r], p1 = rp[r + 1];
      left = p1 - p0;
      const int p = UPPER ? p1 - 1 : p0;
      acc = in[r];
      load_group<G>(A, ci, v, p, step, left);
      load_group<G>(B, ci, v, p + G * step, step, left - G);
      pnext = p + 2 * G * step;
    }
    int apos = 0;
    bool pending = act;
    while (__any_sync(FULL, pending)) {
      if (pending) {
        if (left > 0) {
          int c;
          double2 l;
          pick<G>(A, apos, c, l);
          const double2 s = vld2(out + c);
          if (is_ready(s)) {
            acc = csub(acc, cmul_plain(l, s));
            --left;
            if (++apos == G && left > 0) {
              A = B;  // loaded G consumptions ago
              apos = 0;
              load_group<G>(B, ci, v, pnext, step, left - G);
              pnext += G * step;
            }
          }
        }
        if (left == 0) {
          vst2(out + r, UPPER ? cmul_plain(acc, __ldg(rU + r)) : acc);
          pending = false;
        }
      }
    }
  }
}

// Warp-per-row variant (rows dealt round-robin to warps): lanes fetch 32
// entries at a time, wait only on their own source, and the ordered
// subtraction chain advances over the ready prefix.
template <bool UPPER>
__device__ __forceinline__ void tri_sweep_warp(int n, const int32_t* __restrict__ rp,
                                               const int32_t* __restrict__ ci,
                                               const double2* __restrict__ v,
                                               const double2* __restrict__ rU,
                                               const double2* in, double2* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  long long* const tt = g_tri_times;
  for (int q = wid; q < n; q += nw) {
    const int r = UPPER ? n - 1 - q : q;
    if (tt && lane == 0) tt[2 * r] = clock64();
    const int p0 = rp[r], p1 = rp[r + 1];
    const int total = p1 - p0;
    double2 acc = in[r];
    for (int base = 0; base < total; base += 32) {
      const int e = base + lane;
      const bool act = e < total;
      int c = 0;
      double2 lv = make_double2(0.0, 0.0);
      if (act) {
        const int p = UPPER ? p1 - 1 - e : p0 + e;
        c = __ldg(ci + p);
        lv = __ldg(v + p);
      }
      const int cnt = min(32, total - base);
      bool have = !act;
      double2 prod = make_double2(0.0, 0.0);
      int done = 0;
      unsigned nap = 0;
      while (done < cnt) {
        if (!have) {
          const double2 s = vld2(out + c);
          if (is_ready(s)) {
            prod = cmul_plain(lv, s);
            have = true;
          }
        }
        const unsigned m = __ballot_sync(FULL, have);
        const unsigned pend = ~m;
        int upto = pend ? (__ffs(pend) - 1) : 32;
        if (upto > cnt) upto = cnt;
        if (upto == done) {
          // nothing new: back off so polling warps leave the issue slots to
          // the warp on the critical path (the solve is latency-bound)
          nap = nap ? min(nap * 2, g_tri_nap_max) : g_tri_nap_min;
          if (nap) __nanosleep(nap);
          continue;
        }
        nap = 0;
        for (int k = done; k < upto; ++k) {
          const double px = __shfl_sync(FULL, prod.x, k);
          const double py = __shfl_sync(FULL, prod.y, k);
          acc = csub(acc, make_double2(px, py));
        }
        done = upto;
      }
    }
    if (lane == 0) {
      vst2(out + r, UPPER ? cmul_plain(acc, __ldg(rU + r)) : acc);
      if (tt) tt[2 * r + 1] = clock64();
    }
    __syncwarp();
  }
}

// Warp-per-row with a lane-0 ordered fold.  For each chunk of up to 64
// entries the warp loads (column, value) pairs coalesced, tries each source
// once and stores the product of every source already final into a per-warp
// shared buffer; then lane 0 alone folds the chunk in the reference order,
// reading precomputed products and, for the entries that were not ready,
// polling the source in a tight loop and multiplying itself.  The critical
// hop (last source published -> this row published) is therefore one
// shared-memory poll, one complex multiply-subtract and one 16-byte store.
constexpr int FOLD_CHUNK = 64;

struct FoldBuf {
  int c[FOLD_CHUNK];
  double2 l[FOLD_CHUNK];
  double2 p[FOLD_CHUNK];
  unsigned ok[FOLD_CHUNK / 32];
};

template <bool UPPER>
__device__ __forceinline__ void tri_sweep_fold(int n, const int32_t* __restrict__ rp,
                                               const int32_t* __restrict__ ci,
                                               const double2* __restrict__ v,
                                               const double2* __restrict__ rU,
                                               const double2* in, double2* out,
                                               FoldBuf* bufs) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  FoldBuf& B = bufs[wid];
  for (int q = wid; q < n; q += nw) {
    const int r = UPPER ? n - 1 - q : q;
    const int p0 = rp[r], p1 = rp[r + 1];
    const int total = p1 - p0;
    double2 acc = in[r];
    const double2 rr = UPPER ? __ldg(rU + r) : make_double2(0.0, 0.0);
    for (int base = 0; base < total; base += FOLD_CHUNK) {
      const int cnt = min(FOLD_CHUNK, total - base);
#pragma unroll
      for (int h = 0; h < FOLD_CHUNK / 32; ++h) {
        const int e = h * 32 + lane;
        bool ok = false;
        if (e < cnt) {
          const int p = UPPER ? p1 - 1 - (base + e) : p0 + base + e;
          const int c = __ldg(ci + p);
          const double2 lv = __ldg(v + p);
          B.c[e] = c;
          B.l[e] = lv;
          const double2 s = vld2(out + c);
          if (is_ready(s)) {
            B.p[e] = cmul_plain(lv, s);
            ok = true;
          }
        }
        const unsigned m = __ballot_sync(FULL, ok);
        if (lane == 0) B.ok[h] = m;
      }
      __syncwarp();
      if (lane == 0) {
        for (int e = 0; e < cnt; ++e) {
          double2 pe;
          if ((B.ok[e >> 5] >> (e & 31)) & 1u) {
            pe = B.p[e];
          } else {
            const int c = B.c[e];
            double2 s;
            do {
              s = vld2(out + c);
            } while (!is_ready(s));
            pe = cmul_plain(B.l[e], s);
          }
          acc = csub(acc, pe);
        }
      }
      __syncwarp();
    }
    if (lane == 0) vst2(out + r, UPPER ? cmul_plain(acc, rr) : acc);
    __syncwarp();
  }
}

// Lane-per-row sweep over the SELL-32 factor layout (sell.cu).  Warp w takes
// slices w, w+W, ...; lane l of slice s owns sweep position 32s+l and folds
// its row's terms in the reference order straight from registers: the next
// 2*G entries sit in two register groups (refilled one group at a time with
// coalesced loads while the other is consumed), each loop iteration polls
// every unconsumed source of the current group at once and folds the ready
// prefix.  A row's far terms (sources finished long before) fold at G terms
// per iteration; its last term -- the row just published -- costs one poll,
// one complex multiply-subtract and the publishing store.  No shuffles, no
// cross-lane fold: 32 rows advance per warp instruction.
template <int G>
struct SellGroup {
  int c[G];
  double2 l[G];
};

template <int G>
__device__ __forceinline__ void sell_load(SellGroup<G>& g, const int32_t* __restrict__ cp,
                                          const double2* __restrict__ vp, int k, int w) {
#pragma unroll
  for (int j = 0; j < G; ++j) {
    if (k + j < w) {
      g.c[j] = __ldg(cp + 32 * (k + j));
      g.l[j] = __ldg(vp + 32 * (k + j));
    } else {
      g.c[j] = -1;
    }
  }
}

template <bool UPPER, int G = 4>
__device__ __forceinline__ void tri_sweep_sell(int n, const int32_t* __restrict__ sptr,
                                               const int32_t* __restrict__ sci,
                                               const double2* __restrict__ sv,
                                               const double2* __restrict__ rU,
                                               const double2* in, double2* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int nsl = (n + 31) >> 5;
  for (int s = wid; s < nsl; s += nw) {
    const int q = 32 * s + lane;
    const bool act = q < n;
    const int r = UPPER ? n - 1 - q : q;
    const int32_t p0 = __ldg(sptr + s);
    const int w = (__ldg(sptr + s + 1) - p0) >> 5;
    const int32_t* cp = sci + p0 + lane;
    const double2* vp = sv + p0 + lane;
    double2 acc = act ? in[r] : make_double2(0.0, 0.0);
    const double2 rr = (UPPER && act) ? __ldg(rU + r) : make_double2(0.0, 0.0);
    SellGroup<G> A, B;
    sell_load<G>(A, cp, vp, 0, w);
    sell_load<G>(B, cp, vp, G, w);
    int k = 0, apos = 0;
    bool pending = act;
    if (pending && A.c[0] < 0) {  // empty row
      vst2(out + r, UPPER ? cmul_plain(acc, rr) : acc);
      pending = false;
    }
    while (__any_sync(FULL, pending)) {
      if (pending) {
        double2 src[G];
#pragma unroll
        for (int j = 0; j < G; ++j)
          src[j] = (j >= apos && A.c[j] >= 0) ? vld2(out + A.c[j]) : make_double2(0.0, 0.0);
        bool stop = false;
#pragma unroll
        for (int j = 0; j < G; ++j) {
          if (j >= apos && !stop) {
            if (A.c[j] >= 0 && is_ready(src[j])) {
              acc = csub(acc, cmul_plain(A.l[j], src[j]));
              apos = j + 1;
            } else {
              stop = true;
            }
          }
        }
        bool done = false;
#pragma unroll
        for (int j = 0; j < G; ++j)
          if (j == apos) done = A.c[j] < 0;  // next term is padding: row complete
        if (apos == G) {
          k += G;
          A = B;
          sell_load<G>(B, cp, vp, k + G, w);
          apos = 0;
          done = A.c[0] < 0;
        }
        if (done) {
          vst2(out + r, UPPER ? cmul_plain(acc, rr) : acc);
          pending = false;
        }
      }
    }
  }
}

// Unit-lower solve: out[r] = in[r] - sum_{c<r, ascending} L[r,c] out[c]
// (reference lower_solve, _ckernels.pyx:53-67).  out pre-filled with the
// sentinel.
__device__ __noinline__ static void lower_solve(int n, const int32_t* __restrict__ rp,
                                                const int32_t* __restrict__ ci,
                                                const double2* __restrict__ v,
                                                const double2* in, double2* out) {
  tri_sweep_warp<false>(n, rp, ci, v, nullptr, in, out);
}

// Upper solve: out[r] = (in[r] - sum_{c>r, descending} U[r,c] out[c]) *
// recipc(U_rr) (reference upper_solve, _ckernels.pyx:70-85).
__device__ __noinline__ static void upper_solve(int n, const int32_t* __restrict__ rp,
                                                const int32_t* __restrict__ ci,
                                                const double2* __restrict__ v,
                                                const double2* __restrict__ rU,
                                                const double2* in, double2* out) {
  tri_sweep_warp<true>(n, rp, ci, v, rU, in, out);
}

}  // namespace cta
}  // namespace rs
