// Sync-free, level-ordered sparse triangular sweeps across the whole GPU: the
// preconditioner apply of systems too large for one CTA (config 3, the
// block-Jacobi blocks of config 5).  Bit-identical to the reference
// lower_solve / upper_solve (_ckernels.pyx:53-85): every row folds its terms
// in the reference order (ascending column for L, descending for U, then
// x_c = y_c * recipc(U_cc)); only independent rows run concurrently.
//
// Data: the level-ordered SELL layout built by levels.cu.  A warp owns one
// slice (H = 32/G rows of ONE level, G lanes per row).  Step k: every lane
// loads its entry (coalesced), waits until the source value y[col] has been
// published (readiness travels with the value: outputs start as a sentinel
// NaN and are published with one 16-byte store, cta_ops.cuh), multiplies, and
// the G products of a row are subtracted in lane order through shuffles, so
// the fold order is the storage order.  Padding subtracts +0, which changes
// nothing.  Rows of one slice never depend on each other, and a slice only
// waits on slices of earlier levels, which sit at lower slice numbers: with
// slices taken in ascending order by co-resident (or ticketed) warps nothing
// can deadlock.
#pragma once
#include "common.cuh"
#include "cta_ops.cuh"

namespace rs {

struct TriSell {
  const int32_t* order;  // [nslices * H] global row per sorted position, -1 = padding
  const int32_t* sptr;   // [nslices + 1] entry offsets (multiples of 32)
  const int32_t* sci;    // global column per entry, -1 = padding
  const double2* sv;
  int32_t nslices;
  int32_t G;  // lanes per row (1, 4 or 32); H = 32 / G rows per slice
  // Warps per CTA that take part in the sweep (0 = all).  Every waiting lane
  // polls a value near the sweep's frontier, so a narrow DAG (config 3: ~3
  // rows per level) swept by every resident warp turns the frontier's L2
  // sectors into a hot spot (measured: 41 us per level with 2,368 warps);
  // the window of slices in flight only needs to cover the pre-fold latency.
  int32_t apw;
};

namespace tri {

// tuning hook: per-slice (start, first step done, end) global-timer stamps [3 * nslices]
__device__ unsigned long long* g_slice_times = nullptr;
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Ordered fold of one step's products into the row accumulators: the G lanes
// of a row subtract their products in lane order (= storage order).
template <int G>
__device__ __forceinline__ void fold_step(double2& acc, double2 p, int r) {
  constexpr unsigned FULL = 0xffffffffu;
  if (G == 1) {
    acc = csub(acc, p);
  } else {
#pragma unroll
    for (int j = 0; j < G; ++j) {
      const double px = __shfl_sync(FULL, p.x, r * G + j);
      const double py = __shfl_sync(FULL, p.y, r * G + j);
      acc = csub(acc, make_double2(px, py));
    }
  }
}

// One slice.  rhs: right-hand side (final values); out: solution vector
// (sentinel-initialised, published per row); rd: recipc(U_cc) (UPPER).
//
// Waiting is decoupled from folding.  A slice of up to KREG steps (the sparse
// factors of config 5) keeps all its entries in registers: every source value
// is requested at once, the not-yet-published ones are re-polled together,
// and the fold runs from registers -- so a dependency hop costs one L2 round
// trip, not one per step.  Wider slices first wait for every source (loads
// four steps deep), then stream the fold with plain pipelined loads.
constexpr int KREG = 8;

template <bool UPPER, int G>
__device__ __noinline__ void sweep_slice(const TriSell& T, int32_t s, const double2* rhs,
                                         double2* out, const double2* rd) {
  constexpr int H = 32 / G;
  const int lane = threadIdx.x & 31;
  const int r = lane / G;
  const int32_t row = __ldg(T.order + (int64_t)s * H + r);
  const int32_t base = __ldg(T.sptr + s);
  const int32_t w = (__ldg(T.sptr + s + 1) - base) >> 5;
  unsigned long long* const tt = (!UPPER && lane == 0) ? g_slice_times : nullptr;
  if (tt) tt[3 * (int64_t)s] = gtime();
  double2 acc = row >= 0 ? __ldcg(rhs + row) : make_double2(0.0, 0.0);
  const int32_t* ci = T.sci + base + lane;
  const double2* av = T.sv + base + lane;
  if (w <= KREG) {
    int32_t c[KREG];
    double2 a[KREG], y[KREG];
#pragma unroll
    for (int k = 0; k < KREG; ++k) {
      c[k] = -1;
      if (k < w) {
        c[k] = __ldg(ci + 32 * k);
        a[k] = ldg2(av + 32 * k);
      }
    }
    unsigned pend = 0;
#pragma unroll
    for (int k = 0; k < KREG; ++k)
      if (c[k] >= 0) y[k] = cta::vld2(out + c[k]);
#pragma unroll
    for (int k = 0; k < KREG; ++k)
      if (c[k] >= 0 && !cta::is_ready(y[k])) pend |= 1u << k;
    while (pend) {
#pragma unroll
      for (int k = 0; k < KREG; ++k)
        if ((pend >> k) & 1u) y[k] = cta::vld2(out + c[k]);
#pragma unroll
      for (int k = 0; k < KREG; ++k)
        if (((pend >> k) & 1u) && cta::is_ready(y[k])) pend &= ~(1u << k);
    }
    if (tt) tt[3 * (int64_t)s + 1] = gtime();
#pragma unroll
    for (int k = 0; k < KREG; ++k) {
      if (k < w) {  // warp-uniform
        const double2 p = c[k] >= 0 ? cmul_plain(a[k], y[k]) : make_double2(0.0, 0.0);
        fold_step<G>(acc, p, r);
      }
    }
  } else {
    // phase A: every source of this lane is published (four steps in flight)
    for (int32_t k0 = 0; k0 < w; k0 += 4) {
      int32_t c[4];
      double2 y[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) c[u] = (k0 + u < w) ? __ldg(ci + 32 * (k0 + u)) : -1;
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c[u] >= 0) y[u] = cta::vld2(out + c[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c[u] >= 0)
          while (!cta::is_ready(y[u])) y[u] = cta::vld2(out + c[u]);
    }
    if (tt) tt[3 * (int64_t)s + 1] = gtime();
    // phase B: ordered fold, plain loads (published values never change)
    for (int32_t k0 = 0; k0 < w; k0 += 4) {
      int32_t c[4];
      double2 a[4], y[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        c[u] = -1;
        if (k0 + u < w) {
          c[u] = __ldg(ci + 32 * (k0 + u));
          a[u] = ldg2(av + 32 * (k0 + u));
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (c[u] >= 0) y[u] = __ldcg(out + c[u]);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (k0 + u < w) {
          const double2 p = c[u] >= 0 ? cmul_plain(a[u], y[u]) : make_double2(0.0, 0.0);
          fold_step<G>(acc, p, r);
        }
      }
    }
  }
  if (row >= 0 && lane % G == 0) {
    if (UPPER) acc = cmul_plain(acc, rd[row]);
    cta::vst2(out + row, acc);
  }
  if (tt) tt[3 * (int64_t)s + 2] = gtime();
}

template <bool UPPER>
__device__ __forceinline__ void sweep_slice_g(const TriSell& T, int32_t s, const double2* rhs,
                                              double2* out, const double2* rd) {
  switch (T.G) {  // the layouts levels.cu is asked for: 32, 8 or 1 rows per slice
    case 1: sweep_slice<UPPER, 1>(T, s, rhs, out, rd); break;
    case 4: sweep_slice<UPPER, 4>(T, s, rhs, out, rd); break;
    default: sweep_slice<UPPER, 32>(T, s, rhs, out, rd); break;
  }
}

// The whole sweep from inside a grid-wide kernel: the first apw warps of
// every CTA take slices in ascending order, consecutive slices going to
// different CTAs.  All participants are co-resident, so waits cannot deadlock.
template <bool UPPER>
__device__ __noinline__ void sweep_grid(const TriSell& T, const double2* rhs, double2* out,
                                           const double2* rd) {
  const int wpc = blockDim.x >> 5;
  const int apw = (T.apw > 0 && T.apw < wpc) ? T.apw : wpc;
  const int lw = threadIdx.x >> 5;
  if (lw >= apw) return;
  const int32_t stride = apw * (int32_t)gridDim.x;
  for (int32_t s = lw * (int32_t)gridDim.x + blockIdx.x; s < T.nslices; s += stride)
    sweep_slice_g<UPPER>(T, s, rhs, out, rd);
}

}  // namespace tri
}  // namespace rs
