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
  const int32_t* skey;   // per chunk of KREG steps: its dependency of the highest level (-1: none)
  int32_t nslices;
  int32_t G;  // lanes per row (1, 2, 4 or 32); H = 32 / G rows per slice
  // Warps per CTA that take part in the sweep (0 = all).  Every waiting lane
  // polls a value near the sweep's frontier, so a narrow DAG (config 3: ~3
  // rows per level) swept by every resident warp turns the frontier's L2
  // sectors into a hot spot (measured: 41 us per level with 2,368 warps);
  // the window of slices in flight only needs to cover the pre-fold latency.
  int32_t apw;
  int32_t mode;  // tuning: 1 = wait for every chunk's key before the first chunk
};

namespace tri {

// tuning hook: per-slice (start, first step done, end) global-timer stamps [3 * nslices]
__device__ unsigned long long* g_slice_times = nullptr;
__device__ int g_slice_clock_mode = 0;  // 1: slots hold clock64 deltas (key seen->loaded, loaded->published)
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Ordered fold of one step's products into the row accumulators: the G lanes
// of a row subtract their products in lane order (= storage order).
// `live`: ballot of the lanes holding a real entry in this step; trailing
// lane positions that are padding in every row of the slice are skipped
// (subtracting their +0 would change nothing).
template <int G>
__device__ __forceinline__ void fold_step(double2& acc, double2 p, int r, unsigned live) {
  constexpr unsigned FULL = 0xffffffffu;
  if (G == 1) {
    acc = csub(acc, p);
  } else {
    unsigned m = live;
#pragma unroll
    for (int sh = G; sh < 32; sh <<= 1) m |= m >> sh;
    m &= (G == 32) ? 0xffffffffu : ((1u << G) - 1u);
    const int cnt = 32 - __clz(m);  // lane positions 0 .. cnt-1 of a row are in use
#pragma unroll 1
    for (int j = 0; j < cnt; ++j) {
      const double px = __shfl_sync(FULL, p.x, r * G + j);
      const double py = __shfl_sync(FULL, p.y, r * G + j);
      acc = csub(acc, make_double2(px, py));
    }
  }
}

// One slice.  rhs: right-hand side (final values); out: solution vector
// (sentinel-initialised, published per row); rd: recipc(U_cc) (UPPER).
//
// Waiting is decoupled from loading and folding.  The slice is consumed in
// chunks of KREG steps held in registers: a chunk's factor entries are loaded
// with KREG independent loads per lane, every source value is requested at
// once, the not-yet-published ones are re-polled together, and the fold runs
// from registers in storage order.  The static loads of a slice's first chunk
// are issued before any waiting, so a dependency hop costs one L2 round trip
// plus the fold -- not one round trip per step (measured: 30 us per level with
// step-by-step loads on config 5).
constexpr int KREG = 8;

template <bool UPPER, int G>
__device__ __forceinline__ void sweep_slice(const TriSell& T, int32_t s, const double2* rhs,
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
  double2 rdv = make_double2(1.0, 0.0);
  if (UPPER && row >= 0) rdv = ldg2(rd + row);
  const int32_t* ci = T.sci + base + lane;
  const double2* av = T.sv + base + lane;
  const int32_t* keys = T.skey + ((base >> 5) / KREG + s);
  if (T.mode == 1) {  // tuning: serialize the whole slice behind its latest dependency
    for (int32_t k0 = 0; k0 < w; k0 += KREG) {
      const int32_t key = __ldg(keys + k0 / KREG);
      if (key >= 0) {
        double2 kv = cta::vld2(out + key);
        while (!__all_sync(0xffffffffu, cta::is_ready(kv))) kv = cta::vld2(out + key);
      }
    }
  }
  long long ck_seen = 0;
  for (int32_t k0 = 0; k0 < w; k0 += KREG) {
    int32_t c[KREG];
    double2 a[KREG], y[KREG];
#pragma unroll
    for (int k = 0; k < KREG; ++k) {
      c[k] = -1;
      if (k0 + k < w) {
        c[k] = __ldg(ci + 32 * (k0 + k));
        a[k] = ldg2(av + 32 * (k0 + k));
      }
    }
    {
      // The warp watches this chunk's latest dependency (highest level) while
      // the entry loads above are in flight; when it is published the chunk's
      // other sources almost always are.  Early chunks hold the oldest
      // sources, so they are folded long before the chain arrives and only
      // the last chunk sits on the critical path.  (Polling every source from
      // every waiting lane -- 1,184 warps x 32 lanes x 8 loads on config 5 --
      // saturates L2 and stretches a dependency hop to ~16 us.)
      // Every lane loads the same address (one broadcast request per poll) and
      // the loop is warp-uniform: a lone polling lane with the other 31 parked
      // at a __syncwarp cost ~2,000 cycles of re-convergence per hop.
      const int32_t key = __ldg(keys + k0 / KREG);
      if (key >= 0) {
        double2 kv = cta::vld2(out + key);
        while (!__all_sync(0xffffffffu, cta::is_ready(kv))) kv = cta::vld2(out + key);
      }
    }
    const long long ck0 = (tt && g_slice_clock_mode) ? clock64() : 0;
    unsigned pend = 0;
#pragma unroll
    for (int k = 0; k < KREG; ++k)
      if (c[k] >= 0) y[k] = cta::vld2(out + c[k]);
#pragma unroll
    for (int k = 0; k < KREG; ++k)
      if (c[k] >= 0 && !cta::is_ready(y[k])) pend |= 1u << k;
    while (__any_sync(0xffffffffu, pend != 0)) {  // warp-uniform: stragglers only
#pragma unroll
      for (int k = 0; k < KREG; ++k)
        if ((pend >> k) & 1u) y[k] = cta::vld2(out + c[k]);
#pragma unroll
      for (int k = 0; k < KREG; ++k)
        if (((pend >> k) & 1u) && cta::is_ready(y[k])) pend &= ~(1u << k);
    }
    if (tt && k0 == 0) tt[3 * (int64_t)s + 1] = g_slice_clock_mode ? (unsigned long long)(clock64() - ck0) : gtime();
    ck_seen = (tt && g_slice_clock_mode) ? clock64() : 0;
#pragma unroll
    for (int k = 0; k < KREG; ++k) {
      if (k0 + k < w) {  // warp-uniform
        const double2 p = c[k] >= 0 ? cmul_plain(a[k], y[k]) : make_double2(0.0, 0.0);
        fold_step<G>(acc, p, r, G == 1 ? 0u : __ballot_sync(0xffffffffu, c[k] >= 0));
      }
    }
  }
  if (tt && g_slice_clock_mode) tt[3 * (int64_t)s] = (unsigned long long)(clock64() - ck_seen);
  if (row >= 0 && lane % G == 0) {
    if (UPPER) acc = cmul_plain(acc, rdv);
    cta::vst2(out + row, acc);
  }
  if (tt) tt[3 * (int64_t)s + 2] = g_slice_clock_mode ? (unsigned long long)(clock64() - ck_seen) : gtime();
}

// The whole sweep from inside a grid-wide kernel: the first apw warps of
// every CTA take slices in ascending order, consecutive slices going to
// different CTAs.  All participants are co-resident, so waits cannot deadlock.
// One out-of-line body per (triangle, lanes per row) with the slice code
// inlined into its loop: called through the ABI per slice, sweep_slice saved
// and restored ~0.5-1 KB of registers in local memory on every call and a
// dependency hop took 4,460 cycles from "sources loaded" to "published".
template <bool UPPER, int G>
__device__ __noinline__ void sweep_loop(const TriSell& T, const double2* rhs, double2* out,
                                        const double2* rd, int32_t first, int32_t stride) {
  for (int32_t s = first; s < T.nslices; s += stride) sweep_slice<UPPER, G>(T, s, rhs, out, rd);
}

// The sweep bodies are reached through a table of function pointers, i.e. by
// an INDIRECT call: that forces the standard ABI on them (compiled on their
// own with the full register budget; the caller saves what it needs around
// the call, once per sweep).  Called directly from the solver kernel, ptxas'
// interprocedural register allocation confined them to the registers the
// Krylov code leaves free (R144 and up) and the polling loop spilled on every
// step: the same sweeps ran 1.9x slower inside grid_solver_kernel than in
// grid_apply_kernel (2.70 + 1.57 ms vs 1.38 + 0.85 ms per apply on config 5).
typedef void (*sweep_fn_t)(const TriSell&, const double2*, double2*, const double2*, int32_t,
                           int32_t);
__device__ sweep_fn_t g_sweep_table[2][4] = {
    {sweep_loop<false, 1>, sweep_loop<false, 2>, sweep_loop<false, 4>, sweep_loop<false, 32>},
    {sweep_loop<true, 1>, sweep_loop<true, 2>, sweep_loop<true, 4>, sweep_loop<true, 32>}};

template <bool UPPER>
__device__ __forceinline__ void sweep_grid(const TriSell& T, const double2* rhs, double2* out,
                                           const double2* rd) {
  const int wpc = blockDim.x >> 5;
  const int apw = (T.apw > 0 && T.apw < wpc) ? T.apw : wpc;
  const int lw = threadIdx.x >> 5;
  if (lw >= apw) return;
  const int32_t stride = apw * (int32_t)gridDim.x;
  const int32_t first = lw * (int32_t)gridDim.x + blockIdx.x;
  // the layouts levels.cu is asked for: 32, 16, 8 or 1 rows per slice
  const int idx = T.G == 1 ? 0 : T.G == 2 ? 1 : T.G == 4 ? 2 : 3;
  sweep_fn_t fn = *(volatile sweep_fn_t*)&g_sweep_table[UPPER ? 1 : 0][idx];
  fn(T, rhs, out, rd, first, stride);
}

}  // namespace tri
}  // namespace rs
