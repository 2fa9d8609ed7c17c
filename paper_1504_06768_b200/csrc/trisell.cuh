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
  int32_t G;  // lanes per row (1, 2, 4, 8, 16, 32); H = 32 / G rows per slice
};

namespace tri {

// One slice.  rhs: right-hand side (final values, plain loads); out: solution
// vector (sentinel-initialised, published per row); rd: recipc(U_cc) (UPPER).
template <bool UPPER, int G>
__device__ __forceinline__ void sweep_slice(const TriSell& T, int32_t s, const double2* rhs,
                                            double2* out, const double2* rd) {
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int H = 32 / G;
  const int lane = threadIdx.x & 31;
  const int r = lane / G;
  const int32_t row = __ldg(T.order + (int64_t)s * H + r);
  const int32_t base = __ldg(T.sptr + s);
  const int32_t w = (__ldg(T.sptr + s + 1) - base) >> 5;
  double2 acc = row >= 0 ? __ldcg(rhs + row) : make_double2(0.0, 0.0);
  int32_t c_n = -1;
  double2 a_n = make_double2(0.0, 0.0);
  if (w > 0) {
    c_n = __ldg(T.sci + base + lane);
    a_n = ldg2(T.sv + base + lane);
  }
  for (int32_t k = 0; k < w; ++k) {
    const int32_t c = c_n;
    const double2 a = a_n;
    if (k + 1 < w) {  // next step's entry is in flight while this one waits
      c_n = __ldg(T.sci + base + 32 * (k + 1) + lane);
      a_n = ldg2(T.sv + base + 32 * (k + 1) + lane);
    }
    double2 p = make_double2(0.0, 0.0);
    if (c >= 0) {
      double2 yv = cta::vld2(out + c);
      while (!cta::is_ready(yv)) yv = cta::vld2(out + c);
      p = cmul_plain(a, yv);
    }
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
  if (row >= 0 && lane % G == 0) {
    if (UPPER) acc = cmul_plain(acc, rd[row]);
    cta::vst2(out + row, acc);
  }
}

template <bool UPPER>
__device__ __forceinline__ void sweep_slice_g(const TriSell& T, int32_t s, const double2* rhs,
                                              double2* out, const double2* rd) {
  switch (T.G) {
    case 1: sweep_slice<UPPER, 1>(T, s, rhs, out, rd); break;
    case 2: sweep_slice<UPPER, 2>(T, s, rhs, out, rd); break;
    case 4: sweep_slice<UPPER, 4>(T, s, rhs, out, rd); break;
    case 8: sweep_slice<UPPER, 8>(T, s, rhs, out, rd); break;
    case 16: sweep_slice<UPPER, 16>(T, s, rhs, out, rd); break;
    default: sweep_slice<UPPER, 32>(T, s, rhs, out, rd); break;
  }
}

}  // namespace tri
}  // namespace rs
