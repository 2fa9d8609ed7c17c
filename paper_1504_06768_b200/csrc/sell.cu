// Sliced-ELL (SELL-32) layout of the triangular factors for the lane-per-row
// sweeps (cta_ops.cuh tri_sweep_sell).
//
// The sweep visits rows in "sweep order" q = 0..n-1 (L: row q, ascending;
// U: row n-1-q, descending), and each row folds its terms in the reference
// order (L: ascending column, U: descending column; _ckernels.pyx:53-85).
// Slice s holds sweep positions 32s..32s+31, one per lane; entry k of lane l
// sits at sptr[s] + 32k + l, so when the 32 lanes of a warp consume their
// k-th terms together the loads are one coalesced 128-byte index line and
// four 128-byte value lines.  A slice is as wide as its longest row; shorter
// rows are padded with column -1, which also marks the end of a row.
//
// sptr is absolute over the block-diagonal batch: system b's slices are
// sptr[b*nsl .. b*nsl + nsl] with nsl = ceil(n/32).
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.cuh"

namespace rs {

namespace {
inline unsigned grid_of(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }
}  // namespace

__global__ void sell_width_kernel(int B, int32_t n, int upper, const int32_t* __restrict__ rp,
                                  int32_t* __restrict__ width) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)B * n) return;
  const int64_t b = t / n;
  const int32_t q = (int32_t)(t % n);
  const int32_t r = upper ? n - 1 - q : q;
  const int64_t row = b * n + r;
  const int32_t len = rp[row + 1] - rp[row];
  const int32_t nsl = (n + 31) >> 5;
  // 32 * (max length in the slice): the slice's entry count
  atomicMax(&width[b * nsl + (q >> 5)], 32 * len);
}

__global__ void sell_fill_kernel(int B, int32_t n, int upper, const int32_t* __restrict__ rp,
                                 const int32_t* __restrict__ ci, const double2* __restrict__ v,
                                 const int32_t* __restrict__ sptr, int32_t* __restrict__ sci,
                                 double2* __restrict__ sv) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int32_t nsl = (n + 31) >> 5;
  if (t >= (int64_t)B * nsl * 32) return;
  const int64_t b = t / ((int64_t)nsl * 32);
  const int32_t qq = (int32_t)(t % ((int64_t)nsl * 32));
  const int32_t s = qq >> 5, l = qq & 31;
  const int32_t p0 = sptr[b * nsl + s];
  const int32_t w = (sptr[b * nsl + s + 1] - p0) >> 5;
  int32_t len = 0, e0 = 0;
  if (qq < n) {
    const int32_t r = upper ? n - 1 - qq : qq;
    const int64_t row = b * n + r;
    e0 = rp[row];
    len = rp[row + 1] - e0;
  }
  for (int32_t k = 0; k < w; ++k) {
    const int32_t o = p0 + 32 * k + l;
    if (k < len) {
      const int32_t e = upper ? e0 + len - 1 - k : e0 + k;
      sci[o] = ci[e];
      sv[o] = v[e];
    } else {
      sci[o] = -1;
      sv[o] = make_double2(0.0, 0.0);
    }
  }
}

int sell_build(int B, int32_t n, int upper, const int32_t* rp, const int32_t* ci,
               const double2* v, int32_t* sptr, int32_t* sci, double2* sv, int64_t* total,
               cudaStream_t st) {
  const int32_t nsl = (n + 31) >> 5;
  const int64_t nslices = (int64_t)B * nsl;
  if (!sci) {
    // pass 1: slice sizes -> sptr, total padded entries
    int32_t* width = nullptr;
    RS_CUDA_TRY(cudaMallocAsync(&width, sizeof(int32_t) * (nslices + 1), st));
    RS_CUDA_TRY(cudaMemsetAsync(width, 0, sizeof(int32_t) * (nslices + 1), st));
    if (B > 0 && n > 0) {
      sell_width_kernel<<<grid_of((int64_t)B * n, 256), 256, 0, st>>>(B, n, upper, rp, width);
      ::rs::count_launch();
      RS_CUDA_TRY(cudaGetLastError());
    }
    // 64-bit scan on the host side would need a copy; entries fit int32 when
    // the padded total does (checked below).
    int64_t tot = 0;
    int rc = scan_counts(width, sptr, nslices, &tot, st);
    cudaFreeAsync(width, st);
    if (rc) return rc;
    if (tot < 0 || tot >= ((int64_t)1 << 31)) {
      set_error("sell_build: %lld padded entries exceed int32 indexing", (long long)tot);
      return RS_ERR_OVERFLOW;
    }
    if (total) *total = tot;
    return RS_OK;
  }
  if (B > 0 && n > 0) {
    sell_fill_kernel<<<grid_of(nslices * 32, 256), 256, 0, st>>>(B, n, upper, rp, ci, v, sptr,
                                                                 sci, sv);
    ::rs::count_launch();
    RS_CUDA_TRY(cudaGetLastError());
  }
  return RS_OK;
}

}  // namespace rs
