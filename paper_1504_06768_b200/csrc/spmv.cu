// Complex128 CSR SpMV, y = A x, bit-exact with the reference csr_matvec
// (pkg/src/rhosolve/kernels/_ckernels.pyx:34-50): every row is summed
// sequentially in storage order, the first term is a product (not 0 + p),
// complex products use the plain two-rounding formula, and empty rows give 0.
//
// B200 layout: a CTA owns ROWS consecutive rows.  Their column indices and
// values form one contiguous slice of the CSR arrays, which the CTA streams
// into shared memory with fully coalesced 16-byte loads (int32 indices,
// double2 values; 20 B per nonzero, the algorithmic minimum).  Each thread then
// runs the sequential sum for its own row out of shared memory, gathering x
// through the read-only path (the RCM band keeps x accesses L1/L2 local).
// Slices larger than the staging buffer (the trace row of the modified
// Liouvillian, ~D+15 entries) fall back to direct global reads for that CTA.
//
// Batches of B equal-size systems are stored block-diagonally: row_ptr spans
// all B*n rows, column indices are local to their system, and system b reads
// x[b*n ...].  A single system is B = 1.
#include "common.cuh"
#include "kernels.cuh"

namespace rs {

constexpr int SPMV_ROWS = 128;
constexpr int SPMV_CAP = 3072;  // staged nonzeros per CTA (60 KB)

__global__ void __launch_bounds__(SPMV_ROWS)
spmv_staged_kernel(int64_t nrows, int32_t n, const int32_t* __restrict__ rp,
                   const int32_t* __restrict__ ci,
                   const double2* __restrict__ v,
                   const double2* __restrict__ x, double2* __restrict__ y) {
  extern __shared__ __align__(16) unsigned char smem[];
  double2* s_v = reinterpret_cast<double2*>(smem);
  int32_t* s_c = reinterpret_cast<int32_t*>(s_v + SPMV_CAP);

  const int64_t r0 = (int64_t)blockIdx.x * SPMV_ROWS;
  if (r0 >= nrows) return;
  const int64_t r1 = min(r0 + SPMV_ROWS, nrows);
  const int32_t base = rp[r0];
  const int32_t cnt = rp[r1] - base;
  const int64_t row = r0 + threadIdx.x;
  const bool staged = cnt <= SPMV_CAP;
  if (staged) {
    for (int e = threadIdx.x; e < cnt; e += SPMV_ROWS) {
      s_v[e] = ldg2(v + base + e);
      s_c[e] = __ldg(ci + base + e);
    }
    __syncthreads();
  }
  if (row >= r1) return;
  const double2* xs = x + (row / n) * (int64_t)n;
  const int32_t p0 = rp[row], p1 = rp[row + 1];
  double2 s = make_double2(0.0, 0.0);
  if (p0 < p1) {
    if (staged) {
      int q = p0 - base;
      const int qe = p1 - base;
      s = cmul_plain(s_v[q], ldg2(xs + s_c[q]));
      for (++q; q < qe; ++q) s = cadd(s, cmul_plain(s_v[q], ldg2(xs + s_c[q])));
    } else {
      int q = p0;
      s = cmul_plain(ldg2(v + q), ldg2(xs + __ldg(ci + q)));
      for (++q; q < p1; ++q)
        s = cadd(s, cmul_plain(ldg2(v + q), ldg2(xs + __ldg(ci + q))));
    }
  }
  y[row] = s;
}

int launch_spmv(int64_t nrows, int32_t n, const int32_t* rp, const int32_t* ci,
                const double2* v, const double2* x, double2* y,
                cudaStream_t st) {
  if (nrows == 0) return RS_OK;
  static bool attr_set = false;
  const size_t smem = SPMV_CAP * (sizeof(double2) + sizeof(int32_t));
  if (!attr_set) {
    RS_CUDA_TRY(cudaFuncSetAttribute(spmv_staged_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    attr_set = true;
  }
  const int64_t grid = (nrows + SPMV_ROWS - 1) / SPMV_ROWS;
  spmv_staged_kernel<<<(unsigned)grid, SPMV_ROWS, smem, st>>>(nrows, n, rp, ci,
                                                              v, x, y); ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

}  // namespace rs
