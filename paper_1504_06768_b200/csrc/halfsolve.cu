// In-place triangular half-solves on the raw CSC factors: the device
// equivalents of the reference seam's lower_solve / upper_solve
// (_ckernels.pyx:53-67, 70-85; bound at kernels/__init__.py:21-24).
//
// The reference loops are executed verbatim, column by column, by ONE warp per
// system: a column's off-diagonal entries update distinct rows of y, so their
// order within the column is free and they are applied lane-parallel; a
// __syncwarp orders them before the next column reads its own y entry.  Every
// y[i] therefore receives its subtractions in ascending (L) / descending (U)
// column order, exactly as the scalar loops produce them -- bit-identical.
// No allocation, no synchronisation: the calls are stream-ordered.  The fused
// preconditioner apply of the solvers (colsweep.cuh) is the fast path; these
// two exist so that the reference's own factor.solve_lu runs unmodified on
// the device kernels.
#include "common.cuh"
#include "kernels.cuh"

namespace rs {

template <bool UPPER>
__global__ void __launch_bounds__(32) half_solve_kernel(int32_t n, const int32_t* __restrict__ cp,
                                                        const int32_t* __restrict__ ci,
                                                        const double2* __restrict__ cx,
                                                        int64_t cap, double2* y) {
  const int64_t b = blockIdx.x;
  const int lane = threadIdx.x;
  cp += b * (n + 1);
  ci += b * cap;
  cx += b * cap;
  y += b * n;
  if (!UPPER) {
    int32_t p1 = cp[0];
    for (int32_t c = 0; c < n; ++c) {
      const int32_t p0 = p1 + 1;  // skip the unit diagonal
      p1 = cp[c + 1];
      const double2 xc = y[c];
      for (int32_t p = p0 + lane; p < p1; p += 32) {
        const int32_t i = ci[p];
        y[i] = csub(y[i], cmul_plain(cx[p], xc));
      }
      __syncwarp();
    }
  } else {
    int32_t e = cp[n];
    for (int32_t c = n - 1; c >= 0; --c) {
      const int32_t p1 = e - 1;  // the pivot is the column's last entry
      const int32_t p0 = cp[c];
      e = p0;
      const double2 xc = cmul_plain(y[c], recipc(cx[p1]));
      __syncwarp();  // every lane has read y[c]
      if (lane == 0) y[c] = xc;
      for (int32_t p = p0 + lane; p < p1; p += 32) {
        const int32_t i = ci[p];
        y[i] = csub(y[i], cmul_plain(cx[p], xc));
      }
      __syncwarp();
    }
  }
}

int half_solve(int upper, int B, int32_t n, const int32_t* cp, const int32_t* ci,
               const double2* cx, int64_t cap, double2* y, cudaStream_t st) {
  if (!B || !n) return RS_OK;
  if (upper) half_solve_kernel<true><<<B, 32, 0, st>>>(n, cp, ci, cx, cap, y);
  else half_solve_kernel<false><<<B, 32, 0, st>>>(n, cp, ci, cx, cap, y);
  count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

}  // namespace rs
