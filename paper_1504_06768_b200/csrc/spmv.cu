// Complex128 CSR SpMV, y = A x, bit-exact with the reference csr_matvec
// (pkg/src/rhosolve/kernels/_ckernels.pyx:34-50): every row is summed
// sequentially in storage order, the first term is a product (not 0 + p),
// complex products use the plain two-rounding formula, and empty rows give 0.
//
// B200 layout -- products element-parallel, sums row-sequential.  The only
// ordering constraint of the reference is the left fold of each row's
// products; the products themselves are independent.  A CTA owns SPMV_T
// consecutive rows, whose nonzeros form one contiguous slice of the CSR
// arrays.  Pass 1 streams that slice in chunks of SPMV_CHUNK entries: thread t
// takes entries t, t+T, ... (fully coalesced 4-byte index and 16-byte value
// loads, SPMV_UNROLL independent loads in flight per thread), gathers x
// through the read-only path and writes the complex product to shared memory.
// Pass 2: thread t folds its own row's products out of shared memory in
// storage order, carrying the partial sum across chunks -- so rows of any
// length (the modified Liouvillian's trace row) need no special path.  The
// kernel streams 20 B per nonzero once: the HBM roofline case.
//
// Batches of B equal-size systems are stored block-diagonally: row_ptr spans
// all B*n rows, column indices are local to their system, and system b reads
// x[b*n ...].  A CTA can straddle system boundaries; the element offsets at
// which a new system starts inside the CTA's slice sit in a small shared
// table.  A single system is B = 1.
#include "common.cuh"
#include "kernels.cuh"

namespace rs {

constexpr int SPMV_T = 256;        // threads = rows per CTA
constexpr int SPMV_CHUNK = 2048;   // products staged per pass (32 KB)
constexpr int SPMV_UNROLL = SPMV_CHUNK / SPMV_T;
constexpr int SPMV_MAXSYS = SPMV_T + 2;

__global__ void __launch_bounds__(SPMV_T)
spmv_kernel(int64_t nrows, int32_t n, const int32_t* __restrict__ rp,
            const int32_t* __restrict__ ci, const double2* __restrict__ v,
            const double2* __restrict__ x, double2* __restrict__ y) {
  __shared__ __align__(16) double2 s_p[SPMV_CHUNK];
  __shared__ int32_t s_sysbeg[SPMV_MAXSYS];  // element where each later system starts
  __shared__ int s_nb;

  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * SPMV_T;
  const int64_t r1 = min(r0 + SPMV_T, nrows);
  const int64_t row = r0 + tid;
  const bool have = row < r1;
  const int32_t base = __ldg(rp + r0), end = __ldg(rp + r1);
  const int32_t p0 = have ? __ldg(rp + row) : 0, p1 = have ? __ldg(rp + row + 1) : 0;

  // system boundaries inside [r0, r1): rows that are multiples of n
  const int64_t s0 = r0 / n;
  if (tid == 0) s_nb = 0;
  __syncthreads();
  if (have && row > r0 && row % n == 0) {
    const int k = (int)(row / n - s0) - 1;
    s_sysbeg[k] = p0;
    atomicMax(&s_nb, k + 1);
  }
  __syncthreads();
  const int nb = s_nb;

  double2 acc = make_double2(0.0, 0.0);
  for (int32_t cb = base; cb < end; cb += SPMV_CHUNK) {
    const int32_t ce = min(cb + SPMV_CHUNK, end);
    int c[SPMV_UNROLL];
    double2 a[SPMV_UNROLL];
#pragma unroll
    for (int u = 0; u < SPMV_UNROLL; ++u) {
      const int32_t e = cb + u * SPMV_T + tid;
      if (e < ce) {
        c[u] = __ldg(ci + e);
        a[u] = ldg2(v + e);
      }
    }
#pragma unroll
    for (int u = 0; u < SPMV_UNROLL; ++u) {
      const int32_t e = cb + u * SPMV_T + tid;
      if (e < ce) {
        int64_t sys = s0;
        for (int k = 0; k < nb && e >= s_sysbeg[k]; ++k) ++sys;
        s_p[e - cb] = cmul_plain(a[u], ldg2(x + sys * n + c[u]));
      }
    }
    __syncthreads();
    const int32_t qa = max(p0, cb), qb = min(p1, ce);
    for (int32_t q = qa; q < qb; ++q) {
      const double2 pq = s_p[q - cb];
      acc = (q == p0) ? pq : cadd(acc, pq);
    }
    __syncthreads();
  }
  if (have) y[row] = acc;
}

int launch_spmv(int64_t nrows, int32_t n, const int32_t* rp, const int32_t* ci,
                const double2* v, const double2* x, double2* y,
                cudaStream_t st) {
  if (nrows == 0) return RS_OK;
  RS_CHECK_ARG(n > 0, "n must be positive");
  const int64_t grid = (nrows + SPMV_T - 1) / SPMV_T;
  spmv_kernel<<<(unsigned)grid, SPMV_T, 0, st>>>(nrows, n, rp, ci, v, x, y);
  ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

}  // namespace rs
