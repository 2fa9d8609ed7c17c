// Complex128 CSR SpMV, y = A x, bit-exact with the reference csr_matvec
// (pkg/src/rhosolve/kernels/_ckernels.pyx:34-50): every row is summed
// sequentially in storage order, the first term is a product (not 0 + p),
// complex products use the plain two-rounding formula, and empty rows give 0.
//
// B200 layout -- products element-parallel, sums row-sequential.  The only
// ordering constraint of the reference is the left fold of each row's
// products; the products themselves are independent.  Each warp owns 32
// consecutive rows, whose nonzeros form one contiguous slice of the CSR
// arrays.  Pass 1 streams that slice in chunks of 32*UNROLL entries: lane l
// takes entries l, l+32, ... (fully coalesced 4-byte index and 16-byte value
// loads, UNROLL independent loads in flight per lane), gathers x through the
// read-only path and writes the complex product to a warp-private shared
// buffer.  Pass 2: lane l folds its own row's products in storage order,
// carrying the partial sum across chunks -- so rows of any length (the
// modified Liouvillian's trace row) need no special path.  Warps never wait
// on each other (no CTA barrier), so load and fold phases of different warps
// overlap.  The kernel streams 20 B per nonzero once: the HBM roofline case.
// Tuning (tools/spmv_probe.py): CTA-wide staging with 256-row CTAs reached
// 2.27-2.86 TB/s on the c4 batch, this warp-granular form 2.86 TB/s (158 MB)
// and 3.77 TB/s (633 MB); software-pipelining the next chunk spilled and lost.
//
// Batches of B equal-size systems are stored block-diagonally: row_ptr spans
// all B*n rows, column indices are local to their system, and system b reads
// x[b*n ...].  A CTA can straddle system boundaries; the element offsets at
// which a new system starts inside the CTA's slice sit in a small shared
// table.  A single system is B = 1.
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace rs {

// shared slot of staged product e (CTA-relative): one pad slot per 8 keeps
// the row-sequential fold (lane t reads ~8t + q for ~8-entry rows) off a
// single bank quad
template <bool PAD>
__device__ __forceinline__ int slot_of(int e) { return PAD ? e + (e >> 3) : e; }

// Warp-granular variant: each warp owns 32 consecutive rows and stages its
// own products in a private shared buffer, so warps never wait on each other
// (no CTA barrier) and load / fold phases of different warps overlap.
template <int UNROLL, int MINB>
__global__ void __launch_bounds__(256, MINB)
spmv_warp_kernel(int64_t nrows, int32_t n, const int32_t* __restrict__ rp,
                 const int32_t* __restrict__ ci, const double2* __restrict__ v,
                 const double2* __restrict__ x, double2* __restrict__ y) {
  constexpr int CH = 32 * UNROLL;
  __shared__ __align__(16) double2 s_buf[8][CH + CH / 8];
  __shared__ int32_t s_beg[8][34];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double2* s_p = s_buf[wid];
  int32_t* s_sysbeg = s_beg[wid];
  const int64_t r0 = ((int64_t)blockIdx.x * 8 + wid) * 32;
  if (r0 >= nrows) return;
  const int64_t r1 = min(r0 + 32, nrows);
  const int64_t row = r0 + lane;
  const bool have = row < r1;
  const int32_t base = __ldg(rp + r0), end = __ldg(rp + r1);
  const int32_t p0 = have ? __ldg(rp + row) : 0, p1 = have ? __ldg(rp + row + 1) : 0;
  const int64_t s0 = r0 / n;
  // system starts inside the warp's rows (ballot-compacted, ascending)
  const bool starts = have && row > r0 && row % n == 0;
  const unsigned sm = __ballot_sync(0xffffffffu, starts);
  if (starts) s_sysbeg[__popc(sm & ((1u << lane) - 1u))] = p0;
  const int nb = __popc(sm);
  __syncwarp();
  double2 acc = make_double2(0.0, 0.0);
  for (int32_t cb = base; cb < end; cb += CH) {
    const int32_t ce = min(cb + CH, end);
    int c[UNROLL];
    double2 a[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int32_t e = cb + 32 * u + lane;
      if (e < ce) {
        c[u] = __ldg(ci + e);
        a[u] = ldg2(v + e);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const int32_t e = cb + 32 * u + lane;
      if (e < ce) {
        int64_t sys = s0;
        for (int k = 0; k < nb && e >= s_sysbeg[k]; ++k) ++sys;
        s_p[slot_of<true>(e - cb)] = cmul_plain(a[u], ldg2(x + sys * n + c[u]));
      }
    }
    __syncwarp();
    const int32_t qa = max(p0, cb), qb = min(p1, ce);
    for (int32_t q = qa; q < qb; ++q) {
      const double2 pq = s_p[slot_of<true>(q - cb)];
      acc = (q == p0) ? pq : cadd(acc, pq);
    }
    __syncwarp();
  }
  if (have) y[row] = acc;
}

int launch_spmv(int64_t nrows, int32_t n, const int32_t* rp, const int32_t* ci,
                const double2* v, const double2* x, double2* y,
                cudaStream_t st) {
  if (nrows == 0) return RS_OK;
  RS_CHECK_ARG(n > 0, "n must be positive");
  // 8 warps x 32 rows per CTA; 4 chunks of 32 products per warp pass
  const unsigned grid = (unsigned)((nrows + 255) / 256);
  static const int variant = getenv("RHOSOLVE_SPMV_VARIANT") ? atoi(getenv("RHOSOLVE_SPMV_VARIANT")) : 0;
  switch (variant) {  // tuning hook (tools/spmv_c5.py); 0 = the measured best
    case 1: spmv_warp_kernel<4, 5><<<grid, 256, 0, st>>>(nrows, n, rp, ci, v, x, y); break;
    case 2: spmv_warp_kernel<4, 6><<<grid, 256, 0, st>>>(nrows, n, rp, ci, v, x, y); break;
    case 3: spmv_warp_kernel<2, 6><<<grid, 256, 0, st>>>(nrows, n, rp, ci, v, x, y); break;
    case 4: spmv_warp_kernel<2, 8><<<grid, 256, 0, st>>>(nrows, n, rp, ci, v, x, y); break;
    case 5: spmv_warp_kernel<8, 3><<<grid, 256, 0, st>>>(nrows, n, rp, ci, v, x, y); break;
    case 6: spmv_warp_kernel<8, 4><<<grid, 256, 0, st>>>(nrows, n, rp, ci, v, x, y); break;
    default: spmv_warp_kernel<4, 4><<<grid, 256, 0, st>>>(nrows, n, rp, ci, v, x, y); break;
  }
  ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

}  // namespace rs
