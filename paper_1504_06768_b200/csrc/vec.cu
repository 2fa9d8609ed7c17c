// Grid-wide vector kernels for the large-system (multi-kernel) solver path
// -- config 5, n = 2.56M, where one CTA per system is far too little:
//   * deterministic multi-pair vdot / squared norms / max-abs: a fixed grid
//     of per-CTA partials (fixed thread->element map, shuffle tree, fixed
//     cross-warp order) reduced by one CTA in fixed order, so results are
//     bitwise reproducible run to run;
//   * fused linear combinations out = sum_k c_k v_k (k <= 4) with host
//     complex coefficients -- one HBM pass per BiCGStab update;
//   * block-diagonal extraction (block-Jacobi preconditioner blocks).
#include "common.cuh"
#include "kernels.cuh"

namespace rs {

constexpr int RED_BLOCKS = 592;  // 4 x 148 SMs
constexpr int RED_THREADS = 256;

struct VecPairs {
  const double2* x[4];
  const double2* y[4];
};

// partial[b*(2*np) + 2k + {0,1}] = sum over this CTA's elements of conj(x_k) y_k
__global__ void __launch_bounds__(RED_THREADS) vdot_partial_kernel(int64_t n, int np,
                                                                   VecPairs P, double* partial) {
  __shared__ double red[8][2 * 4];
  double acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < np) {
        const double2 a = P.x[k][i], b = P.y[k][i];
        acc[2 * k] = __fma_rn(a.x, b.x, __fma_rn(a.y, b.y, acc[2 * k]));
        acc[2 * k + 1] = __fma_rn(a.x, b.y, __fma_rn(-a.y, b.x, acc[2 * k + 1]));
      }
    }
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 8; ++k)
    for (int o = 16; o; o >>= 1) acc[k] = __dadd_rn(acc[k], __shfl_xor_sync(0xffffffffu, acc[k], o));
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 8; ++k) red[wid][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < 2 * np) {
    double s = red[0][threadIdx.x];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) s = __dadd_rn(s, red[w][threadIdx.x]);
    partial[(int64_t)blockIdx.x * (2 * np) + threadIdx.x] = s;
  }
}

__global__ void sum_partials_kernel(int nparts, int width, const double* partial, double* out) {
  const int k = threadIdx.x;
  if (k >= width) return;
  double s = 0.0;
  for (int b = 0; b < nparts; ++b) s = __dadd_rn(s, partial[(int64_t)b * width + k]);
  out[k] = s;
}

int vec_vdots(int64_t n, int np, const double2* const* xs, const double2* const* ys, double* out,
              double* scratch, cudaStream_t st) {
  if (np < 1 || np > 4) {
    set_error("vdots: 1..4 pairs supported");
    return RS_ERR_ARG;
  }
  VecPairs P{};
  for (int k = 0; k < np; ++k) {
    P.x[k] = xs[k];
    P.y[k] = ys[k];
  }
  vdot_partial_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, np, P, scratch); ::rs::count_launch();
  sum_partials_kernel<<<1, 32, 0, st>>>(RED_BLOCKS, 2 * np, scratch, out); ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

__global__ void __launch_bounds__(RED_THREADS) amax_partial_kernel(int64_t n, const double2* x,
                                                                   double* partial) {
  __shared__ double red[8];
  double m = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, hypot(x[i].x, x[i].y));
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) s = fmax(s, red[w]);
    partial[blockIdx.x] = s;
  }
}

__global__ void max_partials_kernel(int nparts, const double* partial, double* out) {
  __shared__ double red[32];
  double m = 0.0;
  for (int b = threadIdx.x; b < nparts; b += blockDim.x) m = fmax(m, partial[b]);
  for (int o = 16; o; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = red[0];
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) s = fmax(s, red[w]);
    out[0] = s;
  }
}

int vec_amax(int64_t n, const double2* x, double* out, double* scratch, cudaStream_t st) {
  amax_partial_kernel<<<RED_BLOCKS, RED_THREADS, 0, st>>>(n, x, scratch); ::rs::count_launch();
  max_partials_kernel<<<1, 256, 0, st>>>(RED_BLOCKS, scratch, out); ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

struct Lin {
  const double2* v[4];
  double2 c[4];
};

// out = sum_{k<nv} c_k * v_k  (out may alias any v_k)
__global__ void lincomb_kernel(int64_t n, int nv, Lin L, double2* out) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (k < nv) {
        const double2 a = L.c[k], b = L.v[k][i];
        acc.x += a.x * b.x - a.y * b.y;
        acc.y += a.x * b.y + a.y * b.x;
      }
    }
    out[i] = acc;
  }
}

int vec_lincomb(int64_t n, int nv, const double2* const* vs, const double* coef_re,
                const double* coef_im, double2* out, cudaStream_t st) {
  if (nv < 1 || nv > 4) {
    set_error("lincomb: 1..4 vectors supported");
    return RS_ERR_ARG;
  }
  Lin L{};
  for (int k = 0; k < nv; ++k) {
    L.v[k] = vs[k];
    L.c[k] = make_double2(coef_re[k], coef_im[k]);
  }
  const int64_t want = (n + 255) / 256;
  const unsigned grid = (unsigned)(want < 148 * 16 ? want : 148 * 16);
  if (n > 0) {
    lincomb_kernel<<<grid, 256, 0, st>>>(n, nv, L, out); ::rs::count_launch();
  }
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

// ---- block-diagonal extraction --------------------------------------------
// Rows [g*m, (g+1)*m) of an nrows x ncols CSR (columns offset by col0), kept
// entries with columns in the same block, re-indexed locally: the nblk
// diagonal blocks of size m as a block-diagonal batch (block-Jacobi).
template <bool FILL>
__global__ void block_extract_kernel(int64_t nrows, int32_t m, int32_t col0, const int32_t* rp,
                                     const int32_t* ci, const double2* v, int32_t* counts,
                                     const int32_t* out_rp, int32_t* out_ci, double2* out_v) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int32_t lo = (int32_t)((r / m) * m), hi = lo + m;
  int32_t cnt = 0;
  int32_t o = FILL ? out_rp[r] : 0;
  for (int32_t p = rp[r]; p < rp[r + 1]; ++p) {
    const int32_t c = ci[p] - col0;
    if (c >= lo && c < hi) {
      if (FILL) {
        out_ci[o] = c - lo;
        out_v[o] = v[p];
        ++o;
      }
      ++cnt;
    }
  }
  if (!FILL) counts[r] = cnt;
}

int block_extract(int64_t nrows, int32_t m, int32_t col0, const int32_t* rp, const int32_t* ci,
                  const double2* v, int32_t* out_rp, int32_t* out_ci, double2* out_v,
                  int64_t* nnz_out, cudaStream_t st) {
  if (nrows % m) {
    set_error("block size %d does not divide %lld rows", m, (long long)nrows);
    return RS_ERR_ARG;
  }
  const unsigned grid = (unsigned)((nrows + 255) / 256);
  if (!out_ci) {
    int32_t* counts = nullptr;
    RS_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (nrows + 1), st));
    block_extract_kernel<false><<<grid, 256, 0, st>>>(nrows, m, col0, rp, ci, v, counts, nullptr,
                                                      nullptr, nullptr); ::rs::count_launch();
    const int rc = scan_counts(counts, out_rp, nrows, nnz_out, st);
    cudaFreeAsync(counts, st);
    return rc;
  }
  block_extract_kernel<true><<<grid, 256, 0, st>>>(nrows, m, col0, rp, ci, v, nullptr, out_rp,
                                                   out_ci, out_v); ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

}  // namespace rs
