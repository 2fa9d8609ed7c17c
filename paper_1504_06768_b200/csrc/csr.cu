// Structure-changing CSR kernels: scans, stable transpose, symmetric
// permutation, the shifted / trace-modified variants, row norms and the
// CSC-factor -> row-oriented CSR conversion used by the triangular solves.
//
// All kernels take a block-diagonal batch of B systems of size n: row_ptr is
// global over B*n rows (absolute positions), column indices are local to the
// system.  B = 1 is a single system.
#include <cub/cub.cuh>

#include "common.cuh"
#include "kernels.cuh"

namespace rs {

// ---------------------------------------------------------------- scans ----
int scan_counts(const int32_t* counts, int32_t* offsets, int64_t n,
                int64_t* total_host, cudaStream_t st) {
  // offsets[0] = 0, offsets[i+1] = sum(counts[0..i])
  RS_CUDA_TRY(cudaMemsetAsync(offsets, 0, sizeof(int32_t), st));
  if (n > 0) {
    size_t tmp_bytes = 0;
    RS_CUDA_TRY(cub::DeviceScan::InclusiveSum(nullptr, tmp_bytes, counts, offsets + 1,
                                              (int)n, st));
    void* tmp = nullptr;
    RS_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, st));
    cudaError_t e = cub::DeviceScan::InclusiveSum(tmp, tmp_bytes, counts, offsets + 1,
                                                  (int)n, st);
    cudaFreeAsync(tmp, st);
    RS_CUDA_TRY(e);
  }
  if (total_host) {
    int32_t t = 0;
    RS_CUDA_TRY(cudaMemcpyAsync(&t, offsets + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    RS_CUDA_TRY(cudaStreamSynchronize(st));
    *total_host = t;
  }
  return RS_OK;
}

// ------------------------------------------------------------ transpose ----
__global__ void expand_rows_kernel(int64_t nrows, const int32_t* rp, int32_t* rowid) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  for (int32_t p = rp[r]; p < rp[r + 1]; ++p) rowid[p] = (int32_t)r;
}

__global__ void transpose_keys_kernel(int64_t nnz, int32_t n, const int32_t* rowid,
                                      const int32_t* ci, int32_t* key, int32_t* idx,
                                      int32_t* counts) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= nnz) return;
  const int32_t r = rowid[p];
  const int32_t b = r / n;
  const int32_t k = b * n + ci[p];  // global output row
  key[p] = k;
  idx[p] = (int32_t)p;
  atomicAdd(counts + k, 1);
}

__global__ void transpose_gather_kernel(int64_t nnz, int32_t n, const int32_t* sorted_idx,
                                       const int32_t* rowid, const double2* v,
                                       int32_t* out_ci, double2* out_v) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nnz) return;
  const int32_t p = sorted_idx[q];
  out_ci[q] = rowid[p] % n;
  if (out_v) out_v[q] = v[p];
}

static inline unsigned grid_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

int csr_transpose(int B, int32_t n, const int32_t* rp, const int32_t* ci, const double2* v,
                  int32_t* out_rp, int32_t* out_ci, double2* out_v, cudaStream_t st) {
  const int64_t nrows = (int64_t)B * n;
  int32_t nnz32 = 0;
  RS_CUDA_TRY(cudaMemcpyAsync(&nnz32, rp + nrows, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RS_CUDA_TRY(cudaStreamSynchronize(st));
  const int64_t nnz = nnz32;
  int32_t *rowid = nullptr, *key = nullptr, *idx = nullptr, *key2 = nullptr, *idx2 = nullptr,
          *counts = nullptr;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  int rc = RS_OK;
  RS_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (nrows + 1), st));
  RS_CUDA_TRY(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (nrows + 1), st));
  if (nnz > 0) {
    RS_CUDA_TRY(cudaMallocAsync(&rowid, sizeof(int32_t) * nnz, st));
    RS_CUDA_TRY(cudaMallocAsync(&key, sizeof(int32_t) * nnz, st));
    RS_CUDA_TRY(cudaMallocAsync(&idx, sizeof(int32_t) * nnz, st));
    RS_CUDA_TRY(cudaMallocAsync(&key2, sizeof(int32_t) * nnz, st));
    RS_CUDA_TRY(cudaMallocAsync(&idx2, sizeof(int32_t) * nnz, st));
    expand_rows_kernel<<<grid_for(nrows, 256), 256, 0, st>>>(nrows, rp, rowid); ::rs::count_launch();
    transpose_keys_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(nnz, n, rowid, ci, key, idx,
                                                              counts); ::rs::count_launch();
    int end_bit = 1;
    while (end_bit < 31 && ((int64_t)1 << end_bit) < nrows) ++end_bit;
    RS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key, key2, idx, idx2,
                                                (int)nnz, 0, end_bit, st));
    RS_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, st));
    RS_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key2, idx, idx2,
                                                (int)nnz, 0, end_bit, st));
    transpose_gather_kernel<<<grid_for(nnz, 256), 256, 0, st>>>(nnz, n, idx2, rowid, v,
                                                                out_ci, out_v); ::rs::count_launch();
  }
  rc = scan_counts(counts, out_rp, nrows, nullptr, st);
  cudaFreeAsync(counts, st);
  if (nnz > 0) {
    cudaFreeAsync(rowid, st);
    cudaFreeAsync(key, st);
    cudaFreeAsync(idx, st);
    cudaFreeAsync(key2, st);
    cudaFreeAsync(idx2, st);
    cudaFreeAsync(tmp, st);
  }
  RS_CUDA_TRY(cudaGetLastError());
  return rc;
}

// -------------------------------------------------------------- permute ----
// B[f[i], f[j]] = A[i, j]  (sparse.permute, sparse.py:276-282).  inv = f^-1.
__global__ void permute_count_kernel(int64_t nrows, int32_t n, const int32_t* rp,
                                     const int32_t* inv, int32_t* counts) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int64_t b = r / n;
  const int64_t src = b * n + inv[r];
  counts[r] = rp[src + 1] - rp[src];
}

__global__ void permute_fill_kernel(int64_t nrows, int32_t n, const int32_t* rp,
                                    const int32_t* ci, const double2* v, const int32_t* fwd,
                                    const int32_t* inv, const int32_t* out_rp,
                                    int32_t* out_ci, double2* out_v) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int64_t b = r / n;
  const int32_t* f = fwd + b * n;
  const int64_t src = b * n + inv[r];
  const int32_t p0 = rp[src], p1 = rp[src + 1];
  const int32_t o = out_rp[r];
  // insertion sort by new column while copying (rows are short; the trace
  // row of the modified variant is the only long one)
  for (int32_t p = p0; p < p1; ++p) {
    const int32_t c = f[ci[p]];
    const double2 val = v[p];
    int32_t q = o + (p - p0);
    while (q > o && out_ci[q - 1] > c) {
      out_ci[q] = out_ci[q - 1];
      out_v[q] = out_v[q - 1];
      --q;
    }
    out_ci[q] = c;
    out_v[q] = val;
  }
}

int csr_permute(int B, int32_t n, const int32_t* rp, const int32_t* ci, const double2* v,
                const int32_t* fwd, const int32_t* inv, int32_t* out_rp, int32_t* out_ci,
                double2* out_v, cudaStream_t st) {
  const int64_t nrows = (int64_t)B * n;
  int32_t* counts = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (nrows + 1), st));
  permute_count_kernel<<<grid_for(nrows, 256), 256, 0, st>>>(nrows, n, rp, inv, counts); ::rs::count_launch();
  int rc = scan_counts(counts, out_rp, nrows, nullptr, st);
  cudaFreeAsync(counts, st);
  if (rc) return rc;
  permute_fill_kernel<<<grid_for(nrows, 128), 128, 0, st>>>(nrows, n, rp, ci, v, fwd, inv,
                                                            out_rp, out_ci, out_v); ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

// ---------------------------------------------------------------- shift ----
// L - sigma I with every diagonal stored (liouville.shift, liouville.py:80-96):
// from_coo(prune=False) sums the existing L_ii (first) with -sigma.
__global__ void shift_count_kernel(int64_t nrows, int32_t n, const int32_t* rp,
                                   const int32_t* ci, int32_t* counts) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int32_t d = (int32_t)(r % n);
  bool has = false;
  for (int32_t p = rp[r]; p < rp[r + 1]; ++p) has |= (ci[p] == d);
  counts[r] = rp[r + 1] - rp[r] + (has ? 0 : 1);
}

__global__ void shift_fill_kernel(int64_t nrows, int32_t n, const int32_t* rp,
                                  const int32_t* ci, const double2* v, double sigma,
                                  const int32_t* out_rp, int32_t* out_ci, double2* out_v) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int32_t d = (int32_t)(r % n);
  const double2 ms = make_double2(-sigma, 0.0);
  int32_t o = out_rp[r];
  bool placed = false;
  for (int32_t p = rp[r]; p < rp[r + 1]; ++p) {
    const int32_t c = ci[p];
    if (!placed && c > d) {
      out_ci[o] = d;
      out_v[o] = ms;
      ++o;
      placed = true;
    }
    if (c == d) {
      out_ci[o] = c;
      out_v[o] = cadd(v[p], ms);
      placed = true;
    } else {
      out_ci[o] = c;
      out_v[o] = v[p];
    }
    ++o;
  }
  if (!placed) {
    out_ci[o] = d;
    out_v[o] = ms;
  }
}

int csr_shift(int B, int32_t n, const int32_t* rp, const int32_t* ci, const double2* v,
              double sigma, int32_t* out_rp, int32_t* out_ci, double2* out_v,
              int64_t* nnz_out, cudaStream_t st) {
  const int64_t nrows = (int64_t)B * n;
  int32_t* counts = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (nrows + 1), st));
  shift_count_kernel<<<grid_for(nrows, 256), 256, 0, st>>>(nrows, n, rp, ci, counts); ::rs::count_launch();
  int rc = scan_counts(counts, out_rp, nrows, nnz_out, st);
  cudaFreeAsync(counts, st);
  if (rc || !out_ci) return rc;
  shift_fill_kernel<<<grid_for(nrows, 256), 256, 0, st>>>(nrows, n, rp, ci, v, sigma, out_rp,
                                                          out_ci, out_v); ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

// ------------------------------------------------------- trace modified ----
// Row 0 += w at columns k(D+1) (liouville.build_modified, liouville.py:114-138;
// from_coo(prune=False) adds L[0,c] (first) + w).
__global__ void modify_count_kernel(int64_t nrows, int32_t n, int32_t D, const int32_t* rp,
                                    const int32_t* ci, int32_t* counts) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int32_t cnt = rp[r + 1] - rp[r];
  if (r % n == 0) {
    // merge count: trace columns not already present
    int32_t missing = D;
    for (int32_t p = rp[r]; p < rp[r + 1]; ++p) {
      const int32_t c = ci[p];
      if (c % (D + 1) == 0 && c / (D + 1) < D) --missing;
    }
    cnt += missing;
  }
  counts[r] = cnt;
}

__global__ void modify_fill_kernel(int64_t nrows, int32_t n, int32_t D, const int32_t* rp,
                                   const int32_t* ci, const double2* v, const double* w,
                                   const int32_t* out_rp, int32_t* out_ci, double2* out_v) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int32_t o = out_rp[r];
  const int32_t p0 = rp[r], p1 = rp[r + 1];
  if (r % n != 0) {
    for (int32_t p = p0; p < p1; ++p, ++o) {
      out_ci[o] = ci[p];
      out_v[o] = v[p];
    }
    return;
  }
  const double2 wv = make_double2(w[r / n], 0.0);
  int32_t p = p0;
  for (int32_t k = 0; k < D; ++k) {
    const int32_t tc = k * (D + 1);
    while (p < p1 && ci[p] < tc) {
      out_ci[o] = ci[p];
      out_v[o] = v[p];
      ++o;
      ++p;
    }
    if (p < p1 && ci[p] == tc) {
      out_ci[o] = tc;
      out_v[o] = cadd(v[p], wv);
      ++p;
    } else {
      out_ci[o] = tc;
      out_v[o] = wv;
    }
    ++o;
  }
  for (; p < p1; ++p, ++o) {
    out_ci[o] = ci[p];
    out_v[o] = v[p];
  }
}

int csr_modify(int B, int32_t n, int32_t D, const int32_t* rp, const int32_t* ci,
               const double2* v, const double* w, int32_t* out_rp, int32_t* out_ci,
               double2* out_v, int64_t* nnz_out, cudaStream_t st) {
  const int64_t nrows = (int64_t)B * n;
  int32_t* counts = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (nrows + 1), st));
  modify_count_kernel<<<grid_for(nrows, 256), 256, 0, st>>>(nrows, n, D, rp, ci, counts); ::rs::count_launch();
  int rc = scan_counts(counts, out_rp, nrows, nnz_out, st);
  cudaFreeAsync(counts, st);
  if (rc || !out_ci) return rc;
  modify_fill_kernel<<<grid_for(nrows, 256), 256, 0, st>>>(nrows, n, D, rp, ci, v, w, out_rp,
                                                           out_ci, out_v); ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

// default_weight (liouville.py:99-111): mean |L_ii| over the plain diagonal
// ("abs") or |mean L_ii| ("signed"), one CTA per system, fixed order.
__global__ void default_weight_kernel(int32_t n, const int32_t* rp, const int32_t* ci,
                                      const double2* v, int signed_mode, double* w) {
  __shared__ double red[2][32];
  const int b = blockIdx.x;
  double a0 = 0.0, a1 = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const int64_t r = (int64_t)b * n + i;
    double2 d = make_double2(0.0, 0.0);
    for (int32_t p = rp[r]; p < rp[r + 1]; ++p)
      if (ci[p] == i) d = v[p];
    if (signed_mode) {
      a0 += d.x;
      a1 += d.y;
    } else {
      a0 += hypot(d.x, d.y);
    }
  }
  for (int o = 16; o; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = a0;
    red[1][threadIdx.x >> 5] = a1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) {
      s0 += red[0][k];
      s1 += red[1][k];
    }
    w[b] = signed_mode ? hypot(s0 / n, s1 / n) : s0 / n;
  }
}

int csr_default_weight(int B, int32_t n, const int32_t* rp, const int32_t* ci,
                       const double2* v, int signed_mode, double* w, cudaStream_t st) {
  default_weight_kernel<<<B, 256, 0, st>>>(n, rp, ci, v, signed_mode, w); ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

// ------------------------------------------------------------ row norms ----
// factor.py:84-88: per-row max of |re|+|im|.
__global__ void row_norms_kernel(int64_t nrows, const int32_t* rp, const double2* v,
                                 double* rn) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  double m = 0.0;
  for (int32_t p = rp[r]; p < rp[r + 1]; ++p) m = fmax(m, cabs1(v[p]));
  rn[r] = m;
}

int csr_row_norms(int64_t nrows, const int32_t* rp, const double2* v, double* rn,
                  cudaStream_t st) {
  if (nrows == 0) return RS_OK;
  row_norms_kernel<<<grid_for(nrows, 256), 256, 0, st>>>(nrows, rp, v, rn); ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

// ---------------------------------------------- factor CSC -> solve CSR ----
// Per-system CSC columns (Lp/Li/Lx at offset b*cap) -> a block-diagonal
// "column-major" CSR of the factor transpose without the stored diagonals:
// L drops its leading unit diagonal, U its trailing pivot (whose recipc goes
// to rU).  A transpose then yields the row-oriented factors.
__global__ void factor_strip_count_kernel(int B, int32_t n, const int32_t* cp, int64_t cap,
                                          int lower, int32_t* counts) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= (int64_t)B * n) return;
  const int64_t b = r / n, k = r % n;
  const int32_t* p = cp + b * (n + 1);
  counts[r] = p[k + 1] - p[k] - 1;
  (void)cap;
  (void)lower;
}

// one warp per factor column: coalesced copy of its off-diagonal entries
__global__ void factor_strip_fill_kernel(int B, int32_t n, const int32_t* cp,
                                         const int32_t* ri, const double2* rv, int64_t cap,
                                         int lower, const int32_t* out_rp, int32_t* out_ci,
                                         double2* out_v, double2* rU) {
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r >= (int64_t)B * n) return;
  const int64_t b = r / n, k = r % n;
  const int32_t* p = cp + b * (n + 1);
  const int32_t* I = ri + b * cap;
  const double2* X = rv + b * cap;
  const int32_t o = out_rp[r];
  const int32_t s = lower ? p[k] + 1 : p[k];
  const int32_t e = lower ? p[k + 1] : p[k + 1] - 1;
  for (int32_t q = s + lane; q < e; q += 32) {
    out_ci[o + (q - s)] = I[q];
    out_v[o + (q - s)] = X[q];
  }
  if (!lower && lane == 0) rU[r] = recipc(X[p[k + 1] - 1]);
}

int factor_to_csr(int B, int32_t n, const int32_t* cp, const int32_t* ri, const double2* rv,
                  int64_t cap, int lower, int32_t* out_rp, int32_t* out_ci, double2* out_v,
                  double2* rU, int64_t* nnz_out, cudaStream_t st) {
  // pass 1 (out_ci == null): count only, returns nnz; pass 2: fill + transpose
  const int64_t nrows = (int64_t)B * n;
  int32_t* counts = nullptr;
  int32_t* crp = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (nrows + 1), st));
  RS_CUDA_TRY(cudaMallocAsync(&crp, sizeof(int32_t) * (nrows + 1), st));
  factor_strip_count_kernel<<<grid_for(nrows, 256), 256, 0, st>>>(B, n, cp, cap, lower, counts); ::rs::count_launch();
  int64_t nnz = 0;
  int rc = scan_counts(counts, crp, nrows, &nnz, st);
  cudaFreeAsync(counts, st);
  if (nnz_out) *nnz_out = nnz;
  if (rc || !out_ci) {
    cudaFreeAsync(crp, st);
    return rc;
  }
  int32_t* cci = nullptr;
  double2* cv = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&cci, sizeof(int32_t) * (nnz + 1), st));
  RS_CUDA_TRY(cudaMallocAsync(&cv, sizeof(double2) * (nnz + 1), st));
  factor_strip_fill_kernel<<<grid_for(nrows * 32, 256), 256, 0, st>>>(B, n, cp, ri, rv, cap,
                                                                      lower, crp, cci, cv, rU); ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  rc = csr_transpose(B, n, crp, cci, cv, out_rp, out_ci, out_v, st);
  cudaFreeAsync(crp, st);
  cudaFreeAsync(cci, st);
  cudaFreeAsync(cv, st);
  return rc;
}

}  // namespace rs
