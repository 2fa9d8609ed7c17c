// Level analysis and the level-ordered SELL layout of the triangular factors
// for the grid-wide preconditioner apply (trisell.cuh, grid.cu).
//
// A sparse triangular solve in row form is a DAG: row i needs the results of
// the rows its off-diagonal columns name.  level(i) = 1 + max level of its
// dependencies.  The reference's column sweeps (_ckernels.pyx:53-85) fix only
// the order in which each y[i] receives its subtractions (ascending column
// for L, descending for U); rows of one level are independent, so they can be
// solved concurrently as long as every row folds its own terms in that order.
//
// Layout: rows sorted by (level, row), every level padded to a multiple of H
// rows (H = 32/G, G = lanes per row), so a warp always works on H rows of ONE
// level -- no lane ever waits on another lane of its warp.  Slice s holds
// sorted positions H*s .. H*s+H-1; lane (r*G + j) of the warp owns entries
// j, j+G, j+2G, ... of the slice's r-th row, in the reference fold order, and
// entry (k, lane) sits at sptr[s] + 32*k + lane: the k-th step of a slice is
// one coalesced 128-byte index line and four 128-byte value lines.  Padding
// has column -1.  Column indices are global over the block-diagonal batch
// (block b's column c is b*n + c), so block-Jacobi blocks need no special
// handling: their DAGs are simply disjoint.
#include <cub/cub.cuh>

#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace rs {

namespace {

inline unsigned grid_of(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Levels by Kahn's topological sweep over the raw CSC factor (column c lists
// the rows that depend on row c): one launch per level, the frontier of rows
// whose dependencies are all settled handed from launch to launch through two
// device buffers, so the work is O(nnz) plus one small launch per level and
// nothing ever spins.  (A first version propagated levels row by row with
// spinning warps: 31.7 s on config 5's 2.56M-row factor -- every waiting lane
// polling hammers L2 and starves the rows that could progress.)
__global__ void kahn_init_kernel(int64_t N, const int32_t* __restrict__ rp,
                                 int32_t* __restrict__ indeg, int32_t* __restrict__ frontier,
                                 int32_t* __restrict__ counts) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= N) return;
  const int32_t d = rp[g + 1] - rp[g];
  indeg[g] = d;
  if (d == 0) frontier[atomicAdd(counts, 1)] = (int32_t)g;
}

// one warp per frontier row
__global__ void __launch_bounds__(256) kahn_level_kernel(
    int32_t lev, int32_t n, int upper, const int32_t* __restrict__ cp,
    const int32_t* __restrict__ ri, int64_t cap, const int32_t* __restrict__ cur,
    int32_t* __restrict__ nxt, int32_t* counts, int32_t* indeg, int32_t* __restrict__ level,
    unsigned long long* processed) {
  const int32_t m = counts[lev];
  if (blockIdx.x == 0 && threadIdx.x == 0 && m > 0) atomicAdd(processed, (unsigned long long)m);
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; t < m; t += nw) {
    const int32_t g = cur[t];
    if (lane == 0) level[g] = lev;
    const int64_t b = g / n;
    const int32_t c = g - (int32_t)(b * n);
    const int32_t* col = cp + b * (n + 1);
    // L: skip the unit diagonal (first); U: skip the pivot (last)
    const int32_t p0 = upper ? col[c] : col[c] + 1;
    const int32_t p1 = upper ? col[c + 1] - 1 : col[c + 1];
    const int32_t* rows = ri + b * cap;
    for (int32_t p = p0 + lane; p < p1; p += 32) {
      const int32_t i = (int32_t)(b * n) + rows[p];
      if (atomicSub(indeg + i, 1) == 1) nxt[atomicAdd(counts + lev + 1, 1)] = i;
    }
  }
}

__global__ void level_hist_kernel(int64_t N, const int32_t* __restrict__ level,
                                  int32_t* __restrict__ hist) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < N) atomicAdd(hist + level[g], 1);
}

__global__ void level_pad_kernel(int64_t nlev, int32_t H, const int32_t* __restrict__ hist,
                                 int32_t* __restrict__ padded) {
  const int64_t l = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (l < nlev) padded[l] = (hist[l] + H - 1) / H * H;
}

// sort key (level, longest row first); value = row.  Rows of one level are
// independent, so their order is free: sorting them by length gives slices of
// uniform width (less padding, and most slices fit one register chunk).
__global__ void sort_keys_kernel(int64_t N, const int32_t* __restrict__ level,
                                 const int32_t* __restrict__ rp, unsigned long long* __restrict__ key,
                                 int32_t* __restrict__ v) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= N) return;
  const unsigned len = (unsigned)(rp[g + 1] - rp[g]);
  key[g] = ((unsigned long long)(unsigned)level[g] << 32) | (0xffffffffu - len);
  v[g] = (int32_t)g;
}

// sorted index k (rows sorted by level, ties by row) -> padded position
__global__ void level_place_kernel(int64_t N, const unsigned long long* __restrict__ key_sorted,
                                   const int32_t* __restrict__ row_sorted,
                                   const int32_t* __restrict__ off,
                                   const int32_t* __restrict__ poff,
                                   int32_t* __restrict__ order) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const int32_t l = (int32_t)(key_sorted[k] >> 32);
  order[poff[l] + ((int32_t)k - off[l])] = row_sorted[k];
}

__global__ void trisell_width_kernel(int64_t npos, int32_t H, const int32_t* __restrict__ order,
                                     const int32_t* __restrict__ rp,
                                     int32_t* __restrict__ width) {
  const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= npos) return;
  const int32_t g = order[pos];
  if (g < 0) return;
  const int32_t G = 32 / H;
  const int32_t len = rp[g + 1] - rp[g];
  atomicMax(width + pos / H, 32 * ((len + G - 1) / G));
}

// The dependency of the highest level per CHUNK of KCH steps of every slice
// (packed level:column, max): what the slice's warp watches before it touches
// that chunk's sources.  Chunk j of slice s has index (sptr[s]/32)/KCH + s + j.
constexpr int KCH = 8;  // = tri::KREG (trisell.cuh)
__global__ void trisell_key_kernel(int64_t npos, int32_t n, int32_t H, int upper,
                                   const int32_t* __restrict__ order,
                                   const int32_t* __restrict__ rp,
                                   const int32_t* __restrict__ ci,
                                   const int32_t* __restrict__ level,
                                   const int32_t* __restrict__ sptr,
                                   unsigned long long* __restrict__ best) {
  const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= npos) return;
  const int32_t g = order[pos];
  if (g < 0) return;
  const int32_t G = 32 / H;
  const int64_t s = pos / H;
  const int64_t cbase = (sptr[s] >> 5) / KCH + s;
  const int32_t cb = (g / n) * n;
  const int32_t e0 = rp[g], len = rp[g + 1] - e0;
  for (int32_t e = 0; e < len; ++e) {  // e-th term in fold order
    const int32_t src = upper ? e0 + len - 1 - e : e0 + e;
    const int32_t c = cb + ci[src];
    const unsigned long long k = ((unsigned long long)(unsigned)(level[c] + 1) << 32) | (unsigned)c;
    atomicMax(best + cbase + (e / G) / KCH, k);
  }
}
__global__ void trisell_key_out_kernel(int64_t nkeys, const unsigned long long* __restrict__ best,
                                       int32_t* __restrict__ skey) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s < nkeys) skey[s] = best[s] ? (int32_t)(best[s] & 0xffffffffu) : -1;
}

// one thread per (slice, lane)
__global__ void trisell_fill_kernel(int64_t nslices, int32_t n, int32_t H, int upper,
                                    const int32_t* __restrict__ order,
                                    const int32_t* __restrict__ rp,
                                    const int32_t* __restrict__ ci,
                                    const double2* __restrict__ v,
                                    const int32_t* __restrict__ sptr, int32_t* __restrict__ sci,
                                    double2* __restrict__ sv) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nslices * 32) return;
  const int64_t s = t >> 5;
  const int32_t lane = (int32_t)(t & 31);
  const int32_t G = 32 / H;
  const int32_t r = lane / G, j = lane % G;
  const int32_t p0 = sptr[s];
  const int32_t w = (sptr[s + 1] - p0) >> 5;
  const int32_t g = order[s * H + r];
  int32_t len = 0, e0 = 0, cb = 0;
  if (g >= 0) {
    e0 = rp[g];
    len = rp[g + 1] - e0;
    cb = (g / n) * n;  // block base of the global column index
  }
  for (int32_t k = 0; k < w; ++k) {
    const int32_t o = p0 + 32 * k + lane;
    const int32_t e = k * G + j;
    if (e < len) {
      const int32_t src = upper ? e0 + len - 1 - e : e0 + e;
      sci[o] = cb + ci[src];
      sv[o] = v[src];
    } else {
      sci[o] = -1;
      sv[o] = make_double2(0.0, 0.0);
    }
  }
}

}  // namespace

int tri_levels(int B, int32_t n, int upper, const int32_t* rp, const int32_t* cp,
               const int32_t* ri, int64_t cap, int32_t* level, int64_t* nlev_host,
               cudaStream_t st) {
  const int64_t N = (int64_t)B * n;
  *nlev_host = 0;
  if (N == 0) return RS_OK;
  int32_t *indeg = nullptr, *fr = nullptr, *counts = nullptr;
  unsigned long long* processed = nullptr;
  auto cleanup = [&]() {
    for (void* p : {(void*)indeg, (void*)fr, (void*)counts, (void*)processed})
      if (p) cudaFreeAsync(p, st);
  };
#define LV_TRY(expr)                                                        \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) {                                                \
      ::rs::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,            \
                      cudaGetErrorString(_e));                              \
      cleanup();                                                            \
      return RS_ERR_CUDA;                                                   \
    }                                                                       \
  } while (0)
  LV_TRY(cudaMallocAsync(&indeg, sizeof(int32_t) * N, st));
  LV_TRY(cudaMallocAsync(&fr, sizeof(int32_t) * 2 * N, st));
  LV_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (N + 2), st));
  LV_TRY(cudaMallocAsync(&processed, sizeof(unsigned long long), st));
  LV_TRY(cudaMemsetAsync(counts, 0, sizeof(int32_t) * (N + 2), st));
  LV_TRY(cudaMemsetAsync(processed, 0, sizeof(unsigned long long), st));
  kahn_init_kernel<<<grid_of(N, 256), 256, 0, st>>>(N, rp, indeg, fr, counts);
  count_launch();
  int dev = 0, sms = 0;
  LV_TRY(cudaGetDevice(&dev));
  LV_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid = (unsigned)(4 * sms);
  int64_t lev = 0;
  unsigned long long done = 0;
  while (done < (unsigned long long)N && lev <= N) {
    for (int k = 0; k < 64 && lev <= N; ++k, ++lev) {
      kahn_level_kernel<<<grid, 256, 0, st>>>((int32_t)lev, n, upper, cp, ri, cap,
                                              fr + (lev & 1) * N, fr + ((lev + 1) & 1) * N, counts,
                                              indeg, level, processed);
      count_launch();
    }
    LV_TRY(cudaGetLastError());
    LV_TRY(cudaMemcpyAsync(&done, processed, sizeof(done), cudaMemcpyDeviceToHost, st));
    LV_TRY(cudaStreamSynchronize(st));
  }
  if (done != (unsigned long long)N) {
    cleanup();
    set_error("tri_levels: dependency structure is not triangular");
    return RS_ERR_ARG;
  }
  // number of levels = leading non-empty frontiers
  std::vector<int32_t> h((size_t)lev);
  LV_TRY(cudaMemcpyAsync(h.data(), counts, sizeof(int32_t) * (size_t)lev, cudaMemcpyDeviceToHost,
                         st));
  LV_TRY(cudaStreamSynchronize(st));
#undef LV_TRY
  int64_t nl = 0;
  while (nl < lev && h[(size_t)nl] > 0) ++nl;
  cleanup();
  *nlev_host = nl;
  return RS_OK;
}

// order[pos] = global row (or -1) with every level padded to a multiple of H.
// order must hold N + H * nlev entries; *npos_host = positions used.
int tri_order(int B, int32_t n, const int32_t* level, const int32_t* rp, int64_t nlev, int32_t H,
              int32_t* order, int64_t* npos_host, cudaStream_t st) {
  const int64_t N = (int64_t)B * n;
  *npos_host = 0;
  if (N == 0 || nlev == 0) return RS_OK;
  int32_t *hist = nullptr, *padded = nullptr, *off = nullptr, *poff = nullptr, *rows = nullptr,
          *rows_in = nullptr;
  unsigned long long *keys = nullptr, *keys_in = nullptr;
  void* tmp = nullptr;
  auto cleanup = [&]() {
    for (void* p : {(void*)hist, (void*)padded, (void*)off, (void*)poff, (void*)keys,
                    (void*)keys_in, (void*)rows, (void*)rows_in, tmp})
      if (p) cudaFreeAsync(p, st);
  };
#define LV_TRY(expr)                                                        \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) {                                                \
      ::rs::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,            \
                      cudaGetErrorString(_e));                              \
      cleanup();                                                            \
      return RS_ERR_CUDA;                                                   \
    }                                                                       \
  } while (0)
  LV_TRY(cudaMallocAsync(&hist, sizeof(int32_t) * nlev, st));
  LV_TRY(cudaMallocAsync(&padded, sizeof(int32_t) * nlev, st));
  LV_TRY(cudaMallocAsync(&off, sizeof(int32_t) * (nlev + 1), st));
  LV_TRY(cudaMallocAsync(&poff, sizeof(int32_t) * (nlev + 1), st));
  LV_TRY(cudaMallocAsync(&keys, sizeof(unsigned long long) * N, st));
  LV_TRY(cudaMallocAsync(&keys_in, sizeof(unsigned long long) * N, st));
  LV_TRY(cudaMallocAsync(&rows, sizeof(int32_t) * N, st));
  LV_TRY(cudaMallocAsync(&rows_in, sizeof(int32_t) * N, st));
  LV_TRY(cudaMemsetAsync(hist, 0, sizeof(int32_t) * nlev, st));
  level_hist_kernel<<<grid_of(N, 256), 256, 0, st>>>(N, level, hist);
  count_launch();
  level_pad_kernel<<<grid_of(nlev, 256), 256, 0, st>>>(nlev, H, hist, padded);
  count_launch();
  int rc = scan_counts(hist, off, nlev, nullptr, st);
  int64_t npos = 0;
  if (!rc) rc = scan_counts(padded, poff, nlev, &npos, st);
  if (rc) {
    cleanup();
    return rc;
  }
  // stable sort of the rows by (level, longest first); ties keep ascending rows
  sort_keys_kernel<<<grid_of(N, 256), 256, 0, st>>>(N, level, rp, keys_in, rows_in);
  count_launch();
  int bits = 1;
  while (((int64_t)1 << bits) < nlev) ++bits;
  size_t tmp_bytes = 0;
  LV_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, keys_in, keys, rows_in, rows, (int)N,
                                         0, 32 + bits, st));
  LV_TRY(cudaMallocAsync(&tmp, tmp_bytes, st));
  LV_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, keys_in, keys, rows_in, rows, (int)N, 0,
                                         32 + bits, st));
  LV_TRY(cudaMemsetAsync(order, 0xff, sizeof(int32_t) * npos, st));
  level_place_kernel<<<grid_of(N, 256), 256, 0, st>>>(N, keys, rows, off, poff, order);
  count_launch();
  LV_TRY(cudaGetLastError());
#undef LV_TRY
  cleanup();
  *npos_host = npos;
  return RS_OK;
}

// entries of the per-chunk key array for `total` padded entries in `nslices` slices
int64_t tri_sell_keys(int64_t total, int64_t nslices) { return (total >> 5) / KCH + nslices + 1; }

// Pass 1 (sci == null): sptr[npos/H + 1] and *total (padded entries, host).
// Pass 2 (*total as returned by pass 1): fill sci / sv / skey[tri_sell_keys()].
int tri_sell(int B, int32_t n, int upper, const int32_t* rp, const int32_t* ci, const double2* v,
             const int32_t* order, int64_t npos, int32_t H, const int32_t* level, int32_t* sptr,
             int32_t* sci, double2* sv, int32_t* skey, int64_t* total, cudaStream_t st) {
  const int64_t nslices = npos / H;
  if (!sci) {
    int32_t* width = nullptr;
    RS_CUDA_TRY(cudaMallocAsync(&width, sizeof(int32_t) * (nslices + 1), st));
    RS_CUDA_TRY(cudaMemsetAsync(width, 0, sizeof(int32_t) * (nslices + 1), st));
    if (npos > 0) {
      trisell_width_kernel<<<grid_of(npos, 256), 256, 0, st>>>(npos, H, order, rp, width);
      count_launch();
    }
    int64_t tot = 0;
    const int rc = scan_counts(width, sptr, nslices, &tot, st);
    cudaFreeAsync(width, st);
    if (rc) return rc;
    if (tot < 0 || tot >= ((int64_t)1 << 31)) {
      set_error("tri_sell: %lld padded entries exceed int32 indexing", (long long)tot);
      return RS_ERR_OVERFLOW;
    }
    if (total) *total = tot;
    return RS_OK;
  }
  if (nslices > 0) {
    trisell_fill_kernel<<<grid_of(nslices * 32, 256), 256, 0, st>>>(nslices, n, H, upper, order,
                                                                    rp, ci, v, sptr, sci, sv);
    count_launch();
    if (skey) {  // per chunk: the latest dependency, what the slice's warp watches
      const int64_t nkeys = tri_sell_keys(total ? *total : 0, nslices);
      unsigned long long* best = nullptr;
      RS_CUDA_TRY(cudaMallocAsync(&best, sizeof(unsigned long long) * nkeys, st));
      RS_CUDA_TRY(cudaMemsetAsync(best, 0, sizeof(unsigned long long) * nkeys, st));
      trisell_key_kernel<<<grid_of(npos, 256), 256, 0, st>>>(npos, n, H, upper, order, rp, ci,
                                                             level, sptr, best);
      count_launch();
      trisell_key_out_kernel<<<grid_of(nkeys, 256), 256, 0, st>>>(nkeys, best, skey);
      count_launch();
      cudaFreeAsync(best, st);
    }
    RS_CUDA_TRY(cudaGetLastError());
  }
  return RS_OK;
}

}  // namespace rs
