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

#include "common.cuh"
#include "kernels.cuh"

namespace rs {

namespace {

inline unsigned grid_of(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

__device__ __forceinline__ int ld_lvl(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_lvl(int32_t* p, int v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Levels by propagation in sweep order.  Warps claim rows through a ticket
// (4 at a time), so a row only ever waits on rows claimed before it: no
// deadlock whatever the number of resident CTAs.  level[] starts at -1.
constexpr int CLAIM = 4;
__global__ void __launch_bounds__(256) tri_level_kernel(int64_t N, int32_t n, int upper,
                                                        const int32_t* __restrict__ rp,
                                                        const int32_t* __restrict__ ci,
                                                        int32_t* level,
                                                        unsigned long long* next) {
  const int lane = threadIdx.x & 31;
  while (true) {
    unsigned long long q0 = 0;
    if (lane == 0) q0 = atomicAdd(next, (unsigned long long)CLAIM);
    q0 = __shfl_sync(0xffffffffu, q0, 0);
    if (q0 >= (unsigned long long)N) break;
    const int64_t q1 = min((int64_t)q0 + CLAIM, N);
    for (int64_t q = (int64_t)q0; q < q1; ++q) {
      const int64_t b = q / n;
      const int32_t j = (int32_t)(q % n);
      const int64_t g = b * n + (upper ? n - 1 - j : j);
      const int32_t p0 = rp[g], p1 = rp[g + 1];
      int m = 0;
      for (int32_t p = p0 + lane; p < p1; p += 32) {
        const int32_t* d = level + b * n + ci[p];
        int lv;
        do {
          lv = ld_lvl(d);
        } while (lv < 0);
        m = max(m, lv + 1);
      }
      for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      if (lane == 0) st_lvl(level + g, m);
      __syncwarp();
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

__global__ void iota_kernel(int64_t N, int32_t* __restrict__ v) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < N) v[g] = (int32_t)g;
}

// sorted index k (rows sorted by level, ties by row) -> padded position
__global__ void level_place_kernel(int64_t N, const int32_t* __restrict__ lev_sorted,
                                   const int32_t* __restrict__ row_sorted,
                                   const int32_t* __restrict__ off,
                                   const int32_t* __restrict__ poff,
                                   int32_t* __restrict__ order) {
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= N) return;
  const int32_t l = lev_sorted[k];
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

int tri_levels(int B, int32_t n, int upper, const int32_t* rp, const int32_t* ci, int32_t* level,
               int64_t* nlev_host, cudaStream_t st) {
  const int64_t N = (int64_t)B * n;
  if (N == 0) {
    *nlev_host = 0;
    return RS_OK;
  }
  unsigned long long* next = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&next, 16, st));
  RS_CUDA_TRY(cudaMemsetAsync(next, 0, 16, st));
  RS_CUDA_TRY(cudaMemsetAsync(level, 0xff, sizeof(int32_t) * N, st));
  int dev = 0, sms = 0;
  RS_CUDA_TRY(cudaGetDevice(&dev));
  RS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const unsigned grid = (unsigned)std::min<int64_t>((N + 8 * CLAIM - 1) / (8 * CLAIM), 8 * sms);
  tri_level_kernel<<<grid, 256, 0, st>>>(N, n, upper, rp, ci, level, next);
  count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  // max level -> host
  int32_t* dmax = reinterpret_cast<int32_t*>(next + 1);
  size_t tmp_bytes = 0;
  RS_CUDA_TRY(cub::DeviceReduce::Max(nullptr, tmp_bytes, level, dmax, (int)N, st));
  void* tmp = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, st));
  cudaError_t e = cub::DeviceReduce::Max(tmp, tmp_bytes, level, dmax, (int)N, st);
  cudaFreeAsync(tmp, st);
  RS_CUDA_TRY(e);
  int32_t mx = 0;
  RS_CUDA_TRY(cudaMemcpyAsync(&mx, dmax, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RS_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFreeAsync(next, st);
  *nlev_host = (int64_t)mx + 1;
  return RS_OK;
}

// order[pos] = global row (or -1) with every level padded to a multiple of H.
// order must hold N + H * nlev entries; *npos_host = positions used.
int tri_order(int B, int32_t n, const int32_t* level, int64_t nlev, int32_t H, int32_t* order,
              int64_t* npos_host, cudaStream_t st) {
  const int64_t N = (int64_t)B * n;
  *npos_host = 0;
  if (N == 0 || nlev == 0) return RS_OK;
  int32_t *hist = nullptr, *padded = nullptr, *off = nullptr, *poff = nullptr, *keys = nullptr,
          *rows = nullptr, *rows_in = nullptr;
  void* tmp = nullptr;
  auto cleanup = [&]() {
    for (void* p : {(void*)hist, (void*)padded, (void*)off, (void*)poff, (void*)keys,
                    (void*)rows, (void*)rows_in, tmp})
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
  LV_TRY(cudaMallocAsync(&keys, sizeof(int32_t) * N, st));
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
  // stable sort of the rows by level (ties keep ascending row order)
  iota_kernel<<<grid_of(N, 256), 256, 0, st>>>(N, rows_in);
  count_launch();
  int bits = 1;
  while (((int64_t)1 << bits) < nlev) ++bits;
  size_t tmp_bytes = 0;
  LV_TRY(cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, level, keys, rows_in, rows, (int)N,
                                         0, bits, st));
  LV_TRY(cudaMallocAsync(&tmp, tmp_bytes, st));
  LV_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, level, keys, rows_in, rows, (int)N, 0,
                                         bits, st));
  LV_TRY(cudaMemsetAsync(order, 0xff, sizeof(int32_t) * npos, st));
  level_place_kernel<<<grid_of(N, 256), 256, 0, st>>>(N, keys, rows, off, poff, order);
  count_launch();
  LV_TRY(cudaGetLastError());
#undef LV_TRY
  cleanup();
  *npos_host = npos;
  return RS_OK;
}

// Pass 1 (sci == null): sptr[npos/H + 1] and *total (padded entries, host).
// Pass 2: fill sci / sv.
int tri_sell(int B, int32_t n, int upper, const int32_t* rp, const int32_t* ci, const double2* v,
             const int32_t* order, int64_t npos, int32_t H, int32_t* sptr, int32_t* sci,
             double2* sv, int64_t* total, cudaStream_t st) {
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
    RS_CUDA_TRY(cudaGetLastError());
  }
  return RS_OK;
}

}  // namespace rs
