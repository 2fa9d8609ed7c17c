// Reverse Cuthill-McKee ordering, bit-identical to the reference
// ordering.rcm (pkg/src/rhosolve/ordering.py:82-118):
//   * graph = stored structure of A + A^T, self-loops removed, deduplicated
//     (_symmetric_adjacency, ordering.py:62-79); deg = #distinct neighbours;
//   * each component starts at the unvisited node of minimum (deg, index);
//   * queue BFS, a popped node appends its unvisited neighbours sorted by
//     (deg, index);
//   * the Cuthill-McKee order is reversed (Permutation.from_order(order[::-1]),
//     sparse.py:166-171).
//
// Level-synchronous restatement (provably the same order): the queue visits
// level l in its CM order; a node u of level l+1 is appended by its
// earliest-positioned neighbour in level l, and children of one parent follow
// the (deg, index) order.  So level l+1 = unvisited neighbours of level l
// sorted by (parent_pos, deg, index), with parent_pos = min position of a
// level-l neighbour (an integer atomicMin; the first thread to lower it from
// "unreached" claims u for the candidate list).  The sort is a counting sort
// on parent_pos followed by a per-parent insertion sort on (deg, index).
//
// One CTA per system (batches = the config-4 sweep); every phase is a
// barrier-separated sweep, integer-only and deterministic.
#include "common.cuh"
#include "kernels.cuh"

namespace rs {

constexpr int32_t UNREACHED = 0x7fffffff;

// ---- symmetric adjacency (count / fill passes) -----------------------------
template <bool FILL>
__global__ void sym_adj_kernel(int64_t nrows, int32_t n, const int32_t* rp, const int32_t* ci,
                               const int32_t* trp, const int32_t* tci, int32_t* counts,
                               const int32_t* out_rp, int32_t* out_ci) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  const int32_t self = (int32_t)(r % n);
  int32_t a = rp[r], ae = rp[r + 1], b = trp[r], be = trp[r + 1];
  int32_t cnt = 0, last = -1;
  int32_t o = FILL ? out_rp[r] : 0;
  while (a < ae || b < be) {
    int32_t c;
    if (b >= be || (a < ae && ci[a] <= tci[b])) c = ci[a++];
    else c = tci[b++];
    if (c == self || c == last) continue;
    last = c;
    if (FILL) out_ci[o++] = c;
    ++cnt;
  }
  if (!FILL) counts[r] = cnt;
}

struct RcmArgs {
  int32_t n;
  const int32_t* arp;  // adjacency row pointers [B*n+1] (absolute)
  const int32_t* aci;  // local neighbours
  int32_t* parent;     // [B*n] scratch
  int32_t* order;      // [B*n] scratch
  int32_t* tmp;        // [B*n]
  int32_t* bcnt;       // [B*n]
  int32_t* boff;       // [B*n]
  int32_t* fwd;        // out [B*n]
  int32_t* inv;        // out [B*n]
};

__device__ __forceinline__ int32_t deg_of(const int32_t* arp, int32_t u) {
  return arp[u + 1] - arp[u];
}

__global__ void __launch_bounds__(1024) rcm_kernel(RcmArgs a) {
  const int b = blockIdx.x;
  const int32_t n = a.n;
  const int64_t bn = (int64_t)b * n;
  const int32_t* arp = a.arp + bn;
  const int32_t* aci = a.aci;
  int32_t* parent = a.parent + bn;
  int32_t* order = a.order + bn;
  int32_t* tmp = a.tmp + bn;
  int32_t* bcnt = a.bcnt + bn;
  int32_t* boff = a.boff + bn;
  __shared__ int32_t s_ncand;
  __shared__ unsigned long long s_min;
  __shared__ int32_t s_scan[1024];
  __shared__ int32_t s_carry;

  for (int32_t i = threadIdx.x; i < n; i += blockDim.x) {
    parent[i] = UNREACHED;
    bcnt[i] = 0;
  }
  __syncthreads();
  int32_t filled = 0;
  while (filled < n) {
    // component start: unvisited node of minimum (deg, index)
    if (threadIdx.x == 0) s_min = ~0ull;
    __syncthreads();
    unsigned long long best = ~0ull;
    for (int32_t i = threadIdx.x; i < n; i += blockDim.x)
      if (parent[i] == UNREACHED) {
        const unsigned long long key =
            ((unsigned long long)(uint32_t)deg_of(arp, i) << 32) | (uint32_t)i;
        best = key < best ? key : best;
      }
    atomicMin(&s_min, best);
    __syncthreads();
    const int32_t start = (int32_t)(s_min & 0xffffffffu);
    if (threadIdx.x == 0) {
      parent[start] = -1;
      order[filled] = start;
      s_ncand = 0;
    }
    __syncthreads();
    int32_t lvl_start = filled;
    int32_t lvl_end = filled + 1;
    filled = lvl_end;
    while (lvl_start < lvl_end) {
      // A: claim unvisited neighbours, record earliest parent position
      const int32_t width = lvl_end - lvl_start;
      for (int32_t q = threadIdx.x; q < width; q += blockDim.x) {
        const int32_t pos = lvl_start + q;
        const int32_t v = order[pos];
        for (int32_t e = arp[v]; e < arp[v + 1]; ++e) {
          const int32_t u = aci[e];
          const int32_t pu = *(volatile int32_t*)(parent + u);
          if (pu < lvl_start) continue;  // visited in an earlier level
          const int32_t old = atomicMin(parent + u, pos);
          if (old == UNREACHED) tmp[atomicAdd(&s_ncand, 1)] = u;
        }
      }
      __syncthreads();
      const int32_t nc = s_ncand;
      if (nc == 0) break;
      // B: bucket sizes per parent position
      for (int32_t j = threadIdx.x; j < nc; j += blockDim.x)
        atomicAdd(bcnt + (parent[tmp[j]] - lvl_start), 1);
      __syncthreads();
      // C: exclusive scan of bcnt[0..width) -> boff
      if (threadIdx.x == 0) s_carry = 0;
      __syncthreads();
      for (int32_t base = 0; base < width; base += blockDim.x) {
        const int32_t idx = base + threadIdx.x;
        const int32_t v = idx < width ? bcnt[idx] : 0;
        s_scan[threadIdx.x] = v;
        __syncthreads();
        for (int off = 1; off < (int)blockDim.x; off <<= 1) {
          const int32_t add = threadIdx.x >= (unsigned)off ? s_scan[threadIdx.x - off] : 0;
          __syncthreads();
          s_scan[threadIdx.x] += add;
          __syncthreads();
        }
        if (idx < width) {
          boff[idx] = s_carry + s_scan[threadIdx.x] - v;
          bcnt[idx] = 0;  // reused as the fill counter
        }
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_carry += s_scan[threadIdx.x];
        __syncthreads();
      }
      // D: place candidates into their parent bucket (order inside the bucket
      // is fixed by E)
      for (int32_t j = threadIdx.x; j < nc; j += blockDim.x) {
        const int32_t u = tmp[j];
        const int32_t bk = parent[u] - lvl_start;
        order[lvl_end + boff[bk] + atomicAdd(bcnt + bk, 1)] = u;
      }
      __syncthreads();
      // E: per-bucket insertion sort by (deg, index); reset counters
      for (int32_t bk = threadIdx.x; bk < width; bk += blockDim.x) {
        const int32_t s = lvl_end + boff[bk];
        const int32_t e = s + bcnt[bk];
        for (int32_t x = s + 1; x < e; ++x) {
          const int32_t u = order[x];
          const int32_t du = deg_of(arp, u);
          int32_t y = x;
          while (y > s) {
            const int32_t w = order[y - 1];
            const int32_t dw = deg_of(arp, w);
            if (dw < du || (dw == du && w < u)) break;
            order[y] = w;
            --y;
          }
          order[y] = u;
        }
        bcnt[bk] = 0;
      }
      if (threadIdx.x == 0) s_ncand = 0;
      __syncthreads();
      lvl_start = lvl_end;
      lvl_end += nc;
      filled = lvl_end;
    }
    __syncthreads();
  }
  // reverse: inverse[k] = order[n-1-k]; forward[inverse[k]] = k
  for (int32_t k = threadIdx.x; k < n; k += blockDim.x) {
    const int32_t u = order[n - 1 - k];
    a.inv[bn + k] = u;
    a.fwd[bn + u] = k;
  }
}

static inline unsigned gridr(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

int rcm_order(int B, int32_t n, const int32_t* rp, const int32_t* ci, int32_t* fwd,
              int32_t* inv, cudaStream_t st) {
  const int64_t nrows = (int64_t)B * n;
  int32_t nnz32 = 0;
  RS_CUDA_TRY(cudaMemcpyAsync(&nnz32, rp + nrows, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RS_CUDA_TRY(cudaStreamSynchronize(st));
  int32_t *trp = nullptr, *tci = nullptr, *counts = nullptr, *arp = nullptr, *aci = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&trp, sizeof(int32_t) * (nrows + 1), st));
  RS_CUDA_TRY(cudaMallocAsync(&tci, sizeof(int32_t) * ((int64_t)nnz32 + 1), st));
  int rc = csr_transpose(B, n, rp, ci, nullptr, trp, tci, nullptr, st);
  if (rc) return rc;
  RS_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (nrows + 1), st));
  RS_CUDA_TRY(cudaMallocAsync(&arp, sizeof(int32_t) * (nrows + 1), st));
  sym_adj_kernel<false><<<gridr(nrows, 256), 256, 0, st>>>(nrows, n, rp, ci, trp, tci, counts,
                                                          nullptr, nullptr); ::rs::count_launch();
  int64_t annz = 0;
  rc = scan_counts(counts, arp, nrows, &annz, st);
  if (rc) return rc;
  RS_CUDA_TRY(cudaMallocAsync(&aci, sizeof(int32_t) * (annz + 1), st));
  sym_adj_kernel<true><<<gridr(nrows, 256), 256, 0, st>>>(nrows, n, rp, ci, trp, tci, nullptr,
                                                         arp, aci); ::rs::count_launch();
  RcmArgs a;
  a.n = n;
  a.arp = arp;
  a.aci = aci;
  int32_t* scratch = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&scratch, sizeof(int32_t) * nrows * 5, st));
  a.parent = scratch;
  a.order = scratch + nrows;
  a.tmp = scratch + 2 * nrows;
  a.bcnt = scratch + 3 * nrows;
  a.boff = scratch + 4 * nrows;
  a.fwd = fwd;
  a.inv = inv;
  rcm_kernel<<<B, 1024, 0, st>>>(a); ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  cudaFreeAsync(scratch, st);
  cudaFreeAsync(trp, st);
  cudaFreeAsync(tci, st);
  cudaFreeAsync(counts, st);
  cudaFreeAsync(arp, st);
  cudaFreeAsync(aci, st);
  return RS_OK;
}

__global__ void same_pattern_init_kernel(int32_t* same) { *same = 1; }

// Every system of the batch stores system 0's pattern?  (rs_same_pattern)
__global__ void same_pattern_kernel(int32_t B, int32_t n, int64_t per,
                                    const int32_t* __restrict__ rp,
                                    const int32_t* __restrict__ ci, int32_t* same) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t nnz = per * B;
  bool bad = false;
  if (t < nnz && t >= per) bad = ci[t] != ci[t % per];
  if (t < (int64_t)B * n) {  // row extents, relative to the system's first entry
    const int64_t b = t / n;
    bad = bad || (int64_t)rp[t] - b * per != (int64_t)rp[t - b * n];
  }
  if (t == 0) bad = bad || rp[(int64_t)B * n] != nnz;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *same = 0;
}

int same_pattern(int32_t B, int32_t n, const int32_t* rp, const int32_t* ci, int64_t nnz,
                 int32_t* same, cudaStream_t st) {
  const bool candidate = B > 1 && n > 0 && nnz % B == 0;
  RS_CUDA_TRY(cudaMemsetAsync(same, 0, sizeof(int32_t), st));
  if (!candidate) return RS_OK;
  same_pattern_init_kernel<<<1, 1, 0, st>>>(same);
  const int64_t work = nnz > (int64_t)B * n ? nnz : (int64_t)B * n;
  same_pattern_kernel<<<(unsigned)((work + 255) / 256), 256, 0, st>>>(B, n, nnz / B, rp, ci, same);
  ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

}  // namespace rs
