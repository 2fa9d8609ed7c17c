// Column-oriented triangular sweeps: the reference lower_solve / upper_solve
// loops (_ckernels.pyx:53-85) executed verbatim, so bit-exactness is by
// construction:
//
//   lower:  for c ascending:  y[Li[p]] -= Lx[p] * y[c]   (unit diagonal skipped)
//   upper:  for c descending: y[c] *= recipc(U_cc); y[Ui[p]] -= Ux[p] * y[c]
//
// Why this shape on B200: under RCM the factors' dependency DAG is almost a
// chain (c4 U: ~1 level per row), so the sweep is latency-bound on the
// column-to-column hand-off.  A row-oriented sweep pays an inter-warp
// hand-off (>= 130-200 cycles through shared memory) per row.  Here ONE warp
// (the consumer) carries the whole chain and the hand-off is intra-warp:
// column c's entries are applied lane-parallel (distinct rows, so their order
// is free) as shared-memory read-modify-writes of y, and a __syncwarp orders
// them before column c+1 reads y[c+1].
//
// A single warp is bound by its own dependent-instruction latency, so the
// consumer's per-column work is cut to the minimum by a precomputed COLUMN
// STREAM (built once per factorization, sell.cu col_stream_build): the
// columns in sweep order (L ascending, U descending), each padded to whole
// 32-entry rows (row index -1 = padding), every row tagged "continues the
// previous column" or not, and U's first rows carrying recipc(U_cc).
// PRODUCER warps copy stream rows into a shared-memory ring (coalesced, four
// rows in flight per warp); the consumer reads one ring row per step, with
// the next row prefetched into registers while the current one is applied.
// Per column the critical path is one shared load of y[c] (and of y[i]), one
// complex multiply-subtract, the store and a __syncwarp.
//
// y must be in shared memory (n <= ~7-12k complex per CTA); larger systems
// use the row-oriented sweeps of cta_ops.cuh.
#pragma once
#include "common.cuh"
#include "cta_ops.cuh"

namespace rs {
namespace cta {

// One triangle's column stream for one system.
struct ColStream {
  const int32_t* idx;   // [rows * 32], -1 = padding
  const double2* val;   // [rows * 32]
  const int32_t* meta;  // [rows]: 1 = continues the previous column
  const double2* rd;    // [rows]: recipc(U_cc) on U's first rows (U only)
  int rows;
};

struct ColRing {
  int32_t* idx;  // [S * 32]
  double2* val;  // [S * 32]
  double2* rd;   // [S]
  int* seq;      // [S]: (stream row << 1) | continuation, -1 = empty
  int* head;     // consumer progress (rows fully consumed)
  int S;         // slots (power of two)
};

__host__ __device__ inline size_t col_ring_bytes(int S) {
  return (size_t)S * 32 * (sizeof(int32_t) + sizeof(double2)) + (size_t)S * sizeof(double2) +
         sizeof(int) * ((size_t)S + 4);
}

// Carve a ring out of shared memory at p (16-byte aligned).
__device__ __forceinline__ ColRing col_ring_at(unsigned char* p, int S) {
  ColRing g;
  g.val = reinterpret_cast<double2*>(p);
  g.rd = g.val + 32 * S;
  g.idx = reinterpret_cast<int32_t*>(g.rd + S);
  g.seq = g.idx + 32 * S;
  g.head = g.seq + S;
  g.S = S;
  return g;
}

__device__ __forceinline__ unsigned saddr(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
// CTA-scope acquire / release on the ring's control words: a slot's sequence
// word is published with release after its entries and read with acquire
// before them.
__device__ __forceinline__ int ld_acq(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];" : "=r"(v) : "r"(saddr(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"(saddr(p)), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_rlx(const int* p) {
  int v;
  asm volatile("ld.volatile.shared.b32 %0, [%1];" : "=r"(v) : "r"(saddr(p)));
  return v;
}
__device__ __forceinline__ void st_rlx(int* p, int v) {
  asm volatile("st.volatile.shared.b32 [%0], %1;" ::"r"(saddr(p)), "r"(v) : "memory");
}
// explicit shared accesses for the sweep vector (asm volatile keeps order)
__device__ __forceinline__ double2 lds2(unsigned a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts2(unsigned a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}

// All threads of the CTA: reset the ring before a sweep.
__device__ __forceinline__ void col_ring_reset(const ColRing& g) {
  for (int s = threadIdx.x; s < g.S; s += blockDim.x) g.seq[s] = -1;
  if (threadIdx.x == 0) *g.head = 0;
}

// Producer warp pw of P: rows pw, pw + P, ... of the stream into the ring,
// four rows' loads in flight before the first store.
__device__ __forceinline__ void col_ring_produce(const ColRing& g, const ColStream& cs,
                                                 bool upper, int pw, int P) {
  constexpr int U = 4;
  const int lane = threadIdx.x & 31;
  for (int r0 = pw; r0 < cs.rows; r0 += U * P) {
    int ci[U], mt[U];
    double2 cv[U], rd[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * P;
      if (r < cs.rows) {
        ci[u] = __ldg(cs.idx + 32 * (int64_t)r + lane);
        cv[u] = __ldg(cs.val + 32 * (int64_t)r + lane);
        mt[u] = __ldg(cs.meta + r);
        if (upper) rd[u] = __ldg(cs.rd + r);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int r = r0 + u * P;
      if (r >= cs.rows) break;
      // slot r % S last held row r - S: wait until it is consumed
      if (r >= g.S) {
        if (lane == 0)
          while (ld_rlx(g.head) <= r - g.S) __nanosleep(20);
        __syncwarp();
      }
      const int slot = r & (g.S - 1);
      g.idx[32 * slot + lane] = ci[u];
      g.val[32 * slot + lane] = cv[u];
      if (upper && lane == 0) g.rd[slot] = rd[u];
      __syncwarp();
      if (lane == 0) st_rel(g.seq + slot, (r << 1) | (mt[u] & 1));
    }
  }
}

// One staged stream row in registers.
struct ColRow {
  int i;       // this lane's row index (-1 = padding)
  double2 v;   // this lane's factor entry
  double2 rd;  // recipc(U_cc) (U first rows)
  int cont;    // continues the previous column
};

__device__ __forceinline__ void col_row_fetch(const ColRing& g, int r, bool upper, ColRow& x) {
  const int lane = threadIdx.x & 31;
  const int slot = r & (g.S - 1);
  int s;
  while (((s = ld_acq(g.seq + slot)) >> 1) != r) {
  }
  x.cont = s & 1;
  x.i = g.idx[32 * slot + lane];
  x.v = g.val[32 * slot + lane];
  if (upper) x.rd = g.rd[slot];
}

// Consumer warp: the whole sweep, in place on y (shared memory).
template <bool UPPER>
__device__ __forceinline__ void col_consume(int n, int rows, const ColRing& g, double2* y) {
  const int lane = threadIdx.x & 31;
  const unsigned yb = saddr(y);
  int c = UPPER ? n : -1;
  double2 xc = make_double2(0.0, 0.0);
  ColRow nxt;
  if (rows > 0) col_row_fetch(g, 0, UPPER, nxt);
  for (int r = 0; r < rows; ++r) {
    const ColRow cur = nxt;
    if (!cur.cont) {  // first row of the next column (warp-uniform)
      c += UPPER ? -1 : 1;
      xc = lds2(yb + 16u * c);
      if (UPPER) {
        xc = cmul_plain(xc, cur.rd);
        if (lane == 0) sts2(yb + 16u * c, xc);
      }
    }
    double2 yi;
    if (cur.i >= 0) yi = lds2(yb + 16u * cur.i);
    if (r + 1 < rows) col_row_fetch(g, r + 1, UPPER, nxt);
    if (cur.i >= 0) sts2(yb + 16u * cur.i, csub(yi, cmul_plain(cur.v, xc)));
    __syncwarp();
    if (lane == 0 && (r & 3) == 3) st_rlx(g.head, r + 1);
  }
}

// CTA-level in-place M^{-1} sweeps on y (shared memory): warp 0 consumes,
// warps 1..P produce.  Must be called by all threads (contains
// __syncthreads).
__device__ __forceinline__ void col_lu_sweeps(int n, const ColStream& Ls, const ColStream& Us,
                                              const ColRing& g, double2* y) {
  const int wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int P = max(1, min(nw - 1, 4));
  col_ring_reset(g);
  __syncthreads();
  if (wid == 0) col_consume<false>(n, Ls.rows, g, y);
  else if (wid <= P) col_ring_produce(g, Ls, false, wid - 1, P);
  __syncthreads();
  col_ring_reset(g);
  __syncthreads();
  if (wid == 0) col_consume<true>(n, Us.rows, g, y);
  else if (wid <= P) col_ring_produce(g, Us, true, wid - 1, P);
  __syncthreads();
}

}  // namespace cta
}  // namespace rs
