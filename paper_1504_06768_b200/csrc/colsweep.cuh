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
// 64-entry rows (row index -1 = padding), every row tagged "continues the
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

// Stream row width: two entries per lane, so the typical banded column
// (~50-70 off-diagonal entries) is one or two consumer steps.
constexpr int CW = 64;

// One triangle's column stream for one system.
struct ColStream {
  const int32_t* idx;   // [rows * CW], -1 = padding
  const double2* val;   // [rows * CW]
  const int32_t* meta;  // [rows]: 1 = continues the previous column
  const double2* rd;    // [rows]: recipc(U_cc) on U's first rows (U only)
  int rows;
};

struct ColRing {
  int32_t* idx;  // [S * CW]
  double2* val;  // [S * CW]
  double2* rd;   // [S]
  int* seq;      // [S]: (stream row << 1) | continuation, -1 = empty
  int* head;     // consumer progress (rows fully consumed)
  int S;         // slots (power of two)
};

// shared bytes of the sweep vector: y[0..n-1] plus one dummy slot
__host__ __device__ inline size_t col_y_bytes(int n) { return 16 * ((size_t)n + 1); }

__host__ __device__ inline size_t col_ring_bytes(int S) {
  return (size_t)S * CW * (sizeof(int32_t) + sizeof(double2)) + (size_t)S * sizeof(double2) +
         sizeof(int) * ((size_t)S + 4);
}

// Carve a ring out of shared memory at p (16-byte aligned).
__device__ __forceinline__ ColRing col_ring_at(unsigned char* p, int S) {
  ColRing g;
  g.val = reinterpret_cast<double2*>(p);
  g.rd = g.val + CW * S;
  g.idx = reinterpret_cast<int32_t*>(g.rd + S);
  g.seq = g.idx + CW * S;
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

// Where the sweep vector lives: shared memory (32-bit addresses) when it
// fits the CTA, else global memory (the consumer warp is its only reader and
// writer during a sweep, so L1 serves its re-reads; __syncwarp orders lanes).
template <typename AT>
struct YMem;
template <>
struct YMem<unsigned> {
  __device__ static unsigned base(double2* y) { return saddr(y); }
  __device__ static double2 ld(unsigned a) { return lds2(a); }
  __device__ static void st(unsigned a, double2 v) { sts2(a, v); }
};
template <>
struct YMem<unsigned long long> {
  __device__ static unsigned long long base(double2* y) {
    return reinterpret_cast<unsigned long long>(y);
  }
  __device__ static double2 ld(unsigned long long a) {
    double2 v;
    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(a));
    return v;
  }
  __device__ static void st(unsigned long long a, double2 v) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(a), "d"(v.x), "d"(v.y) : "memory");
  }
};

// All threads of the CTA: reset the ring before a sweep.
__device__ __forceinline__ void col_ring_reset(const ColRing& g) {
  for (int s = threadIdx.x; s < g.S; s += blockDim.x) g.seq[s] = -1;
  if (threadIdx.x == 0) *g.head = 0;
}

// cp.async helpers (16-byte global -> shared copies that bypass registers)
__device__ __forceinline__ void cp16(unsigned dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Producer warp pw of P: batches of PB consecutive rows (batch k = pw, pw+P,
// ...) copied into the ring with cp.async (no registers held: two batches
// in flight per warp), each batch published once it has landed.
constexpr int PB = 4;

__device__ __forceinline__ void col_ring_produce(const ColRing& g, const ColStream& cs,
                                                 bool upper, int pw, int P) {
  const int lane = threadIdx.x & 31;
  const int nb = (cs.rows + PB - 1) / PB;
  const unsigned sidx = saddr(g.idx), sval = saddr(g.val), srd = saddr(g.rd);
  int pend = -1;       // batch issued but not yet published
  int pend_meta = 0;   // lane j < PB: meta of row j of the pending batch
  auto publish = [&]() {
    __syncwarp();
    __threadfence_block();
    const int r0 = pend * PB;
    if (lane < min(PB, cs.rows - r0)) {
      const int r = r0 + lane;
      st_rlx(g.seq + (r & (g.S - 1)), (r << 1) | (pend_meta & 1));
    }
    pend = -1;
  };
  for (int k = pw; k < nb; k += P) {
    const int r0 = k * PB;
    const int cnt = min(PB, cs.rows - r0);
    const int meta = lane < cnt ? __ldg(cs.meta + r0 + lane) : 0;
    // space: slots of rows r0 .. r0+cnt-1 last held rows - S.  Never block
    // while holding an unpublished batch (the consumer may need it first).
    const int need = r0 + cnt - g.S;
    if (need > 0) {
      int h = 0;
      if (lane == 0) h = ld_rlx(g.head);
      h = __shfl_sync(FULL, h, 0);
      if (h < need) {
        if (pend >= 0) {
          cp_wait<0>();
          publish();
        }
        if (lane == 0)
          while (ld_rlx(g.head) < need) __nanosleep(20);
        __syncwarp();
      }
    }
    for (int j = 0; j < cnt; ++j) {
      const int r = r0 + j;
      const int slot = r & (g.S - 1);
      // idx row: 256 B = 16 x 16 B; val row: 1 KB = 64 x 16 B
      if (lane < 16)
        cp16(sidx + (unsigned)(CW * 4 * slot + 16 * lane), cs.idx + CW * (int64_t)r + 4 * lane);
      cp16(sval + (unsigned)(CW * 16 * slot + 16 * lane), cs.val + CW * (int64_t)r + lane);
      cp16(sval + (unsigned)(CW * 16 * slot + 16 * (lane + 32)),
           cs.val + CW * (int64_t)r + lane + 32);
      if (upper && lane == 0) cp16(srd + 16u * slot, cs.rd + r);
    }
    cp_commit();
    if (pend >= 0) {  // the previous batch has had a batch's time to land
      cp_wait<1>();
      publish();
    }
    pend = k;
    pend_meta = meta;
  }
  if (pend >= 0) {
    cp_wait<0>();
    publish();
  }
}

// One staged stream row in registers.
template <typename AT>
struct ColRow {
  AT a0, a1;        // addresses of this lane's two y entries (dummy slot for padding)
  double2 v0, v1;   // this lane's two factor entries
  double2 rd;       // recipc(U_cc) (U first rows)
  int cont;         // continues the previous column
};

// tuning hook: per-row consumer clocks [3 * rows] of the first system's L sweep
__device__ long long* g_col_times = nullptr;

// Raw ring row r (known staged) in registers; the y addresses are derived
// from it one step later (col_row_addr), after the current row's math, so
// the consumer never stalls on these loads.
struct ColRaw {
  int seq, i0, i1;
  double2 v0, v1, rd;
};
template <bool UPPER>
__device__ __forceinline__ void col_row_raw(const ColRing& g, int r, ColRaw& x) {
  const int lane = threadIdx.x & 31;
  const int slot = r & (g.S - 1);
  x.seq = g.seq[slot];
  x.i0 = g.idx[CW * slot + lane];
  x.i1 = g.idx[CW * slot + 32 + lane];
  x.v0 = g.val[CW * slot + lane];
  x.v1 = g.val[CW * slot + 32 + lane];
  if (UPPER) x.rd = g.rd[slot];
}
template <typename AT>
__device__ __forceinline__ void col_row_addr(const ColRaw& w, AT yb, AT dummy, ColRow<AT>& x) {
  x.cont = w.seq & 1;
  x.a0 = w.i0 >= 0 ? yb + (AT)16 * (AT)w.i0 : dummy;
  x.a1 = w.i1 >= 0 ? yb + (AT)16 * (AT)w.i1 : dummy;
  x.v0 = w.v0;
  x.v1 = w.v1;
  x.rd = w.rd;
}
template <bool UPPER, typename AT>
__device__ __forceinline__ void col_row_load(const ColRing& g, int r, AT yb, AT dummy,
                                             ColRow<AT>& x) {
  ColRaw w;
  col_row_raw<UPPER>(g, r, w);
  col_row_addr(w, yb, dummy, x);
}

// Rows below the returned bound are staged: the warp checks the next 32
// slots at once (one acquire load per lane + ballot), so the common-case
// per-row cost is a uniform compare.
__device__ __forceinline__ int col_ring_ready(const ColRing& g, int r, int rows) {
  const int lane = threadIdx.x & 31;
  while (true) {
    const int rr = r + lane;
    const bool ok = rr >= rows || ((ld_acq(g.seq + (rr & (g.S - 1))) >> 1) == rr);
    const unsigned bad = __ballot_sync(FULL, !ok);
    const int cnt = bad ? __ffs(bad) - 1 : 32;
    if (cnt > 0) return r + cnt;
  }
}

// One consumer step: apply row r (cur) and stage row r+1 (nxt).  Order:
// issue the y loads of row r, issue the raw ring loads of row r+1, do row
// r's math and stores, then derive row r+1's addresses.
template <bool UPPER, typename AT>
__device__ __forceinline__ void col_step(const ColRing& g, int r, int rows, AT yb, AT dummy,
                                         int& c, double2& xc, int& ready,
                                         const ColRow<AT>& cur, ColRow<AT>& nxt, long long* tt) {
  using M = YMem<AT>;
  const int lane = threadIdx.x & 31;
  if (tt) tt[3 * r] = clock64();
  // first row of a column: xc = y[c'] (U: times recipc(U_cc), stored back)
  const int cn = cur.cont ? c : c + (UPPER ? -1 : 1);
  double2 xn = M::ld(yb + (AT)16 * (AT)cn);
  const double2 y0 = M::ld(cur.a0), y1 = M::ld(cur.a1);
  const bool more = r + 1 < rows;
  ColRaw w;
  if (more) {
    if (r + 1 >= ready) ready = col_ring_ready(g, r + 1, rows);
    col_row_raw<UPPER>(g, r + 1, w);
  }
  if (tt) tt[3 * r + 1] = clock64();
  if (UPPER) xn = cmul_plain(xn, cur.rd);
  xc = cur.cont ? xc : xn;
  c = cn;
  if (UPPER && lane == 0 && !cur.cont) M::st(yb + (AT)16 * (AT)cn, xc);
  M::st(cur.a0, csub(y0, cmul_plain(cur.v0, xc)));
  M::st(cur.a1, csub(y1, cmul_plain(cur.v1, xc)));
  __syncwarp();
  if (more) col_row_addr(w, yb, dummy, nxt);
  if (tt) tt[3 * r + 2] = clock64();
  if (lane == 0 && (r & 7) == 7) st_rlx(g.head, r + 1);
}

// Consumer warp: the whole sweep, in place on y (shared memory, with one
// dummy slot after y[n-1] absorbing padding updates).
template <bool UPPER, typename AT>
__device__ __forceinline__ void col_consume(int n, int rows, const ColRing& g, double2* y) {
  const int lane = threadIdx.x & 31;
  const AT yb = YMem<AT>::base(y), dummy = yb + (AT)16 * (AT)n;
  long long* const tt = (!UPPER && blockIdx.x == 0 && lane == 0) ? g_col_times : nullptr;
  int c = UPPER ? n : -1;
  double2 xc = make_double2(0.0, 0.0);
  if (rows <= 0) return;
  int ready = col_ring_ready(g, 0, rows);
  ColRow<AT> A, B;
  col_row_load<UPPER, AT>(g, 0, yb, dummy, A);
  for (int r = 0; r < rows; r += 2) {  // unrolled by two: no register moves
    col_step<UPPER, AT>(g, r, rows, yb, dummy, c, xc, ready, A, B, tt);
    if (r + 1 >= rows) break;
    col_step<UPPER, AT>(g, r + 1, rows, yb, dummy, c, xc, ready, B, A, tt);
  }
}

// Several consumer warps for long columns (config 3: ~175 entries per L / U
// column = 3 stream rows).  The rows of ONE column update distinct entries of
// y, so up to W of them are applied by W warps at once; columns stay strictly
// ordered by a named barrier among the consumers (which also orders their y
// accesses: same CTA), so every y[i] still receives its subtractions in column
// order -- bit-identical.  Per group: the consumers read the next W ring
// slots' sequence words, take g = the leading rows that belong to the current
// column (the first row plus its continuations, at most W), warp j < g applies
// row r + j, all meet at the barrier, r += g.
template <bool UPPER, typename AT>
__device__ __forceinline__ void col_consume_multi(int n, int rows, const ColRing& g, double2* y,
                                                  int W, int widx) {
  using M = YMem<AT>;
  const int lane = threadIdx.x & 31;
  const AT yb = M::base(y), dummy = yb + (AT)16 * (AT)n;
  int c = UPPER ? n : -1;
  double2 xc = make_double2(0.0, 0.0);
  int r = 0;
  while (r < rows) {
    // the next W rows staged?  lane j watches row r + j
    int sq;
    while (true) {
      const int rr = r + lane;
      sq = (lane < W && rr < rows) ? ld_acq(g.seq + (rr & (g.S - 1))) : ((rr << 1) | 0);
      const bool ok = lane >= W || rr >= rows || (sq >> 1) == rr;
      if (__all_sync(FULL, ok)) break;
    }
    // group size: row r, then continuation rows
    const unsigned contm = __ballot_sync(FULL, lane < W && r + lane < rows && (sq & 1)) & ~1u;
    const int avail = min(W, rows - r);
    int gsz = 1;
    while (gsz < avail && ((contm >> gsz) & 1u)) ++gsz;
    const int cont0 = __shfl_sync(FULL, sq, 0) & 1;
    // the column of this group (uniform across the consumers)
    if (!cont0) {
      c += UPPER ? -1 : 1;
      double2 xn = M::ld(yb + (AT)16 * (AT)c);
      if (UPPER) xn = cmul_plain(xn, g.rd[r & (g.S - 1)]);
      xc = xn;
    }
    if (widx < gsz) {
      const int slot = (r + widx) & (g.S - 1);
      const int i0 = g.idx[CW * slot + lane], i1 = g.idx[CW * slot + 32 + lane];
      const double2 v0 = g.val[CW * slot + lane], v1 = g.val[CW * slot + 32 + lane];
      const AT a0 = i0 >= 0 ? yb + (AT)16 * (AT)i0 : dummy;
      const AT a1 = i1 >= 0 ? yb + (AT)16 * (AT)i1 : dummy;
      const double2 y0 = M::ld(a0), y1 = M::ld(a1);
      M::st(a0, csub(y0, cmul_plain(v0, xc)));
      M::st(a1, csub(y1, cmul_plain(v1, xc)));
    }
    r += gsz;
    asm volatile("bar.sync 1, %0;" ::"r"(32 * W) : "memory");
    // U: the solved entry replaces y[c] once every consumer has read the
    // unsolved one (no row of this or a later column targets it)
    if (UPPER && !cont0 && widx == 0 && lane == 0) M::st(yb + (AT)16 * (AT)c, xc);
    if (widx == 0 && lane == 0) st_rlx(g.head, r);
  }
}

// A sliding shared-memory window over a sweep vector that is too large for
// shared memory (config 3: n = 57,600).  Column c only touches rows within
// `reach` of it (the factor's bandwidth in pivotal coordinates), so a window
// of WIN = 2^k >= reach + panel + 1 rows, addressed modulo WIN, holds every
// row a panel of columns can touch; at a panel boundary the rows that can no
// longer be touched go back to global memory and the same slots receive the
// rows that enter.  With several consumer warps the global vector would be
// re-read from L2 on every step (each warp's stores invalidate the others'
// L1 lines: 650 ns per column group measured); in the window a step costs
// shared-memory latency.
struct YWindow {
  double2* s;   // [WIN + 1] shared (slot WIN: dummy for padding entries)
  double2* g;   // the whole vector in global memory
  int mask;     // WIN - 1
  int panel;    // columns per panel = WIN - reach - 1
};

template <bool UPPER>
__device__ __forceinline__ void col_consume_win(int n, int rows, const ColRing& g,
                                                const YWindow& w, int W, int widx) {
  const int lane = threadIdx.x & 31;
  const int ct = widx * 32 + lane, cn = 32 * W;  // consumer thread index / count
  const int WIN = w.mask + 1;
  const unsigned sb = saddr(w.s), dummy = sb + 16u * (unsigned)WIN;
  auto bar = [&]() { asm volatile("bar.sync 1, %0;" ::"r"(32 * W) : "memory"); };
  // window: L covers rows [edge, edge + WIN), U covers (edge - WIN, edge]
  int edge = UPPER ? n - 1 : 0;
  if (!UPPER) {
    for (int j = ct; j < min(WIN, n); j += cn) w.s[j & w.mask] = w.g[j];
  } else {
    for (int j = n - 1 - ct; j >= 0 && j > n - 1 - WIN; j -= cn) w.s[j & w.mask] = w.g[j];
  }
  bar();
  int c = UPPER ? n : -1;
  double2 xc = make_double2(0.0, 0.0);
  int r = 0;
  while (r < rows) {
    int sq;
    while (true) {
      const int rr = r + lane;
      sq = (lane < W && rr < rows) ? ld_acq(g.seq + (rr & (g.S - 1))) : ((rr << 1) | 0);
      const bool ok = lane >= W || rr >= rows || (sq >> 1) == rr;
      if (__all_sync(FULL, ok)) break;
    }
    const unsigned contm = __ballot_sync(FULL, lane < W && r + lane < rows && (sq & 1)) & ~1u;
    const int avail = min(W, rows - r);
    int gsz = 1;
    while (gsz < avail && ((contm >> gsz) & 1u)) ++gsz;
    const int cont0 = __shfl_sync(FULL, sq, 0) & 1;
    if (!cont0) {
      c += UPPER ? -1 : 1;
      // panel boundary: every update of the leaving rows is behind the last
      // barrier; swap them for the entering rows, slot for slot
      if (!UPPER && c >= edge + w.panel) {
        for (int j = edge + ct; j < edge + w.panel; j += cn) {
          w.g[j] = w.s[j & w.mask];
          if (j + WIN < n) w.s[j & w.mask] = w.g[j + WIN];
        }
        edge += w.panel;
        bar();
      } else if (UPPER && c <= edge - w.panel) {
        for (int j = edge - ct; j > edge - w.panel; j -= cn) {
          w.g[j] = w.s[j & w.mask];
          if (j - WIN >= 0) w.s[j & w.mask] = w.g[j - WIN];
        }
        edge -= w.panel;
        bar();
      }
      double2 xn = lds2(sb + 16u * (unsigned)(c & w.mask));
      if (UPPER) xn = cmul_plain(xn, g.rd[r & (g.S - 1)]);
      xc = xn;
    }
    if (widx < gsz) {
      const int slot = (r + widx) & (g.S - 1);
      const int i0 = g.idx[CW * slot + lane], i1 = g.idx[CW * slot + 32 + lane];
      const double2 v0 = g.val[CW * slot + lane], v1 = g.val[CW * slot + 32 + lane];
      const unsigned a0 = i0 >= 0 ? sb + 16u * (unsigned)(i0 & w.mask) : dummy;
      const unsigned a1 = i1 >= 0 ? sb + 16u * (unsigned)(i1 & w.mask) : dummy;
      const double2 y0 = lds2(a0), y1 = lds2(a1);
      sts2(a0, csub(y0, cmul_plain(v0, xc)));
      sts2(a1, csub(y1, cmul_plain(v1, xc)));
    }
    r += gsz;
    bar();
    if (UPPER && !cont0 && widx == 0 && lane == 0) sts2(sb + 16u * (unsigned)(c & w.mask), xc);
    if (widx == 0 && lane == 0) st_rlx(g.head, r);
  }
  bar();
  // what is still in the window goes back
  if (!UPPER) {
    for (int j = edge + ct; j < min(edge + WIN, n); j += cn) w.g[j] = w.s[j & w.mask];
  } else {
    for (int j = edge - ct; j >= 0 && j > edge - WIN; j -= cn) w.g[j] = w.s[j & w.mask];
  }
}

// CTA-level in-place M^{-1} sweeps on y (shared memory): warp 0 consumes,
// warps 1..P produce.  Must be called by all threads (contains
// __syncthreads).  consumers > 1 (long columns, lone large systems): warps
// 0..consumers-1 consume together (col_consume_multi), the rest produce.
template <typename AT>
__device__ __forceinline__ void col_lu_sweeps(int n, const ColStream& Ls, const ColStream& Us,
                                              const ColRing& g, double2* y, int consumers = 1,
                                              const YWindow* win = nullptr) {
  const int wid = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  const int W = max(1, min(consumers, nw - 1));
  const int P = max(1, min(nw - W, 8));
  col_ring_reset(g);
  __syncthreads();
  if (win) {  // y in global memory behind a sliding shared-memory window
    if (wid < W) col_consume_win<false>(n, Ls.rows, g, *win, W, wid);
    else if (wid < W + P) col_ring_produce(g, Ls, false, wid - W, P);
    __syncthreads();
    col_ring_reset(g);
    __syncthreads();
    if (wid < W) col_consume_win<true>(n, Us.rows, g, *win, W, wid);
    else if (wid < W + P) col_ring_produce(g, Us, true, wid - W, P);
    __syncthreads();
    return;
  }
  if (W == 1) {
    if (wid == 0) col_consume<false, AT>(n, Ls.rows, g, y);
    else if (wid <= P) col_ring_produce(g, Ls, false, wid - 1, P);
  } else {
    if (wid < W) col_consume_multi<false, AT>(n, Ls.rows, g, y, W, wid);
    else if (wid < W + P) col_ring_produce(g, Ls, false, wid - W, P);
  }
  __syncthreads();
  col_ring_reset(g);
  __syncthreads();
  if (W == 1) {
    if (wid == 0) col_consume<true, AT>(n, Us.rows, g, y);
    else if (wid <= P) col_ring_produce(g, Us, true, wid - 1, P);
  } else {
    if (wid < W) col_consume_multi<true, AT>(n, Us.rows, g, y, W, wid);
    else if (wid < W + P) col_ring_produce(g, Us, true, wid - W, P);
  }
  __syncthreads();
}

}  // namespace cta
}  // namespace rs
