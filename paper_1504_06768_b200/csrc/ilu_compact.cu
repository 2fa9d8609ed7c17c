// Complete LU with partial pivoting, column-pipelined like ilu.cu, with every
// warp's working column held COMPACTLY in shared memory: the batch kernel of
// the c4 sweep (512 systems of order 1600, four systems per SM).
//
// Same semantics and the same bits as the reference `factorize`
// (pkg/src/rhosolve/kernels/_ckernels.pyx:144-385) with drop_tol = 0 and no
// fill cap, and the same pipeline as ilutp_pipeline_kernel (warp w owns
// columns w, w+W, ...; pending pivotal columns in a per-warp bitmap, popped
// in ascending order below the finished-column frontier; see ilu.cu for why
// that reproduces the reference's heap order).  What differs is where the
// column lives.  ilu.cu keeps a dense n-vector per warp in global memory
// (x[row], marker[row], pattern list): every access pays a 64-bit address
// computation and an L1/L2 round trip, and the ncu source view of the batch
// (profiles/r02_ncu_c4_pipeline_source.txt) shows the kernel issue-bound on
// exactly that: ~415 warp instructions per applied L column.  Here
//   * the values of the column's pattern sit in shared memory BY POSITION
//     (xs[pos], discovery order = the reference's pattern order) next to the
//     row of every position (pats[pos], u16), so the pivot search and both
//     emissions are plain scans over positions;
//   * the row -> position map: when the structural bound on a column's
//     pattern (3w+1 for half-bandwidth w, see launch_lu_compact) is <= 248 it
//     is one byte per row in shared memory (POS8), kept exact -- 0xff =
//     absent, and a column clears its own rows when it leaves -- so membership
//     and position are one load; else an int32 per row in per-warp global
//     scratch validated as a sparse set (row i is in the pattern iff
//     p = pos[i] < npat and pats[p] == i: never cleared, stale contents are
//     harmless);
//   * pinv / prow (u16 shadows), Lp, the pending bitmaps, the U positions of
//     the column and Up[k] (a ring handed from column to column) are shared
//     memory too, all addressed with explicit 32-bit ld/st.shared.
// With POS8 the only global traffic of a pop is the L column itself.  A
// column whose pattern outgrows the per-warp capacity (int32 variant only)
// stops the system untouched (state stays FAC_RUNNING) and ilu.cu's general
// kernel factors it afterwards; capacity overflow of the output and zero
// pivots are reported exactly as ilu.cu does.
#include <stdlib.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace rs {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ int warp_min_i(int v) {
  return (int)__reduce_min_sync(FULL, v);
}

}  // namespace

// shared-memory bytes per CTA for `warps` warps and `capx` positions each
// (pos8: the row -> position map lives in shared memory as one byte per row)
size_t lu_compact_smem_bytes(int32_t n, int warps, int capx, int pos8, int ucap = 0) {
  const size_t nwords = ((size_t)n + 31) / 32;
  size_t b = 16 * (size_t)warps * capx + 4 * ((size_t)n + 1) + 4 * nwords * warps + 16 + 128 +
             2 * 2 * (size_t)n + 2 * (size_t)warps * capx;
  if (pos8) b += (size_t)warps * n + (size_t)warps * ucap;  // + U positions of the column
  return b;
}

// Shared memory is addressed with explicit 32-bit shared-state-space
// accesses: under the 64-register cap (four systems per SM) the compiler
// otherwise re-derives every base (CTA window + warp slice + offset) from
// constants at each use -- a third of the instructions of the first version.
__device__ __forceinline__ double2 lds2(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts2(uint32_t a, double2 v) {
  asm volatile("st.shared.v2.f64 [%0], {%1,%2};" ::"r"(a), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ int lds32(uint32_t a) {
  int v;
  asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, int v) {
  asm volatile("st.shared.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int lds16(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return (int)v;
}
__device__ __forceinline__ void sts16(uint32_t a, int v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ int lds8(uint32_t a) {
  unsigned short v;
  asm volatile("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
  return (int)v;
}
__device__ __forceinline__ void sts8(uint32_t a, int v) {
  asm volatile("st.shared.u8 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ void atoms_or(uint32_t a, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void atoms_and(uint32_t a, uint32_t v) {
  asm volatile("red.shared.and.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
// keeps a pointer in registers (opaque to rematerialisation from constants)
template <typename T>
__device__ __forceinline__ T* pin(T* p) {
  asm volatile("" : "+l"(p));
  return p;
}

// POS8: row -> position map as one byte per row in shared memory (capx <= 248, 0xff = absent);
// otherwise int32 per row in per-warp global scratch.
template <int MAXT, int MINB, bool POS8>
__global__ void __launch_bounds__(MAXT, MINB) lu_compact_kernel(FactorArgs a, int capx, int ucap) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, W = blockDim.x >> 5;
  const int b = blockIdx.x + a.b0;
  const int32_t n = a.n;
  const int nwords = (n + 31) >> 5;
  int32_t* state = a.state + 3 * (int64_t)b;
  if (state[0] != FAC_RUNNING) return;

  // shared layout: xs[W][capx] c128 | Lp[n+1] i32 | bits[W][nwords] | ctl[4] | Up ring[32] |
  //                pinv[n] prow[n] u16 (0xffff: none) | pats[W][capx] u16 | pos8[W][n] u8
  const uint32_t s0 = (uint32_t)__cvta_generic_to_shared(smem);
  uint32_t XS = s0 + 16u * (uint32_t)(wid * capx);  // this warp's values by position
  uint32_t LPS = s0 + 16u * (uint32_t)(W * capx);
  uint32_t BITS = LPS + 4u * ((uint32_t)n + 1u) + 4u * (uint32_t)(wid * nwords);
  const uint32_t CTL = LPS + 4u * ((uint32_t)n + 1u) + 4u * (uint32_t)(W * nwords);
  const uint32_t UPR = CTL + 16u;  // Up[k], handed from column k-1's owner to column k's (k mod 32)
  uint32_t PINV = UPR + 128u;                                   // prow at +2n
  uint32_t PATS = PINV + 4u * (uint32_t)n + 2u * (uint32_t)(wid * capx);  // rows by position
  uint32_t POS = PINV + 4u * (uint32_t)n + 2u * (uint32_t)(W * capx) + (uint32_t)(wid * n);
  uint32_t UPOS = PINV + 4u * (uint32_t)n + 2u * (uint32_t)(W * capx) + (uint32_t)(W * n) +
                  (uint32_t)(wid * ucap);  // POS8: positions of the column's U entries, pop order
  asm volatile("" : "+r"(XS), "+r"(LPS), "+r"(PINV), "+r"(BITS), "+r"(PATS), "+r"(POS), "+r"(UPOS));
  const uint32_t n2 = 2u * (uint32_t)n;
#define PROW (PINV + n2)
  constexpr int NONE = 0xffff;

  const int64_t bn = (int64_t)b * n;
  int32_t* const gLp = a.Lp + (int64_t)b * (n + 1);
  int32_t* const gUp = a.Up + (int64_t)b * (n + 1);
  int32_t* const Li = pin(a.Li + (int64_t)b * a.capL);
  double2* const Lx = pin(a.Lx + (int64_t)b * a.capL);
  int32_t* const gpinv = a.pinv + bn;
  const int32_t* const Ap = a.Ap + bn;
  // per-warp global scratch: position of a row (sparse set), U positions of the column
  const int64_t ws = ((int64_t)b * W + wid) * n;
  int32_t* const pos_of = pin(a.wflag + ws);
  auto pos_get = [&](int i) -> int { return POS8 ? lds8(POS + (uint32_t)i) : pos_of[i]; };
  auto pos_set = [&](int i, int p) {
    if (POS8) sts8(POS + (uint32_t)i, p);
    else pos_of[i] = p;
  };
  int32_t* const upos = a.wurow + ws;

  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    sts16(PINV + 2u * i, NONE);
    sts16(PROW + 2u * i, NONE);
    gpinv[i] = -1;
    sts32(LPS + 4u * i, 0);
  }
  for (int w = lane; w < nwords; w += 32) sts32(BITS + 4u * w, 0);
  if (POS8)  // the byte map is kept exact: 0xff = not in the working column
    for (int i = lane; i < n; i += 32) sts8(POS + (uint32_t)i, 0xff);
  if (threadIdx.x == 0) {
    sts32(LPS + 4u * (uint32_t)n, 0);
    sts32(CTL, 0);
    sts32(CTL + 4, 0);
    sts32(UPR, 0);
    gLp[0] = 0;
    gUp[0] = 0;
  }
  __syncthreads();

  for (int k = wid; k < n; k += W) {
    int scanned = lds32(CTL);
    if (lds32(CTL + 4)) break;
    __threadfence_block();
    // ---- 1. scatter column k; seed pending with columns already finished ----
    const int32_t c0 = Ap[k], c1 = Ap[k + 1];
    int npat = c1 - c0;
    if (npat > capx) {
      if (lane == 0) sts32(CTL + 4, 2);
      break;
    }
    int lowc = 0x7fffffff;
    for (int e = c0 + lane; e < c1; e += 32) {
      const int i = a.Ai[e];
      sts2(XS + 16u * (e - c0), a.Ax[e]);
      sts16(PATS + 2u * (e - c0), i);
      pos_set(i, e - c0);
      const int pv = lds16(PINV + 2u * i);
      if (pv < scanned) {  // (NONE = 0xffff is never below the frontier)
        atoms_or(BITS + 4u * (pv >> 5), 1u << (pv & 31));
        lowc = min(lowc, pv);
      }
    }
    lowc = warp_min_i(lowc);
    __syncwarp();

    // ---- 2. updates in ascending pivotal order, gated by the frontier -------
    int unum = 0;
    int w = (lowc == 0x7fffffff) ? ((scanned + 31) >> 5) : (lowc >> 5);
    int stop = 0;  // 1: another warp aborted, 2: pattern capacity exceeded
    while (true) {
      const int wend = (scanned + 31) >> 5;
      int c = -1;
      if (w < wend) {  // the current word first: one broadcast load, no vote
        const uint32_t word = (uint32_t)lds32(BITS + 4u * w);
        if (word) c = (w << 5) + __ffs(word) - 1;
        else ++w;
      }
      while (c < 0 && w < wend) {
        const int ww = w + lane;
        const uint32_t bv = (ww < wend) ? (uint32_t)lds32(BITS + 4u * ww) : 0u;
        const unsigned m = __ballot_sync(FULL, bv != 0u);
        if (m) {
          const int src = __ffs(m) - 1;
          const uint32_t word = __shfl_sync(FULL, bv, src);
          w += src;
          c = (w << 5) + __ffs(word) - 1;
          break;
        }
        w += 32;
      }
      if (c < 0) {
        if (scanned == k) break;
        // advance the frontier over newly finished columns; the owner of the
        // next column to finish polls hot, the others nap with their distance
        int d;
        const int dist = k - scanned - 1;
        const unsigned nap =
            dist <= 0 ? (unsigned)a.hot_nap : (dist < 4 ? a.nap_step * dist : 8u * a.nap_step);
        int ab = 0;
        while ((d = lds32(CTL)) == scanned && !(ab = lds32(CTL + 4))) {
          if (nap) __nanosleep(nap);
        }
        if (ab || lds32(CTL + 4)) {
          stop = 1;
          break;
        }
        __threadfence_block();
        int newlow = 0x7fffffff;
        for (int m = scanned + lane; m < d; m += 32) {
          const int r = lds16(PROW + 2u * m);
          const int p = pos_get(r);
          if (POS8 ? p != 0xff : ((unsigned)p < (unsigned)npat && lds16(PATS + 2u * p) == r)) {
            atoms_or(BITS + 4u * (m >> 5), 1u << (m & 31));
            newlow = min(newlow, m);
          }
        }
        newlow = warp_min_i(newlow);
        __syncwarp();
        w = (newlow == 0x7fffffff) ? ((d + 31) >> 5) : (newlow >> 5);
        scanned = d;
        continue;
      }
      // pop column c.  The loads of L[:,c] are issued first (64 entries a
      // pass, 96 when the column is longer: every c4 column in one pass); the
      // U entry -- the value of c's pivot row, final by now -- and the
      // bookkeeping overlap their latency.
      const int32_t p0 = lds32(LPS + 4u * c) + 1, p1 = lds32(LPS + 4u * c + 4u);
      double2 xc = make_double2(0.0, 0.0);
      if (POS8 && unum >= ucap) {  // (cannot happen within the structural bound)
        stop = 2;
        break;
      }
      // one pass over NH x 32 entries from `base`; returns false on capacity overflow
      auto pass = [&](auto nh, int base) -> bool {
        constexpr int NH = decltype(nh)::value;
        const int cnt = p1 - base;  // warp-uniform
        const int pa = base + lane;
        bool act[NH];
        int ii[NH], ff[NH];
        double2 ll[NH], xx[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          act[h] = lane + 32 * h < cnt;
          ii[h] = 0;
          ll[h] = make_double2(0.0, 0.0);
          if (act[h]) {
            ii[h] = Li[pa + 32 * h];
            ll[h] = Lx[pa + 32 * h];
          }
        }
        if (base == p0) {
          const int pp = pos_get(lds16(PROW + 2u * c));
          xc = lds2(XS + 16u * pp);
          if (lane == 0) {
            atoms_and(BITS + 4u * w, ~(1u << (c & 31)));
            if (POS8) sts8(UPOS + (uint32_t)unum, pp);
            else upos[unum] = pp;
          }
          ++unum;
        }
        bool in[NH];
        int rr[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          ff[h] = act[h] ? pos_get(ii[h]) : 0x7fffffff;
          in[h] = POS8 ? (act[h] && ff[h] != 0xff) : (unsigned)ff[h] < (unsigned)npat;
        }
#pragma unroll
        for (int h = 0; h < NH; ++h) {  // row check and value of a candidate position together
          rr[h] = -1;
          xx[h] = make_double2(0.0, 0.0);
          if (in[h]) {
            if (!POS8) rr[h] = lds16(PATS + 2u * ff[h]);  // sparse-set check (int32 map only)
            xx[h] = lds2(XS + 16u * ff[h]);
          }
        }
        unsigned mm[NH], any = 0;
        bool nw[NH];
#pragma unroll
        for (int h = 0; h < NH; ++h) {
          nw[h] = act[h] && !(in[h] && (POS8 || rr[h] == ii[h]));
          mm[h] = __ballot_sync(FULL, nw[h]);
          any |= mm[h];
        }
        if (any) {  // fill rows join the pattern in discovery order
          int tot = 0;
#pragma unroll
          for (int h = 0; h < NH; ++h) tot += __popc(mm[h]);
          if (npat + tot > capx) return false;
          const unsigned lt = lanemask_lt();
          int at = npat;
#pragma unroll
          for (int h = 0; h < NH; ++h) {
            if (nw[h]) {
              ff[h] = at + __popc(mm[h] & lt);
              xx[h] = make_double2(0.0, 0.0);
              sts16(PATS + 2u * ff[h], ii[h]);
              pos_set(ii[h], ff[h]);
              const int v = lds16(PINV + 2u * ii[h]);
              if (v < scanned) atoms_or(BITS + 4u * (v >> 5), 1u << (v & 31));
            }
            at += __popc(mm[h]);
          }
          npat = at;
          __syncwarp();
        }
#pragma unroll
        for (int h = 0; h < NH; ++h)
          if (act[h]) sts2(XS + 16u * ff[h], csub(xx[h], cmul_plain(ll[h], xc)));
        return true;
      };
      {
        bool ok = true;
        int base = p0;
        do {
          const int cnt = p1 - base;
          if (cnt > 64) ok = pass(std::integral_constant<int, 3>(), base), base += 96;
          else ok = pass(std::integral_constant<int, 2>(), base), base += 64;
        } while (ok && base < p1);
        if (!ok) stop = 2;
      }
      if (stop) break;
      __syncwarp();
    }
    if (stop) {
      if (stop == 2 && lane == 0) sts32(CTL + 4, 2);
      break;
    }
    __threadfence_block();  // acquire: every column < k is final

    // ---- 3. pivot: max |re|+|im| over non-pivotal rows, ties -> lowest row --
    double best = -1.0;
    int ipiv = -1, ipos = -1, lnum = 0;
    for (int blk = 0; blk < npat; blk += 128) {
      int iu[4];
      bool cand[4];
      double2 xv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = blk + 32 * u + lane;
        iu[u] = t < npat ? lds16(PATS + 2u * t) : -1;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = blk + 32 * u + lane;
        cand[u] = iu[u] >= 0 && lds16(PINV + 2u * iu[u]) == NONE;
        xv[u] = cand[u] ? lds2(XS + 16u * t) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        lnum += __popc(__ballot_sync(FULL, cand[u]));
        if (cand[u]) {
          const double mag = cabs1(xv[u]);
          if (mag > best || (mag == best && iu[u] < ipiv)) {
            best = mag;
            ipiv = iu[u];
            ipos = blk + 32 * u + lane;
          }
        }
      }
    }
    // warp argmax of (magnitude, lowest row) with three redux.sync: non-negative
    // doubles order like their bit patterns; a lane without a candidate (best
    // = -1) contributes key 0 like a zero magnitude, and a best of 0 fails the
    // pivot test below either way.  (A NaN never becomes a lane's best: the
    // reference's comparisons fail on it too.)
    const unsigned long long km =
        best >= 0.0 ? (unsigned long long)__double_as_longlong(best) : 0ull;
    const unsigned khi = (unsigned)(km >> 32), klo = (unsigned)km;
    const unsigned mh = __reduce_max_sync(FULL, khi);
    const unsigned ml = __reduce_max_sync(FULL, khi == mh ? klo : 0u);
    const bool top = ipiv >= 0 && khi == mh && klo == ml;
    const unsigned br = __reduce_min_sync(FULL, top ? (unsigned)ipiv : 0xffffffffu);
    const int gipiv = br == 0xffffffffu ? -1 : (int)br;
    const double gbest = __longlong_as_double((long long)(((unsigned long long)mh << 32) | ml));
    if (gipiv < 0 || gbest == 0.0) {
      if (lane == 0) {
        state[0] = FAC_ZERO_PIVOT;
        state[1] = k;
        sts32(CTL + 4, 1);
      }
      break;
    }
    const unsigned om = __ballot_sync(FULL, ipiv == gipiv);
    const int gpos = __shfl_sync(FULL, ipos, __ffs(om) - 1);
    const double2 piv = lds2(XS + 16u * gpos);

    // ---- 4. emit L (unit diagonal first), publish the column, then U -------
    const int32_t lnnz = lds32(LPS + 4u * k);
    const int32_t unnz = lds32(UPR + 4u * (k & 31));
    if ((int64_t)unnz + unum + 1 > a.capU || (int64_t)lnnz + lnum > a.capL) {
      if (lane == 0) {
        state[0] = FAC_OVERFLOW;
        state[1] = k;
        sts32(CTL + 4, 1);
      }
      break;
    }
    const double2 rp = recipc(piv);
    if (lane == 0) {
      Li[lnnz] = gipiv;
      Lx[lnnz] = make_double2(1.0, 0.0);
    }
    int off = lnnz + 1;
    for (int blk = 0; blk < npat; blk += 128) {
      int iu[4];
      bool kp[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int t = blk + 32 * u + lane;
        iu[u] = t < npat ? lds16(PATS + 2u * t) : -1;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        kp[u] = iu[u] >= 0 && iu[u] != gipiv && lds16(PINV + 2u * iu[u]) == NONE;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned m = __ballot_sync(FULL, kp[u]);
        if (kp[u]) {
          const int o = off + __popc(m & lanemask_lt());
          Li[o] = iu[u];
          Lx[o] = cmul_plain(lds2(XS + 16u * (blk + 32 * u + lane)), rp);
        }
        off += __popc(m);
      }
    }
    __threadfence_block();
    __syncwarp();
    if (lane == 0) {
      // only shared-memory state is published on the critical path (the fence
      // has no global store of this lane to wait for); the global copies the
      // kernel itself never reads follow the release
      sts32(LPS + 4u * k + 4u, off);
      sts16(PINV + 2u * gipiv, k);
      sts16(PROW + 2u * k, gipiv);
      sts32(UPR + 4u * ((k + 1) & 31), unnz + unum + 1);
      __threadfence_block();  // release column k
      sts32(CTL, k + 1);
      gUp[k + 1] = unnz + unum + 1;
      gLp[k + 1] = off;
      gpinv[gipiv] = k;
    }
    // U column k (pops were ascending; pivot last): no later column reads it,
    // so it is written after the release, off the critical path
    int32_t* const Ui = a.Ui + (int64_t)b * a.capU;
    double2* const Ux = a.Ux + (int64_t)b * a.capU;
    for (int t = lane; t < unum; t += 32) {
      const int p = POS8 ? lds8(UPOS + (uint32_t)t) : upos[t];
      Ui[unnz + t] = lds16(PINV + 2u * lds16(PATS + 2u * p));
      Ux[unnz + t] = lds2(XS + 16u * p);
    }
    if (lane == 0) {
      Ui[unnz + unum] = k;
      Ux[unnz + unum] = piv;
    }
    if (POS8)  // the column leaves the byte map
      for (int t = lane; t < npat; t += 32) sts8(POS + (uint32_t)lds16(PATS + 2u * t), 0xff);
    __syncwarp();
  }
  __syncthreads();
  if (lds32(CTL + 4)) return;  // zero pivot / overflow recorded; 2: left to the general kernel
  // ---- finish: remap L rows to pivotal indices --------------------------------
  const int32_t lnnz = gLp[n];
  for (int p = threadIdx.x; p < lnnz; p += blockDim.x) Li[p] = lds16(PINV + 2u * Li[p]);
  if (threadIdx.x == 0) {
    state[0] = FAC_DONE;
    state[1] = -1;
  }
#undef PROW
}

// Half-bandwidth of the batch's pattern, max |row - col| (CSC, local rows).
__global__ void band_kernel(int64_t cols, int32_t n, const int32_t* __restrict__ Ap,
                            const int32_t* __restrict__ Ai, int32_t* out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int d = 0;
  if (t < cols) {
    const int j = (int)(t % n);
    for (int32_t e = Ap[t]; e < Ap[t + 1]; ++e) d = max(d, abs(Ai[e] - j));
  }
  d = (int)__reduce_max_sync(FULL, d);
  if ((threadIdx.x & 31) == 0 && d > 0) atomicMax(out, d);
}

// Launches the compact kernel when it applies (complete LU, natural column
// order, shared memory for the shadows plus a useful pattern capacity);
// *launched = 0 otherwise.  Systems it could not finish keep FAC_RUNNING.
//
// Planning.  LU with row interchanges of a matrix of half-bandwidth w keeps
// at most w + 1 entries in a column of L and 2w + 1 in a column of U, so a
// column's pattern never exceeds 3w + 1 rows: the capacity to provide.  When
// that is <= 248 the row -> position map fits one byte per row in shared
// memory too (POS8), and the planner takes the largest warp count whose
// capacity reaches the bound (c4: w = 78, bound 235, seven warps per system at
// four systems per SM).  Otherwise the map stays in global scratch and the
// capacity is whatever fits; columns beyond it send the system to ilu.cu.
int launch_lu_compact(const FactorArgs& a, cudaStream_t st, int* launched) {
  *launched = 0;
  if (a.B == 0 || a.n == 0 || a.q || a.cps > 1 || a.n > 65535) return RS_OK;
  if (a.drop_tol > 0.0 || a.fill_cap >= 0 || a.fill_caps || a.pivot_floor > 0.0) return RS_OK;
  int dev = 0, sms = 0, per_sm = 0, max_block = 0;
  RS_CUDA_TRY(cudaGetDevice(&dev));
  RS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  RS_CUDA_TRY(cudaDeviceGetAttribute(&per_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev));
  RS_CUDA_TRY(cudaDeviceGetAttribute(&max_block, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (a.warps != 8 && a.warps != 16) return RS_OK;
  // systems resident per SM: the whole batch in one wave (up to four per SM
  // with 8-warp systems, two with 16-warp systems)
  const int want = std::min(a.warps == 8 ? 4 : 2, std::max(1, (a.B + sms - 1) / sms));
  const size_t budget = std::min<size_t>((size_t)max_block, (size_t)per_sm / want - 1024);
  // structural bound on a column's pattern
  int32_t bw = 0;
  RS_CUDA_TRY(cudaMemsetAsync(a.gctl, 0, sizeof(int32_t), st));
  const int64_t cols = (int64_t)a.B * a.n;
  band_kernel<<<(unsigned)((cols + 255) / 256), 256, 0, st>>>(cols, a.n, a.Ap, a.Ai, a.gctl);
  ::rs::count_launch();
  RS_CUDA_TRY(cudaMemcpyAsync(&bw, a.gctl, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  RS_CUDA_TRY(cudaStreamSynchronize(st));
  const int need = (int)std::min<int64_t>(a.n, 3 * (int64_t)bw + 1);
  const int ucap = (int)std::min<int64_t>(a.n, 2 * (int64_t)bw + 8);
  int W = 0, capx = 0, pos8 = 0;
  if (need <= 248 && !getenv("RHOSOLVE_COMPACT_NOPOS8")) {  // (position 0xff = absent)
    const int cand8[] = {8, 7, 6, 5, 4}, cand16[] = {16, 12, 8};
    const int* cand = a.warps == 8 ? cand8 : cand16;
    const int nc = a.warps == 8 ? 5 : 3;
    for (int i = 0; i < nc && !W; ++i) {
      const size_t fixed = lu_compact_smem_bytes(a.n, cand[i], 0, 1, ucap);
      if (fixed >= budget) continue;
      const int c = std::min(248, (int)((budget - fixed) / (18 * (size_t)cand[i])) & ~7);
      if (c >= need) {
        W = cand[i];
        capx = std::min(c, (need + 7) & ~7);
        pos8 = 1;
      }
    }
  }
  if (!W) {
    W = a.warps;
    const size_t fixed = lu_compact_smem_bytes(a.n, W, 0, 0);
    if (fixed + 18 * (size_t)W * 64 > budget) return RS_OK;
    capx = (int)((budget - fixed) / (18 * (size_t)W)) & ~7;
    // complete LU fills its band, so the bound is nearly reached (c4: 228 of
    // 235): a capacity below it would abandon the system half-way and leave
    // the whole factorization to ilu.cu anyway
    if (capx < need) return RS_OK;
    capx = std::min(capx, (std::max(need, 8) + 7) & ~7);
  }
  if (const char* e = getenv("RHOSOLVE_COMPACT_CAPX")) capx = std::max(8, atoi(e) & ~7);  // tests
  const size_t smem = lu_compact_smem_bytes(a.n, W, capx, pos8, ucap);
  if (smem > (size_t)max_block) return RS_OK;
  auto launch = [&](auto kern) -> int {
    RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<a.B, 32 * W, smem, st>>>(a, capx, ucap);
    ::rs::count_launch();
    RS_CUDA_TRY(cudaGetLastError());
    return RS_OK;
  };
  if (W > 8 && want > 1)  // (two 16-warp systems per SM: 64 registers)
    RS_TRY(pos8 ? launch(lu_compact_kernel<512, 2, true>) : launch(lu_compact_kernel<512, 2, false>));
  else if (W > 8)
    RS_TRY(pos8 ? launch(lu_compact_kernel<512, 1, true>) : launch(lu_compact_kernel<512, 1, false>));
  else if (W <= 7 && want > 1)  // (224 threads: 72 registers at four systems per SM)
    RS_TRY(pos8 ? launch(lu_compact_kernel<224, 4, true>) : launch(lu_compact_kernel<224, 4, false>));
  else if (want > 1)
    RS_TRY(pos8 ? launch(lu_compact_kernel<256, 4, true>) : launch(lu_compact_kernel<256, 4, false>));
  else
    RS_TRY(pos8 ? launch(lu_compact_kernel<256, 1, true>) : launch(lu_compact_kernel<256, 1, false>));
  *launched = 1;
  return RS_OK;
}

}  // namespace rs
