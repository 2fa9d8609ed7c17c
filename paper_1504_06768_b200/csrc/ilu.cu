// Left-looking sparse LU / ILUTP with threshold partial pivoting, dropping and
// a per-column fill cap: the semantics of the reference `factorize`
// (pkg/src/rhosolve/kernels/_ckernels.pyx:144-385, wrapped by
// factor._factor, pkg/src/rhosolve/factor.py:70-112), reproduced bit for bit.
//
// Why it is bit-exact: for every column k the reference
//   1. scatters A[:,q[k]] into a dense accumulator x,
//   2. applies  x[i] -= L[i,c] * x[prow[c]]  for every reachable pivotal
//      column c in strictly ascending c (its binary heap),
//   3. picks the pivot = max |re|+|im| over non-pivotal rows, ties to the
//      lowest row, fails on none/zero,
//   4. drops entries below d * rownorm, caps kept entries by the total order
//      (-mag, U-before-L, index), and emits U (pivot last) and L (unit
//      diagonal first, scaled by recipc(pivot)).
// Each x[i] therefore receives its updates in ascending c, one complex
// multiply-subtract each.  Here the ascending order comes from a bitmap of
// pending pivotal columns; the entries of one L column touch distinct rows,
// so a warp applies them in parallel without changing any rounding.  Newly
// reached rows are appended in the reference's discovery order (ballot +
// prefix), so the raw CSC output matches the reference array for array.
//
// B200 mapping -- a column pipeline.  Column k needs every earlier pivot, so
// the elimination is sequential in its *tail* (the last updates, the pivot
// search, dropping and emission), but the bulk of a column's work -- the
// updates from columns finished long ago -- is not.  One CTA owns one system;
// warp w owns columns k = w, w+W, w+2W, ...  Each warp keeps a private dense
// accumulator and marker array and a private pending bitmap, and advances a
// "swept" frontier over finished columns: when column m completes, every
// warp whose pattern contains prow[m] marks m pending.  A warp pops pending
// columns strictly below its frontier (no smaller one can ever appear), so up
// to W columns are updated concurrently while the critical path shrinks to
// one column's tail.  pinv/prow/Lp (shared) live in shared memory when they
// fit; completion is a single shared counter with release/acquire fences.
// A batch of systems (config-4 sweep) is a grid of CTAs.
//
// Storage: with a cap, nnz(L)+nnz(U) <= n*cap, so the caller preallocates;
// complete LU (cap = -1) may overflow, in which case the kernel stops before
// column k, records it, and the host grows the buffers and resumes.
#include "common.cuh"
#include "kernels.cuh"
#ifndef RS_FENCE
#define RS_FENCE() __threadfence_block()
#endif
#define RS_FENCE_CTA() __threadfence_block()

namespace rs {

namespace {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ int warp_sum_i(int v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}
__device__ __forceinline__ int warp_min_i(int v) {
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(FULL, v, o));
  return v;
}
__device__ __forceinline__ uint64_t mag_key(double2 z) {
  return (uint64_t)__double_as_longlong(cabs1(z));
}
// Cross-warp shared state (pinv / prow / Lp / Up, in shared or global
// memory) is only ever exchanged inside one CTA: CTA-scope relaxed accesses
// (a plain volatile generic access compiles to a system-scope strong load).
// (MULTI: a system spans several CTAs, so the exchange is GPU-scope.)
template <bool MULTI = false>
__device__ __forceinline__ int vload_(const int32_t* p) {
  int v;
  if (MULTI) asm volatile("ld.relaxed.gpu.s32 %0, [%1];" : "=r"(v) : "l"(p));
  else asm volatile("ld.relaxed.cta.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
template <bool MULTI = false>
__device__ __forceinline__ void vstore_(int32_t* p, int v) {
  if (MULTI) asm volatile("st.relaxed.gpu.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
  else asm volatile("st.relaxed.cta.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void probe_mark(unsigned long long* pr, int k, int slot, int lane) {
  if (pr && lane == 0) pr[(size_t)k * 6 + slot] = clock64();
}

}  // namespace

// shared-memory bytes per CTA: pinv, prow, Lp (when shared_in_smem) + the
// per-warp pending bitmaps (when bits_in_smem) + control words.
__host__ __device__ size_t ilutp_smem_bytes(int32_t n, int warps, int shared_in_smem,
                                            int bits_in_smem, int hist) {
  const size_t nwords = ((size_t)n + 31) / 32;
  size_t b = 64 + (hist ? 1024 * (size_t)warps : 0);  // control words + per-warp cap histograms
  if (shared_in_smem) b += 4 * ((size_t)n * 2 + (size_t)n + 1);
  if (bits_in_smem) b += 4 * nwords * (size_t)warps;
  return (b + 15) & ~(size_t)15;
}

// INC = false: complete LU (drop 0, no cap) -- the drop tests, keep flags
// and cap selection compile away.
// MULTI = true: one system spans a.cps CTAs (large systems: c3, the c5
// block-Jacobi blocks).  Warp gw = cta * Wl + wid of the system owns columns
// gw, gw + W, ... with W = cps * Wl; the finished-column counter and abort
// flag live in global memory (a.gctl), exchanges are GPU-scope, and the
// CTA-wide init / finish steps run as separate kernels.
template <int MAXT, int MINB, bool INC, bool MULTI>
__global__ void __launch_bounds__(MAXT, MINB) ilutp_pipeline_kernel(FactorArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int Wl = blockDim.x >> 5;
  const int cps = MULTI ? a.cps : 1;
  const int b = MULTI ? blockIdx.x / cps : blockIdx.x + a.b0;
  const int wid = MULTI ? (blockIdx.x % cps) * Wl + (threadIdx.x >> 5) : (threadIdx.x >> 5);
  const int lw = threadIdx.x >> 5;  // warp index inside this CTA (shared-memory slices)
  const int W = Wl * cps;
  auto vload = [](const int32_t* p) { return vload_<MULTI>(p); };
#define FENCE() (MULTI ? __threadfence() : RS_FENCE_CTA())
  // L columns written by another SM must not be served from a stale L1 line
  auto ldL = [](const auto* p) { return MULTI ? __ldcg(p) : *p; };
  auto vstore = [](int32_t* p, int v) { vstore_<MULTI>(p, v); };
  const int32_t n = a.n;
  const int nwords = (n + 31) >> 5;
  int32_t* state = a.state + 3 * (int64_t)b;
  const int st0 = state[0];
  if (st0 == FAC_DONE || st0 == FAC_ZERO_PIVOT) return;
  const int k0 = (st0 == FAC_OVERFLOW) ? state[1] : 0;

  const int64_t bn = (int64_t)b * n;
  int32_t* gLp = a.Lp + (int64_t)b * (n + 1);
  int32_t* gUp = a.Up + (int64_t)b * (n + 1);
  int32_t* Li = a.Li + (int64_t)b * a.capL;
  double2* Lx = a.Lx + (int64_t)b * a.capL;
  int32_t* Ui = a.Ui + (int64_t)b * a.capU;
  double2* Ux = a.Ux + (int64_t)b * a.capU;
  int32_t* gpinv = a.pinv + bn;
  const double* rn = a.rn ? a.rn + bn : nullptr;
  const int32_t* Ap = a.Ap + bn;
  const double drop = INC ? a.drop_tol : 0.0;

  // control words: ctl[0] = number of finished columns, ctl[1] = abort
  volatile int32_t* ctl = MULTI ? reinterpret_cast<volatile int32_t*>(a.gctl + 2 * (int64_t)b)
                                : reinterpret_cast<volatile int32_t*>(smem);
  // after the per-warp cap histograms (complete LU launched without them: a.hist = 0)
  unsigned char* sp = smem + 64 + (a.hist ? 1024 * (size_t)Wl : 0);
  int32_t *pinv, *prow, *Lp;
  if (a.smem_mode) {
    pinv = reinterpret_cast<int32_t*>(sp);
    prow = pinv + n;
    Lp = prow + n;
    sp += 4 * ((size_t)n * 2 + (size_t)n + 1);
  } else {
    pinv = gpinv;
    prow = a.prow + bn;
    Lp = gLp;
  }
  uint32_t* bits;
  if (a.bits_in_smem) bits = reinterpret_cast<uint32_t*>(sp) + (size_t)lw * nwords;
  else bits = a.wbits + ((int64_t)b * W + wid) * nwords;

  // per-warp private scratch (global, L1/L2 resident)
  const int64_t ws = ((int64_t)b * W + wid) * n;
  double2* x = a.wx + ws;
  int32_t* flag = a.wflag + ws;
  int32_t* pat = a.wpat + ws;
  int32_t* urow = a.wurow + ws;
  double2* uval = a.wuval + ws;
  int32_t* lrow = a.wlrow + ws;
  uint8_t* ukeep = a.wukeep + ws;
  uint8_t* lkeep = a.wlkeep + ws;
  uint64_t* keys = a.wkey + ws;
  unsigned* hist = reinterpret_cast<unsigned*>(smem + 64) + 256 * lw;

  // ---- init -----------------------------------------------------------------
  if (!MULTI) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      if (k0 == 0) gpinv[i] = -1;
      prow[i] = -1;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const int pv = gpinv[i];
      if (a.smem_mode) pinv[i] = pv;
      if (pv >= 0) prow[pv] = i;  // resume after overflow: prow = pinv^-1
    }
    if (a.smem_mode)
      for (int i = threadIdx.x; i <= n; i += blockDim.x) Lp[i] = (i <= k0) ? gLp[i] : 0;
  }
  for (int i = lane; i < n; i += 32) flag[i] = -1;
  for (int w = lane; w < nwords; w += 32) bits[w] = 0u;
  if (!MULTI && threadIdx.x == 0) {
    ctl[0] = k0;
    ctl[1] = 0;
    if (k0 == 0) {
      gLp[0] = 0;
      gUp[0] = 0;
      Lp[0] = 0;
    }
  }
  FENCE();
  __syncthreads();
  const int fill_cap = a.fill_caps ? a.fill_caps[b] : a.fill_cap;
  const bool have_cap = INC && fill_cap >= 0;

  // round-robin columns, starting at the resume point
  for (int k = k0 + wid; k < n; k += W) {
    const int j = a.q ? a.q[bn + k] : k;
    int scanned = ctl[0];
    __syncwarp();
    if (ctl[1]) break;
    FENCE();
    unsigned long long* const pr = (b == 0) ? a.probe : nullptr;
    probe_mark(pr, k, 0, lane);
    // ---- 1. scatter column j; seed pending with columns already finished --
    const int32_t c0 = Ap[j], c1 = Ap[j + 1];
    int npat = c1 - c0;
    int lowc = 0x7fffffff;
    for (int e = c0 + lane; e < c1; e += 32) {
      const int i = a.Ai[e];
      x[i] = a.Ax[e];
      flag[i] = k;
      pat[e - c0] = i;
      const int pv = vload(pinv + i);
      if (pv >= 0 && pv < scanned) {
        atomicOr(&bits[pv >> 5], 1u << (pv & 31));
        lowc = min(lowc, pv);
      }
    }
    lowc = warp_min_i(lowc);
    __syncwarp();

    // ---- 2. updates in ascending pivotal order, gated by the frontier -----
    int unum = 0;
    int kept_u = 0;
    int w = (lowc == 0x7fffffff) ? ((scanned + 31) >> 5) : (lowc >> 5);
    bool aborted = false;
    // first chunk of the next pending column, fetched while the current one
    // is applied (L columns are immutable once published)
    int pre_c = -1, pre_i = 0;
    double2 pre_v = make_double2(0.0, 0.0);
    uint32_t cur_word = 0;
    while (true) {
      const int wend = (scanned + 31) >> 5;
      int c = -1;
      while (w < wend) {
        const int ww = w + lane;
        const uint32_t bv = (ww < wend) ? bits[ww] : 0u;
        const unsigned m = __ballot_sync(FULL, bv != 0u);
        if (m) {
          const int src = __ffs(m) - 1;
          const uint32_t word = __shfl_sync(FULL, bv, src);
          w += src;
          c = (w << 5) + __ffs(word) - 1;
          cur_word = word;
          break;
        }
        w += 32;
      }
      if (c < 0) {
        if (scanned == k) break;
        // advance the frontier over newly finished columns
        int d;
        // the warp owning the next column to finish spins hot; the others
        // back off so they do not steal issue slots from the critical tail
        // nap length grows with the distance to this column's turn
        const int dist = k - scanned - 1;
        const unsigned nap =
            dist <= 0 ? (unsigned)a.hot_nap : (dist < 4 ? a.nap_step * dist : 8u * a.nap_step);
        while ((d = ctl[0]) == scanned && !ctl[1]) {
          if (nap) __nanosleep(nap);
        }
        if (ctl[1]) {
          aborted = true;
          break;
        }
        FENCE();
        int newlow = 0x7fffffff;
        for (int m = scanned + lane; m < d; m += 32) {
          const int r = vload(prow + m);
          if (flag[r] == k) {
            atomicOr(&bits[m >> 5], 1u << (m & 31));
            newlow = min(newlow, m);
          }
        }
        newlow = warp_min_i(newlow);
        __syncwarp();
        w = (newlow == 0x7fffffff) ? ((d + 31) >> 5) : (newlow >> 5);
        scanned = d;
        continue;
      }
      const int pr = vload(prow + c);
      const double2 xc = x[pr];
      const double rnc = (drop > 0.0) ? rn[pr] : 0.0;
      const int32_t p0 = vload(Lp + c) + 1, p1 = vload(Lp + c + 1);
      const bool use_pre = (pre_c == c);
      const int my_pre_i = pre_i;
      const double2 my_pre_v = pre_v;
      {  // prefetch the next pending column below the frontier (same word)
        const uint32_t rest = cur_word & ~((2u << (c & 31)) - 1u);
        pre_c = -1;
        if (rest) {
          const int cn = (w << 5) + __ffs(rest) - 1;
          const int q0 = vload(Lp + cn) + 1 + lane, q1 = vload(Lp + cn + 1);
          pre_c = cn;
          if (q0 < q1) {
            pre_i = ldL(Li + q0);
            pre_v = ldL(Lx + q0);
          }
        }
      }
      // U entry for c: its value is final now, so its drop test is decided
      // here instead of on the column's critical tail
      const bool ukk = !(drop > 0.0 && cabs1(xc) < drop * rnc);
      __syncwarp();
      if (INC && a.early_drop && !ukk) {
        // opt-in Saad-ILUT rule (not the reference's): an entry the drop rule
        // discards is discarded before it eliminates anything
        if (lane == 0) atomicAnd(&bits[w], ~(1u << (c & 31)));
        __syncwarp();
        continue;
      }
      if (lane == 0) {
        atomicAnd(&bits[w], ~(1u << (c & 31)));
        urow[unum] = c;
        uval[unum] = xc;
        if (INC) ukeep[unum] = ukk;
      }
      ++unum;
      kept_u += ukk;
      // apply L[:,c] in blocks of 64 entries: all loads of a block are issued
      // before any is consumed (one memory latency per block, not per entry)
      for (int base = p0; base < p1; base += 64) {
        const int pa = base + lane, pb = pa + 32;
        const bool acta = pa < p1, actb = pb < p1;
        int ia = 0, ib = 0;
        double2 la = make_double2(0.0, 0.0), lb = la;
        if (acta) {
          if (use_pre && base == p0) {
            ia = my_pre_i;
            la = my_pre_v;
          } else {
            ia = ldL(Li + pa);
            la = ldL(Lx + pa);
          }
        }
        if (actb) {
          ib = ldL(Li + pb);
          lb = ldL(Lx + pb);
        }
        const int fa = acta ? flag[ia] : k, fb = actb ? flag[ib] : k;
        double2 xa = acta ? x[ia] : la, xb = actb ? x[ib] : lb;
        const int va = acta ? vload(pinv + ia) : -1, vb = actb ? vload(pinv + ib) : -1;
        const bool newa = acta && fa != k, newb = actb && fb != k;
        const unsigned ma = __ballot_sync(FULL, newa);
        const unsigned mb = __ballot_sync(FULL, newb);
        const unsigned lt = lanemask_lt();
        if (newa) {
          flag[ia] = k;
          xa = make_double2(0.0, 0.0);
          pat[npat + __popc(ma & lt)] = ia;
          if (va >= 0 && va < scanned) atomicOr(&bits[va >> 5], 1u << (va & 31));
        }
        npat += __popc(ma);
        if (newb) {
          flag[ib] = k;
          xb = make_double2(0.0, 0.0);
          pat[npat + __popc(mb & lt)] = ib;
          if (vb >= 0 && vb < scanned) atomicOr(&bits[vb >> 5], 1u << (vb & 31));
        }
        npat += __popc(mb);
        if (acta) x[ia] = csub(xa, cmul_plain(la, xc));
        if (actb) x[ib] = csub(xb, cmul_plain(lb, xc));
      }
      __syncwarp();
    }
    if (aborted) break;
    FENCE();  // acquire: every column < k is final
    probe_mark(pr, k, 1, lane);

    // ---- 3+4. pivot (max |re|+|im| over non-pivotal rows, ties -> lowest
    // row) fused with the L drop test, 256 pattern entries per load batch -
    double best = -1.0;
    int ipiv = -1, ipos = -1, ikeep = 0;
    int lnum = 0, kept_l = 0;
    for (int blk = 0; blk < npat; blk += 256) {
      int iu[8], pv[8];
      double2 xv[8];
      double rv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = blk + 32 * u + lane;
        iu[u] = t < npat ? pat[t] : -1;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool act = iu[u] >= 0;
        pv[u] = act ? vload(pinv + iu[u]) : 0;
        xv[u] = act ? x[iu[u]] : make_double2(0.0, 0.0);
        rv[u] = (act && drop > 0.0) ? rn[iu[u]] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = iu[u];
        const bool cand = i >= 0 && pv[u] < 0;
        const unsigned cm = __ballot_sync(FULL, cand);
        if (cand) {
          const int pos = lnum + __popc(cm & lanemask_lt());
          const double mag = cabs1(xv[u]);
          const bool keep = !(drop > 0.0 && mag < drop * rv[u]);
          lrow[pos] = i;
          if (INC) lkeep[pos] = keep;
          kept_l += keep;
          if (mag > best || (mag == best && i < ipiv)) {
            best = mag;
            ipiv = i;
            ipos = pos;
            ikeep = keep;
          }
        }
        lnum += __popc(cm);
      }
    }
    double gbest = best;
    int gipiv = ipiv;
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(FULL, gbest, o);
      const int oi = __shfl_xor_sync(FULL, gipiv, o);
      if (ob > gbest || (ob == gbest && oi >= 0 && (gipiv < 0 || oi < gipiv))) {
        gbest = ob;
        gipiv = oi;
      }
    }
    if (gipiv < 0 || gbest == 0.0) {
      if (!(a.pivot_floor > 0.0)) {
        if (lane == 0) {
          state[0] = FAC_ZERO_PIVOT;
          state[1] = k;
          ctl[1] = 1;
        }
        break;
      }
      // Opt-in remedy (not in the reference; the block-Jacobi preconditioner
      // of config 5 asks for it): a column with no usable pivot takes the
      // value pivot_floor on the row the reference's tie rule names (the
      // lowest non-pivotal pattern row), or -- when every pattern row is
      // already pivotal -- on the lowest row not yet pivotal, which joins
      // the pattern.  Every column < k is final here, so pinv is exact.
      if (gipiv < 0) {
        int r = 0x7fffffff;
        for (int base = 0; base < n && r == 0x7fffffff; base += 32) {
          const int i = base + lane;
          const bool open = i < n && vload(pinv + i) < 0;
          const unsigned m = __ballot_sync(FULL, open);
          if (m) r = base + __ffs(m) - 1;
        }
        gipiv = r;
        ipiv = -1;
        ipos = -1;
        if (lane == 0) {
          lrow[lnum] = r;
          if (INC) lkeep[lnum] = 0;
          flag[r] = k;
          ipiv = r;
          ipos = lnum;
          ikeep = 0;
        }
        lnum += 1;
      }
      if (lane == 0) {
        x[gipiv] = make_double2(a.pivot_floor, 0.0);
        atomicAdd(&state[2], 1);  // substituted pivots of this system
      }
      __syncwarp();
    }
    // the pivot row is never an L entry: the owning lane clears its keep
    const bool owner = (ipiv == gipiv) && ipos >= 0;
    if (INC && owner) lkeep[ipos] = 0;
    const unsigned om = __ballot_sync(FULL, owner && ikeep);
    kept_l = warp_sum_i(kept_l) - (om ? 1 : 0);
    ipiv = gipiv;
    const double2 piv = x[ipiv];
    __syncwarp();
    probe_mark(pr, k, 2, lane);
    probe_mark(pr, k, 3, lane);

    // ---- 5. fill cap: keep the best (cap-2) by (-mag, U-before-L, index) --
    // Exact top-k: an 8-bit radix select over the magnitude bit patterns
    // (non-negative doubles order like their bits) finds the allowed-th
    // largest key T; ties at T (rare) are resolved by (U-before-L, index)
    // with a bitwise select over the tied candidates only.
    if (have_cap && kept_u + kept_l + 2 > fill_cap && kept_u + kept_l > 0) {
      const int ncand = kept_u + kept_l;
      int allowed = fill_cap - 2;
      if (allowed < 0) allowed = 0;
      if (allowed > ncand) allowed = ncand;
      uint64_t* key = keys;  // [0, unum): U candidates, [unum, unum + lnum): L
      for (int t = lane; t < unum; t += 32) key[t] = ukeep[t] ? mag_key(uval[t]) : ~0ull;
      for (int t = lane; t < lnum; t += 32)
        key[unum + t] = lkeep[t] ? mag_key(x[lrow[t]]) : ~0ull;
      __syncwarp();
      const int ntot = unum + lnum;
      uint64_t T = 0;
      uint32_t S = 0xffffffffu;
      if (allowed > 0) {
        uint64_t prefix = 0, pmask = 0;
        int remaining = allowed;
        for (int shift = 56; shift >= 0; shift -= 8) {
          for (int j = lane; j < 256; j += 32) hist[j] = 0;
          __syncwarp();
          for (int t = lane; t < ntot; t += 32) {
            const uint64_t kk = key[t];
            if (kk != ~0ull && (kk & pmask) == prefix) atomicAdd(&hist[(kk >> shift) & 255], 1u);
          }
          __syncwarp();
          // lane l owns digits 255-8l .. 248-8l (high digits first)
          unsigned c8[8], tot = 0;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            c8[j] = hist[255 - 8 * lane - j];
            tot += c8[j];
          }
          unsigned incl = tot;  // inclusive scan over lanes (high digits first)
          for (int o = 1; o < 32; o <<= 1) {
            const unsigned v = __shfl_up_sync(FULL, incl, o);
            if (lane >= o) incl += v;
          }
          const unsigned excl = incl - tot;
          int digit = -1;
          unsigned above = 0;
          if (excl < (unsigned)remaining && (unsigned)remaining <= incl) {
            unsigned run = excl;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              if (digit < 0 && run + c8[j] >= (unsigned)remaining) {
                digit = 255 - 8 * lane - j;
                above = run;
              }
              run += c8[j];
            }
          }
          const unsigned hit = __ballot_sync(FULL, digit >= 0);
          const int src = __ffs(hit) - 1;
          digit = __shfl_sync(FULL, digit, src);
          above = __shfl_sync(FULL, above, src);
          remaining -= (int)above;
          prefix |= (uint64_t)digit << shift;
          pmask |= 255ull << shift;
          __syncwarp();
        }
        T = prefix;
        int gt = 0, ties = 0;
        for (int t = lane; t < ntot; t += 32) {
          const uint64_t kk = key[t];
          if (kk != ~0ull) {
            gt += kk > T;
            ties += kk == T;
          }
        }
        gt = warp_sum_i(gt);
        ties = warp_sum_i(ties);
        const int need = allowed - gt;  // >= 1 ties at T to take
        if (ties > need) {
          // secondary key (dom<<31 | idx), smallest first, among the ties
          S = 0;
          for (int bit = 31; bit >= 0; --bit) {
            const uint32_t cand = S | (1u << bit);
            int cnt = 0;
            for (int t = lane; t < unum; t += 32)
              cnt += (key[t] == T && (uint32_t)urow[t] < cand);
            for (int t = lane; t < lnum; t += 32)
              cnt += (key[unum + t] == T && ((1u << 31) | (uint32_t)lrow[t]) < cand);
            cnt = warp_sum_i(cnt);
            if (cnt < need) S = cand;
          }
        }
      }
      kept_u = 0;
      kept_l = 0;
      for (int t = lane; t < unum; t += 32) {
        const uint64_t kk = key[t];
        const bool keep = allowed > 0 && kk != ~0ull &&
                          (kk > T || (kk == T && (uint32_t)urow[t] <= S));
        ukeep[t] = keep;
        kept_u += keep;
      }
      for (int t = lane; t < lnum; t += 32) {
        const uint64_t kk = key[unum + t];
        const bool keep = allowed > 0 && kk != ~0ull &&
                          (kk > T || (kk == T && ((1u << 31) | (uint32_t)lrow[t]) <= S));
        lkeep[t] = keep;
        kept_l += keep;
      }
      kept_u = warp_sum_i(kept_u);
      kept_l = warp_sum_i(kept_l);
      __syncwarp();
    }

    // ---- 6. emit L (unit diagonal first), publish the column, then U ------
    const int32_t lnnz = vload(Lp + k);
    const int32_t unnz = vload(gUp + k);
    if ((int64_t)unnz + kept_u + 1 > a.capU || (int64_t)lnnz + kept_l + 1 > a.capL) {
      if (lane == 0) {
        state[0] = FAC_OVERFLOW;
        state[1] = k;
        ctl[1] = 1;
      }
      break;
    }
    const double2 rp = recipc(piv);
    if (lane == 0) {
      Li[lnnz] = ipiv;
      Lx[lnnz] = make_double2(1.0, 0.0);
    }
    int off = lnnz + 1;
    for (int blk = 0; blk < lnum; blk += 256) {
      int ir[8];
      bool kp[8];
      double2 xv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = blk + 32 * u + lane;
        const bool act = t < lnum;
        ir[u] = act ? lrow[t] : 0;
        kp[u] = act && (INC ? lkeep[t] != 0 : ir[u] != ipiv);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) xv[u] = kp[u] ? x[ir[u]] : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const unsigned m = __ballot_sync(FULL, kp[u]);
        if (kp[u]) {
          const int o = off + __popc(m & lanemask_lt());
          Li[o] = ir[u];
          Lx[o] = cmul_plain(xv[u], rp);
        }
        off += __popc(m);
      }
    }
    const int32_t unew = unnz + kept_u + 1;
    FENCE();
    __syncwarp();
    if (lane == 0) {
      vstore(gUp + k + 1, unew);
      vstore(gLp + k + 1, off);
      if (a.smem_mode) vstore(Lp + k + 1, off);
      vstore(pinv + ipiv, k);
      if (a.smem_mode) gpinv[ipiv] = k;
      vstore(prow + k, ipiv);
      FENCE();  // release column k
      ctl[0] = k + 1;
    }
    probe_mark(pr, k, 4, lane);
    // U column k (kept rows ascending, pivot last): not read by later
    // columns, so it is written after the release, off the critical path
    int uo = unnz;
    for (int base = 0; base < unum; base += 32) {
      const int t = base + lane;
      const bool keep = t < unum && (INC ? ukeep[t] != 0 : true);
      const unsigned m = __ballot_sync(FULL, keep);
      if (keep) {
        const int o = uo + __popc(m & lanemask_lt());
        Ui[o] = urow[t];
        Ux[o] = uval[t];
      }
      uo += __popc(m);
    }
    if (lane == 0) {
      Ui[uo] = k;
      Ux[uo] = piv;
    }
    __syncwarp();
  }
  if (MULTI) return;  // finish runs as ilutp_multi_finish_kernel
  __syncthreads();
  if (ctl[1]) return;  // zero pivot or overflow: state already recorded
  // ---- finish: remap L rows to pivotal indices ------------------------------
  const int32_t lnnz = gLp[n];
  for (int p = threadIdx.x; p < lnnz; p += blockDim.x) Li[p] = pinv[Li[p]];
  if (threadIdx.x == 0) {
    state[0] = FAC_DONE;
    state[1] = -1;
  }
}

// MULTI init, pass 1: reset pinv (fresh start) and prow of unfinished systems
__global__ void ilutp_multi_init1_kernel(FactorArgs a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)a.B * a.n) return;
  const int64_t b = t / a.n;
  const int st0 = a.state[3 * b];
  if (st0 == FAC_DONE || st0 == FAC_ZERO_PIVOT) return;
  if (st0 != FAC_OVERFLOW) a.pinv[t] = -1;
  a.prow[t] = -1;
}
// pass 2: prow = pinv^-1 (resume after overflow), control words, Lp/Up[0]
__global__ void ilutp_multi_init2_kernel(FactorArgs a) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)a.B * a.n) return;
  const int64_t b = t / a.n, i = t % a.n;
  const int st0 = a.state[3 * b];
  if (st0 == FAC_DONE || st0 == FAC_ZERO_PIVOT) return;
  const int pv = a.pinv[t];
  if (pv >= 0) a.prow[b * a.n + pv] = (int32_t)i;
  if (i == 0) {
    const int k0 = st0 == FAC_OVERFLOW ? a.state[3 * b + 1] : 0;
    a.gctl[2 * b] = k0;
    a.gctl[2 * b + 1] = 0;
    if (k0 == 0) {
      a.Lp[b * (a.n + 1)] = 0;
      a.Up[b * (a.n + 1)] = 0;
    }
  }
}
// finish: remap L rows to pivotal indices for systems that completed
__global__ void ilutp_multi_finish_kernel(FactorArgs a) {
  const int b = blockIdx.y;
  const int st0 = a.state[3 * b];
  if (st0 == FAC_DONE || st0 == FAC_ZERO_PIVOT || a.gctl[2 * b + 1]) return;
  const int32_t lnnz = a.Lp[(int64_t)b * (a.n + 1) + a.n];
  int32_t* Li = a.Li + (int64_t)b * a.capL;
  const int32_t* pinv = a.pinv + (int64_t)b * a.n;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < lnnz;
       p += (int64_t)gridDim.x * blockDim.x)
    Li[p] = pinv[Li[p]];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.state[3 * b] = FAC_DONE;
    a.state[3 * b + 1] = -1;
  }
}

static int launch_ilutp_multi(const FactorArgs& a, size_t smem, cudaStream_t st) {
  const int64_t N = (int64_t)a.B * a.n;
  const unsigned g = (unsigned)((N + 255) / 256);
  ilutp_multi_init1_kernel<<<g, 256, 0, st>>>(a);
  ::rs::count_launch();
  ilutp_multi_init2_kernel<<<g, 256, 0, st>>>(a);
  ::rs::count_launch();
  const bool inc = a.drop_tol > 0.0 || a.fill_cap >= 0 || a.fill_caps != nullptr;
  void* kern = inc ? (void*)ilutp_pipeline_kernel<512, 1, true, true>
                   : (void*)ilutp_pipeline_kernel<512, 1, false, true>;
  RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  // every CTA of a system waits on the others: cooperative launch guarantees
  // they are co-resident
  FactorArgs aa = a;
  {  // never ask for more co-resident CTAs than the device holds
    int per_sm = 0, dev = 0, sms = 0;
    RS_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 32 * a.warps, smem));
    RS_CUDA_TRY(cudaGetDevice(&dev));
    RS_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int cap = per_sm * sms;
    if (a.B > cap) {
      set_error("multi-CTA factorization: %d systems exceed %d co-resident CTAs", a.B, cap);
      return RS_ERR_UNSUPPORTED;
    }
    if (aa.B * aa.cps > cap) aa.cps = cap / aa.B;
  }
  void* args[] = {&aa};
  RS_CUDA_TRY(cudaLaunchCooperativeKernel(kern, dim3((unsigned)(aa.B * aa.cps)), dim3(32 * a.warps),
                                          args, smem, st));
  ::rs::count_launch();
  ilutp_multi_finish_kernel<<<dim3(64, (unsigned)a.B), 256, 0, st>>>(a);
  ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

int launch_ilutp(const FactorArgs& a, cudaStream_t st) {
  if (a.B == 0 || a.n == 0) return RS_OK;
  const int W = a.warps;
  const size_t smem = ilutp_smem_bytes(a.n, W, a.smem_mode, a.bits_in_smem, a.hist);
  if (a.cps > 1) return launch_ilutp_multi(a, smem, st);
  // one instantiation per block size so each gets its full register budget
  // (a 1024-thread bound caps registers at 64 and spills the tail loops)
  auto launch = [&](auto kern) -> int {
    RS_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
    kern<<<a.B, 32 * W, smem, st>>>(a);
    ::rs::count_launch();
    return RS_OK;
  };
  // batches: keep 4 systems per SM resident (512 systems ~ one wave)
  // (a launch with a system offset shares its SMs with the frontal kernel:
  // always the 64-register build)
  const bool batch = a.B > 148 || a.b0 > 0;
  int rc;
  (void)0;
  const bool inc = a.drop_tol > 0.0 || a.fill_cap >= 0 || a.fill_caps != nullptr;
  auto pick = [&](auto kc, auto ki) -> int { return inc ? launch(ki) : launch(kc); };
  if (W <= 4)
    rc = batch ? pick(ilutp_pipeline_kernel<128, 4, false, false>, ilutp_pipeline_kernel<128, 4, true, false>)
               : pick(ilutp_pipeline_kernel<128, 1, false, false>, ilutp_pipeline_kernel<128, 1, true, false>);
  else if (W <= 6)
    rc = batch ? pick(ilutp_pipeline_kernel<192, 4, false, false>, ilutp_pipeline_kernel<192, 4, true, false>)
               : pick(ilutp_pipeline_kernel<192, 1, false, false>, ilutp_pipeline_kernel<192, 1, true, false>);
  else if (W <= 8)
    rc = batch ? pick(ilutp_pipeline_kernel<256, 4, false, false>, ilutp_pipeline_kernel<256, 4, true, false>)
               : pick(ilutp_pipeline_kernel<256, 1, false, false>, ilutp_pipeline_kernel<256, 1, true, false>);
  else if (W <= 16)
    rc = pick(ilutp_pipeline_kernel<512, 1, false, false>, ilutp_pipeline_kernel<512, 1, true, false>);
  else
    rc = pick(ilutp_pipeline_kernel<1024, 1, false, false>, ilutp_pipeline_kernel<1024, 1, true, false>);
  if (rc) return rc;
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

int ilutp_plan(int32_t n, int warps, int* smem_mode, int* bits_in_smem) {
  int dev = 0, max_smem = 0;
  RS_CUDA_TRY(cudaGetDevice(&dev));
  RS_CUDA_TRY(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  // keep ~96 KB of the carveout as L1 for the per-warp accumulators
  const size_t budget = (size_t)max_smem > 131072 ? (size_t)max_smem - 98304 : 32768;
  *bits_in_smem = ilutp_smem_bytes(n, warps, 0, 1, 1) <= budget;
  *smem_mode = ilutp_smem_bytes(n, warps, 1, *bits_in_smem, 1) <= budget;
  return RS_OK;
}

}  // namespace rs
