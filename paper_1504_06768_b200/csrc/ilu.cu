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
// multiply-subtract each.  Here the same ascending order comes from scanning a
// bitmap of pending pivotal columns; the entries of one L column touch
// distinct rows, so a warp applies them in parallel without changing any
// rounding.  Newly reached rows are appended to the pattern in the
// reference's discovery order (ballot + prefix), so even the raw CSC output
// (column-internal order included) matches the reference.
//
// B200 mapping: column k depends on every earlier pivot choice, so the
// elimination is inherently column-sequential.  One warp owns one system and
// runs warp-synchronously (no CTA barriers on the per-pop critical path);
// x, the touched-row flags, pinv, prow, Lp and the pending bitmap sit in
// shared memory when 32 B/row fits (n <= ~7000: configs 1, 2, 4), otherwise
// in L2-resident global scratch.  A batch of B systems (the config-4 sweep)
// runs one warp per system across the SMs.
//
// Storage: with a cap, nnz(L)+nnz(U) <= n*cap, so the caller preallocates;
// complete LU (cap = -1) may overflow, in which case the kernel stops before
// column k, records it, and the host grows the buffers and resumes.
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

struct SysPtrs {
  double2* x;
  int32_t* flag;
  int32_t* pinv;
  int32_t* prow;
  int32_t* Lp;  // shadow of Lp (smem mode) or the output itself
  uint32_t* bits;
};

}  // namespace

__host__ __device__ size_t ilutp_smem_per_system(int32_t n) {
  const size_t nwords = ((size_t)n + 31) / 32;
  size_t bytes = 16 * (size_t)n + 4 * (size_t)n * 3 + 4 * ((size_t)n + 1) +
                 4 * nwords;
  return (bytes + 15) & ~(size_t)15;
}

__global__ void ilutp_warp_kernel(FactorArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  const int wid = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int b = blockIdx.x * wpb + wid;
  if (b >= a.B) return;
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
  int32_t* gprow = a.prow + bn;
  int32_t* pat = a.wpat + bn;
  int32_t* urow = a.wurow + bn;
  double2* uval = a.wuval + bn;
  int32_t* lrow = a.wlrow + bn;
  uint8_t* ukeep = a.wukeep + bn;
  uint8_t* lkeep = a.wlkeep + bn;
  const double* rn = a.rn ? a.rn + bn : nullptr;
  const int32_t* Ap = a.Ap + bn;
  const double drop = a.drop_tol;

  SysPtrs s;
  if (a.smem_mode) {
    unsigned char* base = smem + (size_t)wid * ilutp_smem_per_system(n);
    s.x = reinterpret_cast<double2*>(base);
    s.flag = reinterpret_cast<int32_t*>(s.x + n);
    s.pinv = s.flag + n;
    s.prow = s.pinv + n;
    s.Lp = s.prow + n;
    s.bits = reinterpret_cast<uint32_t*>(s.Lp + n + 1);
    for (int i = lane; i < n; i += 32) {
      s.flag[i] = -1;
      s.pinv[i] = k0 ? gpinv[i] : -1;
      s.prow[i] = -1;
    }
    for (int i = lane; i <= n; i += 32) s.Lp[i] = (i <= k0) ? gLp[i] : 0;
  } else {
    s.x = a.wx + bn;
    s.flag = a.wflag + bn;
    s.pinv = gpinv;
    s.prow = gprow;
    s.Lp = gLp;
    s.bits = a.wbits + (int64_t)b * nwords;
    for (int i = lane; i < n; i += 32) {
      s.flag[i] = -1;
      if (!k0) s.pinv[i] = -1;
      s.prow[i] = -1;
    }
  }
  __syncwarp();
  if (k0) {  // resumed after a capacity overflow: prow is the inverse of pinv
    for (int i = lane; i < n; i += 32) {
      const int pv = s.pinv[i];
      if (pv >= 0) s.prow[pv] = i;
    }
  }
  for (int w = lane; w < nwords; w += 32) s.bits[w] = 0u;
  if (k0 == 0 && lane == 0) {
    gLp[0] = 0;
    gUp[0] = 0;
    s.Lp[0] = 0;
  }
  __syncwarp();
  int32_t lnnz = k0 ? gLp[k0] : 0;
  int32_t unnz = k0 ? gUp[k0] : 0;
  const bool have_cap = a.fill_cap >= 0;

  for (int k = k0; k < n; ++k) {
    const int j = a.q ? a.q[bn + k] : k;
    // ---- 1. scatter column j, seed the pending set ------------------------
    const int32_t c0 = Ap[j], c1 = Ap[j + 1];
    int npat = c1 - c0;
    int lowc = 0x7fffffff;
    for (int e = c0 + lane; e < c1; e += 32) {
      const int i = a.Ai[e];
      s.x[i] = a.Ax[e];
      s.flag[i] = k;
      pat[e - c0] = i;
      const int pv = s.pinv[i];
      if (pv >= 0) {
        atomicOr(&s.bits[pv >> 5], 1u << (pv & 31));
        lowc = min(lowc, pv);
      }
    }
    lowc = warp_min_i(lowc);
    __syncwarp();

    // ---- 2. left-looking updates in ascending pivotal order ---------------
    int unum = 0;
    const int wend = (k + 31) >> 5;
    int w = (lowc == 0x7fffffff) ? wend : (lowc >> 5);
    while (true) {
      int c = -1;
      while (w < wend) {
        const int ww = w + lane;
        const uint32_t bv = (ww < wend) ? s.bits[ww] : 0u;
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
      if (c < 0) break;
      const int pr = s.prow[c];
      const double2 xc = s.x[pr];
      const int32_t p0 = s.Lp[c] + 1, p1 = s.Lp[c + 1];
      __syncwarp();
      if (lane == 0) {
        atomicAnd(&s.bits[w], ~(1u << (c & 31)));
        urow[unum] = c;
        uval[unum] = xc;
      }
      ++unum;
      for (int base = p0; base < p1; base += 32) {
        const int p = base + lane;
        const bool act = p < p1;
        int i = 0;
        double2 lv = make_double2(0.0, 0.0);
        bool isnew = false;
        if (act) {
          i = Li[p];
          lv = Lx[p];
          isnew = s.flag[i] != k;
        }
        const unsigned nm = __ballot_sync(FULL, isnew);
        if (act) {
          double2 xi;
          if (isnew) {
            s.flag[i] = k;
            xi = make_double2(0.0, 0.0);
            pat[npat + __popc(nm & lanemask_lt())] = i;
            const int pv = s.pinv[i];
            if (pv >= 0) atomicOr(&s.bits[pv >> 5], 1u << (pv & 31));
          } else {
            xi = s.x[i];
          }
          s.x[i] = csub(xi, cmul_plain(lv, xc));
        }
        npat += __popc(nm);
      }
      __syncwarp();
    }

    // ---- 3. pivot: max |re|+|im| over non-pivotal rows, ties -> lowest row -
    double best = -1.0;
    int ipiv = -1;
    int lnum = 0;
    for (int base = 0; base < npat; base += 32) {
      const int t = base + lane;
      const bool act = t < npat;
      const int i = act ? pat[t] : 0;
      const bool cand = act && s.pinv[i] < 0;
      const unsigned cm = __ballot_sync(FULL, cand);
      if (cand) {
        lrow[lnum + __popc(cm & lanemask_lt())] = i;
        const double mag = cabs1(s.x[i]);
        if (mag > best || (mag == best && i < ipiv)) {
          best = mag;
          ipiv = i;
        }
      }
      lnum += __popc(cm);
    }
    for (int o = 16; o; o >>= 1) {
      const double ob = __shfl_xor_sync(FULL, best, o);
      const int oi = __shfl_xor_sync(FULL, ipiv, o);
      if (ob > best || (ob == best && oi >= 0 && (ipiv < 0 || oi < ipiv))) {
        best = ob;
        ipiv = oi;
      }
    }
    if (ipiv < 0 || best == 0.0) {
      if (lane == 0) {
        state[0] = FAC_ZERO_PIVOT;
        state[1] = k;
      }
      if (a.smem_mode) {
        for (int i = lane; i < n; i += 32) {
          gpinv[i] = s.pinv[i];
          gprow[i] = s.prow[i];
        }
      }
      return;
    }
    const double2 piv = s.x[ipiv];
    __syncwarp();

    // ---- 4. dropping ------------------------------------------------------
    int kept_u = 0, kept_l = 0;
    for (int t = lane; t < unum; t += 32) {
      bool keep = true;
      if (drop > 0.0 && cabs1(uval[t]) < drop * rn[s.prow[urow[t]]]) keep = false;
      ukeep[t] = keep;
      kept_u += keep;
    }
    for (int t = lane; t < lnum; t += 32) {
      const int i = lrow[t];
      bool keep = true;
      if (i == ipiv) keep = false;
      else if (drop > 0.0 && cabs1(s.x[i]) < drop * rn[i]) keep = false;
      lkeep[t] = keep;
      kept_l += keep;
    }
    kept_u = warp_sum_i(kept_u);
    kept_l = warp_sum_i(kept_l);
    __syncwarp();

    // ---- 5. fill cap: keep the best (cap-2) by (-mag, U-before-L, index) --
    if (have_cap && kept_u + kept_l + 2 > a.fill_cap && kept_u + kept_l > 0) {
      const int ncand = kept_u + kept_l;
      int allowed = a.fill_cap - 2;
      if (allowed < 0) allowed = 0;
      if (allowed > ncand) allowed = ncand;
      // Threshold T = allowed-th largest magnitude key (keys are the bit
      // patterns of non-negative doubles, so integer order == value order).
      uint64_t T = 0;
      uint32_t S = 0xffffffffu;
      if (allowed > 0) {
        for (int bit = 62; bit >= 0; --bit) {
          const uint64_t cand = T | (1ull << bit);
          int cnt = 0;
          for (int t = lane; t < unum; t += 32)
            cnt += (ukeep[t] && mag_key(uval[t]) >= cand);
          for (int t = lane; t < lnum; t += 32)
            cnt += (lkeep[t] && mag_key(s.x[lrow[t]]) >= cand);
          cnt = warp_sum_i(cnt);
          if (cnt >= allowed) T = cand;
        }
        int gt = 0;
        for (int t = lane; t < unum; t += 32) gt += (ukeep[t] && mag_key(uval[t]) > T);
        for (int t = lane; t < lnum; t += 32)
          gt += (lkeep[t] && mag_key(s.x[lrow[t]]) > T);
        gt = warp_sum_i(gt);
        const int need = allowed - gt;  // >= 1 ties at T to take
        // S = need-th smallest secondary key (dom<<31 | idx) among ties.
        S = 0;
        for (int bit = 31; bit >= 0; --bit) {
          const uint32_t cand = S | (1u << bit);
          int cnt = 0;
          for (int t = lane; t < unum; t += 32)
            cnt += (ukeep[t] && mag_key(uval[t]) == T && (uint32_t)urow[t] < cand);
          for (int t = lane; t < lnum; t += 32)
            cnt += (lkeep[t] && mag_key(s.x[lrow[t]]) == T &&
                    ((1u << 31) | (uint32_t)lrow[t]) < cand);
          cnt = warp_sum_i(cnt);
          if (cnt < need) S = cand;
        }
      }
      kept_u = 0;
      kept_l = 0;
      for (int t = lane; t < unum; t += 32) {
        bool keep = false;
        if (allowed > 0 && ukeep[t]) {
          const uint64_t kk = mag_key(uval[t]);
          keep = kk > T || (kk == T && (uint32_t)urow[t] <= S);
        }
        ukeep[t] = keep;
        kept_u += keep;
      }
      for (int t = lane; t < lnum; t += 32) {
        bool keep = false;
        if (allowed > 0 && lkeep[t]) {
          const uint64_t kk = mag_key(s.x[lrow[t]]);
          keep = kk > T || (kk == T && ((1u << 31) | (uint32_t)lrow[t]) <= S);
        }
        lkeep[t] = keep;
        kept_l += keep;
      }
      kept_u = warp_sum_i(kept_u);
      kept_l = warp_sum_i(kept_l);
      __syncwarp();
    }

    // ---- 6. emit U (kept rows ascending, pivot last) and L (unit first) ---
    if ((int64_t)unnz + kept_u + 1 > a.capU || (int64_t)lnnz + kept_l + 1 > a.capL) {
      if (lane == 0) {
        state[0] = FAC_OVERFLOW;
        state[1] = k;
      }
      if (a.smem_mode) {
        for (int i = lane; i < n; i += 32) {
          gpinv[i] = s.pinv[i];
          gprow[i] = s.prow[i];
        }
      }
      return;
    }
    int off = unnz;
    for (int base = 0; base < unum; base += 32) {
      const int t = base + lane;
      const bool keep = t < unum && ukeep[t];
      const unsigned m = __ballot_sync(FULL, keep);
      if (keep) {
        const int o = off + __popc(m & lanemask_lt());
        Ui[o] = urow[t];
        Ux[o] = uval[t];
      }
      off += __popc(m);
    }
    if (lane == 0) {
      Ui[off] = k;
      Ux[off] = piv;
      gUp[k + 1] = off + 1;
    }
    unnz = off + 1;

    const double2 rp = recipc(piv);
    if (lane == 0) {
      Li[lnnz] = ipiv;
      Lx[lnnz] = make_double2(1.0, 0.0);
    }
    off = lnnz + 1;
    for (int base = 0; base < lnum; base += 32) {
      const int t = base + lane;
      const bool keep = t < lnum && lkeep[t];
      const unsigned m = __ballot_sync(FULL, keep);
      if (keep) {
        const int o = off + __popc(m & lanemask_lt());
        const int i = lrow[t];
        Li[o] = i;
        Lx[o] = cmul_plain(s.x[i], rp);
      }
      off += __popc(m);
    }
    lnnz = off;
    if (lane == 0) {
      gLp[k + 1] = off;
      s.Lp[k + 1] = off;
      s.pinv[ipiv] = k;
      s.prow[k] = ipiv;
    }
    __syncwarp();
  }

  // ---- finish: publish pinv/prow, remap L rows to pivotal indices ---------
  if (a.smem_mode) {
    for (int i = lane; i < n; i += 32) {
      gpinv[i] = s.pinv[i];
      gprow[i] = s.prow[i];
    }
  }
  __syncwarp();
  for (int p = lane; p < lnnz; p += 32) Li[p] = s.pinv[Li[p]];
  if (lane == 0) {
    state[0] = FAC_DONE;
    state[1] = -1;
  }
}

int launch_ilutp(const FactorArgs& a, cudaStream_t st) {
  if (a.B == 0 || a.n == 0) return RS_OK;
  int dev;
  RS_CUDA_TRY(cudaGetDevice(&dev));
  int max_smem = 0;
  RS_CUDA_TRY(cudaDeviceGetAttribute(&max_smem,
                                     cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  const size_t per = ilutp_smem_per_system(a.n);
  int spb = 1;  // systems (warps) per CTA
  size_t smem = 0;
  if (a.smem_mode) {
    spb = (int)((size_t)max_smem / per);
    if (spb < 1) {
      set_error("ilutp smem mode requested but n=%d needs %zu B", a.n, per);
      return RS_ERR_ARG;
    }
    if (spb > 4) spb = 4;
    if (spb > a.B) spb = a.B;
    smem = per * spb;
    RS_CUDA_TRY(cudaFuncSetAttribute(ilutp_warp_kernel,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
  } else {
    spb = a.B < 4 ? a.B : 4;
  }
  const int grid = (a.B + spb - 1) / spb;
  ilutp_warp_kernel<<<grid, 32 * spb, smem, st>>>(a);
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

bool ilutp_fits_smem(int32_t n) {
  int dev = 0, max_smem = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return false;
  if (cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin,
                             dev) != cudaSuccess)
    return false;
  return ilutp_smem_per_system(n) <= (size_t)max_smem;
}

}  // namespace rs
