// Lindblad superoperator assembly straight into CSR (liouville.build_liouvillian,
// pkg/src/rhosolve/liouville.py:54-77), bit-exact in structure and values.
//
// The reference builds L as a chain of sparse.add calls (sparse.py:231-240):
//   L = add(kron(I,H), kron(H^T,I), -1j, +1j)
//   for C in c_ops:  L = add(L, kron(conj C, C))
//                    L = add(L, kron(I, C^dag C), 1, -1/2)
//                    L = add(L, kron((C^dag C)^T, I), 1, -1/2)
// where every add rescales both operands (numpy complex array multiply,
// FMA form on x86-64: re = fma(ar,br,-(ai*bi)), im = fma(ar,bi,ai*br)), sums
// coinciding entries (existing L first) and prunes exact zeros.  The value at
// a position is therefore a fixed left fold over the term sequence with
// rescaling and pruning after every step, which this kernel replays per
// output position.  One thread owns one output row r = i*D + k and merges the
// 2 + 3K sorted term streams of that row by column:
//   kron(I, X)  row (i,k): columns i*D + X[k,:]
//   kron(X, I)  row (i,k): columns X[i,:]*D + k
//   kron(conj X, X): columns X[i,:]*D + X[k,:]
// A count pass and a fill pass (same code) bracket a device scan.
//
// C^dag C (sparse.matmul, sparse.py:243-265: per row, ascending inner index,
// dictionary accumulation starting from 0.0 with numpy scalar products in the
// plain two-rounding form, then pruned) is computed on the device too.
#include <string.h>

#include "common.cuh"
#include "kernels.cuh"

namespace rs {

constexpr int MAX_COPS = 8;

struct OpCSR {
  const int32_t* rp;
  const int32_t* ci;
  const double2* v;
};

struct AssembleArgs {
  int32_t D;
  int32_t K;
  int32_t B;  // systems: every operator is a block-diagonal batch of B D x D CSRs
  OpCSR H, Ht;
  OpCSR C[MAX_COPS], CDC[MAX_COPS], CDCt[MAX_COPS];
};

namespace {

constexpr int32_t END = 0x7fffffff;

__device__ __forceinline__ double2 conjz(double2 a) { return make_double2(a.x, -a.y); }

struct Cursor {
  int32_t p, pe;  // outer range (row i of X for XI / CC, row k of X for IH)
  int32_t t, ts, te;  // inner range (CC only)
};

}  // namespace

// kind: 0 = IH (kron(I,X)), 1 = XI (kron(X,I)), 2 = CC (kron(conj X, X))
__device__ __forceinline__ int32_t cur_col(int kind, const OpCSR& X, const Cursor& c,
                                           int32_t i, int32_t k, int32_t D) {
  if (c.p >= c.pe) return END;
  if (kind == 0) return i * D + X.ci[c.p];
  if (kind == 1) return X.ci[c.p] * D + k;
  return X.ci[c.p] * D + X.ci[c.t];
}
__device__ __forceinline__ double2 cur_val(int kind, const OpCSR& X, const Cursor& c) {
  const double2 one = make_double2(1.0, 0.0);
  if (kind == 0) return cmul_np(one, X.v[c.p]);
  if (kind == 1) return cmul_np(X.v[c.p], one);
  return cmul_np(conjz(X.v[c.p]), X.v[c.t]);
}
__device__ __forceinline__ void cur_next(int kind, Cursor& c) {
  if (kind == 2) {
    if (++c.t < c.te) return;
    c.t = c.ts;
  }
  ++c.p;
}

template <bool FILL>
__global__ void assemble_kernel(AssembleArgs a, int32_t* counts, const int32_t* out_rp,
                                int32_t* out_ci, double2* out_v) {
  const int32_t D = a.D;
  const int64_t n = (int64_t)D * D;
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n * a.B) return;
  const int64_t ob = (r / n) * D;  // first operator row of this system
  const int32_t rl = (int32_t)(r % n);
  const int32_t i = rl / D, k = rl % D;
  const int nt = 2 + 3 * a.K;
  Cursor cur[2 + 3 * MAX_COPS];
  int kinds[2 + 3 * MAX_COPS];
  OpCSR mats[2 + 3 * MAX_COPS];
  for (int t = 0; t < nt; ++t) {
    int kind;
    OpCSR X;
    if (t == 0) {
      kind = 0;
      X = a.H;
    } else if (t == 1) {
      kind = 1;
      X = a.Ht;
    } else {
      const int c = (t - 2) / 3, s = (t - 2) % 3;
      kind = s == 0 ? 2 : (s == 1 ? 0 : 1);
      X = s == 0 ? a.C[c] : (s == 1 ? a.CDC[c] : a.CDCt[c]);
    }
    kinds[t] = kind;
    mats[t] = X;
    Cursor c;
    const int32_t rowsel = (kind == 0) ? k : i;
    c.p = X.rp[ob + rowsel];
    c.pe = X.rp[ob + rowsel + 1];
    c.ts = c.te = c.t = 0;
    if (kind == 2) {
      c.ts = c.t = X.rp[ob + k];
      c.te = X.rp[ob + k + 1];
      if (c.ts == c.te) c.p = c.pe;  // empty inner row: no entries
    }
    cur[t] = c;
  }
  int32_t cnt = 0;
  int32_t o = FILL ? out_rp[r] : 0;
  const double2 one = make_double2(1.0, 0.0);
  const double2 mi = make_double2(0.0, -1.0), pi = make_double2(0.0, 1.0);
  const double2 mhalf = make_double2(-0.5, 0.0);
  while (true) {
    int32_t cm = END;
    for (int t = 0; t < nt; ++t) cm = min(cm, cur_col(kinds[t], mats[t], cur[t], i, k, D));
    if (cm == END) break;
    // fold at column cm
    bool pres = false;
    double2 v = make_double2(0.0, 0.0);
    {
      const bool h0 = cur_col(kinds[0], mats[0], cur[0], i, k, D) == cm;
      const bool h1 = cur_col(kinds[1], mats[1], cur[1], i, k, D) == cm;
      double2 av, bv;
      if (h0) {
        av = cmul_np(mi, cur_val(kinds[0], mats[0], cur[0]));
        cur_next(kinds[0], cur[0]);
      }
      if (h1) {
        bv = cmul_np(pi, cur_val(kinds[1], mats[1], cur[1]));
        cur_next(kinds[1], cur[1]);
      }
      if (h0 && h1) {
        v = cadd(av, bv);
        pres = true;
      } else if (h0) {
        v = av;
        pres = true;
      } else if (h1) {
        v = bv;
        pres = true;
      }
      if (pres && cis_zero(v)) pres = false;
    }
    for (int t = 2; t < nt; ++t) {
      const bool ht = cur_col(kinds[t], mats[t], cur[t], i, k, D) == cm;
      if (pres) v = cmul_np(one, v);
      if (ht) {
        const double2 beta = ((t - 2) % 3 == 0) ? one : mhalf;
        const double2 tv = cmul_np(beta, cur_val(kinds[t], mats[t], cur[t]));
        cur_next(kinds[t], cur[t]);
        if (pres) {
          v = cadd(v, tv);
        } else {
          v = tv;
          pres = true;
        }
      }
      if (pres && cis_zero(v)) pres = false;
    }
    if (pres) {
      if (FILL) {
        out_ci[o] = cm;
        out_v[o] = v;
        ++o;
      }
      ++cnt;
    }
  }
  if (!FILL) counts[r] = cnt;
}

// ---- C^dag C ----------------------------------------------------------------
// One CTA per output row (global over the batch); dense accumulator row in
// global scratch (D complex + presence flags); sequential over the inner index
// j (ascending), parallel over the entries of C's row j (distinct output
// columns).
__global__ void cdc_dense_kernel(int32_t D, OpCSR Ct, OpCSR C, double2* acc, int8_t* pres,
                                 int32_t* counts) {
  const int64_t i = blockIdx.x;
  const int64_t ob = (i / D) * D;  // first operator row of this system
  double2* row = acc + i * D;
  int8_t* pr = pres + i * D;
  for (int32_t c = threadIdx.x; c < D; c += blockDim.x) pr[c] = 0;
  __syncthreads();
  for (int32_t p = Ct.rp[i]; p < Ct.rp[i + 1]; ++p) {
    const int64_t j = ob + Ct.ci[p];
    const double2 vj = make_double2(Ct.v[p].x, -Ct.v[p].y);  // adjoint = conj(transpose)
    for (int32_t t = C.rp[j] + threadIdx.x; t < C.rp[j + 1]; t += blockDim.x) {
      const int32_t c = C.ci[t];
      const double2 prod = cmul_plain(vj, C.v[t]);
      if (pr[c]) row[c] = cadd(row[c], prod);
      else {
        row[c] = cadd(make_double2(0.0, 0.0), prod);
        pr[c] = 1;
      }
    }
    __syncthreads();
  }
  int32_t cnt = 0;
  for (int32_t c = threadIdx.x; c < D; c += blockDim.x)
    if (pr[c] && !cis_zero(row[c])) ++cnt;
  for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  __shared__ int32_t ws[32];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = cnt;
  __syncthreads();
  if (threadIdx.x == 0) {
    int32_t s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += ws[w];
    counts[i] = s;
  }
}

__global__ void cdc_compact_kernel(int64_t rows, int32_t D, const double2* acc,
                                   const int8_t* pres, const int32_t* rp, int32_t* ci,
                                   double2* v) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows) return;
  int32_t o = rp[i];
  for (int32_t c = 0; c < D; ++c) {
    const double2 x = acc[i * D + c];
    if (pres[i * D + c] && !cis_zero(x)) {
      ci[o] = c;
      v[o] = x;
      ++o;
    }
  }
}

// max |H - H^dag| over stored entries (liouville.py:62-64).
__global__ void herm_dev_kernel(int64_t rows, int32_t D, OpCSR H, unsigned long long* out) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= rows) return;
  const int64_t ob = (g / D) * D;
  const int32_t i = (int32_t)(g - ob);
  double m = 0.0;
  for (int32_t p = H.rp[g]; p < H.rp[g + 1]; ++p) {
    const int64_t j = ob + H.ci[p];
    double2 d = H.v[p];
    int32_t lo = H.rp[j], hi = H.rp[j + 1];
    while (lo < hi) {
      const int32_t mid = (lo + hi) >> 1;
      if (H.ci[mid] < i) lo = mid + 1;
      else hi = mid;
    }
    if (lo < H.rp[j + 1] && H.ci[lo] == i) {
      const double2 h = H.v[lo];
      d = make_double2(d.x - h.x, d.y + h.y);
    }
    m = fmax(m, hypot(d.x, d.y));
  }
  atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

static inline unsigned gridn(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

struct OpBufs {
  int32_t *rp = nullptr, *ci = nullptr;
  double2* v = nullptr;
};

static void free_op(OpBufs& b, cudaStream_t st) {
  if (b.rp) cudaFreeAsync(b.rp, st);
  if (b.ci) cudaFreeAsync(b.ci, st);
  if (b.v) cudaFreeAsync(b.v, st);
  b = OpBufs();
}

static int op_transpose(int B, int32_t D, const OpCSR& X, int64_t nnz, OpBufs& out,
                        cudaStream_t st) {
  RS_CUDA_TRY(cudaMallocAsync(&out.rp, sizeof(int32_t) * ((int64_t)B * D + 1), st));
  RS_CUDA_TRY(cudaMallocAsync(&out.ci, sizeof(int32_t) * (nnz + 1), st));
  RS_CUDA_TRY(cudaMallocAsync(&out.v, sizeof(double2) * (nnz + 1), st));
  return csr_transpose(B, D, X.rp, X.ci, X.v, out.rp, out.ci, out.v, st);
}

static int op_cdc(int B, int32_t D, const OpCSR& C, const OpCSR& Ct, OpBufs& out, int64_t* nnz,
                  cudaStream_t st) {
  double2* acc = nullptr;
  int8_t* pres = nullptr;
  int32_t* counts = nullptr;
  const int64_t rows = (int64_t)B * D;
  RS_CUDA_TRY(cudaMallocAsync(&acc, sizeof(double2) * rows * D, st));
  RS_CUDA_TRY(cudaMallocAsync(&pres, rows * D, st));
  RS_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (rows + 1), st));
  RS_CUDA_TRY(cudaMallocAsync(&out.rp, sizeof(int32_t) * (rows + 1), st));
  cdc_dense_kernel<<<(unsigned)rows, 128, 0, st>>>(D, Ct, C, acc, pres, counts); ::rs::count_launch();
  int rc = scan_counts(counts, out.rp, rows, nnz, st);
  if (rc == RS_OK) {
    RS_CUDA_TRY(cudaMallocAsync(&out.ci, sizeof(int32_t) * (*nnz + 1), st));
    RS_CUDA_TRY(cudaMallocAsync(&out.v, sizeof(double2) * (*nnz + 1), st));
    cdc_compact_kernel<<<gridn(rows, 128), 128, 0, st>>>(rows, D, acc, pres, out.rp, out.ci, out.v); ::rs::count_launch();
  }
  cudaFreeAsync(acc, st);
  cudaFreeAsync(pres, st);
  cudaFreeAsync(counts, st);
  RS_CUDA_TRY(cudaGetLastError());
  return rc;
}

// Count pass when out_ci == nullptr (fills out_rp, returns *nnz_out); fill
// pass otherwise (out_rp must hold the count-pass result).
int liouvillian_assemble(int32_t B, int32_t D, const int32_t* Hrp, const int32_t* Hci,
                         const double2* Hv, int64_t Hnnz, int32_t K, const int32_t* const* Crp,
                         const int32_t* const* Cci, const double2* const* Cv,
                         const int64_t* Cnnz, double* herm_dev, int32_t* out_rp,
                         int32_t* out_ci, double2* out_v, int64_t* nnz_out, cudaStream_t st) {
  if (K > MAX_COPS) {
    set_error("at most %d collapse operators supported, got %d", MAX_COPS, K);
    return RS_ERR_UNSUPPORTED;
  }
  const int64_t n = (int64_t)B * D * D;  // output rows over the whole batch
  AssembleArgs a;
  a.D = D;
  a.K = K;
  a.B = B;
  a.H = OpCSR{Hrp, Hci, Hv};
  OpBufs ht, ct[MAX_COPS], cdc[MAX_COPS], cdct[MAX_COPS];
  int rc = op_transpose(B, D, a.H, Hnnz, ht, st);
  a.Ht = OpCSR{ht.rp, ht.ci, ht.v};
  for (int c = 0; c < K && rc == RS_OK; ++c) {
    a.C[c] = OpCSR{Crp[c], Cci[c], Cv[c]};
    rc = op_transpose(B, D, a.C[c], Cnnz[c], ct[c], st);
    if (rc) break;
    int64_t cnnz = 0;
    rc = op_cdc(B, D, a.C[c], OpCSR{ct[c].rp, ct[c].ci, ct[c].v}, cdc[c], &cnnz, st);
    if (rc) break;
    a.CDC[c] = OpCSR{cdc[c].rp, cdc[c].ci, cdc[c].v};
    rc = op_transpose(B, D, a.CDC[c], cnnz, cdct[c], st);
    a.CDCt[c] = OpCSR{cdct[c].rp, cdct[c].ci, cdct[c].v};
  }
  if (rc == RS_OK && herm_dev) {
    unsigned long long* dm = nullptr;
    RS_CUDA_TRY(cudaMallocAsync(&dm, sizeof(unsigned long long), st));
    RS_CUDA_TRY(cudaMemsetAsync(dm, 0, sizeof(unsigned long long), st));
    herm_dev_kernel<<<gridn((int64_t)B * D, 128), 128, 0, st>>>((int64_t)B * D, D, a.H, dm); ::rs::count_launch();
    unsigned long long hv = 0;
    RS_CUDA_TRY(cudaMemcpyAsync(&hv, dm, sizeof(hv), cudaMemcpyDeviceToHost, st));
    RS_CUDA_TRY(cudaStreamSynchronize(st));
    cudaFreeAsync(dm, st);
    double hd;
    memcpy(&hd, &hv, sizeof(hd));
    *herm_dev = hd;
  }
  if (rc == RS_OK) {
    if (!out_ci) {
      int32_t* counts = nullptr;
      RS_CUDA_TRY(cudaMallocAsync(&counts, sizeof(int32_t) * (n + 1), st));
      assemble_kernel<false><<<gridn(n, 128), 128, 0, st>>>(a, counts, nullptr, nullptr,
                                                           nullptr); ::rs::count_launch();
      rc = scan_counts(counts, out_rp, n, nnz_out, st);
      cudaFreeAsync(counts, st);
    } else {
      assemble_kernel<true><<<gridn(n, 128), 128, 0, st>>>(a, nullptr, out_rp, out_ci, out_v); ::rs::count_launch();
    }
  }
  free_op(ht, st);
  for (int c = 0; c < K; ++c) {
    free_op(ct[c], st);
    free_op(cdc[c], st);
    free_op(cdct[c], st);
  }
  RS_CUDA_TRY(cudaGetLastError());
  return rc;
}

}  // namespace rs
