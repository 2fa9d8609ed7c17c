// Solution post-processing, steady._postprocess (pkg/src/rhosolve/steady.py:62-71)
// plus the solution unpermute of steady.py:126-127 / 249-250:
//   x_nat = x_perm[forward]           (omitted on the natural ordering)
//   rho   = unvec(x_nat)              rho[r, c] = x_nat[c*D + r]
//   rho   = 0.5 * (rho + rho^dag)
//   rho  /= trace(rho)                (skipped when the trace is 0)
//   residual = || L_plain vec(rho) ||_2
// One CTA per system; rho is written row-major (D x D complex128), the layout
// numpy returns.
#include "common.cuh"
#include "cta_ops.cuh"
#include "kernels.cuh"

namespace rs {

__global__ void __launch_bounds__(512) postprocess_kernel(
    int32_t D, const double2* x, const int32_t* fwd, const int32_t* Lrp, const int32_t* Lci,
    const double2* Lv, double2* rho, double2* vec_tmp, double* residual, double2* trace_out) {
  __shared__ double red[64];

  const int b = blockIdx.x;
  const int64_t n = (int64_t)D * D;
  const double2* xs = x + b * n;
  const int32_t* f = fwd ? fwd + b * n : nullptr;
  double2* R = rho + b * n;
  double2* vv = vec_tmp + b * n;
  double acc[2] = {0.0, 0.0};
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    const int32_t r = (int32_t)(e / D), c = (int32_t)(e % D);
    const int64_t i1 = (int64_t)c * D + r, i2 = (int64_t)r * D + c;
    const double2 a = xs[f ? f[i1] : i1];
    const double2 bb = xs[f ? f[i2] : i2];
    const double2 s = make_double2(a.x + bb.x, a.y - bb.y);
    const double2 h = make_double2(0.5 * s.x, 0.5 * s.y);
    R[e] = h;
    if (r == c) {
      acc[0] += h.x;
      acc[1] += h.y;
    }
  }
  cta::block_sum<2>(acc, red);
  const double2 tr = make_double2(acc[0], acc[1]);
  const bool nz = !(tr.x == 0.0 && tr.y == 0.0);
  // numpy complex division by a scalar (Smith's method with a reciprocal)
  double rat = 0.0, scl = 0.0;
  const bool real_major = fabs(tr.x) >= fabs(tr.y);
  if (nz) {
    if (real_major) {
      rat = tr.y / tr.x;
      scl = 1.0 / (tr.x + tr.y * rat);
    } else {
      rat = tr.x / tr.y;
      scl = 1.0 / (tr.y + tr.x * rat);
    }
  }
  for (int64_t e = threadIdx.x; e < n; e += blockDim.x) {
    double2 h = R[e];
    if (nz) {
      if (real_major) h = make_double2((h.x + h.y * rat) * scl, (h.y - h.x * rat) * scl);
      else h = make_double2((h.x * rat + h.y) * scl, (h.y * rat - h.x) * scl);
      R[e] = h;
    }
    const int32_t r = (int32_t)(e / D), c = (int32_t)(e % D);
    vv[(int64_t)c * D + r] = h;
  }
  __syncthreads();
  double racc[1] = {0.0};
  const int32_t* rp = Lrp + b * n;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    const int32_t p0 = rp[i], p1 = rp[i + 1];
    double2 s = make_double2(0.0, 0.0);
    if (p0 < p1) {
      s = cmul_plain(Lv[p0], vv[Lci[p0]]);
      for (int32_t p = p0 + 1; p < p1; ++p) s = cadd(s, cmul_plain(Lv[p], vv[Lci[p]]));
    }
    racc[0] = __fma_rn(s.x, s.x, __fma_rn(s.y, s.y, racc[0]));
  }
  cta::block_sum<1>(racc, red);
  if (threadIdx.x == 0) {
    residual[b] = sqrt(racc[0]);
    if (trace_out) trace_out[b] = tr;
  }

}

int postprocess(int B, int32_t D, const double2* x, const int32_t* fwd, const int32_t* Lrp,
                const int32_t* Lci, const double2* Lv, double2* rho, double* residual,
                double2* trace_out, cudaStream_t st) {
  const int64_t n = (int64_t)D * D;
  double2* tmp = nullptr;
  RS_CUDA_TRY(cudaMallocAsync(&tmp, sizeof(double2) * n * B, st));
  postprocess_kernel<<<B, 512, 0, st>>>(D, x, fwd, Lrp, Lci, Lv, rho, tmp, residual, trace_out); ::rs::count_launch();
  cudaFreeAsync(tmp, st);
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

// x_nat[i] = x_perm[fwd[i]] per system (steady.py:249-250).
__global__ void unpermute_kernel(int64_t total, int32_t n, const double2* x, const int32_t* fwd,
                                 double2* out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int64_t b = e / n;
  out[e] = x[b * n + fwd[e]];
}

// prhs[fwd[i]] = rhs[i] per system (steady.py:89-94).
__global__ void scatter_perm_kernel(int64_t total, int32_t n, const double2* x,
                                    const int32_t* fwd, double2* out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const int64_t b = e / n;
  out[b * n + fwd[e]] = x[e];
}

int permute_vector(int B, int32_t n, const double2* x, const int32_t* fwd, double2* out,
                   int gather, cudaStream_t st) {
  const int64_t total = (int64_t)B * n;
  if (!total) return RS_OK;
  const unsigned grid = (unsigned)((total + 255) / 256);
  if (gather) unpermute_kernel<<<grid, 256, 0, st>>>(total, n, x, fwd, out);
  else scatter_perm_kernel<<<grid, 256, 0, st>>>(total, n, x, fwd, out);
  ::rs::count_launch();
  RS_CUDA_TRY(cudaGetLastError());
  return RS_OK;
}

}  // namespace rs
