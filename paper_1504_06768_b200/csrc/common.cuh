// Shared device helpers for the rhosolve-b200 kernels (sm_100a).
//
// complex128 lives in HBM as interleaved double2 (re, im), the layout of
// numpy complex128, so host buffers cross the C ABI without repacking.
//
// Two complex-multiply roundings exist on the reference path and both are
// reproduced bit for bit:
//   * cmul_plain: (ar*br - ai*bi, ar*bi + ai*br), two roundings per part, no
//     FMA.  This is the Cython kernel arithmetic (CYTHON_CCOMPLEX=0 plus
//     -ffp-contract=off, reference pkg/setup.py:13-27, _ckernels.pyx:21-50)
//     and numpy's scalar*scalar path (sparse.matmul, sparse.py:243-265).
//   * cmul_np: (fma(ar,br,-(ai*bi)), fma(ar,bi,ai*br)), the numpy >= 2
//     SIMD array loop used by sparse.kron / sparse.add scaling
//     (sparse.py:202-240) on FMA-capable x86 hosts.
// Every operation uses explicit __d*_rn / __fma_rn intrinsics so nvcc can
// never contract them, independent of -fmad.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rs {

struct cplx {
  double re, im;
};

__host__ __device__ __forceinline__ double2 mk(double r, double i) {
  return make_double2(r, i);
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
}
__device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y));
}
__device__ __forceinline__ double2 cmul_plain(double2 a, double2 b) {
  return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                      __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}
__device__ __forceinline__ double2 cmul_np(double2 a, double2 b) {
  return make_double2(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)),
                      __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}
// conj(z) * (1 / |z|^2): reference recipc, _ckernels.pyx:25-31.
__device__ __forceinline__ double2 recipc(double2 z) {
  double d = __drcp_rn(__dadd_rn(__dmul_rn(z.x, z.x), __dmul_rn(z.y, z.y)));
  return make_double2(__dmul_rn(z.x, d), __dmul_rn(-z.y, d));
}
// |re| + |im|: reference cabs1, _ckernels.pyx:21-22.
__device__ __forceinline__ double cabs1(double2 z) {
  return fabs(z.x) + fabs(z.y);
}
__device__ __forceinline__ bool cis_zero(double2 z) {
  return z.x == 0.0 && z.y == 0.0;
}
__device__ __forceinline__ double cabs2(double2 z) {
  return __dadd_rn(__dmul_rn(z.x, z.x), __dmul_rn(z.y, z.y));
}

// 16-byte read-only load of a complex128 through the non-coherent path.
__device__ __forceinline__ double2 ldg2(const double2* p) { return __ldg(p); }

__device__ __forceinline__ int warp_lane() { return threadIdx.x & 31; }

}  // namespace rs

// Status codes shared with include/rhosolve_b200.h.
#define RS_OK 0
#define RS_ERR_ARG -1
#define RS_ERR_CUDA -2
#define RS_ERR_ALLOC -3
#define RS_ERR_BREAKDOWN -4
#define RS_ERR_NONFINITE -5
#define RS_ERR_OVERFLOW -6
#define RS_ERR_UNSUPPORTED -7
#define RS_ERR_STRUCT_SINGULAR -8

namespace rs {
void set_error(const char* fmt, ...);
// Host-side count of this library's kernel launches (rs_launch_count()).
void count_launch();
}

#define RS_CUDA_TRY(expr)                                                   \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess) {                                                \
      ::rs::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,            \
                      cudaGetErrorString(_e));                              \
      return RS_ERR_CUDA;                                                   \
    }                                                                       \
  } while (0)

#define RS_CHECK_ARG(cond, msg)                                             \
  do {                                                                      \
    if (!(cond)) {                                                          \
      ::rs::set_error("invalid argument: %s", msg);                         \
      return RS_ERR_ARG;                                                    \
    }                                                                       \
  } while (0)

#define RS_TRY(expr)                                                        \
  do {                                                                      \
    int _s = (expr);                                                        \
    if (_s != RS_OK) return _s;                                             \
  } while (0)
