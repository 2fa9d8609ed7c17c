// Dissect the per-hop cost of a warp-round-robin dependency chain (row r
// depends on row r-1, rows dealt to warps round-robin), as in the sparse
// triangular sweep with one entry per row.
#include <cstdio>
#include <cuda_runtime.h>

constexpr unsigned long long SENT = 0x7ff4dead5eedbeefull;
__device__ __forceinline__ double2 lds2(const double2* p) {
  double2 v;
  asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ void sts2(double2* p, double2 v) {
  asm volatile("st.volatile.shared.v2.f64 [%0], {%1, %2};" ::"r"((unsigned)__cvta_generic_to_shared(p)), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ bool ready(double2 s) {
  return __double_as_longlong(s.x) != (long long)SENT && __double_as_longlong(s.y) != (long long)SENT;
}

// MODE 0: minimal: lane0 spins on y[r-1], y[r] = y[r-1]*0.5 (DMUL), store.
// MODE 1: + global loads per row (rp, ci, v, in) before polling.
// MODE 2: MODE 1 + complex cmul/csub.
// MODE 3: MODE 2 + whole-warp participation (ballot + syncwarp per row).
template <int MODE>
__global__ void chain(int n, const int* rp, const int* ci, const double2* v, const double2* in,
                      long long* out) {
  extern __shared__ double2 y[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = make_double2(__longlong_as_double(SENT), __longlong_as_double(SENT));
  __syncthreads();
  if (threadIdx.x == 0) y[0] = make_double2(1.0, 0.0);
  __syncthreads();
  long long t0 = clock64();
  for (int r = 1 + wid; r < n; r += nw) {
    int c = r - 1;
    double2 l = make_double2(0.5, 0.0), acc = make_double2(0.0, 0.0);
    if (MODE >= 1) {
      const int p0 = rp[r];
      c = ci[p0];
      l = v[p0];
      acc = in[r];
    }
    if (MODE == 3) {
      const bool ok = ready(lds2(y + c));
      const unsigned m = __ballot_sync(0xffffffffu, ok);
      (void)m;
      __syncwarp();
    }
    if (lane == 0) {
      double2 s;
      do { s = lds2(y + c); } while (!ready(s));
      double2 res;
      if (MODE >= 2) {
        const double2 p = make_double2(l.x * s.x - l.y * s.y, l.x * s.y + l.y * s.x);
        res = make_double2(acc.x - p.x, acc.y - p.y);
      } else {
        res = make_double2(s.x * 0.5, s.y * 0.5);
      }
      sts2(y + r, res);
    }
    if (MODE == 3) __syncwarp();
  }
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  const int n = 6400;
  int *rp, *ci;
  double2 *v, *in;
  long long* out;
  cudaMalloc(&rp, 4 * (n + 1)); cudaMalloc(&ci, 4 * n); cudaMalloc(&v, 16 * n); cudaMalloc(&in, 16 * n);
  cudaMalloc(&out, 8);
  int* h = new int[n + 1];
  for (int i = 0; i <= n; ++i) h[i] = i > 0 ? i - 1 : 0;
  cudaMemcpy(rp, h, 4 * (n + 1), cudaMemcpyHostToDevice);
  for (int i = 0; i < n; ++i) h[i] = i - 1 < 0 ? 0 : i - 1;
  // row r's single entry is at position r-1 with column r-1
  int* hc = new int[n];
  for (int i = 0; i < n; ++i) hc[i] = i;
  cudaMemcpy(ci, hc, 4 * n, cudaMemcpyHostToDevice);
  cudaMemset(v, 0, 16 * n);
  cudaMemset(in, 0, 16 * n);
  cudaFuncSetAttribute(chain<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * n);
  cudaFuncSetAttribute(chain<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * n);
  cudaFuncSetAttribute(chain<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * n);
  cudaFuncSetAttribute(chain<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 16 * n);
  for (int mode = 0; mode < 4; ++mode)
    for (int threads : {64, 256, 512, 1024}) {
      long long c = 0;
      for (int rep = 0; rep < 2; ++rep) {
        switch (mode) {
          case 0: chain<0><<<1, threads, 16 * n>>>(n, rp, ci, v, in, out); break;
          case 1: chain<1><<<1, threads, 16 * n>>>(n, rp, ci, v, in, out); break;
          case 2: chain<2><<<1, threads, 16 * n>>>(n, rp, ci, v, in, out); break;
          case 3: chain<3><<<1, threads, 16 * n>>>(n, rp, ci, v, in, out); break;
        }
        cudaDeviceSynchronize();
        cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      }
      printf("mode %d threads %4d: %.0f cycles/hop  (%s)\n", mode, threads, (double)c / n,
             cudaGetErrorString(cudaGetLastError()));
    }
}
