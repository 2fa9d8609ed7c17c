// Microbenchmark: latency of a value hand-off between warps of one CTA.
// Warp 0 and warp 1 alternately wait for the other's counter value and
// publish the next one; cycles per hop = total / hops.  Variants: shared vs
// global memory, volatile vs relaxed/acquire, extra warps spinning or not.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ long long ld_vol_s(const long long* p) {
  long long v;
  asm volatile("ld.volatile.shared.s64 %0, [%1];" : "=l"(v) : "r"((unsigned)__cvta_generic_to_shared(p)));
  return v;
}
__device__ __forceinline__ void st_vol_s(long long* p, long long v) {
  asm volatile("st.volatile.shared.s64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "l"(v) : "memory");
}
__device__ __forceinline__ long long ld_rel_g(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.s64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_rel_g(long long* p, long long v) {
  asm volatile("st.relaxed.gpu.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <int MODE>
__global__ void pingpong(long long* g, int hops, int spin_warps, long long* out) {
  __shared__ long long s[64];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x < 64) s[threadIdx.x] = -1;
  if (threadIdx.x == 0) { g[0] = -1; }
  __syncthreads();
  __threadfence();
  __syncthreads();
  long long t0 = clock64();
  if (w < 2) {
    for (long long k = w; k < hops; k += 2) {
      if (k > 0) {
        // wait for value k-1
        if (MODE == 0) { while (ld_vol_s(&s[0]) != k - 1) {} }
        else { while (ld_rel_g(&g[0]) != k - 1) {} }
      }
      if (lane == 0) {
        if (MODE == 0) st_vol_s(&s[0], k);
        else st_rel_g(&g[0], k);
      }
      __syncwarp();
    }
  } else if (w < 2 + spin_warps) {
    // distractors: poll a location that never changes until the end
    while (true) {
      long long v = (MODE == 0) ? ld_vol_s(&s[0]) : ld_rel_g(&g[0]);
      if (v >= hops - 1) break;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = t1 - t0;
}

int main() {
  long long *g, *out;
  cudaMalloc(&g, 1024);
  cudaMalloc(&out, 64);
  const int hops = 20000;
  for (int mode = 0; mode < 2; ++mode)
    for (int spin : {0, 2, 14, 30}) {
      int threads = 32 * (2 + spin);
      for (int rep = 0; rep < 2; ++rep) {
        if (mode == 0) pingpong<0><<<1, threads>>>(g, hops, spin, out);
        else pingpong<1><<<1, threads>>>(g, hops, spin, out);
      }
      cudaDeviceSynchronize();
      long long c;
      cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
      printf("%s spin_warps=%2d: %.1f cycles/hop\n", mode ? "global relaxed.gpu" : "shared volatile  ",
             spin, (double)c / hops);
    }
  return 0;
}
