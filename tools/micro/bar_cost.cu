// Cost of a CTA barrier per step for a 512-thread CTA holding ~222 KB of
// shared memory (the frontal LU's shape): empty steps, steps with a short
// dependent shared-memory chain, and with a global load in flight.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(512, 1) bar_kernel(int steps, int mode, long long* out, int* g) {
  extern __shared__ double2 sm[];
  const int tid = threadIdx.x;
  for (int i = tid; i < 1024; i += 512) sm[i] = make_double2(i, 0);
  __syncthreads();
  long long t0 = clock64();
  double acc = 0;
  int gi = 0;
  for (int k = 0; k < steps; ++k) {
    if (mode >= 1) {  // dependent LDS chain of 8
      int idx = (tid + k) & 1023;
      for (int j = 0; j < 8; ++j) {
        double2 v = sm[idx];
        acc += v.x;
        idx = ((int)v.x + 1) & 1023;
      }
    }
    if (mode == 2 && tid >= 256) gi += g[(k * 512 + tid) & 1048575];
    int ld = 0;
    if (mode == 3 && tid >= 256) ld = g[(k * 4096 + tid * 8) & 1048575];  // consumed after 2 barriers
    if (mode == 4 && tid >= 256) ((int*)g)[(k * 4096 + tid * 8) & 1048575] = k;  // store only
    __syncthreads();
    if (mode >= 1 && tid < 128) sm[tid] = make_double2(acc, 0);
    __syncthreads();
    __syncthreads();
    gi += ld;
  }
  long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = (t1 - t0) / steps;
  if (acc == 12345.0 || gi == 7) out[1000] = 1;
}

int main() {
  long long* d;
  int* g;
  cudaMalloc(&d, 8 * 2048);
  cudaMalloc(&g, 4 << 20);
  cudaMemset(g, 0, 4 << 20);
  cudaFuncSetAttribute(bar_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 222 * 1024);
  for (int mode = 0; mode < 5; ++mode)
    for (int blocks : {1, 148}) {
      bar_kernel<<<blocks, 512, 222 * 1024>>>(2000, mode, d, g);
      long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      printf("mode %d blocks %d: %lld cycles per step (3 barriers)\n", mode, blocks, h);
    }
  return 0;
}
