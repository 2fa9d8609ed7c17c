// FP64 DADD / DMUL dependent-chain latency and SHFL latency (cycles).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* d, long long* out, int n) {
  double a = d[threadIdx.x], b = d[threadIdx.x + 32];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) a = __dmul_rn(a, b);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31);
  long long t3 = clock64();
  int x = threadIdx.x;
  __shared__ int s[64];
  s[threadIdx.x] = threadIdx.x;
  __syncwarp();
  for (int i = 0; i < n; ++i) x = ((volatile int*)s)[x & 31];
  long long t4 = clock64();
  d[threadIdx.x] = a + x;
  if (threadIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t1; out[2] = t3 - t2; out[3] = t4 - t3; }
}
int main() {
  double* d; long long* o; cudaMalloc(&d, 1024); cudaMalloc(&o, 64);
  cudaMemset(d, 0, 1024);
  const int n = 4096;
  k<<<1, 32>>>(d, o, n); k<<<1, 32>>>(d, o, n); cudaDeviceSynchronize();
  long long h[4]; cudaMemcpy(h, o, 32, cudaMemcpyDeviceToHost);
  printf("DADD %.1f  DMUL %.1f  SHFL %.1f  LDS(volatile) %.1f cycles\n", (double)h[0]/n, (double)h[1]/n, (double)h[2]/n, (double)h[3]/n);
}
