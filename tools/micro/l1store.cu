// Does a global store keep/refresh the line in L1 for later loads by the same
// warp?  Dependent load chains over (a) lines only loaded before, (b) lines
// the warp itself stored, (c) lines stored then re-read once.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* a, int* b, long long* out, int n) {
  const int lane = threadIdx.x;
  // warm lines of b by loading
  int x = 0;
  for (int i = lane; i < 1024; i += 32) x += b[i];
  __syncwarp();
  long long t0 = clock64();
  int p = lane;
  for (int i = 0; i < n; ++i) p = b[(p * 33 + 7) & 1023];  // loaded-only lines
  long long t1 = clock64();
  for (int i = lane; i < 1024; i += 32) a[i] = (i * 33 + 7) & 1023;  // store lines
  __syncwarp();
  long long t2 = clock64();
  int q = lane;
  for (int i = 0; i < n; ++i) q = a[q];  // stored lines
  long long t3 = clock64();
  int r = lane;
  for (int i = 0; i < n; ++i) r = a[r];  // again (now loaded)
  long long t4 = clock64();
  if (lane == 0) { out[0] = t1 - t0; out[1] = t3 - t2; out[2] = t4 - t3; }
  b[2048 + lane] = p + q + r + x;
}
int main() {
  int *a, *b; long long* o;
  cudaMalloc(&a, 1 << 16); cudaMalloc(&b, 1 << 16); cudaMalloc(&o, 64);
  int h[4096]; for (int i = 0; i < 4096; ++i) h[i] = (i * 33 + 7) & 1023;
  cudaMemcpy(b, h, sizeof(h), cudaMemcpyHostToDevice);
  const int n = 2000;
  for (int rep = 0; rep < 3; ++rep) k<<<1, 32>>>(a, b, o, n);
  cudaDeviceSynchronize();
  long long r[3]; cudaMemcpy(r, o, 24, cudaMemcpyDeviceToHost);
  printf("load-only lines %.0f cyc/load; after own stores %.0f; re-read %.0f\n",
         (double)r[0] / n, (double)r[1] / n, (double)r[2] / n);
}
