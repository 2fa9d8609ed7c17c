// Dependent-load latency of the load flavours a spin-wait can use (cycles per
// load, one lane, pointer chase through a 64 MB buffer so every load is an L2
// or HBM access), and the cross-SM publish -> observe hop for each flavour.
//   nvcc -O3 -arch=sm_100a -o poll_lat poll_lat.cu && ./poll_lat
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double2 ld_cg(const double2* p) {
  double2 v;
  asm volatile("ld.global.cg.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double2 ld_rlx(const double2* p) {
  double2 v;
  asm volatile("ld.relaxed.gpu.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ double2 ld_vol(const double2* p) {
  double2 v;
  asm volatile("ld.volatile.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p) : "memory");
  return v;
}

template <int MODE>
__global__ void chase(const double2* buf, int steps, long long* out) {
  size_t i = 0;
  double acc = 0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    double2 v = MODE == 0 ? ld_cg(buf + i) : (MODE == 1 ? ld_rlx(buf + i) : ld_vol(buf + i));
    i = (size_t)v.x;
    acc += v.y;
  }
  long long t1 = clock64();
  out[0] = t1 - t0;
  out[1] = (long long)acc;
}

// ping-pong between two CTAs on different SMs: flag value travels with the data
template <int MODE>
__global__ void pingpong(double2* slot, int rounds, long long* out) {
  const int me = blockIdx.x;  // 0 or 1
  if (threadIdx.x != 0) return;
  long long t0 = clock64();
  for (int r = 0; r < rounds; ++r) {
    if ((r & 1) == me) {
      asm volatile("st.relaxed.gpu.global.v2.f64 [%0], {%1, %2};" ::"l"(slot), "d"((double)(r + 1)), "d"(0.0) : "memory");
    } else {
      double2 v;
      do {
        v = MODE == 0 ? ld_cg(slot) : (MODE == 1 ? ld_rlx(slot) : ld_vol(slot));
      } while (v.x != (double)(r + 1));
    }
  }
  long long t1 = clock64();
  if (me == 0) out[0] = t1 - t0;
}

int main() {
  const size_t N = 4 << 20;  // 64 MB of double2
  double2* h = (double2*)malloc(N * sizeof(double2));
  size_t stride = 40503;  // scattered chase
  for (size_t i = 0; i < N; ++i) { h[i].x = (double)((i * 1 + stride * 97) % N); h[i].y = 1.0; }
  size_t cur = 0;
  for (size_t k = 0; k < N; ++k) { size_t nxt = (cur + stride) % N; h[cur].x = (double)nxt; cur = nxt; }
  double2* d; long long* o;
  cudaMalloc(&d, N * sizeof(double2)); cudaMalloc(&o, 64);
  cudaMemcpy(d, h, N * sizeof(double2), cudaMemcpyHostToDevice);
  long long r[2];
  const char* names[3] = {"ld.global.cg", "ld.relaxed.gpu", "ld.volatile"};
  for (int rep = 0; rep < 2; ++rep)
    for (int m = 0; m < 3; ++m) {
      const int steps = 20000;
      if (m == 0) chase<0><<<1, 1>>>(d, steps, o);
      if (m == 1) chase<1><<<1, 1>>>(d, steps, o);
      if (m == 2) chase<2><<<1, 1>>>(d, steps, o);
      cudaDeviceSynchronize();
      cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
      printf("chase %-16s %.0f cycles/load\n", names[m], (double)r[0] / steps);
    }
  for (int m = 0; m < 3; ++m) {
    const int rounds = 20000;
    cudaMemset(d, 0, 16);
    if (m == 0) pingpong<0><<<2, 32>>>(d, rounds, o);
    if (m == 1) pingpong<1><<<2, 32>>>(d, rounds, o);
    if (m == 2) pingpong<2><<<2, 32>>>(d, rounds, o);
    cudaDeviceSynchronize();
    cudaMemcpy(r, o, 16, cudaMemcpyDeviceToHost);
    printf("pingpong %-16s %.0f cycles/hop\n", names[m], (double)r[0] / rounds);
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock %d kHz\n", clk);
  return 0;
}
