// Named-barrier ping-pong latency between two warps (bar.arrive / bar.sync).
#include <cstdio>
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__global__ void k(long long* cyc, int iters, int* out) {
  __shared__ volatile int buf[64];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  long long t0 = clock64();
  int v = 0;
  for (int it = 0; it < iters; ++it) {
    if (warp == 0) {
      if (lane == 0) buf[0] = it;
      bar_arrive(1, 64);   // publish to warp 1
      bar_sync(2, 64);     // wait for the reply
      v += buf[1];
    } else {
      bar_sync(1, 64);
      const int x = buf[0];
      if (lane == 0) buf[1] = x + 1;
      bar_arrive(2, 64);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = v; }
}
__global__ void k_flag(long long* cyc, int iters, int* out) {
  __shared__ volatile int f0, f1;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { f0 = -1; f1 = -1; }
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (warp == 0) { f0 = it; while (f1 != it) {} }
    else { while (f0 != it) {} f1 = it; }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = f1; }
}
int main() {
  long long* c; int* o; cudaMalloc(&c, 8); cudaMalloc(&o, 4);
  int iters = 10000; long long h;
  k<<<1, 64>>>(c, iters, o); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("named barrier ping-pong: %.1f cycles per round trip\n", (double)h / iters);
  k_flag<<<1, 64>>>(c, iters, o); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("volatile smem flag ping-pong: %.1f cycles per round trip\n", (double)h / iters);
  return 0;
}
