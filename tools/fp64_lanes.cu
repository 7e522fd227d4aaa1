// FP64 issue cost per warp instruction vs active lanes (one warp per SM).
#include <cstdio>
__global__ void k(double* out, long long* cyc, int iters, int active) {
  const int lane = threadIdx.x & 31;
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = lane * 1e-3 + i;
  long long t0 = 0, t1 = 0;
  if (lane < active) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 8; ++i) a[i] = fma(a[i], 0.999999, 1e-7);
    }
    t1 = clock64();
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[threadIdx.x] = s;
  if (lane == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096 * 8); cudaMalloc(&c, 1024 * 8);
  int iters = 100000;
  for (int act : {32, 16, 8, 1}) {
    k<<<1, 32>>>(o, c, iters, act);
    cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("active lanes %2d: %.2f cycles per DFMA warp-instruction (8 independent chains)\n", act, (double)h / (iters * 8.0));
  }
  return 0;
}
