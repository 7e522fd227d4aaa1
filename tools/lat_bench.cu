// Latency microbenchmarks for the leaf-chain cost model (single warp, clock64).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(double* out, long long* cyc, int n, double s, int sel) {
  double a = threadIdx.x * 1e-3 + 1.0, b = 1.0000001;
  __shared__ double sh[64];
  sh[threadIdx.x] = a;
  __syncthreads();
  long long t0, t1;
  // 0: dependent DFMA
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, s);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  // 1: dependent DMUL
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = a * b;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
  // 2: dependent shuffle (double)
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = __shfl_sync(0xffffffffu, a, (threadIdx.x + 1) & 31) + s;
  t1 = clock64();
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
  // 3: dependent smem load chain
  int idx = threadIdx.x;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double v = sh[idx];
    idx = ((int)v + i) & 31;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[3] = t1 - t0;
  // 4: dependent reciprocal (1.0 / x)
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = 1.0 / (a + s);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[4] = t1 - t0;
  // 5: data-dependent 5-way switch per iteration
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    int k = ((int)(a * 7.0) + sel + i) % 5;
    switch (k) {
      case 0: a = fma(a, b, 0.1); break;
      case 1: a = fma(a, b, 0.2); break;
      case 2: a = fma(a, b, 0.3); break;
      case 3: a = fma(a, b, 0.4); break;
      default: a = fma(a, b, 0.5); break;
    }
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[5] = t1 - t0;
  // 6: __syncthreads round trip (block of blockDim threads)
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    sh[threadIdx.x & 63] = a;
    __syncthreads();
    a += sh[(threadIdx.x + 1) & 63];
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[6] = t1 - t0;
  // 7: double sqrt chain
  t0 = clock64();
  for (int i = 0; i < n; ++i) a = sqrt(a + s);
  t1 = clock64();
  if (threadIdx.x == 0) cyc[7] = t1 - t0;
  // 8: MUFU.RCP64H estimate + dependent DADD (subtract one DFMA latency)
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double r;
    asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a));
    a = r + s;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[8] = t1 - t0;
  // 9: 64-bit unsigned compare + select chain (the pivot tree's level)
  unsigned long long u = (unsigned long long)__double_as_longlong(a), w = u ^ 0x5555ull;
  t0 = clock64();
  for (int i = 0; i < n; ++i) {
    const bool take = w > u;
    const unsigned long long nu = take ? w : u;
    w = (take ? u : w) + 0x10001ull * (unsigned)i;
    u = nu;
  }
  t1 = clock64();
  if (threadIdx.x == 0) cyc[9] = t1 - t0;
  a += __longlong_as_double((long long)(u ^ w));
  out[threadIdx.x] = a;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 4096 * sizeof(double));
  cudaMallocManaged(&cyc, 16 * sizeof(long long));
  const char* names[] = {"DFMA dep", "DMUL dep", "SHFL dep", "LDS dep", "DDIV(1/x) dep",
                         "switch5+DFMA", "syncthreads", "DSQRT dep", "MUFU.RCP64H+DADD", "cmp64+sel"};
  for (int threads : {32, 256, 512}) {
    int n = 1024;
    lat_kernel<<<1, threads>>>(out, cyc, n, 1e-9, 1);
    cudaDeviceSynchronize();
    lat_kernel<<<1, threads>>>(out, cyc, n, 1e-9, 1);
    cudaDeviceSynchronize();
    printf("block=%d:", threads);
    for (int i = 0; i < 10; ++i) printf("  %s=%.1f", names[i], (double)cyc[i] / n);
    printf("\n");
  }
  return 0;
}
