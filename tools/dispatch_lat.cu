// Cost of a data-dependent 5-way dispatch: jump table (BRX) vs compare chain vs selects.
#include <cstdio>
__device__ int g_j[4096];
template <int MODE>
__global__ void k(double* out, long long* cyc, int iters) {
  __shared__ int js[4096];
  for (int i = threadIdx.x; i < 4096; i += 32) js[i] = g_j[i];
  __syncwarp();
  double a0 = threadIdx.x, a1 = 1, a2 = 2, a3 = 3, a4 = 4;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    int j = js[(it + (int)(a0 * 1e-300)) & 4095];
    if (MODE == 0) {
      switch (j) {
        case 0: a0 = fma(a0, 1.0000001, 1e-9); break;
        case 1: a1 = fma(a1, 1.0000001, 1e-9); break;
        case 2: a2 = fma(a2, 1.0000001, 1e-9); break;
        case 3: a3 = fma(a3, 1.0000001, 1e-9); break;
        default: a4 = fma(a4, 1.0000001, 1e-9); break;
      }
    } else if (MODE == 1) {
      if (j < 2) { if (j == 0) a0 = fma(a0, 1.0000001, 1e-9); else a1 = fma(a1, 1.0000001, 1e-9); }
      else if (j < 4) { if (j == 2) a2 = fma(a2, 1.0000001, 1e-9); else a3 = fma(a3, 1.0000001, 1e-9); }
      else a4 = fma(a4, 1.0000001, 1e-9);
    } else {
      const double n0 = fma(a0, 1.0000001, 1e-9), n1 = fma(a1, 1.0000001, 1e-9), n2 = fma(a2, 1.0000001, 1e-9),
                   n3 = fma(a3, 1.0000001, 1e-9), n4 = fma(a4, 1.0000001, 1e-9);
      a0 = j == 0 ? n0 : a0; a1 = j == 1 ? n1 : a1; a2 = j == 2 ? n2 : a2; a3 = j == 3 ? n3 : a3; a4 = j == 4 ? n4 : a4;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = a0 + a1 + a2 + a3 + a4;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  int h[4096]; unsigned s = 1; for (int i = 0; i < 4096; ++i) { s = s * 1103515245u + 12345u; h[i] = (s >> 16) % 5; }
  cudaMemcpyToSymbol(g_j, h, sizeof h);
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 8);
  const char* names[] = {"switch", "nested if", "selects"};
  int iters = 20000;
#define RUN(M) { k<M><<<1, 32>>>(o, c, iters); cudaDeviceSynchronize(); long long hh; cudaMemcpy(&hh, c, 8, cudaMemcpyDeviceToHost); printf("%-10s %.1f cycles/iter\n", names[M], (double)hh / iters); }
  RUN(0) RUN(1) RUN(2)
  return 0;
}
