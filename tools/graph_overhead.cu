// Per-node cost of a CUDA graph of back-to-back tiny kernels on one stream.
#include <cstdio>
__global__ void empty_k(int* p) { if (threadIdx.x == 0 && p[0] == 12345) p[1] = 1; }
__global__ void small_k(double* p, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0000001 + 1e-9;
}
int main() {
  int* d; double* x; cudaMalloc(&d, 64); cudaMalloc(&x, 1 << 20);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int kind = 0; kind < 3; ++kind) {
    const int N = 10000;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) {
      if (kind == 0) empty_k<<<1, 32, 0, s>>>(d);
      else if (kind == 1) empty_k<<<64, 256, 0, s>>>(d);
      else small_k<<<256, 256, 0, s>>>(x, 65536);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const char* nm[] = {"empty 1x32", "empty 64x256", "small 256x256"};
    printf("%-16s %.2f us per node\n", nm[kind], ms * 1e3 / N);
    // eager
    cudaEventRecord(a, s);
    for (int i = 0; i < N; ++i) {
      if (kind == 0) empty_k<<<1, 32, 0, s>>>(d);
      else if (kind == 1) empty_k<<<64, 256, 0, s>>>(d);
      else small_k<<<256, 256, 0, s>>>(x, 65536);
    }
    cudaEventRecord(b, s); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("%-16s %.2f us per eager launch\n", nm[kind], ms * 1e3 / N);
  }
  return 0;
}
