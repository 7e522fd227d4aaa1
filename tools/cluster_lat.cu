// Graph node-to-node latency of dependent kernels with and without a cluster
// dimension, and overlap of cluster kernels with a 1-CTA-per-SM kernel on another
// stream (models the fused FFT next to the other group's leaf sweep).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void small_k(double* p, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0000001 + 1e-9;
}
// spins ~us microseconds, one CTA per SM sized like the leaf kernel (big smem)
__global__ void __launch_bounds__(384, 1) hog_k(long long cycles, double* p) {
  extern __shared__ double sm[];
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 0 && p) p[blockIdx.x] = sm[0];
}
// FFT-like: 256 threads, 66 KB smem, ~work microseconds
__global__ void __launch_bounds__(256, 2) work_k(long long cycles, double* p) {
  extern __shared__ double sm[];
  long long t0 = clock64();
  while (clock64() - t0 < cycles) {
  }
  if (threadIdx.x == 0 && p) p[blockIdx.x] = sm[0];
}
static float run_chain(cudaStream_t s, int N, int cluster, int ctas, double* x) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < N; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ctas);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cluster ? cluster : 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = (cluster && (cluster > 0) && (i % 2 == 0 || cluster < 100)) ? 1 : 0;
    cudaLaunchKernelEx(&cfg, small_k, x, 65536);
  }
  cudaStreamEndCapture(s, &g);
  if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) return -1.f;
  cudaGraphLaunch(ge, s);
  cudaStreamSynchronize(s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, s);
  cudaGraphLaunch(ge, s);
  cudaEventRecord(b, s);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / N;
}
int main() {
  double* x;
  cudaMalloc(&x, 64 << 20);
  cudaStream_t s, s2;
  cudaStreamCreate(&s);
  cudaStreamCreate(&s2);
  for (int ctas : {32, 256}) {
    printf("chain of 2000 dependent graph nodes, %d CTAs: plain %.2f us/node, cluster4 %.2f, cluster8 %.2f\n", ctas,
           run_chain(s, 2000, 0, ctas, x), run_chain(s, 2000, 4, ctas, x), run_chain(s, 2000, 8, ctas, x));
  }
  // overlap: stream A = hog on nh SMs for 100 us (x20 back to back), stream B = work kernels (cluster or
  // not) of 3200*4 CTAs each ~10 us per CTA.  One graph with two branches.
  cudaFuncSetAttribute(hog_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  cudaFuncSetAttribute(work_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const long long us = 1965;  // cycles per microsecond
  for (int nh : {0, 32, 128}) {
    for (int cluster : {0, 4}) {
      for (int prio = 0; prio < 2; ++prio) {
        cudaGraph_t g;
        cudaGraphExec_t ge;
        cudaEvent_t fork, join;
        cudaEventCreateWithFlags(&fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&join, cudaEventDisableTiming);
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        cudaEventRecord(fork, s);
        cudaStreamWaitEvent(s2, fork, 0);
        if (nh)
          for (int i = 0; i < 20; ++i) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(nh);
            cfg.blockDim = dim3(384);
            cfg.dynamicSmemBytes = 150 * 1024;
            cfg.stream = s2;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributePriority;
            at[0].val.priority = -1;
            cfg.attrs = at;
            cfg.numAttrs = prio ? 1 : 0;
            cudaLaunchKernelEx(&cfg, hog_k, 100 * us, (double*)nullptr);
          }
        cudaEventRecord(join, s2);
        for (int i = 0; i < 4; ++i) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(3200 * 4);
          cfg.blockDim = dim3(256);
          cfg.dynamicSmemBytes = 66 * 1024;
          cfg.stream = s;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeClusterDimension;
          at[0].val.clusterDim.x = 4;
          at[0].val.clusterDim.y = 1;
          at[0].val.clusterDim.z = 1;
          cfg.attrs = at;
          cfg.numAttrs = cluster ? 1 : 0;
          cudaLaunchKernelEx(&cfg, work_k, 10 * us, (double*)nullptr);
        }
        cudaStreamWaitEvent(s, join, 0);
        cudaStreamEndCapture(s, &g);
        if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
          printf("instantiate failed\n");
          return 1;
        }
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a, s);
        cudaGraphLaunch(ge, s);
        cudaEventRecord(b, s);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        // ideal: work alone = 4 * 12800 CTAs * 10 us / 296 slots = 1730 us; hog alone = 2000 us
        printf("hog %3d SMs x 20 x 100us %s | 4 work kernels (12800 CTAs x 10us, %s): %.0f us (%s)\n", nh,
               prio ? "high-prio" : "same-prio", cluster ? "cluster 4" : "no cluster", ms * 1e3,
               cudaGetErrorString(cudaGetLastError()));
      }
    }
  }
  return 0;
}
