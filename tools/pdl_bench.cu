#include <cstdio>
__device__ __forceinline__ void gd_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void gd_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
template <bool PDL>
__global__ void small_k(double* p, int n) {
  if (PDL) { gd_launch(); gd_wait(); }
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = p[i] * 1.0000001 + 1e-9;
}
template <bool PDL>
__global__ void mid_k(double* p, int n) {   // ~ a few us of work
  if (PDL) { gd_launch(); gd_wait(); }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = p[i] * 1.0000001 + 1e-9;
}
int main() {
  double* x; cudaMalloc(&x, 64 << 20);
  cudaStream_t s; cudaStreamCreate(&s);
  for (int kind = 0; kind < 4; ++kind) {
    const int N = 4000;
    bool pdl = kind & 1;
    bool mid = kind >= 2;
    cudaGraph_t g; cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(mid ? 296 : 256); cfg.blockDim = dim3(256); cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at; cfg.numAttrs = pdl ? 1 : 0;
      int n = mid ? (4 << 20) : 65536;
      if (mid) { if (pdl) cudaLaunchKernelEx(&cfg, mid_k<true>, x, n); else cudaLaunchKernelEx(&cfg, mid_k<false>, x, n); }
      else { if (pdl) cudaLaunchKernelEx(&cfg, small_k<true>, x, n); else cudaLaunchKernelEx(&cfg, small_k<false>, x, n); }
    }
    cudaStreamEndCapture(s, &g);
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) { printf("instantiate failed\n"); return 1; }
    cudaGraphLaunch(ge, s); cudaStreamSynchronize(s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s); cudaGraphLaunch(ge, s); cudaEventRecord(b, s); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("%s %s: %.2f us per node (%s)\n", mid ? "mid(32MB rw)" : "small", pdl ? "PDL" : "plain", ms * 1e3 / N,
           cudaGetErrorString(cudaGetLastError()));
  }
}
