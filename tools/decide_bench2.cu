#include <cstdio>
#include "../paper_1302_6945_b200/csrc/common.cuh"
void tr_set_error(const char*, ...) {}
void tr_kernel_begin(int, cudaStream_t) {}
void tr_kernel_end(int, cudaStream_t) {}
__device__ __forceinline__ double rcp_fast(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
template <int P>
__device__ int decide2(const cplx (&phi)[P], const int (&cd)[P], double thr, cplx* mu_out) {
  double a2[P];
#pragma unroll
  for (int i = 0; i < P; ++i) a2[i] = cabs2(phi[i]);
  int dmin = cd[0];
#pragma unroll
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
  // amax2 and the candidate argmax as two small trees
  double k[P];
#pragma unroll
  for (int i = 0; i < P; ++i) k[i] = cd[i] == dmin ? a2[i] : -1.0;
  double m01 = fmax(a2[0], a2[1]), m23 = fmax(a2[2], a2[3]);
  double amax2 = fmax(fmax(m01, m23), a2[4]);
  // first index of the max key (ties -> lowest index)
  int j01 = k[1] > k[0] ? 1 : 0; double v01 = fmax(k[0], k[1]);
  int j23 = k[3] > k[2] ? 3 : 2; double v23 = fmax(k[2], k[3]);
  int j03 = v23 > v01 ? j23 : j01; double v03 = fmax(v01, v23);
  int j = k[4] > v03 ? 4 : j03; double bm = fmax(v03, k[4]);
  if (amax2 == 0.0 || bm < thr * thr * amax2) return -1;
  cplx pj = phi[0];
#pragma unroll
  for (int i = 1; i < P; ++i) pj = (j == i) ? phi[i] : pj;
  const double inv2 = rcp_fast(cabs2(pj));
  const cplx inv = cmk(pj.x * inv2, -pj.y * inv2);
#pragma unroll
  for (int i = 0; i < P; ++i) mu_out[i] = i == j ? cmk(0.0, 0.0) : cneg(cmul(phi[i], inv));
  return j;
}
__global__ void k(double* out, long long* cyc, int n) {
  cplx phi[5], m[5]; int cd[5] = {0, 1, 0, 1, 2};
  for (int i = 0; i < 5; ++i) phi[i] = cmk(1.0 + i + threadIdx.x, 0.5 * i);
  long long t0 = clock64();
  int acc = 0;
  for (int it = 0; it < n; ++it) {
    int j = decide2<5>(phi, cd, 1e-8, m);
    acc += j;
    phi[0] = cadd(phi[0], m[1]);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
  out[threadIdx.x] = phi[0].x + acc;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, c, 256); cudaDeviceSynchronize(); }
  printf("decide2=%.1f cyc\n", c[0] / 256.0);
}
