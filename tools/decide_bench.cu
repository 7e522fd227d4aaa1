// cycles of one decide() / row_update() in isolation (1 warp), for the cost model
#include <cstdio>
#include "../paper_1302_6945_b200/csrc/common.cuh"
void tr_set_error(const char*, ...) {}
void tr_kernel_begin(int, cudaStream_t) {}
void tr_kernel_end(int, cudaStream_t) {}
template <int P>
__device__ int decide(const cplx (&phi)[P], const int (&cd)[P], double thr, cplx* mu_out) {
  double a2[P], amax2 = 0.0;
#pragma unroll
  for (int i = 0; i < P; ++i) { a2[i] = cabs2(phi[i]); amax2 = fmax(amax2, a2[i]); }
  if (amax2 == 0.0) return -1;
  int dmin = cd[0];
#pragma unroll
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
  double bm = -1.0; int j = 0; cplx pj = phi[0];
#pragma unroll
  for (int i = 0; i < P; ++i) if (cd[i] == dmin && a2[i] > bm) { bm = a2[i]; j = i; pj = phi[i]; }
  if (bm < thr * thr * amax2) return -1;
  const double inv2 = 1.0 / cabs2(pj);
  const cplx inv = cmk(pj.x * inv2, -pj.y * inv2);
#pragma unroll
  for (int i = 0; i < P; ++i) mu_out[i] = i == j ? cmk(0.0, 0.0) : cneg(cmul(phi[i], inv));
  return j;
}
template <int P> __device__ cplx sel(const cplx (&v)[P], int j) { cplx r = v[0];
#pragma unroll
  for (int i = 1; i < P; ++i) r = (j == i) ? v[i] : r; return r; }
template <int P> __device__ void row_update(cplx (&r)[P], int j, const cplx* mu, cplx dsig) {
  const cplx rj = sel<P>(r, j); const cplx nj = cmul(rj, dsig);
#pragma unroll
  for (int i = 0; i < P; ++i) r[i] = (i == j) ? nj : cfma(mu[i], rj, r[i]); }
__global__ void k(double* out, long long* cyc, int n) {
  cplx phi[5], m[5]; int cd[5] = {0, 1, 0, 1, 2};
  for (int i = 0; i < 5; ++i) phi[i] = cmk(1.0 + i + threadIdx.x, 0.5 * i);
  long long t0 = clock64();
  int acc = 0;
  for (int it = 0; it < n; ++it) {
    int j = decide<5>(phi, cd, 1e-8, m);
    acc += j;
    phi[0] = cadd(phi[0], m[1]);  // dependency into the next call
  }
  long long t1 = clock64();
  cplx mu[5]; for (int i = 0; i < 5; ++i) mu[i] = cmk(1e-3 * i, 2e-3);
  long long t2 = clock64();
  int j = acc & 3;
  for (int it = 0; it < n; ++it) { row_update<5>(phi, (j + it) % 5, mu, cmk(0.5, 0.25)); }
  long long t3 = clock64();
  long long t4 = clock64();
  for (int it = 0; it < n; ++it) { long long x = clock64(); acc += (int)x; }
  long long t5 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t3 - t2; cyc[2] = t5 - t4; }
  out[threadIdx.x] = phi[0].x + acc;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMallocManaged(&c, 64);
  for (int r = 0; r < 2; ++r) { k<<<1, 32>>>(o, c, 256); cudaDeviceSynchronize(); }
  printf("decide=%.1f cyc  row_update=%.1f cyc  clock64=%.1f cyc\n", c[0] / 256.0, c[1] / 256.0, c[2] / 256.0);
}
