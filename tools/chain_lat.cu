// Latency microbenchmarks for the leaf chain step (one warp, dependent loop).
#include <cstdio>
#include <cstdint>
struct __align__(16) cplx { double x, y; };
__device__ __forceinline__ cplx cmk(double x, double y) { cplx c; c.x = x; c.y = y; return c; }
__device__ __forceinline__ double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ cplx cfma(cplx a, cplx b, cplx c) {
  return cmk(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
__device__ __forceinline__ double rcp_nr(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
constexpr int P = 5;
__device__ __forceinline__ int decide_d(const cplx (&f)[P], const int (&cd)[P], double thr2) {
  double v[P], am[P]; int ix[P]; int dmin = cd[0];
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
  for (int i = 0; i < P; ++i) { am[i] = cabs2(f[i]); v[i] = cd[i] == dmin ? am[i] : -1.0; ix[i] = i; }
  for (int w = 1; w < P; w *= 2)
    for (int i = 0; i + w < P; i += 2 * w) {
      bool take = v[i + w] > v[i]; ix[i] = take ? ix[i + w] : ix[i]; v[i] = take ? v[i + w] : v[i]; am[i] = fmax(am[i], am[i + w]);
    }
  if (am[0] == 0.0 || v[0] < thr2 * am[0]) return -1;
  return ix[0];
}
// integer-compare variant: nonnegative doubles order like their bit patterns
__device__ __forceinline__ int decide_i(const cplx (&f)[P], const int (&cd)[P], double thr2) {
  long long v[P], am[P]; int ix[P]; int dmin = cd[0];
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
  for (int i = 0; i < P; ++i) { long long b = __double_as_longlong(cabs2(f[i])); am[i] = b; v[i] = cd[i] == dmin ? b : -1; ix[i] = i; }
  for (int w = 1; w < P; w *= 2)
    for (int i = 0; i + w < P; i += 2 * w) {
      bool take = v[i + w] > v[i]; ix[i] = take ? ix[i + w] : ix[i]; v[i] = take ? v[i + w] : v[i]; am[i] = max(am[i], am[i + w]);
    }
  double amd = __longlong_as_double(am[0]);
  if (am[0] == 0 || __longlong_as_double(v[0]) < thr2 * amd || v[0] < 0) return -1;
  return ix[0];
}
template <int MODE>
__global__ void k(double* out, long long* cyc, int iters) {
  const int lane = threadIdx.x;
  cplx f[P]; int cd[P];
  for (int i = 0; i < P; ++i) { f[i] = cmk(1.0 + 0.1 * i + lane * 1e-9, 0.3 - 0.05 * i); cd[i] = i & 1; }
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {  // decide (double compares) -> feeds back
      int j = decide_d(f, cd, 1e-16);
      f[0].x += j * 1e-30;
    } else if (MODE == 1) {  // decide (int compares)
      int j = decide_i(f, cd, 1e-16);
      f[0].x += j * 1e-30;
    } else if (MODE == 2) {  // rcp chain: |f|^2 -> rcp -> ci -> mu -> f
      double inv2 = rcp_nr(cabs2(f[1]));
      cplx ci = cmk(-f[1].x * inv2, f[1].y * inv2);
      cplx m = cmul(f[0], ci);
      f[1] = cfma(m, f[2], f[1]);
    } else if (MODE == 3) {  // 20 SHFL (5 complex) broadcast, dependent
      for (int i = 0; i < P; ++i) { f[i].x = __shfl_sync(0xffffffffu, f[i].x, (lane + 1) & 31); f[i].y = __shfl_sync(0xffffffffu, f[i].y, (lane + 1) & 31); }
      f[0].x += f[4].y * 1e-30;
    } else if (MODE == 4) {  // 5-way dispatch on a data value
      int j = (int)(f[0].x * 1e9) % 5;
      if (j == 0) f[1].x += 1e-30; else if (j == 1) f[2].x += 1e-30; else if (j == 2) f[3].x += 1e-30; else if (j == 3) f[4].x += 1e-30; else f[0].y += 1e-30;
      f[0].x += 1e-12;
    } else if (MODE == 5) {  // scaled update: exponent -> scale -> cmsub
      cplx fj = f[1];
      double mx = fmax(fabs(fj.x), fabs(fj.y));
      int e = (__double2hiint(mx) >> 20) & 0x7ff;
      double sc = __hiloint2double((2046 - e) << 20, 0);
      cplx pj = cmk(fj.x * sc, fj.y * sc);
      cplx a = cmul(pj, f[2]); cplx b = cmul(cmk(f[0].x * sc, f[0].y * sc), f[3]);
      f[1] = cmk(a.x - b.x, a.y - b.y);
    } else if (MODE == 6) {  // one DFMA dependent chain (baseline)
      f[0].x = fma(f[0].x, 0.999, 1e-9);
    } else if (MODE == 7) {  // smem round trip (STS by lane 0, LDS broadcast)
      __shared__ cplx buf[8];
      if (lane == 0) buf[it & 7] = f[0];
      __syncwarp();
      f[0] = buf[it & 7]; f[0].x += 1e-30;
    }
  }
  long long t1 = clock64();
  for (int i = 0; i < P; ++i) acc += f[i].x + f[i].y;
  out[lane] = acc;
  if (lane == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 8);
  const char* names[] = {"decide (DSETP tree)", "decide (int tree)", "rcp->mu->cfma chain", "20 SHFL dep", "5-way dispatch", "scaled update", "DFMA dep", "smem round trip"};
  int iters = 20000;
#define RUN(M) { k<M><<<1, 32>>>(o, c, iters); cudaDeviceSynchronize(); long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("%-24s %.1f cycles/iter\n", names[M], (double)h / iters); }
  RUN(0) RUN(1) RUN(2) RUN(3) RUN(4) RUN(5) RUN(6) RUN(7)
  return 0;
}
