// The leaf decider step in isolation (one warp): decide + mu + log + front update.
#include <cstdio>
#include "../paper_1302_6945_b200/csrc/common.cuh"
constexpr unsigned FULL = 0xffffffffu;
TR_D double rcp_nr(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
template <int P> TR_D cplx sel(const cplx (&v)[P], int j) { cplx r = v[0]; for (int i = 1; i < P; ++i) r = (j == i) ? v[i] : r; return r; }
template <int P>
TR_D int decide1(const cplx (&f)[P], const int (&cd)[P], double thr2, cplx& fj) {
  double v[P], am[P]; int ix[P]; cplx fv[P]; int dmin = cd[0];
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
  for (int i = 0; i < P; ++i) { am[i] = cabs2(f[i]); v[i] = cd[i] == dmin ? am[i] : -1.0; ix[i] = i; fv[i] = f[i]; }
  for (int w = 1; w < P; w *= 2)
    for (int i = 0; i + w < P; i += 2 * w) {
      const bool take = v[i + w] > v[i];
      ix[i] = take ? ix[i + w] : ix[i]; v[i] = take ? v[i + w] : v[i]; fv[i] = take ? fv[i + w] : fv[i]; am[i] = fmax(am[i], am[i + w]);
    }
  fj = fv[0];
  if (am[0] == 0.0 || v[0] < thr2 * am[0]) return -1;
  return ix[0];
}
template <int P, int J>
TR_D void mu_j(const cplx (&f)[P], cplx (&mu)[P], int (&cd)[P], cplx fj) {
  const double inv2 = rcp_nr(cabs2(fj));
  const cplx ci = cmk(-fj.x * inv2, fj.y * inv2);
  for (int i = 0; i < P; ++i) mu[i] = (i == J) ? cmk(0.0, 0.0) : cmul(f[i], ci);
  cd[J] += 1;
}
// lean: integer argmax on bit patterns, no mu on the chain (front via ci * qj)
template <int P>
TR_D int decide_int(const cplx (&f)[P], const int (&cd)[P], double thr2, cplx& fj, double& a2j) {
  unsigned long long v[P], am[P]; int ix[P]; cplx fv[P]; int dmin = cd[0];
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
  for (int i = 0; i < P; ++i) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(cabs2(f[i]));
    am[i] = b; v[i] = cd[i] == dmin ? b : 0ull; ix[i] = i; fv[i] = f[i];
  }
  for (int w = 1; w < P; w *= 2)
    for (int i = 0; i + w < P; i += 2 * w) {
      const bool take = v[i + w] > v[i];
      ix[i] = take ? ix[i + w] : ix[i]; v[i] = take ? v[i + w] : v[i]; fv[i] = take ? fv[i + w] : fv[i]; am[i] = am[i] > am[i + w] ? am[i] : am[i + w];
    }
  fj = fv[0];
  a2j = __longlong_as_double((long long)v[0]);
  const double amax = __longlong_as_double((long long)am[0]);
  if (amax == 0.0 || a2j < thr2 * amax) return -1;
  return ix[0];
}
template <int MODE>
__global__ void k(double* out, long long* cyc, int iters) {
  constexpr int P = 5;
  __shared__ cplx lmu[4096 * P];
  __shared__ int lj[4096];
  const int lane = threadIdx.x;
  cplx f[P], pre[P]; int cd[P];
  for (int i = 0; i < P; ++i) { f[i] = cmk(1.0 + 0.37 * i, 0.5 - 0.21 * i); pre[i] = cmk(0.3 * i, 1.0 + 0.1 * i); cd[i] = (i == 1 || i == 2) ? 0 : 5; }
  cplx sf = cmk(1, 0), sp = cmk(0, 1);
  long long t0 = clock64();
  if (MODE == 3) {
    for (int t = 0; t < iters; ++t) {
      cplx fj; double a2j;
      const int j = decide_int<P>(f, cd, 1e-16, fj, a2j);
      const double inv2 = rcp_nr(a2j);
      const cplx ci = cmk(-fj.x * inv2, fj.y * inv2);
      if (lane == 0) { lj[t & 4095] = j; lmu[(t & 4095) * 2] = ci; }
      const cplx qj = sel<P>(pre, j);
      const cplx c2 = cmul(ci, qj);
      const cplx nfj = cmul(qj, csub(sp, sf));
      for (int i = 0; i < P; ++i) {
        const cplx v = cfma(f[i], c2, pre[i]);
        f[i] = (j < 0) ? pre[i] : (i == j) ? nfj : v;
      }
      for (int i = 0; i < P; ++i) cd[i] += (i == j);
      for (int i = 0; i < P; ++i) f[i] = cmk(f[i].x * 0.5 + 0.3 * i, f[i].y * 0.5 - 0.1);
    }
  } else
  for (int t = 0; t < iters; ++t) {
    cplx fj;
    const int j = decide1<P>(f, cd, 1e-16, fj);
    cplx mu[P];
    if (MODE >= 1) {
      switch (j) {
        case 0: mu_j<P, 0>(f, mu, cd, fj); break;
        case 1: mu_j<P, 1>(f, mu, cd, fj); break;
        case 2: mu_j<P, 2>(f, mu, cd, fj); break;
        case 3: mu_j<P, 3>(f, mu, cd, fj); break;
        case 4: mu_j<P, 4>(f, mu, cd, fj); break;
        default: for (int i = 0; i < P; ++i) mu[i] = cmk(0.0, 0.0); break;
      }
    } else {
      for (int i = 0; i < P; ++i) mu[i] = cmul(f[i], fj);
      cd[j & 3] += 1;
    }
    if (MODE >= 2 && lane == 0) { lj[t & 4095] = j; for (int i = 0; i < P; ++i) lmu[(t & 4095) * P + i] = mu[i]; }
    const cplx qj = sel<P>(pre, j);
    const cplx nfj = cmul(qj, csub(sp, sf));
    for (int i = 0; i < P; ++i) {
      const cplx v = cfma(mu[i], qj, pre[i]);
      f[i] = (j < 0) ? pre[i] : (i == j) ? nfj : v;
    }
    // keep magnitudes sane
    for (int i = 0; i < P; ++i) f[i] = cmk(f[i].x * 0.5 + 0.3 * i, f[i].y * 0.5 - 0.1);
  }
  long long t1 = clock64();
  double s = 0; for (int i = 0; i < P; ++i) s += f[i].x + f[i].y;
  out[lane] = s + lj[5];
  if (lane == 0) cyc[0] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 8);
  int iters = 4000; long long h;
  const char* nm[] = {"decide+mul+front", "decide+switch mu+front", "+ log STS", "lean (int argmax, ci qj)"};
#define RUN(M) k<M><<<1, 32>>>(o, c, iters); cudaDeviceSynchronize(); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("%-28s %.1f cycles/step\n", nm[M], (double)h / iters);
  RUN(0) RUN(1) RUN(2) RUN(3)
  return 0;
}
