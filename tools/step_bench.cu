// The fused leaf's decider step in isolation (one warp, P = 5): cycles per step of variants
// of the dependency chain shuffle -> pivot rule -> reciprocal -> own-row update.
//   V0: as leaf_fused3_kernel (two Newton steps, ci = -conj(fj)/|fj|^2, c2 = ci rj)
//   V1: g = -conj(fj) rj beside the reciprocal; 1/x = r0 (1 + e + e^2) (cubic step, one level
//       shorter), folded into c2 = q + q p with q = g r0
//   V2: V1 without the log stores (their issue cost)
//   V3: V0 without the log stores
// POLL > 0: that many extra warps poll the flag with ld.acquire (MIO contention of the holders).
#include <cstdio>
#include <cstdlib>
#include "../paper_1302_6945_b200/csrc/common.cuh"
void tr_set_error(const char*, ...) {}
constexpr unsigned FULL = 0xffffffffu;
constexpr int P = 5;
TR_D cplx shfl_c(cplx v, int src) { return cmk(__shfl_sync(FULL, v.x, src), __shfl_sync(FULL, v.y, src)); }
TR_D double rcp_nr(double x) {
  double r; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0); r = fma(r, e, r); e = fma(-x, r, 1.0); return fma(r, e, r);
}
TR_D cplx sel(const cplx (&v)[P], int j) { cplx r = v[0];
#pragma unroll
  for (int i = 1; i < P; ++i) r = (j == i) ? v[i] : r; return r; }
TR_D int decide_bits(const cplx (&f)[P], const int (&cd)[P], double thr2, cplx& fj, double& a2j) {
  unsigned long long v[P], am[P]; int ix[P]; cplx fv[P]; int dmin = cd[0];
#pragma unroll
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
#pragma unroll
  for (int i = 0; i < P; ++i) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(cabs2(f[i]));
    am[i] = b; v[i] = cd[i] == dmin ? b : 0ull; ix[i] = i; fv[i] = f[i];
  }
#pragma unroll
  for (int w = 1; w < P; w *= 2)
#pragma unroll
    for (int i = 0; i + w < P; i += 2 * w) {
      const bool take = v[i + w] > v[i];
      ix[i] = take ? ix[i + w] : ix[i]; v[i] = take ? v[i + w] : v[i]; fv[i] = take ? fv[i + w] : fv[i];
      am[i] = am[i] > am[i + w] ? am[i] : am[i + w];
    }
  fj = fv[0]; a2j = __longlong_as_double((long long)v[0]);
  const double amax = __longlong_as_double((long long)am[0]);
  if (amax == 0.0 || a2j < thr2 * amax) return -1;
  return ix[0];
}
TR_D unsigned smem_u32(const void* p) { unsigned a = (unsigned)__cvta_generic_to_shared(p); asm volatile("" : "+r"(a)); return a; }
TR_D void sts_c_if(int pred, unsigned addr, cplx v) {
  asm volatile("{ .reg .pred p; setp.ne.s32 p, %0, 0; @p st.shared.v2.f64 [%1], {%2, %3}; }" ::"r"(pred), "r"(addr), "d"(v.x), "d"(v.y) : "memory"); }
TR_D void sts_i_if(int pred, unsigned addr, int v) {
  asm volatile("{ .reg .pred p; setp.ne.s32 p, %0, 0; @p st.shared.u32 [%1], %2; }" ::"r"(pred), "r"(addr), "r"(v) : "memory"); }
TR_D void st_release_if(int pred, unsigned addr, int v) {
  asm volatile("{ .reg .pred p; setp.ne.s32 p, %0, 0; @p st.release.cta.shared.u32 [%1], %2; }" ::"r"(pred), "r"(addr), "r"(v) : "memory"); }
TR_D int ld_acquire(const int* p) { int v; asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"((unsigned)__cvta_generic_to_shared(p)) : "memory"); return v; }

template <int V>
__global__ void __launch_bounds__(384, 1) step_kernel(const cplx* rows, const cplx* sig, int K, int reps, long long* cyc, double* out, int* jout, int mode) {
  extern __shared__ __align__(16) unsigned char raw[];
  cplx* lf = reinterpret_cast<cplx*>(raw);  // [K][P]
  cplx* lci = lf + K * P;                   // [K]
  cplx* lsig = lci + K;                     // [K]
  int* lj = reinterpret_cast<int*>(lsig + K);
  int* flag = lj + K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < K; e += blockDim.x) lsig[e] = sig[e];
  if (tid == 0) flag[0] = 0, flag[1] = 0;
  __syncthreads();
  if (warp == 0) {
    const double thr2 = 1e-16;
    const unsigned a_lf = smem_u32(lf), a_lci = smem_u32(lci), a_lj = smem_u32(lj), a_flag = smem_u32(flag);
    const int pub = lane == 0;
    long long total = 0;
    double acc = 0.0;
    for (int rep = 0; rep < reps; ++rep) {
      int cd[P] = {-48, -48, -48, -48, 0};
      long long t0 = clock64();
      for (int b = 0; b < K / 32; ++b) {
        cplx r[P];
#pragma unroll
        for (int i = 0; i < P; ++i) r[i] = rows[(32 * b + lane) * P + i];
        const cplx sg = lsig[32 * b + lane];
        cplx ci_prev = cmk(0.0, 0.0);
        for (int t = 32 * b; t < 32 * b + 32; ++t) {
          const int src = t & 31;
          cplx f[P];
#pragma unroll
          for (int i = 0; i < P; ++i) f[i] = shfl_c(r[i], src);
          if constexpr (V == 9) {
            if (t > 32 * b) { sts_c_if(pub, a_lci + 16u * (unsigned)(t - 1), ci_prev); st_release_if(pub, a_flag, t); }
          }
          if constexpr (V == 8 || V == 9) {
            const unsigned plf = a_lf + (unsigned)t * (P * 16u);
#pragma unroll
            for (int i = 0; i < P; ++i) sts_c_if(pub, plf + 16u * i, f[i]);
          }
          const cplx sf = lsig[t];
          cplx fj; double a2j;
          const int j = decide_bits(f, cd, thr2, fj, a2j);
          if constexpr (V == 8 || V == 9) sts_i_if(pub, a_lj + 4u * (unsigned)t, j);
          if constexpr (V == 0 || V >= 3) {
            const double inv2 = rcp_nr(a2j);
            const cplx ci = cmk(-fj.x * inv2, fj.y * inv2);
            if constexpr (V == 8) { sts_c_if(pub, a_lci + 16u * (unsigned)t, ci); st_release_if(pub, a_flag, t + 1); }
            if constexpr (V == 9) ci_prev = ci;
            if constexpr (V == 0 || V == 4 || V == 5 || V == 6 || V == 7) {
              const unsigned plf = a_lf + (unsigned)t * (P * 16u);
              if constexpr (V != 5) sts_i_if(pub, a_lj + 4u * (unsigned)t, j);
              sts_c_if(pub, a_lci + 16u * (unsigned)t, ci);
              if constexpr (V == 7) {
                // one STS.128 for the five entries: lane i < P stores f[i]
                cplx pc = f[0];
#pragma unroll
                for (int i = 1; i < P; ++i) pc = (lane == i) ? f[i] : pc;
                sts_c_if(lane < P, plf + 16u * lane, pc);
              } else if constexpr (V != 5) {
#pragma unroll
                for (int i = 0; i < P; ++i) sts_c_if(pub, plf + 16u * i, f[i]);
              }
              if constexpr (V == 0 || V == 5) st_release_if(pub, a_flag, t + 1);
              if constexpr (V == 4) sts_i_if(pub, a_flag, t + 1);
              if constexpr (V == 7) { __syncwarp(); st_release_if(pub, a_flag, t + 1); }
            }
            if (j >= 0) {
              const cplx rj = sel(r, j);
              const cplx c2 = cmul(ci, rj);
              const cplx nj = cmul(rj, csub(sg, sf));
#pragma unroll
              for (int i = 0; i < P; ++i) { const cplx v = cfma(f[i], c2, r[i]); r[i] = (i == j) ? nj : v; }
            }
          } else {
            double r0; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r0) : "d"(a2j));
            const double e = fma(-a2j, r0, 1.0);
            const double p = fma(e, e, e);
            const cplx rj = sel(r, j);
            // g = -conj(fj) rj
            const cplx g = cmk(-(fj.x * rj.x + fj.y * rj.y), fj.y * rj.x - fj.x * rj.y);
            const cplx q = cmk(g.x * r0, g.y * r0);
            const cplx c2 = cmk(fma(q.x, p, q.x), fma(q.y, p, q.y));
            if constexpr (V == 1) {
              const double cx = -fj.x * r0, cy = fj.y * r0;
              const cplx ci = cmk(fma(cx, p, cx), fma(cy, p, cy));
              const unsigned plf = a_lf + (unsigned)t * (P * 16u);
              sts_i_if(pub, a_lj + 4u * (unsigned)t, j);
              sts_c_if(pub, a_lci + 16u * (unsigned)t, ci);
#pragma unroll
              for (int i = 0; i < P; ++i) sts_c_if(pub, plf + 16u * i, f[i]);
              st_release_if(pub, a_flag, t + 1);
            }
            if (j >= 0) {
              const cplx nj = cmul(rj, csub(sg, sf));
#pragma unroll
              for (int i = 0; i < P; ++i) { const cplx v = cfma(f[i], c2, r[i]); r[i] = (i == j) ? nj : v; }
            }
          }
#pragma unroll
          for (int i = 0; i < P; ++i) cd[i] += (i == j);
          if (rep == 0 && lane == 0) jout[t] = j;
        }
        if constexpr (V == 9) { sts_c_if(pub, a_lci + 16u * (unsigned)(32 * b + 31), ci_prev); st_release_if(pub, a_flag, 32 * b + 32); }
#pragma unroll
        for (int i = 0; i < P; ++i) acc += r[i].x + r[i].y;
      }
      total += clock64() - t0;
      if (pub) flag[0] = 0;
      __syncwarp();
    }
    if (lane == 0) cyc[0] = total;
    out[lane] = acc;
  } else if ((warp & 3) != 0) {
    if (mode == 1) {
      // FP64-busy warps (like holders / basis rows replaying): independent DFMA streams, no shared memory
      double a0 = tid, a1 = tid + 1, a2 = tid + 2, a3 = tid + 3;
      while (*(volatile int*)&flag[1] == 0) {
#pragma unroll
        for (int u = 0; u < 16; ++u) { a0 = fma(a0, 1.0000001, 0.5); a1 = fma(a1, 1.0000001, 0.5); a2 = fma(a2, 1.0000001, 0.5); a3 = fma(a3, 1.0000001, 0.5); }
      }
      out[tid] = a0 + a1 + a2 + a3;
      return;
    }
    if (mode == 2) {
      // LDS-busy warps: broadcast LDS.128 streams from the log
      cplx acc2 = cmk(0, 0);
      int k = 0;
      while (*(volatile int*)&flag[1] == 0) {
#pragma unroll
        for (int u = 0; u < 8; ++u) { const volatile double* q = (const volatile double*)&lf[(k + u) % (K * P)]; acc2.x += q[0]; acc2.y += q[1]; }
        k += 8;
      }
      out[tid] = acc2.x + acc2.y;
      return;
    }
    // pollers (never on the decider's scheduler): spin on the flag like the holders / basis rows
    int seen = 0;
    long long spins = 0;
    while (ld_acquire(&flag[1]) == 0) { seen += ld_acquire(&flag[0]); ++spins; }
    if (seen == -1) out[tid] = (double)spins;
  }
  if (warp == 0) { __syncwarp(); if (lane == 0) { flag[1] = 1; __threadfence_block(); } }
}

template <int V>
void run(const char* name, const cplx* rows, const cplx* sig, int K, int reps, int threads, long long* cyc, double* out, int* jout, int mode = 0) {
  const size_t sm = (size_t)K * (P + 2) * sizeof(cplx) + (K + 2) * sizeof(int);
  cudaFuncSetAttribute(step_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  for (int w = 0; w < 2; ++w) { step_kernel<V><<<1, threads, sm>>>(rows, sig, K, reps, cyc, out, jout, mode); cudaDeviceSynchronize(); }
  cudaError_t e = cudaGetLastError();
  double s = 0; for (int i = 0; i < 32; ++i) s += out[i];
  int h[5] = {0, 0, 0, 0, 0}, def = 0; for (int t = 0; t < K; ++t) { if (jout[t] >= 0) h[jout[t]]++; else def++; }
  printf("%-28s threads=%3d  %.1f cycles/step  (pivots %d %d %d %d %d, deferred %d, checksum %.6e) %s\n", name, threads,
         (double)cyc[0] / ((double)reps * K), h[0], h[1], h[2], h[3], h[4], def, s, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  const int K = 192, reps = 50;
  cplx *rows, *sig; long long* cyc; double* out; int* jout;
  cudaMallocManaged(&rows, K * P * sizeof(cplx)); cudaMallocManaged(&sig, K * sizeof(cplx));
  cudaMallocManaged(&cyc, 64); cudaMallocManaged(&out, 512 * sizeof(double)); cudaMallocManaged(&jout, K * sizeof(int));
  srand(7);
  for (int i = 0; i < K * P; ++i) rows[i] = cmk(rand() / (double)RAND_MAX - 0.5, rand() / (double)RAND_MAX - 0.5);
  for (int i = 0; i < K; ++i) { double a = 6.283185307179586 * ((i * 119) % K) / K; sig[i] = cmk(cos(a), sin(a)); }
  for (int threads : {384}) {
    run<0>("V0 current", rows, sig, K, reps, threads, cyc, out, jout);
    run<1>("V1 short chain", rows, sig, K, reps, threads, cyc, out, jout);
    run<3>("V3 current, no log", rows, sig, K, reps, threads, cyc, out, jout);
    run<2>("V2 short chain, no log", rows, sig, K, reps, threads, cyc, out, jout);
    run<4>("V4 current, no fence", rows, sig, K, reps, threads, cyc, out, jout);
    run<5>("V5 ci + release only", rows, sig, K, reps, threads, cyc, out, jout);
    run<6>("V6 data stores, no flag", rows, sig, K, reps, threads, cyc, out, jout);
    run<3>("V3 no log, FP64-busy others", rows, sig, K, reps, threads, cyc, out, jout, 1);
    run<3>("V3 no log, LDS-busy others", rows, sig, K, reps, threads, cyc, out, jout, 2);
    run<5>("V5 ci+rel, FP64-busy others", rows, sig, K, reps, threads, cyc, out, jout, 1);
    run<7>("V7 one STS.128 for f", rows, sig, K, reps, threads, cyc, out, jout);
    run<8>("V8 early f/j stores", rows, sig, K, reps, threads, cyc, out, jout);
    run<9>("V9 V8 + deferred release", rows, sig, K, reps, threads, cyc, out, jout);
  }
  return 0;
}
