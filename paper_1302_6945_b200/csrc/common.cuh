// Shared device helpers for the B200 Tikhonov-Toeplitz solver.
// complex128 values are double2 {re, im}; all arithmetic is FP64.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define TR_HD __host__ __device__ __forceinline__
#define TR_D __device__ __forceinline__

typedef double2 cplx;

TR_HD cplx cmk(double r, double i) { cplx c; c.x = r; c.y = i; return c; }
TR_HD cplx cadd(cplx a, cplx b) { return cmk(a.x + b.x, a.y + b.y); }
TR_HD cplx csub(cplx a, cplx b) { return cmk(a.x - b.x, a.y - b.y); }
TR_HD cplx cmul(cplx a, cplx b) {
  return cmk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a*b + c with fused multiply-adds
TR_D cplx cfma(cplx a, cplx b, cplx c) {
  double re = fma(a.x, b.x, fma(-a.y, b.y, c.x));
  double im = fma(a.x, b.y, fma(a.y, b.x, c.y));
  return cmk(re, im);
}
TR_HD cplx cscale(cplx a, double s) { return cmk(a.x * s, a.y * s); }
TR_HD cplx cconj(cplx a) { return cmk(a.x, -a.y); }
TR_HD double cabs2(cplx a) { return a.x * a.x + a.y * a.y; }
TR_HD cplx cneg(cplx a) { return cmk(-a.x, -a.y); }
// conj(w) when sign < 0
TR_HD cplx csign(cplx w, int sign) { return sign < 0 ? cconj(w) : w; }

// exp(2 pi i k / n) for integer k (any sign), accurate to ~1 ulp.
TR_D cplx unit_root(long long k, long long n) {
  long long r = k % n;
  if (r < 0) r += n;
  // x = 2r/n in [0, 2); fold to [-1, 1) so sincospi works on a small argument
  double x = (2.0 * (double)r) / (double)n;
  if (2 * r >= n) x = (2.0 * (double)(r - n)) / (double)n;
  double s, c;
  sincospi(x, &s, &c);
  return cmk(c, s);
}

// numpy's complex division (Smith's method), so mu matches the reference's
// rounding as closely as a different evaluation order allows.
TR_D cplx cdiv_np(cplx a, cplx b) {
  double br = b.x, bi = b.y;
  if (fabs(br) >= fabs(bi)) {
    double rat = bi / br;
    double scl = 1.0 / (br + bi * rat);
    return cmk((a.x + a.y * rat) * scl, (a.y - a.x * rat) * scl);
  }
  double rat = br / bi;
  double scl = 1.0 / (bi + br * rat);
  return cmk((a.x * rat + a.y) * scl, (a.y * rat - a.x) * scl);
}

// |z| as numpy does (hypot) for the rare places where the exact modulus
// value (not only its ordering) matters.
TR_D double cabs(cplx a) { return hypot(a.x, a.y); }

// order-preserving bit pattern of a non-negative double for atomicMax
TR_D unsigned long long dbits(double v) { return (unsigned long long)__double_as_longlong(v); }
TR_D double dfrom(unsigned long long b) { return __longlong_as_double((long long)b); }

#define TR_CUDA_CHECK(expr)                                                    \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      tr_set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e),         \
                   __FILE__, __LINE__, cudaGetErrorString(_e));                \
      return 4;                                                                \
    }                                                                          \
  } while (0)

void tr_set_error(const char* fmt, ...);

// Kernel classes for launch counting and optional per-class CUDA-event timing
// (tr_kernel_timing / tr_kernel_stats in the C ABI).
enum {
  TRK_ASSEMBLE = 0,
  TRK_FFT,
  TRK_LEAF_PIVOT,
  TRK_LEAF_BUILD,
  TRK_LEAF_CHECK,
  TRK_LEAF_EXACT,
  TRK_UPDATE,
  TRK_COMBINE,
  TRK_NORMAL,
  TRK_FINISH,
  TRK_NCLASS
};
void tr_kernel_begin(int cls, cudaStream_t st);
void tr_kernel_end(int cls, cudaStream_t st);
// algorithmic work of a launch (counted only while timing is enabled)
void tr_kernel_work(int cls, double bytes, double flops);
struct TrKTimer {
  int cls;
  cudaStream_t st;
  TrKTimer(int c, cudaStream_t s) : cls(c), st(s) { tr_kernel_begin(c, s); }
  ~TrKTimer() { tr_kernel_end(cls, st); }
};
