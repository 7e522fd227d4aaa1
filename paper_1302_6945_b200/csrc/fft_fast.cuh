// Compile-time-shaped FFT pass kernels (see fft_fast.cu).
#pragma once
#include "common.cuh"

struct FastArgs {
  const cplx* in;
  long long in_ls;
  int in_len;     // valid values per input line (zero padded beyond)
  cplx* out;
  long long out_ls;
  long long nsub; // lines * J sub-transforms
  int J;          // n / R
  int Ns;         // product of earlier radices (power of two)
  int log2Ns;
  int tws;        // n / (Ns * R)
  const cplx* twN;
  const cplx* twR;
  int sign;
  // optional pointwise factor applied on load: x[e] * mul_scale * mul[line * mul_ls + e]
  const cplx* mul = nullptr;
  long long mul_ls = 0;
  double mul_scale = 1.0;
  // optional twist + fold on load (fft_reg.cu TF variant; the coset update of
  // tree.cu twist_fold_kernel fused into the transform): line = (sys * tf_noff
  // + c) * tf_PP + e reads x[q] = sum_{l = q mod R, l < tf_L} B[sys][e][l] w^(o_c l),
  // w = exp(2 pi i / tf_N) from tf_twN, o_c = c ? tf_o1 : tf_o0
  const cplx* tf_B = nullptr;
  long long tf_bsys = 0, tf_bcap = 0, tf_L = 0, tf_o0 = 0, tf_o1 = 0, tf_N = 0;
  int tf_PP = 0, tf_noff = 1;
  const cplx* tf_twN = nullptr;
};

bool fast_supported(int log2, int q);
int fast_tile(int log2, int q);
// returns 0 on launch, -1 when (log2, q) has no compiled kernel
int fast_launch(int log2, int q, bool small, const FastArgs& a, cudaStream_t st);
// register radix-16 single-pass kernel (fft_reg.cu); -1 when not applicable
int reg_launch(int log2, int q, const FastArgs& a, cudaStream_t st);

// two-pass column/row kernels for n = N1 N2 (fft_col.cu)
struct ColArgs {
  const cplx* in;
  long long in_ls, in_len;
  int in_es;          // element stride inside a sub-transform
  cplx* out;
  long long out_ls;
  int out_es;
  int subs;           // sub-transforms per line
  long long lines;
  const cplx* twR;    // exp(2 pi i k / R)
  const cplx* twN;    // exp(2 pi i k / n)
  const cplx* tw2;    // pass B: exp(2 pi i n2 l / n), [N2][TL]
  int sign;
  // pass A only: pointwise factor on load, x[gi] * mul_scale * mul[line * mul_ls + gi]
  const cplx* mul = nullptr;
  long long mul_ls = 0;
  double mul_scale = 1.0;
  // with mul2 (same strides, full-length lines): mul_scale * (x[gi] mul[gi] +
  // conj(x[(n - gi) mod n]) mul2[gi]) -- the spectrum product of a real sequence
  // transformed as a half-length complex one (solver.cu, real CG refinement)
  const cplx* mul2 = nullptr;
};
// sub-transforms per CTA of the column kernels for transform length R
inline int col_tile(int R) {
  int p = 1;
  while (p < R) p <<= 1;
  int t = 4096 / p;
  return t > 16 ? 16 : (t < 4 ? 4 : t);
}
int col_launch(bool pass_a, int log2, int q, const ColArgs& a, cudaStream_t st);
// both passes in one cluster launch (a: pass A into the scratch slots, b: pass B out of them)
int col2_launch(int a1, int a2, int q2, const ColArgs& a, const ColArgs& b, long long n, cudaStream_t st);
