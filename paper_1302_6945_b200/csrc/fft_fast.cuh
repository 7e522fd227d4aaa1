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
};

bool fast_supported(int log2, int q);
int fast_tile(int log2, int q);
// returns 0 on launch, -1 when (log2, q) has no compiled kernel
int fast_launch(int log2, int q, bool small, const FastArgs& a, cudaStream_t st);
// register radix-16 single-pass kernel (fft_reg.cu); -1 when not applicable
int reg_launch(int log2, int q, const FastArgs& a, cudaStream_t st);
