// Batched complex128 FFT for lengths 2^a * q (q odd, q <= 63).
//
// Multi-pass Stockham autosort: a length-n transform is split into 1-3
// passes of radix R_i <= 4096 (one kernel launch each).  Inside a pass a CTA
// stages a tile of T consecutive butterflies (x LB lines) in shared memory and
// runs the length-R sub-transform there with radix-8/4/2 stages plus at most
// one direct odd-radix stage.  Twiddles come from exp(+2 pi i k / n) tables
// computed in long double on the host (0.5 ulp), conjugated for sign < 0.
//
//   y[k] = sum_j x[j] * exp(sign * 2 pi i j k / n)     (unnormalized)
#pragma once
#include "common.cuh"

struct FftPass {
  int R;       // sub-transform length of this pass
  int Ns;      // product of the radices of earlier passes
  int T;       // consecutive butterflies per CTA tile
  int LB;      // lines per CTA (single-pass plans only)
  int nst;     // number of in-smem stages
  int rad[16]; // in-smem stage radices (first the odd one, then 8/4/2)
  const cplx* twR;  // table exp(2 pi i k / R)
  int log2, q;      // R = q * 2^log2
  bool fast;        // compile-time-shaped kernel available (fft_fast.cu)
};

struct FftPlan {
  long long n = 0;
  int npass = 0;
  FftPass pass[3];
  const cplx* twN = nullptr;  // table exp(2 pi i k / n)
  // two-pass column plan n = N1 N2 (fft_col.cu), N1 = 2^a1, N2 = q 2^a2
  bool col = false;
  int a1 = 0, a2 = 0, q2 = 1;
  const cplx* tw1 = nullptr;
  const cplx* tw2 = nullptr;
  const cplx* twc = nullptr;  // [N2][TL] exp(2 pi i n2 l / n) for pass B
};

// Plan (cached per device and length).  Returns 0 on success.
int fft_plan(long long n, FftPlan* out);
// Largest odd factor a plan may contain.
constexpr int FFT_MAX_ODD = 63;
// True when n = 2^a * q with q odd <= FFT_MAX_ODD.
bool fft_supported(long long n);
// Smallest supported length >= n with cheap factors (cost-ranked).
long long fft_good_len(long long n);

// Batched transform of `lines` lines (optionally of in[e] * mul_scale *
// mul[line * mul_ls + e], the product fused into the load).  Line i of the input starts at
// in + i*in_ls and holds in_len <= n valid values (zero-padded to n); the
// output line i starts at out + i*out_ls.  `scratch` must hold lines*n
// values.  in == out is allowed.  With mul2 (two-pass column plans only,
// full-length lines) the loaded value is mul_scale * (in[e] mul[e] +
// conj(in[(n - e) mod n]) mul2[e]).
int fft_exec(const FftPlan& p, const cplx* in, long long in_ls, long long in_len,
             cplx* out, long long out_ls, cplx* scratch, long long lines, int sign,
             cudaStream_t st,
             const cplx* mul = nullptr, long long mul_ls = 0, double mul_scale = 1.0,
             long long chunk_bytes_override = -1, const cplx* mul2 = nullptr);

// Forward (+1) transform of the twisted, folded basis entries of a coset update
// (tree.cu twist_fold_kernel fused into the loads of the single-pass register
// kernel): output line (sys * noff + c) * PP + e = transform of x[q] = sum_{l = q
// mod n, l < L} B[sys][e][l] w^(o_c l), w = exp(2 pi i / N).  Returns -1 when the
// plan is not a single-pass register plan (the caller runs the two kernels).
int fft_exec_twistfold(const FftPlan& p, const cplx* B, long long b_sys, long long b_cap, int PP, long long L,
                       long long o0, long long o1, int noff, long long N, const cplx* twN, cplx* out,
                       long long lines, cudaStream_t st);

// Twiddle table exp(2 pi i k / n), k < n (cached, device memory).
const cplx* twiddle_table(long long n);

// Single-pass cluster / TMA transform (fft_cl.cu) for n in {8192, 12288,
// 16384, 32768, 65536}: one HBM read and write per element.  Returns -1 when
// the shape or device cannot use it (the caller falls back).
bool fft_cl_supported(long long n);
int fft_cl_exec(long long n, const cplx* in, long long in_ls, long long in_len, cplx* out, long long out_ls,
                long long lines, int sign, const cplx* twN, const cplx* mul, long long mul_ls, double mul_scale,
                cudaStream_t st);
