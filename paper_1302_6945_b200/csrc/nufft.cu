// Nonuniform Fourier sums for the Gramian-Toeplitz setup (ref:
// pkg/src/toepreg/nufft.py:60-72 weighted_fourier_gramian, :106-114 the
// sampled rhs).  The reference forms exp(2 pi i f_k d) densely (O(K n)
// memory); here each term is generated on the fly:
//
//   adjoint  y[d] = sum_k c_k exp(+-2 pi i f_k d),  d < n
//   forward  y[k] = sum_j x_j exp(+-2 pi i f_k j),  k < K
//
// A thread owns RUN consecutive output lags; for every source term the phase
// at the first lag is reduced exactly (f d = p + e with the FMA remainder e,
// the integer part of p dropped) and fed to sincospi, and the next lags follow
// by multiplying with exp(+-2 pi i f_k) (RUN - 1 rotations, |error| ~ RUN ulp).
// Source terms are staged through shared memory in tiles.
#include "kernels.cuh"

namespace {

constexpr int NT = 256;
constexpr int RUN = 8;
constexpr int TILE = 256;

// exp(sign 2 pi i f d) with the phase reduced mod 1 before the rounding of 2 pi f d
TR_D cplx phase_exp(double f, double d, int sign) {
  const double p = f * d;
  const double e = fma(f, d, -p);  // exact: f d = p + e
  const double r = (p - rint(p)) + e;
  double s, c;
  sincospi(2.0 * r, &s, &c);
  return cmk(c, sign < 0 ? -s : s);
}

// y[d] = sum_k c[k] w(f_k, d); c complex
__global__ void __launch_bounds__(NT) nudft_adjoint_kernel(const double* __restrict__ f, const cplx* __restrict__ c,
                                                           long long K, long long n, int sign, cplx* __restrict__ y) {
  __shared__ double sf[TILE];
  __shared__ cplx sc[TILE], sz[TILE];
  const long long d0 = ((long long)blockIdx.x * NT + threadIdx.x) * RUN;
  cplx acc[RUN];
#pragma unroll
  for (int j = 0; j < RUN; ++j) acc[j] = cmk(0.0, 0.0);
  for (long long k0 = 0; k0 < K; k0 += TILE) {
    const int nk = (int)min((long long)TILE, K - k0);
    __syncthreads();
    for (int i = threadIdx.x; i < nk; i += NT) {
      const double fk = f[k0 + i];
      sf[i] = fk;
      sc[i] = c[k0 + i];
      sz[i] = phase_exp(fk, 1.0, sign);
    }
    __syncthreads();
    if (d0 < n) {
      for (int i = 0; i < nk; ++i) {
        const cplx ck = sc[i], z = sz[i];
        cplx w = cmul(ck, phase_exp(sf[i], (double)d0, sign));
#pragma unroll
        for (int j = 0; j < RUN; ++j) {
          acc[j] = cadd(acc[j], w);
          w = cmul(w, z);
        }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < RUN; ++j)
    if (d0 + j < n) y[d0 + j] = acc[j];
}

// y[k] = sum_j x[j] w(f_k, j)
__global__ void __launch_bounds__(NT) nudft_forward_kernel(const double* __restrict__ f, const cplx* __restrict__ x,
                                                           long long K, long long n, int sign, cplx* __restrict__ y) {
  __shared__ cplx sx[TILE];
  const long long k = (long long)blockIdx.x * NT + threadIdx.x;
  const double fk = k < K ? f[k] : 0.0;
  const cplx z = phase_exp(fk, 1.0, sign);
  cplx acc = cmk(0.0, 0.0);
  for (long long j0 = 0; j0 < n; j0 += TILE) {
    const int nj = (int)min((long long)TILE, n - j0);
    __syncthreads();
    for (int i = threadIdx.x; i < nj; i += NT) sx[i] = x[j0 + i];
    __syncthreads();
    if (k < K) {
      for (int i = 0; i < nj; i += RUN) {
        cplx w = phase_exp(fk, (double)(j0 + i), sign);
        const int m = min(RUN, nj - i);
        for (int u = 0; u < m; ++u) {
          acc = cfma(sx[i + u], w, acc);
          w = cmul(w, z);
        }
      }
    }
  }
  if (k < K) y[k] = acc;
}

}  // namespace

int launch_nudft_adjoint(const double* f, const cplx* c, long long K, long long n, int sign, cplx* y,
                         cudaStream_t st) {
  const long long threads = (n + RUN - 1) / RUN;
  { TrKTimer _kt(TRK_ASSEMBLE, st); nudft_adjoint_kernel<<<(unsigned)((threads + NT - 1) / NT), NT, 0, st>>>(f, c, K, n, sign, y); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_nudft_forward(const double* f, const cplx* x, long long K, long long n, int sign, cplx* y,
                         cudaStream_t st) {
  { TrKTimer _kt(TRK_ASSEMBLE, st); nudft_forward_kernel<<<(unsigned)((K + NT - 1) / NT), NT, 0, st>>>(f, x, K, n, sign, y); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}
