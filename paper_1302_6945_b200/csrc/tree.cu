// Divide-and-conquer tree kernels (ref: pkg/src/toepreg/tanint.py:368-393):
//  * coset update: twist + fold of the left basis (ref fftpoly.py:64-89
//    grid_eval), the DFT (fft.cu), then w <- w . B(sigma) in place;
//  * combine: B_left B_right by FFT (fft.cu), P x P x P product per
//    frequency, trim at 1e-14 of the global max and column normalisation
//    (ref fftpoly.py:148-155, :215-249; tanint.py:379-385).
#include "kernels.cuh"

namespace {

__global__ void twist_fold_kernel(cplx* G, const cplx* B, long long b_sys, long long b_cap, int PP,
                                  long long L, long long o0, long long o1, int noff, long long cnt,
                                  long long N, const cplx* twN) {
  long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int ce = blockIdx.y;  // coset * PP + entry
  long long sys = blockIdx.z;
  if (q >= cnt) return;
  int c = ce / PP, e = ce % PP;
  long long oc = c ? o1 : o0;
  const cplx* src = B + sys * b_sys + (long long)e * b_cap;
  cplx acc = cmk(0.0, 0.0);
  if (oc == 0) {
    for (long long l = q; l < L; l += cnt) acc = cadd(acc, src[l]);
  } else {
    // twist index oc l mod N, stepped by oc cnt < N (no 64-bit modulo in the loop)
    long long idx = (oc * q) % N;
    const long long step = (oc * cnt) % N;
    for (long long l = q; l < L; l += cnt) {
      acc = cfma(src[l], __ldg(&twN[idx]), acc);
      idx += step;
      if (idx >= N) idx -= N;
    }
  }
  G[((sys * noff + c) * PP + e) * cnt + q] = acc;
}

template <int P>
__global__ void apply_update_kernel(cplx* W, long long w_sys, const cplx* G, int rows, long long o0,
                                    long long o1, int noff, long long stride, long long cnt) {
  long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int c = blockIdx.y;
  long long sys = blockIdx.z;
  if (t >= cnt) return;
  long long node = (c ? o1 : o0) + stride * t;
  const cplx* g = G + (sys * noff + c) * (long long)P * P * cnt + t;
  cplx* w = W + sys * w_sys + node * rows * P;
  for (int r = 0; r < rows; ++r) {
    cplx old[P];
#pragma unroll
    for (int i = 0; i < P; ++i) old[i] = w[r * P + i];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      cplx acc = cmk(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < P; ++i) acc = cfma(old[i], g[(long long)(i * P + k) * cnt], acc);
      w[r * P + k] = acc;
    }
  }
}

template <int P>
__global__ void pointwise_matmul_kernel(cplx* FA, const cplx* FB, long long R) {
  long long f = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long sys = blockIdx.y;
  if (f >= R) return;
  cplx* a = FA + sys * (long long)P * P * R + f;
  const cplx* b = FB + sys * (long long)P * P * R + f;
  for (int i = 0; i < P; ++i) {
    cplx ar[P];
#pragma unroll
    for (int k = 0; k < P; ++k) ar[k] = a[(long long)(i * P + k) * R];
    cplx cr[P];
#pragma unroll
    for (int jj = 0; jj < P; ++jj) {
      cplx acc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < P; ++k) acc = cfma(ar[k], b[(long long)(k * P + jj) * R], acc);
      cr[jj] = acc;
    }
#pragma unroll
    for (int jj = 0; jj < P; ++jj) a[(long long)(i * P + jj) * R] = cr[jj];
  }
}

__device__ __forceinline__ double block_max256(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double m = sh[0];
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = fmax(m, sh[w]);
  __syncthreads();
  return m;
}

// profile[l] = max_e |F[e][l]|, global max
__global__ void trim1_kernel(TrimArgs a) {
  __shared__ double sh[32];
  long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long sys = blockIdx.y;
  const int PP = a.P * a.P;
  double m = 0.0;
  if (l < a.L) {
    const cplx* F = a.F + sys * PP * a.R + l;
    for (int e = 0; e < PP; ++e) m = fmax(m, cabs(F[(long long)e * a.R]));
    a.prof[sys * a.L + l] = m;
  }
  double bm = block_max256(m, sh);
  if (threadIdx.x == 0) atomicMax(&a.red[sys * (2 + a.P)], dbits(bm));
}

// last significant index (+1)
__global__ void trim2_kernel(TrimArgs a) {
  __shared__ double sh[32];
  long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long sys = blockIdx.y;
  double gmax = dfrom(a.red[sys * (2 + a.P)]);
  double v = -1.0;
  if (l < a.L && a.prof[sys * a.L + l] > 1e-14 * gmax) v = (double)(l + 1);
  double bm = block_max256(v, sh);
  if (threadIdx.x == 0 && bm > 0.0)
    atomicMax(&a.red[sys * (2 + a.P) + 1], (unsigned long long)bm);
}

// per-column max over the kept range
__global__ void trim3_kernel(TrimArgs a) {
  __shared__ double sh[32];
  long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long sys = blockIdx.y;
  const int P = a.P, PP = P * P;
  unsigned long long* red = a.red + sys * (2 + P);
  long long lt = (long long)red[1];
  if (lt < 1) lt = 1;
  const cplx* F = a.F + sys * PP * a.R + l;
  for (int j = 0; j < P; ++j) {
    double m = 0.0;
    if (l < lt && l < a.L)
      for (int i = 0; i < P; ++i) m = fmax(m, cabs(F[(long long)(i * P + j) * a.R]));
    double bm = block_max256(m, sh);
    if (threadIdx.x == 0) atomicMax(&red[2 + j], dbits(bm));
  }
}

__global__ void trim4_kernel(TrimArgs a) {
  long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long sys = blockIdx.y;
  const int P = a.P, PP = P * P;
  const unsigned long long* red = a.red + sys * (2 + P);
  long long lt = (long long)red[1];
  if (lt < 1) lt = 1;
  long long lw = lt < a.cap_node ? lt : a.cap_node;
  if (l < a.cap) {
    const cplx* F = a.F + sys * PP * a.R + l;
    cplx* o = a.out + sys * a.out_sys + l;
    for (int i = 0; i < P; ++i)
      for (int j = 0; j < P; ++j) {
        cplx v = cmk(0.0, 0.0);
        if (l < lw) {
          double cm = dfrom(red[2 + j]);
          double safe = cm > 0.0 ? cm : 1.0;
          cplx f = F[(long long)(i * P + j) * a.R];
          v = cmk(f.x / safe, f.y / safe);
        }
        o[(long long)(i * P + j) * a.cap] = v;
      }
  }
  if (l == 0) {
    double ms = 1.0;
    bool first = true;
    for (int j = 0; j < P; ++j) {
      double cm = dfrom(red[2 + j]) / (double)a.R;
      double safe = cm > 0.0 ? cm : 1.0;
      ms = first ? safe : fmax(ms, safe);
      first = false;
    }
    a.max_scale[sys] = fmax(a.max_scale[sys], ms);
    if (lt > a.cap_node) a.trim_over[sys] += 1;
  }
}

// All four trim phases in one CTA per system (batches of many systems):
// profile + global max, last significant index, column maxima over the kept
// range, scaled write-out.  Same rule as trim1..4 (squared moduli).
constexpr int TF = 512;

__device__ __forceinline__ double bmax512(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double m = sh[0];
#pragma unroll
  for (int w = 1; w < TF / 32; ++w) m = fmax(m, sh[w]);
  return m;
}

template <int P>
__global__ void __launch_bounds__(TF) trim_fused_kernel(TrimArgs a) {
  __shared__ double sh[TF / 32];
  const long long sys = blockIdx.x;
  constexpr int PP = P * P;
  const cplx* F = a.F + sys * PP * a.R;
  double* prof = a.prof + sys * a.L;
  double gm = 0.0;
  for (long long l = threadIdx.x; l < a.L; l += TF) {
    double m = 0.0;
#pragma unroll
    for (int e = 0; e < PP; ++e) m = fmax(m, cabs2(F[(long long)e * a.R + l]));
    prof[l] = m;
    gm = fmax(gm, m);
  }
  gm = bmax512(gm, sh);
  const double thr = 1e-28 * gm;  // (1e-14)^2 on squared moduli
  double last = 0.0;
  for (long long l = threadIdx.x; l < a.L; l += TF)
    if (prof[l] > thr) last = fmax(last, (double)(l + 1));
  last = bmax512(last, sh);
  long long lt = (long long)last;
  if (lt < 1) lt = 1;
  const long long lw = lt < a.cap_node ? lt : a.cap_node;
  double cm[P];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    double m = 0.0;
    for (long long l = threadIdx.x; l < lt && l < a.L; l += TF)
#pragma unroll
      for (int i = 0; i < P; ++i) m = fmax(m, cabs2(F[(long long)(i * P + j) * a.R + l]));
    cm[j] = sqrt(bmax512(m, sh));
  }
  cplx* o = a.out + sys * a.out_sys;
  for (long long l = threadIdx.x; l < a.cap; l += TF) {
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        cplx v = cmk(0.0, 0.0);
        if (l < lw) {
          const double safe = cm[j] > 0.0 ? cm[j] : 1.0;
          const cplx f = F[(long long)(i * P + j) * a.R + l];
          v = cmk(f.x / safe, f.y / safe);
        }
        o[(long long)(i * P + j) * a.cap + l] = v;
      }
  }
  if (threadIdx.x == 0) {
    double ms = 1.0;
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const double c = cm[j] / (double)a.R;
      const double safe = c > 0.0 ? c : 1.0;
      ms = j == 0 ? safe : fmax(ms, safe);
    }
    a.max_scale[sys] = fmax(a.max_scale[sys], ms);
    if (lt > a.cap_node) a.trim_over[sys] += 1;
  }
}

inline dim3 g2(long long n, long long nsys, int th = 256) {
  return dim3((unsigned)((n + th - 1) / th), (unsigned)nsys);
}

}  // namespace

int launch_twist_fold(cplx* G, const cplx* B, long long b_sys, long long b_cap, int PP, long long L,
                      long long o0, long long o1, int noff, long long cnt, long long N,
                      const cplx* twN, long long nsys, cudaStream_t st) {
  dim3 grid((unsigned)((cnt + 255) / 256), noff * PP, (unsigned)nsys);
  tr_kernel_work(TRK_UPDATE, 16.0 * nsys * PP * (double)(L + noff * cnt), 8.0 * nsys * PP * (double)L);
  { TrKTimer _kt(TRK_UPDATE, st); twist_fold_kernel<<<grid, 256, 0, st>>>(G, B, b_sys, b_cap, PP, L, o0, o1, noff, cnt, N, twN); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_apply_update(cplx* W, long long w_sys, const cplx* G, int rows, int P, long long o0,
                        long long o1, int noff, long long stride, long long cnt, long long nsys,
                        cudaStream_t st) {
  dim3 grid((unsigned)((cnt + 127) / 128), noff, (unsigned)nsys);
  tr_kernel_work(TRK_UPDATE, 16.0 * nsys * noff * (double)cnt * (2.0 * rows * P + P * P),
                 8.0 * nsys * noff * (double)cnt * rows * P * P);
  if (P == 5)
    { TrKTimer _kt(TRK_UPDATE, st); apply_update_kernel<5><<<grid, 128, 0, st>>>(W, w_sys, G, rows, o0, o1, noff, stride, cnt); }
  else
    { TrKTimer _kt(TRK_UPDATE, st); apply_update_kernel<7><<<grid, 128, 0, st>>>(W, w_sys, G, rows, o0, o1, noff, stride, cnt); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_pointwise_matmul(cplx* FA, const cplx* FB, int P, long long R, long long nsys,
                            cudaStream_t st) {
  tr_kernel_work(TRK_COMBINE, 48.0 * nsys * P * P * (double)R, 8.0 * nsys * P * P * P * (double)R);
  {
    TrKTimer _kt(TRK_COMBINE, st);
    if (P == 5) pointwise_matmul_kernel<5><<<g2(R, nsys, 128), 128, 0, st>>>(FA, FB, R);
    else pointwise_matmul_kernel<7><<<g2(R, nsys, 128), 128, 0, st>>>(FA, FB, R);
  }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_trim_normalize(const TrimArgs& a, long long nsys, cudaStream_t st) {
  tr_kernel_work(TRK_COMBINE, 16.0 * nsys * a.P * a.P * (double)(a.L + a.cap), 0.0);
  if (nsys >= 32) {  // enough systems to fill the GPU with one CTA each
    {
      TrKTimer _kt(TRK_COMBINE, st);
      if (a.P == 5) trim_fused_kernel<5><<<(unsigned)nsys, TF, 0, st>>>(a);
      else trim_fused_kernel<7><<<(unsigned)nsys, TF, 0, st>>>(a);
    }
    TR_CUDA_CHECK(cudaGetLastError());
    return 0;
  }
  TR_CUDA_CHECK(cudaMemsetAsync(a.red, 0, sizeof(unsigned long long) * (2 + a.P) * nsys, st));
  { TrKTimer _kt(TRK_COMBINE, st); trim1_kernel<<<g2(a.L, nsys), 256, 0, st>>>(a); }
  { TrKTimer _kt(TRK_COMBINE, st); trim2_kernel<<<g2(a.L, nsys), 256, 0, st>>>(a); }
  { TrKTimer _kt(TRK_COMBINE, st); trim3_kernel<<<g2(a.L, nsys), 256, 0, st>>>(a); }
  { TrKTimer _kt(TRK_COMBINE, st); trim4_kernel<<<g2(a.cap, nsys), 256, 0, st>>>(a); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}
