// Divide-and-conquer tree kernels (ref: pkg/src/toepreg/tanint.py:368-393):
//  * coset update: twist + fold of the left basis (ref fftpoly.py:64-89
//    grid_eval), the DFT (fft.cu), then w <- w . B(sigma) in place;
//  * combine: B_left B_right by FFT (fft.cu), P x P x P product per
//    frequency, trim at 1e-14 of the global max and column normalisation
//    (ref fftpoly.py:148-155, :215-249; tanint.py:379-385).
#include <cooperative_groups.h>
#include <stdlib.h>

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
  // the whole B(f) in registers (one load each), then row by row of A(f)
  cplx br[P * P];
#pragma unroll
  for (int e = 0; e < P * P; ++e) br[e] = b[(long long)e * R];
  cplx ar[P];
#pragma unroll
  for (int k = 0; k < P; ++k) ar[k] = a[(long long)k * R];
#pragma unroll
  for (int i = 0; i < P; ++i) {
    cplx an[P];
    if (i + 1 < P) {
#pragma unroll
      for (int k = 0; k < P; ++k) an[k] = a[(long long)((i + 1) * P + k) * R];  // prefetch the next row
    }
    cplx cr[P];
#pragma unroll
    for (int jj = 0; jj < P; ++jj) {
      cplx acc = cmk(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < P; ++k) acc = cfma(ar[k], br[k * P + jj], acc);
      cr[jj] = acc;
    }
#pragma unroll
    for (int jj = 0; jj < P; ++jj) a[(long long)(i * P + jj) * R] = cr[jj];
    if (i + 1 < P) {
#pragma unroll
      for (int k = 0; k < P; ++k) ar[k] = an[k];
    }
  }
}

// Trim + normalise with a cluster of C CTAs per system (C = 1: one CTA):
// every CTA owns a contiguous slice of the coefficient range, the per-system
// reductions (global max, last column above 1e-14 of it, column maxima) are
// combined through distributed shared memory.  One read of F yields the
// profile and the untrimmed column maxima; a column maximum above the trim
// threshold is attained inside the kept range, so it equals the trimmed one
// (the rare column entirely below the threshold is recomputed over l < lt).
constexpr int TC = 256;
template <int P, int C>
__global__ void __launch_bounds__(TC) trim_cl_kernel(TrimArgs a) {
  namespace cg = cooperative_groups;
  constexpr int PP = P * P;
  constexpr int NV = 2 + P;  // gmax, last, colmax[P]
  __shared__ double part[NV];
  __shared__ double wsh[TC / 32][NV];
  __shared__ double glob[NV];
  const int rank = C > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const long long sys = blockIdx.x / C;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long Rs = a.Rs > 0 ? a.Rs : a.R;
  const cplx* F = a.F + sys * PP * Rs;
  double* prof = a.prof + sys * a.L;
  const long long per = (a.L + C - 1) / C;
  const long long lo = rank * per, hi = min(a.L, lo + per);
  // block + cluster max of v[0..n) into glob (all threads see the result)
  auto reduce = [&](double* v, int n) {
    for (int k = 0; k < n; ++k) {
      double x = v[k];
      for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
      if (lane == 0) wsh[warp][k] = x;
    }
    __syncthreads();
    if (tid < n) {
      double x = 0.0;
      for (int w = 0; w < TC / 32; ++w) x = fmax(x, wsh[w][tid]);
      part[tid] = x;
    }
    if constexpr (C > 1) {
      cg::cluster_group cl = cg::this_cluster();
      cl.sync();
      if (tid < n) {
        double x = 0.0;
        for (int r = 0; r < C; ++r) x = fmax(x, cl.map_shared_rank(part, r)[tid]);
        glob[tid] = x;
      }
      cl.sync();  // partners done reading part
    } else {
      __syncthreads();
      if (tid < n) glob[tid] = part[tid];
    }
    __syncthreads();
  };
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  for (long long l = lo + tid; l < hi; l += TC) {
    double m = 0.0;
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        const double q = cabs2(F[(long long)(i * P + j) * Rs + l]);
        m = fmax(m, q);
        v[2 + j] = fmax(v[2 + j], q);
      }
    prof[l] = m;
    v[0] = fmax(v[0], m);
  }
  reduce(v, NV);
  const double gm = glob[0];
  const double thr = 1e-28 * gm;  // (1e-14)^2 on squared moduli
  double cm2[P];
#pragma unroll
  for (int j = 0; j < P; ++j) cm2[j] = glob[2 + j];
  double last = 0.0;
  for (long long l = lo + tid; l < hi; l += TC)
    if (prof[l] > thr) last = fmax(last, (double)(l + 1));
  reduce(&last, 1);
  long long lt = (long long)glob[0];
  if (lt < 1) lt = 1;
  // Coefficients past the planned length: FP64 product rounding (the
  // reference's long-double products keep such tails below its 1e-14 trim
  // threshold; FP64 ones reach ~1e-14 of the maximum) is dropped silently;
  // anything above 1e-10 of the maximum is structure the plan did not
  // provide for and is reported (trim_over -> status 6).
  double dropped = 0.0;
  if (lt > a.cap_node) {  // uniform across the cluster
    for (long long l = (lo > a.cap_node ? lo : a.cap_node) + tid; l < hi && l < lt; l += TC)
      dropped = fmax(dropped, prof[l]);
    reduce(&dropped, 1);
    dropped = glob[0];
    if (a.debug && tid == 0 && rank == 0)
      printf("[trim] sys %lld L %lld cap %lld lt %lld: largest dropped |F|/max %.3e\n", sys, a.L, a.cap_node, lt,
             sqrt(dropped / gm));
  }
  bool slow = false;
#pragma unroll
  for (int j = 0; j < P; ++j) slow |= !(cm2[j] > thr);
  if (slow) {  // uniform across the cluster: same glob values everywhere
    double w[P];
#pragma unroll
    for (int j = 0; j < P; ++j) w[j] = 0.0;
    for (long long l = lo + tid; l < hi && l < lt; l += TC)
#pragma unroll
      for (int j = 0; j < P; ++j)
#pragma unroll
        for (int i = 0; i < P; ++i) w[j] = fmax(w[j], cabs2(F[(long long)(i * P + j) * Rs + l]));
    reduce(w, P);
#pragma unroll
    for (int j = 0; j < P; ++j) cm2[j] = glob[j];
  }
  double cm[P];
#pragma unroll
  for (int j = 0; j < P; ++j) cm[j] = sqrt(cm2[j]);
  const long long lw = lt < a.cap_node ? lt : a.cap_node;
  cplx* o = a.out + sys * a.out_sys;
  const long long cper = (a.cap + C - 1) / C;
  const long long clo = rank * cper, chi = min(a.cap, clo + cper);
  for (long long l = clo + tid; l < chi; l += TC) {
#pragma unroll
    for (int i = 0; i < P; ++i)
#pragma unroll
      for (int j = 0; j < P; ++j) {
        cplx val = cmk(0.0, 0.0);
        if (l < lw) {
          const double safe = cm[j] > 0.0 ? cm[j] : 1.0;
          const cplx f = F[(long long)(i * P + j) * Rs + l];
          val = cmk(f.x / safe, f.y / safe);
        }
        o[(long long)(i * P + j) * a.cap + l] = val;
      }
  }
  if (rank == 0 && tid == 0) {
    double ms = 1.0;
#pragma unroll
    for (int j = 0; j < P; ++j) {
      const double c = cm[j] / (double)a.R;
      const double safe = c > 0.0 ? c : 1.0;
      ms = j == 0 ? safe : fmax(ms, safe);
    }
    a.max_scale[sys] = fmax(a.max_scale[sys], ms);
    if (lt > a.cap_node && dropped > 1e-20 * gm) a.trim_over[sys] += 1;
  }
}

template <int P, int C>
int launch_trim_cl(const TrimArgs& a, long long nsys, cudaStream_t st) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(C * nsys));
  cfg.blockDim = dim3(TC);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = C > 1 ? 1 : 0;
  TrKTimer _kt(TRK_COMBINE, st);
  TR_CUDA_CHECK(cudaLaunchKernelEx(&cfg, trim_cl_kernel<P, C>, a));
  return 0;
}

template <int P>
int dispatch_trim_cl(const TrimArgs& a, long long nsys, cudaStream_t st) {
  // CTAs per system: enough to cover the GPU (2 per SM), slices of >= 256
  // coefficients.  TR_TRIM_CTAS sets the per-SM figure; 4 / 8 / 16 measured no
  // better inside a c5 solve (324.2 / 324.7 / 323.4 ms vs 321.2 ms per step)
  // although the top-level trims alone run at only 1.9 TB/s with 2.
  static const long long per_sm = [] {
    const char* e = getenv("TR_TRIM_CTAS");
    return e ? atoll(e) : 2LL;
  }();
  long long want = (per_sm * 148 + nsys - 1) / nsys;
  long long by_len = (a.L + 255) / 256;
  long long c = want < by_len ? want : by_len;
  if (c >= 8) return launch_trim_cl<P, 8>(a, nsys, st);
  if (c >= 4) return launch_trim_cl<P, 4>(a, nsys, st);
  if (c >= 2) return launch_trim_cl<P, 2>(a, nsys, st);
  return launch_trim_cl<P, 1>(a, nsys, st);
}

inline dim3 g2(long long n, long long nsys, int th = 256) {
  return dim3((unsigned)((n + th - 1) / th), (unsigned)nsys);
}

}  // namespace

namespace {
template <int P>
__global__ void wrap_fix_kernel(cplx* F, long long Rs, long long R, const cplx* A, long long a_cap, long long La,
                                const cplx* B, long long b_cap, long long Lb) {
  const long long sys = blockIdx.x;
  const int e = threadIdx.x;
  if (e >= P * P) return;
  const int i = e / P, j = e - i * P;
  const cplx* a = A + sys * P * P * a_cap;
  const cplx* b = B + sys * P * P * b_cap;
  cplx t = cmk(0.0, 0.0);
#pragma unroll
  for (int k = 0; k < P; ++k) t = cfma(a[(i * P + k) * a_cap + La - 1], b[(k * P + j) * b_cap + Lb - 1], t);
  t = cscale(t, (double)R);  // the inverse transform is unnormalised
  cplx* f = F + (sys * P * P + e) * Rs;
  f[0] = csub(f[0], t);
  f[R] = t;
}
}  // namespace

int launch_wrap_fix(cplx* F, long long Rs, long long R, const cplx* A, long long a_cap, long long La,
                    const cplx* B, long long b_cap, long long Lb, int P, long long nsys, cudaStream_t st) {
  TrKTimer _kt(TRK_COMBINE, st);
  if (P == 5) wrap_fix_kernel<5><<<(unsigned)nsys, 32, 0, st>>>(F, Rs, R, A, a_cap, La, B, b_cap, Lb);
  else wrap_fix_kernel<7><<<(unsigned)nsys, 64, 0, st>>>(F, Rs, R, A, a_cap, La, B, b_cap, Lb);
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

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
  const int rc = a.P == 5 ? dispatch_trim_cl<5>(a, nsys, st) : dispatch_trim_cl<7>(a, nsys, st);
  if (rc) return rc;
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}
