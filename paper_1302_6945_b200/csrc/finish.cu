// Deferred-condition cleanup (ref: pkg/src/toepreg/tanint.py:438-454),
// solution extraction (ref: tanint.py:470-491) and fixed-order norms.
#include <math.h>

#include "kernels.cuh"

namespace {

constexpr int CT = 256;  // cleanup / extract block size
constexpr double GOLDEN = 0.6180339887498949;

__device__ double blk_max(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double m = sh[0];
  for (int w = 1; w < CT / 32; ++w) m = fmax(m, sh[w]);
  __syncthreads();
  return m;
}

__device__ int gcd_i(int a, int b) {
  while (b) { int t = a % b; a = b; b = t; }
  return a;
}

// One CTA per system; only systems with deferred points do work.
template <int P>
__global__ void cleanup_kernel(CleanupArgs a) {
  cplx* tmp = a.tmp;  // [sys][P][cap] column stash
  __shared__ double shd[CT / 32];
  __shared__ cplx shc[CT / 32][P];
  __shared__ int2 pts[512];
  const long long sys = blockIdx.x;
  const int tid = threadIdx.x;
  int nd = a.dcount[sys];
  if (a.blen) {
    if (tid == 0) a.blen[sys] = (int)a.len0;
  }
  if (nd == 0 || a.status[sys] != 0) return;
  if (nd > a.dmax || nd > 512) {
    if (tid == 0) a.status[sys] = 5;
    return;
  }
  // sort by (index, row) (insertion sort; nd is small), then stride order
  if (tid == 0) {
    const int2* src = a.defer + sys * a.dmax;
    for (int i = 0; i < nd; ++i) {
      int2 v = src[i];
      int k = i - 1;
      while (k >= 0 && (pts[k].x > v.x || (pts[k].x == v.x && pts[k].y > v.y))) {
        pts[k + 1] = pts[k];
        --k;
      }
      pts[k + 1] = v;
    }
  }
  __syncthreads();
  int s = 1;
  if (nd > 2) {
    s = (int)nearbyint(GOLDEN * nd);
    while (gcd_i(s, nd) != 1) ++s;
  }
  cplx* B = a.B + sys * a.b_sys;
  cplx* T = tmp + sys * (long long)P * a.cap;
  int cd[P];
  for (int i = 0; i < P; ++i) cd[i] = a.cd[sys * 8 + i];
  long long len = a.len0;
  double thr = fmin(1e-13, a.thr);
  double mscale = a.max_scale[sys];
  for (int t = 0; t < nd; ++t) {
    int2 pt = pts[(nd > 2) ? (int)(((long long)t * s) % nd) : t];
    long long node = pt.x;
    const cplx* w = a.Wp + ((sys * a.N + node) * a.rows + pt.y) * P;
    cplx wv[P];
    for (int i = 0; i < P; ++i) wv[i] = w[i];
    // phi_k = sum_l (sum_i w_i B[i][k][l]) sigma^l
    cplx acc[P];
    for (int k = 0; k < P; ++k) acc[k] = cmk(0.0, 0.0);
    for (long long l = tid; l < len; l += CT) {
      cplx z = __ldg(&a.twN[(node * l) % a.N]);
      for (int k = 0; k < P; ++k) {
        cplx v = cmk(0.0, 0.0);
        for (int i = 0; i < P; ++i) v = cfma(wv[i], B[(long long)(i * P + k) * a.cap + l], v);
        acc[k] = cfma(v, z, acc[k]);
      }
    }
    // fixed-order block reduction
    cplx phi[P];
    for (int k = 0; k < P; ++k) {
      cplx v = acc[k];
      for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_down_sync(0xffffffffu, v.x, o);
        v.y += __shfl_down_sync(0xffffffffu, v.y, o);
      }
      if ((tid & 31) == 0) shc[tid >> 5][k] = v;
    }
    __syncthreads();
    for (int k = 0; k < P; ++k) {
      cplx v = shc[0][k];
      for (int wi = 1; wi < CT / 32; ++wi) v = cadd(v, shc[wi][k]);
      phi[k] = v;
    }
    __syncthreads();
    double ab[P], amax = 0.0;
    for (int i = 0; i < P; ++i) { ab[i] = cabs(phi[i]); amax = fmax(amax, ab[i]); }
    bool small = amax == 0.0;
    int j = 0;
    if (!small) {
      int dmin = cd[0];
      for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
      double bm = -1.0;
      for (int i = 0; i < P; ++i)
        if (cd[i] == dmin && ab[i] > bm) { bm = ab[i]; j = i; }
      small = bm < thr * amax;
    }
    if (small) {  // genuinely singular (ref tanint.py:449-453 with defer=False)
      if (tid == 0) a.status[sys] = 3;
      return;
    }
    if (len + 1 > a.cap) {
      if (tid == 0) a.status[sys] = 5;
      return;
    }
    cplx mu[P];
    for (int i = 0; i < P; ++i) mu[i] = cdiv_np(cneg(phi[i]), phi[j]);
    const cplx sig = __ldg(&a.twN[node % a.N]);
    // stash column j, then update every coefficient
    for (long long e = tid; e < (long long)P * (len + 1); e += CT) {
      long long k = e / (len + 1), l = e % (len + 1);
      T[k * a.cap + l] = l < len ? B[(long long)(k * P + j) * a.cap + l] : cmk(0.0, 0.0);
    }
    __syncthreads();
    for (long long e = tid; e < (long long)P * (len + 1); e += CT) {
      long long k = e / (len + 1), l = e % (len + 1);
      cplx oj = T[k * a.cap + l];
      cplx pv = l > 0 ? T[k * a.cap + l - 1] : cmk(0.0, 0.0);
      for (int i = 0; i < P; ++i)
        if (i != j) {
          cplx* c = &B[(long long)(k * P + i) * a.cap + l];
          *c = cfma(mu[i], oj, *c);
        }
      B[(long long)(k * P + j) * a.cap + l] = cfma(cneg(sig), oj, pv);
    }
    __syncthreads();
    ++len;
    cd[j] += 1;
    if ((t + 1) % 8 == 0) {
      for (int i = 0; i < P; ++i) {
        double m = 0.0;
        for (long long e = tid; e < (long long)P * len; e += CT) {
          long long k = e / len, l = e % len;
          m = fmax(m, cabs(B[(long long)(k * P + i) * a.cap + l]));
        }
        m = blk_max(m, shd);
        if (m > 1e8) {
          for (long long e = tid; e < (long long)P * len; e += CT) {
            long long k = e / len, l = e % len;
            cplx* c = &B[(long long)(k * P + i) * a.cap + l];
            *c = cscale(*c, 1.0 / m);
          }
          mscale = fmax(mscale, m);
        }
        __syncthreads();
      }
    }
  }
  // normalize (ref tanint.py:454)
  for (int i = 0; i < P; ++i) {
    double m = 0.0;
    for (long long e = tid; e < (long long)P * len; e += CT) {
      long long k = e / len, l = e % len;
      m = fmax(m, cabs(B[(long long)(k * P + i) * a.cap + l]));
    }
    m = blk_max(m, shd);
    double safe = m > 0.0 ? m : 1.0;
    for (long long e = tid; e < (long long)P * len; e += CT) {
      long long k = e / len, l = e % len;
      cplx* c = &B[(long long)(k * P + i) * a.cap + l];
      *c = cscale(*c, 1.0 / safe);
    }
    __syncthreads();
  }
  if (tid == 0) {
    for (int i = 0; i < P; ++i) a.cd[sys * 8 + i] = cd[i];
    a.max_scale[sys] = mscale;
    if (a.blen) a.blen[sys] = (int)len;
  }
}

__global__ void extract_kernel(ExtractArgs a) {
  __shared__ double sh[CT / 32];
  const long long sys = blockIdx.x;
  const int P = a.P;
  const int* cd = a.cd + sys * 8;
  int zeros = 0, j = -1;
  for (int i = 0; i < P; ++i)
    if (cd[i] == 0) { ++zeros; if (j < 0) j = i; }
  cplx* x = a.x + sys * a.n;
  bool bad = (zeros != 1) || a.status[sys] != 0;
  long long len = a.blen ? a.blen[sys] : a.cap;
  const cplx* B = a.B + sys * a.b_sys;
  double cm = 0.0;
  if (!bad) {
    for (long long e = threadIdx.x; e < (long long)P * len; e += CT) {
      long long i = e / len, l = e % len;
      cm = fmax(cm, cabs(B[(long long)(i * P + j) * a.cap + l]));
    }
  }
  cm = blk_max(cm, sh);
  cplx cst = bad ? cmk(0.0, 0.0) : B[(long long)((P - 1) * P + j) * a.cap];
  if (!bad && cabs(cst) < 1e-12 * cm) bad = true;
  if (bad) {
    if (threadIdx.x == 0 && a.status[sys] == 0) a.status[sys] = 3;
    for (long long l = threadIdx.x; l < a.n; l += CT) x[l] = cmk(0.0, 0.0);
    return;
  }
  const cplx* col = B + (long long)j * a.cap;  // row 0, column j
  for (long long l = threadIdx.x; l < a.n; l += CT)
    x[l] = l < len ? cdiv_np(col[l], cst) : cmk(0.0, 0.0);
}

__global__ void norm_partial_kernel(const cplx* v, long long n, double* partial, int nchunk) {
  __shared__ double sh[256];
  long long sys = blockIdx.y;
  int c = blockIdx.x;
  long long per = (n + nchunk - 1) / nchunk;
  long long lo = c * per, hi = lo + per < n ? lo + per : n;
  double s = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += 256) s += cabs2(v[sys * n + i]);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[sys * nchunk + c] = sh[0];
}

__global__ void norm_final_kernel(const double* partial, int nchunk, double* out, long long nsys) {
  long long sys = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (sys >= nsys) return;
  double s = 0.0;
  for (int c = 0; c < nchunk; ++c) s += partial[sys * nchunk + c];
  out[sys] = sqrt(s);
}

__global__ void add_kernel(cplx* x, const cplx* d, long long total) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < total) x[i] = cadd(x[i], d[i]);
}

}  // namespace

int launch_cleanup(const CleanupArgs& a, long long nsys, cudaStream_t st) {
  {
    TrKTimer _kt(TRK_FINISH, st);
    if (a.P == 5) cleanup_kernel<5><<<(unsigned)nsys, CT, 0, st>>>(a);
    else cleanup_kernel<7><<<(unsigned)nsys, CT, 0, st>>>(a);
  }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_extract(const ExtractArgs& a, long long nsys, cudaStream_t st) {
  { TrKTimer _kt(TRK_FINISH, st); extract_kernel<<<(unsigned)nsys, CT, 0, st>>>(a); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_norms(const cplx* v, long long n, long long nsys, double* partial, int nchunk,
                 double* out, cudaStream_t st) {
  { TrKTimer _kt(TRK_NORMAL, st); norm_partial_kernel<<<dim3(nchunk, (unsigned)nsys), 256, 0, st>>>(v, n, partial, nchunk); }
  { TrKTimer _kt(TRK_NORMAL, st); norm_final_kernel<<<(unsigned)((nsys + 127) / 128), 128, 0, st>>>(partial, nchunk, out, nsys); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_add_inplace(cplx* x, const cplx* d, long long n, long long nsys, cudaStream_t st) {
  long long total = n * nsys;
  { TrKTimer _kt(TRK_FINISH, st); add_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(x, d, total); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}
