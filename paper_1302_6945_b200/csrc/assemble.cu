// Stage 1-2: circulant extension + roots-of-unity transform of the
// regularised normal system (ref: pkg/src/toepreg/extension.py:84-138,
// :196-273), plus the FFT Toeplitz matvecs behind T^H b and the normal
// operator (ref: toeplitz.py:79-111, solver.py:104-167).
#include "kernels.cuh"

namespace {

// Generator entry i of a block in generator form (top-right -> bottom-left).
TR_D cplx seq_gen(const SeqDesc& s, const cplx* g, long long i) {
  if (s.kind == SEQ_PLAIN) return g[i];
  if (s.kind == SEQ_ADJOINT) return cconj(g[s.len - 1 - i]);
  // SEQ_HERM: full generator of the Hermitian matrix with first column g
  long long n = (s.len + 1) / 2;
  if (i < n - 1) return cconj(g[n - 1 - i]);
  return g[i - (n - 1)];
}

__global__ void ext_seq_kernel(cplx* out, long long N, int nblk, SeqBatch sb, long long nsys) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int blk = blockIdx.y;
  long long sys = blockIdx.z;
  if (i >= N || sys >= nsys) return;
  const SeqDesc& s = sb.d[blk];
  cplx v = cmk(0.0, 0.0);
  const cplx* g = s.g + sys * s.bstride;
  if (s.kind == SEQ_RHS) {
    // ref extension.py:134-138: c[N - len:] = -rhs
    long long start = N - s.len;
    if (i >= start) v = cneg(g[i - start]);
  } else {
    long long k = N - s.len;  // extension count (ref extension.py:84-102)
    if (i >= k) v = seq_gen(s, g, i - k);
    else if (s.echo) v = seq_gen(s, g, (k - 1 - i) % s.len);
  }
  out[(sys * nblk + blk) * N + i] = v;
}

__global__ void emb_col_kernel(cplx* out, long long q, SeqBatch sb, int nblk, long long nsys) {
  // first column of the order-q circulant whose leading corner is the block
  // (ref toeplitz.py:79-90); rows/cols are those of the (possibly adjoint) block
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int blk = blockIdx.y;
  long long sys = blockIdx.z;
  if (i >= q || sys >= nsys) return;
  const SeqDesc& s = sb.d[blk];
  const cplx* g = s.g + sys * s.bstride;
  cplx v = cmk(0.0, 0.0);
  if (i < s.rows) v = seq_gen(s, g, s.cols - 1 + i);
  else if (s.cols > 1 && i >= q - (s.cols - 1)) v = seq_gen(s, g, i - (q - (s.cols - 1)));
  out[(sys * nblk + blk) * q + i] = v;
}

__global__ void assemble_weights_kernel(AsmArgs a) {
  long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long sys = blockIdx.y;
  if (k >= a.N) return;
  const long long N = a.N;
  const cplx* S = a.spec + sys * a.nblk * N;
  auto spec = [&](int b) { return S[b * N + k]; };
  auto npow = [&](long long e) { return __ldg(&a.twN[(k * (e % N)) % N]); };
  cplx w[3][7];
#pragma unroll
  for (int r = 0; r < 3; ++r)
#pragma unroll
    for (int i = 0; i < 7; ++i) w[r][i] = cmk(0.0, 0.0);
  const cplx one = cmk(1.0, 0.0);
  if (a.variant == VAR_L2) {
    double bsq = a.beta_sq[sys * a.beta_bstride];
    w[0][0] = cscale(npow(N - a.n), bsq);
    w[0][1] = spec(0);
    w[0][2] = one;
    w[0][4] = spec(2);
    w[1][0] = cneg(spec(1));
    w[1][1] = npow(N - a.m);
    w[1][3] = one;
  } else if (a.variant == VAR_GENERAL) {
    w[0][1] = spec(0);
    w[0][2] = spec(1);
    w[0][3] = one;
    w[0][6] = spec(2);
    w[1][0] = cneg(spec(3));
    w[1][1] = npow(N - a.m);
    w[1][4] = one;
    w[2][0] = cneg(spec(4));
    w[2][2] = npow(N - a.pl);
    w[2][5] = one;
  } else {  // gramian
    w[0][0] = spec(0);
    w[0][1] = spec(1);
    w[0][2] = one;
    w[0][4] = spec(2);
    w[1][0] = cneg(spec(3));
    w[1][1] = npow(N - a.pl);
    w[1][3] = one;
  }
  const int rows = a.rows, P = a.P;
  cplx* W = a.W + (sys * N + k) * rows * P;
  cplx* Wp = a.Wp ? a.Wp + (sys * N + k) * rows * P : nullptr;
  for (int r = 0; r < rows; ++r)
    for (int i = 0; i < P; ++i) {
      W[r * P + i] = w[r][i];
      if (Wp) Wp[r * P + i] = w[r][i];
    }
}

// out[sys][i] = a[sys][i] * b[sys][i] * scale   (batch stride 0 = shared)
__global__ void spec_mul_kernel(cplx* out, long long out_bs, const cplx* a, long long a_bs,
                                const cplx* b, long long b_bs, long long q, double scale,
                                int conj_b) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long sys = blockIdx.y;
  if (i >= q) return;
  cplx bv = b[sys * b_bs + i];
  if (conj_b) bv = cconj(bv);
  out[sys * out_bs + i] = cscale(cmul(a[sys * a_bs + i], bv), scale);
}

// buf[sys][i] = i < keep ? buf*scale : 0
__global__ void mask_scale_kernel(cplx* buf, long long bs, long long q, long long keep, double scale) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long sys = blockIdx.y;
  if (i >= q) return;
  cplx* p = buf + sys * bs;
  p[i] = i < keep ? cscale(p[i], scale) : cmk(0.0, 0.0);
}

// acc[sys][i] (+)= src[sys][i] * scale for i < n
__global__ void accum_kernel(cplx* acc, long long acc_bs, const cplx* src, long long src_bs,
                             long long n, double scale, int overwrite) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long sys = blockIdx.y;
  if (i >= n) return;
  cplx v = cscale(src[sys * src_bs + i], scale);
  cplx* p = acc + sys * acc_bs + i;
  *p = overwrite ? v : cadd(*p, v);
}

// r = y - (Ax + bsq * x); also writes r for the refinement
__global__ void residual_kernel(cplx* r, const cplx* ax, const cplx* x, const cplx* y,
                                long long n, const double* beta_sq, long long beta_bs,
                                int add_ridge) {
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long sys = blockIdx.y;
  if (i >= n) return;
  long long o = sys * n + i;
  cplx v = ax[o];
  if (add_ridge) v = cadd(v, cscale(x[o], beta_sq[sys * beta_bs]));
  r[o] = csub(y[o], v);
}

inline dim3 grid1(long long n, long long nsys, int threads = 256) {
  return dim3((unsigned)((n + threads - 1) / threads), (unsigned)nsys);
}

}  // namespace

int launch_ext_seq(cplx* out, long long N, const SeqBatch& sb, int nblk, long long nsys,
                   cudaStream_t st) {
  dim3 g((unsigned)((N + 255) / 256), nblk, (unsigned)nsys);
  { TrKTimer _kt(TRK_ASSEMBLE, st); ext_seq_kernel<<<g, 256, 0, st>>>(out, N, nblk, sb, nsys); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_emb_col(cplx* out, long long q, const SeqBatch& sb, int nfill, int nblk, long long nsys,
                   cudaStream_t st) {
  dim3 g((unsigned)((q + 255) / 256), nfill, (unsigned)nsys);
  { TrKTimer _kt(TRK_ASSEMBLE, st); emb_col_kernel<<<g, 256, 0, st>>>(out, q, sb, nblk, nsys); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_assemble(const AsmArgs& a, long long nsys, cudaStream_t st) {
  { TrKTimer _kt(TRK_ASSEMBLE, st); assemble_weights_kernel<<<grid1(a.N, nsys), 256, 0, st>>>(a); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_spec_mul(cplx* out, long long out_bs, const cplx* a, long long a_bs, const cplx* b,
                    long long b_bs, long long q, double scale, long long nsys, cudaStream_t st,
                    int conj_b) {
  { TrKTimer _kt(TRK_NORMAL, st); spec_mul_kernel<<<grid1(q, nsys), 256, 0, st>>>(out, out_bs, a, a_bs, b, b_bs, q, scale, conj_b); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_mask_scale(cplx* buf, long long bs, long long q, long long keep, double scale,
                      long long nsys, cudaStream_t st) {
  { TrKTimer _kt(TRK_NORMAL, st); mask_scale_kernel<<<grid1(q, nsys), 256, 0, st>>>(buf, bs, q, keep, scale); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_accum(cplx* acc, long long acc_bs, const cplx* src, long long src_bs, long long n,
                 double scale, int overwrite, long long nsys, cudaStream_t st) {
  { TrKTimer _kt(TRK_NORMAL, st); accum_kernel<<<grid1(n, nsys), 256, 0, st>>>(acc, acc_bs, src, src_bs, n, scale, overwrite); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_residual(cplx* r, const cplx* ax, const cplx* x, const cplx* y, long long n,
                    const double* beta_sq, long long beta_bs, int add_ridge, long long nsys,
                    cudaStream_t st) {
  { TrKTimer _kt(TRK_NORMAL, st); residual_kernel<<<grid1(n, nsys), 256, 0, st>>>(r, ax, x, y, n, beta_sq, beta_bs, add_ridge); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}
