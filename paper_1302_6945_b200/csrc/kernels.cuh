// Kernel launch interfaces shared by the solver orchestration.
#pragma once
#include "common.cuh"

enum { VAR_GENERAL = 0, VAR_L2 = 1, VAR_GRAMIAN = 2 };
enum { SEQ_PLAIN = 0, SEQ_ADJOINT = 1, SEQ_HERM = 2, SEQ_RHS = 3 };

// One generator-form block (or an rhs vector) feeding the extension /
// circulant embedding kernels.
struct SeqDesc {
  const cplx* g;        // generator (or first column for SEQ_HERM, rhs for SEQ_RHS)
  long long bstride;    // per-system stride in complex elements (0 = shared)
  long long len;        // generator length (2n-1 for SEQ_HERM, vector length for SEQ_RHS)
  int kind;
  int echo;             // echo fill for the extension (ref extension.py:76-102)
  long long rows, cols; // block shape (for the circulant embedding)
};
struct SeqBatch {
  SeqDesc d[6];
};

struct AsmArgs {
  int variant, rows, P, nblk;
  long long N, n, m, pl;
  const cplx* spec;      // [sys][nblk][N] block spectra
  const double* beta_sq; // |beta|^2 per system
  long long beta_bstride;
  const cplx* twN;
  cplx* W;               // [sys][N][rows][P]
  cplx* Wp;              // pristine copy (may be null)
};

int launch_ext_seq(cplx* out, long long N, const SeqBatch& sb, int nblk, long long nsys, cudaStream_t st);
int launch_emb_col(cplx* out, long long q, const SeqBatch& sb, int nfill, int nblk, long long nsys,
                   cudaStream_t st);
int launch_assemble(const AsmArgs& a, long long nsys, cudaStream_t st);
int launch_spec_mul(cplx* out, long long out_bs, const cplx* a, long long a_bs, const cplx* b,
                    long long b_bs, long long q, double scale, long long nsys, cudaStream_t st,
                    int conj_b = 0);
int launch_mask_scale(cplx* buf, long long bs, long long q, long long keep, double scale,
                      long long nsys, cudaStream_t st);
int launch_accum(cplx* acc, long long acc_bs, const cplx* src, long long src_bs, long long n,
                 double scale, int overwrite, long long nsys, cudaStream_t st);
int launch_residual(cplx* r, const cplx* ax, const cplx* x, const cplx* y, long long n,
                    const double* beta_sq, long long beta_bs, int add_ridge, long long nsys,
                    cudaStream_t st);

// ---- tree (tree.cu) ----
// G[sys][c][e][q] = sum_{l = q mod cnt, l < L} B[sys][e][l] w_N^(o_c l)
int launch_twist_fold(cplx* G, const cplx* B, long long b_sys, long long b_cap, int PP, long long L,
                      long long o0, long long o1, int noff, long long cnt, long long N,
                      const cplx* twN, long long nsys, cudaStream_t st);
// W[sys][o_c + s t][r][:] <- W[..][r][:] . Bval(t)   with Bval from G (after the DFT)
int launch_apply_update(cplx* W, long long w_sys, const cplx* G, int rows, int P, long long o0,
                        long long o1, int noff, long long stride, long long cnt, long long nsys,
                        cudaStream_t st);
// wrapped product (transform length R = La + Lb - 2): F[e][0] -= R T_e, F[e][R] = R T_e with
// T = A[:, :, La-1] B[:, :, Lb-1]; F lines of stride Rs = R + 1
int launch_wrap_fix(cplx* F, long long Rs, long long R, const cplx* A, long long a_cap, long long La,
                    const cplx* B, long long b_cap, long long Lb, int P, long long nsys, cudaStream_t st);
// FA[sys][f] <- FA[sys][f] @ FB[sys][f]  (P x P per frequency f < R)
int launch_pointwise_matmul(cplx* FA, const cplx* FB, int P, long long R, long long nsys,
                            cudaStream_t st);
struct TrimArgs {
  const cplx* F;       // [sys][PP][Rs] unnormalised product (x R)
  long long R;         // transform length (the product's scale)
  long long Rs = 0;    // line stride of F (0: R)
  long long L;         // untrimmed product length (<= R)
  int P;
  double* prof;        // [sys][L] scratch
  unsigned long long* red;  // [sys][2 + P] : gmax, last, colmax[P]
  cplx* out;           // [sys][PP][cap]
  long long out_sys, cap, cap_node;
  double* max_scale;   // [sys]
  int* trim_over;      // [sys] count of truncated (beyond bound) products
  int debug = 0;       // TR_TRIM_DEBUG: print truncations (diagnostic)
};
int launch_trim_normalize(const TrimArgs& a, long long nsys, cudaStream_t st);

// Fused combine of two leaf bases (combine_small.cu)
struct CombineArgs {
  const cplx* A;        // left basis [sys][PP][a_cap], La valid coefficients
  long long a_sys, a_cap;
  int La;
  const cplx* B;        // right basis [sys][PP][b_cap], Lb valid coefficients
  long long b_sys, b_cap;
  int Lb;
  cplx* out;            // [sys][PP][cap]
  long long out_sys, cap, cap_node;
  const cplx* twR;      // exp(2 pi i k / R)
  double* max_scale;    // [sys]
  int* trim_over;       // [sys]
  int P, R;
};
// Transform length for a leaf pair of La, Lb coefficients (0: too large)
int combine_small_R(int P, long long La, long long Lb);
int launch_combine_small(const CombineArgs& a, long long nsys, cudaStream_t st);

// Fused coset update after a leaf (combine_small.cu)
struct UpdateArgs {
  const cplx* B;        // left leaf basis [sys][PP][b_cap], Lb valid coefficients
  long long b_sys, b_cap;
  int Lb;
  cplx* W;              // weights [sys][N][rows][P]
  long long w_sys, N;
  int rows, P;
  long long o0, o1, stride;
  int noff, cnt;        // cosets, nodes per coset
  const cplx* twN;
};
int launch_update_small(const UpdateArgs& a, long long nsys, cudaStream_t st);

// ---- finish (finish.cu) ----
struct CleanupArgs {
  cplx* B;             // root basis [sys][PP][cap] (normalized, len = Lroot bound)
  long long b_sys, cap;
  long long len0;      // current (bound) length of the root basis
  int P, rows;
  long long N;
  const cplx* Wp;      // pristine weights
  const cplx* twN;
  int2* defer;
  int* dcount;
  int dmax;
  int* cd;
  double thr;
  double* max_scale;
  int* status;
  int* blen;           // [sys] resulting length
  cplx* tmp;           // [sys][P][cap] scratch
};
int launch_cleanup(const CleanupArgs& a, long long nsys, cudaStream_t st);
struct ExtractArgs {
  const cplx* B;
  long long b_sys, cap;
  const int* blen;      // may be null -> cap
  int P;
  const int* cd;
  long long n;
  cplx* x;              // [sys][n]
  int* status;
};
int launch_extract(const ExtractArgs& a, long long nsys, cudaStream_t st);
// per-system ||v||_2 with a fixed reduction order (chunk partials, then sum)
int launch_norms(const cplx* v, long long n, long long nsys, double* partial, int nchunk,
                 double* out, cudaStream_t st);
int launch_add_inplace(cplx* x, const cplx* d, long long n, long long nsys, cudaStream_t st);

// ---- conjugate gradients (cg.cu) ----
// st[sys][4] = {rho, |rhs|, active, -}; it[sys] = iterations done
int launch_cg_init(cplx* X, cplx* R, cplx* D, const cplx* Y, long long n, double* st, int* it, long long nsys,
                   cudaStream_t s);
int launch_cg_update(cplx* X, cplx* R, cplx* D, const cplx* AD, const double* beta_sq, long long beta_bs,
                     int ridge, long long n, double tol, double* st, int* it, long long nsys, cudaStream_t s,
                     long long ad_ls = 0);
int launch_cg_active(const double* st, long long nsys, int* any, cudaStream_t s);
int launch_cg_warm(cplx* X, cplx* R, cplx* D, const cplx* AX, const cplx* Y, const double* beta_sq,
                   long long beta_bs, int ridge, long long n, double* st, int* it, long long nsys, int* status,
                   int* rescued, const int* trim_over, cudaStream_t s, double* XR = nullptr);
// real CG refinement (solver.cu): x from the real state; P / M factors of the half-length spectrum product
int launch_real_unpack(cplx* X, const double* XR, long long n, long long nsys, cudaStream_t s);
int launch_pm_spectra(cplx* out, long long out_bs, const cplx* E, long long e_bs, long long q, const cplx* twq,
                      long long lines, long long nsys, cudaStream_t s);

// ---- nonuniform Fourier sums (nufft.cu) ----
// adjoint: y[d] = sum_k c_k exp(sign 2 pi i f_k d), d < n; forward: y[k] = sum_j x_j exp(sign 2 pi i f_k j)
int launch_nudft_adjoint(const double* f, const cplx* c, long long K, long long n, int sign, cplx* y,
                         cudaStream_t st);
int launch_nudft_forward(const double* f, const cplx* x, long long K, long long n, int sign, cplx* y,
                         cudaStream_t st);
int launch_cg_check(double* st, const int* it, long long nsys, int cap, const int* rescued, cudaStream_t s);
int launch_cg_restore(cplx* X, const cplx* X0, const double* st, long long n, long long nsys, cudaStream_t s);
int launch_add_masked(cplx* X, const cplx* D, const double* st, long long n, long long nsys, cudaStream_t s);
int launch_refine_apply(cplx* X, const cplx* D, const int* status, const double* st, long long n, long long nsys,
                        cudaStream_t s);
