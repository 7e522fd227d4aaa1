// Conjugate gradients on the normal equations (ref: pkg/src/toepreg/solver.py
// :184-215 cg_solve), batched over systems.  The operator application is the
// FFT NormalOperator of solver.cu (normal_apply); the vector part of one
// iteration -- alpha = rho / Re<d, Ad>, x += alpha d, r -= alpha Ad,
// rho' = |r|^2, the stopping test, d = r + (rho'/rho) d -- is one kernel with
// one CTA per system (two block reductions), so an iteration costs the
// operator's transforms plus one launch and nothing syncs with the host.
#include <cooperative_groups.h>

#include "kernels.cuh"

namespace {

constexpr int CGT = 1024;

__device__ __forceinline__ double blk_sum(double v, double* sh) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) sh[warp] = v;
  __syncthreads();
  double s = 0.0;
  for (int w = 0; w < CGT / 32; ++w) s += sh[w];  // fixed order: deterministic
  return s;
}

__global__ void __launch_bounds__(CGT) cg_init_kernel(cplx* X, cplx* R, cplx* D, const cplx* Y, long long n,
                                                      double* st, int* it) {
  __shared__ double sh[CGT / 32];
  const long long sys = blockIdx.x;
  const cplx* y = Y + sys * n;
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += CGT) {
    const cplx v = y[i];
    X[sys * n + i] = cmk(0.0, 0.0);
    R[sys * n + i] = v;
    D[sys * n + i] = v;
    s += cabs2(v);
  }
  s = blk_sum(s, sh);
  if (threadIdx.x == 0) {
    st[sys * 4 + 0] = s;            // rho
    st[sys * 4 + 1] = sqrt(s);      // |rhs|
    st[sys * 4 + 2] = s > 0.0;      // active
    it[sys] = 0;
  }
}

__global__ void __launch_bounds__(CGT) cg_update_kernel(cplx* X, cplx* R, cplx* D, const cplx* AD,
                                                        long long ad_ls, const double* beta_sq, long long beta_bs,
                                                        int ridge, long long n, double tol, double* st, int* it) {
  __shared__ double sh[CGT / 32];
  const long long sys = blockIdx.x;
  if (st[sys * 4 + 2] != 1.0) return;
  cplx* x = X + sys * n;
  cplx* r = R + sys * n;
  cplx* d = D + sys * n;
  const cplx* ad = AD + sys * ad_ls;
  const double b2 = ridge ? beta_sq[sys * beta_bs] : 0.0;
  // Re <d, A d> (A d = normal operator + |beta|^2 d for the ridge variant)
  double s = 0.0;
  for (long long i = threadIdx.x; i < n; i += CGT) {
    const cplx dv = d[i], av = ad[i];
    s += dv.x * (av.x + b2 * dv.x) + dv.y * (av.y + b2 * dv.y);
  }
  const double dad = blk_sum(s, sh);
  const double rho = st[sys * 4 + 0];
  const double alpha = rho / dad;
  s = 0.0;
  for (long long i = threadIdx.x; i < n; i += CGT) {
    const cplx dv = d[i], av = ad[i];
    const cplx adv = cmk(av.x + b2 * dv.x, av.y + b2 * dv.y);
    x[i] = cmk(x[i].x + alpha * dv.x, x[i].y + alpha * dv.y);
    const cplx rv = cmk(r[i].x - alpha * adv.x, r[i].y - alpha * adv.y);
    r[i] = rv;
    s += cabs2(rv);
  }
  const double rho_next = blk_sum(s, sh);
  const bool stop = sqrt(rho_next) <= tol * st[sys * 4 + 1];
  if (!stop) {
    const double beta = rho_next / rho;
    for (long long i = threadIdx.x; i < n; i += CGT) {
      const cplx rv = r[i], dv = d[i];
      d[i] = cmk(rv.x + beta * dv.x, rv.y + beta * dv.y);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    it[sys] += 1;
    st[sys * 4 + 0] = rho_next;
    if (stop) st[sys * 4 + 2] = 0.0;
  }
}

// warm start from the direct solution x: r = y - A x, d = r; the target is
// a 1e-8 reduction of the recursive residual, enough for the correction on
// any system CG converges on (x error ~ cond(A) 1e-8 of the direct error).
// Rescue: a system whose direct solve failed (status 3: singular under FP64
// rounding where the reference's long-double products succeeded; or a basis
// product outgrew its planned length, trim_over > 0) or whose direct
// solution is no better than zero (|y - A x| >= |y|, or not finite)
// restarts from x = 0 instead; its CG is never abandoned for the direct
// refinement and stops at the iteration cap (rescued = 1).  A system with a
// zero right-hand side keeps status 3 (the operator itself is singular).
//
// XR != nullptr (real data, solver.cu real CG refinement): the CG state is kept
// as real vectors -- x in XR, r in R, d in D, each line n doubles (n / 2
// complex values: the layout the half-length transforms and cg_update read);
// imaginary parts (rounding noise of a real problem) are dropped.
__global__ void __launch_bounds__(CGT) cg_warm_kernel(cplx* X, cplx* R, cplx* D, const cplx* AX,
                                                      const cplx* Y, const double* beta_sq, long long beta_bs,
                                                      int ridge, long long n, double* st, int* it, int* status,
                                                      int* rescued, const int* trim_over, double* XR) {
  __shared__ double sh[CGT / 32];
  __shared__ int rescue_sh;
  const long long sys = blockIdx.x;
  const double b2 = ridge ? beta_sq[sys * beta_bs] : 0.0;
  double* Rr = reinterpret_cast<double*>(R);
  double* Dr = reinterpret_cast<double*>(D);
  double s = 0.0, sy = 0.0;
  for (long long i = threadIdx.x; i < n; i += CGT) {
    const long long o = sys * n + i;
    const cplx x = X[o], ax = AX[o], y = Y[o];
    const cplx r = cmk(y.x - (ax.x + b2 * x.x), y.y - (ax.y + b2 * x.y));
    if (XR) {
      XR[o] = x.x;
      Rr[o] = r.x;
      Dr[o] = r.x;
      s += r.x * r.x;
      sy += y.x * y.x;
    } else {
      R[o] = r;
      D[o] = r;
      s += cabs2(r);
      sy += cabs2(y);
    }
  }
  s = blk_sum(s, sh);
  sy = blk_sum(sy, sh);
  if (threadIdx.x == 0) rescue_sh = sy > 0.0 && (status[sys] == 3 || trim_over[sys] > 0 || !(s < sy));
  __syncthreads();
  const bool rescue = rescue_sh != 0;
  if (rescue) {
    for (long long i = threadIdx.x; i < n; i += CGT) {
      const long long o = sys * n + i;
      const cplx y = Y[o];
      if (XR) {
        XR[o] = 0.0;
        Rr[o] = y.x;
        Dr[o] = y.x;
      } else {
        X[o] = cmk(0.0, 0.0);
        R[o] = y;
        D[o] = y;
      }
    }
    s = sy;
  }
  if (threadIdx.x == 0) {
    // 1e-8 of the initial residual, but not below the FP64 floor of the
    // residual itself (~1e-15 |y|): iterations past it no longer improve x
    const double target = fmax(1e-8 * sqrt(s), 1e-15 * sqrt(sy));
    st[sys * 4 + 0] = s;
    st[sys * 4 + 1] = target;
    st[sys * 4 + 2] = sqrt(s) > target;
    st[sys * 4 + 3] = s;  // initial rho (progress estimate on the host)
    it[sys] = 0;
    rescued[sys] = rescue ? 1 : 0;
    if (rescue) status[sys] = 0;
  }
}

// st[2]: 1 iterating, 0 converged, 2 abandoned.  A system is abandoned when
// its own geometric rate so far projects past `cap` iterations (decided only
// from its own residual history at fixed check points: deterministic and
// independent of the batch it is solved in).
__global__ void cg_check_kernel(double* st, const int* it, long long nsys, int cap, const int* rescued) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (s >= nsys || st[s * 4 + 2] != 1.0) return;
  const int k = it[s];
  if (rescued[s]) {  // CG is this system's solver: run to the cap, keep its x
    if (k >= cap) st[s * 4 + 2] = 0.0;
    return;
  }
  const double r0 = sqrt(st[s * 4 + 3]), rk = sqrt(st[s * 4 + 0]), tgt = st[s * 4 + 1];
  const double rate = pow(rk / r0, 1.0 / k);
  const double need = rate < 1.0 ? log(tgt / rk) / log(rate) : 1e30;
  if (k >= cap || k + need > cap) st[s * 4 + 2] = 2.0;
}

// x = x0 for systems CG did not converge on (the direct refinement restarts
// from the direct solution)
__global__ void cg_restore_kernel(cplx* X, const cplx* X0, const double* st, long long n) {
  const long long sys = blockIdx.y;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n || st[sys * 4 + 2] == 0.0) return;
  X[sys * n + i] = X0[sys * n + i];
}

// x += d where the refinement solve succeeded (status 0) and, after CG, for
// systems CG did not converge on
__global__ void refine_apply_kernel(cplx* X, const cplx* D, const int* status, const double* st, long long n) {
  const long long sys = blockIdx.y;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n || status[sys] != 0 || (st && st[sys * 4 + 2] == 0.0)) return;
  const long long o = sys * n + i;
  X[o] = cadd(X[o], D[o]);
}

// x += d for systems CG did not converge on
__global__ void add_masked_kernel(cplx* X, const cplx* D, const double* st, long long n) {
  const long long sys = blockIdx.y;
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= n || st[sys * 4 + 2] == 0.0) return;
  const long long o = sys * n + i;
  X[o] = cadd(X[o], D[o]);
}

// The same iteration tail with a cluster of C CTAs per system (each owns a
// contiguous slice of the vectors; the two reductions combine the CTAs'
// partial sums through DSMEM in rank order: deterministic for a given n).
constexpr int CGC_T = 256;
template <int C>
__global__ void __launch_bounds__(CGC_T) cg_update_cl_kernel(cplx* X, cplx* R, cplx* D, const cplx* AD,
                                                             long long ad_ls, const double* beta_sq,
                                                             long long beta_bs, int ridge, long long n, double tol,
                                                             double* st, int* it) {
  namespace cg = cooperative_groups;
  __shared__ double wsum[CGC_T / 32];
  __shared__ double part[2];
  const long long sys = blockIdx.x / C;
  const int rank = C > 1 ? (int)cg::this_cluster().block_rank() : 0;
  const bool active = st[sys * 4 + 2] == 1.0;  // uniform over the cluster
  if (!active) return;
  const long long per = (n + C - 1) / C;
  const long long lo = rank * per, hi = min(n, lo + per);
  cplx* x = X + sys * n;
  cplx* r = R + sys * n;
  cplx* d = D + sys * n;
  const cplx* ad = AD + sys * ad_ls;
  const double b2 = ridge ? beta_sq[sys * beta_bs] : 0.0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  auto csum = [&](double v, int slot) -> double {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) wsum[warp] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < CGC_T / 32; ++w) t += wsum[w];
      part[slot] = t;
    }
    double tot;
    if constexpr (C > 1) {
      cg::cluster_group cl = cg::this_cluster();
      cl.sync();
      tot = 0.0;
      for (int q = 0; q < C; ++q) tot += cl.map_shared_rank(part, q)[slot];
    } else {
      __syncthreads();
      tot = part[slot];
    }
    return tot;
  };
  double s = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += CGC_T) {
    const cplx dv = d[i], av = ad[i];
    s += dv.x * (av.x + b2 * dv.x) + dv.y * (av.y + b2 * dv.y);
  }
  const double dad = csum(s, 0);
  const double rho = st[sys * 4 + 0];
  const double alpha = rho / dad;
  s = 0.0;
  for (long long i = lo + threadIdx.x; i < hi; i += CGC_T) {
    const cplx dv = d[i], av = ad[i];
    const cplx adv = cmk(av.x + b2 * dv.x, av.y + b2 * dv.y);
    x[i] = cmk(x[i].x + alpha * dv.x, x[i].y + alpha * dv.y);
    const cplx rv = cmk(r[i].x - alpha * adv.x, r[i].y - alpha * adv.y);
    r[i] = rv;
    s += cabs2(rv);
  }
  const double rho_next = csum(s, 1);
  const bool stop = sqrt(rho_next) <= tol * st[sys * 4 + 1];
  if (!stop) {
    const double beta = rho_next / rho;
    for (long long i = lo + threadIdx.x; i < hi; i += CGC_T) {
      const cplx rv = r[i], dv = d[i];
      d[i] = cmk(rv.x + beta * dv.x, rv.y + beta * dv.y);
    }
  }
  if constexpr (C > 1) cg::this_cluster().sync();  // all ranks read st / the partials before rank 0 writes
  else __syncthreads();
  if (rank == 0 && threadIdx.x == 0) {
    it[sys] += 1;
    st[sys * 4 + 0] = rho_next;
    if (stop) st[sys * 4 + 2] = 0.0;
  }
}

template <int C>
int launch_cg_cl(cplx* X, cplx* R, cplx* D, const cplx* AD, long long ad_ls, const double* beta_sq,
                 long long beta_bs, int ridge, long long n, double tol, double* st, int* it, long long nsys,
                 cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(C * nsys));
  cfg.blockDim = dim3(CGC_T);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = C > 1 ? 1 : 0;
  TrKTimer _kt(TRK_NORMAL, s);
  TR_CUDA_CHECK(cudaLaunchKernelEx(&cfg, cg_update_cl_kernel<C>, X, R, D, AD, ad_ls, beta_sq, beta_bs, ridge, n,
                                   tol, st, it));
  return 0;
}

__global__ void cg_active_kernel(const double* st, long long nsys, int* any) {
  long long s = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int a = (s < nsys && st[s * 4 + 2] == 1.0) ? 1 : 0;
  a = __syncthreads_or(a);
  if (threadIdx.x == 0 && a) atomicOr(any, 1);
}


// x (complex, zero imaginary part) from the real CG state
__global__ void real_unpack_kernel(cplx* X, const double* XR, long long total) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i < total) X[i] = cmk(XR[i], 0.0);
}

// Factors of the half-length spectrum product (ref solver.py:104-167 applies
// the blocks through full-length circulant embeddings).  A real sequence x of
// q values read as h = q / 2 complex ones z_j = x_2j + i x_2j+1 has the
// transform Z; with E the circulant spectrum (length q, forward sign -1) of a
// real block, the h-point inverse transform of
//   V_k = P_k Z_k + M_k conj(Z_(-k mod h)),
//   P_k = (E_k + E_(k+h)) - (E_k - E_(k+h)) sin(2 pi k / q),
//   M_k = i (E_k - E_(k+h)) cos(2 pi k / q)
// is the (real) circulant product E * x in the same interleaved layout.
// out: [line][2 (P, M)][h] for every input line [line][q]; blockIdx.z = system
// (strides out_bs / e_bs).
__global__ void pm_spectra_kernel(cplx* out, long long out_bs, const cplx* E, long long e_bs, long long q,
                                  const cplx* twq, long long lines) {
  const long long h = q / 2;
  const long long line = blockIdx.y;
  const long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (k >= h || line >= lines) return;
  out += blockIdx.z * out_bs;
  E += blockIdx.z * e_bs;
  const cplx e0 = E[line * q + k], e1 = E[line * q + k + h];
  const cplx w = twq[k];  // cos + i sin (2 pi k / q)
  const cplx S = cadd(e0, e1), Dm = csub(e0, e1);
  out[(line * 2 + 0) * h + k] = cmk(S.x - Dm.x * w.y, S.y - Dm.y * w.y);
  out[(line * 2 + 1) * h + k] = cmk(-Dm.y * w.x, Dm.x * w.x);
}
}  // namespace

int launch_cg_init(cplx* X, cplx* R, cplx* D, const cplx* Y, long long n, double* st, int* it, long long nsys,
                   cudaStream_t s) {
  { TrKTimer _kt(TRK_NORMAL, s); cg_init_kernel<<<(unsigned)nsys, CGT, 0, s>>>(X, R, D, Y, n, st, it); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_cg_update(cplx* X, cplx* R, cplx* D, const cplx* AD, const double* beta_sq, long long beta_bs,
                     int ridge, long long n, double tol, double* st, int* it, long long nsys, cudaStream_t s,
                     long long ad_ls) {
  // CTAs per system from n alone (the reduction order must not depend on the batch)
  const long long ls = ad_ls > 0 ? ad_ls : n;
  const long long c = n / 4096;
  int rc = 0;
  if (c >= 8) rc = launch_cg_cl<8>(X, R, D, AD, ls, beta_sq, beta_bs, ridge, n, tol, st, it, nsys, s);
  else if (c >= 4) rc = launch_cg_cl<4>(X, R, D, AD, ls, beta_sq, beta_bs, ridge, n, tol, st, it, nsys, s);
  else if (c >= 2) rc = launch_cg_cl<2>(X, R, D, AD, ls, beta_sq, beta_bs, ridge, n, tol, st, it, nsys, s);
  else {  // one 1024-thread CTA per system
    TrKTimer _kt(TRK_NORMAL, s);
    cg_update_kernel<<<(unsigned)nsys, CGT, 0, s>>>(X, R, D, AD, ls, beta_sq, beta_bs, ridge, n, tol, st, it);
  }
  if (rc) return rc;
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_cg_active(const double* st, long long nsys, int* any, cudaStream_t s) {
  TR_CUDA_CHECK(cudaMemsetAsync(any, 0, sizeof(int), s));
  { TrKTimer _kt(TRK_NORMAL, s); cg_active_kernel<<<(unsigned)((nsys + 255) / 256), 256, 0, s>>>(st, nsys, any); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_cg_warm(cplx* X, cplx* R, cplx* D, const cplx* AX, const cplx* Y, const double* beta_sq,
                   long long beta_bs, int ridge, long long n, double* st, int* it, long long nsys, int* status,
                   int* rescued, const int* trim_over, cudaStream_t s, double* XR) {
  {
    TrKTimer _kt(TRK_NORMAL, s);
    cg_warm_kernel<<<(unsigned)nsys, CGT, 0, s>>>(X, R, D, AX, Y, beta_sq, beta_bs, ridge, n, st, it, status,
                                                  rescued, trim_over, XR);
  }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_cg_check(double* st, const int* it, long long nsys, int cap, const int* rescued, cudaStream_t s) {
  {
    TrKTimer _kt(TRK_NORMAL, s);
    cg_check_kernel<<<(unsigned)((nsys + 127) / 128), 128, 0, s>>>(st, it, nsys, cap, rescued);
  }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_cg_restore(cplx* X, const cplx* X0, const double* st, long long n, long long nsys, cudaStream_t s) {
  dim3 g((unsigned)((n + 255) / 256), (unsigned)nsys);
  { TrKTimer _kt(TRK_NORMAL, s); cg_restore_kernel<<<g, 256, 0, s>>>(X, X0, st, n); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_add_masked(cplx* X, const cplx* D, const double* st, long long n, long long nsys, cudaStream_t s) {
  dim3 g((unsigned)((n + 255) / 256), (unsigned)nsys);
  { TrKTimer _kt(TRK_FINISH, s); add_masked_kernel<<<g, 256, 0, s>>>(X, D, st, n); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_refine_apply(cplx* X, const cplx* D, const int* status, const double* st, long long n, long long nsys,
                        cudaStream_t s) {
  dim3 g((unsigned)((n + 255) / 256), (unsigned)nsys);
  { TrKTimer _kt(TRK_FINISH, s); refine_apply_kernel<<<g, 256, 0, s>>>(X, D, status, st, n); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_real_unpack(cplx* X, const double* XR, long long n, long long nsys, cudaStream_t s) {
  const long long total = n * nsys;
  { TrKTimer _kt(TRK_NORMAL, s); real_unpack_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(X, XR, total); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int launch_pm_spectra(cplx* out, long long out_bs, const cplx* E, long long e_bs, long long q, const cplx* twq,
                      long long lines, long long nsys, cudaStream_t s) {
  dim3 g((unsigned)((q / 2 + 255) / 256), (unsigned)lines, (unsigned)nsys);
  { TrKTimer _kt(TRK_NORMAL, s); pm_spectra_kernel<<<g, 256, 0, s>>>(out, out_bs, E, e_bs, q, twq, lines); }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}
