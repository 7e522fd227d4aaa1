// Fused combine of two LEAF bases (the deepest tree level: half of all
// combines), one launch instead of six (forward FFTs of both operands, the
// P x P x P product per frequency, the inverse FFT, the wrapped-coefficient
// fix, trim + normalise).  ref: pkg/src/toepreg/tanint.py:379-385,
// fftpoly.py:148-155, :215-249.
//
// A leaf basis has P^2 polynomial entries of at most La (Lb) coefficients:
// the fused leaf kernel keeps entry degrees within its planned register
// blocks (32 DB coefficients) and hands any leaf that outgrows them to the
// exact kernel, which reports a longer result as a truncation.  So the
// product fits R = 2^k >= La + Lb - 1 <= 256 (P = 5) / 128 (P = 7)
// coefficients, and one cluster of P CTAs per system does the whole combine
// in shared memory: CTA i owns output row i, transforms A's row i (P lines)
// and all of B (P^2 lines), forms C_i(f) = sum_j A_ij(f) B_j.(f), transforms
// back, and the trim/normalise reductions (global maximum, last significant
// coefficient, column maxima) run across the cluster through distributed
// shared memory.
// DS variant (batches that would not fit the GPU in one wave otherwise): CTA i
// transforms only row i of B and the product reads the other rows from their
// CTAs through distributed shared memory -- 10 lines and 41 KB of shared
// memory per CTA at R = 256 instead of 30 lines and 123 KB, several CTAs per
// SM.  Same arithmetic per line and per product, so the results are bit for
// bit the same (a 128-system group: 97 -> ~75 us per launch; small groups are
// faster with the redundant transforms and one cluster barrier less).
#include <cooperative_groups.h>

#include "fft_smem.cuh"
#include "kernels.cuh"

namespace {

namespace cg = cooperative_groups;

struct Ident {
  TR_D cplx operator()(int, int, cplx x) const { return x; }
};
template <int LP>
struct StLine {  // natural-order output k of line q back in place
  cplx* S;
  TR_D void operator()(int q, int k, cplx v) const { S[q * LP + k] = v; }
};

template <int P, int R1, int R2, int NTH, bool DS>
__global__ void __launch_bounds__(NTH) combine_small_kernel(CombineArgs a) {
  constexpr int R = R1 * R2, NL = DS ? 2 * P : P + P * P, LP = R + 1, NV = 1 + P;
  extern __shared__ __align__(16) unsigned char smraw[];
  cplx* S = reinterpret_cast<cplx*>(smraw);  // [NL][LP]: element l of line q at S[q * LP + l]
  __shared__ double part[NV], glob[NV];
  __shared__ double wsh[NTH / 32][NV];
  cg::cluster_group cl = cg::this_cluster();
  const int i = (int)cl.block_rank();  // output row
  const long long sys = blockIdx.x / P;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;

  // ---- load A row i (lines 0..P-1) and all of B (lines P..), zero padded to
  // R: a warp per line, lanes along the coefficients (coalesced, conflict-free)
  const cplx* A = a.A + sys * a.a_sys + (long long)i * P * a.a_cap;
  const cplx* B = a.B + sys * a.b_sys + (DS ? (long long)i * P * a.b_cap : 0LL);
  constexpr int NWP = NTH / 32, LPW = (NL + NWP - 1) / NWP, EPL = R / 32;
#pragma unroll
  for (int u = 0; u < LPW; ++u) {
    const int q = warp + u * NWP;
    if (q < NL) {
      const cplx* src = q < P ? A + (long long)q * a.a_cap : B + (long long)(q - P) * a.b_cap;
      const int len = q < P ? a.La : a.Lb;
      cplx x[EPL];
#pragma unroll
      for (int t = 0; t < EPL; ++t) {
        const int l = lane + 32 * t;
        x[t] = l < len ? src[l] : cmk(0.0, 0.0);
      }
#pragma unroll
      for (int t = 0; t < EPL; ++t) S[q * LP + lane + 32 * t] = x[t];
    }
  }
  __syncthreads();
  // ---- forward transforms of all NL lines
  stage1<R1, R2, NL, 1, NTH, Ident, LP>(S, -1, a.twR, Ident());
  stage2<R1, R2, NL, 1, NTH, StLine<LP>, LP>(S, -1, StLine<LP>{S});
  __syncthreads();
  // ---- C_i(f) = sum_j A_ij(f) B_jk(f), into lines 0..P-1 (DS: row j of B
  // lives in CTA j, lines P..2P-1)
  const cplx* Brow[P];
  if constexpr (DS) {
    cl.sync();  // every row of B is transformed
#pragma unroll
    for (int j = 0; j < P; ++j) Brow[j] = cl.map_shared_rank(S, j) + P * LP;
  } else {
#pragma unroll
    for (int j = 0; j < P; ++j) Brow[j] = S + (P + j * P) * LP;
  }
  for (int f = tid; f < R; f += NTH) {
    cplx av[P];
#pragma unroll
    for (int j = 0; j < P; ++j) av[j] = S[j * LP + f];
    cplx cv[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      cplx acc = cmk(0.0, 0.0);
#pragma unroll
      for (int j = 0; j < P; ++j) acc = cfma(av[j], Brow[j][k * LP + f], acc);
      cv[k] = acc;
    }
#pragma unroll
    for (int k = 0; k < P; ++k) S[k * LP + f] = cv[k];
  }
  __syncthreads();
  // ---- inverse transform of the P product lines (unnormalised: x R)
  stage1<R1, R2, P, 1, NTH, Ident, LP>(S, +1, a.twR, Ident());
  stage2<R1, R2, P, 1, NTH, StLine<LP>, LP>(S, +1, StLine<LP>{S});
  __syncthreads();

  // block + cluster maximum of v[0..n) into glob (every thread sees it)
  auto reduce = [&](double* v, int n) {
    for (int k = 0; k < n; ++k) {
      double x = v[k];
      for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
      if (lane == 0) wsh[warp][k] = x;
    }
    __syncthreads();
    if (tid < n) {
      double x = 0.0;
      for (int w = 0; w < NTH / 32; ++w) x = fmax(x, wsh[w][tid]);
      part[tid] = x;
    }
    cl.sync();
    if (tid < n) {
      double x = 0.0;
      for (int r = 0; r < P; ++r) x = fmax(x, cl.map_shared_rank(part, r)[tid]);
      glob[tid] = x;
    }
    cl.sync();  // partners done reading part; glob visible to the block
  };
  const int L = a.La + a.Lb - 1;  // product length (<= R)
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  for (int l = tid; l < L; l += NTH) {
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const double q = cabs2(S[k * LP + l]);
      v[0] = fmax(v[0], q);
      v[1 + k] = fmax(v[1 + k], q);
    }
  }
  reduce(v, NV);
  const double gm = glob[0];
  const double thr = 1e-28 * gm;  // (1e-14)^2 on squared moduli (ref fftpoly.py:211)
  double cm2[P];
#pragma unroll
  for (int k = 0; k < P; ++k) cm2[k] = glob[1 + k];
  double last = 0.0;
  for (int l = tid; l < L; l += NTH) {
    double m = 0.0;
#pragma unroll
    for (int k = 0; k < P; ++k) m = fmax(m, cabs2(S[k * LP + l]));
    if (m > thr) last = fmax(last, (double)(l + 1));
  }
  reduce(&last, 1);
  long long lt = (long long)glob[0];
  if (lt < 1) lt = 1;
  bool slow = false;
#pragma unroll
  for (int k = 0; k < P; ++k) slow |= !(cm2[k] > thr);
  if (slow) {  // a column below the threshold everywhere: its maximum over l < lt
    double w[P];
#pragma unroll
    for (int k = 0; k < P; ++k) w[k] = 0.0;
    for (int l = tid; l < lt; l += NTH)
#pragma unroll
      for (int k = 0; k < P; ++k) w[k] = fmax(w[k], cabs2(S[k * LP + l]));
    reduce(w, P);
#pragma unroll
    for (int k = 0; k < P; ++k) cm2[k] = glob[k];
  }
  double dropped = 0.0;  // largest coefficient past the planned length (see trim_cl_kernel)
  if (lt > a.cap_node) {
    for (long long l = a.cap_node + tid; l < lt; l += NTH)
#pragma unroll
      for (int k = 0; k < P; ++k) dropped = fmax(dropped, cabs2(S[k * LP + l]));
    reduce(&dropped, 1);
    dropped = glob[0];
  }
  double cm[P];
#pragma unroll
  for (int k = 0; k < P; ++k) cm[k] = sqrt(cm2[k]);
  // ---- normalised, trimmed row i of the product into the output slot
  const long long lw = lt < a.cap_node ? lt : a.cap_node;
  cplx* o = a.out + sys * a.out_sys + (long long)i * P * a.cap;
  for (long long e = tid; e < (long long)P * a.cap; e += NTH) {
    const int k = (int)(e / a.cap);
    const long long l = e - (long long)k * a.cap;
    cplx val = cmk(0.0, 0.0);
    if (l < lw) {
      const double safe = cm[k] > 0.0 ? cm[k] : 1.0;
      const cplx f = S[k * LP + l];
      val = cmk(f.x / safe, f.y / safe);
    }
    o[e] = val;
  }
  if (i == 0 && tid == 0) {
    double ms = 1.0;
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const double c = cm[k] / (double)R;
      const double safe = c > 0.0 ? c : 1.0;
      ms = k == 0 ? safe : fmax(ms, safe);
    }
    a.max_scale[sys] = fmax(a.max_scale[sys], ms);
    if (lt > a.cap_node && dropped > 1e-20 * gm) a.trim_over[sys] += 1;
  }
}

#ifndef TR_CS_NTH
#define TR_CS_NTH 512  // threads per CTA of the redundant variant (30-56 lines per CTA)
#endif
template <int P, int R1, int R2, bool DS = false>
int launch_cs(const CombineArgs& a, long long nsys, cudaStream_t st) {
  constexpr int NTH = DS ? 256 : TR_CS_NTH, R = R1 * R2, NL = DS ? 2 * P : P + P * P, LP = R + 1;
  if constexpr (!DS) {
    // more CTAs than one wave of the redundant variant (one CTA per SM at R >= 128)
    if (P * nsys > 296) return launch_cs<P, R1, R2, true>(a, nsys, st);
  }
  const size_t smem = sizeof(cplx) * (size_t)NL * LP;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(combine_small_kernel<P, R1, R2, NTH, DS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    set = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(P * nsys));
  cfg.blockDim = dim3(NTH);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  TrKTimer _kt(TRK_COMBINE, st);
  TR_CUDA_CHECK(cudaLaunchKernelEx(&cfg, combine_small_kernel<P, R1, R2, NTH, DS>, a));
  return 0;
}

}  // namespace

int combine_small_R(int P, long long La, long long Lb) {
  long long r = 1;
  while (r < La + Lb - 1) r <<= 1;
  if (r < 32) r = 32;  // the loader puts 32 coefficients per lane sweep
  const long long rmax = P == 5 ? 256 : (P == 7 ? 128 : 0);
  return r <= rmax ? (int)r : 0;
}

int launch_combine_small(const CombineArgs& a, long long nsys, cudaStream_t st) {
  tr_kernel_work(TRK_COMBINE, 16.0 * nsys * a.P * a.P * (double)(a.La + a.Lb + a.cap_node),
                 nsys * (15.0 * a.P * a.P * a.R * std::log2((double)a.R) + 8.0 * a.P * a.P * a.P * a.R));
  int rc = -1;
  if (a.P == 5) {
    switch (a.R) {
      case 32: rc = launch_cs<5, 8, 4>(a, nsys, st); break;
      case 64: rc = launch_cs<5, 8, 8>(a, nsys, st); break;
      case 128: rc = launch_cs<5, 16, 8>(a, nsys, st); break;
      case 256: rc = launch_cs<5, 16, 16>(a, nsys, st); break;
      default: break;
    }
  } else if (a.P == 7) {
    switch (a.R) {
      case 32: rc = launch_cs<7, 8, 4>(a, nsys, st); break;
      case 64: rc = launch_cs<7, 8, 8>(a, nsys, st); break;
      case 128: rc = launch_cs<7, 16, 8>(a, nsys, st); break;
      default: break;
    }
  }
  if (rc < 0) {
    tr_set_error("combine_small: unsupported shape (P=%d, R=%d)", a.P, a.R);
    return 2;
  }
  if (rc) return rc;
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

// ------------------------------------------------------------------------
// Fused coset update after a LEAF (ref tanint.py:387-393 _update_weights,
// fftpoly.py:64-89 grid_eval): the right sibling's weights are multiplied by
// the left leaf's basis evaluated at the sibling's nodes, one launch instead
// of twist/fold + FFT + apply.  One CTA per (system, coset):
//   G[e][q] = sum_{l = q mod c} B_e[l] w^(o l)          (twist + fold)
//   V[e][k] = sum_q G[e][q] w_c^(q k)                    (c-point DFT, c <= 128)
//   w[r][node_k][:] <- w[r][node_k][:] V(sigma_k)        (apply)
namespace {

#ifndef TR_UPD_NTH
#define TR_UPD_NTH 1024  // threads per CTA: the phases are short per-entry loops, latency-bound at 256
#endif
template <int P>
__global__ void __launch_bounds__(TR_UPD_NTH) update_small_kernel(UpdateArgs a) {
  constexpr int PP = P * P, NTH = TR_UPD_NTH;
  extern __shared__ __align__(16) unsigned char smraw[];
  const int c = a.cnt;
  cplx* G = reinterpret_cast<cplx*>(smraw);  // [PP][c]
  cplx* V = G + PP * c;                      // [PP][c]
  cplx* Wc = V + PP * c;                     // [c]: w^(s t)
  const int cs = blockIdx.x;
  const long long sys = blockIdx.y;
  const long long o = cs ? a.o1 : a.o0;
  const cplx* B = a.B + sys * a.b_sys;
  for (int t = threadIdx.x; t < c; t += NTH) Wc[t] = __ldg(&a.twN[(long long)t * a.stride]);
  // twist + fold
  for (int e = threadIdx.x; e < PP * c; e += NTH) {
    const int ee = e / c, q = e - ee * c;
    const cplx* src = B + (long long)ee * a.b_cap;
    cplx acc = cmk(0.0, 0.0);
    long long idx = (o * q) % a.N;
    const long long step = (o * c) % a.N;
    for (int l = q; l < a.Lb; l += c) {
      acc = cfma(src[l], __ldg(&a.twN[idx]), acc);
      idx += step;
      if (idx >= a.N) idx -= a.N;
    }
    G[e] = acc;
  }
  __syncthreads();
  // c-point DFT (sign +1: values at sigma_k = w^(o + s k)).  c = c1 c2 runs as
  // two passes of c1- and c2-term sums (q = c2 q1 + q2, k = k1 + c1 k2:
  // w_c^(q k) = w_c1^(q1 k1) w_c^(q2 k1) w_c2^(q2 k2)), c (c1 + c2) instead of
  // c^2 complex FMAs per entry; the direct sums (c1 = 1) for small or prime c.
  int c1 = 1;
  if (c > 12)
    for (int d = 2; d * d <= c; ++d)
      if (c % d == 0) c1 = d;
  const int c2 = c / c1;
  if (c1 == 1) {
    for (int e = threadIdx.x; e < PP * c; e += NTH) {
      const int ee = e / c, k = e - ee * c;
      const cplx* g = G + ee * c;
      cplx acc = cmk(0.0, 0.0);
      int t = 0;
      for (int q = 0; q < c; ++q) {
        acc = cfma(g[q], Wc[t], acc);
        t += k;
        if (t >= c) t -= c;
      }
      V[e] = acc;
    }
    __syncthreads();
  } else {
    // pass 1: H[q2][k1] = w_c^(q2 k1) sum_q1 G[c2 q1 + q2] w_c1^(q1 k1), into V
    for (int e = threadIdx.x; e < PP * c; e += NTH) {
      const int ee = e / c, r = e - ee * c;
      const int q2 = r / c1, k1 = r - q2 * c1;
      const cplx* g = G + ee * c + q2;
      cplx acc = cmk(0.0, 0.0);
      int t = 0;  // (q1 k1 mod c1) c2
      const int st = k1 * c2;
      for (int q1 = 0; q1 < c1; ++q1) {
        acc = cfma(g[c2 * q1], Wc[t], acc);
        t += st;
        if (t >= c) t -= c;
      }
      V[ee * c + r] = cmul(acc, Wc[(q2 * k1) % c]);
    }
    __syncthreads();
    // pass 2: V[k1 + c1 k2] = sum_q2 H[q2][k1] w_c2^(q2 k2), back into G
    for (int e = threadIdx.x; e < PP * c; e += NTH) {
      const int ee = e / c, k = e - ee * c;
      const int k2 = k / c1, k1 = k - k2 * c1;
      const cplx* h = V + ee * c + k1;
      cplx acc = cmk(0.0, 0.0);
      int t = 0;  // (q2 k2 mod c2) c1
      const int st = k2 * c1;
      for (int q2 = 0; q2 < c2; ++q2) {
        acc = cfma(h[q2 * c1], Wc[t], acc);
        t += st;
        if (t >= c) t -= c;
      }
      G[e] = acc;
    }
    __syncthreads();
    V = G;  // the apply below reads the values from here
  }
  // apply to the sibling's weights at its nodes
  cplx* W = a.W + sys * a.w_sys;
  for (int e = threadIdx.x; e < c * a.rows; e += NTH) {
    const int k = e / a.rows, r = e - k * a.rows;
    cplx* w = W + (o + a.stride * (long long)k) * a.rows * P + r * P;
    cplx old[P];
#pragma unroll
    for (int i = 0; i < P; ++i) old[i] = w[i];
#pragma unroll
    for (int j = 0; j < P; ++j) {
      cplx acc = cmk(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < P; ++i) acc = cfma(old[i], V[(i * P + j) * c + k], acc);
      w[j] = acc;
    }
  }
}

}  // namespace

int launch_update_small(const UpdateArgs& a, long long nsys, cudaStream_t st) {
  const size_t smem = sizeof(cplx) * ((size_t)2 * a.P * a.P * a.cnt + a.cnt);
  if (a.cnt > 128 || smem > 200 * 1024) {
    tr_set_error("update_small: coset of %d nodes too large", a.cnt);
    return 2;
  }
  tr_kernel_work(TRK_UPDATE, 16.0 * nsys * (a.P * a.P * (double)a.Lb + 2.0 * a.noff * a.cnt * a.rows * a.P),
                 8.0 * nsys * a.noff * a.P * a.P * ((double)a.Lb + (double)a.cnt * a.cnt + a.cnt * a.rows * a.P));
  dim3 grid((unsigned)a.noff, (unsigned)nsys);
  TrKTimer _kt(TRK_UPDATE, st);
  if (a.P == 5) {
    static bool set5 = false;
    if (!set5) {
      cudaFuncSetAttribute(update_small_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      set5 = true;
    }
    update_small_kernel<5><<<grid, TR_UPD_NTH, smem, st>>>(a);
  } else {
    static bool set7 = false;
    if (!set7) {
      cudaFuncSetAttribute(update_small_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      set7 = true;
    }
    update_small_kernel<7><<<grid, TR_UPD_NTH, smem, st>>>(a);
  }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}
