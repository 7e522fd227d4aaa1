// Leaf serial sweep, one CTA per system, basis resident in registers.
//
// The reference absorbs a leaf's K conditions one at a time into a p x p
// polynomial basis (ref: pkg/src/toepreg/tanint.py:189-217): evaluate
// phi = w_t . B(sigma_t), pick the pivot column among the lowest-degree
// columns, col_i += mu_i col_j, col_j <- (z - sigma_t) col_j.  Here:
//
//  * Thread (row k, u) owns coefficients B[k][0..P)[u*D .. u*D+D) in
//    registers (TPR threads per row, rows warp-aligned).  Column updates are
//    row-local; the (z - sigma) shift needs one neighbour coefficient, taken
//    by warp shuffle or, across warps, from a double-buffered smem halo.
//  * phi_t is not re-evaluated from coefficients.  Every pending condition s
//    keeps its residual row r_s = w_s . B(sigma_s) (thread s owns it) and
//    updates it in O(P) per step: r_i += mu_i r_j, r_j *= (sigma_s - sigma_t).
//    phi_t = r_t is published through smem: one __syncthreads per step.
//  * Pivot rule, deferral, rescale cadence (every 8th listed condition,
//    skipped on deferred ones), normalisation, the self-residual check
//    (here by coset fold + DFT rather than powers) and the retry orders are
//    the reference's.
#include <stdlib.h>

#include "leaf.cuh"
#include "leaf_split.cuh"

#define TR_TRY_LEAF(expr) \
  do {                    \
    int _rc = (expr);     \
    if (_rc) return _rc;  \
  } while (0)

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr double RESCALE_TRIGGER = 1e8;  // ref tanint.py:41
constexpr int RESCALE_PERIOD = 8;        // ref tanint.py:42

TR_D long long leaf_node(const LeafArgs& a, int p) {
  if (a.noff == 1) return a.o0 + a.stride * (long long)p;
  return ((p & 1) ? a.o1 : a.o0) + a.stride * (long long)(p >> 1);
}

TR_D int leaf_perm(int i, int s, int rev, int count) {
  if (rev) i = count - 1 - i;
  return (int)(((unsigned)i * (unsigned)s) % (unsigned)count);
}

TR_D double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

template <int P, int D, int TPR>
struct Leaf {
  static constexpr int NT = P * TPR;
  static constexpr int NW = NT / 32;
};

// One absorption step for a compile-time pivot column J.
template <int P, int D, int J>
TR_D void step_body(cplx (&c)[D][P], cplx (&r)[P], const cplx (&mu)[P], cplx msig, cplx up,
                    bool do_basis, bool do_res, cplx dsig) {
  if (do_basis) {
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      cplx oj = c[d][J];
      cplx pv = (d > 0) ? c[d - 1][J] : up;
#pragma unroll
      for (int i = 0; i < P; ++i)
        if (i != J) c[d][i] = cfma(mu[i], oj, c[d][i]);
      c[d][J] = cfma(msig, oj, pv);
    }
  }
  if (do_res) {
    cplx rj = r[J];
#pragma unroll
    for (int i = 0; i < P; ++i)
      if (i != J) r[i] = cfma(mu[i], rj, r[i]);
    r[J] = cmul(rj, dsig);
  }
}

// Pivot rule of the reference (ref tanint.py:193-211): among the columns of
// lowest degree take the first with the largest |phi|; defer when it is below
// thr * max|phi|.  Compared on squared moduli; mu = -phi / phi_j.
template <int P>
TR_D void pivot_publish(const cplx (&phi)[P], const int (&cd)[P], double thr, cplx* mu_out,
                        int* j_out, int* small_out) {
  double a2[P], amax2 = 0.0;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    a2[i] = cabs2(phi[i]);
    amax2 = fmax(amax2, a2[i]);
  }
  int small = amax2 == 0.0;
  int j = 0;
  if (!small) {
    int dmin = cd[0];
#pragma unroll
    for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
    double bm = -1.0;
#pragma unroll
    for (int i = 0; i < P; ++i)
      if (cd[i] == dmin && a2[i] > bm) { bm = a2[i]; j = i; }
    small = bm < thr * thr * amax2;
  }
  if (!small) {
    cplx pj = cmk(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < P; ++i)
      if (i == j) pj = phi[i];
    const double inv2 = 1.0 / cabs2(pj);
    const cplx inv = cmk(pj.x * inv2, -pj.y * inv2);
#pragma unroll
    for (int i = 0; i < P; ++i) mu_out[i] = cneg(cmul(phi[i], inv));
  }
  *j_out = j;
  *small_out = small;
}

template <int P, int D>
TR_D cplx top_dyn(const cplx (&c)[D][P], int j) {
  cplx v = c[D - 1][0];
#pragma unroll
  for (int i = 1; i < P; ++i)
    if (j == i) v = c[D - 1][i];
  return v;
}

template <int P, int D, int TPR>
__global__ void __launch_bounds__(P * TPR, 1) leaf_kernel(LeafArgs a) {
  constexpr int NT = P * TPR;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  cplx* phib = reinterpret_cast<cplx*>(smem_raw);        // [2][P]
  cplx* halo = phib + 2 * P;                              // [2][NW][P]
  cplx* sigb = halo + 2 * NW * P;                         // [2] node of condition t
  cplx* gbuf = sigb + 2;                                  // [P*P][M]
  cplx* bvb = gbuf + P * P * a.M;                         // [P*P][M]
  double* red = reinterpret_cast<double*>(bvb + P * P * a.M);  // [NW][P]
  int2* dcur = reinterpret_cast<int2*>(red + NW * P);     // [K]
  int2* dbest = dcur + a.K;                               // [K]
  int* pubi = reinterpret_cast<int*>(dbest + a.K);        // [2] pivot, [2] deferral flag

  const int sys = blockIdx.x;
  if (a.only && a.only[sys] != -2) return;  // exact fallback for flagged systems only
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const int krow = tid / TPR, u = tid % TPR;
  const int rows = a.rows, K = a.K, count = a.count;
  const cplx* W = a.W + (long long)sys * a.w_sys;
  const long long rowstride = (long long)rows * P;  // per node

  // ---- scale = max |w_in| over the leaf's conditions ----
  double sc = 0.0;
  for (int e = tid; e < K * P; e += NT) {
    int pos = e / (rows * P), rem = e % (rows * P);
    long long node = leaf_node(a, pos);
    sc = fmax(sc, cabs(W[node * rowstride + rem]));
  }
  sc = warp_max(sc);
  if (lane == 0) red[warp] = sc;
  __syncthreads();
  double scale = red[0];
  for (int w = 1; w < NW; ++w) scale = fmax(scale, red[w]);
  __syncthreads();

  int cd0[P];
#pragma unroll
  for (int i = 0; i < P; ++i) cd0[i] = a.cd[sys * 8 + i];

  double best_res = 0.0, best_factor = 1.0;
  int best_cd[P];
  int best_ndef = 0, best_len = 1;
  int attempts = 0;

  for (int att = 0; att < a.nattempts; ++att) {
    ++attempts;
    const int ostr = a.ord_stride[att], orev = a.ord_reverse[att];
    // ---- init workspace: identity ----
    cplx c[D][P];
#pragma unroll
    for (int d = 0; d < D; ++d)
#pragma unroll
      for (int i = 0; i < P; ++i)
        c[d][i] = (u * D + d == 0 && i == krow && krow < P) ? cmk(1.0, 0.0) : cmk(0.0, 0.0);
    int cd[P];
#pragma unroll
    for (int i = 0; i < P; ++i) cd[i] = cd0[i];
    int len = 1, ndef = 0;
    double stat_scale = 1.0;
    // residual row of the condition this thread owns
    cplx r[P];
    cplx sig_s = cmk(0.0, 0.0);
    const bool owner = tid < K;
    if (owner) {
      int pos = leaf_perm(tid / rows, ostr, orev, count);
      int rr = tid % rows;
      long long node = leaf_node(a, pos);
      sig_s = __ldg(&a.twN[node]);
#pragma unroll
      for (int i = 0; i < P; ++i) r[i] = W[node * rowstride + rr * P + i];
    } else {
#pragma unroll
      for (int i = 0; i < P; ++i) r[i] = cmk(0.0, 0.0);
    }
    if (tid == 0) {
      pivot_publish<P>(r, cd, a.thr, phib, pubi, pubi + 2);
      sigb[0] = sig_s;
    }
    if (lane == 31) {
#pragma unroll
      for (int i = 0; i < P; ++i) halo[warp * P + i] = c[D - 1][i];
    }
    __syncthreads();

    for (int t = 0; t < K; ++t) {
      const int cur = t & 1, nxt = cur ^ 1;
      // pivot j, deferral flag and multipliers of condition t were computed
      // once by the thread owning condition t (ref tanint.py:193-211)
      const int j = pubi[cur];
      const bool small = pubi[2 + cur] != 0;
      const cplx sig_t = sigb[cur];
      if (small) {
        if (tid == 0) {
          const long long node_t = leaf_node(a, leaf_perm(t / rows, ostr, orev, count));
          dcur[ndef] = make_int2((int)node_t, t % rows);
        }
        ++ndef;
      } else {
        cplx mu[P];
#pragma unroll
        for (int i = 0; i < P; ++i) mu[i] = phib[cur * P + i];
        const cplx msig = cneg(sig_t);
        // neighbour's old top coefficient of column j
        cplx mytop = top_dyn<P, D>(c, j);
        cplx up;
        up.x = __shfl_up_sync(FULL, mytop.x, 1);
        up.y = __shfl_up_sync(FULL, mytop.y, 1);
        if (lane == 0) up = (u == 0) ? cmk(0.0, 0.0) : halo[(cur * NW + warp - 1) * P + j];
        const bool do_basis = (u * D <= len) && krow < P;
        const bool do_res = owner && tid > t;
        const cplx dsig = csub(sig_s, sig_t);
        switch (j) {
          case 0: step_body<P, D, 0>(c, r, mu, msig, up, do_basis, do_res, dsig); break;
          case 1: step_body<P, D, 1>(c, r, mu, msig, up, do_basis, do_res, dsig); break;
          case 2: step_body<P, D, 2>(c, r, mu, msig, up, do_basis, do_res, dsig); break;
          case 3: step_body<P, D, 3>(c, r, mu, msig, up, do_basis, do_res, dsig); break;
          case 4: step_body<P, D, 4>(c, r, mu, msig, up, do_basis, do_res, dsig); break;
          case 5: if (P > 5) step_body<P, D, (P > 5 ? 5 : 0)>(c, r, mu, msig, up, do_basis, do_res, dsig); break;
          case 6: if (P > 6) step_body<P, D, (P > 6 ? 6 : 0)>(c, r, mu, msig, up, do_basis, do_res, dsig); break;
        }
#pragma unroll
        for (int i = 0; i < P; ++i) cd[i] += (i == j);
        ++len;
        if ((t + 1) % RESCALE_PERIOD == 0) {
          // column max over the workspace; divide columns above the trigger
          double loc[P];
#pragma unroll
          for (int i = 0; i < P; ++i) {
            double m = 0.0;
#pragma unroll
            for (int d = 0; d < D; ++d) m = fmax(m, cabs2(c[d][i]));
            loc[i] = warp_max(m);
          }
          if (lane == 0) {
#pragma unroll
            for (int i = 0; i < P; ++i) red[warp * P + i] = loc[i];
          }
          __syncthreads();
#pragma unroll
          for (int i = 0; i < P; ++i) {
            double m = red[i];
            for (int w = 1; w < NW; ++w) m = fmax(m, red[w * P + i]);
            m = sqrt(m);
            if (m > RESCALE_TRIGGER) {
              double inv = 1.0 / m;
#pragma unroll
              for (int d = 0; d < D; ++d) c[d][i] = cscale(c[d][i], inv);
              r[i] = cscale(r[i], inv);
              stat_scale = fmax(stat_scale, m);
            }
          }
        }
      }
      // the owner of condition t+1 decides its pivot; publish the warp's
      // top coefficients for the next shift
      if (owner && tid == t + 1) {
        pivot_publish<P>(r, cd, a.thr, phib + nxt * P, pubi + nxt, pubi + 2 + nxt);
        sigb[nxt] = sig_s;
      }
      if (lane == 31) {
#pragma unroll
        for (int i = 0; i < P; ++i) halo[(nxt * NW + warp) * P + i] = c[D - 1][i];
      }
      __syncthreads();
    }

    // ---- normalize columns (ref tanint.py:179-183) ----
    double factor;
    {
      double loc[P];
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double m = 0.0;
#pragma unroll
        for (int d = 0; d < D; ++d) m = fmax(m, cabs2(c[d][i]));
        loc[i] = warp_max(m);
      }
      if (lane == 0) {
#pragma unroll
        for (int i = 0; i < P; ++i) red[warp * P + i] = loc[i];
      }
      __syncthreads();
      factor = 1.0;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double m = red[i];
        for (int w = 1; w < NW; ++w) m = fmax(m, red[w * P + i]);
        m = sqrt(m);
        double safe = m > 0.0 ? m : 1.0;
        double inv = 1.0 / safe;
#pragma unroll
        for (int d = 0; d < D; ++d) c[d][i] = cscale(c[d][i], inv);
        factor = fmax(factor, safe);
      }
      factor = fmax(factor, stat_scale);
      __syncthreads();
    }

    // ---- write the basis (attempt 0 straight to the output slot) ----
    cplx* dst = (att == 0 ? a.out : a.scratch) + (long long)sys * a.out_sys;
    if (krow < P) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        int l = u * D + d;
        if (l < a.cap) {
#pragma unroll
          for (int i = 0; i < P; ++i) dst[(long long)(krow * P + i) * a.cap + l] = c[d][i];
        }
      }
    }
    // slots may be wider than this leaf: clear the tail
    for (long long e = tid; e < (long long)P * P * (a.cap - TPR * D); e += NT) {
      long long ee = e / (a.cap - TPR * D), l = TPR * D + e % (a.cap - TPR * D);
      dst[ee * a.cap + l] = cmk(0.0, 0.0);
    }
    __syncthreads();

    // ---- self residual on the leaf's own conditions (ref tanint.py:262-270) ----
    double resm = 0.0;
    for (int cs = 0; cs < a.noff; ++cs) {
      const long long oc = cs ? a.o1 : a.o0;
      const int M = a.M;
      for (int e = tid; e < P * P * M; e += NT) {
        int ee = e / M, q = e % M;
        cplx acc = cmk(0.0, 0.0);
        for (int l = q; l < len; l += M) {
          cplx tw = __ldg(&a.twN[(oc * l) % a.N]);
          acc = cfma(dst[(long long)ee * a.cap + l], tw, acc);
        }
        gbuf[ee * M + q] = acc;
      }
      __syncthreads();
      for (int e = tid; e < P * P * M; e += NT) {
        int ee = e / M, tt = e % M;
        cplx acc = cmk(0.0, 0.0);
        for (int q = 0; q < M; ++q) {
          cplx tw = __ldg(&a.twN[(long long)((q * tt) % M) * a.stride]);
          acc = cfma(gbuf[ee * M + q], tw, acc);
        }
        bvb[ee * M + tt] = acc;
      }
      __syncthreads();
      for (int e = tid; e < M * rows * P; e += NT) {
        int tt = e / (rows * P), rem = e % (rows * P);
        int rr = rem / P, jj = rem % P;
        long long node = oc + a.stride * (long long)tt;
        const cplx* wrow = W + node * rowstride + rr * P;
        cplx acc = cmk(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < P; ++i) acc = cfma(wrow[i], bvb[(i * P + jj) * M + tt], acc);
        resm = fmax(resm, cabs(acc));
      }
      __syncthreads();
    }
    resm = warp_max(resm);
    if (lane == 0) red[warp] = resm;
    __syncthreads();
    double res = red[0];
    for (int w = 1; w < NW; ++w) res = fmax(res, red[w]);
    res = (scale == 0.0) ? 0.0 : res / scale;
    __syncthreads();

    if (att == 0 || res < best_res) {
      best_res = res;
      best_factor = factor;
      best_ndef = ndef;
      best_len = len;
#pragma unroll
      for (int i = 0; i < P; ++i) best_cd[i] = cd[i];
      if (tid == 0)
        for (int e = 0; e < ndef; ++e) dbest[e] = dcur[e];
      if (att > 0) {
        cplx* o = a.out + (long long)sys * a.out_sys;
        const cplx* s = a.scratch + (long long)sys * a.out_sys;
        for (long long e = tid; e < (long long)P * P * a.cap; e += NT) o[e] = s[e];
      }
      __syncthreads();
    }
    if (best_res <= a.check_tol) break;
  }

  // the parent's fused combine reads only len_eff coefficients: a nonzero
  // coefficient past them is reported as a truncation (-> CG rescue)
  if (a.len_eff > 0 && a.trim_over && best_len > a.len_eff) {
    const cplx* o = a.out + (long long)sys * a.out_sys;
    int nz = 0;
    for (long long e = tid; e < (long long)P * P * (best_len - a.len_eff); e += NT) {
      const long long ee = e / (best_len - a.len_eff), l = a.len_eff + e % (best_len - a.len_eff);
      const cplx c = o[ee * a.cap + l];
      nz |= (c.x != 0.0 || c.y != 0.0);
    }
    nz = __syncthreads_or(nz);
    if (nz && tid == 0) a.trim_over[sys] += 1;
  }
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < P; ++i) a.cd[sys * 8 + i] = best_cd[i];
    int base = a.dcount[sys];
    int room = a.dmax - base;
    int nput = best_ndef < room ? best_ndef : room;
    for (int e = 0; e < nput; ++e) a.defer[(long long)sys * a.dmax + base + e] = dbest[e];
    a.dcount[sys] = base + best_ndef;
    if (best_ndef > room) a.status[sys] = 5;
    a.max_scale[sys] = fmax(a.max_scale[sys], best_factor);
    if (attempts > 1) a.retried[sys] += 1;
    if (a.res_out) a.res_out[sys] = best_res;
    if (a.len_out) a.len_out[sys] = best_len;
  }
}

template <int P, int D, int TPR>
int launch_t(const LeafArgs& a, int nsys, cudaStream_t st) {
  constexpr int NT = P * TPR, NW = NT / 32;
  if (a.K + 1 > TPR * D || a.K > NT || a.cap < a.K + 1) {
    tr_set_error("leaf of %d conditions does not fit the P=%d kernel", a.K, P);
    return 2;
  }
  size_t smem = sizeof(cplx) * (2 * P + 2 * NW * P + 2 + 2 * (size_t)P * P * a.M) +
                sizeof(double) * NW * P + sizeof(int2) * 2 * (size_t)a.K + 4 * sizeof(int);
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(leaf_kernel<P, D, TPR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    set = true;
  }
  if (smem > 200 * 1024) {
    tr_set_error("leaf shared memory %zu exceeds the limit", smem);
    return 2;
  }
  { TrKTimer _kt(TRK_LEAF_EXACT, st); leaf_kernel<P, D, TPR><<<nsys, NT, smem, st>>>(a); }
  return 0;
}

}  // namespace

bool leaf_supported(int P, int K) {
  if (P == 5) return K + 1 <= 96 * 3;
  if (P == 7) return K + 1 <= 64 * 4;
  return false;
}

int leaf_launch(const LeafArgs& a_in, int nsys, cudaStream_t st, const SplitState* split, bool exact_pass) {
  if (nsys <= 0) return 0;
  LeafArgs a = a_in;
  if (split && leaf_fast_supported(a)) {
    TR_TRY_LEAF(leaf_fast_launch(a, *split, nsys, st));
    a.only = split->need;  // re-run leaves whose rescale speculation failed
    if (!exact_pass) return 0;  // (flagged in split->any_viol: the caller re-runs with the fallback)
  } else if (split && leaf_split_supported(a)) {
    TR_TRY_LEAF(leaf_split_launch(a, *split, nsys, st));
    a.only = split->need;
    if (!exact_pass) return 0;
  }
  int rc;
  if (a.P == 5) rc = launch_t<5, 3, 96>(a, nsys, st);
  else if (a.P == 7) rc = launch_t<7, 4, 64>(a, nsys, st);
  else {
    tr_set_error("unsupported basis dimension %d", a.P);
    return 2;
  }
  if (rc) return rc;
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}
