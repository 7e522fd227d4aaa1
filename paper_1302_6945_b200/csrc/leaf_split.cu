// Split leaf sweep: pivot chain -> basis replay -> self-check, per attempt.
//
// The reference absorbs a leaf's K conditions one at a time (ref:
// pkg/src/toepreg/tanint.py:189-217 _serial_core).  The decisions it takes
// (pivot column, deferral, mu) depend on the basis only through the residual
// rows r_s = w_s . B(sigma_s), which obey r_i += mu_i r_j, r_j *= (sigma_s -
// sigma_t) at every absorbed step.  So one attempt splits into:
//
//   A  leaf_pivot_relay_kernel  the sequential chain on residual rows only
//                          (warp relay, no barriers), writing the per-step
//                          log (pivot j_t or -1, mu_t) to HBM;
//   B  leaf_build_row_kernel    replays the log on one row of the P x P x (K+1)
//                          coefficient cube per CTA (no decisions left);
//   C  leaf_check_kernel   the reference's self-residual check (coset fold +
//                          DFT), best-attempt bookkeeping and the decision to
//                          retry with the next absorption order (ref :395-434).
//
// The reference's mid-sweep rescale (columns above 1e8, every 8th listed
// condition, ref :214-217) changes later decisions, so A assumes it does not
// fire and B verifies that no coefficient ever exceeded the trigger at a
// check point; a leaf that violates it is re-run by the exact coupled kernel
// (leaf.cu).  Attempts are rounds: systems that passed exit immediately.
#include "leaf.cuh"
#include "leaf_split.cuh"

#include <stdlib.h>


namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr double RESCALE_TRIGGER = 1e8;
constexpr int RESCALE_PERIOD = 8;

TR_D long long node_of(const LeafArgs& a, int p) {
  if (a.noff == 1) return a.o0 + a.stride * (long long)p;
  return ((p & 1) ? a.o1 : a.o0) + a.stride * (long long)(p >> 1);
}
TR_D int perm_of(int i, int s, int rev, int count) {
  if (rev) i = count - 1 - i;
  return (int)(((unsigned)i * (unsigned)s) % (unsigned)count);
}
TR_D long long cond_node(const LeafArgs& a, int s, int att) {
  return node_of(a, perm_of(s / a.rows, a.ord_stride[att], a.ord_reverse[att], a.count));
}
TR_D double wmax(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL, v, o));
  return v;
}

// ref tanint.py:193-211 on squared moduli; returns pivot or -1 (deferred)
template <int P>
TR_D int decide(const cplx (&phi)[P], const int (&cd)[P], double thr, cplx* mu_out) {
  double a2[P], amax2 = 0.0;
#pragma unroll
  for (int i = 0; i < P; ++i) {
    a2[i] = cabs2(phi[i]);
    amax2 = fmax(amax2, a2[i]);
  }
  if (amax2 == 0.0) return -1;
  int dmin = cd[0];
#pragma unroll
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
  double bm = -1.0;
  int j = 0;
  cplx pj = phi[0];
#pragma unroll
  for (int i = 0; i < P; ++i)
    if (cd[i] == dmin && a2[i] > bm) { bm = a2[i]; j = i; pj = phi[i]; }
  if (bm < thr * thr * amax2) return -1;
  const double inv2 = 1.0 / cabs2(pj);
  const cplx inv = cmk(pj.x * inv2, -pj.y * inv2);
#pragma unroll
  for (int i = 0; i < P; ++i) mu_out[i] = i == j ? cmk(0.0, 0.0) : cneg(cmul(phi[i], inv));
  return j;
}

// 1/x to ~1 ulp: MUFU reciprocal estimate + two Newton steps (DDIV costs ~80
// cycles of latency on the chain, this ~50)
TR_D double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}

// The same rule as decide() with a short dependency chain (it sits on the
// leaf's critical path once per condition): squared moduli, reciprocals of
// every candidate computed in parallel, max / first-argmax by trees.
template <int P>
TR_D int decide_fast(const cplx (&phi)[P], const int (&cd)[P], double thr, cplx* mu_out) {
  double a2[P], inv2[P], key[P];
#pragma unroll
  for (int i = 0; i < P; ++i) a2[i] = cabs2(phi[i]);
#pragma unroll
  for (int i = 0; i < P; ++i) inv2[i] = rcp_nr(a2[i]);
  int dmin = cd[0];
#pragma unroll
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
#pragma unroll
  for (int i = 0; i < P; ++i) key[i] = cd[i] == dmin ? a2[i] : -1.0;
  // tree: (value, index) with ties to the lower index
  double v[P];
  int ix[P];
#pragma unroll
  for (int i = 0; i < P; ++i) { v[i] = key[i]; ix[i] = i; }
  double am[P];
#pragma unroll
  for (int i = 0; i < P; ++i) am[i] = a2[i];
#pragma unroll
  for (int w = 1; w < P; w *= 2) {
#pragma unroll
    for (int i = 0; i + w < P; i += 2 * w) {
      const bool take = v[i + w] > v[i];
      ix[i] = take ? ix[i + w] : ix[i];
      v[i] = take ? v[i + w] : v[i];
      am[i] = fmax(am[i], am[i + w]);
    }
  }
  const int j = ix[0];
  const double bm = v[0], amax2 = am[0];
  if (amax2 == 0.0 || bm < thr * thr * amax2) return -1;
  cplx pj = phi[0];
  double ij = inv2[0];
#pragma unroll
  for (int i = 1; i < P; ++i) {
    pj = (j == i) ? phi[i] : pj;
    ij = (j == i) ? inv2[i] : ij;
  }
  const cplx inv = cmk(pj.x * ij, -pj.y * ij);
#pragma unroll
  for (int i = 0; i < P; ++i) mu_out[i] = i == j ? cmk(0.0, 0.0) : cneg(cmul(phi[i], inv));
  return j;
}

// Branch-free column selection: a data-dependent switch costs ~200 cycles on
// B200 (indirect branch), a select chain a few ALU ops.
template <int P>
TR_D cplx sel(const cplx (&v)[P], int j) {
  cplx r = v[0];
#pragma unroll
  for (int i = 1; i < P; ++i) r = (j == i) ? v[i] : r;
  return r;
}

// r <- r F_t(sigma_s) with mu_j == 0: r_i += mu_i r_j, r_j <- r_j (sigma_s - sigma_t)
template <int P>
TR_D void row_update(cplx (&r)[P], int j, const cplx* mu, cplx dsig) {
  const cplx rj = sel<P>(r, j);
  const cplx nj = cmul(rj, dsig);
#pragma unroll
  for (int i = 0; i < P; ++i) r[i] = (i == j) ? nj : cfma(mu[i], rj, r[i]);
}

#define TR_SWITCH_J(P, CALL)                     \
  switch (j) {                                   \
    case 0: CALL(0); break;                      \
    case 1: CALL(1); break;                      \
    case 2: CALL(2); break;                      \
    case 3: CALL(3); break;                      \
    case 4: CALL(4); break;                      \
    case 5: if constexpr (P > 5) CALL(5); break; \
    case 6: if constexpr (P > 6) CALL(6); break; \
    default: break;                              \
  }

template <int P, int J>
TR_D void row_step(cplx (&r)[P], const cplx* mu, cplx dsig) {
  const cplx rj = r[J];
#pragma unroll
  for (int i = 0; i < P; ++i)
    if (i != J) r[i] = cfma(mu[i], rj, r[i]);
  r[J] = cmul(rj, dsig);
}

// ---------------------------------------------------- A (relay, no barriers)
// Warp w owns conditions 32w .. 32w+31 (one per lane).  Only the warp that
// owns the next condition is on the critical path: it applies the newest step
// to its rows, evaluates the pivot rule (SIMT; the owner lane's result is
// broadcast by shuffle), appends (j, mu, sigma) to an smem log and bumps a
// volatile head counter.  Every other warp replays the log on its own rows
// in the background and is current by the time the chain reaches it.
TR_D int vload(const int* p) { return *(const volatile int*)p; }
TR_D cplx shfl_c(cplx v, int src) {
  return cmk(__shfl_sync(FULL, v.x, src), __shfl_sync(FULL, v.y, src));
}

template <int P>
__global__ void __launch_bounds__(256) leaf_pivot_relay_kernel(LeafArgs a, SplitState s, int round) {
  const int sys = blockIdx.x;
  if (s.need[sys] != round) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = a.K, rows = a.rows;
  cplx* lmu = reinterpret_cast<cplx*>(smem_raw);   // [K][P]
  cplx* lsig = lmu + (size_t)K * P;                // [K]
  int* lj = reinterpret_cast<int*>(lsig + K);      // [K]
  int* head = lj + K;                              // [1]
  int* nd_s = head + 1;                            // [1]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int att = round;
  const cplx* W = a.W + (long long)sys * a.w_sys;
  const long long rowstride = (long long)rows * P;
  int2* dlog = s.def_try + (long long)sys * s.kcap;

  int cd[P];
#pragma unroll
  for (int i = 0; i < P; ++i) cd[i] = a.cd[sys * 8 + i];
  cplx r[P];
  cplx sg = cmk(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < P; ++i) r[i] = cmk(0.0, 0.0);
  if (tid < K) {
    const long long node = cond_node(a, tid, att);
    sg = __ldg(&a.twN[node]);
    const cplx* wr = W + node * rowstride + (tid % rows) * P;
#pragma unroll
    for (int i = 0; i < P; ++i) r[i] = wr[i];
  }
  if (tid == 0) {
    *head = 0;
    *nd_s = 0;
    s.viol[sys] = 0;
  }
  __syncthreads();

  const int first = 32 * warp;            // first condition this warp decides
  const int last = min(K, first + 32);    // one past its last
  if (first < K) {
    int done = 0;                         // log steps applied to these rows
    // decide condition tn on current rows and publish it (whole warp)
    auto publish = [&](int tn) {
      cplx m[P];
      const int jn = decide_fast<P>(r, cd, a.thr, m);
      const cplx so = sg;
      const int ow = tn & 31;
      if (lane == ow) {
        lj[tn] = jn;
        lsig[tn] = so;
        if (jn >= 0) {
#pragma unroll
          for (int i = 0; i < P; ++i) lmu[tn * P + i] = m[i];
        } else {
          const int nd = vload(nd_s);
          dlog[nd] = make_int2((int)cond_node(a, tn, att), tn % rows);
          *(volatile int*)nd_s = nd + 1;
        }
        __threadfence_block();
        *(volatile int*)head = tn + 1;
      }
      __syncwarp();
    };
    // apply logged step t to these rows
    auto apply = [&](int t) {
      const int j = lj[t];
      if (j >= 0) {
        cplx mu[P];
#pragma unroll
        for (int i = 0; i < P; ++i) mu[i] = lmu[t * P + i];
        const cplx sig_t = lsig[t];
#pragma unroll
        for (int i = 0; i < P; ++i) cd[i] += (i == j);
        if (tid > t && tid < K) row_update<P>(r, j, mu, csub(sg, sig_t));
      }
    };
    if (warp == 0) publish(0);
    // replay until the chain reaches this warp's first condition
    const int need = first > 0 ? first - 1 : 0;
    while (done < need) {
      int h;
      while ((h = vload(head)) <= done) __nanosleep(32);
      __threadfence_block();
      if (h > need) h = need;
      for (; done < h; ++done) apply(done);
    }
    // own the chain for conditions first .. last-1
    for (int tn = (first > 0 ? first : 1); tn < last; ++tn) {
      while (vload(head) < tn) {}
      __threadfence_block();
      apply(tn - 1);
      done = tn;
      publish(tn);
    }
  }
  __syncthreads();
  if (tid == 0) {
    int len = 1;
    int cdf[P];
#pragma unroll
    for (int i = 0; i < P; ++i) cdf[i] = a.cd[sys * 8 + i];
    cplx* mulog = s.mu + (long long)sys * s.kcap * P;
    int* jlog = s.jl + (long long)sys * s.kcap;
    for (int t = 0; t < K; ++t) {
      const int j = lj[t];
      jlog[t] = j;
      if (j >= 0) {
        ++len;
#pragma unroll
        for (int i = 0; i < P; ++i) cdf[i] += (i == j);
      }
    }
    s.ndef_try[sys] = *nd_s;
    s.len_try[sys] = len;
#pragma unroll
    for (int i = 0; i < P; ++i) s.cd_try[sys * 8 + i] = cdf[i];
  }
  // the mu log to HBM for the basis replay (coalesced, all threads)
  cplx* mulog = s.mu + (long long)sys * s.kcap * P;
  for (int e = tid; e < K * P; e += blockDim.x) mulog[e] = lmu[e];
}

// ------------------------------------------------------------------ B
template <int P, int D, int J>
TR_D void basis_step(cplx (&c)[D][P], const cplx* mu_s, cplx msig, cplx up) {
  cplx oj[D];
#pragma unroll
  for (int d = 0; d < D; ++d) oj[d] = c[d][J];
#pragma unroll
  for (int i = 0; i < P; ++i) {
    if (i == J) continue;
    const cplx m = mu_s[i];
#pragma unroll
    for (int d = 0; d < D; ++d) c[d][i] = cfma(m, oj[d], c[d][i]);
  }
#pragma unroll
  for (int d = 0; d < D; ++d) c[d][J] = cfma(msig, oj[d], d > 0 ? oj[d - 1] : up);
}

template <int P, int D>
TR_D cplx pick_top(const cplx (&c)[D][P], int j) {
  cplx v = c[D - 1][0];
#pragma unroll
  for (int i = 1; i < P; ++i)
    if (j == i) v = c[D - 1][i];
  return v;
}

// ------------------------------------------------------- B (one row per CTA)
// Rows of the basis never interact in the replay (B <- B F_t acts on each
// row separately), so row k of system s is CTA (s, k): P x more, much smaller
// CTAs with cheap barriers.  Coefficients are written unnormalised together
// with per-row column maxima; the check kernel normalises.
template <int P, int D, int MAXT>
__global__ void __launch_bounds__(MAXT) leaf_build_row_kernel(LeafArgs a, SplitState s, int round,
                                                              int TPR) {
  const int sys = blockIdx.x, krow = blockIdx.y;
  if (s.need[sys] != round) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = a.K;
  const int NT = blockDim.x, NW = NT / 32;
  cplx* musm = reinterpret_cast<cplx*>(smem_raw);  // [K][P]
  cplx* sgsm = musm + (size_t)K * P;               // [K]
  cplx* halo = sgsm + K;                           // [2][NW][P]
  double* red = reinterpret_cast<double*>(halo + 2 * NW * P);  // [NW][P]
  int* jsm = reinterpret_cast<int*>(red + NW * P); // [K]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int u = tid;
  const bool act = u < TPR;
  const int att = round;
  const cplx* mulog = s.mu + (long long)sys * s.kcap * P;
  const int* jlog = s.jl + (long long)sys * s.kcap;
  for (int e = tid; e < K; e += NT) {
    const int j = jlog[e];
    jsm[e] = j;
    sgsm[e] = __ldg(&a.twN[cond_node(a, e, att)]);
    if (j >= 0)
#pragma unroll
      for (int i = 0; i < P; ++i) musm[e * P + i] = mulog[(long long)e * P + i];
  }
  cplx c[D][P];
#pragma unroll
  for (int d = 0; d < D; ++d)
#pragma unroll
    for (int i = 0; i < P; ++i)
      c[d][i] = (u == 0 && d == 0 && i == krow) ? cmk(1.0, 0.0) : cmk(0.0, 0.0);
  if (lane == 31) {
#pragma unroll
    for (int i = 0; i < P; ++i) halo[warp * P + i] = c[D - 1][i];
  }
  __syncthreads();
  int len = 1, cur = 0;
  bool big = false;
  for (int t = 0; t < K; ++t) {
    const int j = jsm[t];
    if (j < 0) continue;
    const cplx* mu_s = musm + t * P;
    const cplx msig = cneg(sgsm[t]);
    cplx oj[D];
#pragma unroll
    for (int d = 0; d < D; ++d) oj[d] = sel<P>(c[d], j);
    cplx up;
    up.x = __shfl_up_sync(FULL, oj[D - 1].x, 1);
    up.y = __shfl_up_sync(FULL, oj[D - 1].y, 1);
    if (lane == 0 && warp > 0) up = halo[(cur * NW + warp - 1) * P + j];
    if (u == 0) up = cmk(0.0, 0.0);
    if (act && u * D <= len) {
      cplx mu[P];
#pragma unroll
      for (int i = 0; i < P; ++i) mu[i] = mu_s[i];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const cplx nj = cfma(msig, oj[d], d > 0 ? oj[d - 1] : up);
#pragma unroll
        for (int i = 0; i < P; ++i) c[d][i] = (i == j) ? nj : cfma(mu[i], oj[d], c[d][i]);
      }
    }
    ++len;
    if (((t + 1) % RESCALE_PERIOD) == 0) {
#pragma unroll
      for (int d = 0; d < D; ++d)
#pragma unroll
        for (int i = 0; i < P; ++i) big |= cabs2(c[d][i]) > RESCALE_TRIGGER * RESCALE_TRIGGER;
    }
    cur ^= 1;
    if (lane == 31) {
#pragma unroll
      for (int i = 0; i < P; ++i) halo[(cur * NW + warp) * P + i] = c[D - 1][i];
    }
    __syncthreads();
  }
  if (big) atomicOr(&s.viol[sys], 1);
  // per-row column maxima (squared) for the check kernel's normalisation
#pragma unroll
  for (int i = 0; i < P; ++i) {
    double m = 0.0;
#pragma unroll
    for (int d = 0; d < D; ++d) m = fmax(m, cabs2(c[d][i]));
    m = wmax(m);
    if (lane == 0) red[warp * P + i] = m;
  }
  __syncthreads();
  if (tid < P) {
    double m = 0.0;
    for (int w = 0; w < NW; ++w) m = fmax(m, red[w * P + tid]);
    s.colpart[((long long)sys * 8 + krow) * 8 + tid] = m;
  }
  cplx* dst = (round == 0 ? a.out : a.scratch) + (long long)sys * a.out_sys;
  if (act) {
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int l = u * D + d;
      if (l < a.cap) {
#pragma unroll
        for (int i = 0; i < P; ++i) dst[(long long)(krow * P + i) * a.cap + l] = c[d][i];
      }
    }
  }
  const int covered = TPR * D;
  if (a.cap > covered) {
    const int tail = a.cap - covered;
    for (long long e = tid; e < (long long)P * tail; e += NT)
      dst[(long long)(krow * P + e / tail) * a.cap + covered + e % tail] = cmk(0.0, 0.0);
  }
}

// ------------------------------------------------------------------ C
constexpr int CK = 256;

template <int P>
__global__ void __launch_bounds__(CK) leaf_check_kernel(LeafArgs a, SplitState s, int round,
                                                        int norm) {
  const int sys = blockIdx.x;
  if (s.need[sys] != round) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int M = a.M, rows = a.rows, K = a.K;
  cplx* wtab = reinterpret_cast<cplx*>(smem_raw);  // [M]
  cplx* gbuf = wtab + M;                           // [P*P][M]
  cplx* bvb = gbuf + P * P * M;                    // [P*P][M]
  cplx* twl = bvb + P * P * M;                     // [cap] twist factors of one coset
  __shared__ double red[CK / 32];
  __shared__ double csafe[8];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const cplx* W = a.W + (long long)sys * a.w_sys;
  const long long rowstride = (long long)rows * P;
  cplx* src = (round == 0 ? a.out : a.scratch) + (long long)sys * a.out_sys;
  const int len = s.len_try[sys];
  for (int e = tid; e < M; e += CK) wtab[e] = __ldg(&a.twN[(long long)e * a.stride]);
  if (norm) {
    // column normalisation of the row-parallel build (ref tanint.py:179-183)
    if (tid < P) {
      double m = 0.0;
      for (int k = 0; k < P; ++k) m = fmax(m, s.colpart[((long long)sys * 8 + k) * 8 + tid]);
      m = sqrt(m);
      csafe[tid] = m > 0.0 ? m : 1.0;
    }
    __syncthreads();
    if (tid == 0) {
      double f = 1.0;
      for (int i = 0; i < P; ++i) f = fmax(f, csafe[i]);
      s.factor_try[sys] = f;
    }
    for (long long e = tid; e < (long long)P * P * len; e += CK) {
      const long long ee = e / len, l = e % len;
      cplx* p = src + ee * a.cap + l;
      *p = cscale(*p, 1.0 / csafe[ee % P]);
    }
    __syncthreads();
  }
  // scale = max |w_in| over the leaf's conditions
  double sc = 0.0;
  for (int e = tid; e < K * P; e += CK) {
    const int pos = e / (rows * P), rem = e % (rows * P);
    sc = fmax(sc, cabs2(W[node_of(a, pos) * rowstride + rem]));
  }
  sc = wmax(sc);
  if (lane == 0) red[warp] = sc;
  __syncthreads();
  double scale = 0.0;
  for (int w = 0; w < CK / 32; ++w) scale = fmax(scale, red[w]);
  scale = sqrt(scale);
  __syncthreads();
  double resm = 0.0;
  for (int cs = 0; cs < a.noff; ++cs) {
    const long long oc = cs ? a.o1 : a.o0;
    // twist factors w_N^(oc l), l < len, generated incrementally per warp-stride
    for (int l = tid; l < len; l += CK) twl[l] = __ldg(&a.twN[(oc * l) % a.N]);
    __syncthreads();
    for (int e = tid; e < P * P * M; e += CK) {
      const int ee = e / M, q = e % M;
      cplx acc = cmk(0.0, 0.0);
      for (int l = q; l < len; l += M) acc = cfma(src[(long long)ee * a.cap + l], twl[l], acc);
      gbuf[ee * M + q] = acc;
    }
    __syncthreads();
    for (int e = tid; e < P * P * M; e += CK) {
      const int ee = e / M, tt = e % M;
      const cplx* g = gbuf + ee * M;
      cplx acc = cmk(0.0, 0.0);
      int k = 0;
      for (int q = 0; q < M; ++q) {
        acc = cfma(g[q], wtab[k], acc);
        k += tt;
        if (k >= M) k -= M;
      }
      bvb[ee * M + tt] = acc;
    }
    __syncthreads();
    for (int e = tid; e < M * rows * P; e += CK) {
      const int tt = e / (rows * P), rem = e % (rows * P);
      const int rr = rem / P, jj = rem % P;
      const cplx* wrow = W + (oc + a.stride * (long long)tt) * rowstride + rr * P;
      cplx acc = cmk(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < P; ++i) acc = cfma(wrow[i], bvb[(i * P + jj) * M + tt], acc);
      resm = fmax(resm, cabs2(acc));
    }
    __syncthreads();
  }
  resm = wmax(resm);
  if (lane == 0) red[warp] = resm;
  __syncthreads();
  double res = 0.0;
  for (int w = 0; w < CK / 32; ++w) res = fmax(res, red[w]);
  res = (scale == 0.0) ? 0.0 : sqrt(res) / scale;
  const bool better = round == 0 || res < s.res_best[sys];
  const int nd = s.ndef_try[sys];
  if (better) {
    if (round > 0) {
      cplx* o = a.out + (long long)sys * a.out_sys;
      for (long long e = tid; e < (long long)P * P * a.cap; e += CK) o[e] = src[e];
    }
    int2* db = s.def_best + (long long)sys * s.kcap;
    const int2* dt = s.def_try + (long long)sys * s.kcap;
    for (int e = tid; e < nd; e += CK) db[e] = dt[e];
  }
  __syncthreads();
  if (tid == 0) {
    if (better) {
      s.res_best[sys] = res;
      s.ndef_best[sys] = nd;
      s.factor_best[sys] = s.factor_try[sys];
      s.len_best[sys] = s.len_try[sys];
      for (int i = 0; i < P; ++i) s.cd_best[sys * 8 + i] = s.cd_try[sys * 8 + i];
    }
    const bool done = s.res_best[sys] <= a.check_tol || round + 1 >= a.nattempts;
    if (s.viol[sys]) {
      s.need[sys] = SPLIT_EXACT;  // speculation failed: exact coupled kernel
      *s.any_viol = 1;
    } else if (!done) {
      s.need[sys] = round + 1;    // retry with the next absorption order
    } else {
      // commit (ref tanint.py:430-434)
      for (int i = 0; i < P; ++i) a.cd[sys * 8 + i] = s.cd_best[sys * 8 + i];
      const int base = a.dcount[sys];
      const int nb = s.ndef_best[sys];
      const int room = a.dmax - base;
      const int nput = nb < room ? nb : room;
      const int2* db = s.def_best + (long long)sys * s.kcap;
      for (int e = 0; e < nput; ++e) a.defer[(long long)sys * a.dmax + base + e] = db[e];
      a.dcount[sys] = base + nb;
      if (nb > room) a.status[sys] = 5;
      a.max_scale[sys] = fmax(a.max_scale[sys], s.factor_best[sys]);
      if (round > 0) a.retried[sys] += 1;
      if (a.res_out) a.res_out[sys] = s.res_best[sys];
      if (a.len_out) a.len_out[sys] = s.len_best[sys];
      s.need[sys] = SPLIT_DONE;
    }
  }
}

__global__ void need_reset_kernel(int* need, int nsys) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nsys) need[i] = 0;
}

template <int P, int D, int MAXT>
int launch_build_row(const LeafArgs& a, const SplitState& s, int round, int nsys, cudaStream_t st) {
  const int TPR = (a.K + 1 + D - 1) / D;
  const int NT = (TPR + 31) & ~31;
  if (NT > MAXT) return -1;
  const int NW = NT / 32;
  size_t smem = sizeof(cplx) * ((size_t)a.K * P + a.K + 2 * (size_t)NW * P) +
                sizeof(double) * NW * P + sizeof(int) * (a.K + 1);
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(leaf_build_row_kernel<P, D, MAXT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         160 * 1024);
    set = true;
  }
  TrKTimer _kt(TRK_LEAF_BUILD, st);
  leaf_build_row_kernel<P, D, MAXT><<<dim3(nsys, P), NT, smem, st>>>(a, s, round, TPR);
  return 0;
}

size_t check_smem(const LeafArgs& a) {
  return sizeof(cplx) * ((size_t)a.M + 2 * (size_t)a.P * a.P * a.M + a.cap);
}

}  // namespace

bool leaf_split_supported(const LeafArgs& a) {
  if (check_smem(a) > 200 * 1024) return false;
  if (a.K > 256) return false;
  return a.P == 5 || a.P == 7;
}

// One leaf for every system: rounds of (pivot chain, basis replay, check);
// a system leaves the rounds as soon as its self-check passes.
int leaf_split_launch(const LeafArgs& a, const SplitState& s, int nsys, cudaStream_t st) {
  {
    TrKTimer _kt(TRK_LEAF_PIVOT, st);
    need_reset_kernel<<<(nsys + 255) / 256, 256, 0, st>>>(s.need, nsys);
  }
  {  // algorithmic work of one attempt (retry rounds are extra work, not counted)
    const double K = a.K, P = a.P;
    tr_kernel_work(TRK_LEAF_PIVOT, 16.0 * nsys * K * P, 4.0 * nsys * P * K * (K - 1));
    tr_kernel_work(TRK_LEAF_BUILD, 16.0 * nsys * P * P * (K + 1), 4.0 * nsys * P * P * K * (K + 1));
    tr_kernel_work(TRK_LEAF_CHECK, 16.0 * nsys * (P * P * (K + 1) + K * P),
                   8.0 * nsys * (P * P * (K + 1) + (double)a.noff * P * P * a.M * a.M));
  }
  const size_t csm = check_smem(a);
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(leaf_check_kernel<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    cudaFuncSetAttribute(leaf_check_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    set = true;
  }
  for (int round = 0; round < a.nattempts; ++round) {
    {
      TrKTimer _kt(TRK_LEAF_PIVOT, st);
      const size_t rsm = sizeof(cplx) * (size_t)a.K * (a.P + 1) + sizeof(int) * (a.K + 2);
      if (a.P == 5) leaf_pivot_relay_kernel<5><<<nsys, 256, rsm, st>>>(a, s, round);
      else leaf_pivot_relay_kernel<7><<<nsys, 256, rsm, st>>>(a, s, round);
    }
    const int rc = a.P == 5 ? launch_build_row<5, 1, 288>(a, s, round, nsys, st)
                            : launch_build_row<7, 1, 288>(a, s, round, nsys, st);
    if (rc) {
      tr_set_error("leaf split shape unsupported (K=%d, P=%d)", a.K, a.P);
      return 2;
    }
    {
      TrKTimer _kt(TRK_LEAF_CHECK, st);
      if (a.P == 5) leaf_check_kernel<5><<<nsys, CK, csm, st>>>(a, s, round, 1);
      else leaf_check_kernel<7><<<nsys, CK, csm, st>>>(a, s, round, 1);
    }
  }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}
