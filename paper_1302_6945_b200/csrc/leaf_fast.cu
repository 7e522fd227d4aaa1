// Leaf sweep (ref: pkg/src/toepreg/tanint.py:395-434 _serial_leaf, :189-217
// _serial_core, :262-270 _self_residual).
//
// The reference absorbs a leaf's K conditions one at a time into a P x P
// polynomial workspace, then checks the result and retries other absorption
// orders.  The decisions (pivot column, deferral, mu) depend on the basis
// only through the residual rows r_s = w_s . B(sigma_s), which obey
// r_i += mu_i r_j, r_j *= (sigma_s - sigma_t) at every absorbed step.
//
// Default (batches of <= 148 systems): leaf_fused3_kernel, one CTA per
// system-leaf, every attempt of the leaf in one launch:
//   * decider (warp 0, alone on its scheduler): a block of 32 consecutive
//     conditions, one row per lane; a step is shuffle -> pivot rule
//     (branch-free argmax on squared moduli) -> MUFU+Newton reciprocal ->
//     own-row update, published to a shared-memory log with a release store;
//   * holders apply published steps to the later rows (acquire polling) and
//     hand their block to the decider when it gets there;
//   * P basis-row warps replay the log on the coefficient cube (coefficient
//     l = 32 d + lane in registers, structurally-zero blocks skipped); for
//     P = 5 the multipliers mu_i = f_i c_i they all need are formed once per
//     step by the mu warp (warp 4, beside the decider) and read from lmu;
//   * finish_attempt: column normalisation, the self-residual (coset fold +
//     factored M-point DFT) and the retry rule; attempts 0 and 1 run side by
//     side in a 2-CTA cluster when the batch leaves SMs free.
// Larger batches: leaf_chain2_kernel (the same chain with barrier hand-offs)
// then leaf_basis_kernel (row-parallel replay + finish), one launch each per
// attempt round.
//
// The reference's mid-sweep rescale (columns above 1e8 at every 8th
// condition, ref :214-217) would change later decisions; the chain assumes it
// does not fire and the replay checks that no coefficient exceeded the
// trigger at those points.  A leaf that violates this is redone by the exact
// coupled kernel (leaf.cu).
#include <cooperative_groups.h>
#include <stdio.h>
#include <type_traits>
#include <stdlib.h>

#include "leaf.cuh"
#include "leaf_split.cuh"

// chain clock trace of system 0 (diagnostic, tr_debug_chain_trace)
__device__ long long g_chain_trace[4 * 1024];
__device__ int g_chain_trace_on = 0;
#define TR_BTRACE(slot) \
  if (g_chain_trace_on && sys == 0 && round == 0 && tid == 32) g_chain_trace[3072 + (slot)] = clock64();

extern "C" int tr_debug_chain_trace(int enable, long long* out, int n) {
  int on = enable;
  cudaMemcpyToSymbol(g_chain_trace_on, &on, sizeof(int));
  if (out) cudaMemcpyFromSymbol(out, g_chain_trace, sizeof(long long) * (n < 4096 ? n : 4096));
  return 0;
}

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr double RESCALE_TRIGGER = 1e8;
constexpr int RESCALE_PERIOD = 8;
constexpr int NT = 256;  // threads per CTA of both kernels
constexpr int NW = NT / 32;
#ifndef TR_MU_WARP
#define TR_MU_WARP 1  // one warp forms the multipliers mu_i = f_i c_i for all basis rows (leaf_fused3_kernel)
#endif
#ifndef TR_SPIN_NS
#define TR_SPIN_NS 0  // pure acquire polling measured ~1% better than back-off (16-256 ns)
#endif

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
TR_D int vload(const int* p) { return *(const volatile int*)p; }
// release store / acquire load on a shared-memory flag (MEMBAR.ALL.CTA, lighter
// than __threadfence_block's MEMBAR.SC.CTA)
TR_D void st_release(int* p, int v) {
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v)
               : "memory");
}
TR_D int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];"
               : "=r"(v)
               : "r"((unsigned)__cvta_generic_to_shared(p))
               : "memory");
  return v;
}
// Predicated shared-memory stores on precomputed 32-bit shared addresses: the
// decider publishes a step from lane 0 without a divergent branch (the
// branch's lane-0 block -- address rematerialisation through S2R, seven
// stores, the fence -- sat in the middle of every chain step: ~29% of the
// step's stall samples, profiles/r2_leaf_publish.txt)
TR_D unsigned smem_u32(const void* p) {
  unsigned a = (unsigned)__cvta_generic_to_shared(p);
  asm volatile("" : "+r"(a));  // opaque: held in a register, not recomputed per step
  return a;
}
TR_D void sts_c_if(int pred, unsigned addr, cplx v) {
  asm volatile("{ .reg .pred p; setp.ne.s32 p, %0, 0; @p st.shared.v2.f64 [%1], {%2, %3}; }" ::"r"(pred), "r"(addr),
               "d"(v.x), "d"(v.y)
               : "memory");
}
TR_D void sts_i_if(int pred, unsigned addr, int v) {
  asm volatile("{ .reg .pred p; setp.ne.s32 p, %0, 0; @p st.shared.u32 [%1], %2; }" ::"r"(pred), "r"(addr), "r"(v)
               : "memory");
}
TR_D void st_release_if(int pred, unsigned addr, int v) {
  asm volatile("{ .reg .pred p; setp.ne.s32 p, %0, 0; @p st.release.cta.shared.u32 [%1], %2; }" ::"r"(pred),
               "r"(addr), "r"(v)
               : "memory");
}
// wait until the published step counter passes t (backs off so that spinning
// warps leave the shared-memory pipe to the decider)
TR_D int wait_steps(const int* flag, int t, int avail) {
  while (avail <= t) {
    avail = ld_acquire(flag);
    if (TR_SPIN_NS > 0 && avail <= t) __nanosleep(TR_SPIN_NS);
  }
  return avail;
}
TR_D cplx shfl_c(cplx v, int src) {
  return cmk(__shfl_sync(FULL, v.x, src), __shfl_sync(FULL, v.y, src));
}
// 1/x to ~1 ulp: MUFU estimate + two Newton steps
TR_D double rcp_nr(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
// mu_i = f_i c_i with a fixed rounding sequence: the multipliers are formed in three places
// (the mu warp of the fused kernel, its basis rows when no mu warp runs, the chain kernel of
// the split path) and must not depend on how the compiler contracts each of them
TR_D cplx cmul_mu(cplx a, cplx b) {
  return cmk(__fma_rn(a.x, b.x, -__dmul_rn(a.y, b.y)), __fma_rn(a.x, b.y, __dmul_rn(a.y, b.x)));
}
// (P = 7 keeps the plain product in both of its kernels: its leaves run no mu warp, and the
// pinned sequence costs the decider-bound general variant 2% -- config 3: 6.75 -> 6.6 solves/s)
template <int P>
TR_D cplx mu_prod(cplx a, cplx b) {
  if constexpr (P == 5) return cmul_mu(a, b);
  else return cmul(a, b);
}
// a b - c d, the two products in parallel
TR_D cplx cmsub(cplx a, cplx b, cplx c, cplx d) {
  const double ux = fma(a.x, b.x, -a.y * b.y), uy = fma(a.x, b.y, a.y * b.x);
  const double vx = fma(c.x, d.x, -c.y * d.y), vy = fma(c.x, d.y, c.y * d.x);
  return cmk(ux - vx, uy - vy);
}
template <int P>
TR_D cplx sel(const cplx (&v)[P], int j) {
  cplx r = v[0];
#pragma unroll
  for (int i = 1; i < P; ++i) r = (j == i) ? v[i] : r;
  return r;
}
template <int P>
TR_D int sel_i(const int (&v)[P], int j) {
  int r = v[0];
#pragma unroll
  for (int i = 1; i < P; ++i) r = (j == i) ? v[i] : r;
  return r;
}
// r <- r F_t(sigma) with the true multipliers (mu_j = 0)
template <int P>
TR_D void row_update(cplx (&r)[P], int j, const cplx* mu, cplx dsig) {
  const cplx rj = sel<P>(r, j);
  const cplx nj = cmul(rj, dsig);
#pragma unroll
  for (int i = 0; i < P; ++i) {
    const cplx v = cfma(mu[i], rj, r[i]);
    r[i] = (i == j) ? nj : v;
  }
}

// The pivot rule of ref tanint.py:193-211 on squared moduli: among the
// lowest-degree columns the first of largest |phi|; deferred (-1) when that
// is below thr * max|phi| or the row vanishes.  The argmax tree carries the
// winning entry along (fj).
template <int P>
TR_D int chain_decide(const cplx (&f)[P], const cplx (&pre)[P], const int (&cd)[P], double thr2,
                      cplx& fj, cplx& qj, int& jj) {
  double v[P], am[P];
  int ix[P];
  cplx fv[P], pv[P];
  int dmin = cd[0];
#pragma unroll
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
#pragma unroll
  for (int i = 0; i < P; ++i) {
    am[i] = cabs2(f[i]);
    v[i] = cd[i] == dmin ? am[i] : -1.0;
    ix[i] = i;
    fv[i] = f[i];
    pv[i] = pre[i];
  }
#pragma unroll
  for (int w = 1; w < P; w *= 2) {
#pragma unroll
    for (int i = 0; i + w < P; i += 2 * w) {
      const bool take = v[i + w] > v[i];
      ix[i] = take ? ix[i + w] : ix[i];
      v[i] = take ? v[i + w] : v[i];
      fv[i] = take ? fv[i + w] : fv[i];
      pv[i] = take ? pv[i + w] : pv[i];
      am[i] = fmax(am[i], am[i + w]);
    }
  }
  fj = fv[0];
  qj = pv[0];
  jj = ix[0];
  if (am[0] == 0.0 || v[0] < thr2 * am[0]) return -1;
  return ix[0];
}

// One absorbed step with pivot J (compile time: no selects on the chain):
// mu_i = -phi_i / phi_J (mu_J = 0),
//   next front = pre + mu pre_J,  pre_J (s_pre - s_front) in column J;
//   own rows   = r + mu r_J,      r_J (s_row - s_front) in column J.
template <int P, int J>
TR_D void chain_step(cplx (&f)[P], const cplx (&pre)[P], cplx (&r)[P], cplx (&mu)[P], int (&cd)[P],
                     cplx dpf, cplx drf) {
  const cplx fj = f[J];
  const double inv2 = rcp_nr(cabs2(fj));
  const cplx ci = cmk(-fj.x * inv2, fj.y * inv2);
#pragma unroll
  for (int i = 0; i < P; ++i) mu[i] = (i == J) ? cmk(0.0, 0.0) : cmul(f[i], ci);
  const cplx qj = pre[J];
  const cplx rj = r[J];
#pragma unroll
  for (int i = 0; i < P; ++i) {
    if (i == J) {
      f[i] = cmul(qj, dpf);
      r[i] = cmul(rj, drf);
    } else {
      f[i] = cfma(mu[i], qj, pre[i]);
      r[i] = cfma(mu[i], rj, r[i]);
    }
  }
  cd[J] += 1;
}

template <int P>
TR_D void chain_step_any(int j, cplx (&f)[P], const cplx (&pre)[P], cplx (&r)[P], cplx (&mu)[P],
                         int (&cd)[P], cplx dpf, cplx drf) {
  if (j < 0) {
#pragma unroll
    for (int i = 0; i < P; ++i) {
      f[i] = pre[i];
      mu[i] = cmk(0.0, 0.0);
    }
  } else if (j == 0) chain_step<P, 0>(f, pre, r, mu, cd, dpf, drf);
  else if (j == 1) chain_step<P, 1>(f, pre, r, mu, cd, dpf, drf);
  else if (j == 2) chain_step<P, 2>(f, pre, r, mu, cd, dpf, drf);
  else if (j == 3) chain_step<P, 3>(f, pre, r, mu, cd, dpf, drf);
  else if constexpr (P == 5) {
    chain_step<P, 4>(f, pre, r, mu, cd, dpf, drf);
  } else {
    if (j == 4) chain_step<P, 4>(f, pre, r, mu, cd, dpf, drf);
    else if (j == 5) chain_step<P, 5>(f, pre, r, mu, cd, dpf, drf);
    else chain_step<P, 6>(f, pre, r, mu, cd, dpf, drf);
  }
}

// decision only (winning entry carried along)
template <int P>
TR_D int chain_decide1(const cplx (&f)[P], const int (&cd)[P], double thr2, cplx& fj) {
  double v[P], am[P];
  int ix[P];
  cplx fv[P];
  int dmin = cd[0];
#pragma unroll
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
#pragma unroll
  for (int i = 0; i < P; ++i) {
    am[i] = cabs2(f[i]);
    v[i] = cd[i] == dmin ? am[i] : -1.0;
    ix[i] = i;
    fv[i] = f[i];
  }
#pragma unroll
  for (int w = 1; w < P; w *= 2) {
#pragma unroll
    for (int i = 0; i + w < P; i += 2 * w) {
      const bool take = v[i + w] > v[i];
      ix[i] = take ? ix[i + w] : ix[i];
      v[i] = take ? v[i + w] : v[i];
      fv[i] = take ? fv[i + w] : fv[i];
      am[i] = fmax(am[i], am[i + w]);
    }
  }
  fj = fv[0];
  if (am[0] == 0.0 || v[0] < thr2 * am[0]) return -1;
  return ix[0];
}

// decider multipliers for pivot J (compile time): mu_i = -phi_i / phi_J, mu_J = 0
template <int P, int J>
TR_D void decider_mu(const cplx (&f)[P], cplx (&mu)[P], int (&cd)[P], cplx fj) {
  const double inv2 = rcp_nr(cabs2(fj));
  const cplx ci = cmk(-fj.x * inv2, fj.y * inv2);
#pragma unroll
  for (int i = 0; i < P; ++i) mu[i] = (i == J) ? cmk(0.0, 0.0) : cmul(f[i], ci);
  cd[J] += 1;
}

// ---------------------------------------------- chain kernel, warp-specialised
// Warp 0 (the decider) owns the chain: it keeps the row being decided
// ("front", row t through step t-1) and the next one ("pre", row t+1 through
// t-1) replicated in its lanes, decides step t, forms mu_t, publishes
// (j_t, mu_t) and updates pre into the next front.  Warps 1..H (holders) own
// 32 rows each and apply every published step to their rows; the holder of
// row t+2 hands it back (through step t) for the decider's next pre.  The
// hand-offs are named barriers (bar.arrive by the producer, bar.sync by the
// consumers: ~70 cycles one way, with memory ordering), so the decider never
// polls and never updates rows it does not need.
//   barriers 1/3 (step t published, t even/odd): decider + the holders still
//     needed at step t;
//   barriers 2/4 (row t+2 handed back after step t): decider + its holder.
// The decider consumes the hand-back of step t-1 only at the end of step t,
// so the holders' round trip overlaps a whole decision.
TR_D void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
TR_D void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// Pivot rule on the bit patterns of the squared moduli (non-negative doubles
// order like their bits): integer compares and selects instead of FP64
// ones; the winning entry and its squared modulus are carried along.
template <int P>
TR_D int decide_bits(const cplx (&f)[P], const int (&cd)[P], double thr2, cplx& fj, double& a2j) {
  unsigned long long v[P], am[P];
  int ix[P];
  cplx fv[P];
  int dmin = cd[0];
#pragma unroll
  for (int i = 1; i < P; ++i) dmin = min(dmin, cd[i]);
#pragma unroll
  for (int i = 0; i < P; ++i) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(cabs2(f[i]));
    am[i] = b;
    v[i] = cd[i] == dmin ? b : 0ull;
    ix[i] = i;
    fv[i] = f[i];
  }
#pragma unroll
  for (int w = 1; w < P; w *= 2) {
#pragma unroll
    for (int i = 0; i + w < P; i += 2 * w) {
      const bool take = v[i + w] > v[i];
      ix[i] = take ? ix[i + w] : ix[i];
      v[i] = take ? v[i + w] : v[i];
      fv[i] = take ? fv[i + w] : fv[i];
      am[i] = am[i] > am[i + w] ? am[i] : am[i + w];
    }
  }
  fj = fv[0];
  a2j = __longlong_as_double((long long)v[0]);
  const double amax = __longlong_as_double((long long)am[0]);
  if (amax == 0.0 || a2j < thr2 * amax) return -1;
  return ix[0];
}

template <int P, bool SPREAD>
__global__ void __launch_bounds__(SPREAD ? 352 : 288, SPREAD ? 1 : 2) leaf_chain2_kernel(LeafArgs a, SplitState s, int round) {
  const int sys = blockIdx.x;
  if (s.need[sys] != round) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int K = a.K, rows = a.rows;
  // log of step t: the decided row phi_t (lf), c_t = -conj(phi_j)/|phi_j|^2
  // (lci) and j_t; the multipliers are mu_i = phi_i c_t (mu_j = 0)
  cplx* lf = reinterpret_cast<cplx*>(smem_raw);    // [K][P]
  cplx* lci = lf + (size_t)K * P;                  // [K]
  cplx* lsig = lci + K;                            // [K + 2] node of every condition
  cplx* prow = lsig + K + 2;                       // [2][P] handed-back rows
  int* lj = reinterpret_cast<int*>(prow + 2 * P);  // [K] pivot or -1
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(FULL, tid >> 5, 0);  // warp-uniform for ptxas
  const int att = round;
  const cplx* W = a.W + (long long)sys * a.w_sys;
  const long long rowstride = (long long)rows * P;
  int2* dlog = s.def_try + (long long)sys * s.kcap;
  const int H = (K + 31) / 32;  // holder warps
  // holders live on warps 1, 2, 3, 5, 6, 7, 9, 10 (never warp_id = 0 mod 4, the
  // decider's scheduler); holder h >= 1 owns conditions 32 (h - 1) + lane
  // (SPREAD, for one CTA per SM) or on warps 1..H (compact, two CTAs per SM)
  const int hid = SPREAD ? ((warp & 3) ? warp - warp / 4 : 0) : warp;
  const int mine = 32 * (hid - 1) + lane;
  cplx r[P];
  cplx sg = cmk(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < P; ++i) r[i] = cmk(0.0, 0.0);
  if (hid >= 1 && mine < K) {
    const long long node = cond_node(a, mine, att);
    sg = __ldg(&a.twN[node]);
    lsig[mine] = sg;
    const cplx* wr = W + node * rowstride + (mine % rows) * P;
#pragma unroll
    for (int i = 0; i < P; ++i) r[i] = wr[i];
  }
  if (tid < 2) lsig[K + tid] = cmk(0.0, 0.0);
  __syncthreads();

  // participants of barrier 1 at step t: the decider and holders h >= hmin
  auto hmin = [&](int t) { return (t + 2) / 32 + 1; };
  auto nbar1 = [&](int t) { return 32 * (1 + H - hmin(t) + 1); };

  if (warp == 0) {
    // ---------------- decider ----------------
    const double thr2 = a.thr * a.thr;
    int cd[P];
#pragma unroll
    for (int i = 0; i < P; ++i) cd[i] = a.cd[sys * 8 + i];
    cplx f[P], pre[P];
    {
      const long long n0 = cond_node(a, 0, att);
      const cplx* w0 = W + n0 * rowstride;
#pragma unroll
      for (int i = 0; i < P; ++i) f[i] = w0[i];
      if (K > 1) {
        const long long n1 = cond_node(a, 1, att);
        const cplx* w1 = W + n1 * rowstride + (1 % rows) * P;
#pragma unroll
        for (int i = 0; i < P; ++i) pre[i] = w1[i];
      } else {
#pragma unroll
        for (int i = 0; i < P; ++i) pre[i] = cmk(0.0, 0.0);
      }
    }
    cplx sf = lsig[0], sp = lsig[1];
    const bool trace = g_chain_trace_on && sys == 0 && round == 0 && lane == 0;
    for (int t = 0; t < K; ++t) {
      if (trace) g_chain_trace[4 * t] = clock64();
      cplx fj;
      double a2j;
      const int j = decide_bits<P>(f, cd, thr2, fj, a2j);
      const double inv2 = rcp_nr(a2j);
      const cplx ci = cmk(-fj.x * inv2, fj.y * inv2);
      if (trace) g_chain_trace[4 * t + 1] = clock64() + 0 * j;
      if (lane == 0) {
        lj[t] = j;
        lci[t] = ci;
#pragma unroll
        for (int i = 0; i < P; ++i) lf[t * P + i] = f[i];
      }
      // step t to the holders (barrier ids alternate: the decider runs one
      // step ahead of the hand-back)
      if (t + 2 < K) bar_arrive(1 + 2 * (t & 1), nbar1(t));
      if (t + 1 < K) {
        if (t >= 1) {  // pre <- row t+1 through step t-1 (holder step t-1)
          bar_sync(2 + 2 * ((t - 1) & 1), 64);
          if (trace) g_chain_trace[4 * t + 2] = clock64();
          const cplx* src = prow + ((t - 1) & 1) * P;
#pragma unroll
          for (int i = 0; i < P; ++i) pre[i] = src[i];
        }
        // next front: row t+1 through step t = pre + phi (c q_j), q_j (s_p - s_f) in column j
        const cplx qj = sel<P>(pre, j);
        const cplx c2 = cmul(ci, qj);
        const cplx nfj = cmul(qj, csub(sp, sf));
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const cplx v = cfma(f[i], c2, pre[i]);
          f[i] = (j < 0) ? pre[i] : (i == j) ? nfj : v;
        }
      }
#pragma unroll
      for (int i = 0; i < P; ++i) cd[i] += (i == j);
      sf = sp;
      sp = lsig[t + 2];
      if (trace) g_chain_trace[4 * t + 3] = clock64() + 0 * (long long)f[0].x;
    }
  } else if (hid >= 1 && hid <= H) {
    // ---------------- holder ----------------
    for (int t = 0; t + 2 < K && hid >= hmin(t); ++t) {
      bar_sync(1 + 2 * (t & 1), nbar1(t));
      const int j = lj[t];
      if (j >= 0) {
        // r <- r + phi (c r_j), r_j (s_r - s_t) in column j
        const cplx rj = sel<P>(r, j);
        const cplx c2 = cmul(lci[t], rj);
        const cplx nj = cmul(rj, csub(sg, lsig[t]));
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const cplx v = cfma(lf[t * P + i], c2, r[i]);
          r[i] = (i == j) ? nj : v;
        }
      }
      if (hid == hmin(t)) {
        if (lane == (t + 2) % 32) {
          cplx* dst = prow + (t & 1) * P;
#pragma unroll
          for (int i = 0; i < P; ++i) dst[i] = r[i];
        }
        bar_arrive(2 + 2 * (t & 1), 64);
      }
    }
  }
  __syncthreads();
  // epilogue (warp 0): pivot log, basis length, ledger, deferred conditions in
  // step order (ref tanint.py:200-206)
  if (warp == 0) {
    int len = 1, nd = 0;
    int cdf[P];
#pragma unroll
    for (int i = 0; i < P; ++i) cdf[i] = a.cd[sys * 8 + i];
    int* jlog = s.jl + (long long)sys * s.kcap;
    for (int base = 0; base < K; base += 32) {
      const int t = base + lane;
      const int j = t < K ? lj[t] : -2;
      if (t < K) jlog[t] = j;
      const unsigned def = __ballot_sync(FULL, j == -1);
      len += __popc(__ballot_sync(FULL, j >= 0));
      if (j == -1) dlog[nd + __popc(def & ((1u << lane) - 1u))] = make_int2((int)cond_node(a, t, att), t % rows);
      nd += __popc(def);
#pragma unroll
      for (int i = 0; i < P; ++i) cdf[i] += __popc(__ballot_sync(FULL, j == i));
    }
    if (lane == 0) {
      s.ndef_try[sys] = nd;
      s.len_try[sys] = len;
#pragma unroll
      for (int i = 0; i < P; ++i) s.cd_try[sys * 8 + i] = cdf[i];
    }
  }
  // multipliers for the basis replay: mu_i = phi_i c (mu_j = 0)
  cplx* mulog = s.mu + (long long)sys * s.kcap * P;
  for (int e = tid; e < K * P; e += blockDim.x) {
    const int t = e / P, i = e - t * P;
    const int j = lj[t];
    mulog[e] = (j < 0 || i == j) ? cmk(0.0, 0.0) : mu_prod<P>(lf[e], lci[t]);
  }
}

// ------------------------------------------------------------ basis kernel
// One absorbed step on a basis row held as c[d][i] = B[k][i][32 d + lane],
// straight-line over NB blocks (column J is zero beyond them).  Blocks run
// high to low so that block d-1 is still unmodified when block d shifts.
template <int P, int DB, int NB, int J>
TR_D void basis_step(cplx (&c)[DB][P], const cplx (&mu)[P], cplx msig, int lane) {
#pragma unroll
  for (int d = NB - 1; d >= 0; --d) {
    const cplx oj = c[d][J];
    const cplx ojm = d > 0 ? c[d - 1][J] : cmk(0.0, 0.0);
    cplx up = shfl_c(lane == 31 ? ojm : oj, (lane + 31) & 31);
    if (d == 0) up = lane == 0 ? cmk(0.0, 0.0) : up;
#pragma unroll
    for (int i = 0; i < P; ++i)
      if (i != J) c[d][i] = cfma(mu[i], oj, c[d][i]);
    c[d][J] = cfma(msig, oj, up);
  }
}

// the same step with a run-time pivot: selects instead of a dispatch
template <int P, int DB, int NB>
TR_D void basis_step_sel(cplx (&c)[DB][P], int j, const cplx (&mu)[P], cplx msig, int lane) {
  cplx m[P];
#pragma unroll
  for (int i = 0; i < P; ++i) m[i] = (i == j) ? msig : mu[i];
  cplx oj[NB];
#pragma unroll
  for (int d = 0; d < NB; ++d) oj[d] = sel<P>(c[d], j);
#pragma unroll
  for (int d = NB - 1; d >= 0; --d) {
    const cplx ojm = d > 0 ? oj[d - 1] : cmk(0.0, 0.0);
    cplx up = shfl_c(lane == 31 ? ojm : oj[d], (lane + 31) & 31);
    if (d == 0) up = lane == 0 ? cmk(0.0, 0.0) : up;
#pragma unroll
    for (int i = 0; i < P; ++i) c[d][i] = cfma(m[i], oj[d], (i == j) ? up : c[d][i]);
  }
}

template <int P, int DB, int NB>
TR_D void basis_step_j(cplx (&c)[DB][P], int j, const cplx (&mu)[P], cplx msig, int lane) {
  if (j == 0) basis_step<P, DB, NB, 0>(c, mu, msig, lane);
  else if (j == 1) basis_step<P, DB, NB, 1>(c, mu, msig, lane);
  else if (j == 2) basis_step<P, DB, NB, 2>(c, mu, msig, lane);
  else if (j == 3) basis_step<P, DB, NB, 3>(c, mu, msig, lane);
  else if constexpr (P == 5) {
    basis_step<P, DB, NB, 4>(c, mu, msig, lane);
  } else {
    if (j == 4) basis_step<P, DB, NB, 4>(c, mu, msig, lane);
    else if (j == 5) basis_step<P, DB, NB, 5>(c, mu, msig, lane);
    else basis_step<P, DB, NB, 6>(c, mu, msig, lane);
  }
}

struct RowState {
  int dmax;   // structural degree of the row (max over its entries)
  bool big;   // a coefficient passed the rescale trigger at a check point
};

// Steps t.. while the row fits in NB blocks; returns the first step that
// needs more (or K).  deg[i] = structural degree of B[k][i] (-1: zero).
template <int P, int DB, int NB>
TR_D int run_steps(cplx (&c)[DB][P], int (&deg)[P], RowState& st, int t, int K, const int* jsm,
                   const cplx* musm, const cplx* sgsm, int lane) {
  for (; t < K; ++t) {
    const int j = jsm[t];
    cplx mu[P];
#pragma unroll
    for (int i = 0; i < P; ++i) mu[i] = musm[t * P + i];
    const cplx msig = cneg(sgsm[t]);
    if (j >= 0) {
      const int dj = sel_i<P>(deg, j);
      if (dj >= 0) {  // else column j of this row is zero: the step is a no-op here
        const int nd = max(st.dmax, dj + 1);
        if (nd / 32 + 1 > NB) return t;
#pragma unroll
        for (int i = 0; i < P; ++i) deg[i] = (i == j) ? dj + 1 : max(deg[i], dj);
        st.dmax = nd;
        basis_step_j<P, DB, NB>(c, j, mu, msig, lane);
      }
    }
    if (((t + 1) % RESCALE_PERIOD) == 0) {
      // the reference rescales when a coefficient passes the trigger here
      bool b = false;
#pragma unroll
      for (int d = 0; d < NB; ++d)
#pragma unroll
        for (int i = 0; i < P; ++i) b |= cabs2(c[d][i]) > RESCALE_TRIGGER * RESCALE_TRIGGER;
      st.big |= b;
    }
  }
  return t;
}

template <int P, int DB>
TR_D void build_row(cplx (&c)[DB][P], int k, RowState& st, int K, const int* jsm, const cplx* musm,
                    const cplx* sgsm, int lane) {
  int deg[P];
#pragma unroll
  for (int i = 0; i < P; ++i) deg[i] = i == k ? 0 : -1;
  st.dmax = 0;
  st.big = false;
  int t = 0;
  while (t < K) {
    int need = st.dmax / 32 + 1;
    const int j = jsm[t];
    if (j >= 0) {
      const int dj = sel_i<P>(deg, j);
      if (dj >= 0) need = max(need, (dj + 1) / 32 + 1);
    }
#define TR_RUN(NB) \
  case NB: if constexpr (NB <= DB) t = run_steps<P, DB, NB>(c, deg, st, t, K, jsm, musm, sgsm, lane); break;
    if (need > DB) {  // the basis outgrew the planned register blocks
      st.big = true;    // -> exact coupled kernel
      break;
    }
    switch (need) {
      TR_RUN(1) TR_RUN(2) TR_RUN(3) TR_RUN(4) TR_RUN(5) TR_RUN(6) TR_RUN(7) TR_RUN(8) TR_RUN(9)
      default: t = K; break;
    }
#undef TR_RUN
  }
}

struct BasisSmem {
  static size_t bytes(int K, int P, int M, int DB) {
    return sizeof(cplx) * ((size_t)K * P + K + M + 32 * (size_t)DB + 2 * (size_t)P * P * M) +
           sizeof(int) * (size_t)K;
  }
  // + the normalised basis staged for the self-check fold
  static size_t staged(int P, int DB) { return sizeof(cplx) * (size_t)P * P * 32 * DB; }
};

// Column normalisation, basis write-out, self-check and best-attempt
// bookkeeping of one attempt (ref tanint.py:179-183, :262-270, :395-434).
// Warp `row >= 0` holds basis row `row` in c; every thread of the CTA calls.
template <int P, int DB>
TR_D void finish_attempt(const LeafArgs& a, const SplitState& s, int round, int sys, cplx (&c)[DB][P], int row,
                         int stage, cplx* wtab, cplx* twl, cplx* gbuf, cplx* vbuf, cplx* cbuf,
                         double (*red)[8], double* csafe, double* wred, int* sviol, int nw) {
  constexpr int CAPR = 32 * DB;
  constexpr int PP = P * P;
  const int K = a.K, M = a.M, rows = a.rows, cap = a.cap;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nt = blockDim.x;
  if (row >= 0) {
    // column maxima of this row
#pragma unroll
    for (int i = 0; i < P; ++i) {
      double m = 0.0;
#pragma unroll
      for (int d = 0; d < DB; ++d) m = fmax(m, cabs2(c[d][i]));
      m = wmax(m);
      if (lane == 0) red[row][i] = m;
    }
  }
  __syncthreads();
  if (tid < P) {
    double m = 0.0;
    for (int k = 0; k < P; ++k) m = fmax(m, red[k][tid]);
    m = sqrt(m);
    csafe[tid] = m > 0.0 ? m : 1.0;
  }
  __syncthreads();
  // normalise and write the attempt's basis
  cplx* dst = (round == 0 ? a.out : a.scratch) + (long long)sys * a.out_sys;
  if (row >= 0) {
    const int k = row;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const double inv = 1.0 / csafe[i];
#pragma unroll
      for (int d = 0; d < DB; ++d) {
        const int l = 32 * d + lane;
        const cplx v = cscale(c[d][i], inv);
        if (l < cap) dst[(long long)(k * P + i) * cap + l] = v;
        if (stage) cbuf[(k * P + i) * CAPR + l] = v;
      }
    }
  }
  if (cap > CAPR) {
    const int tail = cap - CAPR;
    for (int e = tid; e < PP * tail; e += nt) dst[(long long)(e / tail) * cap + CAPR + e % tail] = cmk(0.0, 0.0);
  }

  // ---- self-residual: fold + M-point DFT, all warps ----
  const cplx* W = a.W + (long long)sys * a.w_sys;
  const long long rowstride = (long long)rows * P;
  double sc = 0.0;
  for (int e = tid; e < K * P; e += nt) {
    const int pos = e / (rows * P), rem = e % (rows * P);
    sc = fmax(sc, cabs2(W[node_of(a, pos) * rowstride + rem]));
  }
  sc = wmax(sc);
  if (lane == 0) wred[warp] = sc;
  // coefficients past the register blocks are zero (an overflow went to the
  // exact kernel), so the staged fold stops at CAPR
  const int len = min(min(s.len_try[sys], cap), stage ? CAPR : cap);
  double resm = 0.0;
  for (int cs = 0; cs < a.noff; ++cs) {
    const long long oc = cs ? a.o1 : a.o0;
    for (int l = tid; l < len; l += nt) twl[l] = __ldg(&a.twN[(oc * l) % a.N]);
    __syncthreads();  // also orders the basis writes above before the reads below
    for (int e = tid; e < PP * M; e += nt) {
      const int pq = e / M, q = e % M;
      const cplx* src = stage ? cbuf + (size_t)pq * CAPR : dst + (long long)pq * cap;
      cplx a0 = cmk(0.0, 0.0), a1 = cmk(0.0, 0.0);
      int l = q;
      for (; l + M < len; l += 2 * M) {
        a0 = cfma(src[l], twl[l], a0);
        a1 = cfma(src[l + M], twl[l + M], a1);
      }
      if (l < len) a0 = cfma(src[l], twl[l], a0);
      gbuf[e] = cadd(a0, a1);
    }
    __syncthreads();
    for (int e = tid; e < P * M; e += nt) {
      const int k = e / M, t = e % M;
      const cplx* g = gbuf + (size_t)k * P * M;
      cplx acc[P];
#pragma unroll
      for (int i = 0; i < P; ++i) acc[i] = cmk(0.0, 0.0);
      int kk = 0;
      for (int q = 0; q < M; ++q) {
        const cplx w = wtab[kk];
#pragma unroll
        for (int i = 0; i < P; ++i) acc[i] = cfma(g[i * M + q], w, acc[i]);
        kk += t;
        if (kk >= M) kk -= M;
      }
#pragma unroll
      for (int i = 0; i < P; ++i) vbuf[(k * P + i) * M + t] = acc[i];
    }
    __syncthreads();
    for (int e = tid; e < M * rows * P; e += nt) {
      const int tt = e / (rows * P), rem = e % (rows * P);
      const int rr = rem / P, jj = rem % P;
      const cplx* wrow = W + (oc + a.stride * (long long)tt) * rowstride + rr * P;
      cplx acc = cmk(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < P; ++i) acc = cfma(wrow[i], vbuf[(i * P + jj) * M + tt], acc);
      resm = fmax(resm, cabs2(acc));
    }
    __syncthreads();
  }
  double scale = 0.0;
  for (int w = 0; w < nw; ++w) scale = fmax(scale, wred[w]);
  scale = sqrt(scale);
  __syncthreads();
  resm = wmax(resm);
  if (lane == 0) wred[warp] = resm;
  __syncthreads();
  double res = 0.0;
  for (int w = 0; w < nw; ++w) res = fmax(res, wred[w]);
  res = (scale == 0.0) ? 0.0 : sqrt(res) / scale;

  // ---- best attempt, retry or commit ----
  double factor = 1.0;
  for (int i = 0; i < P; ++i) factor = fmax(factor, csafe[i]);
  const bool better = round == 0 || res < s.res_best[sys];
  const int nd = s.ndef_try[sys];
  if (better) {
    if (round > 0) {
      cplx* o = a.out + (long long)sys * a.out_sys;
      for (long long e = tid; e < (long long)PP * cap; e += nt) o[e] = dst[e];
    }
    int2* db = s.def_best + (long long)sys * s.kcap;
    const int2* dt = s.def_try + (long long)sys * s.kcap;
    for (int e = tid; e < nd; e += nt) db[e] = dt[e];
  }
  __syncthreads();
  if (tid == 0) {
    const int viol = *sviol;
    s.viol[sys] = viol;
    if (better) {
      s.res_best[sys] = res;
      s.ndef_best[sys] = nd;
      s.factor_best[sys] = factor;
      s.len_best[sys] = s.len_try[sys];
      for (int i = 0; i < P; ++i) s.cd_best[sys * 8 + i] = s.cd_try[sys * 8 + i];
    }
    const bool done = s.res_best[sys] <= a.check_tol || round + 1 >= a.nattempts;
    if (viol) {
      s.need[sys] = SPLIT_EXACT;  // speculation failed: exact coupled kernel
      *s.any_viol = 1;
    } else if (!done) {
      s.need[sys] = round + 1;    // retry with the next absorption order
    } else {
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

template <int P, int DB>
__global__ void __launch_bounds__(NT, (DB <= 3 ? 2 : 1)) leaf_basis_kernel(LeafArgs a, SplitState s, int round,
                                                                           int stage) {
  const int sys = blockIdx.x;
  if (s.need[sys] != round) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int tid = threadIdx.x, lane = tid & 31;
  const int warp = __shfl_sync(FULL, tid >> 5, 0);  // warp-uniform for ptxas (no collective shuffles)
  TR_BTRACE(0);
  constexpr int CAPR = 32 * DB;
  const int K = a.K, M = a.M, rows = a.rows, cap = a.cap;
  constexpr int PP = P * P;
  cplx* musm = reinterpret_cast<cplx*>(smem_raw);  // [K][P]
  cplx* sgsm = musm + (size_t)K * P;               // [K]
  cplx* wtab = sgsm + K;                           // [M] exp(2 pi i q / M)
  cplx* twl = wtab + M;                            // [CAPR] coset twist w_N^(o l)
  cplx* gbuf = twl + CAPR;                         // [P*P][M] folded coefficients
  cplx* vbuf = gbuf + (size_t)PP * M;              // [P*P][M] basis at one coset
  int* jsm = reinterpret_cast<int*>(vbuf + (size_t)PP * M);  // [K]
  // [P*P][CAPR] normalised basis (when staged), 16-byte aligned after jsm
  cplx* cbuf = reinterpret_cast<cplx*>(smem_raw + (((size_t)((unsigned char*)(jsm + K) - smem_raw) + 15) & ~(size_t)15));
  __shared__ double red[8][8];
  __shared__ double csafe[8];
  __shared__ double wred[NW];
  __shared__ int sviol;
  const int att = round;

  {
    const cplx* mulog = s.mu + (long long)sys * s.kcap * P;
    const int* jlog = s.jl + (long long)sys * s.kcap;
    for (int e = tid; e < K; e += NT) {
      jsm[e] = jlog[e];
      sgsm[e] = __ldg(&a.twN[cond_node(a, e, att)]);
    }
    for (int e = tid; e < K * P; e += NT) musm[e] = mulog[e];
    for (int e = tid; e < M; e += NT) wtab[e] = __ldg(&a.twN[(long long)e * a.stride]);
    if (tid == 0) sviol = 0;
  }
  __syncthreads();
  TR_BTRACE(1);

  // ---- replay: warp k builds row k of the basis ----
  cplx c[DB][P];
#pragma unroll
  for (int d = 0; d < DB; ++d)
#pragma unroll
    for (int i = 0; i < P; ++i) c[d][i] = cmk(0.0, 0.0);
  if (warp < P) {
    const int k = warp;
#pragma unroll
    for (int i = 0; i < P; ++i)
      if (i == k && lane == 0) c[0][i] = cmk(1.0, 0.0);
    RowState st;
    build_row<P, DB>(c, k, st, K, jsm, musm, sgsm, lane);
    TR_BTRACE(2);
    if (__any_sync(FULL, st.big) && lane == 0) sviol = 1;
  }
  finish_attempt<P, DB>(a, s, round, sys, c, warp < P ? warp : -1, stage, wtab, twl, gbuf, vbuf, cbuf, red,
                        csafe, wred, &sviol, NW);
}

// ------------------------------------ fused attempts, lane-resident front
// One CTA per system runs every attempt of the leaf: the chain of
// leaf_chain3_kernel (decider warp 0 alone on its scheduler, holders of the
// later blocks), plus P basis-row warps that replay the published steps from
// the log as fast as they can (acquire polling, never on the decider's
// critical path), then the normalisation / self-check of finish_attempt; a
// retry (ref tanint.py:395-434) loops inside the kernel, so a leaf is one
// launch.  Warps != 0 mod 4 carry holders (slots 1..H-1) and basis rows
// (slots H..H+P-1).
template <int P, int DB, int NB>
TR_D int poll_steps(cplx (&c)[DB][P], int (&deg)[P], RowState& st, int t, int& avail, int K, const int* lj,
                    const cplx* lf, const cplx* lci, const cplx* lsig, const int* flag, const cplx* lmu,
                    int lane) {
  for (; t < K; ++t) {
    avail = wait_steps(flag, t, avail);
    const int j = lj[t];
    if (j >= 0) {
      const int dj = sel_i<P>(deg, j);
      if (dj >= 0) {
        const int nd = max(st.dmax, dj + 1);
        if (nd / 32 + 1 > NB) return t;
#pragma unroll
        for (int i = 0; i < P; ++i) deg[i] = (i == j) ? dj + 1 : max(deg[i], dj);
        st.dmax = nd;
        cplx mu[P];
        if (lmu) {  // published by the mu warp (the same products)
#pragma unroll
          for (int i = 0; i < P; ++i) mu[i] = lmu[t * P + i];
        } else {
          const cplx ci = lci[t];
#pragma unroll
          for (int i = 0; i < P; ++i) mu[i] = mu_prod<P>(lf[t * P + i], ci);
        }
        basis_step_j<P, DB, NB>(c, j, mu, cneg(lsig[t]), lane);
      }
    }
    if (((t + 1) % RESCALE_PERIOD) == 0) {
      bool b = false;
#pragma unroll
      for (int d = 0; d < NB; ++d)
#pragma unroll
        for (int i = 0; i < P; ++i) b |= cabs2(c[d][i]) > RESCALE_TRIGGER * RESCALE_TRIGGER;
      st.big |= b;
    }
  }
  return t;
}

// Shared memory of leaf_fused3_kernel: the leaf's weights (natural node
// order, loaded once for every attempt and the self-check), the step log,
// the check buffers and the attempt bookkeeping.
struct Fused3Smem {
  static size_t bytes(int K, int P, int M, int DB) {
    const size_t capr = 32 * (size_t)DB;
    return sizeof(cplx) * ((size_t)K * P /*wl*/ + (size_t)K * P /*lf*/ + 2 * (size_t)K /*lci, lsig*/ +
                           32 * (size_t)P /*xfer*/ + M /*wtab*/ + 2 * capr /*twl x2*/ +
                           2 * (size_t)P * P * M /*gbuf, vbuf*/ + (size_t)P * P * capr /*cbuf*/ +
                           (size_t)K * P /*lmu*/) +
           sizeof(int2) * 2 * (size_t)K /*dtry, dbest*/ + sizeof(int) * ((size_t)K + 4);
  }
};

struct F3Book {  // attempt bookkeeping (ref tanint.py:395-434)
  double res_try, factor_try, res_best, factor_best, scale;
  int nd_try, len_try, viol_try, nd_best, len_best, next;
  int cd_try[8], cd_best[8];
};

// The reference's retry rule applied to one more finished attempt `c`
// (rounds are considered in order): returns bit0 = c becomes the best,
// bit1 = done, bit2 = rescale speculation failed (exact kernel).
TR_D int f3_pick(F3Book& bk, const F3Book& c, int round, int P, int nattempts, double tol) {
  if (c.viol_try) return 4;
  const bool better = round == 0 || c.res_try < bk.res_best;
  if (better) {
    bk.res_best = c.res_try;
    bk.nd_best = c.nd_try;
    bk.factor_best = c.factor_try;
    bk.len_best = c.len_try;
    for (int i = 0; i < P; ++i) bk.cd_best[i] = c.cd_try[i];
  }
  const bool done = bk.res_best <= tol || round + 1 >= nattempts;
  return (better ? 1 : 0) | (done ? 2 : 0);
}

template <int P, int DB, int NTH, bool CL>
__global__ void __launch_bounds__(NTH, 1) leaf_fused3_kernel(LeafArgs a, SplitState s) {
  // CL: a cluster of two CTAs per system runs attempts 0 and 1 side by side
  const int rank = CL ? (int)cooperative_groups::this_cluster().block_rank() : 0;
  const int sys = CL ? blockIdx.x >> 1 : blockIdx.x;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  constexpr int CAPR = 32 * DB;
  constexpr int PP = P * P;
  const int K = a.K, rows = a.rows, M = a.M, cap = a.cap;
  const int RP = rows * P;
  cplx* wl = reinterpret_cast<cplx*>(smem_raw);    // [noff][M][rows][P] leaf weights
  cplx* lf = wl + (size_t)K * P;                   // [K][P] decided rows
  cplx* lci = lf + (size_t)K * P;                  // [K]
  cplx* lsig = lci + K;                            // [K]
  cplx* xfer = lsig + K;                           // [32][P]
  cplx* wtab = xfer + 32 * P;                      // [M]
  cplx* twl = wtab + M;                            // [2][CAPR] coset twists
  cplx* gbuf = twl + 2 * CAPR;                     // [P*P][M]
  cplx* vbuf = gbuf + (size_t)PP * M;              // [P*P][M]
  cplx* cbuf = vbuf + (size_t)PP * M;              // [P*P][CAPR] normalised basis
  cplx* lmu = cbuf + (size_t)PP * CAPR;            // [K][P] multipliers mu_i = f_i c_i (the mu warp)
  int2* dtry = reinterpret_cast<int2*>(lmu + (size_t)K * P);  // [K]
  int2* dbest = dtry + K;                          // [K]
  int* lj = reinterpret_cast<int*>(dbest + K);     // [K]
  int* flag = lj + K;  // [0] published steps, [1] blocks handed over, [2] steps whose multipliers are in lmu
  __shared__ double red[8][8];
  __shared__ double csafe[8];
  __shared__ double wred[16];
  __shared__ F3Book bk;
  __shared__ long long tsm[32];  // clock stamps of system 0 (tr_debug_chain_trace)
  __shared__ int cd0[8];         // column degrees entering the leaf
  const int tid = threadIdx.x, lane = tid & 31, nt = blockDim.x;
  const int warp = __shfl_sync(FULL, tid >> 5, 0);
  const int nw = nt >> 5;
  if (g_chain_trace_on && sys == 0 && rank == 0 && tid == 0) g_chain_trace[3072 + 129] = clock64();  // kernel entry
  const cplx* W = a.W + (long long)sys * a.w_sys;
  const long long rowstride = (long long)RP;
  const int H = (K + 31) / 32;
  // holder warps: blocks 2h-1 and 2h; when the layout leaves a warp unused (P = 5, K = 192:
  // 3 holders + 5 basis rows on 9 warps) the first two blocks -- the ones with the least
  // time to catch up -- get a holder each (TR_EXTRA_HOLDER)
#ifndef TR_EXTRA_HOLDER
#define TR_EXTRA_HOLDER 1
#endif
  const int nslots = a.dense ? nw - 1 : nw - 1 - (nw - 1) / 4;
  const bool extra = P == 5 && TR_EXTRA_HOLDER && !a.dense && H >= 4 && H / 2 + 1 + P <= nslots;
  const int NH = H / 2 + (extra ? 1 : 0);
  // warp roles: the decider alone on its scheduler (warps 4, 8, 12 idle), or -- a.dense,
  // when that would need a 13th warp and with it the 128-register budget of four warps
  // per scheduler -- every warp used (the P = 7 leaves of config 3: 11 instead of 14
  // warps, 168 instead of 128 registers, no 1-2.5 KB of spills per thread)
  const int slot = a.dense ? warp : ((warp & 3) ? warp - warp / 4 : 0);
  const int hold = (slot >= 1 && slot <= NH) ? slot : 0;
  const int brow = (slot > NH && slot <= NH + P) ? slot - NH - 1 : -1;
  // The multipliers mu_i = f_i c_i of a step are the same for every basis row: one warp beside
  // the decider (warp 4, otherwise idle; a few instructions per step, lanes one
  // product each) computes them once and publishes them for the P basis-row warps, which
  // otherwise spend a third to a half of their FP64 work recomputing them -- the consumer
  // schedulers, not the decider, set the pace of the hand-overs (profiles/r2_leaf_decider.txt)
  // (not in the dense layout of the P = 7 leaves: their chain is bound by the decider, measured)
  const bool mu_on = P == 5 && TR_MU_WARP && !a.dense && nw > 4;
  const bool muw = mu_on && warp == 4;
  // blocks held (hb2 < H: two)
  const int hb1 = extra ? (hold <= 2 ? hold : 2 * hold - 3) : 2 * hold - 1;
  const int hb2 = extra ? (hold <= 2 ? H : 2 * hold - 2) : 2 * hold;

  // ---- once per leaf: weights, DFT table, coset twists, weight scale ----
  double sc = 0.0;
  for (int e = tid; e < K * P; e += nt) {
    const int pos = e / RP, rem = e - pos * RP;
    const cplx w = W[node_of(a, pos) * rowstride + rem];
    const int cs = a.noff == 1 ? 0 : (pos & 1), tt = a.noff == 1 ? pos : (pos >> 1);
    wl[(cs * M + tt) * RP + rem] = w;
    sc = fmax(sc, cabs2(w));
  }
  for (int e = tid; e < M; e += nt) wtab[e] = __ldg(&a.twN[(long long)e * a.stride]);
  if (tid < P) cd0[tid] = a.cd[sys * 8 + tid];
  for (int e = tid; e < a.noff * CAPR; e += nt) {
    const int cs = e / CAPR, l = e - cs * CAPR;
    const long long oc = cs ? a.o1 : a.o0;
    twl[e] = __ldg(&a.twN[(oc * l) % a.N]);
  }
  sc = wmax(sc);
  if (lane == 0) wred[warp] = sc;
  __syncthreads();
  if (tid == 0) {
    double m = 0.0;
    for (int w = 0; w < nw; ++w) m = fmax(m, wred[w]);
    bk.scale = sqrt(m);
  }

  int round = rank;
  bool viol = false;
  for (;; ++round) {
    const int att = round;
    cplx r[P], r2[P];
    cplx sg = cmk(0.0, 0.0), sg2 = cmk(0.0, 0.0);
    auto load_row = [&](int m, cplx (&rr)[P], cplx& sgv) {
#pragma unroll
      for (int i = 0; i < P; ++i) rr[i] = cmk(0.0, 0.0);
      if (m < K) {
        const int pidx = perm_of(m / rows, a.ord_stride[att], a.ord_reverse[att], a.count);
        const int cs = a.noff == 1 ? 0 : (pidx & 1), tt = a.noff == 1 ? pidx : (pidx >> 1);
        sgv = __ldg(&a.twN[node_of(a, pidx)]);
        lsig[m] = sgv;
        const cplx* wr = wl + (cs * M + tt) * RP + (m % rows) * P;
#pragma unroll
        for (int i = 0; i < P; ++i) rr[i] = wr[i];
      }
    };
    if (warp == 0) load_row(lane, r, sg);
    if (hold) {
      load_row(32 * hb1 + lane, r, sg);
      if (hb2 < H) load_row(32 * hb2 + lane, r2, sg2);
    }
    if (tid < 3) flag[tid] = 0;
    if (tid == 0) bk.viol_try = 0;
    cplx c[DB][P];  // basis row (basis warps only; set in their branch)
    RowState st;
    st.dmax = 0;
    st.big = false;
    __syncthreads();

    if (warp == 0) {
      // ---------------- decider (as leaf_chain3_kernel) ----------------
      const double thr2 = a.thr * a.thr;
      int cd[P];
#pragma unroll
      for (int i = 0; i < P; ++i) cd[i] = cd0[i];
      int nabs = 0, ndef = 0;  // absorbed / deferred conditions (the chain epilogue, kept on the fly)
      unsigned a_lf = 0, a_lci = 0, a_lj = 0, a_flag = 0;
      if constexpr (P != 7) a_lf = smem_u32(lf), a_lci = smem_u32(lci), a_lj = smem_u32(lj), a_flag = smem_u32(flag);
      const int pub = lane == 0;
      for (int b = 0; b < H; ++b) {
        if (b > 0) {
          long long tw0 = 0;
          if constexpr (P == 5) tw0 = clock64();
          while (ld_acquire(&flag[1]) < b) {
          }
          if constexpr (P == 5)
            if (lane == 0 && b < 8) tsm[24 + b] = clock64() - tw0;  // hand-over wait of block b
#pragma unroll
          for (int i = 0; i < P; ++i) r[i] = xfer[lane * P + i];
          sg = lsig[min(32 * b + lane, K - 1)];
        }
        if (lane == 0 && b < 12) tsm[b] = clock64();
        const int tend = min(K, 32 * b + 32);
        for (int t = 32 * b; t < tend; ++t) {
          const int src = t & 31;
          cplx f[P];
#pragma unroll
          for (int i = 0; i < P; ++i) f[i] = shfl_c(r[i], src);
          const cplx sf = lsig[t];
          cplx fj;
          double a2j;
          const int j = decide_bits<P>(f, cd, thr2, fj, a2j);
          const double inv2 = rcp_nr(a2j);
          const cplx ci = cmk(-fj.x * inv2, fj.y * inv2);
          if constexpr (P == 7) {
            // (the general variant's decider is register-bound: four hoisted addresses cost it
            // spills, config 3 leaf time 399 -> 407 ms; it keeps the lane-0 block)
            if (lane == 0) {
              lj[t] = j;
              lci[t] = ci;
#pragma unroll
              for (int i = 0; i < P; ++i) lf[t * P + i] = f[i];
              st_release(&flag[0], t + 1);
            }
          } else {
            const unsigned plf = a_lf + (unsigned)t * (P * 16u);
            sts_i_if(pub, a_lj + 4u * (unsigned)t, j);
            sts_c_if(pub, a_lci + 16u * (unsigned)t, ci);
#pragma unroll
            for (int i = 0; i < P; ++i) sts_c_if(pub, plf + 16u * i, f[i]);
            st_release_if(pub, a_flag, t + 1);
          }
          // P = 7: pivot-specialised row update (j is warp-uniform), no select chains over
          // seven columns -- 1239 -> 1125 ns per condition at config 3; P = 5 is faster
          // with the selects (534 vs 545 ns: the switch costs the later phases registers)
          auto upd = [&](auto JC) {
            constexpr int J = decltype(JC)::value;
            const cplx rj = r[J];
            const cplx c2 = cmul(ci, rj);
            const cplx nj = cmul(rj, csub(sg, sf));
#pragma unroll
            for (int i = 0; i < P; ++i)
              if (i != J) r[i] = cfma(f[i], c2, r[i]);
            r[J] = nj;
            cd[J] += 1;
          };
          if constexpr (P == 7) {
          switch (j) {
            case 0: upd(std::integral_constant<int, 0>()); break;
            case 1: upd(std::integral_constant<int, 1>()); break;
            case 2: upd(std::integral_constant<int, 2>()); break;
            case 3: upd(std::integral_constant<int, 3>()); break;
            case 4: upd(std::integral_constant<int, 4>()); break;
            case 5: if constexpr (P > 5) upd(std::integral_constant<int, 5>()); break;
            case 6: if constexpr (P > 6) upd(std::integral_constant<int, 6>()); break;
            default: break;
          }
          } else {
          if (j >= 0) {
            const cplx rj = sel<P>(r, j);
            const cplx c2 = cmul(ci, rj);
            const cplx nj = cmul(rj, csub(sg, sf));
#pragma unroll
            for (int i = 0; i < P; ++i) {
              const cplx v = cfma(f[i], c2, r[i]);
              r[i] = (i == j) ? nj : v;
            }
          }
#pragma unroll
          for (int i = 0; i < P; ++i) cd[i] += (i == j);
          }
          nabs += j >= 0;
          if (j == -1) {  // deferred, in step order (ref tanint.py:200-206)
            if (lane == 0) dtry[ndef] = make_int2((int)cond_node(a, t, att), t % rows);
            ++ndef;
          }
        }
      }
      if (lane == 0) {
        bk.nd_try = ndef;
        bk.len_try = 1 + nabs;
#pragma unroll
        for (int i = 0; i < P; ++i) bk.cd_try[i] = cd[i];
      }
      if (lane == 0) tsm[12] = clock64();
    } else if (hold) {
      // ---------------- holder of blocks hb1, hb2: steps < 32 hb ----------------
      auto step_row = [&](int t, int j, cplx (&rr)[P], cplx sgv) {
        const cplx rj = sel<P>(rr, j);
        const cplx c2 = cmul(lci[t], rj);
        const cplx nj = cmul(rj, csub(sgv, lsig[t]));
#pragma unroll
        for (int i = 0; i < P; ++i) {
          const cplx v = cfma(lf[t * P + i], c2, rr[i]);
          rr[i] = (i == j) ? nj : v;
        }
      };
      auto hand_over = [&](int b, const cplx (&rr)[P]) {
        while (ld_acquire(&flag[1]) < b - 1) if (TR_SPIN_NS > 0) __nanosleep(TR_SPIN_NS);
#pragma unroll
        for (int i = 0; i < P; ++i) xfer[lane * P + i] = rr[i];
        __syncwarp();
        if (lane == 0) st_release(&flag[1], b);
      };
      const bool two = hb2 < H;
      int avail = 0, t = 0;
      for (; t < 32 * hb1; ++t) {
        avail = wait_steps(&flag[0], t, avail);
        const int j = lj[t];
        if (j >= 0) {
          step_row(t, j, r, sg);
          if (two) step_row(t, j, r2, sg2);
        }
      }
      hand_over(hb1, r);
      if (two) {
        for (; t < 32 * hb2; ++t) {
          avail = wait_steps(&flag[0], t, avail);
          const int j = lj[t];
          if (j >= 0) step_row(t, j, r2, sg2);
        }
        hand_over(hb2, r2);
      }
    } else if (muw) {
      // ---------------- multipliers of the published steps ----------------
      int done = 0, avail = 0;
      while (done < K) {
        avail = wait_steps(&flag[0], done, avail);
        for (int e = done * P + lane; e < avail * P; e += 32) lmu[e] = mu_prod<P>(lf[e], lci[e / P]);
        __syncwarp();
        if (lane == 0) st_release(&flag[2], avail);
        done = avail;
      }
    } else if (brow >= 0) {
      // ---------------- basis row brow: replay published steps ----------------
      const int* bflag = mu_on ? &flag[2] : &flag[0];
      const cplx* bmu = mu_on ? lmu : nullptr;
      int deg[P];
#pragma unroll
      for (int d = 0; d < DB; ++d)
#pragma unroll
        for (int i = 0; i < P; ++i) c[d][i] = cmk(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < P; ++i) deg[i] = i == brow ? 0 : -1;
#pragma unroll
      for (int i = 0; i < P; ++i)
        if (i == brow && lane == 0) c[0][i] = cmk(1.0, 0.0);
      int tb = 0, avail = 0;
      while (tb < K) {
        int need = st.dmax / 32 + 1;
        avail = wait_steps(bflag, tb, avail);
        const int j = lj[tb];
        if (j >= 0) {
          const int dj = sel_i<P>(deg, j);
          if (dj >= 0) need = max(need, (dj + 1) / 32 + 1);
        }
        if (need > DB) {  // outgrew the register blocks: exact kernel
          st.big = true;
          break;
        }
#define TR_RUN3(NB) \
  case NB: if constexpr (NB <= DB) tb = poll_steps<P, DB, NB>(c, deg, st, tb, avail, K, lj, lf, lci, lsig, bflag, bmu, lane); break;
        switch (need) {
          TR_RUN3(1) TR_RUN3(2) TR_RUN3(3) TR_RUN3(4) TR_RUN3(5) TR_RUN3(6) TR_RUN3(7)
          default: tb = K; break;
        }
#undef TR_RUN3
      }
      // column maxima of this row (ref tanint.py:179-183)
#pragma unroll
      for (int i = 0; i < P; ++i) {
        double m = 0.0;
#pragma unroll
        for (int d = 0; d < DB; ++d) m = fmax(m, cabs2(c[d][i]));
        m = wmax(m);
        if (lane == 0) red[brow][i] = m;
      }
      if (__any_sync(FULL, st.big) && lane == 0) bk.viol_try = 1;
    }
    __syncthreads();
    if (tid == 0) tsm[13] = clock64();
    // ---- column scales (the chain epilogue was kept by the decider) ----
    if (tid < 32 + P && tid >= 32) {
      const int i = tid - 32;
      double m = 0.0;
      for (int k = 0; k < P; ++k) m = fmax(m, red[k][i]);
      m = sqrt(m);
      csafe[i] = m > 0.0 ? m : 1.0;
    }
    __syncthreads();
    if (tid == 0) tsm[22] = clock64();
    // ---- normalise and write the attempt's basis (round 0: out, else scratch) ----
    cplx* dst = (round == 0 ? a.out : a.scratch) + (long long)sys * a.out_sys;
    if (brow >= 0) {
      const int k = brow;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const double inv = 1.0 / csafe[i];
#pragma unroll
        for (int d = 0; d < DB; ++d) {
          const int l = 32 * d + lane;
          const cplx v = cscale(c[d][i], inv);
          if (l < cap) dst[(long long)(k * P + i) * cap + l] = v;
          cbuf[(k * P + i) * CAPR + l] = v;
        }
      }
    }
    if (tid == 0) tsm[23] = clock64();
    if (cap > CAPR) {
      const int tail = cap - CAPR;
      for (int e = tid; e < PP * tail; e += nt) dst[(long long)(e / tail) * cap + CAPR + e % tail] = cmk(0.0, 0.0);
    }
    __syncthreads();
    if (tid == 0) tsm[14] = clock64();
    // ---- self-residual (ref tanint.py:262-270): fold + M-point DFT per coset ----
    const int len = min(min(bk.len_try, cap), CAPR);
    double resm = 0.0;
    int M1 = 1;  // DFT factor M = M1 * M2 (M1 <= M2; 1: direct sums)
    if (M > 12)
      for (int d = 2; d * d <= M; ++d)
        if (M % d == 0) M1 = d;
    const int M2 = M / M1;
    for (int cs = 0; cs < a.noff; ++cs) {
      const cplx* tw = twl + cs * CAPR;
      for (int e = tid; e < PP * M; e += nt) {
        const int pq = e / M, q = e % M;
        const cplx* src = cbuf + (size_t)pq * CAPR;
        cplx a0 = cmk(0.0, 0.0), a1 = cmk(0.0, 0.0);
        int l = q;
        for (; l + M < len; l += 2 * M) {
          a0 = cfma(src[l], tw[l], a0);
          a1 = cfma(src[l + M], tw[l + M], a1);
        }
        if (l < len) a0 = cfma(src[l], tw[l], a0);
        gbuf[e] = cadd(a0, a1);
      }
      __syncthreads();
      if (tid == 0) tsm[16 + 3 * cs] = clock64();
      // M-point DFT of every folded entry (omega^e = wtab[e mod M]).  The
      // check is FP64-throughput-bound, so M = M1 * M2 runs as two passes
      // of M1- and M2-term sums (Cooley-Tukey, twiddle folded into the first
      // pass): P^2 M (M1 + M2) instead of P^2 M^2 complex FMAs.  Node powers
      // run as recurrences re-anchored from the table every 16 terms.
      const cplx* X = vbuf;  // DFT output [P*P][M]
      if (M1 > 1) {
        for (int e = tid; e < P * M; e += nt) {
          const int k = e / M, r = e % M;
          const int n2 = r / M1, k1 = r - n2 * M1;
          const cplx* g = gbuf + (size_t)k * P * M + n2;
          const int st = M2 * k1;  // < M
          const cplx ws = wtab[st];
          int kk = n2 * k1;        // exponent of w (< M)
          cplx w = wtab[kk];
          cplx acc[P];
#pragma unroll
          for (int i = 0; i < P; ++i) acc[i] = cmk(0.0, 0.0);
          for (int n1 = 0; n1 < M1; ++n1) {
            if (n1 && (n1 & 15) == 0) w = wtab[kk];
#pragma unroll
            for (int i = 0; i < P; ++i) acc[i] = cfma(g[i * M + M2 * n1], w, acc[i]);
            w = cmul(w, ws);
            kk += st;
            if (kk >= M) kk -= M;
          }
#pragma unroll
          for (int i = 0; i < P; ++i) vbuf[(k * P + i) * M + r] = acc[i];
        }
        __syncthreads();
        for (int e = tid; e < P * M; e += nt) {
          const int k = e / M, t = e % M;
          const int k2 = t / M1, k1 = t - k2 * M1;
          const cplx* y = vbuf + (size_t)k * P * M + k1;
          const int st = M1 * k2;  // < M
          const cplx ws = wtab[st];
          int kk = 0;
          cplx w = cmk(1.0, 0.0);
          cplx acc[P];
#pragma unroll
          for (int i = 0; i < P; ++i) acc[i] = cmk(0.0, 0.0);
          for (int n2 = 0; n2 < M2; ++n2) {
            if (n2 && (n2 & 15) == 0) w = wtab[kk];
#pragma unroll
            for (int i = 0; i < P; ++i) acc[i] = cfma(y[i * M + n2 * M1], w, acc[i]);
            w = cmul(w, ws);
            kk += st;
            if (kk >= M) kk -= M;
          }
#pragma unroll
          for (int i = 0; i < P; ++i) gbuf[(k * P + i) * M + t] = acc[i];
        }
        X = gbuf;
      } else {
        for (int e = tid; e < P * M; e += nt) {
          const int k = e / M, t = e % M;
          const cplx* g = gbuf + (size_t)k * P * M;
          const cplx wt = wtab[t];
          cplx acc[P];
#pragma unroll
          for (int i = 0; i < P; ++i) acc[i] = cmk(0.0, 0.0);
          cplx w = cmk(1.0, 0.0);
          int kk = 0;
          for (int q = 0; q < M; ++q) {
            if ((q & 15) == 0) w = wtab[kk];
#pragma unroll
            for (int i = 0; i < P; ++i) acc[i] = cfma(g[i * M + q], w, acc[i]);
            w = cmul(w, wt);
            kk += t;
            if (kk >= M) kk -= M;
          }
#pragma unroll
          for (int i = 0; i < P; ++i) vbuf[(k * P + i) * M + t] = acc[i];
        }
      }
      __syncthreads();
      if (tid == 0) tsm[17 + 3 * cs] = clock64();
      for (int e = tid; e < M * RP; e += nt) {
        const int tt = e / RP, rem = e % RP;
        const int rr = rem / P, jj = rem % P;
        const cplx* wrow = wl + (cs * M + tt) * RP + rr * P;
        cplx acc = cmk(0.0, 0.0);
#pragma unroll
        for (int i = 0; i < P; ++i) acc = cfma(wrow[i], X[(i * P + jj) * M + tt], acc);
        resm = fmax(resm, cabs2(acc));
      }
      __syncthreads();
      if (tid == 0) tsm[18 + 3 * cs] = clock64();
    }
    resm = wmax(resm);
    if (lane == 0) wred[warp] = resm;
    __syncthreads();
    if (tid == 0) {
      tsm[15] = clock64();
      if (g_chain_trace_on && sys == 0 && round < 4)
        for (int e = 0; e < 32; ++e) g_chain_trace[3072 + 32 * round + e] = tsm[e];
    }
    // ---- best attempt, retry or commit ----
    if (tid == 0) {
      double rm = 0.0;
      for (int w = 0; w < nw; ++w) rm = fmax(rm, wred[w]);
      bk.res_try = (bk.scale == 0.0) ? 0.0 : sqrt(rm) / bk.scale;
      double factor = 1.0;
      for (int i = 0; i < P; ++i) factor = fmax(factor, csafe[i]);
      bk.factor_try = factor;
    }
    if constexpr (CL) {
      if (round < 2) {
        // attempts 0 and 1 finished side by side: rank 0 applies the retry
        // rule to both in order (the partner's book and deferrals via DSMEM)
        cooperative_groups::cluster_group cl = cooperative_groups::this_cluster();
        cl.sync();
        F3Book* pb = cl.map_shared_rank(&bk, 1);
        int2* pd = cl.map_shared_rank(dtry, 1);
        if (rank == 0) {
          if (tid == 0) {
            int nx = f3_pick(bk, bk, 0, P, a.nattempts, a.check_tol);
            if (!(nx & 6)) {
              const int n1 = f3_pick(bk, *pb, 1, P, a.nattempts, a.check_tol);
              nx = (nx & 1) | (n1 << 3);  // bits 3..5: attempt 1's verdict
            }
            bk.next = nx;
          }
          __syncthreads();
          const int nx = bk.next;
          const int n1 = nx >> 3;
          if ((nx & 1) && !(n1 & 1)) {
            for (int e = tid; e < bk.nd_try; e += nt) dbest[e] = dtry[e];
          }
          if (n1 & 1) {
            const int nd = pb->nd_try;
            for (int e = tid; e < nd; e += nt) dbest[e] = pd[e];
            cplx* o = a.out + (long long)sys * a.out_sys;
            const cplx* sd = a.scratch + (long long)sys * a.out_sys;
            for (long long e = tid; e < (long long)PP * cap; e += nt) o[e] = sd[e];
          }
        }
        cl.sync();  // the partner's shared memory is no longer read
        if (rank == 1) return;
        const int nx = bk.next;
        const int n1 = nx >> 3;
        if ((nx & 4) || (n1 & 4)) {
          viol = true;
          break;
        }
        if ((nx & 2) || (n1 & 2)) break;
        round = 1;  // continue with attempt 2
        __syncthreads();
        continue;
      }
    }
    if (tid == 0) bk.next = f3_pick(bk, bk, round, P, a.nattempts, a.check_tol);
    __syncthreads();
    const int nx = bk.next;
    if (nx & 4) {
      viol = true;
      break;
    }
    if (nx & 1) {
      const int nd = bk.nd_try;
      for (int e = tid; e < nd; e += nt) dbest[e] = dtry[e];
      if (round > 0) {
        cplx* o = a.out + (long long)sys * a.out_sys;
        for (long long e = tid; e < (long long)PP * cap; e += nt) o[e] = dst[e];
      }
    }
    if (nx & 2) break;
    __syncthreads();
  }
  __syncthreads();
  if (g_chain_trace_on && sys == 0 && tid == 0) g_chain_trace[3072 + 128] = clock64();
  // ---- commit (ref tanint.py:430-434) or hand the leaf to the exact kernel ----
  if (viol || (a.force_viol && sys == 0)) {
    if (tid == 0) {
      s.viol[sys] = 1;
      s.need[sys] = SPLIT_EXACT;
      *s.any_viol = 1;
    }
    return;
  }
  const int base = a.dcount[sys];
  const int nb = bk.nd_best;
  const int room = a.dmax - base;
  const int nput = nb < room ? nb : room;
  for (int e = tid; e < nput; e += nt) a.defer[(long long)sys * a.dmax + base + e] = dbest[e];
  if (tid < P) a.cd[sys * 8 + tid] = bk.cd_best[tid];
  if (tid == 0) {
    s.viol[sys] = 0;
    a.dcount[sys] = base + nb;
    if (nb > room) a.status[sys] = 5;
    a.max_scale[sys] = fmax(a.max_scale[sys], bk.factor_best);
    if (round > 0) a.retried[sys] += 1;
    if (a.res_out) a.res_out[sys] = bk.res_best;
    if (a.len_out) a.len_out[sys] = bk.len_best;
    s.need[sys] = SPLIT_DONE;
  }
}

__global__ void fast_need_reset_kernel(int* need, int nsys) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nsys) need[i] = 0;
}

int blocks_for(const LeafArgs& a) { return (a.K + 1 + 31) / 32; }
constexpr int DB5 = 9, DB7 = 7;  // register blocks: K + 1 <= 288 (P = 5), 224 (P = 7)
// blocks for this leaf: the planned structural degree plus slack (a leaf that
// outgrows them is redone by the exact kernel), at most what K allows
int blocks_planned(const LeafArgs& a) {
  const int full = blocks_for(a);
  if (a.dbound <= 0) return full;
  const int b = (a.dbound + 8) / 32 + 1;
  return b < full ? b : full;
}

template <int P, int DB>
int launch_basis(const LeafArgs& a, const SplitState& s, int round, int nsys, cudaStream_t st) {
  size_t smem = BasisSmem::bytes(a.K, P, a.M, DB);
  // stage the basis in shared memory for the check when it still fits the
  // kernel's CTAs per SM
  const size_t limit = DB <= 3 ? 110 * 1024 : 220 * 1024;
  const size_t with = ((smem + 15) & ~(size_t)15) + BasisSmem::staged(P, DB);
  const int stage = with <= limit ? 1 : 0;
  if (stage) smem = with;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(leaf_basis_kernel<P, DB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    set = true;
  }
  TrKTimer _kt(TRK_LEAF_BUILD, st);
  leaf_basis_kernel<P, DB><<<nsys, NT, smem, st>>>(a, s, round, stage);
  return 0;
}

template <int P>
int dispatch_basis(const LeafArgs& a, const SplitState& s, int round, int nsys, cudaStream_t st) {
  switch (blocks_planned(a)) {
    case 1: return launch_basis<P, 1>(a, s, round, nsys, st);
    case 2: return launch_basis<P, 2>(a, s, round, nsys, st);
    case 3: return launch_basis<P, 3>(a, s, round, nsys, st);
    case 4: return launch_basis<P, 4>(a, s, round, nsys, st);
    case 5: return launch_basis<P, 5>(a, s, round, nsys, st);
    case 6: return launch_basis<P, 6>(a, s, round, nsys, st);
    case 7: return launch_basis<P, 7>(a, s, round, nsys, st);
    case 8: if constexpr (P == 5) return launch_basis<P, 8>(a, s, round, nsys, st); else return -1;
    case 9: if constexpr (P == 5) return launch_basis<P, 9>(a, s, round, nsys, st); else return -1;
    default: return -1;
  }
}

}  // namespace

bool leaf_fast_supported(const LeafArgs& a) {
  if (a.P != 5 && a.P != 7) return false;
  if (a.K < 2 || a.K > NT) return false;
  const int db = blocks_planned(a);
  if (db > (a.P == 5 ? DB5 : DB7)) return false;
  return BasisSmem::bytes(a.K, a.P, a.M, db) <= 220 * 1024;
}

template <int P, int DB, int NTH, bool CL>
int launch_f3(const LeafArgs& a, const SplitState& s, int nsys, int nw, size_t fs, cudaStream_t st) {
  static int max_threads = -1;
  if (max_threads < 0) {
    cudaFuncSetAttribute(leaf_fused3_kernel<P, DB, NTH, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncAttributes fa;
    TR_CUDA_CHECK(cudaFuncGetAttributes(&fa, leaf_fused3_kernel<P, DB, NTH, CL>));
    max_threads = fa.maxThreadsPerBlock;
    if (getenv("TR_DEBUG"))
      fprintf(stderr, "fused3<%d,%d,%d,%d>: regs %d max threads %d\n", P, DB, NTH, (int)CL, fa.numRegs,
              fa.maxThreadsPerBlock);
  }
  if (32 * nw > max_threads) return -1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(CL ? 2 * nsys : nsys));
  cfg.blockDim = dim3(32 * nw);
  cfg.dynamicSmemBytes = fs;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = CL ? 1 : 0;
  TR_CUDA_CHECK(cudaLaunchKernelEx(&cfg, leaf_fused3_kernel<P, DB, NTH, CL>, a, s));
  return 0;
}

// fused attempts with the lane-resident chain (leaf_fused3_kernel): one
// launch per leaf; returns -1 when the shape does not fit it
int launch_fused3(const LeafArgs& a, const SplitState& s, int nsys, cudaStream_t st) {
  if (nsys > 148) return -1;
  const int H = (a.K + 31) / 32;
  const int last = H / 2 + a.P;  // highest slot: H/2 holders, then the basis rows
  int nw = 1;
  while (nw - 1 - (nw - 1) / 4 < last) ++nw;
  LeafArgs ad = a;
  ad.dense = 0;
  if (nw > 12 && last + 1 <= 12) {  // every warp used: stays within three warps per scheduler
    nw = last + 1;
    ad.dense = 1;
  }
  if (nw > 16) return -1;
  const int db = blocks_planned(a);
  if (db > (a.P == 5 ? 4 : 3)) return -1;
  const size_t fs = Fused3Smem::bytes(a.K, a.P, a.M, db);
  if (fs > 200 * 1024) return -1;
  {
    const double K = a.K, P = a.P;
    tr_kernel_work(TRK_LEAF_PIVOT, 16.0 * nsys * K * P, 4.0 * nsys * P * K * (K - 1));
    tr_kernel_work(TRK_LEAF_BUILD, 16.0 * nsys * (P * P * (K + 1) + K * P),
                   4.0 * nsys * P * P * K * (K + 1) + 8.0 * nsys * (double)a.noff * P * P * a.M * a.M);
  }
  // attempts 0 and 1 side by side (2-CTA clusters) while the batch leaves
  // SMs idle: the retry tail of a leaf then costs no extra chain time
  const bool cl = a.nattempts > 1 && 2 * nsys <= 148;
  int rc = 0;
  TrKTimer _kt(TRK_LEAF_PIVOT, st);
#define TR_F3N(PP_, DB_, NTH_)                                                                             \
  {                                                                                                        \
    if (cl) rc = launch_f3<PP_, DB_, NTH_, true>(ad, s, nsys, nw, fs, st);                                 \
    else rc = launch_f3<PP_, DB_, NTH_, false>(ad, s, nsys, nw, fs, st);                                   \
  }
#define TR_F3L(PP_, DB_)                  \
  if (nw <= 12) TR_F3N(PP_, DB_, 384)     \
  else TR_F3N(PP_, DB_, 512)
  if (a.P == 5) {
    switch (db) {
      case 1: TR_F3L(5, 1) break;
      case 2: TR_F3L(5, 2) break;
      case 3: TR_F3L(5, 3) break;
      default: TR_F3L(5, 4) break;
    }
  } else {
    switch (db) {
      case 1: TR_F3L(7, 1) break;
      case 2: TR_F3L(7, 2) break;
      default: TR_F3L(7, 3) break;
    }
  }
#undef TR_F3L
#undef TR_F3N
  if (rc) return rc;  // -1: does not fit, the caller falls back
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int leaf_fast_launch(const LeafArgs& a, const SplitState& s, int nsys, cudaStream_t st) {
  {
    const int rc = launch_fused3(a, s, nsys, st);
    if (rc >= 0) return rc;
  }
  {
    TrKTimer _kt(TRK_LEAF_PIVOT, st);
    fast_need_reset_kernel<<<(nsys + 255) / 256, 256, 0, st>>>(s.need, nsys);
  }
  {  // algorithmic work of one attempt (retry rounds are extra work, not counted)
    const double K = a.K, P = a.P;
    tr_kernel_work(TRK_LEAF_PIVOT, 16.0 * nsys * K * P, 4.0 * nsys * P * K * (K - 1));
    tr_kernel_work(TRK_LEAF_BUILD, 16.0 * nsys * (P * P * (K + 1) + K * P),
                   4.0 * nsys * P * P * K * (K + 1) + 8.0 * nsys * (double)a.noff * P * P * a.M * a.M);
  }
  const size_t csm2 = sizeof(cplx) * ((size_t)a.K * a.P + 2 * a.K + 2 + 2 * a.P) + sizeof(int) * a.K;
  const int hk = (a.K + 31) / 32;  // holder warps
  // one CTA per SM when the batch fits the GPU: holders off the decider's
  // scheduler; otherwise the compact layout, two CTAs per SM
  const bool spread = nsys <= 148;
  const int nth2 = 32 * (1 + hk + (spread ? (hk - 1) / 3 : 0));
  for (int round = 0; round < a.nattempts; ++round) {
    {
      TrKTimer _kt(TRK_LEAF_PIVOT, st);
      if (a.P == 5) {
        if (spread) leaf_chain2_kernel<5, true><<<nsys, nth2, csm2, st>>>(a, s, round);
        else leaf_chain2_kernel<5, false><<<nsys, nth2, csm2, st>>>(a, s, round);
      } else {
        if (spread) leaf_chain2_kernel<7, true><<<nsys, nth2, csm2, st>>>(a, s, round);
        else leaf_chain2_kernel<7, false><<<nsys, nth2, csm2, st>>>(a, s, round);
      }
    }
    const int rc = a.P == 5 ? dispatch_basis<5>(a, s, round, nsys, st)
                            : dispatch_basis<7>(a, s, round, nsys, st);
    if (rc) {
      tr_set_error("leaf shape unsupported (K=%d, P=%d)", a.K, a.P);
      return 2;
    }
  }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}
