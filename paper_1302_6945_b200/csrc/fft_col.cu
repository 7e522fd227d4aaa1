// Two-pass batched FFT for n = N1 N2 > 4096 (N1, N2 <= 1024).
//
//   X[k1 + N1 k2] = sum_n2 W_N2^(n2 k2) W_N^(n2 k1) sum_n1 x[N2 n1 + n2] W_N1^(n1 k1)
//
// pass A: for every n2, the length-N1 transform of x[N2 n1 + n2] (n1 < N1),
//         written as Y[n2 N1 + k1] (each transform's outputs contiguous);
// pass B: for every k1, the length-N2 transform of Y[n2 N1 + k1] W_N^(n2 k1),
//         written to X[k1 + N1 k2].
// A CTA owns TL consecutive sub-transforms and maps consecutive threads to
// consecutive sub-transforms, so every strided element access of a pass is a
// contiguous run of TL values across a warp (coalesced).  Pass A's outputs
// go out through a shared-memory transpose (runs of N1 values).  Inside a
// CTA the radix-16 register Stockham stages of fft_reg.cu run on a
// [TL][R + 1] shared tile (odd row pitch: conflict-free across lanes).
#include <stdlib.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <utility>
#include <string.h>
#include <cooperative_groups.h>

#include "fft.cuh"
#include "fft_bfly.cuh"
#include "fft_fast.cuh"

#ifndef FFT_COL_MINB
#define FFT_COL_MINB 2  // resident CTAs per SM the register budget is sized for (3: spills, measured slower)
#endif

namespace {

constexpr int NTH = 256;

__host__ __device__ constexpr int ilog2c(int x) {
  int l = 0;
  while ((1 << l) < x) ++l;
  return l;
}

template <int LOG2, int Q, int TLX = 0>
struct CPlan {
  static constexpr int R = Q << LOG2;
  static constexpr int N16 = LOG2 / 4;
  static constexpr int REM = 1 << (LOG2 % 4);
  static constexpr int NODD = Q == 1 ? 0 : Q == 15 ? 2 : 1;
  static constexpr int NST = N16 + (REM > 1 ? 1 : 0) + NODD;
  TR_HD static constexpr int radix(int s) {
    return s < N16 ? 16
         : (REM > 1 && s == N16) ? REM
         : (Q == 15) ? (s == NST - 2 ? 3 : 5)
         : Q;
  }
  TR_HD static constexpr int ns(int s) {
    int p = 1;
    for (int i = 0; i < s; ++i) p *= radix(i);
    return p;
  }
  static constexpr int TLc = 4096 / (1 << ilog2c(R));
  static constexpr int TL = TLX ? TLX : (TLc > 16 ? 16 : (TLc < 4 ? 4 : TLc));  // sub-transforms per CTA
  static constexpr int T = NTH / TL;                               // threads per sub-transform
  static constexpr int LS = R + 1;                                 // odd pitch
};

template <int RS>
TR_D void tw_apply(cplx (&v)[RS], const cplx* twR, int k, int step, int sign) {
#pragma unroll
  for (int u = 1; u < RS; ++u) {
    cplx w = __ldg(&twR[u * k * step]);
    if (sign < 0) w.y = -w.y;
    v[u] = cmul(v[u], w);
  }
}

// element e of sub-transform s of line: in[line*in_ls + s + e*in_es]
template <int LOG2, int Q, bool PASSA, int S, int TLX = 0, bool LDCG = false, bool M2 = false>
TR_D void col_stage(cplx* sm, const ColArgs& a, long long lbase_in, long long lbase_out, int s, bool live,
                    int tb, const cplx* mrow, const cplx* stg = nullptr) {
  using G = CPlan<LOG2, Q, TLX>;
  constexpr int R = G::R, r = G::radix(S), NS = G::ns(S), B = R / r, T = G::T;
  constexpr int IT = (B + T - 1) / T;
  constexpr bool FIRST = S == 0, LAST = S == G::NST - 1;
  const int sign = a.sign;
  cplx v[IT][r];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int b = tb + it * T;
    if ((B % T == 0 || b < B) && live) {
#pragma unroll
      for (int u = 0; u < r; ++u) {
        const int e = b + u * B;
        if constexpr (FIRST) {
          const long long gi = s + (long long)e * a.in_es;
          // staged tile ([e][TL], zero filled past in_len) or straight from HBM
          cplx x;
          if constexpr (LDCG) {
            // written by other CTAs of the cluster just before: L2 only
            x = __ldcg(&a.in[lbase_in + gi]);
          } else {
            x = stg ? stg[e * G::TL + (int)(threadIdx.x % G::TL)]
                    : (gi < a.in_len ? a.in[lbase_in + gi] : cmk(0.0, 0.0));
          }
          if constexpr (PASSA && M2) {
            // x m + conj(x[-gi]) m2 (full-length lines; no run-time branch, so
            // the unrolled loads of all elements still issue together)
            const long long nn = (long long)R * a.subs;
            const cplx xm = cconj(a.in[lbase_in + (gi ? nn - gi : 0)]);
            const cplx m2 = a.mul2[(mrow - a.mul) + gi];
            x = cscale(cfma(xm, m2, cmul(x, mrow[gi])), a.mul_scale);
          } else if constexpr (PASSA) {
            if (mrow) x = cmul(x, cscale(mrow[gi], a.mul_scale));
          }
          if constexpr (!PASSA) {
            // W_N^(n2 k1) = W_N^(n2 k1h TL) W_N^(n2 k1l), k1 = s = s0 + sl: the first
            // factor is warp-uniform (broadcast), the second a coalesced [N2][TL] row
            const int sl = s % G::TL;
            cplx w1 = __ldg(&a.twN[(long long)e * (s - sl)]);
            cplx w2 = __ldg(&a.tw2[e * G::TL + sl]);
            cplx w = cmul(w1, w2);
            if (sign < 0) w.y = -w.y;
            x = cmul(x, w);
          }
          v[it][u] = x;
        } else {
          v[it][u] = sm[e];
        }
      }
      if constexpr (NS > 1) tw_apply<r>(v[it], a.twR, b % NS, R / (NS * r), sign);
      bfly_any<r>(v[it], sign);
    }
  }
  if constexpr (!FIRST) __syncthreads();
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int b = tb + it * T;
    if ((B % T == 0 || b < B) && live) {
      const int k = b % NS;
      const int base = (b / NS) * NS * r + k;
#pragma unroll
      for (int u = 0; u < r; ++u) {
        const int o = base + u * NS;
        if constexpr (LAST && !PASSA) {
          a.out[lbase_out + s + (long long)o * a.out_es] = v[it][u];
        } else {
          sm[o] = v[it][u];
        }
      }
    }
  }
  if constexpr (!LAST) {
    __syncthreads();
    col_stage<LOG2, Q, PASSA, S + 1, TLX, LDCG, M2>(sm, a, lbase_in, lbase_out, s, live, tb, mrow, nullptr);
  }
}

template <int LOG2, int Q, bool PASSA, bool M2 = false>
__global__ void __launch_bounds__(NTH, FFT_COL_MINB) fft_col_kernel(ColArgs a) {
  using G = CPlan<LOG2, Q>;
  extern __shared__ __align__(16) unsigned char fsm[];
  cplx* tile = reinterpret_cast<cplx*>(fsm);
  const int sl = threadIdx.x % G::TL, tb = threadIdx.x / G::TL;
  const long long sub0 = (long long)blockIdx.x * G::TL;  // TL divides subs
  const long long line = sub0 / a.subs;
  const int s0 = (int)(sub0 - line * a.subs);
  const bool live = line < a.lines;
  const long long lin = line * a.in_ls, lout = line * a.out_ls;
  const cplx* mrow = (PASSA && a.mul) ? a.mul + line * a.mul_ls : nullptr;
  col_stage<LOG2, Q, PASSA, 0, 0, false, M2>(tile + (size_t)sl * G::LS, a, lin, lout, s0 + sl, live, tb, mrow);
  if constexpr (PASSA) {
    // outputs of each sub-transform are contiguous: Y[s R + k]
    __syncthreads();
    if (live) {
      for (int e = threadIdx.x; e < G::TL * G::R; e += NTH) {
        const int t = e / G::R, k = e - t * G::R;
        a.out[lout + (long long)(s0 + t) * G::R + k] = tile[(size_t)t * G::LS + k];
      }
    }
  }
}

template <int LOG2, int Q, bool PASSA, bool M2 = false>
int launch(const ColArgs& a, cudaStream_t st) {
  if constexpr ((Q << LOG2) > 1024 || (Q << LOG2) < 2) {
    return -1;
  } else {
    using G = CPlan<LOG2, Q>;
    if (a.subs % G::TL) return -1;
    if constexpr (PASSA && !M2) {
      if (a.mul2) return launch<LOG2, Q, PASSA, true>(a, st);
    }
    if (M2 && !a.mul) return -1;
    const size_t smem = sizeof(cplx) * (size_t)G::TL * G::LS;
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(fft_col_kernel<LOG2, Q, PASSA, M2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           100 * 1024);
      set = true;
    }
    const long long blocks = a.lines * a.subs / G::TL;
    TrKTimer _kt(TRK_FFT, st);
    fft_col_kernel<LOG2, Q, PASSA, M2><<<(unsigned)blocks, NTH, smem, st>>>(a);
    return 0;
  }
}


// ------------------------------------------------ both passes in one launch
// A cluster of C CTAs owns one line at a time (persistent: cluster c takes
// lines c, c + #clusters, ...).  Its CTAs share the line's pass-A tiles, meet at
// a cluster barrier (release / acquire: pass A's global stores are visible to
// the cluster), then share the pass-B tiles.  The intermediate Y lives in one
// scratch slot per cluster (#clusters * n values, a few tens of MB): it is
// rewritten for every line, so it stays dirty in L2 and HBM sees one read and
// one write per element; the whole transform is one launch whose clusters
// drift out of phase, so loads, butterflies and stores of different lines
// overlap (the chunked two-launch plan runs every CTA in lockstep, 1-2 waves
// per launch).
TR_D void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
TR_D unsigned cluster_rank() { unsigned r; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r)); return r; }
TR_D unsigned cluster_size() { unsigned r; asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r)); return r; }
TR_D unsigned cluster_id() { unsigned r; asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r)); return r; }
TR_D unsigned cluster_count() { unsigned r; asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r)); return r; }

// Free scratch slots as S mailboxes (0 = empty, else slot + 1) with ticket
// counters: a cluster takes ticket t = head++ and empties mailbox t % S
// (waiting while it is empty), and returns its slot with ticket u = tail++
// into mailbox u % S (waiting while it is full).  With at most S clusters
// between take and return, every wait is on a cluster that is already running,
// and after a launch all S slots are back in the mailboxes: the state carries
// over from launch to launch without a reset.
struct Col2Ring {
  unsigned long long head, tail;
  unsigned box[80];
};
constexpr int ring_slots(int C) { return C == 4 ? 76 : 38; }  // >= resident clusters of size C on 148 SMs

template <int LA, int LB, int QB>
__global__ void __launch_bounds__(NTH, FFT_COL_MINB) fft_col2_kernel(ColArgs a, ColArgs b, Col2Ring* ring, int S) {
  using GA = CPlan<LA, 1>;
  using GB = CPlan<LB, QB>;
  extern __shared__ __align__(16) unsigned char fsm[];
  __shared__ int s_slot;
  cplx* tile = reinterpret_cast<cplx*>(fsm);
  const int rank = (int)cluster_rank(), C = (int)cluster_size();
  const long long cid = cluster_id(), ncl = cluster_count();
  const int sla = threadIdx.x % GA::TL, tba = threadIdx.x / GA::TL;
  const int slb = threadIdx.x % GB::TL, tbb = threadIdx.x / GB::TL;
  const int tiles_a = a.subs / GA::TL, tiles_b = b.subs / GB::TL;
  long long slot_id = cid;
  if (ring) {  // more clusters than slots: take a free one
    if (rank == 0 && threadIdx.x == 0) {
      const unsigned long long t = atomicAdd(&ring->head, 1ULL);
      unsigned* box = &ring->box[t % (unsigned)S];
      unsigned v;
      while ((v = atomicExch(box, 0u)) == 0u) __nanosleep(200);
      __threadfence();
      s_slot = (int)v - 1;
    }
    cluster_sync_all();
    slot_id = *cooperative_groups::this_cluster().map_shared_rank(&s_slot, 0);
  }
  const long long slot = slot_id * a.out_ls;  // scratch slot of this cluster (out_ls = n)
  for (long long line = cid; line < a.lines; line += ncl) {
    const long long lin = line * a.in_ls;
    const cplx* mrow = a.mul ? a.mul + line * a.mul_ls : nullptr;
    for (int t = rank; t < tiles_a; t += C) {
      const int s0 = t * GA::TL;
      col_stage<LA, 1, true, 0>(tile + (size_t)sla * GA::LS, a, lin, slot, s0 + sla, true, tba, mrow);
      __syncthreads();
      for (int e = threadIdx.x; e < GA::TL * GA::R; e += NTH) {
        const int u = e / GA::R, k = e - u * GA::R;
        a.out[slot + (long long)(s0 + u) * GA::R + k] = tile[(size_t)u * GA::LS + k];
      }
      __syncthreads();
    }
    cluster_sync_all();
    const long long lout = line * b.out_ls;
    for (int t = rank; t < tiles_b; t += C) {
      const int s0 = t * GB::TL;
      col_stage<LB, QB, false, 0, 0, true>(tile + (size_t)slb * GB::LS, b, slot, lout, s0 + slb, true, tbb, nullptr);
      __syncthreads();
    }
    if (ring || line + ncl < a.lines) cluster_sync_all();  // the slot is rewritten by the next pass A
  }
  if (ring && rank == 0 && threadIdx.x == 0) {
    __threadfence();
    const unsigned long long u = atomicAdd(&ring->tail, 1ULL);
    unsigned* box = &ring->box[u % (unsigned)S];
    while (atomicCAS(box, 0u, (unsigned)slot_id + 1u) != 0u) __nanosleep(200);
  }
}

// mailbox state per (scratch buffer, cluster size), created on first use
Col2Ring* ring_for(const void* scratch, int C, cudaStream_t st) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, Col2Ring*> rings;
  std::lock_guard<std::mutex> lk(mu);
  auto key = std::make_pair(scratch, C);
  auto it = rings.find(key);
  if (it != rings.end()) return it->second;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  Col2Ring h;
  memset(&h, 0, sizeof h);
  const int S = ring_slots(C);
  h.head = 0;
  h.tail = (unsigned long long)S;
  for (int i = 0; i < S; ++i) h.box[i] = (unsigned)i + 1u;
  Col2Ring* d = nullptr;
  if (cudaMalloc(&d, sizeof h) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, &h, sizeof h, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  rings[key] = d;
  return d;
}

// TR_FFT_C2 = 0: off (default), 1: one cluster per line (scratch slots from the mailboxes), 2: persistent clusters
int col2_mode() {
  static const int m = [] {
    const char* e = getenv("TR_FFT_C2");
    return e ? atoi(e) : 0;
  }();
  return m;
}

template <int LA, int LB, int QB>
int launch2(const ColArgs& a, const ColArgs& b, long long n, cudaStream_t st) {
  using GA = CPlan<LA, 1>;
  using GB = CPlan<LB, QB>;
  if (a.subs % GA::TL || b.subs % GB::TL || a.mul2) return -1;
  const size_t sa = sizeof(cplx) * (size_t)GA::TL * GA::LS, sb = sizeof(cplx) * (size_t)GB::TL * GB::LS;
  const size_t smem = sa > sb ? sa : sb;
  auto kern = fft_col2_kernel<LA, LB, QB>;
  // active clusters per cluster size (4, 8), once per instantiation and device
  static int act[2] = {0, 0};
  static bool set = false;
  if (!set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024) != cudaSuccess) return -1;
    for (int i = 0; i < 2; ++i) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 4u << i;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.gridDim = dim3(4u << i);
      cfg.blockDim = dim3(NTH);
      cfg.dynamicSmemBytes = smem;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int nc = 0;
      if (cudaOccupancyMaxActiveClusters(&nc, kern, &cfg) != cudaSuccess) nc = 0;
      act[i] = nc;
    }
    cudaGetLastError();
    set = true;
  }
  // cluster size: 4 for throughput (least barrier wait) when its scratch slots
  // stay L2-sized and there are lines enough to fill the GPU, else 8
  static const long long budget = [] {
    const char* e = getenv("TR_FFT_C2_MB");  // scratch slots of one launch (MB)
    return (long long)((e ? atof(e) : 40.0) * (1 << 20));
  }();
  const long long lb = n * (long long)sizeof(cplx);
  const bool persistent = col2_mode() == 2;
  auto slots = [&](int i) { return persistent ? act[i] : ring_slots(4 << i); };
  int ci = -1;
  static const int force_c = [] {
    const char* e = getenv("TR_FFT_C2_CL");  // 4 / 8: force the cluster size
    return e ? atoi(e) : 0;
  }();
  if (force_c == 4 || force_c == 8) {
    const int i = force_c == 4 ? 0 : 1;
    if (act[i] > 0 && std::min<long long>(slots(i), a.lines) * lb <= budget) ci = i;
  } else {
    // rounds of resident clusters x tiles per CTA and round; ties go to the
    // smaller cluster (fewer CTAs idle at the barriers)
    const int ta = a.subs / GA::TL, tb = b.subs / GB::TL;
    long long best = -1;
    for (int i = 0; i < 2; ++i) {
      const int C = 4 << i;
      if (act[i] <= 0 || std::min<long long>(slots(i), a.lines) * lb > budget) continue;
      const long long rounds = (a.lines + act[i] - 1) / act[i];
      const long long cost = rounds * ((ta + C - 1) / C + (tb + C - 1) / C);
      if (best < 0 || cost < best) {
        best = cost;
        ci = i;
      }
    }
  }
  if (ci < 0) return -1;
  const int C = 4 << ci;
  long long ncl = std::min<long long>(act[ci], a.lines);
  Col2Ring* ring = nullptr;
  int S = 0;
  if (!persistent) {
    ncl = a.lines;
    S = ring_slots(C);
    if (a.lines > S) {
      ring = ring_for(a.out, C, st);
      if (!ring) return -1;
    }
  }
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)C;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.gridDim = dim3((unsigned)(ncl * C));
  cfg.blockDim = dim3(NTH);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  TrKTimer _kt(TRK_FFT, st);
  if (cudaLaunchKernelEx(&cfg, kern, a, b, ring, S) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return 0;
}

}  // namespace

int col_launch(bool pass_a, int log2, int q, const ColArgs& a, cudaStream_t st) {
  if (pass_a) {
    if (q != 1) return -1;
#define TR_LA(L) \
  case L: return launch<L, 1, true>(a, st);
    switch (log2) {
      TR_LA(1) TR_LA(2) TR_LA(3) TR_LA(4) TR_LA(5) TR_LA(6) TR_LA(7) TR_LA(8) TR_LA(9) TR_LA(10)
      default: return -1;
    }
#undef TR_LA
  }
#define TR_L(Q, L) \
  case L: return launch<L, Q, false>(a, st);
#define TR_Q(Q)                                                                            \
  case Q: switch (log2) {                                                                  \
      TR_L(Q, 0) TR_L(Q, 1) TR_L(Q, 2) TR_L(Q, 3) TR_L(Q, 4) TR_L(Q, 5) TR_L(Q, 6) TR_L(Q, 7) \
      TR_L(Q, 8) TR_L(Q, 9) TR_L(Q, 10)                                                     \
      default: return -1;                                                                  \
    }
  switch (q) {
    TR_Q(1) TR_Q(3) TR_Q(5) TR_Q(7) TR_Q(9) TR_Q(15)
    default: return -1;
  }
#undef TR_Q
#undef TR_L
}

// Both passes in one launch (fft_col2_kernel); -1 when the split has no
// instantiation or the scratch slots would outgrow L2 (the caller then runs
// the two launches above).
int col2_launch(int a1, int a2, int q2, const ColArgs& a, const ColArgs& b, long long n, cudaStream_t st) {
#define TR_C2(LA, LB, QB) \
  if (a1 == LA && a2 == LB && q2 == QB) return launch2<LA, LB, QB>(a, b, n, st);
#define TR_C2A(LB, QB) TR_C2(6, LB, QB) TR_C2(7, LB, QB) TR_C2(8, LB, QB)
  TR_C2A(6, 1) TR_C2A(7, 1) TR_C2A(8, 1)
  TR_C2A(5, 3) TR_C2A(6, 3)
  TR_C2A(4, 5) TR_C2A(5, 5)
  TR_C2A(4, 7) TR_C2A(5, 7)
  TR_C2A(4, 9)
  TR_C2A(4, 15)
#undef TR_C2A
#undef TR_C2
  return -1;
}
