// Single-pass batched FFT, register radix-16 Stockham (lengths R = q 2^a <= 4096).
//
// A CTA transforms TL lines with T threads each (T ~ R / 16, TL chosen at
// launch).  Stage s (radix r, Ns = product of the earlier radices, B = R / r
// butterflies) reads its r inputs b + u B, twiddles them by w^(u k) with
// k = b mod Ns, runs the butterfly in registers and writes (b / Ns) Ns r +
// k + u Ns (Stockham autosort: natural order in and out).  Stage 0 reads
// straight from HBM and the last stage writes straight to HBM, both
// coalesced; in between the data sits in shared memory, padded by one value
// per 2^PSH so that the stride-r writes of the first stage are
// conflict-free.  Radix-16 stages first, then the power-of-two remainder,
// then the odd factors: 4096 = 16 16 16 is 3 stages and 2 smem round trips
// (the pass kernels in fft_fast.cu need 4 stages and 5 round trips).
// Twiddles come from the exp(2 pi i m / R) table (0.5 ulp, L1 resident).
#include "fft.cuh"
#include "fft_bfly.cuh"
#include "fft_fast.cuh"

namespace {

constexpr int NTH = 256;

__host__ __device__ constexpr int ilog2c(int x) {
  int l = 0;
  while ((1 << l) < x) ++l;
  return l;
}

// radix plan: 16s, the power-of-two remainder, then the odd factors
template <int LOG2, int Q>
struct Plan {
  static constexpr int R = Q << LOG2;
  static constexpr int N16 = LOG2 / 4;
  static constexpr int REM = 1 << (LOG2 % 4);       // 1, 2, 4, 8
  static constexpr int NODD = Q == 1 ? 0 : Q == 15 ? 2 : 1;
  static constexpr int NST = N16 + (REM > 1 ? 1 : 0) + NODD;
  TR_HD static constexpr int radix(int s) {
    return s < N16 ? 16
         : (REM > 1 && s == N16) ? REM
         : (Q == 15) ? (s == NST - 2 ? 3 : 5)
         : Q;
  }
  TR_HD static constexpr int ns(int s) {  // product of the radices before stage s
    int p = 1;
    for (int i = 0; i < s; ++i) p *= radix(i);
    return p;
  }
  static constexpr int R0 = radix(0);
  // pad one value per 2^PSH (first-stage write stride) when it is a power of two
  static constexpr int PSH = (R0 & (R0 - 1)) == 0 ? ilog2c(R0) : 30;
  static constexpr int Tq = (R + 15) / 16;
  static constexpr int T = Tq >= NTH ? NTH : (1 << ilog2c(Tq));  // threads per line
  static constexpr int TLMAX = NTH / T;                           // lines per CTA (max)
  static constexpr int LS = R + (R >> PSH) + (T < 32 ? 1 : 0);    // smem per line
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

template <int LOG2, int Q, int S, bool TF = false>
TR_D void run_stage(cplx* sm, const FastArgs& a, long long lin, long long lout, bool live, int tb,
                    int sign, const cplx* mrow, long long tf_o = 0) {
  using G = Plan<LOG2, Q>;
  constexpr int R = G::R, r = G::radix(S), NS = G::ns(S), B = R / r, T = G::T;
  constexpr int IT = (B + T - 1) / T;
  constexpr bool FIRST = S == 0, LAST = S == G::NST - 1;
  constexpr int PSH = G::PSH;
  cplx v[IT][r];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int b = tb + it * T;
    if ((B % T == 0 || b < B) && live) {
#pragma unroll
      for (int u = 0; u < r; ++u) {
        const int e = b + u * B;
        if constexpr (FIRST && TF) {
          // (filled below: terms outermost, so the loads of all r values issue together)
        } else if constexpr (FIRST) {
          v[it][u] = e < a.in_len ? a.in[lin + e] : cmk(0.0, 0.0);
          if (mrow) v[it][u] = cmul(v[it][u], cscale(mrow[e], a.mul_scale));
        } else {
          v[it][u] = sm[e + (e >> PSH)];
        }
      }
      if constexpr (FIRST && TF) {
        // twist + fold: x[e] = sum_{l = e mod R, l < L} B[l] w^(o l), the same sums in the
        // same order as twist_fold_kernel (tree.cu)
        const cplx* src = a.tf_B + lin;
        const int N = (int)a.tf_N, L = (int)a.tf_L;
        const int nt = (L + R - 1) / R;
#pragma unroll
        for (int u = 0; u < r; ++u) v[it][u] = cmk(0.0, 0.0);
        if (tf_o == 0) {
          for (int t = 0; t < nt; ++t) {
#pragma unroll
            for (int u = 0; u < r; ++u) {
              const int l = b + u * B + t * R;
              if (l < L) v[it][u] = cadd(v[it][u], src[l]);
            }
          }
        } else {
          const int stepB = (int)((tf_o * B) % N), stepR = (int)((tf_o * R) % N);
          int idx[r];
          idx[0] = (int)((tf_o * b) % N);
#pragma unroll
          for (int u = 1; u < r; ++u) {
            idx[u] = idx[u - 1] + stepB;
            if (idx[u] >= N) idx[u] -= N;
          }
          for (int t = 0; t < nt; ++t) {
#pragma unroll
            for (int u = 0; u < r; ++u) {
              const int l = b + u * B + t * R;
              if (l < L) v[it][u] = cfma(src[l], __ldg(&a.tf_twN[idx[u]]), v[it][u]);
              idx[u] += stepR;
              if (idx[u] >= N) idx[u] -= N;
            }
          }
        }
      }
      if constexpr (NS > 1) tw_apply<r>(v[it], a.twR, b % NS, R / (NS * r), sign);
      bfly_any<r>(v[it], sign);
    }
  }
  if constexpr (!FIRST || LAST) __syncthreads();  // reads done before in-place writes
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    const int b = tb + it * T;
    if ((B % T == 0 || b < B) && live) {
      const int k = b % NS;
      const int base = (b / NS) * NS * r + k;
#pragma unroll
      for (int u = 0; u < r; ++u) {
        const int o = base + u * NS;
        if constexpr (LAST) {
          a.out[lout + o] = v[it][u];
        } else {
          sm[o + (o >> PSH)] = v[it][u];
        }
      }
    }
  }
  if constexpr (!LAST) {
    __syncthreads();
    run_stage<LOG2, Q, S + 1, TF>(sm, a, lin, lout, live, tb, sign, mrow, tf_o);
  }
}

#ifndef FFT_REG_MINB
#define FFT_REG_MINB 2  // resident CTAs per SM the register budget is sized for (3: spills, measured slower)
#endif

// CTA = TL lines x T threads (TL chosen at launch so small batches still
// spread over the SMs)
template <int LOG2, int Q, bool TF = false>
__global__ void __launch_bounds__(NTH, FFT_REG_MINB) fft_reg_kernel(FastArgs a, int TL) {
  using G = Plan<LOG2, Q>;
  extern __shared__ __align__(16) unsigned char fsm[];
  const int sl = threadIdx.x / G::T, tb = threadIdx.x % G::T;
  const long long line = (long long)blockIdx.x * TL + sl;
  const bool live = line < a.nsub;
  cplx* sm = reinterpret_cast<cplx*>(fsm) + (size_t)sl * G::LS;
  if constexpr (TF) {
    // line = (sys * noff + c) * PP + e: basis entry e of system sys, coset c
    const long long sc = line / a.tf_PP;
    const int e = (int)(line - sc * a.tf_PP);
    const long long sys = sc / a.tf_noff;
    const int c = (int)(sc - sys * a.tf_noff);
    run_stage<LOG2, Q, 0, true>(sm, a, sys * a.tf_bsys + (long long)e * a.tf_bcap, line * a.out_ls, live, tb, a.sign,
                                nullptr, c ? a.tf_o1 : a.tf_o0);
  } else {
    const cplx* mrow = a.mul ? a.mul + line * a.mul_ls : nullptr;
    run_stage<LOG2, Q, 0>(sm, a, line * a.in_ls, line * a.out_ls, live, tb, a.sign, mrow);
  }
}

template <int LOG2, int Q, bool TF = false>
int launch(const FastArgs& a, cudaStream_t st) {
  if constexpr ((Q << LOG2) > 4096 || (Q << LOG2) < 2 || (TF && (Q << LOG2) < 128)) {
    return -1;
  } else {
    if constexpr (!TF) {
      if (a.tf_B) return launch<LOG2, Q, true>(a, st);
    }
    using G = Plan<LOG2, Q>;
    // lines per CTA: as many as fit, but keep >= 2 CTAs per SM when the batch allows
    int TL = G::TLMAX;
    const int tlmin = G::T >= 32 ? 1 : 32 / G::T;  // whole warps
    while (TL > tlmin && (a.nsub + TL - 1) / TL < 2 * 148) TL >>= 1;
    const size_t smem = sizeof(cplx) * (size_t)TL * G::LS;
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(fft_reg_kernel<LOG2, Q, TF>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           100 * 1024);
      set = true;
    }
    const long long blocks = (a.nsub + TL - 1) / TL;
    TrKTimer _kt(TRK_FFT, st);
    fft_reg_kernel<LOG2, Q, TF><<<(unsigned)blocks, G::T * TL, smem, st>>>(a, TL);
    return 0;
  }
}

}  // namespace

// single-pass transforms only (J == 1, Ns == 1): nsub = lines
int reg_launch(int log2, int q, const FastArgs& a, cudaStream_t st) {
  if (a.J != 1 || a.Ns != 1) return -1;
#define TR_L(Q, L) \
  case L: return launch<L, Q>(a, st);
#define TR_Q(Q)                                                                   \
  case Q: switch (log2) {                                                         \
      TR_L(Q, 0) TR_L(Q, 1) TR_L(Q, 2) TR_L(Q, 3) TR_L(Q, 4) TR_L(Q, 5) TR_L(Q, 6) \
      TR_L(Q, 7) TR_L(Q, 8) TR_L(Q, 9) TR_L(Q, 10) TR_L(Q, 11) TR_L(Q, 12)         \
      default: return -1;                                                         \
    }
  switch (q) {
    TR_Q(1) TR_Q(3) TR_Q(5) TR_Q(7) TR_Q(9) TR_Q(15)
    default: return -1;
  }
#undef TR_Q
#undef TR_L
}
