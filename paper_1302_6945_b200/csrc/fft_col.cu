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
template <int LOG2, int Q, bool PASSA, int S, int TLX = 0>
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
          cplx x = stg ? stg[e * G::TL + (int)(threadIdx.x % G::TL)]
                       : (gi < a.in_len ? a.in[lbase_in + gi] : cmk(0.0, 0.0));
          if constexpr (PASSA) {
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
    col_stage<LOG2, Q, PASSA, S + 1, TLX>(sm, a, lbase_in, lbase_out, s, live, tb, mrow, nullptr);
  }
}

template <int LOG2, int Q, bool PASSA>
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
  col_stage<LOG2, Q, PASSA, 0>(tile + (size_t)sl * G::LS, a, lin, lout, s0 + sl, live, tb, mrow);
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

template <int LOG2, int Q, bool PASSA>
int launch(const ColArgs& a, cudaStream_t st) {
  if constexpr ((Q << LOG2) > 1024 || (Q << LOG2) < 2) {
    return -1;
  } else {
    using G = CPlan<LOG2, Q>;
    if (a.subs % G::TL) return -1;
    const size_t smem = sizeof(cplx) * (size_t)G::TL * G::LS;
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(fft_col_kernel<LOG2, Q, PASSA>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           100 * 1024);
      set = true;
    }
    const long long blocks = a.lines * a.subs / G::TL;
    TrKTimer _kt(TRK_FFT, st);
    fft_col_kernel<LOG2, Q, PASSA><<<(unsigned)blocks, NTH, smem, st>>>(a);
    return 0;
  }
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
