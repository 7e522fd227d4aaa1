// Compile-time-shaped Stockham pass kernels for sub-transform lengths
// R = q * 2^a, q in {1, 3, 5, 7, 9, 15}, R <= 4096.  All in-CTA index
// arithmetic uses compile-time divisors; the per-sub-transform global bases
// are computed once per CTA.  Radix stages: the odd factors (3/5/7) first,
// then radix-8 stages and a final 4 or 2.  Lengths with other odd factors use
// the generic kernel in fft.cu.
#include "fft.cuh"
#include "fft_fast.cuh"
#include "fft_bfly.cuh"

namespace {

// large tiles: 256 threads x 16 values; small tiles (single-pass R <= 1024):
// 128 threads x 8 values, so small batches still fill the SMs
constexpr int TILE = 4096;

__host__ __device__ constexpr int np2(int x) {
  int p = 1;
  while (p < x) p <<= 1;
  return p;
}
__host__ __device__ constexpr int nodd(int q) {
  int c = 0;
  while (q % 3 == 0) { q /= 3; ++c; }
  while (q % 5 == 0) { q /= 5; ++c; }
  while (q % 7 == 0) { q /= 7; ++c; }
  return c;
}
__host__ __device__ constexpr int odd_at(int q, int s) {
  int c = 0;
  while (q % 3 == 0) { if (c == s) return 3; q /= 3; ++c; }
  while (q % 5 == 0) { if (c == s) return 5; q /= 5; ++c; }
  while (q % 7 == 0) { if (c == s) return 7; q /= 7; ++c; }
  return 1;
}
__host__ __device__ constexpr int npow2st(int l) { return l / 3 + (l % 3 ? 1 : 0); }
__host__ __device__ constexpr int pow2_at(int l, int s) { return s < l / 3 ? 8 : (l % 3 == 2 ? 4 : 2); }

template <int LOG2, int Q, bool SM>
struct Geo {
  static constexpr int FT = SM ? 128 : 256;
  static constexpr int TV = SM ? 1024 : 4096;
  static constexpr int R = Q << LOG2;
  static constexpr int TL = np2(R) >= TV ? 1 : (TV / np2(R) > 256 ? 256 : TV / np2(R));
  static constexpr int LS = R + (TL > 1 ? 1 : 0);
  static constexpr int NEL = TL * R;
  static constexpr int NODD = nodd(Q);
  static constexpr int NST = NODD + npow2st(LOG2);
  TR_HD static constexpr int radix(int s) { return s < NODD ? odd_at(Q, s) : pow2_at(LOG2, s - NODD); }
};

TR_D cplx twl(const cplx* t, int i, int sign) {
  cplx w = __ldg(&t[i]);
  return sign < 0 ? cconj(w) : w;
}

// one Stockham stage over every staged sub-transform
template <int R, int TL, int LS, int RS, int NSS, int FT>
TR_D void stage(cplx* sm, const cplx* twR, int sign) {
  constexpr int PER = R / RS;
  constexpr int TOT = PER * TL;
  constexpr int IT = (TOT + FT - 1) / FT;
  constexpr int TWS = R / (NSS * RS);
  cplx v[IT][RS];
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    int b = threadIdx.x + it * FT;
    if (TOT % FT == 0 || b < TOT) {
      int sl = b / PER, bb = b % PER;
      int k = bb % NSS;
      const cplx* base = sm + sl * LS + bb;
#pragma unroll
      for (int u = 0; u < RS; ++u) {
        cplx x = base[u * PER];
        if (NSS > 1 && u > 0) x = cmul(x, twl(twR, u * k * TWS, sign));
        v[it][u] = x;
      }
      bfly<RS>(v[it], sign);
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < IT; ++it) {
    int b = threadIdx.x + it * FT;
    if (TOT % FT == 0 || b < TOT) {
      int sl = b / PER, bb = b % PER;
      int k = bb % NSS;
      cplx* base = sm + sl * LS + (bb / NSS) * (NSS * RS) + k;
#pragma unroll
      for (int u = 0; u < RS; ++u) base[u * NSS] = v[it][u];
    }
  }
  __syncthreads();
}

template <int LOG2, int Q, bool SM, int S, int NSS>
TR_D void run_stages(cplx* sm, const cplx* twR, int sign) {
  using G = Geo<LOG2, Q, SM>;
  if constexpr (S < G::NST) {
    constexpr int RS = G::radix(S);
    stage<G::R, G::TL, G::LS, RS, NSS, G::FT>(sm, twR, sign);
    run_stages<LOG2, Q, SM, S + 1, NSS * RS>(sm, twR, sign);
  }
}

template <int LOG2, int Q, bool SM>
__global__ void __launch_bounds__(SM ? 128 : 256) fft_fast_kernel(FastArgs a) {
  using G = Geo<LOG2, Q, SM>;
  constexpr int R = G::R, TL = G::TL, LS = G::LS, NEL = G::NEL, FT = G::FT;
  extern __shared__ __align__(16) unsigned char fsm[];
  cplx* sm = reinterpret_cast<cplx*>(fsm);
  __shared__ long long ib[TL], ob[TL];
  __shared__ int jj[TL], kk[TL];
  const long long s0 = (long long)blockIdx.x * TL;
  for (int t = threadIdx.x; t < TL; t += FT) {
    long long s = s0 + t;
    if (s < a.nsub) {
      long long line = s / a.J;
      int j = (int)(s - line * a.J);
      int k = j & (a.Ns - 1);
      ib[t] = line * a.in_ls + j;
      ob[t] = line * a.out_ls + ((long long)(j >> a.log2Ns) << a.log2Ns) * R + k;
      jj[t] = j;
      kk[t] = k;
    } else {
      ib[t] = -1;
      ob[t] = -1;
      jj[t] = 0;
      kk[t] = 0;
    }
  }
  __syncthreads();
  // ---- load with the inter-pass twiddle ----
  if (a.J >= TL) {
#pragma unroll 4
    for (int e = threadIdx.x; e < NEL; e += FT) {
      int sl = e % TL, r = e / TL;
      cplx x = cmk(0.0, 0.0);
      long long b = ib[sl];
      if (b >= 0) {
        int idx = jj[sl] + r * a.J;
        if (idx < a.in_len) x = a.in[b + (long long)r * a.J];
        if (a.Ns > 1 && r > 0) x = cmul(x, twl(a.twN, r * kk[sl] * a.tws, a.sign));
      }
      sm[sl * LS + r] = x;
    }
  } else {
#pragma unroll 4
    for (int e = threadIdx.x; e < NEL; e += FT) {
      int r = e % R, sl = e / R;
      cplx x = cmk(0.0, 0.0);
      long long b = ib[sl];
      if (b >= 0) {
        int idx = jj[sl] + r * a.J;
        if (idx < a.in_len) x = a.in[b + (long long)r * a.J];
        if (a.Ns > 1 && r > 0) x = cmul(x, twl(a.twN, r * kk[sl] * a.tws, a.sign));
      }
      sm[sl * LS + r] = x;
    }
  }
  __syncthreads();
  run_stages<LOG2, Q, SM, 0, 1>(sm, a.twR, a.sign);
  // ---- store ----
  if (a.Ns == 1) {
#pragma unroll 4
    for (int e = threadIdx.x; e < NEL; e += FT) {
      int q = e % R, sl = e / R;
      long long b = ob[sl];
      if (b >= 0) a.out[b + q] = sm[sl * LS + q];
    }
  } else {
#pragma unroll 4
    for (int e = threadIdx.x; e < NEL; e += FT) {
      int sl = e % TL, q = e / TL;
      long long b = ob[sl];
      if (b >= 0) a.out[b + (long long)q * a.Ns] = sm[sl * LS + q];
    }
  }
}

template <int LOG2, int Q, bool SM>
int launch_t(const FastArgs& a, cudaStream_t st) {
  if constexpr ((Q << LOG2) > TILE || (SM && (Q << LOG2) > 1024)) {
    return -1;
  } else {
  using G = Geo<LOG2, Q, SM>;
  size_t smem = sizeof(cplx) * (size_t)G::TL * G::LS;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(fft_fast_kernel<LOG2, Q, SM>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         96 * 1024);
    set = true;
  }
  long long blocks = (a.nsub + G::TL - 1) / G::TL;
  { TrKTimer _kt(TRK_FFT, st); fft_fast_kernel<LOG2, Q, SM><<<(unsigned)blocks, G::FT, smem, st>>>(a); }
  return 0;
  }
}

#define TR_FAST_CASES(Q, MAXLOG)                                  \
  case Q: switch (log2) {                                         \
      TR_L(Q, 0) TR_L(Q, 1) TR_L(Q, 2) TR_L(Q, 3) TR_L(Q, 4)      \
      TR_L(Q, 5) TR_L(Q, 6) TR_L(Q, 7) TR_L(Q, 8) TR_L(Q, 9)      \
      TR_L(Q, 10) TR_L(Q, 11) TR_L(Q, 12)                         \
      default: return -1;                                         \
    }

}  // namespace

int fast_tile(int log2, int q) {
  int R = q << log2;
  int p = np2(R);
  return p >= TILE ? 1 : (TILE / p > 256 ? 256 : TILE / p);
}

bool fast_supported(int log2, int q) {
  if (!(q == 1 || q == 3 || q == 5 || q == 7 || q == 9 || q == 15)) return false;
  return (q << log2) <= TILE && log2 <= 12;
}

int fast_launch(int log2, int q, bool small, const FastArgs& a, cudaStream_t st) {
  if (!fast_supported(log2, q)) return -1;
#define TR_L(Q, L) \
  case L:          \
    return small ? launch_t<L, Q, true>(a, st) : launch_t<L, Q, false>(a, st);
  switch (q) {
    TR_FAST_CASES(1, 12)
    TR_FAST_CASES(3, 10)
    TR_FAST_CASES(5, 9)
    TR_FAST_CASES(7, 9)
    TR_FAST_CASES(9, 8)
    TR_FAST_CASES(15, 8)
    default: return -1;
  }
#undef TR_L
}
