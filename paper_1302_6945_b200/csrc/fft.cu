#include <tuple>
#include <algorithm>
#include <stdlib.h>
#include <cmath>
// Batched complex128 multi-pass Stockham FFT (see fft.cuh).
#include "fft.cuh"
#include "kernels.cuh"

extern thread_local long long g_fft_tag;
thread_local int g_fft_groups = 0;  // set while a solve enqueues work for several concurrent stream groups
#include "fft_fast.cuh"

#include <math.h>
#include <map>
#include <mutex>
#include <vector>

namespace {

constexpr int FFT_THREADS = 256;
constexpr int FFT_TILE = 4096;                 // complex values per CTA tile
constexpr int FFT_MAXE = FFT_TILE / FFT_THREADS;  // values per thread

struct PassArgs {
  long long n;
  int R, Ns, T, LB, LS, nst, sign;
  int rad[16];
  const cplx* twN;
  const cplx* twR;
  const cplx* in;
  long long in_ls, in_len;
  cplx* out;
  long long out_ls;
  long long lines;
  long long tiles;  // n / R / T
};

TR_D cplx tw_lookup(const cplx* tab, long long idx, int sign) {
  cplx w = __ldg(&tab[idx]);
  return sign < 0 ? cconj(w) : w;
}

template <int RS>
TR_D void dft_small(cplx* a, int sign) {
  if (RS == 2) {
    cplx t = a[0];
    a[0] = cadd(t, a[1]);
    a[1] = csub(t, a[1]);
  } else if (RS == 4) {
    cplx t0 = cadd(a[0], a[2]), t1 = csub(a[0], a[2]);
    cplx t2 = cadd(a[1], a[3]), d = csub(a[1], a[3]);
    cplx t3 = sign > 0 ? cmk(-d.y, d.x) : cmk(d.y, -d.x);  // d * (i*sign)
    a[0] = cadd(t0, t2);
    a[2] = csub(t0, t2);
    a[1] = cadd(t1, t3);
    a[3] = csub(t1, t3);
  } else if (RS == 8) {
    cplx e[4] = {a[0], a[2], a[4], a[6]};
    cplx o[4] = {a[1], a[3], a[5], a[7]};
    dft_small<4>(e, sign);
    dft_small<4>(o, sign);
    const double c = 0.70710678118654752440;
    double s = (double)sign;
    // o[v] *= w8^(sign v)
    cplx o1 = cmk(c * (o[1].x - s * o[1].y), c * (o[1].y + s * o[1].x));
    cplx o2 = cmk(-s * o[2].y, s * o[2].x);
    cplx o3 = cmk(-c * (o[3].x + s * o[3].y), c * (s * o[3].x - o[3].y));
    a[0] = cadd(e[0], o[0]);
    a[4] = csub(e[0], o[0]);
    a[1] = cadd(e[1], o1);
    a[5] = csub(e[1], o1);
    a[2] = cadd(e[2], o2);
    a[6] = csub(e[2], o2);
    a[3] = cadd(e[3], o3);
    a[7] = csub(e[3], o3);
  }
}

// One Stockham stage of radix RS over all smem lines (power-of-two radix).
template <int RS>
TR_D void smem_stage_pow2(cplx* s, const PassArgs& a, int NsS, int nlines_tile) {
  const int R = a.R;
  const int per_line = R / RS;
  const int total = per_line * nlines_tile;
  const int mtot = NsS * RS;  // sub-transform length after this stage
  const int twstep = R / mtot;
  cplx v[FFT_MAXE];
#pragma unroll
  for (int it = 0; it < FFT_MAXE / RS; ++it) {
    int bidx = threadIdx.x + it * FFT_THREADS;
    if (bidx < total) {
      int line = bidx / per_line, b = bidx - line * per_line;
      int k = b % NsS;
      cplx* base = s + line * a.LS;
#pragma unroll
      for (int u = 0; u < RS; ++u) {
        cplx x = base[b + u * per_line];
        if (NsS > 1 && u > 0) x = cmul(x, tw_lookup(a.twR, (long long)u * k * twstep, a.sign));
        v[it * RS + u] = x;
      }
      dft_small<RS>(&v[it * RS], a.sign);
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < FFT_MAXE / RS; ++it) {
    int bidx = threadIdx.x + it * FFT_THREADS;
    if (bidx < total) {
      int line = bidx / per_line, b = bidx - line * per_line;
      int k = b % NsS;
      cplx* base = s + line * a.LS;
      int o = (b / NsS) * mtot + k;
#pragma unroll
      for (int u = 0; u < RS; ++u) base[o + u * NsS] = v[it * RS + u];
    }
  }
  __syncthreads();
}

// Direct DFT stage of odd radix q (first stage, so NsS == 1: no twiddles).
TR_D void smem_stage_odd(cplx* s, const PassArgs& a, int q, int nlines_tile) {
  const int R = a.R;
  const int per_line = R / q;
  const int total = R * nlines_tile;  // outputs
  const int wstep = R / q;
  cplx v[FFT_MAXE];
#pragma unroll
  for (int it = 0; it < FFT_MAXE; ++it) {
    int oi = threadIdx.x + it * FFT_THREADS;
    if (oi < total) {
      int line = oi / R, r = oi - line * R;
      int b = r / q, vv = r - b * q;
      const cplx* base = s + line * a.LS;
      cplx acc = cmk(0.0, 0.0);
      for (int u = 0; u < q; ++u) {
        int e = (u * vv) % q;
        acc = cfma(base[b + u * per_line], tw_lookup(a.twR, (long long)e * wstep, a.sign), acc);
      }
      v[it] = acc;
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < FFT_MAXE; ++it) {
    int oi = threadIdx.x + it * FFT_THREADS;
    if (oi < total) {
      int line = oi / R, r = oi - line * R;
      int b = r / q, vv = r - b * q;
      // NsS == 1: output position b*q + vv == r
      s[line * a.LS + b * q + vv] = v[it];
    }
  }
  __syncthreads();
}

__global__ void __launch_bounds__(FFT_THREADS) fft_pass_kernel(PassArgs a) {
  extern __shared__ cplx smem[];
  const int R = a.R, T = a.T, LB = a.LB;
  const long long tile = blockIdx.x;
  const long long line0 = (long long)blockIdx.y * LB;
  const long long j0 = tile * T;
  const long long stride_in = a.n / R;  // distance between butterfly inputs
  const int nel = LB * T * R;
  const int nlines_tile = LB * T;

  // ---- load (t fastest, then r, then line) with the inter-pass twiddle ----
  for (int idx = threadIdx.x; idx < nel; idx += FFT_THREADS) {
    int t = idx % T;
    int r = (idx / T) % R;
    int lb = idx / (T * R);
    long long line = line0 + lb;
    cplx x = cmk(0.0, 0.0);
    if (line < a.lines) {
      long long j = j0 + t;
      long long e = j + (long long)r * stride_in;
      if (e < a.in_len) x = a.in[line * a.in_ls + e];
      if (a.Ns > 1 && r > 0) {
        long long k = j % a.Ns;
        long long m = ((long long)r * k) * (a.n / ((long long)a.Ns * R));
        x = cmul(x, tw_lookup(a.twN, m % a.n, a.sign));
      }
    }
    smem[(lb * T + t) * a.LS + r] = x;
  }
  __syncthreads();

  // ---- length-R sub-transform of every staged line ----
  int NsS = 1;
  for (int st = 0; st < a.nst; ++st) {
    int rs = a.rad[st];
    if (rs == 8) smem_stage_pow2<8>(smem, a, NsS, nlines_tile);
    else if (rs == 4) smem_stage_pow2<4>(smem, a, NsS, nlines_tile);
    else if (rs == 2) smem_stage_pow2<2>(smem, a, NsS, nlines_tile);
    else smem_stage_odd(smem, a, rs, nlines_tile);
    NsS *= rs;
  }

  // ---- store: y[(j/Ns)*Ns*R + q*Ns + (j%Ns)] ----
  for (int idx = threadIdx.x; idx < nel; idx += FFT_THREADS) {
    int t, q, lb;
    if (a.Ns == 1) {  // each j owns a contiguous run of R outputs
      q = idx % R;
      t = (idx / R) % T;
      lb = idx / (T * R);
    } else {
      t = idx % T;
      q = (idx / T) % R;
      lb = idx / (T * R);
    }
    long long line = line0 + lb;
    if (line >= a.lines) continue;
    long long j = j0 + t;
    long long k = j % a.Ns;
    long long o = (j / a.Ns) * (long long)a.Ns * R + (long long)q * a.Ns + k;
    a.out[line * a.out_ls + o] = smem[(lb * T + t) * a.LS + q];
  }
}

struct TwKey {
  int dev;
  long long n;
  bool operator<(const TwKey& o) const { return dev != o.dev ? dev < o.dev : n < o.n; }
};
std::mutex g_mu;
std::map<TwKey, cplx*> g_tw;

void split_pow2(int R, int* rad, int* nst) {
  // odd part first, then 8s, then a 4 or 2 remainder
  int q = R;
  while ((q & 1) == 0) q >>= 1;
  int p2 = R / q;
  int k = 0;
  if (q > 1) rad[k++] = q;
  while (p2 >= 8) { rad[k++] = 8; p2 /= 8; }
  if (p2 == 4) rad[k++] = 4;
  else if (p2 == 2) rad[k++] = 2;
  *nst = k;
}

long long odd_part(long long n) {
  while (n > 0 && (n & 1) == 0) n >>= 1;
  return n;
}

}  // namespace

const cplx* twiddle_table(long long n) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  TwKey key{dev, n};
  auto it = g_tw.find(key);
  if (it != g_tw.end()) return it->second;
  std::vector<cplx> h((size_t)n);
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (long long k = 0; k < n; ++k) {
    // exact symmetric reduction keeps the table symmetric to the last bit
    long long r = k;
    long double ang = two_pi * (long double)r / (long double)n;
    h[(size_t)k] = cmk((double)cosl(ang), (double)sinl(ang));
  }
  // exact values at the quarter points
  if (n % 4 == 0) {
    h[(size_t)(n / 4)] = cmk(0.0, 1.0);
    h[(size_t)(3 * n / 4)] = cmk(0.0, -1.0);
  }
  if (n % 2 == 0) h[(size_t)(n / 2)] = cmk(-1.0, 0.0);
  cplx* d = nullptr;
  if (cudaMalloc(&d, sizeof(cplx) * (size_t)n) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, h.data(), sizeof(cplx) * (size_t)n, cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  g_tw[key] = d;
  return d;
}

// [N2][TL] table exp(2 pi i n2 l / n) (cached)
const cplx* col_twiddles(long long n, long long N2, int TL) {
  int dev = 0;
  cudaGetDevice(&dev);
  static std::map<std::tuple<int, long long, long long, int>, cplx*> cache;
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_tuple(dev, n, N2, TL);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  std::vector<cplx> h((size_t)(N2 * TL));
  const long double two_pi = 6.283185307179586476925286766559005768L;
  for (long long a = 0; a < N2; ++a)
    for (int l = 0; l < TL; ++l) {
      const long long m = (a * l) % n;
      const long double ang = two_pi * (long double)m / (long double)n;
      h[(size_t)(a * TL + l)] = cmk((double)cosl(ang), (double)sinl(ang));
    }
  cplx* d = nullptr;
  if (cudaMalloc(&d, sizeof(cplx) * h.size()) != cudaSuccess) return nullptr;
  if (cudaMemcpy(d, h.data(), sizeof(cplx) * h.size(), cudaMemcpyHostToDevice) != cudaSuccess) {
    cudaFree(d);
    return nullptr;
  }
  cache[key] = d;
  return d;
}

bool fft_supported(long long n) {
  if (n < 1) return false;
  return odd_part(n) <= FFT_MAX_ODD;
}

// measured cost per element of tr_fft on B200 (tools/fft_sweep.py, 8M-element batches)
static const struct { long long n; double c; } kFftCost[] = {
    {16, 0.0145}, {18, 0.0102}, {20, 0.0074}, {24, 0.0091}, {28, 0.0094}, {30, 0.0105},
    {32, 0.0083}, {36, 0.0075}, {40, 0.0079}, {48, 0.0067}, {56, 0.0077}, {60, 0.0085},
    {64, 0.0069}, {72, 0.0071}, {80, 0.0067}, {96, 0.0067}, {112, 0.0064}, {120, 0.0079},
    {128, 0.0057}, {144, 0.0069}, {160, 0.0076}, {192, 0.0069}, {224, 0.0072}, {240, 0.0071},
    {256, 0.0060}, {288, 0.0084}, {320, 0.0083}, {384, 0.0078}, {448, 0.0082}, {480, 0.0091},
    {512, 0.0083}, {576, 0.0087}, {640, 0.0091}, {768, 0.0082}, {896, 0.0086}, {960, 0.0091},
    {1024, 0.0093}, {1152, 0.0096}, {1280, 0.0093}, {1536, 0.0100}, {1792, 0.0090}, {1920, 0.0096},
    {2048, 0.0106}, {2304, 0.0103}, {2560, 0.0113}, {3072, 0.0113}, {3584, 0.0109}, {3840, 0.0099},
    {4096, 0.0120}, {4608, 0.0297}, {5120, 0.0304}, {6144, 0.0370}, {7168, 0.0270}, {7680, 0.0267},
    {8192, 0.0321}, {9216, 0.0246}, {10240, 0.0290}, {12288, 0.0227}, {14336, 0.0252}, {15360, 0.0209},
    {16384, 0.0233}, {18432, 0.0227}, {20480, 0.0293}, {24576, 0.0221}, {28672, 0.0249}, {30720, 0.0189},
    {32768, 0.0236}, {36864, 0.0224}, {40960, 0.0196}, {49152, 0.0215}, {57344, 0.0178}, {61440, 0.0185},
    {65536, 0.0186}, {73728, 0.0225}, {81920, 0.0196}, {98304, 0.0215}, {114688, 0.0177}, {122880, 0.0183},
    {131072, 0.0184},
};

long long fft_good_len(long long n) {
  if (n <= 1) return 1;
  // candidates 2^a * q, q in a small odd set; ranked by the measured cost of
  // this library's kernels (len * cost per element), else len (log2 len + q / 4)
  static const int qs[] = {1, 3, 5, 7, 9, 15};
  long long best = -1;
  double best_cost = 1e300;
  for (int q : qs) {
    long long len = q;
    while (len < n) len *= 2;
    double per = -1.0;
    for (const auto& e : kFftCost)
      if (e.n == len) per = e.c;
    const double cost = per > 0.0 ? (double)len * per
                                  : (double)len * (log2((double)len) + 0.25 * q) * 1e-3;
    if (cost < best_cost) { best_cost = cost; best = len; }
  }
  return best;
}

int fft_plan(long long n, FftPlan* out) {
  if (!fft_supported(n)) {
    tr_set_error("fft length %lld has an odd factor above %d", n, FFT_MAX_ODD);
    return 2;
  }
  FftPlan p;
  p.n = n;
  p.twN = twiddle_table(n);
  if (!p.twN) { tr_set_error("twiddle table allocation failed (n=%lld)", n); return 4; }
  long long q = odd_part(n);
  long long p2 = n / q;
  std::vector<long long> radices;
  if (n <= FFT_TILE) {
    radices.push_back(n);
  } else {
    // passes of radix <= 1024 (tiles of >= 4 sub-transforms keep global
    // accesses in >= 64 B runs).  Leading passes are powers of two so every
    // pass's Ns is a power of two; the odd factor rides in the last pass.
    int a = 0;
    while ((p2 >> a) > 1) ++a;  // p2 = 2^a
    int npass = (n <= 1024LL * 1024LL) ? 2 : 3;
    int lgq = 0;
    while ((1LL << lgq) < q) ++lgq;
    int lg = a + lgq;
    int share = (lg + npass - 1) / npass;
    int b_last = share - lgq;
    if (b_last < 0) b_last = 0;
    int rest = a - b_last;
    std::vector<long long> lead;
    for (int i = 0; i < npass - 1; ++i) {
      int left = npass - 1 - i;
      int b = (rest + left - 1) / left;
      if (b > 10) b = 10;
      lead.push_back(1LL << b);
      rest -= b;
    }
    b_last += rest;  // whatever the leading passes could not take
    long long last = q << b_last;
    if (last > 1024 && q == 1) { tr_set_error("fft length %lld cannot be split", n); return 2; }
    if (last > FFT_TILE) { tr_set_error("fft length %lld cannot be split", n); return 2; }
    for (long long t : lead) radices.push_back(t);
    radices.push_back(last);
  }
  (void)p2;
  if (radices.size() > 3) { tr_set_error("fft length %lld needs too many passes", n); return 2; }
  p.npass = (int)radices.size();
  long long Ns = 1;
  for (int i = 0; i < p.npass; ++i) {
    FftPass& ps = p.pass[i];
    ps.R = (int)radices[i];
    ps.Ns = (int)Ns;
    if (p.npass == 1) {
      ps.T = 1;
      ps.LB = (int)(FFT_TILE / ps.R);
      if (ps.LB > 64) ps.LB = 64;
      if (ps.LB < 1) ps.LB = 1;
    } else {
      ps.LB = 1;
      long long T = FFT_TILE / ps.R;
      long long nj = n / ps.R;
      if (T > nj) T = nj;
      // T must divide n/R
      while (nj % T) T >>= 1;
      ps.T = (int)T;
    }
    split_pow2(ps.R, ps.rad, &ps.nst);
    ps.q = (int)odd_part(ps.R);
    ps.log2 = 0;
    while ((ps.q << ps.log2) < ps.R) ++ps.log2;
    ps.fast = fast_supported(ps.log2, ps.q) && ((Ns & (Ns - 1)) == 0);
    ps.twR = twiddle_table(ps.R);
    if (!ps.twR) { tr_set_error("twiddle table allocation failed (R=%d)", ps.R); return 4; }
    Ns *= ps.R;
  }
  // two-pass column plan (fft_col.cu) when n = N1 N2 with both <= 1024
  if (p.npass >= 2) {
    int a = 0;
    while ((p2 >> a) > 1) ++a;
    int lq = 0;
    while ((1LL << lq) < q) ++lq;
    // balanced split first, then the nearest ones whose tiles divide the
    // sub-transform counts (pass A tile | N2)
    const int amid = (a + lq + 1) / 2;
    for (int d = 0; d <= a && !p.col; ++d) {
      for (int sgn = 0; sgn < 2 && !p.col; ++sgn) {
        const int a1 = sgn ? amid + d : amid - d;
        if (d == 0 && sgn) continue;
        const int a2 = a - a1;
        if (a1 < 1 || a2 < 0) continue;
        const long long N1 = 1LL << a1, N2 = q << a2;
        if (N1 > 1024 || N2 > 1024 || N1 * N2 != n) continue;
        if (N2 % col_tile((int)N1) || N1 % col_tile((int)N2)) continue;
        p.col = true;
        p.a1 = a1;
        p.a2 = a2;
        p.q2 = (int)q;
        p.tw1 = twiddle_table(N1);
        p.tw2 = twiddle_table(N2);
        p.twc = col_twiddles(n, N2, col_tile((int)N2));
        if (!p.tw1 || !p.tw2 || !p.twc) { tr_set_error("twiddle table allocation failed"); return 4; }
      }
    }
  }
  *out = p;
  return 0;
}

static int launch_pass(const FftPlan& p, int i, const cplx* in, long long in_ls, long long in_len,
                       cplx* out, long long out_ls, long long lines, int sign, cudaStream_t st,
                       const cplx* mul = nullptr, long long mul_ls = 0, double mul_scale = 1.0) {
  const FftPass& ps = p.pass[i];
  if (ps.fast) {
    FastArgs f;
    f.mul = mul;
    f.mul_ls = mul_ls;
    f.mul_scale = mul_scale;
    f.in = in;
    f.in_ls = in_ls;
    f.in_len = (int)in_len;
    f.out = out;
    f.out_ls = out_ls;
    f.J = (int)(p.n / ps.R);
    f.nsub = lines * (long long)f.J;
    f.Ns = ps.Ns;
    f.log2Ns = 0;
    while ((1 << f.log2Ns) < ps.Ns) ++f.log2Ns;
    f.tws = (int)(p.n / ((long long)ps.Ns * ps.R));
    f.twN = p.twN;
    f.twR = ps.twR;
    f.sign = sign;
    const bool small = p.npass == 1 && ps.R <= 1024;
    if (p.npass == 1 && reg_launch(ps.log2, ps.q, f, st) == 0) return 0;
    f.mul = nullptr;  // (fft_exec multiplied first when the register kernel cannot fuse it)
    if (fast_launch(ps.log2, ps.q, small, f, st) == 0) return 0;
  }
  PassArgs a;
  a.n = p.n;
  a.R = ps.R;
  a.Ns = ps.Ns;
  a.T = ps.T;
  a.LB = ps.LB;
  int nl = ps.LB * ps.T;
  a.LS = ps.R + (nl > 1 ? 1 : 0);
  a.nst = ps.nst;
  for (int k = 0; k < 16; ++k) a.rad[k] = ps.rad[k];
  a.sign = sign;
  a.twN = p.twN;
  a.twR = ps.twR;
  a.in = in;
  a.in_ls = in_ls;
  a.in_len = in_len;
  a.out = out;
  a.out_ls = out_ls;
  a.lines = lines;
  a.tiles = p.n / ps.R / ps.T;
  size_t smem = sizeof(cplx) * (size_t)nl * a.LS;
  dim3 grid((unsigned)a.tiles, (unsigned)((lines + ps.LB - 1) / ps.LB));
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(fft_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
    attr_set = true;
  }
  { TrKTimer _kt(TRK_FFT, st); fft_pass_kernel<<<grid, FFT_THREADS, smem, st>>>(a); }
  return 0;
}

int fft_exec(const FftPlan& p, const cplx* in, long long in_ls, long long in_len, cplx* out,
             long long out_ls, cplx* scratch, long long lines, int sign, cudaStream_t st,
             const cplx* mul, long long mul_ls, double mul_scale, long long chunk_bytes_override,
             const cplx* mul2) {
  if (lines <= 0) return 0;
  if (in_len > p.n) in_len = p.n;
  const long long n = p.n;
  if (mul2 && (!mul || !p.col || in_len != n)) {
    tr_set_error("fft_exec: the mirrored factor needs a two-pass column plan and full-length lines (n=%lld)", n);
    return 2;
  }
  g_fft_tag = (n << 20) + (lines & ((1 << 20) - 1));
  if (mul) {
    // the column kernels and the single-pass register kernel fuse the factor
    // into their loads; other plans multiply first
    const FftPass& p0 = p.pass[0];
    const int q0 = p0.q;
    const bool reg = p.npass == 1 && p0.fast && p0.R >= 2 && p0.R <= 4096 && p0.log2 <= 12 &&
                     (q0 == 1 || q0 == 3 || q0 == 5 || q0 == 7 || q0 == 9 || q0 == 15);
    if (!p.col && !reg) {
      if (in_len != n) { tr_set_error("fft_exec: fused factor needs full-length lines"); return 2; }
      { const int rc0 = launch_spec_mul(out, out_ls, in, in_ls, mul, mul_ls, n, mul_scale, lines, st); if (rc0) return rc0; }
      in = out;
      in_ls = out_ls;
      mul = nullptr;
    }
  }
  tr_kernel_work(TRK_FFT, 16.0 * lines * (double)(in_len + n),
                 5.0 * lines * (double)n * std::log2((double)n));
  // single pass on a cluster with TMA staging (fft_cl.cu): opt-in with
  // TR_FFT_CL=1.  Measured (tools/fft_lines.py, B200): 0.9-1.1x the two-pass
  // column kernels below (the DSMEM exchange and the cluster barriers cost
  // more than the halved HBM traffic saves at these FP64-latency-bound
  // rates), so the two-pass kernels stay the default.
  static const bool cl_on = [] {
    const char* e = getenv("TR_FFT_CL");
    return e && e[0] == '1';
  }();
  if (cl_on && !mul2 && fft_cl_supported(n) &&
      fft_cl_exec(n, in, in_ls, in_len, out, out_ls, lines, sign, p.twN, mul, mul_ls, mul_scale, st) == 0)
    return 0;
  if (p.col) {
    // Both passes in one cluster launch (fft_col.cu fft_col2_kernel), opt-in
    // with TR_FFT_C2=1 (one cluster per line) or 2 (persistent clusters).
    // Measured on B200 (tools/fft_c2.py, tools/fft_graph_lat.py): 1.3-1.55x the
    // chunked launches on transforms of hundreds of lines run alone (32768 x
    // 3200: 1484 -> 2310 GB/s), but no faster on the few-line transforms of a
    // single system, and inside a solve whose batch is split into stream
    // groups the long cluster launches delay the other groups' leaf sweeps
    // (which need whole SMs): c2 34.7 -> 37.1 ms, c5 360 -> 372 ms per step.
    // The chunked launches below therefore stay the default.
    static const bool c2_on = [] {
      const char* e = getenv("TR_FFT_C2");
      return e && e[0] != '0';
    }();
    static const bool c2_force = [] {
      const char* e = getenv("TR_FFT_C2_GROUPS");  // 1: also with concurrent stream groups
      return e && e[0] == '1';
    }();
    // (a batch split into stream groups keeps the chunked launches: their short
    // kernels interleave with the other groups' leaf sweeps, which need whole SMs
    // and would otherwise wait behind a long cluster launch -- measured slower)
    if (c2_on && (!g_fft_groups || c2_force)) {
      const long long N1 = 1LL << p.a1, N2 = (long long)p.q2 << p.a2;
      ColArgs ca, cb;
      ca.in = in;
      ca.in_ls = in_ls;
      ca.in_len = in_len;
      ca.in_es = (int)N2;
      ca.out = scratch;
      ca.out_ls = n;
      ca.out_es = 1;
      ca.subs = (int)N2;
      ca.lines = lines;
      ca.twR = p.tw1;
      ca.twN = p.twN;
      ca.tw2 = p.twc;
      ca.sign = sign;
      ca.mul = mul;
      ca.mul2 = mul2;
      ca.mul_ls = mul_ls;
      ca.mul_scale = mul_scale;
      cb = ca;
      cb.mul = nullptr;
      cb.mul2 = nullptr;
      cb.in = scratch;
      cb.in_ls = n;
      cb.in_len = n;
      cb.in_es = (int)N1;
      cb.out = out;
      cb.out_ls = out_ls;
      cb.out_es = (int)N1;
      cb.subs = (int)N1;
      cb.twR = p.tw2;
      if (col2_launch(p.a1, p.a2, p.q2, ca, cb, n, st) == 0) {
        TR_CUDA_CHECK(cudaGetLastError());
        return 0;
      }
    }
    // Lines go through both passes in chunks whose intermediate fits in L2
    // (the same scratch region for every chunk): pass B reads pass A's output
    // from L2, and the dirty scratch lines are overwritten by the next chunk
    // instead of being written back, so HBM sees one read and one write per
    // transform.  TR_FFT_L2MB sets the chunk size (0: one chunk).
    static const long long chunk_bytes = [] {
      const char* e = getenv("TR_FFT_L2MB");
      return (long long)(e ? atof(e) : 16.0) * (1LL << 20);
    }();
    long long cl = lines;
    const long long cb = chunk_bytes_override >= 0 ? chunk_bytes_override : chunk_bytes;
    if (cb > 0) {
      cl = cb / (n * (long long)sizeof(cplx));
      if (cl < 1) cl = 1;
      if (cl > lines) cl = lines;
    }
    const long long N1 = 1LL << p.a1, N2 = (long long)p.q2 << p.a2;
    for (long long s0 = 0; s0 < lines; s0 += cl) {
      const long long nl = std::min(cl, lines - s0);
      ColArgs c;
      c.in = in + s0 * in_ls;
      c.in_ls = in_ls;
      c.in_len = in_len;
      c.in_es = (int)N2;
      c.out = scratch;
      c.out_ls = n;
      c.out_es = 1;
      c.subs = (int)N2;
      c.lines = nl;
      c.twR = p.tw1;
      c.twN = p.twN;
      c.tw2 = p.twc;
      c.sign = sign;
      c.mul = mul ? mul + s0 * mul_ls : nullptr;
      c.mul2 = mul2 ? mul2 + s0 * mul_ls : nullptr;
      c.mul_ls = mul_ls;
      c.mul_scale = mul_scale;
      int rc = col_launch(true, p.a1, 1, c, st);
      if (rc) {
        if (s0 == 0) break;  // no column kernel: the pass plan below
        tr_set_error("fft column plan has no kernel for n=%lld", n);
        return 2;
      }
      c.mul = nullptr;
      c.mul2 = nullptr;
      c.in = scratch;
      c.in_ls = n;
      c.in_len = n;
      c.in_es = (int)N1;
      c.out = out + s0 * out_ls;
      c.out_ls = out_ls;
      c.out_es = (int)N1;
      c.subs = (int)N1;
      c.twR = p.tw2;
      rc = col_launch(false, p.a2, p.q2, c, st);
      if (rc) { tr_set_error("fft column plan has no kernel for n=%lld", n); return 2; }
      if (s0 + nl >= lines) {
        TR_CUDA_CHECK(cudaGetLastError());
        return 0;
      }
    }
  }
  if (mul2) {
    tr_set_error("fft_exec: no column kernel for the mirrored factor (n=%lld)", n);
    return 2;
  }
  if (p.npass == 1) {
    launch_pass(p, 0, in, in_ls, in_len, out, out_ls, lines, sign, st, mul, mul_ls, mul_scale);
  } else if (p.npass == 2) {
    launch_pass(p, 0, in, in_ls, in_len, scratch, n, lines, sign, st);
    launch_pass(p, 1, scratch, n, n, out, out_ls, lines, sign, st);
  } else {
    // in -> scratch -> out -> scratch, then copy back into out
    launch_pass(p, 0, in, in_ls, in_len, scratch, n, lines, sign, st);
    launch_pass(p, 1, scratch, n, n, out, out_ls, lines, sign, st);
    launch_pass(p, 2, out, out_ls, n, scratch, n, lines, sign, st);
    TR_CUDA_CHECK(cudaMemcpy2DAsync(out, sizeof(cplx) * out_ls, scratch, sizeof(cplx) * n,
                                    sizeof(cplx) * n, lines, cudaMemcpyDeviceToDevice, st));
  }
  TR_CUDA_CHECK(cudaGetLastError());
  return 0;
}

int fft_exec_twistfold(const FftPlan& p, const cplx* B, long long b_sys, long long b_cap, int PP, long long L,
                       long long o0, long long o1, int noff, long long N, const cplx* twN, cplx* out,
                       long long lines, cudaStream_t st) {
  if (lines <= 0) return 0;
  if (p.npass != 1 || !p.pass[0].fast || p.n < 128 || p.n > 4096) return -1;
  const FftPass& ps = p.pass[0];
  FastArgs f;
  f.in = nullptr;
  f.in_ls = 0;
  f.in_len = 0;
  f.out = out;
  f.out_ls = p.n;
  f.J = 1;
  f.nsub = lines;
  f.Ns = 1;
  f.log2Ns = 0;
  f.tws = 1;
  f.twN = p.twN;
  f.twR = ps.twR;
  f.sign = +1;
  f.tf_B = B;
  f.tf_bsys = b_sys;
  f.tf_bcap = b_cap;
  f.tf_PP = PP;
  f.tf_noff = noff;
  f.tf_L = L;
  f.tf_o0 = o0;
  f.tf_o1 = o1;
  f.tf_N = N;
  f.tf_twN = twN;
  g_fft_tag = (p.n << 20) + (lines & ((1 << 20) - 1));
  if (reg_launch(ps.log2, ps.q, f, st) != 0) return -1;
  tr_kernel_work(TRK_FFT, 16.0 * ((double)lines / noff * L + (double)lines * p.n),
                 5.0 * lines * (double)p.n * std::log2((double)p.n));
  if (cudaGetLastError() != cudaSuccess) return -1;
  return 0;
}
