// In-shared-memory FFT stages for small lengths L = R1 R2 (R1, R2 in
// {2, 3, 4, 5, 7, 8, 9, 16}), used by the cluster transform (fft_cl.cu) and
// the fused small combine (combine_small.cu).
#pragma once
#include "fft_bfly.cuh"

// Length L = R1 R2 transforms of NL lines in shared memory, element e of
// line l at base[l * LS + e * ES] (consecutive threads take consecutive
// lines: conflict-free for LS = 1, or for ES = 1 with an odd line pitch LS).
//   stage1: radix R1 over e = j2 + R2 j1, times W_L^(j2 k1), in place; the
//           value loaded for (l, e) passes through ld(l, e, x) first;
//   stage2: radix R2 over e = R2 k1 + j2; after a barrier the outputs
//           k = k1 + R1 k2 (natural order) go to st(l, k, v) -- any layout,
//           since every read of the buffer is done by then.
template <int R1, int R2, int NL, int ES, int NTH, class Ld, int LS = 1>
TR_D void stage1(cplx* base, int sign, const cplx* twL, Ld ld) {
  constexpr int L = R1 * R2;
  for (int g = threadIdx.x; g < NL * R2; g += NTH) {
    const int l = g % NL, j2 = g / NL;
    cplx v[R1];
#pragma unroll
    for (int j1 = 0; j1 < R1; ++j1) v[j1] = ld(l, j2 + R2 * j1, base[l * LS + (j2 + R2 * j1) * ES]);
    bfly_any<R1>(v, sign);
    if (j2) {
#pragma unroll
      for (int k1 = 1; k1 < R1; ++k1) {
        cplx w = __ldg(&twL[(j2 * k1) % L]);
        if (sign < 0) w.y = -w.y;
        v[k1] = cmul(v[k1], w);
      }
    }
#pragma unroll
    for (int k1 = 0; k1 < R1; ++k1) base[l * LS + (j2 + R2 * k1) * ES] = v[k1];
  }
  __syncthreads();
}

template <int R1, int R2, int NL, int ES, int NTH, class St, int LS = 1>
TR_D void stage2(const cplx* base, int sign, St st) {
  constexpr int NG = (NL * R1 + NTH - 1) / NTH;
  cplx v[NG][R2];
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    const int g = threadIdx.x + q * NTH;
    if (NL * R1 % NTH == 0 || g < NL * R1) {
      const int l = g % NL, k1 = g / NL;
#pragma unroll
      for (int j2 = 0; j2 < R2; ++j2) v[q][j2] = base[l * LS + (R2 * k1 + j2) * ES];
      bfly_any<R2>(v[q], sign);
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < NG; ++q) {
    const int g = threadIdx.x + q * NTH;
    if (NL * R1 % NTH == 0 || g < NL * R1) {
      const int l = g % NL, k1 = g / NL;
#pragma unroll
      for (int k2 = 0; k2 < R2; ++k2) st(l, k1 + R1 * k2, v[q][k2]);
    }
  }
}

