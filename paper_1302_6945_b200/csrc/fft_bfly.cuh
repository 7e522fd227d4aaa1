// In-register FFT butterflies (radix 2, 3, 4, 5, 7, 8, 16), unnormalised:
//   a[k] <- sum_n a[n] exp(sign * 2 pi i n k / RS)
#pragma once
#include "common.cuh"

// cos / sin (2 pi k / RS) for RS = 5, 7 as literals
template <int RS>
TR_HD constexpr double tcos(int k) {
  if (RS == 5) {
    constexpr double c[5] = {1.0, 0.30901699437494742410, -0.80901699437494742410,
                             -0.80901699437494742410, 0.30901699437494742410};
    return c[k];
  }
  constexpr double c[7] = {1.0, 0.62348980185873353053, -0.22252093395631440429,
                           -0.90096886790241912624, -0.90096886790241912624,
                           -0.22252093395631440429, 0.62348980185873353053};
  return c[k];
}
template <int RS>
TR_HD constexpr double tsin(int k) {
  if (RS == 5) {
    constexpr double s[5] = {0.0, 0.95105651629515357212, 0.58778525229247312917,
                             -0.58778525229247312917, -0.95105651629515357212};
    return s[k];
  }
  constexpr double s[7] = {0.0, 0.78183148246802980871, 0.97492791218182360702,
                           0.43388373911755812048, -0.43388373911755812048,
                           -0.97492791218182360702, -0.78183148246802980871};
  return s[k];
}

template <int RS>
TR_D void bfly(cplx* a, int sign) {
  if constexpr (RS == 2) {
    cplx t = a[0];
    a[0] = cadd(t, a[1]);
    a[1] = csub(t, a[1]);
  } else if constexpr (RS == 4) {
    cplx t0 = cadd(a[0], a[2]), t1 = csub(a[0], a[2]);
    cplx t2 = cadd(a[1], a[3]), d = csub(a[1], a[3]);
    cplx t3 = sign > 0 ? cmk(-d.y, d.x) : cmk(d.y, -d.x);
    a[0] = cadd(t0, t2);
    a[2] = csub(t0, t2);
    a[1] = cadd(t1, t3);
    a[3] = csub(t1, t3);
  } else if constexpr (RS == 8) {
    cplx e[4] = {a[0], a[2], a[4], a[6]};
    cplx o[4] = {a[1], a[3], a[5], a[7]};
    bfly<4>(e, sign);
    bfly<4>(o, sign);
    const double c = 0.70710678118654752440;
    const double s = (double)sign;
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
  } else if constexpr (RS == 3) {
    const double h = 0.86602540378443864676;  // sin(2 pi / 3)
    cplx t1 = cadd(a[1], a[2]);
    cplx t2 = cmk(a[0].x - 0.5 * t1.x, a[0].y - 0.5 * t1.y);
    cplx d = csub(a[1], a[2]);
    double s = h * (double)sign;
    cplx t3 = cmk(-s * d.y, s * d.x);  // i * sign * sin * d
    a[0] = cadd(a[0], t1);
    a[1] = cadd(t2, t3);
    a[2] = csub(t2, t3);
  } else {
    // direct DFT for radix 5 / 7 with constant twiddles
    const double sg = (double)sign;
    cplx y[RS];
#pragma unroll
    for (int v = 0; v < RS; ++v) {
      cplx acc = a[0];
#pragma unroll
      for (int u = 1; u < RS; ++u) {
        const int k = (u * v) % RS;
        acc = cfma(a[u], cmk(tcos<RS>(k), sg * tsin<RS>(k)), acc);
      }
      y[v] = acc;
    }
#pragma unroll
    for (int v = 0; v < RS; ++v) a[v] = y[v];
  }
}


// radix 16 = 4 x 4 with the W16 twiddles in between (output in natural order)
TR_D void bfly16(cplx* a, int sign) {
  const double s = (double)sign;
  const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;  // cos, sin(pi/8)
  const double h = 0.70710678118654752440;
  cplx y[4][4];
#pragma unroll
  for (int n2 = 0; n2 < 4; ++n2) {
    cplx t[4] = {a[n2], a[4 + n2], a[8 + n2], a[12 + n2]};
    bfly<4>(t, sign);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) y[n2][k1] = t[k1];
  }
  // y[n2][k1] *= W16^(n2 k1), exponents 0..9
  const double cs[10] = {1.0, c1, h, s1, 0.0, -s1, -h, -c1, -1.0, -c1};
  const double sn[10] = {0.0, s1, h, c1, 1.0, c1, h, s1, 0.0, -s1};
#pragma unroll
  for (int n2 = 1; n2 < 4; ++n2)
#pragma unroll
    for (int k1 = 1; k1 < 4; ++k1) {
      const int e = n2 * k1;
      y[n2][k1] = cmul(y[n2][k1], cmk(cs[e], s * sn[e]));
    }
#pragma unroll
  for (int k1 = 0; k1 < 4; ++k1) {
    cplx t[4] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1]};
    bfly<4>(t, sign);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) a[k1 + 4 * k2] = t[k2];
  }
}

// radix 9 = 3 x 3 with the W9 twiddles in between (output in natural order)
TR_D void bfly9(cplx* a, int sign) {
  const double s = (double)sign;
  // cos / sin (2 pi e / 9), e = 1, 2, 4
  const double c1 = 0.76604444311897803520, s1 = 0.64278760968653932632;
  const double c2 = 0.17364817766693034885, s2 = 0.98480775301220805936;
  const double c4 = -0.93969262078590838405, s4 = 0.34202014332566873304;
  cplx y[3][3];
#pragma unroll
  for (int n2 = 0; n2 < 3; ++n2) {
    cplx t[3] = {a[n2], a[3 + n2], a[6 + n2]};
    bfly<3>(t, sign);
#pragma unroll
    for (int k1 = 0; k1 < 3; ++k1) y[n2][k1] = t[k1];
  }
  y[1][1] = cmul(y[1][1], cmk(c1, s * s1));
  y[1][2] = cmul(y[1][2], cmk(c2, s * s2));
  y[2][1] = cmul(y[2][1], cmk(c2, s * s2));
  y[2][2] = cmul(y[2][2], cmk(c4, s * s4));
#pragma unroll
  for (int k1 = 0; k1 < 3; ++k1) {
    cplx t[3] = {y[0][k1], y[1][k1], y[2][k1]};
    bfly<3>(t, sign);
#pragma unroll
    for (int k2 = 0; k2 < 3; ++k2) a[k1 + 3 * k2] = t[k2];
  }
}

template <int RS>
TR_D void bfly_any(cplx* a, int sign) {
  if constexpr (RS == 16) bfly16(a, sign);
  else if constexpr (RS == 9) bfly9(a, sign);
  else bfly<RS>(a, sign);
}
