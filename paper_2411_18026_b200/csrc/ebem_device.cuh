// Device-side FP64 building blocks of the Galerkin fill: complex arithmetic,
// the H0/H1 Hankel pair, the ten radial kernel scalars, and the 2x2 kernel
// combiners.  Everything lives in registers; the per-medium tables (log-power
// series, Gauss rules) are read from a per-handle context in global memory
// with warp-uniform addresses (L1 broadcast).
//
// Reference formulas followed (behaviour, not code):
//   hankel1_01                proj/src/hankel.cpp:34-71
//   KernelScalars::full       proj/src/kernel_scalars.cpp:214-281
//   KernelScalars::static_part proj/src/kernel_scalars.cpp:283-299
//   KernelScalars::split      proj/src/kernel_scalars.cpp:301-331
//   KernelScalars::remainder  proj/src/kernel_scalars.cpp:346-379
//   integrated_remainder      proj/src/kernel_scalars.cpp:333-344 (+ LogSeries
//                             ::integrate_scaled :108-121)
//   combine_D / combine_N     proj/src/kernels.cpp:22-68
//   q0_kernel                 proj/src/kernels.cpp:70-78
#pragma once

#include <cuda_runtime.h>
#include <math.h>

#include "ebem_ctx.h"
#include "hankel_tables.cuh"

namespace ebem_gpu {

// ----------------------------------------------------------------- complex
struct cplx {
  double re, im;
};
__device__ __forceinline__ cplx mk(double r, double i = 0.0) { return {r, i}; }
__device__ __forceinline__ cplx operator+(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx operator-(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cplx operator-(cplx a) { return {-a.re, -a.im}; }
__device__ __forceinline__ cplx operator*(cplx a, cplx b) {
  return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__device__ __forceinline__ cplx operator*(double s, cplx a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cplx operator*(cplx a, double s) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cplx operator/(cplx a, double s) { return {a.re / s, a.im / s}; }
__device__ __forceinline__ cplx& operator+=(cplx& a, cplx b) { a.re += b.re; a.im += b.im; return a; }
__device__ __forceinline__ cplx& operator-=(cplx& a, cplx b) { a.re -= b.re; a.im -= b.im; return a; }
__device__ __forceinline__ cplx conj(cplx a) { return {a.re, -a.im}; }
// a += s * b  (s real)
__device__ __forceinline__ void axpy(cplx& a, double s, cplx b) {
  a.re = fma(s, b.re, a.re);
  a.im = fma(s, b.im, a.im);
}
// a += b * c (complex)
__device__ __forceinline__ void cfma(cplx& a, cplx b, cplx c) {
  a.re = fma(b.re, c.re, a.re);
  a.re = fma(-b.im, c.im, a.re);
  a.im = fma(b.re, c.im, a.im);
  a.im = fma(b.im, c.re, a.im);
}

// ----------------------------------------------------------------- Hankel
template <int N>
__device__ __forceinline__ double clenshaw01(const double (&c)[N], double u) {
  const double y = 2.0 * u - 1.0;
  const double y2 = 2.0 * y;
  double b1 = 0.0, b2 = 0.0;
#pragma unroll
  for (int j = N - 1; j >= 1; --j) {
    const double t = fma(y2, b1, c[j] - b2);
    b2 = b1;
    b1 = t;
  }
  return fma(y, b1, c[0] - b2);
}

template <int N>
__device__ __forceinline__ double horner(const double (&c)[N], double u) {
  double s = c[N - 1];
#pragma unroll
  for (int j = N - 2; j >= 0; --j) s = fma(s, u, c[j]);
  return s;
}

// Regular parts of J0, J1/x, Y0, Y1 for x <= 8 in t = (x/8)^2: power series
// (one FMA per term) up to kTaylorX, Chebyshev (Clenshaw) above.
__device__ __forceinline__ void small_parts(double x, double t, double& j0, double& j1x,
                                            double& v0, double& v1) {
  if (x <= kTaylorX) {
    j0 = horner(kJ0Taylor, t);
    j1x = horner(kJ1Taylor, t);
    v0 = horner(kV0Taylor, t);
    v1 = horner(kV1Taylor, t);
  } else {
    j0 = clenshaw01(kJ0Small, t);
    j1x = clenshaw01(kJ1Small, t);
    v0 = clenshaw01(kV0Small, t);
    v1 = clenshaw01(kV1Small, t);
  }
}

constexpr double kTwoOverPi = 0.63661977236758134308;
constexpr double kEulerGamma = 0.57721566490153286061;
constexpr double kPio4Hi = 0.78539816339744827900;
constexpr double kPio4Lo = 3.06161699786838301793e-17;
constexpr double kPi = 3.14159265358979323846;

// H0^(1)(x), H1^(1)(x) for real x > 0 (Chebyshev in (x/8)^2 below 8,
// Hankel asymptotic factors in (8/x)^2 above, phase x - pi/4 kept exact with
// a two-sum as in proj/src/hankel.cpp:53-65).
__device__ __forceinline__ void hankel01(double x, cplx& h0, cplx& h1) {
  if (x <= 8.0) {
    const double q = x * 0.125;
    const double t = q * q;
    double j0, j1x, v0, v1;
    small_parts(x, t, j0, j1x, v0, v1);
    const double j1 = j1x * x;
    const double lg = kTwoOverPi * (log(0.5 * x) + kEulerGamma);
    const double y0 = fma(lg, j0, v0);
    const double y1 = v1 * x + lg * j1 - kTwoOverPi / x;
    h0 = mk(j0, y0);
    h1 = mk(j1, y1);
    return;
  }
  const double q = 8.0 / x;
  const double v = q * q;
  const double p0 = clenshaw01(kP0Large, v);
  const double q0 = clenshaw01(kQ0Large, v) / x;
  const double p1 = clenshaw01(kP1Large, v);
  const double q1 = clenshaw01(kQ1Large, v) / x;
  const double amp = sqrt(kTwoOverPi / x);
  const double chi0 = x - kPio4Hi;
  const double resid = (x - chi0) - kPio4Hi;
  const double corr = resid - kPio4Lo;
  double s0, c0;
  sincos(chi0, &s0, &c0);
  const double s0c = fma(corr, c0, s0);
  const double c0c = fma(-corr, s0, c0);
  s0 = s0c;
  c0 = c0c;
  const double c1 = s0;
  const double s1 = -c0;
  h0 = mk(amp * (p0 * c0 - q0 * s0), amp * (p0 * s0 + q0 * c0));
  h1 = mk(amp * (p1 * c1 - q1 * s1), amp * (p1 * s1 + q1 * c1));
}

// ----------------------------------------------------------------- scalars
// Order everywhere: gpsi, gchi, d1, d2, d3, n1, n2, n4, n5, n7.
struct Scalars {
  cplx s[10];
};
struct StaticScalars {
  double s[10];
};

__device__ __forceinline__ void static_part(const DevMedium& m, double r,
                                            StaticScalars& o) {
  const double logr = log(r);
  const double lp2m = m.lam + 2.0 * m.mu;
  o.s[0] = -logr / (2.0 * kPi) + m.cconst * (2.0 * logr + 1.0);
  o.s[1] = 2.0 * m.cconst;
  o.s[2] = m.mu / (2.0 * kPi * lp2m * r);
  o.s[3] = -o.s[2];
  o.s[4] = -8.0 * m.cconst / r;
  const double r2 = r * r;
  o.s[5] = m.mu * m.mu / (kPi * lp2m * r2);
  o.s[6] = m.mu * m.lam / (kPi * lp2m * r2);
  o.s[7] = -8.0 * m.qfactor / r2;
  o.s[8] = m.mu * (m.lam - m.mu) / (kPi * lp2m * r2);
  o.s[9] = 2.0 * m.mu * m.mu / (kPi * lp2m * r2);
}

// {Re a, Im a, Re b, Im b} of power q of series k (warp-uniform address).
__device__ __forceinline__ double4 ld_series(const DevCtx* __restrict__ ctx,
                                             int k, int q) {
  const double2* p = reinterpret_cast<const double2*>(ctx->series) +
                     2 * (k * kMaxSeriesPow + q);
  const double2 a = __ldg(p), b = __ldg(p + 1);
  return make_double4(a.x, a.y, b.x, b.y);
}

// Remainder series below the series radius: sum_q (a_q + b_q ln r) r^q, dense
// power tables (zeros where the series has no term).
__device__ __forceinline__ void series_eval(const DevCtx* __restrict__ ctx,
                                            double r, Scalars& o) {
  const double logr = log(r);
  const int maxq = ctx->series_maxq;
#pragma unroll
  for (int k = 0; k < 10; ++k) o.s[k] = mk(0.0, 0.0);
  double rp = 1.0;
  for (int q = 0; q <= maxq; ++q) {
#pragma unroll
    for (int k = 0; k < 10; ++k) {
      const double4 c = ld_series(ctx, k, q);
      // (a + b ln r) r^q
      const cplx t = mk(fma(c.z, logr, c.x), fma(c.w, logr, c.y));
      axpy(o.s[k], rp, t);
    }
    rp *= r;
  }
}

// Full dynamic scalars at r (> 0), proj/src/kernel_scalars.cpp:214-281.
__device__ __forceinline__ void scalars_full(const DevCtx* __restrict__ ctx,
                                             double r, Scalars& o) {
  const DevMedium& m = ctx->med;
  if (r < m.series_radius) {
    series_eval(ctx, r, o);
    StaticScalars s0;
    static_part(m, r, s0);
#pragma unroll
    for (int k = 0; k < 10; ++k) o.s[k].re += s0.s[k];
    return;
  }
  const double kT = m.kT, kL = m.kL;
  const double zT = kT * r;
  const double zL = kL * r;
  cplx h0T, h1T, h0L, h1L;
  hankel01(zT, h0T, h1T);
  hankel01(zL, h0L, h1L);
  // chi = (i/4) H0; multiplying by i/4: (a+ib) i/4 = (-b/4, a/4)
  auto i4 = [](cplx z) { return mk(-0.25 * z.im, 0.25 * z.re); };
  const cplx chiT = i4(h0T);
  const cplx chiL = i4(h0L);
  const cplx chiT1 = -(kT * i4(h1T));
  const cplx chiL1 = -(kL * i4(h1L));
  const double izT = 1.0 / zT, izL = 1.0 / zL;
  const cplx chiT2 = -(kT * kT) * i4(h0T - h1T * izT);
  const cplx chiL2 = -(kL * kL) * i4(h0L - h1L * izL);
  const cplx chiT3 = -(kT * kT * kT) *
                     i4(-h1T - h0T * izT + (2.0 * izT * izT) * h1T);
  const cplx chiL3 = -(kL * kL * kL) *
                     i4(-h1L - h0L * izL + (2.0 * izL * izL) * h1L);
  const cplx chiT4 = -(kT * kT * kT * kT) *
                     i4(-h0T + (2.0 * izT) * h1T + (3.0 * izT * izT) * h0T -
                        (6.0 * izT * izT * izT) * h1T);
  const cplx chiL4 = -(kL * kL * kL * kL) *
                     i4(-h0L + (2.0 * izL) * h1L + (3.0 * izL * izL) * h0L -
                        (6.0 * izL * izL * izL) * h1L);
  const double ikT2 = 1.0 / (kT * kT);
  const cplx psi1 = (chiT1 - chiL1) * ikT2;
  const cplx psi2 = (chiT2 - chiL2) * ikT2;
  const cplx psi3 = (chiT3 - chiL3) * ikT2;
  const cplx psi4 = (chiT4 - chiL4) * ikT2;
  const double ir = 1.0 / r;
  const double mu = m.mu;
  o.s[0] = chiT + psi1 * ir;
  o.s[1] = psi2 - psi1 * ir;
  const cplx w = o.s[1] * ir;
  const cplx gam = o.s[1] * (ir * ir);
  const cplx bet = (psi3 - 3.0 * w) * ir;
  const cplx alf = psi4 - (6.0 * ir) * psi3 + 15.0 * gam;
  o.s[2] = m.aratio * chiL1 + 2.0 * w;
  o.s[3] = chiT1 + 2.0 * w;
  o.s[4] = 2.0 * (psi3 - 3.0 * w);
  o.s[5] = (-2.0 * mu * ir) * chiT1 - (4.0 * mu) * gam;
  o.s[6] = (-mu) * (chiT2 - chiT1 * ir) - (4.0 * mu) * bet;
  o.s[7] = (-4.0 * mu) * alf;
  o.s[8] = (m.lam * m.aratio * kL * kL) * chiL -
           (4.0 * mu * m.aratio * ir) * chiL1 - (4.0 * mu) * gam;
  o.s[9] = (-2.0 * mu * m.aratio) * (chiL2 - chiL1 * ir) - (4.0 * mu) * bet;
}

// full and remainder together, proj/src/kernel_scalars.cpp:301-331.
__device__ __forceinline__ void scalars_split(const DevCtx* __restrict__ ctx,
                                              double r, Scalars& full,
                                              Scalars& rem) {
  StaticScalars s0;
  static_part(ctx->med, r, s0);
  if (r < ctx->med.series_radius) {
    series_eval(ctx, r, rem);
#pragma unroll
    for (int k = 0; k < 10; ++k) {
      full.s[k] = rem.s[k];
      full.s[k].re += s0.s[k];
    }
    return;
  }
  scalars_full(ctx, r, full);
#pragma unroll
  for (int k = 0; k < 10; ++k) {
    rem.s[k] = full.s[k];
    rem.s[k].re -= s0.s[k];
  }
}

// Highest power of the dense series a remainder at argument <= scale needs:
// ParSeries::rcut counts the parity-form terms t (powers par + 2t) whose
// size exceeds 1e-22 of the largest at that radius (scalars 2..9, the ones
// the Burton-Miller operator uses); the integrated forms only shrink them.
__device__ __forceinline__ int series_maxq_at(const DevCtx* __restrict__ ctx, double scale) {
  int nt = 1;
  for (int t = 1; t < kParTerms; ++t) nt += scale > ctx->pser.rcut[t];
  const int q = 2 * nt + 1;
  return q < ctx->series_maxq ? q : ctx->series_maxq;
}

// Closed form of int_0^1 u^upow rem(scale*u) du per scalar,
// proj/src/kernel_scalars.cpp:108-121,333-344.  Sets *bad when the element is
// too long for the frequency (the reference throws std::domain_error).
// The three weights upow = 1, 2, 3 of integrated_remainder from one pass
// over the series (same operations per weight as three separate calls).
__device__ __forceinline__ void integrated_remainder3(
    const DevCtx* __restrict__ ctx, double scale, Scalars (&o)[3], int* bad) {
  if (!(ctx->med.kT * scale < 2.5)) atomicExch(bad, 1);
  const double logc = log(scale);
  const int maxq = series_maxq_at(ctx, scale);
#pragma unroll
  for (int j = 0; j < 3; ++j)
#pragma unroll
    for (int k = 0; k < 10; ++k) o[j].s[k] = mk(0.0, 0.0);
  double cp = 1.0;
  for (int q = 0; q <= maxq; ++q) {
    double inv[3], inv2[3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      inv[j] = 1.0 / double(q + j + 2);
      inv2[j] = inv[j] * inv[j];
    }
#pragma unroll
    for (int k = 0; k < 10; ++k) {
      const double4 c = ld_series(ctx, k, q);
      const double ar = fma(c.z, logc, c.x), ai = fma(c.w, logc, c.y);
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const cplx t = mk(ar * inv[j] - c.z * inv2[j], ai * inv[j] - c.w * inv2[j]);
        axpy(o[j].s[k], cp, t);
      }
    }
    cp *= scale;
  }
}

__device__ __forceinline__ void integrated_remainder(
    const DevCtx* __restrict__ ctx, double scale, int upow, Scalars& o,
    int* bad) {
  if (!(ctx->med.kT * scale < 2.5)) atomicExch(bad, 1);
  const double logc = log(scale);
  const int maxq = ctx->series_maxq;
#pragma unroll
  for (int k = 0; k < 10; ++k) o.s[k] = mk(0.0, 0.0);
  double cp = 1.0;
  for (int q = 0; q <= maxq; ++q) {
    const double inv = 1.0 / double(q + upow + 1);
    const double inv2 = inv * inv;
#pragma unroll
    for (int k = 0; k < 10; ++k) {
      const double4 c = ld_series(ctx, k, q);
      // c^q [ (a + b ln c) inv - b inv^2 ]
      const cplx t = mk(fma(c.z, logc, c.x) * inv - c.z * inv2,
                        fma(c.w, logc, c.y) * inv - c.w * inv2);
      axpy(o.s[k], cp, t);
    }
    cp *= scale;
  }
}

// ----------------------------------------------------------------- combiners
// 2x2 complex tensor, row-major a11 a12 a21 a22.
struct CMat2 {
  cplx a[4];
};

// D_ij = -(d1 n_j zh_i + d2 ((n.zh) d_ij + n_i zh_j) + d3 (n.zh) zh_i zh_j)
__device__ __forceinline__ void combine_D(const Scalars& s, double zx,
                                          double zy, double nyx, double nyy,
                                          CMat2& m) {
  const double nz = nyx * zx + nyy * zy;
  const cplx d1 = s.s[2], d2 = s.s[3], d3 = s.s[4];
  m.a[0] = -(d1 * (nyx * zx) + d2 * (nz + nyx * zx) + d3 * (nz * zx * zx));
  m.a[1] = -(d1 * (nyy * zx) + d2 * (nyx * zy) + d3 * (nz * zx * zy));
  m.a[2] = -(d1 * (nyx * zy) + d2 * (nyy * zx) + d3 * (nz * zy * zx));
  m.a[3] = -(d1 * (nyy * zy) + d2 * (nz + nyy * zy) + d3 * (nz * zy * zy));
}

// Hypersingular kernel, m = observation normal (nx), n = source normal (ny).
__device__ __forceinline__ void combine_N(const Scalars& s, double zx,
                                          double zy, double mx, double my,
                                          double nx, double ny, CMat2& out) {
  const double mn = mx * nx + my * ny;
  const double mz = mx * zx + my * zy;
  const double nz = nx * zx + ny * zy;
  const double mv[2] = {mx, my}, nv[2] = {nx, ny}, zv[2] = {zx, zy};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double dij = (i == j) ? 1.0 : 0.0;
      const double c1 = mn * dij + nv[i] * mv[j];
      const double c2 = mn * zv[i] * zv[j] + mz * nz * dij + mz * nv[i] * zv[j] +
                        nz * zv[i] * mv[j];
      const double c4 = mz * nz * zv[i] * zv[j];
      const double c5 = mv[i] * nv[j];
      const double c7 = mz * zv[i] * nv[j] + nz * mv[i] * zv[j];
      out.a[2 * i + j] = s.s[5] * c1 + s.s[6] * c2 + s.s[7] * c4 +
                         s.s[8] * c5 + s.s[9] * c7;
    }
  }
}

// Integrated-by-parts static hypersingular kernel (real).
__device__ __forceinline__ void q0_kernel(double qfactor, double r, double zx,
                                          double zy, double q[4]) {
  const double lr = qfactor * log(r);
  q[0] = lr - qfactor * (zx * zx);
  q[1] = -qfactor * (zx * zy);
  q[2] = q[1];
  q[3] = lr - qfactor * (zy * zy);
}

// ------------------------------------------------------- fast D/N path
// The fill only ever needs the traction scalars d1, d2, d3 (always the full
// values) and the hypersingular scalars n1, n2, n4, n5, n7 (full for the
// proxy blocks, remainders for the exact Galerkin pairs): gpsi / gchi feed
// only G, which the Burton-Miller operator never uses.  One ln r per point
// serves the series branch, the Hankel small-argument log terms and q0.

// D/N series (scalars 2..9) staged in shared memory once per CTA, one row
// of 8 coefficients per power (d-series carry odd powers, n-series even
// powers; parity checked on the host).
struct SerSm {
  int ntmax;
  double2 at[kParTerms][8];
  double2 bt[kParTerms][8];
  double rcut[kParTerms];
};

__device__ __forceinline__ void load_sersm(const DevCtx* __restrict__ ctx, SerSm& s) {
  const int tid = threadIdx.x + blockDim.x * threadIdx.y;
  const int nth = blockDim.x * blockDim.y;
  for (int i = tid; i < 8 * kParTerms; i += nth) {
    const int k = i / kParTerms, p = i - k * kParTerms;
    s.at[p][k] = ctx->pser.a[k + 2][p];
    s.bt[p][k] = ctx->pser.b[k + 2][p];
  }
  for (int i = tid; i < kParTerms; i += nth) s.rcut[i] = ctx->pser.rcut[i];
  if (tid == 0) {
    int m = 0;
    for (int k = 0; k < 8; ++k) m = ctx->pser.nt[k + 2] > m ? ctx->pser.nt[k + 2] : m;
    s.ntmax = m;
  }
}

struct DN {
  cplx d[3];  // d1, d2, d3
  cplx n[5];  // n1, n2, n4, n5, n7
};

// H0, H1 with ln(x/2) supplied by the caller (small-argument branch).
__device__ __forceinline__ void hankel01_lg(double x, double log_half_x,
                                            cplx& h0, cplx& h1) {
  if (x <= 8.0) {
    const double q = x * 0.125;
    const double t = q * q;
    double j0, j1x, v0, v1;
    small_parts(x, t, j0, j1x, v0, v1);
    const double j1 = j1x * x;
    const double lg = kTwoOverPi * (log_half_x + kEulerGamma);
    const double y0 = fma(lg, j0, v0);
    const double y1 = v1 * x + lg * j1 - kTwoOverPi / x;
    h0 = mk(j0, y0);
    h1 = mk(j1, y1);
    return;
  }
  hankel01(x, h0, h1);
}

#ifndef EBEM_REAL_LOG
#define EBEM_REAL_LOG 0  // the real-B chains measured slower (426 vs 407 ms near field: schedule)
#endif
// All eight remainder series at once: one loop over powers, 16 independent
// Horner chains in u = r^2, started at the highest of the nt terms used.
// nt: ParSeries::rcut terms for the largest distance the caller sweeps.
__device__ __forceinline__ int series_terms(const SerSm& S, double rmax) {
  int nt = 1;
  for (int t = 1; t < S.ntmax; ++t) nt += rmax > S.rcut[t];
  return nt;
}
__device__ __forceinline__ void series_joint(const SerSm& S, double u, double logr,
                                             double r, int nt, DN& o) {
#if !EBEM_REAL_LOG
  cplx A[8], B[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 a = S.at[nt - 1][k], b = S.bt[nt - 1][k];
    A[k] = mk(a.x, a.y);
    B[k] = mk(b.x, b.y);
  }
  for (int p = nt - 2; p >= 0; --p) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double2 a = S.at[p][k], b = S.bt[p][k];
      A[k] = mk(fma(A[k].re, u, a.x), fma(A[k].im, u, a.y));
      B[k] = mk(fma(B[k].re, u, b.x), fma(B[k].im, u, b.y));
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k)
    o.d[k] = r * mk(fma(B[k].re, logr, A[k].re), fma(B[k].im, logr, A[k].im));
#pragma unroll
  for (int k = 0; k < 5; ++k)
    o.n[k] = mk(fma(B[3 + k].re, logr, A[3 + k].re), fma(B[3 + k].im, logr, A[3 + k].im));
#else
  // the log coefficients are real (the ln r terms come only from the real
  // Y0 part of H0; checked on the host), so B carries no imaginary chain
  cplx A[8];
  double B[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const double2 a = S.at[nt - 1][k];
    A[k] = mk(a.x, a.y);
    B[k] = S.bt[nt - 1][k].x;
  }
  for (int p = nt - 2; p >= 0; --p) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double2 a = S.at[p][k];
      A[k] = mk(fma(A[k].re, u, a.x), fma(A[k].im, u, a.y));
      B[k] = fma(B[k], u, S.bt[p][k].x);
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) o.d[k] = r * mk(fma(B[k], logr, A[k].re), A[k].im);
#pragma unroll
  for (int k = 0; k < 5; ++k) o.n[k] = mk(fma(B[3 + k], logr, A[3 + k].re), A[3 + k].im);
#endif
}

// series_joint with the first kFcTerms coefficients read from the
// __grid_constant__ FillConst: for a compile-time term count the Horner
// steps are DFMAs with constant-bank operands (no shared-memory loads).
template <int NT>
__device__ __forceinline__ void series_horner_c(const FillConst& fc, double u, double logr,
                                                double r, DN& o) {
#if EBEM_REAL_LOG
  cplx A[8];
  double B[8];  // real log coefficients (see series_joint)
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    A[k] = mk(fc.sa[NT - 1][k].x, fc.sa[NT - 1][k].y);
    B[k] = fc.sb[NT - 1][k].x;
  }
#pragma unroll
  for (int p = NT - 2; p >= 0; --p) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      A[k] = mk(fma(A[k].re, u, fc.sa[p][k].x), fma(A[k].im, u, fc.sa[p][k].y));
      B[k] = fma(B[k], u, fc.sb[p][k].x);
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k) o.d[k] = r * mk(fma(B[k], logr, A[k].re), A[k].im);
#pragma unroll
  for (int k = 0; k < 5; ++k) o.n[k] = mk(fma(B[3 + k], logr, A[3 + k].re), A[3 + k].im);
#else
  cplx A[8], B[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    A[k] = mk(fc.sa[NT - 1][k].x, fc.sa[NT - 1][k].y);
    B[k] = mk(fc.sb[NT - 1][k].x, fc.sb[NT - 1][k].y);
  }
#pragma unroll
  for (int p = NT - 2; p >= 0; --p) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      A[k] = mk(fma(A[k].re, u, fc.sa[p][k].x), fma(A[k].im, u, fc.sa[p][k].y));
      B[k] = mk(fma(B[k].re, u, fc.sb[p][k].x), fma(B[k].im, u, fc.sb[p][k].y));
    }
  }
#pragma unroll
  for (int k = 0; k < 3; ++k)
    o.d[k] = r * mk(fma(B[k].re, logr, A[k].re), fma(B[k].im, logr, A[k].im));
#pragma unroll
  for (int k = 0; k < 5; ++k)
    o.n[k] = mk(fma(B[3 + k].re, logr, A[3 + k].re), fma(B[3 + k].im, logr, A[3 + k].im));
#endif
}

#ifndef EBEM_SERIES_CONST
#define EBEM_SERIES_CONST 1
#endif
__device__ __forceinline__ void series_dispatch(const FillConst& fc, const SerSm& S, double u,
                                                double logr, double r, int nt, DN& o) {
#if EBEM_SERIES_CONST
  switch (nt) {
#define EBEM_HC(K) \
  case K:          \
    series_horner_c<K>(fc, u, logr, r, o); \
    return;
    EBEM_HC(1) EBEM_HC(2) EBEM_HC(3) EBEM_HC(4) EBEM_HC(5) EBEM_HC(6)
    EBEM_HC(7) EBEM_HC(8) EBEM_HC(9) EBEM_HC(10) EBEM_HC(11) EBEM_HC(12)
#undef EBEM_HC
    default:
      break;
  }
#endif
  series_joint(S, u, logr, r, nt, o);
}

// The scalars of one point.  kRem = false: full d and n (proxy blocks,
// kernel_cross_block); kRem = true: full d, remainder n
// (PairIntegrator::separated).  The medium constants come from the
// __grid_constant__ FillConst kernel parameter (constant-bank operands).
template <bool kRem>
__device__ __forceinline__ void dn_eval(const FillConst& fc, const SerSm& S,
                                        double r, double ir, double logr, int nt,
                                        DN& o) {
  const DevMedium& m = fc.med;
  const double ir2 = ir * ir;
  if (r < m.series_radius) {
    series_dispatch(fc, S, r * r, logr, r, nt, o);
    o.d[0].re += m.sd1 * ir;
    o.d[1].re -= m.sd1 * ir;
    o.d[2].re += m.sd3 * ir;
    if (!kRem) {
#pragma unroll
      for (int k = 0; k < 5; ++k) o.n[k].re += m.sn[k] * ir2;
    }
    return;
  }
  const double kT = m.kT, kL = m.kL, mu = m.mu, ar = m.aratio;
  cplx h0T, h1T, h0L, h1L;
  hankel01_lg(kT * r, logr + m.log_half_kT, h0T, h1T);
  hankel01_lg(kL * r, logr + m.log_half_kL, h0L, h1L);
  auto i4 = [](cplx z) { return mk(-0.25 * z.im, 0.25 * z.re); };
  const double izT = ir * m.inv_kT, izL = ir * m.inv_kL;
  const cplx chiL = i4(h0L);
  const cplx chiT1 = -(kT * i4(h1T));
  const cplx chiL1 = -(kL * i4(h1L));
  const cplx chiT2 = -(kT * kT) * i4(h0T - h1T * izT);
  const cplx chiL2 = -(kL * kL) * i4(h0L - h1L * izL);
  const cplx chiT3 = -(kT * kT * kT) * i4(-h1T - h0T * izT + (2.0 * izT * izT) * h1T);
  const cplx chiL3 = -(kL * kL * kL) * i4(-h1L - h0L * izL + (2.0 * izL * izL) * h1L);
  const cplx chiT4 = -(kT * kT * kT * kT) *
                     i4(-h0T + (2.0 * izT) * h1T + (3.0 * izT * izT) * h0T -
                        (6.0 * izT * izT * izT) * h1T);
  const cplx chiL4 = -(kL * kL * kL * kL) *
                     i4(-h0L + (2.0 * izL) * h1L + (3.0 * izL * izL) * h0L -
                        (6.0 * izL * izL * izL) * h1L);
  const double ikT2 = m.inv_kT * m.inv_kT;
  const cplx psi1 = (chiT1 - chiL1) * ikT2;
  const cplx psi2 = (chiT2 - chiL2) * ikT2;
  const cplx psi3 = (chiT3 - chiL3) * ikT2;
  const cplx psi4 = (chiT4 - chiL4) * ikT2;
  const cplx gchi = psi2 - psi1 * ir;
  const cplx w = gchi * ir;
  const cplx gam = gchi * ir2;
  const cplx bet = (psi3 - 3.0 * w) * ir;
  const cplx alf = psi4 - (6.0 * ir) * psi3 + 15.0 * gam;
  o.d[0] = ar * chiL1 + 2.0 * w;
  o.d[1] = chiT1 + 2.0 * w;
  o.d[2] = 2.0 * (psi3 - 3.0 * w);
  o.n[0] = (-2.0 * mu * ir) * chiT1 - (4.0 * mu) * gam;
  o.n[1] = (-mu) * (chiT2 - chiT1 * ir) - (4.0 * mu) * bet;
  o.n[2] = (-4.0 * mu) * alf;
  o.n[3] = m.c_n5 * chiL - (4.0 * mu * ar * ir) * chiL1 - (4.0 * mu) * gam;
  o.n[4] = (-2.0 * mu * ar) * (chiL2 - chiL1 * ir) - (4.0 * mu) * bet;
  if (kRem) {
#pragma unroll
    for (int k = 0; k < 5; ++k) o.n[k].re -= m.sn[k] * ir2;
  }
}

__device__ __forceinline__ void combine_D(const DN& s, double zx, double zy,
                                          double nyx, double nyy, CMat2& m) {
  const double nz = nyx * zx + nyy * zy;
  const cplx d1 = s.d[0], d2 = s.d[1], d3 = s.d[2];
  m.a[0] = -(d1 * (nyx * zx) + d2 * (nz + nyx * zx) + d3 * (nz * zx * zx));
  m.a[1] = -(d1 * (nyy * zx) + d2 * (nyx * zy) + d3 * (nz * zx * zy));
  m.a[2] = -(d1 * (nyx * zy) + d2 * (nyy * zx) + d3 * (nz * zy * zx));
  m.a[3] = -(d1 * (nyy * zy) + d2 * (nz + nyy * zy) + d3 * (nz * zy * zy));
}

__device__ __forceinline__ void combine_N(const DN& s, double zx, double zy,
                                          double mx, double my, double nx,
                                          double ny, CMat2& out) {
  const double mn = mx * nx + my * ny;
  const double mz = mx * zx + my * zy;
  const double nz = nx * zx + ny * zy;
  const double mv[2] = {mx, my}, nv[2] = {nx, ny}, zv[2] = {zx, zy};
#pragma unroll
  for (int i = 0; i < 2; ++i) {
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double dij = (i == j) ? 1.0 : 0.0;
      const double c1 = mn * dij + nv[i] * mv[j];
      const double c2 = mn * zv[i] * zv[j] + mz * nz * dij + mz * nv[i] * zv[j] +
                        nz * zv[i] * mv[j];
      const double c4 = mz * nz * zv[i] * zv[j];
      const double c5 = mv[i] * nv[j];
      const double c7 = mz * zv[i] * nv[j] + nz * mv[i] * zv[j];
      out.a[2 * i + j] = s.n[0] * c1 + s.n[1] * c2 + s.n[2] * c4 +
                         s.n[3] * c5 + s.n[4] * c7;
    }
  }
}

}  // namespace ebem_gpu
