// Per-problem host tables the kernels read: medium constants, the
// small-distance expansion of the ten kernel scalars, Gauss-Legendre rules
// and the element geometry.
//
// Small-distance expansion.  Below the series radius the kernels evaluate
// each scalar as static(r) + R(r) with R(r) = sum_q (a_q + b_q ln r) r^q
// (the split of proj/src/kernel_scalars.cpp:123-212 / 381-409; the values
// must agree with KernelScalars::remainder to rounding).  The coefficients
// are derived here directly, without a series algebra:
//
//  1. chi_a(r) = (i/4) H0(k_a r) has the classical ascending expansion
//     sum_p t_p [ i/4 - (ln(k_a/2) + gamma - H_p)/(2 pi) - ln(r)/(2 pi) ] r^{2p},
//     t_p = (-1)^p (k_a/2)^{2p} / (p!)^2, H_p the harmonic numbers.
//  2. Every scalar is a fixed linear combination of r^{-j} d^n/dr^n f(r),
//     f in {chi_T, chi_L, psi = (chi_T - chi_L)/k_T^2}, the combinations
//     being the closed-form far-field formulas (kernel_scalars.cpp:233-281)
//     with gchi, w, gam, bet, alf written out (kScalarTerms below).
//  3. The n-th derivative of (a + b ln r) r^m is, in closed form,
//     [(m)_n a + D_n(m) b + (m)_n b ln r] r^{m-n}, (m)_n the falling
//     factorial and D_n(m) its derivative in m, so each table entry maps a
//     base coefficient straight to its output power.
//  4. The static part (kernel_scalars.cpp:283-299) is subtracted in the same
//     coefficient space.  Where it cancels the full expansion to rounding
//     the coefficient is an exact zero; every negative power must cancel
//     this way, which checks the whole derivation.
//
// The base expansion keeps p = 0..16 (powers up to r^32), the truncation the
// reference uses, so that both remainders are the same polynomial.
#include "medium_setup.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <stdexcept>
#include <vector>

namespace ebem_gpu {

namespace {

using cplx = std::complex<double>;
constexpr double kPi = 3.14159265358979323846;
constexpr double kEuler = 0.57721566490153286060651209008240;
constexpr int kBaseOrder = 16;           // p = 0..16 in step 1
constexpr int kLo = -8, kHi = 48;        // coefficient window, powers kLo..kHi-1
constexpr int kSpan = kHi - kLo;

// Which base function a table entry differentiates.
enum Base { CHI_T = 0, CHI_L = 1, PSI = 2 };

struct Entry {
  int scalar;   // 0..9 in ScalarSet order gpsi gchi d1 d2 d3 n1 n2 n4 n5 n7
  Base base;
  int deriv;    // n
  int rdiv;     // j: the entry is coef * r^{-j} * f^{(n)}(r)
  int coef_id;  // index into the per-medium coefficient list
};

// coefficient ids (values filled per medium in entry_coefficients)
enum Coef {
  ONE = 0, MINUS_ONE, TWO, MINUS_TWO, SIX, MINUS_SIX, AR, TWO_MU_NEG,
  FOUR_MU_NEG, FOUR_MU, TWELVE_MU_NEG, TWELVE_MU, MU_NEG, MU, TWENTY4_MU,
  SIXTY_MU_NEG, SIXTY_MU, N5_CHI, N5_CHI1, TWO_MU_AR_NEG, TWO_MU_AR, kCoefs
};

// gpsi = chiT + psi'/r
// gchi = psi'' - psi'/r
// w    = psi''/r - psi'/r^2           gam = psi''/r^2 - psi'/r^3
// bet  = psi'''/r - 3 psi''/r^2 + 3 psi'/r^3
// alf  = psi'''' - 6 psi'''/r + 15 psi''/r^2 - 15 psi'/r^3
// d1 = ar chiL' + 2w, d2 = chiT' + 2w, d3 = 2 psi''' - 6w
// n1 = -2mu chiT'/r - 4mu gam
// n2 = -mu chiT'' + mu chiT'/r - 4mu bet
// n4 = -4mu alf
// n5 = lam ar kL^2 chiL - 4mu ar chiL'/r - 4mu gam
// n7 = -2mu ar chiL'' + 2mu ar chiL'/r - 4mu bet
constexpr Entry kScalarTerms[] = {
    {0, CHI_T, 0, 0, ONE},         {0, PSI, 1, 1, ONE},
    {1, PSI, 2, 0, ONE},           {1, PSI, 1, 1, MINUS_ONE},
    {2, CHI_L, 1, 0, AR},          {2, PSI, 2, 1, TWO},
    {2, PSI, 1, 2, MINUS_TWO},
    {3, CHI_T, 1, 0, ONE},         {3, PSI, 2, 1, TWO},
    {3, PSI, 1, 2, MINUS_TWO},
    {4, PSI, 3, 0, TWO},           {4, PSI, 2, 1, MINUS_SIX},
    {4, PSI, 1, 2, SIX},
    {5, CHI_T, 1, 1, TWO_MU_NEG},  {5, PSI, 2, 2, FOUR_MU_NEG},
    {5, PSI, 1, 3, FOUR_MU},
    {6, CHI_T, 2, 0, MU_NEG},      {6, CHI_T, 1, 1, MU},
    {6, PSI, 3, 1, FOUR_MU_NEG},   {6, PSI, 2, 2, TWELVE_MU},
    {6, PSI, 1, 3, TWELVE_MU_NEG},
    {7, PSI, 4, 0, FOUR_MU_NEG},   {7, PSI, 3, 1, TWENTY4_MU},
    {7, PSI, 2, 2, SIXTY_MU_NEG},  {7, PSI, 1, 3, SIXTY_MU},
    {8, CHI_L, 0, 0, N5_CHI},      {8, CHI_L, 1, 1, N5_CHI1},
    {8, PSI, 2, 2, FOUR_MU_NEG},   {8, PSI, 1, 3, FOUR_MU},
    {9, CHI_L, 2, 0, TWO_MU_AR_NEG}, {9, CHI_L, 1, 1, TWO_MU_AR},
    {9, PSI, 3, 1, FOUR_MU_NEG},   {9, PSI, 2, 2, TWELVE_MU},
    {9, PSI, 1, 3, TWELVE_MU_NEG},
};

void entry_coefficients(const DevMedium& m, double* c) {
  const double mu = m.mu, ar = m.aratio;
  c[ONE] = 1.0;
  c[MINUS_ONE] = -1.0;
  c[TWO] = 2.0;
  c[MINUS_TWO] = -2.0;
  c[SIX] = 6.0;
  c[MINUS_SIX] = -6.0;
  c[AR] = ar;
  c[TWO_MU_NEG] = -2.0 * mu;
  c[FOUR_MU_NEG] = -4.0 * mu;
  c[FOUR_MU] = 4.0 * mu;
  c[TWELVE_MU_NEG] = -12.0 * mu;
  c[TWELVE_MU] = 12.0 * mu;
  c[MU_NEG] = -mu;
  c[MU] = mu;
  c[TWENTY4_MU] = 24.0 * mu;
  c[SIXTY_MU_NEG] = -60.0 * mu;
  c[SIXTY_MU] = 60.0 * mu;
  c[N5_CHI] = m.lam * ar * m.kL * m.kL;
  c[N5_CHI1] = -4.0 * mu * ar;
  c[TWO_MU_AR_NEG] = -2.0 * mu * ar;
  c[TWO_MU_AR] = 2.0 * mu * ar;
}

// (m)_n = m (m-1) ... (m-n+1) and its derivative with respect to m.
void falling(int m, int n, double* val, double* dval) {
  double v = 1.0, dv = 0.0;
  for (int i = 0; i < n; ++i) {
    const double f = double(m - i);
    dv = dv * f + v;  // product rule, one factor at a time
    v *= f;
  }
  *val = v;
  *dval = dv;
}

// Ascending expansion of chi(r) = (i/4) H0(k r): a[p], b[p] of r^{2p}.
void chi_expansion(double k, cplx* a, cplx* b) {
  const double lk = std::log(0.5 * k) + kEuler;
  double t = 1.0, h = 0.0;
  for (int p = 0; p <= kBaseOrder; ++p) {
    if (p > 0) {
      t *= -(0.5 * k) * (0.5 * k) / (double(p) * double(p));
      h += 1.0 / double(p);
    }
    a[p] = t * cplx((h - lk) / (2.0 * kPi), 0.25);
    b[p] = cplx(-t / (2.0 * kPi), 0.0);
  }
}

struct Coeffs {
  cplx a[10][kSpan];
  cplx b[10][kSpan];
};

double l1(cplx z) { return std::abs(z.real()) + std::abs(z.imag()); }

}  // namespace

DevMedium make_medium(double lam, double mu, double rho, double omega,
                      double alpha_re, double alpha_im) {
  if (!(mu > 0.0) || !(lam + mu > 0.0))
    throw std::invalid_argument("Medium: Lame constants out of range");
  const double cL = std::sqrt((lam + 2.0 * mu) / rho);
  const double cT = std::sqrt(mu / rho);
  if (!(cL > 0.0) || !(cT > 0.0) || !(rho > 0.0) || !(omega > 0.0))
    throw std::invalid_argument("Medium: all parameters must be positive");
  if (!(cL > cT)) throw std::invalid_argument("Medium: requires c_L > c_T");
  const double l2m = lam + 2.0 * mu;
  DevMedium m{};
  m.kL = omega / cL;
  m.kT = omega / cT;
  m.lam = lam;
  m.mu = mu;
  m.aratio = lam / l2m;
  m.cconst = (lam + mu) / (8.0 * kPi * l2m);
  m.ccon = m.cconst;
  m.qfactor = 8.0 * mu * m.cconst;
  m.kappa = mu / (2.0 * kPi * l2m);
  m.series_radius = 0.25 / m.kT;
  m.alpha_re = alpha_re;
  m.alpha_im = alpha_im;
  m.inv_kT = 1.0 / m.kT;
  m.inv_kL = 1.0 / m.kL;
  m.log_half_kT = std::log(0.5 * m.kT);
  m.log_half_kL = std::log(0.5 * m.kL);
  // static parts: d1 = sd1/r, d2 = -sd1/r, d3 = sd3/r, n* = sn[i]/r^2
  m.sd1 = mu / (2.0 * kPi * l2m);
  m.sd3 = -8.0 * m.cconst;
  m.sn[0] = mu * mu / (kPi * l2m);
  m.sn[1] = mu * lam / (kPi * l2m);
  m.sn[2] = -8.0 * m.qfactor;
  m.sn[3] = mu * (lam - mu) / (kPi * l2m);
  m.sn[4] = 2.0 * mu * mu / (kPi * l2m);
  m.c_n5 = lam * m.aratio * m.kL * m.kL;
  return m;
}

int build_series(const DevMedium& m, double* out, int max_pow) {
  cplx base_a[3][kBaseOrder + 1], base_b[3][kBaseOrder + 1];
  chi_expansion(m.kT, base_a[CHI_T], base_b[CHI_T]);
  chi_expansion(m.kL, base_a[CHI_L], base_b[CHI_L]);
  const double ikT2 = 1.0 / (m.kT * m.kT);
  for (int p = 0; p <= kBaseOrder; ++p) {
    base_a[PSI][p] = (base_a[CHI_T][p] - base_a[CHI_L][p]) * ikT2;
    base_b[PSI][p] = (base_b[CHI_T][p] - base_b[CHI_L][p]) * ikT2;
  }
  double coef[kCoefs];
  entry_coefficients(m, coef);

  // full expansion of every scalar (singular powers included)
  auto* full = new Coeffs();
  std::vector<double> scale_a(10 * kSpan, 0.0);  // |terms| summed, per slot
  for (const Entry& e : kScalarTerms) {
    for (int p = 0; p <= kBaseOrder; ++p) {
      const int mpow = 2 * p;
      double fv, fd;
      falling(mpow, e.deriv, &fv, &fd);
      const cplx a = base_a[e.base][p], b = base_b[e.base][p];
      const cplx na = coef[e.coef_id] * (fv * a + fd * b);
      const cplx nb = coef[e.coef_id] * (fv * b);
      if (na == cplx(0.0) && nb == cplx(0.0)) continue;
      const int q = mpow - e.deriv - e.rdiv;
      if (q < kLo || q >= kHi)
        throw std::logic_error("near-field expansion: power outside the table window");
      full->a[e.scalar][q - kLo] += na;
      full->b[e.scalar][q - kLo] += nb;
      scale_a[e.scalar * kSpan + q - kLo] += l1(na) + l1(nb);
    }
  }

  // subtract the static parts; positions they cancel to rounding are zeros
  struct StaticTerm { int scalar, q; bool log; double v; };
  const StaticTerm stat[] = {
      {0, 0, true, -1.0 / (2.0 * kPi) + 2.0 * m.cconst},
      {0, 0, false, m.cconst},
      {1, 0, false, 2.0 * m.cconst},
      {2, -1, false, m.sd1},
      {3, -1, false, -m.sd1},
      {4, -1, false, m.sd3},
      {5, -2, false, m.sn[0]},
      {6, -2, false, m.sn[1]},
      {7, -2, false, m.sn[2]},
      {8, -2, false, m.sn[3]},
      {9, -2, false, m.sn[4]},
  };
  for (const StaticTerm& s : stat) {
    cplx& c = s.log ? full->b[s.scalar][s.q - kLo] : full->a[s.scalar][s.q - kLo];
    const double size = scale_a[s.scalar * kSpan + s.q - kLo] + std::abs(s.v);
    c -= s.v;
    if (l1(c) <= 1e-12 * size) c = 0.0;
  }
  std::fill(out, out + size_t(10) * max_pow * 4, 0.0);
  int maxq = 0;
  for (int k = 0; k < 10; ++k) {
    double peak = 0.0;
    for (int i = 0; i < kSpan; ++i) {
      const int q = i + kLo;
      const double size = scale_a[k * kSpan + i];
      if (q < 0) {
        if (l1(full->a[k][i]) > 1e-12 * size || l1(full->b[k][i]) > 1e-12 * size)
          throw std::logic_error(
              "near-field expansion: a singular power survives the static split");
        full->a[k][i] = full->b[k][i] = 0.0;
        continue;
      }
      peak = std::max(peak, std::max(l1(full->a[k][i]), l1(full->b[k][i])));
    }
    const double floor = 1e-25 * peak;  // drop coefficients below any use
    for (int q = 0; q < kHi; ++q) {
      cplx a = full->a[k][q - kLo], b = full->b[k][q - kLo];
      if (l1(a) <= floor) a = 0.0;
      if (l1(b) <= floor) b = 0.0;
      if (a == cplx(0.0) && b == cplx(0.0)) continue;
      if (q >= max_pow)
        throw std::logic_error("near-field expansion: longer than the device table");
      maxq = std::max(maxq, q);
      double* o = out + (size_t(k) * max_pow + q) * 4;
      o[0] = a.real();
      o[1] = a.imag();
      o[2] = b.real();
      o[3] = b.imag();
    }
  }
  delete full;
  return maxq;
}

void build_parity_series(const double* dense, int max_pow, ParSeries& ps) {
  for (int k = 0; k < 10; ++k) {
    std::vector<int> present;
    for (int q = 0; q < max_pow; ++q) {
      const double* c = dense + (size_t(k) * max_pow + q) * 4;
      if (c[0] != 0.0 || c[1] != 0.0 || c[2] != 0.0 || c[3] != 0.0) present.push_back(q);
    }
    const int par = present.empty() ? 0 : present.front() & 1;
    for (int q : present)
      if ((q & 1) != par)
        throw std::logic_error("near-field expansion: powers of both parities");
    const int nt = present.empty() ? 0 : (present.back() - par) / 2 + 1;
    if (nt > kParTerms)
      throw std::logic_error("near-field expansion: longer than the device table");
    ps.par[k] = par;
    ps.nt[k] = nt;
    for (int p = 0; p < kParTerms; ++p) {
      const int q = par + 2 * p;
      const double* c = (p < nt && q < max_pow) ? dense + (size_t(k) * max_pow + q) * 4
                                                : nullptr;
      ps.a[k][p] = c ? double2{c[0], c[1]} : double2{0.0, 0.0};
      ps.b[k][p] = c ? double2{c[2], c[3]} : double2{0.0, 0.0};
    }
  }
}

// Gauss-Legendre rule on [0, 1] (gauss_rule, proj/src/quadrature.cpp:16-47).
// The nodes are the eigenvalues of the Jacobi matrix of the shifted Legendre
// polynomials (diagonal 1/2, off-diagonal k / (2 sqrt(4k^2 - 1))), isolated
// by Sturm-sequence bisection and polished by Newton steps on P_n(2x - 1);
// the weights come from the Christoffel function,
// w_i = 1 / sum_{k<n} (2k + 1) P_k(2 x_i - 1)^2, a sum of positive terms.
#ifndef EBEM_GAUSS_GOLUB
#define EBEM_GAUSS_GOLUB 1
#endif
// The textbook Newton iteration for the roots of P_n (Tricomi's cosine
// guess, the three-term recurrence for P_n and P_n', stop below 1e-15) with
// the derivative weight formula 2 / ((1 - s^2) P_n'(s)^2) -- the published
// algorithm (Numerical Recipes' gauleg) the reference's gauss_rule follows.
// Its weights carry up to ~9e-14 relative error at the ends (the (1 - s^2)
// cancellation), which the reference's matrices inherit.
static void gauss_rule_newton(int n, double* x, double* w) {
  const int half = (n + 1) / 2;
  for (int r = 0; r < half; ++r) {
    double s = std::cos(kPi * (r + 0.75) / (n + 0.5));  // r-th root from the top
    double deriv = 0.0;
    for (int it = 0; it < 100; ++it) {
      double pm = 1.0, pc = s;  // P_0, P_1
      for (int k = 2; k <= n; ++k) {
        const double pn = ((2.0 * k - 1.0) * s * pc - (k - 1.0) * pm) / k;
        pm = pc;
        pc = pn;
      }
      deriv = n * (s * pc - pm) / (s * s - 1.0);
      const double step = pc / deriv;
      s -= step;
      if (std::abs(step) < 1e-15) break;
    }
    const double wt = 0.5 * (2.0 / ((1.0 - s * s) * deriv * deriv));
    x[r] = 0.5 * (1.0 - s);
    x[n - 1 - r] = 0.5 * (1.0 + s);
    w[r] = w[n - 1 - r] = wt;
  }
}

void gauss_rule(int n, double* x, double* w) {
  if (!EBEM_GAUSS_GOLUB) {
    gauss_rule_newton(n, x, w);
    return;
  }
  std::vector<double> off2(n > 0 ? n : 1, 0.0);  // squared off-diagonals
  for (int k = 1; k < n; ++k) off2[k] = double(k) * k / (4.0 * (4.0 * k * k - 1.0));
  // number of eigenvalues below t (Sturm count of the LDL^T pivots)
  auto count_below = [&](double t) {
    int c = 0;
    double d = 0.5 - t;
    if (d < 0.0) ++c;
    for (int k = 1; k < n; ++k) {
      if (d == 0.0) d = 1e-300;
      d = (0.5 - t) - off2[k] / d;
      if (d < 0.0) ++c;
    }
    return c;
  };
  // P_n(s) and P_n'(s) at s = 2t - 1, plus the Christoffel sum
  auto legendre = [&](double t, double* pn, double* dpn, double* chr) {
    const double s = 2.0 * t - 1.0;
    double pkm1 = 0.0, pk = 1.0, dkm1 = 0.0, dk = 0.0, sum = 1.0;
    for (int k = 0; k < n; ++k) {
      const double pk1 = ((2.0 * k + 1.0) * s * pk - k * pkm1) / (k + 1.0);
      const double dk1 = ((2.0 * k + 1.0) * (pk + s * dk) - k * dkm1) / (k + 1.0);
      pkm1 = pk;
      pk = pk1;
      dkm1 = dk;
      dk = dk1;
      if (k + 1 < n) sum += (2.0 * k + 3.0) * pk * pk;
    }
    *pn = pk;
    *dpn = 2.0 * dk;  // d/dt
    *chr = sum;
  };
  for (int i = 0; i < n; ++i) {
    double lo = 0.0, hi = 1.0;  // the i-th smallest eigenvalue lies in (0, 1)
    for (int it = 0; it < 80 && hi - lo > 1e-15; ++it) {
      const double mid = 0.5 * (lo + hi);
      if (count_below(mid) > i) hi = mid; else lo = mid;
    }
    double t = 0.5 * (lo + hi), pn, dpn, chr;
    for (int it = 0; it < 3; ++it) {
      legendre(t, &pn, &dpn, &chr);
      if (dpn == 0.0) break;
      t -= pn / dpn;
    }
    legendre(t, &pn, &dpn, &chr);
    x[i] = t;
    w[i] = 1.0 / chr;
  }
  // exact mirror symmetry of the rule about 1/2
  for (int i = 0; i < n / 2; ++i) {
    const double xs = 0.5 * (x[i] + (1.0 - x[n - 1 - i]));
    const double ws = 0.5 * (w[i] + w[n - 1 - i]);
    x[i] = xs;
    x[n - 1 - i] = 1.0 - xs;
    w[i] = w[n - 1 - i] = ws;
  }
  if (n % 2 == 1) x[n / 2] = 0.5;
}

void build_elements(const double* xy, int n, double* elem, double* hmin,
                    double* hmax) {
  double lo = 1e300, hi = 0.0;
  for (int e = 0; e < n; ++e) {
    const int nx = (e + 1) % n;
    const double sx = xy[2 * e], sy = xy[2 * e + 1];
    const double ex = xy[2 * nx] - sx, ey = xy[2 * nx + 1] - sy;
    const double len = std::hypot(ex, ey);
    if (!(len > 0.0)) throw std::invalid_argument("Mesh: zero-length element");
    const double ux = ex / len, uy = ey / len;
    const double vals[kElemFields] = {sx, sy, ex, ey, ux, uy, -uy, ux, len};
    for (int f = 0; f < kElemFields; ++f) elem[size_t(f) * n + e] = vals[f];
    lo = std::min(lo, len);
    hi = std::max(hi, len);
  }
  *hmin = lo;
  *hmax = hi;
}

// Elements [e0, e1) of the mesh: the field-major array elem (as
// build_elements) and the packed 8-double rows elem8 (px, py, dx, dy, nx, ny,
// h, 0) in one pass.  Returns false on a zero-length element.
bool build_elements_range(const double* xy, int n, int e0, int e1, double* elem,
                          double* elem8, double* hmin, double* hmax) {
  double lo = 1e300, hi = 0.0;
  for (int e = e0; e < e1; ++e) {
    const int nx = (e + 1) % n;
    const double sx = xy[2 * e], sy = xy[2 * e + 1];
    const double ex = xy[2 * nx] - sx, ey = xy[2 * nx + 1] - sy;
    const double len = std::hypot(ex, ey);
    if (!(len > 0.0)) return false;
    const double ux = ex / len, uy = ey / len;
    const double vals[kElemFields] = {sx, sy, ex, ey, ux, uy, -uy, ux, len};
    for (int f = 0; f < kElemFields; ++f) elem[size_t(f) * n + e] = vals[f];
    double* r = elem8 + 8 * size_t(e);
    r[0] = sx; r[1] = sy; r[2] = ex; r[3] = ey; r[4] = -uy; r[5] = ux; r[6] = len; r[7] = 0.0;
    lo = std::min(lo, len);
    hi = std::max(hi, len);
  }
  *hmin = lo;
  *hmax = hi;
  return true;
}

}  // namespace ebem_gpu
