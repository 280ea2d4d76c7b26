// Host-side setup of the per-medium tables the kernels read: the log-power
// remainder series of the ten kernel scalars, Gauss-Legendre rules, element
// geometry.  Restated from the reference's published algorithm:
//   KernelScalars ctor    proj/src/kernel_scalars.cpp:123-212 (LogSeries ops
//                         :28-106)
//   make_rule             proj/src/quadrature.cpp:16-47
//   Mesh ctor             proj/src/geometry.cpp:15-37
#include "host_setup.h"

#include <algorithm>
#include <cmath>
#include <complex>
#include <map>
#include <stdexcept>

namespace ebem_gpu {

namespace {

using cd = std::complex<double>;
constexpr double kPiD = 3.14159265358979323846;
constexpr double kGamma = 0.57721566490153286060651209008240;
constexpr int kTerms = 16;  // retained powers r^{2p}, p = 0..16

double mag(cd z) { return std::abs(z.real()) + std::abs(z.imag()); }

// sum_q (a_q + b_q ln r) r^q keyed by the power q.
class PowLog {
 public:
  void add(int q, cd a, cd b) {
    auto it = t_.find(q);
    if (it == t_.end()) {
      t_.emplace(q, std::make_pair(a, b));
    } else {
      it->second.first += a;
      it->second.second += b;
    }
  }
  PowLog d() const {  // d/dr: (q a + b + q b ln r) r^{q-1}
    PowLog o;
    for (const auto& [q, ab] : t_) {
      const cd a = double(q) * ab.first + ab.second;
      const cd b = double(q) * ab.second;
      if (a != cd(0.0) || b != cd(0.0)) o.add(q - 1, a, b);
    }
    return o;
  }
  PowLog over_r(int p = 1) const {
    PowLog o;
    for (const auto& [q, ab] : t_) o.add(q - p, ab.first, ab.second);
    return o;
  }
  PowLog times(cd f) const {
    PowLog o;
    for (const auto& [q, ab] : t_) o.add(q, f * ab.first, f * ab.second);
    return o;
  }
  PowLog plus(const PowLog& other, cd f = cd(1.0)) const {
    PowLog o = *this;
    for (const auto& [q, ab] : other.t_) o.add(q, f * ab.first, f * ab.second);
    return o;
  }
  double peak() const {
    double p = 0.0;
    for (const auto& kv : t_)
      p = std::max(p, std::max(mag(kv.second.first), mag(kv.second.second)));
    return p;
  }
  void prune(double rel = 1e-25) {
    const double cut = rel * peak();
    std::map<int, std::pair<cd, cd>> kept;
    for (const auto& [q, ab] : t_) {
      const cd a = mag(ab.first) > cut ? ab.first : cd(0.0);
      const cd b = mag(ab.second) > cut ? ab.second : cd(0.0);
      if (a != cd(0.0) || b != cd(0.0)) kept.emplace(q, std::make_pair(a, b));
    }
    t_.swap(kept);
  }
  void drop_log(int q) {
    const double p = peak();
    auto it = t_.find(q);
    if (it == t_.end()) return;
    if (mag(it->second.second) > 1e-10 * p)
      throw std::logic_error("LogSeries: log coefficient is not negligible");
    it->second.second = cd(0.0);
  }
  int min_q() const { return t_.empty() ? 0 : t_.begin()->first; }
  int max_q() const { return t_.empty() ? 0 : t_.rbegin()->first; }
  const std::map<int, std::pair<cd, cd>>& terms() const { return t_; }

 private:
  std::map<int, std::pair<cd, cd>> t_;
};

// chi_a + ln(r)/(2 pi) with chi_a = (i/4) H0(k r), as a series in r^{2p}.
PowLog chi_regular(double k) {
  PowLog s;
  const cd c0 = cd(0.0, 0.25) - (std::log(0.5 * k) + kGamma) / (2.0 * kPiD);
  double ap = 1.0, harm = 0.0;
  for (int p = 0; p <= kTerms; ++p) {
    if (p > 0) {
      ap *= -0.25 * k * k / (double(p) * double(p));
      harm += 1.0 / double(p);
    }
    const cd A = ap * (c0 + harm / (2.0 * kPiD));
    const cd B = (p == 0) ? cd(0.0) : cd(-ap / (2.0 * kPiD));
    s.add(2 * p, A, B);
  }
  return s;
}

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
  DevMedium m{};
  m.kL = omega / cL;
  m.kT = omega / cT;
  m.lam = lam;
  m.mu = mu;
  m.aratio = lam / (lam + 2.0 * mu);
  m.cconst = (lam + mu) / (8.0 * kPiD * (lam + 2.0 * mu));
  m.qfactor = 8.0 * mu * m.cconst;
  m.series_radius = 0.25 / m.kT;
  m.kappa = mu / (2.0 * kPiD * (lam + 2.0 * mu));
  m.ccon = (lam + mu) / (8.0 * kPiD * (lam + 2.0 * mu));
  m.alpha_re = alpha_re;
  m.alpha_im = alpha_im;
  m.inv_kT = 1.0 / m.kT;
  m.inv_kL = 1.0 / m.kL;
  m.log_half_kT = std::log(0.5 * m.kT);
  m.log_half_kL = std::log(0.5 * m.kL);
  const double l2m = lam + 2.0 * mu;
  m.sd1 = mu / (2.0 * kPiD * l2m);
  m.sd3 = -8.0 * m.cconst;
  m.sn[0] = mu * mu / (kPiD * l2m);
  m.sn[1] = mu * lam / (kPiD * l2m);
  m.sn[2] = -8.0 * m.qfactor;
  m.sn[3] = mu * (lam - mu) / (kPiD * l2m);
  m.sn[4] = 2.0 * mu * mu / (kPiD * l2m);
  m.c_n5 = lam * m.aratio * m.kL * m.kL;
  return m;
}

int build_series(const DevMedium& m, double* out, int max_pow) {
  const double kT = m.kT, kL = m.kL, lam = m.lam, mu = m.mu;
  const double ar = m.aratio, cc = m.cconst;
  const PowLog chiT = chi_regular(kT);
  const PowLog chiL = chi_regular(kL);
  PowLog psi = chiT.plus(chiL, cd(-1.0)).times(cd(1.0 / (kT * kT)));
  psi.add(2, cd(0.0), cd(-cc));
  psi.drop_log(2);
  psi.prune();
  const PowLog psi1 = psi.d(), psi2 = psi1.d(), psi3 = psi2.d(), psi4 = psi3.d();
  const PowLog chiT1 = chiT.d(), chiT2 = chiT1.d();
  const PowLog chiL1 = chiL.d(), chiL2 = chiL1.d();

  PowLog gpsi = chiT.plus(psi1.over_r());
  PowLog gchi = psi2.plus(psi1.over_r(), cd(-1.0));
  gchi.prune();
  const PowLog w = gchi.over_r();
  const PowLog gam = gchi.over_r(2);
  PowLog bet = psi3.plus(w, cd(-3.0)).over_r();
  bet.prune();
  PowLog alf = psi4.plus(psi3.over_r(), cd(-6.0)).plus(gam, cd(15.0));
  alf.prune();
  PowLog d1 = chiL1.times(cd(ar)).plus(w, cd(2.0));
  PowLog d2 = chiT1.plus(w, cd(2.0));
  PowLog d3 = psi3.plus(w, cd(-3.0)).times(cd(2.0));
  PowLog n1 = chiT1.over_r().times(cd(-2.0 * mu)).plus(gam, cd(-4.0 * mu));
  PowLog n2 = chiT2.plus(chiT1.over_r(), cd(-1.0)).times(cd(-mu)).plus(bet, cd(-4.0 * mu));
  PowLog n4 = alf.times(cd(-4.0 * mu));
  PowLog n5 = chiL.times(cd(lam * ar * kL * kL))
                  .plus(chiL1.over_r(), cd(-4.0 * mu * ar))
                  .plus(gam, cd(-4.0 * mu));
  n5.add(0, cd(0.0), cd(-lam * ar * kL * kL / (2.0 * kPiD)));
  PowLog n7 = chiL2.plus(chiL1.over_r(), cd(-1.0))
                  .times(cd(-2.0 * mu * ar))
                  .plus(bet, cd(-4.0 * mu));
  PowLog all[10] = {gpsi, gchi, d1, d2, d3, n1, n2, n4, n5, n7};
  int maxq = 0;
  std::fill(out, out + 10 * max_pow * 4, 0.0);
  for (int k = 0; k < 10; ++k) {
    all[k].prune();
    if (all[k].min_q() < 0)
      throw std::logic_error("KernelScalars: remainder series kept a negative power");
    maxq = std::max(maxq, all[k].max_q());
    if (all[k].max_q() >= max_pow)
      throw std::logic_error("KernelScalars: series longer than the device table");
    for (const auto& [q, ab] : all[k].terms()) {
      double* o = out + (k * max_pow + q) * 4;
      o[0] = ab.first.real();
      o[1] = ab.first.imag();
      o[2] = ab.second.real();
      o[3] = ab.second.imag();
    }
  }
  return maxq;
}

void build_parity_series(const double* dense, int max_pow, ParSeries& ps) {
  for (int k = 0; k < 10; ++k) {
    int lo = -1, hi = -1;
    for (int q = 0; q < max_pow; ++q) {
      const double* c = dense + (k * max_pow + q) * 4;
      if (c[0] != 0.0 || c[1] != 0.0 || c[2] != 0.0 || c[3] != 0.0) {
        if (lo < 0) lo = q;
        hi = q;
        if ((q - lo) % 2 != 0)
          throw std::logic_error("KernelScalars: series of mixed parity");
      }
    }
    ps.par[k] = lo < 0 ? 0 : lo % 2;
    ps.nt[k] = lo < 0 ? 0 : (hi - ps.par[k]) / 2 + 1;
    if (ps.nt[k] > kParTerms)
      throw std::logic_error("KernelScalars: series longer than the device table");
    for (int p = 0; p < kParTerms; ++p) {
      const int q = ps.par[k] + 2 * p;
      const double* c = (p < ps.nt[k] && q < max_pow) ? dense + (k * max_pow + q) * 4 : nullptr;
      ps.a[k][p] = c ? double2{c[0], c[1]} : double2{0.0, 0.0};
      ps.b[k][p] = c ? double2{c[2], c[3]} : double2{0.0, 0.0};
    }
  }
}

void gauss_rule(int n, double* x, double* w) {
  for (int i = 0; i < (n + 1) / 2; ++i) {
    double z = std::cos(kPiD * (i + 0.75) / (n + 0.5));
    double dp = 0.0;
    for (int iter = 0; iter < 100; ++iter) {
      double p0 = 1.0, p1 = z;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (z * p1 - p0) / (z * z - 1.0);
      const double dz = p1 / dp;
      z -= dz;
      if (std::abs(dz) < 1e-15) break;
    }
    const double wt = 2.0 / ((1.0 - z * z) * dp * dp);
    x[i] = 0.5 * (1.0 - z);
    w[i] = 0.5 * wt;
    x[n - 1 - i] = 0.5 * (1.0 + z);
    w[n - 1 - i] = 0.5 * wt;
  }
}

void build_elements(const double* xy, int n, double* elem, double* hmin,
                    double* hmax) {
  *hmin = 1e300;
  *hmax = 0.0;
  for (int e = 0; e < n; ++e) {
    const int f = e + 1 == n ? 0 : e + 1;
    const double px = xy[2 * e], py = xy[2 * e + 1];
    const double dx = xy[2 * f] - px, dy = xy[2 * f + 1] - py;
    const double h = std::hypot(dx, dy);
    if (!(h > 0.0)) throw std::invalid_argument("Mesh: zero-length element");
    const double tx = dx / h, ty = dy / h;
    elem[size_t(EPX) * n + e] = px;
    elem[size_t(EPY) * n + e] = py;
    elem[size_t(EDX) * n + e] = dx;
    elem[size_t(EDY) * n + e] = dy;
    elem[size_t(ETX) * n + e] = tx;
    elem[size_t(ETY) * n + e] = ty;
    elem[size_t(ENX) * n + e] = -ty;
    elem[size_t(ENY) * n + e] = tx;
    elem[size_t(EH) * n + e] = h;
    *hmin = std::min(*hmin, h);
    *hmax = std::max(*hmax, h);
  }
}

}  // namespace ebem_gpu
