#pragma once
// Host tables of one problem: medium constants, the small-distance expansion
// of the kernel scalars, Gauss-Legendre rules, element geometry
// (medium_setup.cpp).
#include "ebem_ctx.h"

namespace ebem_gpu {

DevMedium make_medium(double lam, double mu, double rho, double omega,
                      double alpha_re, double alpha_im);
// Remainder expansion of the ten scalars: out[10][max_pow][4] =
// (Re a_q, Im a_q, Re b_q, Im b_q) of sum_q (a_q + b_q ln r) r^q; returns the
// largest power present.
int build_series(const DevMedium& m, double* out, int max_pow);
// The same coefficients regrouped by parity for Horner in r^2 on the device.
void build_parity_series(const double* dense, int max_pow, ParSeries& ps);
// n-point Gauss-Legendre rule on [0, 1], nodes ascending.
void gauss_rule(int n, double* x, double* w);
// Element table (ElemField planes) of the closed polygon through xy.
void build_elements(const double* xy, int n, double* elem, double* hmin,
                    double* hmax);
bool build_elements_range(const double* xy, int n, int e0, int e1, double* elem,
                          double* elem8, double* hmin, double* hmax);

}  // namespace ebem_gpu
