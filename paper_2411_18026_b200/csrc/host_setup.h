#pragma once

#include "ebem_ctx.h"

namespace ebem_gpu {

DevMedium make_medium(double lam, double mu, double rho, double omega,
                      double alpha_re, double alpha_im);
// Fills out[10][max_pow][4]; returns the largest power present.
int build_series(const DevMedium& m, double* out, int max_pow);
void build_parity_series(const double* dense, int max_pow, ParSeries& ps);
void gauss_rule(int n, double* x, double* w);
void build_elements(const double* xy, int n, double* elem, double* hmin,
                    double* hmax);

}  // namespace ebem_gpu
