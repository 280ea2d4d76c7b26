// Dense reference solver on the device: the full Galerkin matrix
// (BlockAssembler::dense, proj/src/assembly.cpp:311-330) factored once by
// partial-pivoted LU (ConvSolver, proj/src/dense_solver.cpp:9-29; LuFactor,
// proj/src/lapack.cpp:31-99).  The matrix is filled by the symmetric
// near-field machinery (one evaluation per element pair for both
// orientations, the same ordered gather as true_block, so sub-blocks equal
// true_block), factored by the blocked LU, and the 1-norm condition number is
// estimated with LAPACK zlacn2's iteration (the estimator zgecon uses) on
// device solves with A and A^H.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <string>
#include <vector>

#include "ebem_kernels.h"
#include "runtime.h"

namespace ebem_gpu {

namespace {
constexpr double kConditionWarningThreshold = 1e-12;  // dense_solver.cpp:6
double now_s() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
}  // namespace

void Conv::assemble(Problem& P, double* dest) {
  const int n = P.n();
  std::vector<int> nodes(n);
  for (int i = 0; i < n; ++i) nodes[i] = i;
  FillPlan plan(n, P.proxy_cfg().m_prime, P.proxy_cfg().n_gauss);
  plan.add_sym_diag(nodes, dest, 2 * n);
  P.execute(plan);
  P.check_domain();
}

void Conv::check_size(const Problem& P) {
  const size_t d = 2 * size_t(P.n());
  if (d * d * 16 > P.asm_cfg().max_dense_bytes)
    throw Error(EBEM_LENGTH_ERROR,
                "BlockAssembler::dense: matrix exceeds the configured memory budget");
}

Conv::Conv(Problem& p) : P_(p), d_(2 * p.n()) {
  check_size(P_);
  cudaStream_t st = P_.stream();
  const size_t dd = size_t(d_) * d_;
  lu_.alloc(2 * dd + 2);
  ipiv_.alloc(d_ + 1);
  info_.alloc(1);
  double t0 = now_s();
  assemble(P_, lu_.get());
  // ||A||_1 before the factorization (LuFactor ctor, lapack.cpp:36-39)
  DBuf<double> cs;
  cs.alloc(d_ + 1);
  launch_col_abs_sum(lu_.get(), d_, d_, cs.get(), st);
  std::vector<double> h(d_);
  CK(cudaMemcpyAsync(h.data(), cs.get(), 8 * size_t(d_), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  stats_.assemble_seconds = now_s() - t0;
  norm1_ = 0.0;
  for (double v : h) norm1_ = std::max(norm1_, v);
  t0 = now_s();
  LuTask t{};
  t.a = lu_.get();
  t.ipiv = ipiv_.get();
  t.info = info_.get();
  t.n = d_;
  t.ld = d_;
  CK(cudaMemsetAsync(info_.get(), 0, sizeof(int), st));
  run_getrf(P_, {t});
  int info = 0;
  CK(cudaMemcpyAsync(&info, info_.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  stats_.factor_seconds = now_s() - t0;
  if (info > 0)
    throw Error(EBEM_RUNTIME_ERROR, "LuFactor: matrix is singular, zero pivot at index " +
                                        std::to_string(info - 1) + " of " +
                                        std::to_string(d_));
  // min |U_ii| (LuFactor::min_pivot, lapack.cpp:55-59)
  std::vector<double> diag(2 * size_t(d_));
  CK(cudaMemcpy2DAsync(diag.data(), 16, lu_.get(), 16 * (size_t(d_) + 1), 16, d_,
                       cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  double mp = std::numeric_limits<double>::infinity();
  for (int i = 0; i < d_; ++i) mp = std::min(mp, std::hypot(diag[2 * i], diag[2 * i + 1]));
  stats_.min_pivot = d_ == 0 ? 0.0 : mp;
  stats_.rcond = rcond();
  stats_.condition_warning = stats_.rcond < kConditionWarningThreshold;
}

// x := A^-1 x (one column, device)
void Conv::apply_inv(double* x) {
  LuSolveTask s{lu_.get(), ipiv_.get(), x, d_, d_, 1, d_};
  run_getrs(P_, {s});
}

// x := A^-H x
void Conv::apply_inv_h(double* x) {
  launch_getrs_conj(lu_.get(), d_, d_, ipiv_.get(), x, P_.stream());
  CK(cudaGetLastError());
}

// zgecon('1'): rcond = 1 / (||A||_1 est(||A^-1||_1)), the estimate by the
// zlacn2 iteration (Hager / Higham): power steps with sign vectors, at most
// five, then the alternating-sign test vector.
double Conv::rcond() {
  const int n = d_;
  if (n == 0) return 1.0;
  if (norm1_ == 0.0) return 0.0;
  cudaStream_t st = P_.stream();
  DBuf<double> dx;
  dx.alloc(2 * size_t(n) + 2);
  std::vector<double> x(2 * size_t(n)), y(2 * size_t(n));
  auto run = [&](bool herm) {
    CK(cudaMemcpyAsync(dx.get(), x.data(), 16 * size_t(n), cudaMemcpyHostToDevice, st));
    if (herm) apply_inv_h(dx.get());
    else apply_inv(dx.get());
    CK(cudaMemcpyAsync(y.data(), dx.get(), 16 * size_t(n), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  };
  auto sum_abs = [&]() {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += std::hypot(y[2 * i], y[2 * i + 1]);
    return s;
  };
  auto sign_of_y = [&]() {  // x_i = y_i / |y_i| (1 when |y_i| is tiny)
    const double safmin = std::numeric_limits<double>::min();
    for (int i = 0; i < n; ++i) {
      const double a = std::hypot(y[2 * i], y[2 * i + 1]);
      if (a > safmin) {
        x[2 * i] = y[2 * i] / a;
        x[2 * i + 1] = y[2 * i + 1] / a;
      } else {
        x[2 * i] = 1.0;
        x[2 * i + 1] = 0.0;
      }
    }
  };
  auto argmax_abs = [&]() {
    int j = 0;
    double best = -1.0;
    for (int i = 0; i < n; ++i) {
      const double a = std::hypot(y[2 * i], y[2 * i + 1]);
      if (a > best) { best = a; j = i; }
    }
    return j;
  };
  for (int i = 0; i < n; ++i) x[2 * i] = 1.0 / n, x[2 * i + 1] = 0.0;
  run(false);
  double est;
  if (n == 1) {
    est = std::hypot(y[0], y[1]);
  } else {
    est = sum_abs();
    sign_of_y();
    run(true);
    int j = argmax_abs();
    for (int iter = 2; iter <= 5; ++iter) {
      std::fill(x.begin(), x.end(), 0.0);
      x[2 * j] = 1.0;
      run(false);
      const double estold = est;
      est = sum_abs();
      if (est <= estold) break;
      sign_of_y();
      run(true);
      const int jlast = j;
      j = argmax_abs();
      if (std::hypot(y[2 * jlast], y[2 * jlast + 1]) == std::hypot(y[2 * j], y[2 * j + 1]))
        break;
    }
    double altsgn = 1.0;  // x_i = (-1)^i (1 + i / (n - 1))
    for (int i = 0; i < n; ++i) {
      x[2 * i] = altsgn * (1.0 + double(i) / double(n - 1));
      x[2 * i + 1] = 0.0;
      altsgn = -altsgn;
    }
    run(false);
    const double temp = 2.0 * sum_abs() / (3.0 * n);
    if (temp > est) est = temp;
  }
  return est == 0.0 ? 0.0 : (1.0 / est) / norm1_;
}

void Conv::solve_host(const double* rhs, int m, double* x) {
  if (m <= 0 || d_ == 0) return;
  cudaStream_t st = P_.stream();
  DBuf<double> b;
  b.alloc(2 * size_t(d_) * m);
  CK(cudaMemcpyAsync(b.get(), rhs, 16 * size_t(d_) * m, cudaMemcpyHostToDevice, st));
  LuSolveTask s{lu_.get(), ipiv_.get(), b.get(), d_, d_, m, d_};
  run_getrs(P_, {s});
  CK(cudaMemcpyAsync(x, b.get(), 16 * size_t(d_) * m, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
}

void Conv::dense_host(Problem& P, double* out) {
  check_size(P);
  const size_t d = 2 * size_t(P.n());
  DBuf<double> a;
  a.alloc(2 * d * d + 2);
  assemble(P, a.get());
  CK(cudaMemcpyAsync(out, a.get(), 16 * d * d, cudaMemcpyDeviceToHost, P.stream()));
  CK(cudaStreamSynchronize(P.stream()));
}

}  // namespace ebem_gpu
