// C entry points over the reference library compiled in place -- TEST
// INFRASTRUCTURE ONLY (the checker and the CPU baseline, never the product).
//
// oracle/Makefile compiles /root/reference/proj/src/{hankel,geometry,
// kernel_scalars,kernels,quadrature,assembly,lapack,compression,fds,
// dense_solver}.cpp where they lie, against oracle/eigen_shim, and links this
// file into oracle/_ref/libebem_ref.so.  Only tests/, bench.py's reference arm
// and __graft_entry__.smoke() load it.
//
// Every function forwards to the reference's own public API:
//   hankel1_01                   proj/src/hankel.cpp:34
//   KernelScalars::full/...      proj/src/kernel_scalars.cpp:214-379
//   gauss_rule                   proj/src/quadrature.cpp:49
//   BlockAssembler::true_block   proj/src/assembly.cpp:332
//   kernel_cross_block           proj/src/assembly.cpp:424
//   build_proxy                  proj/src/compression.cpp:25
//   AssemblerSource::cell_basis  proj/src/compression.cpp:132
//   Cpqr                         proj/src/lapack.cpp:101-158
//   LuFactor                     proj/src/lapack.cpp:31-99
//   FdsSolver                    proj/src/fds.cpp:18-268
//   ConvSolver                   proj/src/dense_solver.cpp:9-29
//   BlockAssembler::rhs          proj/include/ebem/assembly.hpp:94-119
#include <omp.h>

#include <algorithm>
#include <complex>
#include <cstring>
#include <exception>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "ebem/assembly.hpp"
#include "ebem/compression.hpp"
#include "ebem/dense_solver.hpp"
#include "ebem/postprocess.hpp"
#include "ebem/fds.hpp"
#include "ebem/geometry.hpp"
#include "ebem/hankel.hpp"
#include "ebem/kernels.hpp"
#include "ebem/lapack.hpp"
#include "ebem/medium.hpp"
#include "ebem/quadrature.hpp"
#include "ebem/scalars.hpp"

using namespace ebem;

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::domain_error& e) {
    g_err = std::string("domain_error: ") + e.what();
    return 3;
  } catch (const std::length_error& e) {
    g_err = std::string("length_error: ") + e.what();
    return 4;
  } catch (const std::runtime_error& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = std::string("exception: ") + e.what();
    return 5;
  }
}

void put(const Eigen::MatrixXcd& m, double* out) {
  std::memcpy(out, m.data(), sizeof(cd) * std::size_t(m.rows() * m.cols()));
}

Eigen::MatrixXcd get(const double* in, int rows, int cols) {
  Eigen::MatrixXcd m(rows, cols);
  std::memcpy(m.data(), in, sizeof(cd) * std::size_t(rows) * cols);
  return m;
}

std::array<std::vector<int>, 2> lists(const int* a, int na, const int* b,
                                      int nb) {
  return {std::vector<int>(a, a + na), std::vector<int>(b, b + nb)};
}

// Records every cell_basis call the FdsSolver makes (keyed by node range), so
// tests can compare skeletons and ranks cell by cell.  Thread-safe.
class RecordingSource : public BlockSource {
 public:
  explicit RecordingSource(const BlockSource& inner) : inner_(inner) {}
  int n_nodes() const override { return inner_.n_nodes(); }
  Eigen::MatrixXcd block(
      const std::array<std::vector<int>, 2>& rows,
      const std::array<std::vector<int>, 2>& cols) const override {
    return inner_.block(rows, cols);
  }
  CellBasis cell_basis(const std::array<std::vector<int>, 2>& rows,
                       const std::array<std::vector<int>, 2>& cols,
                       int node_begin, int node_end,
                       double epsilon) const override {
    CellBasis b = inner_.cell_basis(rows, cols, node_begin, node_end, epsilon);
    if (record_) {
      std::lock_guard<std::mutex> lock(mu_);
      Rec& r = recs_[{node_begin, node_end}];
      r.rows = rows;
      r.cols = cols;
      r.basis = b;
    }
    return b;
  }
  struct Rec {
    std::array<std::vector<int>, 2> rows, cols;
    CellBasis basis;
  };
  bool record_ = true;
  mutable std::mutex mu_;
  mutable std::map<std::pair<int, int>, Rec> recs_;

 private:
  const BlockSource& inner_;
};

struct Problem {
  Mesh mesh;
  Medium medium;
  AssemblyConfig acfg;
  ProxyConfig pcfg;
  cd alpha;
  std::unique_ptr<BlockAssembler> assembler;
  std::unique_ptr<AssemblerSource> source;
  std::unique_ptr<RecordingSource> recorder;
};

struct Fds {
  Problem* prob;
  std::unique_ptr<ClusterTree> tree;
  std::unique_ptr<FdsSolver> solver;
};

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_set_threads(int n) { omp_set_num_threads(n > 0 ? n : 1); }
int ref_max_threads() { return omp_get_max_threads(); }

int ref_hankel1_01(const double* x, int n, double* out) {
  return guarded([&] {
    for (int i = 0; i < n; ++i) {
      cd h0, h1;
      hankel1_01(x[i], h0, h1);
      out[4 * i + 0] = h0.real();
      out[4 * i + 1] = h0.imag();
      out[4 * i + 2] = h1.real();
      out[4 * i + 3] = h1.imag();
    }
  });
}

// which: 0 = full, 1 = remainder, 2 = static (real parts only, imag 0).
int ref_scalars(double lam, double mu, double rho, double omega,
                const double* r, int n, int which, double* out) {
  return guarded([&] {
    const KernelScalars ks(Medium::from_lame(lam, mu, rho, omega));
    for (int i = 0; i < n; ++i) {
      ScalarSet s;
      if (which == 0) s = ks.full(r[i]);
      else if (which == 1) s = ks.remainder(r[i]);
      else s = to_complex(ks.static_part(r[i]));
      const cd v[10] = {s.gpsi, s.gchi, s.d1, s.d2, s.d3,
                        s.n1,   s.n2,   s.n4, s.n5, s.n7};
      for (int k = 0; k < 10; ++k) {
        out[20 * i + 2 * k] = v[k].real();
        out[20 * i + 2 * k + 1] = v[k].imag();
      }
    }
  });
}

int ref_integrated_remainder(double lam, double mu, double rho, double omega,
                             double scale, int upow, double* out) {
  return guarded([&] {
    const KernelScalars ks(Medium::from_lame(lam, mu, rho, omega));
    const std::array<cd, 10> v = ks.integrated_remainder(scale, upow);
    for (int k = 0; k < 10; ++k) {
      out[2 * k] = v[k].real();
      out[2 * k + 1] = v[k].imag();
    }
  });
}

int ref_gauss_rule(int n, double* x, double* w) {
  return guarded([&] {
    const GaussRule& g = gauss_rule(n);
    for (int i = 0; i < n; ++i) {
      x[i] = g.x[i];
      w[i] = g.w[i];
    }
  });
}

int ref_problem_new(const double* xy, int n, double lam, double mu,
                    double rho, double omega, double alpha_re,
                    double alpha_im, const int* icfg /*corner,far,rhs,m'*/,
                    const double* dcfg /*refine,radius_factor*/, int n_gauss,
                    void** out) {
  return guarded([&] {
    std::vector<Vec2> nodes(n);
    for (int i = 0; i < n; ++i) nodes[i] = Vec2{xy[2 * i], xy[2 * i + 1]};
    auto* p = new Problem{Mesh(std::move(nodes)),
                          Medium::from_lame(lam, mu, rho, omega),
                          AssemblyConfig{},
                          ProxyConfig{},
                          cd(alpha_re, alpha_im),
                          nullptr,
                          nullptr,
                          nullptr};
    p->acfg.corner_nodes = icfg[0];
    p->acfg.far_nodes = icfg[1];
    p->acfg.rhs_nodes = icfg[2];
    p->acfg.refine = dcfg[0];
    p->pcfg.radius_factor = dcfg[1];
    p->pcfg.m_prime = icfg[3];
    p->pcfg.n_gauss = n_gauss;
    try {
      p->assembler = std::make_unique<BlockAssembler>(p->mesh, p->medium,
                                                      p->alpha, p->acfg);
    } catch (...) {
      delete p;
      throw;
    }
    p->source = std::make_unique<AssemblerSource>(*p->assembler, p->pcfg);
    p->recorder = std::make_unique<RecordingSource>(*p->source);
    *out = p;
  });
}

void ref_problem_free(void* h) { delete static_cast<Problem*>(h); }

int ref_true_block(void* h, const int* r0, int nr0, const int* r1, int nr1,
                   const int* c0, int nc0, const int* c1, int nc1,
                   double* out) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    put(p->assembler->true_block(lists(r0, nr0, r1, nr1),
                                 lists(c0, nc0, c1, nc1)),
        out);
  });
}

int ref_dense(void* h, double* out) {
  return guarded([&] { put(static_cast<Problem*>(h)->assembler->dense(), out); });
}

// Proxy geometry: out3 = {cx, cy, radius}; enclosed written when cap allows.
int ref_build_proxy(void* h, int begin, int end, double* out3,
                    int* n_enclosed, int* enclosed, int cap) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    const ProxySurface s = build_proxy(p->mesh, begin, end, p->pcfg);
    out3[0] = s.center.x;
    out3[1] = s.center.y;
    out3[2] = s.radius;
    *n_enclosed = int(s.enclosed.size());
    if (enclosed && cap >= int(s.enclosed.size()))
      std::copy(s.enclosed.begin(), s.enclosed.end(), enclosed);
  });
}

// The two interaction matrices of AssemblerSource::cell_basis
// (proj/src/compression.cpp:139-166), built with the same calls.
// mv: (2m'+2|enc|) x (nc0+nc1); mu: (nr0+nr1) x (2m'+2|enc|).
int ref_cell_mats(void* h, const int* r0, int nr0, const int* r1, int nr1,
                  const int* c0, int nc0, const int* c1, int nc1, int begin,
                  int end, int* n_outside, double* mv, double* mu) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    const ProxySurface proxy = build_proxy(p->mesh, begin, end, p->pcfg);
    const int m = proxy.polygon.size();
    std::vector<int> poly(m);
    for (int j = 0; j < m; ++j) poly[j] = j;
    const std::array<std::vector<int>, 2> pn{poly, poly};
    const std::array<std::vector<int>, 2> enc{proxy.enclosed, proxy.enclosed};
    const auto rows = lists(r0, nr0, r1, nr1);
    const auto cols = lists(c0, nc0, c1, nc1);
    const KernelScalars& ks = p->assembler->integrator().scalars();
    *n_outside = 2 * m + 2 * int(proxy.enclosed.size());
    if (!mv || !mu) return;
    Eigen::MatrixXcd a = kernel_cross_block(proxy.polygon, pn, p->mesh, cols,
                                            ks, p->alpha, p->pcfg.n_gauss);
    if (!proxy.enclosed.empty()) {
      const Eigen::MatrixXcd near = p->assembler->true_block(enc, cols);
      a.conservativeResize(a.rows() + near.rows(), Eigen::NoChange);
      a.bottomRows(near.rows()) = near;
    }
    put(a, mv);
    Eigen::MatrixXcd b = kernel_cross_block(p->mesh, rows, proxy.polygon, pn,
                                            ks, p->alpha, p->pcfg.n_gauss);
    if (!proxy.enclosed.empty()) {
      const Eigen::MatrixXcd near = p->assembler->true_block(rows, enc);
      b.conservativeResize(Eigen::NoChange, b.cols() + near.cols());
      b.rightCols(near.cols()) = near;
    }
    put(b, mu);
  });
}

// AssemblerSource::cell_basis.  Outputs: k, saturated, skeletons (4 x k),
// u0 (nr0 x k), u1 (nr1 x k), v0 (k x nc0), v1 (k x nc1).  Pass null
// buffers to query k only.
int ref_cell_basis(void* h, const int* r0, int nr0, const int* r1, int nr1,
                   const int* c0, int nc0, const int* c1, int nc1, int begin,
                   int end, double eps, int* k_out, int* saturated,
                   int* skel /* rs0 rs1 cs0 cs1, k each */, double* u0,
                   double* u1, double* v0, double* v1) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    const CellBasis b = p->source->cell_basis(
        lists(r0, nr0, r1, nr1), lists(c0, nc0, c1, nc1), begin, end, eps);
    *k_out = b.k;
    *saturated = b.saturated ? 1 : 0;
    if (!skel) return;
    const int k = b.k;
    for (int i = 0; i < k; ++i) {
      skel[i] = b.row_skeleton[0][i];
      skel[k + i] = b.row_skeleton[1][i];
      skel[2 * k + i] = b.col_skeleton[0][i];
      skel[3 * k + i] = b.col_skeleton[1][i];
    }
    put(b.u[0], u0);
    put(b.u[1], u1);
    put(b.v[0], v0);
    put(b.v[1], v1);
  });
}

// Cpqr on an m x n column-major matrix: writes pivot order (0-based) and
// |R_kk| for all k < min(m,n), eps_rank for each eps, and (optionally) the
// interpolation coefficients at rank k_interp (k x n).
int ref_cpqr(const double* a, int m, int n, int* jpvt, double* rdiag,
             const double* eps, int n_eps, int* ranks, int k_interp,
             double* coeff) {
  return guarded([&] {
    const Cpqr q(get(a, m, n));
    for (int k = 0; k < q.max_rank(); ++k) rdiag[k] = q.pivot_magnitude(k);
    for (int i = 0; i < n_eps; ++i) ranks[i] = q.eps_rank(eps[i]);
    if (coeff && k_interp > 0) put(q.interpolation(k_interp).coeff, coeff);
    // Recover the pivot order: interpolation(k) exposes the first k pivots.
    if (jpvt) {
      const Interpolation all = q.interpolation(q.max_rank());
      for (int j = 0; j < q.max_rank(); ++j) jpvt[j] = all.skeleton[j];
    }
  });
}

int ref_lu_solve(const double* a, int n, const double* b, int m, double* x,
                 double* min_pivot) {
  return guarded([&] {
    const LuFactor lu(get(a, n, n));
    if (min_pivot) *min_pivot = lu.min_pivot();
    put(lu.solve(get(b, n, m)), x);
  });
}

int ref_fds_new(void* h, int depth, double eps, int ell0, int record,
                void** out, double* stats /* upward, top, basis_cpu, top_dim,
                                              saturated */,
                int* max_rank /* depth+1 */) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    auto f = std::make_unique<Fds>();
    f->prob = p;
    f->tree = std::make_unique<ClusterTree>(p->mesh.size(), depth);
    p->recorder->record_ = record != 0;
    p->recorder->recs_.clear();
    const BlockSource& src =
        record ? static_cast<const BlockSource&>(*p->recorder)
               : static_cast<const BlockSource&>(*p->source);
    f->solver = std::make_unique<FdsSolver>(src, *f->tree,
                                            FdsConfig{eps, ell0});
    const FdsStats& s = f->solver->stats();
    if (stats) {
      stats[0] = s.upward_seconds;
      stats[1] = s.top_factor_seconds;
      stats[2] = s.basis_cpu_seconds;
      stats[3] = s.top_dim;
      stats[4] = s.saturated ? 1.0 : 0.0;
    }
    if (max_rank)
      for (int l = 0; l <= depth; ++l) max_rank[l] = s.max_rank[l];
    *out = f.release();
  });
}

void ref_fds_free(void* f) { delete static_cast<Fds*>(f); }

int ref_fds_solve(void* f, const double* rhs, int m, double* x,
                  double* timing3) {
  return guarded([&] {
    auto* s = static_cast<Fds*>(f);
    const int n = s->prob->mesh.size();
    FdsSolveTiming t;
    put(s->solver->solve(get(rhs, 2 * n, m), &t), x);
    if (timing3) {
      timing3[0] = t.upward_seconds;
      timing3[1] = t.top_seconds;
      timing3[2] = t.downward_seconds;
    }
  });
}

int ref_fds_rank_of(void* f, int cell) {
  return static_cast<Fds*>(f)->solver->rank_of(cell);
}

// Recorded basis of the cell owning [begin, end): sizes, then (when the
// buffers are non-null) sequences and skeletons.
int ref_fds_cell(void* f, int begin, int end, int* sizes /* nr0 nr1 nc0 nc1 k */,
                 int* rows, int* cols, int* skel) {
  return guarded([&] {
    auto* s = static_cast<Fds*>(f);
    auto& recs = s->prob->recorder->recs_;
    auto it = recs.find({begin, end});
    if (it == recs.end()) throw std::invalid_argument("no such cell recorded");
    const auto& r = it->second;
    sizes[0] = int(r.rows[0].size());
    sizes[1] = int(r.rows[1].size());
    sizes[2] = int(r.cols[0].size());
    sizes[3] = int(r.cols[1].size());
    sizes[4] = r.basis.k;
    if (rows) {
      std::copy(r.rows[0].begin(), r.rows[0].end(), rows);
      std::copy(r.rows[1].begin(), r.rows[1].end(), rows + sizes[0]);
    }
    if (cols) {
      std::copy(r.cols[0].begin(), r.cols[0].end(), cols);
      std::copy(r.cols[1].begin(), r.cols[1].end(), cols + sizes[2]);
    }
    if (skel) {
      const int k = r.basis.k;
      for (int i = 0; i < k; ++i) {
        skel[i] = r.basis.row_skeleton[0][i];
        skel[k + i] = r.basis.row_skeleton[1][i];
        skel[2 * k + i] = r.basis.col_skeleton[0][i];
        skel[3 * k + i] = r.basis.col_skeleton[1][i];
      }
    }
  });
}

int ref_rhs_plane_p(void* h, const double* angles, int m, double amplitude,
                    double* out) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    const int n = p->mesh.size();
    for (int j = 0; j < m; ++j) {
      const PlanePWave wave(p->medium, amplitude, angles[j]);
      const Eigen::VectorXcd b = p->assembler->rhs(wave);
      std::memcpy(out + 4 * std::size_t(n) * j, b.data(), sizeof(cd) * 2 * n);
    }
  });
}

int ref_conv_solve(void* h, const double* rhs, int m, double* x,
                   double* rcond) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    const ConvSolver conv(p->mesh, p->medium, p->alpha, p->acfg);
    if (rcond) *rcond = conv.stats().rcond;
    const int n = p->mesh.size();
    put(conv.solve(get(rhs, 2 * n, m)), x);
  });
}

// evaluate_scattered / evaluate_field (proj/src/postprocess.cpp:56-119);
// angle < -10: scattered only.  out: (u1, u2) complex per point.
int ref_evaluate_field(void* h, const double* u, const double* pts, int m, int ng,
                       double angle, double amplitude, double* out) {
  return guarded([&] {
    auto* p = static_cast<Problem*>(h);
    const int n = p->mesh.size();
    Eigen::VectorXcd bu(2 * n);
    std::memcpy(bu.data(), u, sizeof(cd) * 2 * n);
    std::vector<Vec2> x(m);
    for (int i = 0; i < m; ++i) x[i] = Vec2{pts[2 * i], pts[2 * i + 1]};
    if (angle < -10.0) {
      const std::vector<CVec2> s = evaluate_scattered(p->mesh, p->medium, bu, x, ng);
      for (int i = 0; i < m; ++i) {
        std::memcpy(out + 4 * i, &s[i].x, sizeof(cd));
        std::memcpy(out + 4 * i + 2, &s[i].y, sizeof(cd));
      }
    } else {
      const PlanePWave wave(p->medium, amplitude, angle);
      const std::vector<FieldSample> s = evaluate_field(p->mesh, p->medium, wave, bu, x, ng);
      for (int i = 0; i < m; ++i) {
        std::memcpy(out + 4 * i, &s[i].displacement.x, sizeof(cd));
        std::memcpy(out + 4 * i + 2, &s[i].displacement.y, sizeof(cd));
      }
    }
  });
}

}  // extern "C"
