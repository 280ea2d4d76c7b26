// Drop-in C++ facade (include/ebem/fds_gpu.hpp) over the C ABI of
// libebem_gpu.so.  Built against the reference headers (proj/include) by
// facade/Makefile; see INTEGRATION.md.
#include "ebem/fds_gpu.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>

namespace ebem::gpu {

namespace {

// Rethrows a C-ABI status as the reference's exception type and message.
void check(int rc) {
  if (rc == EBEM_OK) return;
  const std::string msg = ebem_gpu_last_error();
  switch (rc) {
    case EBEM_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case EBEM_DOMAIN_ERROR: throw std::domain_error(msg);
    case EBEM_LENGTH_ERROR: throw std::length_error(msg);
    case EBEM_LOGIC_ERROR: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

const double* cbuf(const Eigen::MatrixXcd& m) {
  return reinterpret_cast<const double*>(m.data());
}
double* cbuf(Eigen::MatrixXcd& m) { return reinterpret_cast<double*>(m.data()); }

// column-major interleaved complex buffer -> MatrixXcd
Eigen::MatrixXcd from_buf(const double* p, int rows, int cols) {
  Eigen::MatrixXcd m(rows, cols);
  if (rows > 0 && cols > 0)
    std::memcpy(m.data(), p, sizeof(double) * 2 * size_t(rows) * cols);
  return m;
}

}  // namespace

// ------------------------------------------------------------ AssemblerSource

AssemblerSource::AssemblerSource(const BlockAssembler& assembler, const ProxyConfig& proxy,
                                 const AssemblyConfig& assembly) {
  const Mesh& mesh = assembler.mesh();
  n_ = mesh.size();
  std::vector<double> xy(2 * size_t(n_));
  for (int i = 0; i < n_; ++i) {
    xy[2 * i] = mesh.node(i).x;
    xy[2 * i + 1] = mesh.node(i).y;
  }
  // The kernels depend on the medium only through lambda, mu, k_T, k_L:
  // with rho = mu (c_T = 1) and omega = k_T the library reproduces both
  // wave numbers (k_L = k_T sqrt(mu / (lambda + 2 mu)))
  const KernelScalars& ks = assembler.integrator().scalars();
  const double lam = ks.lambda(), mu = ks.mu(), kT = ks.k_T();
  const ebem_assembly_config ac{assembly.corner_nodes, assembly.far_nodes, assembly.rhs_nodes,
                                assembly.refine, assembly.max_dense_bytes};
  const ebem_proxy_config pc{proxy.radius_factor, proxy.m_prime, proxy.n_gauss};
  const cd alpha = assembler.alpha();
  check(ebem_gpu_problem_create(xy.data(), n_, lam, mu, mu, kT, alpha.real(), alpha.imag(),
                                &ac, &pc, &h_));
}

AssemblerSource::~AssemblerSource() { ebem_gpu_problem_destroy(h_); }

Eigen::MatrixXcd AssemblerSource::block(const std::array<std::vector<int>, 2>& rows,
                                        const std::array<std::vector<int>, 2>& cols) const {
  const int nr = int(rows[0].size() + rows[1].size());
  const int nc = int(cols[0].size() + cols[1].size());
  Eigen::MatrixXcd out(nr, nc);
  check(ebem_gpu_true_block(h_, rows[0].data(), int(rows[0].size()), rows[1].data(),
                            int(rows[1].size()), cols[0].data(), int(cols[0].size()),
                            cols[1].data(), int(cols[1].size()), cbuf(out)));
  return out;
}

CellBasis AssemblerSource::cell_basis(const std::array<std::vector<int>, 2>& rows,
                                      const std::array<std::vector<int>, 2>& cols,
                                      int node_begin, int node_end, double epsilon) const {
  const int nr0 = int(rows[0].size()), nr1 = int(rows[1].size());
  const int nc0 = int(cols[0].size()), nc1 = int(cols[1].size());
  int k = 0, sat = 0;
  auto call = [&](int* skel, double* u0, double* u1, double* v0, double* v1) {
    check(ebem_gpu_cell_basis(h_, rows[0].data(), nr0, rows[1].data(), nr1, cols[0].data(),
                              nc0, cols[1].data(), nc1, node_begin, node_end, epsilon, &k,
                              &sat, skel, u0, u1, v0, v1));
  };
  call(nullptr, nullptr, nullptr, nullptr, nullptr);  // rank query
  std::vector<int> skel(4 * size_t(k) + 1);
  std::vector<double> u0(2 * size_t(nr0) * k + 2), u1(2 * size_t(nr1) * k + 2);
  std::vector<double> v0(2 * size_t(nc0) * k + 2), v1(2 * size_t(nc1) * k + 2);
  call(skel.data(), u0.data(), u1.data(), v0.data(), v1.data());
  CellBasis b;
  b.k = k;
  b.saturated = sat != 0;
  b.row_skeleton[0].assign(skel.begin(), skel.begin() + k);
  b.row_skeleton[1].assign(skel.begin() + k, skel.begin() + 2 * k);
  b.col_skeleton[0].assign(skel.begin() + 2 * k, skel.begin() + 3 * k);
  b.col_skeleton[1].assign(skel.begin() + 3 * k, skel.begin() + 4 * k);
  b.u[0] = from_buf(u0.data(), nr0, k);
  b.u[1] = from_buf(u1.data(), nr1, k);
  b.v[0] = from_buf(v0.data(), k, nc0);
  b.v[1] = from_buf(v1.data(), k, nc1);
  return b;
}

// ------------------------------------------------------------------ FdsSolver

// Host callbacks of ebem_gpu_fds_create_source: the BlockSource's virtual
// interface, with its exception carried across the C ABI and rethrown.
struct FdsSolver::Callbacks {
  const BlockSource* src;
  std::exception_ptr err;

  static std::array<std::vector<int>, 2> lists(const int* a, int na, const int* b, int nb) {
    return {std::vector<int>(a, a + na), std::vector<int>(b, b + nb)};
  }
  static int block(void* user, const int* r0, int nr0, const int* r1, int nr1, const int* c0,
                   int nc0, const int* c1, int nc1, double* out) {
    auto* self = static_cast<Callbacks*>(user);
    try {
      const Eigen::MatrixXcd m = self->src->block(lists(r0, nr0, r1, nr1), lists(c0, nc0, c1, nc1));
      if (m.rows() != nr0 + nr1 || m.cols() != nc0 + nc1)
        throw std::logic_error("BlockSource::block returned a block of the wrong shape");
      std::memcpy(out, m.data(), sizeof(double) * 2 * size_t(m.rows()) * m.cols());
      return 0;
    } catch (...) {
      self->err = std::current_exception();
      return EBEM_RUNTIME_ERROR;
    }
  }
  static int basis(void* user, const int* r0, int nr0, const int* r1, int nr1, const int* c0,
                   int nc0, const int* c1, int nc1, int b, int e, double eps, int* k, int* sat,
                   int* skel, double* u0, double* u1, double* v0, double* v1) {
    auto* self = static_cast<Callbacks*>(user);
    try {
      const CellBasis cb =
          self->src->cell_basis(lists(r0, nr0, r1, nr1), lists(c0, nc0, c1, nc1), b, e, eps);
      *k = cb.k;
      *sat = cb.saturated ? 1 : 0;
      const int kk = cb.k;
      for (int i = 0; i < kk; ++i) {
        skel[i] = cb.row_skeleton[0][i];
        skel[kk + i] = cb.row_skeleton[1][i];
        skel[2 * kk + i] = cb.col_skeleton[0][i];
        skel[3 * kk + i] = cb.col_skeleton[1][i];
      }
      auto put = [](const Eigen::MatrixXcd& m, double* o) {
        if (m.size()) std::memcpy(o, m.data(), sizeof(double) * 2 * size_t(m.size()));
      };
      put(cb.u[0], u0);
      put(cb.u[1], u1);
      put(cb.v[0], v0);
      put(cb.v[1], v1);
      return 0;
    } catch (...) {
      self->err = std::current_exception();
      return EBEM_RUNTIME_ERROR;
    }
  }
};

FdsSolver::FdsSolver(const BlockSource& source, const ClusterTree& tree, const FdsConfig& config)
    : tree_(tree), config_(config) {
  if (tree_.n_nodes() != source.n_nodes())
    throw std::invalid_argument("FdsSolver: tree and source node counts differ");
  const ebem_fds_config cfg{config_.epsilon, config_.ell0};
  ebem_fds_stats st{};
  if (const auto* dev = dynamic_cast<const AssemblerSource*>(&source)) {
    check(ebem_gpu_fds_create(dev->handle(), tree_.depth(), &cfg, &h_, &st));
  } else {
    Callbacks cb{&source, nullptr};
    const int rc = ebem_gpu_fds_create_source(tree_.n_nodes(), tree_.depth(), &cfg,
                                              &Callbacks::block, &Callbacks::basis, &cb, &h_,
                                              &st);
    if (rc != EBEM_OK && cb.err) std::rethrow_exception(cb.err);
    check(rc);
  }
  stats_.max_rank.assign(st.max_rank, st.max_rank + tree_.depth() + 1);
  stats_.top_dim = st.top_dim;
  stats_.saturated = st.saturated != 0;
  stats_.upward_seconds = st.upward_seconds;
  stats_.top_factor_seconds = st.top_factor_seconds;
  stats_.basis_cpu_seconds = st.basis_cpu_seconds;
  device_seconds_ = st.factorize_device_seconds;
}

FdsSolver::~FdsSolver() { ebem_gpu_fds_destroy(h_); }

Eigen::MatrixXcd FdsSolver::solve(const Eigen::MatrixXcd& rhs, FdsSolveTiming* timing) const {
  const int n2 = 2 * tree_.n_nodes();
  if (rhs.rows() != n2)
    throw std::invalid_argument("FdsSolver: right-hand side has " + std::to_string(rhs.rows()) +
                                " rows, need " + std::to_string(n2));
  Eigen::MatrixXcd x(n2, rhs.cols());
  ebem_fds_solve_timing t{};
  check(ebem_gpu_fds_solve(h_, cbuf(rhs), int(rhs.cols()), cbuf(x), &t));
  if (timing) {
    timing->upward_seconds = t.upward_seconds;
    timing->top_seconds = t.top_seconds;
    timing->downward_seconds = t.downward_seconds;
  }
  return x;
}

Eigen::VectorXcd FdsSolver::solve(const Eigen::VectorXcd& rhs, FdsSolveTiming* timing) const {
  Eigen::MatrixXcd m(rhs.rows(), 1);
  for (Eigen::Index i = 0; i < rhs.rows(); ++i) m(i, 0) = rhs(i);
  const Eigen::MatrixXcd x = solve(m, timing);
  Eigen::VectorXcd out(x.rows());
  for (Eigen::Index i = 0; i < x.rows(); ++i) out(i) = x(i, 0);
  return out;
}

int FdsSolver::rank_of(int cell) const { return ebem_gpu_fds_rank_of(h_, cell); }

}  // namespace ebem::gpu
