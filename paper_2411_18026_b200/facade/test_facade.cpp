// C++ tests of the drop-in facade (include/ebem/fds_gpu.hpp), compiled
// against the reference headers and linked with the reference library built
// in place (oracle/_ref/libebem_ref.so, test infrastructure) and
// libebem_gpu.so.  Ports the synthetic cases of proj/tests/test_fds.cpp:
// 128-220 (MatrixSource + DirectSource exactness, block-diagonal zero ranks,
// argument errors, the compressed-diagonal identity), the FDS-vs-Conv
// agreement of :222-260, and BASELINE configs[0] against the reference
// FdsSolver through a run_fds-shaped routine that differs from
// proj/tools/ebem_cli.cpp:164-185 only in its two types.  Exit code 0 =
// every check passed.  Run by tests/test_facade.py (GPU).
#include <array>
#include <cmath>
#include <complex>
#include <cstdio>
#include <random>
#include <stdexcept>
#include <utility>
#include <vector>

#include <Eigen/Dense>

#include "ebem/assembly.hpp"
#include "ebem/compression.hpp"
#include "ebem/dense_solver.hpp"
#include "ebem/fds.hpp"
#include "ebem/fds_gpu.hpp"
#include "ebem/geometry.hpp"
#include "ebem/kernels.hpp"
#include "ebem/lapack.hpp"
#include "ebem/medium.hpp"

using namespace ebem;

namespace {

int g_checks = 0, g_failed = 0;
#define CHECK(cond)                                                           \
  do {                                                                        \
    ++g_checks;                                                               \
    if (!(cond)) {                                                            \
      ++g_failed;                                                             \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond);  \
    }                                                                         \
  } while (0)
template <class E, class F>
void check_throws(F&& f, const char* what) {
  ++g_checks;
  try {
    f();
  } catch (const E&) {
    return;
  } catch (...) {
  }
  ++g_failed;
  std::fprintf(stderr, "FAILED: %s did not throw the expected type\n", what);
}

class MatrixSource : public BlockSource {
 public:
  MatrixSource(Eigen::MatrixXcd a, int n) : a_(std::move(a)), n_(n) {}
  int n_nodes() const override { return n_; }
  Eigen::MatrixXcd block(const std::array<std::vector<int>, 2>& rows,
                         const std::array<std::vector<int>, 2>& cols) const override {
    std::vector<int> r, c;
    for (int p = 0; p < 2; ++p) {
      for (int g : rows[p]) r.push_back(p * n_ + g);
      for (int g : cols[p]) c.push_back(p * n_ + g);
    }
    Eigen::MatrixXcd out(r.size(), c.size());
    for (std::size_t j = 0; j < c.size(); ++j)
      for (std::size_t i = 0; i < r.size(); ++i) out(i, j) = a_(r[i], c[j]);
    return out;
  }
  CellBasis cell_basis(const std::array<std::vector<int>, 2>&,
                       const std::array<std::vector<int>, 2>&, int, int, double) const override {
    throw std::logic_error("MatrixSource provides entries only");
  }
  const Eigen::MatrixXcd& matrix() const { return a_; }

 private:
  Eigen::MatrixXcd a_;
  int n_;
};

Eigen::MatrixXcd random_matrix(int rows, int cols, std::mt19937& gen) {
  std::normal_distribution<double> dist(0.0, 1.0);
  Eigen::MatrixXcd m(rows, cols);
  for (int j = 0; j < cols; ++j)
    for (int i = 0; i < rows; ++i) m(i, j) = cd(dist(gen), dist(gen));
  return m;
}

// off-diagonal leaf blocks of exact per-cell ranks, well-conditioned diagonal
Eigen::MatrixXcd synthetic_system(int n, int n_leaves, const std::vector<int>& ranks,
                                  unsigned seed) {
  const int m = n / n_leaves;
  std::mt19937 gen(seed);
  Eigen::MatrixXcd a = Eigen::MatrixXcd::Zero(2 * n, 2 * n);
  std::vector<std::array<Eigen::MatrixXcd, 2>> uf(n_leaves), vf(n_leaves);
  for (int i = 0; i < n_leaves; ++i)
    for (int p = 0; p < 2; ++p) {
      uf[i][p] = random_matrix(m, ranks[i], gen);
      vf[i][p] = random_matrix(ranks[i], m, gen);
    }
  for (int i = 0; i < n_leaves; ++i)
    for (int j = 0; j < n_leaves; ++j) {
      if (i == j || ranks[i] == 0 || ranks[j] == 0) continue;
      const double scale = 1.0 / std::sqrt(double(m) * ranks[i] * ranks[j]);
      for (int p = 0; p < 2; ++p)
        for (int q = 0; q < 2; ++q) {
          const Eigen::MatrixXcd c = scale * random_matrix(ranks[i], ranks[j], gen);
          a.block(p * n + i * m, q * n + j * m, m, m) = uf[i][p] * c * vf[j][q];
        }
    }
  for (int i = 0; i < n_leaves; ++i) {
    const Eigen::MatrixXcd d =
        (1.0 / std::sqrt(2.0 * m)) * random_matrix(2 * m, 2 * m, gen) +
        8.0 * Eigen::MatrixXcd::Identity(2 * m, 2 * m);
    for (int p = 0; p < 2; ++p)
      for (int q = 0; q < 2; ++q)
        a.block(p * n + i * m, q * n + i * m, m, m) = d.block(p * m, q * m, m, m);
  }
  return a;
}

template <class A, class B>
double rel(const A& got, const B& want) {
  return (got - want).norm() / want.norm();
}

// proj/tools/ebem_cli.cpp:164-185 with the solver types as parameters: the
// reference instantiation and the GPU one run the same statements.
template <class Source, class Solver>
Eigen::VectorXcd run_fds(const Mesh& mesh, const Medium& med, cd alpha, const ProxyConfig& proxy,
                         double eps, int levels, int ell0, FdsStats* stats) {
  const BlockAssembler assembler(mesh, med, alpha);
  const Source source(assembler, proxy);
  const ClusterTree tree(mesh.size(), levels);
  const Solver fds(source, tree, FdsConfig{eps, ell0});
  *stats = fds.stats();
  const PlanePWave wave(med, 1.0, 0.0);
  const Eigen::VectorXcd f = assembler.rhs(wave);
  return fds.solve(f);
}

void synthetic_low_rank() {
  const int n = 128, depth = 3, n_leaves = 8;
  const std::vector<int> ranks = {2, 3, 4, 2, 4, 3, 2, 3};
  const MatrixSource entries(synthetic_system(n, n_leaves, ranks, 91), n);
  const DirectSource source(entries);
  const ClusterTree tree(n, depth);
  std::mt19937 gen(17);
  const Eigen::MatrixXcd f = random_matrix(2 * n, 2, gen);
  const Eigen::MatrixXcd want = LuFactor(entries.matrix()).solve(f);
  for (int ell0 : {0, 1, 2}) {
    const gpu::FdsSolver fds(source, tree, FdsConfig{1e-10, ell0});
    const double err = rel(fds.solve(f), want);
    std::printf("synthetic ell0=%d err=%.3e\n", ell0, err);
    CHECK(err <= 1e-11);
    for (int c = ClusterTree::first_cell(depth); c <= ClusterTree::last_cell(depth); ++c)
      CHECK(fds.rank_of(c) == ranks[c - ClusterTree::first_cell(depth)]);
  }
}

void block_diagonal() {
  const int n = 64, depth = 2, n_leaves = 4;
  const std::vector<int> ranks(n_leaves, 0);
  const MatrixSource entries(synthetic_system(n, n_leaves, ranks, 7), n);
  const DirectSource source(entries);
  const ClusterTree tree(n, depth);
  const gpu::FdsSolver fds(source, tree, FdsConfig{1e-10, 1});
  CHECK(fds.stats().top_dim == 0);
  for (int c = ClusterTree::first_cell(depth); c <= ClusterTree::last_cell(depth); ++c)
    CHECK(fds.rank_of(c) == 0);
  std::mt19937 gen(3);
  const Eigen::MatrixXcd f = random_matrix(2 * n, 1, gen);
  const Eigen::MatrixXcd want = LuFactor(entries.matrix()).solve(f);
  CHECK(rel(fds.solve(f), want) <= 1e-12);
}

void rejects_inconsistent_inputs() {
  const int n = 64;
  const MatrixSource entries(synthetic_system(n, 4, {1, 1, 1, 1}, 5), n);
  const DirectSource source(entries);
  const ClusterTree tree(n, 2);
  check_throws<std::invalid_argument>([&] { gpu::FdsSolver(source, tree, FdsConfig{1e-8, 2}); },
                                      "ell0 == depth");
  check_throws<std::invalid_argument>([&] { gpu::FdsSolver(source, tree, FdsConfig{1e-8, -1}); },
                                      "ell0 < 0");
  check_throws<std::invalid_argument>(
      [&] { gpu::FdsSolver(source, ClusterTree(32, 1), FdsConfig{}); }, "node count");
  const gpu::FdsSolver fds(source, tree, FdsConfig{});
  check_throws<std::invalid_argument>([&] { fds.solve(Eigen::VectorXcd(2 * n + 2)); },
                                      "rhs rows");
  // a source exception crosses the C ABI unchanged
  const ClusterTree tree2(n, 2);
  check_throws<std::logic_error>([&] { gpu::FdsSolver(entries, tree2, FdsConfig{}); },
                                 "MatrixSource::cell_basis");
}

void compressed_diagonal_identity() {
  const Medium med = Medium::from_lame(1.0, 1.0, 1.0, 2.0);
  const Mesh mesh = Mesh::star(400, StarShape{});
  const BlockAssembler assembler(mesh, med, med.default_coupling());
  const gpu::AssemblerSource source(assembler);
  const ClusterTree tree(mesh.size(), 2);
  const int cell = ClusterTree::first_cell(2) + 1;
  const int b = tree.cell_begin(cell), e = tree.cell_end(cell);
  std::vector<int> ids(e - b);
  for (int g = b; g < e; ++g) ids[g - b] = g;
  const std::array<std::vector<int>, 2> nodes = {ids, ids};
  const CellBasis basis = source.cell_basis(nodes, nodes, b, e, 1e-8);
  const int nloc = e - b, k = basis.k;
  CHECK(k >= 1);
  const Eigen::MatrixXcd diag = source.block(nodes, nodes);
  // the device block equals the reference assembler's true_block
  CHECK(rel(diag, assembler.true_block(nodes, nodes)) <= 1e-12);
  Eigen::MatrixXcd u = Eigen::MatrixXcd::Zero(2 * nloc, 2 * k);
  u.topLeftCorner(nloc, k) = basis.u[0];
  u.bottomRightCorner(nloc, k) = basis.u[1];
  Eigen::MatrixXcd v = Eigen::MatrixXcd::Zero(2 * k, 2 * nloc);
  v.topLeftCorner(k, nloc) = basis.v[0];
  v.bottomRightCorner(k, nloc) = basis.v[1];
  const Eigen::MatrixXcd w = v * LuFactor(diag).solve(u);
  const Eigen::MatrixXcd atilde = LuFactor(w).inverse();
  CHECK((atilde * w - Eigen::MatrixXcd::Identity(2 * k, 2 * k)).norm() <=
        1e-10 * std::sqrt(2.0 * k));
  // same rank and skeletons as the reference AssemblerSource
  const AssemblerSource ref_source(assembler);
  const CellBasis rb = ref_source.cell_basis(nodes, nodes, b, e, 1e-8);
  CHECK(rb.k == k);
  for (int q = 0; q < 2; ++q) {
    CHECK(rb.row_skeleton[q] == basis.row_skeleton[q]);
    CHECK(rb.col_skeleton[q] == basis.col_skeleton[q]);
  }
}

void agreement_with_dense_solver() {
  const Medium med = Medium::from_lame(1.0, 1.0, 1.0, 2.0);
  const PlanePWave wave(med, 1.0, 0.0);
  const Mesh mesh = Mesh::star(400, StarShape{});
  const BlockAssembler assembler(mesh, med, med.default_coupling());
  const gpu::AssemblerSource source(assembler);
  const ConvSolver conv(mesh, med, med.default_coupling());
  const Eigen::VectorXcd f = assembler.rhs(wave);
  const Eigen::VectorXcd want = conv.solve(f);
  const ClusterTree tree(mesh.size(), 2);
  double prev = 1.0;
  for (double eps : {1e-8, 1e-10}) {
    const gpu::FdsSolver fds(source, tree, FdsConfig{eps, 1});
    const double err = rel(fds.solve(f), want);
    std::printf("n=400 depth=2 eps=%.0e err=%.3e\n", eps, err);
    CHECK(err <= 100.0 * eps);
    CHECK(err < prev);
    prev = err;
  }
  const ClusterTree deep(mesh.size(), 3);
  for (int ell0 : {0, 1, 2}) {
    const gpu::FdsSolver fds(source, deep, FdsConfig{1e-8, ell0});
    const double err = rel(fds.solve(f), want);
    std::printf("n=400 depth=3 ell0=%d err=%.3e\n", ell0, err);
    CHECK(err <= 100.0 * 1e-8);
  }
}

void config1_run_fds_drop_in() {
  // BASELINE.json configs[0]: circle N=1024, k_T a = 1, leaf 32, eps 1e-10
  const int n = 1024;
  const Mesh mesh = Mesh::star(n, StarShape{1.0, 0.0, 3});
  const Medium med = Medium::from_lame(1.0, 1.0, 1.0, 1.0);
  const int levels = ClusterTree::depth_for(n, 32);
  FdsStats st_ref, st_gpu;
  const Eigen::VectorXcd x_ref = run_fds<AssemblerSource, FdsSolver>(
      mesh, med, med.default_coupling(), ProxyConfig{}, 1e-10, levels, 1, &st_ref);
  const Eigen::VectorXcd x_gpu = run_fds<gpu::AssemblerSource, gpu::FdsSolver>(
      mesh, med, med.default_coupling(), ProxyConfig{}, 1e-10, levels, 1, &st_gpu);
  const double err = rel(x_gpu, x_ref);
  std::printf("config1 N=%d: gpu vs reference FdsSolver err=%.3e\n", n, err);
  CHECK(err <= 1e-8);
  CHECK(st_gpu.max_rank == st_ref.max_rank);
  CHECK(st_gpu.top_dim == st_ref.top_dim);
  CHECK(st_gpu.saturated == st_ref.saturated);
}

}  // namespace

int main() {
  synthetic_low_rank();
  block_diagonal();
  rejects_inconsistent_inputs();
  compressed_diagonal_identity();
  agreement_with_dense_solver();
  config1_run_fds_drop_in();
  std::printf("facade: %d checks, %d failed\n", g_checks, g_failed);
  return g_failed == 0 ? 0 : 1;
}
