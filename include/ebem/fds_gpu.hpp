// ebem/fds_gpu.hpp -- drop-in C++ facade of the B200 solver path for code
// written against the reference `ebem` library (/root/reference/proj).
//
// Compiled against the reference's own headers (proj/include) and Eigen, it
// mirrors the two reference types on the hot path and forwards to the C ABI
// of libebem_gpu.so (include/ebem_gpu.h):
//
//   ebem::gpu::AssemblerSource  the production BlockSource
//                               (proj/include/ebem/compression.hpp:106-123):
//                               same constructor (BlockAssembler, ProxyConfig);
//                               entries, bases and everything downstream are
//                               computed on the device.
//   ebem::gpu::FdsSolver        FdsSolver (proj/include/ebem/fds.hpp:55-67):
//                               same constructor (const BlockSource&,
//                               const ClusterTree&, const FdsConfig&), solve,
//                               stats, tree, rank_of.  With a
//                               gpu::AssemblerSource the whole factorization
//                               runs on the device; any other BlockSource
//                               (the reference tests' MatrixSource,
//                               DirectSource, a CPU ebem::AssemblerSource)
//                               supplies entries and bases through its
//                               virtual interface and the merges and solves
//                               run on the device.
//
// Switching the reference's run_fds (proj/tools/ebem_cli.cpp:164-185) is the
// two type changes AssemblerSource -> gpu::AssemblerSource and FdsSolver ->
// gpu::FdsSolver.  Errors are rethrown as the exception
// types and messages the reference uses (std::invalid_argument,
// std::runtime_error, std::domain_error, ...).
#pragma once

#include <Eigen/Dense>
#include <memory>
#include <vector>

#include "ebem/assembly.hpp"
#include "ebem/compression.hpp"
#include "ebem/fds.hpp"
#include "ebem/geometry.hpp"
#include "ebem_gpu.h"

namespace ebem::gpu {

// BlockSource whose entries (BlockAssembler::true_block) and cell bases
// (AssemblerSource::cell_basis) come from the device.  The medium is taken
// from the assembler's kernel scalars (lambda, mu, k_T, k_L), the geometry
// from its mesh; the AssemblyConfig cannot be read back from a
// BlockAssembler, so pass it when it is not the default.
class AssemblerSource : public BlockSource {
 public:
  explicit AssemblerSource(const BlockAssembler& assembler, const ProxyConfig& proxy = {},
                           const AssemblyConfig& assembly = {});
  ~AssemblerSource() override;
  AssemblerSource(const AssemblerSource&) = delete;
  AssemblerSource& operator=(const AssemblerSource&) = delete;

  int n_nodes() const override { return n_; }
  Eigen::MatrixXcd block(const std::array<std::vector<int>, 2>& rows,
                         const std::array<std::vector<int>, 2>& cols) const override;
  CellBasis cell_basis(const std::array<std::vector<int>, 2>& rows,
                       const std::array<std::vector<int>, 2>& cols, int node_begin,
                       int node_end, double epsilon) const override;

  ebem_gpu_problem* handle() const { return h_; }

 private:
  ebem_gpu_problem* h_ = nullptr;
  int n_ = 0;
};

class FdsSolver {
 public:
  FdsSolver(const BlockSource& source, const ClusterTree& tree, const FdsConfig& config = {});
  ~FdsSolver();
  FdsSolver(const FdsSolver&) = delete;
  FdsSolver& operator=(const FdsSolver&) = delete;

  Eigen::MatrixXcd solve(const Eigen::MatrixXcd& rhs, FdsSolveTiming* timing = nullptr) const;
  Eigen::VectorXcd solve(const Eigen::VectorXcd& rhs, FdsSolveTiming* timing = nullptr) const;

  const FdsStats& stats() const { return stats_; }
  const ClusterTree& tree() const { return tree_; }
  int rank_of(int cell) const;
  // CUDA-event time of the whole factorization (not in the reference stats)
  double factorize_device_seconds() const { return device_seconds_; }

 private:
  struct Callbacks;
  ClusterTree tree_;
  FdsConfig config_;
  FdsStats stats_;
  double device_seconds_ = 0.0;
  ebem_gpu_fds* h_ = nullptr;
};

}  // namespace ebem::gpu
