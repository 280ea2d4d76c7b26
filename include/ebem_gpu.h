/*
 * ebem_gpu.h -- C ABI of the B200-native (sm_100a) fast direct solver path.
 *
 * Drop-in boundary for the reference library's hot path (the `ebem` C++
 * library, /root/reference/proj).  Each entry point names the reference
 * interface it replaces; plain pointers and sizes only.  Complex matrices are
 * column-major with interleaved (re, im) doubles, exactly the memory layout
 * of Eigen::MatrixXcd.  Node lists are per displacement component; local
 * vectors are component-major (component 1 over the list, then component 2),
 * global vectors are [u1(0..N-1); u2(0..N-1)] (proj/src/fds.cpp:174-182).
 *
 * Every function returns EBEM_OK (0) or a status naming the exception type
 * the reference throws in the same situation; ebem_gpu_last_error() returns
 * the message of the last failure on the calling thread.
 *
 * Thread safety: every entry point takes one process-wide mutex and runs on
 * one process-wide CUDA stream (the device scratch is shared by all
 * handles), so calls from several threads are safe and serialised.
 */
#ifndef EBEM_GPU_H
#define EBEM_GPU_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum ebem_status {
  EBEM_OK = 0,
  EBEM_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  EBEM_RUNTIME_ERROR = 2,    /* std::runtime_error (singular LU, ...) */
  EBEM_DOMAIN_ERROR = 3,     /* std::domain_error (element too long) */
  EBEM_LENGTH_ERROR = 4,     /* std::length_error (memory budget) */
  EBEM_CUDA_ERROR = 5,       /* no device / CUDA failure */
  EBEM_LOGIC_ERROR = 6       /* std::logic_error */
};

/* AssemblyConfig, proj/include/ebem/assembly.hpp:21-30 */
typedef struct ebem_assembly_config {
  int corner_nodes; /* 10 */
  int far_nodes;    /* 4 */
  int rhs_nodes;    /* 8 */
  double refine;    /* 1.0 */
  size_t max_dense_bytes;
} ebem_assembly_config;

/* ProxyConfig, proj/include/ebem/compression.hpp:14-23 */
typedef struct ebem_proxy_config {
  double radius_factor; /* 1.5 */
  int m_prime;          /* 64 */
  int n_gauss;          /* 6 */
} ebem_proxy_config;

/* FdsConfig, proj/include/ebem/fds.hpp:13-19 */
typedef struct ebem_fds_config {
  double epsilon; /* 1e-8 */
  int ell0;       /* 1 */
} ebem_fds_config;

#define EBEM_MAX_LEVELS 32

/* FdsStats, proj/include/ebem/fds.hpp:21-36 */
typedef struct ebem_fds_stats {
  int depth;
  int max_rank[EBEM_MAX_LEVELS]; /* index = level, 0 at/above ell0 */
  int top_dim;
  int saturated;
  double upward_seconds;
  double top_factor_seconds;
  double basis_cpu_seconds; /* wall time of the basis phase (fill + ID) */
  double factorize_device_seconds; /* CUDA events around the whole build */
} ebem_fds_stats;

/* FdsSolveTiming, proj/include/ebem/fds.hpp:38-42 */
typedef struct ebem_fds_solve_timing {
  double upward_seconds;
  double top_seconds;
  double downward_seconds;
  double device_seconds; /* CUDA events around the whole solve */
} ebem_fds_solve_timing;

typedef struct ebem_gpu_problem ebem_gpu_problem;
typedef struct ebem_gpu_fds ebem_gpu_fds;
typedef struct ebem_gpu_conv ebem_gpu_conv;

/* ConvStats (proj/include/ebem/dense_solver.hpp:10-19). */
typedef struct ebem_conv_stats {
  double assemble_seconds;
  double factor_seconds;
  double rcond;      /* 1-norm reciprocal condition estimate (zgecon's zlacn2) */
  double min_pivot;  /* min |U_ii| */
  int condition_warning;
} ebem_conv_stats;

const char* ebem_gpu_last_error(void);

/* Describes the device the library runs on; EBEM_CUDA_ERROR without one. */
int ebem_gpu_device_info(char* buf, int len);

/* Mesh(std::vector<Vec2>) + Medium::from_lame(lambda, mu, rho, omega) +
 * BlockAssembler(mesh, medium, alpha, AssemblyConfig) +
 * AssemblerSource(assembler, ProxyConfig)
 * (proj/include/ebem/geometry.hpp:32, medium.hpp:30-39, assembly.hpp:74-75,
 * compression.hpp:109-110).  nodes_xy: 2*n_nodes doubles (x0,y0,x1,y1,...).
 * NULL configs mean the reference defaults. */
int ebem_gpu_problem_create(const double* nodes_xy, int n_nodes, double lambda,
                            double mu, double rho, double omega,
                            double alpha_re, double alpha_im,
                            const ebem_assembly_config* assembly,
                            const ebem_proxy_config* proxy,
                            ebem_gpu_problem** out);
void ebem_gpu_problem_destroy(ebem_gpu_problem* p);
int ebem_gpu_problem_size(const ebem_gpu_problem* p);

/* BlockSource::block == BlockAssembler::true_block
 * (proj/include/ebem/compression.hpp:74-76, proj/src/assembly.cpp:332-409).
 * out: (nr0+nr1) x (nc0+nc1) complex, host memory. */
int ebem_gpu_true_block(ebem_gpu_problem* p, const int* rows0, int nr0,
                        const int* rows1, int nr1, const int* cols0, int nc0,
                        const int* cols1, int nc1, double* out);

/* BlockSource::cell_basis == AssemblerSource::cell_basis
 * (proj/include/ebem/compression.hpp:80-86, proj/src/compression.cpp:132-169).
 * Pass skel == NULL to query k only; otherwise skel holds 4*k ints
 * (row_skeleton[0], row_skeleton[1], col_skeleton[0], col_skeleton[1]) and
 * u0 (nr0 x k), u1 (nr1 x k), v0 (k x nc0), v1 (k x nc1) complex. */
int ebem_gpu_cell_basis(ebem_gpu_problem* p, const int* rows0, int nr0,
                        const int* rows1, int nr1, const int* cols0, int nc0,
                        const int* cols1, int nc1, int node_begin, int node_end,
                        double epsilon, int* k, int* saturated, int* skel,
                        double* u0, double* u1, double* v0, double* v1);

/* cell_basis for a batch of contiguous cells [begin_i, end_i) with
 * rows = cols = the cell's nodes, in one batched device pass (the level
 * path of the factorization; BASELINE config 5 microbenchmark).  Writes the
 * shared ranks; skel_out (may be NULL; capacity 4 * sum(end_i - begin_i))
 * gets, cell after cell, the row skeletons of both components then the
 * column skeletons, k_i entries each, in pivot order (CellBasis::
 * row_skeleton / col_skeleton, compression.hpp:35-44); device_seconds (may
 * be NULL) gets the CUDA-event time. */
int ebem_gpu_cell_bases(ebem_gpu_problem* p, int count, const int* begins,
                        const int* ends, double epsilon, int* k_out,
                        int* skel_out, double* device_seconds);

/* The two interaction matrices cell_basis compresses
 * (proj/src/compression.cpp:139-166): mv (n_out x (nc0+nc1)) and
 * mu ((nr0+nr1) x n_out), n_out = 2 m' + 2 |enclosed|.  NULL buffers query
 * n_out only. */
int ebem_gpu_cell_mats(ebem_gpu_problem* p, const int* rows0, int nr0,
                       const int* rows1, int nr1, const int* cols0, int nc0,
                       const int* cols1, int nc1, int node_begin, int node_end,
                       int* n_out, double* mv, double* mu);

/* build_proxy geometry and enclosed nodes (proj/src/compression.cpp:25-69).
 * out3 = {cx, cy, radius}; enclosed written when cap suffices. */
int ebem_gpu_build_proxy(ebem_gpu_problem* p, int node_begin, int node_end,
                         double* out3, int* n_enclosed, int* enclosed, int cap);

/* BlockAssembler::rhs / rhs_batch for plane waves
 * (proj/include/ebem/assembly.hpp:94-124, proj/src/assembly.cpp:411-422).
 * kind 0: PlanePWave (proj/src/kernels.cpp:99-118); kind 1: plane SV wave
 * (not in the reference).  out: 2N x m complex, host memory. */
int ebem_gpu_rhs_plane(ebem_gpu_problem* p, int kind, const double* angles,
                       int m, double amplitude, double* out);

/* evaluate_scattered / evaluate_field (proj/src/postprocess.cpp:56-119):
 * displacement at m points (points_xy: x0 y0 x1 y1 ...) off the boundary from
 * the nodal solution boundary_u (2N complex), Gauss order n_gauss per element;
 * wave_kind < 0: scattered part only, 0: + incident plane P wave, 1: + plane
 * SV wave (angle, amplitude).  out_u: 2 complex per point (u1, u2);
 * out_intensity: |u1|^2 + |u2|^2 per point (may be null).  invalid_argument
 * status for a point within one element length of the curve. */
int ebem_gpu_field(ebem_gpu_problem* p, const double* boundary_u, const double* points_xy,
                   int m, int n_gauss, int wave_kind, double angle, double amplitude,
                   double* out_u, double* out_intensity);

/* BlockAssembler::dense (proj/src/assembly.cpp:311-330): the full 2N x 2N
 * Galerkin matrix into out (host, column-major complex); length_error
 * status past AssemblyConfig::max_dense_bytes. */
int ebem_gpu_dense(ebem_gpu_problem* p, double* out);

/* ConvSolver(mesh, medium, alpha, config) on the problem's geometry: dense
 * assembly + partial-pivoted LU (proj/src/dense_solver.cpp:9-22).  The
 * problem must outlive the solver. */
int ebem_gpu_conv_create(ebem_gpu_problem* p, ebem_gpu_conv** out,
                         ebem_conv_stats* stats);
/* ConvSolver::solve (proj/src/dense_solver.cpp:24-29): rhs, x 2N x m, host. */
int ebem_gpu_conv_solve(ebem_gpu_conv* c, const double* rhs, int m, double* x);
void ebem_gpu_conv_destroy(ebem_gpu_conv* c);

/* FdsSolver(source, ClusterTree(N, depth), FdsConfig): factorization
 * (proj/src/fds.cpp:18-154).  The problem must outlive the solver. */
int ebem_gpu_fds_create(ebem_gpu_problem* p, int depth,
                        const ebem_fds_config* cfg, ebem_gpu_fds** out,
                        ebem_fds_stats* stats);
void ebem_gpu_fds_destroy(ebem_gpu_fds* f);

/* FdsSolver::solve (proj/src/fds.cpp:156-263): rhs and x are 2N x m complex
 * in host memory (x may alias rhs). */
int ebem_gpu_fds_solve(ebem_gpu_fds* f, const double* rhs, int m, double* x,
                       ebem_fds_solve_timing* timing);
/* Same with device pointers on the solver's stream (no host copies). */
int ebem_gpu_fds_solve_device(ebem_gpu_fds* f, const double* rhs_dev, int m,
                              double* x_dev);

/* Any other BlockSource (compression.hpp:66-87), e.g. the reference tests'
 * MatrixSource / DirectSource: entries and bases come from host callbacks;
 * the merges (LU, A^-1 U, W, atilde) and every solve run on the device.
 * Callbacks return 0 on success.  block: out (nr0+nr1) x (nc0+nc1).
 * basis: k <= min(nr0, nr1, nc0, nc1); skel holds 4*k ids (rs0 rs1 cs0 cs1),
 * u0 (nr0 x k), u1 (nr1 x k), v0 (k x nc0), v1 (k x nc1), column-major. */
typedef int (*ebem_block_fn)(void* user, const int* rows0, int nr0,
                             const int* rows1, int nr1, const int* cols0,
                             int nc0, const int* cols1, int nc1, double* out);
typedef int (*ebem_basis_fn)(void* user, const int* rows0, int nr0,
                             const int* rows1, int nr1, const int* cols0,
                             int nc0, const int* cols1, int nc1,
                             int node_begin, int node_end, double epsilon,
                             int* k, int* saturated, int* skel, double* u0,
                             double* u1, double* v0, double* v1);
int ebem_gpu_fds_create_source(int n_nodes, int depth,
                               const ebem_fds_config* cfg,
                               ebem_block_fn block, ebem_basis_fn basis,
                               void* user, ebem_gpu_fds** out,
                               ebem_fds_stats* stats);

/* FdsSolver::rank_of (proj/include/ebem/fds.hpp:67). */
int ebem_gpu_fds_rank_of(const ebem_gpu_fds* f, int cell);
/* Introspection for parity tests: sizes = {nr0, nr1, nc0, nc1, k}; when
 * non-NULL, skel holds 4*k node ids (rs0, rs1, cs0, cs1). */
int ebem_gpu_fds_cell(const ebem_gpu_fds* f, int cell, int* sizes, int* skel);

/* Point evaluations of the device special functions (parity hooks):
 * hankel: out[4i..4i+3] = H0(x_i), H1(x_i); scalars: 10 complex per r,
 * which = 0 full, 1 remainder, 2 static (proj/src/kernel_scalars.cpp). */
int ebem_gpu_eval_hankel(const double* x, int n, double* out);
int ebem_gpu_eval_scalars(ebem_gpu_problem* p, const double* r, int n,
                          int which, double* out);
/* Host-only table hooks (no device needed; CPU tests): the remainder
 * expansion of the ten kernel scalars for a medium, out[10][max_pow][4] =
 * (Re a_q, Im a_q, Re b_q, Im b_q) of sum_q (a_q + b_q ln r) r^q
 * (KernelScalars::remainder below the series radius,
 * proj/src/kernel_scalars.cpp:123-212, 381-409), *max_q the largest power;
 * and the n-point Gauss-Legendre rule on [0, 1] (gauss_rule,
 * proj/src/quadrature.cpp:16-56). */
int ebem_gpu_series_table(double lambda, double mu, double rho, double omega,
                          double* out, int max_pow, int* max_q);
int ebem_gpu_gauss_rule(int n, double* x, double* w);

/* Parity hook of the ID's TSQR stage (the reduction before Cpqr,
 * proj/src/lapack.cpp:101-119): reduces the rows x n complex block a
 * (column-major, ld) to *r_rows x n rows with the same Gram matrix
 * (an upper-triangular n x n R when n <= 128); r holds rows x n. */
int ebem_gpu_tall_reduce(const double* a, int rows, int n, int ld, double* r,
                         int* r_rows);

/* Number of kernel launches issued by the library since load (bench). */
long long ebem_gpu_launch_count(void);

/* Per-kernel device timing with CUDA events on the launching stream
 * (measurement hooks for bench.py).  prof_read fills n entries of
 * milliseconds, launch counts and algorithmic work units (point
 * evaluations for the fill kernels, flops or bytes for the others). */
int ebem_gpu_prof_enable(int on);
int ebem_gpu_prof_read(int reset, double* ms, long long* count, double* units,
                       int n);
const char* ebem_gpu_prof_name(int id);
/* Algorithmic HBM bytes per kernel kind since the last prof_read reset
 * (operands read once, results written once; 0 for the fill kernels). */
int ebem_gpu_prof_bytes(double* bytes, int n);
int ebem_gpu_prof_kernels(void);
/* Measured FP64 FMA throughput of the device (TFLOP/s), the roofline
 * denominator of the fill kernels. */
int ebem_gpu_fp64_peak(double* tflops);

/* Debug hook: copies a cell's device factor (0 LU, 1 pivots, 2 A^-1 U,
 * 3 V = [v0 v1], 4 atilde) into host memory. */
int ebem_gpu_fds_debug_cell(const ebem_gpu_fds* f, int cell, int which,
                            double* out);

#ifdef __cplusplus
}
#endif

#endif /* EBEM_GPU_H */
