// Task descriptors and launch wrappers of the batched dense kernels
// (ebem_dense.cu).  Complex matrices are column-major interleaved doubles.
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

namespace ebem_gpu {

constexpr int kSmemCap = 200 * 1024;  // dynamic shared memory per CTA
constexpr int kMaxCpqrCols = 256;

struct QrTask {  // R (n x n, dst_ld) of the rows x n block at src (ld)
  const double* src;
  double* dst;
  int rows, n, ld, dst_ld;
  int in_smem;
  int pad;
  long long ws_off;  // global workspace offset (complex) when !in_smem
};

struct CpqrTask {
  const double* src;  // rows x n, ld
  int rows, n, ld;
  int in_smem;
  double stop_rel;  // stop at the first |R_ii| <= stop_rel |R_00|
  int* jpvt;        // n, zero-based pivot order
  double* rdiag;    // |R_ii| of the computed steps (+ the stopping one)
  int* steps;       // number of completed steps (= eps_rank(stop_rel))
  double* r_out;    // steps x n, ld r_ld (upper trapezoid, pivoted order)
  int r_ld;
  int pad;
  long long ws_off;
};

struct InterpTask {
  const double* r;  // k x n upper trapezoid, ld r_ld
  const int* jpvt;
  double* out;      // k x n (ld out_ld) or n x k when adjoint
  int k, n, r_ld, out_ld;
  int adjoint;
  int pad;
};

struct LuTask {
  double* a;  // n x n, ld, factored in place
  int* ipiv;  // zero-based row interchanges
  int* info;  // 0, or 1 + index of the first exactly-zero pivot
  int n, ld;
  int in_smem;
  int pad;
  long long ws_off;
  int* perm;  // optional (n <= kPermMaxN): the interchanges composed into one permutation
};
constexpr int kPermMaxN = 1024;

struct LuSolveTask {
  const double* lu;
  const int* ipiv;
  double* b;
  int n, ld, nrhs, ldb;
  // optional: row r of the permuted right-hand side is row perm[r] of b (the
  // interchanges ipiv applied in order); spares the few-column solves their
  // serial interchange loop
  const int* perm;
};

// trans: 0 = N, 1 = T, 2 = C (conjugate transpose)
struct GemmTask {
  const double* a;
  const double* b;
  double* c;
  int m, n, k;
  int lda, ldb, ldc;
  int trans_a, trans_b;
  double alpha_re, alpha_im, beta_re, beta_im;
};

struct CopyTask {  // dst(i, j) = src(i, j) (0 when src is null; transpose 1:
                   // dst(j, i); 2: identity)
  const double* src;
  double* dst;
  int rows, cols, src_ld, dst_ld;
  int conj, transpose;
};

void dense_init();
void launch_qr_reduce(const QrTask* tasks, int n, size_t smem, double2* gws,
                      cudaStream_t st);
void launch_cpqr(const CpqrTask* tasks, int n, size_t smem, double2* gws,
                 cudaStream_t st);
// blocks of at most 32 x 32: one warp per matrix (k_cpqr_warp)
void launch_cpqr_warp(const CpqrTask* tasks, int n, cudaStream_t st);
// Team-layout Householder kernels (ebem_qr.cu), same task descriptors.
void launch_qr_team(const QrTask* tasks, int n, size_t smem, double2* gws,
                    cudaStream_t st);
void launch_cpqr_team(const CpqrTask* tasks, int n, size_t smem, double2* gws,
                      cudaStream_t st);
// Streaming TSQR (ebem_tsqr.cu): same QrTask (in_smem / ws_off unused);
// n <= kTsqrMaxCols in two variants (tsqr_variant: 0 for n <= 64, 1 above),
// smem = tsqr_smem_bytes(n) for the largest n of a launch.
constexpr int kTsqrMaxCols = 128;
int tsqr_variant(int n);  // -1: not supported (n > kTsqrMaxCols)
int tsqr_block_rows(int n);
int tsqr_ctas_per_sm(int n);
size_t tsqr_smem_bytes(int n);
void launch_tsqr(const QrTask* tasks, int n_tasks, int variant, size_t smem,
                 cudaStream_t st);
// L2 warm-up of byte ranges (prefetch.global.L2, one line per thread step):
// the solve's upper tree levels are few, latency-bound launches whose
// factors fit the L2.
struct PrefetchTask {
  const void* p;
  unsigned long long bytes;
};
void launch_prefetch_l2(const PrefetchTask* tasks, int n, cudaStream_t st);
// perm of every task that asks for one, from its ipiv (one warp per task).
void launch_pivots_to_perm(const LuTask* tasks, int n, cudaStream_t st);
void launch_interp(const InterpTask* tasks, int n, int max_k, cudaStream_t st);
void launch_getrf(const LuTask* tasks, int n, size_t smem, double2* gws,
                  cudaStream_t st);
// CTAs per task for a batch whose largest LU has order max_n
// right-hand sides per warp for a batch (0: the unstaged one-warp-per-column
// kernel for at most kNarrowRhs columns; getrs_blocks then counts warps)
// -1: one CTA per column (orders above kGetrsWarpMaxN for few columns, and
// 256 < n <= kGetrsCtaMaxN for any count).
constexpr int kNarrowRhs = 8;
constexpr int kGetrsWarpMaxN = 128;
constexpr int kGetrsCtaMaxN = 2048;
// -2: blocked panels for many columns (ebem_dense.cu k_getrs_blk)
#ifndef EBEM_BLK_MIN_N
#define EBEM_BLK_MIN_N 64
#endif
constexpr int kBlkMinRhs = 16;
constexpr int kBlkMinN = EBEM_BLK_MIN_N;
constexpr int kGetrsBlkMaxN = 512;
int getrs_cpw(int max_nrhs, int max_n);
int getrs_blocks(int nrhs, int max_n, int cpw);
// Dense-solver helpers (ebem_lu.cu): column sums of |a_ij| (1-norm), and
// x := A^-H x with A's LU (one right-hand side, one CTA).
void launch_col_abs_sum(const double* a, int n, int ld, double* out, cudaStream_t st);
void launch_getrs_conj(const double* lu, int n, int ld, const int* ipiv, double* x,
                       cudaStream_t st);
// Blocked LU (ebem_lu.cu) of the tasks with in_smem == 0, in place.
void launch_lu_blocked(const LuTask* tasks, int n_tasks, int max_n, cudaStream_t st);
void launch_getrs(const LuSolveTask* tasks, const int* block_off, int n_tasks,
                  int n_blocks, cudaStream_t st, int smem_bytes, int max_n, int cpw);
// Dynamic shared memory that stages an n x n LU (0 when it does not fit).
int getrs_smem_bytes(int n);
// Narrow products (at most kNarrow columns, no transposes) run as a GEMV
// kernel: gemm_narrow gives its column template (1 or kNarrow; 0 = tiled GEMM);
// a launch uses one kind for all its tasks (the smallest common one).
constexpr int kNarrow = 4;
int gemm_narrow(const GemmTask& g);
int gemm_blocks(const GemmTask& g, int narrow);
void launch_gemm(const GemmTask* tasks, const int* block_off, int n_tasks,
                 int n_blocks, cudaStream_t st, int narrow);
int copy_blocks(int rows, int cols);
void launch_copy(const CopyTask* tasks, const int* block_off, int n_tasks,
                 int n_blocks, cudaStream_t st);

}  // namespace ebem_gpu
