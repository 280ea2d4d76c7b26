// Streaming Householder TSQR: R factor of a tall rows x n complex block.
//
// The pivoted QR of an interaction matrix depends on its columns only through
// their Gram matrix, so the tall matrices are first reduced to an n x n R
// (same column norms, same zlaqp2 pivot sequence) before the column-pivoted
// pass (Cpqr, proj/src/lapack.cpp:101-119).  One CTA owns a row range of one
// matrix and keeps R (packed upper triangle) in shared memory; it streams the
// rows through in blocks B of kRows = LANES * kRpt rows held in registers and
// folds each block into R with the structured reflectors of [R; B]:
//   column i:  x = [R_ii; B(:, i)],  beta = -sign(Re R_ii) ||x||,
//              tau = (beta - R_ii) / beta,  v = B(:, i) / (R_ii - beta)
//   columns j > i:  s = R_ij + v^H B(:, j),  f = conj(tau) s,
//                   R_ij -= f,  B(:, j) -= v f
// (zlarfg / zlarf semantics, the sign convention of k_qr_reduce).
// Layout: LANES consecutive lanes own one column, lane g holds rows
// g, g + LANES, ... of the block; the group owning column i + 1 updates it
// first and immediately generates reflector i + 1 (look-ahead), so every step
// costs one barrier.  The R factors of several row pieces of one matrix are
// stacked and reduced again by the same kernel.
#include <cuda_runtime.h>

#include <cstdio>

#include "ebem_dense.h"

namespace ebem_gpu {

namespace {

constexpr int kTsqrThreads = 1024;
constexpr int kRpt = 8;  // block rows per lane

__device__ __forceinline__ int pidx(int i, int j) { return ((j * (j + 1)) >> 1) + i; }

template <int LANES>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = LANES >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int LANES>
__device__ __forceinline__ void make_reflector(double2 (&B)[kRpt], bool mine, int i,
                                               int g, double2* R, double2* vout,
                                               double2* tau_out) {
  double p = 0.0;
  if (mine) {
#pragma unroll
    for (int k = 0; k < kRpt; ++k) p = fma(B[k].x, B[k].x, fma(B[k].y, B[k].y, p));
  }
  const double xnorm2 = group_sum<LANES>(p);
  if (!mine) return;
  const double2 alpha = R[pidx(i, i)];
#ifdef EBEM_TSQR_DEBUG
  if (g == 0 && !(isfinite(xnorm2) && isfinite(alpha.x) && isfinite(alpha.y)))
    printf("tsqr blk %d col %d: xnorm2 %g alpha %g %g\n", blockIdx.x, i, xnorm2, alpha.x, alpha.y);
#endif
  double2 tau = make_double2(0.0, 0.0);
  if (!(xnorm2 == 0.0 && alpha.y == 0.0)) {
    const double nrm = sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xnorm2);
    const double beta = alpha.x >= 0.0 ? -nrm : nrm;
    tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
    // scal = 1 / (alpha - beta), Smith's division: the residues of columns
    // that are already eliminated shrink geometrically, and |alpha - beta|^2
    // would underflow long before |alpha - beta| does
    const double ar = alpha.x - beta, ai = alpha.y;
    double2 scal;
    if (fabs(ar) >= fabs(ai)) {
      const double q = ai / ar, d = ar + ai * q;
      scal = make_double2(1.0 / d, -q / d);
    } else {
      const double q = ar / ai, d = ai + ar * q;
      scal = make_double2(q / d, -1.0 / d);
    }
#pragma unroll
    for (int k = 0; k < kRpt; ++k)
      B[k] = make_double2(scal.x * B[k].x - scal.y * B[k].y,
                          scal.x * B[k].y + scal.y * B[k].x);
    if (g == 0) R[pidx(i, i)] = make_double2(beta, 0.0);
  }
#pragma unroll
  for (int k = 0; k < kRpt; ++k) vout[g + LANES * k] = B[k];
  if (g == 0) *tau_out = tau;
}

template <int LANES>
__global__ void __launch_bounds__(kTsqrThreads, 1)
k_tsqr(const QrTask* __restrict__ tasks) {
  constexpr int kRows = LANES * kRpt;
  extern __shared__ double2 R[];  // packed upper triangle, then v[2][kRows], tau[2]
  const QrTask T = tasks[blockIdx.x];
  const int n = T.n, rows = T.rows, ld = T.ld;
  double2* vbuf = R + ((n * (n + 1)) >> 1);
  double2* tbuf = vbuf + 2 * kRows;
  const int g = threadIdx.x % LANES;
  const int j = threadIdx.x / LANES;  // owned column
  constexpr int kGroupsPerWarp = 32 / LANES;
  const int wfirst = (threadIdx.x >> 5) * kGroupsPerWarp;  // first column of the warp
  const int wlast = wfirst + kGroupsPerWarp - 1;
  for (int t = threadIdx.x; t < ((n * (n + 1)) >> 1); t += blockDim.x)
    R[t] = make_double2(0.0, 0.0);
  const double2* src = reinterpret_cast<const double2*>(T.src) + (size_t)j * ld;
  const bool own = j < n;
  __syncthreads();
  for (int r0 = 0; r0 < rows; r0 += kRows) {
    double2 B[kRpt];
#pragma unroll
    for (int k = 0; k < kRpt; ++k) {
      const int r = r0 + g + LANES * k;
      B[k] = (own && r < rows) ? src[r] : make_double2(0.0, 0.0);
    }
    if (own && r0 + kRows < rows) {  // warm L2 for the next block
      const int r = r0 + kRows + g * kRpt;
      if (r < rows) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + r));
    }
    if (wfirst == 0) make_reflector<LANES>(B, j == 0, 0, g, R, vbuf, tbuf);
    __syncthreads();
    for (int i = 0; i < n; ++i) {
      const int cur = i & 1;
      if (wlast > i && wfirst < n) {  // warp-uniform: some column j > i here
        const bool act = own && j > i;
        const double2* v = vbuf + cur * kRows;
        double sr0 = 0.0, si0 = 0.0, sr1 = 0.0, si1 = 0.0;
#pragma unroll
        for (int k = 0; k < kRpt; k += 2) {
          const double2 a = v[g + LANES * k], b = B[k];
          sr0 = fma(a.x, b.x, fma(a.y, b.y, sr0));
          si0 = fma(a.x, b.y, fma(-a.y, b.x, si0));
          const double2 c = v[g + LANES * (k + 1)], d = B[k + 1];
          sr1 = fma(c.x, d.x, fma(c.y, d.y, sr1));
          si1 = fma(c.x, d.y, fma(-c.y, d.x, si1));
        }
        double sr = group_sum<LANES>(sr0 + sr1);
        double si = group_sum<LANES>(si0 + si1);
        if (act) {
          const double2 rij = R[pidx(i, j)];
          sr += rij.x;
          si += rij.y;
          const double2 tau = tbuf[cur];
          // f = conj(tau) s
          const double fr = tau.x * sr + tau.y * si;
          const double fi = tau.x * si - tau.y * sr;
#pragma unroll
          for (int k = 0; k < kRpt; ++k) {
            const double2 a = v[g + LANES * k];
            B[k].x = fma(-a.x, fr, fma(a.y, fi, B[k].x));
            B[k].y = fma(-a.x, fi, fma(-a.y, fr, B[k].y));
          }
          if (g == 0) R[pidx(i, j)] = make_double2(rij.x - fr, rij.y - fi);
#ifdef EBEM_TSQR_DEBUG
          if (g == 0 && !(isfinite(fr) && isfinite(fi)) && isfinite(rij.x))
            printf("tsqr r0 %d step %d col %d: s %g %g tau %g %g rij %g %g\n", r0, i, j, sr, si,
                   tbuf[cur].x, tbuf[cur].y, rij.x, rij.y);
#endif
        }
        if (i + 1 < n && wfirst <= i + 1 && i + 1 <= wlast)
          make_reflector<LANES>(B, j == i + 1, i + 1, g, R, vbuf + (cur ^ 1) * kRows,
                                tbuf + (cur ^ 1));
      }
      __syncthreads();
    }
  }
  double2* out = reinterpret_cast<double2*>(T.dst);
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int c = idx / n, r = idx - c * n;
    out[(size_t)c * T.dst_ld + r] = r <= c ? R[pidx(r, c)] : make_double2(0.0, 0.0);
  }
}

}  // namespace

int tsqr_lanes(int n) { return n <= 64 ? 16 : n <= kTsqrMaxCols ? 8 : 0; }
int tsqr_block_rows(int n) { return tsqr_lanes(n) * kRpt; }
size_t tsqr_smem_bytes(int n) {
  return sizeof(double2) * (size_t(n) * (n + 1) / 2 + 2 * size_t(tsqr_block_rows(n)) + 2);
}

void launch_tsqr(const QrTask* tasks, int n_tasks, int lanes, size_t smem,
                 cudaStream_t st) {
  if (n_tasks <= 0) return;
  if (lanes == 16) {
    static bool once = [] {
      cudaFuncSetAttribute(k_tsqr<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           227 * 1024);
      return true;
    }();
    (void)once;
    k_tsqr<16><<<n_tasks, kTsqrThreads, smem, st>>>(tasks);
  } else {
    static bool once = [] {
      cudaFuncSetAttribute(k_tsqr<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           227 * 1024);
      return true;
    }();
    (void)once;
    k_tsqr<8><<<n_tasks, kTsqrThreads, smem, st>>>(tasks);
  }
}

}  // namespace ebem_gpu
