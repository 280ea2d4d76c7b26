// Batched complex-double dense linear algebra for the skeletonization and the
// merges (sm_100a).  One CTA per small matrix; matrices live in shared memory
// when they fit (<= kSmemCap bytes) and are worked on in place in global
// memory (L2/L1 resident) otherwise.
//
//   k_qr_reduce  unpivoted Householder QR of a row block -> R (n x n); tall
//                interaction matrices are reduced block by block (TSQR) before
//                the pivoted factorization, which keeps the column norms and
//                therefore the pivot sequence of the full matrix.
//   k_cpqr       column-pivoted Householder QR with LAPACK zlaqp2 pivoting
//                (first index of the largest partial norm, norm downdating
//                with recomputation below sqrt(eps)), stopping at the first
//                |R_kk| <= stop_rel |R_00| (Cpqr, proj/src/lapack.cpp:101-138;
//                kPivotFloor, proj/src/compression.cpp:15,93-99)
//   k_interp     [I, R11^-1 R12] scattered by pivot (Cpqr::interpolation,
//                proj/src/lapack.cpp:140-158), optionally conj-transposed
//   k_getrf      partial-pivoted LU, pivot = first max |Re|+|Im| (zgetrf as
//                called by LuFactor, proj/src/lapack.cpp:31-53)
//   k_getrs      row swaps + unit-lower + upper triangular solves
//                (LuFactor::solve, proj/src/lapack.cpp:73-89)
//   k_gemm       C = alpha op(A) op(B) + beta C, ragged batch
//   k_copy       batched block copies (optionally conjugated)
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <cstdlib>

#include "ebem_dense.h"

namespace ebem_gpu {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
#ifndef EBEM_QR_THREADS
#define EBEM_QR_THREADS 512
#endif
constexpr int kQrThreads = EBEM_QR_THREADS;  // QR / CPQR / LU CTAs
#ifndef EBEM_GETRF_LA
#define EBEM_GETRF_LA 1  // look-ahead k_getrf (one barrier per column); 0: the unblocked sequence
#endif

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 zconj(double2 a) { return make_double2(a.x, -a.y); }
// a - b*c
__device__ __forceinline__ double2 zfms(double2 a, double2 b, double2 c) {
  return make_double2(fma(-b.y, -c.y, fma(-b.x, c.x, a.x)),
                      fma(-b.y, c.x, fma(-b.x, c.y, a.y)));
}
// a + b*c
__device__ __forceinline__ double2 zfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(-b.y, c.y, fma(b.x, c.x, a.x)),
                      fma(b.y, c.x, fma(b.x, c.y, a.y)));
}
// a + conj(b)*c
__device__ __forceinline__ double2 zfmac(double2 a, double2 b, double2 c) {
  return make_double2(fma(b.y, c.y, fma(b.x, c.x, a.x)),
                      fma(-b.y, c.x, fma(b.x, c.y, a.y)));
}
__device__ __forceinline__ double2 zdiv(double2 a, double2 b) {
  // Smith's algorithm
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  }
  const double r = b.x / b.y, d = b.y + b.x * r;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}
__device__ __forceinline__ double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double2 warp_sum2(double2 v) {
  return make_double2(warp_sum(v.x), warp_sum(v.y));
}

// Block-wide sum of one double per thread (all threads must call).
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    s = warp_sum(s);
    if (threadIdx.x == 0) red[0] = s;
  }
  __syncthreads();
  s = red[0];
  __syncthreads();
  return s;
}

// Load an m x n block (ld) into a dense workspace (ld m).
__device__ void load_block(const double2* __restrict__ src, int m, int n, int ld,
                           double2* __restrict__ dst) {
  for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
    const int j = idx / m, i = idx - j * m;
    dst[idx] = src[(size_t)j * ld + i];
  }
}

// Generate the Householder reflector of column `col` rows [i, m) of A (ld m):
// returns tau, overwrites A[i,col] with beta and A[i+1:,col] with v.
// Semantics of zlarfg (beta = -sign(alpha_r) ||(alpha, x)||).
__device__ double2 householder(double2* A, int m, int ld, int i, int col,
                               double* red, double* beta_out) {
  double2* c = A + (size_t)col * ld;
  double part = 0.0;
  for (int r = i + 1 + threadIdx.x; r < m; r += blockDim.x) {
    const double2 v = c[r];
    part = fma(v.x, v.x, fma(v.y, v.y, part));
  }
  const double xnorm2 = block_sum(part, red);
  const double2 alpha = c[i];
  double2 tau = make_double2(0.0, 0.0);
  double beta;
  if (xnorm2 == 0.0 && alpha.y == 0.0) {
    beta = alpha.x;  // H = I
  } else {
    const double nrm = sqrt(alpha.x * alpha.x + alpha.y * alpha.y + xnorm2);
    beta = alpha.x >= 0.0 ? -nrm : nrm;
    tau = make_double2((beta - alpha.x) / beta, -alpha.y / beta);
    const double2 scal = zdiv(make_double2(1.0, 0.0),
                              make_double2(alpha.x - beta, alpha.y));
    for (int r = i + 1 + threadIdx.x; r < m; r += blockDim.x) c[r] = zmul(scal, c[r]);
  }
  __syncthreads();
  if (threadIdx.x == 0) c[i] = make_double2(beta, 0.0);
  __syncthreads();
  *beta_out = beta;
  return tau;
}

// Apply H^H = I - conj(tau) v v^H (v_i = 1, v stored below A[i,col]) to the
// columns cols [c0, n) of A, rows [i, m).  One warp per column.
__device__ void apply_reflector(double2* A, int m, int ld, int i, int col,
                                double2 tau, int c0, int n) {
  if (tau.x == 0.0 && tau.y == 0.0) return;
  const double2 ctau = zconj(tau);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const double2* v = A + (size_t)col * ld;
  const int nw = blockDim.x >> 5;
  for (int j = c0 + w; j < n; j += nw) {
    double2* cj = A + (size_t)j * ld;
    // s = v^H c_j
    double2 s = make_double2(0.0, 0.0);
    for (int r = i + l; r < m; r += 32) {
      const double2 vr = (r == i) ? make_double2(1.0, 0.0) : v[r];
      s = zfmac(s, vr, cj[r]);
    }
    s = warp_sum2(s);
    const double2 f = zmul(ctau, s);
    for (int r = i + l; r < m; r += 32) {
      const double2 vr = (r == i) ? make_double2(1.0, 0.0) : v[r];
      cj[r] = zfms(cj[r], vr, f);
    }
  }
}

}  // namespace

// ------------------------------------------------------------ QR reduction
__global__ void __launch_bounds__(kQrThreads)
k_qr_reduce(const QrTask* __restrict__ tasks, double2* __restrict__ gws) {
  extern __shared__ double2 smem[];
  __shared__ double red[33];
  const QrTask T = tasks[blockIdx.x];
  const int m = T.rows, n = T.n;
  double2* A = T.in_smem ? smem : gws + T.ws_off;
  load_block(reinterpret_cast<const double2*>(T.src), m, n, T.ld, A);
  __syncthreads();
  const int steps = m < n ? m : n;
  for (int i = 0; i < steps; ++i) {
    double beta;
    const double2 tau = householder(A, m, m, i, i, red, &beta);
    apply_reflector(A, m, m, i, i, tau, i + 1, n);
    __syncthreads();
  }
  double2* R = reinterpret_cast<double2*>(T.dst);
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int j = idx / n, i = idx - j * n;
    R[(size_t)j * T.dst_ld + i] = (i <= j && i < m) ? A[(size_t)j * m + i]
                                                    : make_double2(0.0, 0.0);
  }
}

// --------------------------------------------------------------------- CPQR
__global__ void __launch_bounds__(kQrThreads)
k_cpqr(const CpqrTask* __restrict__ tasks, double2* __restrict__ gws) {
  extern __shared__ double2 smem[];
  __shared__ double red[33];
  const int nw = blockDim.x >> 5;
  __shared__ double vn1[kMaxCpqrCols], vn2[kMaxCpqrCols];
  __shared__ int jp[kMaxCpqrCols];
  __shared__ int s_pvt;
  __shared__ double s_r00;
  const CpqrTask T = tasks[blockIdx.x];
  const int m = T.rows, n = T.n;
  double2* A = T.in_smem ? smem : gws + T.ws_off;
  load_block(reinterpret_cast<const double2*>(T.src), m, n, T.ld, A);
  for (int j = threadIdx.x; j < n; j += blockDim.x) jp[j] = j;
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  // initial column norms
  for (int j = w; j < n; j += nw) {
    const double2* c = A + (size_t)j * m;
    double s = 0.0;
    for (int r = l; r < m; r += 32) s = fma(c[r].x, c[r].x, fma(c[r].y, c[r].y, s));
    s = warp_sum(s);
    if (l == 0) vn1[j] = vn2[j] = sqrt(s);
  }
  __syncthreads();
  const double tol3z = 1.0536712127723509e-08;  // sqrt(2^-53)
  const int mn = m < n ? m : n;
  int steps = mn;
  double* rdiag = T.rdiag;
  for (int i = 0; i < mn; ++i) {
    // pivot: first index of the largest partial norm (idamax)
    if (w == 0) {
      double best = -1.0;
      int bi = i;
      for (int j = i + l; j < n; j += 32) {
        const double v = vn1[j];
        if (v > best) { best = v; bi = j; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (l == 0) s_pvt = bi;
    }
    __syncthreads();
    const int pvt = s_pvt;
    if (pvt != i) {
      double2* a = A + (size_t)pvt * m;
      double2* b = A + (size_t)i * m;
      for (int r = threadIdx.x; r < m; r += blockDim.x) {
        const double2 t = a[r];
        a[r] = b[r];
        b[r] = t;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const int t = jp[pvt];
        jp[pvt] = jp[i];
        jp[i] = t;
        vn1[pvt] = vn1[i];
        vn2[pvt] = vn2[i];
      }
      __syncthreads();
    }
    double beta;
    const double2 tau = householder(A, m, m, i, i, red, &beta);
    const double rii = fabs(beta);
    if (threadIdx.x == 0) {
      rdiag[i] = rii;
      if (i == 0) s_r00 = rii;
    }
    __syncthreads();
    const double r00 = s_r00;
    if (r00 == 0.0 || rii <= T.stop_rel * r00) {
      steps = i;
      break;
    }
    apply_reflector(A, m, m, i, i, tau, i + 1, n);
    __syncthreads();
    // partial norm downdate (zlaqp2)
    for (int j = i + 1 + w; j < n; j += nw) {
      const double v1 = vn1[j];
      if (v1 == 0.0) continue;
      const double2 aij = A[(size_t)j * m + i];
      double temp = hypot(aij.x, aij.y) / v1;
      temp = 1.0 - temp * temp;
      temp = temp > 0.0 ? temp : 0.0;
      const double ratio = v1 / vn2[j];
      const double temp2 = temp * ratio * ratio;
      if (temp2 <= tol3z) {
        double nv = 0.0;
        if (i + 1 < m) {
          const double2* c = A + (size_t)j * m;
          double s = 0.0;
          for (int r = i + 1 + l; r < m; r += 32) s = fma(c[r].x, c[r].x, fma(c[r].y, c[r].y, s));
          nv = sqrt(warp_sum(s));
        }
        if (l == 0) vn1[j] = vn2[j] = nv;
      } else {
        if (l == 0) vn1[j] = v1 * sqrt(temp);
      }
    }
    __syncthreads();
  }
  // outputs: pivots, steps, R rows [0, steps) in pivoted order (ld n)
  for (int j = threadIdx.x; j < n; j += blockDim.x) T.jpvt[j] = jp[j];
  if (threadIdx.x == 0) *T.steps = steps;
  double2* R = reinterpret_cast<double2*>(T.r_out);
  for (int idx = threadIdx.x; idx < steps * n; idx += blockDim.x) {
    const int j = idx / steps, i = idx - j * steps;
    R[(size_t)j * T.r_ld + i] = (i <= j) ? A[(size_t)j * m + i] : make_double2(0.0, 0.0);
  }
}

// ------------------------------------------------------------- interpolation
// coeff = [I, R11^-1 R12] (k x n) with column jpvt[j] <- column j.  Output
// (k x n, ld out_ld) or its conjugate transpose (n x k) when T.adjoint.
__global__ void __launch_bounds__(kThreads)
k_interp(const InterpTask* __restrict__ tasks) {
  const InterpTask T = tasks[blockIdx.x];
  const int k = T.k, n = T.n;
  if (k == 0) return;
  const double2* R = reinterpret_cast<const double2*>(T.r);
  double2* out = reinterpret_cast<double2*>(T.out);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  // R11 (k x k upper triangle) staged in shared memory once per task, so
  // the back substitutions' dependent steps read ~30-cycle shared memory,
  // not L2; then one warp per column j >= k of R12, lanes over rows
  extern __shared__ double2 col[];  // R11 [k][k] | Smith terms [k] | kWarps * k | branch [k]
  double2* Rs = col;
  double2* sd = col + (size_t)k * k;  // (ratio, denominator) of zdiv by R_rr
  double2* x = col + (size_t)k * k + k + w * k;
  int* br = reinterpret_cast<int*>(col + (size_t)k * k + k + kWarps * k);
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
    const int c = idx / k, r = idx - c * k;
    Rs[idx] = r <= c ? R[(size_t)c * T.r_ld + r] : make_double2(0.0, 0.0);
  }
  __syncthreads();
  // the divisor-only half of Smith's algorithm (zdiv), once per diagonal
  // entry, so each substitution step keeps two independent divisions
  for (int r = threadIdx.x; r < k; r += blockDim.x) {
    const double2 b = Rs[(size_t)r * k + r];
    br[r] = fabs(b.x) >= fabs(b.y);
    if (br[r]) {
      const double q = b.y / b.x;
      sd[r] = make_double2(q, b.x + b.y * q);
    } else {
      const double q = b.x / b.y;
      sd[r] = make_double2(q, b.y + b.x * q);
    }
  }
  __syncthreads();
  for (int j = k + w; j < n; j += kWarps) {
    for (int r = l; r < k; r += 32) x[r] = R[(size_t)j * T.r_ld + r];
    __syncwarp();
    for (int r = k - 1; r >= 0; --r) {
      if (l == 0) {  // x[r] / R_rr, Smith's algorithm (as zdiv)
        const double2 a = x[r], q = sd[r];
        if (br[r])
          x[r] = make_double2((a.x + a.y * q.x) / q.y, (a.y - a.x * q.x) / q.y);
        else
          x[r] = make_double2((a.x * q.x + a.y) / q.y, (a.y * q.x - a.x) / q.y);
      }
      __syncwarp();
      const double2 xr = x[r];
      for (int q = l; q < r; q += 32) x[q] = zfms(x[q], Rs[(size_t)r * k + q], xr);
      __syncwarp();
    }
    const int dc = T.jpvt[j];
    for (int r = l; r < k; r += 32) {
      if (T.adjoint) out[(size_t)r * T.out_ld + dc] = zconj(x[r]);
      else out[(size_t)dc * T.out_ld + r] = x[r];
    }
    __syncwarp();
  }
  // identity part
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
    const int j = idx / k, r = idx - j * k;
    const int dc = T.jpvt[j];
    const double2 v = make_double2(r == j ? 1.0 : 0.0, 0.0);
    if (T.adjoint) out[(size_t)r * T.out_ld + dc] = v;
    else out[(size_t)dc * T.out_ld + r] = v;
  }
}

// ----------------------------------------------------------------------- LU
__global__ void __launch_bounds__(kQrThreads)
k_getrf(const LuTask* __restrict__ tasks, double2* __restrict__ gws) {
  extern __shared__ double2 smem[];
  __shared__ int s_p;
  __shared__ int s_info;
  const LuTask T = tasks[blockIdx.x];
  const int n = T.n;
  double2* G = reinterpret_cast<double2*>(T.a);
  double2* A = T.in_smem ? smem : gws + T.ws_off;
  load_block(G, n, n, T.ld, A);
  if (threadIdx.x == 0) s_info = 0;
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#if EBEM_GETRF_LA
  // Look-ahead elimination, one CTA barrier per column: in step k warp 0
  // finishes column k + 1 (interchange and update by column k, then its
  // pivot search, interchange and scaling) while the other warps interchange
  // and update the columns right of it and interchange the L columns left of
  // k.  Every element sees the same operations in the same order as the
  // unblocked sequence below (bitwise-identical factors).
  const int nw = blockDim.x >> 5;
  auto pivot_col = [&](int k) {  // warp 0: pivot of column k, interchange + scale it
    double best = -1.0;
    int bi = k;
    for (int r = k + l; r < n; r += 32) {
      const double v = cabs1(A[(size_t)k * n + r]);
      if (v > best) { best = v; bi = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (l == 0) {
      s_p = bi;
      T.ipiv[k] = bi;
      if (best == 0.0 && s_info == 0) s_info = k + 1;
    }
    if (bi != k && l == 0) {
      const double2 t = A[(size_t)k * n + k];
      A[(size_t)k * n + k] = A[(size_t)k * n + bi];
      A[(size_t)k * n + bi] = t;
    }
    __syncwarp();
    const double2 piv = A[(size_t)k * n + k];
    if (piv.x != 0.0 || piv.y != 0.0) {
      const double2 rp = zdiv(make_double2(1.0, 0.0), piv);
      for (int r = k + 1 + l; r < n; r += 32)
        A[(size_t)k * n + r] = zmul(A[(size_t)k * n + r], rp);
    }
  };
  if (w == 0) pivot_col(0);
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    const int p = s_p;  // pivot of column k (applied to column k, which is scaled)
    __syncthreads();    // everyone read s_p before warp 0 overwrites it
    auto swap_update = [&](int j) {  // column j > k: interchange rows k, p; update
      if (p != k && l == 0) {
        const double2 t = A[(size_t)j * n + k];
        A[(size_t)j * n + k] = A[(size_t)j * n + p];
        A[(size_t)j * n + p] = t;
      }
      __syncwarp();
      const double2 akj = A[(size_t)j * n + k];
      for (int r = k + 1 + l; r < n; r += 32)
        A[(size_t)j * n + r] = zfms(A[(size_t)j * n + r], A[(size_t)k * n + r], akj);
      __syncwarp();
    };
    if (w == 0) {
      if (k + 1 < n) {
        swap_update(k + 1);
        pivot_col(k + 1);
      }
    } else {
      for (int j = k + 2 + (w - 1); j < n; j += nw - 1) swap_update(j);
      if (p != k)
        for (int j = (w - 1) * 32 + l; j < k; j += (nw - 1) * 32) {
          const double2 t = A[(size_t)j * n + k];
          A[(size_t)j * n + k] = A[(size_t)j * n + p];
          A[(size_t)j * n + p] = t;
        }
    }
    __syncthreads();
  }
#else
  for (int k = 0; k < n; ++k) {
    if (w == 0) {
      double best = -1.0;
      int bi = k;
      for (int r = k + l; r < n; r += 32) {
        const double v = cabs1(A[(size_t)k * n + r]);
        if (v > best) { best = v; bi = r; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (l == 0) {
        s_p = bi;
        T.ipiv[k] = bi;
        if (best == 0.0 && s_info == 0) s_info = k + 1;
      }
    }
    __syncthreads();
    const int p = s_p;
    if (p != k) {
      for (int j = threadIdx.x; j < n; j += blockDim.x) {
        const double2 t = A[(size_t)j * n + k];
        A[(size_t)j * n + k] = A[(size_t)j * n + p];
        A[(size_t)j * n + p] = t;
      }
      __syncthreads();
    }
    const double2 piv = A[(size_t)k * n + k];
    if (piv.x != 0.0 || piv.y != 0.0) {
      const double2 rp = zdiv(make_double2(1.0, 0.0), piv);
      for (int r = k + 1 + threadIdx.x; r < n; r += blockDim.x)
        A[(size_t)k * n + r] = zmul(A[(size_t)k * n + r], rp);
    }
    __syncthreads();
    // rank-1 update of the trailing block, one warp per column
    for (int j = k + 1 + w; j < n; j += (int)(blockDim.x >> 5)) {
      const double2 akj = A[(size_t)j * n + k];
      for (int r = k + 1 + l; r < n; r += 32)
        A[(size_t)j * n + r] = zfms(A[(size_t)j * n + r], A[(size_t)k * n + r], akj);
    }
    __syncthreads();
  }
#endif
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int j = idx / n, i = idx - j * n;
    G[(size_t)j * T.ld + i] = A[idx];
  }
  if (threadIdx.x == 0) *T.info = s_info;
}

// ---------------------------------------------------------------- LU solve
// One warp per right-hand-side column.  grid = (task, column group).  The
// LU factors (and the columns) are staged in shared memory when they fit, so
// the dependent substitution steps hit ~30-cycle shared memory, not L2.
__global__ void __launch_bounds__(kThreads)
k_getrs(const LuSolveTask* __restrict__ tasks, const int* __restrict__ block_off,
        int n_tasks, int cap) {
  extern __shared__ double2 sm[];
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (block_off[mid] <= (int)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const LuSolveTask T = tasks[lo];
  const int n = T.n;
  const bool stage = (long long)n * n + (long long)kWarps * n <= cap;
  const double2* A = reinterpret_cast<const double2*>(T.lu);
  size_t lda = T.ld;
  if (stage) {
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
      const int j = idx / n, i = idx - j * n;
      sm[idx] = A[(size_t)j * lda + i];
    }
    A = sm;
    lda = n;
  }
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int col = (blockIdx.x - block_off[lo]) * kWarps + w;
  if (col >= T.nrhs) return;
  double2* bg = reinterpret_cast<double2*>(T.b) + (size_t)col * T.ldb;
  double2* b = bg;
  if (stage) {
    b = sm + (size_t)n * n + (size_t)w * n;
    for (int r = l; r < n; r += 32) b[r] = bg[r];
    __syncwarp();
  }
  // row interchanges in order
  if (l == 0) {
    for (int k = 0; k < n; ++k) {
      const int p = T.ipiv[k];
      if (p != k) {
        const double2 t = b[k];
        b[k] = b[p];
        b[p] = t;
      }
    }
  }
  __syncwarp();
  // L y = b (unit lower)
  for (int k = 0; k < n; ++k) {
    const double2 bk = b[k];
    for (int r = k + 1 + l; r < n; r += 32) b[r] = zfms(b[r], A[(size_t)k * lda + r], bk);
    __syncwarp();
  }
  // U x = y
  for (int k = n - 1; k >= 0; --k) {
    if (l == 0) b[k] = zdiv(b[k], A[(size_t)k * lda + k]);
    __syncwarp();
    const double2 xk = b[k];
    for (int r = l; r < k; r += 32) b[r] = zfms(b[r], A[(size_t)k * lda + r], xk);
    __syncwarp();
  }
  if (stage)
    for (int r = l; r < n; r += 32) bg[r] = b[r];
}

// --------------------------------------------------------------------- GEMM
// C = alpha op(A) op(B) + beta C; 32x32 output tile per CTA, 256 threads,
// each thread 4 outputs; K staged through shared memory in chunks of 16.
constexpr int kTile = 32;
constexpr int kKc = 16;

__global__ void __launch_bounds__(kThreads)
k_gemm(const GemmTask* __restrict__ tasks, const int* __restrict__ block_off,
       int n_tasks) {
  __shared__ double2 As[kKc][kTile + 1];
  __shared__ double2 Bs[kKc][kTile + 1];
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (block_off[mid] <= (int)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const GemmTask T = tasks[lo];
  const int tiles_m = (T.m + kTile - 1) / kTile;
  const int tile = blockIdx.x - block_off[lo];
  const int tm = tile % tiles_m, tn = tile / tiles_m;
  const int r0 = tm * kTile, c0 = tn * kTile;
  const double2* A = reinterpret_cast<const double2*>(T.a);
  const double2* B = reinterpret_cast<const double2*>(T.b);
  double2* C = reinterpret_cast<double2*>(T.c);
  const int tr = threadIdx.x & 31;        // row in tile
  const int tc = (threadIdx.x >> 5) * 4;  // 4 columns per thread
  double2 acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < T.k; k0 += kKc) {
    // stage A tile (rows r0.., k k0..) and B tile (k k0.., cols c0..)
    for (int idx = threadIdx.x; idx < kKc * kTile; idx += kThreads) {
      const int kk = idx / kTile, rr = idx - kk * kTile;
      const int gr = r0 + rr, gk = k0 + kk;
      double2 va = make_double2(0.0, 0.0);
      if (gr < T.m && gk < T.k) {
        va = T.trans_a ? A[(size_t)gr * T.lda + gk] : A[(size_t)gk * T.lda + gr];
        if (T.trans_a == 2) va = zconj(va);
      }
      As[kk][rr] = va;
      const int gc = c0 + rr;
      double2 vb = make_double2(0.0, 0.0);
      if (gc < T.n && gk < T.k) {
        vb = T.trans_b ? B[(size_t)gk * T.ldb + gc] : B[(size_t)gc * T.ldb + gk];
        if (T.trans_b == 2) vb = zconj(vb);
      }
      Bs[kk][rr] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kKc; ++kk) {
      const double2 a = As[kk][tr];
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[q] = zfma(acc[q], a, Bs[kk][tc + q]);
    }
    __syncthreads();
  }
  const double2 alpha = make_double2(T.alpha_re, T.alpha_im);
  const double2 beta = make_double2(T.beta_re, T.beta_im);
  const int gr = r0 + tr;
  if (gr >= T.m) return;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int gc = c0 + tc + q;
    if (gc >= T.n) continue;
    double2* cp = C + (size_t)gc * T.ldc + gr;
    double2 v = zmul(alpha, acc[q]);
    if (beta.x != 0.0 || beta.y != 0.0) v = zfma(v, beta, *cp);
    *cp = v;
  }
}

// ------------------------------------------------- GEMM on FP64 tensor cores
// The same product on the FP64 MMA units: mma.sync.m8n8k4 f64 (DMMA), one
// 8x8x4 real product per warp instruction (8 x the work of a DFMA warp
// instruction).  A complex product is four real MMAs on split re / im
// fragments (C_re += A_re B_re - A_im B_im, C_im += A_re B_im + A_im B_re),
// the same operation count as the SIMT kernel and no 3-multiply trick, so the
// rounding stays that of a plain complex dot product.
//   CTA 128 threads = 4 warps, 32 x 32 complex output tile, warp 16 x 16
//   (2 x 2 MMA blocks).  K in chunks of 16 complex, staged by cp.async into a
//   two-stage ring of [row][k] tiles (the copy of chunk c+1 overlaps the
//   MMAs of chunk c); out-of-range elements are zero-filled by the copy.
//   The 20-element row pitch (80 words = 16 mod 32) makes the 16-byte
//   fragment loads (re and im of one element together) conflict-free.
constexpr int kMmaThreads = 128;
constexpr int kMmaKc = 16;
constexpr int kMmaPitch = kMmaKc + 4;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// 16-byte async copy; src_bytes = 0 zero-fills the destination
__device__ __forceinline__ void cp16z(void* dst, const void* src, int src_bytes) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src),
               "r"(src_bytes));
}

__global__ void __launch_bounds__(kMmaThreads)
k_gemm_mma(const GemmTask* __restrict__ tasks, const int* __restrict__ block_off,
           int n_tasks) {
  __shared__ double2 As[2][kTile][kMmaPitch];
  __shared__ double2 Bs[2][kTile][kMmaPitch];
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (block_off[mid] <= (int)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const GemmTask& T = tasks[lo];
  const int m = T.m, n = T.n, kdim = T.k, lda = T.lda, ldb = T.ldb;
  const int ta = T.trans_a, tb = T.trans_b;
  const int tiles_m = (m + kTile - 1) / kTile;
  const int tile = blockIdx.x - block_off[lo];
  const int r0 = (tile % tiles_m) * kTile, c0 = (tile / tiles_m) * kTile;
  const double2* __restrict__ A = reinterpret_cast<const double2*>(T.a);
  const double2* __restrict__ B = reinterpret_cast<const double2*>(T.b);
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  // chunk copy: 4 elements of A and 4 of B per thread; consecutive threads
  // on consecutive global addresses
  auto issue = [&](int k0, int st) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int idx = tid + kMmaThreads * q;
      int row, kk;
      if (ta) { row = idx / kMmaKc; kk = idx % kMmaKc; }
      else { row = idx % kTile; kk = idx / kTile; }
      int gr = r0 + row, gk = k0 + kk;
      bool ok = gr < m && gk < kdim;
      const double2* src = ok ? (ta ? A + (size_t)gr * lda + gk : A + (size_t)gk * lda + gr) : A;
      cp16z(&As[st][row][kk], src, ok ? 16 : 0);
      int col;
      if (tb) { col = idx % kTile; kk = idx / kTile; }
      else { col = idx / kMmaKc; kk = idx % kMmaKc; }
      const int gc = c0 + col;
      gk = k0 + kk;
      ok = gc < n && gk < kdim;
      src = ok ? (tb ? B + (size_t)gk * ldb + gc : B + (size_t)gc * ldb + gk) : B;
      cp16z(&Bs[st][col][kk], src, ok ? 16 : 0);
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  double acc[2][2][2][2];  // [row block][col block][re, im][2]
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int c = 0; c < 2; ++c) acc[i][j][c][0] = acc[i][j][c][1] = 0.0;
  const int wr = (w & 1) * 16, wc = (w >> 1) * 16;
  const int fr = lane >> 2, fk = lane & 3;
  const bool live_r[2] = {r0 + wr < m, r0 + wr + 8 < m};
  const bool live_c[2] = {c0 + wc < n, c0 + wc + 8 < n};
  const double sa = ta == 2 ? -1.0 : 1.0, sb = tb == 2 ? -1.0 : 1.0;  // conjugation
  const int nck = (kdim + kMmaKc - 1) / kMmaKc;
  issue(0, 0);
  for (int c = 0; c < nck; ++c) {
    const int st = c & 1;
    if (c + 1 < nck) {
      issue((c + 1) * kMmaKc, st ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const int ks_end = min(kMmaKc, kdim - c * kMmaKc);
#pragma unroll
    for (int ks = 0; ks < kMmaKc; ks += 4) {
      if (ks >= ks_end) break;
      double ar[2], ai[2], an[2], br[2], bi[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const double2 a = As[st][wr + 8 * i + fr][ks + fk];
        const double2 b = Bs[st][wc + 8 * i + fr][ks + fk];
        ar[i] = a.x;
        ai[i] = sa * a.y;
        an[i] = -ai[i];
        br[i] = b.x;
        bi[i] = sb * b.y;
      }
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          // 8 x 8 sub-tiles wholly outside m x n (the padding of m = k, n = 2k
          // to 32 x 32 tiles) issue no MMAs (warp-uniform)
          if (!live_r[i] || !live_c[j]) continue;
          dmma(acc[i][j][0][0], acc[i][j][0][1], ar[i], br[j]);
          dmma(acc[i][j][0][0], acc[i][j][0][1], an[i], bi[j]);
          dmma(acc[i][j][1][0], acc[i][j][1][1], ar[i], bi[j]);
          dmma(acc[i][j][1][0], acc[i][j][1][1], ai[i], br[j]);
        }
    }
    __syncthreads();  // stage st is refilled by the next iteration's copy
  }
  const double2 alpha = make_double2(T.alpha_re, T.alpha_im);
  const double2 beta = make_double2(T.beta_re, T.beta_im);
  const bool acc_c = beta.x != 0.0 || beta.y != 0.0;
  double2* C = reinterpret_cast<double2*>(T.c);
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int gr = r0 + wr + 8 * i + fr;
    if (gr >= m) continue;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gc = c0 + wc + 8 * j + 2 * fk + h;
        if (gc >= n) continue;
        double2* cp = C + (size_t)gc * T.ldc + gr;
        double2 v = zmul(alpha, make_double2(acc[i][j][0][h], acc[i][j][1][h]));
        if (acc_c) v = zfma(v, beta, *cp);
        *cp = v;
      }
  }
}

// ------------------------------------------------------ narrow GEMM (GEMV)
// C = alpha A B + beta C with at most kNarrow columns in B and C and no
// transposes: the solve's per-cell products with one or a few right-hand
// sides, bound by reading A once.  One CTA per 32-row tile: lane = row
// (coalesced column reads of A), the 8 warps split K and are summed through
// shared memory in a fixed order (deterministic).
template <int NR>
__global__ void __launch_bounds__(kThreads)
k_gemv(const GemmTask* __restrict__ tasks, const int* __restrict__ block_off, int n_tasks) {
  __shared__ double2 part[kWarps][NR][32];
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (block_off[mid] <= (int)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const GemmTask T = tasks[lo];
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int r = (blockIdx.x - block_off[lo]) * 32 + l;
  const double2* A = reinterpret_cast<const double2*>(T.a);
  const double2* B = reinterpret_cast<const double2*>(T.b);
  double2 acc[NR];
#pragma unroll
  for (int c = 0; c < NR; ++c) acc[c] = make_double2(0.0, 0.0);
  if (r < T.m) {
#pragma unroll 4
    for (int k = w; k < T.k; k += kWarps) {
      const double2 a = __ldg(A + (size_t)k * T.lda + r);
#pragma unroll
      for (int c = 0; c < NR; ++c)
        if (c < T.n) acc[c] = zfma(acc[c], a, __ldg(B + (size_t)c * T.ldb + k));
    }
  }
#pragma unroll
  for (int c = 0; c < NR; ++c) part[w][c][l] = acc[c];
  __syncthreads();
  if (w != 0 || r >= T.m) return;
  const double2 alpha = make_double2(T.alpha_re, T.alpha_im);
  const double2 beta = make_double2(T.beta_re, T.beta_im);
  double2* C = reinterpret_cast<double2*>(T.c);
#pragma unroll
  for (int c = 0; c < NR; ++c) {
    if (c >= T.n) break;
    double2 s = part[0][c][l];
#pragma unroll
    for (int q = 1; q < kWarps; ++q) s = make_double2(s.x + part[q][c][l].x, s.y + part[q][c][l].y);
    double2* cp = C + (size_t)c * T.ldc + r;
    double2 v = zmul(alpha, s);
    if (beta.x != 0.0 || beta.y != 0.0) v = zfma(v, beta, *cp);
    *cp = v;
  }
}

// Warp-per-tile variant (the default): CTA = 8 independent warps, warp =
// one 32-row tile of one task running over all of K (no K split, no
// shared-memory sum, no CTA barrier), 8 columns of A in flight per lane;
// the right-hand-side entries are read 32 at a time by the lanes and
// broadcast by shuffles.  8x fewer CTAs than k_gemv for the same tiles:
// the solve's per-cell products are a few KB each, so per-CTA overhead, not
// HBM, bounded k_gemv.
template <int NR>
__global__ void __launch_bounds__(kThreads)
k_gemv_w(const GemmTask* __restrict__ tasks, const int* __restrict__ tile_off, int n_tasks,
         int n_tiles) {
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int tile = blockIdx.x * kWarps + w;
  if (tile >= n_tiles) return;
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(tile_off + mid) <= tile) lo = mid;
    else hi = mid - 1;
  }
  const GemmTask& T = tasks[lo];
  const int m = T.m, kdim = T.k, ncol = T.n;
  const size_t lda = T.lda, ldb = T.ldb;
  const int r = (tile - __ldg(tile_off + lo)) * 32 + l;
  const bool live = r < m;
  const double2* __restrict__ A = reinterpret_cast<const double2*>(T.a) + (live ? r : 0);
  const double2* __restrict__ B = reinterpret_cast<const double2*>(T.b);
  double2 acc[NR];
#pragma unroll
  for (int c = 0; c < NR; ++c) acc[c] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < kdim; k0 += 32) {
    const int kk = min(32, kdim - k0);
    double2 xb[NR];
#pragma unroll
    for (int c = 0; c < NR; ++c)
      xb[c] = (c < ncol && l < kk) ? __ldg(B + (size_t)c * ldb + k0 + l) : make_double2(0.0, 0.0);
#pragma unroll 8
    for (int j = 0; j < kk; ++j) {
      const double2 a = live ? __ldg(A + (size_t)(k0 + j) * lda) : make_double2(0.0, 0.0);
#pragma unroll
      for (int c = 0; c < NR; ++c) {
        const double2 x = make_double2(__shfl_sync(0xffffffffu, xb[c].x, j),
                                       __shfl_sync(0xffffffffu, xb[c].y, j));
        acc[c] = zfma(acc[c], a, x);
      }
    }
  }
  if (!live) return;
  const double2 alpha = make_double2(T.alpha_re, T.alpha_im);
  const double2 beta = make_double2(T.beta_re, T.beta_im);
  double2* C = reinterpret_cast<double2*>(T.c);
#pragma unroll
  for (int c = 0; c < NR; ++c) {
    if (c >= ncol) break;
    double2* cp = C + (size_t)c * T.ldc + r;
    double2 v = zmul(alpha, acc[c]);
    if (beta.x != 0.0 || beta.y != 0.0) v = zfma(v, beta, *cp);
    *cp = v;
  }
}

// --------------------------------------------------------------------- copy
constexpr int kCopyUnit = 128;  // elements per warp
__global__ void __launch_bounds__(kThreads)
k_copy(const CopyTask* __restrict__ tasks, const int* __restrict__ unit_off,
       int n_tasks, int n_units) {
  // one warp per unit of kCopyUnit elements (most solve copies are a few
  // dozen elements: a CTA per task would idle 7 of its 8 warps)
  const int unit = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (unit >= n_units) return;
  const int l = threadIdx.x & 31;
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(unit_off + mid) <= unit) lo = mid;
    else hi = mid - 1;
  }
  const CopyTask T = tasks[lo];
  const long long base = (long long)(unit - __ldg(unit_off + lo)) * kCopyUnit;
  const double2* S = reinterpret_cast<const double2*>(T.src);
  double2* D = reinterpret_cast<double2*>(T.dst);
  const long long total = (long long)T.rows * T.cols;
  for (int q = 0; q < kCopyUnit / 32; ++q) {
    const long long idx = base + q * 32 + l;
    if (idx >= total) break;
    const int j = int(idx / T.rows), i = int(idx - (long long)j * T.rows);
    double2 v = T.src ? S[(size_t)j * T.src_ld + i] : make_double2(0.0, 0.0);
    if (T.transpose == 2) v = make_double2(i == j ? 1.0 : 0.0, 0.0);  // identity
    if (T.conj) v = zconj(v);
    if (T.transpose == 1) D[(size_t)i * T.dst_ld + j] = v;
    else D[(size_t)j * T.dst_ld + i] = v;
  }
}

// ----------------------------------------------------- LU solve, registers
// One warp per kCpw right-hand sides; lane l holds rows l, l + 32, ... of
// each (kMaxS slots).  The LU (and 1 / U_kk) is staged in shared memory when
// it fits and shared by the CTA's 8 warps; every row value travels by
// shuffle, so the substitutions need no warp barriers and no division.
constexpr int kCpw = 4;  // right-hand sides per warp for wide batches (1 for narrow)

__device__ __forceinline__ double2 zrcp(double2 a) {
  // 1 / a by Smith's method with reciprocals only
  if (fabs(a.x) >= fabs(a.y)) {
    const double r = a.y * (1.0 / a.x), d = 1.0 / fma(a.y, r, a.x);
    return make_double2(d, -r * d);
  }
  const double r = a.x * (1.0 / a.y), d = 1.0 / fma(a.x, r, a.y);
  return make_double2(r * d, -d);
}

template <int kMaxS>
__device__ __forceinline__ double2 pick(const double2 (&v)[kMaxS], int s) {
  double2 o = v[0];
#pragma unroll
  for (int q = 1; q < kMaxS; ++q)
    if (q == s) o = v[q];
  return o;
}
template <int kMaxS>
__device__ __forceinline__ void put(double2 (&v)[kMaxS], int s, double2 x) {
#pragma unroll
  for (int q = 0; q < kMaxS; ++q)
    if (q == s) v[q] = x;
}
__device__ __forceinline__ double2 shfl2(double2 v, int src) {
  return make_double2(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}

template <int kMaxS, int CPW>
__global__ void __launch_bounds__(kThreads)
k_getrs_reg(const LuSolveTask* __restrict__ tasks, const int* __restrict__ block_off,
            int n_tasks, int cap) {
  extern __shared__ double2 sm[];
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (block_off[mid] <= (int)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const LuSolveTask T = tasks[lo];
  const int n = T.n;
  const bool stage = (long long)n * n + n <= cap;
  const double2* A = reinterpret_cast<const double2*>(T.lu);
  size_t lda = T.ld;
  double2* invd = sm + (stage ? (size_t)n * n : 0);
  if (stage) {
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
      const int j = idx / n, i = idx - j * n;
      sm[idx] = A[(size_t)j * lda + i];
    }
    A = sm;
    lda = n;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < n; k += blockDim.x) invd[k] = zrcp(A[(size_t)k * lda + k]);
  __syncthreads();
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int col0 = ((blockIdx.x - block_off[lo]) * kWarps + w) * CPW;
  if (col0 >= T.nrhs) return;
  double2 b[CPW][kMaxS];
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    const int col = col0 + c;
    const double2* bg = reinterpret_cast<const double2*>(T.b) + (size_t)col * T.ldb;
#pragma unroll
    for (int s = 0; s < kMaxS; ++s) {
      const int r = l + 32 * s;
      b[c][s] = (col < T.nrhs && r < n) ? bg[r] : make_double2(0.0, 0.0);
    }
  }
  // row interchanges in order (warp-uniform pivots)
  for (int k = 0; k < n; ++k) {
    const int p = __ldg(T.ipiv + k);
    if (p == k) continue;
    const int sk = k >> 5, lk = k & 31, sp = p >> 5, lp = p & 31;
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      const double2 vk = shfl2(pick(b[c], sk), lk);
      const double2 vp = shfl2(pick(b[c], sp), lp);
      if (l == lk) put(b[c], sk, vp);
      if (l == lp) put(b[c], sp, vk);
    }
  }
  // L y = b (unit lower)
  for (int k = 0; k < n - 1; ++k) {
    const int sk = k >> 5, lk = k & 31;
    double2 bk[CPW];
#pragma unroll
    for (int c = 0; c < CPW; ++c) bk[c] = shfl2(pick(b[c], sk), lk);
    const double2* Ak = A + (size_t)k * lda;
#pragma unroll
    for (int s = 0; s < kMaxS; ++s) {
      const int r = l + 32 * s;
      if (r > k && r < n) {
        const double2 a = Ak[r];
#pragma unroll
        for (int c = 0; c < CPW; ++c) b[c][s] = zfms(b[c][s], a, bk[c]);
      }
    }
  }
  // U x = y
  for (int k = n - 1; k >= 0; --k) {
    const int sk = k >> 5, lk = k & 31;
    const double2 ik = invd[k];
    double2 xk[CPW];
#pragma unroll
    for (int c = 0; c < CPW; ++c) {
      xk[c] = zmul(shfl2(pick(b[c], sk), lk), ik);
      if (l == lk) put(b[c], sk, xk[c]);
    }
    const double2* Ak = A + (size_t)k * lda;
#pragma unroll
    for (int s = 0; s < kMaxS; ++s) {
      const int r = l + 32 * s;
      if (r < k) {
        const double2 a = Ak[r];
#pragma unroll
        for (int c = 0; c < CPW; ++c) b[c][s] = zfms(b[c][s], a, xk[c]);
      }
    }
  }
#pragma unroll
  for (int c = 0; c < CPW; ++c) {
    const int col = col0 + c;
    if (col >= T.nrhs) break;
    double2* bg = reinterpret_cast<double2*>(T.b) + (size_t)col * T.ldb;
#pragma unroll
    for (int s = 0; s < kMaxS; ++s) {
      const int r = l + 32 * s;
      if (r < n) bg[r] = b[c][s];
    }
  }
}

// ------------------------------------------------- LU solve, one warp each
// For a few right-hand sides every LU entry is read once, so staging the LU in
// shared memory buys nothing: one warp per (task, right-hand side), the CTA's
// warps serve different cells, lane l holds rows l, l + 32, ... and the next
// column of L / U (and the next reciprocal diagonal) is loaded one step ahead
// of the substitution that needs it.
template <int kMaxS>
__global__ void __launch_bounds__(kThreads)
k_getrs_warp(const LuSolveTask* __restrict__ tasks, const int* __restrict__ warp_off,
             int n_tasks, int n_warps) {
  const int gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const int l = threadIdx.x & 31;
  if (gw >= n_warps) return;  // warp-uniform
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(warp_off + mid) <= gw) lo = mid;
    else hi = mid - 1;
  }
  const LuSolveTask T = tasks[lo];
  const int n = T.n;
  const int col = gw - __ldg(warp_off + lo);
  if (col >= T.nrhs || n <= 0) return;
  const double2* A = reinterpret_cast<const double2*>(T.lu);
  const size_t lda = T.ld;
  double2* bg = reinterpret_cast<double2*>(T.b) + (size_t)col * T.ldb;
  double2 b[kMaxS];
#pragma unroll
  for (int s = 0; s < kMaxS; ++s) {
    const int r = l + 32 * s;
    b[s] = r < n ? bg[r] : make_double2(0.0, 0.0);
  }
  auto load_col = [&](int k, double2 (&c)[kMaxS]) {
    const double2* Ak = A + (size_t)k * lda;
#pragma unroll
    for (int s = 0; s < kMaxS; ++s) {
      const int r = l + 32 * s;
      c[s] = r < n ? __ldg(Ak + r) : make_double2(0.0, 0.0);
    }
  };
  int piv[kMaxS];  // lane l holds ipiv[l + 32 s]
#pragma unroll
  for (int s = 0; s < kMaxS; ++s) {
    const int r = l + 32 * s;
    piv[s] = r < n ? __ldg(T.ipiv + r) : r;
  }
  double2 cur[kMaxS], nxt[kMaxS];
  load_col(0, nxt);
  for (int k = 0; k < n; ++k) {  // row interchanges in order (warp-uniform)
    const int sk = k >> 5, lk = k & 31;
    int p = piv[0];
#pragma unroll
    for (int s = 1; s < kMaxS; ++s)
      if (s == sk) p = piv[s];
    p = __shfl_sync(0xffffffffu, p, lk);
    if (p == k) continue;
    const int sp = p >> 5, lp = p & 31;
    const double2 vk = shfl2(pick(b, sk), lk);
    const double2 vp = shfl2(pick(b, sp), lp);
    if (l == lk) put(b, sk, vp);
    if (l == lp) put(b, sp, vk);
  }
  // L y = b (unit lower)
  for (int k = 0; k < n - 1; ++k) {
#pragma unroll
    for (int s = 0; s < kMaxS; ++s) cur[s] = nxt[s];
    if (k + 1 < n - 1) load_col(k + 1, nxt);
    const double2 bk = shfl2(pick(b, k >> 5), k & 31);
#pragma unroll
    for (int s = 0; s < kMaxS; ++s) {
      const int r = l + 32 * s;
      if (r > k && r < n) b[s] = zfms(b[s], cur[s], bk);
    }
  }
  // U x = y
  load_col(n - 1, nxt);
  double2 dnext = __ldg(A + (size_t)(n - 1) * lda + (n - 1));
  for (int k = n - 1; k >= 0; --k) {
#pragma unroll
    for (int s = 0; s < kMaxS; ++s) cur[s] = nxt[s];
    const double2 ik = zrcp(dnext);
    if (k > 0) {
      load_col(k - 1, nxt);
      dnext = __ldg(A + (size_t)(k - 1) * lda + (k - 1));
    }
    const int sk = k >> 5, lk = k & 31;
    const double2 xk = zmul(shfl2(pick(b, sk), lk), ik);
    if (l == lk) put(b, sk, xk);
#pragma unroll
    for (int s = 0; s < kMaxS; ++s) {
      const int r = l + 32 * s;
      if (r < k) b[s] = zfms(b[s], cur[s], xk);
    }
  }
#pragma unroll
  for (int s = 0; s < kMaxS; ++s) {
    const int r = l + 32 * s;
    if (r < n) bg[r] = b[s];
  }
}

// The row interchanges of an LU composed into one permutation: perm[r] is the
// row of b that ends up in row r (swaps applied in order to the identity).
// One warp per task; the serial part runs on shared memory.
constexpr int kPermWarps = 4;
__global__ void __launch_bounds__(32 * kPermWarps)
k_pivots_to_perm(const LuTask* __restrict__ tasks, int n_tasks) {
  __shared__ int sm[kPermWarps][2 * kPermMaxN];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = blockIdx.x * kPermWarps + warp;
  if (task >= n_tasks) return;
  const LuTask T = tasks[task];
  if (T.perm == nullptr || T.n > kPermMaxN) return;
  int* idx = sm[warp];
  int* piv = idx + kPermMaxN;
  for (int r = lane; r < T.n; r += 32) {
    idx[r] = r;
    piv[r] = T.ipiv[r];
  }
  __syncwarp();
  if (lane == 0)
    for (int k = 0; k < T.n; ++k) {
      const int p = piv[k];
      if (p != k) {
        const int v = idx[k];
        idx[k] = idx[p];
        idx[p] = v;
      }
    }
  __syncwarp();
  for (int r = lane; r < T.n; r += 32) T.perm[r] = idx[r];
}

// ------------------------------------------------ LU solve, one CTA each
// One CTA (kThreads) per (task, right-hand side) for orders up to
// kThreads * kS: thread t keeps rows t, t + kThreads, ... in registers and
// loads its part of the next column of L / U one step ahead; the new x_k goes
// through a two-slot shared-memory broadcast, one barrier per step.  The row
// interchanges run in shared memory first (LAPACK order, one thread).
template <int kS>
__global__ void __launch_bounds__(kThreads)
k_getrs_cta(const LuSolveTask* __restrict__ tasks, const int* __restrict__ block_off,
            int n_tasks) {
  // columns of L / U stream PF steps ahead through a per-thread shared-memory
  // ring filled by cp.async (a CTA barrier would wait for register loads,
  // not for these); each thread reads back only the entries it copied
  constexpr int PF = kS >= 8 ? 2 : 16 / kS;
  extern __shared__ double2 sx[];  // ring [PF][kS][kThreads] | x (n) | ipiv (n ints)
  __shared__ double2 bc[2];
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (block_off[mid] <= (int)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const LuSolveTask T = tasks[lo];
  const int col = blockIdx.x - block_off[lo];
  if (col >= T.nrhs) return;
  const int n = T.n;
  if (n <= 0) return;
  const int t = threadIdx.x;
  const double2* A = reinterpret_cast<const double2*>(T.lu);
  const size_t lda = T.ld;
  double2* bg = reinterpret_cast<double2*>(T.b) + (size_t)col * T.ldb;
  double2* ring = sx;
  double2* xs = sx + PF * kS * kThreads;
  int* sp = reinterpret_cast<int*>(xs + n);
  auto slot = [&](int q, int s) -> double2& { return ring[(q * kS + s) * kThreads + t]; };
  auto fetch = [&](int k, int q) {  // column k -> slot q (own rows), one group
    if (k >= 0 && k < n) {
      const double2* Ak = A + (size_t)k * lda;
#pragma unroll
      for (int s = 0; s < kS; ++s) {
        const int r = t + kThreads * s;
        if (r < n) {
          const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(&slot(q, s)));
          asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(Ak + r));
        }
      }
    }
    asm volatile("cp.async.commit_group;\n" ::);
  };
  auto wait_oldest = [] { asm volatile("cp.async.wait_group %0;\n" ::"n"(PF - 1) : "memory"); };
  const bool permuted = T.perm != nullptr;  // CTA-uniform
  for (int r = t; r < n; r += kThreads) {
    if (permuted) {
      xs[r] = bg[__ldg(T.perm + r)];
    } else {
      xs[r] = bg[r];
      sp[r] = __ldg(T.ipiv + r);
    }
  }
#pragma unroll
  for (int q = 0; q < PF; ++q) fetch(q < n - 1 ? q : -1, q);
  __syncthreads();
  if (t == 0 && !permuted)
    for (int k = 0; k < n; ++k) {
      const int p = sp[k];
      if (p != k) {
        const double2 v = xs[k];
        xs[k] = xs[p];
        xs[p] = v;
      }
    }
  __syncthreads();
  double2 b[kS];
#pragma unroll
  for (int s = 0; s < kS; ++s) {
    const int r = t + kThreads * s;
    b[s] = r < n ? xs[r] : make_double2(0.0, 0.0);
  }
  // 1 / U_rr of the thread's own rows, formed here so that the division is
  // off the substitution chain of the U phase (same operations, same bits)
  double2 rinv[kS];
#pragma unroll
  for (int s = 0; s < kS; ++s) {
    const int r = t + kThreads * s;
    rinv[s] = r < n ? zrcp(__ldg(A + (size_t)r * lda + r)) : make_double2(0.0, 0.0);
  }
  // L y = b: x_0 is b_0; the owner of row k + 1 publishes it after step k
  if (t == 0) bc[0] = b[0];
  __syncthreads();
  for (int k0 = 0; k0 < n - 1; k0 += PF) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int k = k0 + q;
      if (k < n - 1) {  // CTA-uniform
        wait_oldest();
        const double2 xk = bc[k & 1];
#pragma unroll
        for (int s = 0; s < kS; ++s) {
          const int r = t + kThreads * s;
          if (r > k && r < n) b[s] = zfms(b[s], slot(q, s), xk);
          if (r == k + 1) bc[(k + 1) & 1] = b[s];
        }
        fetch(k + PF < n - 1 ? k + PF : -1, q);
        __syncthreads();
      }
    }
  }
  // U x = y: column k in slot (n - 1 - k) % PF; the owner of row k - 1
  // divides by U_{k-1,k-1} (next slot) and publishes x_{k-1}
#pragma unroll
  for (int q = 0; q < PF; ++q) fetch(n - 1 - q, q);
  wait_oldest();
#pragma unroll
  for (int s = 0; s < kS; ++s)
    if (t + kThreads * s == n - 1) {
      b[s] = zmul(b[s], rinv[s]);
      bc[(n - 1) & 1] = b[s];
    }
  __syncthreads();
  for (int k0 = n - 1; k0 >= 1; k0 -= PF) {
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int k = k0 - q;
      if (k >= 1) {  // CTA-uniform
        // column k (slot q) is complete; column k - 1 (next slot) is the
        // group after it: wait for both
        asm volatile("cp.async.wait_group %0;\n" ::"n"(PF - 2 > 0 ? PF - 2 : 0) : "memory");
        const double2 xk = bc[k & 1];
#pragma unroll
        for (int s = 0; s < kS; ++s) {
          const int r = t + kThreads * s;
          if (r < k) b[s] = zfms(b[s], slot(q, s), xk);
          if (r == k - 1) {
            b[s] = zmul(b[s], rinv[s]);
            bc[(k - 1) & 1] = b[s];
          }
        }
        fetch(k - PF, q);
        __syncthreads();
      }
    }
  }
#pragma unroll
  for (int s = 0; s < kS; ++s) {
    const int r = t + kThreads * s;
    if (r < n) bg[r] = b[s];
  }
}

// ----------------------------------------- LU solve, blocked, many columns
// kBlkRhs right-hand sides per CTA held in shared memory (rows permuted on
// load); L then U in 32-row panels: the panel's triangular solve by the
// warps (lane = row, two columns per warp, shuffles), then the trailing rows
// by a register-tiled update (thread = 4 columns x Q rows, the LU column
// reads coalesced across the 64 row lanes).  Orders up to 64 Q.
constexpr int kBlkRhs = 16;
constexpr int kBlkPanel = 32;
#ifndef EBEM_GETRS_MMA
#define EBEM_GETRS_MMA 1
#endif
// Trailing update of a panel on the FP64 tensor cores:
//   X[r][0..16) -= A[r][k0 .. k0 + pw) X[k0 .. k0 + pw)[0..16),  ra <= r < rb,
// A the LU (column-major, lda), X the CTA's right-hand sides ([col][row],
// ld n).  Warps take 8-row tiles; per tile 8 k-steps of 4 x 2 column tiles
// x 4 real m8n8k4 products (complex as four real MMAs), the tile's A
// fragments loaded from global memory up front, X's from shared memory.
__device__ __forceinline__ void blk_update_mma(const double2* __restrict__ A, size_t lda,
                                               double2* X, int n, int k0, int pw, int ra,
                                               int rb, int w, int l) {
  const int fr = l >> 2, fk = l & 3;
  const int mtiles = (rb - ra + 7) >> 3;
  for (int mt = w; mt < mtiles; mt += kWarps) {
    const int r = ra + 8 * mt + fr;
    double2 a[kBlkPanel / 4];
#pragma unroll
    for (int ks = 0; ks < kBlkPanel / 4; ++ks) {
      const int kk = 4 * ks + fk;
      a[ks] = (r < rb && kk < pw) ? __ldg(A + (size_t)(k0 + kk) * lda + r)
                                  : make_double2(0.0, 0.0);
    }
    double acc[2][2][2];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int c = 0; c < 2; ++c) acc[nt][c][0] = acc[nt][c][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < kBlkPanel / 4; ++ks) {
      const int kk = 4 * ks + fk;
      if (4 * ks >= pw) break;  // warp-uniform
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const double2 b = kk < pw ? X[(size_t)(8 * nt + fr) * n + k0 + kk] : make_double2(0.0, 0.0);
        dmma(acc[nt][0][0], acc[nt][0][1], a[ks].x, b.x);
        dmma(acc[nt][0][0], acc[nt][0][1], -a[ks].y, b.y);
        dmma(acc[nt][1][0], acc[nt][1][1], a[ks].x, b.y);
        dmma(acc[nt][1][0], acc[nt][1][1], a[ks].y, b.x);
      }
    }
    const int row = ra + 8 * mt + fr;
    if (row < rb)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double2& xr = X[(size_t)(8 * nt + 2 * fk + h) * n + row];
          xr = make_double2(xr.x - acc[nt][0][h], xr.y - acc[nt][1][h]);
        }
  }
}
template <int Q>
__global__ void __launch_bounds__(kThreads)
k_getrs_blk(const LuSolveTask* __restrict__ tasks, const int* __restrict__ block_off,
            int n_tasks) {
  static_assert(kThreads == 256 && kBlkRhs == 16, "layout: 4 column groups x 64 row lanes");
  extern __shared__ double2 X[];  // [kBlkRhs][n] | perm (n ints)
  __shared__ double2 Dp[kBlkPanel][kBlkPanel + 1];  // panel diagonal block, [col][row]
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (block_off[mid] <= (int)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const LuSolveTask T = tasks[lo];
  const int n = T.n;
  const int c0 = (blockIdx.x - block_off[lo]) * kBlkRhs;
  if (n <= 0 || c0 >= T.nrhs) return;
  const int nc = min(kBlkRhs, T.nrhs - c0);
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
  const double2* A = reinterpret_cast<const double2*>(T.lu);
  const size_t lda = T.ld;
  double2* Bg = reinterpret_cast<double2*>(T.b) + (size_t)c0 * T.ldb;
  int* perm = reinterpret_cast<int*>(X + (size_t)kBlkRhs * n);
  // row r of the permuted system is row perm[r] of b (LAPACK interchanges)
  for (int r = t; r < n; r += kThreads) perm[r] = r;
  __syncthreads();
  if (t == 0)
    for (int k = 0; k < n; ++k) {
      const int p = __ldg(T.ipiv + k);
      if (p != k) {
        const int v = perm[k];
        perm[k] = perm[p];
        perm[p] = v;
      }
    }
  __syncthreads();
  for (int idx = t; idx < kBlkRhs * n; idx += kThreads) {
    const int c = idx / n, r = idx - c * n;
    X[idx] = c < nc ? Bg[(size_t)c * T.ldb + perm[r]] : make_double2(0.0, 0.0);
  }
  const int cg = t >> 6, rl = t & 63;  // update layout: columns 4 cg .. 4 cg + 3
  // ---- L y = b (unit lower)
  for (int k0 = 0; k0 < n; k0 += kBlkPanel) {
    const int k1 = min(k0 + kBlkPanel, n), pw = k1 - k0;
    for (int idx = t; idx < kBlkPanel * kBlkPanel; idx += kThreads) {
      const int kk = idx >> 5, rr = idx & 31;
      Dp[kk][rr] = (kk < pw && rr < pw) ? __ldg(A + (size_t)(k0 + kk) * lda + k0 + rr)
                                        : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      double2* xc = X + (size_t)(2 * w + cc) * n + k0;
      double2 x = l < pw ? xc[l] : make_double2(0.0, 0.0);
      for (int kk = 0; kk < pw - 1; ++kk) {
        const double2 xk = shfl2(x, kk);
        if (l > kk) x = zfms(x, Dp[kk][l], xk);
      }
      if (l < pw) xc[l] = x;
    }
    __syncthreads();
    if (EBEM_GETRS_MMA && k1 < n) {
      blk_update_mma(A, lda, X, n, k0, pw, k1, n, w, l);
    } else if (k1 < n) {
      double2 acc[Q][4];
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[q][j] = make_double2(0.0, 0.0);
      for (int kk = 0; kk < pw; ++kk) {
        double2 xv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) xv[j] = X[(size_t)(4 * cg + j) * n + k0 + kk];
        const double2* Ak = A + (size_t)(k0 + kk) * lda;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int r = k1 + rl + 64 * q;
          if (r < n) {
            const double2 a = __ldg(Ak + r);
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[q][j] = zfma(acc[q][j], a, xv[j]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int r = k1 + rl + 64 * q;
        if (r < n)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            double2& xr = X[(size_t)(4 * cg + j) * n + r];
            xr = make_double2(xr.x - acc[q][j].x, xr.y - acc[q][j].y);
          }
      }
    }
    __syncthreads();
  }
  // ---- U x = y, panels from the bottom
  for (int k1 = n; k1 > 0; k1 -= kBlkPanel) {
    const int k0 = max(0, k1 - kBlkPanel), pw = k1 - k0;
    for (int idx = t; idx < kBlkPanel * kBlkPanel; idx += kThreads) {
      const int kk = idx >> 5, rr = idx & 31;
      double2 v = (kk < pw && rr < pw) ? __ldg(A + (size_t)(k0 + kk) * lda + k0 + rr)
                                       : make_double2(0.0, 0.0);
      if (kk == rr && kk < pw) v = zrcp(v);  // the diagonal as its reciprocal
      Dp[kk][rr] = v;
    }
    __syncthreads();
#pragma unroll
    for (int cc = 0; cc < 2; ++cc) {
      double2* xc = X + (size_t)(2 * w + cc) * n + k0;
      double2 x = l < pw ? xc[l] : make_double2(0.0, 0.0);
      for (int kk = pw - 1; kk >= 0; --kk) {
        if (l == kk) x = zmul(x, Dp[kk][kk]);
        const double2 xk = shfl2(x, kk);
        if (l < kk) x = zfms(x, Dp[kk][l], xk);
      }
      if (l < pw) xc[l] = x;
    }
    __syncthreads();
    if (EBEM_GETRS_MMA && k0 > 0) {
      blk_update_mma(A, lda, X, n, k0, pw, 0, k0, w, l);
    } else if (k0 > 0) {
      double2 acc[Q][4];
#pragma unroll
      for (int q = 0; q < Q; ++q)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[q][j] = make_double2(0.0, 0.0);
      for (int kk = 0; kk < pw; ++kk) {
        double2 xv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) xv[j] = X[(size_t)(4 * cg + j) * n + k0 + kk];
        const double2* Ak = A + (size_t)(k0 + kk) * lda;
#pragma unroll
        for (int q = 0; q < Q; ++q) {
          const int r = rl + 64 * q;
          if (r < k0) {
            const double2 a = __ldg(Ak + r);
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[q][j] = zfma(acc[q][j], a, xv[j]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        const int r = rl + 64 * q;
        if (r < k0)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            double2& xr = X[(size_t)(4 * cg + j) * n + r];
            xr = make_double2(xr.x - acc[q][j].x, xr.y - acc[q][j].y);
          }
      }
    }
    __syncthreads();
  }
  for (int idx = t; idx < kBlkRhs * n; idx += kThreads) {
    const int c = idx / n, r = idx - c * n;
    if (c < nc) Bg[(size_t)c * T.ldb + r] = X[idx];
  }
}

// ------------------------------------------ LU solve, large n (> 256)
// One CTA per right-hand side, column-oriented substitutions: step k reads
// one (coalesced) column of L or U and updates the remaining rows in
// parallel, one barrier per step.  x lives in shared memory when it fits.
constexpr int kBigThreads = 1024;
__global__ void __launch_bounds__(kBigThreads)
k_getrs_big(const LuSolveTask* __restrict__ tasks, const int* __restrict__ block_off,
            int n_tasks, int smem_cap) {
  extern __shared__ double2 sx[];
  int lo = 0, hi = n_tasks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (block_off[mid] <= (int)blockIdx.x) lo = mid;
    else hi = mid - 1;
  }
  const LuSolveTask T = tasks[lo];
  const int col = blockIdx.x - block_off[lo];
  if (col >= T.nrhs) return;
  const int n = T.n;
  const double2* A = reinterpret_cast<const double2*>(T.lu);
  const size_t lda = T.ld;
  double2* bg = reinterpret_cast<double2*>(T.b) + (size_t)col * T.ldb;
  const bool in_smem = n <= smem_cap;
  double2* x = in_smem ? sx : bg;
  if (in_smem)
    for (int r = threadIdx.x; r < n; r += blockDim.x) x[r] = bg[r];
  __syncthreads();
  if (threadIdx.x == 0)
    for (int k = 0; k < n; ++k) {
      const int p = T.ipiv[k];
      if (p != k) {
        const double2 t = x[k];
        x[k] = x[p];
        x[p] = t;
      }
    }
  __syncthreads();
  for (int k = 0; k < n - 1; ++k) {  // unit lower
    const double2 xk = x[k];
    const double2* Lk = A + (size_t)k * lda;
    for (int r = k + 1 + threadIdx.x; r < n; r += blockDim.x) x[r] = zfms(x[r], Lk[r], xk);
    __syncthreads();
  }
  for (int k = n - 1; k >= 0; --k) {  // upper
    const double2* Uk = A + (size_t)k * lda;
    const double2 xk = zdiv(x[k], Uk[k]);
    __syncthreads();
    if (threadIdx.x == 0) x[k] = xk;
    for (int r = threadIdx.x; r < k; r += blockDim.x) x[r] = zfms(x[r], Uk[r], xk);
    __syncthreads();
  }
  if (in_smem)
    for (int r = threadIdx.x; r < n; r += blockDim.x) bg[r] = x[r];
}

// ----------------------------------------------------------- host wrappers
static void set_smem_attr(const void* f) {
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCap);
}

void dense_init() {
  static bool done = false;
  if (done) return;
  set_smem_attr((const void*)k_qr_reduce);
  set_smem_attr((const void*)k_cpqr);
  set_smem_attr((const void*)k_getrf);
  set_smem_attr((const void*)k_getrs);
  set_smem_attr((const void*)k_getrs_big);
  set_smem_attr((const void*)k_getrs_reg<2, 1>);
  set_smem_attr((const void*)k_getrs_reg<4, 1>);
  set_smem_attr((const void*)k_getrs_reg<8, 1>);
  set_smem_attr((const void*)k_getrs_reg<2, kCpw>);
  set_smem_attr((const void*)k_getrs_reg<4, kCpw>);
  set_smem_attr((const void*)k_getrs_reg<8, kCpw>);
  done = true;
}

void launch_qr_reduce(const QrTask* tasks, int n, size_t smem, double2* gws,
                      cudaStream_t st) {
  if (n <= 0) return;
  k_qr_reduce<<<n, kQrThreads, smem, st>>>(tasks, gws);
}
void launch_cpqr(const CpqrTask* tasks, int n, size_t smem, double2* gws,
                 cudaStream_t st) {
  if (n <= 0) return;
  k_cpqr<<<n, kQrThreads, smem, st>>>(tasks, gws);
}
void launch_interp(const InterpTask* tasks, int n, int max_k, cudaStream_t st) {
  if (n <= 0) return;
  const int kk = max_k > 0 ? max_k : 1;
  const size_t smem = (size_t(kk) * kk + kk + size_t(kWarps) * kk) * sizeof(double2) +
                      size_t(kk) * sizeof(int);
  static bool attr = [] {
    cudaFuncSetAttribute(k_interp, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCap);
    return true;
  }();
  (void)attr;
  if (smem > size_t(kSmemCap)) throw std::length_error("interpolation: rank too large");
  k_interp<<<n, kThreads, smem, st>>>(tasks);
}
__global__ void __launch_bounds__(256)
k_prefetch_l2(const PrefetchTask* __restrict__ tasks, int n) {
  const unsigned long long tid = blockIdx.x * 256ull + threadIdx.x;
  const unsigned long long nth = gridDim.x * 256ull;
  for (int i = 0; i < n; ++i) {
    const char* p = static_cast<const char*>(tasks[i].p);
    const unsigned long long lines = (tasks[i].bytes + 127) >> 7;
    for (unsigned long long q = tid; q < lines; q += nth)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(p + (q << 7)));
  }
}
void launch_prefetch_l2(const PrefetchTask* tasks, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_prefetch_l2<<<148 * 4, 256, 0, st>>>(tasks, n);
}
void launch_pivots_to_perm(const LuTask* tasks, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_pivots_to_perm<<<(n + kPermWarps - 1) / kPermWarps, 32 * kPermWarps, 0, st>>>(tasks, n);
}
void launch_getrf(const LuTask* tasks, int n, size_t smem, double2* gws,
                  cudaStream_t st) {
  if (n <= 0) return;
  k_getrf<<<n, kQrThreads, smem, st>>>(tasks, gws);
}
int getrs_cpw(int max_nrhs, int max_n) {
  if (max_nrhs >= kBlkMinRhs && max_n >= kBlkMinN && max_n <= kGetrsBlkMaxN) return -2;
  if (max_n > 256 && max_n <= kGetrsCtaMaxN) return -1;  // one CTA per column
  if (max_nrhs <= kNarrowRhs && max_n <= kGetrsWarpMaxN) return 0;  // one warp per column
  if (max_nrhs <= kNarrowRhs && max_n <= 256) return -1;
  return max_nrhs <= kWarps ? 1 : kCpw;
}
int getrs_blocks(int nrhs, int max_n, int cpw) {
  if (cpw == 0) return nrhs;  // warps
  if (cpw == -2) return (nrhs + kBlkRhs - 1) / kBlkRhs;
  if (cpw < 0) return nrhs;   // CTAs
  const int per = max_n <= 256 ? kWarps * cpw : 1;  // large n: one CTA per column
  return (nrhs + per - 1) / per;
}
void launch_getrs(const LuSolveTask* tasks, const int* block_off, int n_tasks,
                  int n_blocks, cudaStream_t st, int smem_bytes, int max_n, int cpw) {
  if (n_blocks <= 0) return;
  if (cpw == 0) {  // n_blocks counts warps
    const int grid = (n_blocks + kWarps - 1) / kWarps;
    if (max_n <= 64) k_getrs_warp<2><<<grid, kThreads, 0, st>>>(tasks, block_off, n_tasks, n_blocks);
    else k_getrs_warp<4><<<grid, kThreads, 0, st>>>(tasks, block_off, n_tasks, n_blocks);
    return;
  }
  if (cpw == -2) {  // blocked, kBlkRhs columns per CTA
    const size_t sm = size_t(max_n) * (kBlkRhs * 16 + 4) + 16;
    static const bool attr = [] {
      cudaFuncSetAttribute(k_getrs_blk<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      cudaFuncSetAttribute(k_getrs_blk<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      return true;
    }();
    (void)attr;
    if (max_n <= 256) k_getrs_blk<4><<<n_blocks, kThreads, sm, st>>>(tasks, block_off, n_tasks);
    else k_getrs_blk<8><<<n_blocks, kThreads, sm, st>>>(tasks, block_off, n_tasks);
    return;
  }
  if (cpw < 0) {  // one CTA per column, orders up to kThreads * 8
    const int pf = max_n <= kThreads ? 16 : max_n <= 2 * kThreads ? 8 : max_n <= 4 * kThreads ? 4 : 2;
    const int ks = max_n <= kThreads ? 1 : max_n <= 2 * kThreads ? 2 : max_n <= 4 * kThreads ? 4 : 8;
    const size_t sm = 16 * size_t(pf) * ks * kThreads + 20 * size_t(std::max(max_n, 2)) + 16;
    static const bool attr = [] {
      const int cap = 160 * 1024;
      cudaFuncSetAttribute(k_getrs_cta<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
      cudaFuncSetAttribute(k_getrs_cta<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
      cudaFuncSetAttribute(k_getrs_cta<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
      cudaFuncSetAttribute(k_getrs_cta<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, cap);
      return true;
    }();
    (void)attr;
    if (max_n <= kThreads) k_getrs_cta<1><<<n_blocks, kThreads, sm, st>>>(tasks, block_off, n_tasks);
    else if (max_n <= 2 * kThreads) k_getrs_cta<2><<<n_blocks, kThreads, sm, st>>>(tasks, block_off, n_tasks);
    else if (max_n <= 4 * kThreads) k_getrs_cta<4><<<n_blocks, kThreads, sm, st>>>(tasks, block_off, n_tasks);
    else k_getrs_cta<8><<<n_blocks, kThreads, sm, st>>>(tasks, block_off, n_tasks);
    return;
  }
  // LU staged when it fits (smem_bytes covers the largest staged one);
  // 1 / U_kk always needs n slots
  const int bytes = std::max(smem_bytes, 16 * std::max(max_n, 1));
  const int cap = smem_bytes / 16;
#define EBEM_GETRS(S, C) \
  k_getrs_reg<S, C><<<n_blocks, kThreads, size_t(bytes), st>>>(tasks, block_off, n_tasks, cap)
  if (max_n <= 64) {
    if (cpw == 1) EBEM_GETRS(2, 1); else EBEM_GETRS(2, kCpw);
  } else if (max_n <= 128) {
    if (cpw == 1) EBEM_GETRS(4, 1); else EBEM_GETRS(4, kCpw);
  } else if (max_n <= 256) {
    if (cpw == 1) EBEM_GETRS(8, 1); else EBEM_GETRS(8, kCpw);
  } else {
    const int xcap = kSmemCap / 16;
    k_getrs_big<<<n_blocks, kBigThreads, size_t(std::min(max_n, xcap)) * 16, st>>>(
        tasks, block_off, n_tasks, xcap);
  }
#undef EBEM_GETRS
}

int getrs_smem_bytes(int n) {
  // staged LU + 1 / U_kk (register kernel, n <= 256); larger n stage only x
  if (n > 256) return 0;
  const long long b = ((long long)n * n + n) * 16;
  return b <= kSmemCap ? int(b) : 0;
}
int gemm_narrow(const GemmTask& g) {
  if (g.trans_a || g.trans_b || g.n > kNarrow) return 0;
  return g.n <= 1 ? 1 : kNarrow;
}
// EBEM_GEMM_MMA=0 selects the SIMT k_gemm (A/B measurements).
bool gemm_use_mma() {
  static const bool on = [] {
    const char* e = std::getenv("EBEM_GEMM_MMA");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}
int gemm_blocks(const GemmTask& g, int narrow) {
  if (narrow) return (g.m + 31) / 32;
  return ((g.m + kTile - 1) / kTile) * ((g.n + kTile - 1) / kTile);
}
void launch_gemm(const GemmTask* tasks, const int* block_off, int n_tasks,
                 int n_blocks, cudaStream_t st, int narrow) {
  if (n_blocks <= 0) return;
  static const bool warp_gemv = [] {  // EBEM_GEMV_WARP=0: the K-split k_gemv (A/B)
    const char* e = std::getenv("EBEM_GEMV_WARP");
    return e == nullptr || std::atoi(e) != 0;
  }();
  // few tiles (the upper levels): the K-split kernel keeps more loads in
  // flight per tile than one warp running down K
  static const int warp_min = [] {
    const char* e = std::getenv("EBEM_GEMV_WARP_MIN");
    return e ? std::atoi(e) : 4096;
  }();
  const int wgrid = (n_blocks + kWarps - 1) / kWarps;
  if (narrow && warp_gemv && n_blocks >= warp_min) {
    if (narrow == 1)
      k_gemv_w<1><<<wgrid, kThreads, 0, st>>>(tasks, block_off, n_tasks, n_blocks);
    else
      k_gemv_w<kNarrow><<<wgrid, kThreads, 0, st>>>(tasks, block_off, n_tasks, n_blocks);
  } else if (narrow == 1) k_gemv<1><<<n_blocks, kThreads, 0, st>>>(tasks, block_off, n_tasks);
  else if (narrow) k_gemv<kNarrow><<<n_blocks, kThreads, 0, st>>>(tasks, block_off, n_tasks);
  else if (gemm_use_mma()) k_gemm_mma<<<n_blocks, kMmaThreads, 0, st>>>(tasks, block_off, n_tasks);
  else k_gemm<<<n_blocks, kThreads, 0, st>>>(tasks, block_off, n_tasks);
}
int copy_blocks(int rows, int cols) {  // warp units
  const long long t = (long long)rows * cols;
  return int((t + kCopyUnit - 1) / kCopyUnit);
}
void launch_copy(const CopyTask* tasks, const int* block_off, int n_tasks,
                 int n_blocks, cudaStream_t st) {
  if (n_blocks <= 0) return;
  k_copy<<<(n_blocks + kWarps - 1) / kWarps, kThreads, 0, st>>>(tasks, block_off, n_tasks,
                                                                 n_blocks);
}

}  // namespace ebem_gpu
