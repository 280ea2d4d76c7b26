// Blocked right-looking LU with partial pivoting for the diagonal blocks
// (and the top block) too large for one CTA's shared memory: zgetrf as
// called by LuFactor (proj/src/lapack.cpp:31-53), pivot = first row of the
// largest |Re| + |Im| in the column, row interchanges applied to the whole
// matrix (LAPACK's ipiv convention), info = 1 + the first exactly-zero pivot.
//
// Per panel of kNb columns: k_lu_panel factors the panel in place (one CTA
// per matrix), k_lu_rest applies the panel's interchanges to the other
// columns and solves L11 U12 = A12 for the panel rows (one warp per column),
// k_lu_update does A22 -= L21 U12 in 64 x 64 register-blocked tiles.  The
// trailing update carries the O(n^3) work on every SM instead of one.
#include <cuda_runtime.h>

#include <algorithm>

#include "ebem_dense.h"

namespace ebem_gpu {

namespace {

constexpr int kNb = 32;
#ifndef EBEM_LU_MMA
#define EBEM_LU_MMA 1  // trailing update on the FP64 tensor cores (0: SIMT register tiles)
#endif
__device__ __forceinline__ void mma_f64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
constexpr int kPanelThreads = 512;
constexpr int kTile = 64;

__device__ __forceinline__ double cabs1(double2 a) { return fabs(a.x) + fabs(a.y); }
__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a - b c
__device__ __forceinline__ double2 zfms(double2 a, double2 b, double2 c) {
  return make_double2(fma(-b.y, -c.y, fma(-b.x, c.x, a.x)),
                      fma(-b.y, c.x, fma(-b.x, c.y, a.y)));
}
__device__ __forceinline__ double2 zrcp(double2 a) {
  if (fabs(a.x) >= fabs(a.y)) {
    const double r = a.y * (1.0 / a.x), d = 1.0 / fma(a.y, r, a.x);
    return make_double2(d, -r * d);
  }
  const double r = a.x * (1.0 / a.y), d = 1.0 / fma(a.x, r, a.y);
  return make_double2(r * d, -d);
}

__global__ void __launch_bounds__(kPanelThreads)
k_lu_panel(const LuTask* __restrict__ tasks, int j0) {
  const LuTask T = tasks[blockIdx.x];
  const int n = T.n;
  if (j0 >= n || T.in_smem) return;
  double2* A = reinterpret_cast<double2*>(T.a);
  const size_t ld = T.ld;
  const int nbc = min(kNb, n - j0);
  __shared__ double s_best[kPanelThreads / 32];
  __shared__ int s_idx[kPanelThreads / 32];
  __shared__ int s_p;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (j0 == 0 && threadIdx.x == 0) *T.info = 0;  // the pivot writer below
  for (int jj = 0; jj < nbc; ++jj) {
    const int col = j0 + jj;
    double2* ac = A + (size_t)col * ld;
    // pivot: first index of the largest cabs1 at or below the diagonal
    double best = -1.0;
    int bi = n;
    for (int r = col + threadIdx.x; r < n; r += blockDim.x) {
      const double v = cabs1(ac[r]);
      if (v > best) { best = v; bi = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    if (l == 0) { s_best[w] = best; s_idx[w] = bi; }
    __syncthreads();
    if (w == 0) {
      best = l < (int)(blockDim.x >> 5) ? s_best[l] : -1.0;
      bi = l < (int)(blockDim.x >> 5) ? s_idx[l] : n;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (l == 0) {
        if (best <= 0.0) {  // exactly zero column: no interchange, no scaling
          bi = col;
          if (*T.info == 0) *T.info = col + 1;
        }
        s_p = bi;
        T.ipiv[col] = bi;
      }
    }
    __syncthreads();
    const int p = s_p;
    if (p != col && threadIdx.x < nbc) {  // interchange within the panel
      double2* c = A + (size_t)(j0 + threadIdx.x) * ld;
      const double2 t = c[col];
      c[col] = c[p];
      c[p] = t;
    }
    __syncthreads();
    const double2 piv = ac[col];
    if (piv.x != 0.0 || piv.y != 0.0) {
      const double2 rp = zrcp(piv);
      for (int r = col + 1 + threadIdx.x; r < n; r += blockDim.x) ac[r] = zmul(ac[r], rp);
    }
    __syncthreads();
    // rank-1 update of the panel's remaining columns
    const int rows = n - col - 1, cols = nbc - jj - 1;
    for (int idx = threadIdx.x; idx < rows * cols; idx += blockDim.x) {
      const int c = idx / rows, r = col + 1 + (idx - c * rows);
      double2* cc = A + (size_t)(col + 1 + c) * ld;
      cc[r] = zfms(cc[r], ac[r], cc[col]);
    }
    __syncthreads();
  }
}

// Interchanges of the panel on every other column; U12 = L11^-1 A12 for the
// columns right of the panel.  One warp per column, lane l = panel row l.
__global__ void __launch_bounds__(256)
k_lu_rest(const LuTask* __restrict__ tasks, int j0) {
  const LuTask T = tasks[blockIdx.x];
  const int n = T.n;
  if (j0 >= n || T.in_smem) return;
  const int nbc = min(kNb, n - j0);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int c = blockIdx.y * 8 + w;  // column index among the non-panel columns
  const int col = c < j0 ? c : c + nbc;
  if (col >= n) return;
  double2* A = reinterpret_cast<double2*>(T.a);
  const size_t ld = T.ld;
  double2* a = A + (size_t)col * ld;
  if (l == 0) {
    for (int k = j0; k < j0 + nbc; ++k) {
      const int p = T.ipiv[k];
      if (p != k) {
        const double2 t = a[k];
        a[k] = a[p];
        a[p] = t;
      }
    }
  }
  __syncwarp();
  if (col < j0) return;
  double2 v = l < nbc ? a[j0 + l] : make_double2(0.0, 0.0);
  for (int k = 0; k < nbc - 1; ++k) {
    const double2 xk = make_double2(__shfl_sync(0xffffffffu, v.x, k),
                                    __shfl_sync(0xffffffffu, v.y, k));
    if (l > k && l < nbc) v = zfms(v, A[(size_t)(j0 + k) * ld + j0 + l], xk);
  }
  if (l < nbc) a[j0 + l] = v;
}

// A22 -= L21 U12 on 64 x 64 tiles (4 x 4 entries per thread).
__global__ void __launch_bounds__(256)
k_lu_update(const LuTask* __restrict__ tasks, int j0) {
  const LuTask T = tasks[blockIdx.x];
  const int n = T.n;
  if (T.in_smem) return;
  const int s = j0 + kNb;  // first trailing row / column
  if (s >= n) return;
  const int m = n - s;
  const int tiles = (m + kTile - 1) / kTile;
  const int tr = blockIdx.y % tiles, tc = blockIdx.y / tiles;
  if (tc >= tiles) return;
  constexpr int kK = 16;  // k chunk staged per pass (2 x 16.6 KB of shared memory)
  __shared__ double2 Ls[kK][kTile + 1];  // L21 tile, [k][row]
  __shared__ double2 Us[kK][kTile + 1];  // U12 tile, [k][col]
  double2* A = reinterpret_cast<double2*>(T.a);
  const size_t ld = T.ld;
  const int r0 = s + tr * kTile, c0 = s + tc * kTile;
  const int ty = threadIdx.x >> 4, tx = threadIdx.x & 15;  // rows ty + 16 a, cols tx + 16 b
#if EBEM_LU_MMA
  double macc[8][2][2];  // [column tile][re, im][2]
#pragma unroll
  for (int t = 0; t < 8; ++t)
#pragma unroll
    for (int c = 0; c < 2; ++c) macc[t][c][0] = macc[t][c][1] = 0.0;
  (void)ty;
  (void)tx;
#endif
  double2 acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = make_double2(0.0, 0.0);
  for (int k0 = 0; k0 < kNb; k0 += kK) {
    for (int idx = threadIdx.x; idx < kK * kTile; idx += blockDim.x) {
      const int k = idx / kTile, i = idx - k * kTile;
      Ls[k][i] = (r0 + i < n) ? A[(size_t)(j0 + k0 + k) * ld + r0 + i] : make_double2(0.0, 0.0);
    }
    for (int idx = threadIdx.x; idx < kK * kTile; idx += blockDim.x) {
      const int i = idx / kK, k = idx - i * kK;  // consecutive threads: down a column
      Us[k][i] = (c0 + i < n) ? A[(size_t)(c0 + i) * ld + j0 + k0 + k] : make_double2(0.0, 0.0);
    }
    __syncthreads();
#if EBEM_LU_MMA
    {
      // FP64 tensor cores: warp w owns output rows 8w .. 8w + 7 of the tile,
      // all 8 column tiles; per k-step one A fragment, eight B fragments,
      // 8 x 4 real m8n8k4 products (complex as four real MMAs)
      const int w = threadIdx.x >> 5, l = threadIdx.x & 31, fr = l >> 2, fk = l & 3;
#pragma unroll
      for (int k = 0; k < kK; k += 4) {
        const double2 a = Ls[k + fk][8 * w + fr];
        const double an = -a.y;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          const double2 b = Us[k + fk][8 * t + fr];
          mma_f64(macc[t][0][0], macc[t][0][1], a.x, b.x);
          mma_f64(macc[t][0][0], macc[t][0][1], an, b.y);
          mma_f64(macc[t][1][0], macc[t][1][1], a.x, b.y);
          mma_f64(macc[t][1][0], macc[t][1][1], a.y, b.x);
        }
      }
    }
#else
#pragma unroll 4
    for (int k = 0; k < kK; ++k) {
      double2 lv[4], uv[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) lv[a] = Ls[k][ty + 16 * a];
#pragma unroll
      for (int b = 0; b < 4; ++b) uv[b] = Us[k][tx + 16 * b];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          acc[a][b].x = fma(lv[a].x, uv[b].x, fma(-lv[a].y, uv[b].y, acc[a][b].x));
          acc[a][b].y = fma(lv[a].x, uv[b].y, fma(lv[a].y, uv[b].x, acc[a][b].y));
        }
    }
#endif
    __syncthreads();
  }
#if EBEM_LU_MMA
  {
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31, fr = l >> 2, fk = l & 3;
    const int r = r0 + 8 * w + fr;
    if (r < n)
#pragma unroll
      for (int t = 0; t < 8; ++t)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int c = c0 + 8 * t + 2 * fk + h;
          if (c >= n) continue;
          double2* e = A + (size_t)c * ld + r;
          *e = make_double2(e->x - macc[t][0][h], e->y - macc[t][1][h]);
        }
  }
#else
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const int c = c0 + tx + 16 * b;
    if (c >= n) continue;
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int r = r0 + ty + 16 * a;
      if (r >= n) continue;
      double2* e = A + (size_t)c * ld + r;
      *e = make_double2(e->x - acc[a][b].x, e->y - acc[a][b].y);
    }
  }
#endif
}

}  // namespace

int lu_blocked_panel() { return kNb; }

void launch_lu_blocked(const LuTask* tasks, int n_tasks, int max_n, cudaStream_t st) {
  if (n_tasks <= 0 || max_n <= 0) return;
  for (int j0 = 0; j0 < max_n; j0 += kNb) {
    k_lu_panel<<<n_tasks, kPanelThreads, 0, st>>>(tasks, j0);
    const int others = max_n - std::min(kNb, max_n - j0);
    if (others > 0) {
      dim3 g(n_tasks, (others + 7) / 8);
      k_lu_rest<<<g, 256, 0, st>>>(tasks, j0);
    }
    const int m = max_n - j0 - kNb;
    if (m > 0) {
      const int tiles = (m + kTile - 1) / kTile;
      dim3 g(n_tasks, tiles * tiles);
      k_lu_update<<<g, 256, 0, st>>>(tasks, j0);
    }
  }
}

}  // namespace ebem_gpu

// ----------------------------------------------- dense-solver helpers
// (ConvSolver, proj/src/dense_solver.cpp:9-29; LuFactor, proj/src/lapack.cpp)
namespace ebem_gpu {
namespace {

// sum_i |a_ij| of every column (one warp per column)
__global__ void __launch_bounds__(256)
k_col_abs_sum(const double2* __restrict__ a, int n, int ld, double* __restrict__ out) {
  const int col = blockIdx.x * 8 + (threadIdx.x >> 5), l = threadIdx.x & 31;
  if (col >= n) return;
  const double2* c = a + (size_t)col * ld;
  double s = 0.0;
  for (int r = l; r < n; r += 32) s += hypot(c[r].x, c[r].y);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (l == 0) out[col] = s;
}

__device__ double2 zdiv_robust(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  }
  const double r = b.x / b.y, d = b.y + b.x * r;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}

__device__ double2 block_sum2(double2 v, double2* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
    v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double2 s = make_double2(0.0, 0.0);
  for (int k = 0; k < int(blockDim.x >> 5); ++k) s = make_double2(s.x + red[k].x, s.y + red[k].y);
  return s;
}

// x := A^-H x for A = P L U (LAPACK ipiv): U^H y = x, L^H z = y, x = P z.
__global__ void __launch_bounds__(1024)
k_getrs_conj(const double2* __restrict__ lu, int n, int ld, const int* __restrict__ ipiv,
             double2* __restrict__ x) {
  __shared__ double2 red[32];
  for (int i = 0; i < n; ++i) {  // U^H is lower triangular
    const double2* ui = lu + (size_t)i * ld;
    double2 p = make_double2(0.0, 0.0);
    for (int k = threadIdx.x; k < i; k += blockDim.x) {
      const double2 u = ui[k], y = x[k];  // conj(u) y
      p.x += u.x * y.x + u.y * y.y;
      p.y += u.x * y.y - u.y * y.x;
    }
    const double2 s = block_sum2(p, red);
    if (threadIdx.x == 0) {
      const double2 d = make_double2(ui[i].x, -ui[i].y);
      x[i] = zdiv_robust(make_double2(x[i].x - s.x, x[i].y - s.y), d);
    }
    __syncthreads();
  }
  for (int i = n - 1; i >= 0; --i) {  // L^H is unit upper triangular
    const double2* li = lu + (size_t)i * ld;
    double2 p = make_double2(0.0, 0.0);
    for (int k = i + 1 + threadIdx.x; k < n; k += blockDim.x) {
      const double2 l = li[k], z = x[k];
      p.x += l.x * z.x + l.y * z.y;
      p.y += l.x * z.y - l.y * z.x;
    }
    const double2 s = block_sum2(p, red);
    if (threadIdx.x == 0) x[i] = make_double2(x[i].x - s.x, x[i].y - s.y);
    __syncthreads();
  }
  if (threadIdx.x == 0)
    for (int k = n - 1; k >= 0; --k) {
      const int p = ipiv[k];
      if (p != k) {
        const double2 t = x[k];
        x[k] = x[p];
        x[p] = t;
      }
    }
}

}  // namespace

void launch_col_abs_sum(const double* a, int n, int ld, double* out, cudaStream_t st) {
  if (n <= 0) return;
  k_col_abs_sum<<<(n + 7) / 8, 256, 0, st>>>(reinterpret_cast<const double2*>(a), n, ld, out);
}

void launch_getrs_conj(const double* lu, int n, int ld, const int* ipiv, double* x,
                       cudaStream_t st) {
  if (n <= 0) return;
  k_getrs_conj<<<1, 1024, 0, st>>>(reinterpret_cast<const double2*>(lu), n, ld, ipiv,
                                   reinterpret_cast<double2*>(x));
}

}  // namespace ebem_gpu
