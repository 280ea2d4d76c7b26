// Streaming TSQR with compact-WY panels whose block reflectors are applied
// on the FP64 tensor cores.
//
// Same job as k_tsqr (the R factor of a tall rows x n complex block, rows
// streamed through 32-row blocks B folded into R by the structured
// reflectors of [R; B], zlarfg/zlarf conventions), but the n columns are cut
// into panels of 8, one warp per panel, and a panel's 8 reflectors reach the
// other warps as ONE block reflector Q_p^H = I - V T^H V^H (zlarft forward,
// columnwise; V = [I_8 at R rows 8p..8p+7 ; Y], Y the 32 x 8 block part):
//   W = R[8p.., c] + Y^H B[:, c]      (8 x 8 per consumer warp, m8n8k4 DMMA)
//   W' = T^H W;  R[8p.., c] -= W'
//   B[:, c] -= Y W'                    (DMMA, accumulating into B in place)
// instead of 8 reflector-at-a-time SIMT updates, each behind its own
// cross-warp hand-off.  Only the 8 reflectors inside a panel form a chain,
// and that chain stays inside the owning warp.
//
// Register layout.  Lane l of a warp owns column 8w + (l >> 2) and block rows
// 8t + 2g + h (g = l & 3, t = 0..kTg-1, h = 0..1).  With the k-steps of the
// products taken over the rows {8t + 2g + h : g} (any order of a sum is
// allowed), these registers are at once the B operand of W = Y^H B and the
// accumulator of B^T -= W'^T Y^T: the block never leaves registers.
#include <cuda_runtime.h>

#include <algorithm>

#include "ebem_dense.h"

namespace ebem_gpu {

namespace {

constexpr int kWyThreads = 512;  // 16 warps: panels of 8 columns, n <= 128
constexpr int kWyWarps = kWyThreads / 32;
constexpr int kPw = 8;   // panel width (columns per warp)
#ifndef EBEM_WY_ROWS
#define EBEM_WY_ROWS 64
#endif
constexpr int kBr = EBEM_WY_ROWS;  // block rows (64: half the reflector chains per row of 32)
constexpr int kTg = kBr / 8;       // row groups of 8 (t index)
#ifndef EBEM_WY_RING
#define EBEM_WY_RING 4
#endif
constexpr int kRing = EBEM_WY_RING;  // panel slots (panel tag b P + p lives in slot tag % kRing)

__device__ __forceinline__ int wpidx(int i, int j) { return ((j * (j + 1)) >> 1) + i; }

__device__ __forceinline__ void dmma_wy(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double gsum4(double v) {  // the 4 lanes of a column
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

struct WySlot {
  double2 y[kBr][kPw];  // block part of the panel's reflectors
  double2 t[kPw][kPw];  // T (upper triangle), T[i][i] = tau_i
};

__device__ __forceinline__ void wy_fence() { __threadfence_block(); }

__global__ void __launch_bounds__(kWyThreads, 1)
k_tsqr_wy(const QrTask* __restrict__ tasks) {
  extern __shared__ double2 sm[];
  __shared__ int seq[kRing];      // the panel tag a slot holds
  __shared__ int prog[kWyWarps];  // 1 + tag of the last panel a warp applied
  const QrTask T = tasks[blockIdx.x];
  const int n = T.n, rows = T.rows, ld = T.ld;
  const int P = (n + kPw - 1) / kPw;
  const int rsz = (n * (n + 1)) >> 1;
  double2* R = sm;
  WySlot* ring = reinterpret_cast<WySlot*>(sm + rsz);
  double2* wscr = reinterpret_cast<double2*>(ring + kRing);  // [warp][8][8]
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  const int g = l & 3, jj = l >> 2;
  const int col = w * kPw + jj;
  const bool own = w < P && col < n;
  for (int q = threadIdx.x; q < rsz; q += blockDim.x) R[q] = make_double2(0.0, 0.0);
  if (threadIdx.x < kWyWarps) prog[threadIdx.x] = 0;
  if (threadIdx.x < kRing) seq[threadIdx.x] = -1;
  __syncthreads();
  volatile int* vseq = seq;
  volatile int* vprog = prog;
  if (w < P) {
    double2* ws = wscr + w * (kPw * kPw);
    const double2* src = reinterpret_cast<const double2*>(T.src) + (size_t)(own ? col : 0) * ld;
    for (int r0 = 0, b = 0; r0 < rows; r0 += kBr, ++b) {
      double2 B[kTg][2];
#pragma unroll
      for (int t = 0; t < kTg; ++t)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = r0 + 8 * t + 2 * g + h;
          B[t][h] = (own && r < rows) ? src[r] : make_double2(0.0, 0.0);
        }
      if (own && r0 + kBr < rows) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + r0 + kBr + 8 * g));
      // ---- the block reflectors of panels 0 .. w - 1 of this block
      for (int p = 0; p < w; ++p) {
        const int tag = b * P + p;
        while (vseq[tag % kRing] != tag) __nanosleep(20);
        wy_fence();
        const WySlot& S = ring[tag % kRing];
        const int i = l >> 2;  // W row (reflector) of this lane's accumulator
        // W = R[8p + i][c] + Y^H B  (C fragment: W[i][2g + h'])
        double wr[2], wi[2];
#pragma unroll
        for (int hp = 0; hp < 2; ++hp) {
          const int c = w * kPw + 2 * g + hp;
          const double2 v = c < n ? R[wpidx(kPw * p + i, c)] : make_double2(0.0, 0.0);
          wr[hp] = v.x;
          wi[hp] = v.y;
        }
#pragma unroll
        for (int t = 0; t < kTg; ++t)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const double2 y = S.y[8 * t + 2 * g + h][i];  // A = conj(Y)^T fragment
            dmma_wy(wr[0], wr[1], y.x, B[t][h].x);
            dmma_wy(wr[0], wr[1], y.y, B[t][h].y);
            dmma_wy(wi[0], wi[1], y.x, B[t][h].y);
            dmma_wy(wi[0], wi[1], -y.y, B[t][h].x);
          }
#pragma unroll
        for (int hp = 0; hp < 2; ++hp) ws[i * kPw + 2 * g + hp] = make_double2(wr[hp], wi[hp]);
        __syncwarp();
        // W' = T^H W, R -= W'
        double2 wp[2];
#pragma unroll
        for (int hp = 0; hp < 2; ++hp) {
          const int cc = 2 * g + hp;
          double ar = 0.0, ai = 0.0;
          for (int m = 0; m <= i; ++m) {  // conj(T[m][i]) W[m][cc]
            const double2 tv = S.t[m][i], wv = ws[m * kPw + cc];
            ar = fma(tv.x, wv.x, fma(tv.y, wv.y, ar));
            ai = fma(tv.x, wv.y, fma(-tv.y, wv.x, ai));
          }
          wp[hp] = make_double2(ar, ai);
          const int c = w * kPw + cc, rr = kPw * p + i;
          if (c < n && rr < n) {
            double2& rv = R[wpidx(rr, c)];
            rv = make_double2(rv.x - ar, rv.y - ai);
          }
        }
        __syncwarp();
#pragma unroll
        for (int hp = 0; hp < 2; ++hp) ws[i * kPw + 2 * g + hp] = wp[hp];
        __syncwarp();
        // B^T -= W'^T Y^T: accumulator = this lane's B (column jj, rows 8t + 2g + h)
#pragma unroll
        for (int t = 0; t < kTg; ++t)
#pragma unroll
          for (int kq = 0; kq < 2; ++kq) {
            const double2 a = ws[(4 * kq + g) * kPw + jj];  // W'[i][jj], negated below
            const double2 y = S.y[8 * t + jj][4 * kq + g];  // Y^T[i][row 8t + jj]
            dmma_wy(B[t][0].x, B[t][1].x, -a.x, y.x);
            dmma_wy(B[t][0].x, B[t][1].x, a.y, y.y);
            dmma_wy(B[t][0].y, B[t][1].y, -a.x, y.y);
            dmma_wy(B[t][0].y, B[t][1].y, -a.y, y.x);
          }
        __syncwarp();
        if (l == 0) {
          wy_fence();
          vprog[w] = tag + 1;
        }
      }
      // ---- this warp's panel: 8 reflectors, then T; publish in slot w
      {
        const int tag = b * P + w;
        if (tag >= kRing) {  // slot reuse: the consumers of tag - kRing applied it
          const int old = tag - kRing, po = old % P;
          for (;;) {
            const int v = (l > po && l < P) ? vprog[l] : 0x7fffffff;
            if (__reduce_min_sync(0xffffffffu, v) >= old + 1) break;
            __nanosleep(20);
          }
          wy_fence();
        }
        WySlot& S = ring[tag % kRing];
        for (int i = 0; i < kPw; ++i) {
          const int ci = w * kPw + i;
          const bool mine = jj == i;
          double p4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int t = 0; t < kTg; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              p4[(2 * t + h) & 3] = fma(B[t][h].x, B[t][h].x, fma(B[t][h].y, B[t][h].y, p4[(2 * t + h) & 3]));
          const double xnorm2 = gsum4((p4[0] + p4[1]) + (p4[2] + p4[3]));
          double2 tau = make_double2(0.0, 0.0);
          if (mine && ci < n) {
            const double2 alpha = R[wpidx(ci, ci)];
            if (!(xnorm2 == 0.0 && alpha.y == 0.0)) {
              // zlarfg without true divisions (as k_tsqr's make_reflector)
              const double x2 = fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, xnorm2));
              const double s = rsqrt(x2);
              const double nrm = x2 * s;
              const bool pos = alpha.x >= 0.0;
              const double beta = pos ? -nrm : nrm;
              const double ib = pos ? -s : s;
              tau = make_double2((beta - alpha.x) * ib, -alpha.y * ib);
              const double arn = fma(alpha.x, s, pos ? 1.0 : -1.0);
              const double ain = alpha.y * s;
              const double id = s / fma(arn, arn, ain * ain);
              const double2 scal = make_double2(arn * id, -ain * id);
#pragma unroll
              for (int t = 0; t < kTg; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                  B[t][h] = make_double2(scal.x * B[t][h].x - scal.y * B[t][h].y,
                                         scal.x * B[t][h].y + scal.y * B[t][h].x);
              if (g == 0) R[wpidx(ci, ci)] = make_double2(beta, 0.0);
            }
          }
          if (mine) {  // the reflector's block part (zeros for a missing column)
#pragma unroll
            for (int t = 0; t < kTg; ++t)
#pragma unroll
              for (int h = 0; h < 2; ++h)
                S.y[8 * t + 2 * g + h][i] = ci < n ? B[t][h] : make_double2(0.0, 0.0);
            if (g == 0) S.t[i][i] = tau;
          }
          __syncwarp();
          {  // apply reflector i to the panel's later columns (shuffles warp-uniform)
            const bool act = jj > i && own;
            const double2 tv = S.t[i][i];
            double ar[4] = {0.0, 0.0, 0.0, 0.0}, ai[4] = {0.0, 0.0, 0.0, 0.0};
            if (act) {
#pragma unroll
              for (int t = 0; t < kTg; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const int q = (2 * t + h) & 3;
                  const double2 y = S.y[8 * t + 2 * g + h][i];
                  ar[q] = fma(y.x, B[t][h].x, fma(y.y, B[t][h].y, ar[q]));
                  ai[q] = fma(y.x, B[t][h].y, fma(-y.y, B[t][h].x, ai[q]));
                }
            }
            double sr = gsum4((ar[0] + ar[1]) + (ar[2] + ar[3]));
            double si = gsum4((ai[0] + ai[1]) + (ai[2] + ai[3]));
            if (act) {
              const double2 rij = R[wpidx(ci, col)];
              sr += rij.x;
              si += rij.y;
              const double fr = tv.x * sr + tv.y * si;  // f = conj(tau) s
              const double fi = tv.x * si - tv.y * sr;
#pragma unroll
              for (int t = 0; t < kTg; ++t)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                  const double2 y = S.y[8 * t + 2 * g + h][i];
                  B[t][h].x = fma(-y.x, fr, fma(y.y, fi, B[t][h].x));
                  B[t][h].y = fma(-y.x, fi, fma(-y.y, fr, B[t][h].y));
                }
              if (g == 0) R[wpidx(ci, col)] = make_double2(rij.x - fr, rij.y - fi);
            }
          }
          __syncwarp();
        }
        // G[m][i] = y_m^H y_i (m < i): column i's lanes, from their own y_i
        for (int m = 0; m < kPw - 1; ++m) {
          double pr[4] = {0.0, 0.0, 0.0, 0.0}, pi[4] = {0.0, 0.0, 0.0, 0.0};
          if (jj > m) {
#pragma unroll
            for (int t = 0; t < kTg; ++t)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int q = (2 * t + h) & 3;
                const double2 ym = S.y[8 * t + 2 * g + h][m];
                const double2 yi = B[t][h];  // this column's own reflector (scaled)
                pr[q] = fma(ym.x, yi.x, fma(ym.y, yi.y, pr[q]));
                pi[q] = fma(ym.x, yi.y, fma(-ym.y, yi.x, pi[q]));
              }
          }
          const double gr = gsum4((pr[0] + pr[1]) + (pr[2] + pr[3]));
          const double gi = gsum4((pi[0] + pi[1]) + (pi[2] + pi[3]));
          if (jj > m && g == 0) ws[m * kPw + jj] = make_double2(gr, gi);
        }
        __syncwarp();
        // T[k][i] = -tau_i sum_{m = k}^{i-1} T[k][m] G[m][i]  (zlarft forward)
        for (int i = 1; i < kPw; ++i) {
          if (l < i) {
            const double2 ti = S.t[i][i];
            double ar = 0.0, ai = 0.0;
            for (int m = l; m < i; ++m) {
              const double2 tk = S.t[l][m], gm = ws[m * kPw + i];
              ar = fma(tk.x, gm.x, fma(-tk.y, gm.y, ar));
              ai = fma(tk.x, gm.y, fma(tk.y, gm.x, ai));
            }
            S.t[l][i] = make_double2(-(ti.x * ar - ti.y * ai), -(ti.x * ai + ti.y * ar));
          }
          __syncwarp();
        }
        if (l == 0) {
          wy_fence();
          vseq[tag % kRing] = tag;
        }
        __syncwarp();
      }
    }
  }
  __syncthreads();
  double2* out = reinterpret_cast<double2*>(T.dst);
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int c = idx / n, r = idx - c * n;
    out[(size_t)c * T.dst_ld + r] = r <= c ? R[wpidx(r, c)] : make_double2(0.0, 0.0);
  }
}

}  // namespace

size_t tsqr_wy_smem_bytes(int n) {
  return sizeof(double2) * (size_t(n) * (n + 1) / 2) + sizeof(WySlot) * kRing +
         sizeof(double2) * size_t(kWyWarps) * kPw * kPw;
}
int tsqr_wy_block_rows() { return kBr; }

int tsqr_wy_max_n() {
  int n = kWyWarps * kPw;
  while (n > 0 && tsqr_wy_smem_bytes(n) > size_t(kSmemCap)) --n;
  return n;
}

void launch_tsqr_wy(const QrTask* tasks, int n_tasks, size_t smem, cudaStream_t st) {
  if (n_tasks <= 0) return;
  static bool once = [] {
    cudaFuncSetAttribute(k_tsqr_wy, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCap);
    return true;
  }();
  (void)once;
  k_tsqr_wy<<<n_tasks, kWyThreads, smem, st>>>(tasks);
}

}  // namespace ebem_gpu
