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
//
// Layout: LANES consecutive lanes own one column, lane g holds rows
// g, g + LANES, ... of the block.  The step sequence is a chain: reflector
// t + 1 needs column t + 1 updated by reflector t.  The group owning column
// t + 1 applies reflector t to its columns first and immediately generates
// reflector t + 1 (look-ahead).  Reflectors travel through a ring of D
// shared-memory slots (full: a per-slot sequence number; empty: per-warp
// progress counters), and warps are coupled only through
// the reflectors they consume.  A warp needs reflectors 0 .. wlast - 1 of a
// block only, so it proceeds to the next block as soon as its own columns
// are eliminated: the reflector chains of consecutive blocks overlap in a
// wavefront instead of the CTA stepping through n reflectors per block.  The
// R factors of several row pieces of one matrix are stacked and reduced again
// by the same kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdint.h>

#include "ebem_dense.h"

namespace ebem_gpu {

namespace {

#ifndef EBEM_TSQR_RPT
#define EBEM_TSQR_RPT 8
#endif
constexpr int kRpt = EBEM_TSQR_RPT;  // block rows per lane
// (lanes per column, CTA threads) of the two variants: n <= 64 and n <= 128.
// Smaller CTAs put several independent reflector chains on one SM.
#ifndef EBEM_TSQR_S_LANES
#define EBEM_TSQR_S_LANES 4
#endif
#ifndef EBEM_TSQR_S_THREADS
#define EBEM_TSQR_S_THREADS 256
#endif
#ifndef EBEM_TSQR_M_LANES
#define EBEM_TSQR_M_LANES 4
#endif
#ifndef EBEM_TSQR_M_THREADS
#define EBEM_TSQR_M_THREADS 512
#endif
static_assert(EBEM_TSQR_S_THREADS / EBEM_TSQR_S_LANES >= 64, "small variant: 64 columns");
static_assert(EBEM_TSQR_M_THREADS / EBEM_TSQR_M_LANES >= kTsqrMaxCols, "medium variant");
// reflector ring depth of the two variants (one block's reflectors for
// n <= 64 lets the column groups drift a whole block apart)
#ifndef EBEM_TSQR_S_SLOTS
#define EBEM_TSQR_S_SLOTS 64
#endif
#ifndef EBEM_TSQR_M_SLOTS
#define EBEM_TSQR_M_SLOTS 128
#endif

__device__ __forceinline__ int pidx(int i, int j) { return ((j * (j + 1)) >> 1) + i; }

template <int LANES>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = LANES >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Slot reuse: each warp publishes how many reflectors (global index,
// block-major) it no longer needs; a producer may overwrite the slot of
// reflector t - D once every warp has moved past it.  (Counters rather than
// an "empty" mbarrier: a warp with no column right of reflector i never reads
// it, and must not hold the ring back while it works on the next block.)
template <int W>
__device__ __forceinline__ void wait_slot(const volatile int* prog, int need) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    const int v = lane < W ? prog[lane] : 0x7fffffff;
    if (__reduce_min_sync(0xffffffffu, v) >= need) break;
    __nanosleep(32);
  }
  __threadfence_block();
}

// Reflector of column i from the owning group's registers (warp-uniform call;
// only the `mine` lanes write).  Waits for the ring slot to be free first.
#ifdef EBEM_TSQR_TIMING
#define TSQR_T0(v) const long long v = clock64()
#define TSQR_ACC(acc, v) acc += clock64() - v
#else
#define TSQR_T0(v)
#define TSQR_ACC(acc, v)
#endif
template <int LANES, int RPT, int D, int W>
__device__ __forceinline__ void make_reflector(double2 (&B)[RPT], bool mine, int i,
                                               int g, double2* R, int t,
                                               double2* vring, double2* tring,
                                               volatile int* seq, const volatile int* prog,
                                               long long& t_slot) {
  constexpr int kRows = LANES * RPT;
  double p[4] = {0.0, 0.0, 0.0, 0.0};
  double2 alpha = make_double2(0.0, 0.0);
  if (mine) {
    alpha = R[pidx(i, i)];
#pragma unroll
    for (int k = 0; k < RPT; ++k)
      p[k & 3] = fma(B[k].x, B[k].x, fma(B[k].y, B[k].y, p[k & 3]));
  }
  const double xnorm2 = group_sum<LANES>((p[0] + p[1]) + (p[2] + p[3]));
  double2 tau = make_double2(0.0, 0.0);
  if (mine && !(xnorm2 == 0.0 && alpha.y == 0.0)) {
    // x2 = |alpha|^2 + ||x||^2;  s = 1 / sqrt(x2);  beta = -+ x2 s.
    // With ar = Re(alpha) - beta (|ar| >= 1/s >= |ai|) scaled to O(1):
    // 1 / (alpha - beta) = s (ar s - i ai s) / ((ar s)^2 + (ai s)^2).
    // Two special functions on the chain, no true division with a zero
    // numerator (that sends it down its slow path), no underflow in the
    // squares of the geometrically shrinking residues of eliminated columns.
    const double x2 = fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, xnorm2));
    const double s = rsqrt(x2);
    const double nrm = x2 * s;
    const bool pos = alpha.x >= 0.0;
    const double beta = pos ? -nrm : nrm;
    const double ib = pos ? -s : s;
    tau = make_double2((beta - alpha.x) * ib, -alpha.y * ib);
    const double arn = fma(alpha.x, s, pos ? 1.0 : -1.0);  // (alpha.x - beta) s
    const double ain = alpha.y * s;
    const double id = s / fma(arn, arn, ain * ain);
    const double2 scal = make_double2(arn * id, -ain * id);
#pragma unroll
    for (int k = 0; k < RPT; ++k)
      B[k] = make_double2(scal.x * B[k].x - scal.y * B[k].y,
                          scal.x * B[k].y + scal.y * B[k].x);
    if (g == 0) R[pidx(i, i)] = make_double2(beta, 0.0);
  }
  {
    TSQR_T0(c0);
    if (t >= D) wait_slot<W>(prog, t - D + 1);
    TSQR_ACC(t_slot, c0);
  }
  const int slot = t % D;
  if (mine) {
    double2* v = vring + slot * kRows;
#pragma unroll
    for (int k = 0; k < RPT; ++k) v[g + LANES * k] = B[k];
    if (g == 0) tring[slot] = tau;
  }
  __syncwarp();
  if (mine && g == 0) {
    __threadfence_block();
    seq[slot] = t;  // the slot now holds reflector t
  }
}

// Wait until the slot holds reflector t.  A sequence number, not an mbarrier
// phase: a warp that skipped reflector t - D (no column right of it) may get
// here before t - D was even produced, and a parity test would then mistake
// phase t/D - 2 for t/D.
#ifndef EBEM_TSQR_SLEEP
#define EBEM_TSQR_SLEEP 20
#endif
__device__ __forceinline__ void wait_seq(const volatile int* seq, int slot, int t) {
  while (seq[slot] != t) {
    if (EBEM_TSQR_SLEEP > 0) __nanosleep(EBEM_TSQR_SLEEP);
  }
  __threadfence_block();
}

// registers per thread the CTA size is sized for (the medium variant is one
// CTA per SM by shared memory anyway: R up to 132 KB plus the ring)
#ifndef EBEM_TSQR_REGS
#define EBEM_TSQR_REGS 64
#endif
#ifndef EBEM_TSQR_M_REGS
#define EBEM_TSQR_M_REGS 128
#endif
// Block-skewed wavefront: warp w owns columns [wfirst, wlast] and, per row
// block, consumes reflectors 0 .. wlast - 1 only.  Reflector i of block b+1
// needs column i of block b+1 (its owner) and R_ii after block b (same
// owner), so a warp whose columns are done moves on to the next block at
// once: the reflector chains of consecutive blocks overlap instead of the
// whole CTA stepping through n reflectors per block in lock step.
template <int LANES, int RPT, int THREADS, int D, int REGS>
__global__ void __launch_bounds__(THREADS, (65536 / (THREADS * REGS)) > 0 ? 65536 / (THREADS * REGS) : 1)
k_tsqr(const QrTask* __restrict__ tasks) {
  constexpr int kWarpsPerCta = THREADS / 32;
  constexpr int kRows = LANES * RPT;
  constexpr int kGroupsPerWarp = 32 / LANES;
  extern __shared__ double2 R[];  // packed upper triangle | v ring | tau ring
  __shared__ int seq_s[D];
  __shared__ int prog[kWarpsPerCta];
  const QrTask T = tasks[blockIdx.x];
  const int n = T.n, rows = T.rows, ld = T.ld;
  double2* vring = R + ((n * (n + 1)) >> 1);
  double2* tring = vring + D * kRows;
  const int g = threadIdx.x % LANES;
  const int j = threadIdx.x / LANES;  // owned column
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wfirst = warp * kGroupsPerWarp;  // first column of the warp
  const int wlast = min(wfirst + kGroupsPerWarp - 1, n - 1);  // last real column
  for (int q = threadIdx.x; q < ((n * (n + 1)) >> 1); q += blockDim.x)
    R[q] = make_double2(0.0, 0.0);
  for (int q = threadIdx.x; q < D; q += blockDim.x) seq_s[q] = -1;
  if (threadIdx.x < kWarpsPerCta) prog[threadIdx.x] = 0;
  const double2* src = reinterpret_cast<const double2*>(T.src) + (size_t)j * ld;
  const bool own = j < n;
  __syncthreads();
  volatile int* vprog = prog;
  volatile int* seq = seq_s;
  long long t_slot = 0, t_seq = 0, t_make = 0, t_load = 0;
  TSQR_T0(c_all);
  if (wfirst >= n) {  // no columns: never holds the ring back
    if (lane == 0) vprog[warp] = 0x7fffffff;
  } else {
    for (int r0 = 0, b = 0; r0 < rows; r0 += kRows, ++b) {
      const int t0 = b * n;  // global index of reflector 0 of this block
      double2 B[RPT];
      TSQR_T0(c_ld);
#pragma unroll
      for (int k = 0; k < RPT; ++k) {
        const int r = r0 + g + LANES * k;
        B[k] = (own && r < rows) ? src[r] : make_double2(0.0, 0.0);
      }
#ifdef EBEM_TSQR_TIMING
      if (B[0].x == 1.2345e300) t_load += 1;  // (forces the loads to complete here)
#endif
      TSQR_ACC(t_load, c_ld);
      if (own && r0 + kRows < rows) {  // warm L2 for the next block
        const int r = r0 + kRows + g * RPT;
        if (r < rows) asm volatile("prefetch.global.L2 [%0];" ::"l"(src + r));
      }
      if (wfirst == 0) {
        TSQR_T0(c_mk);
        make_reflector<LANES, RPT, D, kWarpsPerCta>(B, j == 0, 0, g, R, t0, vring, tring, seq,
                                               vprog, t_slot);
        TSQR_ACC(t_make, c_mk);
      }
      for (int i = 0; i < wlast; ++i) {
        const int t = t0 + i;
        const int slot = t % D;
        {
          TSQR_T0(c_sq);
          wait_seq(seq, slot, t);
          TSQR_ACC(t_seq, c_sq);
        }
        const bool act = own && j > i;
        const double2* v = vring + slot * kRows;
        double2 rij = make_double2(0.0, 0.0);
        if (act) rij = R[pidx(i, j)];
        double ar[4] = {0.0, 0.0, 0.0, 0.0}, ai[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < RPT; ++k) {
          const double2 a = v[g + LANES * k], bb = B[k];
          ar[k & 3] = fma(a.x, bb.x, fma(a.y, bb.y, ar[k & 3]));
          ai[k & 3] = fma(a.x, bb.y, fma(-a.y, bb.x, ai[k & 3]));
        }
        double sr = group_sum<LANES>((ar[0] + ar[1]) + (ar[2] + ar[3]));
        double si = group_sum<LANES>((ai[0] + ai[1]) + (ai[2] + ai[3]));
        const double2 tau = tring[slot];
        if (act) {
          sr += rij.x;
          si += rij.y;
          // f = conj(tau) s
          const double fr = tau.x * sr + tau.y * si;
          const double fi = tau.x * si - tau.y * sr;
#pragma unroll
          for (int k = 0; k < RPT; ++k) {
            const double2 a = v[g + LANES * k];
            B[k].x = fma(-a.x, fr, fma(a.y, fi, B[k].x));
            B[k].y = fma(-a.x, fi, fma(-a.y, fr, B[k].y));
          }
          if (g == 0) R[pidx(i, j)] = make_double2(rij.x - fr, rij.y - fi);
        }
        __syncwarp();
        // progress (slot reuse) published every fourth reflector and before
        // the warp's own reflectors: a fence and a store less per step
        if (lane == 0 && ((i & 3) == 3 || i + 1 >= wfirst)) {  // slots <= t read by this warp
          __threadfence_block();
          vprog[warp] = t + 1;
        }
        if (i + 1 >= wfirst) {  // the warp owns column i + 1 (i + 1 <= wlast)
          TSQR_T0(c_mk);
          make_reflector<LANES, RPT, D, kWarpsPerCta>(B, j == i + 1, i + 1, g, R, t + 1, vring,
                                                 tring, seq, vprog, t_slot);
          TSQR_ACC(t_make, c_mk);
        }
      }
      if (lane == 0) {  // nothing else of this block is read by this warp
        __threadfence_block();
        vprog[warp] = t0 + n;
      }
    }
  }
#ifdef EBEM_TSQR_TIMING
  if (lane == 0 && blockIdx.x == gridDim.x / 2 && wfirst < n)
    printf("tsqr n=%d rows=%d warp=%d all=%lld load=%lld seq=%lld make=%lld (slot=%lld)\n", n, rows,
           warp, clock64() - c_all, t_load, t_seq, t_make, t_slot);
#endif
  __syncthreads();
  double2* out = reinterpret_cast<double2*>(T.dst);
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int c = idx / n, r = idx - c * n;
    out[(size_t)c * T.dst_ld + r] = r <= c ? R[pidx(r, c)] : make_double2(0.0, 0.0);
  }
}

// ---------------------------------------------------------------------------
// Warp-private TSQR (variants 3 and 4): one warp per row piece, lane = column.
//
// The wavefront kernel above couples the warps of a CTA through the reflector
// ring, so its chain (one hand-off per reflector per row block) sets the
// time.  Here every warp streams its own piece into its own R and nothing
// crosses warps: lane l owns column l (variant 3, n <= 32; rows in blocks of
// 32) or columns l and n - 32 + l ... see col_of (variant 4, n <= 64; blocks
// of 16 rows), the block's rows of its columns live in the lane's registers
// and R (packed upper triangle, row-major, so R(i, .) of consecutive lanes is
// contiguous) lives in the warp's slice of shared memory.  Column c of R is
// only ever touched by the lane that owns column c, so the only exchange is
// the reflector itself: the owner of column i writes v and tau into a
// double-buffered warp slot, one __syncwarp, every lane reads it as a
// broadcast.  Same zlarfg / zlarf arithmetic as make_reflector / k_tsqr:
//   x = [R_ii; B(:, i)], beta = -sign(Re R_ii) ||x||, tau = (beta - R_ii) / beta,
//   v = B(:, i) / (R_ii - beta);  s = R_ij + v^H B(:, j), f = conj(tau) s,
//   R_ij -= f, B(:, j) -= v f.
// Latency is hidden across warps (10-12 independent chains per SM) instead
// of inside one chain; the pieces' R factors are stacked and reduced again
// by the next round of reduce_tall.
template <int SLOTS>
struct LaneCfg;
template <>
struct LaneCfg<1> {
  static constexpr int kBr = 16, kWpc = 4, kMinB = 3;
};
template <>
struct LaneCfg<2> {
  static constexpr int kBr = 16, kWpc = 2, kMinB = 4;
};

__device__ __forceinline__ int roff(int i, int n) { return i * n - ((i * (i - 1)) >> 1); }

template <int BR>
__device__ __forceinline__ void lane_reflector(double2 (&B)[BR], double2* Rs, int i, int n,
                                               double2* vb, double2* tb) {
  double p[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
  for (int k = 0; k < BR; ++k) p[k & 3] = fma(B[k].x, B[k].x, fma(B[k].y, B[k].y, p[k & 3]));
  const double xnorm2 = (p[0] + p[1]) + (p[2] + p[3]);
  double2 alpha = Rs[roff(i, n)];
  double2 tau = make_double2(0.0, 0.0);
  if (!(xnorm2 == 0.0 && alpha.y == 0.0)) {
    double x2 = fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, xnorm2));
    // Stacked R factors drive later columns through cascades of rounding
    // residues whose squares leave the normal range; the approximate rsqrt
    // flushes those, so such columns are scaled by 2^600 first (exact).
    double sc = 1.0;
    if (x2 < 0x1p-960) {
      sc = 0x1p600;
      double q[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < BR; ++k) {
        const double bx = B[k].x * sc, by = B[k].y * sc;
        q[k & 3] = fma(bx, bx, fma(by, by, q[k & 3]));
      }
      alpha = make_double2(alpha.x * sc, alpha.y * sc);
      x2 = fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, (q[0] + q[1]) + (q[2] + q[3])));
    }
    // rsqrt and the reciprocal below by the hardware approximations and
    // Newton steps (x2 normal, den in [1, 2]): the library versions carry
    // slow-path calls that spill the lane's block registers
    double s;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(s) : "d"(x2));
#pragma unroll
    for (int it = 0; it < 3; ++it) {
      const double e = fma(-x2 * s, s, 1.0);
      s = fma(0.5 * s, e, s);
    }
    const double nrm = x2 * s;
    const bool pos = alpha.x >= 0.0;
    const double beta = pos ? -nrm : nrm;
    const double ib = pos ? -s : s;
    tau = make_double2((beta - alpha.x) * ib, -alpha.y * ib);
    const double arn = fma(alpha.x, s, pos ? 1.0 : -1.0);
    const double ain = alpha.y * s;
    const double den = fma(arn, arn, ain * ain);
    double rc;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(rc) : "d"(den));
#pragma unroll
    for (int it = 0; it < 3; ++it) {
      const double e = fma(-den, rc, 1.0);
      rc = fma(rc, e, rc);
    }
    const double id = s * rc * sc;
    const double2 scal = make_double2(arn * id, -ain * id);
#pragma unroll
    for (int k = 0; k < BR; ++k)
      vb[k] = make_double2(scal.x * B[k].x - scal.y * B[k].y, scal.x * B[k].y + scal.y * B[k].x);
    Rs[roff(i, n)] = make_double2(beta * (1.0 / sc), 0.0);
  } else {
#pragma unroll
    for (int k = 0; k < BR; ++k) vb[k] = B[k];
  }
  *tb = tau;
}

// s = R_ij + v^H B(:, j) for one column slot, then R_ij -= f, B -= v f
// (dots of both slots first so their chains overlap; see k_tsqr_lane)
template <int BR>
__device__ __forceinline__ void lane_update(double2 (&B)[BR], const double2* v, double2 tau,
                                            double sr, double si, double2* rij) {
  const double2 r = *rij;
  sr += r.x;
  si += r.y;
  const double fr = tau.x * sr + tau.y * si;
  const double fi = tau.x * si - tau.y * sr;
#pragma unroll
  for (int k = 0; k < BR; ++k) {
    const double2 a = v[k];
    B[k].x = fma(-a.x, fr, fma(a.y, fi, B[k].x));
    B[k].y = fma(-a.x, fi, fma(-a.y, fr, B[k].y));
  }
  *rij = make_double2(r.x - fr, r.y - fi);
}

template <int BR>
__device__ __forceinline__ void lane_dot(const double2 (&B)[BR], const double2* v, double& sr,
                                         double& si) {
  double ar[2] = {0.0, 0.0}, ai[2] = {0.0, 0.0};
#pragma unroll
  for (int k = 0; k < BR; ++k) {
    const double2 a = v[k], bb = B[k];
    ar[k & 1] = fma(a.x, bb.x, fma(a.y, bb.y, ar[k & 1]));
    ai[k & 1] = fma(a.x, bb.y, fma(-a.y, bb.x, ai[k & 1]));
  }
  sr = ar[0] + ar[1];
  si = ai[0] + ai[1];
}

template <int SLOTS>
__global__ void __launch_bounds__(LaneCfg<SLOTS>::kWpc * 32, LaneCfg<SLOTS>::kMinB)
k_tsqr_lane(const QrTask* __restrict__ tasks, int n_tasks, int wstride) {
  constexpr int BR = LaneCfg<SLOTS>::kBr;
  extern __shared__ double2 sm_lane[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int task = blockIdx.x * LaneCfg<SLOTS>::kWpc + warp;
  if (task >= n_tasks) return;  // warps are independent: no CTA barrier below
  const QrTask T = tasks[task];
  const int n = T.n, rows = T.rows, ld = T.ld;
  const int nr = (n * (n + 1)) >> 1;
  double2* Rs = sm_lane + size_t(warp) * wstride;
  double2* vbuf = Rs + nr;  // 2 x BR
  double2* tbuf = vbuf + 2 * BR;
  // slot 0: column n2 + lane; slot 1 (variant 4): column lane < n2.  The low
  // columns sit in slot 1 so that slot retires after n2 reflectors.
  const int n2 = SLOTS == 2 ? n - 32 : 0;
  const int c0 = n2 + lane;
  const bool v0 = c0 < n;
  const bool v1 = SLOTS == 2 && lane < n2;
  for (int q = lane; q < nr; q += 32) Rs[q] = make_double2(0.0, 0.0);
  __syncwarp();
  const double2* src = reinterpret_cast<const double2*>(T.src);
  const double2* s0 = src + size_t(v0 ? c0 : 0) * ld;
  const double2* s1 = src + size_t(v1 ? lane : 0) * ld;
  for (int r0 = 0; r0 < rows; r0 += BR) {
    double2 B0[BR], B1[BR];  // B1 unused (eliminated) for SLOTS == 1
#pragma unroll
    for (int k = 0; k < BR; ++k) {
      const int r = r0 + k;
      B0[k] = (v0 && r < rows) ? __ldg(s0 + r) : make_double2(0.0, 0.0);
      B1[k] = (SLOTS == 2 && v1 && r < rows) ? __ldg(s1 + r) : make_double2(0.0, 0.0);
    }
    if (r0 + BR < rows) {  // warm L2 for the next block of this lane's columns
      if (v0) asm volatile("prefetch.global.L2 [%0];" ::"l"(s0 + r0 + BR));
      if (SLOTS == 2 && v1) asm volatile("prefetch.global.L2 [%0];" ::"l"(s1 + r0 + BR));
    }
    for (int i = 0; i < n; ++i) {
      double2* vb = vbuf + (i & 1) * BR;
      double2* tb = tbuf + (i & 1);
      if constexpr (SLOTS == 2) {
        if (i < n2) {
          if (lane == i) lane_reflector<BR>(B1, Rs, i, n, vb, tb);
        } else if (lane == i - n2) {
          lane_reflector<BR>(B0, Rs, i, n, vb, tb);
        }
      } else {
        if (lane == i) lane_reflector<BR>(B0, Rs, i, n, vb, tb);
      }
      __syncwarp();
      if (i + 1 >= n) break;
      const double2 tau = *tb;
      const int ro = roff(i, n) - i;  // R(i, c) = Rs[ro + c]
      if constexpr (SLOTS == 2) {
        if (i + 1 < n2) {  // both slots have columns right of i (every slot-0 column)
          double sr0, si0, sr1, si1;
          lane_dot<BR>(B0, vb, sr0, si0);
          lane_dot<BR>(B1, vb, sr1, si1);
          if (v0) lane_update<BR>(B0, vb, tau, sr0, si0, Rs + ro + c0);
          if (v1 && lane > i) lane_update<BR>(B1, vb, tau, sr1, si1, Rs + ro + lane);
          continue;
        }
      }
      double sr0, si0;
      lane_dot<BR>(B0, vb, sr0, si0);
      if (v0 && c0 > i) lane_update<BR>(B0, vb, tau, sr0, si0, Rs + ro + c0);
    }
  }
  // R (n x n, column-major, zeros below the diagonal); each lane its columns
  double2* out = reinterpret_cast<double2*>(T.dst);
  if (v0)
    for (int r = 0; r < n; ++r)
      out[size_t(c0) * T.dst_ld + r] = r <= c0 ? Rs[roff(r, n) + c0 - r] : make_double2(0.0, 0.0);
  if (SLOTS == 2 && v1)
    for (int r = 0; r < n; ++r)
      out[size_t(lane) * T.dst_ld + r] = r <= lane ? Rs[roff(r, n) + lane - r] : make_double2(0.0, 0.0);
}

}  // namespace

static bool lane_tsqr_enabled() {  // EBEM_TSQR_LANE=0: the wavefront kernel (A/B)
  static const bool on = [] {
    const char* e = std::getenv("EBEM_TSQR_LANE");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}

static int lane_wstride(int n, int slots) {
  const int br = slots == 1 ? LaneCfg<1>::kBr : LaneCfg<2>::kBr;
  return (n * (n + 1)) / 2 + 2 * br + 2;
}

// variant 2: n <= 32 (the leaf blocks), 128 threads, so more independent
// reflector chains share an SM
constexpr int kTinyThreads = 128;
// variant 5: 64 < n <= 96 on 384-thread CTAs (12 warps x 8 columns) with
// 16 rows per lane (64-row blocks): the kernel's time is (row blocks) x
// (reflectors) x (the last warp's ~800 cycles per consumed reflector), and
// 170 registers per thread hold a block twice as tall, so the same chain
// covers twice the rows (EBEM_TSQR_TALL=0: variant 1 for these, A/B).
constexpr int kTallCols = 96, kTallThreads = 384, kTallRpt = 16, kTallSlots = 128;
// variant 7: 96 < n <= 112 (the two top levels at the bench size) on 512
// threads with 12 rows per lane (48-row blocks; 128 registers, a few spilled
// bytes), R (<= 101 KB) beside a 128-slot ring (EBEM_TSQR_TALL7=0: variant 1).
constexpr int kTall7Cols = 112, kTall7Threads = 512, kTall7Rpt = 12, kTall7Slots = 128;
static bool tall7_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("EBEM_TSQR_TALL7");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}
static bool tall_tsqr_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("EBEM_TSQR_TALL");
    return e == nullptr || std::atoi(e) != 0;
  }();
  return on;
}
static int tsqr_slots(int n) {
  if (tsqr_variant(n) == 5) return kTallSlots;
  if (tsqr_variant(n) == 7) return kTall7Slots;
  return n <= 64 ? EBEM_TSQR_S_SLOTS : EBEM_TSQR_M_SLOTS;
}
int tsqr_variant(int n) {
  if (lane_tsqr_enabled() && n <= 64) return n <= 32 ? 3 : 4;
  if (tall_tsqr_enabled() && n > 64 && n <= kTallCols) return 5;
  if (tall_tsqr_enabled() && tall7_enabled() && n > kTallCols && n <= kTall7Cols) return 7;
  return n <= 32 ? 2 : n <= 64 ? 0 : n <= kTsqrMaxCols ? 1 : -1;
}
int tsqr_block_rows(int n) {
  if (tsqr_variant(n) == 3) return LaneCfg<1>::kBr;
  if (tsqr_variant(n) == 4) return LaneCfg<2>::kBr;
  if (tsqr_variant(n) == 5) return EBEM_TSQR_M_LANES * kTallRpt;
  if (tsqr_variant(n) == 7) return EBEM_TSQR_M_LANES * kTall7Rpt;
  return tsqr_variant(n) == 1 ? EBEM_TSQR_M_LANES * kRpt : EBEM_TSQR_S_LANES * kRpt;
}
int tsqr_ctas_per_sm(int n) {
  if (tsqr_variant(n) == 3 || tsqr_variant(n) == 4) {  // resident warps (= tasks) per SM
    const int slots = tsqr_variant(n) == 3 ? 1 : 2;
    const int wpc = slots == 1 ? LaneCfg<1>::kWpc : LaneCfg<2>::kWpc;
    const int minb = slots == 1 ? LaneCfg<1>::kMinB : LaneCfg<2>::kMinB;
    const int by_smem = int((227 * 1024) / (tsqr_smem_bytes(n) + 1024));
    return wpc * std::max(1, std::min(minb, by_smem));
  }
  if (tsqr_variant(n) >= 5) return 1;
  const bool small = tsqr_variant(n) != 1;
  const int t = tsqr_variant(n) == 2 ? kTinyThreads : small ? EBEM_TSQR_S_THREADS : EBEM_TSQR_M_THREADS;
  const int by_regs = std::max(1, 65536 / (t * (small ? EBEM_TSQR_REGS : EBEM_TSQR_M_REGS)));
  const int by_smem = std::max(1, int((227 * 1024) / (tsqr_smem_bytes(n) + 1024)));
  return std::min(std::min(by_regs, by_smem), 2048 / t);
}
size_t tsqr_smem_bytes(int n) {
  if (tsqr_variant(n) == 3 || tsqr_variant(n) == 4) {
    const int slots = tsqr_variant(n) == 3 ? 1 : 2;
    const int wpc = slots == 1 ? LaneCfg<1>::kWpc : LaneCfg<2>::kWpc;
    return sizeof(double2) * size_t(wpc) * lane_wstride(n, slots);
  }
  return sizeof(double2) *
         (size_t(n) * (n + 1) / 2 + size_t(tsqr_slots(n)) * (tsqr_block_rows(n) + 1));
}

template <int L, int RPT, int T, int D, int G>
static void launch_variant(const QrTask* tasks, int n_tasks, size_t smem, cudaStream_t st) {
  static bool once = [] {
    cudaFuncSetAttribute(k_tsqr<L, RPT, T, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         216 * 1024);
    return true;
  }();
  (void)once;
  k_tsqr<L, RPT, T, D, G><<<n_tasks, T, smem, st>>>(tasks);
}

void launch_tsqr(const QrTask* tasks, int n_tasks, int variant, size_t smem,
                 cudaStream_t st) {
  if (n_tasks <= 0) return;
  if (variant == 3 || variant == 4) {
    // smem was sized for the launch's largest n: recover that n's stride
    const int slots = variant == 3 ? 1 : 2;
    const int wpc = slots == 1 ? LaneCfg<1>::kWpc : LaneCfg<2>::kWpc;
    const int wstride = int(smem / (sizeof(double2) * wpc));
    const int grid = (n_tasks + wpc - 1) / wpc;
    static bool once = [] {
      cudaFuncSetAttribute(k_tsqr_lane<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_tsqr_lane<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      return true;
    }();
    (void)once;
    if (slots == 1)
      k_tsqr_lane<1><<<grid, wpc * 32, smem, st>>>(tasks, n_tasks, wstride);
    else
      k_tsqr_lane<2><<<grid, wpc * 32, smem, st>>>(tasks, n_tasks, wstride);
    return;
  }
  if (variant == 2)
    launch_variant<EBEM_TSQR_S_LANES, kRpt, kTinyThreads, EBEM_TSQR_S_SLOTS, EBEM_TSQR_REGS>(tasks, n_tasks, smem, st);
  else if (variant == 0)
    launch_variant<EBEM_TSQR_S_LANES, kRpt, EBEM_TSQR_S_THREADS, EBEM_TSQR_S_SLOTS, EBEM_TSQR_REGS>(tasks, n_tasks, smem, st);
  else if (variant == 5)
    launch_variant<EBEM_TSQR_M_LANES, kTallRpt, kTallThreads, kTallSlots, 170>(tasks, n_tasks, smem, st);
  else if (variant == 7)
    launch_variant<EBEM_TSQR_M_LANES, kTall7Rpt, kTall7Threads, kTall7Slots, 128>(tasks, n_tasks, smem, st);
  else
    launch_variant<EBEM_TSQR_M_LANES, kRpt, EBEM_TSQR_M_THREADS, EBEM_TSQR_M_SLOTS, EBEM_TSQR_M_REGS>(tasks, n_tasks, smem, st);
}

}  // namespace ebem_gpu
