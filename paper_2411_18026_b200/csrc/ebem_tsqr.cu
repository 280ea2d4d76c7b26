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
template <int LANES, int D, int W>
__device__ __forceinline__ void make_reflector(double2 (&B)[kRpt], bool mine, int i,
                                               int g, double2* R, int t,
                                               double2* vring, double2* tring,
                                               volatile int* seq, const volatile int* prog) {
  constexpr int kRows = LANES * kRpt;
  double p[4] = {0.0, 0.0, 0.0, 0.0};
  double2 alpha = make_double2(0.0, 0.0);
  if (mine) {
    alpha = R[pidx(i, i)];
#pragma unroll
    for (int k = 0; k < kRpt; ++k)
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
    for (int k = 0; k < kRpt; ++k)
      B[k] = make_double2(scal.x * B[k].x - scal.y * B[k].y,
                          scal.x * B[k].y + scal.y * B[k].x);
    if (g == 0) R[pidx(i, i)] = make_double2(beta, 0.0);
  }
  if (t >= D) wait_slot<W>(prog, t - D + 1);
  const int slot = t % D;
  if (mine) {
    double2* v = vring + slot * kRows;
#pragma unroll
    for (int k = 0; k < kRpt; ++k) v[g + LANES * k] = B[k];
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
template <int LANES, int THREADS, int D, int REGS>
__global__ void __launch_bounds__(THREADS, (65536 / (THREADS * REGS)) > 0 ? 65536 / (THREADS * REGS) : 1)
k_tsqr(const QrTask* __restrict__ tasks) {
  constexpr int kWarpsPerCta = THREADS / 32;
  constexpr int kRows = LANES * kRpt;
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
  if (wfirst >= n) {  // no columns: never holds the ring back
    if (lane == 0) vprog[warp] = 0x7fffffff;
  } else {
    for (int r0 = 0, b = 0; r0 < rows; r0 += kRows, ++b) {
      const int t0 = b * n;  // global index of reflector 0 of this block
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
      if (wfirst == 0)
        make_reflector<LANES, D, kWarpsPerCta>(B, j == 0, 0, g, R, t0, vring, tring, seq,
                                               vprog);
      for (int i = 0; i < wlast; ++i) {
        const int t = t0 + i;
        const int slot = t % D;
        wait_seq(seq, slot, t);
        const bool act = own && j > i;
        const double2* v = vring + slot * kRows;
        double2 rij = make_double2(0.0, 0.0);
        if (act) rij = R[pidx(i, j)];
        double ar[4] = {0.0, 0.0, 0.0, 0.0}, ai[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < kRpt; ++k) {
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
          for (int k = 0; k < kRpt; ++k) {
            const double2 a = v[g + LANES * k];
            B[k].x = fma(-a.x, fr, fma(a.y, fi, B[k].x));
            B[k].y = fma(-a.x, fi, fma(-a.y, fr, B[k].y));
          }
          if (g == 0) R[pidx(i, j)] = make_double2(rij.x - fr, rij.y - fi);
        }
        __syncwarp();
        if (lane == 0) {  // slot t read by this warp
          __threadfence_block();
          vprog[warp] = t + 1;
        }
        if (i + 1 >= wfirst)  // the warp owns column i + 1 (i + 1 <= wlast)
          make_reflector<LANES, D, kWarpsPerCta>(B, j == i + 1, i + 1, g, R, t + 1, vring,
                                                 tring, seq, vprog);
      }
      if (lane == 0) {  // nothing else of this block is read by this warp
        __threadfence_block();
        vprog[warp] = t0 + n;
      }
    }
  }
  __syncthreads();
  double2* out = reinterpret_cast<double2*>(T.dst);
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int c = idx / n, r = idx - c * n;
    out[(size_t)c * T.dst_ld + r] = r <= c ? R[pidx(r, c)] : make_double2(0.0, 0.0);
  }
}

}  // namespace

// variant 2: n <= 32 (the leaf blocks), 128 threads, so more independent
// reflector chains share an SM
constexpr int kTinyThreads = 128;
static int tsqr_slots(int n) { return n <= 64 ? EBEM_TSQR_S_SLOTS : EBEM_TSQR_M_SLOTS; }
int tsqr_variant(int n) { return n <= 32 ? 2 : n <= 64 ? 0 : n <= kTsqrMaxCols ? 1 : -1; }
int tsqr_block_rows(int n) {
  return tsqr_variant(n) == 1 ? EBEM_TSQR_M_LANES * kRpt : EBEM_TSQR_S_LANES * kRpt;
}
int tsqr_ctas_per_sm(int n) {
  const bool small = tsqr_variant(n) != 1;
  const int t = tsqr_variant(n) == 2 ? kTinyThreads : small ? EBEM_TSQR_S_THREADS : EBEM_TSQR_M_THREADS;
  const int by_regs = std::max(1, 65536 / (t * (small ? EBEM_TSQR_REGS : EBEM_TSQR_M_REGS)));
  const int by_smem = std::max(1, int((227 * 1024) / (tsqr_smem_bytes(n) + 1024)));
  return std::min(std::min(by_regs, by_smem), 2048 / t);
}
size_t tsqr_smem_bytes(int n) {
  return sizeof(double2) *
         (size_t(n) * (n + 1) / 2 + size_t(tsqr_slots(n)) * (tsqr_block_rows(n) + 1));
}

template <int L, int T, int D, int G>
static void launch_variant(const QrTask* tasks, int n_tasks, size_t smem, cudaStream_t st) {
  static bool once = [] {
    cudaFuncSetAttribute(k_tsqr<L, T, D, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return true;
  }();
  (void)once;
  k_tsqr<L, T, D, G><<<n_tasks, T, smem, st>>>(tasks);
}

void launch_tsqr(const QrTask* tasks, int n_tasks, int variant, size_t smem,
                 cudaStream_t st) {
  if (n_tasks <= 0) return;
  if (variant == 2)
    launch_variant<EBEM_TSQR_S_LANES, kTinyThreads, EBEM_TSQR_S_SLOTS, EBEM_TSQR_REGS>(tasks, n_tasks, smem, st);
  else if (variant == 0)
    launch_variant<EBEM_TSQR_S_LANES, EBEM_TSQR_S_THREADS, EBEM_TSQR_S_SLOTS, EBEM_TSQR_REGS>(tasks, n_tasks, smem, st);
  else
    launch_variant<EBEM_TSQR_M_LANES, EBEM_TSQR_M_THREADS, EBEM_TSQR_M_SLOTS, EBEM_TSQR_M_REGS>(tasks, n_tasks, smem, st);
}

}  // namespace ebem_gpu
