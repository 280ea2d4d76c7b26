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
// reflector t + 1 (look-ahead).  Reflectors travel through a ring of kSlots
// shared-memory slots guarded by mbarriers (full: the producing group's lanes
// arrive; empty: every warp arrives once it has read the slot), so warps are
// coupled only through the reflectors they consume: the step time is the
// producer chain, not a CTA-wide barrier plus the slowest warp.  The R
// factors of several row pieces of one matrix are stacked and reduced again
// by the same kernel.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdint.h>

#include "ebem_dense.h"

namespace ebem_gpu {

namespace {

constexpr int kRpt = 8;    // block rows per lane
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
constexpr int kSlots = 8;  // reflector ring depth

__device__ __forceinline__ int pidx(int i, int j) { return ((j * (j + 1)) >> 1) + i; }

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

template <int LANES>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = LANES >> 1; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Reflector of column i from the owning group's registers (warp-uniform call;
// only the `mine` lanes write).  Waits for the slot to be free first.
template <int LANES>
__device__ __forceinline__ void make_reflector(double2 (&B)[kRpt], bool mine, int i,
                                               int g, double2* R, long long t,
                                               double2* vring, double2* tring,
                                               uint64_t* full, uint64_t* empty) {
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
  if (!mine) return;
  double2 tau = make_double2(0.0, 0.0);
  if (!(xnorm2 == 0.0 && alpha.y == 0.0)) {
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
  const int slot = int(t % kSlots);
  if (t >= kSlots) mbar_wait(empty + slot, uint32_t(((t / kSlots) + 1) & 1));
  double2* v = vring + slot * kRows;
#pragma unroll
  for (int k = 0; k < kRpt; ++k) v[g + LANES * k] = B[k];
  if (g == 0) tring[slot] = tau;
  mbar_arrive(full + slot);
}

#ifndef EBEM_TSQR_REGS
#define EBEM_TSQR_REGS 64  // registers per thread the CTA size is sized for
#endif
template <int LANES, int THREADS>
__global__ void __launch_bounds__(THREADS, (65536 / (THREADS * EBEM_TSQR_REGS)) > 0 ? 65536 / (THREADS * EBEM_TSQR_REGS) : 1)
k_tsqr(const QrTask* __restrict__ tasks) {
  constexpr int kWarpsPerCta = THREADS / 32;
  constexpr int kRows = LANES * kRpt;
  constexpr int kGroupsPerWarp = 32 / LANES;
  extern __shared__ double2 R[];  // packed upper triangle | v ring | tau ring
  __shared__ uint64_t full[kSlots], empty[kSlots];
  const QrTask T = tasks[blockIdx.x];
  const int n = T.n, rows = T.rows, ld = T.ld;
  double2* vring = R + ((n * (n + 1)) >> 1);
  double2* tring = vring + kSlots * kRows;
  const int g = threadIdx.x % LANES;
  const int j = threadIdx.x / LANES;  // owned column
  const int lane = threadIdx.x & 31;
  const int wfirst = (threadIdx.x >> 5) * kGroupsPerWarp;  // first column of the warp
  const int wlast = wfirst + kGroupsPerWarp - 1;
  for (int q = threadIdx.x; q < ((n * (n + 1)) >> 1); q += blockDim.x)
    R[q] = make_double2(0.0, 0.0);
  if (threadIdx.x < kSlots) {
    mbar_init(full + threadIdx.x, LANES);
    mbar_init(empty + threadIdx.x, kWarpsPerCta);
  }
  const double2* src = reinterpret_cast<const double2*>(T.src) + (size_t)j * ld;
  const bool own = j < n;
  __syncthreads();
  long long t = 0;  // global reflector index (block-major)
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
    if (wfirst == 0)
      make_reflector<LANES>(B, j == 0, 0, g, R, t, vring, tring, full, empty);
    for (int i = 0; i < n; ++i, ++t) {
      const int slot = int(t % kSlots);
      mbar_wait(full + slot, uint32_t((t / kSlots) & 1));
      if (wlast > i && wfirst < n) {  // warp-uniform: some column j > i here
        const bool act = own && j > i;
        const double2* v = vring + slot * kRows;
        double2 rij = make_double2(0.0, 0.0);
        if (act) rij = R[pidx(i, j)];
        double ar[4] = {0.0, 0.0, 0.0, 0.0}, ai[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int k = 0; k < kRpt; ++k) {
          const double2 a = v[g + LANES * k], b = B[k];
          ar[k & 3] = fma(a.x, b.x, fma(a.y, b.y, ar[k & 3]));
          ai[k & 3] = fma(a.x, b.y, fma(-a.y, b.x, ai[k & 3]));
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
        if (lane == 0) mbar_arrive(empty + slot);  // slot read by this warp
        if (i + 1 < n && wfirst <= i + 1 && i + 1 <= wlast)
          make_reflector<LANES>(B, j == i + 1, i + 1, g, R, t + 1, vring, tring, full,
                                empty);
      } else {
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + slot);
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

int tsqr_variant(int n) { return n <= 64 ? 0 : n <= kTsqrMaxCols ? 1 : -1; }
int tsqr_block_rows(int n) {
  return tsqr_variant(n) == 0 ? EBEM_TSQR_S_LANES * kRpt : EBEM_TSQR_M_LANES * kRpt;
}
int tsqr_ctas_per_sm(int n) {
  const int t = tsqr_variant(n) == 0 ? EBEM_TSQR_S_THREADS : EBEM_TSQR_M_THREADS;
  const int by_regs = std::max(1, 65536 / (t * EBEM_TSQR_REGS));
  const int by_smem = std::max(1, int((227 * 1024) / (tsqr_smem_bytes(n) + 1024)));
  return std::min(std::min(by_regs, by_smem), 2048 / t);
}
size_t tsqr_smem_bytes(int n) {
  return sizeof(double2) *
         (size_t(n) * (n + 1) / 2 + kSlots * size_t(tsqr_block_rows(n)) + kSlots);
}

template <int L, int T>
static void launch_variant(const QrTask* tasks, int n_tasks, size_t smem, cudaStream_t st) {
  static bool once = [] {
    cudaFuncSetAttribute(k_tsqr<L, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    return true;
  }();
  (void)once;
  k_tsqr<L, T><<<n_tasks, T, smem, st>>>(tasks);
}

void launch_tsqr(const QrTask* tasks, int n_tasks, int variant, size_t smem,
                 cudaStream_t st) {
  if (n_tasks <= 0) return;
  if (variant == 0)
    launch_variant<EBEM_TSQR_S_LANES, EBEM_TSQR_S_THREADS>(tasks, n_tasks, smem, st);
  else
    launch_variant<EBEM_TSQR_M_LANES, EBEM_TSQR_M_THREADS>(tasks, n_tasks, smem, st);
}

}  // namespace ebem_gpu
