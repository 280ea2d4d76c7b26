// Householder QR kernels of the skeletonization, "team" layout (sm_100a).
//
// One CTA (512 threads) per matrix block held in shared memory; the 512
// threads form 64 teams of 8 consecutive lanes and team t owns columns
// t, t+64, ...  Every Householder step needs only two block barriers: the
// owner team of column i generates the reflector (norm by an 8-lane shuffle
// reduction), then every team applies it to its own columns (8-lane dot
// products, update of the rows the same lanes read).  A team's 8 lanes read
// 8 consecutive rows = one 128-byte shared-memory wavefront.
//
//   k_qr_team    unpivoted QR of a row block -> R (TSQR reduction rounds)
//   k_cpqr_team  column-pivoted QR with LAPACK zlaqp2 pivoting and the
//                early stop at |R_ii| <= stop_rel |R_00|
//                (Cpqr, proj/src/lapack.cpp:101-138; zlaqp2 semantics:
//                first index of the largest partial norm, norm downdate
//                t = 1 - (|a_ij| / vn1_j)^2 with recomputation when
//                t (vn1_j / vn2_j)^2 <= sqrt(eps))
#include <cuda_runtime.h>

#include "ebem_dense.h"

namespace ebem_gpu {

namespace {

#ifndef EBEM_TEAM_THREADS
#define EBEM_TEAM_THREADS 256
#endif
#ifndef EBEM_TEAM_LANES
#define EBEM_TEAM_LANES 8
#endif
constexpr int kTeamThreads = EBEM_TEAM_THREADS;
constexpr int kTeamLanes = EBEM_TEAM_LANES;
constexpr int kTeams = kTeamThreads / kTeamLanes;  // 32 (256 x 8: CPQR 29.7 -> 27.5 ms at 2N = 2^19)

// The 8 lanes of this thread's team (teams of one warp may diverge).
__device__ __forceinline__ unsigned team_mask() {
  constexpr unsigned kLaneBits = (1u << kTeamLanes) - 1u;
  return kLaneBits << ((threadIdx.x & 31) & ~(kTeamLanes - 1));
}

__device__ __forceinline__ double team_sum(double v) {
  const unsigned mk = team_mask();
#pragma unroll
  for (int o = 1; o < kTeamLanes; o <<= 1) v += __shfl_xor_sync(mk, v, o);
  return v;
}

__device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__device__ __forceinline__ double2 zdiv(double2 a, double2 b) {
  if (fabs(b.x) >= fabs(b.y)) {
    const double r = b.y / b.x, d = b.x + b.y * r;
    return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
  }
  const double r = b.x / b.y, d = b.y + b.x * r;
  return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
}

struct HH {  // reflector broadcast
  double2 tau;
  double beta;
};

// Householder reflector of column i (rows i..m-1) by its owner team:
// zlarfg semantics (beta = -sign(Re alpha) ||(alpha, x)||, H = I when x = 0
// and Im alpha = 0).  Writes v below the diagonal, beta on it.
__device__ __forceinline__ void team_reflector(double2* __restrict__ c, int m,
                                               int i, int sub, HH* out) {
  double part = 0.0;
  for (int r = i + 1 + sub; r < m; r += kTeamLanes)
    part = fma(c[r].x, c[r].x, fma(c[r].y, c[r].y, part));
  const double xn2 = team_sum(part);
  const double2 alpha = c[i];
  double2 tau = make_double2(0.0, 0.0);
  double beta;
  if (xn2 == 0.0 && alpha.y == 0.0) {
    beta = alpha.x;
  } else {
    // zlarfg with reciprocals only (a true division with a zero numerator,
    // e.g. alpha.y = 0, takes the slow path); see make_reflector in
    // ebem_tsqr.cu for the scaled form of 1 / (alpha - beta)
    const double x2 = fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, xn2));
    const double s = rsqrt(x2);
    const bool pos = alpha.x >= 0.0;
    beta = pos ? -(x2 * s) : x2 * s;
    const double ib = pos ? -s : s;
    tau = make_double2((beta - alpha.x) * ib, -alpha.y * ib);
    const double arn = fma(alpha.x, s, pos ? 1.0 : -1.0);
    const double ain = alpha.y * s;
    const double id = s / fma(arn, arn, ain * ain);
    const double2 scal = make_double2(arn * id, -ain * id);
    for (int r = i + 1 + sub; r < m; r += kTeamLanes) c[r] = zmul(scal, c[r]);
  }
  __syncwarp(team_mask());
  if (sub == 0) {
    c[i] = make_double2(beta, 0.0);
    out->tau = tau;
    out->beta = beta;
  }
}

// Apply H^H = I - conj(tau) v v^H to column cj (rows i..m-1) by a team.
__device__ __forceinline__ void team_apply(const double2* __restrict__ v,
                                           double2* __restrict__ cj, int m, int i,
                                           int sub, double2 ctau) {
  double sx = 0.0, sy = 0.0;
  for (int r = i + sub; r < m; r += kTeamLanes) {
    const double2 vr = (r == i) ? make_double2(1.0, 0.0) : v[r];
    const double2 a = cj[r];
    // conj(v) * a
    sx = fma(vr.x, a.x, fma(vr.y, a.y, sx));
    sy = fma(vr.x, a.y, fma(-vr.y, a.x, sy));
  }
  sx = team_sum(sx);
  sy = team_sum(sy);
  const double2 f = zmul(ctau, make_double2(sx, sy));
  for (int r = i + sub; r < m; r += kTeamLanes) {
    const double2 vr = (r == i) ? make_double2(1.0, 0.0) : v[r];
    double2 a = cj[r];
    a.x = fma(-vr.x, f.x, fma(vr.y, f.y, a.x));
    a.y = fma(-vr.x, f.y, fma(-vr.y, f.x, a.y));
    cj[r] = a;
  }
}

__device__ void load_block(const double2* __restrict__ src, int m, int n, int ld,
                           double2* __restrict__ dst) {
  for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
    const int j = idx / m, i = idx - j * m;
    dst[idx] = src[(size_t)j * ld + i];
  }
}

}  // namespace

// The shared-memory and the global-workspace variants are separate
// instantiations so the shared one compiles to LDS/STS (a pointer that may
// point to either space forces generic loads).
template <bool kSmem>
__device__ __forceinline__ void qr_team_body(const QrTask& T, double2* __restrict__ A,
                                             HH& hh) {
  const int m = T.rows, n = T.n;
  load_block(reinterpret_cast<const double2*>(T.src), m, n, T.ld, A);
  __syncthreads();
  const int team = threadIdx.x / kTeamLanes, sub = threadIdx.x % kTeamLanes;
  const int steps = m < n ? m : n;
  for (int i = 0; i < steps; ++i) {
    if (team == (i % kTeams)) team_reflector(A + (size_t)i * m, m, i, sub, &hh);
    __syncthreads();
    const double2 ctau = make_double2(hh.tau.x, -hh.tau.y);
    if (ctau.x != 0.0 || ctau.y != 0.0) {
      const double2* v = A + (size_t)i * m;
      for (int j = team; j < n; j += kTeams)
        if (j > i) team_apply(v, A + (size_t)j * m, m, i, sub, ctau);
    }
    __syncthreads();
  }
  double2* R = reinterpret_cast<double2*>(T.dst);
  for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
    const int j = idx / n, i = idx - j * n;
    R[(size_t)j * T.dst_ld + i] = (i <= j && i < m) ? A[(size_t)j * m + i]
                                                    : make_double2(0.0, 0.0);
  }
}

__global__ void __launch_bounds__(kTeamThreads)
k_qr_team(const QrTask* __restrict__ tasks, double2* __restrict__ gws) {
  extern __shared__ double2 smem[];
  __shared__ HH hh;
  const QrTask T = tasks[blockIdx.x];
  if (T.in_smem) qr_team_body<true>(T, smem, hh);
  else qr_team_body<false>(T, gws + T.ws_off, hh);
}

struct CpqrShared {
  HH hh;
  double vn1[kMaxCpqrCols], vn2[kMaxCpqrCols];
  int jp[kMaxCpqrCols];
  int s_pvt;
  double s_r00;
};

template <bool kSmem>
__device__ __forceinline__ void cpqr_team_body(const CpqrTask& T, double2* __restrict__ A,
                                               CpqrShared& sh) {
  HH& hh = sh.hh;
  double* vn1 = sh.vn1;
  double* vn2 = sh.vn2;
  int* jp = sh.jp;
  int& s_pvt = sh.s_pvt;
  double& s_r00 = sh.s_r00;
  const int m = T.rows, n = T.n;
  load_block(reinterpret_cast<const double2*>(T.src), m, n, T.ld, A);
  for (int j = threadIdx.x; j < n; j += blockDim.x) jp[j] = j;
  __syncthreads();
  const int team = threadIdx.x / kTeamLanes, sub = threadIdx.x % kTeamLanes;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  // initial column norms (dznrm2 of every column)
  for (int j = team; j < n; j += kTeams) {
    const double2* c = A + (size_t)j * m;
    double s = 0.0;
    for (int r = sub; r < m; r += kTeamLanes) s = fma(c[r].x, c[r].x, fma(c[r].y, c[r].y, s));
    s = team_sum(s);
    if (sub == 0) vn1[j] = vn2[j] = sqrt(s);
  }
  __syncthreads();
  const double tol3z = 1.0536712127723509e-08;  // sqrt(2^-53)
  const int mn = m < n ? m : n;
  int steps = mn;
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
    // the step's team swaps the pivot column in and builds the reflector
    if (team == (i % kTeams)) {
      if (pvt != i) {
        double2* a = A + (size_t)pvt * m;
        double2* b = A + (size_t)i * m;
        for (int r = sub; r < m; r += kTeamLanes) {
          const double2 t = a[r];
          a[r] = b[r];
          b[r] = t;
        }
        if (sub == 0) {
          const int t = jp[pvt];
          jp[pvt] = jp[i];
          jp[i] = t;
          vn1[pvt] = vn1[i];
          vn2[pvt] = vn2[i];
        }
        __syncwarp(team_mask());
      }
      team_reflector(A + (size_t)i * m, m, i, sub, &hh);
      if (sub == 0) {
        const double r = fabs(hh.beta);
        T.rdiag[i] = r;
        if (i == 0) s_r00 = r;
      }
    }
    __syncthreads();
    const double rii = fabs(hh.beta);
    const double r00 = s_r00;
    if (r00 == 0.0 || rii <= T.stop_rel * r00) {
      steps = i;
      break;
    }
    const double2 ctau = make_double2(hh.tau.x, -hh.tau.y);
    const double2* v = A + (size_t)i * m;
    for (int j = team; j < n; j += kTeams) {
      if (j <= i) continue;
      double2* cj = A + (size_t)j * m;
      if (ctau.x != 0.0 || ctau.y != 0.0) team_apply(v, cj, m, i, sub, ctau);
      // partial norm downdate (zlaqp2), by the same team
      const double v1 = vn1[j];
      if (v1 == 0.0) continue;
      __syncwarp(team_mask());
      const double2 aij = cj[i];
      const double iv1 = 1.0 / v1;
      double temp = hypot(aij.x, aij.y) * iv1;
      temp = 1.0 - temp * temp;
      temp = temp > 0.0 ? temp : 0.0;
      const double ratio = v1 * (1.0 / vn2[j]);
      const double temp2 = temp * ratio * ratio;
      if (temp2 <= tol3z) {
        double s = 0.0;
        for (int r = i + 1 + sub; r < m; r += kTeamLanes)
          s = fma(cj[r].x, cj[r].x, fma(cj[r].y, cj[r].y, s));
        s = team_sum(s);
        if (sub == 0) vn1[j] = vn2[j] = (i + 1 < m) ? sqrt(s) : 0.0;
      } else {
        if (sub == 0) vn1[j] = v1 * sqrt(temp);
      }
    }
    __syncthreads();
  }
  for (int j = threadIdx.x; j < n; j += blockDim.x) T.jpvt[j] = jp[j];
  if (threadIdx.x == 0) *T.steps = steps;
  double2* R = reinterpret_cast<double2*>(T.r_out);
  for (int idx = threadIdx.x; idx < steps * n; idx += blockDim.x) {
    const int j = idx / steps, i = idx - j * steps;
    R[(size_t)j * T.r_ld + i] = (i <= j) ? A[(size_t)j * m + i] : make_double2(0.0, 0.0);
  }
}

__global__ void __launch_bounds__(kTeamThreads)
k_cpqr_team(const CpqrTask* __restrict__ tasks, double2* __restrict__ gws) {
  extern __shared__ double2 smem[];
  __shared__ CpqrShared sh;
  const CpqrTask T = tasks[blockIdx.x];
  if (T.in_smem) cpqr_team_body<true>(T, smem, sh);
  else cpqr_team_body<false>(T, gws + T.ws_off, sh);
}

void qr_team_init() {
  static bool done = false;
  if (done) return;
  cudaFuncSetAttribute((const void*)k_qr_team, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCap);
  cudaFuncSetAttribute((const void*)k_cpqr_team, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemCap);
  done = true;
}

void launch_qr_team(const QrTask* tasks, int n, size_t smem, double2* gws,
                    cudaStream_t st) {
  if (n <= 0) return;
  qr_team_init();
  k_qr_team<<<n, kTeamThreads, smem, st>>>(tasks, gws);
}

// Warp-per-matrix pivoted QR for blocks of at most 32 x 32 (the leaf
// level's reduced ID inputs): lane j holds column j in registers, so a step
// needs no barrier -- the pivot is a shuffle argmax, the column swap and the
// reflector broadcast are shuffles, and every lane updates its own column.
// Same zlaqp2 decisions and zlarfg arithmetic as cpqr_team_body (the sums
// run in row order here, so partial norms may differ in the last bit).
constexpr int kCpqrWarps = 4;  // matrices per CTA
__global__ void __launch_bounds__(kCpqrWarps * 32)
k_cpqr_warp(const CpqrTask* __restrict__ tasks, int n_tasks) {
  const int task = blockIdx.x * kCpqrWarps + (threadIdx.x >> 5);
  if (task >= n_tasks) return;
  const int l = threadIdx.x & 31;
  const CpqrTask T = tasks[task];
  const int m = T.rows, n = T.n;
  const bool own = l < n;
  const double2* src = reinterpret_cast<const double2*>(T.src) + (size_t)l * T.ld;
  double2 c[32];
#pragma unroll
  for (int r = 0; r < 32; ++r) c[r] = (own && r < m) ? src[r] : make_double2(0.0, 0.0);
  double vn1 = 0.0;
#pragma unroll
  for (int r = 0; r < 32; ++r) vn1 = fma(c[r].x, c[r].x, fma(c[r].y, c[r].y, vn1));
  vn1 = own ? sqrt(vn1) : -1.0;
  double vn2 = vn1;
  int jp = l;
  const double tol3z = 1.0536712127723509e-08;  // sqrt(2^-53)
  const int mn = m < n ? m : n;
  int steps = mn;
  double r00 = 0.0;
  for (int i = 0; i < mn; ++i) {
    // pivot: first index of the largest partial norm among columns >= i
    double best = l >= i ? vn1 : -2.0;
    int bi = l;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const int pvt = bi;
    if (pvt != i) {  // swap columns i and pvt; vn of pvt takes i's (zlaqp2)
      const int from = l == i ? pvt : (l == pvt ? i : l);
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        c[r].x = __shfl_sync(0xffffffffu, c[r].x, from);
        c[r].y = __shfl_sync(0xffffffffu, c[r].y, from);
      }
      jp = __shfl_sync(0xffffffffu, jp, from);
      const double a1 = __shfl_sync(0xffffffffu, vn1, i);
      const double a2 = __shfl_sync(0xffffffffu, vn2, i);
      if (l == pvt) { vn1 = a1; vn2 = a2; }
    }
    // reflector of column i (zlarfg, the arithmetic of team_reflector)
    double2 tau = make_double2(0.0, 0.0);
    double beta = 0.0;
    if (l == i) {
      double xn2 = 0.0;
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (r > i && r < m) xn2 = fma(c[r].x, c[r].x, fma(c[r].y, c[r].y, xn2));
      double2 alpha = make_double2(0.0, 0.0);
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (r == i) alpha = c[r];
      if (xn2 == 0.0 && alpha.y == 0.0) {
        beta = alpha.x;
      } else {
        const double x2 = fma(alpha.x, alpha.x, fma(alpha.y, alpha.y, xn2));
        const double sr = rsqrt(x2);
        const bool pos = alpha.x >= 0.0;
        beta = pos ? -(x2 * sr) : x2 * sr;
        const double ib = pos ? -sr : sr;
        tau = make_double2((beta - alpha.x) * ib, -alpha.y * ib);
        const double arn = fma(alpha.x, sr, pos ? 1.0 : -1.0);
        const double ain = alpha.y * sr;
        const double id = sr / fma(arn, arn, ain * ain);
        const double2 scal = make_double2(arn * id, -ain * id);
#pragma unroll
        for (int r = 0; r < 32; ++r)
          if (r > i && r < m) c[r] = zmul(scal, c[r]);
      }
#pragma unroll
      for (int r = 0; r < 32; ++r)
        if (r == i) c[r] = make_double2(beta, 0.0);
    }
    beta = __shfl_sync(0xffffffffu, beta, i);
    tau.x = __shfl_sync(0xffffffffu, tau.x, i);
    tau.y = __shfl_sync(0xffffffffu, tau.y, i);
    const double rii = fabs(beta);
    if (l == 0) T.rdiag[i] = rii;
    if (i == 0) r00 = rii;
    if (r00 == 0.0 || rii <= T.stop_rel * r00) {
      steps = i;
      break;
    }
    // apply H^H = I - conj(tau) v v^H to the columns right of i
    // v (lane i's column below the diagonal) is broadcast row by row in
    // both passes; lane i's registers are not modified by this step
    const double2 ctau = make_double2(tau.x, -tau.y);
    const bool apply = ctau.x != 0.0 || ctau.y != 0.0;  // warp-uniform
    if (apply) {
      double sx = 0.0, sy = 0.0;
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        if (r < i || r >= m) continue;
        double2 vr = make_double2(__shfl_sync(0xffffffffu, c[r].x, i),
                                  __shfl_sync(0xffffffffu, c[r].y, i));
        if (r == i) vr = make_double2(1.0, 0.0);
        sx = fma(vr.x, c[r].x, fma(vr.y, c[r].y, sx));
        sy = fma(vr.x, c[r].y, fma(-vr.y, c[r].x, sy));
      }
      const double2 f = zmul(ctau, make_double2(sx, sy));
#pragma unroll
      for (int r = 0; r < 32; ++r) {
        if (r < i || r >= m) continue;
        double2 vr = make_double2(__shfl_sync(0xffffffffu, c[r].x, i),
                                  __shfl_sync(0xffffffffu, c[r].y, i));
        if (r == i) vr = make_double2(1.0, 0.0);
        if (own && l > i) {
          c[r].x = fma(-vr.x, f.x, fma(vr.y, f.y, c[r].x));
          c[r].y = fma(-vr.x, f.y, fma(-vr.y, f.x, c[r].y));
        }
      }
    }
    if (own && l > i) {
      // partial norm downdate (zlaqp2)
      if (vn1 != 0.0) {
        double2 aij = make_double2(0.0, 0.0);
#pragma unroll
        for (int r = 0; r < 32; ++r)
          if (r == i) aij = c[r];
        const double iv1 = 1.0 / vn1;
        double temp = hypot(aij.x, aij.y) * iv1;
        temp = 1.0 - temp * temp;
        temp = temp > 0.0 ? temp : 0.0;
        const double ratio = vn1 * (1.0 / vn2);
        const double temp2 = temp * ratio * ratio;
        if (temp2 <= tol3z) {
          double s2 = 0.0;
#pragma unroll
          for (int r = 0; r < 32; ++r)
            if (r > i && r < m) s2 = fma(c[r].x, c[r].x, fma(c[r].y, c[r].y, s2));
          vn1 = vn2 = (i + 1 < m) ? sqrt(s2) : 0.0;
        } else {
          vn1 = vn1 * sqrt(temp);
        }
      }
    }
  }
  if (own) T.jpvt[l] = jp;
  if (l == 0) *T.steps = steps;
  if (own) {
    double2* R = reinterpret_cast<double2*>(T.r_out) + (size_t)l * T.r_ld;
#pragma unroll
    for (int r = 0; r < 32; ++r)
      if (r < steps) R[r] = (r <= l) ? c[r] : make_double2(0.0, 0.0);
  }
}

void launch_cpqr_warp(const CpqrTask* tasks, int n, cudaStream_t st) {
  if (n <= 0) return;
  k_cpqr_warp<<<(n + kCpqrWarps - 1) / kCpqrWarps, kCpqrWarps * 32, 0, st>>>(tasks, n);
}

void launch_cpqr_team(const CpqrTask* tasks, int n, size_t smem, double2* gws,
                      cudaStream_t st) {
  if (n <= 0) return;
  qr_team_init();
  k_cpqr_team<<<n, kTeamThreads, smem, st>>>(tasks, gws);
}

}  // namespace ebem_gpu
