// Galerkin fill kernels (sm_100a, FP64):
//   k_proxy_pairs     proxy polygon <-> curve element pairs, n_g x n_g Gauss,
//                     full kernel, both orientations from one scalar
//                     evaluation (kernel_cross_block, proj/src/assembly.cpp:424-509)
//   k_sym_count       quadrature-tier class of every near element pair + counts
//   k_sym_scatter     per-pair records written straight into their class ranges
//   k_near_sym        separated element pairs, tiered tensor Gauss with the
//                     static hypersingular part integrated by parts
//                     (PairIntegrator::separated, proj/src/assembly.cpp:248-286);
//                     both near blocks of a cell from one evaluation, or one
//                     orientation for plain true blocks
//   k_near_singular   coincident (closed form + integrated series) and
//                     adjacent (Duffy) pairs (proj/src/assembly.cpp:70-246)
//   k_gather          ordered scatter of bundles into output blocks
//                     (proj/src/assembly.cpp:373-407, :493-506)
#include <stdexcept>
#include <cstdlib>
#include <cuda_runtime.h>

#include <algorithm>

#include "ebem_device.cuh"
#include "ebem_jobs.h"
#include "ebem_kernels.h"

namespace ebem_gpu {

namespace {

__device__ __forceinline__ double ef(const DevCtx* __restrict__ c, int f, int e) {
  return __ldg(c->elem + size_t(f) * c->n_nodes + e);
}

// Largest j in [0, n) with off[j] <= x (off ascending, off[0] == 0).
template <class T>
__device__ __forceinline__ int find_job(const T* __restrict__ off, int n, T x) {
  int lo = 0, hi = n - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (__ldg(off + mid) <= x) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ double pt_seg_dist(double px, double py, double ax,
                                              double ay, double bx, double by) {
  const double abx = bx - ax, aby = by - ay;
  const double len2 = abx * abx + aby * aby;
  double t = len2 > 0.0 ? ((px - ax) * abx + (py - ay) * aby) / len2 : 0.0;
  t = fmin(fmax(t, 0.0), 1.0);
  return hypot(px - (ax + t * abx), py - (ay + t * aby));
}

// Element geometry from the element-major copy: g = {px, py, dx, dy, nx, ny, h, 0}.
struct Elem8 {
  double px, py, dx, dy, nx, ny, h;
};
__device__ __forceinline__ Elem8 load_elem8(const DevCtx* __restrict__ c, int e) {
  const double2* p = reinterpret_cast<const double2*>(c->elem8) + 4 * (long long)e;
  const double2 a = __ldg(p), b = __ldg(p + 1), d = __ldg(p + 2), h = __ldg(p + 3);
  return Elem8{a.x, a.y, b.x, b.y, d.x, d.y, h.x};
}

// Mesh::element_distance, proj/src/geometry.cpp:83-96, on loaded geometry.
__device__ __forceinline__ double element_distance8(const Elem8& A, const Elem8& B) {
  const double a0x = A.px, a0y = A.py;
  const double a1x = a0x + A.dx, a1y = a0y + A.dy;
  const double b0x = B.px, b0y = B.py;
  const double b1x = b0x + B.dx, b1y = b0y + B.dy;
  double d = pt_seg_dist(a0x, a0y, b0x, b0y, b1x, b1y);
  d = fmin(d, pt_seg_dist(a1x, a1y, b0x, b0y, b1x, b1y));
  d = fmin(d, pt_seg_dist(b0x, b0y, a0x, a0y, a1x, a1y));
  d = fmin(d, pt_seg_dist(b1x, b1y, a0x, a0y, a1x, a1y));
  return d;
}

// tier_nodes, proj/src/assembly.cpp:27-38.
__device__ __forceinline__ int tier_nodes(double q, int far, double refine) {
  int n = far;
  if (q >= 8.0) {
  } else if (q >= 4.0) {
    n += 2;
  } else if (q >= 2.0) {
    n += 5;
  } else {
    n += 9;
  }
  return int(n * refine + 0.5);
}

// Bundle storage, component-plane major: entry k = bidx(la, lb, i, j) of
// slot p lives at ((i, j) plane) * 4 nb + 4 p + (la, lb), so the gather of one
// component block reads a slot's four shape entries as one 64-byte chunk.
__device__ __forceinline__ long long bslot(long long p, int k, long long nb) {
  return (long long)(k & 3) * nb * 4 + p * 4 + (k >> 2);
}

__device__ __forceinline__ void store_bundle(double* __restrict__ out, long long p,
                                             const cplx (&v)[kBundle], long long nb) {
  double2* o = reinterpret_cast<double2*>(out);
#pragma unroll
  for (int k = 0; k < kBundle; ++k) o[bslot(p, k, nb)] = make_double2(v[k].re, v[k].im);
}

// bundle index: ((la * 2 + lb) * 2 + i) * 2 + j
__device__ __forceinline__ int bidx(int la, int lb, int i, int j) {
  return ((la * 2 + lb) * 2 + i) * 2 + j;
}

}  // namespace

// ---------------------------------------------------------------- singular
namespace {

// The four integrated remainders of a coincident pair (weights u^0 .. u^3,
// proj/src/kernel_scalars.cpp:333-344), only the scalars the bundle uses,
// with the series terms split over the warp's lanes (lane l: powers l,
// l + 32) and summed in a fixed butterfly order.  Call with all 32 lanes.
struct CoincRem {
  cplx n0[5], n1[5], n3[5];  // u^0, u^1, u^3: n1 n2 n4 n5 n7
  cplx d1[2], d2[2];         // u^1, u^2: d1 d2
};
__device__ __forceinline__ void coincident_remainders(const DevCtx* __restrict__ ctx,
                                                      double scale, int lane,
                                                      CoincRem& o, int* bad) {
  if (lane == 0 && !(ctx->med.kT * scale < 2.5)) atomicExch(bad, 1);
  const double logc = log(scale);
  const int maxq = series_maxq_at(ctx, scale);
  double acc[38];
#pragma unroll
  for (int k = 0; k < 38; ++k) acc[k] = 0.0;
  for (int q = lane; q <= maxq; q += 32) {
    // c^q by squaring (deterministic per q)
    double cq = 1.0, base = scale;
    for (int e = q; e > 0; e >>= 1) {
      if (e & 1) cq *= base;
      base *= base;
    }
    auto term = [&](int k, int upow, double* dst) {
      const double4 c = ld_series(ctx, k, q);
      const double inv = 1.0 / double(q + upow + 1), inv2 = inv * inv;
      dst[0] = fma(cq, fma(c.z, logc, c.x) * inv - c.z * inv2, dst[0]);
      dst[1] = fma(cq, fma(c.w, logc, c.y) * inv - c.w * inv2, dst[1]);
    };
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      term(5 + k, 0, acc + 2 * k);
      term(5 + k, 1, acc + 10 + 2 * k);
      term(5 + k, 3, acc + 20 + 2 * k);
    }
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      term(2 + k, 1, acc + 30 + 2 * k);
      term(2 + k, 2, acc + 34 + 2 * k);
    }
  }
#pragma unroll
  for (int k = 0; k < 38; ++k)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    o.n0[k] = mk(acc[2 * k], acc[2 * k + 1]);
    o.n1[k] = mk(acc[10 + 2 * k], acc[10 + 2 * k + 1]);
    o.n3[k] = mk(acc[20 + 2 * k], acc[20 + 2 * k + 1]);
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    o.d1[k] = mk(acc[30 + 2 * k], acc[30 + 2 * k + 1]);
    o.d2[k] = mk(acc[34 + 2 * k], acc[34 + 2 * k + 1]);
  }
}

__device__ void coincident_bundle(const DevCtx* __restrict__ ctx, int e,
                                  cplx (&v)[kBundle], int* bad, int lane) {
  const double h = ef(ctx, EH, e);
  CoincRem rm;
  coincident_remainders(ctx, h, lane, rm, bad);
  if (lane != 0) return;
  const double tx = ef(ctx, ETX, e), ty = ef(ctx, ETY, e);
  const double nx = ef(ctx, ENX, e), ny = ef(ctx, ENY, e);
  const double logh = log(h);
  const double qfac = ctx->med.qfactor;
  const double kappa = ctx->med.kappa;
  const cplx alpha = mk(ctx->med.alpha_re, ctx->med.alpha_im);
  cplx D[kBundle], Nn[kBundle];
#pragma unroll
  for (int k = 0; k < kBundle; ++k) D[k] = Nn[k] = mk(0.0, 0.0);
  const double M[2][2] = {{h / 3.0, h / 6.0}, {h / 6.0, h / 3.0}};

  // traction, static: principal values -+ 1/2 on the off-diagonal shapes
  const double dcoef = 0.5 * kappa * h;
  D[bidx(0, 1, 0, 1)] += mk(dcoef);
  D[bidx(0, 1, 1, 0)] += mk(-dcoef);
  D[bidx(1, 0, 0, 1)] += mk(-dcoef);
  D[bidx(1, 0, 1, 0)] += mk(dcoef);

  const cplx i1 = rm.d2[0] - rm.d1[0];
  const cplx i2 = rm.d2[1] - rm.d1[1];
  const double h2 = h * h;
  const double tv[2] = {tx, ty}, nv[2] = {nx, ny};
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const cplx val = (-h2) * (i1 * (tv[i] * nv[j]) + i2 * (nv[i] * tv[j]));
      D[bidx(0, 1, i, j)] += val;
      D[bidx(1, 0, i, j)] -= val;
    }
// hypersingular, static part by parts
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      const double sgn = (a == b) ? 1.0 : -1.0;
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const double dij = (i == j) ? 1.0 : 0.0;
          Nn[bidx(a, b, i, j)] += mk(sgn * qfac * ((logh - 1.5) * dij - tv[i] * tv[j]));
        }
    }
  // hypersingular remainder: even reduction weights (n scalars only:
  // combine_N reads s[5..9])
  Scalars sdiag, soff;
#pragma unroll
  for (int k = 0; k < 10; ++k) sdiag.s[k] = soff.s[k] = mk(0.0);
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    sdiag.s[5 + k] = rm.n3[k] / 3.0 - rm.n1[k] + (2.0 * rm.n0[k]) / 3.0;
    soff.s[5 + k] = (rm.n0[k] - rm.n3[k]) / 3.0;
  }
  CMat2 nd, no;
  combine_N(sdiag, tx, ty, nx, ny, nx, ny, nd);
  combine_N(soff, tx, ty, nx, ny, nx, ny, no);
#pragma unroll
  for (int e4 = 0; e4 < 4; ++e4) {
    Nn[bidx(0, 0, 0, 0) + e4] += h2 * nd.a[e4];
    Nn[bidx(1, 1, 0, 0) + e4] += h2 * nd.a[e4];
    Nn[bidx(0, 1, 0, 0) + e4] += h2 * no.a[e4];
    Nn[bidx(1, 0, 0, 0) + e4] += h2 * no.a[e4];
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int k = bidx(a, b, i, j);
          cplx val = D[k] + alpha * Nn[k];
          if (i == j) val.re += 0.5 * M[a][b];
          v[k] = val;
        }
}

// Points p = part, part + nparts, ... of the 2 n corner-rule points (both
// Duffy triangles); the caller sums the parts.
__device__ void adjacent_bundle(const DevCtx* __restrict__ ctx, int ea, int eb,
                                bool end_start, cplx (&v)[kBundle], int* bad,
                                int part = 0, int nparts = 1) {
  const double hx = ef(ctx, EH, ea), hy = ef(ctx, EH, eb);
  double txx, txy, tyx, tyy;
  double bx0[2], bx1[2], by0[2], by1[2];
  if (end_start) {
    txx = -ef(ctx, ETX, ea); txy = -ef(ctx, ETY, ea);
    bx0[0] = 0.0; bx1[0] = 1.0; bx0[1] = 1.0; bx1[1] = -1.0;
    tyx = ef(ctx, ETX, eb); tyy = ef(ctx, ETY, eb);
    by0[0] = 1.0; by1[0] = -1.0; by0[1] = 0.0; by1[1] = 1.0;
  } else {
    txx = ef(ctx, ETX, ea); txy = ef(ctx, ETY, ea);
    bx0[0] = 1.0; bx1[0] = -1.0; bx0[1] = 0.0; bx1[1] = 1.0;
    tyx = -ef(ctx, ETX, eb); tyy = -ef(ctx, ETY, eb);
    by0[0] = 0.0; by1[0] = 1.0; by0[1] = 1.0; by1[1] = -1.0;
  }
  const double nxx = ef(ctx, ENX, ea), nxy = ef(ctx, ENY, ea);
  const double nyx = ef(ctx, ENX, eb), nyy = ef(ctx, ENY, eb);
  const double qfac = ctx->med.qfactor;
  const double hxy = hx * hy;
  const cplx alpha = mk(ctx->med.alpha_re, ctx->med.alpha_im);
  Scalars dhat;
#pragma unroll
  for (int k = 0; k < 10; ++k) dhat.s[k] = mk(0.0);
  dhat.s[2] = mk(ctx->med.kappa);
  dhat.s[3] = mk(-ctx->med.kappa);
  dhat.s[4] = mk(-8.0 * ctx->med.ccon);

  cplx acc[kBundle];
#pragma unroll
  for (int k = 0; k < kBundle; ++k) acc[k] = mk(0.0);
  const int n = ctx->corner_n;
  const double* gx = ctx->gx + gauss_offset(n);
  const double* gw = ctx->gw + gauss_offset(n);
  for (int pt = part; pt < 2 * n; pt += nparts) {
    const int tri = pt >= n ? 1 : 0;
    const int wi = pt - tri * n;
    {
      const double w = gx[wi];
      const double wt = gw[wi];
      double zvx, zvy;
      if (tri == 0) {
        zvx = hx * txx - (w * hy) * tyx;
        zvy = hx * txy - (w * hy) * tyy;
      } else {
        zvx = (w * hx) * txx - hy * tyx;
        zvy = (w * hx) * txy - hy * tyy;
      }
      const double g = hypot(zvx, zvy);
      const double ig = 1.0 / g;
      const double zhx = ig * zvx, zhy = ig * zvy;
      const double logg = log(g);
      CMat2 dmat[3], nmat[3];
      {
        Scalars s3[3];
        integrated_remainder3(ctx, g, s3, bad);
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          combine_D(s3[j], zhx, zhy, nyx, nyy, dmat[j]);
          combine_N(s3[j], zhx, zhy, nxx, nxy, nyx, nyy, nmat[j]);
        }
      }
      CMat2 dstat;
      combine_D(dhat, zhx, zhy, nyx, nyy, dstat);
      const double ql = qfac * (logg * 0.5 - 0.25);
      const double qz = qfac * 0.5;
      const double qm[4] = {ql - qz * zhx * zhx, -qz * zhx * zhy,
                            -qz * zhy * zhx, ql - qz * zhy * zhy};
#pragma unroll
      for (int a = 0; a < 2; ++a) {
#pragma unroll
        for (int b = 0; b < 2; ++b) {
          const double t0 = bx0[a], u0 = by0[b];
          const double t1 = (tri == 0) ? bx1[a] : bx1[a] * w;
          const double u1 = (tri == 0) ? by1[b] * w : by1[b];
          const double c[3] = {t0 * u0, t0 * u1 + t1 * u0, t1 * u1};
          const double cint = c[0] / 1.0 + c[1] / 2.0 + c[2] / 3.0;
          const double fs = wt * hxy * cint / g;
          const double sgn = (a == b) ? 1.0 : -1.0;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            cplx d = fs * dstat.a[e];
            cplx nn = mk(wt * sgn * qm[e]);
#pragma unroll
            for (int j = 0; j < 3; ++j) {
              const double f = wt * hxy * c[j];
              axpy(d, f, dmat[j].a[e]);
              axpy(nn, f, nmat[j].a[e]);
            }
            acc[(a * 2 + b) * 4 + e] += d + alpha * nn;
          }
        }
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kBundle; ++k) v[k] = acc[k];
}

}  // namespace

// One warp per touching pair: the adjacent (Duffy) rule's points are split
// over the lanes and summed in a fixed butterfly order; a coincident pair
// (one closed form plus four 1-D series integrals) is done by lane 0.
__global__ void __launch_bounds__(128)
k_near_singular(const DevCtx* __restrict__ ctx, const long long* __restrict__ pairs,
                const int* __restrict__ pair_elems, int n, double* __restrict__ bundles,
                long long nb, int* bad) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= n) return;  // warp-uniform
  const int ea = pair_elems[2 * t], eb = pair_elems[2 * t + 1];
  const int N = ctx->n_nodes;
  cplx v[kBundle];
  if (ea == eb) {
    coincident_bundle(ctx, ea, v, bad, lane);  // all lanes: split series sums
    if (lane == 0) store_bundle(bundles, pairs[t], v, nb);
    return;
  }
  const bool end_start = (ea + 1 == N ? 0 : ea + 1) == eb;
  adjacent_bundle(ctx, ea, eb, end_start, v, bad, lane, 32);
#pragma unroll
  for (int k = 0; k < kBundle; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      v[k].re += __shfl_xor_sync(0xffffffffu, v[k].re, o);
      v[k].im += __shfl_xor_sync(0xffffffffu, v[k].im, o);
    }
  if (lane < kBundle) {
    cplx mine = v[0];
#pragma unroll
    for (int k = 1; k < kBundle; ++k)
      if (lane == k) mine = v[k];
    reinterpret_cast<double2*>(bundles)[bslot(pairs[t], lane, nb)] =
        make_double2(mine.re, mine.im);
  }
}

// ------------------------------------------------------- symmetric near
// Bucketing of the symmetric near pairs by quadrature class (kSymClasses,
// ebem_jobs.h) as a two-pass count-and-scatter: pass 1 classifies every pair
// and counts the classes, pass 2 writes each non-skipped pair's record
// straight into its class range.  Within a CTA the pairs of one class keep
// their pair order (warp ballots + a per-warp prefix), so consecutive records
// still address consecutive bundle slots; one global atomic per class per CTA.
constexpr int kBucketThreads = 256;
// counts / cursors live after the bounds in the same small device array
constexpr int kBoundsCounts = 16, kBoundsCursors = 32, kBoundsInts = 48;

__global__ void __launch_bounds__(kBucketThreads)
k_sym_count(const DevCtx* __restrict__ ctx, const SymJob* __restrict__ jobs,
            const long long* __restrict__ job_off, int n_jobs,
            const int* __restrict__ elems, long long n_pairs,
            unsigned char* __restrict__ keys, int* __restrict__ pair_job,
            int* __restrict__ bounds) {
  __shared__ int s_cnt[kSymClasses];
  if (threadIdx.x < kSymClasses) s_cnt[threadIdx.x] = 0;
  __syncthreads();
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (p < n_pairs) {
    const int jb = find_job(job_off, n_jobs, p);
    const SymJob J = jobs[jb];
    const long long local = p - J.local_off;
    const int a = int(local / J.nE);
    const int q = int(local - (long long)a * J.nE);
    const int ea = __ldg(elems + J.a_off + a);
    const int eb = __ldg(elems + J.e_off + q);
    const int N = ctx->n_nodes;
    const int na = ea + 1 == N ? 0 : ea + 1;
    const int nb = eb + 1 == N ? 0 : eb + 1;
    unsigned char key = kSymClasses - 1;  // skip
    if (!(ea == eb || na == eb || nb == ea) && !(J.tri && a >= q)) {
      const Elem8 A = load_elem8(ctx, ea), B = load_elem8(ctx, eb);
      // most pairs are far (tier 0): the midpoint distance minus the two
      // half-lengths bounds the segment distance from below, so a pair whose
      // bound clears 8 h_max (with a 1e-9 relative margin for rounding) is
      // tier 0 without the four point-segment distances
      const double hmax = fmax(A.h, B.h);
      const double cx = (A.px + 0.5 * A.dx) - (B.px + 0.5 * B.dx);
      const double cy = (A.py + 0.5 * A.dy) - (B.py + 0.5 * B.dy);
      const double thr = 8.0 * hmax * (1.0 + 1e-9) + 0.5 * (A.h + B.h) * (1.0 + 1e-9);
      int tier = 0;
      const double c2 = fma(cx, cx, cy * cy);
      if (c2 < thr * thr) {
        const double rq = element_distance8(A, B) / hmax;
        tier = rq >= 8.0 ? 0 : rq >= 4.0 ? 1 : rq >= 2.0 ? 2 : 3;
      } else if (ctx->very_far_tier) {
        // the same lower bound on the segment distance, against kVeryFar h_max
        const double vf = kVeryFar * hmax + 0.5 * (A.h + B.h);
        if (c2 >= vf * vf) tier = 4;
      }
      key = tier + (J.onesided ? kSymTiers : 0);
    }
    keys[p] = key;
    pair_job[p] = jb;  // read back by the scatter pass (no second search)
    atomicAdd(&s_cnt[key], 1);
  }
  __syncthreads();
  if (threadIdx.x < kSymClasses && s_cnt[threadIdx.x])
    atomicAdd(bounds + kBoundsCounts + threadIdx.x, s_cnt[threadIdx.x]);
}

// One record per non-skipped near pair, at bounds[class] + its rank: the
// element geometry and output slots the near-field kernel needs, laid out so
// one CTA stages a whole group of pairs with contiguous async copies (no
// dependent index chain on the compute kernel's critical path).  CTA 0 also
// publishes the class bounds (exclusive prefix of the counts, bounds[9] = n).
__global__ void __launch_bounds__(kBucketThreads)
k_sym_scatter(const DevCtx* __restrict__ ctx, const SymJob* __restrict__ jobs,
              const int* __restrict__ elems, const unsigned char* __restrict__ keys,
              const int* __restrict__ pair_job, long long n_pairs,
              int* __restrict__ bounds, double* __restrict__ recs) {
  constexpr int kWarps = kBucketThreads / 32;
  __shared__ int s_start[kSymClasses];       // class starts (prefix of counts)
  __shared__ int s_wcnt[kWarps][kSymClasses];
  __shared__ int s_base[kSymClasses];
  constexpr int kRecPad = kSymRec / 2 + 1;  // 144-byte rows: conflict-free 16-byte stores
  __shared__ double2 s_rec[kWarps * 32 * kRecPad];
  __shared__ long long s_idx[kWarps][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    int s = 0;
    for (int c = 0; c < kSymClasses; ++c) {
      s_start[c] = s;
      if (blockIdx.x == 0) bounds[c] = s;
      s += bounds[kBoundsCounts + c];
    }
    if (blockIdx.x == 0) bounds[kSymClasses] = s;
  }
  const long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int key = p < n_pairs ? int(__ldg(keys + p)) : kSymClasses - 1;
  // per-warp ranks of each lane within its class (pair order kept)
  const unsigned same = __match_any_sync(0xffffffffu, key);
  const int rank = __popc(same & ((1u << lane) - 1u));
  if (lane < kSymClasses) s_wcnt[warp][lane] = 0;
  __syncwarp();
  if (rank == 0) s_wcnt[warp][key] = __popc(same);
  __syncthreads();
  if (threadIdx.x < kSymClasses - 1) {  // the skip class gets no records
    const int c = threadIdx.x;
    int tot = 0;
    for (int w = 0; w < kWarps; ++w) {
      const int v = s_wcnt[w][c];
      s_wcnt[w][c] = tot;
      tot += v;
    }
    s_base[c] = tot ? s_start[c] + atomicAdd(bounds + kBoundsCursors + c, tot) : 0;
  }
  __syncthreads();
  // records go through shared memory so that each store instruction writes
  // 512 contiguous bytes (a warp's records of one class are contiguous)
  double2* const wrec = s_rec + warp * (32 * kRecPad);
  if (key != kSymClasses - 1) {
    const long long idx = (long long)s_base[key] + s_wcnt[warp][key] + rank;
    const SymJob J = jobs[__ldg(pair_job + p)];
    const long long local = p - J.local_off;
    const int a = int(local / J.nE);
    const int q = int(local - (long long)a * J.nE);
    const int ea = __ldg(elems + J.a_off + a);
    const int eb = __ldg(elems + J.e_off + q);
    const Elem8 A = load_elem8(ctx, ea), B = load_elem8(ctx, eb);
    double r[kSymRec] = {A.px, A.py, A.dx, A.dy, A.nx, A.ny,
                         B.px, B.py, B.dx, B.dy, B.nx, B.ny};
    r[SR_VD] = __longlong_as_double(J.v_off + local);
    r[SR_UD] = __longlong_as_double(J.u_off + (long long)q * J.nA + a);
    r[SR_HH] = A.h * B.h;
    r[15] = 0.0;
#pragma unroll
    for (int k = 0; k < kSymRec / 2; ++k)
      wrec[lane * kRecPad + k] = make_double2(r[2 * k], r[2 * k + 1]);
    s_idx[warp][lane] = idx;
  } else {
    s_idx[warp][lane] = -1;
  }
  __syncwarp();
  double2* const o = reinterpret_cast<double2*>(recs);
#pragma unroll
  for (int c = lane; c < 32 * (kSymRec / 2); c += 32) {
    const int rr = c / (kSymRec / 2), piece = c - rr * (kSymRec / 2);
    const long long idx = s_idx[warp][rr];
    if (idx >= 0) o[idx * (kSymRec / 2) + piece] = wrec[rr * kRecPad + piece];
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n"); }
__device__ __forceinline__ void cp_async_wait1() {
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
}

// r = |z|, 1/r and ln r of one quadrature point.  EBEM_FAST_R: from
// r^2 = zx^2 + zy^2 by one reciprocal square root (ln r = ln(r^2) / 2)
// instead of the overflow-safe hypot, a true division and ln r: the same
// accuracy (a few ulp) at fewer instructions; the points never come near
// the under/overflow range hypot guards against (r ~ h .. diam of the curve).
#ifndef EBEM_FAST_R
#define EBEM_FAST_R 1
#endif
__device__ __forceinline__ void point_radius(double zx, double zy, double& r, double& ir,
                                             double& logr) {
#if EBEM_FAST_R
  const double r2 = fma(zx, zx, zy * zy);
  ir = rsqrt(r2);
  r = r2 * ir;
  logr = 0.5 * log(r2);
#else
  r = hypot(zx, zy);
  ir = 1.0 / r;
  logr = log(r);
#endif
}

// CTA = P pairs x n threads; thread (pair, i) fixes the test point s_i on the
// enclosed element and sweeps the n points on the cell element, evaluating
// the scalars once for both orientations (r is symmetric).  The records of
// the next pair group are copied into shared memory (cp.async) while the
// current group is evaluated.
// Small CTAs (measured at 2N = 2^19: 256 x 1 -> 64 x 4 saves 5 % of the
// near-field time; the CTA barrier then couples 2 warps, not 8); 254
// registers either way, 8 warps per SM.
#ifndef EBEM_SYM_THREADS
#define EBEM_SYM_THREADS 64
#endif
#ifndef EBEM_SYM_MINB
#define EBEM_SYM_MINB 4
#endif
#ifndef EBEM_PRX_THREADS
#define EBEM_PRX_THREADS 128
#endif
#ifndef EBEM_PRX_MINB
#define EBEM_PRX_MINB 2
#endif
// PROXY: the proxy blocks (kernel_cross_block, assembly.cpp:424-509) — full
// n scalars, no static hypersingular part, records with a negative V slot
// are padding.
#ifndef EBEM_J_UNROLL
#define EBEM_J_UNROLL 1
#endif
constexpr int kJUnroll = EBEM_J_UNROLL;  // trial-point loop unroll (experiments)
template <bool BOTH, bool PROXY>
__device__ __forceinline__ void near_body(const DevCtx* __restrict__ ctx, const FillConst& fc,
                                          const double* __restrict__ recs, int first,
                                          int count, int n, double* __restrict__ bundles,
                                          long long nb) {
  // dynamic: [P * n][8 V + 8 U cplx + 2 (Q as re/im pairs)], then the two
  // record buffers [2][P][kSymRec]
  extern __shared__ double2 sh[];
  __shared__ SerSm S;
  __shared__ double sgx[kMaxGauss], sgw[kMaxGauss];
  const int P = blockDim.x / n;
  if ((int)blockIdx.x * P >= count) return;  // uniform per CTA
  double* const s_rec = reinterpret_cast<double*>(sh + blockDim.x * 18);  // [2][P][rec]
  const double* __restrict__ crec = recs + (long long)first * kSymRec;
  // stage the records of the group starting at pair g (16 B per copy)
  auto stage = [&](int g, int buf) {
    const int np = min(P, count - g);
    const double* src = crec + (long long)g * kSymRec;
    for (int c = threadIdx.x; c < np * (kSymRec / 2); c += blockDim.x)
      cp_async16(s_rec + buf * P * kSymRec + 2 * c, src + 2 * c);
  };
  stage(blockIdx.x * P, 0);
  cp_async_commit();
  load_sersm(ctx, S);
  __shared__ double sws[2 * kMaxGauss];  // w_i (1 - s_i), w_i s_i
  if (threadIdx.x < n) {
    const double x = ctx->gx[gauss_offset(n) + threadIdx.x];
    const double w = ctx->gw[gauss_offset(n) + threadIdx.x];
    sgx[threadIdx.x] = x;
    sgw[threadIdx.x] = w;
    sws[threadIdx.x] = w * (1.0 - x);
    sws[kMaxGauss + threadIdx.x] = w * x;
  }
  const int lp = threadIdx.x / n;
  const int i = threadIdx.x - lp * n;
  const double* gx = sgx;
  const double* gw = sgw;
  // persistent CTAs stride over the class's pair groups
  int buf = 0;
  for (int base = blockIdx.x * P; base < count; base += gridDim.x * P, buf ^= 1) {
  const int nxt = base + gridDim.x * P;
  if (nxt < count) stage(nxt, buf ^ 1);
  cp_async_commit();  // (possibly empty group: keeps the wait count uniform)
  cp_async_wait1();
  __syncthreads();
  const double* rec_all = s_rec + buf * P * kSymRec;
  const int idx = base + lp;
  const double* R = rec_all + lp * kSymRec;
  const bool active = lp < P && idx < count &&
                      (!PROXY || __double_as_longlong(R[SR_VD]) >= 0);
  if (active) {
    const double pax = R[SR_A + 0], pay = R[SR_A + 1];
    const double dax = R[SR_A + 2], day = R[SR_A + 3];
    const double nax = R[SR_A + 4], nay = R[SR_A + 5];
    const double pbx = R[SR_B + 0], pby = R[SR_B + 1];
    const double dbx = R[SR_B + 2], dby = R[SR_B + 3];
    const double nbx = R[SR_B + 4], nby = R[SR_B + 5];
    const cplx alpha = mk(fc.med.alpha_re, fc.med.alpha_im);
    const double qfac = fc.med.qfactor;
    const double s = gx[i];
    const double xx = pax + s * dax, xy = pay + s * day;
    // series terms for the farthest trial point (a segment's farthest point
    // from x is an endpoint): one count per thread, not per point
#ifndef EBEM_NT_PER_POINT
#define EBEM_NT_PER_POINT 0
#endif
    const bool per_point = EBEM_NT_PER_POINT && !PROXY;
    int nt = 0;
    if (!per_point) {
      const double rmax =
          fmax(hypot(xx - pbx, xy - pby), hypot(xx - pbx - dbx, xy - pby - dby));
      nt = series_terms(S, rmax);
    }
    cplx rv[2][4], ru[2][4];
    double Q[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) rv[b][e] = ru[b][e] = mk(0.0);
#pragma unroll (kJUnroll)
    for (int j = 0; j < n; ++j) {
      const double t = gx[j];
      const double wj = gw[j];
      const double zx = xx - (pbx + t * dbx);
      const double zy = xy - (pby + t * dby);
      double r, ir, logr;
      point_radius(zx, zy, r, ir, logr);
      const double zhx = ir * zx, zhy = ir * zy;
      DN dn;
      dn_eval<!PROXY>(fc, S, r, ir, logr, per_point ? series_terms(S, r) : nt, dn);
      const double pt[2] = {wj * (1.0 - t), wj * t};
      CMat2 dm, nm;
      // V: test on the enclosed element (normal na), trial on the cell element
      combine_D(dn, zhx, zhy, nbx, nby, dm);
      combine_N(dn, zhx, zhy, nax, nay, nbx, nby, nm);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const cplx k = dm.a[e] + alpha * nm.a[e];
        axpy(rv[0][e], pt[0], k);
        axpy(rv[1][e], pt[1], k);
      }
      if (BOTH) {
        // U: test on the cell element, trial on the enclosed element
        // N_U = N_V^T (combine_N is symmetric under z -> -z, m <-> n, i <-> j)
        combine_D(dn, -zhx, -zhy, nax, nay, dm);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const cplx k = dm.a[e] + alpha * nm.a[(e >> 1) | ((e & 1) << 1)];
          axpy(ru[0][e], pt[0], k);
          axpy(ru[1][e], pt[1], k);
        }
      }
      if (!PROXY) {
        // integrated-by-parts static hypersingular kernel (even in zh)
        const double lq = qfac * logr;
        Q[0] = fma(wj, lq - qfac * (zhx * zhx), Q[0]);
        Q[1] = fma(wj, -qfac * (zhx * zhy), Q[1]);
        Q[3] = fma(wj, lq - qfac * (zhy * zhy), Q[3]);
      }
    }
    Q[2] = Q[1];
    double2* my = sh + threadIdx.x * 18;
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        my[b * 4 + e] = make_double2(rv[b][e].re, rv[b][e].im);
        my[8 + b * 4 + e] = make_double2(ru[b][e].re, ru[b][e].im);
      }
    if (!PROXY) {
      my[16] = make_double2(Q[0], Q[1]);
      my[17] = make_double2(Q[2], Q[3]);
    }
  }
  __syncthreads();
  // reduction over i: threads stride over (pair, orientation, 16 outputs),
  // consecutive threads on consecutive shape entries of one component plane
  // (64-byte store runs).  Output (la, lb, e) of orientation o sums
  // fma(w_i phi_x(s_i), row_i[slot], .) over i in order, x = la (V) or lb (U),
  // with the shape weights from the per-CTA table sws.
  const cplx alpha = mk(fc.med.alpha_re, fc.med.alpha_im);
  constexpr int kOrient = BOTH ? 2 : 1;
  for (int o = threadIdx.x; o < P * kOrient * kBundle; o += blockDim.x) {
    const int lp2 = o / (kOrient * kBundle);
    const int rem = o - lp2 * (kOrient * kBundle);
    const int orient = rem >> 4;
    const int kk = rem & 15;
    const int e = kk >> 2, l = kk & 3;  // plane-major: kk = e * 4 + (la, lb)
    const int idx2 = base + lp2;
    if (idx2 >= count) continue;
    const double* R2 = rec_all + lp2 * kSymRec;
    if (PROXY && __double_as_longlong(R2[SR_VD]) < 0) continue;
    const int la = l >> 1, lb = l & 1;
    const int slot = orient == 0 ? (lb * 4 + e) : (8 + la * 4 + e);
    const double* wsh = sws + (orient == 0 ? la : lb) * kMaxGauss;
    const double2* row = sh + (lp2 * n) * 18;
    const double* qrow = reinterpret_cast<const double*>(sh + (lp2 * n) * 18 + 16) + e;
    double ar = 0.0, ai = 0.0, qs = 0.0;
#pragma unroll 4
    for (int ii = 0; ii < n; ++ii) {
      const double2 v = row[ii * 18 + slot];
      const double w = wsh[ii];
      ar = fma(w, v.x, ar);
      ai = fma(w, v.y, ai);
      if (!PROXY) qs = fma(sgw[ii], qrow[ii * 36], qs);
    }
    const double hh = R2[SR_HH];
    const double sg = (la == lb) ? 1.0 : -1.0;  // slope_la * slope_lb
    const double re = PROXY ? hh * ar : fma(hh, ar, sg * qs * alpha.re);
    const double im = PROXY ? hh * ai : fma(hh, ai, sg * qs * alpha.im);
    const long long dst = __double_as_longlong(orient == 0 ? R2[SR_VD] : R2[SR_UD]);
    reinterpret_cast<double2*>(bundles)[bslot(dst, (l << 2) | e, nb)] = make_double2(re, im);
  }
  __syncthreads();  // shared row sums and pair records are reused
  }
}

// Thread-per-pair variant of near_body: one thread owns one element pair and
// sweeps all n x n points (test point s_i outer, trial point t_j inner), so
// no shared-memory reduction over i and no CTA barrier between evaluation
// and output.  After each test point the thread folds its trial sums into
// its bundle accumulators, acc[x][y][e] += w_i phi_x(s_i) r[y][e], kept in
// the thread's own shared-memory column (thread-major, conflict-free); the
// arithmetic (fma(w_i phi, r, acc) from i = 0 upward, Q summed the same way)
// is that of the reduction in near_body, so both variants give the same bits.
// The bundle is written from the thread's column at the end of the pair.
#ifndef EBEM_PP_THREADS
#define EBEM_PP_THREADS 64
#endif
#ifndef EBEM_PP_MINB
#define EBEM_PP_MINB 4
#endif
constexpr int kPpRecPitch = kSymRec + 2;  // 144-byte record rows: conflict-free LDS.128
// thread per pair only for launches that fill the grid several times over:
// its unit of work is a whole pair, so a small launch would idle most SMs
#ifndef EBEM_PP_MIN_ROUNDS
#define EBEM_PP_MIN_ROUNDS 3
#endif
constexpr int kPpMinRounds = EBEM_PP_MIN_ROUNDS;
template <bool BOTH, bool PROXY>
__device__ __forceinline__ void near_body_pp(const DevCtx* __restrict__ ctx,
                                             const FillConst& fc,
                                             const double* __restrict__ recs, int first,
                                             int count, int n, double* __restrict__ bundles,
                                             long long nb) {
  constexpr int kOrient = BOTH ? 2 : 1;
  constexpr int kAcc = 16 * kOrient;  // complex accumulators per thread
  // dynamic: [kAcc][T] accumulators, then one record buffer [T][pitch]
  extern __shared__ double2 sh[];
  __shared__ SerSm S;
  __shared__ double sgx[kMaxGauss], sgw[kMaxGauss];
  const int T = blockDim.x;
  const int tid = threadIdx.x;
  if ((int)blockIdx.x * T >= count) return;  // uniform per CTA
  double2* const acc = sh + tid;              // acc[k * T]
  double* const s_rec = reinterpret_cast<double*>(sh + kAcc * T);
  const double* __restrict__ crec = recs + (long long)first * kSymRec;
  auto stage = [&](int g) {
    const int np = min(T, count - g);
    const double* src = crec + (long long)g * kSymRec;
    for (int c = tid; c < np * (kSymRec / 2); c += T) {
      const int p = c / (kSymRec / 2), q = c - p * (kSymRec / 2);
      cp_async16(s_rec + p * kPpRecPitch + 2 * q, src + 2 * c);
    }
    cp_async_commit();
  };
  stage(blockIdx.x * T);
  load_sersm(ctx, S);
  if (tid < n) {
    sgx[tid] = ctx->gx[gauss_offset(n) + tid];
    sgw[tid] = ctx->gw[gauss_offset(n) + tid];
  }
  const cplx alpha = mk(fc.med.alpha_re, fc.med.alpha_im);
  const double qfac = fc.med.qfactor;
  for (int base = blockIdx.x * T; base < count; base += gridDim.x * T) {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
    __syncthreads();
    // the record goes to registers; the buffer then takes the next group
    const double2* R2 = reinterpret_cast<const double2*>(s_rec + tid * kPpRecPitch);
    const double2 r0 = R2[0], r1 = R2[1], r2 = R2[2], r3 = R2[3], r4 = R2[4], r5 = R2[5],
                  r6 = R2[6], r7 = R2[7];
    __syncthreads();
    const int nxt = base + gridDim.x * T;
    if (nxt < count) stage(nxt);
    const int idx = base + tid;
    const bool active =
        idx < count && (!PROXY || __double_as_longlong(r6.x) >= 0);
    if (active) {
      const double pax = r0.x, pay = r0.y, dax = r1.x, day = r1.y, nax = r2.x, nay = r2.y;
      const double pbx = r3.x, pby = r3.y, dbx = r4.x, dby = r4.y, nbx = r5.x, nby = r5.y;
      const long long vd = __double_as_longlong(r6.x), ud = __double_as_longlong(r6.y);
      const double hh = r7.x;
      double qs[3] = {0.0, 0.0, 0.0};
#pragma unroll 1
      for (int i = 0; i < n; ++i) {
        const double s = sgx[i];
        const double wi = sgw[i];
        const double xx = pax + s * dax, xy = pay + s * day;
        const double rmax =
            fmax(hypot(xx - pbx, xy - pby), hypot(xx - pbx - dbx, xy - pby - dby));
        const int nt = series_terms(S, rmax);
        cplx rv[2][4], ru[2][4];
        double Q[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
          for (int e = 0; e < 4; ++e) rv[b][e] = ru[b][e] = mk(0.0);
#pragma unroll 1
        for (int j = 0; j < n; ++j) {
          const double t = sgx[j];
          const double wj = sgw[j];
          const double zx = xx - (pbx + t * dbx);
          const double zy = xy - (pby + t * dby);
          double r, ir, logr;
          point_radius(zx, zy, r, ir, logr);
          const double zhx = ir * zx, zhy = ir * zy;
          DN dn;
          dn_eval<!PROXY>(fc, S, r, ir, logr, nt, dn);
          const double pt[2] = {wj * (1.0 - t), wj * t};
          CMat2 dm, nm;
          combine_D(dn, zhx, zhy, nbx, nby, dm);
          combine_N(dn, zhx, zhy, nax, nay, nbx, nby, nm);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const cplx k = dm.a[e] + alpha * nm.a[e];
            axpy(rv[0][e], pt[0], k);
            axpy(rv[1][e], pt[1], k);
          }
          if (BOTH) {
            combine_D(dn, -zhx, -zhy, nax, nay, dm);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const cplx k = dm.a[e] + alpha * nm.a[(e >> 1) | ((e & 1) << 1)];
              axpy(ru[0][e], pt[0], k);
              axpy(ru[1][e], pt[1], k);
            }
          }
          if (!PROXY) {
            const double lq = qfac * logr;
            Q[0] = fma(wj, lq - qfac * (zhx * zhx), Q[0]);
            Q[1] = fma(wj, -qfac * (zhx * zhy), Q[1]);
            Q[2] = fma(wj, lq - qfac * (zhy * zhy), Q[2]);
          }
        }
        // fold: acc[o][x][y][e] (+)= w_i phi_x(s_i) r_o[y][e]
        const double wsh[2] = {wi * (1.0 - s), wi * s};
#pragma unroll
        for (int x = 0; x < 2; ++x)
#pragma unroll
          for (int y = 0; y < 2; ++y)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int kv = (x * 2 + y) * 4 + e;
              double2 a = i ? acc[kv * T] : make_double2(0.0, 0.0);
              a.x = fma(wsh[x], rv[y][e].re, a.x);
              a.y = fma(wsh[x], rv[y][e].im, a.y);
              acc[kv * T] = a;
              if (BOTH) {
                double2 b = i ? acc[(16 + kv) * T] : make_double2(0.0, 0.0);
                b.x = fma(wsh[x], ru[y][e].re, b.x);
                b.y = fma(wsh[x], ru[y][e].im, b.y);
                acc[(16 + kv) * T] = b;
              }
            }
        if (!PROXY) {
#pragma unroll
          for (int e = 0; e < 3; ++e) qs[e] = fma(wi, Q[e], qs[e]);
        }
      }
      // bundle entries: k = bidx(la, lb, i, j), component e = k & 3
      double2* const out = reinterpret_cast<double2*>(bundles);
#pragma unroll
      for (int o = 0; o < kOrient; ++o) {
        const long long dst = o == 0 ? vd : ud;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const double q = qs[e == 3 ? 2 : (e == 0 ? 0 : 1)];
#pragma unroll
          for (int l = 0; l < 4; ++l) {
            const int la = l >> 1, lb = l & 1;
            // V: acc[la][lb][e]; U: acc[lb][la][e] (its test shape is lb)
            const int kv = o == 0 ? (la * 2 + lb) * 4 + e : 16 + (lb * 2 + la) * 4 + e;
            const double2 a = acc[kv * T];
            const double sg = (la == lb) ? 1.0 : -1.0;
            const double re = PROXY ? hh * a.x : fma(hh, a.x, sg * q * alpha.re);
            const double im = PROXY ? hh * a.y : fma(hh, a.y, sg * q * alpha.im);
            out[bslot(dst, (l << 2) | e, nb)] = make_double2(re, im);
          }
        }
      }
    }
  }
}

__global__ void __launch_bounds__(EBEM_PP_THREADS, EBEM_PP_MINB)
k_proxy_pp(const DevCtx* __restrict__ ctx, const __grid_constant__ FillConst fc,
           const double* __restrict__ recs, int n_slots, int ng,
           double* __restrict__ bundles, long long nb) {
  near_body_pp<true, true>(ctx, fc, recs, 0, n_slots, ng, bundles, nb);
}

template <bool BOTH>
__global__ void __launch_bounds__(EBEM_SYM_THREADS, EBEM_SYM_MINB)
k_near_sym(const DevCtx* __restrict__ ctx, const __grid_constant__ FillConst fc,
           const double* __restrict__ recs, const int* __restrict__ class_bounds,
           int cls, int n, double* __restrict__ bundles, long long nb) {
  // this class's pairs, from the device-side bucket bounds (no host sync)
  const int first = __ldg(class_bounds + cls);
  const int count = __ldg(class_bounds + cls + 1) - first;
  near_body<BOTH, false>(ctx, fc, recs, first, count, n, bundles, nb);
}

// ------------------------------------------------------------------- proxy
// Proxy blocks: one record per (polygon element, curve element) slot of each
// job's CTA tiles (kProxyTile slots per tile; the tail of a job's last tile
// is padding, marked by a negative V slot).  The polygon element is the test
// side of V ("a"), the curve element the trial side ("b").
constexpr int kProxyThreads = 256;

__global__ void __launch_bounds__(256)
k_proxy_records(const DevCtx* __restrict__ ctx, const ProxyJob* __restrict__ jobs,
                const int* __restrict__ job_block_off, int n_jobs,
                const int* __restrict__ elems, long long n_slots, int tile,
                double* __restrict__ recs) {
  constexpr int kRecPad = kSymRec / 2 + 1;  // 144-byte rows, as in k_sym_scatter
  __shared__ double2 s_rec[8 * 32 * kRecPad];
  const long long t0 = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31);
  const long long t = t0 + (threadIdx.x & 31);
  const int lane = threadIdx.x & 31;
  double2* const wrec = s_rec + (threadIdx.x >> 5) * (32 * kRecPad);
  if (t < n_slots) {
  const int blk = int(t / tile);
  const int jb = find_job(job_block_off, n_jobs, blk);
  const ProxyJob J = jobs[jb];
  const int m = ctx->m_prime;
  const int pair = (blk - J.block_off) * tile + int(t - (long long)blk * tile);
  double r[kSymRec];
#pragma unroll
  for (int k = 0; k < kSymRec; ++k) r[k] = 0.0;
  if (pair >= m * J.nE) {
    r[SR_VD] = __longlong_as_double(-1LL);
  } else {
    const int pe = pair / J.nE;
    const int q = pair - pe * J.nE;
    const int eb = __ldg(elems + J.e_off + q);
    // polygon element pe: node pe -> node (pe+1) mod m (Mesh ctor, geometry.cpp:15-37)
    const int pn = pe + 1 == m ? 0 : pe + 1;
    const double p0x = J.cx + J.radius * ctx->poly_cs[2 * pe];
    const double p0y = J.cy + J.radius * ctx->poly_cs[2 * pe + 1];
    const double p1x = J.cx + J.radius * ctx->poly_cs[2 * pn];
    const double p1y = J.cy + J.radius * ctx->poly_cs[2 * pn + 1];
    const double pdx = p1x - p0x, pdy = p1y - p0y;
    const double hp = hypot(pdx, pdy);
    const double ptx = pdx / hp, pty = pdy / hp;
    r[SR_A + 0] = p0x;
    r[SR_A + 1] = p0y;
    r[SR_A + 2] = pdx;
    r[SR_A + 3] = pdy;
    r[SR_A + 4] = -pty;
    r[SR_A + 5] = ptx;
    const Elem8 B = load_elem8(ctx, eb);
    r[SR_B + 0] = B.px;
    r[SR_B + 1] = B.py;
    r[SR_B + 2] = B.dx;
    r[SR_B + 3] = B.dy;
    r[SR_B + 4] = B.nx;
    r[SR_B + 5] = B.ny;
    r[SR_VD] = __longlong_as_double(J.v_off + pair);
    r[SR_UD] = __longlong_as_double(J.u_off + (long long)q * m + pe);
    r[SR_HH] = hp * B.h;
  }
#pragma unroll
  for (int k = 0; k < kSymRec / 2; ++k)
    wrec[lane * kRecPad + k] = make_double2(r[2 * k], r[2 * k + 1]);
  }
  __syncwarp();
  // the warp's records are consecutive: 512-byte store runs
  if (t0 >= n_slots) return;
  const int live = n_slots - t0 < 32 ? int(n_slots - t0) : 32;
  double2* const o = reinterpret_cast<double2*>(recs + t0 * kSymRec);
#pragma unroll
  for (int c = lane; c < 32 * (kSymRec / 2); c += 32) {
    const int rr = c / (kSymRec / 2);
    if (rr < live) o[c] = wrec[rr * kRecPad + c - rr * (kSymRec / 2)];
  }
}

// Same evaluation as the near-field kernel (thread (pair, i) fixes the
// polygon quadrature point s_i and sweeps the curve points t_j), full scalars.
__global__ void __launch_bounds__(EBEM_PRX_THREADS, EBEM_PRX_MINB)
k_proxy_pairs(const DevCtx* __restrict__ ctx, const __grid_constant__ FillConst fc,
              const double* __restrict__ recs, int n_slots, int ng,
              double* __restrict__ bundles, long long nb) {
  near_body<true, true>(ctx, fc, recs, 0, n_slots, ng, bundles, nb);
}

// ------------------------------------------------------------------ gather
__global__ void __launch_bounds__(kGatherTile)
k_gather(const GatherJob* __restrict__ jobs, const int* __restrict__ job_block_off,
         int n_jobs, const NodeDesc* __restrict__ desc,
         const double* __restrict__ bundles, long long nb) {
  __shared__ int s_jb;
  if (threadIdx.x == 0) s_jb = find_job(job_block_off, n_jobs, int(blockIdx.x));
  __syncthreads();
  const int jb = s_jb;
  const GatherJob& J = jobs[jb];
  const long long local =
      (long long)(blockIdx.x - __ldg(job_block_off + jb)) * kGatherTile + threadIdx.x;
  if (local >= (long long)J.nrows * J.ncols) return;
  // consecutive threads -> consecutive destination addresses: down a column
  // for plain blocks, along a row for the conjugate-transposed ones
  int r, c;
  if (J.trans) {
    r = int(local / J.ncols);
    c = int(local - (long long)r * J.ncols);
  } else {
    c = int(local / J.nrows);
    r = int(local - (long long)c * J.nrows);
  }
  const NodeDesc rd = desc[J.rdesc_off + r];
  const NodeDesc cd = desc[J.cdesc_off + c];
  const int i = rd.bits >> 2, j = cd.bits >> 2;
  const int ra[2] = {rd.e1, rd.e2}, la[2] = {rd.bits & 1, (rd.bits >> 1) & 1};
  const int cb[2] = {cd.e1, cd.e2}, lb[2] = {cd.bits & 1, (cd.bits >> 1) & 1};
  const double2* B = reinterpret_cast<const double2*>(bundles);
  double re = 0.0, im = 0.0;
#pragma unroll
  for (int x = 0; x < 2; ++x)
#pragma unroll
    for (int y = 0; y < 2; ++y) {
      const long long pidx = J.pair_off + (long long)ra[x] * J.nces + cb[y];
      const double2 v = __ldg(B + bslot(pidx, bidx(la[x], lb[y], i, j), nb));
      re += v.x;
      im += v.y;
    }
  double2* D = reinterpret_cast<double2*>(J.dest);
  if (J.trans) D[rd.dest * (long long)J.ld + cd.dest] = make_double2(re, -im);
  else D[cd.dest * (long long)J.ld + rd.dest] = make_double2(re, im);
}

// ------------------------------------------------------------ cross-level reuse
// One warp per (task, column): the column's listed enclosed rows, both
// components, from the child's matrix to the cell's.  Row pairs are runs of
// consecutive positions in both matrices, so the lanes read and write
// consecutive addresses.
__global__ void __launch_bounds__(32 * kReuseCols)
k_reuse_copy(const ReuseTask* __restrict__ tasks, const int* __restrict__ task_block_off,
             int n_tasks, const int2* __restrict__ row_pairs,
             const int2* __restrict__ col_pairs) {
  __shared__ int s_t;
  if (threadIdx.x == 0) s_t = find_job(task_block_off, n_tasks, int(blockIdx.x));
  __syncthreads();
  const ReuseTask T = tasks[s_t];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int c = (int(blockIdx.x) - __ldg(task_block_off + s_t)) * kReuseCols + warp;
  if (c >= T.n_cols) return;
  const int2 cp = __ldg(col_pairs + T.col_off + c);
  const double2* src = reinterpret_cast<const double2*>(T.src) + (long long)cp.x * T.src_ld;
  double2* dst = reinterpret_cast<double2*>(T.dst) + (long long)cp.y * T.dst_ld;
  const int2* rp = row_pairs + T.row_off;
  for (int r = lane; r < T.n_rows; r += 32) {
    const int2 q = __ldg(rp + r);
    dst[T.dst_row0 + q.y] = __ldg(src + T.src_row0 + q.x);
    dst[T.dst_row0 + T.dst_ne + q.y] = __ldg(src + T.src_row0 + T.src_ne + q.x);
  }
}

// One CTA per task; consecutive threads on consecutive destination rows.
__global__ void __launch_bounds__(128)
k_map_copy(const MapTask* __restrict__ tasks, const int2* __restrict__ row_pairs,
           const int2* __restrict__ col_pairs) {
  const MapTask T = tasks[blockIdx.x];
  const double2* src = reinterpret_cast<const double2*>(T.src);
  double2* dst = reinterpret_cast<double2*>(T.dst);
  const int2* rp = row_pairs + T.row_off;
  const int2* cp = col_pairs + T.col_off;
  const int total = T.n_rows * T.n_cols;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int c = idx / T.n_rows, r = idx - c * T.n_rows;
    const int2 rr = __ldg(rp + r), cc = __ldg(cp + c);
    double2 v;
    if (T.swap) {
      v = __ldg(src + (long long)rr.x * T.src_ld + cc.x);
      v.y = -v.y;
    } else {
      v = __ldg(src + (long long)cc.x * T.src_ld + rr.x);
    }
    dst[(long long)cc.y * T.dst_ld + rr.y] = v;
  }
}

// ------------------------------------------------------------ host wrappers

void launch_map_copy(const MapTask* tasks, int n_tasks, const int2* row_pairs,
                     const int2* col_pairs, cudaStream_t st) {
  if (n_tasks <= 0) return;
  k_map_copy<<<n_tasks, 128, 0, st>>>(tasks, row_pairs, col_pairs);
}

void launch_reuse_copy(const ReuseTask* tasks, const int* task_block_off, int n_tasks,
                       int n_blocks, const int2* row_pairs, const int2* col_pairs,
                       cudaStream_t st) {
  if (n_blocks <= 0) return;
  k_reuse_copy<<<n_blocks, 32 * kReuseCols, 0, st>>>(tasks, task_block_off, n_tasks, row_pairs,
                                                     col_pairs);
}


// Thread-per-pair proxy body (near_body_pp); EBEM_FILL_PP=0 selects the
// (pair, test point) thread mapping with the shared-memory reduction.  (The
// near field measured slower with it, 407 -> 436 ms at 2N = 2^19: n = 4
// points per side leave too little work per pair to hide the fold and the
// per-thread bundle stores; the proxy blocks, 36 points of full scalars per
// pair, gain 134 -> 121 ms.)
static bool fill_pp() {
  static const bool on = [] {
    const char* e = std::getenv("EBEM_FILL_PP");
    return e ? std::atoi(e) != 0 : true;
  }();
  return on;
}

void launch_sym_bucket(const DevCtx* ctx, const SymJob* jobs, const long long* job_off,
                       int n_jobs, const int* elems, long long n_pairs,
                       unsigned char* keys, int* pair_job, int* bounds, double* recs,
                       cudaStream_t st) {
  if (n_pairs <= 0) return;
  cudaMemsetAsync(bounds + kBoundsCounts, 0,
                  size_t(kBoundsInts - kBoundsCounts) * sizeof(int), st);
  const unsigned grid = (unsigned)((n_pairs + kBucketThreads - 1) / kBucketThreads);
  k_sym_count<<<grid, kBucketThreads, 0, st>>>(ctx, jobs, job_off, n_jobs, elems, n_pairs,
                                               keys, pair_job, bounds);
  k_sym_scatter<<<grid, kBucketThreads, 0, st>>>(ctx, jobs, elems, keys, pair_job, n_pairs,
                                                 bounds, recs);
}

int sym_bounds_ints() { return kBoundsInts; }

void launch_near_sym(const DevCtx* ctx, const FillConst& fc, const double* recs, const int* class_bounds,
                     int cls, long long max_count, int n, bool both, double* bundles,
                     long long nb, cudaStream_t st) {
  if (max_count <= 0) return;
  const int P = EBEM_SYM_THREADS / n;
  const int threads = P * n;
  const size_t smem = size_t(threads) * 18 * sizeof(double2) +
                      size_t(2 * P) * kSymRec * sizeof(double);
  // persistent grid: a few CTAs per SM, never more than the largest count needs
  static const int n_sm = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  const long long need = (max_count + P - 1) / P;
  const int grid = int(std::min<long long>(need, 4LL * n_sm));
#define EBEM_SYM_LAUNCH(B)                                                          \
  do {                                                                              \
    cudaFuncSetAttribute(k_near_sym<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                         EBEM_SYM_THREADS * (18 * (int)sizeof(double2) +        \
                                             2 * kSymRec * (int)sizeof(double)));  \
    k_near_sym<B><<<grid, threads, smem, st>>>(ctx, fc, recs, class_bounds, cls, n,  \
                                               bundles, nb);                        \
  } while (0)
  if (both) EBEM_SYM_LAUNCH(true);
  else EBEM_SYM_LAUNCH(false);
#undef EBEM_SYM_LAUNCH
}

void launch_near_singular(const DevCtx* ctx, const long long* pairs,
                          const int* pair_elems, int n, double* bundles, long long nb,
                          int* bad, cudaStream_t st) {
  if (n <= 0) return;
  const int bs = 128;  // 4 pairs per CTA, one warp each
  k_near_singular<<<(unsigned)((n + 3) / 4), bs, 0, st>>>(ctx, pairs, pair_elems, n,
                                                          bundles, nb, bad);
}

int proxy_pairs_per_block(int n_gauss) {
  return n_gauss >= kProxyThreads ? 1 : kProxyThreads / n_gauss;
}

int proxy_blocks_for(int m_prime, int nE, int n_gauss) {
  const int p = proxy_pairs_per_block(n_gauss);
  return (m_prime * nE + p - 1) / p;
}

void launch_proxy_pairs(const DevCtx* ctx, const FillConst& fc, int n_gauss,
                        const ProxyJob* jobs, const int* job_block_off, int n_jobs,
                        int n_blocks, const int* elems, double* recs, double* bundles,
                        long long nb, cudaStream_t st) {
  if (n_blocks <= 0) return;
  const int tile = proxy_pairs_per_block(n_gauss);
  const long long n_slots = (long long)n_blocks * tile;
  k_proxy_records<<<(unsigned)((n_slots + 255) / 256), 256, 0, st>>>(
      ctx, jobs, job_block_off, n_jobs, elems, n_slots, tile, recs);
  static const int n_sm = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  if (fill_pp() && n_slots >= (long long)kPpMinRounds * EBEM_PP_MINB * n_sm * EBEM_PP_THREADS) {
    const int T = EBEM_PP_THREADS;
    const size_t smem_pp = size_t(T) * 32 * sizeof(double2) +
                           size_t(T) * kPpRecPitch * sizeof(double);
    static bool attr_pp = [smem_pp] {
      cudaFuncSetAttribute(k_proxy_pp, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem_pp));
      return true;
    }();
    (void)attr_pp;
    const long long need_pp = (n_slots + T - 1) / T;
    const int grid_pp = int(std::min<long long>(need_pp, (long long)EBEM_PP_MINB * n_sm));
    k_proxy_pp<<<grid_pp, T, smem_pp, st>>>(ctx, fc, recs, int(n_slots), n_gauss, bundles, nb);
    return;
  }
  const int P = EBEM_PRX_THREADS / n_gauss;
  const int threads = P * n_gauss;
  const size_t smem = size_t(threads) * 18 * sizeof(double2) +
                      size_t(2 * P) * kSymRec * sizeof(double);
  static bool attr = [] {
    cudaFuncSetAttribute(k_proxy_pairs, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         EBEM_PRX_THREADS * (18 * (int)sizeof(double2) +
                                             2 * kSymRec * (int)sizeof(double)));
    return true;
  }();
  (void)attr;
  const long long need = (n_slots + P - 1) / P;
  const int grid = int(std::min<long long>(need, 4LL * n_sm));
  k_proxy_pairs<<<grid, threads, smem, st>>>(ctx, fc, recs, int(n_slots), n_gauss, bundles,
                                             nb);
}

void launch_gather(const GatherJob* jobs, const int* job_block_off, int n_jobs,
                   int n_blocks, const NodeDesc* desc, const double* bundles,
                   long long nb, cudaStream_t st) {
  if (n_blocks <= 0) return;
  k_gather<<<(unsigned)n_blocks, kGatherTile, 0, st>>>(jobs, job_block_off, n_jobs,
                                                       desc, bundles, nb);
}

}  // namespace ebem_gpu
