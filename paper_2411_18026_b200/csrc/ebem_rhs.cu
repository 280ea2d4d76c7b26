// Incident-field right-hand sides and point evaluations of the special
// functions (the latter only back the parity tests of the device math).
//
//   k_rhs_plane   BlockAssembler::rhs with a plane P wave (PlanePWave,
//                 proj/src/kernels.cpp:99-118; proj/include/ebem/assembly.hpp:94-119)
//                 or a plane SV wave (config 4; not in the reference, derived
//                 from the same constitutive law).  One thread per
//                 node sums its two supporting elements in ascending element
//                 order, Gauss points in rule order, as the reference loop does.
#include <cuda_runtime.h>

#include "ebem_device.cuh"
#include "ebem_kernels.h"

namespace ebem_gpu {

namespace {

__device__ __forceinline__ double efr(const DevCtx* __restrict__ c, int f, int e) {
  return __ldg(c->elem + size_t(f) * c->n_nodes + e);
}

// Plane wave with unit direction d: P (kind 0) u = A d e^{-i kL d.x};
// SV (kind 1) u = A p e^{-i kT d.x} with p = (-d_y, d_x).
__device__ __forceinline__ void wave_at(const DevMedium& m, int kind, double dx,
                                        double dy, double amp, double x,
                                        double y, double nx, double ny,
                                        cplx& ux, cplx& uy, cplx& tx, cplx& ty) {
  const double k = kind == 0 ? m.kL : m.kT;
  double sn, cs;
  sincos(-k * (dx * x + dy * y), &sn, &cs);
  const cplx ph = mk(amp * cs, amp * sn);
  const cplx f = mk(0.0, -k) * ph;  // -i k A e^{...}
  const double nd = nx * dx + ny * dy;
  if (kind == 0) {
    ux = ph * dx;
    uy = ph * dy;
    tx = f * (m.lam * nx + 2.0 * m.mu * nd * dx);
    ty = f * (m.lam * ny + 2.0 * m.mu * nd * dy);
  } else {
    const double px = -dy, py = dx;
    const double np = nx * px + ny * py;
    ux = ph * px;
    uy = ph * py;
    tx = f * (m.mu * (nd * px + np * dx));
    ty = f * (m.mu * (nd * py + np * dy));
  }
}

}  // namespace

// out: 2N x m complex, column-major (component-major rows).
__global__ void k_rhs_plane(const DevCtx* __restrict__ ctx, int kind,
                            const double* __restrict__ angles, int m,
                            double amp, int rhs_n, double* __restrict__ out) {
  const int N = ctx->n_nodes;
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)N * m) return;
  const int col = int(t / N);
  const int g = int(t - (long long)col * N);
  const double ang = angles[col];
  double dys, dxs;
  sincos(ang, &dys, &dxs);
  const cplx alpha = mk(ctx->med.alpha_re, ctx->med.alpha_im);
  const double* gx = ctx->gx + gauss_offset(rhs_n);
  const double* gw = ctx->gw + gauss_offset(rhs_n);
  // supporting elements of node g in ascending order, with local shape index
  int es[2], as[2];
  if (g == 0) {
    es[0] = 0; as[0] = 0; es[1] = N - 1; as[1] = 1;
  } else {
    es[0] = g - 1; as[0] = 1; es[1] = g; as[1] = 0;
  }
  cplx b1 = mk(0.0), b2 = mk(0.0);
  for (int q = 0; q < 2; ++q) {
    const int e = es[q];
    const double h = efr(ctx, EH, e);
    const double px = efr(ctx, EPX, e), py = efr(ctx, EPY, e);
    const double ddx = efr(ctx, EDX, e), ddy = efr(ctx, EDY, e);
    const double nx = efr(ctx, ENX, e), ny = efr(ctx, ENY, e);
    for (int k = 0; k < rhs_n; ++k) {
      const double s = gx[k];
      cplx ux, uy, tx, ty;
      wave_at(ctx->med, kind, dxs, dys, amp, px + s * ddx, py + s * ddy, nx, ny,
              ux, uy, tx, ty);
      const cplx v1 = ux + alpha * tx;
      const cplx v2 = uy + alpha * ty;
      const double wh = gw[k] * h;
      const double p = as[q] == 0 ? (1.0 - s) * wh : s * wh;
      axpy(b1, p, v1);
      axpy(b2, p, v2);
    }
  }
  double2* o = reinterpret_cast<double2*>(out) + (long long)col * 2 * N;
  o[g] = make_double2(b1.re, b1.im);
  o[N + g] = make_double2(b2.re, b2.im);
}

// ------------------------------------------------------- field evaluation
// boundary_distance (proj/src/postprocess.cpp:24-30): one CTA per point
__global__ void __launch_bounds__(256)
k_boundary_distance(const DevCtx* __restrict__ ctx, const double* __restrict__ pts,
                    double* __restrict__ out) {
  __shared__ double red[8];
  const int N = ctx->n_nodes;
  const double x = pts[2 * blockIdx.x], y = pts[2 * blockIdx.x + 1];
  double best = 1e300;
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const double ax = efr(ctx, EPX, e), ay = efr(ctx, EPY, e);
    const double bx = efr(ctx, EDX, e), by = efr(ctx, EDY, e);  // b - a
    const double len2 = bx * bx + by * by;
    double t = len2 > 0.0 ? ((x - ax) * bx + (y - ay) * by) / len2 : 0.0;
    t = fmin(fmax(t, 0.0), 1.0);
    best = fmin(best, hypot(x - (ax + t * bx), y - (ay + t * by)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < int(blockDim.x >> 5); ++w) best = fmin(best, red[w]);
    out[blockIdx.x] = fmin(best, red[0]);
  }
}

// evaluate_scattered / evaluate_field (proj/src/postprocess.cpp:56-119):
// u_s(x) = -sum_e sum_q w_q h_e D(x, y_q, n_e) u(y_q), u linear on each
// element; one CTA per point, elements strided over the threads.  Optional
// incident plane wave (kind 0 P, 1 SV; < 0 none) and intensity.
__global__ void __launch_bounds__(256)
k_field(const DevCtx* __restrict__ ctx, const double* __restrict__ bu,
        const double* __restrict__ pts, int ng, int kind, double angle, double amp,
        double* __restrict__ out_u, double* __restrict__ out_int) {
  __shared__ cplx red[8][2];
  const int N = ctx->n_nodes;
  const double x = pts[2 * blockIdx.x], y = pts[2 * blockIdx.x + 1];
  const double* gx = ctx->gx + gauss_offset(ng);
  const double* gw = ctx->gw + gauss_offset(ng);
  const double2* u = reinterpret_cast<const double2*>(bu);
  cplx a1 = mk(0.0), a2 = mk(0.0);
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    const int e2 = e + 1 == N ? 0 : e + 1;
    const double px = efr(ctx, EPX, e), py = efr(ctx, EPY, e);
    const double dx = efr(ctx, EDX, e), dy = efr(ctx, EDY, e);
    const double nx = efr(ctx, ENX, e), ny = efr(ctx, ENY, e);
    const double len = efr(ctx, EH, e);
    const double2 ua1 = u[e], ua2 = u[N + e], ub1 = u[e2], ub2 = u[N + e2];
    for (int q = 0; q < ng; ++q) {
      const double t = gx[q];
      const double zx = x - (px + t * dx), zy = y - (py + t * dy);
      const double r = hypot(zx, zy);
      Scalars s;
      scalars_full(ctx, r, s);
      CMat2 d;
      combine_D(s, zx / r, zy / r, nx, ny, d);
      const cplx u1 = mk((1.0 - t) * ua1.x + t * ub1.x, (1.0 - t) * ua1.y + t * ub1.y);
      const cplx u2 = mk((1.0 - t) * ua2.x + t * ub2.x, (1.0 - t) * ua2.y + t * ub2.y);
      const double w = gw[q] * len;
      axpy(a1, w, d.a[0] * u1 + d.a[1] * u2);
      axpy(a2, w, d.a[2] * u1 + d.a[3] * u2);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a1.re += __shfl_xor_sync(0xffffffffu, a1.re, o);
    a1.im += __shfl_xor_sync(0xffffffffu, a1.im, o);
    a2.re += __shfl_xor_sync(0xffffffffu, a2.re, o);
    a2.im += __shfl_xor_sync(0xffffffffu, a2.im, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5][0] = a1;
    red[threadIdx.x >> 5][1] = a2;
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  cplx s1 = mk(0.0), s2 = mk(0.0);
  for (int w = 0; w < int(blockDim.x >> 5); ++w) {
    s1 += red[w][0];
    s2 += red[w][1];
  }
  s1 = -s1;
  s2 = -s2;
  if (kind >= 0) {
    double dys, dxs;
    sincos(angle, &dys, &dxs);
    cplx ux, uy, tx, ty;
    wave_at(ctx->med, kind, dxs, dys, amp, x, y, 0.0, 0.0, ux, uy, tx, ty);
    s1 += ux;
    s2 += uy;
  }
  out_u[4 * blockIdx.x] = s1.re;
  out_u[4 * blockIdx.x + 1] = s1.im;
  out_u[4 * blockIdx.x + 2] = s2.re;
  out_u[4 * blockIdx.x + 3] = s2.im;
  if (out_int) out_int[blockIdx.x] = s1.re * s1.re + s1.im * s1.im + s2.re * s2.re + s2.im * s2.im;
}

__global__ void k_eval_hankel(const double* __restrict__ x, int n,
                              double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  cplx h0, h1;
  hankel01(x[t], h0, h1);
  out[4 * t] = h0.re;
  out[4 * t + 1] = h0.im;
  out[4 * t + 2] = h1.re;
  out[4 * t + 3] = h1.im;
}

__global__ void k_eval_scalars(const DevCtx* __restrict__ ctx,
                               const double* __restrict__ r, int n, int which,
                               double* __restrict__ out) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  Scalars s;
  if (which == 0) {
    scalars_full(ctx, r[t], s);
  } else if (which == 1) {
    Scalars f;
    scalars_split(ctx, r[t], f, s);
  } else {
    StaticScalars s0;
    static_part(ctx->med, r[t], s0);
    for (int k = 0; k < 10; ++k) s.s[k] = mk(s0.s[k]);
  }
  for (int k = 0; k < 10; ++k) {
    out[20 * t + 2 * k] = s.s[k].re;
    out[20 * t + 2 * k + 1] = s.s[k].im;
  }
}

// FP64 FMA throughput probe: 8 independent dependency chains per thread.
__global__ void __launch_bounds__(256) k_fp64_peak(int iters, double seed,
                                                   double* sink) {
  double a[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = seed + q + threadIdx.x;
  const double b = 1.0 - 1e-9, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) a[q] = fma(a[q], b, c);
  }
  double s = 0.0;
#pragma unroll
  for (int q = 0; q < 8; ++q) s += a[q];
  if (s == 12345.678) sink[0] = s;
}

double measure_fp64_peak_tflops() {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* sink = nullptr;
  cudaMalloc(&sink, 8);
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  k_fp64_peak<<<blocks, threads>>>(64, 1.0, sink);  // warm-up
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_fp64_peak<<<blocks, threads>>>(iters, 1.0, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(sink);
  const double flops = 2.0 * 8.0 * double(iters) * blocks * threads;
  return ms > 0 ? flops / (1e-3 * ms) / 1e12 : 0.0;
}

void launch_rhs_plane(const DevCtx* ctx, int n_nodes, int kind,
                        const double* angles, int m, double amplitude,
                        int rhs_n, double* out, cudaStream_t st) {
  const long long total = (long long)n_nodes * m;
  if (total <= 0) return;
  const int bs = 128;
  k_rhs_plane<<<(unsigned)((total + bs - 1) / bs), bs, 0, st>>>(
      ctx, kind, angles, m, amplitude, rhs_n, out);
}

void launch_boundary_distance(const DevCtx* ctx, const double* pts, int m, double* out,
                              cudaStream_t st) {
  if (m <= 0) return;
  k_boundary_distance<<<m, 256, 0, st>>>(ctx, pts, out);
}

void launch_field(const DevCtx* ctx, const double* bu, const double* pts, int m, int ng,
                  int kind, double angle, double amp, double* out_u, double* out_int,
                  cudaStream_t st) {
  if (m <= 0) return;
  k_field<<<m, 256, 0, st>>>(ctx, bu, pts, ng, kind, angle, amp, out_u, out_int);
}

void launch_eval_hankel(const double* x, int n, double* out, cudaStream_t st) {
  if (n <= 0) return;
  k_eval_hankel<<<(n + 127) / 128, 128, 0, st>>>(x, n, out);
}

void launch_eval_scalars(const DevCtx* ctx, const double* r, int n, int which,
                         double* out, cudaStream_t st) {
  if (n <= 0) return;
  k_eval_scalars<<<(n + 127) / 128, 128, 0, st>>>(ctx, r, n, which, out);
}

}  // namespace ebem_gpu
