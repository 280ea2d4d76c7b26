// Plain-data structures shared by the host runtime (C++) and the sm_100a
// kernels (CUDA).  No torch types, no STL.
#pragma once

#include <stdint.h>
#include <vector_types.h>

namespace ebem_gpu {

constexpr int kMaxSeriesPow = 48;  // dense power tables r^0 .. r^47
constexpr int kMaxGauss = 40;      // Gauss-Legendre orders 1 .. 40 on device
constexpr int kGaussSlots = kMaxGauss * (kMaxGauss + 1) / 2;

// Medium constants (proj/include/ebem/medium.hpp, kernel_scalars.cpp:123-131,
// assembly.cpp:42-50).
struct DevMedium {
  double kL, kT, lam, mu;
  double aratio;         // lam / (lam + 2 mu)
  double cconst;         // (lam + mu) / (8 pi (lam + 2 mu))
  double qfactor;        // 8 mu cconst
  double series_radius;  // 0.25 / kT
  double kappa;          // mu / (2 pi (lam + 2 mu))
  double ccon;           // (lam + mu) / (8 pi (lam + 2 mu))
  double alpha_re, alpha_im;
  // derived constants of the fast kernel path (host-computed once)
  double inv_kT, inv_kL;
  double log_half_kT, log_half_kL;  // ln(k/2): ln(k r / 2) = ln r + ln(k/2)
  double sd1, sd3;                  // static d1 = sd1 / r, d3 = sd3 / r
  double sn[5];                     // static n1, n2, n4, n5, n7 = sn[i] / r^2
  double c_n5;                      // lam * aratio * kL^2
};

// Remainder series of one scalar in parity form:
//   sum_p (a_p + b_p ln r) r^(par + 2p),  p = 0 .. nt-1
// (every series carries powers of a single parity: d's odd, n's even).
constexpr int kParTerms = 26;
struct ParSeries {
  int par[10], nt[10];
  double2 a[10][kParTerms];
  double2 b[10][kParTerms];
  // Per-point truncation of the D/N series (scalars 2..9): a point at
  // distance r needs 1 + #{t >= 1 : r > rcut[t]} terms (+inf past nt).
  double rcut[kParTerms];
};

// Fill-kernel parameter block, passed by value as a __grid_constant__ kernel
// argument: the medium constants are then constant-bank operands.
// The leading D/N series terms (scalars 2..9, parity form) ride along, so
// the Horner steps of the series branch take their coefficients as
// constant-bank operands instead of shared-memory loads.
constexpr int kFcTerms = 12;
struct FillConst {
  DevMedium med;
  double2 sa[kFcTerms][8];
  double2 sb[kFcTerms][8];
};

// Element geometry, structure of arrays over the N elements (element e runs
// from node e to node (e+1) mod N): p = start node, d = end - start, t = unit
// tangent, n = unit normal (+90 deg rotation of t), h = length.
enum ElemField { EPX = 0, EPY, EDX, EDY, ETX, ETY, ENX, ENY, EH, kElemFields };

struct DevCtx {
  DevMedium med;
  int n_nodes;
  int series_maxq;
  // Remainder series of the ten scalars: series[(k * kMaxSeriesPow + q) * 4 +
  // {0,1,2,3}] = {Re a_q, Im a_q, Re b_q, Im b_q} of sum (a_q + b_q ln r) r^q.
  alignas(16) double series[10 * kMaxSeriesPow * 4];
  ParSeries pser;
  // Gauss-Legendre rules on [0,1]; order n occupies [n(n-1)/2, n(n+1)/2).
  double gx[kGaussSlots];
  double gw[kGaussSlots];
  // Quadrature knobs (AssemblyConfig, proj/include/ebem/assembly.hpp:21-30).
  int far_nodes;
  int corner_n;   // scaled corner_nodes
  int proxy_n;    // ProxyConfig::n_gauss
  int m_prime;    // ProxyConfig::m_prime
  double refine;
  int very_far_tier;  // 1: pairs beyond kVeryFar element lengths take the 3 x 3 rule
  // cos/sin of 2 pi j / m' (host libm), for the proxy polygons.
  double poly_cs[2 * 512];
  // Element geometry (device pointer, kElemFields * n_nodes doubles).
  const double* elem;
  // The same geometry element-major for gathers: 8 doubles per element
  // {px, py, dx, dy, nx, ny, h, 0} (one 64-byte line per element).
  const double* elem8;
  const double* node_xy;  // 2 * n_nodes, interleaved x, y
};

__host__ __device__ inline int gauss_offset(int n) { return n * (n - 1) / 2; }

}  // namespace ebem_gpu
