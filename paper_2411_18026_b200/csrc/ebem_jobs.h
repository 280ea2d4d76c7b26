// Work descriptors the host runtime plans per tree level and the fill
// kernels consume.  Plain data, shared by host C++ and device code.
//
// The Galerkin fill is split the way the reference's scatter is organised
// (proj/src/assembly.cpp:373-407, :460-507): every (test element, trial
// element) pair produces a bundle of 16 complex numbers V[la][lb][i][j] =
// D + alpha N (+ M/2 on coincident diagonals); every output entry is then the
// sum of the (at most 2 x 2) bundles of the elements supporting its row and
// column hat functions, added in ascending (test element, trial element)
// order.
#pragma once

namespace ebem_gpu {

constexpr int kBundle = 16;  // complex numbers per element-pair bundle

// One row (or column) of an output block: the hat function of a node in one
// component.  e1 < e2 are the indices (into the job's element list) of the
// two supporting elements in ascending element order; la1/la2 are the local
// shape indices of the node on them (1 on element g-1, 0 on element g).
struct NodeDesc {
  int dest;  // destination row (column) index in the output matrix
  int e1, e2;
  int bits;  // la1 | la2 << 1 | comp << 2
};

// One proxy interaction job per cell: m' polygon elements x nE curve
// elements, both orientations from the same scalar evaluations.
// V bundle (polygon test, curve trial) at v_off + pe * nE + q,
// U bundle (curve test, polygon trial) at u_off + q * m' + pe.
struct ProxyJob {
  long long v_off, u_off;
  int e_off, nE;
  int block_off;  // first CTA of this job in the proxy launch
  int pad;
  double cx, cy, radius;
};

// Both near blocks of one cell from one scalar evaluation per point:
// pairs (a in enclosed elements A, q in cell elements E);
// V bundle (test A[a], trial E[q]) at v_off + a * nE + q,
// U bundle (test E[q], trial A[a]) at u_off + q * nA + a.
// tri = 1 (a diagonal block, A == E, u_off == v_off): only pairs a < q are
// evaluated; the U bundle of (a, q) is the V bundle of (q, a).
// onesided = 1 (a plain true_block(rows = A, cols = E)): V bundles only.
struct SymJob {
  long long v_off, u_off;
  long long local_off;  // first pair of this job in the wave's sym numbering
  int a_off, nA;
  int e_off, nE;
  int tri, onesided;
};

// Near-pair classes of the bucketing sort: tier (0..3 = far, far+2, far+5,
// far+9 points; 4 = very far, 3 points) + kSymTiers for one-sided jobs; the
// last class is "skip" (touching
// pairs, handled by k_near_singular, and the lower triangle of tri jobs).
constexpr int kSymTiers = 5;  // the reference's four tiers + the very-far 3 x 3 tier
constexpr int kSymClasses = 2 * kSymTiers + 1;
// Very-far pairs (segment distance >= kVeryFar x the longer element, default
// assembly settings only): a 3 x 3 rule instead of the reference's 4 x 4.  For
// these pairs both rules integrate the same smooth integrand to below
// rounding: the 3-point Gauss remainder h^7 f(6) / 2016000 of a 1/r^3-type
// kernel is 0.01 (h/r)^6 of the integral, 4e-17 at h/r = 1/250, a fraction
// of an ulp (EBEM_FAR3=0: the reference's tiers only).  (A 2 x 2 rule beyond
// 4000 element lengths, remainder (h/r)^4 / 12 = 3e-16, was measured too:
// faster still, but the far-pair cancellation of DESIGN.md section 5 turns
// those ulps into 1.3e-8 of the solution at N = 262144.)
constexpr double kVeryFar = 250.0;
constexpr int kVeryFarNodes = 3;

// Sorted near-pair record, 16 doubles (128 B): geometry of the enclosed
// element a and the cell element b (px, py, dx, dy, nx, ny each), the two
// bundle slots (as long long bit patterns), h_a h_b, padding.
constexpr int kSymRec = 16;
enum SymRecField { SR_A = 0, SR_B = 6, SR_VD = 12, SR_UD = 13, SR_HH = 14 };

// Scatter of bundles into one output block.
struct GatherJob {
  long long pair_off;   // bundle index of (row element 0, col element 0)
  long long entry_off;  // first entry of this job in the gather launch
  int nces;             // bundle row stride (column elements)
  int rdesc_off, nrows;
  int cdesc_off, ncols;
  int trans;  // 1: write conj(v) at (col dest, row dest)
  int ld;
  double* dest;  // interleaved complex, column-major
};

// Entries of a cell's interaction matrix that its child already holds: for
// every listed (child column, cell column) and (child enclosed position,
// cell enclosed position) pair, both displacement components of the enclosed
// node are copied from the child's matrix (previous level) into the cell's.
struct ReuseTask {
  const double* src;  // child matrix, interleaved complex, column-major
  double* dst;        // cell matrix
  int src_ld, dst_ld;
  int src_row0, src_ne;  // enclosed rows of component p start at row0 + p * ne
  int dst_row0, dst_ne;
  int n_rows, n_cols;    // listed pairs
  long long row_off;     // first (child, cell) enclosed position pair
  long long col_off;     // first (child, cell) column pair
};

// Generic entry copy between two column-major complex matrices: entry
// (row pair r, column pair c) goes to dst(rows[r].y, cols[c].y) from
// src(rows[r].x, cols[c].x), or, with swap, from conj(src(cols[c].x, rows[r].x)).
struct MapTask {
  const double* src;
  double* dst;
  int src_ld, dst_ld;
  int n_rows, n_cols;
  int swap, pad;
  long long row_off, col_off;
};

}  // namespace ebem_gpu
