// Host-callable launch wrappers of the sm_100a kernels (defined in *.cu).
#pragma once

#include <cuda_runtime.h>

#include "ebem_ctx.h"
#include "ebem_jobs.h"

namespace ebem_gpu {

// ---- fill (ebem_fill.cu)
// Bundles (element-pair results, kBundle complex each) are stored
// component-plane major over the wave's nb slots (bslot in ebem_fill.cu).
void launch_near_singular(const DevCtx* ctx, const long long* pairs,
                          const int* pair_elems, int n, double* bundles, long long nb,
                          int* bad, cudaStream_t st);
// Bucketing of the wave's symmetric near pairs by class (count pass, then a
// scatter pass that writes each non-skipped pair's record, kSymRec doubles:
// both elements' geometry, the two bundle slots, the Jacobian product, into
// its class range).  bounds holds sym_bounds_ints() ints: the class starts
// bounds[0..kSymClasses] (bounds[kSymClasses] = n_pairs), then counters.
void launch_sym_bucket(const DevCtx* ctx, const SymJob* jobs, const long long* job_off,
                       int n_jobs, const int* elems, long long n_pairs,
                       unsigned char* keys, int* pair_job, int* bounds, double* recs,
                       cudaStream_t st);
int sym_bounds_ints();
// One launch per near-pair class cls; the class's range of the bucketed pair
// records is read from class_bounds on the device (max_count bounds the grid).
void launch_near_sym(const DevCtx* ctx, const FillConst& fc, const double* recs, const int* class_bounds,
                     int cls, long long max_count, int n, bool both, double* bundles,
                     long long nb, cudaStream_t st);
int proxy_blocks_for(int m_prime, int nE, int n_gauss);
// Proxy blocks: writes the slot records into recs (proxy_blocks x
// proxy_pairs_per_block(n_gauss) x kSymRec doubles), then evaluates them.
int proxy_pairs_per_block(int n_gauss);
void launch_proxy_pairs(const DevCtx* ctx, const FillConst& fc, int n_gauss,
                        const ProxyJob* jobs, const int* job_block_off, int n_jobs,
                        int n_blocks, const int* elems, double* recs, double* bundles,
                        long long nb, cudaStream_t st);
constexpr int kGatherTile = 256;  // output entries per gather CTA
void launch_gather(const GatherJob* jobs, const int* job_block_off, int n_jobs,
                   int n_blocks, const NodeDesc* desc, const double* bundles,
                   long long nb, cudaStream_t st);
// Cross-level reuse: copies the listed entries of the children's interaction
// matrices into the cells' (kReuseCols columns per CTA, one warp each).
constexpr int kReuseCols = 4;
void launch_reuse_copy(const ReuseTask* tasks, const int* task_block_off, int n_tasks,
                       int n_blocks, const int2* row_pairs, const int2* col_pairs,
                       cudaStream_t st);
// Entry copies of the sibling blocks (one CTA per task).
void launch_map_copy(const MapTask* tasks, int n_tasks, const int2* row_pairs,
                     const int2* col_pairs, cudaStream_t st);

// ---- incident-field right-hand sides (ebem_rhs.cu)
// Post-processing (proj/src/postprocess.cpp): distance of m points to the
// boundary, and the scattered (+ incident) displacement at m points.
void launch_boundary_distance(const DevCtx* ctx, const double* pts, int m, double* out,
                              cudaStream_t st);
void launch_field(const DevCtx* ctx, const double* bu, const double* pts, int m, int ng,
                  int kind, double angle, double amp, double* out_u, double* out_int,
                  cudaStream_t st);
void launch_rhs_plane(const DevCtx* ctx, int n_nodes, int kind,
                      const double* angles, int m, double amplitude, int rhs_n,
                      double* out, cudaStream_t st);

// ---- special functions, exposed for parity tests (ebem_rhs.cu)
double measure_fp64_peak_tflops();
void launch_eval_hankel(const double* x, int n, double* out, cudaStream_t st);
void launch_eval_scalars(const DevCtx* ctx, const double* r, int n, int which,
                         double* out, cudaStream_t st);

}  // namespace ebem_gpu
