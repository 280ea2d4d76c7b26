// The C ABI (include/ebem_gpu.h): argument checks, exception-to-status
// mapping, host<->device copies around the runtime classes.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>

#include "ebem_kernels.h"
#include "medium_setup.h"
#include "runtime.h"

using namespace ebem_gpu;

struct ebem_gpu_problem {
  Problem* p;
};
struct ebem_gpu_conv {
  Conv* c;
};

struct ebem_gpu_fds {
  Fds* f;
  Problem* own = nullptr;  // source-only problem owned by the solver
  HostSource hs{};
};

namespace {

thread_local std::string g_err;

std::recursive_mutex& api_mutex() {
  static std::recursive_mutex m;
  return m;
}

template <class F>
int guarded(F&& f) {
  std::lock_guard<std::recursive_mutex> lock(api_mutex());
  try {
    f();
    return EBEM_OK;
  } catch (const Error& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return EBEM_LENGTH_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return EBEM_RUNTIME_ERROR;
  }
}

Lists lists(const int* a, int na, const int* b, int nb) {
  if (na < 0 || nb < 0) throw Error(EBEM_INVALID_ARGUMENT, "negative list length");
  return {std::vector<int>(a, a + na), std::vector<int>(b, b + nb)};
}

void check_nodes(const Lists& l, int n) {
  for (int p = 0; p < 2; ++p)
    for (int g : l[p])
      if (g < 0 || g >= n) throw Error(EBEM_INVALID_ARGUMENT, "node index out of range");
}

ebem_assembly_config default_assembly() {
  ebem_assembly_config a;
  a.corner_nodes = 10;
  a.far_nodes = 4;
  a.rhs_nodes = 8;
  a.refine = 1.0;
  a.max_dense_bytes = size_t(4) << 30;
  return a;
}

ebem_proxy_config default_proxy() {
  ebem_proxy_config p;
  p.radius_factor = 1.5;
  p.m_prime = 64;
  p.n_gauss = 6;
  return p;
}

}  // namespace

extern "C" {

const char* ebem_gpu_last_error(void) { return g_err.c_str(); }

long long ebem_gpu_launch_count(void) { return g_launches.load(); }

int ebem_gpu_prof_enable(int on) {
  return guarded([&] {
    g_prof.collect();
    g_prof.on = on != 0;
  });
}

int ebem_gpu_prof_bytes(double* bytes, int n) {
  return guarded([&] {
    g_prof.collect();
    for (int i = 0; i < n && i < KP_COUNT; ++i) bytes[i] = g_prof.bytes[i];
  });
}

int ebem_gpu_prof_read(int reset, double* ms, long long* count, double* units,
                       int n) {
  return guarded([&] {
    g_prof.collect();
    for (int i = 0; i < n && i < KP_COUNT; ++i) {
      ms[i] = g_prof.ms[i];
      count[i] = g_prof.count[i];
      units[i] = g_prof.units[i];
    }
    if (reset) g_prof.reset();
  });
}

const char* ebem_gpu_prof_name(int id) { return kernel_name(id); }

int ebem_gpu_fp64_peak(double* tflops) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      throw Error(EBEM_CUDA_ERROR, "no CUDA device");
    *tflops = measure_fp64_peak_tflops();
    CK(cudaGetLastError());
  });
}
int ebem_gpu_prof_kernels(void) { return KP_COUNT; }

int ebem_gpu_device_info(char* buf, int len) {
  return guarded([&] {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
      throw Error(EBEM_CUDA_ERROR, "no CUDA device");
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    if (buf && len > 0)
      std::snprintf(buf, size_t(len), "%s sm_%d%d %d SMs %.1f GiB", prop.name,
                    prop.major, prop.minor, prop.multiProcessorCount,
                    prop.totalGlobalMem / double(1 << 30));
  });
}

int ebem_gpu_problem_create(const double* nodes_xy, int n_nodes, double lambda,
                            double mu, double rho, double omega,
                            double alpha_re, double alpha_im,
                            const ebem_assembly_config* assembly,
                            const ebem_proxy_config* proxy,
                            ebem_gpu_problem** out) {
  return guarded([&] {
    if (!out || !nodes_xy) throw Error(EBEM_INVALID_ARGUMENT, "null argument");
    const ebem_assembly_config a = assembly ? *assembly : default_assembly();
    const ebem_proxy_config p = proxy ? *proxy : default_proxy();
    auto* h = new ebem_gpu_problem{nullptr};
    try {
      h->p = new Problem(nodes_xy, n_nodes, lambda, mu, rho, omega, alpha_re,
                         alpha_im, a, p);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

void ebem_gpu_problem_destroy(ebem_gpu_problem* p) {
  if (!p) return;
  std::lock_guard<std::recursive_mutex> lock(api_mutex());
  delete p->p;
  delete p;
}

int ebem_gpu_problem_size(const ebem_gpu_problem* p) { return p ? p->p->n() : -1; }

int ebem_gpu_true_block(ebem_gpu_problem* p, const int* rows0, int nr0,
                        const int* rows1, int nr1, const int* cols0, int nc0,
                        const int* cols1, int nc1, double* out) {
  return guarded([&] {
    const Lists r = lists(rows0, nr0, rows1, nr1);
    const Lists c = lists(cols0, nc0, cols1, nc1);
    check_nodes(r, p->p->n());
    check_nodes(c, p->p->n());
    p->p->true_block_host(r, c, out);
  });
}

int ebem_gpu_cell_mats(ebem_gpu_problem* p, const int* rows0, int nr0,
                       const int* rows1, int nr1, const int* cols0, int nc0,
                       const int* cols1, int nc1, int node_begin, int node_end,
                       int* n_out, double* mv, double* mu) {
  return guarded([&] {
    Problem& P = *p->p;
    const Lists r = lists(rows0, nr0, rows1, nr1);
    const Lists c = lists(cols0, nc0, cols1, nc1);
    check_nodes(r, P.n());
    check_nodes(c, P.n());
    const ProxyGeom g = P.build_proxy(node_begin, node_end);
    const int no = 2 * P.proxy_cfg().m_prime + 2 * int(g.enclosed.size());
    *n_out = no;
    if (!mv || !mu) return;
    std::vector<BasisReq> req{BasisReq{&r, &c, node_begin, node_end}};
    std::vector<ProxyGeom> geom;
    std::vector<size_t> tv, tu;
    std::vector<int> nout;
    DBuf<double> tbuf;
    P.interaction(req, geom, tv, tu, nout, tbuf);
    P.check_domain();
    const int ncol = nc0 + nc1, nrow = nr0 + nr1;
    CK(cudaMemcpyAsync(mv, tbuf.get() + 2 * tv[0], 16 * size_t(no) * ncol,
                       cudaMemcpyDeviceToHost, P.stream()));
    std::vector<double> tuh(2 * size_t(no) * nrow);
    CK(cudaMemcpyAsync(tuh.data(), tbuf.get() + 2 * tu[0], 16 * size_t(no) * nrow,
                       cudaMemcpyDeviceToHost, P.stream()));
    CK(cudaStreamSynchronize(P.stream()));
    // mu = T_U^H
    for (int i = 0; i < nrow; ++i)
      for (int j = 0; j < no; ++j) {
        const double* s = tuh.data() + 2 * (size_t(i) * no + j);
        double* d = mu + 2 * (size_t(j) * nrow + i);
        d[0] = s[0];
        d[1] = -s[1];
      }
  });
}

int ebem_gpu_build_proxy(ebem_gpu_problem* p, int node_begin, int node_end,
                         double* out3, int* n_enclosed, int* enclosed, int cap) {
  return guarded([&] {
    const ProxyGeom g = p->p->build_proxy(node_begin, node_end);
    out3[0] = g.cx;
    out3[1] = g.cy;
    out3[2] = g.radius;
    *n_enclosed = int(g.enclosed.size());
    if (enclosed && cap >= int(g.enclosed.size()))
      std::memcpy(enclosed, g.enclosed.data(), 4 * g.enclosed.size());
  });
}

int ebem_gpu_cell_basis(ebem_gpu_problem* p, const int* rows0, int nr0,
                        const int* rows1, int nr1, const int* cols0, int nc0,
                        const int* cols1, int nc1, int node_begin, int node_end,
                        double epsilon, int* k, int* saturated, int* skel,
                        double* u0, double* u1, double* v0, double* v1) {
  return guarded([&] {
    Problem& P = *p->p;
    if (!(epsilon > 0.0))
      throw Error(EBEM_INVALID_ARGUMENT, "Cpqr: truncation epsilon must be positive");
    const Lists r = lists(rows0, nr0, rows1, nr1);
    const Lists c = lists(cols0, nc0, cols1, nc1);
    check_nodes(r, P.n());
    check_nodes(c, P.n());
    std::vector<BasisReq> req{BasisReq{&r, &c, node_begin, node_end}};
    std::vector<BasisRes> res;
    DBuf<double> vb, ub;
    P.bases(req, epsilon, res, vb, ub);
    const BasisRes& b = res[0];
    *k = b.k;
    *saturated = b.saturated ? 1 : 0;
    if (!skel) return;
    const int kk = b.k;
    for (int i = 0; i < kk; ++i) {
      skel[i] = b.srow[0][i];
      skel[kk + i] = b.srow[1][i];
      skel[2 * kk + i] = b.scol[0][i];
      skel[3 * kk + i] = b.scol[1][i];
    }
    if (kk == 0) return;
    const double* vd = vb.get() + 2 * b.v_off;
    const double* ud = ub.get() + 2 * b.u_off;
    CK(cudaMemcpyAsync(v0, vd, 16 * size_t(kk) * nc0, cudaMemcpyDeviceToHost, P.stream()));
    CK(cudaMemcpyAsync(v1, vd + 2 * size_t(kk) * nc0, 16 * size_t(kk) * nc1,
                       cudaMemcpyDeviceToHost, P.stream()));
    CK(cudaMemcpyAsync(u0, ud, 16 * size_t(kk) * nr0, cudaMemcpyDeviceToHost, P.stream()));
    CK(cudaMemcpyAsync(u1, ud + 2 * size_t(kk) * nr0, 16 * size_t(kk) * nr1,
                       cudaMemcpyDeviceToHost, P.stream()));
    CK(cudaStreamSynchronize(P.stream()));
  });
}

int ebem_gpu_cell_bases(ebem_gpu_problem* p, int count, const int* begins,
                        const int* ends, double epsilon, int* k_out,
                        int* skel_out, double* device_seconds) {
  return guarded([&] {
    Problem& P = *p->p;
    if (count < 0) throw Error(EBEM_INVALID_ARGUMENT, "negative cell count");
    std::vector<Lists> lists_(count);
    std::vector<BasisReq> req(count);
    for (int c = 0; c < count; ++c) {
      if (begins[c] < 0 || ends[c] > P.n() || begins[c] >= ends[c])
        throw Error(EBEM_INVALID_ARGUMENT, "build_proxy: bad node range");
      std::vector<int> r(ends[c] - begins[c]);
      for (int i = 0; i < int(r.size()); ++i) r[i] = begins[c] + i;
      lists_[c] = Lists{r, r};
      req[c] = BasisReq{&lists_[c], &lists_[c], begins[c], ends[c]};
    }
    std::vector<BasisRes> res;
    DBuf<double> vb, ub;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0, P.stream()));
    P.bases(req, epsilon, res, vb, ub);
    CK(cudaEventRecord(e1, P.stream()));
    CK(cudaEventSynchronize(e1));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (device_seconds) *device_seconds = 1e-3 * ms;
    size_t o = 0;
    for (int c = 0; c < count; ++c) {
      k_out[c] = res[c].k;
      if (!skel_out) continue;
      for (const auto* l : {&res[c].srow[0], &res[c].srow[1], &res[c].scol[0],
                            &res[c].scol[1]})
        for (int v : *l) skel_out[o++] = v;
    }
  });
}

int ebem_gpu_series_table(double lambda, double mu, double rho, double omega,
                          double* out, int max_pow, int* max_q) {
  return guarded([&] {
    if (max_pow < 1) throw Error(EBEM_INVALID_ARGUMENT, "table too short");
    const DevMedium m = make_medium(lambda, mu, rho, omega, 0.0, 0.0);
    const int q = build_series(m, out, max_pow);
    if (max_q) *max_q = q;
  });
}

int ebem_gpu_gauss_rule(int n, double* x, double* w) {
  return guarded([&] {
    if (n < 1 || n > 64) throw Error(EBEM_INVALID_ARGUMENT, "gauss_rule: order out of range");
    gauss_rule(n, x, w);
  });
}

int ebem_gpu_rhs_plane(ebem_gpu_problem* p, int kind, const double* angles,
                       int m, double amplitude, double* out) {
  return guarded([&] {
    if (kind != 0 && kind != 1) throw Error(EBEM_INVALID_ARGUMENT, "unknown wave kind");
    p->p->rhs_plane(kind, angles, m, amplitude, out);
  });
}

int ebem_gpu_fds_create(ebem_gpu_problem* p, int depth,
                        const ebem_fds_config* cfg, ebem_gpu_fds** out,
                        ebem_fds_stats* stats) {
  return guarded([&] {
    ebem_fds_config c;
    c.epsilon = 1e-8;
    c.ell0 = 1;
    if (cfg) c = *cfg;
    auto* h = new ebem_gpu_fds{};
    try {
      h->f = new Fds(*p->p, depth, c);
    } catch (...) {
      delete h;
      throw;
    }
    if (stats) *stats = h->f->stats();
    *out = h;
  });
}

int ebem_gpu_field(ebem_gpu_problem* p, const double* boundary_u, const double* points_xy,
                   int m, int n_gauss, int wave_kind, double angle, double amplitude,
                   double* out_u, double* out_intensity) {
  return guarded([&] {
    if (!p || (m > 0 && (!boundary_u || !points_xy || !out_u)))
      throw Error(EBEM_INVALID_ARGUMENT, "evaluate_scattered: null argument");
    if (wave_kind > 1) throw Error(EBEM_INVALID_ARGUMENT, "evaluate_field: unknown wave kind");
    p->p->field(boundary_u, points_xy, m, n_gauss, wave_kind, angle, amplitude, out_u,
                out_intensity);
  });
}

int ebem_gpu_dense(ebem_gpu_problem* p, double* out) {
  return guarded([&] {
    if (!p || !out) throw Error(EBEM_INVALID_ARGUMENT, "dense: null argument");
    Conv::dense_host(*p->p, out);
  });
}

int ebem_gpu_conv_create(ebem_gpu_problem* p, ebem_gpu_conv** out,
                         ebem_conv_stats* stats) {
  return guarded([&] {
    if (!p || !out) throw Error(EBEM_INVALID_ARGUMENT, "ConvSolver: null argument");
    *out = nullptr;
    std::unique_ptr<Conv> c(new Conv(*p->p));
    if (stats) {
      const ConvStatsC& s = c->stats();
      stats->assemble_seconds = s.assemble_seconds;
      stats->factor_seconds = s.factor_seconds;
      stats->rcond = s.rcond;
      stats->min_pivot = s.min_pivot;
      stats->condition_warning = s.condition_warning ? 1 : 0;
    }
    *out = new ebem_gpu_conv{c.release()};
  });
}

int ebem_gpu_conv_solve(ebem_gpu_conv* c, const double* rhs, int m, double* x) {
  return guarded([&] {
    if (!c || (m > 0 && (!rhs || !x)))
      throw Error(EBEM_INVALID_ARGUMENT, "ConvSolver: null argument");
    if (m < 0) throw Error(EBEM_INVALID_ARGUMENT, "ConvSolver: negative column count");
    c->c->solve_host(rhs, m, x);
  });
}

void ebem_gpu_conv_destroy(ebem_gpu_conv* c) {
  if (!c) return;
  std::lock_guard<std::recursive_mutex> lock(api_mutex());
  delete c->c;
  delete c;
}

void ebem_gpu_fds_destroy(ebem_gpu_fds* f) {
  if (!f) return;
  std::lock_guard<std::recursive_mutex> lock(api_mutex());
  delete f->f;
  delete f->own;
  delete f;
}

int ebem_gpu_fds_create_source(int n_nodes, int depth, const ebem_fds_config* cfg,
                               ebem_block_fn block, ebem_basis_fn basis,
                               void* user, ebem_gpu_fds** out,
                               ebem_fds_stats* stats) {
  return guarded([&] {
    if (!block || !basis || !out) throw Error(EBEM_INVALID_ARGUMENT, "null argument");
    ebem_fds_config c;
    c.epsilon = 1e-8;
    c.ell0 = 1;
    if (cfg) c = *cfg;
    auto* h = new ebem_gpu_fds{};
    try {
      h->hs = HostSource{block, basis, user};
      h->own = new Problem(n_nodes);
      h->f = new Fds(*h->own, depth, c, &h->hs);
    } catch (...) {
      delete h->f;
      delete h->own;
      delete h;
      throw;
    }
    if (stats) *stats = h->f->stats();
    *out = h;
  });
}

int ebem_gpu_fds_solve(ebem_gpu_fds* f, const double* rhs, int m, double* x,
                       ebem_fds_solve_timing* timing) {
  return guarded([&] {
    if (m < 0) throw Error(EBEM_INVALID_ARGUMENT, "negative column count");
    if (m == 0) return;
    Problem& P = f->f->problem();
    const size_t bytes = 32 * size_t(P.n()) * m;
    DBuf<double> d;
    d.alloc(4 * size_t(P.n()) * m);
    CK(cudaMemcpyAsync(d.get(), rhs, bytes, cudaMemcpyHostToDevice, P.stream()));
    f->f->solve_device(d.get(), m, d.get(), timing);
    CK(cudaMemcpyAsync(x, d.get(), bytes, cudaMemcpyDeviceToHost, P.stream()));
    CK(cudaStreamSynchronize(P.stream()));
  });
}

int ebem_gpu_fds_solve_device(ebem_gpu_fds* f, const double* rhs_dev, int m,
                              double* x_dev) {
  return guarded([&] {
    if (m <= 0) return;
    f->f->solve_device(rhs_dev, m, x_dev, nullptr);
  });
}

int ebem_gpu_fds_rank_of(const ebem_gpu_fds* f, int cell) {
  return f->f->rank_of(cell);
}

int ebem_gpu_fds_cell(const ebem_gpu_fds* f, int cell, int* sizes, int* skel) {
  return guarded([&] { f->f->cell_info(cell, sizes, skel); });
}

// Debug hook: copies a cell's device factor (0 lu, 1 ipiv, 2 A^-1 U, 3 V,
// 4 atilde) to host memory.
int ebem_gpu_fds_debug_cell(const ebem_gpu_fds* f, int cell, int which,
                            double* out) {
  return guarded([&] { f->f->debug_cell(cell, which, out); });
}

int ebem_gpu_eval_hankel(const double* x, int n, double* out) {
  return guarded([&] {
    if (n <= 0) return;
    scratch();  // the device check (no CPU fallback)
    DBuf<double> dx, dout;
    dx.alloc(n);
    dout.alloc(4 * size_t(n));
    copy_sync(dx.get(), x, 8 * size_t(n));
    launch_eval_hankel(dx.get(), n, dout.get(), scratch_stream());
    ++g_launches;  // test hook
    CK(cudaGetLastError());
    copy_sync(out, dout.get(), 32 * size_t(n));
  });
}

int ebem_gpu_tall_reduce(const double* a, int rows, int n, int ld, double* r,
                         int* r_rows) {
  return guarded([&] {
    if (rows <= 0 || n <= 0 || ld < rows || !a || !r || !r_rows)
      throw Error(EBEM_INVALID_ARGUMENT, "tall_reduce: bad arguments");
    scratch();
    cudaStream_t st = scratch_stream();
    DBuf<double> da;
    da.alloc(2 * size_t(ld) * n);
    copy_sync(da.get(), a, 16 * size_t(ld) * n);
    std::vector<TallBlock> q{TallBlock{da.get(), rows, n, ld}};
    reduce_tall(q, st, true);
    ++g_launches;  // test hook
    CK(cudaGetLastError());
    const TallBlock& x = q[0];
    std::vector<double> tmp(2 * size_t(x.ld) * n);
    copy_sync(tmp.data(), x.p, 16 * size_t(x.ld) * n);
    for (int j = 0; j < n; ++j)
      std::memcpy(r + 2 * size_t(j) * x.rows, tmp.data() + 2 * size_t(j) * x.ld,
                  16 * size_t(x.rows));
    *r_rows = x.rows;
  });
}

int ebem_gpu_eval_scalars(ebem_gpu_problem* p, const double* r, int n,
                          int which, double* out) {
  return guarded([&] {
    if (n <= 0) return;
    Problem& P = *p->p;
    DBuf<double> dr, dout;
    dr.alloc(n);
    dout.alloc(20 * size_t(n));
    CK(cudaMemcpyAsync(dr.get(), r, 8 * size_t(n), cudaMemcpyHostToDevice, P.stream()));
    launch_eval_scalars(P.dctx(), dr.get(), n, which, dout.get(), P.stream());
    ++g_launches;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(out, dout.get(), 160 * size_t(n), cudaMemcpyDeviceToHost, P.stream()));
    CK(cudaStreamSynchronize(P.stream()));
  });
}

}  // extern "C"
