// Native host runtime: planning and driving the batched sm_100a kernels.
//
// Reference behaviour mirrored here (the arithmetic itself runs on device):
//   build_proxy                   proj/src/compression.cpp:25-69
//   AssemblerSource::cell_basis   proj/src/compression.cpp:132-169
//   basis_from_interactions       proj/src/compression.cpp:71-118
//   BlockAssembler::true_block    proj/src/assembly.cpp:332-409 (element sets,
//                                 scatter order)
//   FdsSolver::build / solve      proj/src/fds.cpp:56-263
#include "runtime.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <limits>
#include <cstdio>
#include <cstdlib>
#include <condition_variable>
#include <exception>
#include <mutex>
#include <thread>

#include "ebem_kernels.h"
#include "medium_setup.h"

namespace ebem_gpu {

std::atomic<long long> g_launches{0};
Profiler g_prof;

namespace {
double wall_now() {
  return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}
std::vector<std::pair<std::string, double>>& phases() {
  static std::vector<std::pair<std::string, double>> v;
  return v;
}
}  // namespace

int verbose_level() {
  static const int v = [] {
    const char* e = std::getenv("EBEM_VERBOSE");
    return e ? std::atoi(e) : 0;
  }();
  return v;
}

void host_phase_add(const char* name, double seconds) {
  for (auto& kv : phases())
    if (kv.first == name) {
      kv.second += seconds;
      return;
    }
  phases().emplace_back(name, seconds);
}

void host_phase_dump() {
  if (!verbose_level()) return;
  double tot = 0.0;
  for (auto& kv : phases()) tot += kv.second;
  std::fprintf(stderr, "[ebem] host phases (total %.3f s):\n", tot);
  for (auto& kv : phases())
    std::fprintf(stderr, "[ebem]   %-18s %8.3f s\n", kv.first.c_str(), kv.second);
  phases().clear();
}

PhaseTimer::PhaseTimer(const char* name, cudaStream_t st)
    : name_(name), st_(st), t0_(verbose_level() ? wall_now() : 0.0) {}

PhaseTimer::~PhaseTimer() {
  if (!verbose_level()) return;
  if (verbose_level() >= 2 && st_) cudaStreamSynchronize(st_);
  host_phase_add(name_, wall_now() - t0_);
}

const char* kernel_name(int id) {
  static const char* names[KP_COUNT] = {
      "k_proxy_pairs", "k_near_onesided", "k_near_singular", "k_gather",
      "k_qr_reduce", "k_cpqr", "k_interp", "k_getrf", "k_getrs", "k_gemm",
      "k_copy", "k_rhs_plane", "k_near_sym", "k_sym_bucket", "k_reuse_copy"};
  return (id >= 0 && id < KP_COUNT) ? names[id] : "?";
}

cudaEvent_t Profiler::ev() {
  if (!pool_.empty()) {
    cudaEvent_t e = pool_.back();
    pool_.pop_back();
    return e;
  }
  cudaEvent_t e;
  CK(cudaEventCreate(&e));
  return e;
}

void Profiler::begin(cudaStream_t st) {
  if (!on) return;
  cur_ = ev();
  CK(cudaEventRecord(cur_, st));
}

void Profiler::end(int id, cudaStream_t st, double u, double by) {
  ++g_launches;
  if (!on || !cur_) return;
  cudaEvent_t b = ev();
  CK(cudaEventRecord(b, st));
  pending_.push_back(Rec{id, cur_, b, u, -1, by});
  cur_ = nullptr;
}

void Profiler::end_counted(int id, cudaStream_t st, const int* dev_bounds, double mult) {
  ++g_launches;
  if (!on || !cur_) return;
  cudaEvent_t b = ev();
  CK(cudaEventRecord(b, st));
  if (counts_used_ == counts_cap_) {  // pinned pairs, grown by doubling
    int* nc = nullptr;
    const int cap = counts_cap_ ? 2 * counts_cap_ : 256;
    CK(cudaMallocHost(reinterpret_cast<void**>(&nc), sizeof(int) * 2 * cap));
    if (counts_) {
      CK(cudaStreamSynchronize(st));
      std::memcpy(nc, counts_, sizeof(int) * 2 * counts_used_);
      CK(cudaFreeHost(counts_));
    }
    counts_ = nc;
    counts_cap_ = cap;
  }
  const int slot = counts_used_++;
  CK(cudaMemcpyAsync(counts_ + 2 * slot, dev_bounds, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
  pending_.push_back(Rec{id, cur_, b, mult, slot, 0.0});
  cur_ = nullptr;
}

void Profiler::collect() {
  if (pending_.empty()) return;
  CK(cudaDeviceSynchronize());
  for (Rec& r : pending_)
    if (r.slot >= 0) r.units *= double(counts_[2 * r.slot + 1] - counts_[2 * r.slot]);
  counts_used_ = 0;
  for (size_t k = 0; k < pending_.size(); ++k) {
    const Rec& r = pending_[k];
    float t = 0.f;
    CK(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.id] += t;
    count[r.id] += 1;
    units[r.id] += r.units;
    bytes[r.id] += r.bytes;
    if (k > 0) {  // one stream: the span between two recorded kernels
      float g = 0.f;
      CK(cudaEventElapsedTime(&g, pending_[k - 1].b, r.a));
      gap_ms[r.id] += g;
    }
  }
  for (const Rec& r : pending_) {
    pool_.push_back(r.a);
    pool_.push_back(r.b);
  }
  if (verbose_level() >= 1 && !pending_.empty()) {
    double tot = 0.0;
    for (int i = 0; i < KP_COUNT; ++i) tot += gap_ms[i];
    std::fprintf(stderr, "[ebem] device gaps before kernels (total %.1f ms):", tot);
    for (int i = 0; i < KP_COUNT; ++i)
      if (gap_ms[i] > 0.05) std::fprintf(stderr, " %s %.1f", kernel_name(i), gap_ms[i]);
    std::fprintf(stderr, "\n");
  }
  pending_.clear();
}

void Profiler::reset() {
  collect();
  for (int i = 0; i < KP_COUNT; ++i)
    ms[i] = 0.0, count[i] = 0, units[i] = 0.0, bytes[i] = 0.0, gap_ms[i] = 0.0;
}

void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(EBEM_CUDA_ERROR, std::string("CUDA error in ") + what + ": " +
                                     cudaGetErrorString(e));
}

Staging::~Staging() {
  for (Slot& x : s_) {
    if (x.ev) cudaEventSynchronize(x.ev);
    if (x.up) cudaEventSynchronize(x.up);
    if (x.host) cudaFreeHost(x.host);
    if (x.dev) cudaFree(x.dev);
    if (x.ev) cudaEventDestroy(x.ev);
    if (x.up) cudaEventDestroy(x.up);
  }
  if (copy_) cudaStreamDestroy(copy_);
}

static double g_staged_bytes = 0.0;  // timeline statistics
static long g_staged_copies = 0;
char* Staging::put(const Pack& pk, cudaStream_t st) {
  cur_ = (cur_ + 1) % int(s_.size());
  Slot& x = s_[cur_];
  if (!x.ev) CK(cudaEventCreateWithFlags(&x.ev, cudaEventDisableTiming));
  if (!x.up) CK(cudaEventCreateWithFlags(&x.up, cudaEventDisableTiming));
  if (!copy_) CK(cudaStreamCreateWithFlags(&copy_, cudaStreamNonBlocking));
  if (x.pending) {  // the slot's previous kernels (and so its upload) are done
    CK(cudaEventSynchronize(x.ev));
    x.pending = false;
  }
  if (x.uploading) {  // a put without a fence: its copy may still read x.host
    CK(cudaEventSynchronize(x.up));
    x.uploading = false;
  }
  const size_t bytes = pk.bytes();
  if (bytes > x.cap) {
    // grow to the largest size any slot has needed so far: the slots rotate,
    // and each regrowth frees device memory (a device-wide synchronisation)
    static size_t high_water = 0;
    high_water = std::max(high_water, std::max(std::max(bytes + bytes / 2, 2 * x.cap), size_t(32) << 20));
    const size_t cap = high_water;
    if (x.host) CK(cudaFreeHost(x.host));
    if (x.dev) CK(cudaFree(x.dev));
    CK(cudaMallocHost(reinterpret_cast<void**>(&x.host), cap));
    CK(cudaMalloc(reinterpret_cast<void**>(&x.dev), cap));
    x.cap = cap;
  }
  if (bytes) {
    std::memcpy(x.host, pk.data(), bytes);
    CK(cudaMemcpyAsync(x.dev, x.host, bytes, cudaMemcpyHostToDevice, copy_));
    CK(cudaEventRecord(x.up, copy_));
    CK(cudaStreamWaitEvent(st, x.up, 0));
    x.uploading = true;
    g_staged_bytes += double(bytes);
    ++g_staged_copies;
  }
  return x.dev;
}

void Staging::fence(cudaStream_t st) {
  if (cur_ < 0) return;
  Slot& x = s_[cur_];
  CK(cudaEventRecord(x.ev, st));
  x.pending = true;
}

void Pack::upload(DBuf<char>& dev, cudaStream_t st) {
  if (buf_.empty()) return;
  dev.ensure(buf_.size());
  CK(cudaMemcpyAsync(dev.get(), buf_.data(), buf_.size(), cudaMemcpyHostToDevice, st));
}

namespace {

double now() {
  return std::chrono::duration<double>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

constexpr long long kMaxBundlesPerWave = 8ll << 20;  // 2 GiB of bundles
// The first wave of a plan is closed at the end of the first planning batch
// that brings it to this size: the device starts while the host plans on.
constexpr long long kFirstWaveBundles = 1ll << 20;

}  // namespace

// ------------------------------------------------------------ NodeBoxTree
int NodeBoxTree::make(const double* xy, int lo, int hi) {
  Box b{lo, hi, -1, -1, 0, 0, 0, 0};
  if (hi - lo <= 16) {
    b.x0 = b.y0 = std::numeric_limits<double>::infinity();
    b.x1 = b.y1 = -std::numeric_limits<double>::infinity();
    for (int g = lo; g < hi; ++g) {
      b.x0 = std::min(b.x0, xy[2 * g]);
      b.x1 = std::max(b.x1, xy[2 * g]);
      b.y0 = std::min(b.y0, xy[2 * g + 1]);
      b.y1 = std::max(b.y1, xy[2 * g + 1]);
    }
  } else {
    const int mid = lo + (hi - lo) / 2;
    b.left = make(xy, lo, mid);
    b.right = make(xy, mid, hi);
    const Box& L = boxes_[b.left];
    const Box& R = boxes_[b.right];
    b.x0 = std::min(L.x0, R.x0);
    b.x1 = std::max(L.x1, R.x1);
    b.y0 = std::min(L.y0, R.y0);
    b.y1 = std::max(L.y1, R.y1);
  }
  boxes_.push_back(b);
  return int(boxes_.size()) - 1;
}

void NodeBoxTree::build(const double* xy, int n) {
  boxes_.clear();
  boxes_.reserve(size_t(n / 8 + 4));
  root_ = make(xy, 0, n);
}

void NodeBoxTree::enclosed(const double* xy, double cx, double cy,
                           double radius, int begin, int end,
                           std::vector<int>& out) const {
  out.clear();
  // explicit stack, left before right -> ascending node order
  int stack[128];
  int sp = 0;
  stack[sp++] = root_;
  const double slack = radius * (1.0 + 1e-9) + 1e-300;
  while (sp) {
    const Box& b = boxes_[stack[--sp]];
    const double dx = std::max(std::max(b.x0 - cx, cx - b.x1), 0.0);
    const double dy = std::max(std::max(b.y0 - cy, cy - b.y1), 0.0);
    if (std::hypot(dx, dy) > slack) continue;
    if (b.left < 0) {
      for (int g = b.lo; g < b.hi; ++g) {
        if (g >= begin && g < end) continue;
        // exactly the reference predicate: (node - center).norm() < radius
        if (std::hypot(xy[2 * g] - cx, xy[2 * g + 1] - cy) < radius)
          out.push_back(g);
      }
    } else {
      stack[sp++] = b.right;
      stack[sp++] = b.left;
    }
  }
}

// ------------------------------------------------------------- timeline
// EBEM_TIMELINE=1 (development aid): events + host clocks at the level
// loop's hand-off points; printed after the build as (GPU ms, host ms, lag).
// A lag near zero means the GPU had drained its queue when the host got
// there: device idle waiting for host planning.
namespace {
struct Timeline {
  bool on = false;
  cudaStream_t st = nullptr;
  double h0 = 0.0;
  cudaEvent_t e0 = nullptr;
  std::vector<std::string> names;
  std::vector<cudaEvent_t> ev;
  std::vector<double> host;
};
Timeline& tl() {
  static Timeline t;
  return t;
}
bool tl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("EBEM_TIMELINE");
    return e && std::atoi(e) != 0;
  }();
  return on;
}
}  // namespace
void tl_begin(cudaStream_t st) {
  Timeline& t = tl();
  t.on = tl_enabled();
  if (!t.on) return;
  t.st = st;
  t.names.clear();
  t.ev.clear();
  t.host.clear();
  g_staged_bytes = 0.0;
  g_staged_copies = 0;
  if (!t.e0) cudaEventCreate(&t.e0);
  cudaEventRecord(t.e0, st);
  cudaEventSynchronize(t.e0);
  t.h0 = now();
}
void tl_mark(const std::string& name) {
  Timeline& t = tl();
  if (!t.on) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, t.st);
  t.names.push_back(name);
  t.ev.push_back(e);
  t.host.push_back(now() - t.h0);
}
void tl_dump() {
  Timeline& t = tl();
  if (!t.on) return;
  cudaStreamSynchronize(t.st);
  double idle = 0.0, prev_g = 0.0;
  for (size_t i = 0; i < t.ev.size(); ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.e0, t.ev[i]);
    const double h = 1e3 * t.host[i];
    // the GPU reached this mark no earlier than the host recorded it: when
    // it got there within 20 us of the host, it waited (since the previous
    // mark at the latest) for the host
    const double lag = ms - h;
    if (lag < 0.02) idle += std::max(0.0, ms - std::max(prev_g, 0.0)) ;
    std::fprintf(stderr, "[tl] %-28s gpu %9.3f ms  host %9.3f ms  lag %8.3f\n", t.names[i].c_str(), ms, h, lag);
    prev_g = ms;
    cudaEventDestroy(t.ev[i]);
  }
  std::fprintf(stderr, "[tl] upper bound of host-bound device time: %.1f ms; staged %.1f MB in %ld copies\n",
               idle, g_staged_bytes / 1e6, g_staged_copies);
  g_staged_bytes = 0.0;
  g_staged_copies = 0;
  t.ev.clear();
  t.on = false;
}

// ---------------------------------------------------------------- Problem
Scratch& scratch() {
  // leaked on purpose: CUDA resources must not be released after the
  // runtime's own teardown at process exit
  static Scratch* s = [] {
    auto* x = new Scratch();
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw Error(EBEM_CUDA_ERROR, "no CUDA device available (the B200 path has no CPU fallback)");
    CK(cudaStreamCreateWithFlags(&x->st, cudaStreamNonBlocking));
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = ~uint64_t(0);
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    return x;
  }();
  return *s;
}

cudaStream_t scratch_stream() { return scratch().st; }

void copy_sync(void* dst, const void* src, size_t bytes) {
  if (!bytes) return;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, scratch().st));
  CK(cudaStreamSynchronize(scratch().st));
}

Problem::Problem(const double* xy, int n, double lam, double mu, double rho,
                 double omega, double are, double aim,
                 const ebem_assembly_config& a, const ebem_proxy_config& p)
    : staging(scratch().staging),
      tbuf_(scratch().tbuf),
      qr_rounds_(scratch().qr_rounds),
      id_jp_(scratch().id_jp),
      id_steps_(scratch().id_steps),
      id_rd_(scratch().id_rd),
      id_r_(scratch().id_r),
      sym_keys_(scratch().sym_keys),
      sym_vals_(scratch().sym_vals),
      sym_recs_(scratch().sym_recs),
      sym_bounds_(scratch().sym_bounds),
      bundles(scratch().bundles),
      gws(scratch().gws),
      n_(n),
      acfg_(a),
      pcfg_(p) {
  if (n < 4) throw Error(EBEM_INVALID_ARGUMENT, "Mesh: needs at least 4 nodes");
  if (n < 8) throw Error(EBEM_INVALID_ARGUMENT, "PairIntegrator: mesh too coarse");
  const double tc0 = now();
  xy_.assign(xy, xy + 2 * size_t(n));
  // element geometry straight into pinned staging memory (process-wide,
  // grow-only), built on the planning threads: field-major array, packed
  // 8-double rows and the node coordinates, uploaded below
  const size_t n9 = size_t(kElemFields) * n;
  double* const h_elem = scratch().h_geom.ensure(n9 + 10 * size_t(n));
  double* const h_e8 = h_elem + n9;
  double* const h_xy = h_e8 + 8 * size_t(n);
  {
    const int nch = std::max(1, std::min(n / 4096, 4 * planning_threads()));
    std::vector<double> lo(nch, 1e300), hi(nch, 0.0);
    std::vector<char> okv(nch, 1);
    parallel_for(nch, [&](int k) {
      const int e0 = int(size_t(n) * k / nch), e1 = int(size_t(n) * (k + 1) / nch);
      okv[k] = build_elements_range(xy_.data(), n, e0, e1, h_elem, h_e8, &lo[k], &hi[k]);
      std::memcpy(h_xy + 2 * size_t(e0), xy_.data() + 2 * size_t(e0), 16 * size_t(e1 - e0));
    });
    hmin_ = 1e300;
    hmax_ = 0.0;
    for (int k = 0; k < nch; ++k) {
      if (!okv[k]) throw Error(EBEM_INVALID_ARGUMENT, "Mesh: zero-length element");
      hmin_ = std::min(hmin_, lo[k]);
      hmax_ = std::max(hmax_, hi[k]);
    }
  }
  DevMedium med;
  try {
    med = make_medium(lam, mu, rho, omega, are, aim);
  } catch (const std::invalid_argument& e) {
    throw Error(EBEM_INVALID_ARGUMENT, e.what());
  }
  auto scaled = [&](int q) { return int(q * a.refine + 0.5); };
  const double tc1 = now();
  hctx_.med = med;
  hctx_.n_nodes = n;
  // the series tables depend on the medium only: kept for the next problem
  // with the same medium (API calls are serialised by the API mutex)
  struct SeriesCache {
    bool valid = false;
    double key[6];
    int maxq;
    unsigned char series[sizeof(hctx_.series)];
    ParSeries pser;
  };
  static SeriesCache scache;
  const double skey[6] = {lam, mu, rho, omega, are, aim};
  const bool cached = scache.valid && std::memcmp(scache.key, skey, sizeof(skey)) == 0;
  fc_.med = med;
  if (cached) {
    hctx_.series_maxq = scache.maxq;
    std::memcpy(hctx_.series, scache.series, sizeof(hctx_.series));
    hctx_.pser = scache.pser;
  }
  try {
    if (!cached) {
    hctx_.series_maxq = build_series(med, hctx_.series, kMaxSeriesPow);
    build_parity_series(hctx_.series, kMaxSeriesPow, hctx_.pser);
    for (int k = 2; k < 10; ++k)  // series_joint drops the imaginary log chain
      for (int p = 0; p < kParTerms; ++p)
        if (hctx_.pser.b[k][p].y != 0.0)
          throw std::logic_error("near-field expansion: complex log coefficient");
    for (int k = 0; k < 8; ++k) {  // series_joint hard-codes d odd, n even
      const int par = hctx_.pser.par[k + 2];
      if (par != (k < 3 ? 1 : 0))
        throw std::logic_error("near-field expansion: unexpected parity of a D/N series");
    }
    // The fill evaluates the D/N series only below the series radius: drop
    // the terms whose size there is below 1e-21 of the series' largest term
    // (the reference keeps them; they cannot change a double result).
    const double rmax = med.series_radius, lr = std::fabs(std::log(rmax));
    for (int k = 2; k < 10; ++k) {
      ParSeries& ps = hctx_.pser;
      double big = 0.0;
      std::vector<double> mag(ps.nt[k]);
      for (int p = 0; p < ps.nt[k]; ++p) {
        const double2 a = ps.a[k][p], b = ps.b[k][p];
        mag[p] = (std::hypot(a.x, a.y) + std::hypot(b.x, b.y) * lr) *
                 std::pow(rmax, ps.par[k] + 2 * p);
        big = std::max(big, mag[p]);
      }
      int nt = ps.nt[k];
      while (nt > 1 && mag[nt - 1] <= 1e-21 * big) --nt;
      for (int p = nt; p < kParTerms; ++p) ps.a[k][p] = ps.b[k][p] = double2{0.0, 0.0};
      ps.nt[k] = nt;
    }
    // The same criterion point by point: on a fine geometric grid below the
    // series radius find how many terms each r needs (the largest count over
    // scalars 2..9, evaluated at the upper end of each grid interval), and
    // record the radius past which t + 1 terms are needed.
    {
      ParSeries& ps = hctx_.pser;
      int ntmax = 1;
      for (int k = 2; k < 10; ++k) ntmax = std::max(ntmax, ps.nt[k]);
      // coefficient magnitudes once, powers of r incrementally
      double amag[10][kParTerms], bmag[10][kParTerms];
      for (int k = 2; k < 10; ++k)
        for (int p = 0; p < ps.nt[k]; ++p) {
          amag[k][p] = std::hypot(ps.a[k][p].x, ps.a[k][p].y);
          bmag[k][p] = std::hypot(ps.b[k][p].x, ps.b[k][p].y);
        }
      auto need = [&](double r) {
        const double lr = std::fabs(std::log(r));
        const double r2 = r * r;
        int worst = 1;
        for (int k = 2; k < 10; ++k) {
          double big = 0.0, mag[kParTerms];
          double rp = ps.par[k] == 0 ? 1.0 : std::pow(r, ps.par[k]);
          for (int p = 0; p < ps.nt[k]; ++p, rp *= r2) {
            mag[p] = (amag[k][p] + bmag[k][p] * lr) * rp;
            big = std::max(big, mag[p]);
          }
          int nt = ps.nt[k];
          while (nt > 1 && mag[nt - 1] <= 1e-22 * big) --nt;
          worst = std::max(worst, nt);
        }
        return worst;
      };
      for (int t = 0; t < kParTerms; ++t) ps.rcut[t] = t < ntmax ? 0.0 : HUGE_VAL;
      // walking down from the series radius: rcut[t] = the largest grid r at
      // and below which every grid point needs <= t terms
      std::vector<int> needs;
      std::vector<double> rs;
      for (double r = rmax; r > rmax * 1e-12; r *= 0.98) {
        rs.push_back(r);
        needs.push_back(need(r));
      }
      for (int t = 1; t < ntmax; ++t) {
        int g = int(rs.size());  // first index of the tail with need <= t
        while (g > 0 && needs[g - 1] <= t) --g;
        if (g < int(rs.size())) ps.rcut[t] = rs[g];
        if (g == 0) ps.rcut[t] = HUGE_VAL;
      }
      if (getenv("EBEM_VERBOSE") && atoi(getenv("EBEM_VERBOSE")) >= 2)
        for (int t = 1; t < ntmax; ++t)
          fprintf(stderr, "series: r > %.3e needs > %d terms\n", ps.rcut[t], t);
    }
    scache.valid = false;
    std::memcpy(scache.key, skey, sizeof(skey));
    scache.maxq = hctx_.series_maxq;
    std::memcpy(scache.series, hctx_.series, sizeof(hctx_.series));
    scache.pser = hctx_.pser;
    scache.valid = true;
    }
  } catch (const std::logic_error& e) {
    throw Error(EBEM_LOGIC_ERROR, e.what());
  }
  for (int p = 0; p < kFcTerms; ++p)
    for (int k = 0; k < 8; ++k) {
      const bool in = p < kParTerms;
      fc_.sa[p][k] = in ? hctx_.pser.a[k + 2][p] : double2{0.0, 0.0};
      fc_.sb[p][k] = in ? hctx_.pser.b[k + 2][p] : double2{0.0, 0.0};
    }
  {
    // Gauss-Legendre rules 1 .. kMaxGauss: computed once per process
    static const std::vector<double> rules = [] {
      const size_t len = size_t(gauss_offset(kMaxGauss)) + kMaxGauss;
      std::vector<double> r(2 * len);
      for (int q = 1; q <= kMaxGauss; ++q)
        gauss_rule(q, r.data() + gauss_offset(q), r.data() + len + gauss_offset(q));
      return r;
    }();
    const size_t len = rules.size() / 2;
    std::memcpy(hctx_.gx, rules.data(), len * sizeof(double));
    std::memcpy(hctx_.gw, rules.data() + len, len * sizeof(double));
  }
  hctx_.far_nodes = a.far_nodes;
  hctx_.refine = a.refine;
  {
    // the very-far 3 x 3 tier only with the default far rule (4 points, no
    // refinement), whose value it reproduces to rounding
    static const bool far2 = [] {
      const char* e = std::getenv("EBEM_FAR3");
      return e == nullptr || std::atoi(e) != 0;
    }();
    hctx_.very_far_tier = (far2 && a.far_nodes == 4 && a.refine == 1.0) ? 1 : 0;
  }
  hctx_.corner_n = scaled(a.corner_nodes);
  hctx_.proxy_n = p.n_gauss;
  hctx_.m_prime = p.m_prime;
  const int max_tier = scaled(a.far_nodes + 9);
  if (hctx_.corner_n < 1 || hctx_.corner_n > kMaxGauss || max_tier > kMaxGauss ||
      scaled(a.far_nodes) < 1 || scaled(a.rhs_nodes) < 1 ||
      scaled(a.rhs_nodes) > kMaxGauss)
    throw Error(EBEM_INVALID_ARGUMENT, "gauss_rule: order out of range");
  if (p.n_gauss < 1 || p.n_gauss > kMaxGauss)
    throw Error(EBEM_INVALID_ARGUMENT, "gauss_rule: order out of range");
  if (p.radius_factor <= 1.0)
    throw Error(EBEM_INVALID_ARGUMENT,
                "build_proxy: radius_factor must exceed 1 so the circle "
                "encloses the cell");
  if (p.m_prime < 3)
    throw Error(EBEM_INVALID_ARGUMENT, "build_proxy: polygon needs >= 3 nodes");
  if (p.m_prime > 512)
    throw Error(EBEM_INVALID_ARGUMENT, "build_proxy: m_prime above 512 unsupported");
  for (int j = 0; j < p.m_prime; ++j) {
    const double t = 2.0 * 3.14159265358979323846 * j / p.m_prime;
    hctx_.poly_cs[2 * j] = std::cos(t);
    hctx_.poly_cs[2 * j + 1] = std::sin(t);
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    throw Error(EBEM_CUDA_ERROR, "no CUDA device available (the B200 path has no CPU fallback)");
  const double tc2 = now();
  st_ = scratch().st;
  delem_.alloc(n9);
  dxy_.alloc(xy_.size());
  delem8_.alloc(8 * size_t(n));
  CK(cudaMemcpyAsync(delem_.get(), h_elem, n9 * 8, cudaMemcpyHostToDevice, st_));
  CK(cudaMemcpyAsync(dxy_.get(), h_xy, xy_.size() * 8, cudaMemcpyHostToDevice, st_));
  CK(cudaMemcpyAsync(delem8_.get(), h_e8, 64 * size_t(n), cudaMemcpyHostToDevice, st_));
  hctx_.elem = delem_.get();
  hctx_.elem8 = delem8_.get();
  // (the stream is synchronised below, before the staging memory can be reused)
  hctx_.node_xy = dxy_.get();
  dctx_.alloc(1);
  CK(cudaMemcpyAsync(dctx_.get(), &hctx_, sizeof(DevCtx), cudaMemcpyHostToDevice, st_));
  bad.alloc(1);
  CK(cudaMemsetAsync(bad.get(), 0, sizeof(int), st_));
  CK(cudaStreamSynchronize(st_));
  dense_init();
  const double tc3 = now();
  tree_.build(xy_.data(), n);
  if (verbose_level())
    std::fprintf(stderr, "[ebem] problem setup: geometry %.1f ms, tables %.1f ms, upload %.1f ms, box tree %.1f ms\n",
                 1e3 * (tc1 - tc0), 1e3 * (tc2 - tc1), 1e3 * (tc3 - tc2), 1e3 * (now() - tc3));
}

Problem::Problem(int n)
    : staging(scratch().staging),
      tbuf_(scratch().tbuf),
      qr_rounds_(scratch().qr_rounds),
      id_jp_(scratch().id_jp),
      id_steps_(scratch().id_steps),
      id_rd_(scratch().id_rd),
      id_r_(scratch().id_r),
      sym_keys_(scratch().sym_keys),
      sym_vals_(scratch().sym_vals),
      sym_recs_(scratch().sym_recs),
      sym_bounds_(scratch().sym_bounds),
      bundles(scratch().bundles),
      gws(scratch().gws),
      n_(n) {
  if (n <= 0) throw Error(EBEM_INVALID_ARGUMENT, "FdsSolver: node count must be positive");
  acfg_ = ebem_assembly_config{10, 4, 8, 1.0, size_t(4) << 30};
  pcfg_ = ebem_proxy_config{1.5, 64, 6};
  st_ = scratch().st;
  bad.alloc(1);
  CK(cudaMemsetAsync(bad.get(), 0, sizeof(int), st_));
  dense_init();
}

Problem::~Problem() {
  if (st_) cudaStreamSynchronize(st_);  // the stream is process-wide
}

ProxyGeom Problem::build_proxy(int begin, int end) const {
  const int n = n_;
  if (begin < 0 || end > n || begin >= end)
    throw Error(EBEM_INVALID_ARGUMENT, "build_proxy: bad node range");
  double xmin = std::numeric_limits<double>::infinity(), xmax = -xmin;
  double ymin = xmin, ymax = -xmin;
  for (int g = begin - 1; g <= end; ++g) {
    const int w = (g % n + n) % n;
    xmin = std::min(xmin, xy_[2 * w]);
    xmax = std::max(xmax, xy_[2 * w]);
    ymin = std::min(ymin, xy_[2 * w + 1]);
    ymax = std::max(ymax, xy_[2 * w + 1]);
  }
  ProxyGeom g;
  g.cx = 0.5 * (xmin + xmax);
  g.cy = 0.5 * (ymin + ymax);
  const double half_diag = 0.5 * std::hypot(xmax - xmin, ymax - ymin);
  g.radius = pcfg_.radius_factor * std::max(half_diag, 1e-300);
  tree_.enclosed(xy_.data(), g.cx, g.cy, g.radius, begin, end, g.enclosed);
  return g;
}

void Problem::check_domain() {
  int h = 0;
  CK(cudaMemcpyAsync(&h, bad.get(), sizeof(int), cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
  if (h) {
    CK(cudaMemsetAsync(bad.get(), 0, sizeof(int), st_));
    throw Error(EBEM_DOMAIN_ERROR,
                "KernelScalars: element too long for this frequency (needs "
                "several elements per wavelength)");
  }
}

// ------------------------------------------------------- planning threads
namespace {

class PlanPool {
 public:
  PlanPool() {
    const unsigned hw = std::thread::hardware_concurrency();
    n_ = int(std::min(16u, std::max(1u, hw)));
    if (const char* e = std::getenv("EBEM_PLAN_THREADS")) n_ = std::max(1, std::atoi(e));
    for (int i = 1; i < n_; ++i) th_.emplace_back([this] { loop(); });
  }
  ~PlanPool() {
    {
      std::lock_guard<std::mutex> lk(m_);
      stop_ = true;
    }
    cv_.notify_all();
    for (std::thread& t : th_) t.join();
  }
  int size() const { return n_; }
  // Items are claimed under the mutex and tagged with the generation of the
  // call: a worker still leaving the previous call can neither take an item
  // of the next one with a stale count nor miss its completion signal.
  void run(int n, const std::function<void(int)>& f) {
    if (n <= 0) return;
    if (n_ == 1 || n == 1 || in_pool_) {  // (a nested call runs serially)
      for (int i = 0; i < n; ++i) f(i);
      return;
    }
    struct Mark {
      Mark() { in_pool_ = true; }
      ~Mark() { in_pool_ = false; }
    } mark;
    unsigned long g;
    {
      std::lock_guard<std::mutex> lk(m_);
      f_ = &f;
      total_ = n;
      next_ = 0;
      done_ = 0;
      err_ = nullptr;
      g = ++gen_;
    }
    cv_.notify_all();
    work(g);
    std::unique_lock<std::mutex> lk(m_);
    done_cv_.wait(lk, [&] { return done_ == total_; });
    f_ = nullptr;
    if (err_) std::rethrow_exception(err_);
  }

 private:
  void work(unsigned long g) {
    for (;;) {
      int i;
      const std::function<void(int)>* f;
      {
        std::lock_guard<std::mutex> lk(m_);
        if (gen_ != g || next_ >= total_) return;
        i = next_++;
        f = f_;
      }
      std::exception_ptr e;
      try {
        (*f)(i);
      } catch (...) {
        e = std::current_exception();
      }
      std::lock_guard<std::mutex> lk(m_);
      if (e && !err_) err_ = e;
      if (++done_ == total_) done_cv_.notify_all();
    }
  }
  void loop() {
    in_pool_ = true;
    unsigned long seen = 0;
    for (;;) {
      {
        std::unique_lock<std::mutex> lk(m_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
      }
      work(seen);
    }
  }
  int n_ = 1;
  std::vector<std::thread> th_;
  std::mutex m_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(int)>* f_ = nullptr;
  int total_ = 0, next_ = 0, done_ = 0;
  std::exception_ptr err_;
  unsigned long gen_ = 0;
  bool stop_ = false;
  static thread_local bool in_pool_;
};
thread_local bool PlanPool::in_pool_ = false;

PlanPool& plan_pool() {
  static PlanPool* p = new PlanPool();  // never destroyed: no join at exit
  return *p;
}

}  // namespace

void parallel_for(int n, const std::function<void(int)>& f) { plan_pool().run(n, f); }
int planning_threads() { return plan_pool().size(); }

// ---------------------------------------------------------------- FillPlan
void FillPlan::clear() {
  has_one_sided_ = has_two_sided_ = false;
  bundles_ = entries_ = 0;
  sym_pairs_ = 0;
  sym_.clear();
  sym_off_.clear();
  proxy_blocks_ = 0;
  poly_desc_off_ = -1;
  elems_.clear();
  sing_pair_.clear();
  sing_elems_.clear();
  proxy_.clear();
  proxy_boff_.clear();
  gather_.clear();
  gather_off_.clear();
  desc_.clear();
}

void FillPlan::append(const FillPlan& o) {
  const int eb = int(elems_.size());
  const long long bb = bundles_, sb = sym_pairs_, entb = entries_;
  const int db = int(desc_.size()), pb = proxy_blocks_;
  elems_.insert(elems_.end(), o.elems_.begin(), o.elems_.end());
  for (long long x : o.sing_pair_) sing_pair_.push_back(x + bb);
  sing_elems_.insert(sing_elems_.end(), o.sing_elems_.begin(), o.sing_elems_.end());
  for (SymJob J : o.sym_) {
    J.v_off += bb;
    J.u_off += bb;
    J.local_off += sb;
    J.a_off += eb;
    J.e_off += eb;
    sym_.push_back(J);
  }
  for (long long x : o.sym_off_) sym_off_.push_back(x + sb);
  for (ProxyJob J : o.proxy_) {
    J.v_off += bb;
    J.u_off += bb;
    J.e_off += eb;
    J.block_off += pb;
    proxy_.push_back(J);
  }
  for (int x : o.proxy_boff_) proxy_boff_.push_back(x + pb);
  for (GatherJob G : o.gather_) {
    G.pair_off += bb;
    G.entry_off += entb;
    G.rdesc_off += db;
    G.cdesc_off += db;
    gather_.push_back(G);
  }
  for (long long x : o.gather_off_) gather_off_.push_back(x + entb);
  desc_.insert(desc_.end(), o.desc_.begin(), o.desc_.end());
  bundles_ += o.bundles_;
  sym_pairs_ += o.sym_pairs_;
  entries_ += o.entries_;
  proxy_blocks_ += o.proxy_blocks_;
  has_one_sided_ = has_one_sided_ || o.has_one_sided_;
  has_two_sided_ = has_two_sided_ || o.has_two_sided_;
  // o's polygon descriptors were copied with its descriptors; this plan's own
  // (if any) stay where they are
}

void FillPlan::append_many(const std::vector<FillPlan>& parts, int k0, int k1) {
  const int np = k1 - k0;
  if (np <= 0) return;
  bool regular = np > 1;  // one offset per job, two elements per singular pair
  for (int k = k0; k < k1 && regular; ++k) {
    const FillPlan& o = parts[k];
    regular = o.sym_off_.size() == o.sym_.size() && o.proxy_boff_.size() == o.proxy_.size() &&
              o.gather_off_.size() == o.gather_.size() &&
              o.sing_elems_.size() == 2 * o.sing_pair_.size();
  }
  if (!regular) {
    for (int k = k0; k < k1; ++k) append(parts[k]);
    return;
  }
  struct Base {
    size_t elems, sing, sym, proxy, gather, desc;
    long long bundles, sym_pairs, entries;
    int proxy_blocks;
  };
  std::vector<Base> base(np + 1);
  base[0] = Base{elems_.size(), sing_pair_.size(), sym_.size(), proxy_.size(), gather_.size(),
                 desc_.size(), bundles_, sym_pairs_, entries_, proxy_blocks_};
  for (int i = 0; i < np; ++i) {
    const FillPlan& o = parts[k0 + i];
    Base b = base[i];
    b.elems += o.elems_.size();
    b.sing += o.sing_pair_.size();
    b.sym += o.sym_.size();
    b.proxy += o.proxy_.size();
    b.gather += o.gather_.size();
    b.desc += o.desc_.size();
    b.bundles += o.bundles_;
    b.sym_pairs += o.sym_pairs_;
    b.entries += o.entries_;
    b.proxy_blocks += o.proxy_blocks_;
    base[i + 1] = b;
    has_one_sided_ = has_one_sided_ || o.has_one_sided_;
    has_two_sided_ = has_two_sided_ || o.has_two_sided_;
  }
  const Base& e = base[np];
  elems_.resize(e.elems);
  sing_pair_.resize(e.sing);
  sing_elems_.resize(2 * e.sing);
  sym_.resize(e.sym);
  sym_off_.resize(e.sym);
  proxy_.resize(e.proxy);
  proxy_boff_.resize(e.proxy);
  gather_.resize(e.gather);
  gather_off_.resize(e.gather);
  desc_.resize(e.desc);
  parallel_for(np, [&](int i) {
    const FillPlan& o = parts[k0 + i];
    const Base& b = base[i];
    const int eb = int(b.elems), db = int(b.desc), pb = b.proxy_blocks;
    const long long bb = b.bundles, sb = b.sym_pairs, entb = b.entries;
    std::copy(o.elems_.begin(), o.elems_.end(), elems_.begin() + b.elems);
    for (size_t q = 0; q < o.sing_pair_.size(); ++q) sing_pair_[b.sing + q] = o.sing_pair_[q] + bb;
    std::copy(o.sing_elems_.begin(), o.sing_elems_.end(), sing_elems_.begin() + 2 * b.sing);
    for (size_t q = 0; q < o.sym_.size(); ++q) {
      SymJob J = o.sym_[q];
      J.v_off += bb;
      J.u_off += bb;
      J.local_off += sb;
      J.a_off += eb;
      J.e_off += eb;
      sym_[b.sym + q] = J;
      sym_off_[b.sym + q] = o.sym_off_[q] + sb;
    }
    for (size_t q = 0; q < o.proxy_.size(); ++q) {
      ProxyJob J = o.proxy_[q];
      J.v_off += bb;
      J.u_off += bb;
      J.e_off += eb;
      J.block_off += pb;
      proxy_[b.proxy + q] = J;
      proxy_boff_[b.proxy + q] = o.proxy_boff_[q] + pb;
    }
    for (size_t q = 0; q < o.gather_.size(); ++q) {
      GatherJob G = o.gather_[q];
      G.pair_off += bb;
      G.entry_off += entb;
      G.rdesc_off += db;
      G.cdesc_off += db;
      gather_[b.gather + q] = G;
      gather_off_[b.gather + q] = o.gather_off_[q] + entb;
    }
    std::copy(o.desc_.begin(), o.desc_.end(), desc_.begin() + b.desc);
  });
  bundles_ = e.bundles;
  sym_pairs_ = e.sym_pairs;
  entries_ = e.entries;
  proxy_blocks_ = e.proxy_blocks;
}

// Elements supporting the hat functions of the listed nodes (node g owns
// elements g-1 and g), ascending and unique (proj/src/assembly.cpp:342-368).
void FillPlan::elements_of(const Lists& nodes, std::vector<int>& out) const {
  out.clear();
  const bool s0 = std::is_sorted(nodes[0].begin(), nodes[0].end());
  const bool s1 = std::is_sorted(nodes[1].begin(), nodes[1].end());
  if (s0 && s1) {
    // Linear path for ascending lists (enclosed sets, leaf ranges): node g
    // contributes g-1, g, already in order; node 0's element N-1 goes last.
    auto gen = [&](const std::vector<int>& v, std::vector<int>& o) {
      o.clear();
      o.reserve(2 * v.size());
      bool wrap = false;
      for (int g : v) {
        if (g == 0) {
          wrap = true;
        } else if (o.empty() || o.back() != g - 1) {
          o.push_back(g - 1);
        }
        if (o.empty() || o.back() != g) o.push_back(g);
      }
      if (wrap && (o.empty() || o.back() != N_ - 1)) o.push_back(N_ - 1);
    };
    thread_local std::vector<int> a, b;
    gen(nodes[0], a);
    if (nodes[1] == nodes[0]) {
      out = a;
      return;
    }
    gen(nodes[1], b);
    out.resize(a.size() + b.size());
    out.erase(std::set_union(a.begin(), a.end(), b.begin(), b.end(), out.begin()),
              out.end());
    return;
  }
  out.reserve(4 * (nodes[0].size() + nodes[1].size()));
  for (int p = 0; p < 2; ++p)
    for (int g : nodes[p]) {
      out.push_back(g);
      out.push_back(g == 0 ? N_ - 1 : g - 1);
    }
  std::sort(out.begin(), out.end());
  out.erase(std::unique(out.begin(), out.end()), out.end());
}

void FillPlan::node_descs(const Lists& nodes, const std::vector<int>& elems,
                          const int dest_off[2], std::vector<NodeDesc>& out,
                          const std::vector<int>* const* pos) const {
  auto idx = [&](int e) {
    return int(std::lower_bound(elems.begin(), elems.end(), e) - elems.begin());
  };
  const int last = idx(N_ - 1);
  for (int p = 0; p < 2; ++p) {
    const std::vector<int>& v = nodes[p];
    const bool sorted = std::is_sorted(v.begin(), v.end());
    int cur = 0;  // two-pointer position for ascending lists
    for (size_t k = 0; k < v.size(); ++k) {
      const int g = v[k];
      NodeDesc d;
      d.dest = dest_off[p] + (pos ? (*pos[p])[k] : int(k));
      int la1, la2;
      if (g == 0) {  // elements 0 (shape 0) and N-1 (shape 1)
        d.e1 = idx(0);
        d.e2 = last;
        la1 = 0;
        la2 = 1;
      } else {  // elements g-1 (shape 1) and g (shape 0), adjacent in elems
        if (sorted) {
          while (elems[cur] < g - 1) ++cur;
          d.e1 = cur;
        } else {
          d.e1 = idx(g - 1);
        }
        d.e2 = d.e1 + 1;
        la1 = 1;
        la2 = 0;
      }
      d.bits = la1 | (la2 << 1) | (p << 2);
      out.push_back(d);
    }
  }
}

void FillPlan::add_true_block(const Lists& rows, const Lists& cols,
                              double* dest, int ld, const int drow[2],
                              const int dcol[2], int trans,
                              const std::vector<int>* const* rpos,
                              const std::vector<int>* const* cpos) {
  const int nr = int(rows[0].size() + rows[1].size());
  const int nc = int(cols[0].size() + cols[1].size());
  if (nr == 0 || nc == 0) return;
  std::vector<int> res, ces;
  elements_of(rows, res);
  elements_of(cols, ces);
  // a one-sided job of the near-field kernel: test = row elements (A),
  // trial = column elements (E), bundle (a, q) at v_off + a nE + q
  SymJob J;
  J.tri = 0;
  J.onesided = 1;
  has_one_sided_ = true;
  J.nA = int(res.size());
  J.nE = int(ces.size());
  J.a_off = int(elems_.size());
  elems_.insert(elems_.end(), res.begin(), res.end());
  J.e_off = int(elems_.size());
  elems_.insert(elems_.end(), ces.begin(), ces.end());
  const long long np = (long long)J.nA * J.nE;
  J.v_off = J.u_off = bundles_;
  J.local_off = sym_pairs_;
  sym_.push_back(J);
  sym_off_.push_back(sym_pairs_);
  sym_pairs_ += np;
  // touching pairs (coincident / adjacent) go to the singular kernel;
  // search from the shorter element list into the longer one
  const bool rows_short = res.size() <= ces.size();
  const std::vector<int>& sh = rows_short ? res : ces;
  const std::vector<int>& lg = rows_short ? ces : res;
  for (int i = 0; i < int(sh.size()); ++i) {
    const int e = sh[i];
    const int cand[3] = {e == 0 ? N_ - 1 : e - 1, e, e + 1 == N_ ? 0 : e + 1};
    for (int c : cand) {
      auto it = std::lower_bound(lg.begin(), lg.end(), c);
      if (it != lg.end() && *it == c) {
        const int j = int(it - lg.begin());
        const int ra = rows_short ? i : j, cb = rows_short ? j : i;
        sing_pair_.push_back(J.v_off + (long long)ra * J.nE + cb);
        sing_elems_.push_back(res[ra]);
        sing_elems_.push_back(ces[cb]);
      }
    }
  }
  GatherJob G;
  G.pair_off = J.v_off;
  G.entry_off = entries_;
  G.nces = J.nE;
  G.rdesc_off = int(desc_.size());
  node_descs(rows, res, drow, desc_, rpos);
  G.nrows = nr;
  G.cdesc_off = int(desc_.size());
  node_descs(cols, ces, dcol, desc_, cpos);
  G.ncols = nc;
  G.trans = trans;
  G.ld = ld;
  G.dest = dest;
  gather_.push_back(G);
  gather_off_.push_back(entries_);
  entries_ += (long long)nr * nc;
  bundles_ += np;
}

void FillPlan::add_sym_near(const std::vector<int>& enc, const Lists& rows,
                            const Lists& cols, double* tv, int ld_v, double* tu,
                            int ld_u) {
  const int rdest[2] = {0, int(rows[0].size())};
  const int cdest[2] = {0, int(cols[0].size())};
  add_sym_near_part(enc, nullptr, int(enc.size()), rows, rdest, cols, cdest, tv, ld_v, tu,
                    ld_u);
}

void FillPlan::add_sym_near_part(const std::vector<int>& enc, const std::vector<int>* enc_pos,
                                 int ne_total, const Lists& rows, const int rdest[2],
                                 const Lists& cols, const int cdest[2], double* tv,
                                 int ld_v, double* tu, int ld_u) {
  if (enc.empty()) return;
  const int nr = int(rows[0].size() + rows[1].size());
  const int nc = int(cols[0].size() + cols[1].size());
  if (nr == 0 && nc == 0) return;
  const Lists encl{enc, enc};
  std::vector<int> A, E;
  elements_of(encl, A);
  Lists both;
  both[0] = rows[0];
  both[0].insert(both[0].end(), rows[1].begin(), rows[1].end());
  both[1] = cols[0];
  both[1].insert(both[1].end(), cols[1].begin(), cols[1].end());
  elements_of(both, E);
  SymJob J;
  J.tri = 0;
  J.onesided = 0;
  has_two_sided_ = true;
  J.nA = int(A.size());
  J.nE = int(E.size());
  J.a_off = int(elems_.size());
  elems_.insert(elems_.end(), A.begin(), A.end());
  J.e_off = int(elems_.size());
  elems_.insert(elems_.end(), E.begin(), E.end());
  const long long np = (long long)J.nA * J.nE;
  J.v_off = bundles_;
  J.u_off = bundles_ + np;
  J.local_off = sym_pairs_;
  sym_.push_back(J);
  sym_off_.push_back(sym_pairs_);
  sym_pairs_ += np;
  bundles_ += 2 * np;
  // touching pairs: both orientations through the singular kernel
  for (int q = 0; q < J.nE; ++q) {
    const int e = E[q];
    const int cand[3] = {e == 0 ? N_ - 1 : e - 1, e, e + 1 == N_ ? 0 : e + 1};
    for (int c : cand) {
      auto it = std::lower_bound(A.begin(), A.end(), c);
      if (it != A.end() && *it == c) {
        const int a = int(it - A.begin());
        sing_pair_.push_back(J.v_off + (long long)a * J.nE + q);
        sing_elems_.push_back(A[a]);
        sing_elems_.push_back(E[q]);
        sing_pair_.push_back(J.u_off + (long long)q * J.nA + a);
        sing_elems_.push_back(E[q]);
        sing_elems_.push_back(A[a]);
      }
    }
  }
  const int ne = int(enc.size());
  const int denc[2] = {2 * m_, 2 * m_ + ne_total};  // enclosed rows per component
  const std::vector<int>* const epos2[2] = {enc_pos, enc_pos};
  const std::vector<int>* const* epos = enc_pos ? epos2 : nullptr;
  if (nc > 0) {  // T_V rows 2m'.. : true_block(enc x 2, cols)
    GatherJob G;
    G.pair_off = J.v_off;
    G.entry_off = entries_;
    G.nces = J.nE;
    G.rdesc_off = int(desc_.size());
    node_descs(encl, A, denc, desc_, epos);
    G.nrows = 2 * ne;
    G.cdesc_off = int(desc_.size());
    node_descs(cols, E, cdest, desc_);
    G.ncols = nc;
    G.trans = 0;
    G.ld = ld_v;
    G.dest = tv;
    gather_.push_back(G);
    gather_off_.push_back(entries_);
    entries_ += (long long)G.nrows * G.ncols;
  }
  if (nr > 0) {  // T_U rows 2m'.. : conj(true_block(rows, enc x 2))
    GatherJob G;
    G.pair_off = J.u_off;
    G.entry_off = entries_;
    G.nces = J.nA;
    G.rdesc_off = int(desc_.size());
    node_descs(rows, E, rdest, desc_);
    G.nrows = nr;
    G.cdesc_off = int(desc_.size());
    node_descs(encl, A, denc, desc_, epos);
    G.ncols = 2 * ne;
    G.trans = 1;
    G.ld = ld_u;
    G.dest = tu;
    gather_.push_back(G);
    gather_off_.push_back(entries_);
    entries_ += (long long)G.nrows * G.ncols;
  }
}

void FillPlan::add_sym_diag(const std::vector<int>& nodes, double* dest,
                            int ld) {
  if (nodes.empty()) return;
  const Lists L{nodes, nodes};
  std::vector<int> E;
  elements_of(L, E);
  SymJob J;
  J.tri = 1;
  J.onesided = 0;
  has_two_sided_ = true;
  J.nA = J.nE = int(E.size());
  J.a_off = J.e_off = int(elems_.size());
  elems_.insert(elems_.end(), E.begin(), E.end());
  const long long np = (long long)J.nA * J.nE;
  J.v_off = J.u_off = bundles_;
  J.local_off = sym_pairs_;
  sym_.push_back(J);
  sym_off_.push_back(sym_pairs_);
  sym_pairs_ += np;
  bundles_ += np;
  // touching pairs (coincident, adjacent): every ordered pair once
  for (int a = 0; a < J.nA; ++a) {
    const int e = E[a];
    const int cand[3] = {e == 0 ? N_ - 1 : e - 1, e, e + 1 == N_ ? 0 : e + 1};
    for (int c : cand) {
      auto it = std::lower_bound(E.begin(), E.end(), c);
      if (it != E.end() && *it == c) {
        const int q = int(it - E.begin());
        sing_pair_.push_back(J.v_off + (long long)a * J.nE + q);
        sing_elems_.push_back(E[a]);
        sing_elems_.push_back(E[q]);
      }
    }
  }
  GatherJob G;
  G.pair_off = J.v_off;
  G.entry_off = entries_;
  G.nces = J.nE;
  G.rdesc_off = int(desc_.size());
  const int off[2] = {0, int(nodes.size())};
  node_descs(L, E, off, desc_);
  G.nrows = 2 * int(nodes.size());
  G.cdesc_off = G.rdesc_off;
  G.ncols = G.nrows;
  G.trans = 0;
  G.ld = ld;
  G.dest = dest;
  gather_.push_back(G);
  gather_off_.push_back(entries_);
  entries_ += (long long)G.nrows * G.ncols;
}

// Descriptors of the 2 m' polygon hat functions (both components); the
// polygon element list is 0..m'-1 itself.
int FillPlan::poly_descs() {
  if (poly_desc_off_ >= 0) return poly_desc_off_;
  poly_desc_off_ = int(desc_.size());
  for (int p = 0; p < 2; ++p)
    for (int j = 0; j < m_; ++j) {
      NodeDesc d;
      d.dest = p * m_ + j;
      int la1, la2;
      if (j == 0) {
        d.e1 = 0;
        d.e2 = m_ - 1;
        la1 = 0;
        la2 = 1;
      } else {
        d.e1 = j - 1;
        d.e2 = j;
        la1 = 1;
        la2 = 0;
      }
      d.bits = la1 | (la2 << 1) | (p << 2);
      desc_.push_back(d);
    }
  return poly_desc_off_;
}

void FillPlan::add_proxy(double cx, double cy, double radius, const Lists& rows,
                         const Lists& cols, double* tv, int ld_v, double* tu,
                         int ld_u) {
  Lists both;
  both[0] = rows[0];
  both[0].insert(both[0].end(), rows[1].begin(), rows[1].end());
  both[1] = cols[0];
  both[1].insert(both[1].end(), cols[1].begin(), cols[1].end());
  std::vector<int> E;
  elements_of(both, E);
  ProxyJob J;
  J.e_off = int(elems_.size());
  J.nE = int(E.size());
  elems_.insert(elems_.end(), E.begin(), E.end());
  J.v_off = bundles_;
  J.u_off = bundles_ + (long long)m_ * J.nE;
  J.block_off = proxy_blocks_;
  J.pad = 0;
  J.cx = cx;
  J.cy = cy;
  J.radius = radius;
  proxy_.push_back(J);
  proxy_boff_.push_back(proxy_blocks_);
  proxy_blocks_ += proxy_blocks_for(m_, J.nE, ng_);
  bundles_ += 2ll * m_ * J.nE;
  const int pd = poly_descs();
  const int nr = int(rows[0].size() + rows[1].size());
  const int nc = int(cols[0].size() + cols[1].size());
  // T_V poly rows: M_V(poly (i, pj), col (j, c))
  if (nc > 0) {
    GatherJob G;
    G.pair_off = J.v_off;
    G.entry_off = entries_;
    G.nces = J.nE;
    G.rdesc_off = pd;
    G.nrows = 2 * m_;
    G.cdesc_off = int(desc_.size());
    const int dcol[2] = {0, int(cols[0].size())};
    node_descs(cols, E, dcol, desc_);
    G.ncols = nc;
    G.trans = 0;
    G.ld = ld_v;
    G.dest = tv;
    gather_.push_back(G);
    gather_off_.push_back(entries_);
    entries_ += (long long)G.nrows * G.ncols;
  }
  // T_U poly rows: conj(M_U(row (i, r), poly (j, pj)))
  if (nr > 0) {
    GatherJob G;
    G.pair_off = J.u_off;
    G.entry_off = entries_;
    G.nces = m_;
    G.rdesc_off = int(desc_.size());
    const int drow[2] = {0, int(rows[0].size())};
    node_descs(rows, E, drow, desc_);
    G.nrows = nr;
    G.cdesc_off = pd;
    G.ncols = 2 * m_;
    G.trans = 1;
    G.ld = ld_u;
    G.dest = tu;
    gather_.push_back(G);
    gather_off_.push_back(entries_);
    entries_ += (long long)G.nrows * G.ncols;
  }
}

void Problem::execute(FillPlan& plan) {
  if (plan.empty()) return;
  PhaseTimer t_exec("fill_execute", st_);
  Pack pk;
  const size_t o_el = pk.add(plan.elems_);
  const size_t o_sp = pk.add(plan.sing_pair_);
  const size_t o_se = pk.add(plan.sing_elems_);
  const size_t o_sj = pk.add(plan.sym_);
  const size_t o_so = pk.add(plan.sym_off_);
  const size_t o_pj = pk.add(plan.proxy_);
  const size_t o_pb = pk.add(plan.proxy_boff_);
  const size_t o_gj = pk.add(plan.gather_);
  // CTA tiles of kGatherTile entries, each job starting on its own tile
  std::vector<int> gblk(plan.gather_.size());
  int n_gblk = 0;
  for (size_t g = 0; g < plan.gather_.size(); ++g) {
    gblk[g] = n_gblk;
    const long long e = (long long)plan.gather_[g].nrows * plan.gather_[g].ncols;
    n_gblk += int((e + kGatherTile - 1) / kGatherTile);
  }
  const size_t o_go = pk.add(gblk);
  const size_t o_de = pk.add(plan.desc_);
  char* base;
  {
    PhaseTimer t_up("fill_upload", nullptr);
    base = staging.put(pk, st_);
  }
  {
    PhaseTimer t_al("fill_bundle_alloc", nullptr);
    // grow-only, sized for a full wave up front (a realloc synchronises)
    const size_t need = size_t(plan.bundles_) * kBundle * 2;
    if (need > bundles.size())
      bundles.ensure(std::max(need, size_t(kMaxBundlesPerWave) * kBundle * 2 * 5 / 4));
  }
  const int* el = Pack::at<int>(base, o_el);
  // symmetric near pairs: bucket by tier (count + scatter, async); the class
  // bounds stay on the device, the near-field launches read them there
  const long long nsym = plan.sym_pairs_;
  // pair records: the bucketed near pairs, then the proxy slots
  const long long proxy_slots =
      (long long)plan.proxy_blocks_ * proxy_pairs_per_block(pcfg_.n_gauss);
  if (nsym == 0 && proxy_slots > 0) sym_recs_.ensure(size_t(kSymRec) * proxy_slots);
  const SymJob* sj = nullptr;
  const long long* so = nullptr;
  if (nsym > 0) {
    sj = Pack::at<SymJob>(base, o_sj);
    so = Pack::at<long long>(base, o_so);
    sym_keys_.ensure(size_t(nsym));
    sym_vals_.ensure(size_t(nsym));  // job of each pair
    if (!sym_bounds_.get()) sym_bounds_.alloc(size_t(sym_bounds_ints()));
    sym_recs_.ensure(size_t(kSymRec) * (nsym + proxy_slots));
    g_prof.begin(st_);
    launch_sym_bucket(dctx(), sj, so, int(plan.sym_.size()), el, nsym, sym_keys_.get(),
                      sym_vals_.get(), sym_bounds_.get(), sym_recs_.get(), st_);
    g_prof.end(KP_BUCKET, st_, double(nsym));
    g_launches += 2;
  }
  if (!plan.proxy_.empty()) {
    double pts = 0.0;
    for (const ProxyJob& j : plan.proxy_)
      pts += double(pcfg_.m_prime) * j.nE * pcfg_.n_gauss * pcfg_.n_gauss;
    g_prof.begin(st_);
    launch_proxy_pairs(dctx(), fc_, pcfg_.n_gauss, Pack::at<ProxyJob>(base, o_pj),
                       Pack::at<int>(base, o_pb), int(plan.proxy_.size()),
                       plan.proxy_blocks_, el, sym_recs_.get() + size_t(kSymRec) * nsym,
                       bundles.get(), plan.bundles_, st_);
    g_prof.end(KP_PROXY, st_, pts);
  }
  if (nsym > 0) {
    // one launch per class, sized by the wave's pair count; each reads its
    // range from the device-side bounds (no host round trip)
    const int add[4] = {0, 2, 5, 9};
    for (int c = 0; c < kSymClasses - 1; ++c) {  // the last class is "skip"
      const int tier = c % kSymTiers;
      const bool both = c < kSymTiers;  // the upper classes: one-sided true blocks
      if (both ? !plan.has_two_sided_ : !plan.has_one_sided_) continue;
      if (tier == 4 && !hctx_.very_far_tier) continue;
      const int nq = tier == 4 ? kVeryFarNodes : int((acfg_.far_nodes + add[tier]) * acfg_.refine + 0.5);
      g_prof.begin(st_);
      launch_near_sym(dctx(), fc_, sym_recs_.get(), sym_bounds_.get(), c, nsym, nq, both,
                      bundles.get(), plan.bundles_, st_);
      // points = class count x nq^2, read back at collect time
      g_prof.end_counted(both ? KP_NEAR_SYM : KP_NEAR_1S, st_, sym_bounds_.get() + c,
                         double(nq) * nq);
    }
  }

  if (!plan.sing_pair_.empty()) {
    g_prof.begin(st_);
    launch_near_singular(dctx(), Pack::at<long long>(base, o_sp),
                         Pack::at<int>(base, o_se), int(plan.sing_pair_.size()),
                         bundles.get(), plan.bundles_, bad.get(), st_);
    g_prof.end(KP_NEAR_SING, st_, double(plan.sing_pair_.size()));
  }
  g_prof.begin(st_);
  launch_gather(Pack::at<GatherJob>(base, o_gj), Pack::at<int>(base, o_go),
                int(plan.gather_.size()), n_gblk, Pack::at<NodeDesc>(base, o_de),
                bundles.get(), plan.bundles_, st_);
  // bytes: 4 bundle reads (16 B each) + one 16 B store per entry
  g_prof.end(KP_GATHER, st_, 80.0 * double(plan.entries_));
  CK(cudaGetLastError());
  staging.fence(st_);
  plan.clear();
}

namespace {

// Common nodes of a cell's enclosed list P and its child's C, as (position in
// C, position in P) pairs in P order, and the positions of P not in C.
void intersect_enclosed(const std::vector<int>& P, const std::vector<int>& C,
                        std::vector<int2>& common, std::vector<int>& rest) {
  common.clear();
  rest.clear();
  if (std::is_sorted(P.begin(), P.end()) && std::is_sorted(C.begin(), C.end())) {
    size_t j = 0;
    for (size_t i = 0; i < P.size(); ++i) {
      while (j < C.size() && C[j] < P[i]) ++j;
      if (j < C.size() && C[j] == P[i]) common.push_back(make_int2(int(j), int(i)));
      else rest.push_back(int(i));
    }
    return;
  }
  std::vector<std::pair<int, int>> idx(C.size());
  for (size_t j = 0; j < C.size(); ++j) idx[j] = {C[j], int(j)};
  std::sort(idx.begin(), idx.end());
  for (size_t i = 0; i < P.size(); ++i) {
    auto it = std::lower_bound(idx.begin(), idx.end(), std::make_pair(P[i], -1));
    if (it != idx.end() && it->first == P[i]) common.push_back(make_int2(it->second, int(i)));
    else rest.push_back(int(i));
  }
}

// Reuse copies planned by one planning thread (offsets local to the part).
struct ReusePart {
  std::vector<ReuseTask> tasks;
  std::vector<int2> rows, cols;
  long long entries = 0;
};

// EBEM_REUSE: 0 = every level computes all its entries (A/B); 1 = only the
// copies that reproduce the computed entries bit for bit (same bundles, same
// summation order); 2 (default) = also the sibling-block entries taken from
// the other orientation of a symmetric evaluation (equal up to rounding).
int reuse_level() {
  static const int lv = [] {
    const char* e = std::getenv("EBEM_REUSE");
    return e == nullptr ? 2 : std::atoi(e);
  }();
  return lv;
}
bool reuse_enabled() { return reuse_level() >= 1; }

}  // namespace

void Problem::interaction(const std::vector<BasisReq>& req,
                          std::vector<ProxyGeom>& geom,
                          std::vector<size_t>& tv_off,
                          std::vector<size_t>& tu_off, std::vector<int>& n_out,
                          DBuf<double>& tbuf, const PrevLevel* prev) {
  const int m = pcfg_.m_prime;
  const size_t nc_ = req.size();
  geom.resize(nc_);
  tv_off.resize(nc_);
  tu_off.resize(nc_);
  n_out.resize(nc_);
  size_t run = 0;
  {
    PhaseTimer t_geom("proxy_geometry", nullptr);
    parallel_for(int(nc_), [&](int c) { geom[c] = build_proxy(req[c].begin, req[c].end); });
  }
  for (size_t c = 0; c < nc_; ++c) {
    n_out[c] = 2 * m + 2 * int(geom[c].enclosed.size());
    const size_t ncol = (*req[c].cols)[0].size() + (*req[c].cols)[1].size();
    const size_t nrow = (*req[c].rows)[0].size() + (*req[c].rows)[1].size();
    tv_off[c] = run;
    run += size_t(n_out[c]) * ncol;
    tu_off[c] = run;
    run += size_t(n_out[c]) * nrow;
  }
  {
    PhaseTimer t_alloc("alloc_tbuf", nullptr);
    tbuf.ensure(2 * run + 2);
  }
  if (prev && !(prev->valid && reuse_enabled())) prev = nullptr;
  const double* pbase = nullptr;
  if (prev) pbase = (prev->buf ? scratch().tbuf_alt : scratch().tbuf).get();
  // Cells are planned in contiguous chunks on the planning threads and the
  // chunk plans appended in cell order: the same jobs, offsets and gather
  // order as a serial pass.
  double* base = tbuf.get();
  const int nchunk = int(std::min<size_t>(nc_, size_t(8 * planning_threads())));
  std::vector<FillPlan> parts(nchunk, FillPlan(n_, m, pcfg_.n_gauss));
  std::vector<ReusePart> rparts(nchunk);
  // Cross-level reuse (chained calls): the entry (enclosed node b, skeleton a
  // of child ch) of this cell's near blocks is the entry (b, a) of the
  // child's, whenever b was enclosed by the child's proxy circle too -- the
  // same element-pair bundles summed in the same order.  Those entries are
  // copied from the child's matrices (previous level, other buffer); the
  // near-field fill of the cell covers the remaining enclosed nodes only,
  // one job per child.
  // What the near-field jobs of one cell look like: whether its enclosed
  // nodes split per child (reuse), and which of them each child's job keeps.
  struct NearPrep {
    bool split = false;
    int kc[2] = {0, 0};
    std::vector<int> rest[2];
    bool whole[2] = {true, true};  // child x keeps every enclosed node
  };
  auto prep_near = [&](NearPrep& np, ReusePart& rp, size_t c) {
    double* tv = base + 2 * tv_off[c];
    double* tu = base + 2 * tu_off[c];
    const Lists& rows = *req[c].rows;
    const Lists& cols = *req[c].cols;
    const int no = n_out[c];
    const std::vector<int>& enc = geom[c].enclosed;
    const int ne = int(enc.size());
    bool ok = prev != nullptr && ne > 0;
    int ch[2] = {-1, -1};
    int (&kc)[2] = np.kc;
    for (int x = 0; ok && x < 2; ++x) {
      ch[x] = req[c].child[x];
      ok = ch[x] >= 0 && ch[x] < int(prev->geom.size());
      if (ok) kc[x] = int(prev->spos[ch[x]][0].size());
    }
    // the cell's lists must be the children's skeletons, child 0 first
    for (int a = 0; ok && a < 4; ++a) {
      const std::vector<int>& L = a < 2 ? cols[a] : rows[a - 2];
      ok = int(L.size()) == kc[0] + kc[1];
      for (int x = 0; ok && x < 2; ++x) {
        const std::vector<int>& sn = prev->snode[ch[x]][a];
        ok = int(sn.size()) == kc[x] &&
             std::equal(sn.begin(), sn.end(), L.begin() + (x ? kc[0] : 0));
      }
    }
    std::vector<int2> common[2];
    if (ok) {
      for (int x = 0; x < 2; ++x)
        intersect_enclosed(enc, prev->geom[ch[x]].enclosed, common[x], np.rest[x]);
      ok = !common[0].empty() || !common[1].empty();
    }
    np.split = ok;
    if (!ok) return;
    const int nc0 = int(cols[0].size()), nr0 = int(rows[0].size());
    for (int x = 0; x < 2; ++x) {
      const int j0 = x ? kc[0] : 0, k = kc[x];
      np.whole[x] = common[x].empty();
      if (k == 0 || common[x].empty()) continue;
      // copies: T_V columns from the child's cols skeletons, T_U from rows
      const int cc = ch[x];
      const int cne = int(prev->geom[cc].enclosed.size());
      const long long row_off = (long long)rp.rows.size();
      rp.rows.insert(rp.rows.end(), common[x].begin(), common[x].end());
      for (int w = 0; w < 2; ++w) {  // 0: T_V, 1: T_U
        ReuseTask T{};
        T.src = pbase + 2 * (w ? prev->tu_off[cc] : prev->tv_off[cc]);
        T.dst = w ? tu : tv;
        T.src_ld = prev->n_out[cc];
        T.dst_ld = no;
        T.src_row0 = 2 * m;
        T.src_ne = cne;
        T.dst_row0 = 2 * m;
        T.dst_ne = ne;
        T.n_rows = int(common[x].size());
        T.n_cols = 2 * k;
        T.row_off = row_off;
        T.col_off = (long long)rp.cols.size();
        const int shalf = w ? prev->nr0[cc] : prev->nc0[cc];
        const int dhalf = w ? nr0 : nc0;
        for (int p = 0; p < 2; ++p) {
          const std::vector<int>& sp = prev->spos[cc][2 * w + p];
          for (int j = 0; j < k; ++j)
            rp.cols.push_back(make_int2(p * shalf + sp[j], p * dhalf + j0 + j));
        }
        rp.tasks.push_back(T);
        rp.entries += 2ll * T.n_rows * T.n_cols;
      }
    }
  };
  // Number of enclosed nodes the job of child x (x = -1: the unsplit cell) keeps.
  auto near_count = [&](const NearPrep& np, size_t c, int x) {
    if (x < 0 || np.whole[x]) return int(geom[c].enclosed.size());
    return int(np.rest[x].size());
  };
  // The near-field job of child x of cell c over the kept enclosed nodes
  // [lo, hi) (all of them: the job the unsplit planner makes).
  auto plan_piece = [&](FillPlan& fp, const NearPrep& np, size_t c, int x, int lo, int hi) {
    double* tv = base + 2 * tv_off[c];
    double* tu = base + 2 * tu_off[c];
    const Lists& rows = *req[c].rows;
    const Lists& cols = *req[c].cols;
    const int no = n_out[c];
    const std::vector<int>& enc = geom[c].enclosed;
    const int ne = int(enc.size());
    const int nc0 = int(cols[0].size()), nr0 = int(rows[0].size());
    const bool all = lo == 0 && hi == near_count(np, c, x);
    const bool identity = x < 0 || np.whole[x];
    std::vector<int> sub, pos;
    if (!(all && identity)) {
      sub.resize(hi - lo);
      pos.resize(hi - lo);
      for (int i = lo; i < hi; ++i) {
        pos[i - lo] = identity ? i : np.rest[x][i];
        sub[i - lo] = enc[pos[i - lo]];
      }
    }
    const std::vector<int>& nodes = (all && identity) ? enc : sub;
    const std::vector<int>* pp = (all && identity) ? nullptr : &pos;
    if (x < 0) {
      const int rdest[2] = {0, nr0}, cdest[2] = {0, nc0};
      fp.add_sym_near_part(nodes, pp, ne, rows, rdest, cols, cdest, tv, no, tu, no);
      return;
    }
    const int j0 = x ? np.kc[0] : 0, k = np.kc[x];
    if (k == 0) return;
    Lists rs, cs;
    for (int p = 0; p < 2; ++p) {
      rs[p].assign(rows[p].begin() + j0, rows[p].begin() + j0 + k);
      cs[p].assign(cols[p].begin() + j0, cols[p].begin() + j0 + k);
    }
    const int rdest[2] = {j0, nr0 + j0}, cdest[2] = {j0, nc0 + j0};
    fp.add_sym_near_part(nodes, pp, ne, rs, rdest, cs, cdest, tv, no, tu, no);
  };
  auto plan_near = [&](FillPlan& fp, ReusePart& rp, size_t c) {
    NearPrep np;
    prep_near(np, rp, c);
    if (!np.split) {
      plan_piece(fp, np, c, -1, 0, near_count(np, c, -1));
      return;
    }
    for (int x = 0; x < 2; ++x) plan_piece(fp, np, c, x, 0, near_count(np, c, x));
  };
  // Chunks are planned a batch (one chunk per planning thread) at a time and
  // every wave is executed as soon as its chunks are planned, so the device
  // starts on the first wave while the host plans the rest.
  // waves: consecutive chunks until the bundle count passes the cap (the
  // chunk that crosses it closes the wave), concatenated in parallel
  FillPlan plan(n_, m, pcfg_.n_gauss);
  // Upper levels (few cells, each with a near field of 10^4 .. 10^5 enclosed
  // nodes that takes milliseconds to plan): the proxy blocks, quick to plan,
  // go first as a wave of their own, so the device works on them while the
  // host plans the near field.
  const bool proxy_first = nc_ <= 512 && nc_ > 0;
  if (proxy_first) {
    {
      PhaseTimer t_plan("fill_plan", nullptr);
      parallel_for(nchunk, [&](int k) {
        const size_t c0 = nc_ * size_t(k) / nchunk, c1 = nc_ * size_t(k + 1) / nchunk;
        for (size_t c = c0; c < c1; ++c)
          parts[k].add_proxy(geom[c].cx, geom[c].cy, geom[c].radius, *req[c].rows,
                             *req[c].cols, base + 2 * tv_off[c], n_out[c],
                             base + 2 * tu_off[c], n_out[c]);
      });
    }
    plan.append_many(parts, 0, nchunk);
    for (int q = 0; q < nchunk; ++q) parts[q] = FillPlan(n_, m, pcfg_.n_gauss);
    tl_mark("  proxy wave planned");
    execute(plan);
    // The near fields in pieces of kPiece enclosed nodes per job: a cell's
    // near field is planned by many threads at once and the first wave is
    // ready after one piece per thread, not after whole cells.
    constexpr int kPiece = 8192;
    std::vector<NearPrep> preps(nc_);
    rparts.assign(nc_, ReusePart{});
    {
      PhaseTimer t_plan("fill_plan", nullptr);
      parallel_for(int(nc_), [&](int c) { prep_near(preps[c], rparts[c], size_t(c)); });
    }
    struct Item {
      int c, x, lo, hi;
    };
    std::vector<Item> items;
    for (size_t c = 0; c < nc_; ++c)
      for (int x = preps[c].split ? 0 : -1; x < (preps[c].split ? 2 : 0); ++x) {
        if (x >= 0 && preps[c].kc[x] == 0) continue;
        const int cnt = near_count(preps[c], c, x);
        for (int lo = 0; lo < cnt; lo += kPiece)
          items.push_back(Item{int(c), x, lo, std::min(cnt, lo + kPiece)});
      }
    const int nitems = int(items.size());
    std::vector<FillPlan> iparts(nitems, FillPlan(n_, m, pcfg_.n_gauss));
    const int ibatch = std::max(1, planning_threads());
    int i0 = 0;
    long long iacc = 0;
    for (int ib = 0; ib < nitems; ib += ibatch) {
      const int ie = std::min(nitems, ib + ibatch);
      {
        PhaseTimer t_plan("fill_plan", nullptr);
        parallel_for(ie - ib, [&](int kk) {
          const Item& it = items[ib + kk];
          plan_piece(iparts[ib + kk], preps[it.c], size_t(it.c), it.x, it.lo, it.hi);
        });
      }
      for (int k = ib; k < ie; ++k) {
        iacc += iparts[k].bundles();
        const bool first_early = i0 == 0 && k == ie - 1 && iacc >= kFirstWaveBundles;
        if (iacc > kMaxBundlesPerWave || k == nitems - 1 || first_early) {
          {
            PhaseTimer t_app("fill_plan_append", nullptr);
            plan.append_many(iparts, i0, k + 1);
            for (int q = i0; q <= k; ++q) iparts[q] = FillPlan(n_, m, pcfg_.n_gauss);
          }
          tl_mark("  wave planned");
          execute(plan);
          i0 = k + 1;
          iacc = 0;
        }
      }
    }
  }
  int k0 = 0;
  long long acc = 0;
  const int batch = std::max(1, planning_threads());
  for (int kb = 0; !proxy_first && kb < nchunk; kb += batch) {
    const int ke = std::min(nchunk, kb + batch);
    {
      PhaseTimer t_plan("fill_plan", nullptr);
      parallel_for(ke - kb, [&](int kk) {
        const int k = kb + kk;
        const size_t c0 = nc_ * size_t(k) / nchunk, c1 = nc_ * size_t(k + 1) / nchunk;
        for (size_t c = c0; c < c1; ++c) {
          const Lists& rows = *req[c].rows;
          const Lists& cols = *req[c].cols;
          double* tv = base + 2 * tv_off[c];
          double* tu = base + 2 * tu_off[c];
          const int no = n_out[c];
          if (!proxy_first)
            parts[k].add_proxy(geom[c].cx, geom[c].cy, geom[c].radius, rows, cols, tv,
                               no, tu, no);
          plan_near(parts[k], rparts[k], c);
        }
      });
    }
    for (int k = kb; k < ke; ++k) {
      acc += parts[k].bundles();
      const bool first_early = k0 == 0 && k == ke - 1 && acc >= kFirstWaveBundles;
      if (acc > kMaxBundlesPerWave || k == nchunk - 1 || first_early) {
        {
          PhaseTimer t_app("fill_plan_append", nullptr);
          plan.append_many(parts, k0, k + 1);
          for (int q = k0; q <= k; ++q) parts[q] = FillPlan(n_, m, pcfg_.n_gauss);
        }
        tl_mark("  wave planned");
        execute(plan);
        k0 = k + 1;
        acc = 0;
      }
    }
  }
  // the reuse copies of the level: one launch
  std::vector<ReuseTask> rtasks;
  std::vector<int2> rrows, rcols;
  long long rentries = 0;
  for (ReusePart& rp : rparts) {
    for (ReuseTask T : rp.tasks) {
      T.row_off += (long long)rrows.size();
      T.col_off += (long long)rcols.size();
      rtasks.push_back(T);
    }
    rrows.insert(rrows.end(), rp.rows.begin(), rp.rows.end());
    rcols.insert(rcols.end(), rp.cols.begin(), rp.cols.end());
    rentries += rp.entries;
  }
  if (!rtasks.empty()) {
    std::vector<int> boff(rtasks.size());
    int nblk = 0;
    for (size_t i = 0; i < rtasks.size(); ++i) {
      boff[i] = nblk;
      nblk += (rtasks[i].n_cols + kReuseCols - 1) / kReuseCols;
    }
    Pack pk;
    const size_t o_t = pk.add(rtasks);
    const size_t o_b = pk.add(boff);
    const size_t o_r = pk.add(rrows);
    const size_t o_c = pk.add(rcols);
    char* tb = staging.put(pk, st_);
    g_prof.begin(st_);
    launch_reuse_copy(Pack::at<ReuseTask>(tb, o_t), Pack::at<int>(tb, o_b), int(rtasks.size()),
                      nblk, Pack::at<int2>(tb, o_r), Pack::at<int2>(tb, o_c), st_);
    g_prof.end(KP_REUSE, st_, double(rentries), 32.0 * double(rentries));
    CK(cudaGetLastError());
    staging.fence(st_);
  }
}

void Problem::plan_sibling_block(FillPlan& plan, MapPart& mp, int ca, int cb,
                                 const Lists& rows, const Lists& cols, double* dest, int ld,
                                 const int drow[2], const int dcol[2]) {
  const int m = pcfg_.m_prime;
  bool ok = prev_.valid && reuse_enabled() && ca >= 0 && cb >= 0 &&
            ca < int(prev_.geom.size()) && cb < int(prev_.geom.size());
  for (int p = 0; ok && p < 2; ++p)
    ok = rows[p] == prev_.snode[ca][2 + p] && cols[p] == prev_.snode[cb][p];
  if (!ok) {
    plan.add_true_block(rows, cols, dest, ld, drow, dcol, 0);
    return;
  }
  const std::vector<int>& encA = prev_.geom[ca].enclosed;
  const std::vector<int>& encB = prev_.geom[cb].enclosed;
  const bool sa = std::is_sorted(encA.begin(), encA.end());
  const bool sb = std::is_sorted(encB.begin(), encB.end());
  auto find = [](const std::vector<int>& enc, bool sorted, int node) {
    if (sorted) {
      auto it = std::lower_bound(enc.begin(), enc.end(), node);
      return (it != enc.end() && *it == node) ? int(it - enc.begin()) : -1;
    }
    auto it = std::find(enc.begin(), enc.end(), node);
    return it != enc.end() ? int(it - enc.begin()) : -1;
  };
  const int neA = int(encA.size()), neB = int(encB.size());
  const double* pbase = (prev_.buf ? scratch().tbuf_alt : scratch().tbuf).get();
  // rows whose node lies inside cb's circle: whole rows from cb's T_V
  Lists rest_r, rest_c;
  std::vector<int> rpos[2], cpos[2];
  std::vector<int2> rows_v, cols_all, rows_u, cols_u;
  for (int p = 0; p < 2; ++p)
    for (int ia = 0; ia < int(rows[p].size()); ++ia) {
      const int ib = find(encB, sb, rows[p][ia]);
      if (ib >= 0) {
        rows_v.push_back(make_int2(2 * m + p * neB + ib, drow[p] + ia));
      } else {
        rest_r[p].push_back(rows[p][ia]);
        rpos[p].push_back(ia);
        rows_u.push_back(make_int2(p * prev_.nr0[ca] + prev_.spos[ca][2 + p][ia], drow[p] + ia));
      }
    }
  const bool other = reuse_level() >= 2;
  for (int q = 0; q < 2; ++q)
    for (int jb = 0; jb < int(cols[q].size()); ++jb) {
      cols_all.push_back(make_int2(q * prev_.nc0[cb] + prev_.spos[cb][q][jb], dcol[q] + jb));
      const int ja = other ? find(encA, sa, cols[q][jb]) : -1;
      if (ja >= 0) {
        cols_u.push_back(make_int2(2 * m + q * neA + ja, dcol[q] + jb));
      } else {
        rest_c[q].push_back(cols[q][jb]);
        cpos[q].push_back(jb);
      }
    }
  if (!rows_v.empty()) {
    MapTask T{};
    T.src = pbase + 2 * prev_.tv_off[cb];
    T.dst = dest;
    T.src_ld = prev_.n_out[cb];
    T.dst_ld = ld;
    T.n_rows = int(rows_v.size());
    T.n_cols = int(cols_all.size());
    T.swap = 0;
    T.row_off = (long long)mp.rows.size();
    T.col_off = (long long)mp.cols.size();
    mp.rows.insert(mp.rows.end(), rows_v.begin(), rows_v.end());
    mp.cols.insert(mp.cols.end(), cols_all.begin(), cols_all.end());
    mp.tasks.push_back(T);
  }
  if (!rows_u.empty() && !cols_u.empty()) {
    // the remaining rows against the columns inside ca's circle: ca's
    // T_U = M_U^H holds conj(K(row, enclosed)) at (enclosed, row)
    MapTask T{};
    T.src = pbase + 2 * prev_.tu_off[ca];
    T.dst = dest;
    T.src_ld = prev_.n_out[ca];
    T.dst_ld = ld;
    T.n_rows = int(rows_u.size());
    T.n_cols = int(cols_u.size());
    T.swap = 1;
    T.row_off = (long long)mp.rows.size();
    T.col_off = (long long)mp.cols.size();
    mp.rows.insert(mp.rows.end(), rows_u.begin(), rows_u.end());
    mp.cols.insert(mp.cols.end(), cols_u.begin(), cols_u.end());
    mp.tasks.push_back(T);
  }
  const std::vector<int>* const rp[2] = {&rpos[0], &rpos[1]};
  const std::vector<int>* const cp[2] = {&cpos[0], &cpos[1]};
  plan.add_true_block(rest_r, rest_c, dest, ld, drow, dcol, 0, rp, cp);
}

void Problem::run_map_copies(std::vector<MapPart>& parts) {
  std::vector<MapTask> tasks;
  std::vector<int2> rows, cols;
  double entries = 0.0;
  for (MapPart& mp : parts) {
    for (MapTask T : mp.tasks) {
      T.row_off += (long long)rows.size();
      T.col_off += (long long)cols.size();
      entries += double(T.n_rows) * T.n_cols;
      tasks.push_back(T);
    }
    rows.insert(rows.end(), mp.rows.begin(), mp.rows.end());
    cols.insert(cols.end(), mp.cols.begin(), mp.cols.end());
    mp = MapPart{};
  }
  if (tasks.empty()) return;
  Pack pk;
  const size_t o_t = pk.add(tasks);
  const size_t o_r = pk.add(rows);
  const size_t o_c = pk.add(cols);
  char* tb = staging.put(pk, st_);
  g_prof.begin(st_);
  launch_map_copy(Pack::at<MapTask>(tb, o_t), int(tasks.size()), Pack::at<int2>(tb, o_r),
                  Pack::at<int2>(tb, o_c), st_);
  g_prof.end(KP_REUSE, st_, entries, 32.0 * entries);
  CK(cudaGetLastError());
  staging.fence(st_);
}

// TSQR rounds until each block is an n x n R or fits one CTA's shared memory
// (then the column-pivoted pass takes it directly); updates q in place to
// point at the reduced blocks (scratch().qr_rounds).
void reduce_tall(std::vector<TallBlock>& q, cudaStream_t st, bool force) {
  Scratch& S = scratch();
  std::vector<DBuf<double>>& qr_rounds_ = S.qr_rounds;
  DBuf<double2>& gws = S.gws;
  Staging& staging = S.staging;
  // ---- TSQR rounds until each input is an n x n R or fits one CTA's shared
  // memory.  Inputs with n <= kTsqrMaxCols stream through k_tsqr (row pieces
  // sized so a round fills the GPU, the pieces' R factors stacked for the next
  // round); wider ones use the chunked k_qr_reduce tree.
  static const int n_sm = [] {
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    return v > 0 ? v : 148;
  }();
  static const int forced_pieces = [] {  // experiments: EBEM_TSQR_PIECES
    const char* e = std::getenv("EBEM_TSQR_PIECES");
    return e ? std::atoi(e) : 0;
  }();
  size_t round = 0;
  for (;;) {
    std::vector<QrTask> tasks, streamv[8];
    std::vector<size_t> out_off(q.size(), 0);
    size_t out_total = 0, ws_total = 0;
    std::vector<int> pieces(q.size(), 0);
    std::vector<char> streamed(q.size(), 0);
    double work = 0.0;  // streamed rows x steps x (n + 64) / block rows
    for (size_t i = 0; i < q.size(); ++i) {
      const TallBlock& x = q[i];
      const size_t bytes = size_t(x.rows) * x.n * 16;
      // blocks that fit one CTA go straight to the pivoted QR unless they are
      // tall enough that reducing them first is cheaper (EBEM_TSQR_RATIO:
      // rows / n above which a block is reduced anyway; 0 = never; measured
      // at 2N = 2^19: 3 saves ~7 ms over 0)
      static const double ratio = [] {
        const char* e = std::getenv("EBEM_TSQR_RATIO");
        return e ? std::atof(e) : 3.0;
      }();
      const bool tall = ratio > 0.0 && x.rows > ratio * x.n && tsqr_variant(x.n) >= 0;
      if ((bytes <= size_t(kSmemCap) && !force && !tall) || x.rows <= x.n) continue;
      if (tsqr_variant(x.n) >= 0) {
        streamed[i] = 1;
        work += double(x.rows) * x.n * (x.n + 64) / tsqr_block_rows(x.n);
      } else if (x.rows > 2 * x.n) {
        const int chunk = std::max(2 * x.n, int(kSmemCap / (16 * size_t(x.n))));
        pieces[i] = (x.rows + chunk - 1) / chunk;
      }
    }
    int cps = 1;  // resident CTAs per SM of the streamed inputs' variants
    for (size_t i = 0; i < q.size(); ++i)
      if (streamed[i]) cps = std::max(cps, tsqr_ctas_per_sm(q[i].n));
    static const double waves = [] {  // experiments: EBEM_TSQR_WAVES
      const char* e = std::getenv("EBEM_TSQR_WAVES");
      return e ? std::atof(e) : 4.0;
    }();
    const double per_cta = work / (waves * n_sm * cps);
    for (size_t i = 0; i < q.size(); ++i) {
      if (!streamed[i]) continue;
      const TallBlock& x = q[i];
      const double w = double(x.rows) * x.n * (x.n + 64) / tsqr_block_rows(x.n);
      const int cap = std::max(1, x.rows / (4 * x.n));
      pieces[i] = std::min(cap, std::max(1, int(std::ceil(w / per_cta))));
      if (forced_pieces > 0) pieces[i] = std::min(forced_pieces, std::max(1, x.rows / x.n));
    }
    for (size_t i = 0; i < q.size(); ++i) {
      if (!pieces[i]) continue;
      out_off[i] = out_total;
      out_total += size_t(pieces[i]) * q[i].n * q[i].n;
    }
    if (out_total == 0) break;
    if (qr_rounds_.size() <= round) qr_rounds_.emplace_back();
    qr_rounds_[round].ensure(2 * out_total);
    double* ob = qr_rounds_[round].get();
    ++round;
    size_t smemv[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (size_t i = 0; i < q.size(); ++i) {
      if (!pieces[i]) continue;
      const TallBlock& x = q[i];
      const int chunk = (x.rows + pieces[i] - 1) / pieces[i];
      const int ld_out = pieces[i] * x.n;
      for (int pc = 0; pc < pieces[i]; ++pc) {
        const int r0 = pc * chunk;
        const int rr = std::min(chunk, x.rows - r0);
        QrTask t{};
        t.src = x.p + 2 * size_t(r0);
        t.dst = ob + 2 * (out_off[i] + size_t(pc) * x.n);
        t.rows = rr;
        t.n = x.n;
        t.ld = x.ld;
        t.dst_ld = ld_out;
        if (streamed[i]) {
          const int v = tsqr_variant(x.n);
          streamv[v].push_back(t);
          smemv[v] = std::max(smemv[v], tsqr_smem_bytes(x.n));
          continue;
        }
        t.in_smem = size_t(rr) * x.n * 16 <= size_t(kSmemCap);
        t.ws_off = (long long)ws_total;
        if (!t.in_smem) ws_total += size_t(rr) * x.n;
        tasks.push_back(t);
      }
    }
    gws.ensure(ws_total + 1);
    Pack pk;
    const size_t o = pk.add(tasks);
    size_t ov[8];
    for (int v = 0; v < 8; ++v) ov[v] = pk.add(streamv[v]);
    char* tb = staging.put(pk, st);
    size_t smem = 0;
    for (const QrTask& t : tasks)
      if (t.in_smem) smem = std::max(smem, size_t(t.rows) * t.n * 16);
    double fl = 0.0;
    double by = 0.0;  // the block read once, its reduced rows written once
    for (const auto* v : {&tasks, &streamv[0], &streamv[1], &streamv[2], &streamv[3], &streamv[4], &streamv[5], &streamv[6], &streamv[7]})
      for (const QrTask& t : *v) {
        const double mm = t.rows, nn = std::min(t.rows, t.n);
        // complex Householder QR with k = min(m, n) reflectors:
        // 16 m n k - 8 (m + n) k^2 + 16 k^3 / 3 real flops (8 m n^2 - 8 n^3 / 3 at k = n)
        fl += 16.0 * mm * t.n * nn - 8.0 * (mm + t.n) * nn * nn + 16.0 / 3.0 * nn * nn * nn;
        by += 16.0 * (mm + nn) * t.n;
      }
    g_prof.begin(st);
    // (the team-layout k_qr_team measured slower on these shapes: 485 vs 404 ms)
    launch_qr_reduce(Pack::at<QrTask>(tb, o), int(tasks.size()), smem, gws.get(), st);
    for (int v = 0; v < 8; ++v)
      launch_tsqr(Pack::at<QrTask>(tb, ov[v]), int(streamv[v].size()), v, smemv[v], st);
    g_prof.end(KP_QR, st, fl, by);
    CK(cudaGetLastError());
    staging.fence(st);
    for (size_t i = 0; i < q.size(); ++i) {
      if (!pieces[i]) continue;
      q[i].p = ob + 2 * out_off[i];
      q[i].rows = pieces[i] * q[i].n;
      q[i].ld = q[i].rows;
    }
  }
}

void Problem::bases(const std::vector<BasisReq>& req, double eps,
                    std::vector<BasisRes>& res, DBuf<double>& vbuf,
                    DBuf<double>& ubuf, double* fill_seconds, bool chain, bool defer_lists) {
  const size_t ncell = req.size();
  res.assign(ncell, BasisRes{});
  if (ncell == 0) return;
  std::vector<ProxyGeom> geom;
  std::vector<size_t> tv_off, tu_off;
  std::vector<int> n_out;
  // chained calls alternate between the two interaction buffers, so the
  // previous level's matrices outlive this level's fill (cross-level reuse)
  if (!chain) prev_.valid = false;
  const int cur_buf = prev_.valid ? 1 - prev_.buf : 0;
  DBuf<double>& tbuf = cur_buf ? scratch().tbuf_alt : tbuf_;
  const double t0 = now();
  tl_mark("  bases start");
  interaction(req, geom, tv_off, tu_off, n_out, tbuf, chain ? &prev_ : nullptr);
  tl_mark("  fill enq");
  if (fill_seconds) {
    CK(cudaStreamSynchronize(st_));
    *fill_seconds = now() - t0;
  }

  // ---- the four ID inputs per cell: column halves of T_V and T_U
  std::vector<TallBlock> q(4 * ncell);
  for (size_t c = 0; c < ncell; ++c) {
    const Lists& rows = *req[c].rows;
    const Lists& cols = *req[c].cols;
    const int nc0 = int(cols[0].size()), nc1 = int(cols[1].size());
    const int nr0 = int(rows[0].size()), nr1 = int(rows[1].size());
    if (nc0 == 0 || nc1 == 0 || nr0 == 0 || nr1 == 0)
      throw Error(EBEM_INVALID_ARGUMENT, "Cpqr: empty matrix");
    const int no = n_out[c];
    const double* tv = tbuf.get() + 2 * tv_off[c];
    const double* tu = tbuf.get() + 2 * tu_off[c];
    q[4 * c + 0] = {tv, no, nc0, no};
    q[4 * c + 1] = {tv + 2 * size_t(no) * nc0, no, nc1, no};
    q[4 * c + 2] = {tu, no, nr0, no};
    q[4 * c + 3] = {tu + 2 * size_t(no) * nr0, no, nr1, no};
  }
  PhaseTimer* t_qr = new PhaseTimer("id_tsqr", st_);
  reduce_tall(q, st_);
  delete t_qr;
  PhaseTimer t_cpqr("id_cpqr+interp", st_);
  // ---- pivoted QR of every input
  const size_t nq = q.size();
  size_t jp_total = 0, r_total = 0, ws_total = 0;
  std::vector<size_t> jp_off(nq), r_off(nq);
  for (size_t i = 0; i < nq; ++i) {
    jp_off[i] = jp_total;
    jp_total += size_t(q[i].n) + 1;
    r_off[i] = r_total;
    r_total += size_t(q[i].n) * q[i].n;
  }
  DBuf<int>& d_jp = id_jp_;
  DBuf<int>& d_steps = id_steps_;
  DBuf<double>& d_rd = id_rd_;
  DBuf<double>& d_r = id_r_;
  d_jp.ensure(jp_total);
  d_steps.ensure(nq);
  d_rd.ensure(jp_total);
  d_r.ensure(2 * r_total);
  std::vector<CpqrTask> ct(nq);
  size_t smem = 0;
  for (size_t i = 0; i < nq; ++i) {
    if (q[i].n > kMaxCpqrCols)
      throw Error(EBEM_INVALID_ARGUMENT, "Cpqr: more columns than supported");
    CpqrTask& t = ct[i];
    t.src = q[i].p;
    t.rows = q[i].rows;
    t.n = q[i].n;
    t.ld = q[i].ld;
    t.in_smem = size_t(t.rows) * t.n * 16 <= size_t(kSmemCap);
    t.stop_rel = 1e-14;  // kPivotFloor, proj/src/compression.cpp:15
    t.jpvt = d_jp.get() + jp_off[i];
    t.rdiag = d_rd.get() + jp_off[i];
    t.steps = d_steps.get() + i;
    t.r_out = d_r.get() + 2 * r_off[i];
    t.r_ld = t.n;
    t.ws_off = (long long)ws_total;
    if (!t.in_smem) ws_total += size_t(t.rows) * t.n;
    else smem = std::max(smem, size_t(t.rows) * t.n * 16);
  }
  gws.ensure(ws_total + 1);
  {
    // blocks of at most 32 x 32 run one warp per matrix (EBEM_CPQR_WARP=0: all
    // through the team kernel, A/B)
    static const bool warp_cpqr = [] {
      const char* e = std::getenv("EBEM_CPQR_WARP");
      return e == nullptr || std::atoi(e) != 0;
    }();
    std::vector<CpqrTask> ct_w, ct_t;
    for (const CpqrTask& t : ct)
      ((warp_cpqr && t.n <= 32 && t.rows <= 32) ? ct_w : ct_t).push_back(t);
    Pack pk;
    const size_t o = pk.add(ct_t);
    const size_t ow = pk.add(ct_w);
    char* tb = staging.put(pk, st_);
    double fl = 0.0;  // full-rank bound of the pivoted QR flops
    double by = 0.0;  // the (reduced) block read once, R written once
    for (const CpqrTask& t : ct) {
      const double mm = t.rows, nn = std::min(t.rows, t.n);
      // full-rank bound of the pivoted QR: 16 m n k - 8 (m + n) k^2 + 16 k^3 / 3
      fl += 16.0 * mm * t.n * nn - 8.0 * (mm + t.n) * nn * nn + 16.0 / 3.0 * nn * nn * nn;
      by += 16.0 * (mm + nn) * t.n;
    }
    g_prof.begin(st_);
    launch_cpqr_team(Pack::at<CpqrTask>(tb, o), int(ct_t.size()), smem, gws.get(), st_);
    launch_cpqr_warp(Pack::at<CpqrTask>(tb, ow), int(ct_w.size()), st_);
    g_prof.end(KP_CPQR, st_, fl, by);
    CK(cudaGetLastError());
    staging.fence(st_);
  }
  int* const h_jp = scratch().h_jp.ensure(jp_total);
  int* const h_steps = scratch().h_steps.ensure(nq);
  double* const h_rd = scratch().h_rd.ensure(jp_total);
  CK(cudaMemcpyAsync(h_jp, d_jp.get(), jp_total * 4, cudaMemcpyDeviceToHost, st_));
  CK(cudaMemcpyAsync(h_steps, d_steps.get(), nq * 4, cudaMemcpyDeviceToHost, st_));
  CK(cudaMemcpyAsync(h_rd, d_rd.get(), jp_total * 8, cudaMemcpyDeviceToHost, st_));
  tl_mark("  id enq");
  CK(cudaStreamSynchronize(st_));
  tl_mark("  readback");
  check_domain();  // the fill's element-length guard, read after the sync

  // ---- shared rank (basis_from_interactions, compression.cpp:92-99), on the
  // planning threads; the offsets follow serially
  {
    const int nch = int(std::min<size_t>(ncell, size_t(4 * planning_threads())));
    parallel_for(nch, [&](int kq) {
      const size_t c0 = ncell * size_t(kq) / nch, c1 = ncell * size_t(kq + 1) / nch;
      for (size_t c = c0; c < c1; ++c) {
        int k = 0, cap = std::numeric_limits<int>::max();
        for (int a = 0; a < 4; ++a) {
          const size_t i = 4 * c + a;
          const double* rd = h_rd + jp_off[i];
          const int steps = h_steps[i];
          const int mn = std::min(q[i].rows, q[i].n);
          // eps_rank(eps): first j with |R_jj| <= eps |R_00| (0 if R_00 == 0)
          int er;
          if (steps == 0 && mn > 0 && rd[0] == 0.0) {
            er = 0;
          } else {
            er = std::min(steps, mn);
            const int lim = std::min(steps + 1, mn);
            for (int j = 0; j < lim; ++j)
              if (rd[j] <= eps * rd[0]) { er = j; break; }
          }
          k = std::max(k, er);
          cap = std::min(cap, steps);
        }
        k = std::min(k, cap);
        const Lists& rows = *req[c].rows;
        const Lists& cols = *req[c].cols;
        BasisRes& r = res[c];
        r.k = k;
        r.saturated = k >= std::min(std::min(cols[0].size(), cols[1].size()),
                                    std::min(rows[0].size(), rows[1].size()));
      }
    });
  }
  size_t v_total = 0, u_total = 0;
  for (size_t c = 0; c < ncell; ++c) {
    const Lists& rows = *req[c].rows;
    const Lists& cols = *req[c].cols;
    BasisRes& r = res[c];
    r.v_off = v_total;
    v_total += size_t(r.k) * (cols[0].size() + cols[1].size());
    r.u_off = u_total;
    u_total += size_t(r.k) * (rows[0].size() + rows[1].size());
  }
  // (the skeleton lists are filled in after the interpolation launch below:
  // the device needs only the ranks)
  // ---- interpolation coefficients
  vbuf.ensure(2 * v_total + 2);
  ubuf.ensure(2 * u_total + 2);
  std::vector<InterpTask> it;
  int max_k = 1;
  for (size_t c = 0; c < ncell; ++c) {
    const int k = res[c].k;
    if (k == 0) continue;
    max_k = std::max(max_k, k);
    const Lists& rows = *req[c].rows;
    const Lists& cols = *req[c].cols;
    size_t vo = res[c].v_off, uo = res[c].u_off;
    for (int a = 0; a < 4; ++a) {
      const size_t i = 4 * c + a;
      InterpTask t{};
      t.r = d_r.get() + 2 * r_off[i];
      t.jpvt = d_jp.get() + jp_off[i];
      t.k = k;
      t.n = q[i].n;
      t.r_ld = q[i].n;
      if (a < 2) {
        t.out = vbuf.get() + 2 * vo;
        t.out_ld = k;
        t.adjoint = 0;
        vo += size_t(k) * (a == 0 ? cols[0].size() : cols[1].size());
      } else {
        t.out = ubuf.get() + 2 * uo;
        t.out_ld = t.n;
        t.adjoint = 1;
        uo += size_t(k) * (a == 2 ? rows[0].size() : rows[1].size());
      }
      it.push_back(t);
    }
  }
  if (!it.empty()) {
    Pack pk;
    const size_t o = pk.add(it);
    char* tb = staging.put(pk, st_);
    double fl = 0.0;
    for (const InterpTask& t : it) fl += 4.0 * t.k * t.k * double(t.n - t.k);
    g_prof.begin(st_);
    launch_interp(Pack::at<InterpTask>(tb, o), int(it.size()), max_k, st_);
    g_prof.end(KP_INTERP, st_, fl);
    CK(cudaGetLastError());
    staging.fence(st_);
  }
  // ---- skeleton lists in pivot order and, for chained calls, what the next
  // level's reuse needs of this one: finish_bases (deferred by the level
  // loop until its merges are enqueued -- the device needs only the ranks)
  pend_.active = true;
  pend_.chain = chain;
  pend_.cur_buf = cur_buf;
  pend_.req = &req;
  pend_.res = &res;
  pend_.h_jp = h_jp;
  pend_.jp_off = std::move(jp_off);
  pend_.geom = std::move(geom);
  pend_.tv_off = std::move(tv_off);
  pend_.tu_off = std::move(tu_off);
  pend_.n_out = std::move(n_out);
  if (!defer_lists) finish_bases();
}

void Problem::finish_bases() {
  if (!pend_.active) return;
  pend_.active = false;
  const std::vector<BasisReq>& req = *pend_.req;
  std::vector<BasisRes>& res = *pend_.res;
  const size_t ncell = req.size();
  const bool chain = pend_.chain;
  const int* h_jp = pend_.h_jp;
  const std::vector<size_t>& jp_off = pend_.jp_off;
  if (chain) {
    prev_.valid = true;
    prev_.buf = pend_.cur_buf;
    prev_.geom = std::move(pend_.geom);
    prev_.tv_off = std::move(pend_.tv_off);
    prev_.tu_off = std::move(pend_.tu_off);
    prev_.n_out = std::move(pend_.n_out);
    prev_.nc0.resize(ncell);
    prev_.nr0.resize(ncell);
    prev_.spos.resize(ncell);  // (the per-cell vectors are reassigned below)
    prev_.snode.resize(ncell);
  }
  const int nchunk = int(std::min<size_t>(ncell, size_t(4 * planning_threads())));
  parallel_for(nchunk, [&](int kq) {
    const size_t c0 = ncell * size_t(kq) / nchunk, c1 = ncell * size_t(kq + 1) / nchunk;
    for (size_t c = c0; c < c1; ++c) {
      const Lists& rows = *req[c].rows;
      const Lists& cols = *req[c].cols;
      BasisRes& r = res[c];
      const int k = r.k;
      for (int a = 0; a < 4; ++a) {
        const int* jp = h_jp + jp_off[4 * c + a];
        const std::vector<int>& src = a == 0 ? cols[0] : a == 1 ? cols[1] : a == 2 ? rows[0] : rows[1];
        std::vector<int>& dst = a == 0 ? r.scol[0] : a == 1 ? r.scol[1] : a == 2 ? r.srow[0] : r.srow[1];
        dst.resize(k);
        for (int j = 0; j < k; ++j) dst[j] = src[jp[j]];
        if (chain) {
          prev_.spos[c][a].assign(jp, jp + k);
          prev_.snode[c][a] = dst;
        }
      }
      if (chain) {
        prev_.nc0[c] = int(cols[0].size());
        prev_.nr0[c] = int(rows[0].size());
      }
    }
  });
}

void Problem::true_block_host(const Lists& rows, const Lists& cols, double* out) {
  const int nr = int(rows[0].size() + rows[1].size());
  const int nc = int(cols[0].size() + cols[1].size());
  if (nr == 0 || nc == 0) return;
  for (const auto& l : {rows[0], rows[1], cols[0], cols[1]})
    for (int g : l)
      if (g < 0 || g >= n_) throw Error(EBEM_INVALID_ARGUMENT, "true_block: node out of range");
  DBuf<double> d;
  d.alloc(2 * size_t(nr) * nc);
  FillPlan plan(n_, pcfg_.m_prime, pcfg_.n_gauss);
  const int drow[2] = {0, int(rows[0].size())};
  const int dcol[2] = {0, int(cols[0].size())};
  plan.add_true_block(rows, cols, d.get(), nr, drow, dcol, 0);
  execute(plan);
  check_domain();
  CK(cudaMemcpyAsync(out, d.get(), 16 * size_t(nr) * nc, cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
}

void Problem::rhs_plane(int kind, const double* angles, int m, double amp,
                        double* out_host) {
  if (m <= 0) return;
  DBuf<double> da, dout;
  da.alloc(m);
  dout.alloc(4 * size_t(n_) * m);
  CK(cudaMemcpyAsync(da.get(), angles, 8 * size_t(m), cudaMemcpyHostToDevice, st_));
  const int rn = int(acfg_.rhs_nodes * acfg_.refine + 0.5);
  g_prof.begin(st_);
  launch_rhs_plane(dctx(), n_, kind, da.get(), m, amp, rn, dout.get(), st_);
  g_prof.end(KP_RHS, st_, 2.0 * n_ * m * rn);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_host, dout.get(), 32 * size_t(n_) * m, cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
}

void Problem::field(const double* boundary_u, const double* pts, int m, int n_gauss,
                    int kind, double angle, double amp, double* out_u, double* out_int) {
  if (m <= 0) return;
  if (n_gauss < 1 || n_gauss > kMaxGauss)
    throw Error(EBEM_INVALID_ARGUMENT, "gauss_rule: unsupported order " + std::to_string(n_gauss));
  double h = 0.0;  // Mesh::max_length
  for (int e = 0; e < n_; ++e) {
    const int f = e + 1 == n_ ? 0 : e + 1;
    h = std::max(h, std::hypot(xy_[2 * f] - xy_[2 * e], xy_[2 * f + 1] - xy_[2 * e + 1]));
  }
  DBuf<double> dp, dd, du, dout, dint;
  dp.alloc(2 * size_t(m));
  dd.alloc(m);
  CK(cudaMemcpyAsync(dp.get(), pts, 16 * size_t(m), cudaMemcpyHostToDevice, st_));
  launch_boundary_distance(dctx(), dp.get(), m, dd.get(), st_);
  std::vector<double> dist(m);
  CK(cudaMemcpyAsync(dist.data(), dd.get(), 8 * size_t(m), cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
  for (int p = 0; p < m; ++p)
    if (dist[p] <= h)
      throw Error(EBEM_INVALID_ARGUMENT,
                  "evaluate_scattered: point (" + std::to_string(pts[2 * p]) + ", " +
                      std::to_string(pts[2 * p + 1]) + ") is " + std::to_string(dist[p]) +
                      " from the boundary; offset it beyond one element length (" +
                      std::to_string(h) + ")");
  du.alloc(4 * size_t(n_));
  dout.alloc(4 * size_t(m));
  if (out_int) dint.alloc(m);
  CK(cudaMemcpyAsync(du.get(), boundary_u, 32 * size_t(n_), cudaMemcpyHostToDevice, st_));
  launch_field(dctx(), du.get(), dp.get(), m, n_gauss, kind, angle, amp, dout.get(),
               out_int ? dint.get() : nullptr, st_);
  ++g_launches;
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out_u, dout.get(), 32 * size_t(m), cudaMemcpyDeviceToHost, st_));
  if (out_int)
    CK(cudaMemcpyAsync(out_int, dint.get(), 8 * size_t(m), cudaMemcpyDeviceToHost, st_));
  CK(cudaStreamSynchronize(st_));
}

// ------------------------------------------------------------ batched LA
namespace {
// k_getrs stages the LU in shared memory up to this many bytes per launch
// (shared by all tasks of the launch; larger tasks read L2).
int g_getrs_smem = 0;
int g_getrs_maxn = 0;
int g_getrs_cpw = 1;
int g_gemm_narrow = 0;  // GEMV template of the current k_gemm launch (0: tiled)

// Algorithmic HBM bytes of one batched-LA task: operands read once, the
// result written once (complex double = 16 B).
double task_bytes(const CopyTask& c) { return 32.0 * c.rows * c.cols; }
double task_bytes(const GemmTask& g) {
  const bool acc = g.beta_re != 0.0 || g.beta_im != 0.0;
  return 16.0 * (double(g.m) * g.k + double(g.k) * g.n + (acc ? 2.0 : 1.0) * g.m * g.n);
}
double task_bytes(const LuSolveTask& s) {
  return 16.0 * (double(s.n) * s.n + 2.0 * double(s.n) * s.nrhs);
}

template <class T, class F, class U>
void run_blocked(Problem& P, const std::vector<T>& t, F blocks_of,
                 void (*launch)(const T*, const int*, int, int, cudaStream_t),
                 int id, U units_of) {
  if (t.empty()) return;
  std::vector<int> boff(t.size());
  int total = 0;
  for (size_t i = 0; i < t.size(); ++i) {
    boff[i] = total;
    total += blocks_of(t[i]);
  }
  if (total == 0) return;
  if (P.recorder) {
    P.recorder->add(id, t, boff, total,
                    id == KP_GETRS ? g_getrs_smem : id == KP_GEMM ? g_gemm_narrow : 0,
                    id == KP_GETRS ? (g_getrs_maxn | ((g_getrs_cpw + 2) << 16)) : 0);
    return;
  }
  Pack pk;
  const size_t o1 = pk.add(t);
  const size_t o2 = pk.add(boff);
  char* tb = P.staging.put(pk, P.stream());
  double units = 0.0, bytes = 0.0;
  for (const T& x : t) units += units_of(x), bytes += task_bytes(x);
  g_prof.begin(P.stream());
  launch(Pack::at<T>(tb, o1), Pack::at<int>(tb, o2), int(t.size()), total,
         P.stream());
  g_prof.end(id, P.stream(), units, bytes);
  P.staging.fence(P.stream());
  CK(cudaGetLastError());

}
}  // namespace

namespace {
std::vector<char>& recorder_pool() {  // host task buffer of the last recording (API mutex held)
  static std::vector<char> pool;
  return pool;
}
}  // namespace

void Recorder::begin() { pk_.adopt(std::move(recorder_pool())); }

void Recorder::finalize(cudaStream_t st) {
  if (!pk_.bytes()) return;
  dev_.alloc(pk_.bytes());
  for (const Launch& l : launches_)  // the warm-ups cover the task arrays too
    if (l.kind == kPrefetchKind) {
      PrefetchTask* pt = reinterpret_cast<PrefetchTask*>(pk_.mutable_data() + l.task_off);
      pt[l.n_tasks - 1] = PrefetchTask{dev_.get(), pk_.bytes()};
    }
  CK(cudaMemcpyAsync(dev_.get(), pk_.data(), pk_.bytes(), cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  recorder_pool() = pk_.take();  // the host copy is not needed again
}

void Recorder::replay(cudaStream_t st, int phase) {
  char* base = dev_.get();
  for (int i = marks_[phase]; i < marks_[phase + 1]; ++i) {
    const Launch& l = launches_[i];
    const int* boff = Pack::at<int>(base, l.boff_off);
    switch (l.kind) {
      case KP_COPY:
        launch_copy(Pack::at<CopyTask>(base, l.task_off), boff, l.n_tasks, l.n_blocks, st);
        break;
      case KP_GEMM:
        launch_gemm(Pack::at<GemmTask>(base, l.task_off), boff, l.n_tasks, l.n_blocks, st,
                    l.aux);
        break;
      case KP_GETRS:
        launch_getrs(Pack::at<LuSolveTask>(base, l.task_off), boff, l.n_tasks, l.n_blocks, st,
                     l.aux, l.aux2 & 0xffff, (l.aux2 >> 16) - 2);
        break;
      case kPrefetchKind:
        launch_prefetch_l2(Pack::at<PrefetchTask>(base, l.task_off), l.n_tasks, st);
        break;
      default:
        throw Error(EBEM_LOGIC_ERROR, "Recorder: unexpected kernel kind");
    }
  }
}

void run_copies(Problem& P, const std::vector<CopyTask>& t) {
  run_blocked(P, t, [](const CopyTask& c) { return copy_blocks(c.rows, c.cols); },
              launch_copy, KP_COPY,
              [](const CopyTask& c) { return 32.0 * c.rows * c.cols; });
}
namespace {
void launch_gemm_cur(const GemmTask* t, const int* boff, int nt, int nb, cudaStream_t st) {
  launch_gemm(t, boff, nt, nb, st, g_gemm_narrow);
}
}  // namespace

void run_gemms(Problem& P, const std::vector<GemmTask>& t) {
  int narrow = t.empty() ? 0 : 1;  // the smallest kind every task fits
  for (const GemmTask& g : t) {
    const int k = gemm_narrow(g);
    if (k == 0) { narrow = 0; break; }
    narrow = std::max(narrow, k);
  }
  if (narrow == 0) {
    // EBEM_GEMM_LOG: per-launch shape summary of the tiled merge GEMMs
    static const bool log = std::getenv("EBEM_GEMM_LOG") != nullptr;
    if (log) {
      long long tiles = 0;
      double mnk = 0, mn = 0;
      int mmax = 0, nmax = 0, kmax = 0, kmin = 1 << 30;
      for (const GemmTask& g : t) {
        if (g.k <= 0) continue;
        tiles += gemm_blocks(g, 0);
        mnk += double(g.m) * g.n * g.k;
        mn += double(g.m) * g.n;
        mmax = std::max(mmax, g.m); nmax = std::max(nmax, g.n);
        kmax = std::max(kmax, g.k); kmin = std::min(kmin, g.k);
      }
      std::fprintf(stderr,
                   "gemm launch: tasks %zu tiles %lld mean m*n %.0f "
                   "mean k %.1f k [%d, %d] max m %d max n %d flops %.3g\n",
                   t.size(), tiles, mn / t.size(), mnk / mn, kmin, kmax, mmax, nmax,
                   8 * mnk);
    }
  }
  g_gemm_narrow = narrow;
  run_blocked(P, t, [narrow](const GemmTask& g) { return g.k > 0 ? gemm_blocks(g, narrow) : 0; },
              launch_gemm_cur, KP_GEMM,
              [](const GemmTask& g) { return 8.0 * g.m * g.n * double(g.k); });
}
namespace {
void launch_getrs_staged(const LuSolveTask* t, const int* boff, int nt, int nb,
                         cudaStream_t st) {
  launch_getrs(t, boff, nt, nb, st, g_getrs_smem, g_getrs_maxn, g_getrs_cpw);
}
}  // namespace

void run_getrs(Problem& P, const std::vector<LuSolveTask>& t) {
  int smem = 0, maxn = 0, maxr = 0;
  for (const LuSolveTask& x : t) maxn = std::max(maxn, x.n), maxr = std::max(maxr, x.nrhs);
  const int cpw = getrs_cpw(maxr, maxn);
  g_getrs_cpw = cpw;
  for (const LuSolveTask& x : t)
    if (maxn <= 256 || x.n > 0) smem = std::max(smem, getrs_smem_bytes(x.n));
  g_getrs_smem = smem;
  g_getrs_maxn = maxn;
  run_blocked(P, t, [maxn, cpw](const LuSolveTask& s) { return s.n > 0 ? getrs_blocks(s.nrhs, maxn, cpw) : 0; },
              launch_getrs_staged, KP_GETRS,
              [](const LuSolveTask& s) { return 8.0 * s.n * double(s.n) * s.nrhs; });
}
void run_getrf(Problem& P, std::vector<LuTask> t) {
  if (t.empty()) return;
  size_t smem = 0, ws = 0;
  for (size_t i = 0; i < t.size(); ++i) {
    const size_t bytes = size_t(t[i].n) * t[i].n * 16;
    t[i].in_smem = bytes <= size_t(kSmemCap);
    t[i].ws_off = (long long)ws;
    if (t[i].in_smem) smem = std::max(smem, bytes);
    else ws += size_t(t[i].n) * t[i].n;
  }
  P.gws.ensure(ws + 1);
  // shared-memory LUs: one CTA each; larger ones: blocked, in place
  std::vector<LuTask> small, big;
  int big_n = 0;
  for (const LuTask& x : t) {
    if (x.in_smem) small.push_back(x);
    else {
      big.push_back(x);
      big_n = std::max(big_n, x.n);
    }
  }
  Pack pk;
  const size_t o = pk.add(small);
  const size_t ob = pk.add(big);
  char* tb = P.staging.put(pk, P.stream());
  double fl = 0.0, by = 0.0;
  for (const LuTask& x : t) {
    fl += 8.0 / 3.0 * double(x.n) * x.n * x.n;
    by += 32.0 * double(x.n) * x.n;  // the block read and the factors written
  }
  g_prof.begin(P.stream());
  launch_getrf(Pack::at<LuTask>(tb, o), int(small.size()), smem, P.gws.get(), P.stream());
  launch_lu_blocked(Pack::at<LuTask>(tb, ob), int(big.size()), big_n, P.stream());
  bool any_perm = false;
  for (const LuTask& x : t) any_perm = any_perm || x.perm != nullptr;
  if (any_perm) {  // the interchanges composed for the few-column solves
    launch_pivots_to_perm(Pack::at<LuTask>(tb, o), int(small.size()), P.stream());
    launch_pivots_to_perm(Pack::at<LuTask>(tb, ob), int(big.size()), P.stream());
  }
  g_prof.end(KP_GETRF, P.stream(), fl, by);
  P.staging.fence(P.stream());
  CK(cudaGetLastError());
}

namespace {
CopyTask copy_task(const double* src, int src_ld, double* dst, int dst_ld,
                   int rows, int cols) {
  CopyTask c{};
  c.src = src;
  c.dst = dst;
  c.rows = rows;
  c.cols = cols;
  c.src_ld = src_ld;
  c.dst_ld = dst_ld;
  return c;
}
GemmTask gemm_task(const double* a, int lda, const double* b, int ldb, double* c,
                   int ldc, int m, int n, int k, double beta) {
  GemmTask g{};
  g.a = a;
  g.b = b;
  g.c = c;
  g.m = m;
  g.n = n;
  g.k = k;
  g.lda = lda;
  g.ldb = ldb;
  g.ldc = ldc;
  g.alpha_re = 1.0;
  g.beta_re = beta;
  return g;
}
void singular_error(int info, int n) {
  if (std::getenv("EBEM_DEBUG_NOTHROW")) {
    std::fprintf(stderr, "[ebem] singular: pivot %d of %d\n", info - 1, n);
    return;
  }
  throw Error(EBEM_RUNTIME_ERROR,
              "LuFactor: matrix is singular, zero pivot at index " +
                  std::to_string(info - 1) + " of " + std::to_string(n));
}
}  // namespace

// -------------------------------------------------------------------- Fds
Fds::Fds(Problem& p, int depth, const ebem_fds_config& cfg,
         const HostSource* hs)
    : P_(p), depth_(depth), cfg_(cfg), hs_(hs) {
  const int n = P_.n();
  if (depth < 0) throw Error(EBEM_INVALID_ARGUMENT, "ClusterTree: negative depth");
  if (depth >= EBEM_MAX_LEVELS - 1)
    throw Error(EBEM_INVALID_ARGUMENT, "ClusterTree: depth too large");
  const int leaves = 1 << depth;
  if (n <= 0 || n % leaves != 0)
    throw Error(EBEM_INVALID_ARGUMENT,
                "ClusterTree: node count must be divisible by 2^depth (got " +
                    std::to_string(n) + " nodes, depth " + std::to_string(depth) + ")");
  if (cfg_.ell0 < 0 || cfg_.ell0 >= depth)
    throw Error(EBEM_INVALID_ARGUMENT,
                "FdsSolver: dense level must lie strictly above the leaves (got " +
                    std::to_string(cfg_.ell0) + " with depth " + std::to_string(depth) + ")");
  if (!(cfg_.epsilon > 0.0))
    throw Error(EBEM_INVALID_ARGUMENT, "Cpqr: truncation epsilon must be positive");
  build();
}

int* Fds::lu_info(int n) {
  info_n_.push_back(n);
  if (info_n_.size() > info_.size())
    throw Error(EBEM_LOGIC_ERROR, "FdsSolver: LU info slots exhausted");
  return info_.get() + (info_n_.size() - 1);
}

void Fds::reduced_diagonal(FillPlan& plan, std::vector<CopyTask>& copies,
                           int cell, double* dest, int ld, int off, MapPart* mp) {
  // proj/src/fds.cpp:33-54
  const Cell& c1 = cells_[2 * cell + 1];
  const Cell& c2 = cells_[2 * cell + 2];
  const int k1 = c1.k, k2 = c2.k, np = k1 + k2;
  for (int p = 0; p < 2; ++p)
    for (int q = 0; q < 2; ++q) {
      if (k1 > 0)
        copies.push_back(copy_task(c1.atilde + 2 * (size_t(q) * k1 * 2 * k1 + size_t(p) * k1),
                                   2 * k1,
                                   dest + 2 * (size_t(off + q * np) * ld + off + p * np),
                                   ld, k1, k1));
      if (k2 > 0)
        copies.push_back(copy_task(c2.atilde + 2 * (size_t(q) * k2 * 2 * k2 + size_t(p) * k2),
                                   2 * k2,
                                   dest + 2 * (size_t(off + q * np + k1) * ld + off + p * np + k1),
                                   ld, k2, k2));
    }
  double* base = dest + 2 * (size_t(off) * ld + off);
  const int drow12[2] = {0, np}, dcol12[2] = {k1, np + k1};
  const int drow21[2] = {k1, np + k1}, dcol21[2] = {0, np};
  if (mp) {
    // the children are consecutive cells of the level below (the previous
    // chained bases call): entries they already hold are copied
    int lv = 0;
    while (last(lv) < cell) ++lv;
    const int i1 = 2 * cell + 1 - first(lv + 1);
    P_.plan_sibling_block(plan, *mp, i1, i1 + 1, c1.srow, c2.scol, base, ld, drow12, dcol12);
    P_.plan_sibling_block(plan, *mp, i1 + 1, i1, c2.srow, c1.scol, base, ld, drow21, dcol21);
    return;
  }
  plan.add_true_block(c1.srow, c2.scol, base, ld, drow12, dcol12, 0);
  plan.add_true_block(c2.srow, c1.scol, base, ld, drow21, dcol21, 0);
}

void Fds::build() {
  const double t_start = now();
  cudaEvent_t ev0, ev1;
  CK(cudaEventCreate(&ev0));
  CK(cudaEventCreate(&ev1));
  CK(cudaEventRecord(ev0, P_.stream()));
  tl_begin(P_.stream());
  const int n = P_.n();
  const int ncells = (2 << depth_) - 1;
  cells_.assign(ncells, Cell{});
  store_.resize(depth_ + 1);
  stats_ = ebem_fds_stats{};
  stats_.depth = depth_;
  const int leaf = n >> depth_;
  info_.alloc(2 * size_t(ncells) + 2);
  CK(cudaMemsetAsync(info_.get(), 0, 4 * (2 * size_t(ncells) + 2), P_.stream()));
  info_n_.clear();
  for (int l = 0; l <= depth_; ++l)
    for (int c = first(l); c <= last(l); ++c) {
      cells_[c].begin = (c - first(l)) * (n >> l);
      cells_[c].end = cells_[c].begin + (n >> l);
    }
  for (int c = first(depth_); c <= last(depth_); ++c) {
    Cell& C = cells_[c];
    std::vector<int> r(leaf);
    for (int i = 0; i < leaf; ++i) r[i] = C.begin + i;
    C.jrow = {r, r};
    C.jcol = {r, r};
    C.nloc = leaf;
  }
  double basis_seconds = 0.0;
  P_.reset_chain();
  const int m = P_.proxy_cfg().m_prime;
  (void)m;
  for (int level = depth_; level > cfg_.ell0; --level) {
    const int f = first(level), L = last(level);
    const int nlev = L - f + 1;
    Store& S = store_[level];
    // ---- diagonal blocks (leaf: exact; above: reduced from the children's
    // skeletons and Atilde) into the LU arena, and their LU.  They depend on
    // level+1 only, so they are enqueued before this level's bases: the GPU
    // fills and factors them while the host plans the interaction fill.
    size_t lu_total = 0, piv_total = 0;
    std::vector<size_t> lu_off(nlev), piv_off(nlev);
    for (int i = 0; i < nlev; ++i) {
      const Cell& C = cells_[f + i];
      lu_off[i] = lu_total;
      lu_total += size_t(2 * C.nloc) * (2 * C.nloc);
      piv_off[i] = piv_total;
      piv_total += 2 * C.nloc;
    }
    S.lu.alloc(2 * lu_total + 2);
    S.ipiv.alloc(2 * piv_total + 2);  // interchanges, then the composed permutations
    for (int i = 0; i < nlev; ++i) {
      Cell& C = cells_[f + i];
      C.lu = S.lu.get() + 2 * lu_off[i];
      C.ipiv = S.ipiv.get() + piv_off[i];
      C.perm = 2 * C.nloc <= kPermMaxN ? S.ipiv.get() + piv_total + 1 + piv_off[i] : nullptr;
    }
    // A host BlockSource sees the reference's callback order (cell_basis of
    // a cell before its diagonal block, fds.cpp:77-89), so for it this
    // step runs after the bases.
    auto diagonal_and_lu = [&]() {
    {
      PhaseTimer tp("fill_diagonal", P_.stream());
      FillPlan plan(n, P_.proxy_cfg().m_prime, P_.proxy_cfg().n_gauss);
      std::vector<CopyTask> copies;
      std::vector<MapPart> mparts;
      for (int i = 0; hs_ && i < nlev; ++i) {  // host source: assemble on host
        Cell& C = cells_[f + i];
        const int d = 2 * C.nloc;
        std::vector<double> h;
        if (level == depth_) {
          h = host_block(C.jrow, C.jcol);
        } else {
          h.assign(2 * size_t(d) * d, 0.0);
          host_reduced_diagonal(f + i, h.data(), d);
        }
        if (d) copy_sync(C.lu, h.data(), 16 * size_t(d) * d);
      }
      if (!hs_) {
        // planned in contiguous chunks on the planning threads, appended in
        // cell order (same jobs and order as a serial pass)
        const int nchunk = std::min(nlev, 8 * planning_threads());
        std::vector<FillPlan> parts(nchunk, FillPlan(n, P_.proxy_cfg().m_prime,
                                                     P_.proxy_cfg().n_gauss));
        std::vector<std::vector<CopyTask>> pcopies(nchunk);
        mparts.assign(nchunk, MapPart{});
        // a batch of chunks (one per planning thread) at a time, each wave
        // executed as soon as its chunks are planned
        const int batch = std::max(1, planning_threads());
        int k0 = 0;
        long long acc = 0;
        for (int kb = 0; kb < nchunk; kb += batch) {
          const int ke = std::min(nchunk, kb + batch);
          parallel_for(ke - kb, [&](int kk) {
            const int k = kb + kk;
            const int i0 = int(size_t(nlev) * k / nchunk), i1 = int(size_t(nlev) * (k + 1) / nchunk);
            for (int i = i0; i < i1; ++i) {
              Cell& C = cells_[f + i];
              const int d = 2 * C.nloc;
              if (level == depth_) {
                parts[k].add_sym_diag(C.jrow[0], C.lu, d);  // leaf: jrow == jcol, ascending
              } else {
                reduced_diagonal(parts[k], pcopies[k], f + i, C.lu, d, 0, &mparts[k]);
              }
            }
          });
          for (int k = kb; k < ke; ++k) {
            copies.insert(copies.end(), pcopies[k].begin(), pcopies[k].end());
            acc += parts[k].bundles();
            const bool first_early = k0 == 0 && k == ke - 1 && acc >= kFirstWaveBundles;
            if (acc > kMaxBundlesPerWave || k == nchunk - 1 || first_early) {
              plan.append_many(parts, k0, k + 1);
              for (int q = k0; q <= k; ++q)
                parts[q] = FillPlan(n, P_.proxy_cfg().m_prime, P_.proxy_cfg().n_gauss);
              tl_mark("  diag wave planned");
              P_.execute(plan);
              k0 = k + 1;
              acc = 0;
            }
          }
        }
      }
      P_.execute(plan);
      run_copies(P_, copies);
      P_.run_map_copies(mparts);
      // element-length guard: read at the bases' synchronisation below
    }
    {
      PhaseTimer tp("merge_getrf", P_.stream());
      std::vector<LuTask> lt;
      for (int i = 0; i < nlev; ++i) {
        Cell& C = cells_[f + i];
        LuTask t{};
        t.a = C.lu;
        t.ipiv = C.ipiv;
        t.perm = C.perm;
        t.n = 2 * C.nloc;
        t.ld = 2 * C.nloc;
        lt.push_back(t);
      }
      for (LuTask& t : lt) t.info = lu_info(t.n);
      run_getrf(P_, lt);
    }
    };
    tl_mark("L" + std::to_string(level) + " start");
    if (!hs_) diagonal_and_lu();
    tl_mark("L" + std::to_string(level) + " diag+lu enq");
    // ---- bases of every cell of the level
    std::vector<BasisReq> req(nlev);
    for (int c = f; c <= L; ++c)
      req[c - f] = BasisReq{&cells_[c].jrow, &cells_[c].jcol, cells_[c].begin, cells_[c].end};
    if (level < depth_)  // children 2c+1, 2c+2: consecutive cells of the level below
      for (int i = 0; i < nlev; ++i) {
        req[i].child[0] = 2 * i;
        req[i].child[1] = 2 * i + 1;
      }
    std::vector<BasisRes> br;
    DBuf<double>& ubuf = ubuf_;
    const double tb = now();
    if (hs_) host_bases(level, br, S.v, ubuf);
    else P_.bases(req, cfg_.epsilon, br, S.v, ubuf, nullptr, true, true);
    PhaseTimer t_after("level_after_bases", nullptr);
    tl_mark("L" + std::to_string(level) + " bases done");
    basis_seconds += now() - tb;
    if (hs_) diagonal_and_lu();
    size_t au_total = 0, at_total = 0;
    std::vector<size_t> au_off(nlev), at_off(nlev);
    for (int i = 0; i < nlev; ++i) {
      Cell& C = cells_[f + i];
      C.k = br[i].k;
      au_off[i] = au_total;
      au_total += size_t(2 * C.nloc) * (2 * C.k);
      at_off[i] = at_total;
      at_total += size_t(2 * C.k) * (2 * C.k);
      stats_.max_rank[level] = std::max(stats_.max_rank[level], C.k);
      stats_.saturated = stats_.saturated || br[i].saturated;
    }
    S.ainv_u.alloc(2 * au_total + 2);
    S.atilde.alloc(2 * at_total + 2);
    for (int i = 0; i < nlev; ++i) {
      Cell& C = cells_[f + i];
      C.ainv_u = S.ainv_u.get() + 2 * au_off[i];
      C.atilde = S.atilde.get() + 2 * at_off[i];
      C.v = S.v.get() + 2 * br[i].v_off;
    }
    tl_mark("  merge alloc");
    // ---- A^-1 U with U = blockdiag(u0, u1)
    {
      PhaseTimer tp("merge_ainv_u", P_.stream());
      std::vector<CopyTask> ct;
      std::vector<LuSolveTask> st;
      for (int i = 0; i < nlev; ++i) {
        Cell& C = cells_[f + i];
        const int nl = C.nloc, k = C.k;
        if (k == 0) continue;
        const int d = 2 * nl;
        // off-diagonal zero blocks (tasks of one launch must not overlap)
        ct.push_back(copy_task(nullptr, 0, C.ainv_u + 2 * size_t(nl), d, nl, k));
        ct.push_back(copy_task(nullptr, 0, C.ainv_u + 2 * size_t(k) * d, d, nl, k));
        const double* u = ubuf.get() + 2 * br[i].u_off;
        ct.push_back(copy_task(u, nl, C.ainv_u, d, nl, k));
        ct.push_back(copy_task(u + 2 * size_t(nl) * k, nl,
                               C.ainv_u + 2 * (size_t(k) * d + nl), d, nl, k));
        st.push_back(LuSolveTask{C.lu, C.ipiv, C.ainv_u, d, d, 2 * k, d});
      }
      run_copies(P_, ct);
      run_getrs(P_, st);
    }
    tl_mark("  ainv_u enq");
    // ---- W = [v0 A^-1U_top ; v1 A^-1U_bottom], atilde = W^-1
    {
      PhaseTimer tp("merge_atilde", P_.stream());
      DBuf<double>& wbuf = wbuf_;
      DBuf<int>& wpiv = wpiv_;
      wbuf.ensure(2 * at_total + 2);
      wpiv.ensure(at_total + 1);
      std::vector<GemmTask> gt;
      std::vector<LuTask> lt;
      std::vector<CopyTask> ct;
      std::vector<LuSolveTask> st;
      size_t poff = 0;
      for (int i = 0; i < nlev; ++i) {
        Cell& C = cells_[f + i];
        const int nl = C.nloc, k = C.k;
        if (k == 0) continue;
        const int d = 2 * nl, kk = 2 * k;
        double* w = wbuf.get() + 2 * at_off[i];
        gt.push_back(gemm_task(C.v, k, C.ainv_u, d, w, kk, k, kk, nl, 0.0));
        gt.push_back(gemm_task(C.v + 2 * size_t(k) * nl, k, C.ainv_u + 2 * size_t(nl), d,
                               w + 2 * size_t(k), kk, k, kk, nl, 0.0));
        LuTask t{};
        t.a = w;
        t.ipiv = wpiv.get() + poff;
        t.n = kk;
        t.ld = kk;
        lt.push_back(t);
        CopyTask id = copy_task(nullptr, 0, C.atilde, kk, kk, kk);
        id.transpose = 2;  // identity
        ct.push_back(id);
        st.push_back(LuSolveTask{w, wpiv.get() + poff, C.atilde, kk, kk, kk, kk});
        poff += kk;
      }
      run_gemms(P_, gt);
      for (LuTask& t : lt) t.info = lu_info(t.n);
      run_getrf(P_, lt);
      run_copies(P_, ct);
      run_getrs(P_, st);
    }
    tl_mark("  merges enq");
    // ---- skeleton lists (deferred: the merges above needed only the ranks)
    if (!hs_) P_.finish_bases();
    tl_mark("  lists");
    // ---- parent sequences: concatenated child skeletons per component
    {
      const int pf = first(level - 1), np = last(level - 1) - pf + 1;
      const int nch = std::min(np, 4 * planning_threads());
      parallel_for(nch, [&](int kq) {
        const int p0 = int(size_t(np) * kq / nch), p1 = int(size_t(np) * (kq + 1) / nch);
        for (int c = pf + p0; c < pf + p1; ++c) {
          Cell& Pc = cells_[c];
          Cell& c1 = cells_[2 * c + 1];
          Cell& c2 = cells_[2 * c + 2];
          c1.srow = std::move(br[2 * c + 1 - f].srow);
          c1.scol = std::move(br[2 * c + 1 - f].scol);
          c2.srow = std::move(br[2 * c + 2 - f].srow);
          c2.scol = std::move(br[2 * c + 2 - f].scol);
          for (int comp = 0; comp < 2; ++comp) {
            Pc.jrow[comp] = c1.srow[comp];
            Pc.jrow[comp].insert(Pc.jrow[comp].end(), c2.srow[comp].begin(), c2.srow[comp].end());
            Pc.jcol[comp] = c1.scol[comp];
            Pc.jcol[comp].insert(Pc.jcol[comp].end(), c2.scol[comp].begin(), c2.scol[comp].end());
          }
          Pc.nloc = c1.k + c2.k;
        }
      });
    }
  }
  tl_mark("upward enq");
  tl_dump();
  CK(cudaStreamSynchronize(P_.stream()));
  stats_.upward_seconds = now() - t_start;
  stats_.basis_cpu_seconds = basis_seconds;

  // ---- dense system over the cells of level ell0 (proj/src/fds.cpp:131-152)
  PhaseTimer tp_top("top", P_.stream());
  const double t_top = now();
  const int tf = first(cfg_.ell0), tl = last(cfg_.ell0);
  top_off_.assign(tl - tf + 2, 0);
  for (int i = 0; i <= tl - tf; ++i) top_off_[i + 1] = top_off_[i] + 2 * cells_[tf + i].nloc;
  top_dim_ = top_off_.back();
  stats_.top_dim = top_dim_;
  top_lu_.alloc(2 * size_t(top_dim_) * top_dim_ + 2);
  top_ipiv_.alloc(2 * size_t(top_dim_) + 2);  // interchanges, then the composed permutation
  if (hs_ && top_dim_ > 0) {  // host source: the dense top system on the host
    std::vector<double> h(2 * size_t(top_dim_) * top_dim_, 0.0);
    for (int i = 0; i <= tl - tf; ++i) {
      const Cell& ci = cells_[tf + i];
      for (int j = 0; j <= tl - tf; ++j) {
        const Cell& cj = cells_[tf + j];
        const int ri = 2 * ci.nloc, cjn = 2 * cj.nloc;
        if (!ri || !cjn) continue;
        std::vector<double> blk;
        if (i == j) {
          blk.assign(2 * size_t(ri) * ri, 0.0);
          host_reduced_diagonal(tf + i, blk.data(), ri);
        } else {
          blk = host_block(ci.jrow, cj.jcol);
        }
        for (int c = 0; c < cjn; ++c)
          std::memcpy(h.data() + 2 * (size_t(top_off_[j] + c) * top_dim_ + top_off_[i]),
                      blk.data() + 2 * size_t(c) * ri, 16 * size_t(ri));
      }
    }
    copy_sync(top_lu_.get(), h.data(), h.size() * 8);
  }
  {
    FillPlan plan(n, P_.proxy_cfg().m_prime, P_.proxy_cfg().n_gauss);
    std::vector<CopyTask> copies;
    std::vector<MapPart> mparts(1);
    for (int i = 0; !hs_ && i <= tl - tf; ++i) {
      const Cell& ci = cells_[tf + i];
      for (int j = 0; j <= tl - tf; ++j) {
        const Cell& cj = cells_[tf + j];
        if (i == j) {
          reduced_diagonal(plan, copies, tf + i, top_lu_.get(), top_dim_, top_off_[i],
                           &mparts[0]);
        } else {
          const int drow[2] = {top_off_[i], top_off_[i] + ci.nloc};
          const int dcol[2] = {top_off_[j], top_off_[j] + cj.nloc};
          plan.add_true_block(ci.jrow, cj.jcol, top_lu_.get(), top_dim_, drow, dcol, 0);
        }
      }
    }
    P_.execute(plan);
    run_copies(P_, copies);
    P_.run_map_copies(mparts);
    P_.check_domain();
    if (top_dim_ > 0) {
      LuTask t{};
      t.a = top_lu_.get();
      t.ipiv = top_ipiv_.get();
      t.perm = top_dim_ <= kPermMaxN ? top_ipiv_.get() + top_dim_ + 1 : nullptr;
      t.n = top_dim_;
      t.ld = top_dim_;
      t.info = lu_info(top_dim_);
      run_getrf(P_, {t});
    }
  }
  CK(cudaStreamSynchronize(P_.stream()));
  stats_.top_factor_seconds = now() - t_top;
  CK(cudaEventRecord(ev1, P_.stream()));
  CK(cudaEventSynchronize(ev1));
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, ev0, ev1));
  stats_.factorize_device_seconds = 1e-3 * ms;
  host_phase_dump();
  // zero pivots, checked once (in factorization order) instead of a sync per LU
  std::vector<int> info(info_n_.size());
  if (!info.empty())
    copy_sync(info.data(), info_.get(), 4 * info.size());
  for (size_t i = 0; i < info.size(); ++i)
    if (info[i]) singular_error(info[i], info_n_[i]);
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
}

void Fds::debug_cell(int cell, int which, double* out) const {
  const Cell& C = cells_.at(cell);
  const size_t d = 2 * size_t(C.nloc), kk = 2 * size_t(C.k);
  const void* src = nullptr;
  size_t bytes = 0;
  switch (which) {
    case 0: src = C.lu; bytes = 16 * d * d; break;
    case 1: src = C.ipiv; bytes = 4 * d; break;
    case 2: src = C.ainv_u; bytes = 16 * d * kk; break;
    case 3: src = C.v; bytes = 16 * kk * C.nloc; break;
    case 4: src = C.atilde; bytes = 16 * kk * kk; break;
    default: throw Error(EBEM_INVALID_ARGUMENT, "debug_cell: bad selector");
  }
  if (src && bytes) copy_sync(out, src, bytes);
}

std::vector<double> Fds::host_block(const Lists& rows, const Lists& cols) {
  const int nr = int(rows[0].size() + rows[1].size());
  const int nc = int(cols[0].size() + cols[1].size());
  std::vector<double> out(2 * size_t(nr) * nc, 0.0);
  if (!nr || !nc) return out;
  const int rc = hs_->block(hs_->user, rows[0].data(), int(rows[0].size()),
                            rows[1].data(), int(rows[1].size()), cols[0].data(),
                            int(cols[0].size()), cols[1].data(), int(cols[1].size()),
                            out.data());
  if (rc) throw Error(rc, "BlockSource::block callback failed");
  return out;
}

// FdsSolver::reduced_diagonal (proj/src/fds.cpp:33-54) on the host.
void Fds::host_reduced_diagonal(int cell, double* out, int ld) {
  const Cell& c1 = cells_[2 * cell + 1];
  const Cell& c2 = cells_[2 * cell + 2];
  const int k1 = c1.k, k2 = c2.k, np = k1 + k2;
  std::vector<double> a1(2 * size_t(4) * k1 * k1), a2(2 * size_t(4) * k2 * k2);
  if (k1) copy_sync(a1.data(), c1.atilde, a1.size() * 8);
  if (k2) copy_sync(a2.data(), c2.atilde, a2.size() * 8);
  const std::vector<double> x12 = host_block(c1.srow, c2.scol);
  const std::vector<double> x21 = host_block(c2.srow, c1.scol);
  auto put = [&](int r, int c, const double* src, int sld, int sr, int sc) {
    out[2 * (size_t(c) * ld + r)] = src[2 * (size_t(sc) * sld + sr)];
    out[2 * (size_t(c) * ld + r) + 1] = src[2 * (size_t(sc) * sld + sr) + 1];
  };
  for (int p = 0; p < 2; ++p)
    for (int q = 0; q < 2; ++q) {
      for (int jj = 0; jj < k1; ++jj)
        for (int ii = 0; ii < k1; ++ii)
          put(p * np + ii, q * np + jj, a1.data(), 2 * k1, p * k1 + ii, q * k1 + jj);
      for (int jj = 0; jj < k2; ++jj)
        for (int ii = 0; ii < k2; ++ii)
          put(p * np + k1 + ii, q * np + k1 + jj, a2.data(), 2 * k2, p * k2 + ii, q * k2 + jj);
      for (int jj = 0; jj < k2; ++jj)
        for (int ii = 0; ii < k1; ++ii)
          put(p * np + ii, q * np + k1 + jj, x12.data(), 2 * k1, p * k1 + ii, q * k2 + jj);
      for (int jj = 0; jj < k1; ++jj)
        for (int ii = 0; ii < k2; ++ii)
          put(p * np + k1 + ii, q * np + jj, x21.data(), 2 * k2, p * k2 + ii, q * k1 + jj);
    }
}

void Fds::host_bases(int level, std::vector<BasisRes>& br, DBuf<double>& vbuf,
                     DBuf<double>& ubuf) {
  const int f = first(level), L = last(level), nlev = L - f + 1;
  br.assign(nlev, BasisRes{});
  std::vector<double> hv, hu;
  for (int i = 0; i < nlev; ++i) {
    Cell& C = cells_[f + i];
    const int nr0 = int(C.jrow[0].size()), nr1 = int(C.jrow[1].size());
    const int nc0 = int(C.jcol[0].size()), nc1 = int(C.jcol[1].size());
    if (!nr0 || !nr1 || !nc0 || !nc1) throw Error(EBEM_INVALID_ARGUMENT, "Cpqr: empty matrix");
    const int kmax = std::min(std::min(nr0, nr1), std::min(nc0, nc1));
    std::vector<int> skel(4 * size_t(kmax) + 4);
    std::vector<double> u0(2 * size_t(nr0) * kmax + 2), u1(2 * size_t(nr1) * kmax + 2);
    std::vector<double> v0(2 * size_t(nc0) * kmax + 2), v1(2 * size_t(nc1) * kmax + 2);
    int k = 0, sat = 0;
    const int rc = hs_->basis(hs_->user, C.jrow[0].data(), nr0, C.jrow[1].data(), nr1,
                              C.jcol[0].data(), nc0, C.jcol[1].data(), nc1, C.begin,
                              C.end, cfg_.epsilon, &k, &sat, skel.data(), u0.data(),
                              u1.data(), v0.data(), v1.data());
    if (rc) throw Error(rc, "BlockSource::cell_basis callback failed");
    if (k < 0 || k > kmax) throw Error(EBEM_LOGIC_ERROR, "BlockSource::cell_basis: rank out of range");
    BasisRes& r = br[i];
    r.k = k;
    r.saturated = sat != 0;
    r.srow[0].assign(skel.begin(), skel.begin() + k);
    r.srow[1].assign(skel.begin() + k, skel.begin() + 2 * k);
    r.scol[0].assign(skel.begin() + 2 * k, skel.begin() + 3 * k);
    r.scol[1].assign(skel.begin() + 3 * k, skel.begin() + 4 * k);
    r.v_off = hv.size() / 2;
    hv.insert(hv.end(), v0.begin(), v0.begin() + 2 * size_t(k) * nc0);
    hv.insert(hv.end(), v1.begin(), v1.begin() + 2 * size_t(k) * nc1);
    r.u_off = hu.size() / 2;
    hu.insert(hu.end(), u0.begin(), u0.begin() + 2 * size_t(k) * nr0);
    hu.insert(hu.end(), u1.begin(), u1.begin() + 2 * size_t(k) * nr1);
  }
  vbuf.ensure(hv.size() + 2);
  ubuf.ensure(hu.size() + 2);
  if (!hv.empty()) copy_sync(vbuf.get(), hv.data(), hv.size() * 8);
  if (!hu.empty()) copy_sync(ubuf.get(), hu.data(), hu.size() * 8);
}

int Fds::rank_of(int cell) const {
  if (cell < 0 || cell >= int(cells_.size())) return -1;
  return cells_[cell].k;
}

void Fds::cell_info(int cell, int* sizes, int* skel) const {
  if (cell < 0 || cell >= int(cells_.size()))
    throw Error(EBEM_INVALID_ARGUMENT, "FdsSolver: cell out of range");
  const Cell& C = cells_[cell];
  sizes[0] = int(C.jrow[0].size());
  sizes[1] = int(C.jrow[1].size());
  sizes[2] = int(C.jcol[0].size());
  sizes[3] = int(C.jcol[1].size());
  sizes[4] = C.k;
  if (skel) {
    const int k = C.k;
    for (int i = 0; i < k && i < int(C.srow[0].size()); ++i) {
      skel[i] = C.srow[0][i];
      skel[k + i] = C.srow[1][i];
      skel[2 * k + i] = C.scol[0][i];
      skel[3 * k + i] = C.scol[1][i];
    }
  }
}

void Fds::record_solve(int m) {
  const double tr0 = now();
  plan_.reset(new SolvePlan());
  SolvePlan& S = *plan_;
  S.m = m;
  const int n = P_.n();
  const int ncells = int(cells_.size());
  const int leaf = n >> depth_;
  // per-cell row offsets of the f/x (2 nloc) and ftilde/t (2k) blocks
  std::vector<size_t> fo(ncells, 0), ko(ncells, 0);
  size_t ftot = 0, ktot = 0;
  for (int c = 0; c < ncells; ++c) {
    fo[c] = ftot;
    ftot += 2 * size_t(cells_[c].nloc);
    ko[c] = ktot;
    ktot += 2 * size_t(cells_[c].k);
  }
  ws_f_.ensure(2 * ftot * m + 2);
  ws_ft_.ensure(2 * ktot * m + 2);
  ws_t_.ensure(2 * ktot * m + 2);
  ws_x_.ensure(2 * size_t(top_dim_) * m + 2);
  S.rhs.alloc(4 * size_t(n) * m);
  S.x.alloc(4 * size_t(n) * m);
  const double* rhs = S.rhs.get();
  double* x = S.x.get();
  auto F = [&](int c) { return ws_f_.get() + 2 * fo[c] * m; };
  auto FT = [&](int c) { return ws_ft_.get() + 2 * ko[c] * m; };
  auto TT = [&](int c) { return ws_t_.get() + 2 * ko[c] * m; };
  const double tr_alloc = now();
  P_.recorder = &S.rec;
  S.rec.begin();
  S.rec.mark();
  // task lists recycled across recordings (fresh vectors of this size cost
  // thousands of page faults; API calls are serialised)
  static std::vector<CopyTask> s_ct, s_back;
  static std::vector<LuSolveTask> s_st;
  static std::vector<GemmTask> s_g1, s_g2;
  // leaves: f = [rhs[a:a+s]; rhs[N+a:N+a+s]]
  {
    std::vector<CopyTask>& ct = s_ct;
    ct.clear();
    for (int c = first(depth_); c <= last(depth_); ++c) {
      const int a = cells_[c].begin;
      ct.push_back(copy_task(rhs + 2 * size_t(a), 2 * n, F(c), 2 * leaf, leaf, m));
      ct.push_back(copy_task(rhs + 2 * size_t(n + a), 2 * n, F(c) + 2 * size_t(leaf), 2 * leaf, leaf, m));
    }
    run_copies(P_, ct);
  }
  // The upper levels are few-CTA, latency-bound launches: warm the L2 with
  // their factors (and the task arrays) right before the first of them.
  // lp = the lowest level such that the factors of levels ell0+1 .. lp and
  // the top LU fit half the L2 (EBEM_SOLVE_PREFETCH_MB, 0 = off).
  int lp = -1;
  std::vector<PrefetchTask> warm;
  {
    static const double cap_mb = [] {
      const char* e = std::getenv("EBEM_SOLVE_PREFETCH_MB");
      return e ? std::atof(e) : 64.0;
    }();
    auto bytes_of = [&](const Store& s) {
      return 8.0 * (s.lu.size() + s.ainv_u.size() + s.v.size() + s.atilde.size()) +
             4.0 * s.ipiv.size();
    };
    double acc = 8.0 * top_lu_.size();
    for (int l = cfg_.ell0 + 1; l <= depth_; ++l) {
      acc += bytes_of(store_[l]);
      if (acc > cap_mb * 1048576.0) break;
      lp = l;
    }
    if (lp > cfg_.ell0) {
      warm.push_back(PrefetchTask{top_lu_.get(), 8ull * top_lu_.size()});
      warm.push_back(PrefetchTask{top_ipiv_.get(), 4ull * top_ipiv_.size()});
      for (int l = cfg_.ell0 + 1; l <= lp; ++l) {
        const Store& s = store_[l];
        warm.push_back(PrefetchTask{s.lu.get(), 8ull * s.lu.size()});
        warm.push_back(PrefetchTask{s.ipiv.get(), 4ull * s.ipiv.size()});
        warm.push_back(PrefetchTask{s.ainv_u.get(), 8ull * s.ainv_u.size()});
        warm.push_back(PrefetchTask{s.v.get(), 8ull * s.v.size()});
        warm.push_back(PrefetchTask{s.atilde.get(), 8ull * s.atilde.size()});
      }
    }
  }
  for (int level = depth_; level > cfg_.ell0; --level) {
    if (level == lp) S.rec.add_prefetch(warm);
    std::vector<LuSolveTask>& st = s_st;
    std::vector<GemmTask>&g1 = s_g1, &g2 = s_g2;
    st.clear();
    g1.clear();
    g2.clear();
    for (int c = first(level); c <= last(level); ++c) {
      const Cell& C = cells_[c];
      const int nl = C.nloc, d = 2 * nl, k = C.k, kk = 2 * k;
      st.push_back(LuSolveTask{C.lu, C.ipiv, F(c), d, d, m, d, C.perm});  // ainvf in place
      if (k == 0) continue;
      g1.push_back(gemm_task(C.v, k, F(c), d, TT(c), kk, k, m, nl, 0.0));
      g1.push_back(gemm_task(C.v + 2 * size_t(k) * nl, k, F(c) + 2 * size_t(nl), d,
                             TT(c) + 2 * size_t(k), kk, k, m, nl, 0.0));
      g2.push_back(gemm_task(C.atilde, kk, TT(c), kk, FT(c), kk, kk, m, kk, 0.0));
    }
    run_getrs(P_, st);
    run_gemms(P_, g1);
    run_gemms(P_, g2);
    // parent f = [ft1 top; ft2 top; ft1 bottom; ft2 bottom]
    std::vector<CopyTask>& ct = s_ct;
    ct.clear();
    for (int c = first(level - 1); c <= last(level - 1); ++c) {
      const int c1 = 2 * c + 1, c2 = 2 * c + 2;
      const int k1 = cells_[c1].k, k2 = cells_[c2].k, np = k1 + k2;
      const int ld = 2 * np;
      if (ld == 0) continue;
      if (k1) {
        ct.push_back(copy_task(FT(c1), 2 * k1, F(c), ld, k1, m));
        ct.push_back(copy_task(FT(c1) + 2 * size_t(k1), 2 * k1, F(c) + 2 * size_t(np), ld, k1, m));
      }
      if (k2) {
        ct.push_back(copy_task(FT(c2), 2 * k2, F(c) + 2 * size_t(k1), ld, k2, m));
        ct.push_back(copy_task(FT(c2) + 2 * size_t(k2), 2 * k2, F(c) + 2 * size_t(np + k1), ld, k2, m));
      }
    }
    run_copies(P_, ct);
  }
  S.rec.mark();
  // top: stack, solve, unstack (x of the top cells lives in their f blocks)
  {
    const int tf = first(cfg_.ell0), tl = last(cfg_.ell0);
    std::vector<CopyTask>&ct = s_ct, &back = s_back;
    ct.clear();
    back.clear();
    for (int i = 0; i <= tl - tf; ++i) {
      const int c = tf + i;
      const int d = 2 * cells_[c].nloc;
      if (d == 0) continue;
      ct.push_back(copy_task(F(c), d, ws_x_.get() + 2 * size_t(top_off_[i]), top_dim_, d, m));
      back.push_back(copy_task(ws_x_.get() + 2 * size_t(top_off_[i]), top_dim_, F(c), d, d, m));
    }
    run_copies(P_, ct);
    if (top_dim_ > 0)
      run_getrs(P_, {LuSolveTask{top_lu_.get(), top_ipiv_.get(), ws_x_.get(), top_dim_,
                                 top_dim_, m, top_dim_,
                                 top_dim_ <= kPermMaxN ? top_ipiv_.get() + top_dim_ + 1 : nullptr}});
    run_copies(P_, back);
  }
  S.rec.mark();
  // downward: x_child = ainvf + ainv_u (atilde y - ftilde)
  for (int level = cfg_.ell0; level < depth_; ++level) {
    std::vector<CopyTask>& ct = s_ct;
    std::vector<GemmTask>&g1 = s_g1, &g2 = s_g2;
    ct.clear();
    g1.clear();
    g2.clear();
    for (int c = first(level); c <= last(level); ++c) {
      const int c1 = 2 * c + 1, c2 = 2 * c + 2;
      const int k1 = cells_[c1].k, k2 = cells_[c2].k, np = k1 + k2;
      for (int side = 0; side < 2; ++side) {
        const int cc = side == 0 ? c1 : c2;
        const Cell& C = cells_[cc];
        const int k = C.k, kk = 2 * k, d = 2 * C.nloc;
        if (k == 0) continue;
        const int row0 = side == 0 ? 0 : k1;
        ct.push_back(copy_task(F(c) + 2 * size_t(row0), 2 * np, TT(cc), kk, k, m));
        ct.push_back(copy_task(F(c) + 2 * size_t(np + row0), 2 * np, TT(cc) + 2 * size_t(k), kk, k, m));
        GemmTask a = gemm_task(C.atilde, kk, TT(cc), kk, FT(cc), kk, kk, m, kk, -1.0);
        g1.push_back(a);
        g2.push_back(gemm_task(C.ainv_u, d, FT(cc), kk, F(cc), d, d, m, kk, 1.0));
      }
    }
    run_copies(P_, ct);
    run_gemms(P_, g1);
    run_gemms(P_, g2);
  }
  {
    std::vector<CopyTask>& ct = s_ct;
    ct.clear();
    for (int c = first(depth_); c <= last(depth_); ++c) {
      const int a = cells_[c].begin;
      ct.push_back(copy_task(F(c), 2 * leaf, x + 2 * size_t(a), 2 * n, leaf, m));
      ct.push_back(copy_task(F(c) + 2 * size_t(leaf), 2 * leaf, x + 2 * size_t(n + a), 2 * n, leaf, m));
    }
    run_copies(P_, ct);
  }
  S.rec.mark();
  P_.recorder = nullptr;
  const double tr1 = now();
  S.rec.finalize(P_.stream());
  const double tr2 = now();
  for (int q = 0; q < 4; ++q) CK(cudaEventCreate(&S.ev[q]));
  // one graph per phase (upward, top, downward); timing events go between
  for (int ph = 0; ph < 3; ++ph) {
    CK(cudaStreamBeginCapture(P_.stream(), cudaStreamCaptureModeThreadLocal));
    S.rec.replay(P_.stream(), ph);
    CK(cudaStreamEndCapture(P_.stream(), &S.graph[ph]));
    CK(cudaGraphInstantiate(&S.exec[ph], S.graph[ph], 0));
  }
  if (verbose_level())
    std::fprintf(stderr, "[ebem] record_solve(%d): workspaces %.1f ms, tasks %.1f ms, upload %.1f ms, graphs %.1f ms (%zu launches)\n",
                 m, 1e3 * (tr_alloc - tr0), 1e3 * (tr1 - tr_alloc), 1e3 * (tr2 - tr1), 1e3 * (now() - tr2), S.rec.n_launches());
}

Fds::~Fds() = default;  // SolvePlan releases its graphs

void Fds::solve_device(const double* rhs, int m, double* x,
                       ebem_fds_solve_timing* timing) {
  const int n = P_.n();
  if (!plan_ || plan_->m != m) record_solve(m);
  SolvePlan& S = *plan_;
  const size_t bytes = 32 * size_t(n) * m;
  CK(cudaMemcpyAsync(S.rhs.get(), rhs, bytes, cudaMemcpyDefault, P_.stream()));
  for (int ph = 0; ph < 3; ++ph) {
    CK(cudaEventRecord(S.ev[ph], P_.stream()));
    CK(cudaGraphLaunch(S.exec[ph], P_.stream()));
  }
  CK(cudaEventRecord(S.ev[3], P_.stream()));
  CK(cudaMemcpyAsync(x, S.x.get(), bytes, cudaMemcpyDefault, P_.stream()));
  CK(cudaStreamSynchronize(P_.stream()));
  float a = 0.f, b = 0.f, c = 0.f;
  CK(cudaEventElapsedTime(&a, S.ev[0], S.ev[1]));
  CK(cudaEventElapsedTime(&b, S.ev[1], S.ev[2]));
  CK(cudaEventElapsedTime(&c, S.ev[2], S.ev[3]));
  last_solve_device_seconds_ = 1e-3 * (a + b + c);
  g_launches += long(S.rec.n_launches());
  if (timing) {
    timing->upward_seconds = 1e-3 * a;
    timing->top_seconds = 1e-3 * b;
    timing->downward_seconds = 1e-3 * c;
    timing->device_seconds = last_solve_device_seconds_;
  }
}

}  // namespace ebem_gpu
