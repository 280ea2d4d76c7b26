// Native host runtime of the B200 solver path: device buffers, the per-level
// work planner, the batched basis / merge / sweep drivers.  The C ABI
// (capi.cpp) is a thin shell over the classes declared here.
#pragma once

#include <cuda_runtime.h>

#include <array>
#include <atomic>
#include <cstddef>
#include <cstring>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ebem_ctx.h"
#include "ebem_dense.h"
#include "ebem_gpu.h"
#include "ebem_jobs.h"

namespace ebem_gpu {

using Lists = std::array<std::vector<int>, 2>;

// ------------------------------------------------------------------ errors
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
void cuda_check(cudaError_t e, const char* what);
#define CK(x) ::ebem_gpu::cuda_check((x), #x)

extern std::atomic<long long> g_launches;

// ---------------------------------------------------------------- profiler
// Optional per-kernel device timing (CUDA events on the launching stream)
// and algorithmic work units (quadrature point evaluations for the fill
// kernels, bytes or flops for the rest); enabled by ebem_gpu_prof_enable.
enum KernelId {
  KP_PROXY = 0, KP_NEAR_1S, KP_NEAR_SING, KP_GATHER, KP_QR, KP_CPQR,
  KP_INTERP, KP_GETRF, KP_GETRS, KP_GEMM, KP_COPY, KP_RHS, KP_NEAR_SYM, KP_BUCKET, KP_REUSE, KP_COUNT
};
const char* kernel_name(int id);

class Profiler {
 public:
  bool on = false;
  void begin(cudaStream_t st);
  // bytes: algorithmic HBM bytes of the launch (operands read once, results
  // written once), for the HBM roofline of the ID / solve kernels
  void end(int id, cudaStream_t st, double units, double bytes = 0.0);
  // units = mult x (dev_bounds[1] - dev_bounds[0]), read back at collect()
  void end_counted(int id, cudaStream_t st, const int* dev_bounds, double mult);
  void collect();
  void reset();
  double ms[KP_COUNT] = {};
  long long count[KP_COUNT] = {};
  double units[KP_COUNT] = {};
  double bytes[KP_COUNT] = {};
  double gap_ms[KP_COUNT] = {};  // device idle right before each kernel kind

 private:
  struct Rec { int id; cudaEvent_t a, b; double units; int slot; double bytes; };
  int* counts_ = nullptr;  // pinned (first, last) pairs of end_counted
  int counts_used_ = 0, counts_cap_ = 0;
  std::vector<Rec> pending_;
  std::vector<cudaEvent_t> pool_;
  cudaEvent_t cur_ = nullptr;
  cudaEvent_t ev();
};
extern Profiler g_prof;



// Host-side phase timers (EBEM_VERBOSE=1 prints them after a factorization;
// EBEM_VERBOSE=2 also synchronises the stream at each scope end so device
// work is attributed to the phase that issued it).
int verbose_level();
void host_phase_add(const char* name, double seconds);
void host_phase_dump();
class PhaseTimer {
 public:
  PhaseTimer(const char* name, cudaStream_t st);
  ~PhaseTimer();

 private:
  const char* name_;
  cudaStream_t st_;
  double t0_;
};

// The process-wide stream every handle uses (created with the scratch pool).
cudaStream_t scratch_stream();
// cudaMemcpyAsync on that stream + synchronise.
void copy_sync(void* dst, const void* src, size_t bytes);

// ----------------------------------------------------------------- buffers
template <class T>
class DBuf {
 public:
  DBuf() = default;
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p_(o.p_), n_(o.n_) { o.p_ = nullptr; o.n_ = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) { release(); p_ = o.p_; n_ = o.n_; o.p_ = nullptr; o.n_ = 0; }
    return *this;
  }
  ~DBuf() { release(); }
  // Stream-ordered allocation from the device's default memory pool (kept
  // cached: release threshold = max), on the process-wide stream: no
  // implicit device synchronisation, no re-mapping of freed pages.
  void alloc(size_t n) {
    PhaseTimer t("cuda_malloc_free", nullptr);
    release();
    if (n == 0) return;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&p_), n * sizeof(T), scratch_stream()));
    n_ = n;
  }
  // grow-only
  void ensure(size_t n) {
    if (n <= n_) return;
    alloc(n + n / 4);
  }
  void release() {
    if (p_) cudaFreeAsync(p_, scratch_stream());
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// Grow-only pinned host buffer (device-to-host readbacks at full speed).
template <class T>
class PinnedBuf {
 public:
  PinnedBuf() = default;
  PinnedBuf(const PinnedBuf&) = delete;
  PinnedBuf& operator=(const PinnedBuf&) = delete;
  ~PinnedBuf() { if (p_) cudaFreeHost(p_); }
  T* ensure(size_t n) {
    if (n > n_) {
      if (p_) cudaFreeHost(p_);
      p_ = nullptr;
      n_ = 0;
      const size_t cap = n + n / 4 + 64;
      CK(cudaMallocHost(reinterpret_cast<void**>(&p_), cap * sizeof(T)));
      n_ = cap;
    }
    return p_;
  }

 private:
  T* p_ = nullptr;
  size_t n_ = 0;
};

// Packs host arrays into one device upload (16-byte aligned segments).
class Pack {
 public:
  template <class T>
  size_t add(const std::vector<T>& v) {
    return add_raw(v.data(), v.size() * sizeof(T));
  }
  size_t add_raw(const void* p, size_t bytes) {
    const size_t off = (buf_.size() + 15) & ~size_t(15);
    buf_.resize(off + bytes);
    if (bytes) std::memcpy(buf_.data() + off, p, bytes);
    return off;
  }
  void upload(DBuf<char>& dev, cudaStream_t st);
  template <class T>
  T* at(const DBuf<char>& dev, size_t off) const {
    return reinterpret_cast<T*>(dev.get() + off);
  }
  template <class T>
  static T* at(char* base, size_t off) {
    return reinterpret_cast<T*>(base + off);
  }
  size_t bytes() const { return buf_.size(); }
  const char* data() const { return buf_.data(); }
  char* mutable_data() { return buf_.data(); }
  // Buffer recycling (a fresh 10 MB vector costs thousands of page faults):
  // start from a used buffer's capacity / hand the buffer back.
  void adopt(std::vector<char>&& b) {
    buf_ = std::move(b);
    buf_.clear();
  }
  std::vector<char> take() { return std::move(buf_); }

 private:
  std::vector<char> buf_;
};

// Ring of pinned host + device staging slots for task/plan uploads: the
// host copies a pack into a pinned slot and enqueues an async H2D, so it can
// keep planning while the device works; a slot is reused only after the
// kernels that read it (fenced by an event) have finished.
class Staging {
 public:
  explicit Staging(int slots = 8) : s_(slots) {}
  ~Staging();
  char* put(const Pack& pk, cudaStream_t st);
  void fence(cudaStream_t st);

 private:
  struct Slot {
    char* host = nullptr;
    char* dev = nullptr;
    size_t cap = 0;
    cudaEvent_t ev = nullptr;  // the kernels reading the slot are done
    cudaEvent_t up = nullptr;  // the slot's upload is done
    bool pending = false;
    bool uploading = false;    // `up` recorded since the last host rewrite
  };
  std::vector<Slot> s_;
  int cur_ = -1;
  // uploads run on their own stream, so a wave's task arrays cross PCIe
  // while the previous wave computes; the compute stream waits on `up`
  cudaStream_t copy_ = nullptr;
};

// ------------------------------------------------------------ segment tree
// Bounding boxes over node index ranges, for the enclosed-node search of
// build_proxy (proj/src/compression.cpp:62-66): same predicate, node order
// and result, visiting only boxes that can intersect the circle.
class NodeBoxTree {
 public:
  void build(const double* xy, int n);
  void enclosed(const double* xy, double cx, double cy, double radius,
                int begin, int end, std::vector<int>& out) const;

 private:
  struct Box { int lo, hi, left, right; double x0, y0, x1, y1; };
  int make(const double* xy, int lo, int hi);
  std::vector<Box> boxes_;
  int root_ = -1;
};

// ------------------------------------------------------------------ problem
struct ProxyGeom {
  double cx, cy, radius;
  std::vector<int> enclosed;
};

struct BasisReq {  // one cell_basis call
  const Lists* rows;
  const Lists* cols;
  int begin, end;
  // Chained level-by-level calls (Fds::build): indices of the cell's two
  // children in the previous chained call, whose interaction matrices still
  // hold the entries (enclosed node of both, child skeleton) this cell needs
  // again; -1: none (leaf cells, single cell_basis calls).
  int child[2] = {-1, -1};
};

// What a chained bases() call leaves for the next level: where each cell's
// interaction matrices are and which of their columns its skeletons were.
struct PrevLevel {
  bool valid = false;
  int buf = 0;  // which of the two interaction buffers holds the matrices
  std::vector<ProxyGeom> geom;
  std::vector<size_t> tv_off, tu_off;
  std::vector<int> n_out, nc0, nr0;
  // per cell: column positions (within the component's half) and nodes of
  // the k skeletons of cols[0], cols[1], rows[0], rows[1]
  std::vector<std::array<std::vector<int>, 4>> spos, snode;
};

struct BasisRes {
  int k = 0;
  bool saturated = false;
  Lists srow, scol;
  size_t v_off = 0;  // V0 (k x nc0) then V1 (k x nc1) in the V buffer
  size_t u_off = 0;  // U0 (nr0 x k) then U1 (nr1 x k) in the U buffer
};

class FillPlan;

// Entry copies planned by one planning thread (offsets local to the part).
struct MapPart {
  std::vector<MapTask> tasks;
  std::vector<int2> rows, cols;
};

// Records batched LA launches (copies, GEMMs, LU solves) instead of issuing
// them: the task arrays of a whole solve are uploaded once and the launch
// sequence is captured into a CUDA graph that each solve replays.
class Recorder {
 public:
  template <class T>
  void add(int kind, const std::vector<T>& t, const std::vector<int>& boff,
           int total, int aux = 0, int aux2 = 0) {
    Launch l;
    l.kind = kind;
    l.aux2 = aux2;
    l.task_off = pk_.add(t);
    l.boff_off = pk_.add(boff);
    l.n_tasks = int(t.size());
    l.n_blocks = total;
    l.aux = aux;
    launches_.push_back(l);
  }
  void mark() { marks_.push_back(int(launches_.size())); }
  // An L2 warm-up of the given ranges plus this recording's own task arrays
  // (their range is filled in by finalize).
  void add_prefetch(std::vector<PrefetchTask> ranges) {
    ranges.push_back(PrefetchTask{nullptr, 0});
    Launch l{};
    l.kind = kPrefetchKind;
    l.task_off = pk_.add(ranges);
    l.n_tasks = int(ranges.size());
    launches_.push_back(l);
  }
  static constexpr int kPrefetchKind = 1000;
  // Starts a recording on the process-wide recycled host buffer.
  void begin();
  void finalize(cudaStream_t st);
  // launches between marks a and b (phase a of the recording)
  void replay(cudaStream_t st, int phase);
  int n_marks() const { return int(marks_.size()); }
  size_t n_launches() const { return launches_.size(); }

 private:
  struct Launch {
    int kind;
    size_t task_off, boff_off;
    int n_tasks, n_blocks;
    int aux;  // k_getrs: dynamic shared memory bytes
    int aux2;  // k_getrs: largest LU order of the batch
  };
  Pack pk_;
  std::vector<Launch> launches_;
  std::vector<int> marks_;
  DBuf<char> dev_;
};

// Process-wide device scratch and stream shared by every handle: new
// problems and solvers reuse warm buffers (GBs of bundles, pinned staging)
// instead of reallocating them.  All C ABI entry points serialise on
// api_mutex(), so one stream orders every use of the shared buffers.
struct Scratch {
  cudaStream_t st = nullptr;
  Staging staging;
  DBuf<double> tbuf, tbuf_alt;  // interaction matrices (two: level l and l+1)
  std::vector<DBuf<double>> qr_rounds;
  DBuf<int> id_jp, id_steps;
  DBuf<double> id_rd, id_r;
  DBuf<unsigned char> sym_keys;
  DBuf<int> sym_vals;
  DBuf<double> sym_recs;  // kSymRec doubles per sorted near pair
  DBuf<int> sym_bounds;
  DBuf<double> bundles;
  DBuf<double2> gws;
  PinnedBuf<double> h_geom;      // element geometry staging of a problem setup
  PinnedBuf<int> h_jp, h_steps;  // pivoted-QR readbacks
  PinnedBuf<double> h_rd;
};
Scratch& scratch();

// Runs f(i) for i in [0, n) on the process's planning threads (the calling
// thread takes part).  f must not throw.
void parallel_for(int n, const std::function<void(int)>& f);
int planning_threads();

// A tall complex block (column-major, ld) whose R factor the ID needs.
struct TallBlock {
  const double* p;
  int rows, n, ld;
};
// force: also reduce blocks that fit shared memory (parity hook).
void reduce_tall(std::vector<TallBlock>& q, cudaStream_t st, bool force = false);

class Problem {
 public:
  Problem(const double* xy, int n, double lam, double mu, double rho,
          double omega, double are, double aim, const ebem_assembly_config& a,
          const ebem_proxy_config& p);
  // Source-only handle (host BlockSource callbacks): no geometry on device.
  explicit Problem(int n);
  ~Problem();

  int n() const { return n_; }
  cudaStream_t stream() const { return st_; }
  const ebem_proxy_config& proxy_cfg() const { return pcfg_; }
  const ebem_assembly_config& asm_cfg() const { return acfg_; }
  const DevCtx* dctx() const { return dctx_.get(); }
  const double* xy() const { return xy_.data(); }

  ProxyGeom build_proxy(int begin, int end) const;
  // Runs a fill plan (bundles + gathers) on the stream.
  void execute(FillPlan& plan);
  // Raises std::domain_error semantics when a singular-pair series check
  // failed since the last call.
  void check_domain();
  // Shared-rank bases of a batch of cells (AssemblerSource::cell_basis).
  // V/U coefficient blocks land in vbuf/ubuf (device), offsets in res.
  void bases(const std::vector<BasisReq>& req, double eps,
             std::vector<BasisRes>& res, DBuf<double>& vbuf,
             DBuf<double>& ubuf, double* fill_seconds = nullptr, bool chain = false,
             bool defer_lists = false);
  // Fills in the skeleton lists of the last bases() call made with
  // defer_lists (req and res must still be alive), and records the level
  // for the next chained call.
  void finish_bases();
  // Forget the previous chained level (start of a factorization).
  void reset_chain() { prev_.valid = false; }
  // true_block(rows, cols) of two sibling cells' skeletons (the off-diagonal
  // blocks of a reduced diagonal, fds.cpp:33-54): rows = srow of the child
  // with index ca in the previous chained level, cols = scol of child cb.
  // Entries whose row node lies inside cb's proxy circle are copied from cb's
  // T_V, those whose column node lies inside ca's circle from ca's T_U
  // (conjugate-transposed); the rest is planned as a true block.
  void plan_sibling_block(FillPlan& plan, MapPart& mp, int ca, int cb, const Lists& rows,
                          const Lists& cols, double* dest, int ld, const int drow[2],
                          const int dcol[2]);
  // Runs the entry copies planned by plan_sibling_block (one launch).
  void run_map_copies(std::vector<MapPart>& parts);
  // Interaction matrices (device, column-major) of a batch of cells:
  // T_V = M_V (n_out x ncols) and T_U = M_U^H (n_out x nrows).
  void interaction(const std::vector<BasisReq>& req,
                   std::vector<ProxyGeom>& geom, std::vector<size_t>& tv_off,
                   std::vector<size_t>& tu_off, std::vector<int>& n_out,
                   DBuf<double>& tbuf, const PrevLevel* prev = nullptr);
  void true_block_host(const Lists& rows, const Lists& cols, double* out);
  void rhs_plane(int kind, const double* angles, int m, double amp,
                 double* out_host);
  // evaluate_scattered / evaluate_field (proj/src/postprocess.cpp:56-119);
  // kind < 0: scattered only.  Host buffers.
  void field(const double* boundary_u, const double* pts, int m, int n_gauss, int kind,
             double angle, double amp, double* out_u, double* out_int);

  // scratch shared by the drivers (process-wide, see Scratch)
  Staging& staging;
  DBuf<double>& tbuf_;     // interaction matrices of the current basis batch
  std::vector<DBuf<double>>& qr_rounds_;  // TSQR round outputs (grow-only)
  DBuf<int>& id_jp_;
  DBuf<int>& id_steps_;
  DBuf<double>& id_rd_;
  DBuf<double>& id_r_;
  DBuf<unsigned char>& sym_keys_;   // 2 x pairs (in, out)
  DBuf<int>& sym_vals_;             // 2 x pairs (in, out)
  DBuf<double>& sym_recs_;          // sorted pair records (geometry, outputs)
  DBuf<int>& sym_bounds_;
  DBuf<double>& bundles;
  DBuf<double2>& gws;
  DBuf<int> bad;
  Recorder* recorder = nullptr;  // set while a solve is being recorded

 private:
  int n_;
  std::vector<double> xy_, elem_;
  double hmin_ = 0, hmax_ = 0;
  ebem_assembly_config acfg_;
  ebem_proxy_config pcfg_;
  DevCtx hctx_{};
  FillConst fc_{};
  DBuf<DevCtx> dctx_;
  DBuf<double> delem_, delem8_, dxy_;
  cudaStream_t st_ = nullptr;
  NodeBoxTree tree_;
  PrevLevel prev_;
  struct PendingBases {
    bool active = false, chain = false;
    int cur_buf = 0;
    const std::vector<BasisReq>* req = nullptr;
    std::vector<BasisRes>* res = nullptr;
    const int* h_jp = nullptr;
    std::vector<size_t> jp_off, tv_off, tu_off;
    std::vector<ProxyGeom> geom;
    std::vector<int> n_out;
  } pend_;
};

// Work planner for one batch of Galerkin fills.
class FillPlan {
 public:
  FillPlan(int n_nodes, int m_prime, int n_gauss)
      : N_(n_nodes), m_(m_prime), ng_(n_gauss) {}
  // true_block(rows, cols) into dest with per-component destination offsets;
  // trans writes conj(v) at (col, row).
  // rpos / cpos (optional, per component): destination position of each
  // listed node relative to drow / dcol instead of its index in the list.
  void add_true_block(const Lists& rows, const Lists& cols, double* dest,
                      int ld, const int drow[2], const int dcol[2], int trans,
                      const std::vector<int>* const* rpos = nullptr,
                      const std::vector<int>* const* cpos = nullptr);
  // Both proxy blocks of one cell: polygon rows -> T_V rows [0, 2m'),
  // polygon cols of M_U -> T_U rows [0, 2m') (conj-transposed).
  void add_proxy(double cx, double cy, double radius, const Lists& rows,
                 const Lists& cols, double* tv, int ld_v, double* tu, int ld_u);
  // Both near blocks of a cell: true_block(enc x 2, cols) into T_V rows
  // [2m', 2m' + 2|enc|) and true_block(rows, enc x 2)^H into T_U rows, from
  // one scalar evaluation per point (enc ascending).
  void add_sym_near(const std::vector<int>& enc, const Lists& rows,
                    const Lists& cols, double* tv, int ld_v, double* tu,
                    int ld_u);
  // The same for a part of the cell's blocks: the enclosed nodes enc (row
  // position enc_pos[k] of the cell's ne_total enclosed nodes) against the
  // row / column sub-lists, whose first entries sit at rdest / cdest.
  void add_sym_near_part(const std::vector<int>& enc, const std::vector<int>* enc_pos,
                         int ne_total, const Lists& rows, const int rdest[2],
                         const Lists& cols, const int cdest[2], double* tv, int ld_v,
                         double* tu, int ld_u);
  // true_block(J, J) for an ascending node list J (the leaf diagonal) from
  // the upper triangle of element pairs, both orientations per evaluation.
  void add_sym_diag(const std::vector<int>& nodes, double* dest, int ld);
  long long bundles() const { return bundles_; }
  bool empty() const { return gather_.empty(); }
  bool has_one_sided_ = false, has_two_sided_ = false;  // kinds of near jobs
  void clear();
  // Appends another plan (built independently, e.g. on another host thread)
  // with its element, bundle, pair, descriptor and entry offsets relocated.
  void append(const FillPlan& o);
  // append(parts[k0]), ..., append(parts[k1 - 1]) with the copies and
  // relocations of the parts done in parallel on the planning threads.
  void append_many(const std::vector<FillPlan>& parts, int k0, int k1);

 private:
  friend class Problem;
  void elements_of(const Lists& nodes, std::vector<int>& out) const;
  void node_descs(const Lists& nodes, const std::vector<int>& elems,
                  const int dest_off[2], std::vector<NodeDesc>& out,
                  const std::vector<int>* const* pos = nullptr) const;
  int poly_descs();
  int N_, m_, ng_;
  long long bundles_ = 0;
  long long entries_ = 0;
  int proxy_blocks_ = 0;
  int poly_desc_off_ = -1;
  std::vector<int> elems_;
  std::vector<long long> sing_pair_;
  std::vector<int> sing_elems_;
  std::vector<SymJob> sym_;
  std::vector<long long> sym_off_;
  long long sym_pairs_ = 0;
  std::vector<ProxyJob> proxy_;
  std::vector<int> proxy_boff_;
  std::vector<GatherJob> gather_;
  std::vector<long long> gather_off_;
  std::vector<NodeDesc> desc_;
};

// ----------------------------------------------------------------- solver
struct HostSource {
  ebem_block_fn block;
  ebem_basis_fn basis;
  void* user;
};

class Fds {
 public:
  Fds(Problem& p, int depth, const ebem_fds_config& cfg,
      const HostSource* hs = nullptr);
  void solve_device(const double* rhs, int m, double* x, ebem_fds_solve_timing* t);
  const ebem_fds_stats& stats() const { return stats_; }
  int rank_of(int cell) const;
  void debug_cell(int cell, int which, double* out) const;
  void cell_info(int cell, int* sizes, int* skel) const;
  Problem& problem() { return P_; }

 private:
  struct Cell {
    int begin = 0, end = 0;
    Lists jrow, jcol, srow, scol;
    int nloc = 0, k = 0;
    // device factors
    double* lu = nullptr;
    int* ipiv = nullptr;
    int* perm = nullptr;  // the interchanges composed (single-RHS solves)
    double* ainv_u = nullptr;  // 2n x 2k
    double* v = nullptr;       // V0 (k x n) then V1 (k x n)
    double* atilde = nullptr;  // 2k x 2k
  };
  struct Store {
    DBuf<double> lu, ainv_u, v, atilde;
    DBuf<int> ipiv;
  };
  void build();
  // host-source path (callbacks): bases, exact blocks, reduced diagonals
  void host_bases(int level, std::vector<BasisRes>& br, DBuf<double>& vbuf,
                  DBuf<double>& ubuf);
  std::vector<double> host_block(const Lists& rows, const Lists& cols);
  void host_reduced_diagonal(int cell, double* out, int ld);
  const HostSource* hs_ = nullptr;
  void reduced_diagonal(FillPlan& plan, std::vector<CopyTask>& copies, int cell,
                        double* dest, int ld, int off, MapPart* mp = nullptr);
  int first(int l) const { return (1 << l) - 1; }
  int last(int l) const { return (2 << l) - 2; }

  Problem& P_;
  int depth_;
  ebem_fds_config cfg_;
  std::vector<Cell> cells_;
  std::vector<Store> store_;
  std::vector<int> top_off_;
  DBuf<double> top_lu_;
  DBuf<int> top_ipiv_;
  int top_dim_ = 0;
  ebem_fds_stats stats_{};
  double last_solve_device_seconds_ = 0.0;
  int* lu_info(int n);
  DBuf<int> info_;            // zero-pivot flags of every LU of the build
  std::vector<int> info_n_;   // their matrix sizes (for the error message)
  DBuf<double> ubuf_, wbuf_;  // per-level temporaries (grow-only)
  DBuf<int> wpiv_;
  // solve workspaces and the recorded solve (one cached plan, per m)
  DBuf<double> ws_f_, ws_ainvf_, ws_ft_, ws_x_, ws_t_;
  void record_solve(int m);
  struct SolvePlan {
    int m = -1;
    Recorder rec;
    DBuf<double> rhs, x;
    cudaGraph_t graph[3] = {nullptr, nullptr, nullptr};  // up, top, down
    cudaGraphExec_t exec[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    SolvePlan() = default;
    SolvePlan(const SolvePlan&) = delete;
    SolvePlan& operator=(const SolvePlan&) = delete;
    ~SolvePlan() {  // a re-recorded plan releases its graphs and events
      for (int ph = 0; ph < 3; ++ph) {
        if (exec[ph]) cudaGraphExecDestroy(exec[ph]);
        if (graph[ph]) cudaGraphDestroy(graph[ph]);
      }
      for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
    }
  };
  std::unique_ptr<SolvePlan> plan_;

 public:
  ~Fds();
};

// ------------------------------------------------------------ batched LA
// Thin host helpers that upload task arrays and launch the dense kernels.
// Dense reference solver (ConvSolver, proj/src/dense_solver.cpp:9-29).
struct ConvStatsC {
  double assemble_seconds = 0.0, factor_seconds = 0.0, rcond = 1.0, min_pivot = 0.0;
  bool condition_warning = false;
};
class Conv {
 public:
  explicit Conv(Problem& p);
  const ConvStatsC& stats() const { return stats_; }
  int size() const { return d_; }
  void solve_host(const double* rhs, int m, double* x);
  // BlockAssembler::dense into a host buffer (2N x 2N, column-major)
  static void dense_host(Problem& P, double* out);

 private:
  static void check_size(const Problem& P);
  static void assemble(Problem& P, double* dest);
  void apply_inv(double* x);
  void apply_inv_h(double* x);
  double rcond();
  Problem& P_;
  int d_;
  DBuf<double> lu_;
  DBuf<int> ipiv_, info_;
  double norm1_ = 0.0;
  ConvStatsC stats_;
};

void run_copies(Problem& P, const std::vector<CopyTask>& t);
void run_gemms(Problem& P, const std::vector<GemmTask>& t);
void run_getrs(Problem& P, const std::vector<LuSolveTask>& t);
// Factors in place; zero-pivot flags land in each task's info pointer.
void run_getrf(Problem& P, std::vector<LuTask> t);

}  // namespace ebem_gpu
