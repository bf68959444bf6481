// Host runtime of libsvd1: plan, Alg 6.1 orchestration, the O(n)
// decision logic of Alg 6.2 (sorting, deflation, merge), and the FMM tree
// / interaction lists.  Every O(n^2) and O(rows*n)
// step runs in the CUDA kernels of kernels_spectral.cu / kernels_apply.cu.
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl.so.2 is opened at run time when a plan spans ranks

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <memory>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <numeric>
#include <string>
#include <thread>
#include <vector>

#include "svd1_internal.cuh"

using namespace svd1;

namespace {

double now_ms() {
  using namespace std::chrono;
  return duration<double, std::milli>(steady_clock::now().time_since_epoch()).count();
}

// Allocations made by the library (device, stream-ordered pool, pinned host) since the
// process started: svd1_report.allocations is the difference over one call.  The plan
// sizes its workspaces at creation (svd1_plan_create), so an update allocates only if its
// FMM plan outgrows the create-time estimate of a plan-dependent buffer.
std::atomic<int64_t> g_allocs{0};

// grow-only device buffer
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  bool pooled = false;  // from cudaMallocAsync (stream-ordered pool)
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() {
    if (p) {
      if (pooled) cudaFreeAsync(p, nullptr);
      else cudaFree(p);
    }
  }
  // Create-time sizing (and the test hooks): cudaMalloc of exactly `count` elements.
  template <class T>
  svd1_status reserve(size_t count) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    if (bytes <= cap) return SVD1_OK;
    release();
    ++g_allocs;
    if (cudaMalloc(&p, bytes) != cudaSuccess) {
      cudaGetLastError();
      p = nullptr;
      return SVD1_E_NOMEM;
    }
    cap = bytes;
    return SVD1_OK;
  }
  void release() {
    if (p) {
      if (pooled) cudaFreeAsync(p, nullptr);
      else cudaFree(p);
    }
    p = nullptr;
    cap = 0;
    pooled = false;
  }
  // Inside an update: a buffer that outgrows its create-time size grows geometrically
  // in stream order on `st` (the stream of its first use; cudaFreeAsync / cudaMallocAsync
  // from the device's pool): no device-wide synchronisation.
  template <class T>
  svd1_status get(size_t count, T** out, cudaStream_t st) {
    const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
    if (bytes > cap) {
      const size_t want = std::max(bytes + bytes / 2, size_t(4096));
      if (p) {
        if (pooled) cudaFreeAsync(p, st);
        else cudaFree(p);  // (a create-time buffer that was too small: one-off)
      }
      p = nullptr;
      cap = 0;
      ++g_allocs;
      if (cudaMallocAsync(&p, want, st) != cudaSuccess) {
        cudaGetLastError();
        p = nullptr;
        return SVD1_E_NOMEM;
      }
      pooled = true;
      cap = want;
    }
    *out = static_cast<T*>(p);
    return SVD1_OK;
  }
  // sized at creation: never grows
  template <class T>
  svd1_status get_fixed(size_t count, T** out) {
    if (std::max<size_t>(count, 1) * sizeof(T) > cap) return SVD1_E_NOMEM;
    *out = static_cast<T*>(p);
    return SVD1_OK;
  }
};

// pinned host buffer sized at creation (grows, counted, only if an estimate was short)
svd1_status pinned_reserve(void** buf, size_t* cap, size_t bytes) {
  if (bytes <= *cap) return SVD1_OK;
  if (*buf) cudaFreeHost(*buf);
  *buf = nullptr;
  *cap = 0;
  ++g_allocs;
  if (cudaMallocHost(buf, bytes) != cudaSuccess) {
    cudaGetLastError();
    *buf = nullptr;
    return SVD1_E_NOMEM;
  }
  *cap = bytes;
  return SVD1_OK;
}

constexpr int kMaxPairTracked = 256;  // D5: repeated-sigma columns tracked for clusters beyond the probes
constexpr int kMaxBatch = 28;  // svd1_update_batch: buffers are sized for this many updates per call

// ---- NCCL, opened at run time (no link-time dependency; in a process that already
// loaded torch's libnccl.so.2 the same library is reused)
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
const NcclApi& nccl_api() {
  static const NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    auto sym = [h](const char* nm) { return dlsym(h, nm); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommSplit = reinterpret_cast<decltype(a.CommSplit)>(sym("ncclCommSplit"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommSplit && a.AllGather && a.GroupStart && a.GroupEnd &&
           a.CommDestroy && a.GetErrorString;
    return a;
  }();
  return api;
}

svd1_status nccl_fail(ncclResult_t r, const char* what) {
  const NcclApi& A = nccl_api();
  std::fprintf(stderr, "[svd1] NCCL error %d (%s) in %s\n", int(r), A.GetErrorString ? A.GetErrorString(r) : "?",
               what);
  return SVD1_E_NCCL;
}
#define NCCL_TRY(expr)                                  \
  do {                                                  \
    ncclResult_t _r = (expr);                           \
    if (_r != ncclSuccess) return nccl_fail(_r, #expr); \
  } while (0)

// Rank r's slice [lo, hi) of n indices: contiguous blocks of c = ceil(n / G), so rank r's
// results sit at [r c, r c + c) of a G c buffer -- the in-place all-gather layout.
struct Slice {
  int c, lo, hi;
};
inline Slice slice_of(int n, int G, int r) {
  const int c = (n + G - 1) / G;
  const int lo = std::min(n, r * c);
  return Slice{c, lo, std::min(n, lo + c)};
}

#define TRY(expr)                       \
  do {                                  \
    svd1_status _s = (expr);            \
    if (_s != SVD1_OK) return _s;       \
  } while (0)

// 2x2 symmetric Schur split of [[beta, 1], [1, 0]]: rho1 > 0 > rho2 =
// -1/rho1, Q = [[rho1, -1], [1, rho1]] / sqrt(1 + rho1^2) (columns = eigenvectors).
struct Split {
  double rho1, rho2, q00, q01, q10, q11;
};
Split schur_split(double beta) {
  Split s;
  s.rho1 = 0.5 * (beta + std::hypot(beta, 2.0));
  s.rho2 = -1.0 / s.rho1;
  const double h = std::hypot(1.0, s.rho1);
  s.q00 = s.rho1 / h;
  s.q10 = 1.0 / h;
  s.q01 = -1.0 / h;
  s.q11 = s.rho1 / h;
  return s;
}

// Reading D9 (oracle balance_factor): c = 2^floor(e / 2) with
// x / y = f 2^e, f in [0.5, 1); 1 if either norm is 0 or not finite.  A side's Schur split
// takes the rank-1 term as (c a)(b / c)^T with its two vectors' norms within a
// factor of 2 of each other: [[beta, 1], [1, 0]] is not invariant under that exact rewriting,
// and with ||a|| >> ||A b|| its two eigen-updates cancel to eps ||a||^2.  A power of two
// keeps the rescaled vectors exact and makes (2^t a, b / 2^t) give bitwise the same update.
double balance_factor(double x, double y) {
  if (!(x > 0.0 && y > 0.0 && std::isfinite(x) && std::isfinite(y))) return 1.0;
  int ex = 0, ey = 0, e2 = 0;
  const double mx = std::frexp(x, &ex), my = std::frexp(y, &ey);
  std::frexp(mx / my, &e2);
  const int e = ex - ey + e2;
  return std::ldexp(1.0, e >= 0 ? e / 2 : -((1 - e) / 2));  // floor(e / 2)
}

struct FmmHost {
  int L = 0, ncells = 0;
  int ecells = 0;     // expansion columns / p: the cells, then one slot per fused P2L pair
  int64_t cap_cells = 0;  // expansion columns / p the plan's workspaces hold (0: no slots)
  std::vector<FmmCell> cells;
  std::vector<FmmOpDesc> ops;
  std::vector<FmmTerm> terms;
  std::vector<FmmTask> tasks;
  std::vector<int> pass_begin;  // task index where each pass starts (+ end sentinel)
  std::vector<int> pass_bn;     // tile width (16 or 32) of each pass
  std::vector<int> pass_kind;   // 0 P2M, 1 M2M band, 2 M2L, 3 L2L band, 4 final (L2P + M2P + P2P)
  int64_t ops_rows = 0;         // ops buffer: rows of 16 doubles
  int64_t flops_per_row = 0;    // algorithmic flops per row (level by level)
  int64_t flops_exec_per_row = 0;  // flops the plan executes per row (level bands included)
  int64_t flops_cost_per_row = 0;  // the same without the sibling pairs' zero blocks (the
                                   // depth search's cost: pairing does not change it)
  int n_near_pairs = 0, n_m2l_pairs = 0, max_near = 0;
};

// secular FMM plan (host side; see secfmm_plan)
struct SecPlanHost {
  int L = 0, ncells = 0, nleaf = 0;
  std::vector<SecFmmCell> cells;  // ncells + 1 (sentinel carries the partner count)
  std::vector<SecFmmPart> parts;
  std::vector<int32_t> leaf_lo, leaf_cell, near_off, near_lo, near_hi;
  std::vector<int32_t> direct;  // roots outside every target interval (direct sum)
};

struct CauchyPrep {
  bool fmm = false;
  int p = 16;
  int na = 0;
  int64_t rows = 0;
  double flops = 0.0;       // algorithmic
  double flops_exec = 0.0;  // executed by the plan
  FmmHost F;
  std::vector<int32_t> col2src;  // input column -> active source (-1: none); empty = identity
  int n_in = 0;                  // columns of the input buffer
  int n_out = 0;                 // columns of the output buffer
  DevBuf blob, d_ops, d_maps;  // blob: cells, descs, terms, tasks, col2src (one copy)
  FmmCell* dcells = nullptr;
  FmmOpDesc* ddescs = nullptr;
  FmmTerm* dterms = nullptr;
  FmmTask* dtasks = nullptr;
  int32_t* dcol2src = nullptr;
  size_t o_cells = 0, o_descs = 0, o_terms = 0, o_tasks = 0, o_c2s = 0;
  FmmMaps* h_maps = nullptr;  // pinned staging of the TMA descriptors (copied on the apply stream)
  size_t h_maps_cap = 0;
  std::vector<cudaEvent_t> gev;  // events around each GEMM pass of the last launch
  int ngev = 0;
  bool ops_ready = false;  // operator blocks already built (batch mode: on the upload stream)
  ~CauchyPrep() {
    if (h_maps) cudaFreeHost(h_maps);
    for (auto e : gev) cudaEventDestroy(e);
  }
  // device time of the GEMM passes of the last launch (after it completed)
  double gemm_ms() const {
    double t = 0.0;
    for (int i = 0; i + 1 < ngev; i += 2) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, gev[i], gev[i + 1]) == cudaSuccess) t += ms;
      else cudaGetLastError();
    }
    return t;
  }
};

// Everything one RankOneUpdate (Alg 6.2) needs at apply time.
// Host worker threads (apply planners, the U chain, the apply launchers: ~7 per update) are
// taken from a cache of persistent threads instead of being created and destroyed each
// time: a job starts on an idle worker (or on a new one when none is idle, so a job that
// waits for another never starves it), and the handle's join() waits for that job only.
// SVD1_THREAD_POOL=0 falls back to one std::thread per job (experiments).
class WorkerPool {
 public:
  struct Done {
    std::mutex m;
    std::condition_variable cv;
    std::atomic<bool> done{false};
  };
  static WorkerPool& get() {
    static WorkerPool* pool = new WorkerPool;  // never destroyed: idle workers outlive exit
    return *pool;
  }
  // spin up to kSpinUs before blocking on a condition variable: a job's start and its join
  // are on the update's critical path, and a futex wake-up costs tens of microseconds
  static constexpr int kSpinUs = 60;
  template <class Pred>
  static bool spin(Pred ready) {
    const auto t0 = std::chrono::steady_clock::now();
    for (int i = 0;; ++i) {
      if (ready()) return true;
      if ((i & 63) == 63 &&
          std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(kSpinUs))
        return false;
    }
  }
  std::shared_ptr<Done> submit(std::function<void()> f) {
    auto d = std::make_shared<Done>();
    Worker* w = nullptr;
    {
      std::lock_guard<std::mutex> lk(m_);
      if (!idle_.empty()) {
        w = idle_.back();
        idle_.pop_back();
      } else {
        all_.push_back(std::make_unique<Worker>());
        w = all_.back().get();
        std::thread([this, w] { loop(w); }).detach();
      }
    }
    {
      std::lock_guard<std::mutex> lk(w->m);
      w->job = [f = std::move(f), d] {
        f();
        {
          std::lock_guard<std::mutex> l2(d->m);
          d->done.store(true, std::memory_order_release);
        }
        d->cv.notify_all();
      };
      w->has_job.store(true, std::memory_order_release);
    }
    w->cv.notify_one();
    return d;
  }
  static void wait(Done& d) {
    if (spin([&d] { return d.done.load(std::memory_order_acquire); })) return;
    std::unique_lock<std::mutex> lk(d.m);
    d.cv.wait(lk, [&d] { return d.done.load(std::memory_order_acquire); });
  }

 private:
  struct Worker {
    std::mutex m;
    std::condition_variable cv;
    std::function<void()> job;
    std::atomic<bool> has_job{false};
  };
  void loop(Worker* w) {
    for (;;) {
      std::function<void()> job;
      spin([w] { return w->has_job.load(std::memory_order_acquire); });
      {
        std::unique_lock<std::mutex> lk(w->m);
        w->cv.wait(lk, [w] { return w->has_job.load(std::memory_order_acquire); });
        job = std::move(w->job);
        w->has_job.store(false, std::memory_order_relaxed);
      }
      job();
      job = nullptr;
      std::lock_guard<std::mutex> lk(m_);
      idle_.push_back(w);
    }
  }
  std::mutex m_;
  std::vector<Worker*> idle_;
  std::vector<std::unique_ptr<Worker>> all_;
};

// std::thread-like handle (start at construction, joinable(), join()) over the pool
class WorkThread {
 public:
  WorkThread() = default;
  template <class F>
  explicit WorkThread(F&& f) {
    static const bool pooled = [] {
      const char* e = std::getenv("SVD1_THREAD_POOL");
      return !(e && atoi(e) == 0);
    }();
    if (pooled) d_ = WorkerPool::get().submit(std::function<void()>(std::forward<F>(f)));
    else t_ = std::thread(std::forward<F>(f));
  }
  WorkThread(WorkThread&&) = default;
  WorkThread& operator=(WorkThread&& o) {
    if (joinable()) std::terminate();  // as std::thread: never overwrite a running job
    d_ = std::move(o.d_);
    t_ = std::move(o.t_);
    return *this;
  }
  ~WorkThread() {
    if (joinable()) std::terminate();
  }
  bool joinable() const { return bool(d_) || t_.joinable(); }
  void join() {
    if (d_) {
      WorkerPool::wait(*d_);
      d_.reset();
    }
    if (t_.joinable()) t_.join();
  }

 private:
  std::shared_ptr<WorkerPool::Done> d_;
  std::thread t_;
};

struct StepRecord {
  int N = 0;                          // size of the eigenproblem (columns of the buffer)
  int na = 0;                         // active (secular) size
  int nap = 0;                        // na padded to world * slice (all-gather layout)
  double rho = 0.0;
  std::vector<int32_t> h_goff, h_cols;  // Householder groups (buffer columns)
  std::vector<double> h_hv;
  int h_maxlen() const {  // longest Householder group
    int mx = 0;
    for (size_t g = 0; g + 1 < h_goff.size(); ++g) mx = std::max(mx, h_goff[g + 1] - h_goff[g]);
    return mx;
  }
  std::vector<int32_t> src_cols;      // active source i -> input buffer column
  std::vector<int32_t> pass_src, pass_dst;  // deflated: input col -> output position
  std::vector<double> pass_scale;
  std::vector<int32_t> tgt_pos;       // active target j -> output position q
  std::vector<int32_t> dst_cols, pass_dst_cols;  // output buffer columns
  std::vector<double> da, mu, tau_h, cs_h;  // host copies (tree + sign folding)
  std::vector<int32_t> k_h;
  int max_iter = 0;
  double mean_iter = 0.0;
  double spectral_ms = 0.0;
  int ev0 = 0, nc = 0;
  int64_t rows = 0;
  std::vector<int32_t> perm;
  std::vector<int> act, dfl;
  std::vector<double> ds;
  std::vector<std::vector<double>> cs_sorted;
  std::vector<double> Dn;              // next eigenvalues / carries (recycled storage)
  std::vector<std::vector<double>> cn;
  // host-only carries (D5, clusters larger than the probes): the coordinates of a repeated
  // singular value's original columns in this step's basis, through the deflation
  // reflections and the merge only (their active entries are not needed: set to 0)
  std::vector<std::vector<double>>* gcar = nullptr;
  std::vector<std::vector<double>> gs_sorted, gn;
  double* rb = nullptr;  // pinned read-back
  size_t rb_cap = 0;
  cudaEvent_t done_ev = nullptr;  // recorded after the read-back copy
  double plan_ms = 0.0;           // host time of the last apply_plan (diagnostics)
  bool pending = false;           // spectral work in flight (wait on done_ev)
  WorkThread plan_thread;             // apply_plan on a worker thread (plan-owned: it may
  std::atomic<bool> planned{false};   // outlive the update_impl call that started it)
  void join_plan() {
    if (plan_thread.joinable()) plan_thread.join();
  }
  ~StepRecord() {
    join_plan();
    if (rb) cudaFreeHost(rb);
    if (done_ev) cudaEventDestroy(done_ev);
  }
  void clear_host() {
    spectral_ms = 0.0;
    N = na = 0;
    rho = 0.0;
    max_iter = 0;
    h_goff.clear(); h_cols.clear(); h_hv.clear(); src_cols.clear(); pass_src.clear();
    pass_dst.clear(); pass_scale.clear(); tgt_pos.clear(); da.clear(); mu.clear();
    tau_h.clear(); cs_h.clear(); k_h.clear();
  }
  // device arrays
  DevBuf d_zhat, d_scratch, d_in, d_out;
  DevBuf d_ctr;  // last-block counters of the Loewner / norm kernels (kept zero)
  DevBuf blob;  // apply data (Householder groups, column maps, scales, FMM plan): one copy
  int32_t *dgoff = nullptr, *dhcols = nullptr, *dsrc = nullptr, *ddst = nullptr, *dpsrc = nullptr,
          *dpdst = nullptr;
  double *dhv = nullptr, *dcs = nullptr, *dpscale = nullptr;
  std::vector<double> stage;
  CauchyPrep cp;
  SecPlanHost sec;          // secular FMM plan (large active sizes)
  DevBuf sec_blob, sec_scr;
  int sec_fmm_used = 0;
  DevBuf rot_goff, rot_cols, rot_mats;  // pairing rotations (the V2 step's record)
};



}  // namespace

// Kernel launches are counted per host thread (the U- and V-side chains of an update run on
// two threads) and flushed into the plan's atomic total at the chains' ends.
thread_local int64_t tl_launches = 0;

struct svd1_plan_s {
  svd1_config cfg{};
  cudaStream_t st = nullptr;
  int p = 16, leaf = 32;
  // ranks: the spectral phase of every eigen-update is sliced -- roots,
  // Loewner weights and column norms of rank r's index range -- and all-gathered over NCCL,
  // one communicator per side chain (U: 0, V: 1), so each chain's collectives are issued
  // in the same order on every rank whatever the host scheduler interleaves
  int world = 1, rank = 0;
  bool use_nccl = false;  // world > 1, or SVD1_FORCE_NCCL
  bool emulate = false;   // SVD1_EMULATE_RANKS: this process computes every rank's slices
  ncclComm_t comm[2] = {nullptr, nullptr};
  uint64_t probe_seed = 0x1707083691234567ull;
  std::atomic<int64_t> launches{0};
  DevBuf ctr;  // last-block counters for the test hooks (kept zero)
  DevBuf W_u, W_v, proj, partial, status, iters, ops, fmm_cells, fmm_descs, fmm_terms,
      fmm_tasks, scratch_i, scratch_d;
  DevBuf phi[2], psi[2];         // FMM expansions per side (U applies, V applies)
  DevBuf tile_ctr[2];            // per side: the GEMM passes' tile counters of one apply
  DevBuf upad[2];                // even-ld copy of an apply input TMA cannot read in place
  DevBuf probes;                 // 4 x u_rows sign probes
  bool probes_ready = false;
  cudaStream_t st2 = nullptr;    // V-side applies run here, concurrently with the U side
  cudaStream_t sp[4] = {};       // batch mode: spectral + carried-row streams (U, V side),
                                 // then upload streams for the FMM plans (U, V side)
  // svd1_update_batch: the projections of updates 1.. (project_many) run here while update
  // 0's spectral phase runs; proj_ev marks them (and their copies) done
  cudaStream_t st_proj = nullptr;
  cudaEvent_t proj_ev = nullptr;
  cudaEvent_t sync_ev[4] = {};
  StepRecord steps[4];
  // batch mode (svd1_update_batch): step records per update parity (the
  // next update's spectral phase runs while this one's applies are in flight), carried
  // projection rows (ping-pong per side), and the events marking each parity's applies done
  StepRecord bsteps[2][4];
  DevBuf RU[2], RV[2], few_scr[2], bproj, bgram;
  const double* batch_b = nullptr;  // svd1_update_batch's b's during the call (thin V)
  int64_t batch_ldb = 0;
  cudaEvent_t bdone[2][2] = {};  // [parity][side]
  bool bdone_rec[2] = {false, false};
  // batch mode: each side's remaining apply launches of the last update (its second apply
  // waits for its FMM plan) run on a launcher thread, so the next update's spectral chain
  // starts without waiting for them; joined before the side's next apply launch
  WorkThread launcher[2];
  svd1_status launcher_status[2] = {SVD1_OK, SVD1_OK};
  int launcher_parity[2] = {-1, -1};  // parity of the update whose launches they are
  cudaEvent_t rb_ev[2] = {};     // carried rows read back (U, V)
  cudaEvent_t maps_ev[2][4] = {};  // [parity] step e's column maps uploaded (spectral stream)
  cudaEvent_t bwin[2][4] = {};   // [parity]: apply start U, V; apply end U, V (timing)
  cudaEvent_t bspan[4] = {};     // the batch's first apply start U, V; last apply end U, V
  // SVD1_TIMELINE diagnostics (batch mode): labelled device events and host stamps
  std::vector<std::pair<std::string, cudaEvent_t>> tl_dev;
  std::vector<std::pair<std::string, double>> tl_host;
  double tl_t0 = 0.0;
  bool tl_on = false;
  bool tl_pre = false;  // the timeline was started by svd1_update_batch's projections
  double* h_pin = nullptr;  // pinned staging for read-backs
  size_t h_pin_cap = 0;
  // pinned upload arenas, one per side stream (U side: st, V side: st2): every
  // host->device upload is copied here first, so the DMA never reads pageable or
  // short-lived host memory; an arena is rewound only after its last copy (`ev`).
  // A ring: `used` is the next write offset; every copy out of the ring is a region with an
  // event, and a reservation waits only for the in-flight regions it would overwrite (the
  // oldest ones, from the previous lap), never for the copies just enqueued.
  struct Arena {
    struct Region {
      size_t lo, hi;
      cudaEvent_t ev;
    };
    char* buf = nullptr;
    size_t cap = 0, used = 0;
    cudaEvent_t ev = nullptr;    // (unused; kept for the create/destroy bookkeeping)
    bool pending = false;
    std::deque<Region> inflight;  // in allocation order
    std::vector<cudaEvent_t> pool;  // recycled events
  } arena[6];  // sides 0, 1: apply streams; 2, 3: batch spectral streams; 4, 5: uploads
  CauchyPrep standalone;    // plan of the standalone svd1_cauchy_apply
  std::vector<int32_t> rot_goff, rot_cols;  // pairing rotations of repeated sigma clusters
  std::vector<double> rot_mats;
  DevBuf d_rot_goff, d_rot_cols, d_rot_mats;
  cudaEvent_t ev[20] = {};  // timing events (spectral / apply phases)
};

namespace {

int64_t* LC(svd1_plan_t) { return &tl_launches; }
void flush_launches(svd1_plan_t P) {
  P->launches += tl_launches;
  tl_launches = 0;
}

svd1_status pinned(svd1_plan_t P, size_t doubles, double** out) {
  void* b = P->h_pin;
  TRY(pinned_reserve(&b, &P->h_pin_cap, doubles * sizeof(double)));  // sized at creation
  P->h_pin = static_cast<double*>(b);
  *out = P->h_pin;
  return SVD1_OK;
}

// counters for the last-block combines: one int per 64-column block, zeroed when the
// buffer is (re)allocated; the kernels leave them zero
svd1_status counters(DevBuf& b, int n, cudaStream_t st, int** out) {
  const void* before = b.p;
  const size_t cap0 = b.cap;
  TRY(b.get<int>(size_t(n / 64 + 16), out, st));
  if (b.p != before || b.cap != cap0) SVD1_CUDA_TRY(cudaMemsetAsync(b.p, 0, b.cap, st));
  return SVD1_OK;
}

svd1_status ensure_st2(svd1_plan_t P) {
  if (!P->st2) SVD1_CUDA_TRY(cudaStreamCreateWithFlags(&P->st2, cudaStreamNonBlocking));
  return SVD1_OK;
}
svd1_status ensure_side(svd1_plan_t P, int side) {
  if (side == 1) return ensure_st2(P);
  if (side >= 4 && !P->sp[side - 2]) {
    SVD1_CUDA_TRY(cudaStreamCreateWithFlags(&P->sp[side - 2], cudaStreamNonBlocking));
  } else if (side >= 2 && !P->sp[side - 2]) {
    // batch mode's spectral streams run at the highest priority: their short kernels
    // gate the next update, the applies they share the GPU with fill in behind them
    int lo = 0, hi = 0;
    SVD1_CUDA_TRY(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    static const bool flat = std::getenv("SVD1_FLAT_PRIORITY") != nullptr;  // experiments
    SVD1_CUDA_TRY(cudaStreamCreateWithPriority(&P->sp[side - 2], cudaStreamNonBlocking, flat ? lo : hi));
  }
  return SVD1_OK;
}
// side 0 (U) works on the plan stream, side 1 (V) on st2
// side 2 (U) and 3 (V): the batch mode's spectral streams
cudaStream_t side_stream(svd1_plan_t P, int side) {
  return side == 0 ? P->st : side == 1 ? P->st2 : P->sp[side - 2];
}

// Wait for the uploads in flight and rewind the arenas (called at API entry points).
svd1_status arena_reset(svd1_plan_t P, int side) {
  auto& A = P->arena[side];
  // the side's copies run in order on one stream: its newest region is the last to finish
  if (!A.inflight.empty()) SVD1_CUDA_TRY(cudaEventSynchronize(A.inflight.back().ev));
  for (auto& R : A.inflight) A.pool.push_back(R.ev);
  A.inflight.clear();
  A.pending = false;
  A.used = 0;
  return SVD1_OK;
}
svd1_status arena_reset(svd1_plan_t P) {
  for (int side = 0; side < 6; ++side) TRY(arena_reset(P, side));
  return SVD1_OK;
}

// reserve `bytes` of side's ring (growing it only if a single request exceeds it): offset.
// Waits for the in-flight copies that still read [off, off + bytes).
svd1_status arena_reserve(svd1_plan_t P, int side, size_t bytes, size_t* off_out) {
  auto& A = P->arena[side];
  if (bytes > A.cap) {  // sized at creation; an outgrown estimate reallocates (counted)
    TRY(arena_reset(P, side));
    void* b = A.buf;
    TRY(pinned_reserve(&b, &A.cap, std::max<size_t>(bytes * 2, size_t(4) << 20)));
    A.buf = static_cast<char*>(b);
  }
  size_t off = (A.used + 255) & ~size_t(255);
  if (off + bytes > A.cap) off = 0;  // wrap
  const size_t lo = off, hi = off + bytes;
  while (!A.inflight.empty()) {
    const auto& R = A.inflight.front();
    // regions are in allocation order: the front is the oldest; once it does not overlap
    // the new range the newer ones (beyond it in this lap, or behind the head) cannot either
    // -- except after a wrap, where every region of the previous lap above `lo` may overlap
    const bool overlap = R.lo < hi && lo < R.hi;
    if (!overlap) {
      // an older region entirely below lo (this lap) or above hi: check the rest only if it
      // could still overlap (previous-lap regions above lo)
      bool any = false;
      for (const auto& Q : A.inflight)
        if (Q.lo < hi && lo < Q.hi) {
          any = true;
          break;
        }
      if (!any) break;
    }
    SVD1_CUDA_TRY(cudaEventSynchronize(R.ev));
    A.pool.push_back(R.ev);
    A.inflight.pop_front();
  }
  *off_out = off;
  return SVD1_OK;
}

svd1_status arena_commit(svd1_plan_t P, int side, size_t off, size_t bytes, void* dev) {
  auto& A = P->arena[side];
  const cudaStream_t st = side_stream(P, side);
  SVD1_CUDA_TRY(cudaMemcpyAsync(dev, A.buf + off, bytes, cudaMemcpyHostToDevice, st));
  cudaEvent_t ev;
  if (!A.pool.empty()) {
    ev = A.pool.back();
    A.pool.pop_back();
  } else {
    SVD1_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  SVD1_CUDA_TRY(cudaEventRecord(ev, st));
  A.inflight.push_back({off, off + bytes, ev});
  A.pending = true;
  A.used = off + bytes;
  return SVD1_OK;
}

svd1_status arena_put(svd1_plan_t P, const void* src, size_t bytes, void* dev, int side = 0) {
  TRY(ensure_side(P, side));
  size_t off;
  TRY(arena_reserve(P, side, bytes, &off));
  std::memcpy(P->arena[side].buf + off, src, bytes);
  return arena_commit(P, side, off, bytes, dev);
}

// Several host arrays staged as ONE pinned-arena region and ONE host->device copy into
// a grow-only device blob (instead of one copy per array).
struct BlobBuilder {
  struct Part {
    const void* p;
    size_t bytes, off;
  };
  std::vector<Part> parts;
  size_t total = 0;
  template <class T>
  size_t add(const std::vector<T>& v) {
    const size_t off = (total + 255) & ~size_t(255);
    parts.push_back({v.data(), v.size() * sizeof(T), off});
    total = off + v.size() * sizeof(T);
    return off;
  }
};

svd1_status arena_put_blob(svd1_plan_t P, const BlobBuilder& B, DevBuf& dev, char** out, int side = 0) {
  TRY(ensure_side(P, side));
  TRY(dev.get<char>(std::max<size_t>(B.total, 1), out, side_stream(P, side)));
  if (B.total == 0) return SVD1_OK;
  size_t off;
  TRY(arena_reserve(P, side, B.total, &off));
  for (const auto& q : B.parts)
    if (q.bytes) std::memcpy(P->arena[side].buf + off + q.off, q.p, q.bytes);
  return arena_commit(P, side, off, B.total, *out);
}

svd1_status ev_record(svd1_plan_t P, int i, cudaStream_t st = nullptr) {
  if (!P->ev[i]) SVD1_CUDA_TRY(cudaEventCreate(&P->ev[i]));
  SVD1_CUDA_TRY(cudaEventRecord(P->ev[i], st ? st : P->st));
  return SVD1_OK;
}

// `waiter` waits for everything enqueued on `signaller` so far.
svd1_status stream_wait(svd1_plan_t P, int slot, cudaStream_t signaller, cudaStream_t waiter) {
  if (!P->sync_ev[slot])
    SVD1_CUDA_TRY(cudaEventCreateWithFlags(&P->sync_ev[slot], cudaEventDisableTiming));
  SVD1_CUDA_TRY(cudaEventRecord(P->sync_ev[slot], signaller));
  SVD1_CUDA_TRY(cudaStreamWaitEvent(waiter, P->sync_ev[slot], 0));
  return SVD1_OK;
}

// batch mode: record apply-window event q (0/1: start U/V, 2/3: end U/V) of a parity
svd1_status bwin_record(svd1_plan_t P, int par, int q, cudaStream_t st) {
  if (!P->bwin[par][q]) SVD1_CUDA_TRY(cudaEventCreate(&P->bwin[par][q]));
  SVD1_CUDA_TRY(cudaEventRecord(P->bwin[par][q], st));
  return SVD1_OK;
}
// first / last apply of a whole batch (q as for bwin)
svd1_status bspan_record(svd1_plan_t P, int q, cudaStream_t st) {
  if (!P->bspan[q]) SVD1_CUDA_TRY(cudaEventCreate(&P->bspan[q]));
  SVD1_CUDA_TRY(cudaEventRecord(P->bspan[q], st));
  return SVD1_OK;
}
double bspan_ms(svd1_plan_t P) {
  auto el = [&](int a, int b) {
    float ms = 0.f;
    if (!P->bspan[a] || !P->bspan[b] || cudaEventElapsedTime(&ms, P->bspan[a], P->bspan[b]) != cudaSuccess) {
      cudaGetLastError();
      return 0.0;
    }
    return double(ms);
  };
  return std::max(el(0, 2), el(0, 3)) - std::min(0.0, el(0, 1));
}

// first apply start -> last apply end of the update with that parity (after it completed)
double bwin_ms(svd1_plan_t P, int par) {
  auto el = [&](int a, int b) {
    float ms = 0.f;
    if (!P->bwin[par][a] || !P->bwin[par][b] ||
        cudaEventElapsedTime(&ms, P->bwin[par][a], P->bwin[par][b]) != cudaSuccess) {
      cudaGetLastError();
      return 0.0;
    }
    return double(ms);
  };
  return std::max(el(0, 2), el(0, 3)) - std::min(0.0, el(0, 1));
}

std::mutex g_tl_mutex;  // the timeline's vectors (both side threads mark)
void tl_mark(svd1_plan_t P, const std::string& label, cudaStream_t st, bool dev = true) {  // diagnostics
  if (!P->tl_on) return;
  std::lock_guard<std::mutex> lock(g_tl_mutex);
  P->tl_host.push_back({label, now_ms() - P->tl_t0});
  if (dev) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) == cudaSuccess) {
      cudaEventRecord(e, st);
      P->tl_dev.push_back({label, e});
    }
  }
}

double ev_ms(svd1_plan_t P, int a, int b) {
  float ms = 0.f;
  if (P->ev[a] && P->ev[b] && cudaEventElapsedTime(&ms, P->ev[a], P->ev[b]) == cudaSuccess) return ms;
  cudaGetLastError();
  return 0.0;
}

template <class T>
svd1_status upload(svd1_plan_t P, DevBuf& buf, const std::vector<T>& v, T** out, int side = 0) {
  TRY(ensure_side(P, side));
  TRY(buf.get<T>(v.size(), out, side_stream(P, side)));
  if (!v.empty()) TRY(arena_put(P, v.data(), v.size() * sizeof(T), *out, side));
  return SVD1_OK;
}

int choose_p(double eps) {
  // P:701 STEP 1: p = log5(1/eps); rounded up to a multiple of 4 (DMMA k-step), 4 <= p <= 32
  if (!(eps > 0.0 && eps < 1.0)) eps = 1e-10;
  int p = int(std::ceil(std::log(1.0 / eps) / std::log(5.0) - 1e-9));
  p = std::max(4, std::min(kMaxP, (p + 3) & ~3));
  return p;
}

// ------------------------------------------------------------------ FMM tree
// Binary tree of depth L over the active indices [0, na) (cells = index ranges;
// geometry = hull of the sources d_i and targets mu_j of the range).
// Splits are count-balanced (the tree of P:706 generalised to non-uniform spectra),
// except that a cell whose points have a gap of at least half its width is split
// at that gap when the capacities allow (isolated outlier
// eigenvalues, e.g. the large singular values a rank-1 update creates, would
// otherwise blow one leaf up to the whole spectrum).  Leaves hold <= s points.
// Interaction lists use the symmetric admissibility
//   |c_X - c_Y| >= max(3 r_X + r_Y, r_X + 3 r_Y)
// (the paper's |x0 - y0| > 4r at equal radii).
namespace {

// pts: the 2n merged points (sorted); is_src[q]; nsrc[q] = sources among pts[0, q).
struct Merged {
  std::vector<double> pts;
  std::vector<int32_t> nsrc;
};

Merged merge_points(const std::vector<double>& da, const std::vector<double>& mu) {
  // two sorted sequences -> one (ties: source first), O(n)
  const int n = int(da.size());
  Merged M;
  M.pts.resize(2 * n);
  M.nsrc.resize(2 * n + 1);
  M.nsrc[0] = 0;
  int i = 0, j = 0;
  for (int q = 0; q < 2 * n; ++q) {
    const bool take_src = j >= n || (i < n && da[i] <= mu[j]);
    M.pts[q] = take_src ? da[i++] : mu[j++];
    M.nsrc[q + 1] = M.nsrc[q] + (take_src ? 1 : 0);
  }
  return M;
}

bool fmm_cells(FmmHost& F, int s, int L, const Merged& M) {
  const int np = int(M.pts.size());
  const int64_t leafcap = 2 * int64_t(s);  // merged points per leaf (<= s+1 targets when interlaced)
  F.L = L;
  F.ncells = (1 << (L + 1)) - 1;
  F.cells.assign(F.ncells, FmmCell{0.0, 0.0, 0, 0, 0, 0, 0, 0});
  F.cells[0].lo = 0;
  F.cells[0].hi = np;
  const std::vector<double>& P = M.pts;
  for (int l = 0; l < L; ++l) {
    const int64_t cap = leafcap << (L - l - 1);  // capacity of each child
    for (int i = 0; i < (1 << l); ++i) {
      const int c = (1 << l) - 1 + i;
      const int lo = F.cells[c].lo, hi = F.cells[c].hi, nc = hi - lo;
      int t;
      if (nc <= 1) {
        t = hi;
      } else {
        const int tmin = int(std::max<int64_t>(lo + 1, hi - cap));
        const int tmax = int(std::min<int64_t>(hi - 1, lo + cap));
        if (tmin > tmax) return false;
        t = std::min(std::max(lo + nc / 2, tmin), tmax);
        const double width = P[hi - 1] - P[lo];
        double best = -1.0;
        int tb = t;
        for (int u = tmin; u <= tmax; ++u) {
          const double g = P[u] - P[u - 1];
          if (g > best) {
            best = g;
            tb = u;
          }
        }
        if (best >= 0.5 * width) t = tb;  // split isolated points off at a dominant gap
      }
      F.cells[2 * c + 1].lo = lo;
      F.cells[2 * c + 1].hi = t;
      F.cells[2 * c + 2].lo = t;
      F.cells[2 * c + 2].hi = hi;
    }
  }
  for (int i = 0; i < (1 << L); ++i) {
    const FmmCell& C = F.cells[(1 << L) - 1 + i];
    if (C.hi - C.lo > leafcap) return false;
  }
  for (int c = 0; c < F.ncells; ++c) {
    FmmCell& C = F.cells[c];
    C.slo = M.nsrc[C.lo];
    C.shi = M.nsrc[C.hi];
    C.tlo = C.lo - C.slo;
    C.thi = C.hi - C.shi;
    if (C.hi <= C.lo) continue;
    const double a = P[C.lo], b = P[C.hi - 1];
    C.c = 0.5 * (a + b);
    double r = std::max(C.c - a, b - C.c);
    C.r = std::max(r, std::max(std::fabs(C.c) * 0x1.0p-50, 1e-300));
  }
  return true;
}

// ---- secular FMM plan: tree over the oriented sources d (ascending),
// target interval of a cell = [d_lo, d_next] (the brackets of its roots), dual traversal
// with the symmetric admissibility of the apply's tree; far partners -> M2L (P2L when
// the partner holds fewer than kSecP sources) into the left or right expansion, leaf
// pairs -> near ranges evaluated directly by each root.
void secfmm_plan(const double* d, int n, SecPlanHost& S) {
  Merged M;
  M.pts.assign(d, d + n);
  M.nsrc.resize(n + 1);
  for (int q = 0; q <= n; ++q) M.nsrc[q] = q;
  const int s = 16;  // leaves of <= 2 s = 32 sources
  int L0 = 0;
  while ((int64_t(n) + (int64_t(1) << L0) - 1) / (int64_t(1) << L0) > 2 * s) ++L0;
  FmmHost F;
  for (int L = L0; L <= L0 + 2; ++L) {
    FmmHost F2;
    if (!fmm_cells(F2, s, L, M)) continue;
    double rmax = 0.0;
    for (int i = 0; i < (1 << L); ++i) rmax = std::max(rmax, F2.cells[(1 << L) - 1 + i].r);
    F = std::move(F2);
    if (!(rmax >= 0.25 * F.cells[0].r && F.cells[0].r > 0.0)) break;  // no outlier-wide leaf
  }
  const int L = F.L, nc = F.ncells;
  S.L = L;
  S.ncells = nc;
  S.cells.assign(nc + 1, SecFmmCell{0, 0, 0, 0, 0.0, 0.0, 0.0, 0.0});
  // Target intervals bottom-up.  A leaf's is [d_lo, d_hi] (the brackets of its roots)
  // unless the gap to the next leaf is wider than its own hull (an outlier gap): then it
  // is the hull [d_lo, d_{hi-1}] and the one root bracketed by the gap sums directly
  // (pad = 1), so no leaf is near-field to a whole side of the spectrum.  A parent's
  // interval is the hull of its children's, so every expansion contains its descendants'.
  std::vector<double> tlo(nc, 0.0), thi(nc, -1.0);
  const int first_leaf0 = (1 << L) - 1;
  for (int c = nc - 1; c >= 0; --c) {
    const FmmCell& C = F.cells[c];
    SecFmmCell& X = S.cells[c];
    X.lo = C.lo;
    X.hi = C.hi;
    X.c = C.c;
    X.r = C.r;
    X.pad = 0;
    if (C.hi <= C.lo) continue;
    if (c >= first_leaf0) {
      const double a = d[C.lo], h = d[C.hi - 1], b = d[std::min(C.hi, n - 1)];
      tlo[c] = a;
      thi[c] = b;
      if (C.hi < n && b - h > h - a) {
        thi[c] = h;
        X.pad = 1;
      }
    } else {
      bool any = false;
      for (int ch = 2 * c + 1; ch <= 2 * c + 2; ++ch) {
        if (thi[ch] < tlo[ch]) continue;
        tlo[c] = any ? std::min(tlo[c], tlo[ch]) : tlo[ch];
        thi[c] = any ? std::max(thi[c], thi[ch]) : thi[ch];
        any = true;
      }
    }
    X.ct = 0.5 * (tlo[c] + thi[c]);
    X.rt = std::max(std::max(X.ct - tlo[c], thi[c] - X.ct), std::max(std::fabs(X.ct) * 0x1.0p-50, 1e-300));
  }
  auto has_src = [&](int c) { return S.cells[c].hi > S.cells[c].lo; };
  auto has_tgt = [&](int c) { return S.cells[c].hi > S.cells[c].lo && S.cells[c].lo <= n - 2; };
  auto adm = [&](int x, int y) {
    const SecFmmCell &X = S.cells[x], &Y = S.cells[y];
    return std::fabs(X.c - Y.ct) >= std::max(3.0 * X.r + Y.rt, X.r + 3.0 * Y.rt);
  };
  const int first_leaf = (1 << L) - 1;
  auto is_leaf = [&](int c) { return c >= first_leaf; };
  std::vector<std::pair<int, int>> m2l_pairs, near_pairs, p2l_pairs;
  // one-sided separation of near leaves (as the apply's, §4.4): X's sources far enough from
  // the target interval of Y for Y's local expansion -> P2L instead of the direct sum
  static const bool one_sided = [] {
    const char* e = std::getenv("SVD1_ONE_SIDED");
    return !(e && atoi(e) == 0);
  }();
  std::vector<std::pair<int, int>> stack{{0, 0}};
  while (!stack.empty()) {
    const auto [x, y] = stack.back();
    stack.pop_back();
    if (!has_src(x) || !has_tgt(y)) continue;
    if (x != y && adm(x, y)) {
      m2l_pairs.push_back({y, x});
      continue;
    }
    if (is_leaf(x) && is_leaf(y)) {
      const SecFmmCell &X = S.cells[x], &Y = S.cells[y];
      if (one_sided && x != y && std::fabs(X.c - Y.ct) - X.r >= 3.0 * Y.rt) p2l_pairs.push_back({y, x});
      else near_pairs.push_back({y, x});
      continue;
    }
    const bool split_x = is_leaf(y) || (!is_leaf(x) && S.cells[x].r > S.cells[y].rt);
    if (split_x) {
      stack.push_back({2 * x + 2, y});
      stack.push_back({2 * x + 1, y});
    } else {
      stack.push_back({x, 2 * y + 2});
      stack.push_back({x, 2 * y + 1});
    }
  }
  // group the pairs by target cell with a counting sort (partners ascending per cell)
  auto group = [nc](std::vector<std::pair<int, int>>& pairs, std::vector<int>& off, std::vector<int>& val) {
    off.assign(nc + 1, 0);
    for (const auto& pr : pairs) ++off[pr.first + 1];
    for (int c = 0; c < nc; ++c) off[c + 1] += off[c];
    val.resize(pairs.size());
    std::vector<int> fill(off.begin(), off.end() - 1);
    for (const auto& pr : pairs) val[fill[pr.first]++] = pr.second;
    for (int c = 0; c < nc; ++c)
      if (off[c + 1] - off[c] > 1) std::sort(val.begin() + off[c], val.begin() + off[c + 1]);
  };
  std::vector<int> m_off, m_val, o_off, o_val;
  group(m2l_pairs, m_off, m_val);
  group(p2l_pairs, o_off, o_val);
  S.parts.clear();
  S.parts.reserve(m_val.size() + o_val.size());
  for (int c = 0; c < nc; ++c) {
    S.cells[c].m2l_off = int32_t(S.parts.size());
    for (int q = m_off[c]; q < m_off[c + 1]; ++q) {
      const int x = m_val[q];
      const SecFmmCell& X = S.cells[x];
      int32_t fl = X.c > S.cells[c].ct ? 1 : 0;
      if (X.hi - X.lo < kSecP) fl |= 2;
      S.parts.push_back(SecFmmPart{x, fl});
    }
    for (int q = o_off[c]; q < o_off[c + 1]; ++q) {  // one-sided: always from the sources
      const int x = o_val[q];
      S.parts.push_back(SecFmmPart{x, int32_t((S.cells[x].c > S.cells[c].ct ? 1 : 0) | 2)});
    }
  }
  S.cells[nc].m2l_off = int32_t(S.parts.size());
  // leaves (non-empty, in index order) and their near source ranges
  S.leaf_lo.clear();
  S.leaf_cell.clear();
  std::vector<int> leaf_of_cell(nc, -1);
  for (int i = 0; i < (1 << L); ++i) {
    const int c = first_leaf + i;
    if (!has_src(c)) continue;
    leaf_of_cell[c] = int(S.leaf_cell.size());
    S.leaf_lo.push_back(S.cells[c].lo);
    S.leaf_cell.push_back(c);
  }
  S.nleaf = int(S.leaf_cell.size());
  S.leaf_lo.push_back(n);
  S.direct.clear();
  for (int q = 0; q < S.nleaf; ++q)
    if (S.cells[S.leaf_cell[q]].pad) S.direct.push_back(S.leaf_lo[q + 1] - 1);
  S.direct.push_back(n - 1);
  std::vector<int> n_off, n_val;
  group(near_pairs, n_off, n_val);
  S.near_off.assign(S.nleaf + 1, 0);
  S.near_lo.clear();
  S.near_hi.clear();
  for (int lf = 0; lf < S.nleaf; ++lf) {
    const int c = S.leaf_cell[lf];
    S.near_off[lf] = int32_t(S.near_lo.size());
    for (int q = n_off[c]; q < n_off[c + 1]; ++q) {
      const SecFmmCell& X = S.cells[n_val[q]];
      if (S.near_off[lf] < int32_t(S.near_lo.size()) && S.near_hi.back() == X.lo)
        S.near_hi.back() = X.hi;  // merge adjacent ranges
      else {
        S.near_lo.push_back(X.lo);
        S.near_hi.push_back(X.hi);
      }
    }
  }
  S.near_off[S.nleaf] = int32_t(S.near_lo.size());
  if (std::getenv("SVD1_DEBUG")) {
    int64_t tot = 0, mx = 0;
    for (int lf = 0; lf < S.nleaf; ++lf) {
      int64_t k = 0;
      for (int g = S.near_off[lf]; g < S.near_off[lf + 1]; ++g) k += S.near_hi[g] - S.near_lo[g];
      tot += k * (S.leaf_lo[lf + 1] - S.leaf_lo[lf]);
      mx = std::max(mx, k);
    }
    fprintf(stderr, "[svd1] secfmm n=%d L=%d cells=%d leaves=%d m2l parts=%zu near terms/root mean %.1f max %lld\n",
            n, L, nc, S.nleaf, S.parts.size(), double(tot) / n, (long long)mx);
  }
}

// sorted CSR of (row, value) pairs: row r's values in [off[r], off[r+1])
struct Csr {
  std::vector<int> off, val;
  struct Row {
    const int* b;
    const int* e;
    const int* begin() const { return b; }
    const int* end() const { return e; }
    size_t size() const { return size_t(e - b); }
    bool empty() const { return b == e; }
    int operator[](size_t i) const { return b[i]; }
  };
  Csr(std::vector<std::pair<int, int>>& pairs, int rows) : off(rows + 1, 0) {
    std::sort(pairs.begin(), pairs.end());
    val.resize(pairs.size());
    for (size_t q = 0; q < pairs.size(); ++q) {
      ++off[pairs[q].first + 1];
      val[q] = pairs[q].second;
    }
    for (int r = 0; r < rows; ++r) off[r + 1] += off[r];
  }
  Row operator[](int r) const { return Row{val.data() + off[r], val.data() + off[r + 1]}; }
};

void fmm_lists(FmmHost& F, int p, const int32_t* src, int64_t rows) {
  const double tt0 = now_ms();
  const int L = F.L;
  auto has_src = [&](int c) { return F.cells[c].shi > F.cells[c].slo; };
  auto has_tgt = [&](int c) { return F.cells[c].thi > F.cells[c].tlo; };
  auto adm = [&](int x, int y) {
    const FmmCell &X = F.cells[x], &Y = F.cells[y];
    return std::fabs(X.c - Y.c) >= std::max(3.0 * X.r + Y.r, X.r + 3.0 * Y.r);
  };
  // Dual-tree traversal (cells of different levels may interact): a pair is
  // admissible -> M2L into the target cell; two leaves -> near field (P2P);
  // otherwise split the larger cell.  Needed for graded spectra, where a wide
  // target cell only separates from the narrow sources below it at a finer level.
  // interaction lists as CSR (target cell -> sorted partner cells), built from the
  // traversal's pairs with one sort (no per-cell allocations)
  std::vector<std::pair<int, int>> near_pairs, m2l_pairs, p2l_pairs, m2p_pairs;
  // one-sided separation of near leaves (SVD1_ONE_SIDED=0 disables; experiments)
  static const bool one_sided = [] {
    const char* e = std::getenv("SVD1_ONE_SIDED");
    return !(e && atoi(e) == 0);
  }();
  // measured pass rates (TFLOP/s, ncu, C3: profiles/ncu_full_r02_gemm.md) weighing the choice
  static const double kRate16 = std::getenv("SVD1_RATE16") ? atof(std::getenv("SVD1_RATE16")) : 18.0;
  constexpr double kRate32 = 24.5;
  near_pairs.reserve(size_t(F.ncells) * 4);
  m2l_pairs.reserve(size_t(F.ncells) * 4);
  const int first_leaf = (1 << L) - 1;
  auto is_leaf = [&](int c) { return c >= first_leaf; };
  std::vector<std::pair<int, int>> stack;
  stack.push_back({0, 0});
  while (!stack.empty()) {
    const auto [x, y] = stack.back();
    stack.pop_back();
    if (!has_src(x) || !has_tgt(y)) continue;
    if (x != y && adm(x, y)) {
      m2l_pairs.push_back({y, x});
      continue;
    }
    if (is_leaf(x) && is_leaf(y)) {
      // Two leaves that fail the symmetric test may still be separated on one side (the
      // adaptive FMM's X and W lists): X's sources far from Y's box -> P2L into Y's local
      // expansion (Y's Chebyshev interpolant converges as for M2L); Y's targets far from
      // X's box -> M2P, X's far field evaluated at Y's targets.  Each is taken when its
      // estimated time beats the near-field product's (flops over the measured rate of the
      // pass it lands in: the 16-wide M2L pass, the 32-wide final pass).
      if (x != y && one_sided) {
        const FmmCell &X = F.cells[x], &Y = F.cells[y];
        const double D = std::fabs(X.c - Y.c);
        const double ns = X.shi - X.slo, nt = Y.thi - Y.tlo;
        double best = ns * nt / kRate32;  // P2P
        int kind = 0;
        if (D - X.r >= 3.0 * Y.r && ns * p / kRate16 < best) {
          best = ns * p / kRate16;
          kind = 1;
        }
        if (D - Y.r >= 3.0 * X.r && double(p) * nt / kRate32 < best) kind = 2;
        if (kind == 1) {
          p2l_pairs.push_back({y, x});
          continue;
        }
        if (kind == 2) {
          m2p_pairs.push_back({y, x});
          continue;
        }
      }
      near_pairs.push_back({y, x});
      continue;
    }
    const bool split_x = is_leaf(y) || (!is_leaf(x) && F.cells[x].r > F.cells[y].r);
    if (split_x) {
      stack.push_back({2 * x + 2, y});
      stack.push_back({2 * x + 1, y});
    } else {
      stack.push_back({x, 2 * y + 2});
      stack.push_back({x, 2 * y + 1});
    }
  }
  const Csr near(near_pairs, F.ncells), m2l(m2l_pairs, F.ncells), p2l(p2l_pairs, F.ncells),
      m2p(m2p_pairs, F.ncells);
  auto has_local = [&](int y) { return !m2l[y].empty() || !p2l[y].empty(); };  // Psi_y non-zero
  // Fused P2L (SVD1_P2L_FUSED=1; experiments, off): the P2L pairs computed in the P2M
  // pass, which reads the same source windows of U, each into a slot of its own past the
  // cells' columns of Phi, and the M2L pass adding a target's slots with identity operators
  // (2 p^2 per pair instead of re-reading the sources from DRAM).  Needs room for the slots
  // in the plan's expansion workspace.  Measured at C3: P2M 39 -> 52 us, M2L 98 -> 93 us,
  // the stream 444-454 -> 442-448 updates/s, hence off.
  static const bool p2l_fuse_env = [] {
    const char* e = std::getenv("SVD1_P2L_FUSED");
    return e && atoi(e) != 0;
  }();
  const int npl = int(p2l.val.size());
  const bool p2l_fused = p2l_fuse_env && npl > 0 && int64_t(F.ncells) + npl <= F.cap_cells;
  F.ecells = F.ncells + (p2l_fused ? npl : 0);
  std::vector<std::vector<std::pair<int, int>>> p2l_by_src;  // x -> (target y, slot)
  if (p2l_fused) {
    p2l_by_src.resize(F.ncells);
    for (int y = 0; y < F.ncells; ++y)
      for (int q = p2l.off[y]; q < p2l.off[y + 1]; ++q) p2l_by_src[p2l.val[q]].push_back({y, F.ncells + q});
  }
  const double tt1 = now_ms();
  // A term's op (K x N) is stored chunk-transposed (FmmTerm): new_term reserves its
  // ceil(K/16) chunks of [npad][16] doubles; add_op adds a block of its rows.
  // kreal: rows that carry work (window rows of absent sources are zero): flop count
  auto new_term = [&](int in_kind, int col0, int K, int N, int kreal) {
    FmmTerm t;
    t.in_kind = in_kind;
    t.col0 = col0;
    t.K = K;
    t.npad = (N + 15) & ~15;
    t.op_row = F.ops_rows;
    F.ops_rows += int64_t((K + 15) / 16) * t.npad;
    F.terms.push_back(t);
    F.flops_exec_per_row += 2ll * kreal * N;
  };
  auto add_op = [&](int kind, int a, int b, int rows, int cols, int kb, int nb = 0) {
    const FmmTerm& t = F.terms.back();
    FmmOpDesc D;
    D.kind = kind;
    D.a = a;
    D.b = b;
    D.rows = rows;
    D.cols = cols;
    D.kb = kb;
    D.nb = nb;
    D.npad = t.npad;
    D.op_row = t.op_row;
    D.c0 = 0;
    D.s_hi = 0;
    F.ops.push_back(D);
  };
  int64_t adj = 0;  // level-by-level M2M / L2L flops minus the banded ones
  int64_t zero_flops = 0;  // executed, not algorithmic: sibling-pair zero blocks, fused-P2L accumulation
  // sources [s_lo, s_hi) (a contiguous range of the sorted active sources) read through
  // their physical input columns src[s]: windows of nearby columns (gaps <= 8 are
  // bridged by zero op rows), each starting at an even column
  std::vector<int> pc;
  // (b2 >= 0: a task over the sibling pair (b, b2) -- b's block in op columns 0..N/2-1,
  // b2's in N/2..N-1; a negative b targets only the second half)
  auto add_src = [&](int kind, int s_lo, int s_hi, int b, int N, int b2 = -1) {
    pc.resize(s_hi - s_lo);
    bool up = true, down = true;  // monotone maps (identity, reversal) need no sort
    for (int s2 = s_lo; s2 < s_hi; ++s2) {
      pc[s2 - s_lo] = src ? src[s2] : s2;
      if (s2 > s_lo) {
        up = up && pc[s2 - s_lo] > pc[s2 - s_lo - 1];
        down = down && pc[s2 - s_lo] < pc[s2 - s_lo - 1];
      }
    }
    if (down) std::reverse(pc.begin(), pc.end());
    else if (!up) std::sort(pc.begin(), pc.end());
    size_t a = 0;
    while (a < pc.size()) {
      size_t e = a;
      while (e + 1 < pc.size() && pc[e + 1] - pc[e] <= 8) ++e;
      // TMA needs 16-byte aligned box starts: windows start at an even column (a
      // column in front of the term's sources gets a zero op row)
      const int c0 = pc[a] & ~1, len = pc[e] + 1 - c0;
      new_term(IO_U, c0, len, N, int(e - a + 1));
      if (b2 == -1) {
        add_op(kind, s_lo, b, len, N, 0);
        F.ops.back().c0 = c0;
        F.ops.back().s_hi = s_hi;
      } else {
        const int half = N / 2;
        if (b >= 0) {
          add_op(kind, s_lo, b, len, half, 0, 0);
          F.ops.back().c0 = c0;
          F.ops.back().s_hi = s_hi;
        }
        if (b2 >= 0) {
          add_op(kind, s_lo, b2, len, half, 0, half);
          F.ops.back().c0 = c0;
          F.ops.back().s_hi = s_hi;
        }
        if (b < 0 || b2 < 0) zero_flops += 2ll * (e - a + 1) * half;
      }
      a = e + 1;
    }
  };
  int tb = 0;
  auto begin_task = [&]() { tb = int(F.terms.size()); };
  // tasks wider than 32 columns are split along N (they share their terms)
  auto end_task = [&](int out_kind, int col0, int N) {
    for (int c0 = 0; c0 < N; c0 += 32) {
      FmmTask T;
      T.out_kind = out_kind;
      T.col0 = col0 + c0;
      T.N = std::min(32, N - c0);
      T.t_begin = tb;
      T.t_end = int(F.terms.size());
      T.op_col0 = c0;
      F.tasks.push_back(T);
    }
  };
  // consecutive partners -> one term over adjacent columns of U (sources) or Phi
  auto add_runs = [&](const auto& xs, int in_kind, int op_kind, int y, int N) {
    size_t a = 0;
    while (a < xs.size()) {
      size_t b = a;
      if (in_kind == IO_U) {
        while (b + 1 < xs.size() && F.cells[xs[b + 1]].slo == F.cells[xs[b]].shi) ++b;
        add_src(op_kind, F.cells[xs[a]].slo, F.cells[xs[b]].shi, y, N);
        a = b + 1;
        continue;
      }
      while (b + 1 < xs.size() && xs[b + 1] == xs[b] + 1) ++b;
      const int K = int(b - a + 1) * p;
      new_term(in_kind, xs[a] * p, K, N, K);
      for (size_t q = a; q <= b; ++q) add_op(op_kind, xs[q], y, p, N, int(q - a) * p);
      a = b + 1;
    }
  };
  // longest tasks first inside each pass (persistent CTAs take tiles in this order)
  std::vector<std::pair<int64_t, int>> order;
  std::vector<FmmTask> tmp;
  auto sort_pass = [&](int b) {
    const int e = int(F.tasks.size());
    order.clear();
    for (int q = b; q < e; ++q) {
      int64_t k = 0;
      for (int t = F.tasks[q].t_begin; t < F.tasks[q].t_end; ++t) k += F.terms[t].K;
      order.push_back({-k, q});
    }
    std::sort(order.begin(), order.end());  // (cost desc, index asc): stable
    tmp.assign(F.tasks.begin() + b, F.tasks.end());
    for (int q = b; q < e; ++q) F.tasks[q] = tmp[order[q - b].second - b];
  };
  F.ops.reserve(size_t(F.ncells) * 8);
  F.terms.reserve(size_t(F.ncells) * 6);
  F.tasks.reserve(size_t(F.ncells) * 3);
  const int lf0 = (1 << L) - 1, nleaf = 1 << L;
  // Levels are grouped into bands computed by ONE pass each (a launch costs about
  // launch_row flops per row of work): a level joins the current band when the extra
  // flops of reaching back to the band's input level stay below that.
  const double launch_row = 2.0e8 / double(std::max<int64_t>(rows, 1));
  auto first_desc = [](int c, int depth) { return ((c + 1) << depth) - 1; };
  // where the full local expansion of a cell lives (IO_PSI: its M2L part alone, IO_PHI:
  // accumulated with its ancestors' by a band pass; -1: none)
  std::vector<int> loc(F.ncells, -1);
  if (L >= 1) {
    // P2M (STEP 5) in the scaled far-field form
    F.pass_begin.push_back(int(F.tasks.size()));
    F.pass_bn.push_back(p);
    F.pass_kind.push_back(0);
    for (int i = 0; i < nleaf; ++i) {
      const int x = lf0 + i;
      if (!has_src(x)) continue;
      begin_task();
      add_src(OP_P2M, F.cells[x].slo, F.cells[x].shi, x, p);
      end_task(IO_PHI, x * p, p);
      if (p2l_fused)
        for (const auto& [y, slot] : p2l_by_src[x]) {  // fused P2L: same window, next task
          begin_task();
          add_src(OP_P2L, F.cells[x].slo, F.cells[x].shi, y, p);
          end_task(IO_PHI, slot * p, p);
        }
    }
    sort_pass(F.pass_begin.back());
    // M2M (STEP 6; operator re-derived), levels L-1 .. 1 in
    // bands: every level of a band reads the band's input level f directly (the M2M
    // operator of any descendant D -> ancestor c has the same closed form).
    std::vector<int> ds;
    int f = L;
    while (f - 1 >= 1) {
      int lo = f - 1;
      while (lo - 1 >= 1) {
        const int l2 = lo - 1;
        double extra = 0.0;  // flops per row beyond the level-by-level M2M
        for (int i = 0; i < (1 << l2); ++i) {
          const int c = (1 << l2) - 1 + i;
          if (!has_src(c)) continue;
          const int d0 = first_desc(c, f - l2);
          int nd = 0;
          for (int q = 0; q < (1 << (f - l2)); ++q) nd += has_src(d0 + q);
          int nch = has_src(2 * c + 1) + has_src(2 * c + 2);
          extra += 2.0 * double(nd - nch) * p * p;
        }
        if (extra > launch_row) break;
        lo = l2;
      }
      F.pass_begin.push_back(int(F.tasks.size()));
      F.pass_bn.push_back(p);
      F.pass_kind.push_back(1);
      for (int l = f - 1; l >= lo; --l)
        for (int i = 0; i < (1 << l); ++i) {
          const int c = (1 << l) - 1 + i;
          if (!has_src(c)) continue;
          ds.clear();
          const int d0 = first_desc(c, f - l);
          for (int q = 0; q < (1 << (f - l)); ++q)
            if (has_src(d0 + q)) ds.push_back(d0 + q);
          adj += 2ll * p * p * (has_src(2 * c + 1) + has_src(2 * c + 2) - int(ds.size()));
          begin_task();
          add_runs(ds, IO_PHI, OP_M2M, c, p);
          end_task(IO_PHI, c * p, p);
        }
      sort_pass(F.pass_begin.back());
      f = lo;
    }
    // downward (STEP 8; M2L re-derived), restructured:
    // (a) one pass with the M2L (and P2L) contributions of EVERY cell, all levels at
    //     once (no dependence between them), into Psi;
    // (b) L2L for levels 2..L-1 in bands: the full local expansion of a band cell Y is
    //     sum over its ancestors A in the band (A = Y included) of Psi_A S(A -> Y), plus
    //     full(anchor) S(anchor -> Y) for its ancestor at the level above the band;
    //     exact, since the local expansion is a polynomial and L2L re-interpolates it.
    //     Full expansions are stored in Phi (dead after the M2L pass);
    // (c) leaves take L2L from their parent folded into the final pass (evaluating
    //     the parent's local polynomial at the targets is exactly L2L then L2P).
    // Sibling pairs (SVD1_PAIRS: bit 0 the M2L pass, bit 1 the L2L bands; experiments,
    // off by default): the siblings (2P+1, 2P+2) run as ONE 2p-wide task over the union
    // of their inputs (each input's op holds a block per sibling it serves, zero
    // otherwise), so each input window is read once for both.  Measured at C3 (DESIGN.md
    // §4.4): the M2L pass 85 -> 120-190 us (the traversal's partner lists of siblings
    // overlap little: the union's zero blocks cost more than the halved A reads save),
    // the L2L bands about even; the stream 430 -> 405 (both) / 424 (L2L only).
    static const int pair_mask = std::getenv("SVD1_PAIRS") ? atoi(std::getenv("SVD1_PAIRS")) : 0;
    bool pairs = 2 * p <= 32 && (pair_mask & 1);
    auto pair_of = [&](int y) {  // the right sibling when y is a left child that pairs
      return (pairs && (y & 1) && y + 1 < F.ncells) ? y + 1 : -1;
    };
    F.pass_begin.push_back(int(F.tasks.size()));
    F.pass_bn.push_back(pairs ? 2 * p : p);
    F.pass_kind.push_back(2);
    std::vector<int> via_phi, via_src;
    std::vector<std::pair<int, int>> uni;  // (partner, 1: of y | 2: of y2)
    std::vector<int> xs;
    for (int y = 1; y < F.ncells; ++y) {
      if (!has_local(y) || !has_tgt(y)) continue;
      const int y2 = pair_of(y);
      if (y2 > 0 && has_tgt(y2) && !m2l[y2].empty() && p2l[y].empty() && p2l[y2].empty() && !m2l[y].empty()) {
        uni.clear();
        size_t i1 = 0, i2 = 0;
        const auto A1 = m2l[y], A2 = m2l[y2];
        while (i1 < A1.size() || i2 < A2.size()) {
          if (i2 == A2.size() || (i1 < A1.size() && A1[i1] < A2[i2])) uni.push_back({A1[i1++], 1});
          else if (i1 == A1.size() || A2[i2] < A1[i1]) uni.push_back({A2[i2++], 2});
          else {
            uni.push_back({A1[i1], 3});
            ++i1;
            ++i2;
          }
        }
        begin_task();
        for (int pass_src = 0; pass_src < 2; ++pass_src) {
          size_t a = 0;
          while (a < uni.size()) {
            const int x = uni[a].first;
            const bool src_kind = F.cells[x].shi - F.cells[x].slo < p;
            if (src_kind != (pass_src == 1)) {
              ++a;
              continue;
            }
            if (src_kind) {  // P2L: one source window per partner, blocks for its targets
              const int m = uni[a].second;
              add_src(OP_P2L, F.cells[x].slo, F.cells[x].shi, (m & 1) ? y : -2, 2 * p, (m & 2) ? y2 : -2);
              ++a;
              continue;
            }
            // M2L: consecutive partner cells -> one long-K term over adjacent Phi columns
            size_t b = a;
            while (b + 1 < uni.size() && uni[b + 1].first == uni[b].first + 1 &&
                   F.cells[uni[b + 1].first].shi - F.cells[uni[b + 1].first].slo >= p)
              ++b;
            const int K = int(b - a + 1) * p;
            new_term(IO_PHI, x * p, K, 2 * p, K);
            for (size_t q = a; q <= b; ++q) {
              const int m = uni[q].second;
              if (m & 1) add_op(OP_M2L, uni[q].first, y, p, p, int(q - a) * p, 0);
              if (m & 2) add_op(OP_M2L, uni[q].first, y2, p, p, int(q - a) * p, p);
              if (m != 3) zero_flops += 2ll * p * p;
            }
            a = b + 1;
          }
        }
        F.n_m2l_pairs += int(m2l[y].size() + m2l[y2].size());
        end_task(IO_PSI, y * p, 2 * p);
        ++y;  // y2 done
        continue;
      }
      begin_task();
      // partners with fewer than p sources are cheaper as P2L (K = #sources < p)
      via_phi.clear();
      via_src.clear();
      for (int x : m2l[y]) (F.cells[x].shi - F.cells[x].slo >= p ? via_phi : via_src).push_back(x);
      add_runs(via_phi, IO_PHI, OP_M2L, y, p);
      add_runs(via_src, IO_U, OP_P2L, y, p);
      if (p2l_fused) {  // one-sided: the slots the P2M pass filled, by identity operators
        if (!p2l[y].empty()) {
          const int cnt = int(p2l[y].size()), c0 = F.ncells + p2l.off[y];
          new_term(IO_PHI, c0 * p, cnt * p, p, cnt * p);
          for (int q = 0; q < cnt; ++q) add_op(OP_ID, y, y, p, p, q * p);
          zero_flops += 2ll * cnt * p * p;  // accumulation, not algorithmic work
        }
      } else {  // one-sided: sources straight into Psi_y
        xs.assign(p2l[y].begin(), p2l[y].end());
        add_runs(xs, IO_U, OP_P2L, y, p);
      }
      F.n_m2l_pairs += int(m2l[y].size() + p2l[y].size());
      end_task(IO_PSI, y * p, p);
    }
    sort_pass(F.pass_begin.back());
    for (int i = 0; i < 2 && i < (1 << L); ++i) {
      const int y = 1 + i;  // level 1: full = the M2L part
      if (L >= 1 && has_tgt(y) && has_local(y)) loc[y] = IO_PSI;
    }
    pairs = 2 * p <= 32 && (pair_mask & 2);
    int a = 1;  // anchor level: full expansions known
    while (a + 1 <= L - 1) {
      int hi = a + 1;
      while (hi + 1 <= L - 1) {
        double extra = 0.0;  // ancestors beyond the parent, per target cell of level hi+1
        const int l2 = hi + 1;
        for (int i = 0; i < (1 << l2); ++i) {
          const int y = (1 << l2) - 1 + i;
          if (!has_tgt(y)) continue;
          int na2 = 0;
          for (int A = (y - 1) / 2, l3 = l2 - 1; l3 >= a + 1; A = (A - 1) / 2, --l3) na2 += !m2l[A].empty();
          extra += 2.0 * double(std::max(na2 - 1, 0)) * p * p;
        }
        if (extra > launch_row) break;
        hi = l2;
      }
      const int pb = int(F.tasks.size());
      // (cell, input) pairs of y: Psi of the band ancestors with an M2L part, then the
      // anchor's full expansion; adj: level by level, Psi_y = Psi_y I + full(parent) S
      // when the parent has one, minus the band's terms
      auto chain = [&](int y, int l, int* Acell, int* Akind) {
        int nA = 0, A = y;
        for (int l3 = l; l3 >= a + 1; --l3, A = (A - 1) / 2)
          if (!m2l[A].empty()) {
            Acell[nA] = A;
            Akind[nA++] = IO_PSI;
          }
        if (loc[A] >= 0) {  // A is now the ancestor at the anchor level a
          Acell[nA] = A;
          Akind[nA++] = loc[A];
        }
        const int par = (y - 1) / 2;
        if (loc[par] >= 0) adj += 2ll * p * p * ((m2l[y].empty() ? 0 : 1) + 1);
        if (!(nA == 0 || (nA == 1 && Acell[0] == y))) adj -= 2ll * p * p * nA;
        return nA;
      };
      for (int l = a + 1; l <= hi; ++l)
        for (int i = 0; i < (1 << l); ++i) {
          const int y = (1 << l) - 1 + i;
          if (!has_tgt(y)) continue;
          int Acell[32], Akind[32];
          const int nA = chain(y, l, Acell, Akind);
          if (nA == 0 || (nA == 1 && Acell[0] == y)) {  // nothing to accumulate
            loc[y] = nA ? IO_PSI : -1;
            continue;
          }
          const int y2 = pair_of(y);
          if (y2 > 0 && has_tgt(y2)) {
            // sibling pair (as in the M2L pass): the ancestors and the anchor are shared,
            // one 2p-wide task; the siblings' own Psi are adjacent columns (one term)
            int Bcell[32], Bkind[32];
            const int nB = chain(y2, l, Bcell, Bkind);
            const int o1 = Acell[0] == y ? 1 : 0, o2 = Bcell[0] == y2 ? 1 : 0;
            if (nA - o1 != nB - o2 || nB - o2 <= 0) {
              fprintf(stderr, "[svd1] internal: sibling chains differ (%d %d)\n", y, y2);
              std::abort();
            }
            begin_task();
            if (o1 || o2) {
              const int c0 = o1 ? y : y2, K = (o1 + o2) * p;
              new_term(IO_PSI, c0 * p, K, 2 * p, K);
              if (o1) add_op(OP_ID, y, y, p, p, 0, 0);
              if (o2) add_op(OP_ID, y2, y2, p, p, o1 ? p : 0, p);
              zero_flops += 2ll * K * 2 * p - 2ll * (o1 + o2) * p * p;
            }
            for (int q = o1; q < nA; ++q) {
              new_term(Akind[q], Acell[q] * p, p, 2 * p, p);
              add_op(OP_L2L, Acell[q], y, p, p, 0, 0);
              add_op(OP_L2L, Acell[q], y2, p, p, 0, p);
            }
            end_task(IO_PHI, y * p, 2 * p);
            loc[y] = loc[y2] = IO_PHI;
            ++i;  // y2 done
            continue;
          }
          begin_task();
          for (int q = 0; q < nA; ++q) {
            new_term(Akind[q], Acell[q] * p, p, p, p);
            add_op(Acell[q] == y ? OP_ID : OP_L2L, Acell[q], y, p, p, 0);
          }
          end_task(IO_PHI, y * p, p);
          loc[y] = IO_PHI;
        }
      if (int(F.tasks.size()) > pb) {
        F.pass_begin.push_back(pb);
        F.pass_bn.push_back(pairs ? 2 * p : p);
        F.pass_kind.push_back(3);
        sort_pass(pb);
      }
      a = hi;
    }
  }
  // final: L2P (STEP 9) + P2P near field (STEP 10); two launches by
  // output width (leaves with <= 16 targets use the 16-wide tile)
  int n_narrow = 0, n_wide = 0;
  for (int i = 0; i < nleaf; ++i) {
    const int y = lf0 + i;
    if (!has_tgt(y)) continue;
    (F.cells[y].thi - F.cells[y].tlo > 16 ? n_wide : n_narrow)++;
  }
  // a separate 16-wide launch only pays when it carries a real share of the leaves
  const bool split_narrow = n_narrow >= 16 || n_wide == 0;
  for (int wide = 0; wide < 2; ++wide) {
  if (!split_narrow && wide == 0) continue;
  F.pass_begin.push_back(int(F.tasks.size()));
  F.pass_bn.push_back(wide ? 32 : 16);
  F.pass_kind.push_back(4);
  for (int i = 0; i < nleaf; ++i) {
    const int y = lf0 + i;
    if (!has_tgt(y)) continue;
    const int ty = F.cells[y].thi - F.cells[y].tlo;
    if (split_narrow && (ty > 16) != (wide == 1)) continue;
    begin_task();
    const int par = (y - 1) / 2;
    if (has_local(y)) {
      new_term(IO_PSI, y * p, p, ty, p);
      add_op(OP_L2P, y, y, p, ty, 0);
    }
    if (!m2p[y].empty()) {  // one-sided: far fields of near-ish narrow leaves at the targets
      std::vector<int> ws(m2p[y].begin(), m2p[y].end());
      add_runs(ws, IO_PHI, OP_M2P, y, ty);
    }
    if (par >= 1 && loc[par] >= 0) {
      new_term(loc[par], par * p, p, ty, p);
      add_op(OP_L2P_FROM, par, y, p, ty, 0);
    }
    add_runs(near[y], IO_U, OP_P2P, y, ty);
    F.n_near_pairs += int(near[y].size());
    F.max_near = std::max<int>(F.max_near, int(near[y].size()));
    end_task(IO_U, F.cells[y].tlo, ty);
  }
  sort_pass(F.pass_begin.back());
  }
  F.pass_begin.push_back(int(F.tasks.size()));
  for (int& bn : F.pass_bn) bn = bn <= 16 ? 16 : 32;
  F.flops_per_row = F.flops_exec_per_row - zero_flops + adj;
  F.flops_cost_per_row = F.flops_exec_per_row - zero_flops;
  if (std::getenv("SVD1_DEBUG"))
    fprintf(stderr, "[svd1] lists: traversal %.3f ms, generation %.3f ms (ops %zu terms %zu tasks %zu)\n",
            tt1 - tt0, now_ms() - tt1, F.ops.size(), F.terms.size(), F.tasks.size());
}

}  // namespace

int64_t max_cells(int64_t N, int leaf);

void fmm_build_host(FmmHost& F, int na, int leaf, int p, const std::vector<double>& da,
                    const std::vector<double>& mu, const int32_t* src, int64_t rows) {
  const Merged M = merge_points(da, mu);
  int L0 = 0;
  while ((2 * int64_t(na) + (int64_t(1) << L0) - 1) / (int64_t(1) << L0) > 2 * leaf) ++L0;
  // The candidate depths L0, L0 + 1, L0 + 2 are built concurrently (the plan is on the
  // critical path of the stream: an apply starts when its plan is ready); the choice is then
  // made over the results in depth order exactly as a sequential search would make it.
  struct Cand {
    FmmHost F;
    int state = 0;  // 0 infeasible, 1 skipped (wide leaf), 2 built
  };
  const int Lhi = std::min(L0 + 2, 22);
  std::vector<Cand> cand(size_t(std::max(0, Lhi - L0 + 1)));
  auto build = [&](int L) {
    Cand& C = cand[size_t(L - L0)];
    if (!fmm_cells(C.F, leaf, L, M)) return;
    C.F.cap_cells = max_cells(na, leaf);
    // a leaf whose hull spans a quarter of the spectrum (outliers packed with bulk points
    // because the capacities left no room for a gap split) is near to every leaf: such a
    // tree is skipped when a deeper one is still to come
    if (L < L0 + 2) {
      double rmax = 0.0;
      for (int i = 0; i < (1 << L); ++i) rmax = std::max(rmax, C.F.cells[(1 << L) - 1 + i].r);
      if (rmax >= 0.25 * C.F.cells[0].r && C.F.cells[0].r > 0.0) {
        C.state = 1;
        return;
      }
    }
    fmm_lists(C.F, p, src, rows);
    C.state = 2;
  };
  auto cost_of = [rows](const FmmHost& H) {
    return double(H.flops_cost_per_row) + 2.0e8 / double(std::max<int64_t>(rows, 1)) * double(H.pass_bn.size());
  };
  static const bool parallel = std::getenv("SVD1_PLAN_PARALLEL") != nullptr;  // (experiments)
  if (const char* e = std::getenv("SVD1_FMM_FORCE_L")) {  // (experiments) one depth: L0 + value
    const int L = std::min(Lhi, L0 + std::max(0, atoi(e)));
    build(L);
    if (cand[size_t(L - L0)].state == 2) F = std::move(cand[size_t(L - L0)].F);
    return;
  }
  if (parallel) {
    std::vector<std::thread> th;
    for (int L = L0 + 1; L <= Lhi; ++L) th.emplace_back(build, L);
    if (L0 <= Lhi) build(L0);
    for (auto& t : th) t.join();
  } else {  // sequential, building only the depths the search below looks at
    int ib = -1;  // best built so far (the same rule as the selection loop)
    for (int L = L0; L <= Lhi; ++L) {
      if (ib >= 0 && cand[size_t(ib)].F.max_near <= 8) break;
      build(L);
      Cand& C = cand[size_t(L - L0)];
      if (C.state == 2 && (ib < 0 || cost_of(C.F) < cost_of(cand[size_t(ib)].F))) ib = L - L0;
    }
  }
  // cost: executed flops plus one launch-equivalent per pass
  auto cost = [rows](const FmmHost& H) {
    return double(H.flops_cost_per_row) + 2.0e8 / double(std::max<int64_t>(rows, 1)) * double(H.pass_bn.size());
  };
  FmmHost best;
  bool have = false;
  for (int L = L0; L <= Lhi; ++L) {
    // a deeper tree only pays when the shallower one has wide leaves (outliers)
    if (have && best.max_near <= 8) break;
    Cand& C = cand[size_t(L - L0)];
    if (std::getenv("SVD1_DEBUG")) {
      if (C.state == 0) fprintf(stderr, "[svd1] fmm L=%d infeasible\n", L);
      if (C.state == 1) fprintf(stderr, "[svd1] fmm L=%d skipped (wide leaf)\n", L);
      if (C.state == 2)
        fprintf(stderr, "[svd1] fmm L=%d flops/row=%lld max_near=%d m2l=%d near=%d\n", L,
                (long long)C.F.flops_per_row, C.F.max_near, C.F.n_m2l_pairs, C.F.n_near_pairs);
    }
    if (C.state != 2) continue;
    if (!have || cost(C.F) < cost(best)) {
      best = std::move(C.F);
      have = true;
    }
  }
  F = std::move(best);
  if (std::getenv("SVD1_DEBUG"))
    for (size_t q = 0; q + 1 < F.pass_begin.size(); ++q) {
      double fl = 0.0;
      for (int t = F.pass_begin[q]; t < F.pass_begin[q + 1]; ++t)
        for (int u = F.tasks[t].t_begin; u < F.tasks[t].t_end; ++u) fl += 2.0 * F.terms[u].K * F.tasks[t].N;
      fprintf(stderr, "[svd1]   pass %zu: %d tasks, %.0f flops/row (window)\n", q,
              F.pass_begin[q + 1] - F.pass_begin[q], fl);
    }
}

int apply_leaf(int p) {
  int leaf = std::min(2 * p, kMaxLeaf);  // STEP 2: s ~ 2p, capped by the tile
  if (const char* e = std::getenv("SVD1_LEAF")) leaf = std::max(4, std::min(kMaxLeaf, atoi(e)));  // tuning
  return leaf;
}

// Cells of the deepest tree fmm_build_host can choose for na <= N active points: depth
// L0 + 2, L0 the smallest depth with <= 2 leaf merged points per leaf (STEP 2).
int64_t max_cells(int64_t N, int leaf) {
  int L0 = 0;
  while ((2 * std::max<int64_t>(N, 1) + (int64_t(1) << L0) - 1) / (int64_t(1) << L0) > 2 * leaf) ++L0;
  const int L = std::min(L0 + 2, 22);
  return (int64_t(1) << (L + 1)) - 1;
}

// Expansion workspace (Phi or Psi) of one side: rows x (cells * p) doubles
size_t expansion_elems(int64_t rows, int64_t N, int p) {
  return size_t(std::max<int64_t>(rows, 1)) * size_t(max_cells(N, apply_leaf(p))) * size_t(p);
}

// Cauchy apply of one step, split in a host phase (decide FMM vs direct, build the
// tree and task lists, stage their upload) and a launch phase (operators + passes).
// U_out[:, dst[j]] = cs_j sum_i U_in[:, src[i]] zhat_i / ((d_i - d_kj) - tau_j)


// host compute only (thread-safe: touches nothing but C)
// src: active source i -> input column (nullptr: identity), n_in: input columns
void cauchy_plan(const svd1_config& cfg, CauchyPrep& C, int64_t rows, int na,
                 const std::vector<double>& da, const std::vector<double>& mu, int p,
                 const int32_t* src, int n_in) {
  const int minn = cfg.fmm_min_n > 0 ? cfg.fmm_min_n : 384;
  const int leaf = apply_leaf(p);
  bool fmm = (cfg.flags & SVD1_FORCE_FMM) ? (na > leaf) : (na >= minn);
  if (cfg.flags & SVD1_FORCE_DIRECT) fmm = false;
  C.fmm = fmm;
  C.p = p;
  C.na = na;
  C.rows = rows;
  C.flops = C.flops_exec = 2.0 * double(rows) * double(na) * double(na);
  if (!fmm) return;
  fmm_build_host(C.F, na, leaf, p, da, mu, src, rows);
  C.flops = double(C.F.flops_per_row) * double(rows);
  C.flops_exec = double(C.F.flops_exec_per_row) * double(rows);
  C.col2src.clear();
  C.n_in = n_in;
  C.n_out = n_in;
  if (src) {
    C.col2src.assign(size_t(n_in), -1);
    for (int i = 0; i < na; ++i) C.col2src[src[i]] = i;
  }
}

// the FMM plan's device arrays as parts of a blob (cauchy_bind sets the pointers)
void cauchy_stage(CauchyPrep& C, BlobBuilder& B) {
  if (!C.fmm) return;
  C.o_cells = B.add(C.F.cells);
  C.o_descs = B.add(C.F.ops);
  C.o_terms = B.add(C.F.terms);
  C.o_tasks = B.add(C.F.tasks);
  C.o_c2s = B.add(C.col2src);
}

svd1_status cauchy_bind(CauchyPrep& C, char* base, cudaStream_t st) {
  if (!C.fmm) return SVD1_OK;
  C.dcells = reinterpret_cast<FmmCell*>(base + C.o_cells);
  C.ddescs = reinterpret_cast<FmmOpDesc*>(base + C.o_descs);
  C.dterms = reinterpret_cast<FmmTerm*>(base + C.o_terms);
  C.dtasks = reinterpret_cast<FmmTask*>(base + C.o_tasks);
  C.dcol2src = C.col2src.empty() ? nullptr : reinterpret_cast<int32_t*>(base + C.o_c2s);
  double* ops;
  TRY(C.d_ops.get<double>(size_t(std::max<int64_t>(C.F.ops_rows, 1)) * 16, &ops, st));
  return SVD1_OK;
}

svd1_status cauchy_upload(svd1_plan_t P, CauchyPrep& C) {
  if (!C.fmm) return SVD1_OK;
  BlobBuilder B;
  cauchy_stage(C, B);
  char* base;
  TRY(arena_put_blob(P, B, C.blob, &base));
  return cauchy_bind(C, base, P->st);
}

svd1_status cauchy_prepare(svd1_plan_t P, CauchyPrep& C, int64_t rows, int na,
                           const std::vector<double>& da, const std::vector<double>& mu, int p) {
  cauchy_plan(P->cfg, C, rows, na, da, mu, p, nullptr, na);
  return cauchy_upload(P, C);
}

size_t cauchy_exp_elems(const CauchyPrep& C) {
  return C.fmm ? size_t(std::max(C.F.ecells, C.F.ncells)) * size_t(C.p) * size_t(C.rows) : 0;
}

// K5: every operator block of the plan into the ops buffer (zeroed first: op chunks are
// zero past K and N, which the GEMM relies on)
svd1_status cauchy_build_ops(svd1_plan_t P, CauchyPrep& C, const double* d_da, const int32_t* d_k,
                             const double* d_tau, const double* d_zhat, const double* d_cs, cudaStream_t st) {
  if (!C.fmm) return SVD1_OK;
  FmmHost& F = C.F;
  auto* ops = static_cast<double*>(C.d_ops.p);
  SVD1_CUDA_TRY(cudaMemsetAsync(ops, 0, size_t(std::max<int64_t>(F.ops_rows, 1)) * 16 * sizeof(double), st));
  return fmm_build_ops(int(F.ops.size()), C.ddescs, C.dcells, C.p, d_da, d_k, d_tau, d_zhat, d_cs, C.dcol2src, ops,
                       std::max<int64_t>(F.ops_rows, 1) * 16, st, LC(P));
}

constexpr int kMapSlots = 64;  // TMA descriptor sets per apply (one per row chunk, §4.11)
constexpr int kMaxPasses = 64; // GEMM passes per apply (tile counters)

// rows_n >= 0: the apply over rows_n rows starting at U_in / U_out (a row chunk of the fused
// per-side pass), its TMA descriptors in slot `slot`; the operator blocks
// are built by the first launch of the apply (or beforehand on the upload stream)
svd1_status cauchy_launch(svd1_plan_t P, CauchyPrep& C, const double* d_da, const int32_t* d_k,
                          const double* d_tau, const double* d_zhat, const double* d_cs,
                          const double* U_in, int64_t ld_in, const int32_t* d_src, double* U_out,
                          int64_t ld_out, const int32_t* d_dst, cudaStream_t st, int side,
                          int64_t rows_n = -1, int slot = 0, bool last_chunk = true) {
  const int64_t rows = rows_n >= 0 ? rows_n : C.rows;
  if (rows <= 0) return SVD1_OK;
  if (!C.fmm)
    return apply_direct(rows, C.na, d_da, d_k, d_tau, d_zhat, d_cs, U_in, ld_in, d_src, U_out, ld_out,
                        d_dst, st, LC(P));
  FmmHost& F = C.F;
  const int p = C.p;
  double *phi, *psi;
  const size_t exp_elems = cauchy_exp_elems(C);
  TRY(P->phi[side].get<double>(exp_elems, &phi, st));  // sized at creation (no growth here)
  TRY(P->psi[side].get<double>(exp_elems, &psi, st));
  const int64_t ldE = int64_t(std::max(F.ecells, F.ncells)) * p;
  FmmCell* dc = C.dcells;
  FmmOpDesc* dd = C.ddescs;
  FmmTerm* dt = C.dterms;
  FmmTask* dk = C.dtasks;
  auto* ops = static_cast<double*>(C.d_ops.p);
  const int32_t* c2s = C.dcol2src;
  if (!C.ops_ready) TRY(cauchy_build_ops(P, C, d_da, d_k, d_tau, d_zhat, d_cs, st));
  C.ops_ready = !last_chunk;  // later chunks of the same apply reuse the operator blocks
  (void)dd;
  (void)c2s;
  // TMA reads U_in: 16-byte aligned base and even leading dimension, else a padded copy
  if ((reinterpret_cast<uintptr_t>(U_in) & 15) || (ld_in & 1)) {
    const int64_t ldp = (C.n_in + 1) & ~int64_t(1);
    double* pad;
    TRY(P->upad[side].get<double>(size_t(rows) * size_t(ldp), &pad, st));
    SVD1_CUDA_TRY(cudaMemcpy2DAsync(pad, size_t(ldp) * 8, U_in, size_t(ld_in) * 8, size_t(C.n_in) * 8,
                                    size_t(rows), cudaMemcpyDeviceToDevice, st));
    U_in = pad;
    ld_in = ldp;
  }
  // descriptors live in global memory (one copy per apply, written on the apply's own
  // stream; the kernel acquires them through the tensormap proxy before use)
  {
    void* hm = C.h_maps;  // sized at creation
    TRY(pinned_reserve(&hm, &C.h_maps_cap, sizeof(FmmMaps) * kMapSlots));
    C.h_maps = static_cast<FmmMaps*>(hm);
  }
  if (slot < 0 || slot >= kMapSlots) return SVD1_E_INVALID;
  TRY(fmm_make_maps(C.h_maps + slot, rows, U_in, C.n_in, ld_in, phi, psi, ldE));
  FmmMaps* maps;
  TRY(C.d_maps.get<FmmMaps>(kMapSlots, &maps, st));
  maps += slot;
  SVD1_CUDA_TRY(cudaMemcpyAsync(maps, C.h_maps + slot, sizeof(FmmMaps), cudaMemcpyHostToDevice, st));
  const bool dbg = std::getenv("SVD1_DEBUG") != nullptr;
  if (dbg) {  // host-side validation of the task lists
    for (const FmmTask& T : F.tasks) {
      if (T.N < 1 || T.N > 32 || T.t_begin < 0 || T.t_end > int(F.terms.size()) || T.t_begin > T.t_end)
        fprintf(stderr, "[svd1] bad task out=%d/%d N=%d terms=[%d,%d)\n", T.out_kind, T.col0, T.N,
                T.t_begin, T.t_end);
      for (int t = T.t_begin; t < T.t_end; ++t) {
        const FmmTerm& R = F.terms[t];
        if (R.K < 1 || R.op_row < 0 || R.op_row + int64_t((R.K + 15) / 16) * R.npad > F.ops_rows ||
            T.op_col0 + T.N > R.npad)
          fprintf(stderr, "[svd1] bad term %d: kind=%d col0=%d K=%d row=%lld\n", t, R.in_kind, R.col0,
                  R.K, (long long)R.op_row);
      }
    }
    fprintf(stderr, "[svd1] fmm na=%d L=%d cells=%d tasks=%zu terms=%zu ops=%lld rows=%lld p=%d\n",
            C.na, F.L, F.ncells, F.tasks.size(), F.terms.size(), (long long)F.ops_rows * 16,
            (long long)rows, p);
  }
  if (std::getenv("SVD1_PASSSTATS")) {  // per pass: tasks, algorithmic vs tile-padded flops
    for (size_t s = 0; s + 1 < F.pass_begin.size(); ++s) {
      const int b = F.pass_begin[s], e = F.pass_begin[s + 1], bn = F.pass_bn[s];
      double fa = 0.0, fp = 0.0;
      int64_t kmax = 0;
      for (int t = b; t < e; ++t) {
        const FmmTask& T = F.tasks[t];
        int64_t ks = 0;
        for (int q = T.t_begin; q < T.t_end; ++q) {
          fa += 2.0 * F.terms[q].K * T.N;
          fp += 2.0 * ((F.terms[q].K + 15) / 16 * 16) * bn;
          ks += F.terms[q].K;
        }
        kmax = std::max(kmax, ks);
      }
      fprintf(stderr, "[svd1] pass %zu bn=%d tasks=%d flops=%.3e padded=%.3e (x%.2f) kmax=%lld\n", s, bn,
              e - b, fa * rows, fp * rows, fa > 0 ? fp / fa : 0.0, (long long)kmax);
    }
  }
  if (std::getenv("SVD1_CHECK_PASSES")) {  // diagnostics: a pass must not read what it writes
    for (size_t s = 0; s + 1 < F.pass_begin.size(); ++s) {
      std::vector<char> wphi(ldE, 0), wpsi(ldE, 0), wu(std::max(C.n_in, 1) + 64, 0);
      for (int t = F.pass_begin[s]; t < F.pass_begin[s + 1]; ++t) {
        const FmmTask& T = F.tasks[t];
        for (int j = 0; j < T.N; ++j) {
          if (T.out_kind == IO_PHI) wphi[T.col0 + j] = 1;
          if (T.out_kind == IO_PSI) wpsi[T.col0 + j] = 1;
        }
      }
      int bad = 0;
      for (int t = F.pass_begin[s]; t < F.pass_begin[s + 1]; ++t) {
        const FmmTask& T = F.tasks[t];
        for (int u = T.t_begin; u < T.t_end; ++u) {
          const FmmTerm& R = F.terms[u];
          const int kend = (R.K + 15) / 16 * 16;
          for (int k = 0; k < kend; ++k) {
            const int c = R.col0 + k;
            if (R.in_kind == IO_PHI && c < ldE && wphi[c]) ++bad;
            if (R.in_kind == IO_PSI && c < ldE && wpsi[c]) ++bad;
          }
        }
      }
      if (bad) fprintf(stderr, "[svd1] CHECK pass %zu: %d reads of columns written by the same pass\n", s, bad);
    }
  }
  const bool ptime = std::getenv("SVD1_PASSTIME") != nullptr;  // diagnostics (syncs)
  std::vector<cudaEvent_t> pev;
  auto pmark = [&]() {
    if (!ptime) return;
    cudaEvent_t e;
    cudaEventCreate(&e);
    cudaEventRecord(e, st);
    pev.push_back(e);
  };
  struct PassTimePrinter {
    std::vector<cudaEvent_t>* ev;
    ~PassTimePrinter() {
      if (ev->size() < 2) return;
      cudaEventSynchronize(ev->back());
      fprintf(stderr, "[svd1] pass us:");
      for (size_t i = 1; i < ev->size(); ++i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, (*ev)[i - 1], (*ev)[i]);
        fprintf(stderr, " %.1f", 1e3 * ms);
      }
      fprintf(stderr, "\n");
      for (auto e : *ev) cudaEventDestroy(e);
    }
  } ptp{&pev};
  pmark();
  C.ngev = 0;
  const bool gtime = std::getenv("SVD1_GEMM_EVENTS") != nullptr;  // diagnostics (host cost)
  auto gmark = [&]() -> svd1_status {  // events bracketing each GEMM pass
    if (!gtime) return SVD1_OK;
    if (C.ngev == int(C.gev.size())) {
      cudaEvent_t e;
      SVD1_CUDA_TRY(cudaEventCreate(&e));
      C.gev.push_back(e);
    }
    SVD1_CUDA_TRY(cudaEventRecord(C.gev[C.ngev++], st));
    return SVD1_OK;
  };
  // one tile counter per pass, zeroed for this launch (stream-ordered)
  int* ctrs;
  TRY(P->tile_ctr[side].get<int>(kMaxPasses, &ctrs, st));
  if (F.pass_begin.size() > size_t(kMaxPasses)) return SVD1_E_INVALID;
  SVD1_CUDA_TRY(cudaMemsetAsync(ctrs, 0, sizeof(int) * kMaxPasses, st));
  // pass kinds whose tiles run row-block-major (bit k: pass_kind k): every 16-wide pass
  // (P2M, M2M, M2L, L2L) -- the CTAs in flight cover a few row blocks and every task, so
  // the input rows they share (U windows, expansion windows of neighbouring cells) are read
  // from DRAM once.  C3 stream, 4 runs each: P2M only 447, P2M + M2L + L2L 454, all four
  // 457 updates/s; the final pass (32-wide, compute-bound) stays task-major (253 -> 270 us
  // row-block-major).  SVD1_RB_KINDS overrides the mask, SVD1_TILE_ORDER=rb sets every pass.
  static const unsigned rb_kinds = [] {
    const char* e = std::getenv("SVD1_TILE_ORDER");
    if (e && std::string(e) == "rb") return ~0u;
    const char* m = std::getenv("SVD1_RB_KINDS");
    return m ? unsigned(strtoul(m, nullptr, 0)) : 15u;
  }();
  for (size_t s = 0; s + 1 < F.pass_begin.size(); ++s) {
    const int b = F.pass_begin[s], e = F.pass_begin[s + 1];
    if (e <= b) continue;
    TRY(gmark());
    TRY(fmm_run_tasks(e - b, dk + b, dt, F.pass_bn[s], rows, maps, U_out, ld_out, d_dst, phi, psi, ldE,
                      C.n_out, int64_t(exp_elems), ops, F.ops_rows, ctrs + s, (rb_kinds >> F.pass_kind[s]) & 1, st, LC(P)));
    TRY(gmark());
    pmark();
    if (dbg) {
      cudaError_t err = cudaStreamSynchronize(st);
      fprintf(stderr, "[svd1] pass %zu tasks [%d,%d): %s\n", s, b, e, cudaGetErrorString(err));
      if (err != cudaSuccess) return SVD1_E_CUDA;
    }
  }
  return SVD1_OK;
}

svd1_status ensure_expansions(svd1_plan_t P, int side, size_t elems) {
  // zeroed when (re)allocated: a K chunk may reach past a term into columns no pass wrote
  // (they meet zero op rows, but 0 * NaN would not be 0).  Sized for the deepest tree at
  // creation; growth (a smaller eps than the plan's, or the standalone apply's sizes) is
  // stream-ordered on the side's apply stream, behind the applies that used the old buffer.
  const cudaStream_t st = side_stream(P, side);
  for (DevBuf* b : {&P->phi[side], &P->psi[side]}) {
    const void* before = b->p;
    const size_t cap0 = b->cap;  // (a new allocation may reuse the old address)
    double* x;
    TRY(b->get<double>(elems, &x, st));
    if (b->p != before || b->cap != cap0) SVD1_CUDA_TRY(cudaMemsetAsync(b->p, 0, b->cap, st));
  }
  return SVD1_OK;
}

// Secular FMM: plan from the oriented sources (host), one-copy upload, device view.
// Active size from which the secular solve uses the FMM far field.  In a stream
// (svd1_update_batch) the solve shares the GPU with the previous update's applies, and
// the FMM's smaller GPU work pays from C3's size on (measured 400 -> 410 updates/s); one
// call per update it pays only at C5's (its host plan and launches are on the critical
// path there).  SVD1_SEC_FMM_MIN overrides both.
int sec_fmm_min(bool stream) {
  static const int v = [] {
    const char* e = std::getenv("SVD1_SEC_FMM_MIN");
    return e ? std::max(64, atoi(e)) : 0;
  }();
  return v ? v : (stream ? 3072 : 6144);
}

bool use_sec_fmm(uint32_t flags, int n, bool stream) {
  if (flags & SVD1_SECULAR_DIRECT) return false;
  if (flags & SVD1_SECULAR_FMM) return n > 64;
  return n >= sec_fmm_min(stream);
}

svd1_status secfmm_prepare(svd1_plan_t P, SecPlanHost& H, DevBuf& blob, DevBuf& scr, const double* dr,
                           int n, int side, SecFmmDev* out) {
  static const bool report = std::getenv("SVD1_SECTIME") != nullptr;
  const double t0 = now_ms();
  secfmm_plan(dr, n, H);
  if (report) {
    int64_t mx = 0, tot = 0;
    int npad = 0, mxleaf = 0;
    for (int q = 0; q < H.nleaf; ++q) {
      int64_t s = 0;
      for (int g = H.near_off[q]; g < H.near_off[q + 1]; ++g) s += H.near_hi[g] - H.near_lo[g];
      const int cnt = H.leaf_lo[q + 1] - H.leaf_lo[q];
      tot += s * cnt;
      mx = std::max(mx, s);
      mxleaf = std::max(mxleaf, cnt);
      npad += H.cells[H.leaf_cell[q]].pad;
    }
    std::fprintf(stderr,
                 "secfmm_plan n=%d L=%d cells=%d leaves=%d parts=%zu near=%zu max_near_terms=%lld "
                 "mean=%.1f max_leaf=%d pad=%d: %.3f ms\n",
                 n, H.L, H.ncells, H.nleaf, H.parts.size(), H.near_lo.size(), (long long)mx,
                 double(tot) / n, mxleaf, npad, now_ms() - t0);
  }
  BlobBuilder B;
  const size_t o_cells = B.add(H.cells), o_parts = B.add(H.parts), o_llo = B.add(H.leaf_lo),
               o_lc = B.add(H.leaf_cell), o_no = B.add(H.near_off), o_nlo = B.add(H.near_lo),
               o_nhi = B.add(H.near_hi), o_dir = B.add(H.direct);
  char* base;
  TRY(arena_put_blob(P, B, blob, &base, side));
  double* sc;
  TRY(scr.get<double>(size_t(3) * H.ncells * kSecP, &sc, side_stream(P, side)));
  SecFmmDev F;
  F.L = H.L;
  F.ncells = H.ncells;
  F.nleaf = H.nleaf;
  F.ndirect = int(H.direct.size());
  F.direct = reinterpret_cast<const int32_t*>(base + o_dir);
  F.cells = reinterpret_cast<const SecFmmCell*>(base + o_cells);
  F.parts = reinterpret_cast<const SecFmmPart*>(base + o_parts);
  F.leaf_lo = reinterpret_cast<const int32_t*>(base + o_llo);
  F.leaf_cell = reinterpret_cast<const int32_t*>(base + o_lc);
  F.near_off = reinterpret_cast<const int32_t*>(base + o_no);
  F.near_lo = reinterpret_cast<const int32_t*>(base + o_nlo);
  F.near_hi = reinterpret_cast<const int32_t*>(base + o_nhi);
  F.phi = sc;
  F.psiL = sc + size_t(H.ncells) * kSecP;
  F.psiR = sc + size_t(2) * H.ncells * kSecP;
  *out = F;
  return SVD1_OK;
}

// joins its threads on scope exit (early error returns included)
struct Joiner {
  std::vector<WorkThread> ts;
  void add(WorkThread&& t) { ts.push_back(std::move(t)); }
  void join() {
    for (auto& t : ts)
      if (t.joinable()) t.join();
    ts.clear();
  }
  ~Joiner() { join(); }
};

// read-back words of one eigen-update's spectral results (see spectral_launch)
size_t spectral_words(int nap, int nc, int G) {
  return size_t(nap) * (3 + nc) + size_t(nap + 1) / 2 + size_t(G + 1) / 2 + 1;
}

// In-place all-gather of every rank's slice [r c, r c + c) of each part, one NCCL group on
// the chain's communicator and stream (no-op on one process or in the emulation mode,
// where every slice was computed here).
struct GatherPart {
  void* base;
  int count;  // c: elements per rank
  ncclDataType_t type;
  int elem;   // bytes per element
};
svd1_status exchange(svd1_plan_t P, int chain, cudaStream_t st, const std::vector<GatherPart>& parts) {
  if (!P->use_nccl) return SVD1_OK;
  const NcclApi& A = nccl_api();
  NCCL_TRY(A.GroupStart());
  for (const GatherPart& g : parts) {
    char* base = static_cast<char*>(g.base);
    const ncclResult_t r = A.AllGather(base + size_t(P->rank) * g.count * g.elem, base, size_t(g.count), g.type,
                                       P->comm[chain], st);
    if (r != ncclSuccess) {
      A.GroupEnd();
      return nccl_fail(r, "ncclAllGather");
    }
  }
  NCCL_TRY(A.GroupEnd());
  return SVD1_OK;
}

// --------------------------------------------------------- Alg 6.2 spectral
// One RankOneUpdate on the small vectors, in two halves so that the U- and
// V-side eigen-updates run on the GPU together and the host builds FMM trees meanwhile.
// spectral_launch: sort (stable, ties by column), deflate, enqueue the
// secular solve (STEP 2), Loewner, column norms and carried X^T v, and their read-back.
svd1_status spectral_launch(svd1_plan_t P, StepRecord& S, const std::vector<double>& D,
                            const std::vector<double>& z, double rho,
                            const std::vector<std::vector<double>>& carries, int ev0, int side, int chain) {
  TRY(ensure_side(P, side));
  const cudaStream_t st = side_stream(P, side);
  const double th_start = now_ms();
  const int N = int(D.size());
  S.clear_host();  // device buffers are kept (grow-only)
  S.N = N;
  S.rho = rho;
  S.ev0 = ev0;
  std::vector<int32_t>& perm = S.perm;
  perm.resize(N);
  std::iota(perm.begin(), perm.end(), 0);
  // stable ascending order; D is usually already ascending (second eigen-update) or
  // strictly descending (user's sigma order) -> O(n) fast paths
  bool asc = true, desc_strict = true;
  for (int q = 1; q < N; ++q) {
    if (D[q] < D[q - 1]) asc = false;
    if (!(D[q] < D[q - 1])) desc_strict = false;
  }
  if (!asc) {
    if (desc_strict) {
      std::reverse(perm.begin(), perm.end());
    } else {
      std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return D[a] < D[b]; });
    }
  }
  std::vector<double>& ds = S.ds;
  ds.resize(N);
  std::vector<double> zs(N);
  for (int s = 0; s < N; ++s) {
    ds[s] = D[perm[s]];
    zs[s] = z[perm[s]];
  }
  const int nc = int(carries.size());
  S.nc = nc;
  auto& cs_sorted = S.cs_sorted;  // capacity kept across steps
  cs_sorted.resize(nc);
  for (int q = 0; q < nc; ++q) {
    cs_sorted[q].resize(N);
    double* dstq = cs_sorted[q].data();
    const double* srcq = carries[q].data();
    for (int s = 0; s < N; ++s) dstq[s] = srcq[perm[s]];
  }
  const int ng = S.gcar ? int(S.gcar->size()) : 0;
  S.gs_sorted.resize(ng);
  for (int q = 0; q < ng; ++q) {
    S.gs_sorted[q].resize(N);
    for (int s = 0; s < N; ++s) S.gs_sorted[q][s] = (*S.gcar)[q][perm[s]];
  }
  // deflation (DESIGN.md §3.2 D1): (i) zero weights, (iii) exact repeats
  double zn2 = 0.0;
  for (double v : zs) zn2 += v * v;
  const double tol = 8.0 * kEps * std::sqrt(zn2);
  std::vector<char> alive(N, 1);
  for (int s = 0; s < N; ++s)
    if (!(std::fabs(zs[s]) > tol)) {
      alive[s] = 0;
      zs[s] = 0.0;
    }
  S.h_goff.push_back(0);
  {
    std::vector<int> surv;
    for (int s = 0; s < N; ++s)
      if (alive[s]) surv.push_back(s);
    size_t t = 0;
    while (t < surv.size()) {
      size_t u = t;
      while (u + 1 < surv.size() && ds[surv[u + 1]] == ds[surv[t]]) ++u;
      if (u > t) {
        double nrm2 = 0.0;
        for (size_t q = t; q <= u; ++q) nrm2 += zs[surv[q]] * zs[surv[q]];
        const double zl = zs[surv[u]];
        const double alpha = -std::copysign(std::sqrt(nrm2), zl);
        std::vector<double> v;
        for (size_t q = t; q <= u; ++q) v.push_back(zs[surv[q]]);
        v.back() -= alpha;
        double vv = 0.0;
        for (double x : v) vv += x * x;
        for (size_t q = t; q <= u; ++q) {
          S.h_cols.push_back(perm[surv[q]]);
          S.h_hv.push_back(v[q - t]);
        }
        S.h_goff.push_back(int32_t(S.h_cols.size()));
        // same reflection on the carried coefficient vectors: c <- c - v (2 v.c / v.v)
        for (int qq = 0; qq < nc; ++qq) {
          double dot = 0.0;
          for (size_t q = t; q <= u; ++q) dot += v[q - t] * cs_sorted[qq][surv[q]];
          const double f = 2.0 * dot / vv;
          for (size_t q = t; q <= u; ++q) cs_sorted[qq][surv[q]] -= f * v[q - t];
        }
        for (int qq = 0; qq < ng; ++qq) {
          double dot = 0.0;
          for (size_t q = t; q <= u; ++q) dot += v[q - t] * S.gs_sorted[qq][surv[q]];
          const double f = 2.0 * dot / vv;
          for (size_t q = t; q <= u; ++q) S.gs_sorted[qq][surv[q]] -= f * v[q - t];
        }
        for (size_t q = t; q < u; ++q) {
          zs[surv[q]] = 0.0;
          alive[surv[q]] = 0;
        }
        zs[surv[u]] = alpha;
      }
      t = u + 1;
    }
  }
  S.act.clear();
  S.dfl.clear();
  for (int s = 0; s < N; ++s) (alive[s] ? S.act : S.dfl).push_back(s);
  const int na = int(S.act.size());
  S.na = na;
  std::vector<double> za(na);
  S.da.resize(na);
  S.src_cols.resize(na);
  for (int i = 0; i < na; ++i) {
    S.da[i] = ds[S.act[i]];
    za[i] = zs[S.act[i]];
    S.src_cols[i] = perm[S.act[i]];
  }
  if (na == 0) return SVD1_OK;
  const double th0 = now_ms();
  // one upload [d_a | z_a | carries] and one read-back
  // [k (nap words) | tau | cs | carry_out (nc*nap) | iters (int32) | status (G int32)]
  // (nap = G c >= na: every rank's slice of c indices, the in-place all-gather layout)
  const int G = P->world;
  const int c_sl = slice_of(na, G, 0).c;
  const int nap = G * c_sl;
  S.nap = nap;
  const size_t in_words = size_t(na) * (4 + nc);
  const size_t words = spectral_words(nap, nc, G);
  double* din;
  double* dout;
  TRY(S.d_in.get<double>(in_words, &din, st));
  TRY(S.d_out.get<double>(words, &dout, st));
  double* stage;  // built in place in the pinned arena (no intermediate copies)
  size_t stage_off;
  {
    TRY(ensure_side(P, side));
    TRY(arena_reserve(P, side, in_words * sizeof(double), &stage_off));
    stage = reinterpret_cast<double*>(P->arena[side].buf + stage_off);
    std::memcpy(stage, S.da.data(), na * sizeof(double));
    std::memcpy(stage + na, za.data(), na * sizeof(double));
    // the secular solver's view: rho > 0 orientation (reflected for rho < 0), z squared
    double* dr = stage + 2 * na;
    double* z2r = stage + 3 * na;
    for (int i = 0; i < na; ++i) {
      const int src = rho < 0.0 ? na - 1 - i : i;
      dr[i] = rho < 0.0 ? -S.da[src] : S.da[src];
      z2r[i] = za[src] * za[src];
    }
    for (int q = 0; q < nc; ++q) {
      double* cq = stage + size_t(4 + q) * na;
      const double* src = cs_sorted[q].data();
      for (int i = 0; i < na; ++i) cq[i] = src[S.act[i]];
    }
    TRY(arena_commit(P, side, stage_off, in_words * sizeof(double), din));
  }
  double* dda = din;
  double* dza = din + na;
  double* ddr = din + 2 * na;
  double* dz2r = din + 3 * na;
  double* dcar = din + 4 * na;
  int32_t* dk = reinterpret_cast<int32_t*>(dout);
  double* dtau = dout + nap;
  double* dcs = dout + 2 * nap;
  double* dco = dout + 3 * nap;
  int32_t* dit = reinterpret_cast<int32_t*>(dout + size_t(3 + nc) * nap);
  int32_t* dst = reinterpret_cast<int32_t*>(dout + size_t(3 + nc) * nap + size_t(nap + 1) / 2);
  double* dzh;
  TRY(S.d_zhat.get<double>(nap, &dzh, st));
  SVD1_CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(int32_t) * G, st));
  TRY(ev_record(P, ev0, st));
  tl_mark(P, "  ev" + std::to_string(ev0) + " uploaded", st);
  double* scr;
  TRY(S.d_scratch.get<double>(size_t(spectral_scratch_elems(na, nc)), &scr, st));
  int* ctr;
  TRY(counters(S.d_ctr, na, st, &ctr));
  S.sec_fmm_used = use_sec_fmm(P->cfg.flags, na, side >= 2);  // sides 2, 3: batch mode
  // this process's ranks: its own, or every rank's slice in the emulation test mode
  const int r_lo = P->emulate ? 0 : P->rank, r_hi = P->emulate ? G : P->rank + 1;
  SecFmmDev F;
  if (S.sec_fmm_used)  // (reads the oriented sources from the staging region before its own upload)
    TRY(secfmm_prepare(P, S.sec, S.sec_blob, S.sec_scr, stage + 2 * na, na, side, &F));
  for (int r = r_lo; r < r_hi; ++r) {  // STEP 2 on the roots of rank r's slice
    const Slice sl = slice_of(na, G, r);
    // output index range [lo, hi); the solver works in the rho > 0 view (reflected for rho < 0)
    const int j0 = rho < 0.0 ? na - sl.hi : sl.lo, j1 = rho < 0.0 ? na - sl.lo : sl.hi;
    if (S.sec_fmm_used)  // with the far field by FMM
      TRY(secular_fmm(ddr, dz2r, rho, na, j0, j1, F, dk, dtau, dit, dst + r, st, LC(P)));
    else
      TRY(secular(ddr, dz2r, rho, na, j0, j1, dk, dtau, dit, dst + r, st, LC(P)));
  }
  TRY(exchange(P, chain, st, {{dk, c_sl, ncclInt32, 4}, {dtau, c_sl, ncclFloat64, 8}, {dit, c_sl, ncclInt32, 4},
                              {dst, 1, ncclInt32, 4}}));
  tl_mark(P, "  ev" + std::to_string(ev0) + " secular done", st);
  for (int r = r_lo; r < r_hi; ++r) {
    const Slice sl = slice_of(na, G, r);
    TRY(loewner(dda, dk, dtau, rho, dza, na, sl.lo, sl.hi, dzh, scr, ctr, st, LC(P)));
  }
  TRY(exchange(P, chain, st, {{dzh, c_sl, ncclFloat64, 8}}));
  tl_mark(P, "  ev" + std::to_string(ev0) + " loewner done", st);
  for (int r = r_lo; r < r_hi; ++r) {
    const Slice sl = slice_of(na, G, r);
    TRY(colnorm_carry(dda, dk, dtau, dzh, na, sl.lo, sl.hi, dcar, nc, dcs, dco, nap, dst + r, scr, ctr, st,
                      LC(P)));
  }
  {
    std::vector<GatherPart> parts{{dcs, c_sl, ncclFloat64, 8}, {dst, 1, ncclInt32, 4}};
    for (int q = 0; q < nc; ++q) parts.push_back({dco + size_t(q) * nap, c_sl, ncclFloat64, 8});
    TRY(exchange(P, chain, st, parts));
  }
  tl_mark(P, "  ev" + std::to_string(ev0) + " colnorm done", st);
  TRY(ev_record(P, ev0 + 1, st));
  {
    void* rb = S.rb;  // sized at creation
    TRY(pinned_reserve(&rb, &S.rb_cap, words * sizeof(double)));
    S.rb = static_cast<double*>(rb);
  }
  SVD1_CUDA_TRY(cudaMemcpyAsync(S.rb, dout, words * sizeof(double), cudaMemcpyDeviceToHost, st));
  if (!S.done_ev) SVD1_CUDA_TRY(cudaEventCreateWithFlags(&S.done_ev, cudaEventDisableTiming));
  SVD1_CUDA_TRY(cudaEventRecord(S.done_ev, st));
  S.pending = true;
  if (std::getenv("SVD1_TIMING"))
    fprintf(stderr, "[svd1] spectral_launch N=%d: host prep %.3f ms, stage+launch %.3f ms\n", N,
            th0 - th_start, now_ms() - th0);
  return SVD1_OK;
}

// spectral_finish (after a stream sync): status, mu, merge of mu with the deflated
// eigenvalues (stable ascending, deflated first on ties), the new eigenvalues D and
// carried vectors indexed by output position.
svd1_status spectral_finish(svd1_plan_t P, StepRecord& S, std::vector<double>& D,
                            std::vector<std::vector<double>>& carries) {
  const int N = S.N, na = S.na, nc = S.nc;
  const double* carry_out = nullptr;
  if (S.pending) {  // this step's kernels and read-back only (the other side may still run)
    SVD1_CUDA_TRY(cudaEventSynchronize(S.done_ev));
    S.pending = false;
  }
  const int nap = S.nap;
  if (na > 0) {
    const double* rb = S.rb;
    int32_t st_h = 0;  // every rank's status word
    {
      const int32_t* sw = reinterpret_cast<const int32_t*>(rb + size_t(3 + nc) * nap + size_t(nap + 1) / 2);
      for (int r = 0; r < P->world; ++r) st_h |= sw[r];
    }
    S.k_h.resize(na);
    std::memcpy(S.k_h.data(), rb, na * sizeof(int32_t));
    S.tau_h.assign(rb + nap, rb + nap + na);
    S.cs_h.assign(rb + 2 * nap, rb + 2 * nap + na);
    carry_out = rb + 3 * nap;
    const int32_t* it = reinterpret_cast<const int32_t*>(rb + size_t(3 + nc) * nap);
    double sum_it = 0.0;
    for (int j = 0; j < na; ++j) {
      S.max_iter = std::max(S.max_iter, it[j]);
      sum_it += it[j];
    }
    S.mean_iter = sum_it / na;
#ifdef SVD1_SECPROF  // iters hold per-root kilocycles: print the slowest roots
    {
      std::vector<int> ord(na);
      std::iota(ord.begin(), ord.end(), 0);
      std::partial_sort(ord.begin(), ord.begin() + std::min(na, 6), ord.end(),
                        [&](int x, int y) { return it[x] > it[y]; });
      std::fprintf(stderr, "secprof na=%d fmm=%d:", na, int(S.sec_fmm_used));
      for (int q = 0; q < std::min(na, 6); ++q)
        std::fprintf(stderr, " j%d=%dk/%dit", ord[q], it[ord[q]] >> 8, it[ord[q]] & 255);
      std::vector<int> v(it, it + na);
      std::nth_element(v.begin(), v.begin() + na / 2, v.end());
      std::fprintf(stderr, " median=%dk rho=%.3e dk=%.3e tau=%.3e\n", v[na / 2] >> 8, S.rho,
                   S.da[S.k_h[ord[0]]], S.tau_h[ord[0]]);
    }
#endif
    S.spectral_ms = ev_ms(P, S.ev0, S.ev0 + 1);
    if (st_h & 1) return SVD1_E_NOCONV;
    if (st_h & 2) return SVD1_E_POLE;
    if (st_h & 4) return SVD1_E_ZEROCOL;
  }
  S.mu.resize(na);
  for (int j = 0; j < na; ++j) S.mu[j] = S.da[S.k_h[j]] + S.tau_h[j];
  struct Item {
    double v;
    int flag, pos;
  };
  // both lists are ascending (deflated d in sorted order; roots interlace) -> O(n) merge
  // (stable ascending, deflated first on ties); fall back to a sort if mu is not sorted
  std::vector<Item> items;  // (local: spectral_finish runs on the main thread only)
  items.reserve(N);
  bool mu_sorted = true;
  for (int j = 1; j < na; ++j)
    if (S.mu[j] < S.mu[j - 1]) mu_sorted = false;
  if (mu_sorted) {
    size_t a = 0;
    int j = 0;
    while (a < S.dfl.size() || j < na) {
      if (j >= na || (a < S.dfl.size() && S.ds[S.dfl[a]] <= S.mu[j])) {
        items.push_back({S.ds[S.dfl[a]], 0, S.dfl[a]});
        ++a;
      } else {
        items.push_back({S.mu[j], 1, j});
        ++j;
      }
    }
  } else {
    for (int s : S.dfl) items.push_back({S.ds[s], 0, s});
    for (int j = 0; j < na; ++j) items.push_back({S.mu[j], 1, j});
    std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) {
      if (a.v != b.v) return a.v < b.v;
      if (a.flag != b.flag) return a.flag < b.flag;
      return a.pos < b.pos;
    });
  }
  S.tgt_pos.assign(na, -1);
  std::vector<double>& Dn = S.Dn;  // swapped with D / carries below: storage recycles
  std::vector<std::vector<double>>& cn = S.cn;
  Dn.resize(N);
  cn.resize(nc);
  for (auto& v : cn) v.resize(N);
  for (int q = 0; q < N; ++q) {
    const Item& it = items[q];
    Dn[q] = it.v;
    if (it.flag == 0) {
      S.pass_src.push_back(S.perm[it.pos]);
      S.pass_dst.push_back(q);
      S.pass_scale.push_back(1.0);
      for (int qq = 0; qq < nc; ++qq) cn[qq][q] = S.cs_sorted[qq][it.pos];
    } else {
      S.tgt_pos[it.pos] = q;
      for (int qq = 0; qq < nc; ++qq) cn[qq][q] = carry_out[size_t(qq) * nap + it.pos];
    }
  }
  D.swap(Dn);
  carries.swap(cn);
  if (S.gcar) {  // host-only carries: deflated entries move with their columns, active ones 0
    const int ng = int(S.gcar->size());
    S.gn.resize(ng);
    for (int qq = 0; qq < ng; ++qq) {
      S.gn[qq].resize(N);
      for (int q = 0; q < N; ++q) S.gn[qq][q] = items[q].flag == 0 ? S.gs_sorted[qq][items[q].pos] : 0.0;
    }
    S.gcar->swap(S.gn);
  }
  return SVD1_OK;
}

// Host half of one apply: column maps, Householder data, Cauchy plan; staged uploads.
// out_col(q) = reverse ? (N - 1 - q) : q.
// Host half of one apply, in two parts: apply_plan (pure host compute, thread-safe per
// step: column maps and the Cauchy/FMM plan) and apply_upload (staged uploads).
// out_col(q) = reverse ? (N - 1 - q) : q.
// output buffer columns of the step (main thread, before its plan is spawned)
void set_out_cols(StepRecord& S, int64_t rows, bool reverse) {
  const int N = S.N;
  S.rows = rows;
  auto oc = [&](int q) { return reverse ? N - 1 - q : q; };
  S.dst_cols.resize(S.na);
  for (int j = 0; j < S.na; ++j) S.dst_cols[j] = oc(S.tgt_pos[j]);
  S.pass_dst_cols.resize(S.pass_dst.size());
  for (size_t q = 0; q < S.pass_dst.size(); ++q) S.pass_dst_cols[q] = oc(S.pass_dst[q]);
}

// the step's Cauchy/FMM plan (worker thread: touches S.cp and S.plan_ms only)
void apply_plan(const svd1_config& cfg, int p, StepRecord& S) {
  const double t0 = now_ms();
  struct Stamp {
    StepRecord& S;
    double t0;
    ~Stamp() { S.plan_ms = now_ms() - t0; }
  } stamp{S, t0};
  if (S.rows <= 0) return;
  if (S.na > 0) cauchy_plan(cfg, S.cp, S.rows, S.na, S.da, S.mu, p, S.src_cols.data(), S.N);
}

// batch mode: the column maps, Householder groups and scales alone (what the carried
// rows need; no plan), and the FMM plan separately once it is built
svd1_status upload_maps(svd1_plan_t P, StepRecord& S, int side) {
  BlobBuilder B;
  const size_t o_goff = B.add(S.h_goff), o_hcols = B.add(S.h_cols), o_hv = B.add(S.h_hv);
  const size_t o_src = B.add(S.src_cols), o_dst = B.add(S.dst_cols);
  const size_t o_cs = B.add(S.cs_h);
  const size_t o_ps = B.add(S.pass_src), o_pd = B.add(S.pass_dst_cols), o_pc = B.add(S.pass_scale);
  char* base;
  TRY(arena_put_blob(P, B, S.blob, &base, side));
  S.dgoff = reinterpret_cast<int32_t*>(base + o_goff);
  S.dhcols = reinterpret_cast<int32_t*>(base + o_hcols);
  S.dhv = reinterpret_cast<double*>(base + o_hv);
  S.dsrc = reinterpret_cast<int32_t*>(base + o_src);
  S.ddst = reinterpret_cast<int32_t*>(base + o_dst);
  S.dcs = reinterpret_cast<double*>(base + o_cs);
  S.dpsrc = reinterpret_cast<int32_t*>(base + o_ps);
  S.dpdst = reinterpret_cast<int32_t*>(base + o_pd);
  S.dpscale = reinterpret_cast<double*>(base + o_pc);
  return SVD1_OK;
}
svd1_status upload_fmm(svd1_plan_t P, StepRecord& S, int side) {
  if (S.rows <= 0 || S.na <= 0 || !S.cp.fmm) return SVD1_OK;
  BlobBuilder B;
  cauchy_stage(S.cp, B);
  char* base;
  TRY(arena_put_blob(P, B, S.cp.blob, &base, side));
  return cauchy_bind(S.cp, base, side_stream(P, side));
}

svd1_status apply_upload(svd1_plan_t P, StepRecord& S, int side) {
  if (S.rows <= 0) return SVD1_OK;
  BlobBuilder B;
  const size_t o_goff = B.add(S.h_goff), o_hcols = B.add(S.h_cols), o_hv = B.add(S.h_hv);
  const size_t o_src = B.add(S.src_cols), o_dst = B.add(S.dst_cols);
  const size_t o_cs = B.add(S.cs_h);  // cs_h may carry the sign alignment
  const size_t o_ps = B.add(S.pass_src), o_pd = B.add(S.pass_dst_cols), o_pc = B.add(S.pass_scale);
  if (S.na > 0) cauchy_stage(S.cp, B);
  char* base;
  TRY(arena_put_blob(P, B, S.blob, &base, side));
  S.dgoff = reinterpret_cast<int32_t*>(base + o_goff);
  S.dhcols = reinterpret_cast<int32_t*>(base + o_hcols);
  S.dhv = reinterpret_cast<double*>(base + o_hv);
  S.dsrc = reinterpret_cast<int32_t*>(base + o_src);
  S.ddst = reinterpret_cast<int32_t*>(base + o_dst);
  S.dcs = reinterpret_cast<double*>(base + o_cs);
  S.dpsrc = reinterpret_cast<int32_t*>(base + o_ps);
  S.dpdst = reinterpret_cast<int32_t*>(base + o_pd);
  S.dpscale = reinterpret_cast<double*>(base + o_pc);
  if (S.na > 0) TRY(cauchy_bind(S.cp, base, side_stream(P, side)));
  return SVD1_OK;
}

// One row chunk [r0, r0 + rows) of a step's apply (Householder in place on U_in, Cauchy
// apply, passthrough): the whole apply is the chunk r0 = 0, rows = S.rows.
svd1_status apply_chunk(svd1_plan_t P, StepRecord& S, double* U_in, int64_t ld_in, double* U_out,
                        int64_t ld_out, int64_t r0, int64_t rows, cudaStream_t st, int side, int slot,
                        bool last_chunk) {
  if (rows <= 0) return SVD1_OK;
  U_in += r0 * ld_in;
  U_out += r0 * ld_out;
  if (S.h_goff.size() > 1)
    TRY(householder_cols(rows, U_in, ld_in, int(S.h_goff.size()) - 1, S.dgoff, S.dhcols, S.dhv, S.h_maxlen(), st,
                         LC(P)));
  if (S.na > 0)
    TRY(cauchy_launch(P, S.cp, static_cast<double*>(S.d_in.p), static_cast<int32_t*>(S.d_out.p),
                      static_cast<double*>(S.d_out.p) + S.nap, static_cast<double*>(S.d_zhat.p), S.dcs,
                      U_in, ld_in, S.dsrc, U_out, ld_out, S.ddst, st, side, rows, slot, last_chunk));
  if (!S.pass_src.empty())
    TRY(passthrough(rows, int(S.pass_src.size()), U_in, ld_in, S.dpsrc, U_out, ld_out, S.dpdst, S.dpscale,
                    st, LC(P)));
  return SVD1_OK;
}

// Device half: Householder (in place on U_in), Cauchy apply, passthrough.
svd1_status apply_launch(svd1_plan_t P, StepRecord& S, double* U_in, int64_t ld_in, double* U_out,
                         int64_t ld_out, int ev0, cudaStream_t st, int side) {
  const int64_t rows = S.rows;
  if (rows <= 0) return SVD1_OK;
  TRY(ev_record(P, ev0, st));
  TRY(apply_chunk(P, S, U_in, ld_in, U_out, ld_out, 0, rows, st, side, 0, true));
  TRY(ev_record(P, ev0 + 1, st));
  if (std::getenv("SVD1_NANCHECK")) {  // diagnostics: first non-finite output column
    SVD1_CUDA_TRY(cudaStreamSynchronize(st));
    std::vector<double> hb(size_t(rows) * ld_out);
    SVD1_CUDA_TRY(cudaMemcpy(hb.data(), U_out, hb.size() * sizeof(double), cudaMemcpyDeviceToHost));
    int64_t bad = -1, nbad = 0;
    for (int64_t r = 0; r < rows; ++r)
      for (int64_t c2 = 0; c2 < S.N; ++c2)
        if (!std::isfinite(hb[r * ld_out + c2])) {
          ++nbad;
          if (bad < 0) bad = c2;
        }
    double csmin = 1e300, csmax = 0.0;
    for (double v : S.cs_h) {
      csmin = std::min(csmin, std::fabs(v));
      csmax = std::max(csmax, std::fabs(v));
    }
    fprintf(stderr, "[svd1] apply ev%d N=%d na=%d hh_groups=%zu pass=%zu: non-finite %lld (first col %lld) cs [%.3e, %.3e]\n",
            ev0, S.N, S.na, S.h_goff.size() - 1, S.pass_src.size(), (long long)nbad, (long long)bad, csmin, csmax);
    int ncs = 0, ntau = 0;
    for (double v : S.cs_h) ncs += !std::isfinite(v);
    for (double v : S.tau_h) ntau += !std::isfinite(v);
    std::vector<double> zh(S.na);
    cudaMemcpy(zh.data(), S.d_zhat.p, S.na * sizeof(double), cudaMemcpyDeviceToHost);
    int nzh = 0;
    for (double v : zh) nzh += !std::isfinite(v);
    if (bad >= 0) {
      int wj = -1, wq = -1, nw = 0;
      for (int j = 0; j < S.na; ++j)
        if (S.dst_cols[j] == bad) wj = j, ++nw;
      for (size_t q = 0; q < S.pass_dst_cols.size(); ++q)
        if (S.pass_dst_cols[q] == bad) wq = int(q), ++nw;
      std::vector<double> inb(size_t(rows) * ld_in);
      cudaMemcpy(inb.data(), U_in, inb.size() * sizeof(double), cudaMemcpyDeviceToHost);
      int64_t nin = 0;
      for (double v : inb) nin += !std::isfinite(v);
      fprintf(stderr, "   col %lld written by j %d q %d (%d writers); non-finite in U_in %lld; pass_scale %g\n", (long long)bad, wj, wq, nw,
              (long long)nin, wq >= 0 ? S.pass_scale[wq] : 0.0);
      if (wj >= 0) fprintf(stderr, "   j %d: k %d tau %.17g cs %g\n", wj, S.k_h[wj], S.tau_h[wj], S.cs_h[wj]);
    }
    fprintf(stderr, "   nonfinite cs %d tau %d zhat %d; j0: k %d tau %.17g cs %.6g mu %.6g d0 %.17g d1 %.6g zhat0 %.6g dst0 %d\n", ncs, ntau, nzh,
            S.k_h[0], S.tau_h[0], S.cs_h[0], S.mu[0], S.da[0], S.na > 1 ? S.da[1] : 0.0, zh[0], S.dst_cols[0]);
  }
  return SVD1_OK;
}

bool all_finite(const double* x, size_t n) {
  for (size_t i = 0; i < n; ++i)
    if (!std::isfinite(x[i])) return false;
  return true;
}

// ---- create-time workspaces ("the plan owns its workspace, sized at create
// time").  Sizes depend on (m, n, row blocks, p) only; the FMM plan's own arrays (operator
// blocks, interaction lists) depend on the tree and get a generous estimate here: an
// update that outgrows one grows it in stream order (no device synchronisation) and
// reports it in svd1_report.allocations.
size_t fmm_blob_estimate(int64_t N, int p) {
  const int64_t cells = max_cells(N, apply_leaf(p));
  return size_t(cells) * 2048 + size_t(N) * 8 + (size_t(64) << 10);
}
size_t ops_estimate(int64_t N) { return size_t(std::max<int64_t>(N, 64)) * 1024 + (size_t(64) << 10); }
size_t maps_blob_bytes(int64_t N) { return size_t(N + 1) * 48 + 4096; }  // upload_maps / apply_upload

svd1_status reserve_step(StepRecord& S, int64_t N, int p, int G) {
  const int nc = kMaxCarry;
  const int nap = G * slice_of(int(N), G, 0).c;
  TRY(S.d_in.reserve<double>(size_t(N) * (4 + nc)));
  TRY(S.d_out.reserve<double>(spectral_words(nap, nc, G)));
  TRY(S.d_zhat.reserve<double>(size_t(nap)));
  TRY(S.d_scratch.reserve<double>(size_t(spectral_scratch_elems(int(N), nc))));
  TRY(S.d_ctr.reserve<int>(size_t(N / 64 + 16)));
  SVD1_CUDA_TRY(cudaMemset(S.d_ctr.p, 0, S.d_ctr.cap));
  {
    void* rb = S.rb;
    TRY(pinned_reserve(&rb, &S.rb_cap, spectral_words(nap, nc, G) * sizeof(double)));
    S.rb = static_cast<double*>(rb);
  }
  TRY(S.blob.reserve<char>(maps_blob_bytes(N) + fmm_blob_estimate(N, p)));
  TRY(S.cp.blob.reserve<char>(fmm_blob_estimate(N, p)));
  TRY(S.cp.d_ops.reserve<double>(ops_estimate(N)));
  TRY(S.cp.d_maps.reserve<FmmMaps>(kMapSlots));
  {
    void* hm = S.cp.h_maps;
    TRY(pinned_reserve(&hm, &S.cp.h_maps_cap, sizeof(FmmMaps) * kMapSlots));
    S.cp.h_maps = static_cast<FmmMaps*>(hm);
  }
  TRY(S.sec_blob.reserve<char>(size_t(N) * 64 + (size_t(64) << 10)));
  TRY(S.sec_scr.reserve<double>(size_t(3) * size_t(N + 64) * kSecP));
  TRY(S.rot_goff.reserve<int32_t>(size_t(N / 2 + 2)));
  TRY(S.rot_cols.reserve<int32_t>(size_t(N + 1)));
  TRY(S.rot_mats.reserve<double>(size_t(N) * kNumProbes + size_t(kMaxPairTracked) * kMaxPairTracked + 16));
  return SVD1_OK;
}

svd1_status plan_reserve(svd1_plan_t P) {
  const svd1_config& c = P->cfg;
  const int64_t m = c.m, n = c.n;
  const bool thin = (c.flags & SVD1_THIN_V) != 0;
  const int64_t nv = thin ? m + 1 : n;
  const int p = P->p;
  // stream-ordered growth keeps its memory in the pool (no release at synchronisations)
  {
    int dev = 0;
    cudaMemPool_t pool;
    SVD1_CUDA_TRY(cudaGetDevice(&dev));
    SVD1_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t thr = ~uint64_t(0);
    SVD1_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  TRY(ensure_st2(P));
  for (int sd = 2; sd < 6; ++sd) TRY(ensure_side(P, sd));
  const size_t nproj = size_t(5 * m + n + 6);
  TRY(P->W_u.reserve<double>(size_t(c.u_rows) * m));
  TRY(P->W_v.reserve<double>(size_t(c.v_rows) * nv));
  TRY(P->proj.reserve<double>(nproj));
  TRY(P->partial.reserve<double>(size_t(project_partial_elems(c.u_rows, m, c.v_rows, n))));
  TRY(P->probes.reserve<double>(size_t(4 * std::max<int64_t>(c.u_rows, 1))));
  for (int sd = 0; sd < 2; ++sd) TRY(P->tile_ctr[sd].reserve<int>(kMaxPasses));
  TRY(fill_probes(P->probe_seed, c.u_row0, c.u_rows, static_cast<double*>(P->probes.p), P->st, LC(P)));
  P->probes_ready = true;
  // Phi, Psi of both sides for the deepest tree (zeroed: see ensure_expansions)
  for (int side = 0; side < 2; ++side) {
    const size_t e = expansion_elems(side ? c.v_rows : c.u_rows, side ? nv : m, p);
    for (DevBuf* b : {&P->phi[side], &P->psi[side]}) {
      TRY(b->reserve<double>(e));
      SVD1_CUDA_TRY(cudaMemsetAsync(b->p, 0, b->cap, P->st));
    }
  }
  // step records: per-update (steps) and the batch mode's two parities (bsteps)
  for (int e = 0; e < 4; ++e) {
    const int64_t N = e < 2 ? m : nv;
    TRY(reserve_step(P->steps[e], N, p, P->world));
    TRY(reserve_step(P->bsteps[0][e], N, p, P->world));
    TRY(reserve_step(P->bsteps[1][e], N, p, P->world));
  }
  // batch mode (svd1_update_batch): projections, carried rows, few-rows scratch, Gram
  const int ru_max = 4 + (kMaxBatch - 1), rv_max = kMaxBatch - 1;
  TRY(P->bproj.reserve<double>(size_t(kMaxBatch) * nproj));
  for (int q = 0; q < 2; ++q) {
    TRY(P->RU[q].reserve<double>(size_t(ru_max) * m));
    TRY(P->RV[q].reserve<double>(size_t(rv_max) * n));
  }
  TRY(P->few_scr[0].reserve<double>(size_t(few_rows_scratch_elems(ru_max, int(m)))));
  TRY(P->few_scr[1].reserve<double>(size_t(few_rows_scratch_elems(rv_max, int(nv)))));
  TRY(P->bgram.reserve<double>(size_t(kMaxBatch) * kMaxBatch));
  TRY(P->d_rot_goff.reserve<int32_t>(size_t(m / 2 + 2)));
  // pinned host: read-backs and the upload arenas
  {
    void* b = P->h_pin;
    TRY(pinned_reserve(&b, &P->h_pin_cap,
                       (std::max(nproj + size_t(m), size_t(kMaxBatch) * nproj + size_t(m) + size_t(5 * m + n))) *
                           sizeof(double)));
    P->h_pin = static_cast<double*>(b);
  }
  const int64_t Nmax = std::max(m, nv);
  const size_t arena_bytes = std::max<size_t>(size_t(4) << 20, 2 * (size_t(Nmax) * (8 * (4 + kMaxCarry) + 64) +
                                                                   fmm_blob_estimate(Nmax, p) + maps_blob_bytes(Nmax)));
  for (auto& A : P->arena) {
    void* b = A.buf;
    TRY(pinned_reserve(&b, &A.cap, arena_bytes));
    A.buf = static_cast<char*>(b);
    if (!A.ev) SVD1_CUDA_TRY(cudaEventCreateWithFlags(&A.ev, cudaEventDisableTiming));
  }
  SVD1_CUDA_TRY(cudaStreamSynchronize(P->st));
  return SVD1_OK;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

const char* svd1_status_string(svd1_status s) {
  switch (s) {
    case SVD1_OK: return "ok";
    case SVD1_E_INVALID: return "invalid argument";
    case SVD1_E_NONFINITE: return "non-finite input";
    case SVD1_E_NOCONV: return "secular iteration did not converge";
    case SVD1_E_POLE: return "root coincides with a pole";
    case SVD1_E_ZEROCOL: return "zero or non-finite column norm";
    case SVD1_E_CUDA: return "CUDA error";
    case SVD1_E_NOMEM: return "out of memory";
    case SVD1_E_NCCL: return "NCCL error";
  }
  return "unknown status";
}

const char* svd1_version(void) { return "svd1 0.2 (sm_100a, fp64 DMMA)"; }

svd1_status svd1_nccl_unique_id(void* out) {
  if (!out) return SVD1_E_INVALID;
  const NcclApi& A = nccl_api();
  if (!A.ok) return SVD1_E_NCCL;
  ncclUniqueId id;
  NCCL_TRY(A.GetUniqueId(&id));
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(out, &id, sizeof(id));
  return SVD1_OK;
}

svd1_status svd1_plan_create(const svd1_config* cfg, svd1_plan_t* out) {
  if (!cfg || !out) return SVD1_E_INVALID;
  if (cfg->m < 1 || cfg->n < cfg->m || cfg->u_rows < 0 || cfg->v_rows < 0) return SVD1_E_INVALID;
  if (cfg->u_row0 < 0 || cfg->v_row0 < 0 || cfg->u_row0 + cfg->u_rows > cfg->m ||
      cfg->v_row0 + cfg->v_rows > cfg->n)
    return SVD1_E_INVALID;
  if (!(cfg->eps > 0.0 && cfg->eps < 1.0)) return SVD1_E_INVALID;
  const int world = std::max(1, int(cfg->world));
  if (cfg->rank < 0 || cfg->rank >= world) return SVD1_E_INVALID;
  const bool emulate = (cfg->flags & SVD1_EMULATE_RANKS) != 0;
  const bool use_nccl = !emulate && (world > 1 || (cfg->flags & SVD1_FORCE_NCCL));
  if (use_nccl && !cfg->nccl_id) return SVD1_E_INVALID;
  svd1_plan_t P = new (std::nothrow) svd1_plan_s();
  if (!P) return SVD1_E_NOMEM;
  P->cfg = *cfg;
  P->st = static_cast<cudaStream_t>(cfg->stream);
  P->p = choose_p(cfg->eps);
  P->leaf = 2 * P->p;
  P->world = world;
  P->rank = emulate ? 0 : int(cfg->rank);
  P->emulate = emulate && world > 1;
  P->use_nccl = use_nccl;
  if (use_nccl) {  // collective: every rank creates its plan
    const NcclApi& A = nccl_api();
    if (!A.ok) {
      delete P;
      return SVD1_E_NCCL;
    }
    ncclUniqueId id;
    std::memcpy(&id, cfg->nccl_id, sizeof(id));
    ncclResult_t r = A.CommInitRank(&P->comm[0], world, id, int(cfg->rank));
    if (r == ncclSuccess) r = A.CommSplit(P->comm[0], 0, int(cfg->rank), &P->comm[1], nullptr);
    if (r != ncclSuccess) {
      nccl_fail(r, "communicator creation");
      svd1_plan_destroy(P);
      return SVD1_E_NCCL;
    }
  }
  const svd1_status st = plan_reserve(P);
  if (st != SVD1_OK) {
    svd1_plan_destroy(P);
    return st;
  }
  *out = P;
  return SVD1_OK;
}

svd1_status svd1_plan_destroy(svd1_plan_t P) {
  if (!P) return SVD1_E_INVALID;
  for (auto& th : P->launcher)
    if (th.joinable()) th.join();
  cudaStreamSynchronize(P->st);
  if (P->st2) cudaStreamSynchronize(P->st2);
  for (auto& q : P->sp)
    if (q) cudaStreamSynchronize(q);
  if (P->h_pin) cudaFreeHost(P->h_pin);
  for (auto& pe : P->bdone)
    for (auto& e : pe)
      if (e) cudaEventDestroy(e);
  for (auto& e : P->rb_ev)
    if (e) cudaEventDestroy(e);
  for (auto& A : P->arena) {
    if (A.buf) cudaFreeHost(A.buf);
    if (A.ev) cudaEventDestroy(A.ev);
    for (auto& R : A.inflight) cudaEventDestroy(R.ev);
    for (auto e : A.pool) cudaEventDestroy(e);
  }
  for (auto& e : P->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : P->sync_ev)
    if (e) cudaEventDestroy(e);
  if (P->st2) {
    cudaStreamSynchronize(P->st2);
    cudaStreamDestroy(P->st2);
  }
  for (auto& q : P->sp)
    if (q) cudaStreamDestroy(q);
  if (P->st_proj) {
    cudaStreamSynchronize(P->st_proj);
    cudaStreamDestroy(P->st_proj);
  }
  if (P->proj_ev) cudaEventDestroy(P->proj_ev);
  for (auto& cm : P->comm)
    if (cm) nccl_api().CommDestroy(cm);
  delete P;
  return SVD1_OK;
}

svd1_status svd1_project(svd1_plan_t P, const double* U, int64_t ldu, const double* V, int64_t ldv,
                         const double* a, const double* b, double* proj) {
  if (!P || !proj || !a || !b) return SVD1_E_INVALID;
  const svd1_config& c = P->cfg;
  const bool thin = (c.flags & SVD1_THIN_V) != 0;
  if ((c.u_rows && (!U || ldu < c.m)) || (c.v_rows && (!V || ldv < (thin ? c.m + 1 : c.n))))
    return SVD1_E_INVALID;
  double* part;
  const int64_t need = project_partial_elems(c.u_rows, c.m, c.v_rows, c.n);
  TRY(P->partial.get<double>(size_t(need), &part, P->st));
  if (!P->probes_ready) {  // the probes depend only on (seed, global row): once per plan
    double* g;
    TRY(P->probes.get<double>(size_t(4 * std::max<int64_t>(c.u_rows, 1)), &g, P->st));
    TRY(fill_probes(P->probe_seed, c.u_row0, c.u_rows, g, P->st, LC(P)));
    P->probes_ready = true;
  }
  return project(U, ldu, c.u_rows, c.m, c.u_row0, V, ldv, c.v_rows, c.n, c.v_row0, a, b, part, need,
                 proj, static_cast<double*>(P->probes.p), P->st, LC(P), thin ? c.m : c.n);
}

}  // extern "C"

namespace {
// Batch mode context of one update (svd1_update_batch).
struct BatchCtx {
  int parity = 0, t = 0;
  const double* h_proj = nullptr;   // host: [x_a | x_g (4) | y_b | dots] of this update
  std::vector<double>* sig = nullptr;  // in: sigma_t (descending), out: sigma_{t+1}
  int ru_rows = 0, rv_rows = 0;     // carried rows to transform (U: m wide, V: n wide)
  double* h_next = nullptr;         // pinned: read-back of the next update's x_a | x_g | y_b
  double* prev_win = nullptr;       // receives the apply window (ms) of the update two back
  double* prev_gemm = nullptr;      // and its GEMM pass times (4; SVD1_GEMM_EVENTS)
  // thin V (SVD1_THIN_V): b_t (device), y_t = V_t^T b_t (device, first m entries), the
  // Gram matrix of the batch's b's (device, K x K)
  const double* b_dev = nullptr;
  const double* y_dev = nullptr;
  const double* gram = nullptr;
  int K = 0;
  int ru_next = -1, rv_next = -1;   // carried row index of the next update's a / b (-1: none)
  cudaEvent_t rows_wait = nullptr;  // update 0 of svd1_update_batch: the carried rows' initial
                                    // values (project_many) land after this event
};

// carried rows through one step's transform: Householder (in place on `in`), Cauchy
// product of the few rows, passthrough of the deflated columns
svd1_status apply_rows(svd1_plan_t P, StepRecord& S, double* in, double* out, int64_t ld, int rows,
                       cudaStream_t st, int side) {
  if (rows <= 0) return SVD1_OK;
  if (S.h_goff.size() > 1)
    TRY(householder_cols(rows, in, ld, int(S.h_goff.size()) - 1, S.dgoff, S.dhcols, S.dhv, S.h_maxlen(), st,
                         LC(P)));
  if (S.na > 0) {
    double* scr;
    TRY(P->few_scr[side].get<double>(size_t(few_rows_scratch_elems(rows, S.na)), &scr, st));
    TRY(apply_few_rows(rows, S.na, static_cast<double*>(S.d_in.p), static_cast<int32_t*>(S.d_out.p),
                       static_cast<double*>(S.d_out.p) + S.nap, static_cast<double*>(S.d_zhat.p), S.dcs, in, ld,
                       S.dsrc, out, ld, S.ddst, scr, st, LC(P)));
  }
  if (!S.pass_src.empty())
    TRY(passthrough(rows, int(S.pass_src.size()), in, ld, S.dpsrc, out, ld, S.dpdst, S.dpscale, st,
                    LC(P)));
  return SVD1_OK;
}

// expansions are sized at creation for the deepest tree; this only grows them (stream-
// ordered on the side's apply stream, no device synchronisation) if the call's eps is
// smaller than the plan's
svd1_status rare_grow_fn(svd1_plan_t P, StepRecord& Se, int side) {
  if (Se.rows > 0 && Se.na > 0 && cauchy_exp_elems(Se.cp) > P->phi[side].cap / sizeof(double))
    TRY(ensure_expansions(P, side, cauchy_exp_elems(Se.cp)));
  return SVD1_OK;
}

// batch mode: step e's FMM plan on the side's upload stream (never queued behind compute),
// its operator blocks (K5) built there as soon as the plan and the step's maps (column
// scales, with V2's sign alignment) are on the device; the apply stream waits for that work
// and for the maps only.  (This record's ops buffer was last read by the applies of update
// t - 2, which have completed.)
svd1_status upload_step_batch(svd1_plan_t P, StepRecord* S, int e) {
  const int side = e < 2 ? 0 : 1;
  const int par = S == P->bsteps[1] ? 1 : 0;  // (the records' parity: a launcher of update t may
                                              // run while update t + 1 records its own maps)
  TRY(ensure_side(P, side + 4));
  const cudaStream_t as = side_stream(P, side), us = side_stream(P, side + 4);
  SVD1_CUDA_TRY(cudaStreamWaitEvent(as, P->maps_ev[par][e], 0));
  TRY(upload_fmm(P, S[e], side + 4));
  if (S[e].rows > 0 && S[e].na > 0 && S[e].cp.fmm) {
    SVD1_CUDA_TRY(cudaStreamWaitEvent(us, P->maps_ev[par][e], 0));
    TRY(cauchy_build_ops(P, S[e].cp, static_cast<double*>(S[e].d_in.p), static_cast<int32_t*>(S[e].d_out.p),
                         static_cast<double*>(S[e].d_out.p) + S[e].nap, static_cast<double*>(S[e].d_zhat.p),
                         S[e].dcs, us));
    S[e].cp.ops_ready = true;
  }
  return stream_wait(P, e, us, as);
}

// One side's remaining apply launches of a batch update (everything by value: it runs on the
// plan's launcher thread after update_impl has returned): the first apply if it was deferred
// (its input had a Householder group), then, once the second step's plan is ready, the second
// apply (V: pairing rotations), and the events the next updates wait on.
struct SideJob {
  int side = 0, parity = 0, t = 0;
  bool first_done = false;
  StepRecord* S = nullptr;
  double *X = nullptr, *W = nullptr;
  int64_t ldx = 0, ldw = 0;
  cudaStream_t st = nullptr;
  // thin V: the null direction before a deferred first V apply
  bool thin = false;
  int64_t v_rows = 0, m = 0, v_row0 = 0;
  const double *b_dev = nullptr, *y_dev = nullptr;
  double inv_beta = 0.0;
  int nrot = 0;  // V: pairing rotation groups of this update
  int rot_maxk = 0;  // and the largest group's size
  std::string ut;
};
svd1_status side_job(svd1_plan_t P, const SideJob& J) {
  const int e1 = J.side ? 2 : 0, e2 = e1 + 1;
  StepRecord* S = J.S;
  if (!J.first_done) {
    TRY(ev_record(P, J.side ? 18 : 16, J.st));
    TRY(bwin_record(P, J.parity, J.side, J.st));
    if (J.t == 0) TRY(bspan_record(P, J.side, J.st));
    if (J.side && J.thin && J.v_rows)
      TRY(null_direction(J.v_rows, J.X, J.ldx, J.m, J.b_dev, J.v_row0, J.y_dev, J.inv_beta, J.st, LC(P)));
    TRY(apply_launch(P, S[e1], J.X, J.ldx, J.W, J.ldw, 2 * e1, J.st, J.side));
  }
  S[e2].join_plan();
  TRY(rare_grow_fn(P, S[e2], J.side));
  TRY(upload_step_batch(P, S, e2));
  tl_mark(P, J.ut + (J.side ? "V2 apply" : "U2 apply"), J.st);
  TRY(apply_launch(P, S[e2], J.W, J.ldw, J.X, J.ldx, 2 * e2, J.st, J.side));
  if (J.side && J.nrot > 0)
    TRY(col_rotate(S[3].rows, J.X, J.ldx, J.nrot, static_cast<int32_t*>(S[3].rot_goff.p),
                   static_cast<int32_t*>(S[3].rot_cols.p), static_cast<double*>(S[3].rot_mats.p), J.st, LC(P),
                   J.rot_maxk));
  tl_mark(P, J.ut + (J.side ? "V2 end" : "U2 end"), J.st);
  TRY(bwin_record(P, J.parity, 2 + J.side, J.st));
  SVD1_CUDA_TRY(cudaEventRecord(P->bdone[J.parity][J.side], J.st));  // (created by update_impl)
  return SVD1_OK;
}

svd1_status join_launcher(svd1_plan_t P, int side) {
  if (P->launcher[side].joinable()) P->launcher[side].join();
  P->launcher_parity[side] = -1;
  const svd1_status s = P->launcher_status[side];
  P->launcher_status[side] = SVD1_OK;
  return s;
}

// a batch update's apply statistics (its plans complete)
void fill_apply_fields(svd1_report& R, const StepRecord* S) {
  for (int e = 0; e < 4; ++e) {
    const bool has = S[e].rows > 0 && S[e].na > 0;
    R.apply_flops[e] = has ? S[e].cp.flops : 0.0;
    R.apply_flops_exec[e] = has ? S[e].cp.flops_exec : 0.0;
    R.fmm_used[e] = has ? S[e].cp.fmm : 0;
    R.fmm_levels[e] = (has && S[e].cp.fmm) ? S[e].cp.F.L : 0;
    R.fmm_max_near[e] = (has && S[e].cp.fmm) ? S[e].cp.F.max_near : 0;
  }
}

// Rows per chunk of the fused per-side pass: the chunk's U/V rows and W rows (read and
// written) plus the larger step's expansions (Phi, Psi over the tree's non-empty cells)
// within ~64 MB of L2, a multiple of the GEMM's 128-row blocks, at most kMapSlots chunks
// (SVD1_FUSED_ROWS overrides).
int64_t fused_chunk_rows(const StepRecord& S1, const StepRecord& S2, int64_t ldx, int64_t ldw, int64_t rows) {
  static const int64_t env = [] {
    const char* e = std::getenv("SVD1_FUSED_ROWS");
    return e ? std::max<int64_t>(1, atoll(e)) : 0;
  }();
  int64_t rc = env;
  if (!rc) {
    int64_t used = 0;
    for (const StepRecord* S : {&S1, &S2})
      if (S->na > 0 && S->cp.fmm) {
        int64_t u = 0;
        for (const FmmCell& C : S->cp.F.cells) u += C.hi > C.lo;
        used = std::max(used, u * S->cp.p);
      }
    const int64_t per_row = 8 * (ldx + ldw + 2 * used);
    rc = std::max<int64_t>(128, ((int64_t(64) << 20) / std::max<int64_t>(per_row, 1)) / 128 * 128);
  }
  rc = std::max(rc, (rows + kMapSlots - 1) / kMapSlots);
  return std::min(rc, rows);
}

svd1_status update_impl(svd1_plan_t P, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                        const double* proj, double eps, svd1_report* rep, BatchCtx* B,
                        const double* b_dev = nullptr) {
  if (!P || (!B && (!sigma || !proj)) || (B && (!B->h_proj || !B->sig))) return SVD1_E_INVALID;
  const svd1_config& c = P->cfg;
  const int64_t m = c.m, n = c.n;
  // thin right factor: the V side works in the basis [V[:, :m], q] of
  // size nv = m + 1, q = the unit direction of b outside span(V) (column m of V)
  const bool thin = (c.flags & SVD1_THIN_V) != 0;
  const int64_t nv = thin ? m + 1 : n;
  if (B) b_dev = B->b_dev;
  if (thin && ((c.v_rows && !b_dev) || (B && (!B->y_dev || !B->gram)))) return SVD1_E_INVALID;
  if ((c.u_rows && (!U || ldu < m)) || (c.v_rows && (!V || ldv < nv))) return SVD1_E_INVALID;
  if (m > (int64_t(1) << 30) || n > (int64_t(1) << 30)) return SVD1_E_INVALID;
  flush_launches(P);
  const int64_t launches0 = P->launches;
  const int64_t allocs0 = g_allocs.load();
  const double t0 = now_ms();
  if (B) {  // (the rings of the batch streams recycle themselves: no wait here)
  } else {
    TRY(arena_reset(P));
  }
  svd1_report R;
  std::memset(&R, 0, sizeof(R));
  P->p = choose_p(eps > 0.0 ? eps : c.eps);
  R.p = P->p;
  // ---- read back the projections and sigma (one sync); batch mode: given on the host
  const size_t nproj = size_t(5 * m + n + 6);
  double* h;
  if (B) {
    h = const_cast<double*>(B->h_proj);
    if (!all_finite(h, nproj) || !all_finite(B->sig->data(), size_t(m))) return SVD1_E_NONFINITE;
  } else {
    TRY(pinned(P, nproj + size_t(m), &h));
    SVD1_CUDA_TRY(cudaMemcpyAsync(h, proj, nproj * sizeof(double), cudaMemcpyDeviceToHost, P->st));
    SVD1_CUDA_TRY(cudaMemcpyAsync(h + nproj, sigma, size_t(m) * sizeof(double), cudaMemcpyDeviceToHost, P->st));
    SVD1_CUDA_TRY(cudaStreamSynchronize(P->st));
    if (!all_finite(h, nproj + size_t(m))) return SVD1_E_NONFINITE;
  }
  const double* xa = h;
  const double* xg = h + m;
  const double* yb = h + 5 * m;
  const double* ag = h + 5 * m + n;
  const double alpha = ag[4], beta = ag[5];
  std::vector<double> sig = B ? *B->sig : std::vector<double>(h + nproj, h + nproj + m);
  // Reading D10: a run of more than kNumProbes + 2 singular values within
  // 64 eps of each other relative to their size is taken as one repeated value (the run's
  // largest), a backward perturbation of A by <= 64 eps ||A||.  Such a run is otherwise
  // solved as distinct poles whose final columns the probes cannot pair (D5); as a bitwise
  // repetition it deflates (D1) and its columns are paired from their tracked coordinates.
  // (Runs of graded or random spectra are far apart relative to themselves: untouched.)
  for (int64_t i0 = 0; i0 < m;) {
    int64_t i1 = i0 + 1;
    while (i1 < m && sig[i1] > 0.0 &&
           std::fabs(sig[i1 - 1] - sig[i1]) <= 64.0 * kEps * std::max(sig[i1 - 1], sig[i1]))
      ++i1;
    if (i1 - i0 >= kNumProbes + 3 && sig[i0] > 0.0)
      for (int64_t t = i0 + 1; t < i1; ++t) sig[t] = sig[i0];  // (adjacent in the given order)
    i0 = i1;
  }
  R.t_ms[0] = now_ms() - t0;
  if (alpha == 0.0 || beta == 0.0) {  // A_hat = A
    R.noop = 1;
    flush_launches(P);
    R.kernel_launches = P->launches - launches0;
    R.allocations = g_allocs.load() - allocs0;
    if (rep) *rep = R;
    return SVD1_OK;
  }
  // ---- STEPS 2-3: Schur splits; Q2: right side uses rho3, rho4
  // D9: per-side balance of the rank-1 term, ||b~|| = ||Sigma V^T b||, ||a~|| = ||Sigma^T U^T a||
  double bt2 = 0.0, at2 = 0.0;
  for (int64_t i = 0; i < m; ++i) {
    bt2 += (sig[i] * yb[i]) * (sig[i] * yb[i]);
    at2 += (sig[i] * xa[i]) * (sig[i] * xa[i]);
  }
  const double c_u = balance_factor(std::sqrt(bt2), std::sqrt(alpha));
  const double c_v = balance_factor(std::sqrt(beta), std::sqrt(at2));
  const Split su = schur_split(beta / (c_u * c_u)), sv = schur_split(alpha * (c_v * c_v));
  // small vectors in the U and V column bases (B7 identities):
  // U^T b~ = Sigma (V^T b)[:m],  V^T a~ = Sigma^T (U^T a)
  std::vector<double> z1(m), Du(m), z3(nv), Dv(nv, 0.0);
  std::vector<std::vector<double>> cu, cv;
  cu.emplace_back(m);
  cv.emplace_back(nv);
  for (int q = 0; q < kNumProbes; ++q) {
    cu.emplace_back(xg + q * m, xg + (q + 1) * m);
    cv.emplace_back(nv, 0.0);
  }
  for (int64_t i = 0; i < m; ++i) {
    const double sx = sig[i] * yb[i] / c_u, xu = c_u * xa[i];  // (D9)
    z1[i] = su.q00 * xu + su.q10 * sx;     // U^T a1, [a b~] Q_u = [a1 b1]
    cu[0][i] = su.q01 * xu + su.q11 * sx;  // U^T b1
    Du[i] = sig[i] * sig[i];
    Dv[i] = Du[i];
  }
  // thin: the coordinate of b along q is beta_perp = ||b - V V^T b|| (a~ = A^T a has none)
  double beta_perp = 0.0;
  if (thin) {
    double yy = 0.0;
    for (int64_t i = 0; i < m; ++i) yy += yb[i] * yb[i];
    const double r2 = beta - yy;
    beta_perp = r2 > 64.0 * kEps * beta ? std::sqrt(r2) : 0.0;  // b in span(V): no null part
  }
  for (int64_t i = 0; i < nv; ++i) {
    const double sxa = i < m ? sig[i] * xa[i] : 0.0;
    const double ybi = thin && i == m ? beta_perp : yb[i];
    z3[i] = sv.q00 * (ybi / c_v) + sv.q10 * (c_v * sxa);     // V^T a2, [b a~] Q_v = [a2 b2] (D9)
    cv[0][i] = sv.q01 * (ybi / c_v) + sv.q11 * (c_v * sxa);  // V^T b2
    for (int q = 0; q < kNumProbes; ++q)     // V^T A_hat^T g = Sigma^T U^T g + (V^T b)(a.g)
      cv[1 + q][i] = (i < m ? sig[i] * xg[q * m + i] : 0.0) + ybi * ag[q];
  }
  // ---- workspaces for the applies (sized up front: a mid-stream realloc would sync)
  TRY(ensure_st2(P));
  double *Wu = nullptr, *Wv = nullptr;
  if (c.u_rows) TRY(P->W_u.get<double>(size_t(c.u_rows) * m, &Wu, P->st));  // sized at creation
  if (c.v_rows) TRY(P->W_v.get<double>(size_t(c.v_rows) * nv, &Wv, P->st2));
  // expansions for the deepest tree the planner can choose at this p (sized at creation
  // for the plan's eps; a smaller eps per call grows them once, stream-ordered)
  TRY(ensure_expansions(P, 0, expansion_elems(c.u_rows, m, P->p)));
  TRY(ensure_expansions(P, 1, expansion_elems(c.v_rows, nv, P->p)));
  const bool one_stream = !B && std::getenv("SVD1_ONE_STREAM") != nullptr;  // diagnostics
  const bool fused = (c.flags & SVD1_FUSED_SIDE) != 0;
  // spectral work and uploads: the apply streams' sides (0, 1), or in batch mode the
  // spectral streams (2, 3), so the next update's spectral phase is not queued behind
  // this update's applies
  const int sp0 = B ? 2 : 0, sp1 = B ? 3 : (one_stream ? 0 : 1);
  if (B) {
    TRY(ensure_side(P, 2));
    TRY(ensure_side(P, 3));
  }
  cudaStream_t stv = one_stream ? P->st : P->st2;
  // ---- spectral phase.  Each side is a chain on its own stream (U: the plan stream,
  // V: st2): STEP 4 -> STEP 5 and STEP 6 -> STEP 7.  The chains are
  // interleaved on the host, so each side's host step (finish one eigen-update, launch
  // the next) overlaps the other side's GPU work; the FMM plan of each apply is built on
  // a worker thread as soon as its eigen-update is known, and a first apply whose input
  // is not transformed in place (no Householder group) starts as soon as it is planned:
  // it writes only the workspace W, so U, Sigma and V stay untouched until every
  // eigen-update has succeeded.
  const double t1 = now_ms();
  StepRecord* S = B ? P->bsteps[B->parity] : P->steps;
  if (B)  // launchers still holding this parity's records (update t - 2 when t - 1 was a no-op)
    for (int sd = 0; sd < 2; ++sd)
      if (P->launcher_parity[sd] == B->parity) TRY(join_launcher(P, sd));
  if (B && P->bdone_rec[B->parity]) {  // the applies that last used these records are done
    SVD1_CUDA_TRY(cudaEventSynchronize(P->bdone[B->parity][0]));
    SVD1_CUDA_TRY(cudaEventSynchronize(P->bdone[B->parity][1]));
    P->bdone_rec[B->parity] = false;
    if (B->prev_win) *B->prev_win = bwin_ms(P, B->parity);
    if (B->prev_gemm)
      for (int e = 0; e < 4; ++e)
        B->prev_gemm[e] = (S[e].rows > 0 && S[e].na > 0 && S[e].cp.fmm) ? S[e].cp.gemm_ms() : 0.0;
  }
  {
    std::vector<double> zu = z1, zv = z3;
    std::vector<std::vector<double>> cu1(cu.begin() + 1, cu.end()), cv1(cv.begin() + 1, cv.end());
    // carry 0 = the chained vector U^T b1 / V^T b2, carries 1.. = probes
    cu1.insert(cu1.begin(), cu[0]);
    cv1.insert(cv1.begin(), cv[0]);
    cu.swap(cu1);
    cv.swap(cv1);
    z1.swap(zu);
    z3.swap(zv);
  }
  // D5 for clusters larger than the probes: a singular value repeated k >= kNumProbes + 3
  // times in Sigma keeps k - 2 copies after the update, in bases the two sides choose
  // independently.  Those columns are deflated ones: their coordinates over the original
  // group's columns follow from the deflation reflections and the merges alone (host-only
  // carries gcu / gcv, unit vectors of the group's original columns), and since
  // A V_G = sigma U_G and the deflated columns are orthogonal to U_G^T a and V_G^T b,
  // U_c^T A_hat V_c = sigma Tu^T Tv (see the pairing below).  At most kMaxPairTracked columns.
  std::vector<std::vector<double>> gcu, gcv;
  std::vector<int32_t> gidx;
  {
    int64_t i0 = 0;
    while (i0 < m) {
      int64_t i1 = i0 + 1;
      while (i1 < m && sig[i1] == sig[i0]) ++i1;
      if (i1 - i0 >= kNumProbes + 3 && sig[i0] > 0.0) {
        if (int64_t(gidx.size()) + (i1 - i0) > kMaxPairTracked) return SVD1_E_UNSUPPORTED;  // nothing written yet
        for (int64_t g = i0; g < i1; ++g) gidx.push_back(int32_t(g));
      }
      i0 = i1;
    }
    for (int32_t g : gidx) {
      gcu.emplace_back(m, 0.0);
      gcu.back()[g] = 1.0;
      gcv.emplace_back(nv, 0.0);
      gcv.back()[g] = 1.0;
    }
    for (int e = 0; e < 4; ++e) S[e].gcar = gidx.empty() ? nullptr : (e < 2 ? &gcu : &gcv);
  }
  const double tA = now_ms();
  const svd1_config pcfg = P->cfg;
  const int pp = P->p;
  // plan threads still running if an error returns early are joined here (they touch only
  // plan-owned step records)
  struct PlanJoin {
    StepRecord* S;
    bool active = true;
    ~PlanJoin() {
      if (active)
        for (int e = 0; e < 4; ++e) S[e].join_plan();
    }
  };
  PlanJoin plan_join_on_error{S};
  auto rare_grow = [&](int e, int side) -> svd1_status { return rare_grow_fn(P, S[e], side); };
  // Host scheduler of the two chains: each round takes the first ready action in
  // priority order — launch a planned first apply (GPU work as early as possible), then
  // finish an eigen-update whose read-back has landed (and launch its successor / start
  // its plan on a worker thread).  Readiness is polled (cudaEventQuery, atomic flags),
  // so neither side's host step waits behind the other side's GPU work.
  auto spawn_plan = [&](int e, bool reverse, int64_t rows) {
    StepRecord* Se = &S[e];
    Se->join_plan();
    set_out_cols(*Se, rows, reverse);
    Se->planned.store(false, std::memory_order_relaxed);
    Se->plan_thread = WorkThread([Se, pcfg, pp] {
      apply_plan(pcfg, pp, *Se);
      Se->planned.store(true, std::memory_order_release);
    });
  };
  auto landed = [&](int e) {
    if (!S[e].pending) return true;
    const cudaError_t q = cudaEventQuery(S[e].done_ev);
    if (q == cudaErrorNotReady) return false;
    return true;  // success, or an error that spectral_finish reports
  };
  bool fin[4] = {false, false, false, false};
  bool launched_u1 = false, launched_v1 = false, uploaded_u1 = false, uploaded_v1 = false;
  double t_fin[4] = {0, 0, 0, 0}, t_dbg[4] = {0, 0, 0, 0};
  auto nrot_v = [&]() { return c.v_rows > 0 ? int(P->rot_goff.size()) - 1 : 0; };
  auto rot_maxk = [&]() {
    int mk = 0;
    for (size_t g = 0; g + 1 < P->rot_goff.size(); ++g) mk = std::max(mk, P->rot_goff[g + 1] - P->rot_goff[g]);
    return mk;
  };
  auto upload_rot = [&](int us) -> svd1_status {  // pairing rotations (set before step 3's upload)
    if (nrot_v() <= 0) return SVD1_OK;
    int32_t *g, *cl;
    double* mt;
    TRY(upload(P, S[3].rot_goff, P->rot_goff, &g, us));
    TRY(upload(P, S[3].rot_cols, P->rot_cols, &cl, us));
    TRY(upload(P, S[3].rot_mats, P->rot_mats, &mt, us));
    return SVD1_OK;
  };
  // batch mode, as soon as step e's eigen-update is known (no plan needed): its column
  // maps on its spectral stream, and the carried projection rows of later updates
  // through the step's transform there (apply_rows); after the second step of a side
  // the next update's rows are read back, so the next update can start while this
  // one's applies are still being planned and launched
  auto rows_step = [&](int e) -> svd1_status {
    const int side = e < 2 ? 0 : 1;
    const int us = side + 2;
    const cudaStream_t ss = side_stream(P, us);
    TRY(upload_maps(P, S[e], us));
    if (e == 3) TRY(upload_rot(us));
    cudaEvent_t& mev = P->maps_ev[B->parity][e];
    if (!mev) SVD1_CUDA_TRY(cudaEventCreateWithFlags(&mev, cudaEventDisableTiming));
    SVD1_CUDA_TRY(cudaEventRecord(mev, ss));
    DevBuf* R = side ? P->RV : P->RU;
    const int rows = side ? B->rv_rows : B->ru_rows;
    const int64_t ld = side ? nv : m;
    const bool second = e == 1 || e == 3;  // R[0] -> R[1] (first step), R[1] -> R[0]
    double* rin = static_cast<double*>(R[second ? 1 : 0].p);
    double* rout = static_cast<double*>(R[second ? 0 : 1].p);
    if (B->rows_wait) SVD1_CUDA_TRY(cudaStreamWaitEvent(ss, B->rows_wait, 0));
    if (thin && e == 2)  // the later b's coordinates along this update's q
      TRY(thin_carry(rows, rin, ld, m, B->y_dev, B->gram, B->t, B->K, beta_perp > 0.0 ? 1.0 / beta_perp : 0.0,
                     ss, LC(P)));
    TRY(apply_rows(P, S[e], rin, rout, ld, rows, ss, side));
    if (e == 3 && rows > 0 && nrot_v() > 0)
      TRY(col_rotate(rows, rout, ld, nrot_v(), static_cast<int32_t*>(S[3].rot_goff.p),
                     static_cast<int32_t*>(S[3].rot_cols.p), static_cast<double*>(S[3].rot_mats.p), ss,
                     LC(P), rot_maxk()));
    if (second) {  // read back the next update's rows: x_a | x_g (U side), y_b (V side)
      if (!P->rb_ev[side]) SVD1_CUDA_TRY(cudaEventCreateWithFlags(&P->rb_ev[side], cudaEventDisableTiming));
      if (side == 0 && B->ru_next >= 0) {
        SVD1_CUDA_TRY(cudaMemcpyAsync(B->h_next, rout + int64_t(B->ru_next) * m, m * sizeof(double),
                                      cudaMemcpyDeviceToHost, ss));
        SVD1_CUDA_TRY(cudaMemcpyAsync(B->h_next + m, rout, 4 * m * sizeof(double), cudaMemcpyDeviceToHost, ss));
      }
      if (side == 1 && B->rv_next >= 0)  // (thin: the first m entries; the rest stays 0)
        SVD1_CUDA_TRY(cudaMemcpyAsync(B->h_next + 5 * m, rout + int64_t(B->rv_next) * ld,
                                      (thin ? m : n) * sizeof(double), cudaMemcpyDeviceToHost, ss));
      SVD1_CUDA_TRY(cudaEventRecord(P->rb_ev[side], ss));
    }
    return SVD1_OK;
  };
  // upload step e's apply data (batch mode: its FMM plan on the side's upload stream,
  // which never queues behind compute; the apply stream waits for that copy and for the
  // step's maps, not for the spectral work queued after them)
  auto upload_step = [&](int e) -> svd1_status {
    const int side = e < 2 ? 0 : 1;
    if (!B) return apply_upload(P, S[e], one_stream ? 0 : side);
    return upload_step_batch(P, S, e);
  };
  // thin V: column m of V <- q before the first V apply reads it (V side's apply stream)
  auto null_dir = [&]() -> svd1_status {
    if (!thin || !c.v_rows) return SVD1_OK;
    return null_direction(c.v_rows, V, ldv, m, b_dev, c.v_row0, B ? B->y_dev : proj + 5 * m,
                          beta_perp > 0.0 ? 1.0 / beta_perp : 0.0, stv, LC(P));
  };
  // Fused per-side pass (SVD1_FUSED_SIDE): once both steps
  // of a side are planned, the side's rows go through X1 then X2 in chunks sized so that a
  // chunk's U/V rows, its W rows and its expansions stay in L2: U and V are read and written
  // once per update instead of twice.  Per chunk: Householder (step 1) on the chunk's rows,
  // apply 1, passthrough 1, Householder (step 2), apply 2, passthrough 2 (V: pairing
  // rotations); the operator blocks are built once per step.
  auto fused_side = [&](int side) -> svd1_status {
    const int e1 = side ? 2 : 0, e2 = e1 + 1;
    const cudaStream_t st = side ? stv : P->st;
    double* X = side ? V : U;
    const int64_t ldx = side ? ldv : ldu;
    double* Wb = side ? Wv : Wu;
    const int64_t ldw = side ? nv : m;
    const int64_t rows = side ? c.v_rows : c.u_rows;
    if (rows <= 0) return SVD1_OK;
    TRY(ev_record(P, side ? 18 : 16, st));
    if (B) TRY(bwin_record(P, B->parity, side, st));
    if (B && B->t == 0) TRY(bspan_record(P, side, st));
    if (side) TRY(null_dir());
    TRY(ev_record(P, 2 * e1, st));
    const int64_t rc = fused_chunk_rows(S[e1], S[e2], ldx, ldw, rows);
    int slot = 0;
    for (int64_t r0 = 0; r0 < rows; r0 += rc, ++slot) {
      const int64_t nr = std::min(rc, rows - r0);
      const bool last = r0 + nr >= rows;
      TRY(apply_chunk(P, S[e1], X, ldx, Wb, ldw, r0, nr, st, side, slot, last));
      TRY(apply_chunk(P, S[e2], Wb, ldw, X, ldx, r0, nr, st, side, slot, last));
      if (side && nrot_v() > 0)
        TRY(col_rotate(nr, X + r0 * ldx, ldx, nrot_v(), static_cast<int32_t*>(S[3].rot_goff.p),
                       static_cast<int32_t*>(S[3].rot_cols.p), static_cast<double*>(S[3].rot_mats.p), st,
                       LC(P), rot_maxk()));
    }
    // the side's whole time is reported on its first step (apply_ms[e1]); the second's is 0
    TRY(ev_record(P, 2 * e1 + 1, st));
    TRY(ev_record(P, 2 * e2, st));
    TRY(ev_record(P, 2 * e2 + 1, st));
    return SVD1_OK;
  };
  auto first_apply = [&](int e) -> svd1_status {  // upload (+ launch when nothing in place)
    const int side = e == 0 ? 0 : 1;
    TRY(rare_grow(e, side));
    TRY(upload_step(e));
    if (!fused && S[e].h_goff.size() <= 1) {  // nothing transformed in place: start now
      if (e == 0) {
        TRY(ev_record(P, 16, P->st));
        if (B) TRY(bwin_record(P, B->parity, 0, P->st));
        if (B && B->t == 0) TRY(bspan_record(P, 0, P->st));
        tl_mark(P, (B ? "u" + std::to_string(B->t) : std::string()) + " U1 apply", P->st);
        TRY(apply_launch(P, S[0], U, ldu, Wu, m, 0, P->st, 0));
        launched_u1 = true;
      } else {
        TRY(ev_record(P, 18, stv));
        if (B) TRY(bwin_record(P, B->parity, 1, stv));
        if (B && B->t == 0) TRY(bspan_record(P, 1, stv));
        tl_mark(P, (B ? "u" + std::to_string(B->t) : std::string()) + " V1 apply", stv);
        TRY(null_dir());
        TRY(apply_launch(P, S[2], V, ldv, Wv, nv, 4, stv, 1));
        launched_v1 = true;
      }
    }
    return SVD1_OK;
  };
  // The two sides' chains (U: STEP 4 -> STEP 5, V: STEP 6 -> STEP 7) are
  // independent until the sign alignment: each runs on its own host thread (the V side on
  // a second thread), so one side's host work (sort / deflation / secular-FMM plan before a
  // launch, merge and maps after a read-back) overlaps the other side's, and each polls
  // only its own readiness (cudaEventQuery, atomic plan flags).  Per side: launch step 1;
  // when its read-back lands, finish it (host merge), start its FMM plan on a worker
  // thread, transform the carried rows (batch mode), launch step 2; launch the first apply
  // as soon as its plan is ready; finish step 2 and start its plan.
  const std::string ut = B ? "u" + std::to_string(B->t) + " " : "";
  auto chain = [&](int side) -> svd1_status {
    const int e1 = side ? 2 : 0, e2 = e1 + 1;
    const int sps = side ? sp1 : sp0;
    std::vector<double>& Dd = side ? Dv : Du;
    std::vector<std::vector<double>>& cc = side ? cv : cu;
    bool& uploaded = side ? uploaded_v1 : uploaded_u1;
    const int64_t rows = side ? c.v_rows : c.u_rows;
    const double rho1 = side ? sv.rho1 : su.rho1, rho2 = side ? sv.rho2 : su.rho2;
    const char* nm = side ? "V" : "U";
    tl_mark(P, ut + nm + "1 spectral", side_stream(P, sps));
    TRY(spectral_launch(P, S[e1], Dd, side ? z3 : z1, rho1, cc, side ? 12 : 8, sps, side));
    while (!landed(e1)) std::this_thread::yield();
    t_dbg[side ? 3 : 0] = now_ms();
    TRY(spectral_finish(P, S[e1], Dd, cc));
    fin[e1] = true;
    spawn_plan(e1, false, rows);
    if (B) TRY(rows_step(e1));
    {
      std::vector<double> z2 = cc[0];
      cc.erase(cc.begin());
      tl_mark(P, ut + nm + "1 finished; " + nm + "2 spectral", side_stream(P, sps));
      TRY(spectral_launch(P, S[e2], Dd, z2, rho2, cc, side ? 14 : 10, sps, side));
    }
    t_fin[e1] = now_ms();
    while (!fin[e2]) {
      if (!uploaded && S[e1].planned.load(std::memory_order_acquire)) {
        S[e1].join_plan();
        if (B) TRY(join_launcher(P, side));  // the previous update's launches on this side first
        TRY(first_apply(e1));
        uploaded = true;
        continue;
      }
      if (landed(e2)) {
        TRY(spectral_finish(P, S[e2], Dd, cc));
        fin[e2] = true;
        tl_mark(P, ut + nm + "2 finished", nullptr, false);
        spawn_plan(e2, true, rows);
        if (B && side == 0) TRY(rows_step(1));  // (V2's rows need the sign alignment)
        t_fin[e2] = now_ms();
        continue;
      }
      std::this_thread::yield();
    }
    if (!uploaded) {
      S[e1].join_plan();
      if (B) TRY(join_launcher(P, side));
      TRY(first_apply(e1));
      uploaded = true;
    }
    return SVD1_OK;
  };
  // U-side applies (they need every eigen-update to have succeeded -- the factors stay
  // untouched on a numerical error -- but not the sign alignment, which only scales V2's
  // columns): launched from the U thread as soon as the V chain has finished.
  auto u_applies = [&]() -> svd1_status {
    if (fused) {  // both steps of the side row chunk by row chunk (§4.11)
      S[1].join_plan();
      TRY(rare_grow(1, 0));
      TRY(upload_step(1));
      TRY(fused_side(0));
    } else {
      if (!launched_u1) {  // (its input had a Householder group: deferred to here)
        TRY(ev_record(P, 16, P->st));
        if (B) TRY(bwin_record(P, B->parity, 0, P->st));
        if (B && B->t == 0) TRY(bspan_record(P, 0, P->st));
        TRY(apply_launch(P, S[0], U, ldu, Wu, m, 0, P->st, 0));
      }
      S[1].join_plan();
      TRY(rare_grow(1, 0));
      TRY(upload_step(1));
      tl_mark(P, ut + "U2 apply", P->st);
      TRY(apply_launch(P, S[1], Wu, m, U, ldu, 2, P->st, 0));
    }
    if (B) {
      tl_mark(P, ut + "U2 end", P->st);
      TRY(bwin_record(P, B->parity, 2, P->st));
      if (!P->bdone[B->parity][0])
        SVD1_CUDA_TRY(cudaEventCreateWithFlags(&P->bdone[B->parity][0], cudaEventDisableTiming));
      SVD1_CUDA_TRY(cudaEventRecord(P->bdone[B->parity][0], P->st));
    }
    return SVD1_OK;
  };
  // U chain + U applies on a second host thread, V chain here; the sign alignment (below)
  // waits for both chains' spectral results.  States: 0 running, 1 succeeded, 2 failed.
  std::atomic<int> u_state{0}, v_state{0};
  svd1_status st_u = SVD1_OK, st_ua = SVD1_OK;
  Joiner u_thread;
  if (one_stream) {  // (diagnostics: both chains on one stream and one arena -> one thread)
    st_u = chain(0);
    u_state = st_u == SVD1_OK ? 1 : 2;
  } else {
    u_thread.add(WorkThread([&] {
      st_u = chain(0);
      u_state.store(st_u == SVD1_OK ? 1 : 2, std::memory_order_release);
      if (st_u == SVD1_OK) {
        int v;
        while ((v = v_state.load(std::memory_order_acquire)) == 0) std::this_thread::yield();
        if (v == 1 && (!B || fused)) st_ua = u_applies();  // (batch: the U launcher, below)
      }
      flush_launches(P);
    }));
  }
  {
    const svd1_status st_v = chain(1);
    v_state.store(st_v == SVD1_OK ? 1 : 2, std::memory_order_release);
    while (u_state.load(std::memory_order_acquire) == 0) std::this_thread::yield();
    if (st_v != SVD1_OK || st_u != SVD1_OK) {
      u_thread.join();
      TRY(st_u);
      return st_v;
    }
  }
  // batch mode: the U side's remaining apply launches (a deferred first apply, the second
  // apply once its plan is ready) go to the U launcher thread now -- every eigen-update has
  // succeeded -- so neither this update's return nor the next update's spectral chain waits
  // for the U2 plan
  const bool launchers = B && !fused && !one_stream;
  if (launchers) {
    u_thread.join();  // (the U chain is done; its thread only ran the chain in this mode)
    TRY(join_launcher(P, 0));
    SideJob ju;
    ju.side = 0;
    ju.parity = B->parity;
    ju.t = B->t;
    ju.first_done = launched_u1;
    ju.S = S;
    ju.X = U;
    ju.ldx = ldu;
    ju.W = Wu;
    ju.ldw = m;
    ju.st = P->st;
    ju.ut = ut;
    if (!P->bdone[B->parity][0])
      SVD1_CUDA_TRY(cudaEventCreateWithFlags(&P->bdone[B->parity][0], cudaEventDisableTiming));
    P->launcher_parity[0] = B->parity;
    P->launcher[0] = WorkThread([P, ju] {
      P->launcher_status[0] = side_job(P, ju);
      flush_launches(P);
    });
  }
  if (std::getenv("SVD1_TIMING"))
    fprintf(stderr, "[svd1] host: launch1 %.3f finished U1 %.3f U2 %.3f V1 %.3f V2 %.3f (plans %.3f %.3f) U1 landed %.3f finish %.3f spawn %.3f\n",
            tA - t1, t_fin[0] - t1, t_fin[1] - t1, t_fin[2] - t1, t_fin[3] - t1, S[0].plan_ms, S[2].plan_ms,
            t_dbg[0] - t1, t_dbg[1] - t1, t_dbg[2] - t1);
  const double t3 = now_ms();
  R.t_ms[1] = t3 - t1;
  // ---- sign alignment: final column i = position N-1-i
  std::vector<double> sgn(m, 1.0);
  for (int64_t i = 0; i < m; ++i) {
    const int64_t qu = m - 1 - i, qv = nv - 1 - i;
    int kb = 0;
    double best = -1.0;
    for (int q = 0; q < kNumProbes; ++q)
      if (std::fabs(cu[q][qu]) > best) {
        best = std::fabs(cu[q][qu]);
        kb = q;
      }
    if (cu[kb][qu] * cv[kb][qv] < 0.0) {
      sgn[i] = -1.0;
      ++R.sign_flips;
    }
  }
  // Exactly (or numerically) repeated final singular values: the U- and V-side bases
  // of that singular subspace are computed independently, so the sign rule is
  // generalised to a k x k pairing rotation (DESIGN.md §3.2 D5): with probes,
  // q_c = M^T p_c for M = U_c^T A_hat V_c = sigma W, so M^T = Q P^T (P P^T)^-1 from the
  // 4 probes, W = orthonormalised M / sigma, and V_c <- V_c W^T after the last apply.
  P->rot_goff.assign(1, 0);
  P->rot_cols.clear();
  P->rot_mats.clear();
  {
    const double dmax = std::max(Du[m - 1], 0.0);
    const double tolc = 64.0 * kEps * dmax;
    // a cluster (gaps <= 64 eps D_1) whose gaps are also within 64 eps of its own values: its
    // columns are not determined one by one (a graded tail's clusters are: its relative gaps
    // are far above eps, and the solver's relative accuracy fixes each column up to sign)
    auto self_near = [&](int64_t a0, int64_t a1) {
      for (int64_t t = a0 + 1; t < a1; ++t)
        if (Du[m - 1 - (t - 1)] - Du[m - 1 - t] > 64.0 * kEps * Du[m - 1 - (t - 1)]) return false;
      return true;
    };
    int64_t i0 = 0;
    while (i0 < m) {
      int64_t i1 = i0 + 1;
      while (i1 < m && Du[m - 1 - (i1 - 1)] - Du[m - 1 - i1] <= tolc) ++i1;
      const int k = int(i1 - i0);
      if (k >= 2 && k <= kNumProbes && Du[m - 1 - i0] > 0.0) {
        // P (k x K), Q (k x K)
        double Pm[kNumProbes][kNumProbes], Qm[kNumProbes][kNumProbes];
        for (int a = 0; a < k; ++a)
          for (int q = 0; q < kNumProbes; ++q) {
            Pm[a][q] = cu[q][m - 1 - (i0 + a)];
            Qm[a][q] = cv[q][nv - 1 - (i0 + a)];
          }
        double G[kNumProbes][2 * kNumProbes], H[kNumProbes][kNumProbes];
        for (int a = 0; a < k; ++a)
          for (int b = 0; b < k; ++b) {
            double g = 0.0, h = 0.0;
            for (int q = 0; q < kNumProbes; ++q) {
              g += Pm[a][q] * Pm[b][q];
              h += Qm[a][q] * Pm[b][q];
            }
            G[a][b] = g;
            G[a][k + b] = (a == b) ? 1.0 : 0.0;
            H[a][b] = h;
          }
        // G^-1 by Gauss-Jordan with partial pivoting (k <= 4)
        bool ok = true;
        for (int c2 = 0; c2 < k && ok; ++c2) {
          int piv = c2;
          for (int r2 = c2 + 1; r2 < k; ++r2)
            if (std::fabs(G[r2][c2]) > std::fabs(G[piv][c2])) piv = r2;
          if (G[piv][c2] == 0.0) {
            ok = false;
            break;
          }
          if (piv != c2)
            for (int t = 0; t < 2 * k; ++t) std::swap(G[piv][t], G[c2][t]);
          const double inv = 1.0 / G[c2][c2];
          for (int t = 0; t < 2 * k; ++t) G[c2][t] *= inv;
          for (int r2 = 0; r2 < k; ++r2)
            if (r2 != c2) {
              const double f = G[r2][c2];
              for (int t = 0; t < 2 * k; ++t) G[r2][t] -= f * G[c2][t];
            }
        }
        if (ok) {
          // M^T = H G^-1 ;  W = M / sigma  -> columns of W: W[:, b] = (M^T)[b, :]
          double W[kNumProbes][kNumProbes];
          const double sig_c = std::sqrt(Du[m - 1 - i0]);
          for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) {
              double mt = 0.0;  // (M^T)[a][b]
              for (int t = 0; t < k; ++t) mt += H[a][t] * G[t][k + b];
              W[b][a] = mt / sig_c;  // M[b][a]
            }
          // modified Gram-Schmidt on the columns of W (W ~ orthogonal)
          for (int b = 0; b < k; ++b) {
            for (int b2 = 0; b2 < b; ++b2) {
              double dot = 0.0;
              for (int a = 0; a < k; ++a) dot += W[a][b] * W[a][b2];
              for (int a = 0; a < k; ++a) W[a][b] -= dot * W[a][b2];
            }
            double nr = 0.0;
            for (int a = 0; a < k; ++a) nr += W[a][b] * W[a][b];
            nr = std::sqrt(nr);
            for (int a = 0; a < k; ++a) W[a][b] /= nr;
          }
          // V_c <- V_c W^T : new col b = sum_a old col a * W[b][a]; stored row-major
          // as R[a][b] = W[b][a] (the kernel computes out[b] = sum_a in[a] R[a][b])
          for (int a = 0; a < k; ++a) {
            P->rot_cols.push_back(int32_t(i0 + a));
            sgn[i0 + a] = 1.0;  // the rotation carries the sign
          }
          for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) P->rot_mats.push_back(W[b][a]);
          P->rot_goff.push_back(int32_t(P->rot_cols.size()));
          ++R.pair_rotations;
        }
      } else if (k > kNumProbes && !gidx.empty() && Du[m - 1 - i0] > 0.0) {
        // W = Tu^T Tv from the tracked coordinates (Tu[g][a]: original U column g in final
        // column i0 + a); used only if every cluster column lies in the tracked span
        const int ng = int(gidx.size());
        bool inside = true;
        for (int a = 0; a < k && inside; ++a) {
          double nu = 0.0, nvv = 0.0;
          for (int g = 0; g < ng; ++g) {
            nu += gcu[g][m - 1 - (i0 + a)] * gcu[g][m - 1 - (i0 + a)];
            nvv += gcv[g][nv - 1 - (i0 + a)] * gcv[g][nv - 1 - (i0 + a)];
          }
          inside = std::fabs(nu - 1.0) <= 1e-8 && std::fabs(nvv - 1.0) <= 1e-8;
        }
        if (inside) {
          std::vector<double> W(size_t(k) * k);  // W[b * k + a] = M[b][a] / sigma
          for (int b = 0; b < k; ++b)
            for (int a = 0; a < k; ++a) {
              double t = 0.0;
              for (int g = 0; g < ng; ++g) t += gcu[g][m - 1 - (i0 + b)] * gcv[g][nv - 1 - (i0 + a)];
              W[size_t(b) * k + a] = t;
            }
          for (int b = 0; b < k; ++b) {  // modified Gram-Schmidt on the columns (index b)
            for (int b2 = 0; b2 < b; ++b2) {
              double dot = 0.0;
              for (int a = 0; a < k; ++a) dot += W[size_t(a) * k + b] * W[size_t(a) * k + b2];
              for (int a = 0; a < k; ++a) W[size_t(a) * k + b] -= dot * W[size_t(a) * k + b2];
            }
            double nr = 0.0;
            for (int a = 0; a < k; ++a) nr += W[size_t(a) * k + b] * W[size_t(a) * k + b];
            nr = std::sqrt(nr);
            for (int a = 0; a < k; ++a) W[size_t(a) * k + b] /= nr;
          }
          for (int a = 0; a < k; ++a) {
            P->rot_cols.push_back(int32_t(i0 + a));
            sgn[i0 + a] = 1.0;
          }
          for (int a = 0; a < k; ++a)
            for (int b = 0; b < k; ++b) P->rot_mats.push_back(W[size_t(b) * k + a]);
          P->rot_goff.push_back(int32_t(P->rot_cols.size()));
          ++R.pair_rotations;
        } else if (self_near(i0, i1)) {
          ++R.unpaired_clusters;
        }
      } else if (k > kNumProbes && Du[m - 1 - i0] > 0.0 && self_near(i0, i1)) {
        ++R.unpaired_clusters;
      }
      i0 = i1;
    }
  }
  for (int e = 0; e < 4; ++e) S[e].gcar = nullptr;
  for (int j = 0; j < S[3].na; ++j) {
    const int64_t col = nv - 1 - S[3].tgt_pos[j];
    if (col < m) S[3].cs_h[j] *= sgn[col];
  }
  for (size_t q = 0; q < S[3].pass_dst.size(); ++q) {
    const int64_t col = nv - 1 - S[3].pass_dst[q];
    if (col < m) S[3].pass_scale[q] *= sgn[col];
  }
  R.sign_flips = 0;
  for (int64_t i = 0; i < m; ++i) R.sign_flips += sgn[i] < 0.0;
  if (B) TRY(rows_step(3));  // V2 maps carry the sign alignment and pairing rotations
  // ---- STEP 8: sigma = sqrt(max(D, 0)), descending
  std::vector<double> sig_new(m);
  for (int64_t i = 0; i < m; ++i) {
    const double dv = Du[m - 1 - i];
    if (dv < 0.0) ++R.neg_clamped;
    sig_new[i] = std::sqrt(std::max(dv, 0.0));
  }
  for (int e = 0; e < 4; ++e) {
    R.n_active[e] = S[e].na;
    R.n_deflated[e] = S[e].N - S[e].na;
    R.max_iter[e] = S[e].max_iter;
  }
  // ---- applies (vector parts of STEPS 4-7): U -> W_u -> U, V -> W_v -> V.  Every
  // eigen-update succeeded: the first applies that transform their input in place can
  // start now; the second applies follow as soon as their plans are uploaded.
  const double t4 = now_ms();
  if (launchers) {  // the V side's remaining launches likewise (they carry the sign alignment)
    TRY(join_launcher(P, 1));
    SideJob jv;
    jv.side = 1;
    jv.parity = B->parity;
    jv.t = B->t;
    jv.first_done = launched_v1;
    jv.S = S;
    jv.X = V;
    jv.ldx = ldv;
    jv.W = Wv;
    jv.ldw = nv;
    jv.st = stv;
    jv.thin = thin;
    jv.v_rows = c.v_rows;
    jv.m = m;
    jv.v_row0 = c.v_row0;
    jv.b_dev = b_dev;
    jv.y_dev = B->y_dev;
    jv.inv_beta = beta_perp > 0.0 ? 1.0 / beta_perp : 0.0;
    jv.nrot = nrot_v();
    jv.rot_maxk = rot_maxk();
    jv.ut = ut;
    if (!P->bdone[B->parity][1])
      SVD1_CUDA_TRY(cudaEventCreateWithFlags(&P->bdone[B->parity][1], cudaEventDisableTiming));
    P->launcher_parity[1] = B->parity;
    P->launcher[1] = WorkThread([P, jv] {
      P->launcher_status[1] = side_job(P, jv);
      flush_launches(P);
    });
    P->bdone_rec[B->parity] = true;
    R.t_ms[2] = now_ms() - t4;
    *B->sig = sig_new;
    for (int e = 0; e < 4; ++e) {
      R.spectral_ms[e] = S[e].spectral_ms;
      R.mean_iter[e] = S[e].mean_iter;
    }
    // (apply flops / tree statistics: filled by the batch loop once this update's launchers
    // have been joined -- the second steps' plans may still be running now)
    R.t_ms[4] = now_ms() - t0;
    flush_launches(P);
    R.kernel_launches = P->launches - launches0;
    R.allocations = g_allocs.load() - allocs0;
    if (rep) *rep = R;
    plan_join_on_error.active = false;  // the second steps' plans belong to the launchers now
    return SVD1_OK;
  }
  if (one_stream) TRY(u_applies());
  if (fused) {  // both steps of a side row chunk by row chunk (§4.11)
    S[3].join_plan();
    TRY(rare_grow(3, 1));
    TRY(upload_step(3));  // carries the sign alignment
    if (!B) TRY(upload_rot(one_stream ? 0 : 1));
    TRY(fused_side(1));
  }
  if (!fused && !launched_v1) {
    TRY(ev_record(P, 18, stv));
    if (B) TRY(bwin_record(P, B->parity, 1, stv));
    if (B && B->t == 0) TRY(bspan_record(P, 1, stv));
    TRY(null_dir());
    TRY(apply_launch(P, S[2], V, ldv, Wv, nv, 4, stv, 1));
  }
  if (!fused) {
    S[3].join_plan();
    TRY(rare_grow(3, 1));
    TRY(upload_step(3));  // carries the sign alignment
    if (!B) TRY(upload_rot(one_stream ? 0 : 1));
    tl_mark(P, (B ? "u" + std::to_string(B->t) : std::string()) + " V2 apply", stv);
    TRY(apply_launch(P, S[3], Wv, nv, V, ldv, 6, stv, 1));
    if (nrot_v() > 0)
      TRY(col_rotate(c.v_rows, V, ldv, nrot_v(), static_cast<int32_t*>(S[3].rot_goff.p),
                     static_cast<int32_t*>(S[3].rot_cols.p), static_cast<double*>(S[3].rot_mats.p), stv,
                     LC(P), rot_maxk()));
  }
  u_thread.join();  // the U-side applies are queued
  TRY(st_ua);
  if (B) {  // no join, no sync: the next update's spectral phase overlaps these applies
    tl_mark(P, "u" + std::to_string(B->t) + " V2 end", stv);
    TRY(bwin_record(P, B->parity, 3, stv));
    if (!P->bdone[B->parity][1])
      SVD1_CUDA_TRY(cudaEventCreateWithFlags(&P->bdone[B->parity][1], cudaEventDisableTiming));
    SVD1_CUDA_TRY(cudaEventRecord(P->bdone[B->parity][1], stv));
    P->bdone_rec[B->parity] = true;
    R.t_ms[2] = now_ms() - t4;
    *B->sig = sig_new;
    for (int e = 0; e < 4; ++e) {
      const bool has = S[e].rows > 0 && S[e].na > 0;
      R.apply_flops[e] = has ? S[e].cp.flops : 0.0;
      R.apply_flops_exec[e] = has ? S[e].cp.flops_exec : 0.0;
      R.fmm_used[e] = has ? S[e].cp.fmm : 0;
      if (R.fmm_used[e]) {
        R.fmm_levels[e] = S[e].cp.F.L;
        R.fmm_max_near[e] = S[e].cp.F.max_near;
      }
      R.spectral_ms[e] = S[e].spectral_ms;
      R.mean_iter[e] = S[e].mean_iter;
    }
    R.t_ms[4] = now_ms() - t0;
    flush_launches(P);
    R.kernel_launches = P->launches - launches0;
    R.allocations = g_allocs.load() - allocs0;
    if (rep) *rep = R;
    return SVD1_OK;
  }
  TRY(stream_wait(P, 2, P->st2, P->st));  // join
  TRY(ev_record(P, 17, P->st));           // apply phase end
  R.t_ms[2] = now_ms() - t4;
  std::memcpy(h, sig_new.data(), size_t(m) * sizeof(double));
  SVD1_CUDA_TRY(cudaMemcpyAsync(sigma, h, size_t(m) * sizeof(double), cudaMemcpyHostToDevice, P->st));
  SVD1_CUDA_TRY(cudaStreamSynchronize(P->st));
  SVD1_CUDA_TRY(cudaGetLastError());
  R.t_ms[3] = now_ms() - t3;
  for (int e = 0; e < 4; ++e) {
    const bool has = S[e].rows > 0;
    R.apply_ms[e] = has ? ev_ms(P, 2 * e, 2 * e + 1) : 0.0;
    R.apply_flops[e] = (has && S[e].na > 0) ? S[e].cp.flops : 0.0;
    R.apply_flops_exec[e] = (has && S[e].na > 0) ? S[e].cp.flops_exec : 0.0;
    R.gemm_ms[e] = (has && S[e].na > 0 && S[e].cp.fmm) ? S[e].cp.gemm_ms() : 0.0;
    R.fmm_used[e] = (has && S[e].na > 0) ? S[e].cp.fmm : 0;
    if (R.fmm_used[e]) {
      R.fmm_levels[e] = S[e].cp.F.L;
      R.fmm_max_near[e] = S[e].cp.F.max_near;
    }
    R.spectral_ms[e] = S[e].spectral_ms;
    R.mean_iter[e] = S[e].mean_iter;
  }
  R.t_ms[4] = now_ms() - t0;
  R.t_ms[5] = std::max(ev_ms(P, 16, 17), ev_ms(P, 18, 17));  // both sides' applies
  if (std::getenv("SVD1_TIMING")) {  // device timeline relative to the first spectral launch
    const char* nm[4] = {"U1", "U2", "V1", "V2"};
    for (int e = 0; e < 4; ++e)
      fprintf(stderr, "[svd1] dev %s spectral %.3f..%.3f apply %.3f..%.3f\n", nm[e],
              ev_ms(P, 8, 8 + 2 * e), ev_ms(P, 8, 9 + 2 * e), ev_ms(P, 8, 2 * e), ev_ms(P, 8, 2 * e + 1));
    fprintf(stderr, "[svd1] dev end %.3f; host: spectral rounds %.3f, t4 %.3f, end %.3f\n", ev_ms(P, 8, 17),
            t3 - t1, t4 - t1, now_ms() - t1);
  }
  flush_launches(P);
  R.kernel_launches = P->launches - launches0;
  R.allocations = g_allocs.load() - allocs0;
  if (rep) *rep = R;
  return SVD1_OK;
}
svd1_status batch_run(svd1_plan_t P, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                      const double* proj, const double* Bv, int64_t ldb, int64_t K, double eps,
                      svd1_report* reps, const std::function<svd1_status()>& many);
}  // namespace

extern "C" {

svd1_status svd1_update_projected(svd1_plan_t P, double* U, int64_t ldu, double* sigma, double* V,
                                  int64_t ldv, const double* proj, const double* a, const double* b,
                                  double eps, svd1_report* rep) {
  (void)a;
  return update_impl(P, U, ldu, sigma, V, ldv, proj, eps, rep, nullptr, b);
}

svd1_status svd1_update_batch(svd1_plan_t P, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                              const double* A, int64_t lda, const double* Bv, int64_t ldb, int64_t K,
                              double eps, svd1_report* reps) {
  if (!P || !U || !V || !sigma || (K > 0 && (!A || !Bv)) || K < 0 || K > kMaxBatch) return SVD1_E_INVALID;
  const svd1_config& c = P->cfg;
  const int64_t m = c.m, n = c.n;
  const bool thin = (c.flags & SVD1_THIN_V) != 0;
  if (c.u_rows != m || c.v_rows != n || ldu < m || ldv < (thin ? m + 1 : n) || lda < m || ldb < n)
    return SVD1_E_INVALID;
  if (K == 0) return SVD1_OK;
  // every update's STEP-1 projections against the initial factors
  const size_t nproj = size_t(5 * m + n + 6);
  double* pj;
  // (a previous call that failed part-way may have left its project_many in flight)
  if (P->st_proj) SVD1_CUDA_TRY(cudaStreamSynchronize(P->st_proj));
  TRY(P->bproj.get<double>(size_t(kMaxBatch) * nproj, &pj, P->st));
  P->tl_on = std::getenv("SVD1_TIMELINE") != nullptr;
  P->tl_t0 = now_ms();
  P->tl_pre = P->tl_on;
  tl_mark(P, "batch enter", P->st);
  // update 0 in full (its probe block too), updates 1.. with one pass over U and V per
  // 8 of them (only their x_a, y_b and dots are used: the probes are carried)
  TRY(svd1_project(P, U, ldu, V, ldv, A, Bv, pj));
  tl_mark(P, "update 0 projected", P->st);
  // updates 1.. on their own stream, alongside update 0's spectral phase: launched by
  // batch_run once update 0's projection has been read back (its blocks would otherwise
  // hold the SMs the plan stream's small copies need)
  std::function<svd1_status()> many;
  if (K > 1) {
    double* part;
    const int64_t need = project_partial_elems(c.u_rows, m, c.v_rows, n);
    TRY(P->partial.get<double>(size_t(need), &part, P->st));
    if (!P->st_proj) SVD1_CUDA_TRY(cudaStreamCreateWithFlags(&P->st_proj, cudaStreamNonBlocking));
    if (!P->proj_ev) SVD1_CUDA_TRY(cudaEventCreateWithFlags(&P->proj_ev, cudaEventDisableTiming));
    many = [=]() -> svd1_status {
      TRY(project_many(U, ldu, c.u_rows, m, c.u_row0, V, ldv, c.v_rows, n, c.v_row0, thin ? m : n, A + lda, lda,
                       Bv + ldb, ldb, int(K) - 1, static_cast<double*>(P->probes.p), part, need, pj + nproj,
                       int64_t(nproj), P->st_proj, LC(P)));
      tl_mark(P, "projections queued", P->st_proj);
      return SVD1_OK;
    };
  }
  return batch_run(P, U, ldu, sigma, V, ldv, pj, Bv, ldb, K, eps, reps, many);
}

svd1_status svd1_update_batch_projected(svd1_plan_t P, double* U, int64_t ldu, double* sigma, double* V,
                                        int64_t ldv, const double* proj, const double* Bv, int64_t ldb,
                                        int64_t K, double eps, svd1_report* reps) {
  return batch_run(P, U, ldu, sigma, V, ldv, proj, Bv, ldb, K, eps, reps, nullptr);
}
}  // extern "C"

namespace {
// The pipelined stream.  many (svd1_update_batch): launches the
// projections of updates 1..K-1 on st_proj; only update 0's are complete in stream order
// on the plan stream.  Their results are needed by update 0's carried-row transforms and
// the dots by update 1; every apply waits for them (they read the initial factors).
svd1_status batch_run(svd1_plan_t P, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                      const double* proj, const double* Bv, int64_t ldb, int64_t K, double eps,
                      svd1_report* reps, const std::function<svd1_status()>& many) {
  const bool deferred = bool(many);

  if (!P || !sigma || (K > 0 && !proj) || K < 0 || K > kMaxBatch) return SVD1_E_INVALID;
  const svd1_config& c = P->cfg;
  const int64_t m = c.m, n = c.n;
  const bool thin = (c.flags & SVD1_THIN_V) != 0;
  const int64_t nv = thin ? m + 1 : n;  // width of the carried V rows
  // thin V needs the b's themselves (null directions, Gram matrix)
  if (thin && (!Bv || ldb < n)) return SVD1_E_INVALID;
  P->batch_b = thin ? Bv : nullptr;
  P->batch_ldb = ldb;
  struct ResetB {
    svd1_plan_t P;
    ~ResetB() { P->batch_b = nullptr; }
  } reset_b{P};
  if ((c.u_rows && (!U || ldu < m)) || (c.v_rows && (!V || ldv < nv))) return SVD1_E_INVALID;
  if (K == 0) return SVD1_OK;
  const int k = int(K);
  tl_mark(P, "batch_run", nullptr, false);
  TRY(arena_reset(P));
  tl_mark(P, "arenas reset", nullptr, false);
  TRY(ensure_st2(P));
  TRY(ensure_side(P, 2));
  TRY(ensure_side(P, 3));
  // buffers sized for the largest batch whatever K is: no reallocation (and its
  // implicit device synchronisation) between batches of different lengths
  const size_t nproj = size_t(5 * m + n + 6);
  const double* pj = proj;
  // carried rows (row-major, m resp. n wide): U side [x_g (4) | x_a(K-1) .. x_a(1)],
  // V side [y_b(K-1) .. y_b(1)]; update t transforms the rows of updates t+1.. only
  const int ru_max = 4 + (kMaxBatch - 1), rv_max = kMaxBatch - 1;
  double *ru0, *ru1, *rv0, *rv1;
  TRY(P->RU[0].get<double>(size_t(ru_max) * m, &ru0, P->st));  // all sized at creation
  TRY(P->RU[1].get<double>(size_t(ru_max) * m, &ru1, P->st));
  TRY(P->RV[0].get<double>(size_t(rv_max) * n, &rv0, P->st));
  TRY(P->RV[1].get<double>(size_t(rv_max) * n, &rv1, P->st));
  double* scr;  // few-rows scratch at its largest
  TRY(P->few_scr[0].get<double>(size_t(few_rows_scratch_elems(ru_max, int(m))), &scr, P->st));
  TRY(P->few_scr[1].get<double>(size_t(few_rows_scratch_elems(rv_max, int(nv))), &scr, P->st));
  // (deferred: the rows of updates 1.. are copied on st_proj after project_many; the
  // buffers above are ordered on P->st, which st_proj joins first)
  const cudaStream_t qs = deferred ? P->st_proj : P->st;
  SVD1_CUDA_TRY(cudaMemcpyAsync(ru0, pj + m, 4 * m * sizeof(double), cudaMemcpyDeviceToDevice, P->st));
  auto carried_copies = [&]() -> svd1_status {  // the later updates' x_a, y_b as carried rows
    TRY(copy_rows_rev(ru0, m, 4 + (k - 1), pj, int64_t(nproj), m, k - 1, qs, LC(P)));
    TRY(copy_rows_rev(rv0, nv, k - 1, pj + 5 * m, int64_t(nproj), thin ? m : n, k - 1, qs, LC(P)));
    return SVD1_OK;
  };
  if (!deferred) TRY(carried_copies());
  double* gram = nullptr;  // thin: b_t . b_s
  if (thin) {
    TRY(P->bgram.get<double>(size_t(kMaxBatch) * kMaxBatch, &gram, P->st));
    TRY(gram_rows(k, P->batch_b, P->batch_ldb, n, gram, P->st, LC(P)));
  }
  // host copies of the projections (dots of every update; x's of update 0) and sigma
  double* h;
  TRY(pinned(P, size_t(kMaxBatch) * nproj + size_t(m) + size_t(5 * m + n), &h));
  SVD1_CUDA_TRY(cudaMemcpyAsync(h, pj, size_t(deferred ? 1 : k) * nproj * sizeof(double), cudaMemcpyDeviceToHost,
                                P->st));
  SVD1_CUDA_TRY(cudaMemcpyAsync(h + size_t(k) * nproj, sigma, size_t(m) * sizeof(double), cudaMemcpyDeviceToHost,
                                P->st));
  tl_mark(P, "read-backs queued", P->st);
  SVD1_CUDA_TRY(cudaStreamSynchronize(P->st));  // also orders the copies before the V stream
  tl_mark(P, "read-backs done", nullptr, false);
  if (deferred) {  // (after the plan stream's read-backs: copy queues are in order)
    TRY(many());
    TRY(carried_copies());
    SVD1_CUDA_TRY(cudaEventRecord(P->proj_ev, qs));
  }
  if (deferred)  // no apply writes U or V before project_many has read them
    for (cudaStream_t q : {P->st, P->st2}) SVD1_CUDA_TRY(cudaStreamWaitEvent(q, P->proj_ev, 0));
  double* hn = h + size_t(k) * nproj + m;  // next update's x_a | x_g | y_b (read back)
  std::memset(hn, 0, size_t(5 * m + n) * sizeof(double));  // (thin: y_b past m stays 0)
  std::vector<double> sig(h + size_t(k) * nproj, h + size_t(k) * nproj + m);
  std::vector<double> hp(h, h + nproj);
  svd1_status st = SVD1_OK;
  P->tl_on = std::getenv("SVD1_TIMELINE") != nullptr;
  if (!P->tl_pre) P->tl_t0 = now_ms();  // (svd1_update_batch marked its projections)
  P->tl_pre = false;
  tl_mark(P, "batch start", P->st);
  const bool launched_by_launchers = (c.flags & SVD1_FUSED_SIDE) == 0;  // (see update_impl)
  int pending = -1;  // the update whose launchers are in flight (its report still to complete)
  for (int t = 0; t < k && st == SVD1_OK; ++t) {
    if (t == 1 && deferred) SVD1_CUDA_TRY(cudaStreamSynchronize(qs));  // the later updates' dots
    if (t > 0) {  // x's from the carried rows, dots from update t's projection
      std::memcpy(hp.data(), hn, size_t(5 * m + n) * sizeof(double));
      std::memcpy(hp.data() + 5 * m + n, h + size_t(t) * nproj + 5 * m + n, 6 * sizeof(double));
    }
    BatchCtx b;
    b.parity = t & 1;
    b.t = t;
    b.h_proj = hp.data();
    b.sig = &sig;
    b.ru_rows = t + 1 < k ? 4 + (k - 1 - t) : 0;
    b.rv_rows = t + 1 < k ? k - 1 - t : 0;
    b.ru_next = t + 1 < k ? 4 + (k - 2 - t) : -1;
    b.rv_next = t + 1 < k ? k - 2 - t : -1;
    b.h_next = hn;
    b.rows_wait = (deferred && t == 0) ? P->proj_ev : nullptr;
    b.prev_win = (reps && t >= 2) ? &reps[t - 2].t_ms[5] : nullptr;
    b.prev_gemm = (reps && t >= 2) ? reps[t - 2].gemm_ms : nullptr;
    if (thin) {
      b.b_dev = P->batch_b + int64_t(t) * P->batch_ldb;
      b.y_dev = t == 0 ? pj + 5 * m : rv0 + int64_t(k - 1 - t) * nv;
      b.gram = gram;
      b.K = k;
    }
    svd1_report R;
    st = update_impl(P, U, ldu, sigma, V, ldv, nullptr, eps, &R, &b);
    if (reps) reps[t] = R;
    if (t == 0 && deferred && k > 1)  // the 6 dots of updates 1.. (project_many is long done)
      SVD1_CUDA_TRY(cudaMemcpy2DAsync(h + nproj + 5 * m + n, nproj * sizeof(double), pj + nproj + 5 * m + n,
                                      nproj * sizeof(double), 6 * sizeof(double), size_t(k - 1),
                                      cudaMemcpyDeviceToHost, qs));
    if (launched_by_launchers && st == SVD1_OK && !R.noop) {
      // update t joined the launchers of the previous such update before its own applies:
      // that update's plans are complete, its apply statistics can be reported
      if (pending >= 0 && reps) fill_apply_fields(reps[pending], P->bsteps[pending & 1]);
      pending = t;
    }
    if (st != SVD1_OK || t + 1 >= k) break;
    if (R.noop) {  // nothing transformed: the next rows are where they were
      SVD1_CUDA_TRY(cudaDeviceSynchronize());
      SVD1_CUDA_TRY(cudaMemcpy(hn, ru0 + int64_t(b.ru_next) * m, m * sizeof(double), cudaMemcpyDeviceToHost));
      SVD1_CUDA_TRY(cudaMemcpy(hn + m, ru0, 4 * m * sizeof(double), cudaMemcpyDeviceToHost));
      SVD1_CUDA_TRY(cudaMemcpy(hn + 5 * m, rv0 + int64_t(b.rv_next) * nv, (thin ? m : n) * sizeof(double),
                               cudaMemcpyDeviceToHost));
    } else {
      SVD1_CUDA_TRY(cudaEventSynchronize(P->rb_ev[0]));
      SVD1_CUDA_TRY(cudaEventSynchronize(P->rb_ev[1]));
    }
  }
  // the last update's launchers: its remaining apply launches are queued after this
  for (int sd = 0; sd < 2; ++sd) {
    const svd1_status ls = join_launcher(P, sd);
    if (st == SVD1_OK) st = ls;
  }
  if (pending >= 0 && reps) fill_apply_fields(reps[pending], P->bsteps[pending & 1]);
  const bool span_ok = st == SVD1_OK;
  if (span_ok) {
    TRY(bspan_record(P, 2, P->st));
    TRY(bspan_record(P, 3, P->st2));
  }
  // drain every stream; the factors now hold updates 0..t; sigma of the last success
  for (cudaStream_t q : {P->st, P->st2, P->sp[0], P->sp[1], P->sp[2], P->sp[3], P->st_proj})
    if (q || q == P->st) SVD1_CUDA_TRY(cudaStreamSynchronize(q));
  if (P->tl_on) {  // host stamps and device times (ms from the batch start)
    cudaEvent_t base = P->tl_dev.empty() ? nullptr : P->tl_dev.front().second;
    for (size_t q = 0; q < P->tl_host.size(); ++q) fprintf(stderr, "[tl] host %8.3f %s\n", P->tl_host[q].second, P->tl_host[q].first.c_str());
    for (auto& pr : P->tl_dev) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, base, pr.second);
      fprintf(stderr, "[tl] dev  %8.3f %s\n", ms, pr.first.c_str());
    }
    for (auto& pr : P->tl_dev) cudaEventDestroy(pr.second);
    P->tl_dev.clear();
    P->tl_host.clear();
    P->tl_on = false;
  }
  if (reps && span_ok) reps[k - 1].t_ms[6] = bspan_ms(P);  // whole batch's apply span
  if (reps && st == SVD1_OK)  // apply windows of the last two updates
    for (int t = std::max(0, k - 2); t < k; ++t)
      if (P->bdone_rec[t & 1]) {
        reps[t].t_ms[5] = bwin_ms(P, t & 1);
        for (int e = 0; e < 4; ++e) {
          StepRecord& Se = P->bsteps[t & 1][e];
          reps[t].gemm_ms[e] = (Se.rows > 0 && Se.na > 0 && Se.cp.fmm) ? Se.cp.gemm_ms() : 0.0;
        }
      }
  P->bdone_rec[0] = P->bdone_rec[1] = false;
  std::memcpy(h + size_t(k) * nproj, sig.data(), size_t(m) * sizeof(double));
  SVD1_CUDA_TRY(cudaMemcpyAsync(sigma, h + size_t(k) * nproj, size_t(m) * sizeof(double), cudaMemcpyHostToDevice,
                                P->st));
  SVD1_CUDA_TRY(cudaStreamSynchronize(P->st));
  return st;
}
}  // namespace

extern "C" {

svd1_status svd1_update(svd1_plan_t P, double* U, int64_t ldu, double* sigma, double* V, int64_t ldv,
                        const double* a, const double* b, double eps, svd1_report* rep) {
  if (!P) return SVD1_E_INVALID;
  const svd1_config& c = P->cfg;
  if (c.u_rows != c.m || c.v_rows != c.n) return SVD1_E_INVALID;  // single process only
  double* proj;
  TRY(P->proj.get<double>(size_t(5 * c.m + c.n + 6), &proj, P->st));
  TRY(svd1_project(P, U, ldu, V, ldv, a, b, proj));
  return svd1_update_projected(P, U, ldu, sigma, V, ldv, proj, a, b, eps, rep);
}

svd1_status svd1_cauchy_apply(svd1_plan_t P, int64_t rows, int64_t n, const double* d,
                              const int32_t* k, const double* tau, const double* zhat,
                              const double* colscale, const double* U_in, int64_t ld_in,
                              double* U_out, int64_t ld_out, double eps, int32_t* fmm_used) {
  if (!P || rows < 0 || n < 0 || n > (int64_t(1) << 30)) return SVD1_E_INVALID;
  if (n == 0 || rows == 0) return SVD1_OK;
  if (!d || !k || !tau || !zhat || !colscale || !U_in || !U_out || ld_in < n || ld_out < n)
    return SVD1_E_INVALID;
  const int p = choose_p(eps > 0.0 ? eps : P->cfg.eps);
  TRY(arena_reset(P));
  std::vector<double> dh(n), th(n), mu(n);
  std::vector<int32_t> kh(n);
  SVD1_CUDA_TRY(cudaMemcpyAsync(dh.data(), d, n * sizeof(double), cudaMemcpyDeviceToHost, P->st));
  SVD1_CUDA_TRY(cudaMemcpyAsync(kh.data(), k, n * sizeof(int32_t), cudaMemcpyDeviceToHost, P->st));
  SVD1_CUDA_TRY(cudaMemcpyAsync(th.data(), tau, n * sizeof(double), cudaMemcpyDeviceToHost, P->st));
  SVD1_CUDA_TRY(cudaStreamSynchronize(P->st));
  for (int64_t j = 0; j < n; ++j) {
    if (kh[j] < 0 || kh[j] >= n) return SVD1_E_INVALID;
    if (th[j] == 0.0) return SVD1_E_POLE;
    mu[j] = dh[kh[j]] + th[j];
  }
  bool used = false;
  {
    CauchyPrep& C = P->standalone;
    TRY(cauchy_prepare(P, C, rows, int(n), dh, mu, p));
    TRY(ensure_expansions(P, 0, cauchy_exp_elems(C)));
    TRY(cauchy_launch(P, C, d, k, tau, zhat, colscale, U_in, ld_in, nullptr, U_out, ld_out, nullptr,
                      P->st, 0));
    used = C.fmm;
  }
  if (fmm_used) *fmm_used = used ? 1 : 0;
  SVD1_CUDA_TRY(cudaGetLastError());
  return SVD1_OK;
}

svd1_status svd1_secfmm_plan_stats(int64_t n, const double* d, int64_t* st) {
  if (n < 2 || !d || !st || n > (int64_t(1) << 30)) return SVD1_E_INVALID;
  SecPlanHost H;
  const auto t0 = std::chrono::steady_clock::now();
  secfmm_plan(d, int(n), H);
  const auto t1 = std::chrono::steady_clock::now();
  int64_t mx = 0;
  for (int q = 0; q < H.nleaf; ++q) {
    int64_t s2 = 0;
    for (int g = H.near_off[q]; g < H.near_off[q + 1]; ++g) s2 += H.near_hi[g] - H.near_lo[g];
    mx = std::max(mx, s2);
  }
  st[0] = H.L;
  st[1] = H.ncells;
  st[2] = H.nleaf;
  st[3] = int64_t(H.parts.size());
  st[4] = int64_t(H.near_lo.size());
  st[5] = mx;
  st[6] = int64_t(H.direct.size());
  st[7] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
  return SVD1_OK;
}

svd1_status svd1_fmm_tree_stats(int64_t n, const double* d, const int32_t* k, const double* tau,
                                double eps, int64_t* st) {
  if (n <= 0 || !d || !k || !tau || !st || n > (int64_t(1) << 30)) return SVD1_E_INVALID;
  const int p = choose_p(eps);
  const int leaf = std::min(2 * p, kMaxLeaf);
  std::vector<double> dh(d, d + n), mu(n);
  for (int64_t j = 0; j < n; ++j) {
    if (k[j] < 0 || k[j] >= n) return SVD1_E_INVALID;
    mu[j] = dh[k[j]] + tau[j];
  }
  FmmHost F;
  fmm_build_host(F, int(n), leaf, p, dh, mu, nullptr, n);
  int64_t nonempty = 0, max_leaf = 0;
  for (int c = 0; c < F.ncells; ++c) nonempty += F.cells[c].hi > F.cells[c].lo;
  for (int i = 0; i < (1 << F.L); ++i) {
    const FmmCell& C = F.cells[(1 << F.L) - 1 + i];
    max_leaf = std::max<int64_t>(max_leaf, std::max(C.shi - C.slo, C.thi - C.tlo));
  }
  st[0] = F.L;
  st[1] = nonempty;
  st[2] = max_leaf;
  st[3] = F.max_near;
  st[4] = F.n_near_pairs;
  st[5] = F.n_m2l_pairs;
  st[6] = F.flops_per_row;
  st[8] = F.flops_exec_per_row;
  st[7] = int64_t(F.tasks.size());
  return SVD1_OK;
}

svd1_status svd1_secular_solve(svd1_plan_t P, int64_t n, const double* d, const double* z, double rho,
                               int32_t* k_out, double* tau_out, int32_t* iters) {
  if (!P || n < 0 || !d || !z || !k_out || !tau_out || rho == 0.0) return SVD1_E_INVALID;
  if (n == 0) return SVD1_OK;
  int32_t *dst, *dit;
  TRY(P->status.get<int32_t>(1, &dst, P->st));
  TRY(P->iters.get<int32_t>(size_t(n), &dit, P->st));
  SVD1_CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(int32_t), P->st));
  double* orient;
  TRY(P->scratch_d.get<double>(size_t(2 * n), &orient, P->st));
  TRY(secular_orient(d, z, rho, int(n), orient, orient + n, P->st, LC(P)));
  if (use_sec_fmm(P->cfg.flags, int(n), false)) {  // plan from the oriented sources (host copy)
    std::vector<double> dr(n);
    SVD1_CUDA_TRY(cudaMemcpyAsync(dr.data(), orient, n * sizeof(double), cudaMemcpyDeviceToHost, P->st));
    SVD1_CUDA_TRY(cudaStreamSynchronize(P->st));
    SecFmmDev F;
    TRY(arena_reset(P));
    TRY(secfmm_prepare(P, P->steps[0].sec, P->steps[0].sec_blob, P->steps[0].sec_scr, dr.data(), int(n), 0, &F));
    TRY(secular_fmm(orient, orient + n, rho, int(n), 0, int(n), F, k_out, tau_out, dit, dst, P->st, LC(P)));
  } else {
    TRY(secular(orient, orient + n, rho, int(n), 0, int(n), k_out, tau_out, dit, dst, P->st, LC(P)));
  }
  std::vector<int32_t> it(n);
  int32_t st_h = 0;
  SVD1_CUDA_TRY(cudaMemcpyAsync(it.data(), dit, n * sizeof(int32_t), cudaMemcpyDeviceToHost, P->st));
  SVD1_CUDA_TRY(cudaMemcpyAsync(&st_h, dst, sizeof(int32_t), cudaMemcpyDeviceToHost, P->st));
  SVD1_CUDA_TRY(cudaStreamSynchronize(P->st));
  if (iters) *iters = *std::max_element(it.begin(), it.end());
  if (st_h & 1) return SVD1_E_NOCONV;
  if (st_h & 2) return SVD1_E_POLE;
  return SVD1_OK;
}

svd1_status svd1_loewner(svd1_plan_t P, int64_t n, const double* d, const int32_t* k, const double* tau,
                         double rho, const double* z, double* zhat_out) {
  if (!P || n < 0 || !d || !k || !tau || !z || !zhat_out || rho == 0.0) return SVD1_E_INVALID;
  double* scr;
  TRY(P->scratch_d.get<double>(size_t(spectral_scratch_elems(int(n), 0)), &scr, P->st));
  int* ctr;
  TRY(counters(P->ctr, int(n), P->st, &ctr));
  TRY(loewner(d, k, tau, rho, z, int(n), 0, int(n), zhat_out, scr, ctr, P->st, LC(P)));
  SVD1_CUDA_TRY(cudaStreamSynchronize(P->st));
  return SVD1_OK;
}

svd1_status svd1_colnorms(svd1_plan_t P, int64_t n, const double* d, const int32_t* k,
                          const double* tau, const double* zhat, double* colnorm_out) {
  if (!P || n < 0 || !d || !k || !tau || !zhat || !colnorm_out) return SVD1_E_INVALID;
  if (n == 0) return SVD1_OK;
  int32_t* dst;
  double* cs;
  TRY(P->status.get<int32_t>(1, &dst, P->st));
  TRY(P->scratch_i.get<double>(size_t(n), &cs, P->st));
  double* scr;
  TRY(P->scratch_d.get<double>(size_t(spectral_scratch_elems(int(n), 0)), &scr, P->st));
  SVD1_CUDA_TRY(cudaMemsetAsync(dst, 0, sizeof(int32_t), P->st));
  int* ctr;
  TRY(counters(P->ctr, int(n), P->st, &ctr));
  TRY(colnorm_carry(d, k, tau, zhat, int(n), 0, int(n), nullptr, 0, cs, nullptr, n, dst, scr, ctr, P->st,
                    LC(P)));
  std::vector<double> h(n);
  SVD1_CUDA_TRY(cudaMemcpyAsync(h.data(), cs, n * sizeof(double), cudaMemcpyDeviceToHost, P->st));
  SVD1_CUDA_TRY(cudaStreamSynchronize(P->st));
  for (auto& v : h) v = 1.0 / v;
  TRY(arena_reset(P));
  TRY(arena_put(P, h.data(), n * sizeof(double), colnorm_out));
  SVD1_CUDA_TRY(cudaStreamSynchronize(P->st));
  return SVD1_OK;
}

}  // extern "C"
