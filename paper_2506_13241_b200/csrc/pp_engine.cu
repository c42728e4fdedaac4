// pp_engine.cu -- host orchestration of the B200 Pauli-propagation engine
// and its C-ABI (include/pauliprop_gpu.h).
//
// One engine owns one CUDA device's share of the operator: a z-grouped
// arena store (pp_kernels.cuh) plus the regroup machinery (pp_regroup.cuh).
// The per-gate sequence mirrors Engine::apply_gate (engine.cpp:277-316):
//   branch (+ merge)  ->  budget check  ->  [per-gate cadence] truncate
// and truncate_now mirrors engine.cpp:318-351 (global max, NaN/Inf check,
// threshold epsilon0 * gmax, remove |c| <= threshold).
#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pauliprop_gpu.h"
#include "pp_regroup.cuh"
#include "pp_zz.cuh"
#include "pp_dense.cuh"

namespace ppgpu {

struct EngineError : std::runtime_error {
  int code;
  EngineError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PP_CUDA(x)                                                                                  \
  do {                                                                                              \
    cudaError_t e_ = (x);                                                                           \
    if (e_ != cudaSuccess) {                                                                        \
      if (e_ == cudaErrorMemoryAllocation) {                                                        \
        cudaGetLastError();                                                                         \
        throw EngineError(PP_ERR_RESOURCE, std::string("device memory exhausted: ") + #x);          \
      }                                                                                             \
      throw EngineError(PP_ERR_INTERNAL, std::string(cudaGetErrorString(e_)) + " at " + #x);       \
    }                                                                                               \
  } while (0)

using Clock = std::chrono::steady_clock;
static uint64_t ns_since(Clock::time_point t) {
  return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(Clock::now() - t).count();
}

__global__ void k_clear_cumulative(DevStats* st) {
  st->red[2].live = 0;  // the sync slot, ready for the next readout
  st->red[2].gmax_bits = 0;
  st->red[2].gmin_bits = 0x7ff0000000000000ull;
  st->red[2].nonfinite = 0;
  st->red[2].maxcnt = 0;
  st->records = 0;
  st->removed = 0;
  st->out_elems = 0;
  st->aff_total = 0;
  st->stream_elems = 0;
  st->cliff_records = 0;
  st->dense_groups = 0;
  st->dense_out = 0;
  st->bulk_tiles = 0;
  for (int w = 0; w < kSeenWords; ++w) st->seen[w] = 0;
  for (int k = 0; k < kZZSeenGroups; ++k) st->zz_seen[k][0] = st->zz_seen[k][1] = 0;
}

__global__ void k_reset_stats(DevStats* st, unsigned long long bump) { k_reset_stats_body(st, bump); }

template <int W>
__global__ void k_init_small(ArenaView<W> a, GroupView<W> g, const InitSmall<W> in, DevStats* st) {
  const uint32_t t = threadIdx.x;
  if (t < in.n) {
#pragma unroll
    for (int w = 0; w < W; ++w) a.x[w][t] = in.x[t][w];
    a.c[t] = in.c[t];
  }
  if (t < in.G) {
#pragma unroll
    for (int w = 0; w < W; ++w) g.z[w][t] = in.z[t][w];
    g.off[t] = in.off[t];
    g.cnt[t] = in.cnt[t];
    g.cap[t] = in.cnt[t];
    g.gmax[t] = in.gmax[t];
    g.gmin[t] = in.gmin[t];
    g.flags[t] = in.flags[t];
    g.stamp[t] = 0xffffffffu;
  }
  if (t == 0) k_reset_stats_body(st, in.n);
}

__global__ void k_clear_arena_error(DevStats* st) {
  st->err_arena = 0;
  st->err_unsorted = 0;
  st->err_seq = ~0ull;
}

// ---------------------------------------------------------------------------
// interleaved (reference) <-> plane conversion on the host
// ---------------------------------------------------------------------------
static inline uint64_t compact_even(uint64_t v) {
  v &= 0x5555555555555555ull;
  v = (v | (v >> 1)) & 0x3333333333333333ull;
  v = (v | (v >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v >> 4)) & 0x00FF00FF00FF00FFull;
  v = (v | (v >> 8)) & 0x0000FFFF0000FFFFull;
  v = (v | (v >> 16)) & 0x00000000FFFFFFFFull;
  return v;
}
static inline uint64_t spread_even(uint64_t v) {
  v &= 0xFFFFFFFFull;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
// words[4] -> x[2], z[2]  (x = lo ^ hi, z = hi per site)
static void words_to_planes(const uint64_t* w, uint64_t* x, uint64_t* z) {
  for (int pw = 0; pw < 2; ++pw) {
    uint64_t lo = compact_even(w[2 * pw]) | (compact_even(w[2 * pw + 1]) << 32);
    uint64_t hi = compact_even(w[2 * pw] >> 1) | (compact_even(w[2 * pw + 1] >> 1) << 32);
    x[pw] = lo ^ hi;
    z[pw] = hi;
  }
}
static void planes_to_words(const uint64_t* x, const uint64_t* z, uint64_t* w) {
  for (int pw = 0; pw < 2; ++pw) {
    uint64_t hi = z[pw], lo = x[pw] ^ z[pw];
    w[2 * pw] = spread_even(lo) | (spread_even(hi) << 1);
    w[2 * pw + 1] = spread_even(lo >> 32) | (spread_even(hi >> 32) << 1);
  }
}

// Host<->device transfer accounting (process-wide, every engine): the bytes
// of every explicit copy plus the kernel parameter blocks that carry host
// data (gate lists, initial terms).  bench.py reads the totals around the
// public call to report e2e h2d/d2h bytes as counted, not modelled.
static std::atomic<unsigned long long> g_h2d_bytes{0}, g_d2h_bytes{0};
static inline void count_xfer(cudaMemcpyKind k, size_t n) {
  if (k == cudaMemcpyHostToDevice) g_h2d_bytes.fetch_add(n, std::memory_order_relaxed);
  else if (k == cudaMemcpyDeviceToHost) g_d2h_bytes.fetch_add(n, std::memory_order_relaxed);
}
static inline void count_param_h2d(size_t n) { g_h2d_bytes.fetch_add(n, std::memory_order_relaxed); }
static inline cudaError_t copy_async(void* dst, const void* src, size_t n, cudaMemcpyKind k, cudaStream_t s) {
  count_xfer(k, n);
  return cudaMemcpyAsync(dst, src, n, k, s);
}
static inline cudaError_t copy_sync(void* dst, const void* src, size_t n, cudaMemcpyKind k) {
  count_xfer(k, n);
  return cudaMemcpy(dst, src, n, k);
}

static inline bool is_clifford(const pp_gate& g) {
  return g.cos_theta == 0.0 && (g.sin_theta == 1.0 || g.sin_theta == -1.0);
}

// ---------------------------------------------------------------------------
// device memory: a process-wide caching pool so that creating engines (one
// per simulate() call, like the reference) does not pay cudaMalloc/cudaFree
// every time.  Blocks are reused when they fit within 25 % slack.
// ---------------------------------------------------------------------------
// Called before the pool gives up on an allocation: releases engines parked
// in the engine pool (their buffers come back here), set below.
static void (*g_release_parked_engines)(int device) = nullptr;
// device bytes held by engines parked in the engine pool on `device`
static size_t (*g_parked_engine_bytes)(int device) = nullptr;

class DevicePool {
 public:
  static DevicePool& get() {
    static DevicePool p;
    return p;
  }
  void* acquire(size_t bytes, size_t* got) {
    int dev = 0;
    cudaGetDevice(&dev);
    bytes = (bytes + kGrain - 1) / kGrain * kGrain;
    {
      std::lock_guard<std::mutex> lk(mu_);
      auto& fl = free_[dev];
      auto it = fl.lower_bound(bytes);
      if (it != fl.end() && it->first <= bytes + bytes / 4) {
        void* p = it->second;
        *got = it->first;
        fl.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, bytes);
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      if (g_release_parked_engines) g_release_parked_engines(dev);
      // free cached blocks, largest first, only until the request fits: the
      // rest stays for the next engine (simulate() makes one per call)
      for (;;) {
        e = cudaMalloc(&p, bytes);
        if (e != cudaErrorMemoryAllocation) break;
        cudaGetLastError();
        if (!trim_largest(dev)) break;
      }
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      if (e == cudaErrorMemoryAllocation) {
        size_t fb = 0, tb = 0;
        cudaMemGetInfo(&fb, &tb);
        throw EngineError(PP_ERR_RESOURCE, "device memory exhausted (request " + std::to_string(bytes >> 20) +
                                               " MiB, free " + std::to_string(fb >> 20) + " MiB of " +
                                               std::to_string(tb >> 20) + " MiB)");
      }
      throw EngineError(PP_ERR_INTERNAL, std::string("cudaMalloc: ") + cudaGetErrorString(e));
    }
    *got = bytes;
    return p;
  }
  void release(void* p, size_t bytes) {
    if (!p) return;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu_);
    free_[dev].emplace(bytes, p);
  }
  size_t cached_bytes(int dev) {
    std::lock_guard<std::mutex> lk(mu_);
    size_t b = 0;
    for (auto& kv : free_[dev]) b += kv.first;
    return b;
  }
  size_t largest_cached(int dev) {
    std::lock_guard<std::mutex> lk(mu_);
    auto it = free_.find(dev);
    return it == free_.end() || it->second.empty() ? 0 : it->second.rbegin()->first;
  }
  void trim(int dev) {
    std::lock_guard<std::mutex> lk(mu_);
    for (auto& [b, p] : free_[dev]) cudaFree(p);
    free_[dev].clear();
  }
  bool trim_largest(int dev) {  // frees the largest cached block; false when none is left
    std::lock_guard<std::mutex> lk(mu_);
    auto& fl = free_[dev];
    if (fl.empty()) return false;
    auto it = std::prev(fl.end());
    cudaFree(it->second);
    fl.erase(it);
    return true;
  }

 private:
  static constexpr size_t kGrain = 1u << 20;
  std::mutex mu_;
  std::map<int, std::multimap<size_t, void*>> free_;
};

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void release() {
    if (p) DevicePool::get().release(p, bytes);
    p = nullptr;
    bytes = 0;
  }
  void ensure(size_t b) {
    if (b <= bytes) return;
    release();
    p = DevicePool::get().acquire(std::max<size_t>(b, 256), &bytes);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  ~DevBuf() { release(); }
};

// pinned host mirrors of DevStats, recycled across engines
static std::mutex g_pinned_mu;
static std::vector<DevStats*> g_pinned_free;
static DevStats* pinned_stats() {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (!g_pinned_free.empty()) {
      DevStats* p = g_pinned_free.back();
      g_pinned_free.pop_back();
      return p;
    }
  }
  DevStats* p = nullptr;
  PP_CUDA(cudaMallocHost(&p, sizeof(DevStats)));
  return p;
}
static void release_pinned_stats(DevStats* p) {
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_pinned_free.push_back(p);
}
// pinned staging for the diagonal readout, recycled across engines
constexpr size_t kDiagCap = 4096;  // pinned room for diagonal strings
constexpr size_t kDiagSpec = 256;  // fetched with the readout's single round trip
struct DiagPinned {
  uint64_t z[2 * kDiagCap];
  double c[kDiagCap];
};
static std::vector<DiagPinned*> g_diag_free;
static DiagPinned* pinned_diag() {
  {
    std::lock_guard<std::mutex> lk(g_pinned_mu);
    if (!g_diag_free.empty()) {
      DiagPinned* p = g_diag_free.back();
      g_diag_free.pop_back();
      return p;
    }
  }
  DiagPinned* p = nullptr;
  PP_CUDA(cudaMallocHost(&p, sizeof(DiagPinned)));
  return p;
}
static void release_pinned_diag(DiagPinned* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_pinned_mu);
  g_diag_free.push_back(p);
}

// Streams and events outlive engines (simulate() creates one engine per
// call): recycled per device, like the device memory pool.
struct StreamSet {
  cudaStream_t stream;
  cudaEvent_t ev0, ev1, ev_sync;
};
static std::mutex g_streams_mu;
static std::map<int, std::vector<StreamSet>> g_streams;
static std::vector<std::pair<cudaEvent_t, cudaEvent_t>> g_event_pairs;
static StreamSet acquire_stream_set(int dev) {
  {
    std::lock_guard<std::mutex> lk(g_streams_mu);
    auto& v = g_streams[dev];
    if (!v.empty()) {
      StreamSet s = v.back();
      v.pop_back();
      return s;
    }
  }
  StreamSet s;
  PP_CUDA(cudaStreamCreateWithFlags(&s.stream, cudaStreamNonBlocking));
  PP_CUDA(cudaEventCreate(&s.ev0));
  PP_CUDA(cudaEventCreate(&s.ev1));
  PP_CUDA(cudaEventCreateWithFlags(&s.ev_sync, cudaEventDisableTiming));
  return s;
}
static void release_stream_set(int dev, const StreamSet& s) {
  std::lock_guard<std::mutex> lk(g_streams_mu);
  g_streams[dev].push_back(s);
}
// launch configuration of one (device, W): attributes set once, grids from
// the occupancy calculator
struct LaunchSetup {
  uint32_t zz_grid = 0, branch_grid = 0, sub_grid = 0, small_grid = 0, dense_grid = 0;
};
static std::mutex g_setup_mu;
static std::map<std::pair<int, int>, LaunchSetup> g_setup;

static std::mutex g_graph_mu;
// Executable graphs of X-type runs, shared by engines with identical buffers
// (pooled engines).  Entries are reference counted: an engine holds the ones
// it launched until its stream has synchronised, so evicting the cache never
// destroys an exec another thread is about to launch or has in flight.
struct GraphExecDeleter {
  void operator()(CUgraphExec_st* e) const { cudaGraphExecDestroy(e); }
};
using GraphExecPtr = std::shared_ptr<CUgraphExec_st>;
static std::map<std::string, GraphExecPtr> g_graphs;

class EngineBase {
 public:
  virtual ~EngineBase() = default;
  virtual void set_initial(const uint64_t* words, const double* c, size_t count) = 0;
  virtual void apply_gates(const pp_gate* gates, size_t count) = 0;
  virtual double apply_layer(const pp_gate* gates, size_t count) = 0;
  virtual void truncate_now() = 0;
  virtual uint64_t term_count() = 0;
  virtual double global_max() = 0;
  virtual double expectation() = 0;
  virtual double coefficient(const uint64_t* words) = 0;
  virtual uint64_t export_terms(uint64_t* words, double* c, uint64_t cap) = 0;
  virtual pp_counters take_counters() = 0;
  virtual void take_kernel_stats(double* ms, double* bytes, uint64_t* launches, uint64_t* total) = 0;
  virtual void* stream() const = 0;
  // sharding hooks (multi-GPU orchestration)
  virtual void local_stats(double* gmax, uint32_t* nonfinite, uint64_t* count) = 0;
  virtual uint64_t truncate_threshold(double T) = 0;
  virtual int record_words() const = 0;
  virtual void shard_evict(uint32_t world, uint32_t rank, uint64_t seed, uint64_t* out, uint64_t cap,
                           uint64_t* counts) = 0;
  virtual void shard_ingest(const uint64_t* rec, uint64_t count, bool device) = 0;
  virtual const uint64_t* device_records() const = 0;
  virtual void set_bucket_table(const uint16_t* table) = 0;
  virtual void bucket_histogram(uint64_t seed, uint64_t* hist) = 0;
  virtual void set_spec_reduce(std::function<void(std::vector<unsigned long long>&)> f) = 0;
  virtual void set_global_max(double g) = 0;
  virtual double norm2() = 0;
  virtual void group_sizes(uint64_t* groups, uint64_t* strings) = 0;
  virtual void histogram(int bins, double gmax, double epsilon0, uint64_t* pos, uint64_t* neg) = 0;
  // engine reuse across pp_create/pp_destroy (simulate() makes one per call)
  virtual bool reusable() const = 0;
  virtual size_t device_bytes() const = 0;
  virtual int device() const = 0;
  virtual void on_reuse() = 0;
  virtual void poison() = 0;
};

template <int W>
class EngineImpl final : public EngineBase {
 public:
  explicit EngineImpl(const pp_config& cfg) : cfg_(cfg) {
    PP_CUDA(cudaSetDevice(cfg.device));
    {
      const StreamSet ss = acquire_stream_set(cfg.device);
      stream_ = ss.stream;
      ev0_ = ss.ev0;
      ev1_ = ss.ev1;
      ev_sync_ = ss.ev_sync;
    }
    stats_buf_.ensure(sizeof(DevStats));
    d_stats_ = stats_buf_.as<DevStats>();
    h_stats_ = pinned_stats();
    spin_sync_ = std::getenv("PP_BLOCKING_SYNC") == nullptr;
    defer_ok_ = std::getenv("PP_NO_DEFER") == nullptr;
    {
      std::lock_guard<std::mutex> lk(g_setup_mu);
      LaunchSetup& ls = g_setup[{cfg.device, W}];
      if (!ls.sub_grid) {
        PP_CUDA(cudaFuncSetAttribute(k_branch_x<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)branch_x_smem_bytes<W>()));
        PP_CUDA(cudaFuncSetAttribute(k_branch_sublayer<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)branch_smem_bytes<W>()));
        PP_CUDA(cudaFuncSetAttribute(k_sort_small<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(SortSmem<W>)));
        PP_CUDA(cudaFuncSetAttribute(k_sort_big<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)big_sort_smem()));
        PP_CUDA(cudaFuncSetAttribute(k_spec_small<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)spec_small_smem_bytes<W>()));
        PP_CUDA(cudaFuncSetAttribute(k_dense_sublayer<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)dense_smem_bytes<W>()));
        PP_CUDA(cudaFuncSetAttribute(k_dense_sublayer<W>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        PP_CUDA(cudaFuncSetAttribute(k_branch_x<W>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        PP_CUDA(cudaFuncSetAttribute(k_branch_sublayer<W>, cudaFuncAttributePreferredSharedMemoryCarveout, 100));
        PP_CUDA(cudaFuncSetAttribute(k_branch_zz<W>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)sizeof(ZzSmem<W>)));
        int sms = 148, occ = 1, occ_x = 1, occ_s = 1;
        PP_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cfg.device));
        PP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_branch_zz<W>, kCta, sizeof(ZzSmem<W>)));
        // persistent branch grids: every resident CTA slot of the device
        PP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_x, k_branch_x<W>, kCta, branch_x_smem_bytes<W>()));
        PP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_s, k_branch_sublayer<W>, kCta,
                                                              branch_smem_bytes<W>()));
        ls.zz_grid = (uint32_t)(sms * std::max(occ, 1));
        ls.branch_grid = (uint32_t)(sms * std::max(occ_x, 1));
        ls.sub_grid = (uint32_t)(sms * std::max(occ_s, 1));
        int occ_d = 1;
        PP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_d, k_dense_sublayer<W>, kCta, dense_smem_bytes<W>()));
        ls.dense_grid = (uint32_t)(sms * std::max(occ_d, 1));
        int occ_k = 1;
        PP_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_k, k_spec_small<W>, kSmallWarps * 32,
                                                              spec_small_smem_bytes<W>()));
        ls.small_grid = (uint32_t)(sms * std::max(occ_k, 1));
        if (std::getenv("PP_DEBUG"))
          std::fprintf(stderr, "[pp] W=%d branch CTAs/SM %d, sublayer CTAs/SM %d, smem %zu; dense CTAs/SM %d, smem %zu\n",
                       W, occ_x, occ_s, branch_smem_bytes<W>(), occ_d, dense_smem_bytes<W>());
      }
      zz_grid_ = ls.zz_grid;
      branch_grid_ = ls.branch_grid;
      sub_grid_ = ls.sub_grid;
      dense_grid_ = ls.dense_grid;
      small_grid_ = ls.small_grid;
    }
    keep_zeros_ = cfg.cadence == PP_CADENCE_LAYER;
    seed_ = 0x5eed5eed12345678ull;
    tight_arena_ = std::getenv("PP_TIGHT_ARENA") != nullptr;
    no_dense_ = std::getenv("PP_NO_DENSE") != nullptr;
    if (const char* mk = std::getenv("PP_DENSE_MAXK")) dense_maxk_ = std::max(1, std::atoi(mk));  // test hook
    update_arena_max();
  }
  ~EngineImpl() override {
    // buffers return to the pool of the device they came from: run the
    // teardown on this engine's device whatever the caller's current one is
    int prev_dev = -1;
    cudaGetDevice(&prev_dev);
    cudaSetDevice(cfg_.device);
    cudaStreamSynchronize(stream_);
    if (std::getenv("PP_TRACE"))
      std::fprintf(stderr,
                   "[pp] trace: layers %.3f ms (clifford runs %.3f, rx runs %.3f), %llu syncs waiting %.3f ms, "
                   "launches %llu\n",
                   tr_layer_ns_ * 1e-6, tr_cliff_ns_ * 1e-6, tr_rx_ns_ * 1e-6, (unsigned long long)tr_syncs_,
                   tr_sync_ns_ * 1e-6, (unsigned long long)launches_);
    release_stream_set(cfg_.device, StreamSet{stream_, ev0_, ev1_, ev_sync_});
    {
      std::lock_guard<std::mutex> lk(g_streams_mu);
      for (auto& e : free_events_) g_event_pairs.push_back(e);
      for (auto& e : pending_events_) g_event_pairs.push_back(e);
    }
    release_pinned_stats(h_stats_);
    release_pinned_diag(h_diag_);
    release_all_buffers();  // while cfg_.device is current
    if (prev_dev >= 0) cudaSetDevice(prev_dev);
  }
  // every device buffer the engine holds (the memory plan and the engine
  // pool's size cap count them all)
  template <class F>
  void for_each_buf(F&& f) {
    for (auto& a : arena_) f(a.buf);
    for (auto& g : groups_) f(g.buf);
    for (DevBuf* b : {&evict_cnt_, &evict_buf_, &spec_buf_, &backup_, &stats_buf_, &list_, &items_, &rec_slot_,
                      &table_, &scan_tmp_, &scan_gid_, &scan_off_, &diag_z_, &diag_c_, &cliff_, &thr_, &ztab_,
                      &norms_, &sub_groups_, &buckets_, &spec_done_})
      f(*b);
  }
  size_t device_bytes() const override {
    size_t b = 0;
    const_cast<EngineImpl*>(this)->for_each_buf([&](DevBuf& d) { b += d.bytes; });
    return b;
  }
  int device() const override { return cfg_.device; }
  void release_all_buffers() {
    for_each_buf([](DevBuf& d) { d.release(); });
  }

  bool reusable() const override {
    return !poisoned_ && !sub_pending_ && !g_pending_ && !lazy_open_ && device_bytes() <= (size_t(4) << 30);
  }
  void on_reuse() override {  // set_initial resets the operator; this resets the statistics
    PP_CUDA(cudaSetDevice(cfg_.device));  // as a fresh engine's constructor does
    cudaStreamSynchronize(stream_);
    for (auto& pr : pending_events_) free_events_.push_back(pr);
    pending_events_.clear();
    branch_ms_ = 0.0;
    branch_bytes_ = 0.0;
    branch_launches_ = launches_ = 0;
    branch_in_ = branch_stream_ = 0;
    dense_groups_ = dense_out_ = bulk_tiles_ = 0;
    tr_layer_ns_ = tr_sync_ns_ = tr_syncs_ = tr_cliff_ns_ = tr_rx_ns_ = 0;
    set_initial(nullptr, nullptr, 0);  // the empty operator of a fresh engine
    counters_ = pp_counters{};
  }
  void poison() override { poisoned_ = true; }

  // ---------------------------------------------------------------- set_initial
  void set_initial(const uint64_t* words, const double* c, size_t count) override {
    // Engine::set_initial (engine.cpp:196-205): clear, then upsert in order.
    using K = std::array<uint64_t, 2 * W>;  // z (msw first) then x (msw first)
    std::map<K, double> terms;
    for (size_t i = 0; i < count; ++i) {
      uint64_t x[2], z[2];
      words_to_planes(words + 4 * i, x, z);
      if (W == 1 && (x[1] | z[1])) throw EngineError(PP_ERR_INVALID, "term has sites beyond the engine width");
      K k;
      for (int j = 0; j < W; ++j) {
        k[j] = z[W - 1 - j];
        k[W + j] = x[W - 1 - j];
      }
      auto it = terms.find(k);
      if (it == terms.end()) terms.emplace(k, c[i]);
      else it->second += c[i];
    }
    const uint64_t n = terms.size();
    std::vector<uint64_t> hx(W * std::max<uint64_t>(n, 1)), hz;
    std::vector<double> hc(std::max<uint64_t>(n, 1));
    std::vector<uint64_t> goff, gz;
    std::vector<uint32_t> gcnt;
    std::vector<double> gmx, gmn;
    std::vector<uint32_t> gfl;
    uint64_t i = 0;
    double gmax = 0.0;
    bool has_zero = false;
    K prev{};
    bool first = true;
    for (auto& [k, v] : terms) {
      bool newg = first;
      for (int j = 0; j < W && !newg; ++j) newg = k[j] != prev[j];
      if (newg) {
        goff.push_back(i);
        gcnt.push_back(0);
        for (int j = 0; j < W; ++j) gz.push_back(k[W - 1 - j]);
        gmx.push_back(0.0);
        gmn.push_back(INFINITY);
        gfl.push_back(0);
      }
      first = false;
      prev = k;
      for (int j = 0; j < W; ++j) hx[j * n + i] = k[2 * W - 1 - j];
      hc[i] = v;
      gcnt.back()++;
      double av = std::fabs(v);
      gmx.back() = std::max(gmx.back(), av);
      gmn.back() = std::min(gmn.back(), av);
      if (!std::isfinite(v)) gfl.back() = 1;
      if (v == 0.0) has_zero = true;
      gmax = std::max(gmax, av);  // global_max_abs (sparse_operator.cpp:130-134)
      ++i;
    }
    const uint32_t G = (uint32_t)gcnt.size();
    // fresh buffers
    cur_ = 0;
    // a fresh engine starts on the largest block a previous engine left in
    // the pool (simulate() creates one engine per call), else at 1 Mi strings
    if (arena_[0].cap == 0 && !tight_arena_) {
      const uint64_t warm = DevicePool::get().largest_cached(cfg_.device) / R;
      ensure_arena(0, std::min<uint64_t>(std::max<uint64_t>(warm, 1u << 20), std::max<uint64_t>(arena_max_, 1u << 16)));
    }
    ensure_arena(0, std::max<uint64_t>(1u << 16, 4 * n));
    ensure_groups(0, std::max<uint32_t>(G, 1024));
    gcur_ = 0;
    G_ = G;
    sub_pending_ = false;
    g_pending_ = false;
    unsorted_ = false;
    seen_host_ = {};
    zz_seen_pending_ = false;
    if (n <= kInitSmall && G <= kInitSmall) {
      InitSmall<W> in{};
      in.n = (uint32_t)n;
      in.G = G;
      for (uint64_t i = 0; i < n; ++i) {
        for (int j = 0; j < W; ++j) in.x[i][j] = hx[j * n + i];
        in.c[i] = hc[i];
      }
      for (uint32_t q = 0; q < G; ++q) {
        for (int j = 0; j < W; ++j) in.z[q][j] = gz[q * W + j];
        in.off[q] = goff[q];
        in.cnt[q] = gcnt[q];
        in.flags[q] = gfl[q];
        in.gmax[q] = gmx[q];
        in.gmin[q] = gmn[q];
      }
      count_param_h2d(sizeof(in));  // the initial terms travel in the parameter block
      k_init_small<W><<<1, 32, 0, stream_>>>(aview(0), gview(0), in, d_stats_);
      ++launches_;
      PP_CUDA(cudaGetLastError());
      n_small_init_ = true;
    } else {
      n_small_init_ = false;
    }
    if (n && !n_small_init_) {
      ArenaView<W> a = aview(0);
      for (int j = 0; j < W; ++j)
        PP_CUDA(copy_async(a.x[j], hx.data() + j * n, n * 8, cudaMemcpyHostToDevice, stream_));
      PP_CUDA(copy_async(a.c, hc.data(), n * 8, cudaMemcpyHostToDevice, stream_));
    }
    if (G && !n_small_init_) {
      GroupView<W> g = gview(0);
      std::vector<uint64_t> zt(G);
      for (int j = 0; j < W; ++j) {
        for (uint32_t q = 0; q < G; ++q) zt[q] = gz[q * W + j];
        PP_CUDA(copy_async(g.z[j], zt.data(), G * 8, cudaMemcpyHostToDevice, stream_));
      }
      PP_CUDA(copy_async(g.off, goff.data(), G * 8, cudaMemcpyHostToDevice, stream_));
      PP_CUDA(copy_async(g.cnt, gcnt.data(), G * 4, cudaMemcpyHostToDevice, stream_));
      PP_CUDA(copy_async(g.cap, gcnt.data(), G * 4, cudaMemcpyHostToDevice, stream_));
      PP_CUDA(copy_async(g.gmax, gmx.data(), G * 8, cudaMemcpyHostToDevice, stream_));
      PP_CUDA(copy_async(g.gmin, gmn.data(), G * 8, cudaMemcpyHostToDevice, stream_));
      PP_CUDA(copy_async(g.flags, gfl.data(), G * 4, cudaMemcpyHostToDevice, stream_));
      PP_CUDA(cudaMemsetAsync(g.stamp, 0xff, G * 4, stream_));
    }
    if (!n_small_init_) {
      reset_stats(n);
      PP_CUDA(cudaStreamSynchronize(stream_));
    }
    bump_ = bump_bound_ = n;
    live_ = live_bound_ = n;
    // group statistics a fresh engine would start from (pooled engines and a
    // second set_initial must not keep the previous operator's)
    maxcnt_ = G ? *std::max_element(gcnt.begin(), gcnt.end()) : 0u;
    zfactor_ = 4.0;
    dirty_ = false;
    truncated_since_sync_ = false;
    gmax_stale_ = false;
    may_hold_zeros_ = has_zero || keep_zeros_;
    eseq_ = bseq_ = 0;
    gmax_ = gmax;
    counters_ = pp_counters{};
    gates_applied_ = 0;
    seen_w0_ = 0;
  }

  // ---------------------------------------------------------------- gates
  void apply_gates(const pp_gate* gates, size_t count) override {
    apply_gates_async(gates, count);
    sync_state();  // errors surface at the call, as Engine::apply_gate throws
  }
  // one layer of run_circuit: the gates, then the <0|O|0> readout; errors
  // surface at the readout's sync, inside this call
  double apply_layer(const pp_gate* gates, size_t count) override {
    auto t0 = Clock::now();
    apply_gates_async(gates, count);
    const double v = expectation();
    tr_layer_ns_ += ns_since(t0);
    return v;
  }

  void apply_gates_async(const pp_gate* gates, size_t count) {
    // the partition of a gate list into runs is cached (run_circuit applies
    // the same layer every step); with a term budget, fusion depends on |O|
    const bool cacheable = cfg_.max_terms == 0;
    if (!(cacheable && plan_key_.size() == count &&
          std::memcmp(plan_key_.data(), gates, count * sizeof(pp_gate)) == 0)) {
      plan_key_.clear();
      plan_.clear();
      size_t i = 0;
      // runs are capped so one run always fits a batch window (reserve_window)
      // and an X-type run one sublayer launch
      constexpr size_t kRunCap = kSeenGates / 2;
      static_assert(kMaxSubGates <= kRunCap, "an X-type run fits the window");
      while (i < count) {
        if (fusion_allowed() && is_clifford(gates[i])) {
          size_t j = i;
          while (j < count && j - i < kRunCap && is_clifford(gates[j])) ++j;
          plan_.push_back({0, i, j});
          i = j;
        } else if (is_x_type(gates[i])) {
          size_t j = i;
          while (j < count && j - i < (size_t)kMaxSubGates && is_x_type(gates[j]) &&
                 !(fusion_allowed() && is_clifford(gates[j])))
            ++j;
          plan_.push_back({1, i, j});
          i = j;
        } else {
          plan_.push_back({2, i, i + 1});
          ++i;
        }
      }
      if (cacheable) plan_key_.assign(gates, gates + count);
    }
    const std::vector<PlanRun> plan = plan_;  // a nested call may replace plan_
    for (size_t pi = 0; pi < plan.size(); ++pi) {
      const PlanRun& r = plan[pi];
      reserve_window(r.j - r.i);
      auto t0 = Clock::now();
      if (r.kind == 0) {
        // a Clifford run feeding a dense Rx run leaves its groups unsorted
        const bool next_dense = pi + 1 < plan.size() && plan[pi + 1].kind == 1 &&
                                dense_capable(gates + plan[pi + 1].i, plan[pi + 1].j - plan[pi + 1].i);
        apply_clifford_run(gates + r.i, r.j - r.i, !next_dense);
        tr_cliff_ns_ += ns_since(t0);
      } else if (r.kind == 1) {
        run_rx(gates + r.i, r.j - r.i);
        tr_rx_ns_ += ns_since(t0);
      } else {
        apply_one(gates[r.i]);
      }
    }
  }
  // would run_rx take the dense sublayer for this X-type run (after a
  // Clifford run, which changes neither zeros nor the budget state)?
  bool dense_capable(const pp_gate* gates, size_t count) {
    if (no_dense_ || keep_zeros_ || may_hold_zeros_ || cfg_.max_terms != 0 || count > (size_t)kMaxSubGates) return false;
    if (!(external() || cfg_.epsilon0 == 0.0)) return false;
    if (rx_key_.size() == count && std::memcmp(rx_key_.data(), gates, count * sizeof(pp_gate)) == 0)
      return rx_distinct_;
    for (size_t i = 0; i < count; ++i)
      for (size_t j = 0; j < i; ++j)
        if (std::memcmp(gates[i].words, gates[j].words, sizeof(gates[i].words)) == 0) return false;
    return true;
  }
  // sort the groups a regroup left unsorted (before any consumer that needs
  // x order: the per-gate branch kernels, Z-type pairs, shard eviction)
  // pending_only (a sublayer's unsorted fault): only the groups a regroup
  // left unsorted -- the ones still waiting for the run; the class-major
  // output the run has written already stays as it is (and unsorted_ set)
  void ensure_sorted(bool pending_only = false) {
    if (!unsorted_) return;
    sync_state();
    unsorted_ = pending_only;
    if (!G_) return;
    const int mode = pending_only ? 2 : 1;
    ensure_arena(1 - cur_, std::max<uint64_t>(live_ + 1, 1024));  // merge scratch for big groups
    k_set_distinct<<<1, 1, 0, stream_>>>(d_stats_, G_);
    const uint32_t small_grid = std::max<uint32_t>(1u, std::min<uint32_t>(G_, 148u * 4u));
    const uint32_t big_grid = std::max<uint32_t>(1u, std::min<uint32_t>(G_, 148u * 2u));
    k_sort_small<W><<<small_grid, kCta, sizeof(SortSmem<W>), stream_>>>(gview(gcur_), aview(cur_), keep_zeros_, d_stats_,
                                                                         mode);
    k_sort_big<W><<<big_grid, kCta, big_sort_smem(), stream_>>>(gview(gcur_), aview(cur_), aview(1 - cur_), keep_zeros_,
                                                                 d_stats_, mode);
    launches_ += 3;
    dirty_ = true;
  }
  struct PlanRun {
    int kind;  // 0 Clifford run, 1 X-type run, 2 single gate
    size_t i, j;
  };

  // single-qubit X generator: the z-group preserving branch kernel applies
  static bool is_x_type(const pp_gate& g) {
    uint64_t jx[2], jz[2];
    words_to_planes(g.words, jx, jz);
    return (jz[0] | jz[1]) == 0 && __builtin_popcountll(jx[0]) + __builtin_popcountll(jx[1]) == 1;
  }

  struct RxParam {
    int wq;
    uint64_t mq;
    double cosv, sinv;
  };

  // A run of X-type gates: launched as one CUDA graph (captured once per
  // gate list and buffer set, replayed every layer) or as direct launches.
  // An arena overflow inside the run stops it on the device; the host then
  // compacts and resumes at the failing gate, whose finished groups carry
  // its stamp and are skipped.
  void run_rx(const pp_gate* gates, size_t count) {
    auto t0 = Clock::now();
    // run_circuit passes the same gate list every layer: the host-side plan
    // (parameters, sublayer descriptor, qubit distinctness) is cached
    if (!(rx_key_.size() == count && std::memcmp(rx_key_.data(), gates, count * sizeof(pp_gate)) == 0)) {
      rx_key_.clear();
      if (W == 1)
        for (size_t i = 0; i < count; ++i) {
          uint64_t jx[2], jz[2];
          words_to_planes(gates[i].words, jx, jz);
          if (jx[1]) throw EngineError(PP_ERR_INVALID, "generator has sites beyond the engine width");
        }
      rx_prm_.assign(count, RxParam{});
      for (size_t i = 0; i < count; ++i) {
        uint64_t jx[2], jz[2];
        words_to_planes(gates[i].words, jx, jz);
        rx_prm_[i].wq = jx[0] ? 0 : 1;
        rx_prm_[i].mq = jx[0] ? jx[0] : jx[1];
        rx_prm_[i].cosv = gates[i].cos_theta;
        rx_prm_[i].sinv = gates[i].sin_theta;
      }
      rx_sg_ = SubGates{};
      rx_distinct_ = true;
      rx_sg_.fast = std::getenv("PP_DENSE_CAREFUL") == nullptr ? 1 : 0;  // (test hook: always point by point)
      for (size_t i = 0; i < count; ++i)
        if (!(std::fabs(gates[i].sin_theta) >= 0x1p-100) || !(std::fabs(gates[i].cos_theta) >= 0x1p-100)) rx_sg_.fast = 0;
      if (count <= (size_t)kMaxSubGates) {
        rx_sg_.ng = (int)count;
        for (size_t i = 0; i < count; ++i) {
          rx_sg_.wq[i] = (int8_t)rx_prm_[i].wq;
          rx_sg_.mq[i] = rx_prm_[i].mq;
          rx_sg_.cosv[i] = rx_prm_[i].cosv;
          rx_sg_.sinv[i] = rx_prm_[i].sinv;
          rx_sg_.any[rx_prm_[i].wq] |= rx_prm_[i].mq;
          for (size_t j = 0; j < i && rx_distinct_; ++j)
            if (rx_prm_[i].wq == rx_prm_[j].wq && rx_prm_[i].mq == rx_prm_[j].mq) rx_distinct_ = false;
        }
      }
      rx_key_.assign(gates, gates + count);
    }
    const std::vector<RxParam>& prm = rx_prm_;
    const bool budget = cfg_.max_terms != 0 && !external();
    const bool epi = !external() && !(cfg_.epsilon0 == 0.0 && !budget && !may_hold_zeros_);
    const bool do_trunc = cfg_.cadence == PP_CADENCE_GATE;
    const uint64_t seq0 = bseq_;
    // epsilon0 = 0 (no global threshold), no budget: the whole run in one
    // launch, every group through its gates (k_branch_sublayer)
    const bool no_budget = !budget;
    // sharded eps0 > 0 (pp_sharded): the speculative run with every rank's
    // per-gate maxima combined (spec_reduce_), on every rank whatever its size
    const bool coordinated = external() && spec_reduce_ && cfg_.epsilon0 > 0.0 && do_trunc;
    if (coordinated) {
      if (count > (size_t)kMaxSubGates) throw EngineError(PP_ERR_INTERNAL, "sharded X-type run longer than a sublayer");
      ensure_sorted();
      if (!run_rx_speculative(prm, seq0, t0))
        throw EngineError(PP_ERR_RESOURCE, "sharded run: the speculative sublayer did not fit the device");
      return;
    }
    const bool independent = no_budget && (external() || !do_trunc || (cfg_.epsilon0 == 0.0 && !may_hold_zeros_));
    if (independent && count <= (size_t)kMaxSubGates && G_) {
      SubGates sgates = rx_sg_;
      // dense path (k_branch_sublayer / dense_group): zeros dropped, every
      // gate of the run on its own qubit
      sgates.dense = rx_distinct_ && !keep_zeros_ && !may_hold_zeros_ && !no_dense_;
      sgates.maxk = dense_maxk_;
      if (!g_pending_) sync_state();  // after a deferred regroup |O| and the bump are exact already
      if (bump_ + 2 * live_ > arena_[cur_].cap) gc_into_other(next_arena_target());
      // launched without a round trip: an arena overflow is found and
      // resumed by the next sync_state (resume_sublayer)
      sub_gates_ = sgates;
      sub_seq0_ = seq0;
      launch_sublayer();
      sub_pending_ = true;
      bseq_ = seq0 + count;
      gates_applied_ += count;
      counters_.gates += count;
      counters_.branch_ns += ns_since(t0);
      return;
    }
    ensure_sorted();  // the per-gate kernels pair strings by x order
    // epsilon0 > 0 at per-gate cadence: the whole run in one launch with
    // predicted thresholds, verified bit-exactly and rolled back otherwise
    // (PP_NO_SPECULATE: the per-gate launches below)
    const bool speculate = std::getenv("PP_NO_SPECULATE") == nullptr;
    if (speculate && no_budget && do_trunc && !external() && cfg_.epsilon0 > 0.0 && count <= (size_t)kMaxSubGates &&
        G_ && run_rx_speculative(prm, seq0, t0))
      return;
    // per-gate truncation without a budget: deferred (k_thresh / k_flush)
    const bool lazy = epi && do_trunc && no_budget && !external() && cfg_.epsilon0 > 0.0 && !keep_zeros_ &&
                      count + 2 <= kLazyWindow && std::getenv("PP_EAGER_TRUNCATION") == nullptr;
    if (lazy) thr_.ensure(kLazyWindow * sizeof(double));
    size_t pos = 0;
    while (pos < count && G_) {
      sync_state();
      if (bump_ + 2 * live_ > arena_[cur_].cap) gc_into_other(next_arena_target());
      const bool use_graph = pos == 0 && !(cfg_.flags & PP_FLAG_PROFILE);
      err_base_ = gates_applied_ + pos;  // gates applied before this launch run's gate 0
      push_scalars(seq0 + pos);
      if (lazy) {
        PP_CUDA(cudaMemsetAsync(thr_.p, 0, 2 * sizeof(double), stream_));
        lazy_open_ = true;
        lazy_base_ = seq0 + pos;
        lazy_len_ = (uint32_t)(count - pos);
      }
      if (use_graph) {
        GraphExecPtr exec = rx_graph(prm, epi, do_trunc, budget, lazy);
        held_graphs_.push_back(exec);  // alive until this stream has synchronised
        std::pair<cudaEvent_t, cudaEvent_t> ev = take_event_pair();
        PP_CUDA(cudaEventRecord(ev.first, stream_));
        count_param_h2d(count * sizeof(RxParam));  // the gate parameters baked into the graph
        PP_CUDA(cudaGraphLaunch(exec.get(), stream_));
        PP_CUDA(cudaEventRecord(ev.second, stream_));
        pending_events_.push_back(ev);
        launches_ += count * (epi ? 3 : 1);
      } else {
        for (size_t i = pos; i < count; ++i) {
          std::pair<cudaEvent_t, cudaEvent_t> ev;
          if (cfg_.flags & PP_FLAG_PROFILE) {
            ev = take_event_pair();
            PP_CUDA(cudaEventRecord(ev.first, stream_));
          }
          launch_branch(prm[i], (uint32_t)(i - pos), lazy);
          if (cfg_.flags & PP_FLAG_PROFILE) {
            PP_CUDA(cudaEventRecord(ev.second, stream_));
            pending_events_.push_back(ev);
          }
          if (epi) launch_epilogue((uint32_t)(i - pos), do_trunc, budget, lazy);
        }
      }
      branch_launches_ += count - pos;
      if (keep_zeros_) may_hold_zeros_ = true;
      if (epi && do_trunc) truncated_since_sync_ = true;
      if (!epi && do_trunc && !external()) gmax_stale_ = true;
      dirty_ = true;
      sync_state();
      if (!arena_fault_) break;
      // resume at the first gate that ran out of room
      pos = (size_t)(arena_fault_seq_ - seq0);
      k_clear_arena_error<<<1, 1, 0, stream_>>>(d_stats_);
      ++launches_;
      arena_fault_ = false;
      gc_into_other(next_arena_target());
    }
    bseq_ = seq0 + count;
    gates_applied_ += count;
    counters_.gates += count;
    counters_.branch_ns += ns_since(t0);
  }

  // epsilon0 > 0, per-gate cadence: the whole run in one launch with
  // predicted thresholds, verified bit-exactly against epsilon0 * gmax_k.
  bool run_rx_speculative(const std::vector<RxParam>& prm, uint64_t seq0, Clock::time_point t0) {
    const size_t count = prm.size();
    SubGates sgates = rx_sg_;  // the cached descriptor of this run (run_rx)
    // per-gate path only: it marks every gate's records exactly (a truncation
    // can empty a group in the middle of a dense run)
    sgates.dense = false;
    sgates.maxk = dense_maxk_;
    sgates.sorted = unsorted_ ? 0 : 1;
    sync_state();
    std::vector<double> tpred(count, cfg_.epsilon0 * gmax_);
    spec_buf_.ensure(count * 16 + 64);
    double* d_tpred = spec_buf_.as<double>();
    unsigned long long* d_gmax = reinterpret_cast<unsigned long long*>(d_tpred + count);
    if (std::getenv("PP_NO_DISCOVERY") == nullptr) discover_thresholds(sgates, seq0, tpred);
    int faults = 0;
    uint64_t need = 0;  // arena demand a faulted attempt reported (its bump overshoot)
    for (int attempt = 0; attempt < 8; ++attempt) {
      bool give_up = false;
      sync_state();
      // every gate application writes fresh space (the pre-run regions are
      // the rollback point): reserve ~24 |O| when memory allows
      // (groups keep their intermediate versions in the CTAs' L2 scratch;
      // the arena takes the results and large groups' per-gate versions)
      const uint64_t want = std::max<uint64_t>((faults ? 8 : 3) * live_ + (1u << 16), need);
      if (bump_ + want > arena_[cur_].cap) {
        size_t free_b = 0, total_b = 0;
        PP_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const size_t parked = g_parked_engine_bytes ? g_parked_engine_bytes(cfg_.device) : 0;
        const uint64_t afford =
            (uint64_t)((free_b + DevicePool::get().cached_bytes(cfg_.device) + parked + arena_[1 - cur_].buf.bytes) *
                       0.8) / R;
        give_up = live_ + want > afford && faults > 0;
        if (!give_up) gc_into_other(std::max<uint64_t>(std::min<uint64_t>(live_ + want, afford), next_arena_target()));
      }
      if (spec_reduce_) {  // all ranks give up together
        std::vector<unsigned long long> v{give_up ? 1ull : 0ull};
        spec_reduce_(v);
        give_up = v[0] != 0;
      }
      if (give_up) return false;
      // snapshot of the group table: the rollback point
      const size_t gbytes = (size_t)groups_[gcur_].cap * (8 * W + 8 + 8 + 8 + 4 + 4 + 4 + 4);
      backup_.ensure(gbytes);
      PP_CUDA(copy_async(backup_.p, groups_[gcur_].buf.p, gbytes, cudaMemcpyDeviceToDevice, stream_));
      const uint32_t G_saved = G_;
      const pp_counters saved = counters_;
      const auto saved_seen = seen_host_;
      PP_CUDA(copy_async(d_tpred, tpred.data(), count * 8, cudaMemcpyHostToDevice, stream_));
      PP_CUDA(cudaMemsetAsync(d_gmax, 0, count * 8, stream_));
      push_scalars(seq0);
      const uint64_t bump_before = bump_;
      std::pair<cudaEvent_t, cudaEvent_t> ev = take_event_pair();
      PP_CUDA(cudaEventRecord(ev.first, stream_));
      count_param_h2d(sizeof(sgates));
      // small groups a warp each, the rest (and any that outgrew a warp) a CTA each
      spec_done_.ensure(std::max<uint32_t>(G_, 1));
      PP_CUDA(cudaMemsetAsync(spec_done_.p, 0, std::max<uint32_t>(G_, 1), stream_));
      k_spec_small<W><<<small_grid_, kSmallWarps * 32, spec_small_smem_bytes<W>(), stream_>>>(
          gview(gcur_), aview(cur_), sgates, &d_stats_->work[1], d_tpred, d_gmax, d_stats_, spec_done_.as<uint8_t>());
      k_branch_sublayer<W><<<sub_grid_, kCta, branch_smem_bytes<W>(), stream_>>>(
          gview(gcur_), aview(cur_), sgates, keep_zeros_, &d_stats_->work[0], d_tpred, d_gmax, d_stats_,
          spec_done_.as<uint8_t>());
      ++launches_;
      PP_CUDA(cudaEventRecord(ev.second, stream_));
      pending_events_.push_back(ev);
      ++launches_;
      ++branch_launches_;
      std::vector<unsigned long long> gm(count);
      PP_CUDA(copy_async(gm.data(), d_gmax, count * 8, cudaMemcpyDeviceToHost, stream_));
      dirty_ = true;
      sync_state();  // harvests counters, reads the arena fault flag
      bool any_fault = arena_fault_;
      bool nonfinite = h_stats_->red[2].nonfinite != 0;
      if (spec_reduce_) {
        std::vector<unsigned long long> v(gm);
        v.push_back(any_fault ? 1ull : 0ull);
        v.push_back(nonfinite ? 1ull : 0ull);
        spec_reduce_(v);
        std::copy(v.begin(), v.begin() + count, gm.begin());
        any_fault = v[count] != 0;
        nonfinite = v[count + 1] != 0;
      }
      bool exact = !any_fault;
      std::vector<double> tobs(count);
      for (size_t k = 0; k < count; ++k) {
        tobs[k] = cfg_.epsilon0 * __builtin_bit_cast(double, gm[k]);  // engine.cpp:345
        if (__builtin_bit_cast(uint64_t, tobs[k]) != __builtin_bit_cast(uint64_t, tpred[k])) exact = false;
      }
      if (exact && nonfinite)
        throw EngineError(PP_ERR_NUMERICAL, "non-finite coefficient in gates " + std::to_string(gates_applied_ + 1) +
                                                ".." + std::to_string(gates_applied_ + count));
      if (exact) {
        gmax_ = __builtin_bit_cast(double, gm[count - 1]);
        truncated_since_sync_ = false;
        bseq_ = seq0 + count;
        gates_applied_ += count;
        counters_.gates += count;
        counters_.branch_ns += ns_since(t0);
        spec_attempts_ += attempt + 1;
        if (std::getenv("PP_DEBUG"))
          std::fprintf(stderr, "[pp] speculative run of %zu gates accepted after %d attempt(s)\n", count, attempt + 1);
        return true;
      }
      // roll back: restore the table (the old regions are untouched)
      PP_CUDA(copy_async(groups_[gcur_].buf.p, backup_.p, gbytes, cudaMemcpyDeviceToDevice, stream_));
      G_ = G_saved;
      counters_ = saved;
      seen_host_ = saved_seen;  // the rejected attempt's batch marks
      if (std::getenv("PP_DEBUG")) {
        size_t first = 0;
        while (first < count && __builtin_bit_cast(uint64_t, tobs[first]) == __builtin_bit_cast(uint64_t, tpred[first]))
          ++first;
        if (first < count)
          std::fprintf(stderr, "[pp]   gate %zu: predicted %.17g (%016llx) observed %.17g (%016llx) gmax_=%.17g\n", first,
                       tpred[first], (unsigned long long)__builtin_bit_cast(uint64_t, tpred[first]), tobs[first],
                       (unsigned long long)gm[first], gmax_);
      }
      if (any_fault) {
        // the kernels keep bumping past the capacity: what they asked for,
        // plus the live strings, sizes the next attempt
        need = std::max<uint64_t>(need, (bump_ > bump_before ? bump_ - bump_before : 0) + live_ / 2 + (1u << 16));
        if (spec_reduce_) {  // every rank sizes for the largest demand
          std::vector<unsigned long long> v{need};
          spec_reduce_(v);
          need = v[0];
        }
        if (arena_fault_) {
          k_clear_arena_error<<<1, 1, 0, stream_>>>(d_stats_);
          ++launches_;
          arena_fault_ = false;
        }
        if (++faults >= 4) {  // cannot hold a whole speculative run: gates one by one
          dirty_ = true;
          sync_state();
          gc_into_other(next_arena_target());
          return false;
        }
        // the faulted run saw a subset of the groups: its maxima are lower
        // bounds of the true ones, so they can only raise the prediction
        // (a threshold predicted too low keeps too many strings -- the usual
        // cause of the fault)
        for (size_t k = 0; k < count; ++k)
          if (tobs[k] > tpred[k]) tpred[k] = tobs[k];
      } else {
        tpred = tobs;
      }
      dirty_ = true;
      sync_state();
      if (std::getenv("PP_DEBUG")) {
        size_t first = 0;
        while (first < count && tobs[first] == tpred[first]) ++first;
        std::fprintf(stderr, "[pp] speculative run of %zu gates: attempt %d rejected (faults %d, first mismatch at %zu)\n",
                     count, attempt, faults, first);
      }
    }
    return false;  // did not converge: the caller runs the gates one by one
  }

  // The exact thresholds of the run from the groups that can hold its maxima
  // (k_group_norms / k_select_groups): the speculative sublayer on that
  // subset alone, iterated to a fixed point, outputs discarded (the bump
  // pointer and the statistics are reset afterwards).  On success tpred holds
  // epsilon0 * gmax_k for every gate; otherwise it is left as it was.
  void discover_thresholds(const SubGates& sgates, uint64_t seq0, std::vector<double>& tpred) {
    const size_t count = tpred.size();
    // (sharded: every rank takes part in every collective, empty or not)
    if (!(gmax_ > 0.0) || (G_ == 0 && !spec_reduce_)) return;
    const uint64_t bump0 = bump_;
    norms_.ensure((size_t)G_ * 8 + 64);
    ensure_sub_groups(std::max<uint32_t>(G_, 1));
    double* d_norm = norms_.as<double>();
    unsigned int* d_count = reinterpret_cast<unsigned int*>(d_norm + G_);
    double* d_tp = spec_buf_.as<double>();
    unsigned long long* d_gm = reinterpret_cast<unsigned long long*>(d_tp + count);
    push_scalars(seq0);
    k_group_norms<W><<<persistent_grid(), kCta, 0, stream_>>>(gview(gcur_), aview(cur_), d_stats_, d_norm);
    ++launches_;
    std::vector<double> tp(count, cfg_.epsilon0 * gmax_), tobs(count);
    std::vector<unsigned long long> gm(count);
    double L = 0.25 * gmax_;
    bool ok = false;
    for (int round = 0; round < 4 && !ok; ++round) {
      bool fixed = false;
      for (int attempt = 0; attempt < 8 && !fixed; ++attempt) {
        // a fresh copy of the subset's table entries (the run rewrites them)
        PP_CUDA(cudaMemsetAsync(d_count, 0, 4, stream_));
        k_set_scalars<<<1, 1, 0, stream_>>>(d_stats_, G_, arena_[cur_].cap, seq0, window_index());
        k_select_groups<W><<<std::max<uint32_t>(1u, blocks(G_)), kCta, 0, stream_>>>(gview(gcur_), d_stats_, d_norm, L,
                                                                                     sub_view(), d_count);
        k_use_group_count<<<1, 1, 0, stream_>>>(d_stats_, d_count, bump0);
        launches_ += 2;
        PP_CUDA(copy_async(d_tp, tp.data(), count * 8, cudaMemcpyHostToDevice, stream_));
        PP_CUDA(cudaMemsetAsync(d_gm, 0, count * 8, stream_));
        spec_done_.ensure(std::max<uint32_t>(G_, 1));
        PP_CUDA(cudaMemsetAsync(spec_done_.p, 0, std::max<uint32_t>(G_, 1), stream_));
        k_spec_small<W><<<small_grid_, kSmallWarps * 32, spec_small_smem_bytes<W>(), stream_>>>(
            sub_view(), aview(cur_), sgates, &d_stats_->work[1], d_tp, d_gm, d_stats_, spec_done_.as<uint8_t>());
        k_branch_sublayer<W><<<sub_grid_, kCta, branch_smem_bytes<W>(), stream_>>>(
            sub_view(), aview(cur_), sgates, keep_zeros_, &d_stats_->work[0], d_tp, d_gm, d_stats_,
            spec_done_.as<uint8_t>());
        launches_ += 3;
        PP_CUDA(copy_async(gm.data(), d_gm, count * 8, cudaMemcpyDeviceToHost, stream_));
        fetch_stats();
        PP_CUDA(cudaGetLastError());
        if (spec_reduce_) {
          std::vector<unsigned long long> v(gm);
          v.push_back(h_stats_->err_arena ? 1ull : 0ull);
          spec_reduce_(v);
          std::copy(v.begin(), v.begin() + count, gm.begin());
          if (v[count]) break;
        } else if (h_stats_->err_arena) {
          break;  // no room for the subset's outputs: plain speculation
        }
        fixed = true;
        for (size_t k = 0; k < count; ++k) {
          tobs[k] = cfg_.epsilon0 * __builtin_bit_cast(double, gm[k]);  // engine.cpp:345
          if (__builtin_bit_cast(uint64_t, tobs[k]) != __builtin_bit_cast(uint64_t, tp[k])) fixed = false;
        }
        tp = tobs;
      }
      if (!fixed) break;
      double mn = INFINITY;
      for (size_t k = 0; k < count; ++k) mn = std::min(mn, __builtin_bit_cast(double, gm[k]));
      if (mn >= L) {
        ok = true;
      } else {
        L = 0.5 * mn;  // a max fell below the bound: widen the subset
      }
      if (std::getenv("PP_DEBUG"))
        std::fprintf(stderr, "[pp] discovery round %d: L=%.6g min gmax_k=%.6g subset %u groups -> %s\n", round, L,
                     mn, h_stats_->G_dev, ok ? "ok" : "widen");
    }
    reset_stats(bump0);  // discard the subset runs' outputs and counters
    if (ok) {
      tpred = tp;
      ++discoveries_;
    }
  }
  GroupView<W> sub_view() const {
    GroupView<W> v;
    const uint64_t C = sub_cap_;
    char* b = sub_groups_.template as<char>();
    for (int k = 0; k < W; ++k) v.z[k] = reinterpret_cast<uint64_t*>(b) + k * C;
    char* p = b + W * C * 8;
    v.off = reinterpret_cast<uint64_t*>(p);
    p += C * 8;
    v.gmax = reinterpret_cast<double*>(p);
    p += C * 8;
    v.gmin = reinterpret_cast<double*>(p);
    p += C * 8;
    v.cnt = reinterpret_cast<uint32_t*>(p);
    p += C * 4;
    v.cap = reinterpret_cast<uint32_t*>(p);
    p += C * 4;
    v.flags = reinterpret_cast<uint32_t*>(p);
    p += C * 4;
    v.stamp = reinterpret_cast<uint32_t*>(p);
    return v;
  }
  void ensure_sub_groups(uint32_t n) {
    if (sub_cap_ >= n) return;
    sub_groups_.ensure((size_t)n * (8 * W + 8 + 8 + 8 + 4 + 4 + 4 + 4));
    sub_cap_ = n;
  }

  void launch_sublayer() {
    sub_gates_.sorted = unsorted_ ? 0 : 1;
    push_scalars(sub_seq0_);
    std::pair<cudaEvent_t, cudaEvent_t> ev = take_event_pair();
    PP_CUDA(cudaEventRecord(ev.first, stream_));
    // persistent grid, but no more CTAs than a few per group (tiny layers)
    const uint32_t grid = std::max<uint32_t>(1u, std::min<uint32_t>(sub_grid_, 4u * G_));
    count_param_h2d(sizeof(sub_gates_));  // the run's gate list
    if (sub_gates_.dense && !no_dense_kernel_) {
      // the dense path in its own kernel; what it leaves behind (left_list_,
      // DevStats::left_n) goes through the per-gate path right after it
      left_list_.ensure((size_t)std::max<uint32_t>(2u * G_, 4096u) * sizeof(uint32_t));
      const uint32_t dgrid = std::max<uint32_t>(1u, std::min<uint32_t>(dense_grid_, 4u * G_));
      k_dense_sublayer<W><<<dgrid, kCta, dense_smem_bytes<W>(), stream_>>>(
          gview(gcur_), aview(cur_), sub_gates_, &d_stats_->work[0], d_stats_, left_list_.as<uint32_t>());
      SubGates rest = sub_gates_;
      rest.dense = 0;
      k_branch_sublayer<W><<<grid, kCta, branch_smem_bytes<W>(), stream_>>>(
          gview(gcur_), aview(cur_), rest, keep_zeros_, &d_stats_->work[1], nullptr, nullptr, d_stats_, nullptr,
          left_list_.as<uint32_t>());
      ++launches_;
    } else {
      k_branch_sublayer<W><<<grid, kCta, branch_smem_bytes<W>(), stream_>>>(
          gview(gcur_), aview(cur_), sub_gates_, keep_zeros_, &d_stats_->work[0], nullptr, nullptr, d_stats_);
    }
    PP_CUDA(cudaEventRecord(ev.second, stream_));
    pending_events_.push_back(ev);
    ++launches_;
    ++branch_launches_;
    // a group with several x classes leaves the dense path class-major
    // (kFlagUnsorted | kFlagMinFirst, dense_multi)
    if (sub_gates_.dense && sub_gates_.maxk > 1) unsorted_ = true;
    if (keep_zeros_) may_hold_zeros_ = true;
    if (cfg_.cadence == PP_CADENCE_GATE && !external()) gmax_stale_ = true;
    dirty_ = true;
  }
  // a sublayer stopped on an arena overflow: compact into a larger arena and
  // relaunch; groups that finished carry the run's stamps and are skipped
  void resume_sublayer(bool diag) {
    sub_pending_ = false;
    int unsorted_faults = 0;
    for (int attempt = 0; arena_fault_ || unsorted_fault_; ++attempt) {
      if (attempt > 64) throw EngineError(PP_ERR_RESOURCE, "arena cannot hold the sublayer");
      k_clear_arena_error<<<1, 1, 0, stream_>>>(d_stats_);
      ++launches_;
      if (arena_fault_) {
        arena_fault_ = false;
        // repeated overflows (a dense block larger than the usual growth):
        // at least double the arena
        gc_into_other(attempt >= 2 ? std::max<uint64_t>(next_arena_target(),
                                                        std::min<uint64_t>(2 * arena_[cur_].cap, arena_max_))
                                   : next_arena_target());
      }
      if (unsorted_fault_) {  // groups the per-gate path needs sorted
        unsorted_fault_ = false;
        // (a second fault in a row: a group an earlier dense run left
        // class-major is among them -- sort everything)
        ensure_sorted(/*pending_only=*/unsorted_faults++ == 0);
      }
      launch_sublayer();
      sync_state(diag);
    }
  }

  void launch_branch(const RxParam& p, uint32_t rel, bool lazy) {
    count_param_h2d(sizeof(RxParam));
    k_branch_x<W><<<branch_grid_, kCta, branch_x_smem_bytes<W>(), stream_>>>(
        gview(gcur_), aview(cur_), p.wq, p.mq, p.cosv, p.sinv, keep_zeros_, gview(gcur_).z[p.wq],
        &d_stats_->work[rel & 1], &d_stats_->work[(rel + 1) & 1], rel, d_stats_,
        lazy ? thr_.as<double>() : nullptr, lazy ? &d_stats_->red[rel & 1] : nullptr);
    ++launches_;
  }

  GraphExecPtr rx_graph(const std::vector<RxParam>& prm, bool epi, bool do_trunc, bool budget, bool lazy) {
    std::string key;
    auto put = [&](const void* p, size_t n) { key.append(static_cast<const char*>(p), n); };
    GroupView<W> gv = gview(gcur_);
    ArenaView<W> av = aview(cur_);
    put(&gv, sizeof(gv));
    put(&av, sizeof(av));
    put(&d_stats_, sizeof(d_stats_));
    put(&cfg_.epsilon0, sizeof(double));
    put(&cfg_.max_terms, sizeof(uint64_t));
    int dev = cfg_.device;
    put(&dev, sizeof(dev));
    int w = W;
    put(&w, sizeof(w));
    int flags = (epi ? 1 : 0) | (do_trunc ? 2 : 0) | (budget ? 4 : 0) | (keep_zeros_ ? 8 : 0) | (lazy ? 16 : 0);
    put(&flags, sizeof(flags));
    void* thr = thr_.p;
    put(&thr, sizeof(thr));
    for (const RxParam& p : prm) put(&p, sizeof(p));
    // process-wide cache: engines built one per simulate() call get the same
    // pooled buffers, so their graphs are identical and reused
    std::lock_guard<std::mutex> lk(g_graph_mu);
    auto it = g_graphs.find(key);
    if (it != g_graphs.end()) return it->second;
    if (g_graphs.size() > 64) g_graphs.clear();  // holders keep their execs alive
    cudaGraph_t graph;
    PP_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    const uint64_t saved = launches_;
    for (size_t i = 0; i < prm.size(); ++i) {
      launch_branch(prm[i], (uint32_t)i, lazy);
      if (epi) launch_epilogue((uint32_t)i, do_trunc, budget, lazy);
    }
    launches_ = saved;
    PP_CUDA(cudaStreamEndCapture(stream_, &graph));
    cudaGraphExec_t raw;
    PP_CUDA(cudaGraphInstantiate(&raw, graph, 0));
    cudaGraphDestroy(graph);
    GraphExecPtr exec(raw, GraphExecDeleter{});
    g_graphs.emplace(key, exec);
    return exec;
  }

  // Memory plan: two arenas (current + compaction/regroup target) of at
  // most arena_max_ strings each, plus ~16 B per string of regroup slots and
  // group tables and a fixed reserve.  Re-planned before every arena
  // allocation from what is free now, the pool's cached blocks and this
  // engine's own arenas.
  void update_arena_max() {
    size_t free_b = 0, total_b = 0;
    PP_CUDA(cudaMemGetInfo(&free_b, &total_b));
    // parked engines' buffers are released on demand (DevicePool::acquire),
    // so they count as available
    const size_t parked = g_parked_engine_bytes ? g_parked_engine_bytes(cfg_.device) : 0;
    const size_t avail = free_b + DevicePool::get().cached_bytes(cfg_.device) + parked + arena_[0].buf.bytes +
                         arena_[1].buf.bytes;
    const double frac = cfg_.mem_fraction > 0 && cfg_.mem_fraction <= 1 ? cfg_.mem_fraction : 0.92;
    const double budget = (double)avail * frac - (double)(3ull << 30);
    arena_max_ = budget > 0 ? (uint64_t)(budget / (double)(2 * R + 16)) : (1ull << 20);
    // a coarse grain: free memory wobbles by a few MB from call to call, and an
    // engine that asks for a slightly larger arena than the last one released
    // misses the pool's cached block (a fresh cudaMalloc of tens of GB)
    if (arena_max_ > (1ull << 28)) arena_max_ &= ~((1ull << 26) - 1);
  }

  // memory is short: free this device's parked engines and the pool's cache,
  // then plan again
  void reclaim_parked() {
    if (g_release_parked_engines) g_release_parked_engines(cfg_.device);
    DevicePool::get().trim(cfg_.device);
    update_arena_max();
  }

  // arena capacity for the next compaction: room to grow ~2x without
  // another compaction, generous for small states, never above the memory
  // plan's arena_max_ (the other arena must fit too)
  uint64_t next_arena_target() {
    if (tight_arena_) return live_ + live_ / 8 + 1024;  // test hook: exercise overflow and resume
    if (8 * live_ + 1024 > arena_max_) update_arena_max();  // re-plan only when it matters
    const uint64_t lo = live_ + live_ / 8 + (1u << 16);
    // 8x while the plan allows (fewer compactions), at least 3x
    const uint64_t want = std::max<uint64_t>(3 * live_ + 1024, std::min<uint64_t>(8 * live_, arena_max_));
    uint64_t t = std::min<uint64_t>(std::max<uint64_t>(want, arena_[cur_].cap), arena_max_);
    if (t < lo) {
      if (lo > arena_max_) reclaim_parked();
      if (lo > arena_max_)
        throw EngineError(PP_ERR_RESOURCE, "device memory exhausted: " + std::to_string(live_) +
                                               " live strings exceed the arena plan of " +
                                               std::to_string(arena_max_) + " strings");
      t = lo;
    }
    return t;
  }

  // regroup target arena: the exact output plus slack, within the plan
  uint64_t regroup_arena(uint64_t total) {
    if (2 * total + (1u << 16) > arena_max_) update_arena_max();
    if (total + 1 > arena_max_) reclaim_parked();
    if (total + 1 > arena_max_)
      throw EngineError(PP_ERR_RESOURCE, "device memory exhausted: " + std::to_string(total) +
                                             " strings after regroup exceed the arena plan of " +
                                             std::to_string(arena_max_) + " strings");
    if (tight_arena_) return total + 1024;
    return std::min<uint64_t>(std::max<uint64_t>(total + (1u << 16), total + total / 2), arena_max_);
  }

  void truncate_now() override {
    auto t0 = Clock::now();
    epilogue(/*do_truncate=*/true, /*check_budget=*/false);
    sync_state();
    counters_.truncate_ns += ns_since(t0);
  }

  uint64_t term_count() override {
    sync_state();
    return live_;
  }
  double global_max() override {
    sync_state();
    return gmax_;
  }

  double expectation() override {
    // expectation_zero_state (sparse_operator.cpp:89-97): sum over strings
    // with no X/Y.  Summed on the host in ascending z order with Neumaier
    // compensation, so the value is deterministic.  The diagonal pass shares
    // the sync's round trip (sync_state(true)).
    sync_state(true);
    if (G_ == 0) return 0.0;
    const uint64_t nd = diag_n_;
    std::vector<uint64_t> z(nd * W);
    std::vector<double> c(nd);
    if (nd <= diag_copied_) {
      std::memcpy(z.data(), h_diag_->z, nd * W * 8);
      std::memcpy(c.data(), h_diag_->c, nd * 8);
    } else {
      PP_CUDA(copy_async(z.data(), diag_z_.p, nd * W * 8, cudaMemcpyDeviceToHost, stream_));
      PP_CUDA(copy_async(c.data(), diag_c_.p, nd * 8, cudaMemcpyDeviceToHost, stream_));
      PP_CUDA(cudaStreamSynchronize(stream_));
    }
    std::vector<uint64_t> order(nd);
    for (uint64_t i = 0; i < nd; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
      for (int k = W - 1; k >= 0; --k)
        if (z[a * W + k] != z[b * W + k]) return z[a * W + k] < z[b * W + k];
      return false;
    });
    double s = 0.0, comp = 0.0;
    for (uint64_t i : order) {
      double v = c[i];
      double t = s + v;
      if (std::fabs(s) >= std::fabs(v)) comp += (s - t) + v;
      else comp += (v - t) + s;
      s = t;
    }
    return s + comp;
  }

  double coefficient(const uint64_t* words) override {
    sync_state();
    uint64_t x[2], z[2];
    words_to_planes(words, x, z);
    if (W == 1 && (x[1] | z[1])) return 0.0;
    if (G_ == 0) return 0.0;
    PP_CUDA(cudaStreamSynchronize(stream_));  // legacy-stream copies below
    GroupView<W> g = gview(gcur_);
    std::vector<uint64_t> gz(G_);
    std::vector<uint32_t> match(G_, 1);
    for (int k = 0; k < W; ++k) {
      PP_CUDA(copy_sync(gz.data(), g.z[k], G_ * 8, cudaMemcpyDeviceToHost));
      for (uint32_t i = 0; i < G_; ++i) match[i] &= gz[i] == z[k];
    }
    for (uint32_t i = 0; i < G_; ++i) {
      if (!match[i]) continue;
      uint64_t off;
      uint32_t cnt;
      PP_CUDA(copy_sync(&off, g.off + i, 8, cudaMemcpyDeviceToHost));
      PP_CUDA(copy_sync(&cnt, g.cnt + i, 4, cudaMemcpyDeviceToHost));
      if (!cnt) continue;
      ArenaView<W> a = aview(cur_);
      std::vector<uint64_t> xs(cnt * W);
      std::vector<double> cs(cnt);
      for (int k = 0; k < W; ++k)
        PP_CUDA(copy_sync(xs.data() + k * cnt, a.x[k] + off, cnt * 8, cudaMemcpyDeviceToHost));
      PP_CUDA(copy_sync(cs.data(), a.c + off, cnt * 8, cudaMemcpyDeviceToHost));
      for (uint32_t e = 0; e < cnt; ++e) {
        bool eq = true;
        for (int k = 0; k < W; ++k) eq &= xs[k * cnt + e] == x[k];
        if (eq) return cs[e];
      }
    }
    return 0.0;
  }

  uint64_t export_terms(uint64_t* words, double* c, uint64_t cap) override {
    sync_state();
    if (live_ > cap) throw EngineError(PP_ERR_INVALID, "export capacity too small");
    compact();  // one contiguous live range in the current arena
    // the copies below run on the legacy stream, which does not order with
    // the engine's non-blocking stream
    PP_CUDA(cudaStreamSynchronize(stream_));
    const uint64_t n = live_;
    std::vector<uint64_t> xs(n * W), zs;
    std::vector<double> cs(n);
    std::vector<uint64_t> goff(G_), gz(G_ * W);
    std::vector<uint32_t> gcnt(G_);
    if (n) {
      ArenaView<W> a = aview(cur_);
      for (int k = 0; k < W; ++k)
        PP_CUDA(copy_sync(xs.data() + k * n, a.x[k], n * 8, cudaMemcpyDeviceToHost));
      PP_CUDA(copy_sync(cs.data(), a.c, n * 8, cudaMemcpyDeviceToHost));
    }
    if (G_) {
      GroupView<W> g = gview(gcur_);
      PP_CUDA(copy_sync(goff.data(), g.off, G_ * 8, cudaMemcpyDeviceToHost));
      PP_CUDA(copy_sync(gcnt.data(), g.cnt, G_ * 4, cudaMemcpyDeviceToHost));
      for (int k = 0; k < W; ++k)
        PP_CUDA(copy_sync(gz.data() + k * G_, g.z[k], G_ * 8, cudaMemcpyDeviceToHost));
    }
    std::vector<std::array<uint64_t, 4>> out;
    std::vector<double> outc;
    out.reserve(n);
    outc.reserve(n);
    for (uint32_t gi = 0; gi < G_; ++gi) {
      uint64_t zz[2] = {gz[gi], W == 2 ? gz[G_ + gi] : 0};
      for (uint32_t e = 0; e < gcnt[gi]; ++e) {
        uint64_t p = goff[gi] + e;
        uint64_t xx[2] = {xs[p], W == 2 ? xs[n + p] : 0};
        std::array<uint64_t, 4> w;
        planes_to_words(xx, zz, w.data());
        out.push_back(w);
        outc.push_back(cs[p]);
      }
    }
    std::vector<uint64_t> order(out.size());
    for (uint64_t i = 0; i < order.size(); ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](uint64_t a, uint64_t b) {
      for (int k = 3; k >= 0; --k)
        if (out[a][k] != out[b][k]) return out[a][k] < out[b][k];
      return false;
    });
    for (uint64_t i = 0; i < order.size(); ++i) {
      std::memcpy(words + 4 * i, out[order[i]].data(), 32);
      c[i] = outc[order[i]];
    }
    return order.size();
  }

  void* stream() const override { return (void*)stream_; }

  // ---------------------------------------------------------------- sharding
  void local_stats(double* gmax, uint32_t* nonfinite, uint64_t* count) override {
    dirty_ = true;
    sync_state();
    *gmax = __builtin_bit_cast(double, h_stats_->red[2].gmax_bits);
    *nonfinite = h_stats_->red[2].nonfinite;
    *count = live_;
  }

  uint64_t truncate_threshold(double T) override {
    sync_state();
    const uint64_t before = counters_.removed;
    if (G_) {
      push_scalars(bseq_);
      k_truncate_T<W><<<persistent_grid(), kCta, 0, stream_>>>(gview(gcur_), aview(cur_), T, d_stats_);
      ++launches_;
      dirty_ = true;
      sync_state();
    }
    // gmax_ stays what the orchestrator set (pp_set_global_max): the
    // speculative sharded run predicts its thresholds from it
    return counters_.removed - before;
  }

  int record_words() const override { return 2 * W + 1; }

  // z-groups by size: groups[b] / strings[b] for sizes in [2^b, 2^(b+1))
  void group_sizes(uint64_t* groups, uint64_t* strings) override {
    sync_state();
    for (int b = 0; b < 64; ++b) groups[b] = strings[b] = 0;
    if (G_ == 0) return;
    std::vector<uint32_t> cnt(G_);
    PP_CUDA(copy_sync(cnt.data(), gview(gcur_).cnt, (size_t)G_ * 4, cudaMemcpyDeviceToHost));
    for (uint32_t c : cnt)
      if (c) {
        const int b = 31 - __builtin_clz(c);
        ++groups[b];
        strings[b] += c;
      }
  }
  double norm2() override {
    sync_state();
    if (G_ == 0) return 0.0;
    evict_cnt_.ensure(64);
    double* acc = evict_cnt_.as<double>();
    PP_CUDA(cudaMemsetAsync(acc, 0, 8, stream_));
    push_scalars(bseq_);
    k_norm2<W><<<persistent_grid(), kCta, 0, stream_>>>(gview(gcur_), aview(cur_), d_stats_, acc);
    double h = 0.0;
    PP_CUDA(copy_async(&h, acc, 8, cudaMemcpyDeviceToHost, stream_));
    PP_CUDA(cudaStreamSynchronize(stream_));
    return h;
  }

  void histogram(int bins, double gmax, double epsilon0, uint64_t* pos, uint64_t* neg) override {
    sync_state();
    for (int b = 0; b < bins; ++b) pos[b] = neg[b] = 0;
    if (G_ == 0) return;
    const double lower = std::max(epsilon0, 1e-16);
    // The reference bins ax = |c / gmax| in (lower, 1) by
    // int(bins * (1 - std::log(ax) / log_lower)) (sparse_operator.cpp:177-186),
    // with the host's libm log.  That map is monotone in ax, so it is fixed by
    // its bin edges: edge[b] = the smallest double whose bin is >= b, found
    // here by bisection over the ordered bit patterns with the very same host
    // expression.  The kernel counts edges <= ax -- no device log, so a
    // 1-ulp libm difference cannot move a string across a bin boundary.
    const double log_lower = std::log(lower);
    auto bin_of = [&](double ax) {
      int b = static_cast<int>(bins * (1.0 - std::log(ax) / log_lower));
      return std::clamp(b, 0, bins - 1);
    };
    std::vector<double> edges(bins > 1 ? bins - 1 : 1, 2.0);
    for (int b = 1; b < bins; ++b) {
      uint64_t lo = __builtin_bit_cast(uint64_t, lower), hi = __builtin_bit_cast(uint64_t, 1.0);
      if (!(lower < 1.0) || bin_of(std::nextafter(1.0, 0.0)) < b) {
        edges[b - 1] = 1.0;  // only ax >= 1 (the last bin) reaches it
        continue;
      }
      // invariant: bin(lo) < b or lo == lower (excluded), bin(hi - 1ulp) >= b
      while (hi - lo > 1) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (bin_of(__builtin_bit_cast(double, mid)) >= b) hi = mid;
        else lo = mid;
      }
      edges[b - 1] = __builtin_bit_cast(double, hi);
    }
    const size_t ne = edges.size();
    evict_cnt_.ensure(16 * (size_t)bins + 8 * ne);
    unsigned long long* d = evict_cnt_.as<unsigned long long>();
    double* d_edges = reinterpret_cast<double*>(d + 2 * (size_t)bins);
    PP_CUDA(cudaMemsetAsync(d, 0, 16 * (size_t)bins, stream_));
    PP_CUDA(copy_async(d_edges, edges.data(), 8 * ne, cudaMemcpyHostToDevice, stream_));
    push_scalars(bseq_);
    const size_t smem = 8 * (size_t)((bins + 1) & ~1) + 8 * ne;
    if (smem > 48 * 1024)
      PP_CUDA(cudaFuncSetAttribute(k_histogram<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_histogram<W><<<persistent_grid(), kCta, smem, stream_>>>(gview(gcur_), aview(cur_), d_stats_, bins, gmax,
                                                               lower, d_edges, d, d + bins);
    ++launches_;
    PP_CUDA(copy_async(pos, d, 8 * (size_t)bins, cudaMemcpyDeviceToHost, stream_));
    PP_CUDA(copy_async(neg, d + bins, 8 * (size_t)bins, cudaMemcpyDeviceToHost, stream_));
    PP_CUDA(cudaStreamSynchronize(stream_));
  }

  void shard_evict(uint32_t world, uint32_t rank, uint64_t seed, uint64_t* out, uint64_t cap,
                   uint64_t* counts) override {
    sync_state();
    for (uint32_t d = 0; d < world; ++d) counts[d] = 0;
    if (G_ == 0) return;
    evict_cnt_.ensure(world * 8 * 2);
    unsigned long long* dcnt = evict_cnt_.as<unsigned long long>();
    PP_CUDA(cudaMemsetAsync(dcnt, 0, world * 8, stream_));
    k_evict_count<W><<<blocks(G_), kCta, 0, stream_>>>(gview(gcur_), G_, world, rank, seed, dcnt, bucket_table());
    std::vector<unsigned long long> hc(world);
    PP_CUDA(copy_async(hc.data(), dcnt, world * 8, cudaMemcpyDeviceToHost, stream_));
    PP_CUDA(cudaStreamSynchronize(stream_));
    uint64_t total = 0;
    std::vector<unsigned long long> off(world);
    for (uint32_t d = 0; d < world; ++d) {
      off[d] = total;
      total += hc[d];
      counts[d] = hc[d];
    }
    if (total > cap) throw EngineError(PP_ERR_INVALID, "evict: output capacity too small");
    if (total == 0) return;
    const int rw = 2 * W + 1;
    evict_buf_.ensure(total * rw * 8);
    PP_CUDA(copy_async(dcnt + world, off.data(), world * 8, cudaMemcpyHostToDevice, stream_));
    k_evict_write<W><<<G_, kCta, 0, stream_>>>(gview(gcur_), aview(cur_), world, rank, seed, dcnt + world,
                                               evict_buf_.as<uint64_t>(), bucket_table());
    if (out)  // host-staged exchange; otherwise the records stay in evict_buf_ (device_records())
      PP_CUDA(copy_async(out, evict_buf_.p, total * rw * 8, cudaMemcpyDeviceToHost, stream_));
    PP_CUDA(cudaStreamSynchronize(stream_));
    launches_ += 2;
    dirty_ = true;
    sync_state();
  }

  const uint64_t* device_records() const override { return evict_buf_.as<uint64_t>(); }

  // ---- sharded use (pp_sharded.cuh)
  void set_bucket_table(const uint16_t* table) override {  // kBuckets entries, or nullptr: hash mod world
    if (!table) {
      buckets_on_ = false;
      return;
    }
    buckets_.ensure(kBuckets * sizeof(uint16_t));
    PP_CUDA(copy_async(buckets_.p, table, kBuckets * sizeof(uint16_t), cudaMemcpyHostToDevice, stream_));
    buckets_on_ = true;
  }
  const uint16_t* bucket_table() const { return buckets_on_ ? buckets_.as<uint16_t>() : nullptr; }
  void bucket_histogram(uint64_t seed, uint64_t* hist) override {  // kBuckets strings-per-bucket counts
    sync_state();
    evict_cnt_.ensure(kBuckets * 8);
    unsigned long long* d = evict_cnt_.as<unsigned long long>();
    PP_CUDA(cudaMemsetAsync(d, 0, kBuckets * 8, stream_));
    if (G_) {
      k_bucket_hist<W><<<blocks(G_), kCta, 0, stream_>>>(gview(gcur_), G_, seed, d);
      ++launches_;
    }
    PP_CUDA(copy_async(hist, d, kBuckets * 8, cudaMemcpyDeviceToHost, stream_));
    PP_CUDA(cudaStreamSynchronize(stream_));
  }
  void set_spec_reduce(std::function<void(std::vector<unsigned long long>&)> f) override { spec_reduce_ = std::move(f); }
  void set_global_max(double g) override { gmax_ = g; }

  void shard_ingest(const uint64_t* rec, uint64_t count, bool device) override {
    sync_state();
    if (count == 0) return;
    const int rw = 2 * W + 1;
    if (bump_ + count > arena_[cur_].cap) gc_into_other(std::max<uint64_t>(next_arena_target(), live_ + 2 * count));
    evict_buf_.ensure(count * rw * 8);
    PP_CUDA(copy_async(evict_buf_.p, rec, count * rw * 8,
                            device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, stream_));
    rec_slot_.ensure(count * 4);
    uint32_t* flags = rec_slot_.as<uint32_t>();
    k_run_starts<<<(uint32_t)((count + kCta - 1) / kCta), kCta, 0, stream_>>>(evict_buf_.as<uint64_t>(), count, W, W,
                                                                                flags);
    const uint64_t ntiles = (count + kScanTile - 1) / kScanTile;
    scan_tmp_.ensure((ntiles + 1) * 8);
    scan_gid_.ensure(count * 8);
    device_scan(flags, count, 1, scan_gid_.as<unsigned long long>(), ntiles);
    unsigned long long nruns = 0;
    PP_CUDA(copy_async(&nruns, scan_tmp_.as<unsigned long long>() + ntiles, 8, cudaMemcpyDeviceToHost, stream_));
    PP_CUDA(cudaStreamSynchronize(stream_));
    grow_groups_preserving(G_ + (uint32_t)nruns);
    k_ingest_append<W><<<(uint32_t)((count + kCta - 1) / kCta), kCta, 0, stream_>>>(
        evict_buf_.as<uint64_t>(), count, scan_gid_.as<unsigned long long>(), gview(gcur_), G_, aview(cur_), bump_);
    k_ingest_counts<W><<<blocks(nruns), kCta, 0, stream_>>>(gview(gcur_), G_, (uint32_t)nruns, bump_ + count);
    launches_ += 3;
    G_ += (uint32_t)nruns;
    bump_ += count;
    live_ += count;
    bump_bound_ = bump_;
    live_bound_ = live_;
    reset_stats(bump_);
    IdentityProducer<W> p;
    regroup(p);  // merge groups sharing a z, sort by x, combine equal keys
    dirty_ = true;
  }

  void grow_groups_preserving(uint32_t cap) {
    if (groups_[gcur_].cap >= cap) return;
    const int o = 1 - gcur_;
    ensure_groups(o, std::max<uint32_t>(cap, 2 * groups_[gcur_].cap));
    GroupView<W> a = gview(gcur_), b = gview(o);
    for (int k = 0; k < W; ++k) PP_CUDA(copy_async(b.z[k], a.z[k], G_ * 8ull, cudaMemcpyDeviceToDevice, stream_));
    PP_CUDA(copy_async(b.off, a.off, G_ * 8ull, cudaMemcpyDeviceToDevice, stream_));
    PP_CUDA(copy_async(b.gmax, a.gmax, G_ * 8ull, cudaMemcpyDeviceToDevice, stream_));
    PP_CUDA(copy_async(b.gmin, a.gmin, G_ * 8ull, cudaMemcpyDeviceToDevice, stream_));
    PP_CUDA(copy_async(b.cnt, a.cnt, G_ * 4ull, cudaMemcpyDeviceToDevice, stream_));
    PP_CUDA(copy_async(b.cap, a.cap, G_ * 4ull, cudaMemcpyDeviceToDevice, stream_));
    PP_CUDA(copy_async(b.flags, a.flags, G_ * 4ull, cudaMemcpyDeviceToDevice, stream_));
    PP_CUDA(copy_async(b.stamp, a.stamp, G_ * 4ull, cudaMemcpyDeviceToDevice, stream_));
    gcur_ = o;
  }

  pp_counters take_counters() override {
    sync_state();
    close_window();
    pp_counters out = counters_;
    counters_ = pp_counters{};
    return out;
  }

  void take_kernel_stats(double* ms, double* bytes, uint64_t* launches, uint64_t* total) override {
    sync_state();
    *ms = branch_ms_;
    *bytes = branch_bytes_;
    last_stream_frac_ = branch_in_ ? (double)branch_stream_ / (double)branch_in_ : 0.0;
    if (std::getenv("PP_DEBUG"))
      std::fprintf(stderr, "[pp] dense sublayer: %llu groups, %llu strings written, %llu big-block tiles by bulk copies\n",
                   (unsigned long long)dense_groups_, (unsigned long long)dense_out_,
                   (unsigned long long)bulk_tiles_);
    if (std::getenv("PP_DEBUG")) std::fprintf(stderr, "[pp] branch strings %llu, via long-block stream path %.3f\n",
                                              (unsigned long long)branch_in_, last_stream_frac_);
    branch_in_ = branch_stream_ = 0;
    *launches = branch_launches_;
    *total = launches_;
    branch_ms_ = branch_bytes_ = 0.0;
    branch_launches_ = launches_ = 0;
  }

 private:
  static constexpr size_t R = 8 * W + 8;  // bytes per string in the arena

  static size_t big_sort_smem() { return std::max(sizeof(SortSmem<W>), sizeof(MergeSmem<W>)); }
  static uint32_t blocks(uint64_t n) { return (uint32_t)((n + kCta - 1) / kCta); }

  bool fusion_allowed() const {
    if (cfg_.flags & PP_FLAG_NO_CLIFFORD_FUSION) return false;
    // per-layer cadence keeps each gate's zeroed parents until the layer's
    // truncation, and a later gate may revive one: gate by gate is exact
    if (keep_zeros_) return false;
    // a fused run never exceeds |O|, but the reference's transient count
    // inside a Clifford gate can reach 2|O| before truncation
    return cfg_.max_terms == 0 || 2 * live_ <= cfg_.max_terms;
  }

  // ----- buffers
  struct Arena {
    DevBuf buf;
    uint64_t cap = 0;     // strings of bump space
    uint64_t stride = 0;  // plane stride (cap + scratch tail)
  };
  struct Groups {
    DevBuf buf;
    uint32_t cap = 0;
  };
  ArenaView<W> aview(int i) const {
    ArenaView<W> v;
    uint64_t* b = arena_[i].buf.template as<uint64_t>();
    for (int k = 0; k < W; ++k) v.x[k] = b + k * arena_[i].stride;
    v.c = reinterpret_cast<double*>(b + W * arena_[i].stride);
    return v;
  }
  GroupView<W> gview(int i) const {
    GroupView<W> v;
    const uint64_t C = groups_[i].cap;
    char* b = groups_[i].buf.template as<char>();
    for (int k = 0; k < W; ++k) v.z[k] = reinterpret_cast<uint64_t*>(b) + k * C;
    char* p = b + W * C * 8;
    v.off = reinterpret_cast<uint64_t*>(p);
    p += C * 8;
    v.gmax = reinterpret_cast<double*>(p);
    p += C * 8;
    v.gmin = reinterpret_cast<double*>(p);
    p += C * 8;
    v.cnt = reinterpret_cast<uint32_t*>(p);
    p += C * 4;
    v.cap = reinterpret_cast<uint32_t*>(p);
    p += C * 4;
    v.flags = reinterpret_cast<uint32_t*>(p);
    p += C * 4;
    v.stamp = reinterpret_cast<uint32_t*>(p);
    return v;
  }
  // cap strings of bump space, plus (speculative eps0 > 0 runs) the per-CTA
  // scratch tail of k_branch_sublayer (kSpecScratch)
  void ensure_arena(int i, uint64_t cap) {
    cap = (cap + 1) & ~1ull;  // even plane strides: every plane starts 16-byte aligned (128-bit stores)
    if (arena_[i].cap >= cap) return;
    arena_[i].buf.release();
    arena_[i].cap = arena_[i].stride = 0;
    const uint64_t tail = spec_capable() ? 2ull * kSpecScratch * sub_grid_ : 0;
    arena_[i].buf.ensure((cap + tail) * R);
    arena_[i].cap = cap;
    arena_[i].stride = cap + tail;
  }
  bool spec_capable() const {  // (external engines too: a sharded driver runs them coordinated)
    return cfg_.epsilon0 > 0.0 && cfg_.cadence == PP_CADENCE_GATE && cfg_.max_terms == 0;
  }
  void ensure_groups(int i, uint32_t cap) {
    if (groups_[i].cap >= cap) return;
    groups_[i].buf.release();
    groups_[i].cap = 0;
    groups_[i].buf.ensure((size_t)cap * (8 * W + 8 + 8 + 8 + 4 + 4 + 4 + 4));
    groups_[i].cap = cap;
  }

  void reset_stats(unsigned long long bump) {
    k_reset_stats<<<1, 1, 0, stream_>>>(d_stats_, bump);
    ++launches_;
  }
  // The engine's round trips: spin on an event (lower wake-up latency than a
  // blocking stream sync; the waits are short and frequent)
  void wait_stream() {
    PP_CUDA(cudaEventRecord(ev_sync_, stream_));
    cudaError_t e;
    while ((e = cudaEventQuery(ev_sync_)) == cudaErrorNotReady) {
    }
    PP_CUDA(e);
  }
  void fetch_stats() {
    auto t0 = Clock::now();
    PP_CUDA(copy_async(h_stats_, d_stats_, sizeof(DevStats), cudaMemcpyDeviceToHost, stream_));
    if (spin_sync_) wait_stream();
    else PP_CUDA(cudaStreamSynchronize(stream_));
    held_graphs_.clear();  // every launch so far has completed
    tr_sync_ns_ += ns_since(t0);
    ++tr_syncs_;
  }

  // ----- garbage collection: compact the current arena into the other one
  void mem_report(const char* what, uint64_t arg) {
    if (!std::getenv("PP_DEBUG")) return;
    size_t fb = 0, tb = 0;
    cudaMemGetInfo(&fb, &tb);
    std::fprintf(stderr, "[pp] %s %llu: live %llu bump %llu G %u arenas %llu/%llu (max %llu) free %zu MiB\n", what,
                 (unsigned long long)arg, (unsigned long long)live_, (unsigned long long)bump_, G_,
                 (unsigned long long)arena_[cur_].cap, (unsigned long long)arena_[1 - cur_].cap,
                 (unsigned long long)arena_max_, fb >> 20);
  }
  void gc_into_other(uint64_t new_cap) {
    sync_state();
    mem_report("gc ->", new_cap);
    const int o = 1 - cur_;
    ensure_arena(o, new_cap);
    uint64_t total = 0;
    if (G_) {
      const uint64_t ntiles = (G_ + kScanTile - 1) / kScanTile;
      scan_tmp_.ensure((ntiles + 1) * 8);
      scan_off_.ensure((size_t)G_ * 8);
      unsigned long long* noff = scan_off_.as<unsigned long long>();
      device_scan(gview(gcur_).cnt, G_, 0, noff, ntiles);
      total = live_;  // sync_state above: live_ = sum of the group counts
      if (total) {
        const uint64_t tiles = (total + kGcTile - 1) / kGcTile;
        const uint32_t grid = (uint32_t)std::min<uint64_t>(tiles, 148ull * 8ull);
        k_gc_copy<W><<<grid, kCta, 0, stream_>>>(gview(gcur_), G_, noff, total, aview(cur_), aview(o));
        ++launches_;
      }
      k_gc_finish<W><<<std::min<uint32_t>(blocks(G_), 148u * 8u), kCta, 0, stream_>>>(gview(gcur_), G_, noff);
      ++launches_;
    }
    reset_stats(total);
    PP_CUDA(cudaGetLastError());
    bump_ = bump_bound_ = total;
    cur_ = o;
  }
  void compact() {
    sync_state();
    uint64_t cap = std::max<uint64_t>(arena_[cur_].cap, live_ + 1);
    gc_into_other(cap);
  }
  // ----- per-gate epilogue and host synchronisation
  // Budget check, NaN check and truncation run on the device (k_truncate),
  // so consecutive gates need no host round trip; the host synchronises only
  // when it needs exact sizes (sync_state).
  bool external() const { return (cfg_.flags & PP_FLAG_EXTERNAL_TRUNCATION) != 0; }
  void epilogue(bool do_truncate, bool check_budget) {
    if (sub_pending_) sync_state();  // a sublayer must be complete before the epilogue reads the store
    if (external()) {  // the orchestrator truncates with a global threshold
      dirty_ = true;
      return;
    }
    const bool budget = check_budget && cfg_.max_terms;
    // With epsilon0 == 0 the threshold is 0: only exact zeros go, and the
    // branch/regroup kernels never emit zeros (cadence gate), so unless the
    // store may hold zeros (set_initial) or a budget must be checked the
    // epilogue is a no-op; NaN/Inf is then caught at the next sync.
    if (cfg_.epsilon0 == 0.0 && !budget && !may_hold_zeros_) {
      if (do_truncate) gmax_stale_ = true;
      dirty_ = true;
      return;
    }
    push_scalars(bseq_);
    if (G_) {
      err_base_ = gates_applied_ ? gates_applied_ - 1 : 0;  // the gate(s) just applied are counted already
      launch_epilogue(0, do_truncate, budget);
      if (do_truncate) may_hold_zeros_ = false;
    }
    if (do_truncate) truncated_since_sync_ = true;
    dirty_ = true;
  }
  void post_gate() {
    ++gates_applied_;
    ++counters_.gates;
    epilogue(cfg_.cadence == PP_CADENCE_GATE, true);
  }
  // the diagonal pass of the readout, folded into a sync's single round trip
  // red != nullptr: the group reduction of sync_state in the same launch
  void launch_diag(RedSlot* red = nullptr) {
    PP_CUDA(cudaMemsetAsync(&d_stats_->diag_count, 0, sizeof(unsigned long long), stream_));
    diag_copied_ = 0;
    if (!G_) return;
    diag_z_.ensure((size_t)G_ * W * 8);
    diag_c_.ensure((size_t)G_ * 8);
    if (red)
      k_readout<W><<<blocks(32ull * G_), kCta, 0, stream_>>>(gview(gcur_), g_pending_ ? kKeepG : G_, aview(cur_),
                                                              diag_z_.as<uint64_t>(), diag_c_.as<double>(), d_stats_,
                                                              red);
    else
      k_diag<W><<<blocks(32ull * G_), kCta, 0, stream_>>>(gview(gcur_), g_pending_ ? kKeepG : G_, aview(cur_),
                                                           diag_z_.as<uint64_t>(), diag_c_.as<double>(), d_stats_);
    ++launches_;
    if (!h_diag_) h_diag_ = pinned_diag();
    // diagonal strings are few (at most one per group): fetch a short prefix
    // with the readout's round trip, the rest only if there are more
    diag_copied_ = std::min<uint64_t>(G_, kDiagSpec);
    PP_CUDA(copy_async(h_diag_->z, diag_z_.p, diag_copied_ * W * 8, cudaMemcpyDeviceToHost, stream_));
    PP_CUDA(copy_async(h_diag_->c, diag_c_.p, diag_copied_ * 8, cudaMemcpyDeviceToHost, stream_));
  }

  void sync_state(bool diag = false) {
    if (!dirty_) {
      if (!diag) return;
      launch_diag();  // clean store: the diagonal pass alone
      fetch_stats();
      PP_CUDA(cudaGetLastError());
      diag_n_ = h_stats_->diag_count;
      return;
    }
    if (lazy_open_) {  // apply the deferred truncations of the last launch window
      if (G_) {
        k_flush<W><<<persistent_grid(), kCta, 0, stream_>>>(gview(gcur_), aview(cur_), thr_.as<double>(),
                                                          (uint32_t)lazy_base_, lazy_len_, d_stats_);
        ++launches_;
      }
      lazy_open_ = false;
    }
    if (diag) {
      // group reduction and diagonal search in one launch; k_readout takes the
      // group count as a parameter (or st->G_dev, committed on the device), and
      // red[2] is clean (cleared after every sync and by every reset)
      launch_diag(&d_stats_->red[2]);
    } else {
      push_scalars(bseq_);
      if (G_)
        k_reduce<W><<<std::min<uint32_t>(reduce_grid(), blocks(G_)), kCta, 0, stream_>>>(gview(gcur_), d_stats_,
                                                                                         &d_stats_->red[2]);
      launches_ += G_ ? 1 : 0;
    }
    fetch_stats();
    PP_CUDA(cudaGetLastError());
    const DevStats& st = *h_stats_;
    if (g_pending_) {
      if (st.overflow || st.collision)
        throw EngineError(PP_ERR_INTERNAL, "regroup: slot table overflow or fingerprint collision (deferred check)");
      G_ = st.G_dev;
      g_pending_ = false;
    }
    if (st.cliff_records) {  // Clifford records of a deferred regroup (apply_clifford_run's accounting)
      counters_.records_sent += st.cliff_records;
      counters_.removed += st.cliff_records;
    }
    harvest_seen(st);
    diag_n_ = st.diag_count;
    counters_.records_sent += st.records;
    counters_.removed += st.removed;
    if (st.err_budget) {
      dirty_ = false;
      throw EngineError(PP_ERR_RESOURCE, "term budget exhausted: |O|=" + std::to_string(st.err_live) +
                                             " exceeds max_terms=" + std::to_string(cfg_.max_terms) + " at gate " +
                                             std::to_string(err_base_ + st.err_gate + 1));
    }
    if (st.err_numerical) {
      dirty_ = false;
      throw EngineError(PP_ERR_NUMERICAL, "non-finite coefficient at gate " + std::to_string(err_base_ + st.err_gate + 1) +
                                              ", |O|=" + std::to_string(st.err_live));
    }
    arena_fault_ = st.err_arena != 0;
    unsorted_fault_ = st.err_unsorted != 0;
    arena_fault_seq_ = st.err_seq;
    if (st.red[2].nonfinite && gmax_stale_ && !external()) {
      dirty_ = false;
      throw EngineError(PP_ERR_NUMERICAL, "non-finite coefficient detected at gate " + std::to_string(gates_applied_) +
                                              ", |O|=" + std::to_string(st.red[2].live));
    }
    live_ = live_bound_ = st.red[2].live;
    bump_ = bump_bound_ = st.bump;
    maxcnt_ = G_ ? st.red[2].maxcnt : 0u;
    if (truncated_since_sync_) gmax_ = __builtin_bit_cast(double, st.last_gmax_bits);
    // epsilon0 == 0 fast path: the skipped truncations would have used the
    // max after the last gate, which survives its own truncation
    if (gmax_stale_) gmax_ = __builtin_bit_cast(double, st.red[2].gmax_bits);
    truncated_since_sync_ = false;
    gmax_stale_ = false;
    // harvest branch-kernel timings
    for (auto& pr : pending_events_) {
      float ms = 0.f;
      PP_CUDA(cudaEventElapsedTime(&ms, pr.first, pr.second));
      branch_ms_ += ms;
      free_events_.push_back(pr);
    }
    pending_events_.clear();
    branch_bytes_ += (double)(st.aff_total + st.out_elems) * R;
    branch_in_ += st.aff_total;
    branch_stream_ += st.stream_elems;
    dense_groups_ += st.dense_groups;
    dense_out_ += st.dense_out;
    bulk_tiles_ += st.bulk_tiles;
    k_clear_cumulative<<<1, 1, 0, stream_>>>(d_stats_);
    ++launches_;
    dirty_ = false;
    if (sub_pending_) {
      if (arena_fault_ || unsorted_fault_) resume_sublayer(diag);
      sub_pending_ = false;
    }
  }
  uint32_t persistent_grid() const { return 148u * 8u; }

  void push_scalars(uint64_t seq_base) {
    // window index of gate seq_base: the current run starts at bseq_
    const uint32_t seen_base = window_index() + (uint32_t)(seq_base - bseq_);
    k_set_scalars<<<1, 1, 0, stream_>>>(d_stats_, g_pending_ ? kKeepG : G_, arena_[cur_].cap, seq_base, seen_base);
    ++launches_;
  }
  // per-gate epilogue kernels for gate `rel` of a launch run (red slots by parity)
  void launch_epilogue(uint32_t rel, bool do_truncate, bool budget, bool lazy = false) {
    RedSlot* r = &d_stats_->red[rel & 1];
    RedSlot* rn = &d_stats_->red[(rel + 1) & 1];
    if (lazy) {  // deferred truncation: the branch kernel reduced into r; exact threshold now
      k_thresh<W><<<1, kCta, 0, stream_>>>(cfg_.epsilon0, rel, r, rn, thr_.as<double>(), d_stats_);
      ++launches_;
      return;
    }
    k_reduce<W><<<reduce_grid(), kCta, 0, stream_>>>(gview(gcur_), d_stats_, r);
    k_truncate<W><<<persistent_grid(), kCta, 0, stream_>>>(gview(gcur_), aview(cur_), cfg_.epsilon0,
                                                           do_truncate ? 1 : 0, budget ? cfg_.max_terms : 0, rel, r,
                                                           rn, d_stats_);
    launches_ += 2;
  }
  uint32_t reduce_grid() const { return 148u * 4u; }  // fixed: graphs capture it

  // ----- Z-type generator (x_J = 0): pairs of z-groups (pp_zz.cuh).  Returns
  // false when a pair could exceed one segment; the caller then regroups.
  bool apply_zz(const pp_gate& gate, const uint64_t* jzw) {
    auto t0 = Clock::now();
    ensure_sorted();
    sync_state();
    if (2ull * maxcnt_ > kZSeg) return false;
    const bool budget = cfg_.max_terms != 0 && !external();
    const bool do_trunc = cfg_.cadence == PP_CADENCE_GATE;
    const bool epi = !external() && !(cfg_.epsilon0 == 0.0 && !budget && !may_hold_zeros_);
    const bool lazy = epi && do_trunc && !budget && cfg_.epsilon0 > 0.0 && !keep_zeros_ &&
                      std::getenv("PP_EAGER_TRUNCATION") == nullptr;
    Plane<W> jz;
    for (int k = 0; k < W; ++k) jz.w[k] = jzw[k];
    if (lazy) thr_.ensure(kLazyWindow * sizeof(double));
    for (int attempt = 0; G_ > 0; ++attempt) {
      if (attempt > 64) throw EngineError(PP_ERR_RESOURCE, "arena cannot hold the Z-type gate");
      grow_groups_preserving(2 * G_ + 1024);  // room for a partner per group
      if (bump_ + 2 * live_ > arena_[cur_].cap) gc_into_other(next_arena_target());
      uint64_t tc = 1024;
      while (tc < 2ull * G_) tc <<= 1;
      ztab_.ensure(tc * (8 + 8 * W + 4));
      ZTable<W> t;
      char* tb = ztab_.as<char>();
      t.fp = reinterpret_cast<unsigned long long*>(tb);
      for (int k = 0; k < W; ++k) t.z[k] = reinterpret_cast<uint64_t*>(tb + tc * 8 * (1 + k));
      t.gid = reinterpret_cast<uint32_t*>(tb + tc * 8 * (1 + W));
      t.mask = tc - 1;
      push_scalars(bseq_);
      PP_CUDA(cudaMemsetAsync(&d_stats_->zz_newg, 0, 4 * sizeof(unsigned int), stream_));
      PP_CUDA(cudaMemsetAsync(t.fp, 0, tc * 8, stream_));
      if (lazy) {
        PP_CUDA(cudaMemsetAsync(thr_.p, 0, 2 * sizeof(double), stream_));
        lazy_open_ = true;
        lazy_base_ = bseq_;
        lazy_len_ = 1;
      }
      k_ztab_build<W><<<blocks(G_), kCta, 0, stream_>>>(gview(gcur_), G_, t);
      k_branch_zz<W><<<zz_grid_, kCta, sizeof(ZzSmem<W>), stream_>>>(
          gview(gcur_), G_, aview(cur_), jz, gate.cos_theta, gate.sin_theta, keep_zeros_, t, &d_stats_->work[0],
          &d_stats_->work[1], 0, d_stats_, lazy ? thr_.as<double>() : nullptr, lazy ? &d_stats_->red[0] : nullptr);
      launches_ += 2;
      ++branch_launches_;
      err_base_ = gates_applied_;  // (this gate is counted after its launches)
      if (epi) launch_epilogue(0, do_trunc, budget, lazy);
      dirty_ = true;
      fetch_stats();  // the gate's one round trip: new groups, arena fault
      PP_CUDA(cudaGetLastError());
      if (h_stats_->zz_err) throw EngineError(PP_ERR_INTERNAL, "Z-type gate: pair larger than a segment");
      G_ += h_stats_->zz_newg;
      maxcnt_ = std::max<uint32_t>(maxcnt_, h_stats_->zz_maxcnt);
      if (!h_stats_->err_arena) break;
      k_clear_arena_error<<<1, 1, 0, stream_>>>(d_stats_);  // done pairs carry this gate's stamp
      ++launches_;
      lazy_open_ = false;  // the faulted launch set no threshold
      gc_into_other(next_arena_target());
    }
    if (epi && do_trunc) truncated_since_sync_ = true;
    if (!epi && do_trunc && !external()) gmax_stale_ = true;
    if (keep_zeros_) may_hold_zeros_ = true;
    dirty_ = true;
    bseq_ += 1;
    ++gates_applied_;
    ++counters_.gates;
    counters_.branch_ns += ns_since(t0);
    return true;
  }

  // ----- one gate
  void apply_one(const pp_gate& gate) {
    uint64_t jx[2], jz[2];
    words_to_planes(gate.words, jx, jz);
    if (W == 1 && (jx[1] | jz[1])) throw EngineError(PP_ERR_INVALID, "generator has sites beyond the engine width");
    auto t0 = Clock::now();
    int nx = __builtin_popcountll(jx[0]) + (W == 2 ? __builtin_popcountll(jx[1]) : 0);
    bool zfree = (jz[0] | (W == 2 ? jz[1] : 0)) == 0;
    if (nx == 0 && zfree) {
      // identity generator: commutes with everything, no records
    } else if (zfree && nx == 1) {
      run_rx(&gate, 1);
      return;
    } else if (nx == 0 && std::getenv("PP_ZZ_REGROUP") == nullptr && apply_zz(gate, jz)) {
      return;
    } else {
      GateProducer<W> p;
      for (int k = 0; k < W; ++k) {
        p.jx.w[k] = jx[k];
        p.jz.w[k] = jz[k];
      }
      p.cosv = gate.cos_theta;
      p.sinv = gate.sin_theta;
      p.seen_base = window_index();
      regroup(p);
      counters_.records_sent += h_records_;
    }
    counters_.branch_ns += ns_since(t0);
    h_records_ = 0;
    post_gate();
  }

  std::pair<cudaEvent_t, cudaEvent_t> take_event_pair() {
    if (!free_events_.empty()) {
      auto e = free_events_.back();
      free_events_.pop_back();
      return e;
    }
    {
      std::lock_guard<std::mutex> lk(g_streams_mu);
      if (!g_event_pairs.empty()) {
        auto e = g_event_pairs.back();
        g_event_pairs.pop_back();
        return e;
      }
    }
    std::pair<cudaEvent_t, cudaEvent_t> e;
    PP_CUDA(cudaEventCreate(&e.first));
    PP_CUDA(cudaEventCreate(&e.second));
    return e;
  }

  void ensure_list(uint32_t n) { list_.ensure((size_t)std::max<uint32_t>(n, 1) * 4); }

  // A run of Clifford Z_i Z_j gates (i != j, no X/Y): split into matchings,
  // then into equal-offset groups, and regroup with ZZRunProducer.
  bool try_zz_run(const pp_gate* gates, size_t count, bool sort) {
    // a previous fused ZZ run's edge masks are decoded with zz_edges_: harvest
    // them before zz_edges_ can change
    if (zz_seen_pending_) sync_state();
    if (zz_key_.size() == count && std::memcmp(zz_key_.data(), gates, count * sizeof(pp_gate)) == 0) {
      if (!zz_ok_) return false;
      note_zz_run();
      regroup(zz_prod_, sort);  // the same run as last time (run_circuit layers)
      return true;
    }
    zz_key_.clear();
    std::vector<std::pair<int, int>> edges(count);
    std::vector<int> neg(count);
    for (size_t g = 0; g < count; ++g) {
      uint64_t jx[2], jz[2];
      words_to_planes(gates[g].words, jx, jz);
      if (W == 1 && (jx[1] | jz[1])) throw EngineError(PP_ERR_INVALID, "generator has sites beyond the engine width");
      if (jx[0] | jx[1]) return false;
      int sites[3], ns = 0;
      for (int w = 0; w < 2; ++w)
        for (uint64_t v = jz[w]; v && ns < 3; v &= v - 1) sites[ns++] = 64 * w + __builtin_ctzll(v);
      if (ns != 2) return false;
      edges[g] = {sites[0], sites[1]};
      neg[g] = gates[g].sin_theta < 0;
    }
    // greedy matchings in run order
    std::vector<std::vector<size_t>> matchings;
    std::vector<std::vector<uint8_t>> used;
    for (size_t g = 0; g < count; ++g) {
      size_t k = 0;
      for (; k < matchings.size(); ++k)
        if (!used[k][edges[g].first] && !used[k][edges[g].second]) break;
      if (k == matchings.size()) {
        matchings.emplace_back();
        used.emplace_back(128, 0);
      }
      matchings[k].push_back(g);
      used[k][edges[g].first] = used[k][edges[g].second] = 1;
    }
    ZZRunProducer<W> p;
    p.ng = 0;
    std::vector<ZZEdge> zz_edges;
    using T = typename PlaneInt<W>::T;
    for (auto& mt : matchings) {
      std::map<int, std::pair<T, T>> by_d;
      std::map<int, std::vector<std::pair<int, int>>> edge_gates;  // d -> (bit i, run gate)
      for (size_t g : mt) {
        int i = edges[g].first, d = edges[g].second - edges[g].first;  // first < second (ascending scan)
        auto& e = by_d[d];
        e.first |= (T)1 << i;
        if (neg[g]) e.second |= (T)1 << i;
        edge_gates[d].push_back({i, (int)g});
      }
      for (auto& [d, mm] : by_d) {
        if (p.ng >= kMaxZZGroups) {
          zz_key_.assign(gates, gates + count);
          zz_ok_ = false;
          return false;
        }
        p.grp[p.ng].m = mm.first;
        p.grp[p.ng].neg = mm.second;
        p.grp[p.ng].d = d;
        for (auto [i, g] : edge_gates[d]) zz_edges.push_back({p.ng, i, g});
        ++p.ng;
      }
    }
    zz_key_.assign(gates, gates + count);
    zz_prod_ = p;
    zz_edges_ = zz_edges;
    zz_ok_ = true;
    note_zz_run();
    regroup(p, sort);
    return true;
  }

  // ----- fused Clifford run
  void apply_clifford_run(const pp_gate* gates, size_t count, bool sort = true) {
    auto t0 = Clock::now();
    if (G_ && try_zz_run(gates, count, sort)) {
      // handled by the bit-parallel ZZ producer
    } else if (G_) {
      std::vector<uint64_t> gx(count * W), gz(count * W);
      std::vector<double> gs(count);
      for (size_t i = 0; i < count; ++i) {
        uint64_t jx[2], jz[2];
        words_to_planes(gates[i].words, jx, jz);
        if (W == 1 && (jx[1] | jz[1])) throw EngineError(PP_ERR_INVALID, "generator has sites beyond the engine width");
        for (int k = 0; k < W; ++k) {
          gx[i * W + k] = jx[k];
          gz[i * W + k] = jz[k];
        }
        gs[i] = gates[i].sin_theta;
      }
      cliff_.ensure(count * (2 * W + 1) * 8);
      uint64_t* dgx = cliff_.as<uint64_t>();
      uint64_t* dgz = dgx + count * W;
      double* dgs = reinterpret_cast<double*>(dgz + count * W);
      PP_CUDA(copy_async(dgx, gx.data(), count * W * 8, cudaMemcpyHostToDevice, stream_));
      PP_CUDA(copy_async(dgz, gz.data(), count * W * 8, cudaMemcpyHostToDevice, stream_));
      PP_CUDA(copy_async(dgs, gs.data(), count * 8, cudaMemcpyHostToDevice, stream_));
      CliffordProducer<W> p{dgx, dgz, dgs, (int)count, window_index()};
      regroup(p, sort);
    }
    // Clifford gates zero each moved parent and re-insert it at I xor J;
    // absent a partner pair the reference removes one zero per record.
    counters_.records_sent += h_records_;
    counters_.removed += h_records_;
    h_records_ = 0;
    counters_.exchange_ns += ns_since(t0);
    gates_applied_ += count;
    counters_.gates += count;
    auto t1 = Clock::now();
    // A Clifford run is a signed permutation of the strings: |c| values,
    // hence the global max, are unchanged and no zero or NaN appears, so at
    // epsilon0 = 0 (threshold 0, no zeros held) the truncation is a no-op and
    // the regroup left the store exactly known (no sync needed).
    if (!(cfg_.epsilon0 == 0.0 && !may_hold_zeros_ && !external())) epilogue(cfg_.cadence == PP_CADENCE_GATE, false);
    counters_.truncate_ns += ns_since(t1);
  }

  // ----- regroup: records -> new z-grouped store
  template <class P>
  void regroup(const P& prod, bool sort = true) {
    const int maxrec = P::kMaxRec;
    count_param_h2d(sizeof(P));  // the producer's gate descriptors
    sync_state();
    const uint64_t live = live_;
    if (G_ == 0 || live == 0) return;
    mem_report("regroup maxrec", maxrec);
    if (!sort && defer_ok_ && P::kMaxRec == 1 && live <= kSmallRegroupMax) {
      // a small store feeding a dense Rx run: the whole regroup in one CTA,
      // sizes committed on the device (no round trip, as below)
      const uint32_t tc = small_regroup_tc((uint32_t)live);
      const size_t smem = small_regroup_smem<W>(tc, (uint32_t)live);
      static bool attr_set = false;  // per producer type
      if (!attr_set) {
        PP_CUDA(cudaFuncSetAttribute(k_regroup_small<W, P>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)small_regroup_smem<W>(small_regroup_tc(kSmallRegroupMax), kSmallRegroupMax)));
        attr_set = true;
      }
      const int o = 1 - cur_;
      ensure_groups(1 - gcur_, std::max<uint32_t>((uint32_t)live, 1024));
      ensure_arena(o, std::max<uint64_t>(regroup_arena(live), std::min<uint64_t>(arena_[cur_].cap, arena_max_)));
      // (the kernel resets the statistics itself: no k_reset_stats launch)
      k_regroup_small<W, P><<<1, kSmallRegroupThreads, smem, stream_>>>(gview(gcur_), G_, aview(cur_), prod,
                                                                       gview(1 - gcur_), aview(o), (uint32_t)live,
                                                                       tc, d_stats_, bump_);
      ++launches_;
      PP_CUDA(cudaGetLastError());
      cur_ = o;
      gcur_ = 1 - gcur_;
      G_ = (uint32_t)live;  // upper bound until the sync
      g_pending_ = true;
      unsorted_ = true;
      bump_ = bump_bound_ = live;
      live_ = live_bound_ = live;
      h_records_ = 0;
      dirty_ = true;
      return;
    }
    const uint64_t max_items = (uint64_t)G_ + live / kItem + 1;
    items_.ensure(max_items * sizeof(Item));
    rec_slot_.ensure(live * maxrec * 4);
    const uint64_t records_upper = live * maxrec;
    // small stores: size every buffer by its upper bound so nothing can
    // overflow, let the kernels read counts from the device, and synchronise
    // once at the end
    bool small = records_upper <= (1ull << 22);
    uint64_t tc = 1024;
    if (small) {
      while (tc < 2 * records_upper + 1024) tc <<= 1;
    } else {
      // distinct output z-groups: learned from the previous regroup; an
      // overflow retries with a 4x larger table
      const double est = std::max(2.0, 1.5 * zfactor_) * (double)G_;
      while ((double)tc < 2.0 * std::min<double>((double)records_upper, est) + 1024) tc <<= 1;
      if (std::getenv("PP_TINY_TABLE")) tc = 1024;  // test hook: overflow and the 4x retries
    }
    uint64_t tc_max = 1024;
    while (tc_max < 2 * records_upper + 1024) tc_max <<= 1;
    const int o = 1 - cur_;
    for (int attempt = 0;; ++attempt) {
      if (attempt > 8) throw EngineError(PP_ERR_INTERNAL, "regroup: hash table retries exhausted");
      table_.ensure(tc * (8 + 8 * W + 4 + 4));
      HashTable<W> t = tview(tc);
      PP_CUDA(cudaMemsetAsync(t.fp, 0, tc * 8, stream_));
      PP_CUDA(cudaMemsetAsync(t.count, 0, tc * 4, stream_));
      reset_stats(bump_);
      k_make_items<W><<<blocks(G_), kCta, 0, stream_>>>(gview(gcur_), G_, items_.as<Item>(), maxrec, d_stats_);
      ++launches_;
      uint64_t n_items = max_items;
      if (!small) {
        fetch_stats();
        n_items = h_stats_->items;
      }
      k_insert<W, P><<<(uint32_t)n_items, kCta, 0, stream_>>>(items_.as<Item>(), gview(gcur_), aview(cur_), prod, t,
                                                              rec_slot_.as<uint32_t>(), seed_,
                                                              (uint32_t)std::min<uint64_t>(tc / 2, 0xffffffffu),
                                                              d_stats_);
      ++launches_;
      uint32_t distinct = 0;
      if (!small) {
        fetch_stats();
        PP_CUDA(cudaGetLastError());
        if (h_stats_->overflow) {
          if (tc >= tc_max) throw EngineError(PP_ERR_INTERNAL, "regroup: hash table overflow");
          tc = std::min(tc_max, tc * 4);
          continue;
        }
        distinct = h_stats_->distinct;
      }
      // deterministic ids and offsets from slot order
      const uint64_t ntiles = (tc + kScanTile - 1) / kScanTile;
      scan_tmp_.ensure((ntiles + 1) * 8);
      scan_gid_.ensure(tc * 8);
      scan_off_.ensure(tc * 8);
      if (tc <= kScanPairMax) {
        k_scan_pair_small<<<1, kScanPairThreads, 0, stream_>>>(t.count, (uint32_t)tc, scan_gid_.as<unsigned long long>(),
                                                   scan_off_.as<unsigned long long>(), d_stats_);
        ++launches_;
      } else {
        device_scan(t.count, tc, 1, scan_gid_.as<unsigned long long>(), ntiles);
        device_scan(t.count, tc, 0, scan_off_.as<unsigned long long>(), ntiles);
        PP_CUDA(copy_async(&d_stats_->scan_total, scan_tmp_.as<unsigned long long>() + ntiles, 8,
                                cudaMemcpyDeviceToDevice, stream_));
      }
      uint64_t total_bound = records_upper;
      uint32_t groups_bound = (uint32_t)std::min<uint64_t>(records_upper, 0xffffffffu);
      if (!small) {
        fetch_stats();
        total_bound = h_stats_->scan_total;
        groups_bound = distinct;
      }
      ensure_groups(1 - gcur_, std::max<uint32_t>(groups_bound, 1024));
      // the two arenas alternate between regroups: keep the target as large
      // as the current one (the Rx run after a regroup grows into it; a
      // smaller target would overflow there and compact)
      ensure_arena(o, std::max<uint64_t>(regroup_arena(total_bound), std::min<uint64_t>(arena_[cur_].cap, arena_max_)));
      k_table_emit<W><<<(uint32_t)((tc + kCta - 1) / kCta), kCta, 0, stream_>>>(
          t, scan_gid_.as<unsigned long long>(), scan_off_.as<unsigned long long>(), gview(1 - gcur_), 0,
          P::kMaxRec == 1 ? 1 : 0);
      k_scatter<W, P><<<(uint32_t)n_items, kCta, 0, stream_>>>(items_.as<Item>(), gview(gcur_), aview(cur_), prod, t,
                                                               rec_slot_.as<uint32_t>(), gview(1 - gcur_), aview(o),
                                                               d_stats_, scan_off_.as<unsigned long long>());
      launches_ += 2;
      if (!small) {
        fetch_stats();
        PP_CUDA(cudaGetLastError());
        if (h_stats_->collision) {
          seed_ = mix64(seed_ + 1);
          continue;
        }
      }
      // sort inside groups; the source arena is free now and serves as
      // scratch for the big-group merge passes
      bool source_kept = true;
      if (sort) {
        source_kept = arena_[cur_].cap >= total_bound + 1;
        ensure_arena(cur_, std::min<uint64_t>(total_bound + 1, arena_max_));
        const uint32_t sort_grid = std::max<uint32_t>(1u, std::min<uint32_t>(groups_bound, 148u * 16u));
        const uint32_t small_grid = std::max<uint32_t>(1u, std::min<uint32_t>(groups_bound, 148u * 4u));
        k_sort_small<W><<<small_grid, kCta, sizeof(SortSmem<W>), stream_>>>(gview(1 - gcur_), aview(o),
                                                                             keep_zeros_, d_stats_);
        k_sort_big<W><<<std::min<uint32_t>(sort_grid, 148u * 2u), kCta, big_sort_smem(), stream_>>>(
            gview(1 - gcur_), aview(o), aview(cur_), keep_zeros_, d_stats_);
        launches_ += 2;
      } else {
        // a bijection feeding a dense Rx run: statistics only, groups left
        // unsorted (kFlagUnsorted)
        k_group_stats<W><<<std::max<uint32_t>(1u, std::min<uint32_t>((groups_bound + 7) / 8, 148u * 8u)), kCta, 0,
                           stream_>>>(gview(1 - gcur_), aview(o), d_stats_);
        ++launches_;
      }
      if (small && !sort && defer_ok_) {
        // a small Clifford regroup feeding a dense Rx run: no round trip.  A
        // bijection keeps |O| (no merges, no zeros); the group count stays on
        // the device (kernels read st->G_dev) until the next sync, which also
        // checks the overflow / collision flags and accounts the records.
        k_regroup_commit<<<1, 1, 0, stream_>>>(d_stats_);
        ++launches_;
        PP_CUDA(cudaGetLastError());
        cur_ = o;
        gcur_ = 1 - gcur_;
        G_ = groups_bound;  // upper bound until the sync
        g_pending_ = true;
        unsorted_ = true;
        bump_ = bump_bound_ = live;
        live_ = live_bound_ = live;
        h_records_ = 0;
        dirty_ = true;
        return;
      }
      fetch_stats();
      PP_CUDA(cudaGetLastError());
      if (small && (h_stats_->overflow || h_stats_->collision)) {  // not expected: redo on the careful path
        if (!source_kept) throw EngineError(PP_ERR_INTERNAL, "regroup: fingerprint collision after the source was freed");
        seed_ = mix64(seed_ + 1);
        small = false;
        continue;
      }
      distinct = h_stats_->distinct;
      zfactor_ = std::max(1.0, (double)distinct / (double)std::max<uint32_t>(G_, 1));
      const uint64_t total = h_stats_->scan_total;
      counters_.removed += h_stats_->removed;
      h_records_ = h_stats_->records;
      harvest_seen(*h_stats_);
      cur_ = o;
      gcur_ = 1 - gcur_;
      G_ = distinct;
      unsorted_ = !sort;
      bump_ = bump_bound_ = total;
      live_ = live_bound_ = total - h_stats_->removed;
      reset_stats(bump_);  // cumulative counters were harvested above
      if (keep_zeros_) may_hold_zeros_ = true;
      if ((uint64_t)tc * 48 + live * maxrec * 4 > (64ull << 20)) {
        // large temporaries go back to the pool, where an allocation that
        // does not fit can trim them (the arenas need the room)
        PP_CUDA(cudaStreamSynchronize(stream_));
        table_.release();
        scan_gid_.release();
        scan_off_.release();
        rec_slot_.release();
        items_.release();
      }
      return;
    }
  }

  HashTable<W> tview(uint64_t tc) const {
    HashTable<W> t;
    char* b = table_.as<char>();
    t.fp = reinterpret_cast<unsigned long long*>(b);
    uint64_t* zb = reinterpret_cast<uint64_t*>(b + tc * 8);
    for (int k = 0; k < W; ++k) t.z[k] = zb + k * tc;
    t.count = reinterpret_cast<uint32_t*>(b + tc * 8 + tc * 8 * W);
    t.gid = t.count + tc;
    t.mask = tc - 1;
    return t;
  }

  // exclusive scan of in[0..n) (or of in != 0) into out; total at
  // scan_tmp_[ntiles]
  void device_scan(const uint32_t* in, uint64_t n, int as_flag, unsigned long long* out, uint64_t ntiles) {
    unsigned long long* sums = scan_tmp_.as<unsigned long long>();
    k_scan_tiles<<<(uint32_t)ntiles, kCta, 0, stream_>>>(in, n, as_flag, sums);
    k_scan_sums<<<1, kCta, 0, stream_>>>(sums, ntiles);
    k_scan_apply<<<(uint32_t)ntiles, kCta, 0, stream_>>>(in, n, as_flag, sums, out);
    launches_ += 3;
  }

  pp_config cfg_;
  cudaStream_t stream_ = nullptr;
  DevStats* d_stats_ = nullptr;
  DevStats* h_stats_ = nullptr;
  cudaEvent_t ev0_, ev1_;
  Arena arena_[2];
  Groups groups_[2];
  DevBuf evict_cnt_, evict_buf_, spec_buf_, backup_;
  uint64_t spec_attempts_ = 0;
  DevBuf stats_buf_, list_, items_, rec_slot_, table_, scan_tmp_, scan_gid_, scan_off_, diag_z_, diag_c_, cliff_;
  int cur_ = 0, gcur_ = 0;
  uint32_t G_ = 0;
  uint64_t bump_ = 0, live_ = 0;
  DiagPinned* h_diag_ = nullptr;
  uint64_t diag_n_ = 0, diag_copied_ = 0;
  uint64_t arena_max_ = 0;  // per-arena capacity of the memory plan (strings)
  bool tight_arena_ = false;  // PP_TIGHT_ARENA: minimal arenas (tests of the resume paths)
  static constexpr size_t kLazyWindow = 4096;  // gates per deferred-truncation window
  DevBuf thr_;                // thr[j] = max(T_j .. T_now) over the open window
  std::vector<GraphExecPtr> held_graphs_;  // graphs launched since the last stream sync
  DevBuf norms_, sub_groups_;  // threshold discovery: group norms, the subset's table
  DevBuf buckets_;             // sharded: bucket -> rank table (kBuckets uint16)
  DevBuf spec_done_;           // per group: finished by k_spec_small in this attempt
  bool buckets_on_ = false;
 public:
  // Sharded runs (pp_sharded_*): every rank's observations of a speculative
  // run -- the per-gate maxima and the fault / non-finite / give-up flags --
  // are combined by an element-wise max over the ranks before any decision,
  // so all ranks accept, roll back or give up together.
  std::function<void(std::vector<unsigned long long>&)> spec_reduce_;
 private:
  uint32_t sub_cap_ = 0;
  uint64_t discoveries_ = 0;
  bool lazy_open_ = false;
  uint64_t lazy_base_ = 0;
  uint32_t lazy_len_ = 0;
  double zfactor_ = 4.0;     // distinct output groups per input group at the last regroup
  double gmax_ = 0.0, red_gmax_ = 0.0, red_gmin_ = 0.0;
  uint32_t red_nonfinite_ = 0;
  int keep_zeros_ = 0;
  uint64_t bump_bound_ = 0, live_bound_ = 0;
  bool dirty_ = false, truncated_since_sync_ = false, gmax_stale_ = false, may_hold_zeros_ = false;
  uint64_t eseq_ = 0, bseq_ = 0;
  uint64_t tr_layer_ns_ = 0, tr_sync_ns_ = 0, tr_syncs_ = 0;  // PP_TRACE host timeline
  uint64_t tr_cliff_ns_ = 0, tr_rx_ns_ = 0;
  std::vector<pp_gate> plan_key_;  // apply_gates_async run partition cache
  std::vector<PlanRun> plan_;
  uint64_t dense_groups_ = 0, dense_out_ = 0, bulk_tiles_ = 0;
  std::vector<pp_gate> rx_key_;  // run_rx plan cache
  std::vector<RxParam> rx_prm_;
  SubGates rx_sg_{};
  bool rx_distinct_ = true;
  bool no_dense_ = false;
  int dense_maxk_ = (int)kDenseMaxK;
  std::vector<pp_gate> zz_key_;  // try_zz_run plan cache
  ZZRunProducer<W> zz_prod_{};
  bool zz_ok_ = false;
  cudaEvent_t ev_sync_ = nullptr;
  bool n_small_init_ = false;
  bool poisoned_ = false;  // an operation failed: not reused
  bool g_pending_ = false;        // G_ is an upper bound; the exact count is st->G_dev
  bool defer_ok_ = true;          // PP_NO_DEFER turns the deferred regroup off (test hook)
  // ---- batches_sent (engine.cpp:286-301 at one worker: gates that sent a
  // record).  Gates are indexed from the start of the open window
  // (seen_w0_ = gates_applied_ when it opened); kernels set device bits,
  // every sync ORs them into seen_host_ (idempotent, so a relaunched run
  // cannot count a gate twice), and take_counters closes the window.
  struct ZZEdge {
    int group, bit, gate;  // (group, bit) of the fused ZZ producer -> gate of the run
  };
  std::vector<ZZEdge> zz_edges_;
  uint64_t seen_w0_ = 0;
  std::array<unsigned long long, kSeenWords> seen_host_{};
  bool zz_seen_pending_ = false;
  uint32_t zz_seen_base_ = 0;
  uint32_t window_index() const { return (uint32_t)(gates_applied_ - seen_w0_); }
  void note_zz_run() {
    // settle everything launched so far first: regroup's own sync_state must
    // not harvest (and consume) this run's mask slot before the run exists
    sync_state();
    zz_seen_base_ = window_index();
    zz_seen_pending_ = true;
  }
  void harvest_seen(const DevStats& st) {
    for (int w = 0; w < kSeenWords; ++w) seen_host_[w] |= st.seen[w];
    if (zz_seen_pending_) {
      for (const ZZEdge& e : zz_edges_) {
        if ((st.zz_seen[e.group][e.bit >> 6] >> (e.bit & 63)) & 1ull) {
          const uint32_t b = zz_seen_base_ + (uint32_t)e.gate;
          if (b < (uint32_t)kSeenGates) seen_host_[b >> 6] |= 1ull << (b & 63);
        }
      }
      zz_seen_pending_ = false;
    }
  }
  void close_window() {
    uint64_t n = 0;
    for (auto& w : seen_host_) {
      n += (uint64_t)__builtin_popcountll(w);
      w = 0;
    }
    counters_.batches_sent += n;
    seen_w0_ = gates_applied_;
  }
  // before a run of `count` gates: the window must have room for all of them
  void reserve_window(size_t count) {
    if (window_index() + count <= (size_t)kSeenGates) return;
    sync_state();
    close_window();
    if (count > (size_t)kSeenGates)
      throw EngineError(PP_ERR_INTERNAL, "gate run longer than the batch window");
  }
  bool spin_sync_ = true;
  bool arena_fault_ = false;
  bool unsorted_fault_ = false;  // a sublayer left unsorted groups for the per-gate path
  bool unsorted_ = false;        // the table holds kFlagUnsorted groups
  bool sub_pending_ = false;  // a sublayer launch not yet checked for an arena overflow
  SubGates sub_gates_{};
  uint64_t sub_seq0_ = 0;
  uint64_t arena_fault_seq_ = 0;

  uint32_t branch_grid_ = 148u * 2u;
  uint32_t sub_grid_ = 148u * 2u;
  uint32_t dense_grid_ = 148u * 2u;
  DevBuf left_list_;             // groups the dense kernel left for the per-gate path
  bool no_dense_kernel_ = std::getenv("PP_NO_DENSE_KERNEL") != nullptr;  // dense path inside k_branch_sublayer
  uint32_t small_grid_ = 148u * 3u;
  uint32_t zz_grid_ = 148u * 2u;
  uint32_t maxcnt_ = 0x7fffffffu;  // largest group at the last full sync (bounds Z-type pair sizes)
  DevBuf ztab_;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending_events_, free_events_;
  unsigned long long seed_;
  unsigned long long h_records_ = 0;
  pp_counters counters_{};
  uint64_t gates_applied_ = 0;
  uint64_t err_base_ = 0;  // gates applied before relative gate 0 of the launches in flight (error messages)
  int layer_ = 0;
  double branch_ms_ = 0.0, branch_bytes_ = 0.0;
  uint64_t branch_in_ = 0, branch_stream_ = 0;
 public:
  double last_stream_frac_ = 0.0;
 private:
  uint64_t branch_launches_ = 0, launches_ = 0;
};

}  // namespace ppgpu

#include "pp_sharded.cuh"

// ===========================================================================
// C-ABI
// ===========================================================================
struct pp_engine {
  std::unique_ptr<ppgpu::EngineBase> impl;
  std::string error;
  std::string key;  // configuration + construction-time environment (engine pool)
};

namespace {
// Released engines are kept (a few, small ones) and handed to the next
// pp_create with the same configuration: creating an engine costs stream,
// event and launch-setup work comparable to a small propagation.  The pool
// is never destroyed (no CUDA calls during process teardown).
std::mutex g_engine_pool_mu;
std::vector<std::pair<std::string, ppgpu::EngineBase*>>* g_engine_pool = new std::vector<std::pair<std::string, ppgpu::EngineBase*>>();
constexpr size_t kEnginePoolMax = 4;

// device memory is short: parked engines go (their buffers return to the
// device pool, which then frees its cache)
void release_parked_engines(int device) {
  std::vector<ppgpu::EngineBase*> victims;
  {
    std::lock_guard<std::mutex> lk(g_engine_pool_mu);
    auto& pool = *g_engine_pool;
    for (size_t i = 0; i < pool.size();) {
      if (device < 0 || pool[i].second->device() == device) {
        victims.push_back(pool[i].second);
        pool.erase(pool.begin() + i);
      } else {
        ++i;
      }
    }
  }
  for (auto* v : victims) delete v;  // each destructor runs on its own device
}
size_t parked_engine_bytes(int device) {
  std::lock_guard<std::mutex> lk(g_engine_pool_mu);
  size_t b = 0;
  for (auto& kv : *g_engine_pool)
    if (kv.second->device() == device) b += kv.second->device_bytes();
  return b;
}
struct ParkedEnginesHook {
  ParkedEnginesHook() {
    ppgpu::g_release_parked_engines = &release_parked_engines;
    ppgpu::g_parked_engine_bytes = &parked_engine_bytes;
  }
} g_parked_engines_hook;

std::string engine_key(const pp_config& c) {
  std::string k;
  auto put = [&](const void* p, size_t n) { k.append(static_cast<const char*>(p), n); };
  put(&c.n, sizeof c.n);
  put(&c.epsilon0, sizeof c.epsilon0);
  put(&c.cadence, sizeof c.cadence);
  put(&c.max_terms, sizeof c.max_terms);
  put(&c.workers, sizeof c.workers);
  put(&c.device, sizeof c.device);
  put(&c.flags, sizeof c.flags);
  put(&c.mem_fraction, sizeof c.mem_fraction);
  for (const char* v : {"PP_TIGHT_ARENA", "PP_NO_DENSE", "PP_DENSE_MAXK", "PP_NO_DEFER", "PP_BLOCKING_SYNC", "PP_TRACE",
                        "PP_NO_SPECULATE", "PP_NO_DENSE_KERNEL", "PP_DENSE_CAREFUL"}) {
    const char* x = std::getenv(v);
    k += '|';
    if (x) k += x;
  }
  return k;
}
}  // namespace

namespace {
thread_local std::string g_create_error;

template <class F>
int guarded(pp_engine* e, F&& f) {
  try {
    f();
    return PP_OK;
  } catch (const ppgpu::EngineError& x) {
    if (e) {
      e->error = x.what();
      if (e->impl) e->impl->poison();
    }
    return x.code;
  } catch (const std::bad_alloc&) {
    if (e) {
      e->error = "host memory exhausted";
      if (e->impl) e->impl->poison();
    }
    return PP_ERR_RESOURCE;
  } catch (const std::exception& x) {
    if (e) {
      e->error = x.what();
      if (e->impl) e->impl->poison();
    }
    return PP_ERR_INTERNAL;
  }
}
}  // namespace

extern "C" {

int pp_create(const pp_config* config, pp_engine** out) {
  if (!config || !out) return PP_ERR_INVALID;
  *out = nullptr;
  if (config->n < 1 || config->n > 128) {
    g_create_error = "qubit count out of range";
    return PP_ERR_INVALID;
  }
  if (!(config->epsilon0 >= 0)) {
    g_create_error = "epsilon0 must be >= 0";
    return PP_ERR_INVALID;
  }
  if (config->cadence != PP_CADENCE_GATE && config->cadence != PP_CADENCE_LAYER) {
    g_create_error = "bad cadence";
    return PP_ERR_INVALID;
  }
  auto e = std::make_unique<pp_engine>();
  e->key = engine_key(*config);
  {
    std::lock_guard<std::mutex> lk(g_engine_pool_mu);
    for (auto it = g_engine_pool->begin(); it != g_engine_pool->end(); ++it)
      if (it->first == e->key) {
        e->impl.reset(it->second);
        g_engine_pool->erase(it);
        break;
      }
  }
  if (e->impl) {
    int rc = guarded(e.get(), [&] { e->impl->on_reuse(); });
    if (rc == PP_OK) {
      *out = e.release();
      return PP_OK;
    }
    e->impl.reset();
  }
  int rc = guarded(e.get(), [&] {
    int ndev = 0;
    cudaError_t err = cudaGetDeviceCount(&ndev);
    if (err != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw ppgpu::EngineError(PP_ERR_INTERNAL, "no CUDA device available (the engine has no CPU fallback)");
    }
    if (config->device < 0 || config->device >= ndev) throw ppgpu::EngineError(PP_ERR_INVALID, "bad device ordinal");
    if (config->n <= 64) e->impl = std::make_unique<ppgpu::EngineImpl<1>>(*config);
    else e->impl = std::make_unique<ppgpu::EngineImpl<2>>(*config);
  });
  if (rc) {
    g_create_error = e->error;
    return rc;
  }
  *out = e.release();
  return PP_OK;
}

void pp_destroy(pp_engine* e) {
  if (!e) return;
  if (e->impl && e->impl->reusable()) {
    ppgpu::EngineBase* victim = nullptr;
    {
      std::lock_guard<std::mutex> lk(g_engine_pool_mu);
      if (g_engine_pool->size() >= kEnginePoolMax) {
        victim = g_engine_pool->front().second;
        g_engine_pool->erase(g_engine_pool->begin());
      }
      g_engine_pool->emplace_back(e->key, e->impl.release());
    }
    delete victim;
  }
  delete e;
}

int pp_set_initial(pp_engine* e, const uint64_t* words, const double* coeffs, size_t count) {
  if (!e) return PP_ERR_INVALID;
  return guarded(e, [&] { e->impl->set_initial(words, coeffs, count); });
}

int pp_apply_gate(pp_engine* e, const pp_gate* gate) {
  if (!e || !gate) return PP_ERR_INVALID;
  return guarded(e, [&] { e->impl->apply_gates(gate, 1); });
}

int pp_apply_gates(pp_engine* e, const pp_gate* gates, size_t count) {
  if (!e || (!gates && count)) return PP_ERR_INVALID;
  return guarded(e, [&] { e->impl->apply_gates(gates, count); });
}

int pp_apply_layer(pp_engine* e, const pp_gate* gates, size_t count, double* observable) {
  if (!e || (!gates && count) || !observable) return PP_ERR_INVALID;
  return guarded(e, [&] { *observable = e->impl->apply_layer(gates, count); });
}

int pp_truncate_now(pp_engine* e) {
  if (!e) return PP_ERR_INVALID;
  return guarded(e, [&] { e->impl->truncate_now(); });
}

int pp_term_count(const pp_engine* e, uint64_t* out) {
  if (!e || !out) return PP_ERR_INVALID;
  return guarded(const_cast<pp_engine*>(e), [&] { *out = e->impl->term_count(); });
}

int pp_global_max(const pp_engine* e, double* out) {
  if (!e || !out) return PP_ERR_INVALID;
  return guarded(const_cast<pp_engine*>(e), [&] { *out = e->impl->global_max(); });
}

int pp_expectation_zero_state(pp_engine* e, double* out) {
  if (!e || !out) return PP_ERR_INVALID;
  return guarded(e, [&] { *out = e->impl->expectation(); });
}

int pp_coefficient(pp_engine* e, const uint64_t* words, double* out) {
  if (!e || !words || !out) return PP_ERR_INVALID;
  return guarded(e, [&] { *out = e->impl->coefficient(words); });
}

int pp_export(pp_engine* e, uint64_t* words, double* coeffs, uint64_t cap, uint64_t* count) {
  if (!e || !count) return PP_ERR_INVALID;
  return guarded(e, [&] { *count = e->impl->export_terms(words, coeffs, cap); });
}

int pp_take_counters(pp_engine* e, pp_counters* out) {
  if (!e || !out) return PP_ERR_INVALID;
  *out = e->impl->take_counters();
  return PP_OK;
}

int pp_take_kernel_stats(pp_engine* e, double* branch_ms, double* branch_bytes, uint64_t* branch_launches,
                         uint64_t* total_launches) {
  if (!e) return PP_ERR_INVALID;
  e->impl->take_kernel_stats(branch_ms, branch_bytes, branch_launches, total_launches);
  return PP_OK;
}

void* pp_stream(const pp_engine* e) { return e ? e->impl->stream() : nullptr; }

void pp_transfer_totals(uint64_t* h2d_bytes, uint64_t* d2h_bytes) {
  if (h2d_bytes) *h2d_bytes = ppgpu::g_h2d_bytes.load();
  if (d2h_bytes) *d2h_bytes = ppgpu::g_d2h_bytes.load();
}

int pp_local_stats(pp_engine* e, double* gmax, uint32_t* nonfinite, uint64_t* count) {
  if (!e || !gmax || !nonfinite || !count) return PP_ERR_INVALID;
  return guarded(e, [&] { e->impl->local_stats(gmax, nonfinite, count); });
}

int pp_truncate_threshold(pp_engine* e, double threshold, uint64_t* removed) {
  if (!e) return PP_ERR_INVALID;
  return guarded(e, [&] {
    uint64_t r = e->impl->truncate_threshold(threshold);
    if (removed) *removed = r;
  });
}

int pp_record_words(const pp_engine* e) { return e ? e->impl->record_words() : 0; }

int pp_group_sizes(pp_engine* e, uint64_t* groups, uint64_t* strings) {
  if (!e || !groups || !strings) return PP_ERR_INVALID;
  return guarded(e, [&] { e->impl->group_sizes(groups, strings); });
}

int pp_norm2(pp_engine* e, double* out) {
  if (!e || !out) return PP_ERR_INVALID;
  return guarded(e, [&] { *out = e->impl->norm2(); });
}

int pp_density_histogram(pp_engine* e, int bins, double global_max, double epsilon0, uint64_t* positive,
                         uint64_t* negative) {
  if (!e || !positive || !negative || bins < 1 || bins > ppgpu::kMaxHistBins) return PP_ERR_INVALID;
  return guarded(e, [&] {
    if (e->impl->term_count() > 0 && !(global_max > 0))
      throw ppgpu::EngineError(PP_ERR_INVALID,
                               "density_histogram needs a positive global maximum for a nonempty operator");
    e->impl->histogram(bins, global_max, epsilon0, positive, negative);
  });
}

int pp_shard_evict(pp_engine* e, uint32_t world, uint32_t rank, uint64_t seed, uint64_t* records, uint64_t cap,
                   uint64_t* counts) {
  if (!e || !counts || world == 0 || rank >= world) return PP_ERR_INVALID;
  return guarded(e, [&] { e->impl->shard_evict(world, rank, seed, records, cap, counts); });
}

int pp_shard_ingest(pp_engine* e, const uint64_t* records, uint64_t count) {
  if (!e || (!records && count)) return PP_ERR_INVALID;
  return guarded(e, [&] { e->impl->shard_ingest(records, count, false); });
}

int pp_shard_evict_device(pp_engine* e, uint32_t world, uint32_t rank, uint64_t seed, const uint64_t** records,
                          uint64_t* counts) {
  if (!e || !counts || !records || world == 0 || rank >= world) return PP_ERR_INVALID;
  return guarded(e, [&] {
    e->impl->shard_evict(world, rank, seed, nullptr, ~0ull, counts);
    *records = e->impl->device_records();
  });
}

int pp_shard_ingest_device(pp_engine* e, const uint64_t* records, uint64_t count) {
  if (!e || (!records && count)) return PP_ERR_INVALID;
  return guarded(e, [&] { e->impl->shard_ingest(records, count, true); });
}

uint32_t pp_shard_owner(const uint64_t* words, int n, uint64_t seed, uint32_t world) {
  uint64_t x[2], z[2];
  ppgpu::words_to_planes(words, x, z);
  if (n <= 64) {
    ppgpu::Plane<1> p;
    p.w[0] = z[0];
    return ppgpu::shard_owner<1>(p, seed, world);
  }
  ppgpu::Plane<2> p;
  p.w[0] = z[0];
  p.w[1] = z[1];
  return ppgpu::shard_owner<2>(p, seed, world);
}

const char* pp_last_error(const pp_engine* e) { return e ? e->error.c_str() : g_create_error.c_str(); }

}  // extern "C"

// ---------------------------------------------------------------- sharded engine
struct pp_sharded {
  std::unique_ptr<ppgpu::ShardedDriver> d;
  std::string error;
};
struct pp_hub {
  explicit pp_hub(int w) : hub(w) {}
  ppgpu::ThreadHub hub;
};

namespace {
template <class F>
int guarded_s(pp_sharded* s, F&& f) {
  try {
    f();
    return PP_OK;
  } catch (const ppgpu::EngineError& x) {
    if (s) s->error = x.what();
    return x.code;
  } catch (const std::bad_alloc&) {
    if (s) s->error = "host memory exhausted";
    return PP_ERR_RESOURCE;
  } catch (const std::exception& x) {
    if (s) s->error = x.what();
    return PP_ERR_INTERNAL;
  }
}
int sharded_precheck(const pp_config* c) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    g_create_error = "no CUDA device available";
    return PP_ERR_INTERNAL;
  }
  if (!c || c->n < 1 || c->n > 128 || !(c->epsilon0 >= 0.0) || c->device < 0 || c->device >= ndev) {
    g_create_error = "invalid sharded engine configuration";
    return PP_ERR_INVALID;
  }
  return PP_OK;
}
}  // namespace

int pp_nccl_unique_id(uint8_t id[128]) {
  if (!id) return PP_ERR_INVALID;
  try {
    ncclUniqueId u;
    ncclResult_t r = ppgpu::NcclApi::get().GetUniqueId(&u);
    if (r != ncclSuccess) {
      g_create_error = std::string("ncclGetUniqueId: ") + ppgpu::NcclApi::get().GetErrorString(r);
      return PP_ERR_INTERNAL;
    }
    static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(id, &u, 128);
    return PP_OK;
  } catch (const std::exception& x) {
    g_create_error = x.what();
    return PP_ERR_INTERNAL;
  }
}

int pp_sharded_create(const pp_config* c, int world, int rank, const uint8_t id[128], pp_sharded** out) {
  if (!out || !id || world < 1 || rank < 0 || rank >= world) return PP_ERR_INVALID;
  *out = nullptr;
  if (int rc = sharded_precheck(c)) return rc;
  auto s = std::make_unique<pp_sharded>();
  int rc = guarded_s(s.get(), [&] {
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    s->d = std::make_unique<ppgpu::ShardedDriver>(
        *c, std::make_unique<ppgpu::NcclCollective>(world, rank, u, c->device));
  });
  if (rc != PP_OK) {
    g_create_error = s->error;
    return rc;
  }
  *out = s.release();
  return PP_OK;
}

pp_hub* pp_hub_create(int world) { return world >= 1 ? new pp_hub(world) : nullptr; }
void pp_hub_destroy(pp_hub* h) { delete h; }

int pp_sharded_create_hub(const pp_config* c, pp_hub* hub, int rank, pp_sharded** out) {
  if (!out || !hub || rank < 0 || rank >= hub->hub.world) return PP_ERR_INVALID;
  *out = nullptr;
  if (int rc = sharded_precheck(c)) return rc;
  auto s = std::make_unique<pp_sharded>();
  int rc = guarded_s(s.get(), [&] {
    s->d = std::make_unique<ppgpu::ShardedDriver>(*c, std::make_unique<ppgpu::HubCollective>(&hub->hub, rank,
                                                                                            c->device));
  });
  if (rc != PP_OK) {
    g_create_error = s->error;
    return rc;
  }
  *out = s.release();
  return PP_OK;
}

void pp_sharded_destroy(pp_sharded* s) { delete s; }

int pp_sharded_set_initial(pp_sharded* s, const uint64_t* words, const double* coeffs, size_t count) {
  if (!s || (count && (!words || !coeffs))) return PP_ERR_INVALID;
  return guarded_s(s, [&] { s->d->set_initial(words, coeffs, count); });
}
int pp_sharded_apply_gates(pp_sharded* s, const pp_gate* gates, size_t count) {
  if (!s || (count && !gates)) return PP_ERR_INVALID;
  return guarded_s(s, [&] { s->d->apply_gates(gates, count); });
}
int pp_sharded_apply_layer(pp_sharded* s, const pp_gate* gates, size_t count, double* observable) {
  if (!s || !observable || (count && !gates)) return PP_ERR_INVALID;
  return guarded_s(s, [&] { *observable = s->d->apply_layer(gates, count); });
}
int pp_sharded_truncate_now(pp_sharded* s) {
  if (!s) return PP_ERR_INVALID;
  return guarded_s(s, [&] { s->d->truncate_now(); });
}
int pp_sharded_term_count(pp_sharded* s, uint64_t* out) {
  if (!s || !out) return PP_ERR_INVALID;
  return guarded_s(s, [&] { *out = s->d->term_count(); });
}
int pp_sharded_global_max(pp_sharded* s, double* out) {
  if (!s || !out) return PP_ERR_INVALID;
  return guarded_s(s, [&] { *out = s->d->global_max(); });
}
int pp_sharded_take_counters(pp_sharded* s, pp_counters* out) {
  if (!s || !out) return PP_ERR_INVALID;
  return guarded_s(s, [&] { *out = s->d->take_counters(); });
}
int pp_sharded_stats(pp_sharded* s, pp_shard_stats* out) {
  if (!s || !out) return PP_ERR_INVALID;
  return guarded_s(s, [&] { s->d->stats(out); });
}
int pp_sharded_local_count(pp_sharded* s, uint64_t* out) {
  if (!s || !out) return PP_ERR_INVALID;
  return guarded_s(s, [&] { *out = s->d->engine().term_count(); });
}
int pp_sharded_local_export(pp_sharded* s, uint64_t* words, double* coeffs, uint64_t cap, uint64_t* count) {
  if (!s || !count || (cap && (!words || !coeffs))) return PP_ERR_INVALID;
  return guarded_s(s, [&] { *count = s->d->engine().export_terms(words, coeffs, cap); });
}
void* pp_sharded_stream(const pp_sharded* s) { return s ? s->d->engine().stream() : nullptr; }
int pp_sharded_kernel_stats(pp_sharded* s, double* branch_ms, double* branch_bytes, uint64_t* branch_launches,
                            uint64_t* total_launches) {
  if (!s || !branch_ms || !branch_bytes || !branch_launches || !total_launches) return PP_ERR_INVALID;
  return guarded_s(s, [&] { s->d->engine().take_kernel_stats(branch_ms, branch_bytes, branch_launches, total_launches); });
}
const char* pp_sharded_last_error(const pp_sharded* s) { return s ? s->error.c_str() : g_create_error.c_str(); }
