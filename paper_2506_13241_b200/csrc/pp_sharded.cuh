// pp_sharded.cuh -- the operator sharded over GPUs, one engine per rank, SPMD
// (included by pp_engine.cu, C-ABI pp_sharded_* in
// include/pauliprop_gpu.h).
//
// Ownership: a z-plane hash picks one of kBuckets virtual buckets, a bucket
// table maps buckets to ranks.  An X-type gate keeps z, so every Rx
// branch + merge is rank-local; only Clifford/ZZ runs and Z/Y-carrying
// generators move strings.  After such a step every rank builds the global
// bucket histogram (one all-reduce), all ranks derive the same balanced
// table (largest bucket first onto the least-loaded rank), evict the groups
// they no longer own into a device buffer grouped by destination, and one
// all-to-all (grouped ncclSend/ncclRecv over NVLink) delivers them; the
// receiver merges equal keys exactly like TermMap::add (regroup).
//
// Global quantities are collectives: for eps0 > 0 at per-gate cadence an Rx
// run is ONE speculative launch per rank whose per-gate maxima are max-reduced
// over the ranks (EngineImpl::spec_reduce_) -- one small all-reduce per run
// (and per discovery attempt) instead of a host round trip per gate; after a
// string-moving step the global max and count (engine.cpp:321-345) and the
// <0|O|0> readout are all-reduced.  Every rank issues the same collectives in
// the same order whatever its local size, so no rank waits on a skipped one.
//
// Two transports: NCCL (one process per GPU, bootstrapped with an
// ncclUniqueId the caller distributes) and an in-process hub (ranks as
// threads sharing one device; host barriers and device-to-device copies) that
// runs the same driver on one GPU for tests.
#pragma once

#include <condition_variable>

#include "pp_nccl.h"

namespace ppgpu {

class Collective {
 public:
  virtual ~Collective() = default;
  virtual int world() const = 0;
  virtual int rank() const = 0;
  // element-wise over the ranks, host vectors in and out
  virtual void allreduce_max(std::vector<unsigned long long>& v) = 0;
  virtual void allreduce_sum(std::vector<unsigned long long>& v) = 0;
  virtual void allreduce_sum(std::vector<double>& v) = 0;
  // send[d] words from d_send (grouped by destination, in rank order) to rank
  // d; recv[s] words from rank s land in d_recv in source order.  The device
  // buffers must be ready (the caller synchronised their producer).
  virtual void alltoallv(const uint64_t* d_send, const std::vector<uint64_t>& send, uint64_t* d_recv,
                         const std::vector<uint64_t>& recv) = 0;
};

// ---- NCCL: one rank per process and GPU
class NcclCollective final : public Collective {
 public:
  NcclCollective(int world, int rank, const ncclUniqueId& id, int device) : world_(world), rank_(rank) {
    NcclApi& nc = NcclApi::get();
    PP_CUDA(cudaSetDevice(device));
    PP_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    PP_NCCL(nc.CommInitRank(&comm_, world, id, rank));
  }
  ~NcclCollective() override {
    if (comm_) NcclApi::get().CommDestroy(comm_);
    if (stream_) cudaStreamDestroy(stream_);
  }
  int world() const override { return world_; }
  int rank() const override { return rank_; }
  void allreduce_max(std::vector<unsigned long long>& v) override { reduce(v.data(), v.size(), ncclUint64, ncclMax); }
  void allreduce_sum(std::vector<unsigned long long>& v) override { reduce(v.data(), v.size(), ncclUint64, ncclSum); }
  void allreduce_sum(std::vector<double>& v) override { reduce(v.data(), v.size(), ncclFloat64, ncclSum); }
  void alltoallv(const uint64_t* d_send, const std::vector<uint64_t>& send, uint64_t* d_recv,
                 const std::vector<uint64_t>& recv) override {
    NcclApi& nc = NcclApi::get();
    uint64_t so = 0, ro = 0;
    PP_NCCL(nc.GroupStart());
    for (int p = 0; p < world_; ++p) {
      if (send[p]) PP_NCCL(nc.Send(d_send + so, send[p], ncclUint64, p, comm_, stream_));
      if (recv[p]) PP_NCCL(nc.Recv(d_recv + ro, recv[p], ncclUint64, p, comm_, stream_));
      so += send[p];
      ro += recv[p];
    }
    PP_NCCL(nc.GroupEnd());
    PP_CUDA(cudaStreamSynchronize(stream_));
  }

 private:
  void reduce(void* host, size_t n, ncclDataType_t t, ncclRedOp_t op) {
    if (n == 0) return;
    buf_.ensure(n * 8);
    PP_CUDA(copy_async(buf_.p, host, n * 8, cudaMemcpyHostToDevice, stream_));
    PP_NCCL(NcclApi::get().AllReduce(buf_.p, buf_.p, n, t, op, comm_, stream_));
    PP_CUDA(copy_async(host, buf_.p, n * 8, cudaMemcpyDeviceToHost, stream_));
    PP_CUDA(cudaStreamSynchronize(stream_));
  }
  int world_, rank_;
  ncclComm_t comm_ = nullptr;
  cudaStream_t stream_ = nullptr;
  DevBuf buf_;
};

// ---- in-process hub: ranks as threads of one process on one device
struct ThreadHub {
  explicit ThreadHub(int w) : world(w), slots(w), dslots(w), dev(w, nullptr), offs(w) {}
  int world;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  std::vector<std::vector<unsigned long long>> slots;
  std::vector<std::vector<double>> dslots;
  std::vector<const uint64_t*> dev;
  std::vector<std::vector<uint64_t>> offs;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

class HubCollective final : public Collective {
 public:
  HubCollective(ThreadHub* hub, int rank, int device) : hub_(hub), rank_(rank) {
    PP_CUDA(cudaSetDevice(device));
    PP_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  }
  ~HubCollective() override { cudaStreamDestroy(stream_); }
  int world() const override { return hub_->world; }
  int rank() const override { return rank_; }
  void allreduce_max(std::vector<unsigned long long>& v) override {
    combine(v, [](unsigned long long a, unsigned long long b) { return a > b ? a : b; });
  }
  void allreduce_sum(std::vector<unsigned long long>& v) override {
    combine(v, [](unsigned long long a, unsigned long long b) { return a + b; });
  }
  void allreduce_sum(std::vector<double>& v) override {
    hub_->dslots[rank_] = v;
    hub_->barrier();
    for (size_t i = 0; i < v.size(); ++i) {  // rank order: the same sum on every rank
      double s = 0.0;
      for (int r = 0; r < hub_->world; ++r) s += hub_->dslots[r][i];
      v[i] = s;
    }
    hub_->barrier();
  }
  void alltoallv(const uint64_t* d_send, const std::vector<uint64_t>& send, uint64_t* d_recv,
                 const std::vector<uint64_t>& recv) override {
    std::vector<uint64_t> off(send.size() + 1, 0);
    for (size_t p = 0; p < send.size(); ++p) off[p + 1] = off[p] + send[p];
    hub_->dev[rank_] = d_send;
    hub_->offs[rank_] = off;
    hub_->barrier();
    uint64_t ro = 0;
    for (int s = 0; s < hub_->world; ++s) {
      const uint64_t n = hub_->offs[s][rank_ + 1] - hub_->offs[s][rank_];
      if (n != recv[s]) throw EngineError(PP_ERR_INTERNAL, "hub all-to-all: count mismatch");
      if (n)
        PP_CUDA(cudaMemcpyAsync(d_recv + ro, hub_->dev[s] + hub_->offs[s][rank_], n * 8, cudaMemcpyDeviceToDevice,
                                stream_));
      ro += n;
    }
    PP_CUDA(cudaStreamSynchronize(stream_));
    hub_->barrier();  // every rank holds its copy before any source buffer is reused
  }

 private:
  template <class F>
  void combine(std::vector<unsigned long long>& v, F f) {
    hub_->slots[rank_] = v;
    hub_->barrier();
    for (size_t i = 0; i < v.size(); ++i) {
      unsigned long long a = hub_->slots[0][i];
      for (int r = 1; r < hub_->world; ++r) a = f(a, hub_->slots[r][i]);
      v[i] = a;
    }
    hub_->barrier();
  }
  ThreadHub* hub_;
  int rank_;
  cudaStream_t stream_ = nullptr;
};

// ---- the SPMD driver
class ShardedDriver {
 public:
  static constexpr uint64_t kSeed = 0x243F6A8885A308D3ull;  // fixed: owners agree across ranks

  ShardedDriver(const pp_config& cfg, std::unique_ptr<Collective> coll) : cfg_(cfg), coll_(std::move(coll)) {
    if (cfg.max_terms) throw EngineError(PP_ERR_INVALID, "sharded engine: max_terms is not supported");
    pp_config c = cfg;
    c.flags |= PP_FLAG_EXTERNAL_TRUNCATION;
    if (cfg.n <= 64) eng_ = std::make_unique<EngineImpl<1>>(c);
    else eng_ = std::make_unique<EngineImpl<2>>(c);
    const int world = coll_->world();
    table_.resize(kBuckets);
    for (uint32_t b = 0; b < kBuckets; ++b) table_[b] = (uint16_t)(b % (uint32_t)world);
    eng_->set_bucket_table(table_.data());
    Collective* cl = coll_.get();
    eng_->set_spec_reduce([cl](std::vector<unsigned long long>& v) { cl->allreduce_max(v); });
  }
  EngineBase& engine() { return *eng_; }
  Collective& comm() { return *coll_; }

  void set_initial(const uint64_t* words, const double* c, size_t count) {
    std::vector<uint64_t> w;
    std::vector<double> cc;
    double lmax = 0.0;
    for (size_t i = 0; i < count; ++i) {
      if (owner_of(words + 4 * i) != (uint32_t)coll_->rank()) continue;
      w.insert(w.end(), words + 4 * i, words + 4 * i + 4);
      cc.push_back(c[i]);
      if (std::isfinite(c[i])) lmax = std::max(lmax, std::fabs(c[i]));
    }
    eng_->set_initial(w.data(), cc.data(), cc.size());
    std::vector<unsigned long long> v{__builtin_bit_cast(unsigned long long, lmax)};
    coll_->allreduce_max(v);
    gmax_ = __builtin_bit_cast(double, (uint64_t)v[0]);
    eng_->set_global_max(gmax_);
  }

  // Gates in application order (a layer reversed, as run_circuit does):
  // the plan of sharded.py's ShardedEngine.apply_gates, collectives native.
  void apply_gates(const pp_gate* g, size_t count) {
    const bool per_gate = cfg_.cadence == PP_CADENCE_GATE;
    size_t i = 0;
    while (i < count) {
      if (is_x(g[i]) && !is_clifford(g[i])) {
        size_t j = i;
        while (j < count && j - i < (size_t)kMaxSubGates && is_x(g[j]) && !is_clifford(g[j])) ++j;
        eng_->apply_gates(g + i, j - i);  // rank-local; eps0 > 0: one reduced speculative run
        if (per_gate && cfg_.epsilon0 > 0.0) gmax_ = eng_->global_max();  // the run's reduced max
        i = j;
      } else if (is_clifford(g[i])) {
        size_t j = i;
        while (j < count && is_clifford(g[j])) ++j;
        eng_->apply_gates(g + i, j - i);  // a fused signed permutation: magnitudes only move
        exchange();
        if (per_gate) epilogue(true);
        i = j;
      } else {
        eng_->apply_gates(g + i, 1);
        exchange();
        if (per_gate) epilogue(true);
        ++i;
      }
    }
    if (per_gate && cfg_.epsilon0 == 0.0) epilogue(true);  // keep the global max current
  }

  void truncate_now() { epilogue(true); }

  double apply_layer(const pp_gate* g, size_t count) {
    apply_gates(g, count);
    if (cfg_.cadence == PP_CADENCE_LAYER) epilogue(true);
    return expectation();
  }

  double expectation() {
    std::vector<double> v{eng_->expectation()};
    coll_->allreduce_sum(v);
    return v[0];
  }
  uint64_t term_count() {
    std::vector<unsigned long long> v{eng_->term_count()};
    coll_->allreduce_sum(v);
    return v[0];
  }
  double global_max() const { return gmax_; }

  void stats(pp_shard_stats* s) const { *s = stats_; }

  pp_counters take_counters() {
    pp_counters c = eng_->take_counters();
    std::vector<unsigned long long> v{c.removed, c.batches_sent, c.records_sent};
    coll_->allreduce_sum(v);
    c.removed = v[0];
    c.batches_sent = v[1];
    c.records_sent = v[2];
    return c;
  }

 private:
  static bool is_clifford(const pp_gate& g) {
    return g.cos_theta == 0.0 && (g.sin_theta == 1.0 || g.sin_theta == -1.0);
  }
  static bool is_x(const pp_gate& g) {  // a single X: keeps z, rank-local
    uint64_t x[2], z[2];
    words_to_planes(g.words, x, z);
    return (z[0] | z[1]) == 0 && __builtin_popcountll(x[0]) + __builtin_popcountll(x[1]) == 1;
  }
  uint32_t owner_of(const uint64_t* words) const {
    uint64_t x[2], z[2];
    words_to_planes(words, x, z);
    uint64_t h;
    if (cfg_.n <= 64) {
      Plane<1> p;
      p.w[0] = z[0];
      h = shard_hash<1>(p, kSeed);
    } else {
      Plane<2> p;
      p.w[0] = z[0];
      p.w[1] = z[1];
      h = shard_hash<2>(p, kSeed);
    }
    return table_[h % kBuckets];
  }

  // Balanced bucket table from the global histogram: buckets by decreasing
  // size (ties: lower index) onto the least-loaded rank (ties: lower rank);
  // every rank computes the same table.
  void rebalance() {
    std::vector<unsigned long long> hist(kBuckets);
    eng_->bucket_histogram(kSeed, reinterpret_cast<uint64_t*>(hist.data()));
    coll_->allreduce_sum(hist);
    const int world = coll_->world();
    std::vector<uint32_t> order(kBuckets);
    for (uint32_t b = 0; b < kBuckets; ++b) order[b] = b;
    std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return hist[a] > hist[b]; });
    std::vector<unsigned long long> load(world, 0);
    for (uint32_t b : order) {
      int best = 0;
      for (int r = 1; r < world; ++r)
        if (load[r] < load[best]) best = r;
      table_[b] = (uint16_t)best;
      load[best] += hist[b];
    }
    const auto [lo, hi] = std::minmax_element(load.begin(), load.end());
    stats_.balance = *lo ? (double)*hi / (double)*lo : (*hi ? INFINITY : 1.0);
    eng_->set_bucket_table(table_.data());
  }

  // strings whose owner changed move: evict (device buffer grouped by
  // destination), count matrix (one all-reduce), all-to-all, ingest
  void exchange() {
    auto t0 = Clock::now();
    const int world = coll_->world(), rank = coll_->rank();
    if (world > 1) rebalance();
    std::vector<uint64_t> counts(world, 0);
    eng_->shard_evict(world, rank, kSeed, nullptr, ~0ull, counts.data());
    const uint64_t rw = (uint64_t)eng_->record_words();
    std::vector<unsigned long long> mat((size_t)world * world, 0);
    for (int d = 0; d < world; ++d) mat[(size_t)rank * world + d] = counts[d];
    coll_->allreduce_sum(mat);
    std::vector<uint64_t> send(world), recv(world);
    uint64_t total_recv = 0;
    for (int p = 0; p < world; ++p) {
      send[p] = mat[(size_t)rank * world + p] * rw;
      recv[p] = mat[(size_t)p * world + rank] * rw;
      total_recv += recv[p];
      stats_.records_moved += mat[(size_t)rank * world + p];
    }
    recv_buf_.ensure(std::max<uint64_t>(total_recv, 1) * 8);
    coll_->alltoallv(eng_->device_records(), send, recv_buf_.as<uint64_t>(), recv);
    if (total_recv) eng_->shard_ingest(recv_buf_.as<uint64_t>(), total_recv / rw, true);
    ++stats_.exchanges;
    stats_.exchange_ns += ns_since(t0);
  }

  // truncate_now across ranks (engine.cpp:318-351): global max and NaN flag
  // by one max-reduce, threshold epsilon0 * gmax on every rank
  void epilogue(bool truncate) {
    double lmax = 0.0;
    uint32_t nf = 0;
    uint64_t cnt = 0;
    eng_->local_stats(&lmax, &nf, &cnt);
    std::vector<unsigned long long> v{__builtin_bit_cast(unsigned long long, lmax), nf ? 1ull : 0ull};
    coll_->allreduce_max(v);
    if (v[1]) throw EngineError(PP_ERR_NUMERICAL, "non-finite coefficient (sharded)");
    gmax_ = __builtin_bit_cast(double, (uint64_t)v[0]);
    eng_->set_global_max(gmax_);
    if (truncate) eng_->truncate_threshold(cfg_.epsilon0 * gmax_);
  }

  pp_config cfg_;
  std::unique_ptr<Collective> coll_;
  std::unique_ptr<EngineBase> eng_;
  std::vector<uint16_t> table_;
  DevBuf recv_buf_;
  double gmax_ = 0.0;
  pp_shard_stats stats_{};
};

}  // namespace ppgpu
