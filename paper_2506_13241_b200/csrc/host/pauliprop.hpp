// pauliprop.hpp -- host-side C++ API of the B200 engine.
//
// Mirrors the reference's public C++ surface (namespace pauliprop,
// SURVEY.md section 8b) so callers of the reference compile against it
// unchanged: PauliString (pauli_string.hpp:37-63), Angle/Gate/Circuit
// (circuit.hpp:30-71), Geometry/kicked-Ising builders (models.hpp:29-63),
// EngineConfig/Engine/run_circuit (engine.hpp:99-222).  The Engine forwards
// every hot-path call through the C-ABI in include/pauliprop_gpu.h; nothing
// here touches coefficients except for host conversions.
#pragma once

#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <span>
#include <vector>

struct pp_engine;

namespace pauliprop {

constexpr int kMaxQubits = 128;
constexpr int kIndexWords = (2 * kMaxQubits) / 64;

enum class Pauli : uint8_t { I = 0, X = 1, Y = 2, Z = 3 };

// 2 bits per site, site i in bits (2i, 2i+1): the reference's normative
// layout (pauli_string.hpp:28-38), kept so keys cross the API unchanged.
struct PauliString {
  std::array<uint64_t, kIndexWords> words{};
  bool operator==(const PauliString&) const = default;
  bool is_identity() const {
    uint64_t a = 0;
    for (uint64_t w : words) a |= w;
    return a == 0;
  }
  uint8_t code_at(int site) const { return static_cast<uint8_t>((words[site >> 5] >> (2 * (site & 31))) & 3u); }
  void set_code(int site, uint8_t code) {
    uint64_t& w = words[site >> 5];
    int sh = 2 * (site & 31);
    w = (w & ~(uint64_t{3} << sh)) | (uint64_t{code} << sh);
  }
  PauliString operator^(const PauliString& o) const {
    PauliString r;
    for (int i = 0; i < kIndexWords; ++i) r.words[i] = words[i] ^ o.words[i];
    return r;
  }
};

PauliString single_site(int site, Pauli pauli);
uint64_t hash_string(const PauliString& s);
int local_phase(uint8_t a, uint8_t b);
int phase_exponent(const PauliString& I, const PauliString& J, int n);
bool commutes(const PauliString& I, const PauliString& J, int n);
struct StringProduct {
  PauliString index;
  int phase;
};
StringProduct string_product(const PauliString& I, const PauliString& J, int n);
int pauli_weight(const PauliString& s);
PauliString parse_pauli_label(const std::string& text, int n);
std::string to_dense_label(const PauliString& s, int n);
std::string to_sparse_label(const PauliString& s, int n);
std::string to_hex(const PauliString& s, int n);
PauliString from_hex(const std::string& hex, int n);

// ---------------------------------------------------------------- circuits
struct Angle {
  double radians = 0.0;
  bool in_pi_units = false;
  double pi_units = 0.0;
  static Angle from_radians(double r);
  static Angle from_pi_units(double r);
  double cosine() const;
  double sine() const;
};
Angle parse_angle(const std::string& text);

struct Gate {
  PauliString generator;
  double theta = 0.0;
  double cos_theta = 1.0;
  double sin_theta = 0.0;
  Gate() = default;
  Gate(const PauliString& generator, Angle angle);
};

struct Circuit {
  int n = 0;
  std::vector<std::vector<Gate>> layers;
  size_t total_gates() const;
};
Circuit parse_circuit_text(const std::string& text, int n);
std::string format_circuit(const Circuit& circuit);

// ---------------------------------------------------------------- models
struct Geometry {
  int n = 0;
  std::vector<std::pair<int, int>> edges;
  std::vector<int> edge_colors;
  int color_count = 0;
  bool has_coloring() const { return !edge_colors.empty(); }
};
Geometry load_geometry_text(const std::string& text);
Geometry load_geometry_file(const std::string& path);
// The reference's bundled 127-qubit heavy-hex map (models.cpp:120): same
// edges, colours and edge order, hence the same kicked-Ising gate order.
Geometry heavy_hex_127();
std::vector<int> bfs_ball(const Geometry& geom, int start, int radius);
std::vector<Gate> kicked_ising_layer(const Geometry& geom, Angle theta_x, Angle theta_zz);
Circuit build_kicked_ising(const Geometry& geom, Angle theta_x, Angle theta_zz, int layers);

// ---------------------------------------------------------------- partition
// Kept for EngineConfig compatibility and ledger accounting; the GPU engine's
// results never depend on it (test_engine.cpp:211-258).
struct PartitionSpec {
  uint32_t worker_count = 1;
  uint32_t block_size_bits = 1;
  uint32_t perturbation_s = 1;
  static uint32_t default_block_size(uint32_t workers);
  static PartitionSpec make(uint32_t workers, uint32_t block_size_bits, uint32_t perturbation_s = 1);
};
uint64_t block_sum(const PauliString& index, int n, uint32_t block_size_bits);
uint32_t owner(const PartitionSpec& spec, const PauliString& index, int n);
double uniformity_ratio(const std::vector<size_t>& shard_sizes);
// Owners that can receive a record from worker m for generator J
// (partition.cpp:61-108): every worker when the map is perturbed.
std::vector<uint32_t> destination_set(const PartitionSpec& spec, uint32_t m, const PauliString& J, int n);

// Dense check: <0|U^dag O U|0> by forward state-vector evolution from |0..0>
// (the reference's oracle::evolve_state / expectation, n <= 26).
double state_vector_expectation(const Circuit& circuit, const PauliString& observable);

// ---------------------------------------------------------------- engine
enum class TruncationCadence { PerGate, PerLayer };
struct TruncationPolicy {
  double epsilon0 = 0.0;
  TruncationCadence cadence = TruncationCadence::PerGate;
};

struct LayerRecord {
  int t = 0;
  double observable = 0.0;
  uint64_t term_count = 0;
  double global_max = 0.0;
  uint64_t removed = 0;
  double wall_ms_per_gate = 0.0;
  uint64_t batches_sent = 0;
  uint64_t records_sent = 0;
};

struct RunLedger {
  std::vector<LayerRecord> rows;
  static const char* csv_header();
  static std::string csv_row(const LayerRecord& row);
  std::string to_csv() const;
};

struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ResourceLimitError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct EngineConfig {
  int n = 1;
  PartitionSpec partition;
  TruncationPolicy policy;
  int threads = 0;         // accepted for compatibility; the GPU ignores it
  uint64_t max_terms = 0;  // 0 = unlimited
  bool collect_gate_stats = false;
  int device = 0;
  bool fuse_clifford = true;
  bool profile = false;  // no CUDA graphs, per-launch kernel timing
  bool external_truncation = false;  // sharded: the orchestrator truncates with a global threshold
};

// Host copy of the operator (what Engine::merged() returns).
struct SparseOperator {
  int n = 1;
  std::vector<PauliString> keys;  // sorted ascending (word 3 most significant)
  std::vector<double> values;
  size_t term_count() const { return keys.size(); }
  double coefficient(const PauliString& index) const;
  double expectation_zero_state() const;
};

class Engine {
 public:
  explicit Engine(const EngineConfig& config);
  ~Engine();
  Engine(const Engine&) = delete;
  Engine& operator=(const Engine&) = delete;
  Engine(Engine&&) noexcept;
  Engine& operator=(Engine&&) noexcept;

  int num_qubits() const { return config_.n; }
  const EngineConfig& config() const { return config_; }

  void set_initial(const std::vector<std::pair<PauliString, double>>& terms);
  void apply_gate(const Gate& gate);
  void apply_gates(const std::vector<Gate>& gates);  // in order; fuses Clifford runs
  double apply_layer(const std::vector<Gate>& gates);  // apply_gates + expectation_zero_state, one round trip
  void truncate_now();

  uint64_t term_count() const;
  double global_max() const;
  double expectation_zero_state() const;
  double coefficient(const PauliString& index) const;
  SparseOperator merged() const;
  // Host mirror of the reference's per-worker shards (engine.hpp:161-162):
  // the operator split by the block-sum owner map of config().partition,
  // each shard sorted.  Built on first use, invalidated by every change.
  std::span<const SparseOperator> shards() const;
  std::vector<size_t> shard_sizes() const;

  // engine.hpp:109-118.  The GPU fuses generate and apply into one branch
  // kernel: generate_ns carries the branch+merge time, exchange_ns the
  // regroups after Clifford/ZZ runs, truncate_ns the reductions and
  // truncation, apply_ns the rest of the device time.
  struct PhaseTimers {
    uint64_t generate_ns = 0;
    uint64_t exchange_ns = 0;
    uint64_t apply_ns = 0;
    uint64_t truncate_ns = 0;
    uint64_t total_ns() const { return generate_ns + exchange_ns + apply_ns + truncate_ns; }
  };
  struct Counters {
    uint64_t removed = 0;
    uint64_t batches_sent = 0;
    uint64_t records_sent = 0;
    uint64_t gates = 0;
    uint64_t total_ns = 0;
    PhaseTimers timers;
  };
  Counters take_counters();
  void set_layer_context(int t) { layer_context_ = t; }
  pp_engine* handle() const { return handle_; }

  void check(int rc) const;  // C-ABI return code -> the reference's exception types

 private:
  EngineConfig config_;
  pp_engine* handle_ = nullptr;
  mutable std::vector<SparseOperator> shard_mirror_;
  mutable bool mirror_valid_ = false;
  void invalidate() const { mirror_valid_ = false; }
  int layer_context_ = 0;
};

enum class ReadoutMode { ZeroState, TrackedCoefficient };

struct RunOptions {
  ReadoutMode readout = ReadoutMode::ZeroState;
  // Resume: layers t <= start_layer are already folded into the engine's
  // operator (loaded from checkpoint_t<start_layer>); propagation continues
  // at t = start_layer + 1.  The reference writes checkpoints but has no
  // resume path (runner.cpp:52-77, 180-183).
  int start_layer = 0;
  PauliString tracked_index;
  std::function<void(const LayerRecord&, const Engine&)> on_layer;
  std::function<void(int t, size_t gate_index, double value)> on_gate_readout;
};

// ------------------------------------------------------------ diagnostics and checkpoints
// Coefficient density, log-binned with a sign split (sparse_operator.hpp
// DensityHistogram, sparse_operator.cpp:150-197).  The GPU counts (exact
// integers, pp_density_histogram); positive/negative are the reference's
// normalized values: 1/total summed count times, in the same order of
// additions, so the TSV is byte-identical.
struct DensityHistogram {
  std::vector<double> bin_edges;
  std::vector<double> positive;
  std::vector<double> negative;
  std::vector<uint64_t> positive_counts;
  std::vector<uint64_t> negative_counts;
  uint64_t total_terms = 0;
  std::string to_tsv() const;  // sparse_operator.cpp:136-148
};
DensityHistogram histogram_from_counts(int bins, double epsilon0, const std::vector<uint64_t>& positive_counts,
                                       const std::vector<uint64_t>& negative_counts);
DensityHistogram density_histogram(const Engine& engine, int bins, double epsilon0);
DensityHistogram density_histogram(const Engine& engine, int bins, double epsilon0, double global_max);

// Shard dump: one "<hex index> <%.17g coefficient>" line per string
// (SparseOperator::dump/load_dump, sparse_operator.cpp:99-122).
void dump_operator(std::ostream& out, const SparseOperator& op);
SparseOperator load_dump(std::istream& in, int n);

// Checkpoint directory of runner.cpp:52-77: shard_<m>.txt (or the binary
// shard_<m>.ppb: "PPB1", n, count, count x 4 index words, count doubles) plus
// manifest.json {schema, layer, qubits, workers, ..., epsilon0, files}.
// read_checkpoint accepts the reference's own checkpoints (any worker count;
// duplicate keys across shards are added, which cannot happen for a valid
// sharding) and ours.
struct Checkpoint {
  int layer = 0;
  int qubits = 0;
  double epsilon0 = 0.0;
  SparseOperator op;
};
void write_shard_file(const std::string& path, const SparseOperator& op, bool binary);
void write_checkpoint_manifest(const std::string& dir, int layer, int qubits, double epsilon0,
                               const std::vector<std::pair<std::string, uint64_t>>& files);
void write_checkpoint(const std::string& dir, const Engine& engine, int layer, bool binary = false);
Checkpoint read_checkpoint(const std::string& dir);

// Heisenberg loop of engine.cpp:394-446: layers last to first, gates in
// reverse order, optional per-layer truncation, readout after truncation.
RunLedger run_circuit(Engine& engine, const Circuit& circuit, const RunOptions& options = {});

}  // namespace pauliprop
