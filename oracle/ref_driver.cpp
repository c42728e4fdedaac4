// ref_driver.cpp -- C-ABI harness around the UNMODIFIED reference engine.
//
// TEST INFRASTRUCTURE ONLY.  This file is compiled together with the
// reference's own engine-core sources, in place under
// /root/reference/proj/src (see oracle/build_ref.sh), into
// oracle/_ref/libppref.so.  Only tests/, __graft_entry__.smoke() and
// bench.py (cpu_baseline leg, --impl reference) may load it, and only as the
// checker / CPU baseline -- never as the product path.
//
// Everything below drives the reference through its public C++ API:
//   Engine(EngineConfig)            engine.hpp:131-139
//   Engine::set_initial             engine.hpp:145-146 / engine.cpp:196-205
//   Engine::apply_gate              engine.hpp:150     / engine.cpp:277-316
//   Engine::truncate_now            engine.cpp:318-351
//   run_circuit                     engine.hpp:221-222 / engine.cpp:394-446
//   Gate(PauliString, Angle)        circuit.cpp:89-93
//   Angle::from_pi_units/radians    circuit.cpp:42-55
// No reference source is copied into this repository.

#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "pauliprop/circuit.hpp"
#include "pauliprop/engine.hpp"
#include "pauliprop/models.hpp"
#include "pauliprop/partition.hpp"
#include "pauliprop/pauli_string.hpp"
#include "pauliprop/sparse_operator.hpp"

using namespace pauliprop;

namespace {

thread_local std::string g_error;

enum : int { kOk = 0, kInvalid = 2, kNumerical = 3, kResource = 4, kOther = 5 };

int map_exception() {
  try {
    throw;
  } catch (const NumericalError& e) {
    g_error = e.what();
    return kNumerical;
  } catch (const ResourceLimitError& e) {
    g_error = e.what();
    return kResource;
  } catch (const std::bad_alloc& e) {
    g_error = "bad_alloc";
    return kResource;
  } catch (const std::invalid_argument& e) {
    g_error = e.what();
    return kInvalid;
  } catch (const std::exception& e) {
    g_error = e.what();
    return kOther;
  }
}

PauliString from_words(const uint64_t* w) {
  PauliString s;
  for (int i = 0; i < kIndexWords; ++i) s.words[i] = w[i];
  return s;
}

Gate make_gate(const uint64_t* words, double theta, int pi_units) {
  Angle a = pi_units ? Angle::from_pi_units(theta) : Angle::from_radians(theta);
  return Gate(from_words(words), a);
}

struct Handle {
  Engine engine;
  explicit Handle(const EngineConfig& c) : engine(c) {}
};

}  // namespace

extern "C" {

const char* ppref_last_error() { return g_error.c_str(); }

void* ppref_create(int n, uint32_t workers, int threads, double epsilon0,
                   int cadence, uint64_t max_terms) {
  try {
    EngineConfig config;
    config.n = n;
    config.partition = PartitionSpec::make(
        workers, PartitionSpec::default_block_size(workers));
    config.policy.epsilon0 = epsilon0;
    config.policy.cadence =
        cadence == 1 ? TruncationCadence::PerLayer : TruncationCadence::PerGate;
    config.threads = threads;
    config.max_terms = max_terms;
    return new Handle(config);
  } catch (...) {
    map_exception();
    return nullptr;
  }
}

void ppref_destroy(void* h) { delete static_cast<Handle*>(h); }

int ppref_set_initial(void* h, const uint64_t* words, const double* coeffs,
                      size_t count) {
  try {
    std::vector<std::pair<PauliString, double>> terms;
    terms.reserve(count);
    for (size_t i = 0; i < count; ++i) {
      terms.emplace_back(from_words(words + kIndexWords * i), coeffs[i]);
    }
    static_cast<Handle*>(h)->engine.set_initial(terms);
    return kOk;
  } catch (...) {
    return map_exception();
  }
}

int ppref_apply_gate(void* h, const uint64_t* words, double theta,
                     int pi_units) {
  try {
    static_cast<Handle*>(h)->engine.apply_gate(make_gate(words, theta, pi_units));
    return kOk;
  } catch (...) {
    return map_exception();
  }
}

int ppref_truncate_now(void* h) {
  try {
    static_cast<Handle*>(h)->engine.truncate_now();
    return kOk;
  } catch (...) {
    return map_exception();
  }
}

// Runs the reference's own run_circuit over `nlayers` layers given as a flat
// gate list (4 words + angle per gate) and per-layer sizes.  rows_out gets 8
// doubles per layer in LayerRecord order (engine.hpp:70-79).
int ppref_run_circuit(void* h, int n, const uint64_t* words,
                      const double* theta, const int* pi_units,
                      const int64_t* layer_sizes, int nlayers,
                      double* rows_out) {
  try {
    Circuit circuit;
    circuit.n = n;
    size_t g = 0;
    for (int l = 0; l < nlayers; ++l) {
      std::vector<Gate> layer;
      for (int64_t k = 0; k < layer_sizes[l]; ++k, ++g) {
        layer.push_back(make_gate(words + kIndexWords * g, theta[g], pi_units[g]));
      }
      circuit.layers.push_back(std::move(layer));
    }
    RunLedger ledger = run_circuit(static_cast<Handle*>(h)->engine, circuit);
    for (size_t r = 0; r < ledger.rows.size(); ++r) {
      const LayerRecord& row = ledger.rows[r];
      double* o = rows_out + 8 * r;
      o[0] = row.t;
      o[1] = row.observable;
      o[2] = double(row.term_count);
      o[3] = row.global_max;
      o[4] = double(row.removed);
      o[5] = row.wall_ms_per_gate;
      o[6] = double(row.batches_sent);
      o[7] = double(row.records_sent);
    }
    return kOk;
  } catch (...) {
    return map_exception();
  }
}

// Same Heisenberg loop as run_circuit (engine.cpp:412-427) but timed as a
// whole and counting string-gates = sum over gates of |O| entering the gate.
// Used as the reference CPU baseline for bench.py.
int ppref_time_circuit(void* h, int n, const uint64_t* words,
                       const double* theta, const int* pi_units,
                       const int64_t* layer_sizes, int nlayers,
                       double* seconds_out, double* string_gates_out) {
  try {
    (void)n;
    std::vector<std::vector<Gate>> layers;
    size_t g = 0;
    for (int l = 0; l < nlayers; ++l) {
      std::vector<Gate> layer;
      for (int64_t k = 0; k < layer_sizes[l]; ++k, ++g) {
        layer.push_back(make_gate(words + kIndexWords * g, theta[g], pi_units[g]));
      }
      layers.push_back(std::move(layer));
    }
    Engine& engine = static_cast<Handle*>(h)->engine;
    double sg = 0.0;
    auto start = std::chrono::steady_clock::now();
    for (int t = 1; t <= nlayers; ++t) {
      const auto& layer = layers[nlayers - t];
      for (auto it = layer.rbegin(); it != layer.rend(); ++it) {
        sg += double(engine.term_count());
        engine.apply_gate(*it);
      }
      if (engine.config().policy.cadence == TruncationCadence::PerLayer) {
        engine.truncate_now();
      }
    }
    *seconds_out = std::chrono::duration<double>(
                       std::chrono::steady_clock::now() - start).count();
    *string_gates_out = sg;
    return kOk;
  } catch (...) {
    return map_exception();
  }
}

uint64_t ppref_term_count(void* h) {
  return static_cast<Handle*>(h)->engine.term_count();
}

// Engine::shard_sizes (engine.hpp:162): strings per worker shard.
int ppref_shard_sizes(void* h, uint64_t* out, int cap) {
  std::vector<size_t> sz = static_cast<Handle*>(h)->engine.shard_sizes();
  int k = 0;
  for (; k < cap && k < (int)sz.size(); ++k) out[k] = sz[k];
  return k;
}

double ppref_global_max(void* h) {
  return static_cast<Handle*>(h)->engine.global_max();
}

double ppref_expectation(void* h) {
  return static_cast<Handle*>(h)->engine.expectation_zero_state();
}

// Copies every live term (all shards, shard order) into words/coeffs.
// Returns the number written or -1 if cap is too small.
int64_t ppref_export(void* h, uint64_t* words, double* coeffs, uint64_t cap) {
  const Engine& engine = static_cast<Handle*>(h)->engine;
  uint64_t total = engine.term_count();
  if (total > cap) return -1;
  uint64_t k = 0;
  for (const SparseOperator& shard : engine.shards()) {
    auto keys = shard.store().keys();
    auto values = shard.store().values();
    for (size_t i = 0; i < keys.size(); ++i, ++k) {
      std::memcpy(words + kIndexWords * k, keys[i].words.data(),
                  sizeof(uint64_t) * kIndexWords);
      coeffs[k] = values[i];
    }
  }
  return static_cast<int64_t>(k);
}

double ppref_coefficient(void* h, const uint64_t* words) {
  return static_cast<Handle*>(h)->engine.coefficient(from_words(words));
}

// Label parsing through the reference (pauli_string.cpp:105-177).
int ppref_parse_label(const char* text, int n, uint64_t* words_out) {
  try {
    PauliString s = parse_pauli_label(text, n);
    for (int i = 0; i < kIndexWords; ++i) words_out[i] = s.words[i];
    return kOk;
  } catch (...) {
    return map_exception();
  }
}

int ppref_phase_exponent(const uint64_t* a, const uint64_t* b, int n) {
  return phase_exponent(from_words(a), from_words(b), n);
}

// Angle trig through the reference (circuit.cpp:28-63).
void ppref_angle(double value, int pi_units, double* cos_out, double* sin_out,
                 double* radians_out) {
  Angle a = pi_units ? Angle::from_pi_units(value) : Angle::from_radians(value);
  *cos_out = a.cosine();
  *sin_out = a.sine();
  *radians_out = a.radians;
}

// Bundled heavy-hex geometry (heavy_hex_data.cpp, models.cpp:120).
int ppref_heavy_hex(int* edges_out, int* colors_out, int cap) {
  Geometry g = heavy_hex_127();
  if (static_cast<int>(g.edges.size()) > cap) return -1;
  for (size_t e = 0; e < g.edges.size(); ++e) {
    edges_out[2 * e] = g.edges[e].first;
    edges_out[2 * e + 1] = g.edges[e].second;
    colors_out[e] = g.edge_colors[e];
  }
  return static_cast<int>(g.edges.size());
}

// kicked_ising_layer gate order (models.cpp:149-171) for a geometry given as
// text: writes 4 words per gate; returns the gate count or -1.
int ppref_kicked_layer(const char* geometry_text, uint64_t* words_out,
                       int* is_zz_out, int cap) {
  try {
    Geometry g = load_geometry_text(geometry_text);
    std::vector<Gate> layer = kicked_ising_layer(
        g, Angle::from_radians(0.1), Angle::from_pi_units(-0.5));
    if (static_cast<int>(layer.size()) > cap) return -1;
    for (size_t i = 0; i < layer.size(); ++i) {
      for (int w = 0; w < kIndexWords; ++w) {
        words_out[kIndexWords * i + w] = layer[i].generator.words[w];
      }
      is_zz_out[i] = pauli_weight(layer[i].generator) == 2;
    }
    return static_cast<int>(layer.size());
  } catch (...) {
    map_exception();
    return -1;
  }
}

// density_histogram(shards, global_max, bins, epsilon0).to_tsv()
// (sparse_operator.cpp:136-197).  Returns the TSV length, -1 on error, or
// -(needed + 2) when cap is too small.
int64_t ppref_histogram_tsv(void* h, int bins, double epsilon0, char* buf, uint64_t cap) {
  try {
    const Engine& engine = static_cast<Handle*>(h)->engine;
    std::string tsv =
        density_histogram(engine.shards(), engine.global_max(), bins, epsilon0).to_tsv();
    if (tsv.size() + 1 > cap) return -static_cast<int64_t>(tsv.size() + 3);
    std::memcpy(buf, tsv.c_str(), tsv.size() + 1);
    return static_cast<int64_t>(tsv.size());
  } catch (...) {
    map_exception();
    return -1;
  }
}

// SparseOperator::dump of every shard in shard order (sparse_operator.cpp:99-106),
// i.e. the concatenation of the reference's checkpoint shard files.
int64_t ppref_dump(void* h, char* buf, uint64_t cap) {
  std::ostringstream out;
  for (const SparseOperator& shard : static_cast<Handle*>(h)->engine.shards()) shard.dump(out);
  std::string text = out.str();
  if (text.size() + 1 > cap) return -static_cast<int64_t>(text.size() + 3);
  std::memcpy(buf, text.c_str(), text.size() + 1);
  return static_cast<int64_t>(text.size());
}

// SparseOperator::load_dump (sparse_operator.cpp:108-122) -> words/coeffs.
int64_t ppref_load_dump(const char* text, int n, uint64_t* words, double* coeffs, uint64_t cap) {
  try {
    std::istringstream in(text);
    SparseOperator op = SparseOperator::load_dump(in, n);
    auto keys = op.store().keys();
    auto values = op.store().values();
    if (keys.size() > cap) return -1;
    for (size_t i = 0; i < keys.size(); ++i) {
      std::memcpy(words + kIndexWords * i, keys[i].words.data(), sizeof(uint64_t) * kIndexWords);
      coeffs[i] = values[i];
    }
    return static_cast<int64_t>(keys.size());
  } catch (...) {
    map_exception();
    return -1;
  }
}

}  // extern "C"
