/*
 * pauliprop_gpu.h -- C-ABI of the B200 Pauli-propagation engine.
 *
 * This is the drop-in boundary for the reference's hot path
 * (SURVEY.md section 8b).  Each entry point replaces one call of the
 * reference's C++ operator/gate API (namespace pauliprop):
 *
 *   pp_create / pp_destroy      Engine::Engine(const EngineConfig&), ~Engine
 *                               (reference include/pauliprop/engine.hpp:131-139,
 *                                src/engine.cpp:167-190)
 *   pp_set_initial              Engine::set_initial  (engine.hpp:145-146,
 *                                engine.cpp:196-205)
 *   pp_apply_gate               Engine::apply_gate   (engine.hpp:150,
 *                                engine.cpp:277-316), including the per-gate
 *                                truncation at cadence 0 (engine.cpp:313-315)
 *   pp_apply_gates              a run of Engine::apply_gate calls in order
 *                                (the inner loop of run_circuit,
 *                                engine.cpp:414-418); lets the engine fuse
 *                                runs of Clifford gates bit-exactly
 *   pp_truncate_now             Engine::truncate_now (engine.cpp:318-351)
 *   pp_term_count               Engine::term_count   (engine.cpp:353-357)
 *   pp_global_max               Engine::global_max   (engine.hpp:158)
 *   pp_expectation_zero_state   Engine::expectation_zero_state
 *                                (engine.cpp:359-361, sparse_operator.cpp:89-97)
 *   pp_coefficient              Engine::coefficient  (engine.cpp:363-366)
 *   pp_export                   Engine::merged       (engine.cpp:375-386),
 *                                returned sorted by key
 *   pp_take_counters            Engine::take_counters (engine.hpp:171-178)
 *
 * Pauli strings cross this boundary in the reference's own packed layout
 * (pauli_string.hpp:28-38): 4 x uint64 per string, site i in bits
 * (2i, 2i+1) counted from the least significant end of word i/32,
 * I=00 X=01 Y=10 Z=11, unused high bits zero.  Gate trig is computed on the
 * host exactly as Gate::Gate does (circuit.cpp:89-93) and passed in.
 *
 * Return codes map onto the reference's exceptions:
 *   0 ok
 *   2 invalid argument   (std::invalid_argument)
 *   3 numerical          (pauliprop::NumericalError, engine.cpp:333-339)
 *   4 resource           (pauliprop::ResourceLimitError, engine.cpp:269-273,
 *                         or device memory exhausted -> std::bad_alloc)
 *   5 internal CUDA error (std::runtime_error)
 * pp_last_error() returns the message of the last failure on the engine.
 *
 * Threading: one caller thread per engine, like the reference Engine
 * (not re-entrant).  All entry points are synchronous with respect to the
 * results they return.
 */
#ifndef PAULIPROP_GPU_H
#define PAULIPROP_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PP_OK 0
#define PP_ERR_INVALID 2
#define PP_ERR_NUMERICAL 3
#define PP_ERR_RESOURCE 4
#define PP_ERR_INTERNAL 5

#define PP_CADENCE_GATE 0
#define PP_CADENCE_LAYER 1

/* pp_config.flags */
#define PP_FLAG_NO_CLIFFORD_FUSION 1u /* apply Clifford gates one by one */
#define PP_FLAG_PROFILE 2u            /* no CUDA graphs; time every branch launch */
#define PP_FLAG_EXTERNAL_TRUNCATION 4u /* never truncate or check the budget itself: a
                                          sharded orchestrator calls pp_truncate_threshold
                                          with the global threshold */

typedef struct pp_engine pp_engine;

/* EngineConfig (engine.hpp:99-106) minus the thread pool: worker_count is
 * kept for ledger accounting only -- results never depend on it
 * (test_engine.cpp:211-258). */
typedef struct {
  int n;               /* qubits, 1..128 */
  double epsilon0;     /* relative truncation threshold, >= 0 */
  int cadence;         /* PP_CADENCE_GATE or PP_CADENCE_LAYER */
  uint64_t max_terms;  /* 0 = unlimited */
  uint32_t workers;    /* logical workers (ledger only) */
  int device;          /* CUDA device ordinal */
  uint32_t flags;      /* PP_FLAG_* */
  double mem_fraction; /* share of free device memory the engine may use (0 = default 0.9) */
} pp_config;

/* Gate (circuit.hpp:46-54): generator in the packed layout + host trig. */
typedef struct {
  uint64_t words[4];
  double theta;
  double cos_theta;
  double sin_theta;
} pp_gate;

/* Engine::Counters (engine.hpp:171-178), nanoseconds split by phase. */
typedef struct {
  uint64_t removed;
  uint64_t batches_sent;
  uint64_t records_sent;
  uint64_t gates;
  uint64_t branch_ns;   /* branch+merge kernels (generate+apply) */
  uint64_t exchange_ns; /* regroup / reshuffle after Clifford runs */
  uint64_t truncate_ns; /* max-reduce + truncation */
  uint64_t other_ns;
} pp_counters;

int pp_create(const pp_config* config, pp_engine** out);
void pp_destroy(pp_engine* engine);
int pp_set_initial(pp_engine* engine, const uint64_t* words, const double* coeffs, size_t count);
int pp_apply_gate(pp_engine* engine, const pp_gate* gate);
int pp_apply_gates(pp_engine* engine, const pp_gate* gates, size_t count);

/* One layer of run_circuit (engine.cpp:394-446) with a zero-state readout:
 * pp_apply_gates followed by pp_expectation_zero_state, sharing one device
 * round trip (errors surface here exactly as from pp_apply_gates). */
int pp_apply_layer(pp_engine* engine, const pp_gate* gates, size_t count, double* observable);
int pp_truncate_now(pp_engine* engine);
int pp_term_count(const pp_engine* engine, uint64_t* out);
int pp_global_max(const pp_engine* engine, double* out);
int pp_expectation_zero_state(pp_engine* engine, double* out);
int pp_coefficient(pp_engine* engine, const uint64_t* words, double* out);
/* Copies every live term, sorted ascending by the packed words (word 3 most
 * significant).  cap = capacity of words (4*cap uint64) and coeffs. */
int pp_export(pp_engine* engine, uint64_t* words, double* coeffs, uint64_t cap, uint64_t* count);
int pp_take_counters(pp_engine* engine, pp_counters* out);
const char* pp_last_error(const pp_engine* engine);

/* Device time (ms) of the branch+merge kernel launches since the last call,
 * with the algorithmic bytes they moved; for the roofline in bench.py. */
int pp_take_kernel_stats(pp_engine* engine, double* branch_ms, double* branch_bytes,
                         uint64_t* branch_launches, uint64_t* total_launches);

/* The CUDA stream (cudaStream_t) the engine launches on, so callers can
 * bracket work with their own events. */
void* pp_stream(const pp_engine* engine);

/* Process-wide host<->device byte totals over every engine since load:
 * explicit copies plus kernel parameter blocks carrying host data (gate
 * lists, initial terms).  Callers difference two readings. */
void pp_transfer_totals(uint64_t* h2d_bytes, uint64_t* d2h_bytes);

/* ---- sharding (one engine per GPU; the orchestrator owns the collectives).
 * owner(z) = pp_shard_owner: a hash of the string's z-plane.  An Rx gate keeps
 * z, so it never moves strings between shards; after a Clifford/ZZ run or a
 * Z/Y-carrying gate, pp_shard_evict removes every z-group owned elsewhere and
 * returns it as records [x words, z words, coefficient bits] (pp_record_words
 * words each) grouped by destination rank; the receiver merges them with
 * pp_shard_ingest (equal keys combine exactly like TermMap::add).  The
 * reference's distribution is the block-sum map (partition.cpp:53-59) over
 * in-process workers (engine.hpp:126-130); results never depend on it. */
int pp_local_stats(pp_engine* engine, double* gmax, uint32_t* nonfinite, uint64_t* count);
int pp_truncate_threshold(pp_engine* engine, double threshold, uint64_t* removed);
int pp_record_words(const pp_engine* engine);
int pp_shard_evict(pp_engine* engine, uint32_t world, uint32_t rank, uint64_t seed, uint64_t* records,
                   uint64_t cap, uint64_t* counts);
int pp_shard_ingest(pp_engine* engine, const uint64_t* records, uint64_t count);
uint32_t pp_shard_owner(const uint64_t* words, int n, uint64_t seed, uint32_t world);

/* Device-resident exchange (NCCL / NVLink): pp_shard_evict_device leaves the
 * records in an engine-owned device buffer (*records, valid until the next
 * call on this engine) grouped by destination; pp_shard_ingest_device takes
 * records from device memory on the engine's device (e.g. an NCCL all-to-all
 * receive buffer), with the stream work that produced them complete. */
int pp_shard_evict_device(pp_engine* engine, uint32_t world, uint32_t rank, uint64_t seed, const uint64_t** records,
                          uint64_t* counts);
int pp_shard_ingest_device(pp_engine* engine, const uint64_t* records, uint64_t count);

/* Sum of squared coefficients (conserved at epsilon0 = 0; property checks at
 * sizes the oracle cannot reach). */
int pp_norm2(pp_engine* engine, double* out);

/* Diagnostics: the operator's z-groups (strings sharing a z-plane) by size,
 * log2 bins: groups[b] and strings[b] count groups of [2^b, 2^(b+1))
 * strings (64 entries each). */
int pp_group_sizes(pp_engine* engine, uint64_t* groups, uint64_t* strings);

/* Log-binned coefficient density with a sign split, the reference's
 * density_histogram (sparse_operator.cpp:150-197, written per layer by
 * runner.cpp:173-179): edges exp(log(lower) * (1 - b/bins)), lower =
 * max(epsilon0, 1e-16), x = c / global_max.  Writes exact integer counts per
 * bin (positive[bins], negative[bins]); the reference's normalized values are
 * sums of 1/total over those counts.  1 <= bins <= 4096.  PP_ERR_INVALID if
 * the operator is nonempty and global_max <= 0 (sparse_operator.cpp:156-160). */
int pp_density_histogram(pp_engine* engine, int bins, double global_max, double epsilon0, uint64_t* positive,
                         uint64_t* negative);

/* ---- native sharded engine: one rank per GPU, SPMD, NCCL inside
 * (the multi-GPU form of Engine).  Ownership is a
 * z-plane hash into 4096 buckets, rebalanced from the global bucket
 * histogram at every exchange; Rx runs are rank-local; strings move with one
 * all-to-all after each Clifford/ZZ step; eps0 > 0 runs reduce their
 * per-gate maxima over the ranks once per run.  Every rank calls every entry
 * point in the same order (collective calls).
 *
 * Bootstrap: rank 0 calls pp_nccl_unique_id and hands the 128 bytes to every
 * rank out of band (MPI, a store, a file); each rank then calls
 * pp_sharded_create with its device in config->device.  pp_hub_create makes
 * an in-process transport instead (ranks as threads of one process sharing
 * one device; for tests). */
typedef struct pp_sharded pp_sharded;
typedef struct pp_hub pp_hub;
typedef struct {
  uint64_t exchanges;     /* string exchanges so far */
  uint64_t records_moved; /* strings this rank sent */
  uint64_t exchange_ns;   /* wall time in exchanges (rebalance + all-to-all + ingest) */
  double balance;         /* max / min strings per rank after the last rebalance */
} pp_shard_stats;

int pp_nccl_unique_id(uint8_t id[128]);
int pp_sharded_create(const pp_config* config, int world, int rank, const uint8_t id[128], pp_sharded** out);
pp_hub* pp_hub_create(int world);
void pp_hub_destroy(pp_hub* hub);
int pp_sharded_create_hub(const pp_config* config, pp_hub* hub, int rank, pp_sharded** out);
void pp_sharded_destroy(pp_sharded* s);
/* every rank passes the same terms; each keeps those it owns */
int pp_sharded_set_initial(pp_sharded* s, const uint64_t* words, const double* coeffs, size_t count);
int pp_sharded_apply_gates(pp_sharded* s, const pp_gate* gates, size_t count);
/* one run_circuit layer (gates in application order) + the global <0|O|0> */
int pp_sharded_apply_layer(pp_sharded* s, const pp_gate* gates, size_t count, double* observable);
int pp_sharded_truncate_now(pp_sharded* s);
int pp_sharded_term_count(pp_sharded* s, uint64_t* out);
int pp_sharded_global_max(pp_sharded* s, double* out);
int pp_sharded_take_counters(pp_sharded* s, pp_counters* out); /* removed/batches/records summed over ranks */
int pp_sharded_stats(pp_sharded* s, pp_shard_stats* out);
/* this rank's strings (sorted), for checkpoints and tests */
int pp_sharded_local_count(pp_sharded* s, uint64_t* out);
int pp_sharded_local_export(pp_sharded* s, uint64_t* words, double* coeffs, uint64_t cap, uint64_t* count);
void* pp_sharded_stream(const pp_sharded* s);
/* this rank's branch-kernel device time and algorithmic bytes (pp_take_kernel_stats) */
int pp_sharded_kernel_stats(pp_sharded* s, double* branch_ms, double* branch_bytes, uint64_t* branch_launches,
                            uint64_t* total_launches);
const char* pp_sharded_last_error(const pp_sharded* s);

#ifdef __cplusplus
}
#endif

#endif /* PAULIPROP_GPU_H */
