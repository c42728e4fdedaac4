/*
 * pp_oracle.c -- CPU restatement of the reference's Heisenberg-picture
 * Pauli-propagation step, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the parity checker for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load it.  It is never linked into, or called by, the product library.
 *
 * It restates, single-threaded and with one logical worker (results do not
 * depend on the worker count: test_engine.cpp:211-258), the algorithm of
 *   /root/reference/proj/src/engine.cpp        (generate/apply/truncate)
 *   /root/reference/proj/src/term_map.cpp      (store semantics)
 *   /root/reference/proj/src/sparse_operator.cpp (expectation, max)
 *   /root/reference/proj/src/pauli_string.cpp  (phase table, labels)
 *   /root/reference/proj/src/circuit.cpp       (exact pi-unit trig)
 * Keys use the reference's interleaved 2-bit encoding (pauli_string.hpp:
 * 28-38): 4 x uint64, site i in bits (2i, 2i+1), I=00 X=01 Y=10 Z=11.
 *
 * Parity is pinned in tests/test_oracle.py against the reference compiled
 * from its own sources (oracle/_ref, built by oracle/build_ref.sh) and
 * against the golden values committed under tests/golden/.
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (see __graft_entry__.py).
 * -ffp-contract=off keeps every multiply and add a separate IEEE rounding,
 * as in the reference build.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PPO_WORDS 4
#define PPO_OK 0
#define PPO_INVALID 2
#define PPO_NUMERICAL 3
#define PPO_RESOURCE 4

typedef struct {
  uint64_t w[PPO_WORDS];
} ppo_key;

/* kLocalPhase, pauli_string.cpp:28-34: su(2) structure constants. */
static const int8_t kPhase[16] = {0, 0, 0, 0, 0, 0, 1, -1,
                                  0, -1, 0, 1, 0, 1, -1, 0};

/* mix64 / hash_string, pauli_string.cpp:36-41, 71-75 (used only to index
 * the open-addressing table; any hash would do for a restatement). */
static uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static uint64_t key_hash(const ppo_key* k) {
  uint64_t h = 0;
  for (int i = 0; i < PPO_WORDS; ++i) h = mix64(h ^ k->w[i]);
  return h;
}
static int key_eq(const ppo_key* a, const ppo_key* b) {
  return memcmp(a->w, b->w, sizeof(a->w)) == 0;
}
static int code_at(const ppo_key* k, int site) {
  return (int)((k->w[site >> 5] >> (2 * (site & 31))) & 3u);
}

/* Term store: dense key/value arrays + power-of-two linear-probe index, the
 * TermMap contract of term_map.hpp:36-111 (insertion appends; exact zeros
 * persist until a removal pass). */
typedef struct {
  ppo_key* keys;
  double* vals;
  int64_t* idx;
  size_t size, cap, mask;
} ppo_store;

static int store_reindex(ppo_store* s, size_t buckets) {
  int64_t* idx = (int64_t*)malloc(buckets * sizeof(int64_t));
  if (!idx) return PPO_RESOURCE;
  for (size_t b = 0; b < buckets; ++b) idx[b] = -1;
  for (size_t i = 0; i < s->size; ++i) {
    size_t b = key_hash(&s->keys[i]) & (buckets - 1);
    while (idx[b] >= 0) b = (b + 1) & (buckets - 1);
    idx[b] = (int64_t)i;
  }
  free(s->idx);
  s->idx = idx;
  s->mask = buckets - 1;
  return PPO_OK;
}

static int store_reserve(ppo_store* s, size_t n) {
  if (n > s->cap) {
    size_t cap = s->cap ? s->cap : 16;
    while (cap < n) cap *= 2;
    ppo_key* k = (ppo_key*)realloc(s->keys, cap * sizeof(ppo_key));
    if (!k) return PPO_RESOURCE;
    s->keys = k;
    double* v = (double*)realloc(s->vals, cap * sizeof(double));
    if (!v) return PPO_RESOURCE;
    s->vals = v;
    s->cap = cap;
  }
  if (s->idx == NULL || 2 * n > s->mask + 1) {
    size_t buckets = 16;
    while (buckets < 2 * n) buckets *= 2;
    return store_reindex(s, buckets);
  }
  return PPO_OK;
}

static int64_t store_find(const ppo_store* s, const ppo_key* k) {
  if (!s->idx) return -1;
  size_t b = key_hash(k) & s->mask;
  for (;;) {
    int64_t slot = s->idx[b];
    if (slot < 0) return -1;
    if (key_eq(&s->keys[slot], k)) return slot;
    b = (b + 1) & s->mask;
  }
}

/* TermMap::add, term_map.hpp:66-83: += into an existing slot, else append. */
static int store_add(ppo_store* s, const ppo_key* k, double delta) {
  int rc = store_reserve(s, s->size + 1);
  if (rc) return rc;
  size_t b = key_hash(k) & s->mask;
  for (;;) {
    int64_t slot = s->idx[b];
    if (slot < 0) {
      s->idx[b] = (int64_t)s->size;
      s->keys[s->size] = *k;
      s->vals[s->size] = delta;
      s->size++;
      return PPO_OK;
    }
    if (key_eq(&s->keys[slot], k)) {
      s->vals[slot] += delta;
      return PPO_OK;
    }
    b = (b + 1) & s->mask;
  }
}

/* TermMap::remove_below, term_map.cpp:105-144: drop every |v| <= threshold.
 * The reference's survivor order is an implementation detail; sets and
 * values are what parity compares. */
static size_t store_remove_below(ppo_store* s, double threshold) {
  size_t w = 0, removed = 0;
  for (size_t r = 0; r < s->size; ++r) {
    if (fabs(s->vals[r]) > threshold) {
      s->keys[w] = s->keys[r];
      s->vals[w] = s->vals[r];
      ++w;
    } else {
      ++removed;
    }
  }
  s->size = w;
  if (removed && s->idx) store_reindex(s, s->mask + 1);
  return removed;
}

typedef struct {
  int n;
  double epsilon0;
  int cadence; /* 0 per gate, 1 per layer (sparse_operator.hpp:27-37) */
  uint64_t max_terms;
  ppo_store store;
  double last_global_max;
  /* counters drained per layer (engine.hpp:171-178) */
  uint64_t removed, records, gates, gates_total, batches;
  /* scratch for the records of one gate */
  ppo_key* rec_keys;
  double* rec_vals;
  size_t rec_cap;
} ppo_engine;

ppo_engine* ppo_create(int n, double epsilon0, int cadence,
                       uint64_t max_terms) {
  if (n < 1 || n > 128 || !(epsilon0 >= 0)) return NULL;
  ppo_engine* e = (ppo_engine*)calloc(1, sizeof(ppo_engine));
  if (!e) return NULL;
  e->n = n;
  e->epsilon0 = epsilon0;
  e->cadence = cadence;
  e->max_terms = max_terms;
  return e;
}

void ppo_destroy(ppo_engine* e) {
  if (!e) return;
  free(e->store.keys);
  free(e->store.vals);
  free(e->store.idx);
  free(e->rec_keys);
  free(e->rec_vals);
  free(e);
}

static double store_max_abs(const ppo_store* s, int* nonfinite) {
  double mx = 0.0;
  int nan = 0;
  for (size_t i = 0; i < s->size; ++i) {
    double v = s->vals[i];
    nan |= (v != v);
    double av = fabs(v);
    if (av > mx) mx = av;
  }
  *nonfinite = nan || isinf(mx);
  return mx;
}

/* Engine::set_initial, engine.cpp:196-205 (upsert, so repeated keys add). */
int ppo_set_initial(ppo_engine* e, const uint64_t* words, const double* c,
                    size_t count) {
  e->store.size = 0;
  if (e->store.idx) store_reindex(&e->store, e->store.mask + 1);
  for (size_t i = 0; i < count; ++i) {
    ppo_key k;
    memcpy(k.w, words + PPO_WORDS * i, sizeof(k.w));
    int rc = store_add(&e->store, &k, c[i]);
    if (rc) return rc;
  }
  int nf;
  e->last_global_max = store_max_abs(&e->store, &nf);
  e->removed = e->records = e->gates = e->gates_total = e->batches = 0;
  return PPO_OK;
}

/* Engine::truncate_now, engine.cpp:318-351. */
int ppo_truncate_now(ppo_engine* e) {
  int nonfinite;
  double global = store_max_abs(&e->store, &nonfinite);
  if (nonfinite) return PPO_NUMERICAL;
  e->last_global_max = global;
  double threshold = e->epsilon0 * global; /* engine.cpp:345 */
  e->removed += store_remove_below(&e->store, threshold);
  return PPO_OK;
}

/* remove_below at an explicit threshold (a sharded run's global
 * epsilon0 * gmax); returns the removed count. */
uint64_t ppo_truncate_threshold(ppo_engine* e, double threshold) {
  size_t r = store_remove_below(&e->store, threshold);
  e->removed += r;
  return (uint64_t)r;
}

/* Engine::apply_gate, engine.cpp:277-316, with generate_phase (207-247)
 * and apply_phase (249-264) for a single worker. */
int ppo_apply_gate(ppo_engine* e, const uint64_t* gen, double cos_t,
                   double sin_t) {
  ppo_key J;
  memcpy(J.w, gen, sizeof(J.w));
  /* GatePrep support list, engine.cpp:51-54 */
  int sites[128], codes[128], ns = 0;
  for (int site = 0; site < e->n; ++site) {
    int c = code_at(&J, site);
    if (c) {
      sites[ns] = site;
      codes[ns] = c;
      ++ns;
    }
  }
  ppo_store* s = &e->store;
  size_t nrec = 0;
  size_t n0 = s->size;
  if (e->rec_cap < n0) {
    free(e->rec_keys);
    free(e->rec_vals);
    e->rec_keys = (ppo_key*)malloc((n0 ? n0 : 1) * sizeof(ppo_key));
    e->rec_vals = (double*)malloc((n0 ? n0 : 1) * sizeof(double));
    if (!e->rec_keys || !e->rec_vals) return PPO_RESOURCE;
    e->rec_cap = n0;
  }
  for (size_t i = 0; i < n0; ++i) {
    int phase = 0; /* phase_on_support, engine.cpp:75-81 */
    for (int k = 0; k < ns; ++k) {
      phase += kPhase[(code_at(&s->keys[i], sites[k]) << 2) | codes[k]];
    }
    if ((phase & 1) == 0) continue;
    double pre = s->vals[i];
    s->vals[i] = pre * cos_t; /* engine.cpp:223 */
    int m4 = ((phase % 4) + 4) % 4;
    double sign = m4 == 1 ? 1.0 : -1.0; /* record_sign, engine.cpp:71-73 */
    double delta = sign * sin_t * pre;  /* engine.cpp:224-225 */
    if (delta == 0.0) continue;         /* engine.cpp:226 */
    for (int w = 0; w < PPO_WORDS; ++w) {
      e->rec_keys[nrec].w[w] = s->keys[i].w[w] ^ J.w[w];
    }
    e->rec_vals[nrec] = delta;
    ++nrec;
  }
  for (size_t r = 0; r < nrec; ++r) {
    int rc = store_add(s, &e->rec_keys[r], e->rec_vals[r]);
    if (rc) return rc;
  }
  e->records += nrec;
  /* one worker: the (0, 0) outbox is one non-empty batch iff the gate sent a
     record (engine.cpp:286-301) */
  e->batches += nrec > 0;
  e->gates++;
  e->gates_total++;
  if (e->max_terms && s->size > e->max_terms) return PPO_RESOURCE;
  if (e->cadence == 0) return ppo_truncate_now(e);
  return PPO_OK;
}

uint64_t ppo_term_count(const ppo_engine* e) { return e->store.size; }
double ppo_global_max(const ppo_engine* e) { return e->last_global_max; }

/* is_diagonal + expectation_zero_state, sparse_operator.cpp:32-36, 89-97 */
double ppo_expectation(const ppo_engine* e) {
  double sum = 0.0;
  for (size_t i = 0; i < e->store.size; ++i) {
    uint64_t acc = 0;
    for (int w = 0; w < PPO_WORDS; ++w) {
      uint64_t v = e->store.keys[i].w[w];
      acc |= (v ^ (v >> 1)) & 0x5555555555555555ULL;
    }
    if (acc == 0) sum += e->store.vals[i];
  }
  return sum;
}

double ppo_coefficient(const ppo_engine* e, const uint64_t* words) {
  ppo_key k;
  memcpy(k.w, words, sizeof(k.w));
  int64_t slot = store_find(&e->store, &k);
  return slot < 0 ? 0.0 : e->store.vals[slot];
}

int64_t ppo_export(const ppo_engine* e, uint64_t* words, double* c,
                   uint64_t cap) {
  if (e->store.size > cap) return -1;
  for (size_t i = 0; i < e->store.size; ++i) {
    memcpy(words + PPO_WORDS * i, e->store.keys[i].w, sizeof(uint64_t) * 4);
    c[i] = e->store.vals[i];
  }
  return (int64_t)e->store.size;
}

/* density_histogram, sparse_operator.cpp:150-197, as exact counts per bin
 * (the reference sums 1/total per string; the caller normalizes).  Returns
 * PPO_INVALID for bins < 1 or a nonempty operator with gmax <= 0. */
int ppo_density_histogram(const ppo_engine* e, int bins, double gmax,
                          double epsilon0, uint64_t* pos, uint64_t* neg) {
  if (bins < 1) return PPO_INVALID;
  if (e->store.size > 0 && !(gmax > 0)) return PPO_INVALID;
  double lower = epsilon0 > 1e-16 ? epsilon0 : 1e-16;
  double log_lower = log(lower);
  for (int b = 0; b < bins; ++b) pos[b] = neg[b] = 0;
  for (size_t i = 0; i < e->store.size; ++i) {
    double x = e->store.vals[i] / gmax;
    double ax = fabs(x);
    int b;
    if (ax <= lower) {
      b = 0;
    } else if (ax >= 1.0) {
      b = bins - 1;
    } else {
      b = (int)(bins * (1.0 - log(ax) / log_lower));
      if (b < 0) b = 0;
      if (b > bins - 1) b = bins - 1;
    }
    if (x < 0) neg[b]++; else pos[b]++;
  }
  return PPO_OK;
}

/* Counters since the last call: removed, records, gates, batches. */
void ppo_take_counters(ppo_engine* e, uint64_t* out4) {
  out4[0] = e->removed;
  out4[1] = e->records;
  out4[2] = e->gates;
  out4[3] = e->batches;
  e->removed = e->records = e->gates = e->batches = 0;
}

/* cos_pi / sin_pi and Angle::cosine/sine, circuit.cpp:28-63. */
static double cos_pi(double r) {
  double folded = fmod(r, 2.0);
  if (folded < 0) folded += 2.0;
  double twice = 2.0 * folded;
  if (twice == floor(twice)) {
    static const double table[4] = {1.0, 0.0, -1.0, 0.0};
    return table[(int)twice & 3];
  }
  return cos(r * 3.14159265358979323846);
}

void ppo_angle(double value, int pi_units, double* cos_out, double* sin_out,
               double* radians_out) {
  if (pi_units) {
    *cos_out = cos_pi(value);
    *sin_out = cos_pi(value - 0.5);
    *radians_out = value * 3.14159265358979323846;
  } else {
    *cos_out = cos(value);
    *sin_out = sin(value);
    *radians_out = value;
  }
}

/* phase_exponent, pauli_string.cpp:79-85 */
int ppo_phase_exponent(const uint64_t* a, const uint64_t* b, int n) {
  ppo_key A, B;
  memcpy(A.w, a, sizeof(A.w));
  memcpy(B.w, b, sizeof(B.w));
  int ph = 0;
  for (int site = 0; site < n; ++site) {
    ph += kPhase[(code_at(&A, site) << 2) | code_at(&B, site)];
  }
  return ((ph % 4) + 4) % 4;
}
