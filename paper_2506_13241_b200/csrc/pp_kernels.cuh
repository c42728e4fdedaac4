// pp_kernels.cuh -- sm_100a kernels of the Pauli-propagation hot path.
#ifndef PP_DENSE_LOG
#define PP_DENSE_LOG 13
#endif
#ifndef PP_DENSE_RADIX
#define PP_DENSE_RADIX 4
#endif
#ifndef PP_DENSE_CTAS
#define PP_DENSE_CTAS 2
#endif
//
// Store layout: the operator is a set of
// z-groups.  Every string of a group shares its z-plane, which is stored
// once in the group table; the strings themselves live in an arena as
// structure-of-arrays x-plane words + fp64 coefficient (8W+8 bytes/string),
// sorted ascending by x inside each group's region.
//
// Why z-groups: an Rx gate on qubit q (generator X_q) anticommutes with a
// string iff z_q = 1 and its partner flips only x_q (SURVEY.md section 0,
// fact 2), so a z-group is either untouched by the gate or entirely
// branched, and all children stay inside their group.  The branch+merge of
// one gate therefore reads and writes only the affected groups.
//
// All coefficient arithmetic uses __dmul_rn/__dadd_rn (no FMA contraction)
// so results are bit-identical to the reference's scalar C++ (engine.cpp:
// 223-226, term_map.hpp:77-79).
#pragma once

#include "pp_common.cuh"

namespace ppgpu {

template <int W>
struct ArenaView {
  uint64_t* x[W];
  double* c;
};

template <int W>
struct GroupView {
  uint64_t* z[W];
  uint64_t* off;
  uint32_t* cnt;
  uint32_t* cap;
  double* gmax;
  double* gmin;
  uint32_t* flags;  // bit0: non-finite coefficient present; bit1 (kFlagUnsorted): strings not sorted by x
  uint32_t* stamp;  // sequence number of the last X-type gate applied (makes gates resumable)
};
// A regroup that feeds a dense Rx run skips the per-group sort (the dense
// path scatters by x and writes sorted output); such groups carry this flag
// until the dense path or a sort pass (k_sort_small/k_sort_big with
// only_unsorted) rewrites them.
constexpr uint32_t kFlagUnsorted = 2u;
// bit2: the smallest x of an unsorted group is its first string (dense_multi's class-major output)
constexpr uint32_t kFlagMinFirst = 4u;
// which groups a sort pass takes: only_unsorted = 0 all, 1 the unsorted ones,
// 2 the unsorted ones that are not a dense run's class-major output (what a
// regroup left, i.e. groups still waiting for the current run)
__device__ __forceinline__ bool sort_wanted(uint32_t flags, int only_unsorted) {
  if (only_unsorted == 0) return true;
  if (!(flags & kFlagUnsorted)) return false;
  return only_unsorted == 1 || !(flags & kFlagMinFirst);
}

// deferred truncation helpers (see k_thresh): a pending string is held as
// -0.0 in shared memory (stored values are never zero when truncating per
// gate), and a group's threshold slot follows from its stamp
__device__ __forceinline__ bool is_pending(double c) {
  return __double_as_longlong(c) == (long long)0x8000000000000000ull;
}
__device__ __forceinline__ uint32_t pending_index(uint32_t stamp, uint32_t win_base, uint32_t rel) {
  const uint32_t idx = stamp - win_base;
  return idx > rel ? 0u : idx;
}

// Per-gate scratch lives in small slot arrays so consecutive gates need no
// reset launches: a gate's kernels use slot s and clear slot s^1 for the
// next gate.
struct RedSlot {            // group reduction of one epilogue
  unsigned long long live;
  unsigned long long gmax_bits;
  unsigned long long gmin_bits;
  unsigned int nonfinite;
  unsigned int maxcnt;      // largest group (k_reduce)
};
struct SelSlot {            // affected-group selection of one X-type gate
  unsigned long long aff_elems;
  unsigned int n_aff;
  unsigned int pad;
};

__device__ __forceinline__ void clear_red(RedSlot* r) {
  r->live = 0;
  r->gmax_bits = 0;
  r->gmin_bits = 0x7ff0000000000000ull;
  r->nonfinite = 0;
  r->maxcnt = 0;
}

// batches_sent (engine.cpp:286-301, one worker): a gate counts one batch iff
// it sent at least one record.  Kernels set one bit per gate of the harvest
// window (the gates applied since the host last read the statistics); fused
// ZZ runs record their anticommuting-edge masks per edge group instead, which
// the host maps back to gates.
constexpr int kSeenWords = 16;          // gates per harvest window: 1024
constexpr int kSeenGates = 64 * kSeenWords;
constexpr int kZZSeenGroups = 64;       // = kMaxZZGroups (pp_regroup.cuh)

struct DevStats {
  RedSlot red[3];                  // [0,1]: per-gate epilogues, [2]: host syncs
  SelSlot sel[2];
  unsigned long long bump;         // bump pointer of the target arena
  unsigned long long records;      // nonzero sin-branch records (records_sent)
  unsigned long long removed;      // stored strings dropped (zero or truncated)
  unsigned long long items;        // regroup work items
  unsigned long long rec_total;    // regroup record slots reserved
  unsigned long long scratch_bump; // scratch allocation for big sorts
  unsigned long long diag_count;   // diagonal strings found
  unsigned long long out_elems;    // strings written by branch kernels
  unsigned int overflow;
  unsigned int collision;
  unsigned int distinct;
  unsigned int err_budget;         // sticky: term budget exceeded (check_budget)
  unsigned int err_numerical;      // sticky: NaN/Inf seen by a truncation
  unsigned int pad;
  unsigned long long err_gate;     // gate index of the first error
  unsigned long long err_live;     // |O| at the first error
  unsigned long long last_gmax_bits;  // gmax used by the latest truncation
  unsigned long long aff_total;    // cumulative strings in affected groups
  unsigned int work[2];            // chunk counters of consecutive branch launches
  unsigned long long stream_elems; // strings branched through the long-block stream path
  unsigned long long arena_cap;    // capacity of the current arena (strings)
  unsigned long long seq_base;     // sequence number of gate 0 of the current launch run
  unsigned int G_dev;              // group count of the current table
  unsigned int err_arena;          // sticky: a branch allocation did not fit; run must resume
  unsigned long long err_seq;      // first gate sequence number that overflowed
  unsigned long long scan_total;   // regroup: total records (copied from the scan)
  unsigned int zz_newg;            // Z-type gate: groups created for missing partners
  unsigned int zz_maxcnt;          // Z-type gate: largest group written
  unsigned int zz_err;             // Z-type gate: a pair exceeded the segment (host pre-check failed)
  unsigned int zz_pad;
  unsigned int err_unsorted;        // sticky: a sublayer skipped an unsorted group it could not apply densely
  unsigned int pad2;
  unsigned long long cliff_records; // records of a regroup whose sizes the host reads later (deferred)
  unsigned long long dense_groups;  // groups applied by the dense sublayer path (cumulative)
  unsigned long long dense_out;     // strings those groups wrote
  unsigned long long bulk_tiles;    // dense_passes tiles moved by bulk copies (cumulative)
  unsigned int seen_base;           // window index of gate 0 of the current launch run
  unsigned int left_n;              // groups k_dense_sublayer left for the per-gate path (this launch)
  unsigned long long seen[kSeenWords];            // bit g: window gate g sent a record
  unsigned long long zz_seen[kZZSeenGroups][2];   // fused ZZ run: edges (bit i of group k) that sent one
};

__device__ __forceinline__ void mark_seen(DevStats* st, uint32_t bit) {
  if (bit >= (uint32_t)kSeenGates) return;
  const unsigned long long m = 1ull << (bit & 63);
  unsigned long long* w = &st->seen[bit >> 6];
  if (!(*(volatile unsigned long long*)w & m)) atomicOr(w, m);
}

// Scalars a launch run reads from device memory, so that a captured CUDA
// graph can be replayed for every layer.
constexpr unsigned int kKeepG = 0xffffffffu;  // k_set_scalars / k_diag: the group count is on the device
__global__ void k_set_scalars(DevStats* st, unsigned int G, unsigned long long cap, unsigned long long seq_base,
                              unsigned int seen_base) {
  if (G != kKeepG) st->G_dev = G;
  st->seen_base = seen_base;
  st->arena_cap = cap;
  st->seq_base = seq_base;
  st->work[0] = st->work[1] = 0;
  st->left_n = 0;
  clear_red(&st->red[0]);
  clear_red(&st->red[1]);
  clear_red(&st->red[2]);  // the host-sync slot (only sync_state's k_reduce fills it)
}

// set_initial for a handful of terms (the usual single observable string):
// everything travels as kernel parameters, no copies and no round trip.
constexpr uint32_t kInitSmall = 4;
template <int W>
struct InitSmall {
  uint32_t n, G;
  uint64_t x[kInitSmall][W];
  double c[kInitSmall];
  uint64_t z[kInitSmall][W];
  uint64_t off[kInitSmall];
  uint32_t cnt[kInitSmall], flags[kInitSmall];
  double gmax[kInitSmall], gmin[kInitSmall];
};

// Full reset of the statistics block (bump pointer of the target arena).
__device__ __forceinline__ void k_reset_stats_body(DevStats* st, unsigned long long bump) {
  DevStats s;
  memset(&s, 0, sizeof(s));
  s.bump = bump;
  for (int i = 0; i < 3; ++i) s.red[i].gmin_bits = 0x7ff0000000000000ull;
  s.err_seq = ~0ull;
  *st = s;
}

// Reset of one reduction slot (cumulative counters and sticky errors stay).
__global__ void k_red_reset(RedSlot* r) { clear_red(r); }

__device__ __forceinline__ bool engine_failed(const DevStats* st) {
  return (*(volatile const unsigned int*)&st->err_budget) | (*(volatile const unsigned int*)&st->err_numerical) |
         (*(volatile const unsigned int*)&st->err_arena);
}

template <int W>
__device__ __forceinline__ Plane<W> load_plane(uint64_t* const (&p)[W], uint64_t i) {
  Plane<W> r;
#pragma unroll
  for (int k = 0; k < W; ++k) r.w[k] = p[k][i];
  return r;
}
template <int W>
__device__ __forceinline__ void store_plane(uint64_t* const (&p)[W], uint64_t i, const Plane<W>& v) {
#pragma unroll
  for (int k = 0; k < W; ++k) p[k][i] = v.w[k];
}

// ---------------------------------------------------------------------------
// shared-memory key arrays (SoA: one array per plane word, bank friendly)
// ---------------------------------------------------------------------------
template <int W>
__device__ __forceinline__ Plane<W> sk_load(const uint64_t* base, uint32_t stride, uint32_t i) {
  Plane<W> r;
#pragma unroll
  for (int k = 0; k < W; ++k) r.w[k] = base[k * stride + i];
  return r;
}
template <int W>
__device__ __forceinline__ void sk_store(uint64_t* base, uint32_t stride, uint32_t i, const Plane<W>& v) {
#pragma unroll
  for (int k = 0; k < W; ++k) base[k * stride + i] = v.w[k];
}
// first index in [0, n) with key >= k
template <int W>
__device__ __forceinline__ uint32_t sk_lower_bound(const uint64_t* base, uint32_t stride, uint32_t n,
                                                   const Plane<W>& k) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (plane_lt<W>(sk_load<W>(base, stride, mid), k)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// first index in [0, n) with key > k
template <int W>
__device__ __forceinline__ uint32_t sk_upper_bound(const uint64_t* base, uint32_t stride, uint32_t n,
                                                   const Plane<W>& k) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (!plane_lt<W>(k, sk_load<W>(base, stride, mid))) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// ---------------------------------------------------------------------------
// group selection for an X-type gate
// ---------------------------------------------------------------------------
template <int W>
__global__ void k_select_x(GroupView<W> g, uint32_t G, Plane<W> jx, uint32_t* list, SelSlot* sel, DevStats* st) {
  if (engine_failed(st)) return;
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  bool take = false;
  uint32_t c = 0;
  if (i < G) {
    c = g.cnt[i];
    if (c) take = plane_parity_and<W>(load_plane<W>(g.z, i), jx);
  }
  unsigned mask = __ballot_sync(0xffffffffu, take);
  if (!mask) return;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t base = 0;
  unsigned long long sum = warp_sum64(take ? c : 0);
  if (lane == 0) {
    base = atomicAdd(&sel->n_aff, __popc(mask));
    atomicAdd(&sel->aff_elems, sum);
    atomicAdd(&st->aff_total, sum);
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  if (take) list[base + __popc(mask & ((1u << lane) - 1))] = i;
}

// ---------------------------------------------------------------------------
// K_branch: Rx branch + merge of one affected z-group (one CTA per group).
//
// For the group S (sorted by x) and the gate X_q every string branches:
//   parent   x        -> cos * c                 (engine.cpp:223)
//   child    x ^ e_q  -> (+-sin) * c_parent       (engine.cpp:224-227)
// with sign + for a Z at q (x_q = 0) and - for a Y (x_q = 1)
// (record_sign, engine.cpp:67-73 with the phase table of
// pauli_string.cpp:28-34).  A child landing on an existing string is added
// to its scaled value (TermMap::add, term_map.hpp:77-79); each key gets at
// most one child, so the sum is a single two-operand rounding.
//
// The output is the sorted merge of three sorted streams read from S:
//   A  = S                      (all strings, scaled by cos)
//   T0 = { x | e_q : x_q = 0 }  (children of Z-parents, keys with bit q set)
//   T1 = { x &~e_q : x_q = 1 }  (children of Y-parents, keys with bit q clear)
// T0 and T1 are disjoint, and a T key equal to an A key is a partner pair.
// The CTA streams the three views through shared-memory buffers, merging
// every round all buffered keys <= kmax (the smallest last-buffered key of
// the streams that still have input), then compacts and writes them.
// ---------------------------------------------------------------------------
constexpr uint32_t kBufCap = 2 * kCta;      // per-stream buffer
constexpr uint32_t kRefill = kCta;          // refill threshold
constexpr uint32_t kSlots = 3 * kBufCap;    // output slots per round

template <int W>
struct BranchSmem {
  uint64_t key[3][W * kBufCap];
  double val[3][kBufCap];
  uint64_t skey[W * kSlots];
  double sval[kSlots];
  uint8_t semit[kSlots];
  uint32_t scan[40];
  uint32_t cnt[3];
  uint32_t pos[3];
  uint32_t m[3];
  uint32_t all_done;
};

// Three-stream merge over one range S[src, src + n) of a group (a whole
// block of equal high bits, or a whole group): appends the sorted outputs at
// dst + out_n.  Buffers: BranchSmem.
template <int W>
__device__ void stream_branch_range(BranchSmem<W>& sm, ArenaView<W> ar, uint64_t src, uint32_t n, uint64_t dst,
                                    uint32_t& out_n, int wq, uint64_t mq, double cosv, double sinv, int keep_zeros,
                                    double& vmax, double& vmin, uint32_t& nonfinite, unsigned long long& records,
                                    unsigned long long& removed, double tout, double& vall, double tin = -1.0) {
  const uint32_t tid = threadIdx.x;
  const double nsin = -sinv;
  __syncthreads();
  if (tid == 0) {
    sm.cnt[0] = sm.cnt[1] = sm.cnt[2] = 0;
    sm.pos[0] = sm.pos[1] = sm.pos[2] = 0;
  }
  __syncthreads();
  for (;;) {
    // ---- refill the three stream buffers --------------------------------
#pragma unroll 1
    for (int s = 0; s < 3; ++s) {
      while (sm.cnt[s] < kRefill && sm.pos[s] < n) {
        uint32_t p = sm.pos[s] + tid;
        bool ok = false;
        Plane<W> key;
        double v = 0.0;
        if (p < n) {
          key = load_plane<W>(ar.x, src + p);
          v = ar.c[src + p];
          if (tin >= 0.0 && fabs(v) <= tin) v = -0.0;  // removed by a deferred truncation
          uint32_t cls = (key.w[wq] & mq) ? 1u : 0u;
          ok = (s == 0) || (s == 1 && cls == 0) || (s == 2 && cls == 1);
          if (s) key.w[wq] ^= mq;
        }
        uint32_t total;
        uint32_t o = block_excl_scan(ok ? 1u : 0u, sm.scan, &total);
        if (ok) {
          uint32_t d = sm.cnt[s] + o;
          sk_store<W>(sm.key[s], kBufCap, d, key);
          sm.val[s][d] = v;
        }
        __syncthreads();
        if (tid == 0) {
          sm.cnt[s] += total;
          sm.pos[s] += kCta;
        }
        __syncthreads();
      }
    }
    // ---- choose kmax and the consumed prefix of every stream ------------
    if (tid < 3) {
      Plane<W> kmax = plane_max<W>();
      bool bounded = false;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        if (sm.pos[s] < n) {  // stream still has unread input
          Plane<W> last = sk_load<W>(sm.key[s], kBufCap, sm.cnt[s] - 1);
          if (!bounded || plane_lt<W>(last, kmax)) kmax = last;
          bounded = true;
        }
      }
      uint32_t s = tid;
      sm.m[s] = bounded ? sk_upper_bound<W>(sm.key[s], kBufCap, sm.cnt[s], kmax) : sm.cnt[s];
    }
    __syncthreads();
    const uint32_t mA = sm.m[0], m0 = sm.m[1], m1 = sm.m[2];
    const uint32_t total = mA + m0 + m1;
    for (uint32_t i = tid; i < total; i += kCta) sm.semit[i] = 0;
    __syncthreads();
    // ---- A: scaled parents, plus the partner child if present -------------
    for (uint32_t i = tid; i < mA; i += kCta) {
      Plane<W> k = sk_load<W>(sm.key[0], kBufCap, i);
      double c = sm.val[0][i];
      uint32_t l0 = sk_lower_bound<W>(sm.key[1], kBufCap, m0, k);
      uint32_t l1 = sk_lower_bound<W>(sm.key[2], kBufCap, m1, k);
      uint32_t rank = i + l0 + l1;
      double v = __dmul_rn(c, cosv);
      if (k.w[wq] & mq) {  // bit q set: partner child comes from a Z-parent (T0)
        if (l0 < m0 && plane_eq<W>(sk_load<W>(sm.key[1], kBufCap, l0), k)) {
          double d = __dmul_rn(sinv, sm.val[1][l0]);
          if (d != 0.0) v = __dadd_rn(v, d);
        }
      } else {
        if (l1 < m1 && plane_eq<W>(sk_load<W>(sm.key[2], kBufCap, l1), k)) {
          double d = __dmul_rn(nsin, sm.val[2][l1]);
          if (d != 0.0) v = __dadd_rn(v, d);
        }
      }
      vall = fmax(vall, fabs(v));
      bool emit = tout < 0.0 ? (keep_zeros || v != 0.0) : !(fabs(v) <= tout);  // remove_below: |c| <= T
      const bool pend = tin >= 0.0 && is_pending(c);
      if (pend) ++removed;  // its deferred removal, counted once
      if (!emit && !pend) ++removed;
      sk_store<W>(sm.skey, kSlots, rank, k);
      sm.sval[rank] = v;
      sm.semit[rank] = emit;
    }
    // ---- T0 / T1: children; emitted on their own when no partner exists ---
    for (uint32_t j = tid; j < m0 + m1; j += kCta) {
      const bool t0 = j < m0;
      const uint32_t jj = t0 ? j : j - m0;
      const int s = t0 ? 1 : 2;
      Plane<W> k = sk_load<W>(sm.key[s], kBufCap, jj);
      double d = __dmul_rn(t0 ? sinv : nsin, sm.val[s][jj]);
      if (d != 0.0) ++records;
      uint32_t la = sk_lower_bound<W>(sm.key[0], kBufCap, mA, k);
      if (la < mA && plane_eq<W>(sk_load<W>(sm.key[0], kBufCap, la), k)) continue;  // partner
      if (d == 0.0) continue;  // engine.cpp:226: no record for a zero increment
      vall = fmax(vall, fabs(d));
      if (tout >= 0.0 && fabs(d) <= tout) {  // inserted, then truncated
        ++removed;
        continue;
      }
      uint32_t lo = t0 ? sk_lower_bound<W>(sm.key[2], kBufCap, m1, k) : sk_lower_bound<W>(sm.key[1], kBufCap, m0, k);
      uint32_t rank = jj + la + lo;
      sk_store<W>(sm.skey, kSlots, rank, k);
      sm.sval[rank] = d;
      sm.semit[rank] = 1;
    }
    __syncthreads();
    // ---- compact the slots and stream them out ----------------------------
    for (uint32_t base = 0; base < total; base += kCta) {
      uint32_t s = base + tid;
      bool e = s < total && sm.semit[s];
      uint32_t tot;
      uint32_t o = block_excl_scan(e ? 1u : 0u, sm.scan, &tot);
      if (e) {
        double v = sm.sval[s];
        uint64_t d = dst + out_n + o;
        store_plane<W>(ar.x, d, sk_load<W>(sm.skey, kSlots, s));
        ar.c[d] = v;
        double av = fabs(v);
        if (!(av <= 1.7976931348623157e308)) nonfinite = 1;  // NaN or Inf
        vmax = fmax(vmax, av);
        vmin = fmin(vmin, av);
      }
      out_n += tot;
    }
    // ---- drop the consumed prefixes --------------------------------------
    uint32_t rem[3];
#pragma unroll
    for (int s = 0; s < 3; ++s) rem[s] = sm.cnt[s] - sm.m[s];
    Plane<W> tk[3][kBufCap / kCta];
    double tv[3][kBufCap / kCta];
#pragma unroll
    for (int s = 0; s < 3; ++s) {
#pragma unroll
      for (uint32_t r = 0; r < kBufCap / kCta; ++r) {
        uint32_t i = tid + r * kCta;
        if (i < rem[s]) {
          tk[s][r] = sk_load<W>(sm.key[s], kBufCap, sm.m[s] + i);
          tv[s][r] = sm.val[s][sm.m[s] + i];
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 3; ++s) {
#pragma unroll
      for (uint32_t r = 0; r < kBufCap / kCta; ++r) {
        uint32_t i = tid + r * kCta;
        if (i < rem[s]) {
          sk_store<W>(sm.key[s], kBufCap, i, tk[s][r]);
          sm.val[s][i] = tv[s][r];
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      bool done = true;
#pragma unroll
      for (int s = 0; s < 3; ++s) {
        sm.cnt[s] = rem[s];
        done &= (rem[s] == 0 && sm.pos[s] >= n);
      }
      sm.all_done = done;
    }
    __syncthreads();
    if (sm.all_done) break;
  }

}

// ---------------------------------------------------------------------------
// Segment path.  In a group sorted by x, the gate X_q pairs only strings that
// agree on every x bit above q ("blocks"); inside a block the class-0 strings
// (x_q = 0) precede the class-1 strings.  A block's output is the sorted
// coset list Y = merge(S_0, S_1 &~e_q) followed by Y | e_q.  Whole blocks that
// fit in one shared-memory segment are processed from a single coalesced
// load: per-element ranks by binary search inside the block, per-block output
// bases by a CTA scan, then one compaction and a coalesced store.
// ---------------------------------------------------------------------------
constexpr uint32_t kSeg = 1024;
constexpr uint32_t kVT = kSeg / kCta;
constexpr uint32_t kNone = 0xffffffffu;

template <int W>
struct SegSmem {
  uint64_t key[W * (kSeg + 1)];  // x planes of the segment (+1 lookahead), SoA
  double val[kSeg];
  alignas(16) uint32_t blk[kSeg];  // block id per string (stored as uint4)
  uint32_t bstart[kSeg + 1];     // first string of each block (+ end)
  uint32_t bys[kSeg];            // |Y| (cosets) of each block
  uint32_t bobase[kSeg];         // output slot base of each block
  alignas(16) uint32_t pre[kSeg + 4];  // exclusive prefixes: pairs << 16 | unpaired class-1
  union {
    uint32_t lbv[kSeg];          // partner search result per string (until the values pass)
    uint16_t cpos[2 * kSeg];     // compacted output position per slot (from the compaction on)
  };
  alignas(16) uint8_t f[kSeg];   // bit0 block start, bit1 class-0 with partner, bit2 unpaired class-1
  uint64_t okey[W * 2 * kSeg];
  double oval[2 * kSeg];
  alignas(16) uint8_t oemit[2 * kSeg];
  uint32_t scan[40];
  uint32_t nbc, lc;
};

template <int W>
__device__ __forceinline__ bool same_high(const Plane<W>& a, const Plane<W>& b, int wq, uint64_t hmask) {
  bool eq = true;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    uint64_t d = a.w[k] ^ b.w[k];
    if (k > wq) eq &= d == 0;
    else if (k == wq) eq &= (d & hmask) == 0;
  }
  return eq;
}

// first index in [lo, hi) of smem keys (stride kSeg+1) with key >= k
template <int W>
__device__ __forceinline__ uint32_t seg_lower_bound(const uint64_t* key, uint32_t lo, uint32_t hi, const Plane<W>& k) {
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (plane_lt<W>(sk_load<W>(key, kSeg + 1, mid), k)) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// A pack: several small groups of one gate processed as one segment (their
// strings side by side; a group start is always a block start), so a CTA
// pays the per-segment passes once per ~kSeg strings instead of once per
// group.  Built by k_branch_x; seg_branch<W, true> fills the per-group
// output counts, offsets and statistics.
constexpr uint32_t kMaxPack = 64;             // groups per pack
constexpr uint32_t kPackMaxGroup = kSeg / 2;  // larger groups go one by one

struct PackSmem {
  uint32_t m;                       // groups in the pack
  uint32_t gstart[kMaxPack + 1];    // first string of each group in the segment (+ end)
  uint64_t src[kMaxPack];           // arena offset of each group
  double tin[kMaxPack];             // deferred-truncation threshold per group (-1: none)
  double mx[kMaxPack], mn[kMaxPack];
  uint32_t cnt[kMaxPack], ostart[kMaxPack], nf[kMaxPack], gid[kMaxPack];
};

__device__ __forceinline__ uint32_t pack_group_of(const PackSmem& pk, uint32_t i) {
  uint32_t lo = 0, hi = pk.m;  // largest k with gstart[k] <= i
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (pk.gstart[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Processes the complete blocks at the front of S[p, n); returns how many
// strings were consumed (0: the first block is longer than a segment).
// PACK: the segment is the pack `pk` (all its strings, complete groups).
// Per-string passes are striped (string i on thread i % kCta: conflict-free
// shared memory); the three scans read flag bytes in a blocked layout.
template <int W, bool PACK = false>
__device__ uint32_t seg_branch(SegSmem<W>& sm, ArenaView<W> ar, uint64_t src, uint32_t p, uint32_t n, uint64_t dst,
                               uint32_t& out_n, int wq, uint64_t mq, double cosv, double sinv, int keep_zeros,
                               double& vmax, double& vmin, uint32_t& nonfinite, unsigned long long& records,
                               unsigned long long& removed, double tout, double& vall, double tin = -1.0,
                               PackSmem* pk = nullptr) {
  const uint32_t tid = threadIdx.x;
  const uint64_t hmask = ~((mq << 1) - 1);  // bits above q in word wq
  const uint32_t L = PACK ? pk->gstart[pk->m] : min(kSeg, n - p);
  const uint32_t has_next = (!PACK && p + L < n) ? 1u : 0u;
  const bool lazy = PACK ? pk->tin[0] >= 0.0 : tin >= 0.0;  // deferred truncation (uniform per launch)
  const double nsin = -sinv;
  __syncthreads();  // previous users of the shared buffers are done
  for (uint32_t i = tid; i < L + has_next; i += kCta) {
    uint64_t a;
    double t;
    if (PACK) {
      const uint32_t k = pack_group_of(*pk, i);
      a = pk->src[k] + (i - pk->gstart[k]);
      t = pk->tin[k];
    } else {
      a = src + p + i;
      t = tin;
    }
    sk_store<W>(sm.key, kSeg + 1, i, load_plane<W>(ar.x, a));
    if (i < L) {
      double v = ar.c[a];
      if (t >= 0.0 && fabs(v) <= t) v = -0.0;  // removed by a deferred truncation
      sm.val[i] = v;
    }
  }
  __syncthreads();
  // block starts (string i differs from i-1 above bit q; every group start)
  for (uint32_t i = tid; i < kSeg; i += kCta) {
    bool f = i < L && (i == 0 || !same_high<W>(sk_load<W>(sm.key, kSeg + 1, i - 1), sk_load<W>(sm.key, kSeg + 1, i),
                                               wq, hmask));
    sm.f[i] = f ? 1 : 0;
  }
  if (PACK) {
    __syncthreads();
    if (tid < pk->m) sm.f[pk->gstart[tid]] = 1;
  }
  __syncthreads();
  // scan 1 (blocked): block ids and starts
  {
    const uint32_t fl = reinterpret_cast<const uint32_t*>(sm.f)[tid];  // bytes 4 tid .. 4 tid + 3
    uint32_t cnt = __popc(fl & 0x01010101u);
    uint32_t nb;
    uint32_t run = block_excl_scan(cnt, sm.scan, &nb);
    uint32_t ids[kVT];
#pragma unroll
    for (uint32_t v = 0; v < kVT; ++v) {
      const uint32_t i = tid * kVT + v;
      if ((fl >> (8 * v)) & 1u) sm.bstart[run++] = i;
      ids[v] = run - 1;
    }
    reinterpret_cast<uint4*>(sm.blk)[tid] = make_uint4(ids[0], ids[1], ids[2], ids[3]);
    __syncthreads();
    if (tid == 0) {
      bool last_complete = !has_next || !same_high<W>(sk_load<W>(sm.key, kSeg + 1, L - 1),
                                                      sk_load<W>(sm.key, kSeg + 1, L), wq, hmask);
      uint32_t nbc = last_complete ? nb : nb - 1;
      uint32_t lc = last_complete ? L : sm.bstart[nb - 1];
      sm.nbc = nbc;
      sm.lc = lc;
      sm.bstart[nbc] = lc;
    }
    __syncthreads();
  }
  const uint32_t nbc = sm.nbc, Lc = sm.lc;
  if (nbc == 0) return 0;
  // partners: inside a block (equal bits above q) every class-1 key exceeds
  // every class-0 key, so the lower bound of x | e_q (class 0) lands in the
  // class-1 part and that of x &~e_q (class 1) in the class-0 part: one search
  // over the whole block, no split point needed
  for (uint32_t i = tid; i < kSeg; i += kCta) {
    uint8_t fl = i < kSeg ? sm.f[i] : 0;
    if (i < Lc) {
      const uint32_t b = sm.blk[i], bs = sm.bstart[b], be = sm.bstart[b + 1];
      Plane<W> k = sk_load<W>(sm.key, kSeg + 1, i);
      const bool c1 = (k.w[wq] & mq) != 0;
      k.w[wq] ^= mq;
      const uint32_t lb = seg_lower_bound<W>(sm.key, bs, be, k);
      const bool found = lb < be && plane_eq<W>(sk_load<W>(sm.key, kSeg + 1, lb), k);
      if (!c1 && found) fl |= 2;
      if (c1 && !found) fl |= 4;
      sm.lbv[i] = lb;
    }
    sm.f[i] = fl;
  }
  __syncthreads();
  // scan 2 (blocked): pairs (high half) and unpaired class-1 (low half)
  {
    const uint32_t fl = reinterpret_cast<const uint32_t*>(sm.f)[tid];
    const uint32_t c = (__popc(fl & 0x02020202u) << 16) | __popc(fl & 0x04040404u);
    uint32_t tot;
    uint32_t e = block_excl_scan(c, sm.scan, &tot);
    uint32_t out[kVT];
#pragma unroll
    for (uint32_t v = 0; v < kVT; ++v) {
      out[v] = e;
      const uint32_t b = (fl >> (8 * v)) & 0xffu;
      e += (((b >> 1) & 1u) << 16) | ((b >> 2) & 1u);
    }
    reinterpret_cast<uint4*>(sm.pre)[tid] = make_uint4(out[0], out[1], out[2], out[3]);
    if (tid == 0) sm.pre[kSeg] = tot;
  }
  __syncthreads();
  // scan 3 (blocked over blocks): |Y| per block and output bases
  {
    uint32_t bsum = 0, ys[kVT];
#pragma unroll
    for (uint32_t v = 0; v < kVT; ++v) {
      const uint32_t b = tid * kVT + v;
      ys[v] = 0;
      if (b < nbc) {
        const uint32_t bs = sm.bstart[b], be = sm.bstart[b + 1];
        ys[v] = (be - bs) - ((sm.pre[be] >> 16) - (sm.pre[bs] >> 16));
        sm.bys[b] = ys[v];
      }
      bsum += 2 * ys[v];
    }
    uint32_t s2;
    uint32_t ob = block_excl_scan(bsum, sm.scan, &s2);
#pragma unroll
    for (uint32_t v = 0; v < kVT; ++v) {
      const uint32_t b = tid * kVT + v;
      if (b < nbc) sm.bobase[b] = ob;
      ob += 2 * ys[v];
    }
    if (tid == 0) sm.scan[33] = s2;
  }
  __syncthreads();
  const uint32_t s2 = sm.scan[33];
  bool hole = false;  // this thread left a slot unemitted
  // values: Rx rule (engine.cpp:218-227 + term_map.hpp:77-79); the owner of
  // a coset (its class-0 string, or an unpaired class-1 string) fills both
  // output slots.  Rank in Y = class-0 keys below + unpaired class-1 keys below.
  for (uint32_t i = tid; i < Lc; i += kCta) {
    const uint8_t fl = sm.f[i];
    Plane<W> k = sk_load<W>(sm.key, kSeg + 1, i);
    const bool cls1 = (k.w[wq] & mq) != 0;
    const double c = sm.val[i];
    // a string removed by a deferred truncation is counted once, here; its
    // slot then behaves as absent (0 * cos + child == child, no record of 0)
    const bool pc = lazy && is_pending(c);
    if (pc) ++removed;
    if (cls1 && !(fl & 4)) continue;  // paired class-1: its class-0 partner owns the coset
    const uint32_t b = sm.blk[i], bs = sm.bstart[b];
    const uint32_t lb = sm.lbv[i];
    // unpaired class-1 strings below the block's class-1 part = below its start
    const uint32_t um = sm.pre[bs] & 0xffffu;
    const uint32_t ry = cls1 ? (lb - bs) + ((sm.pre[i] & 0xffffu) - um) : (i - bs) + ((sm.pre[lb] & 0xffffu) - um);
    const uint32_t ysz = sm.bys[b];
    const uint32_t s0 = sm.bobase[b] + ry, s1 = s0 + ysz;
    Plane<W> y = k, y1 = k;
    y.w[wq] &= ~mq;
    y1.w[wq] |= mq;
    double v0, v1;
    bool e0, e1;
    if (!cls1) {  // Z at q: the child y|e_q gets +sin c0
      const double d1 = __dmul_rn(sinv, c);
      if (d1 != 0.0) ++records;
      double s = __dmul_rn(c, cosv);
      if (fl & 2) {
        const double c1 = sm.val[lb];
        const double d0 = __dmul_rn(nsin, c1);  // child of the Y partner lands on y
        if (d0 != 0.0) {
          ++records;
          s = __dadd_rn(s, d0);
        }
        double t = __dmul_rn(c1, cosv);
        if (d1 != 0.0) t = __dadd_rn(t, d1);
        v1 = t;
        e1 = tout < 0.0 ? (keep_zeros || t != 0.0) : !(fabs(t) <= tout);
        if (!e1 && !(lazy && is_pending(c1))) ++removed;
      } else {
        v1 = d1;
        e1 = d1 != 0.0 && !(fabs(d1) <= tout);
        if (d1 != 0.0 && !e1) ++removed;  // inserted, then truncated
      }
      v0 = s;
      e0 = tout < 0.0 ? (keep_zeros || s != 0.0) : !(fabs(s) <= tout);
      if (!e0 && !pc) ++removed;
    } else {  // Y at q, no partner: the child y gets -sin c1
      const double d0 = __dmul_rn(nsin, c);
      if (d0 != 0.0) ++records;
      v0 = d0;
      e0 = d0 != 0.0 && !(fabs(d0) <= tout);
      if (d0 != 0.0 && !e0) ++removed;
      v1 = __dmul_rn(c, cosv);
      e1 = tout < 0.0 ? (keep_zeros || v1 != 0.0) : !(fabs(v1) <= tout);
      if (!e1 && !pc) ++removed;
    }
    vall = fmax(vall, fmax(fabs(v0), fabs(v1)));
    sk_store<W>(sm.okey, 2 * kSeg, s0, y);
    sm.oval[s0] = v0;
    sm.oemit[s0] = e0;
    sk_store<W>(sm.okey, 2 * kSeg, s1, y1);
    sm.oval[s1] = v1;
    sm.oemit[s1] = e1;
    hole |= !(e0 && e1);
  }
  // compaction: holes are exact zeros (removed strings); one blocked scan
  // over the emit bytes gives every slot its output position, then a
  // coalesced store reads the slots in position order.  Without holes (the
  // common case at epsilon0 = 0) the slots are the output as they stand.
  constexpr uint32_t kSV = 2 * kSeg / kCta;
  uint32_t ecnt = s2;
  if (__syncthreads_count(hole)) {
    const uint2 eb = reinterpret_cast<const uint2*>(sm.oemit)[tid];  // slots kSV tid .. kSV tid + 7
    const uint32_t base = tid * kSV;
    uint32_t m0 = 0;
#pragma unroll
    for (uint32_t v = 0; v < kSV; ++v) {
      const uint32_t byte = v < 4 ? (eb.x >> (8 * v)) & 0xffu : (eb.y >> (8 * (v - 4))) & 0xffu;
      if (base + v < s2 && byte) m0 |= 1u << v;
    }
    uint32_t tot;
    uint32_t o = block_excl_scan(__popc(m0), sm.scan, &tot);
    ecnt = tot;
    if (tot != s2) {
#pragma unroll
      for (uint32_t v = 0; v < kSV; ++v)
        if ((m0 >> v) & 1u) sm.cpos[o++] = (uint16_t)(base + v);
    }
  }
  __syncthreads();
  const bool dense = ecnt == s2;
  for (uint32_t i = tid; i < ecnt; i += kCta) {
    const uint32_t sl = dense ? i : sm.cpos[i];
    const double val = sm.oval[sl];
    const uint64_t d = dst + out_n + i;
    store_plane<W>(ar.x, d, sk_load<W>(sm.okey, 2 * kSeg, sl));
    ar.c[d] = val;
    if (!PACK) {
      const double av = fabs(val);
      if (!(av <= 1.7976931348623157e308)) nonfinite = 1;
      vmax = fmax(vmax, av);
      vmin = fmin(vmin, av);
    }
  }
  if (PACK) {
    // a group's slots and hence its outputs are contiguous: output range of
    // group k = emitted slots in [bobase of its first block, next group's)
    const uint32_t m = pk->m;
    if (tid < m) {
      const uint32_t sb = sm.bobase[sm.blk[pk->gstart[tid]]];
      uint32_t lo = 0, hi = ecnt;  // emitted slots below sb
      if (dense) {
        lo = sb;
      } else {
        while (lo < hi) {
          const uint32_t mid = (lo + hi) >> 1;
          if (sm.cpos[mid] < sb) lo = mid + 1;
          else hi = mid;
        }
      }
      pk->ostart[tid] = lo;
    }
    __syncthreads();
    // per-group statistics: one warp per group
    const uint32_t lane = tid & 31;
    for (uint32_t k = tid >> 5; k < m; k += kWarps) {
      const uint32_t o0 = pk->ostart[k], o1 = k + 1 < m ? pk->ostart[k + 1] : ecnt;
      unsigned long long gx = 0ull, gn = 0x7ff0000000000000ull;  // bits of |c|: 0 and +inf
      uint32_t nf = 0;
      for (uint32_t j = o0 + lane; j < o1; j += 32) {
        const unsigned long long ab = (unsigned long long)__double_as_longlong(sm.oval[dense ? j : sm.cpos[j]]) &
                                      0x7fffffffffffffffull;
        if (ab >= 0x7ff0000000000000ull) nf = 1;  // NaN or Inf
        if (ab <= 0x7ff0000000000000ull) {        // NaN takes no part in max/min (like fmax/fmin)
          gx = ab > gx ? ab : gx;
          gn = ab < gn ? ab : gn;
        }
      }
      gx = warp_max_bits(gx);
      gn = warp_min_bits(gn);
      nf = __any_sync(0xffffffffu, nf);
      if (lane == 0) {
        pk->cnt[k] = o1 - o0;
        pk->mx[k] = __longlong_as_double((long long)gx);
        pk->mn[k] = __longlong_as_double((long long)gn);
        pk->nf[k] = nf;
      }
    }
  }
  out_n += ecnt;
  return Lc;
}

// End of the block that starts at p (first index with different high bits),
// searched cooperatively: 256 probes per round narrow [lo, hi).
template <int W>
__device__ uint32_t find_block_end(ArenaView<W> ar, uint64_t src, uint32_t p, uint32_t n, int wq, uint64_t mq,
                                   uint32_t* scan) {
  const uint64_t hmask = ~((mq << 1) - 1);
  const Plane<W> k0 = load_plane<W>(ar.x, src + p);
  uint32_t lo = p, hi = n;  // x[lo] in the block; answer in (lo, hi]
  __shared__ uint32_t s_lo, s_hi;
  while (hi - lo > 1) {
    const uint32_t span = hi - lo - 1;  // candidates lo+1 .. hi-1
    const uint32_t step = (span + kCta - 1) / kCta;
    const uint32_t pos = lo + 1 + threadIdx.x * step;
    const bool valid = pos < hi;
    const bool out = valid && !same_high<W>(k0, load_plane<W>(ar.x, src + pos), wq, hmask);
    if (threadIdx.x == 0) {
      s_lo = lo;
      s_hi = hi;
    }
    __syncthreads();
    if (valid && out) atomicMin(&s_hi, pos);
    if (valid && !out) atomicMax(&s_lo, pos);
    __syncthreads();
    lo = s_lo;
    hi = s_hi;
    __syncthreads();
    if (step == 1) break;
  }
  (void)scan;
  return hi;
}

// Persistent: CTAs grab chunks of kCta groups from a counter, select the
// groups the gate touches (z_q = 1) with one coalesced check, and branch
// them, so selection costs no separate launch.  Each
// group is walked front to back: runs of small blocks go through the
// shared-memory segment path, a block longer than a segment through the
// three-stream merge restricted to that block.
template <int W>
__global__ void __launch_bounds__(kCta) k_branch_x(GroupView<W> g, ArenaView<W> ar, int wq, uint64_t mq,
                                                    double cosv, double sinv, int keep_zeros,
                                                    const uint64_t* __restrict__ zq, unsigned int* work,
                                                    unsigned int* work_next, uint32_t seq_rel, DevStats* st,
                                                    const double* __restrict__ thr, RedSlot* red_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BranchSmem<W>& sm = *reinterpret_cast<BranchSmem<W>*>(smem_raw);
  SegSmem<W>& sg = *reinterpret_cast<SegSmem<W>*>(smem_raw);
  const uint32_t tid = threadIdx.x;
  if (engine_failed(st)) return;
  const uint32_t G = *(volatile const unsigned int*)&st->G_dev;
  const unsigned long long cap = *(volatile const unsigned long long*)&st->arena_cap;
  const uint32_t seq_base = (uint32_t)*(volatile const unsigned long long*)&st->seq_base;
  const uint32_t seq = seq_base + seq_rel;
  const uint32_t chunk = max(1u, min(kCta, (G + gridDim.x - 1) / gridDim.x));  // one selection round when G is small
  unsigned long long aff_elems = 0;
  __shared__ unsigned long long dst_s;
  __shared__ double red_max[kWarps], red_min[kWarps];
  __shared__ unsigned long long red_rec[kWarps], red_rem[kWarps];
  __shared__ uint32_t red_nf[kWarps];
  __shared__ uint32_t glist[kCta];
  __shared__ uint32_t gscan[40];
  __shared__ uint32_t s_chunk, s_nlist;
  __shared__ uint32_t s_pp[kCta + 1], s_pfirst[kCta + 1];
  __shared__ uint64_t s_off[kCta];  // small groups of the chunk: arena offset
  __shared__ double s_tin[kCta];    // and deferred-truncation threshold
  __shared__ PackSmem pk;
  unsigned long long pk_records = 0, pk_removed = 0, pk_out = 0;
  // fused epilogue reduction (red_out): live count, max |c| over live strings
  // and the non-finite flag of every group, taken chunk by chunk after the
  // chunk's groups are rewritten (k_reduce's result, without its launch)
  unsigned long long r_live = 0;
  double r_max = 0.0;
  uint32_t r_nf = 0;
  const double thr0 = (red_out && thr) ? thr[0] : 0.0;
  if (blockIdx.x == 0 && tid == 0) *work_next = 0;  // the next gate's counter
  for (;;) {
  // grab the next chunk of kCta groups and select the affected ones in parallel
  __syncthreads();
  if (tid == 0) s_chunk = atomicAdd(work, 1u);
  __syncthreads();
  const uint32_t g0 = s_chunk * chunk;
  if (g0 >= G) break;
  {
    const uint32_t gi = g0 + tid;
    bool take = false;
    if (tid < chunk && gi < G) {  // three independent loads in flight
      const uint64_t zw = zq[gi];
      const uint32_t cn = g.cnt[gi], sp = g.stamp[gi];
      take = (zw & mq) && cn != 0 && sp != seq;
    }
    uint32_t tot;
    const uint32_t o = block_excl_scan(take ? 1u : 0u, gscan, &tot);
    if (take) glist[o] = gi;
    if (tid == 0) s_nlist = tot;
    __syncthreads();
  }
  const uint32_t nlist = s_nlist;
  // ---- groups of at most kPackMaxGroup strings: packs of up to kMaxPack
  // groups (consecutive in the list) whose start prefix falls in the same
  // half segment, so a pack holds at most kSeg strings
  uint32_t nsmall;
  {
    const bool in = tid < nlist;
    const uint32_t gi = in ? glist[tid] : 0u;
    uint32_t nt = 0, sp = 0;
    uint64_t go = 0;
    if (in) {  // independent loads in flight together
      nt = g.cnt[gi];
      go = g.off[gi];
      sp = g.stamp[gi];
    }
    const bool small = in && nt <= kPackMaxGroup;
    const double tg = (small && thr) ? thr[pending_index(sp, seq_base, seq_rel)] : -1.0;
    uint32_t tsz;
    const uint32_t r = block_excl_scan(small ? 1u : 0u, gscan, &nsmall);
    const uint32_t P = block_excl_scan(small ? nt : 0u, gscan, &tsz);
    if (small) {
      glist[r] = gi;
      s_pp[r] = P;
      s_off[r] = go;
      s_tin[r] = tg;
    } else if (in) {
      glist[nsmall + (tid - r)] = gi;  // the larger groups follow, in order
    }
    if (tid == 0) {
      s_pp[nsmall] = tsz;
      // one allocation for every small group of the chunk
      dst_s = tsz ? atomicAdd(&st->bump, 2ull * tsz) : 0ull;
      if (tsz && dst_s + 2ull * tsz > cap) {  // no room: they stay untouched, the host compacts and resumes
        atomicOr(&st->err_arena, 1u);
        atomicMin(&st->err_seq, (unsigned long long)seq);
      }
    }
    __syncthreads();
    const uint64_t chunk_dst = dst_s;
    const uint32_t npack_groups = (tsz && chunk_dst + 2ull * tsz > cap) ? 0u : nsmall;  // no room: skip (uniform)
    const bool start = tid < npack_groups && (tid % kMaxPack == 0 || s_pp[tid] / kPackMaxGroup !=
                                                                         s_pp[tid - 1] / kPackMaxGroup);
    uint32_t npk;
    const uint32_t q = block_excl_scan(start ? 1u : 0u, gscan, &npk);
    if (start) s_pfirst[q] = tid;
    if (tid == 0) s_pfirst[npk] = npack_groups;
    __syncthreads();
    for (uint32_t pj = 0; pj < npk; ++pj) {
      const uint32_t a = s_pfirst[pj], b = s_pfirst[pj + 1];
      const uint32_t m = b - a;
      const uint32_t base = s_pp[a], total = s_pp[b] - base;
      __syncthreads();  // the previous pack is written back
      if (tid < m) {
        pk.gid[tid] = glist[a + tid];
        pk.gstart[tid] = s_pp[a + tid] - base;
        pk.src[tid] = s_off[a + tid];
        pk.tin[tid] = s_tin[a + tid];
      }
      if (tid == 0) {
        pk.m = m;
        pk.gstart[m] = total;
      }
      __syncthreads();
      const uint64_t dst = chunk_dst + 2ull * base;
      aff_elems += total;
      uint32_t out_n = 0;
      double dmax = 0.0, dmin = 0.0, dall = 0.0;
      uint32_t dnf = 0;
      seg_branch<W, true>(sg, ar, 0, 0, total, dst, out_n, wq, mq, cosv, sinv, keep_zeros, dmax, dmin, dnf,
                          pk_records, pk_removed, -1.0, dall, -1.0, &pk);
      __syncthreads();
      if (tid < m) {
        const uint32_t gid = pk.gid[tid];
        const uint32_t c = pk.cnt[tid];
        g.off[gid] = dst + pk.ostart[tid];
        g.cnt[gid] = c;
        g.cap[gid] = c;
        g.gmax[gid] = c ? pk.mx[tid] : 0.0;
        g.gmin[gid] = c ? pk.mn[tid] : __longlong_as_double(0x7ff0000000000000ll);
        g.flags[gid] = pk.nf[tid];
        g.stamp[gid] = seq;
      }
      pk_out += out_n;
    }
  }
  // ---- larger groups one at a time
  for (uint32_t li = nsmall; li < nlist; ++li) {
    const uint32_t gid = glist[li];
    const uint32_t n = g.cnt[gid];
    const uint64_t src = g.off[gid];
    // deferred truncation: thresholds of the gates since this group was last
    // rewritten (read before this gate overwrites its stamp)
    const double tin = thr ? thr[pending_index(g.stamp[gid], seq_base, seq_rel)] : -1.0;
    __syncthreads();
    if (tid == 0) {
      dst_s = atomicAdd(&st->bump, 2ull * n);
      if (dst_s + 2ull * n > cap) {  // no room: leave the group untouched, the host compacts and resumes
        atomicOr(&st->err_arena, 1u);
        atomicMin(&st->err_seq, (unsigned long long)seq);
      }
    }
    __syncthreads();
    const uint64_t dst = dst_s;
    if (dst + 2ull * n > cap) continue;
    aff_elems += n;
    uint32_t out_n = 0;
    double vmax = 0.0, vmin = __longlong_as_double(0x7ff0000000000000ll);  // +inf
    uint32_t nonfinite = 0;
    unsigned long long records = 0, removed = 0;
    double vall = 0.0;
    uint32_t p = 0;
    while (p < n) {
      uint32_t used = seg_branch<W>(sg, ar, src, p, n, dst, out_n, wq, mq, cosv, sinv, keep_zeros, vmax, vmin,
                                    nonfinite, records, removed, -1.0, vall, tin);
      if (used) {
        p += used;
        continue;
      }
      __syncthreads();
      const uint32_t be = find_block_end<W>(ar, src, p, n, wq, mq, nullptr);
      if (tid == 0) atomicAdd(&st->stream_elems, (unsigned long long)(be - p));
      stream_branch_range<W>(sm, ar, src + p, be - p, dst, out_n, wq, mq, cosv, sinv, keep_zeros, vmax, vmin,
                             nonfinite, records, removed, -1.0, vall, tin);
      p = be;
    }
    // ---- per-group statistics -------------------------------------------
    vmax = warp_max(vmax);
    vmin = warp_min(vmin);
    records = warp_sum64(records);
    removed = warp_sum64(removed);
    nonfinite = __any_sync(0xffffffffu, nonfinite);
    const uint32_t lane = tid & 31, warp = tid >> 5;
    __syncthreads();
    if (lane == 0) {
      red_max[warp] = vmax;
      red_min[warp] = vmin;
      red_rec[warp] = records;
      red_rem[warp] = removed;
      red_nf[warp] = nonfinite;
    }
    __syncthreads();
    if (tid == 0) {
      for (uint32_t w = 1; w < kWarps; ++w) {
        vmax = fmax(vmax, red_max[w]);
        vmin = fmin(vmin, red_min[w]);
        records += red_rec[w];
        removed += red_rem[w];
        nonfinite |= red_nf[w];
      }
      g.off[gid] = dst;
      g.cnt[gid] = out_n;
      g.cap[gid] = 2 * n;
      g.gmax[gid] = out_n ? vmax : 0.0;
      g.gmin[gid] = out_n ? vmin : __longlong_as_double(0x7ff0000000000000ll);
      g.flags[gid] = nonfinite;
      g.stamp[gid] = seq;
      atomicAdd(&st->records, records);
      atomicAdd(&st->removed, removed);
      atomicAdd(&st->out_elems, (unsigned long long)out_n);
      if (records) mark_seen(st, st->seen_base + seq_rel);
    }
  }  // groups of the chunk
  if (red_out) {
    __syncthreads();  // the chunk's group entries are written
    const uint32_t gi = g0 + tid;
    if (tid < chunk && gi < G) {
      const uint32_t c = g.cnt[gi];
      const double gm = g.gmax[gi];
      const uint32_t fl = g.flags[gi];
      if (c) {
        r_live += c;
        // deferred truncation: a group whose max is pending removal is empty
        if (!thr || gm > thr0 || gm > thr[pending_index(g.stamp[gi], seq_base, seq_rel)]) r_max = fmax(r_max, gm);
        r_nf |= fl & 1u;
      }
    }
  }
  }  // chunks
  if (tid == 0 && aff_elems) atomicAdd(&st->aff_total, aff_elems);
  if (red_out) {
    r_live = warp_sum64(r_live);
    r_max = warp_max(r_max);
    r_nf = __any_sync(0xffffffffu, r_nf);
    __syncthreads();
    if ((tid & 31) == 0) {
      red_rec[tid >> 5] = r_live;
      red_max[tid >> 5] = r_max;
      red_nf[tid >> 5] = r_nf;
    }
    __syncthreads();
    if (tid == 0) {
      for (uint32_t w = 1; w < kWarps; ++w) {
        r_live += red_rec[w];
        r_max = fmax(r_max, red_max[w]);
        r_nf |= red_nf[w];
      }
      if (r_live) atomicAdd(&red_out->live, r_live);
      atomic_max_nonneg(reinterpret_cast<double*>(&red_out->gmax_bits), r_max);
      if (r_nf) atomicOr(&red_out->nonfinite, 1u);
    }
  }
  pk_records = warp_sum64(pk_records);
  pk_removed = warp_sum64(pk_removed);
  if ((tid & 31) == 0) {
    if (pk_records) {
      atomicAdd(&st->records, pk_records);
      mark_seen(st, st->seen_base + seq_rel);
    }
    if (pk_removed) atomicAdd(&st->removed, pk_removed);
  }
  if (tid == 0 && pk_out) atomicAdd(&st->out_elems, pk_out);
}

// ---------------------------------------------------------------------------
// K_sublayer: a whole run of X-type gates in ONE launch, for epsilon0 = 0.
// Under X-type gates z-groups evolve independently; the only coupling
// between them in the reference is the per-gate global max, and a threshold
// of 0 * gmax = 0 does not depend on it (exact zeros are dropped as they
// appear).  So each CTA takes a group and applies every gate of the run that
// touches it, in order.  g.stamp = sequence number of the last gate applied:
// after an arena overflow the host compacts and relaunches, and each group
// resumes after its stamp.
// ---------------------------------------------------------------------------
constexpr int kMaxSubGates = 128;
// Speculative (eps0 > 0) runs: each CTA of k_branch_sublayer ping-pongs a
// group's intermediate versions through two halves of its own scratch
// region in the arena tail ([cap + 2 kSpecScratch blockIdx, ...)), reused
// gate after gate and group after group (a small group's versions stay in
// L2); only the run's final strings are written to fresh arena space.  A
// working set beyond a half takes a pair of arena regions grown by doubling.
constexpr uint32_t kSpecScratch = 32768;

struct SubGates {
  int ng;
  int8_t wq[kMaxSubGates];
  uint64_t mq[kMaxSubGates];
  double cosv[kMaxSubGates];
  double sinv[kMaxSubGates];
  uint64_t any[2];  // union of the gate masks per plane word
  int dense;        // dense path allowed: distinct qubits, zeros dropped (k_branch_sublayer)
  int sorted;       // every group is sorted by x (no kFlagUnsorted group in the table)
  int maxk;         // x classes allowed per group on the dense path (<= kDenseMaxK; test hook)
  int fast;         // every |sin|, |cos| >= 2^-100: the dense butterflies may skip the per-point bookkeeping
};

// copy group region [src, src+n) to dst keeping |c| > T (truncation into
// fresh space, so the source stays intact for a rollback); returns the count
// and the kept max / min
template <int W>
__device__ uint32_t copy_truncated(ArenaView<W> ar, uint64_t src, uint32_t n, uint64_t dst, double T, uint32_t* scan,
                                   double& vmax, double& vmin) {
  uint32_t w = 0;
  for (uint32_t base = 0; base < n; base += kCta) {
    const uint32_t p = base + threadIdx.x;
    bool keep = false;
    Plane<W> k;
    double v = 0.0;
    if (p < n) {
      k = load_plane<W>(ar.x, src + p);
      v = ar.c[src + p];
      keep = !(fabs(v) <= T);
    }
    uint32_t tot;
    const uint32_t o = block_excl_scan(keep ? 1u : 0u, scan, &tot);
    if (keep) {
      store_plane<W>(ar.x, dst + w + o, k);
      ar.c[dst + w + o] = v;
      vmax = fmax(vmax, fabs(v));
      vmin = fmin(vmin, fabs(v));
    }
    w += tot;
  }
  return w;
}

// Block-wide reduction of the per-thread group statistics into shared
// scalars (result valid in every thread after the call).
struct GroupStatsSmem {
  double mx[kWarps], mn[kWarps], all[kWarps];
  unsigned long long rec[kWarps], rem[kWarps];
  uint32_t nf[kWarps];
};
__device__ __forceinline__ void reduce_group_stats(GroupStatsSmem& r, double& vmax, double& vmin, double& vall,
                                                   uint32_t& nonfinite, unsigned long long& records,
                                                   unsigned long long& removed) {
  // |c| statistics are non-negative and never NaN (fmax/fmin drop NaN), so
  // their bit patterns reduce with REDUX; per-thread counts fit 32 bits
  const unsigned long long bmax = warp_max_bits((unsigned long long)__double_as_longlong(vmax));
  const unsigned long long bmin = warp_min_bits((unsigned long long)__double_as_longlong(vmin));
  const unsigned long long ball = warp_max_bits((unsigned long long)__double_as_longlong(vall));
  const uint32_t rec = __reduce_add_sync(0xffffffffu, (uint32_t)records);
  const uint32_t rem = __reduce_add_sync(0xffffffffu, (uint32_t)removed);
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) {
    r.mx[warp] = __longlong_as_double((long long)bmax);
    r.mn[warp] = __longlong_as_double((long long)bmin);
    r.all[warp] = __longlong_as_double((long long)ball);
    r.rec[warp] = rec;
    r.rem[warp] = rem;
    r.nf[warp] = nonfinite;
  }
  __syncthreads();
  if (threadIdx.x == 0) {  // one thread folds the warps, every thread reads the result
    double a = r.mx[0], b = r.mn[0], c = r.all[0];
    unsigned long long d = r.rec[0], e = r.rem[0];
    uint32_t f = r.nf[0];
    for (uint32_t w = 1; w < kWarps; ++w) {
      a = fmax(a, r.mx[w]);
      b = fmin(b, r.mn[w]);
      c = fmax(c, r.all[w]);
      d += r.rec[w];
      e += r.rem[w];
      f |= r.nf[w];
    }
    r.mx[0] = a;
    r.mn[0] = b;
    r.all[0] = c;
    r.rec[0] = d;
    r.rem[0] = e;
    r.nf[0] = f;
  }
  __syncthreads();
  vmax = r.mx[0];
  vmin = r.mn[0];
  vall = r.all[0];
  records = r.rec[0];
  removed = r.rem[0];
  nonfinite = r.nf[0];
  __syncthreads();
}

// The same reduction with the result valid in thread 0 only: one barrier.
// (The caller's next writes to `r` come after further barriers.)
__device__ __forceinline__ void reduce_group_stats_t0(GroupStatsSmem& r, double& vmax, double& vmin, double& vall,
                                                      uint32_t& nonfinite, unsigned long long& records,
                                                      unsigned long long& removed) {
  const unsigned long long bmax = warp_max_bits((unsigned long long)__double_as_longlong(vmax));
  const unsigned long long bmin = warp_min_bits((unsigned long long)__double_as_longlong(vmin));
  const unsigned long long ball = warp_max_bits((unsigned long long)__double_as_longlong(vall));
  const uint32_t rec = __reduce_add_sync(0xffffffffu, (uint32_t)records);
  const uint32_t rem = __reduce_add_sync(0xffffffffu, (uint32_t)removed);
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    r.mx[warp] = __longlong_as_double((long long)bmax);
    r.mn[warp] = __longlong_as_double((long long)bmin);
    r.all[warp] = __longlong_as_double((long long)ball);
    r.rec[warp] = rec;
    r.rem[warp] = rem;
    r.nf[warp] = nonfinite;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = r.mx[0], b = r.mn[0], c = r.all[0];
    unsigned long long d = r.rec[0], e = r.rem[0];
    uint32_t f = r.nf[0];
    for (uint32_t w = 1; w < kWarps; ++w) {
      a = fmax(a, r.mx[w]);
      b = fmin(b, r.mn[w]);
      c = fmax(c, r.all[w]);
      d += r.rec[w];
      e += r.rem[w];
      f |= r.nf[w];
    }
    vmax = a;
    vmin = b;
    vall = c;
    records = d;
    removed = e;
    nonfinite = f;
  }
}

// ---------------------------------------------------------------------------
// Dense sublayer path (zeros dropped, distinct qubits, one x-class per group).
//
// A run of Rx gates on distinct qubits acts on a z-group as a tensor product
// of 2x2 rotations over the x bits T = {q : z_q = 1, gate on q in the run}.
// When every string of the group agrees on x outside T (one class, F), the
// group is a vector over the 2^m points of T (m = |T|): string x sits at
// b = pext(x, T) (T bits in ascending position, so b order is x order) and
// every other point is zero.  Gate q is a butterfly over bit rank(q) of b
// with the reference's per-string arithmetic (engine.cpp:218-227,
// term_map.hpp:77-79)
//   v0 = c0 cos [+ d0 = -sin c1 if d0 != 0],  v1 = c1 cos [+ d1 = sin c0 if d1 != 0]
// A zero point is an absent string: zero times cos and a zero delta leave
// every nonzero value unchanged, so the nonzero points after the run are
// the reference's strings bit for bit.  Records (nonzero deltas) and removed
// strings (points present after a gate -- nonzero before it or hit by a
// nonzero delta -- whose value is zero) are counted per point as the
// reference counts them per key.
//
// The group is read once and its output written once, already sorted.  The
// stages run in shared memory when 2^m <= kDenseSmem; larger blocks live in
// the output region's coefficient plane and pass through shared memory
// kDenseSmemLog stages at a time (each pass: the cosets of those stages'
// bits, one shared-memory tile each).
// ---------------------------------------------------------------------------
constexpr uint32_t kDenseSmemLog = PP_DENSE_LOG;
constexpr uint32_t kDenseSmem = 1u << kDenseSmemLog;  // doubles of the dynamic buffer
constexpr int kDenseMaxLog = 24;                      // larger blocks take the per-gate path
constexpr uint32_t kDenseMaxK = 256;                  // x classes per group on the dense path
constexpr uint32_t kDenseMaxOut = 1u << 26;           // K 2^m points per group

// Behind the dense tile in the dynamic buffer: output tables and the x-class
// bookkeeping of the group being processed.
constexpr uint32_t kDenseSlots = 2 * kDenseMaxK;  // class hash set (load <= 1/2)
template <int W>
struct DenseTail {
  Plane<W> xt[3 * 256];                 // b byte k -> x bits (T positions)
  unsigned long long hfp[kDenseSlots];  // class hash set: fingerprint (0 = empty)
  Plane<W> hF[kDenseSlots];             //   its class F
  uint8_t hcls[kDenseSlots];            //   its class index (ascending F)
  uint16_t used[kDenseSlots];           // occupied slots, compacted
  uint32_t ccnt[kDenseMaxK + 1];        // strings per class, then class start offsets
  uint32_t nused;                       // occupied slots
  Plane<W> sF[kDenseMaxK];              // classes in ascending order
};

template <int W>
struct DenseCtl {
  Plane<W> T;                   // touched x bits
  Plane<W> F;                   // the group's x bits outside T
  double scos[kMaxSubGates], ssin[kMaxSubGates];  // per stage
  uint32_t tw[kMaxSubGates / 32];                 // touching gates of the run (from k0)
  uint8_t sbit[kMaxSubGates];   // b bit of each stage, in gate order
  uint8_t sgate[kMaxSubGates];  // gate of each stage
  int m, klast;
  uint32_t P;                   // pass: b bits of its stages
  uint32_t deplo[128], dephi[64];  // pass: tile index -> b offset (low 7 / high 6 index bits)
  uint8_t tpos[32];             // b bit j -> x bit position (ascending)
  unsigned long long dst;
  uint32_t fail;
  uint32_t next;                // class discovery: first unmatched string
  // speculative truncation (epsilon0 > 0, per-gate cadence; tpred != nullptr)
  const double* tpred;          // predicted threshold per gate (shared copy), nullptr: none
  unsigned long long* smax;     // per-CTA max |c| after each gate's apply (bits)
  int ng;
  double tin;                   // threshold of the gates before the first stage (-1: none)
  double strunc[kMaxSubGates];  // threshold of the window after stage s (its gate .. the next stage's)
  unsigned long long wmax[2][kWarps];  // per-warp stage max, by stage parity
  uint32_t zeros;               // multi-class: zero points written (holes to compact)
  uint32_t fast;                // this group's butterflies take dense_stages_fast (see there)
  unsigned long long mbar;      // mbarrier of dense_passes' bulk tile loads (initialised once per CTA)
  uint32_t mphase;              //   its phase parity
  uint32_t bulk_tiles;          //   tiles it moved (diagnostics)
};

template <int W>
__device__ __forceinline__ uint32_t dense_pext(const Plane<W>& x, const Plane<W>& T) {
  uint32_t b = 0, j = 0;
#pragma unroll
  for (int k = 0; k < W; ++k)
    for (uint64_t t = T.w[k]; t; t &= t - 1, ++j)
      if (x.w[k] & t & (~t + 1)) b |= 1u << j;
  return b;
}
template <int W>
__device__ __forceinline__ Plane<W> dense_pdep(uint32_t b, const Plane<W>& T, Plane<W> x) {
  uint32_t j = 0;
#pragma unroll
  for (int k = 0; k < W; ++k)
    for (uint64_t t = T.w[k]; t; t &= t - 1, ++j)
      if ((b >> j) & 1u) x.w[k] |= t & (~t + 1);
  return x;
}
// deposit the low bits of i into the set bits of mask (32-bit index space)
__device__ __forceinline__ uint32_t dense_dep32(uint32_t i, uint32_t mask) {
  uint32_t r = 0;
  for (uint32_t t = mask; t; t &= t - 1, i >>= 1)
    if (i & 1u) r |= t & (~t + 1);
  return r;
}

__device__ __forceinline__ void dense_bfly(double& a, double& b, double cosv, double sinv, double nsin,
                                           unsigned long long& records, unsigned long long& removed) {
  const double c0 = a, c1 = b;
  const double d1 = __dmul_rn(sinv, c0);  // child of the Z parent (x_q = 0), lands at x_q = 1
  const double d0 = __dmul_rn(nsin, c1);  // child of the Y parent (x_q = 1), lands at x_q = 0
  double v0 = __dmul_rn(c0, cosv), v1 = __dmul_rn(c1, cosv);
  if (d0 != 0.0) {
    v0 = __dadd_rn(v0, d0);
    ++records;
  }
  if (d1 != 0.0) {
    v1 = __dadd_rn(v1, d1);
    ++records;
  }
  if ((c0 != 0.0 || d0 != 0.0) && v0 == 0.0) ++removed;
  if ((c1 != 0.0 || d1 != 0.0) && v1 == 0.0) ++removed;
  a = v0;
  b = v1;
}

// butterflies of stages [j0, j1) over a tile of 2^u doubles in shared memory;
// P: the b bits of the tile (stage bit p is tile bit popc(P & (2^p - 1)))
// max |c| of a group after gate k's apply was M: gate k and the following
// gates up to `next` (which do not touch the group; their truncations apply
// to it) see M until a threshold empties the group (engine.cpp:318-351 per
// gate; the old path's `contribute`).
template <int W>
__device__ __forceinline__ void dense_contribute(const DenseCtl<W>& dc, int k, int next, double M) {
  if (!(M > 0.0)) return;
  const unsigned long long bits = (unsigned long long)__double_as_longlong(M);
  atomicMax(&dc.smax[k], bits);
  for (int jj = k + 1; jj < next; ++jj) {
    if (M <= dc.tpred[jj - 1]) break;
    atomicMax(&dc.smax[jj], bits);
  }
}

// Shared-memory bank spreading for the register butterflies.  A thread owns
// the 2^r points its r stage bits span, at b | dep(e) (b: its index with
// zeros at the stage positions).  When stage positions fall among the low 4
// tile bits, the lanes of a half-warp differ only above them and all hit one
// bank (a 16-way conflict at stage bits {0..3}).  Thread t instead keeps
// point b | dep(e ^ g) in register e, g taking the lane bits that land above
// bit 3 onto the low stage positions: the 16 lanes then cover 16 distinct
// banks.  The butterfly of stage i is symmetric under that relabelling up to
// the sign of sin (registers e, e | 2^i hold the upper, lower point when bit
// i of g is set), so each point sees the same products and sums.
__device__ __forceinline__ uint32_t dense_bank_flip(const uint32_t* pm, int r, uint32_t lane) {
  int s = 0;
  for (int i = 0; i < r; ++i) s += pm[i] < 4u;
  uint32_t g = 0;
  for (int i = 0; i < r; ++i)
    if (pm[i] < 4u) {
      int rk = 0;  // rank of pm[i] among the low stage positions
      for (int k = 0; k < r; ++k) rk += pm[k] < pm[i];
      g |= ((lane >> (4 - s + rk)) & 1u) << i;
    }
  return g;
}

template <int W, bool SPEC>
__device__ __forceinline__ void dense_stages_t(double* d, uint32_t u, uint32_t P, int j0, int j1, DenseCtl<W>& dc,
                                               unsigned long long& records, unsigned long long& removed,
                                               uint32_t count, uint32_t& anom) {
  // count: points in the tile (a multiple of 2^(p+1) for every stage), default 2^u
  const uint32_t half = (count ? count : (1u << u)) >> 1;
  constexpr bool spec = SPEC;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int j = j0; j < j1; ++j) {
    if (!SPEC && j + 3 < j1 && half >= 8) {
      // four stages per pass (radix 16): each thread takes the 16 points the
      // four stage bits span and runs all four butterfly stages in registers
      // -- per point the same operations in the same order as stage by
      // stage, a quarter of the shared-memory round trips and barriers
      uint32_t pm[4], q[4];
      double cs[4], sn[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        pm[i] = __popc(P & ((1u << dc.sbit[j + i]) - 1u));
        q[i] = pm[i];
        cs[i] = dc.scos[j + i];
        sn[i] = dc.ssin[j + i];
      }
#pragma unroll
      for (int a = 0; a < 3; ++a)  // ascending insertion positions
#pragma unroll
        for (int b2 = 0; b2 < 3 - a; ++b2)
          if (q[b2] > q[b2 + 1]) {
            const uint32_t t2 = q[b2];
            q[b2] = q[b2 + 1];
            q[b2 + 1] = t2;
          }
      const uint32_t sixteenth = half >> 3;
      const uint32_t g = dense_bank_flip(pm, 4, lane);
      uint32_t dg = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        dg |= ((g >> i) & 1u) << pm[i];
        if ((g >> i) & 1u) sn[i] = -sn[i];
      }
      for (uint32_t t = threadIdx.x; t < sixteenth; t += kCta) {
        uint32_t b = t;
#pragma unroll
        for (int i = 0; i < 4; ++i) b = ((b >> q[i]) << (q[i] + 1)) | (b & ((1u << q[i]) - 1u));
        b |= dg;
        double a[16];
#pragma unroll
        for (int e = 0; e < 16; ++e)
          a[e] = d[b ^ (((e & 1) << pm[0]) | (((e >> 1) & 1) << pm[1]) | (((e >> 2) & 1) << pm[2]) |
                        (((e >> 3) & 1) << pm[3]))];
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int e = 0; e < 16; ++e)
            if (!((e >> i) & 1)) dense_bfly(a[e], a[e | (1 << i)], cs[i], sn[i], -sn[i], records, removed);
#pragma unroll
        for (int e = 0; e < 16; ++e)
          d[b ^ (((e & 1) << pm[0]) | (((e >> 1) & 1) << pm[1]) | (((e >> 2) & 1) << pm[2]) |
                 (((e >> 3) & 1) << pm[3]))] = a[e];
      }
      __syncthreads();
      j += 3;
      continue;
    }
    if (!SPEC && j + 1 < j1) {
      // two stages per pass (radix 4): each thread takes the four points a
      // pair of stage bits spans through both butterflies in registers --
      // the same operations in the same order per point, half the shared
      // memory round trips and barriers
      const uint32_t p1 = __popc(P & ((1u << dc.sbit[j]) - 1u)), p2 = __popc(P & ((1u << dc.sbit[j + 1]) - 1u));
      const uint32_t plo = p1 < p2 ? p1 : p2, phi = p1 < p2 ? p2 : p1;
      const uint32_t m1 = 1u << p1, m2 = 1u << p2;
      const uint32_t pp[2] = {p1, p2};
      const uint32_t g = dense_bank_flip(pp, 2, lane);  // see there
      const uint32_t dg = ((g & 1u) << p1) | (((g >> 1) & 1u) << p2);
      const double c1 = dc.scos[j], c2 = dc.scos[j + 1];
      const double s1 = (g & 1u) ? -dc.ssin[j] : dc.ssin[j], s2 = (g & 2u) ? -dc.ssin[j + 1] : dc.ssin[j + 1];
      const uint32_t quarter = half >> 1;
      for (uint32_t t = threadIdx.x; t < quarter; t += kCta) {
        uint32_t b = ((t >> plo) << (plo + 1)) | (t & ((1u << plo) - 1u));
        b = ((b >> phi) << (phi + 1)) | (b & ((1u << phi) - 1u));
        b |= dg;
        double a00 = d[b], a10 = d[b ^ m1], a01 = d[b ^ m2], a11 = d[b ^ m1 ^ m2];
        dense_bfly(a00, a10, c1, s1, -s1, records, removed);
        dense_bfly(a01, a11, c1, s1, -s1, records, removed);
        dense_bfly(a00, a01, c2, s2, -s2, records, removed);
        dense_bfly(a10, a11, c2, s2, -s2, records, removed);
        d[b] = a00;
        d[b ^ m1] = a10;
        d[b ^ m2] = a01;
        d[b ^ m1 ^ m2] = a11;
      }
      __syncthreads();
      ++j;
      continue;
    }
    const uint32_t p = __popc(P & ((1u << dc.sbit[j]) - 1u));
    // bank spreading (dense_bank_flip): for p < 4 the lanes above bit 3 flip
    // which register holds the lower point
    const uint32_t gflip = p < 4u ? (lane >> 3) & 1u : 0u;
    const double cosv = dc.scos[j], sinv = gflip ? -dc.ssin[j] : dc.ssin[j], nsin = -sinv;
    // speculative mode: the inputs carry the truncations of the previous
    // stage's window; the outputs' max feeds this gate's gmax
    const double tprev = (spec && j > 0) ? dc.strunc[j - 1] : -1.0;
    const uint32_t lo = (1u << p) - 1u;
    double mx = 0.0;
    for (uint32_t t = threadIdx.x; t < half; t += kCta) {
      const uint32_t b0 = (((t & ~lo) << 1) | (t & lo)) | (gflip << p);
      double a = d[b0], b = d[b0 ^ (1u << p)];
      if (tprev >= 0.0) {
        if (a != 0.0 && fabs(a) <= tprev) {  // remove_below: |c| <= T
          a = 0.0;
          ++removed;
        }
        if (b != 0.0 && fabs(b) <= tprev) {
          b = 0.0;
          ++removed;
        }
      }
      dense_bfly(a, b, cosv, sinv, nsin, records, removed);
      if (spec) mx = fmax(mx, fmax(fabs(a), fabs(b)));
      d[b0] = a;
      d[b0 ^ (1u << p)] = b;
    }
    if (spec) {
      mx = __longlong_as_double((long long)warp_max_bits((unsigned long long)__double_as_longlong(mx)));
      if (lane == 0) dc.wmax[j & 1][warp] = (unsigned long long)__double_as_longlong(mx);
    }
    __syncthreads();
    if (spec && threadIdx.x == 0) {
      unsigned long long m = 0;
      for (uint32_t w = 0; w < kWarps; ++w) m = dc.wmax[j & 1][w] > m ? dc.wmax[j & 1][w] : m;
      dense_contribute<W>(dc, dc.sgate[j], j + 1 < dc.m ? dc.sgate[j + 1] : dc.ng, __longlong_as_double((long long)m));
    }
  }
}

// Bookkeeping-free butterflies (SubGates::fast, DenseCtl::fast).  Live values
// entering a stage satisfy |v| >= 2^-890 (kFastLive; checked for the group's
// input and for every stage's outputs) and every |sin|, |cos| >= 2^-100, so a
// delta is zero exactly when its source point is, and "add the delta if it is
// nonzero" (term_map.hpp:77-79) equals always adding it.  Each stage then
// sends one record per live point (counted from the block's 2^R-bit live
// mask: a point is live after a stage when it or its partner was) and removes
// nothing, provided every live point still holds a value >= kFastLive after
// the stage -- one integer min over the high words (sign shifted out) of the
// live outputs.  A smaller value there, the zero of an exact cancellation
// included (cos = sin at pi/4 produces them), raises `anom` and the caller
// redoes the tile point by point (dense_bfly).
constexpr uint32_t kFastLiveHi = (1023u - 890u) << 20;
constexpr double kFastLive = 0x1p-890;

// One pass of R stages (radix 2^R): each thread takes the 2^R points the R
// stage bits span through all R butterfly stages in registers -- per point
// the same operations in the same order as stage by stage.
template <int R>
__device__ __forceinline__ void dense_fast_pass(double* d, uint32_t npts, const uint32_t (&pm)[4],
                                                const double (&cs0)[4], const double (&sn0)[4], uint32_t& records,
                                                uint32_t& anom) {
  constexpr int N = 1 << R;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t q[R];
  double cs[R], sn[R];
#pragma unroll
  for (int i = 0; i < R; ++i) q[i] = pm[i];
#pragma unroll
  for (int a = 0; a < R - 1; ++a)  // ascending insertion positions
#pragma unroll
    for (int b2 = 0; b2 < R - 1 - a; ++b2)
      if (q[b2] > q[b2 + 1]) {
        const uint32_t t2 = q[b2];
        q[b2] = q[b2 + 1];
        q[b2 + 1] = t2;
      }
  const uint32_t g = dense_bank_flip(pm, R, lane);  // see there
  uint32_t dg = 0;
#pragma unroll
  for (int i = 0; i < R; ++i) {
    dg |= ((g >> i) & 1u) << pm[i];
    cs[i] = cs0[i];
    sn[i] = ((g >> i) & 1u) ? -sn0[i] : sn0[i];
  }
  for (uint32_t t = threadIdx.x; t < (npts >> R); t += kCta) {
    uint32_t b = t;
#pragma unroll
    for (int i = 0; i < R; ++i) b = ((b >> q[i]) << (q[i] + 1)) | (b & ((1u << q[i]) - 1u));
    b |= dg;
    double a[N];
    uint32_t off[N];
#pragma unroll
    for (int e = 0; e < N; ++e) {
      uint32_t o = 0;
#pragma unroll
      for (int i = 0; i < R; ++i) o |= (uint32_t)((e >> i) & 1) << pm[i];
      off[e] = b ^ o;
      a[e] = d[off[e]];
    }
    uint32_t mk[4] = {0, 0, 0, 0};  // (four short dependency chains instead of one long one)
#pragma unroll
    for (int e = 0; e < N; ++e)
      if ((uint32_t)__double2hiint(a[e]) << 1) mk[e & 3] |= 1u << e;
    uint32_t mask = (mk[0] | mk[1]) | (mk[2] | mk[3]);
    if (!mask) continue;  // nothing live: nothing to do, nothing to store
#pragma unroll
    for (int i = 0; i < R; ++i) {
      records += __popc(mask);
#pragma unroll
      for (int e = 0; e < N; ++e)
        if (!((e >> i) & 1)) {
          double& x0 = a[e];
          double& x1 = a[e | (1 << i)];
          const double d1 = __dmul_rn(sn[i], x0), d0 = __dmul_rn(-sn[i], x1);
          x0 = __dadd_rn(__dmul_rn(x0, cs[i]), d0);
          x1 = __dadd_rn(__dmul_rn(x1, cs[i]), d1);
        }
      // a point is live after the stage when it or its partner was; every
      // live point must hold a value >= kFastLive (an exact cancellation
      // leaves a zero there: caught like any other small value)
      const uint32_t lowhalf = (i == 0 ? 0x5555u : i == 1 ? 0x3333u : i == 2 ? 0x0f0fu : 0x00ffu) & ((1u << N) - 1u);
      mask |= ((mask & lowhalf) << (1 << i)) | ((mask >> (1 << i)) & lowhalf);
      uint32_t um[4] = {0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu};
      if (mask == (1u << N) - 1u) {
#pragma unroll
        for (int e = 0; e < N; ++e) um[e & 3] = min(um[e & 3], (uint32_t)__double2hiint(a[e]) << 1);
      } else {
#pragma unroll
        for (int e = 0; e < N; ++e)
          if ((mask >> e) & 1u) um[e & 3] = min(um[e & 3], (uint32_t)__double2hiint(a[e]) << 1);
      }
      anom |= min(min(um[0], um[1]), min(um[2], um[3])) < 2u * kFastLiveHi;
    }
#pragma unroll
    for (int e = 0; e < N; ++e) d[off[e]] = a[e];
  }
  __syncthreads();
}

// Stages [j0, j1) over a tile of `count` (default 2^u) doubles in shared
// memory, in ceil(n / 4) passes of near-equal radix.
template <int W>
__device__ __forceinline__ void dense_stages_fast(double* d, uint32_t u, uint32_t P, int j0, int j1, DenseCtl<W>& dc,
                                                  unsigned long long& records, uint32_t count, uint32_t& anom) {
  const uint32_t npts = count ? count : (1u << u);
  const int ns = j1 - j0;
  if (ns <= 0) return;
  const int np = (ns + PP_DENSE_RADIX - 1) / PP_DENSE_RADIX, base = ns / np, extra = ns % np;
  uint32_t rec = 0;
  int j = j0;
  for (int p = 0; p < np; ++p) {
    const int r = base + (p < extra ? 1 : 0);
    uint32_t pm[4];
    double cs[4], sn[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int jj = i < r ? j + i : j;
      pm[i] = __popc(P & ((1u << dc.sbit[jj]) - 1u));
      cs[i] = dc.scos[jj];
      sn[i] = dc.ssin[jj];
    }
    if (r == 4) dense_fast_pass<4>(d, npts, pm, cs, sn, rec, anom);
    else if (r == 3) dense_fast_pass<3>(d, npts, pm, cs, sn, rec, anom);
    else if (r == 2) dense_fast_pass<2>(d, npts, pm, cs, sn, rec, anom);
    else dense_fast_pass<1>(d, npts, pm, cs, sn, rec, anom);
    j += r;
  }
  records += rec;
}

template <int W>
__device__ __forceinline__ void dense_stages(double* d, uint32_t u, uint32_t P, int j0, int j1, DenseCtl<W>& dc,
                                             unsigned long long& records, unsigned long long& removed,
                                             uint32_t count, uint32_t& anom, bool fast) {
  if (dc.tpred) dense_stages_t<W, true>(d, u, P, j0, j1, dc, records, removed, count, anom);
  else if (fast) dense_stages_fast<W>(d, u, P, j0, j1, dc, records, count, anom);
  else dense_stages_t<W, false>(d, u, P, j0, j1, dc, records, removed, count, anom);
}

// ---- bulk copies (TMA engine, cp.async.bulk) between a block in global
// memory and the shared-memory tile, completion on an mbarrier: one
// instruction moves a whole contiguous tile row, no registers, no LSU slots
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, uint32_t arrivals) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(arrivals));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "PP_MBAR_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra PP_MBAR_DONE;\n"
      "bra PP_MBAR_WAIT;\n"
      "PP_MBAR_DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst_smem, const void* src_global, uint32_t bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src_global), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst_global, const void* src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst_global), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void proxy_fence() { asm volatile("fence.proxy.async;" ::: "memory"); }

// Stages of a block of S > kDenseSmem points in global memory (L2): passes
// of up to kDenseSmemLog stages, each over full shared-memory tiles (the
// cosets of the pass's stage bits, padded with low bits).
template <int W>
__device__ void dense_passes(double* dbuf, double* blk, uint32_t S, DenseCtl<W>& dc, unsigned long long& records,
                             unsigned long long& removed, uint32_t& anom, bool fast) {
  const uint32_t tid = threadIdx.x;
  const int m = dc.m;
  for (int j0 = 0; j0 < m; j0 += (int)kDenseSmemLog) {
    const int j1 = min(m, j0 + (int)kDenseSmemLog);
    if (tid == 0) {
      // tile bits: this pass's stage bits, padded with the lowest other
      // bits to a full tile (coalesced gathers, several cosets per tile)
      uint32_t P = 0;
      for (int j = j0; j < j1; ++j) P |= 1u << dc.sbit[j];
      for (uint32_t b = 0; __popc(P) < (int)kDenseSmemLog; ++b) P |= 1u << b;
      dc.P = P;
    }
    __syncthreads();
    const uint32_t P = dc.P, u = kDenseSmemLog, Q = (S - 1u) & ~P;
    {  // deposit tables: tile index bits 0-6 and 7-12 into P
      uint32_t plo = P;
      for (int c = 0; c < 7; ++c) plo &= plo - 1;
      const uint32_t lo_mask = P & ~plo;
      if (tid < 128) dc.deplo[tid] = dense_dep32(tid, lo_mask);
      else if (tid < 192) dc.dephi[tid - 128] = dense_dep32(tid - 128, plo);
    }
    __syncthreads();
    // Tile rows: P's low bits up to its first gap are contiguous in the block,
    // 2^L points per row.  Rows of at least 512 bytes move as bulk copies (one
    // cp.async.bulk per row, completion on the CTA's mbarrier); shorter rows
    // element by element.
    const uint32_t L = (uint32_t)__ffs((int)~P) - 1u;
    const bool bulk = L >= 6 && (reinterpret_cast<uintptr_t>(blk) & 15u) == 0;
    const uint32_t rows = (1u << u) >> L, rbytes = 8u << L;
    if (bulk) proxy_fence();  // this thread's earlier writes to the block, before the copy engine reads it
    __syncthreads();
    for (uint32_t sp = 0; sp < (S >> u); ++sp) {
      const uint32_t base = dense_dep32(sp, Q);
      if (bulk) {
        if (tid == 0) {
          mbar_expect_tx(&dc.mbar, 8u << u);
          ++dc.bulk_tiles;
        }
        for (uint32_t r = tid; r < rows; r += kCta) {
          const uint32_t i = r << L;
          bulk_g2s(dbuf + i, blk + (base | dc.deplo[i & 127] | dc.dephi[i >> 7]), rbytes, &dc.mbar);
        }
        mbar_wait(&dc.mbar, dc.mphase & 1u);
        __syncthreads();
        if (tid == 0) dc.mphase ^= 1u;
      } else {
        // 8 loads in flight per thread (the block sits in L2)
        for (uint32_t i0 = 0; i0 < (1u << u); i0 += 8 * kCta) {
          double t[8];
#pragma unroll
          for (uint32_t e = 0; e < 8; ++e) {
            const uint32_t i = i0 + e * kCta + tid;
            t[e] = blk[base | dc.deplo[i & 127] | dc.dephi[i >> 7]];
          }
#pragma unroll
          for (uint32_t e = 0; e < 8; ++e) dbuf[i0 + e * kCta + tid] = t[e];
        }
        __syncthreads();
      }
      dense_stages<W>(dbuf, u, P, j0, j1, dc, records, removed, 0, anom, fast);
      if (bulk) {
        proxy_fence();  // the tile's generic-proxy writes, before the copy engine reads them
        __syncthreads();
        for (uint32_t r = tid; r < rows; r += kCta) {
          const uint32_t i = r << L;
          bulk_s2g(blk + (base | dc.deplo[i & 127] | dc.dephi[i >> 7]), dbuf + i, rbytes);
        }
        bulk_commit_wait();  // (threads without a row have nothing to wait for)
        proxy_fence();       // the block is read with ordinary loads again afterwards
      } else {
        for (uint32_t i = tid; i < (1u << u); i += kCta) blk[base | dc.deplo[i & 127] | dc.dephi[i >> 7]] = dbuf[i];
      }
      __syncthreads();
    }
  }
}

// Several x classes F_1 < ... < F_K (sorted as planes): one 2^m block each,
// written class-major -- block i holds class F_i in b (= x) order, at
// [i 2^m, (i + 1) 2^m) of the group's region (zeros included, then holes are
// compacted out in place).  The group's x order would interleave the blocks,
// so the group is marked kFlagUnsorted like the output of a regroup (nothing
// on the eps0 = 0 pipeline needs x order: the next regroup and the next dense
// run scatter anyway; consumers that do sort first, EngineImpl::ensure_sorted)
// plus kFlagMinFirst: the group's smallest x (class F_1 at b = 0, the only
// place x = 0 can be) still comes first, which is all the readout needs.
template <int W>
__device__ int dense_multi(double* dbuf, DenseCtl<W>& dc, GroupStatsSmem& gs, uint32_t* scan, GroupView<W> g,
                           ArenaView<W> ar, uint32_t gid, uint32_t n, uint64_t src, uint32_t K, uint32_t seq0,
                           unsigned long long cap, DevStats* st, unsigned long long& aff_elems,
                           const uint32_t* s_touch, uint32_t* s_seen) {
  const uint32_t tid = threadIdx.x;
  const int m = dc.m;
  const Plane<W> T = dc.T;
  DenseTail<W>& tl = *reinterpret_cast<DenseTail<W>*>(dbuf + kDenseSmem);
  const Plane<W>* xt = tl.xt;
  const uint32_t S = 1u << m;
  const unsigned long long KS = (unsigned long long)K * S;
  if (KS > kDenseMaxOut) return 0;
  // region: K 2^m output slots (from an even offset: the output is written
  // two points per 128-bit store), a 2^m scratch block for blocks larger than
  // a shared-memory tile, and the strings' (class, point) codes: unsorted
  // with their rank inside the class, then sorted by class with the values
  const bool big = S > kDenseSmem;
  const bool one_tile = KS <= kDenseSmem;  // every class block in one shared-memory tile: no codes, no sort
  const unsigned long long Sx = big ? S : 0;
  const unsigned long long need = KS + Sx + (one_tile ? 0ull : 2ull * n) + 1;
  if (tid == 0) {
    const unsigned long long d = atomicAdd(&st->bump, need);
    dc.dst = (d + 1) & ~1ull;
    dc.fail = d + need > cap;
    if (dc.fail) {
      atomicOr(&st->err_arena, 1u);
      atomicMin(&st->err_seq, (unsigned long long)(seq0 + dc.sgate[0]));
    }
    dc.zeros = 0;
  }
  if (tid < K) tl.ccnt[tid] = 0;
  __syncthreads();
  if (dc.fail) return -1;
  const uint64_t dst = dc.dst;
  unsigned long long records = 0, removed = 0;
  double vmax = 0.0, vmin = __longlong_as_double(0x7ff0000000000000ll), vall = 0.0;
  uint32_t nonfinite = 0, zeros = 0;
  const bool spec = dc.tpred != nullptr;
  // points (i, b) and (i, b + 1), b even -> [dst + i 2^m + b, + 2) as one
  // 128-bit store per plane word and one for the coefficients
  auto note = [&](double v) {
    if (v == 0.0) {
      ++zeros;
    } else {
      const double av = fabs(v);
      if (!(av <= 1.7976931348623157e308)) nonfinite = 1;
      vmax = fmax(vmax, av);
      vmin = fmin(vmin, av);
    }
  };
  auto emit2 = [&](uint32_t i, uint32_t b, double v0, double v1) {
    if (spec) {  // the last window's truncation
      if (v0 != 0.0 && fabs(v0) <= dc.strunc[m - 1]) {
        v0 = 0.0;
        ++removed;
      }
      if (v1 != 0.0 && fabs(v1) <= dc.strunc[m - 1]) {
        v1 = 0.0;
        ++removed;
      }
    }
    const uint64_t r = dst + ((uint64_t)i << m) + b;  // class-major: block i holds class F_i in b order
    Plane<W> hi = tl.sF[i];
    const Plane<W> a1 = xt[256 + ((b >> 8) & 255u)], a2 = xt[512 + (b >> 16)];
    const Plane<W> l0 = xt[b & 255u], l1 = xt[(b & 255u) + 1u];
#pragma unroll
    for (int w = 0; w < W; ++w) {
      hi.w[w] |= a1.w[w] | a2.w[w];
      *reinterpret_cast<ulonglong2*>(ar.x[w] + r) = make_ulonglong2(hi.w[w] | l0.w[w], hi.w[w] | l1.w[w]);
    }
    *reinterpret_cast<double2*>(ar.c + r) = make_double2(v0, v1);
    note(v0);
    note(v1);
  };
  // each string's class (its slot in the class hash set; the stored F is
  // compared here, a fingerprint collision sends the group to the per-gate
  // path), point and rank inside its class, once
  uint64_t* codes = ar.x[0] + dst + KS;        // class << 56 | rank << 24 | point
  uint64_t* scodes = codes + n;                // sorted by class: class << 32 | point
  double* svals = ar.c + dst + KS + Sx + n;    //   and the values
  if (one_tile) {
    // the usual case: strings go straight to their points of the tile
    const uint32_t cnt = (uint32_t)KS;
    const unsigned long long rec0 = records;
    for (bool fast = dc.fast != 0;; fast = false) {
      for (uint32_t e = 2 * tid; e < cnt; e += 2 * kCta) *reinterpret_cast<double2*>(dbuf + e) = make_double2(0.0, 0.0);
      __syncthreads();
      bool bad = false;
      for (uint32_t i = tid; i < n; i += kCta) {
        const Plane<W> x = load_plane<W>(ar.x, src + i);
        const double v = ar.c[src + i];
        Plane<W> f = x;
#pragma unroll
        for (int w = 0; w < W; ++w) f.w[w] &= ~T.w[w];
        const unsigned long long fp = plane_hash<W>(f, 0x9e3779b97f4a7c15ull) | 1ull;
        uint32_t h = (uint32_t)(fp >> 40) & (kDenseSlots - 1);
        while (tl.hfp[h] != fp) h = (h + 1) & (kDenseSlots - 1);
        bad |= !plane_eq<W>(tl.hF[h], f);
        if (spec && v != 0.0 && fabs(v) <= dc.tin) {
          ++removed;
          continue;
        }
        dbuf[((uint32_t)tl.hcls[h] << m) + dense_pext<W>(x, T)] = v;
      }
      if (__syncthreads_or(bad)) return 0;  // a fingerprint collision (the region is given up)
      uint32_t anom = 0;
      dense_stages<W>(dbuf, (uint32_t)m, S - 1u, 0, m, dc, records, removed, cnt, anom, fast);
      if (!fast || !__syncthreads_or(anom)) break;
      records = rec0;  // a cancellation or an extreme value: redo point by point
    }
    for (uint32_t e = 2 * tid; e < cnt; e += 2 * kCta) {
      const double2 v = *reinterpret_cast<const double2*>(dbuf + e);
      emit2(e >> m, e & (S - 1u), v.x, v.y);
    }
  } else {
  {
    bool bad = false;
    for (uint32_t i = tid; i < n; i += kCta) {
      const Plane<W> x = load_plane<W>(ar.x, src + i);
      Plane<W> f = x;
#pragma unroll
      for (int w = 0; w < W; ++w) f.w[w] &= ~T.w[w];
      const unsigned long long fp = plane_hash<W>(f, 0x9e3779b97f4a7c15ull) | 1ull;
      uint32_t h = (uint32_t)(fp >> 40) & (kDenseSlots - 1);
      while (tl.hfp[h] != fp) h = (h + 1) & (kDenseSlots - 1);
      bad |= !plane_eq<W>(tl.hF[h], f);
      const uint32_t c = tl.hcls[h];
      const uint32_t rk = atomicAdd(&tl.ccnt[c], 1u);
      codes[i] = ((uint64_t)c << 56) | ((uint64_t)rk << 24) | dense_pext<W>(x, T);
    }
    if (__syncthreads_or(bad)) return 0;  // (the region is given up)
  }
  {  // class start offsets
    uint32_t tot;
    const uint32_t c = tid < K ? tl.ccnt[tid] : 0u;
    const uint32_t o = block_excl_scan(c, scan, &tot);
    __syncthreads();
    if (tid < K) tl.ccnt[tid] = o;
    if (tid == 0) tl.ccnt[K] = n;
    __syncthreads();
  }
  for (uint32_t i = tid; i < n; i += kCta) {
    const uint64_t code = codes[i];
    const double v = ar.c[src + i];
    const uint32_t c = (uint32_t)(code >> 56);
    const uint32_t pos = tl.ccnt[c] + (uint32_t)((code >> 24) & 0xffffffffu);
    scodes[pos] = ((uint64_t)c << 32) | (code & 0xffffffu);
    svals[pos] = v;
  }
  __syncthreads();
  if (!big) {
    // batches of whole class blocks in one shared-memory tile
    const uint32_t per = kDenseSmem / S;
    for (uint32_t c0 = 0; c0 < K; c0 += per) {
      const uint32_t c1 = min(K, c0 + per), cnt = (c1 - c0) * S;
      const uint32_t j0 = tl.ccnt[c0], j1 = tl.ccnt[c1];
      const unsigned long long rec0 = records;
      for (bool fast = dc.fast != 0;; fast = false) {
        for (uint32_t e = 2 * tid; e < cnt; e += 2 * kCta) *reinterpret_cast<double2*>(dbuf + e) = make_double2(0.0, 0.0);
        __syncthreads();
        for (uint32_t j = j0 + tid; j < j1; j += kCta) {
          const uint64_t code = scodes[j];
          const double v = svals[j];
          if (spec && v != 0.0 && fabs(v) <= dc.tin) {
            ++removed;
            continue;
          }
          dbuf[((uint32_t)(code >> 32) - c0) * S + (uint32_t)code] = v;
        }
        __syncthreads();
        uint32_t anom = 0;
        dense_stages<W>(dbuf, (uint32_t)m, S - 1u, 0, m, dc, records, removed, cnt, anom, fast);
        if (!fast || !__syncthreads_or(anom)) break;
        records = rec0;  // a cancellation or an extreme value: redo the batch point by point
      }
      for (uint32_t e = 2 * tid; e < cnt; e += 2 * kCta) {
        const double2 v = *reinterpret_cast<const double2*>(dbuf + e);
        emit2(c0 + (e >> m), e & (S - 1u), v.x, v.y);
      }
      __syncthreads();
    }
  } else {
    double* blk = ar.c + dst + KS;  // scratch block (coefficient plane past the output)
    for (uint32_t ci = 0; ci < K; ++ci) {
      const uint32_t j0 = tl.ccnt[ci], j1 = tl.ccnt[ci + 1];
      const unsigned long long rec0 = records;
      for (bool fast = dc.fast != 0;; fast = false) {
        for (uint32_t e = 2 * tid; e < S; e += 2 * kCta) *reinterpret_cast<double2*>(blk + e) = make_double2(0.0, 0.0);
        __syncthreads();
        for (uint32_t j = j0 + tid; j < j1; j += kCta) {
          const uint64_t code = scodes[j];
          const double v = svals[j];
          if (spec && v != 0.0 && fabs(v) <= dc.tin) {
            ++removed;
            continue;
          }
          blk[(uint32_t)code] = v;
        }
        __syncthreads();
        uint32_t anom = 0;
        dense_passes<W>(dbuf, blk, S, dc, records, removed, anom, fast);
        if (!fast || !__syncthreads_or(anom)) break;
        records = rec0;
      }
      for (uint32_t e = 2 * tid; e < S; e += 2 * kCta) {
        const double2 v = *reinterpret_cast<const double2*>(blk + e);
        emit2(ci, e, v.x, v.y);
      }
      __syncthreads();
    }
  }
  }
  // holes (zero points): compact [dst, dst + KS) in place, in rank order
  if (zeros) atomicAdd(&dc.zeros, zeros);
  __syncthreads();
  uint32_t out = (uint32_t)KS;
  if (dc.zeros) {
    out = 0;
    const uint32_t lane = tid & 31, warp = tid >> 5;
    for (unsigned long long base = 0; base < KS; base += kCta) {
      const unsigned long long r = base + tid;
      double v = 0.0;
      Plane<W> x;
      if (r < KS) {
        v = ar.c[dst + r];
        x = load_plane<W>(ar.x, dst + r);
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, v != 0.0);
      if (lane == 0) scan[warp] = __popc(bal);
      __syncthreads();
      if (warp == 0) {
        const uint32_t c = lane < kWarps ? scan[lane] : 0u;
        const uint32_t inc = warp_incl_scan(c);
        if (lane < kWarps) scan[lane] = inc - c;
        if (lane == kWarps - 1) scan[kWarps] = inc;
      }
      __syncthreads();
      if (v != 0.0) {
        const uint32_t o = out + scan[warp] + __popc(bal & ((1u << lane) - 1u));
        store_plane<W>(ar.x, dst + o, x);
        ar.c[dst + o] = v;
      }
      out += scan[kWarps];
      __syncthreads();
    }
  }
  reduce_group_stats_t0(gs, vmax, vmin, vall, nonfinite, records, removed);
  if (tid == 0) {
    g.off[gid] = dst;
    g.cnt[gid] = out;
    g.cap[gid] = (uint32_t)KS;
    g.gmax[gid] = out ? vmax : 0.0;
    g.gmin[gid] = out ? vmin : __longlong_as_double(0x7ff0000000000000ll);
    g.flags[gid] = nonfinite | kFlagUnsorted | kFlagMinFirst;
    g.stamp[gid] = seq0 + (uint32_t)dc.klast;
    if (records) {
      atomicAdd(&st->records, records);
      for (int w = 0; w < kMaxSubGates / 32; ++w) atomicOr(&s_seen[w], s_touch[w]);
    }
    if (removed) atomicAdd(&st->removed, removed);
    atomicAdd(&st->out_elems, (unsigned long long)out);
    atomicAdd(&st->dense_groups, 1ull);
    atomicAdd(&st->dense_out, (unsigned long long)out);
  }
  aff_elems += n;
  return 1;
}

// The group's stage list is in dc (T, m, sbit/sgate/scos/ssin, tpos, klast,
// fast, F of its first string; spec: tin, strunc): x classes, output tables,
// then the butterflies and the output (dense_multi for several classes).
// Returns like dense_group.
template <int W>
__device__ int dense_apply(double* dbuf, DenseCtl<W>& dc, GroupStatsSmem& gs, uint32_t* scan, GroupView<W> g,
                           ArenaView<W> ar, const SubGates& gates, uint32_t gid, uint32_t n, uint64_t src,
                           const uint32_t* s_touch, uint32_t seq0, unsigned long long cap, DevStats* st,
                           unsigned long long& aff_elems, uint32_t* s_seen) {
  const uint32_t tid = threadIdx.x;
  const int m = dc.m;
  const Plane<W> T = dc.T;
  const bool spec = dc.tpred != nullptr;
  DenseTail<W>& tl = *reinterpret_cast<DenseTail<W>*>(dbuf + kDenseSmem);
  uint32_t K = 1;
  Plane<W> F = dc.F;  // one string: one class, its x outside T
  // b -> x bits outside F, one table per byte of b
  Plane<W>* xt = tl.xt;
  for (uint32_t e = tid; e < (uint32_t)((m + 7) / 8) * 256u; e += kCta) {
    Plane<W> p;
#pragma unroll
    for (int w = 0; w < W; ++w) p.w[w] = 0;
    const uint32_t j0 = 8 * (e >> 8);
    for (uint32_t bit = 0; bit < 8; ++bit)
      if (j0 + bit < (uint32_t)m && ((e >> bit) & 1u)) {
        const uint32_t q = dc.tpos[j0 + bit];
        p.w[q >> 6] |= 1ull << (q & 63);
      }
    xt[e] = p;
  }
  if (tid < 3 && tid >= (uint32_t)((m + 7) / 8)) {  // tables past b's bytes: only entry 0 is read
    Plane<W> z0;
#pragma unroll
    for (int w = 0; w < W; ++w) z0.w[w] = 0;
    xt[256 * tid] = z0;
  }
  if (n > 1) {
    // x classes (the distinct x parts F outside T): a shared-memory hash set
    // keyed by a fingerprint of F; the stored F is compared when the strings
    // are placed (dense_multi; one class: below) -- a fingerprint collision
    // sends the group to the per-gate path
    for (uint32_t sl = tid; sl < kDenseSlots; sl += kCta) tl.hfp[sl] = 0ull;
    if (tid == 0) tl.nused = 0;
    __syncthreads();
    bool ok = true;
    for (uint32_t i = tid; i < n; i += kCta) {
      Plane<W> f = load_plane<W>(ar.x, src + i);
  #pragma unroll
      for (int w = 0; w < W; ++w) f.w[w] &= ~T.w[w];
      const unsigned long long fp = plane_hash<W>(f, 0x9e3779b97f4a7c15ull) | 1ull;
      uint32_t h = (uint32_t)(fp >> 40) & (kDenseSlots - 1);
      for (uint32_t probe = 0;; ++probe, h = (h + 1) & (kDenseSlots - 1)) {
        if (probe == kDenseSlots) {
          ok = false;  // more than kDenseSlots classes
          break;
        }
        const unsigned long long old = atomicCAS(&tl.hfp[h], 0ull, fp);
        if (old == 0ull) tl.hF[h] = f;
        if (old == 0ull || old == fp) break;
      }
    }
    __syncthreads();
    // the occupied slots, in any order (the classes are ranked by F below)
    static_assert(kDenseSlots == 2 * kCta, "two hash slots per thread");
    if (tl.hfp[2 * tid] != 0ull) tl.used[atomicAdd(&tl.nused, 1u)] = (uint16_t)(2 * tid);
    if (tl.hfp[2 * tid + 1] != 0ull) tl.used[atomicAdd(&tl.nused, 1u)] = (uint16_t)(2 * tid + 1);
    if (!__syncthreads_and(ok)) return 0;
    K = tl.nused;
    if (K > kDenseMaxK || K > (uint32_t)gates.maxk) return 0;
    if (K == 1) {
      for (uint32_t i = tid; i < n && ok; i += kCta) {
        Plane<W> f = load_plane<W>(ar.x, src + i);
#pragma unroll
        for (int w = 0; w < W; ++w) f.w[w] &= ~T.w[w];
        const unsigned long long fp = plane_hash<W>(f, 0x9e3779b97f4a7c15ull) | 1ull;
        uint32_t h = (uint32_t)(fp >> 40) & (kDenseSlots - 1);
        while (tl.hfp[h] != fp) h = (h + 1) & (kDenseSlots - 1);
        ok = plane_eq<W>(tl.hF[h], f);
      }
      if (!__syncthreads_and(ok)) return 0;
    }
    // classes in ascending F order; class index per slot
    for (uint32_t c = tid; c < K; c += kCta) {
      const uint32_t sl = tl.used[c];
      const Plane<W> f = tl.hF[sl];
      uint32_t r = 0;
      for (uint32_t j = 0; j < K; ++j) r += plane_lt<W>(tl.hF[tl.used[j]], f);
      tl.hcls[sl] = (uint8_t)r;
      tl.sF[r] = f;
    }
    __syncthreads();
    F = tl.sF[0];
  } else {
    __syncthreads();
  }
  if (K > 1) return dense_multi<W>(dbuf, dc, gs, scan, g, ar, gid, n, src, K, seq0, cap, st, aff_elems, s_touch, s_seen);
  const uint32_t S = 1u << m;
  if (tid == 0) {
    const unsigned long long d = atomicAdd(&st->bump, (unsigned long long)S);
    dc.dst = d;
    dc.fail = d + S > cap;
    if (dc.fail) {
      atomicOr(&st->err_arena, 1u);
      atomicMin(&st->err_seq, (unsigned long long)(seq0 + dc.sgate[0]));
    }
  }
  __syncthreads();
  if (dc.fail) return -1;
  const uint64_t dst = dc.dst;
  unsigned long long records = 0, removed = 0;
  double vmax = 0.0, vmin = __longlong_as_double(0x7ff0000000000000ll), vall = 0.0;
  uint32_t nonfinite = 0;
  uint32_t out = 0;
  bool done = false;
  if (n == 1 && !spec) {
    // One string: output point b is the input coefficient times one factor
    // per stage -- cos where b keeps the string's bit, the signed sin where it
    // flips it (+sin from a Z, -sin from a Y) -- multiplied in gate order,
    // exactly the products the butterflies form (no point ever receives two
    // contributions).  Valid when no point ends at zero; then every stage's
    // deltas are nonzero: records = 2^m - 1, nothing removed.
    // The products share prefixes: with c the point's bits in stage order,
    // P_{j+1}[c mod 2^{j+1}] = P_j[c mod 2^j] * f_j(bit j of c).  The first
    // L = min(m, 13) stages build P_L in shared memory (2^{L+1} products);
    // each output point multiplies its P_L by its remaining m - L factors.
    const double c0 = ar.c[src];
    const uint32_t b0 = dense_pext<W>(load_plane<W>(ar.x, src), T);
    const int L = m < (int)kDenseSmemLog ? m : (int)kDenseSmemLog;
    // b (x order) -> c (stage order), one table per byte of b; the class hash
    // storage is free on this path
    uint32_t* cperm = reinterpret_cast<uint32_t*>(tl.hF);
    static_assert(sizeof(DenseTail<1>::hF) >= 3 * 256 * sizeof(uint32_t), "cperm fits the class hash keys");
    for (uint32_t e = tid; e < 3 * 256; e += kCta) {
      if ((e & 255u) && (e >> 8) >= (uint32_t)((m + 7) / 8)) continue;  // only entry 0 of unused tables
      uint32_t c = 0;
      const uint32_t t0 = 8 * (e >> 8);
      for (int j = 0; j < m; ++j) {
        const uint32_t t = dc.sbit[j];
        if (t >= t0 && t < t0 + 8 && ((e >> (t - t0)) & 1u)) c |= 1u << j;
      }
      cperm[e] = c;
    }
    // the first stages (<= 256 products) by warp 0 alone, the rest by the CTA
    const int Lw = L < 8 ? L : 8;
    if (tid < 32) {
      if (tid == 0) dbuf[0] = c0;
      __syncwarp();
      for (int j = 0; j < Lw; ++j) {
        const uint32_t bit = 1u << dc.sbit[j];
        const double fk = dc.scos[j], ff = (b0 & bit) ? -dc.ssin[j] : dc.ssin[j];  // keep / flip the string's bit
        const double f0 = (b0 & bit) ? ff : fk, f1 = (b0 & bit) ? fk : ff;           // stage bit 0 / 1
        for (uint32_t p = tid; p < (1u << j); p += 32) {
          const double v = dbuf[p];
          dbuf[p + (1u << j)] = __dmul_rn(v, f1);
          dbuf[p] = __dmul_rn(v, f0);
        }
        __syncwarp();
      }
    }
    __syncthreads();
    for (int j = Lw; j < L; ++j) {
      const uint32_t bit = 1u << dc.sbit[j];
      const double fk = dc.scos[j], ff = (b0 & bit) ? -dc.ssin[j] : dc.ssin[j];  // keep / flip the string's bit
      const double f0 = (b0 & bit) ? ff : fk, f1 = (b0 & bit) ? fk : ff;           // stage bit 0 / 1
      for (uint32_t p = tid; p < (1u << j); p += kCta) {
        const double v = dbuf[p];
        dbuf[p + (1u << j)] = __dmul_rn(v, f1);
        dbuf[p] = __dmul_rn(v, f0);
      }
      __syncthreads();
    }
    bool zero = false;
    for (uint32_t b = tid; b < S; b += kCta) {
      const uint32_t c = cperm[b & 255u] | cperm[256 + ((b >> 8) & 255u)] | cperm[512 + (b >> 16)];
      double v = dbuf[c & ((1u << L) - 1u)];
      for (int j = L; j < m; ++j) {
        const uint32_t bit = 1u << dc.sbit[j];
        const double f = ((c >> j) & 1u) != ((b0 & bit) != 0u) ? ((b0 & bit) ? -dc.ssin[j] : dc.ssin[j])
                                                                : dc.scos[j];
        v = __dmul_rn(v, f);
      }
      zero |= v == 0.0;
      Plane<W> x = F;
      const Plane<W> a0 = xt[b & 255u], a1 = xt[256 + ((b >> 8) & 255u)], a2 = xt[512 + (b >> 16)];
#pragma unroll
      for (int w = 0; w < W; ++w) x.w[w] |= a0.w[w] | a1.w[w] | a2.w[w];
      store_plane<W>(ar.x, dst + b, x);
      ar.c[dst + b] = v;
      const double av = fabs(v);
      if (!(av <= 1.7976931348623157e308)) nonfinite = 1;
      vmax = fmax(vmax, av);
      vmin = fmin(vmin, av);
    }
    if (!__syncthreads_or(zero)) {
      done = true;
      out = S;
      if (tid == 0) records = S - 1;
    } else {  // an underflow or a zero angle: the general path below
      vmax = 0.0;
      vmin = __longlong_as_double(0x7ff0000000000000ll);
      nonfinite = 0;
    }
  }
  if (!done) {
    const bool in_smem = S <= kDenseSmem;
    double* blk = in_smem ? dbuf : ar.c + dst;  // the dense block
    const unsigned long long rec0 = records;
    for (bool fast = dc.fast != 0;; fast = false) {
      for (uint32_t i = tid; i < S; i += kCta) blk[i] = 0.0;
      __syncthreads();
      for (uint32_t i = tid; i < n; i += kCta) {
        const double c = ar.c[src + i];
        if (spec && c != 0.0 && fabs(c) <= dc.tin) {  // truncated before the first stage
          ++removed;
          continue;
        }
        blk[dense_pext<W>(load_plane<W>(ar.x, src + i), T)] = c;
      }
      __syncthreads();
      uint32_t anom = 0;
      if (in_smem) {
        dense_stages<W>(dbuf, (uint32_t)m, S - 1u, 0, m, dc, records, removed, 0, anom, fast);
      } else {
        dense_passes<W>(dbuf, blk, S, dc, records, removed, anom, fast);
      }
      if (!fast || !__syncthreads_or(anom)) break;
      records = rec0;  // a cancellation or an extreme value: redo point by point
    }
    // nonzero points in b (= x) order, compacted into the output region (in
    // place for a block in global memory: a tile's writes land at or below its
    // own positions, after all of its reads)
    constexpr uint32_t kPer = 8;  // 8 loads in flight per thread per tile
    const uint32_t lane = tid & 31, warp = tid >> 5;
    uint32_t* ocnt = reinterpret_cast<uint32_t*>(dc.deplo);  // kPer x kWarps counts (+ total); passes are done
    for (uint32_t base = 0; base < S; base += kCta * kPer) {
      double v[kPer];
      uint32_t bal[kPer];
  #pragma unroll
      for (uint32_t e = 0; e < kPer; ++e) {  // striped: slot e covers [base + e kCta, base + (e+1) kCta)
        const uint32_t b = base + e * kCta + tid;
        v[e] = b < S ? blk[b] : 0.0;
        if (spec && v[e] != 0.0 && fabs(v[e]) <= dc.strunc[m - 1]) {  // the last window's truncation
          v[e] = 0.0;
          ++removed;
        }
      }
  #pragma unroll
      for (uint32_t e = 0; e < kPer; ++e) {
        bal[e] = __ballot_sync(0xffffffffu, v[e] != 0.0);
        if (lane == 0) ocnt[e * kWarps + warp] = __popc(bal[e]);
      }
      __syncthreads();
      if (warp == 0) {  // exclusive scan of the kPer x kWarps counts (b order), 2 per lane
        static_assert(kPer * kWarps == 64, "two counts per lane");
        const uint32_t c0 = ocnt[2 * lane], c1 = ocnt[2 * lane + 1];
        const uint32_t inc = warp_incl_scan(c0 + c1);
        ocnt[2 * lane] = inc - c0 - c1;
        ocnt[2 * lane + 1] = inc - c1;
        if (lane == 31) ocnt[64] = inc;
      }
      __syncthreads();
  #pragma unroll
      for (uint32_t e = 0; e < kPer; ++e) {
        if (v[e] == 0.0) continue;
        const uint32_t b = base + e * kCta + tid;
        const uint32_t o = out + ocnt[e * kWarps + warp] + __popc(bal[e] & ((1u << lane) - 1u));
        Plane<W> x = F;
        const Plane<W> a0 = xt[b & 255u], a1 = xt[256 + ((b >> 8) & 255u)], a2 = xt[512 + (b >> 16)];
  #pragma unroll
        for (int w = 0; w < W; ++w) x.w[w] |= a0.w[w] | a1.w[w] | a2.w[w];
        store_plane<W>(ar.x, dst + o, x);
        ar.c[dst + o] = v[e];
        const double av = fabs(v[e]);
        if (!(av <= 1.7976931348623157e308)) nonfinite = 1;
        vmax = fmax(vmax, av);
        vmin = fmin(vmin, av);
      }
      out += ocnt[kPer * kWarps];
      __syncthreads();
    }
  }
  reduce_group_stats_t0(gs, vmax, vmin, vall, nonfinite, records, removed);
  if (tid == 0) {
    g.off[gid] = dst;
    g.cnt[gid] = out;
    g.cap[gid] = S;
    g.gmax[gid] = out ? vmax : 0.0;
    g.gmin[gid] = out ? vmin : __longlong_as_double(0x7ff0000000000000ll);
    g.flags[gid] = nonfinite;
    g.stamp[gid] = seq0 + (uint32_t)dc.klast;
    if (records) {
      atomicAdd(&st->records, records);
      for (int w = 0; w < kMaxSubGates / 32; ++w) atomicOr(&s_seen[w], s_touch[w]);
    }
    if (removed) atomicAdd(&st->removed, removed);
    atomicAdd(&st->out_elems, (unsigned long long)out);
    atomicAdd(&st->dense_groups, 1ull);
    atomicAdd(&st->dense_out, (unsigned long long)out);
  }
  aff_elems += n;
  return 1;
}

// Returns 1 when the group was applied, 0 when it is not eligible (the
// caller takes the per-gate path), -1 when its output did not fit the arena
// (the group is untouched and resumes in the next launch).
template <int W>
__device__ int dense_group(double* dbuf, DenseCtl<W>& dc, GroupStatsSmem& gs, uint32_t* scan, GroupView<W> g,
                           ArenaView<W> ar, const SubGates& gates, const SubGates& gp, uint32_t gid, uint32_t n, uint64_t src, int k0,
                           const uint32_t* s_touch, uint32_t seq0, unsigned long long cap, DevStats* st,
                           unsigned long long& aff_elems, uint32_t* s_seen) {
  const uint32_t tid = threadIdx.x;
  // stage list, in parallel: thread k owns gate k (parameters read from the
  // kernel's parameter block once per gate, not serially per group)
  __syncthreads();
  if (tid < W) dc.T.w[tid] = 0;
  if (tid < kMaxSubGates / 32) {
    const uint32_t w0 = (uint32_t)k0 >> 5;
    uint32_t t = tid < w0 ? 0u : s_touch[tid];
    if (tid == w0) t &= ~0u << (k0 & 31);
    dc.tw[tid] = t;
  }
  __syncthreads();
  const int k = (int)tid;
  const bool touch = k < gates.ng && ((dc.tw[k >> 5] >> (k & 31)) & 1u);
  int wq = 0;
  uint64_t mq = 0;
  if (touch) {
    wq = gp.wq[k];
    mq = gp.mq[k];
    atomicOr(reinterpret_cast<unsigned long long*>(&dc.T.w[wq]), (unsigned long long)mq);
  }
  __syncthreads();
  if (touch) {
    const Plane<W> T = dc.T;
    uint32_t r = __popcll(T.w[wq] & (mq - 1));
    for (int w = 0; w < wq; ++w) r += __popcll(T.w[w]);
    uint32_t j = __popc(dc.tw[k >> 5] & ((1u << (k & 31)) - 1u));
    for (int w = 0; w < (k >> 5); ++w) j += __popc(dc.tw[w]);
    if (j < kMaxSubGates) {
      dc.sbit[j] = (uint8_t)r;
      dc.sgate[j] = (uint8_t)k;
      dc.scos[j] = gp.cosv[k];
      dc.ssin[j] = gp.sinv[k];
    }
  }
  if (tid == 0) {
    int m = 0, klast = -1;
    for (int w = 0; w < kMaxSubGates / 32; ++w) {
      m += __popc(dc.tw[w]);
      if (dc.tw[w]) klast = 32 * w + 31 - __clz(dc.tw[w]);
    }
    dc.m = m;
    dc.klast = klast;
    Plane<W> F = load_plane<W>(ar.x, src);
#pragma unroll
    for (int w = 0; w < W; ++w) F.w[w] &= ~dc.T.w[w];
    dc.F = F;
    uint32_t j = 0;
#pragma unroll
    for (int w = 0; w < W; ++w)
      for (uint64_t t = dc.T.w[w]; t && j < 32; t &= t - 1, ++j) dc.tpos[j] = (uint8_t)(64 * w + __ffsll((long long)t) - 1);
  }
  __syncthreads();
  const int m = dc.m;
  if (m == 0 || m > kDenseMaxLog) return 0;
  // bookkeeping-free butterflies (dense_stages_fast) when the run's angles and
  // the group's values are far from underflow; anything else is caught there
  if (tid == 0) dc.fast = (!dc.tpred && gates.fast && g.gmin[gid] >= kFastLive) ? 1u : 0u;
  const Plane<W> T = dc.T;
  const bool spec = dc.tpred != nullptr;
  if (spec) {
    // truncation windows: after stage s, the gates from its own to the next
    // stage's (exclusive); before stage 0, the gates from k0 to its
    if (tid < (uint32_t)m) {
      const int k = dc.sgate[tid], next = (int)tid + 1 < m ? dc.sgate[tid + 1] : dc.ng;
      double t = -1.0;
      for (int jj = k; jj < next; ++jj) t = fmax(t, dc.tpred[jj]);
      dc.strunc[tid] = t;
    }
    if (tid == 0) {
      double t = -1.0;
      const int first = dc.sgate[0];
      const double M = g.gmax[gid];  // the group held its values through those gates
      for (int jj = k0; jj < first; ++jj) {
        t = fmax(t, dc.tpred[jj]);
        if (M > 0.0) atomicMax(&dc.smax[jj], (unsigned long long)__double_as_longlong(M));
        if (M <= dc.tpred[jj]) break;  // emptied: later gates see nothing (t already covers M)
      }
      dc.tin = t;
    }
    __syncthreads();
  }
  return dense_apply<W>(dbuf, dc, gs, scan, g, ar, gates, gid, n, src, s_touch, seq0, cap, st, aff_elems, s_seen);
}

// Modes:
//  tpred == nullptr  (epsilon0 = 0, or per-layer cadence): only groups some
//    gate touches; no truncation inside the run; resumable via stamps.
//  tpred != nullptr  (per-gate cadence, epsilon0 > 0, speculative): every
//    group; gate k truncates with the PREDICTED threshold tpred[k]; the max
//    |c| after each gate's apply (before its truncation) is max-reduced into
//    gmax_out[k] over all groups (untouched groups contribute their current
//    max).  All writes go to fresh arena space, so the host can verify
//    eps * gmax_out[k] == tpred[k] for every k and otherwise roll the group
//    table back and rerun with the observed thresholds.
template <int W>
__global__ void __launch_bounds__(kCta, 2) k_branch_sublayer(GroupView<W> g, ArenaView<W> ar, const SubGates gates,
                                                           int keep_zeros, unsigned int* work, const double* tpred,
                                                           unsigned long long* gmax_out, DevStats* st,
                                                           const uint8_t* spec_done = nullptr,
                                                           const uint32_t* list = nullptr) {
  __shared__ uint32_t s_touch[kMaxSubGates / 32];
  __shared__ uint32_t s_seen[kMaxSubGates / 32];  // gates of the run that sent a record (batches_sent)
  extern __shared__ __align__(16) unsigned char smem_raw[];
  BranchSmem<W>& sm = *reinterpret_cast<BranchSmem<W>*>(smem_raw);
  SegSmem<W>& sg = *reinterpret_cast<SegSmem<W>*>(smem_raw);
  const uint32_t tid = threadIdx.x;
  if (engine_failed(st)) return;
  if (tid < kMaxSubGates / 32) s_seen[tid] = 0;
  const bool spec = tpred != nullptr;
  // list != nullptr: only the groups k_dense_sublayer left behind (pp_dense.cuh)
  const uint32_t G = list ? *(volatile const unsigned int*)&st->left_n : *(volatile const unsigned int*)&st->G_dev;
  if (G == 0) return;
  const unsigned long long cap = *(volatile const unsigned long long*)&st->arena_cap;
  const uint32_t seq0 = (uint32_t)(*(volatile const unsigned long long*)&st->seq_base);
  __shared__ unsigned long long dst_s;
  __shared__ uint32_t s_gid, s_fail;
  __shared__ GroupStatsSmem gs;
  __shared__ unsigned long long smax[kMaxSubGates];  // per-CTA per-gate max (bits)
  __shared__ uint32_t tscan[40];
  __shared__ DenseCtl<W> dc;
  __shared__ SubGates s_gp;  // the run's gates, read from the parameter block once per CTA
  for (int k = tid; k < gates.ng; k += kCta) {
    smax[k] = 0ull;
    s_gp.wq[k] = gates.wq[k];
    s_gp.mq[k] = gates.mq[k];
    s_gp.cosv[k] = gates.cosv[k];
    s_gp.sinv[k] = gates.sinv[k];
  }
  __shared__ double s_tpred[kMaxSubGates];
  if (tpred)
    for (int k = tid; k < gates.ng; k += kCta) s_tpred[k] = tpred[k];
  if (tid == 0) {
    s_gp.ng = gates.ng;
    dc.tpred = tpred ? s_tpred : nullptr;
    dc.smax = smax;
    dc.ng = gates.ng;
    mbar_init(&dc.mbar, 1);
    dc.mphase = 0;
    dc.bulk_tiles = 0;
  }
  __syncthreads();
  unsigned long long aff_elems = 0;
  bool failed = false;
  // contribute the group's current max to gates [a, b)
  auto contribute = [&](int a, int b, double m) {
    if (!spec || m <= 0.0) return;
    const unsigned long long bits = (unsigned long long)__double_as_longlong(m);
    for (int j = a + (int)tid; j < b; j += kCta) atomicMax(&smax[j], bits);
  };
  const uint64_t scr0 = cap + 2ull * kSpecScratch * blockIdx.x;  // this CTA's scratch halves (spec mode)
  auto in_scratch = [&](uint64_t a) { return a >= scr0 && a < scr0 + 2ull * kSpecScratch; };
  // ping-pong of a group's versions through the run: the CTA's scratch halves
  // when n strings fit one, else a pair of arena regions grown by doubling
  // (pair_a, pair_cap: per group), so a large group costs O(its peak) of
  // arena space, not a fresh region per gate
  uint64_t pair_a = ~0ull;
  uint32_t pair_cap = 0;
  auto scratch_dst = [&](uint64_t from, uint32_t n) -> uint64_t {
    if (n <= kSpecScratch) return (in_scratch(from) && from == scr0) ? scr0 + kSpecScratch : scr0;
    if (n <= pair_cap) return from == pair_a ? pair_a + pair_cap : pair_a;
    return ~0ull;  // the caller grows the pair
  };
  auto alloc = [&](uint32_t n, int k) -> bool {
    __syncthreads();
    if (tid == 0) {
      dst_s = atomicAdd(&st->bump, (unsigned long long)n);
      s_fail = dst_s + n > cap;
      if (s_fail) {
        atomicOr(&st->err_arena, 1u);
        atomicMin(&st->err_seq, (unsigned long long)(seq0 + k));
      }
    }
    __syncthreads();
    return !s_fail;
  };
  for (;;) {
    __syncthreads();
    if (tid == 0) s_gid = atomicAdd(work, 1u);
    __syncthreads();
    // dense runs: two sweeps over the table, groups with a large output
    // (n 2^m >= one dense tile) first, so the longest groups start early
    const bool lpt = !spec && gates.dense;
    const uint32_t idx = s_gid;
    if (idx >= (lpt ? 2 * G : G) || failed) break;
    const uint32_t gid = list ? list[idx] : (idx < G ? idx : idx - G);
    Plane<W> z;
#pragma unroll
    for (int k = 0; k < W; ++k) z.w[k] = g.z[k][gid];
    uint32_t n = g.cnt[gid];
    if (n == 0) continue;
    if (spec && spec_done && spec_done[gid]) continue;  // run by k_spec_small
    if (!spec) {
      bool touched = false;
      uint32_t mt = 0;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        touched |= (z.w[k] & gates.any[k]) != 0;
        mt += __popcll(z.w[k] & gates.any[k]);
      }
      if (!touched) continue;
      if (lpt) {
        // the sweep follows from z alone: the count changes when another CTA
        // applies the group (it must not move the group to the other sweep)
        const bool big = mt >= kDenseSmemLog;
        if (big != (idx < G)) continue;
      }
    }
    uint64_t src = g.off[gid];
    uint32_t cap_g = g.cap[gid];
    double curmax = g.gmax[gid], curmin = g.gmin[gid];
    uint32_t curnf = g.flags[gid];
    bool changed = false;
    int k0 = 0;
    pair_a = ~0ull;
    pair_cap = 0;
    if (!spec) {
      const uint32_t stamp = g.stamp[gid];
      k0 = (stamp - seq0 < (uint32_t)gates.ng) ? (int)(stamp - seq0) + 1 : 0;  // resume after the stamp
    }
    int last = -1;  // last gate applied to this group (spec: truncations after it are pending)
    // the gates that touch this group, as a bit mask built by one ballot per warp
    {
      const int k = (int)tid;
      const bool t = k < gates.ng && (z.w[gates.wq[k < kMaxSubGates ? k : 0]] & gates.mq[k < kMaxSubGates ? k : 0]);
      const uint32_t b = __ballot_sync(0xffffffffu, t);
      __syncthreads();  // the previous group's readers of s_touch are done
      if ((tid & 31) == 0 && tid < kMaxSubGates) s_touch[tid >> 5] = b;
      __syncthreads();
    }
    if (gates.dense) {
      const int r = dense_group<W>(reinterpret_cast<double*>(smem_raw), dc, gs, tscan, g, ar, gates, s_gp, gid, n, src, k0,
                                   s_touch, seq0, cap, st, aff_elems, s_seen);
      if (r < 0) {
        failed = true;
        break;
      }
      if (r > 0) continue;
    }
    if (!gates.sorted && (g.flags[gid] & kFlagUnsorted)) {
      // the per-gate path needs the group sorted: leave it (stamp unchanged)
      // for a relaunch after the host's sort pass
      if (tid == 0) atomicOr(&st->err_unsorted, 1u);
      continue;
    }
    // next touching gate at or after k (gates.ng: the end step; ng + 1: done)
    auto next_touch = [&](int k) {
      if (k >= gates.ng) return k;
      for (int w = k >> 5; w < kMaxSubGates / 32; ++w) {
        uint32_t bits = s_touch[w];
        if (w == (k >> 5)) bits &= ~0u << (k & 31);
        if (bits) return min((w << 5) + __ffs(bits) - 1, gates.ng);
      }
      return gates.ng;
    };
    for (int k = next_touch(k0); k <= gates.ng; k = next_touch(k + 1)) {
      const bool end = k == gates.ng;
      if (spec) {
        // gates (last, k) did not touch the group: it held its values, each
        // of those gates' truncations applied to it
        double tp = -1.0;
        for (int j = last + 1; j < k; ++j) tp = fmax(tp, tpred[j]);
        if (n) {
          int j_empty = k;  // first pending gate whose threshold empties the group
          for (int j = last + 1; j < k; ++j)
            if (curmax <= tpred[j]) {
              j_empty = j;
              break;
            }
          contribute(last + 1, j_empty + 1 < k ? j_empty + 1 : k, curmax);
          if (j_empty < k) {  // every string is at or below that gate's threshold: all removed
            if (tid == 0) atomicAdd(&st->removed, (unsigned long long)n);
            n = 0;
          }
        }
        if (n && curmin <= tp) {  // drop what those truncations removed, into fresh space
          // (the run's last truncation of a group goes straight to the arena)
          uint64_t tdst = end ? ~0ull : scratch_dst(src, n);
          if (tdst == ~0ull) {
            if (!alloc(n, k)) {
              failed = true;
              break;
            }
            tdst = dst_s;
          }
          if (pair_cap && tdst != pair_a && tdst != pair_a + pair_cap && !in_scratch(tdst)) {
            pair_a = ~0ull;  // the versions left the pair (final copy)
            pair_cap = 0;
          }
          double mx = 0.0, mn = __longlong_as_double(0x7ff0000000000000ll);
          const uint32_t w = copy_truncated<W>(ar, src, n, tdst, tp, tscan, mx, mn);
          mx = warp_max(mx);
          mn = warp_min(mn);
          double dv = 0.0;
          uint32_t nf0 = 0;
          unsigned long long r0 = 0, rm = n - w;
          if (tid != 0) rm = 0;
          reduce_group_stats(gs, mx, mn, dv, nf0, r0, rm);
          if (tid == 0 && rm) atomicAdd(&st->removed, rm);
          src = tdst;
          cap_g = n;
          n = w;
          curmax = w ? mx : 0.0;
          curmin = w ? mn : __longlong_as_double(0x7ff0000000000000ll);
          changed = true;
        }
      }
      if (end || n == 0) break;
      const int wq = gates.wq[k];
      const uint64_t mq = gates.mq[k];
      uint64_t dst = spec ? scratch_dst(src, 2 * n) : ~0ull;
      if (dst == ~0ull) {
        // (spec: a new pair, twice the need or the old pair, whichever is larger)
        const uint32_t want = spec ? max(2 * n, 2 * pair_cap) : 2 * n;
        if (!alloc(spec ? 2 * want : want, k)) {
          failed = true;
          break;
        }
        dst = dst_s;
        if (spec) {
          pair_a = dst;
          pair_cap = want;
        }
      }
      aff_elems += n;
      uint32_t out_n = 0;
      double vmax = 0.0, vmin = __longlong_as_double(0x7ff0000000000000ll), vall = 0.0;
      uint32_t nonfinite = 0;
      unsigned long long records = 0, removed = 0;
      const double cosv = gates.cosv[k], sinv = gates.sinv[k];
      const double tout = spec ? tpred[k] : -1.0;
      uint32_t p = 0;
      while (p < n) {
        uint32_t used = seg_branch<W>(sg, ar, src, p, n, dst, out_n, wq, mq, cosv, sinv, keep_zeros, vmax, vmin,
                                      nonfinite, records, removed, tout, vall);
        if (used) {
          p += used;
          continue;
        }
        __syncthreads();
        const uint32_t be = find_block_end<W>(ar, src, p, n, wq, mq, nullptr);
        if (tid == 0) atomicAdd(&st->stream_elems, (unsigned long long)(be - p));
        stream_branch_range<W>(sm, ar, src + p, be - p, dst, out_n, wq, mq, cosv, sinv, keep_zeros, vmax, vmin,
                               nonfinite, records, removed, tout, vall);
        p = be;
      }
      reduce_group_stats(gs, vmax, vmin, vall, nonfinite, records, removed);
      if (tid == 0) {
        atomicAdd(&st->records, records);
        atomicAdd(&st->removed, removed);
        atomicAdd(&st->out_elems, (unsigned long long)out_n);
        if (records) atomicOr(&s_seen[k >> 5], 1u << (k & 31));
      }
      if (spec) {
        if (tid == 0 && vall > 0.0) atomicMax(&smax[k], (unsigned long long)__double_as_longlong(vall));
        // gmax as the reference sees it includes a NaN only through the flag
      }
      src = dst;
      cap_g = 2 * n;
      n = out_n;
      curmax = out_n ? vmax : 0.0;
      curmin = out_n ? vmin : __longlong_as_double(0x7ff0000000000000ll);
      curnf = nonfinite;
      changed = true;
      last = k;
      if (!spec && tid == 0) {  // resumable progress (eps = 0 mode)
        g.off[gid] = src;
        g.cnt[gid] = n;
        g.cap[gid] = cap_g;
        g.gmax[gid] = curmax;
        g.gmin[gid] = curmin;
        g.flags[gid] = curnf;
        g.stamp[gid] = seq0 + k;
      }
      __syncthreads();
    }
    if (failed) break;
    if (spec && n && in_scratch(src)) {  // the run's result: out of the scratch, into fresh arena space
      if (!alloc(n, gates.ng)) {
        failed = true;
        break;
      }
      const uint64_t o = dst_s;
      for (uint32_t i = tid; i < n; i += kCta) {
        store_plane<W>(ar.x, o + i, load_plane<W>(ar.x, src + i));
        ar.c[o + i] = ar.c[src + i];
      }
      src = o;
      cap_g = n;
    }
    if (spec && changed && tid == 0) {
      g.off[gid] = src;
      g.cnt[gid] = n;
      g.cap[gid] = cap_g;
      g.gmax[gid] = curmax;
      g.gmin[gid] = curmin;
      g.flags[gid] = curnf;
    } else if (spec && n == 0 && tid == 0) {
      g.cnt[gid] = 0;
    }
  }
  __syncthreads();
  if (spec)
    for (int k = tid; k < gates.ng; k += kCta)
      if (smax[k]) atomicMax(&gmax_out[k], smax[k]);
  // a touched group with a nonzero string sends a record through every gate
  // with sin != 0 that touches it (dense path: the group's vector stays
  // nonzero through the run's rotations); the per-gate path marks exactly
  for (int k = tid; k < gates.ng; k += kCta)
    if (((s_seen[k >> 5] >> (k & 31)) & 1u) && s_gp.sinv[k] != 0.0) mark_seen(st, st->seen_base + k);
  if (tid == 0 && aff_elems) atomicAdd(&st->aff_total, aff_elems);
  if (tid == 0 && dc.bulk_tiles) atomicAdd(&st->bulk_tiles, (unsigned long long)dc.bulk_tiles);
}

// ---------------------------------------------------------------------------
// Threshold discovery for a speculative run (eps0 > 0, per-gate cadence).
// Inside a run of X-type gates a group's strings only rotate among
// themselves and lose strings to truncation, so the group's max |c| after
// any of the run's gates is at most its L2 norm (up to rounding, covered by
// a 1e-9 margin).  If L <= gmax_k for every gate k of the run, the groups
// with norm < L cannot hold any gmax_k: the run's exact thresholds
// epsilon0 * gmax_k follow from the groups with norm >= L alone.  The host
// runs the speculative sublayer on that small subset (a copy of their table
// entries, outputs discarded) until its thresholds are a fixed point, checks
// min_k gmax_k >= L, and then runs the whole table once with them.
// ---------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(kCta) k_group_norms(GroupView<W> g, ArenaView<W> ar, const DevStats* st,
                                                      double* norm) {
  const uint32_t G = *(volatile const unsigned int*)&st->G_dev;
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t gi = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; gi < G; gi += (gridDim.x * blockDim.x) >> 5) {
    const uint32_t n = g.cnt[gi];
    const uint64_t o = g.off[gi];
    double s = 0.0;
    for (uint32_t i = lane; i < n; i += 32) {
      const double v = ar.c[o + i];
      s = fma(v, v, s);
    }
#pragma unroll
    for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
    if (lane == 0) norm[gi] = s;
  }
}

// Copies the table entries of the groups whose norm may reach L (or that
// hold a non-finite value) into `sub`; the subset's group count lands in
// *count.
template <int W>
__global__ void k_select_groups(GroupView<W> g, const DevStats* st, const double* norm, double L, GroupView<W> sub,
                                unsigned int* count) {
  const uint32_t G = *(volatile const unsigned int*)&st->G_dev;
  const uint32_t gi = blockIdx.x * blockDim.x + threadIdx.x;
  if (gi >= G) return;
  const uint32_t n = g.cnt[gi];
  if (!n) return;
  const double nrm = sqrt(norm[gi]) * (1.0 + 1e-9);  // summation and rotation rounding
  if (!(nrm >= L) && !(g.flags[gi] & 1u)) return;
  const uint32_t j = atomicAdd(count, 1u);
#pragma unroll
  for (int k = 0; k < W; ++k) sub.z[k][j] = g.z[k][gi];
  sub.off[j] = g.off[gi];
  sub.cnt[j] = n;
  sub.cap[j] = g.cap[gi];
  sub.gmax[j] = g.gmax[gi];
  sub.gmin[j] = g.gmin[gi];
  sub.flags[j] = g.flags[gi];
  sub.stamp[j] = g.stamp[gi];
}

__global__ void k_use_group_count(DevStats* st, const unsigned int* count, unsigned long long bump) {
  st->G_dev = *count;
  st->bump = bump;
  st->work[0] = st->work[1] = 0;
}

// ---------------------------------------------------------------------------
// k_spec_small: the speculative run (eps0 > 0, per-gate cadence) for small
// z-groups, one WARP per group, the group's strings held in that warp's
// shared memory from the first gate of the run to the last.  Per touching
// gate X_q the strings are hashed by x; a string x pairs with x ^ e_q when
// both are present (one butterfly, the reference's per-key arithmetic:
// v = c cos [+ (+-sin) c_partner], engine.cpp:218-227 + TermMap::add), a
// lone string keeps c cos and appends its child (x ^ e_q, +-sin c); then
// every string with |c| <= T_k goes (truncate_now, engine.cpp:318-351).
// Gates that do not touch the group apply their truncations when the next
// touching gate (or the end) comes, and the group's max feeds their gmax
// until a threshold empties it -- k_branch_sublayer's spec semantics exactly.
// Only the final strings are written (sorted by x, fresh arena space): no
// intermediate version leaves the SM.  A group that outgrows the warp's
// buffer is left untouched for k_branch_sublayer; finished groups are
// flagged in spec_done (cleared per attempt) so k_branch_sublayer skips them.
// ---------------------------------------------------------------------------
// (measured on the config-2 shape: 256 strings x 8 warps 50.5 ms per step, 512 x 4 53.8, 128 x 8 57.4, 1024 x 2 83.3)
#ifndef PP_SMALL_CAP
#define PP_SMALL_CAP 256
#endif
#ifndef PP_SMALL_WARPS
#define PP_SMALL_WARPS 8
#endif
constexpr uint32_t kSmallCap = PP_SMALL_CAP;       // strings per warp buffer
constexpr uint32_t kSmallWarps = PP_SMALL_WARPS;   // warps (groups in flight) per CTA
#ifndef PP_SMALL_MAXIN
#define PP_SMALL_MAXIN (PP_SMALL_CAP / 2)
#endif
constexpr uint32_t kSmallMaxIn = PP_SMALL_MAXIN;   // groups of at most this many strings start here

template <int W>
constexpr size_t spec_small_smem_bytes() {
  return (size_t)kSmallWarps * kSmallCap * (8 * W + 8 + 2 * 4);  // x planes, c, hash (2 slots per string)
}

template <int W>
__device__ __forceinline__ uint32_t small_hash(const uint64_t* xs, uint32_t i) {
  uint64_t h = xs[i] * 0x9E3779B97F4A7C15ull;
  if (W == 2) h ^= xs[kSmallCap + i] * 0xC2B2AE3D27D4EB4Full;
  return (uint32_t)(h >> 40) & (2 * kSmallCap - 1);
}
template <int W>
__device__ __forceinline__ uint32_t small_hash_key(const Plane<W>& x) {
  uint64_t h = x.w[0] * 0x9E3779B97F4A7C15ull;
  if (W == 2) h ^= x.w[1] * 0xC2B2AE3D27D4EB4Full;
  return (uint32_t)(h >> 40) & (2 * kSmallCap - 1);
}

template <int W>
__global__ void __launch_bounds__(kSmallWarps * 32) k_spec_small(GroupView<W> g, ArenaView<W> ar, const SubGates gates,
                                                                 unsigned int* work, const double* __restrict__ tpred,
                                                                 unsigned long long* gmax_out, DevStats* st,
                                                                 uint8_t* spec_done) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* xs = reinterpret_cast<uint64_t*>(smem_raw) + (size_t)warp * W * kSmallCap;  // [W][kSmallCap]
  double* cs = reinterpret_cast<double*>(reinterpret_cast<uint64_t*>(smem_raw) + (size_t)kSmallWarps * W * kSmallCap) +
               (size_t)warp * kSmallCap;
  uint32_t* ht = reinterpret_cast<uint32_t*>(reinterpret_cast<double*>(reinterpret_cast<uint64_t*>(smem_raw) +
                                                                       (size_t)kSmallWarps * W * kSmallCap) +
                                             (size_t)kSmallWarps * kSmallCap) +
                 (size_t)warp * 2 * kSmallCap;
  __shared__ unsigned long long smax[kMaxSubGates];
  __shared__ double s_tp[kMaxSubGates], s_cos[kMaxSubGates], s_sin[kMaxSubGates];
  __shared__ uint64_t s_mq[kMaxSubGates];
  __shared__ int8_t s_wq[kMaxSubGates];
  __shared__ uint32_t s_seen[kMaxSubGates / 32];
  const int ng = gates.ng;
  for (int k = threadIdx.x; k < ng; k += blockDim.x) {
    smax[k] = 0ull;
    s_tp[k] = tpred[k];
    s_cos[k] = gates.cosv[k];
    s_sin[k] = gates.sinv[k];
    s_mq[k] = gates.mq[k];
    s_wq[k] = gates.wq[k];
  }
  if (threadIdx.x < kMaxSubGates / 32) s_seen[threadIdx.x] = 0;
  __syncthreads();
  if (engine_failed(st)) return;
  const uint32_t G = *(volatile const unsigned int*)&st->G_dev;
  const unsigned long long cap = *(volatile const unsigned long long*)&st->arena_cap;
  const uint32_t seq0 = (uint32_t)(*(volatile const unsigned long long*)&st->seq_base);
  const double kInf = __longlong_as_double(0x7ff0000000000000ll);
  unsigned long long w_records = 0, w_removed = 0, w_out = 0, w_in = 0;
  auto contribute = [&](int j, double m) {  // group max m at gate j
    if (m > 0.0) atomicMax(&smax[j], (unsigned long long)__double_as_longlong(m));
  };
  for (;;) {
    uint32_t gid = 0;
    if (lane == 0) gid = atomicAdd(work, 1u);
    gid = __shfl_sync(0xffffffffu, gid, 0);
    if (gid >= G) break;
    uint32_t n = g.cnt[gid];
    if (n == 0 || n > kSmallMaxIn) continue;
    Plane<W> z;
#pragma unroll
    for (int w = 0; w < W; ++w) z.w[w] = g.z[w][gid];
    const uint64_t src = g.off[gid];
    // touching gates (z_q = 1), 4 words of 32
    uint32_t touch[kMaxSubGates / 32];
#pragma unroll
    for (int t = 0; t < kMaxSubGates / 32; ++t) {
      const int k = 32 * t + (int)lane;
      const bool tk = k < ng && (z.w[s_wq[k < ng ? k : 0]] & s_mq[k < ng ? k : 0]);
      touch[t] = __ballot_sync(0xffffffffu, tk);
    }
    // load the group
    double mx = 0.0, mn = kInf;
    for (uint32_t i = lane; i < n; i += 32) {
#pragma unroll
      for (int w = 0; w < W; ++w) xs[w * kSmallCap + i] = ar.x[w][src + i];
      const double v = ar.c[src + i];
      cs[i] = v;
      mx = fmax(mx, fabs(v));
      mn = fmin(mn, fabs(v));
    }
    mx = warp_max_nn(mx);
    mn = warp_min_nn(mn);
    __syncwarp();
    w_in += n;
    uint32_t nonfinite = 0;
    unsigned long long g_records = 0, g_removed = 0;
    uint32_t seen_local[kMaxSubGates / 32] = {0, 0, 0, 0};
    bool abort = false;
    int last = -1;
    // truncation |c| <= T of the n strings (in place, order kept); returns the count kept
    auto truncate = [&](double T) {
      uint32_t out = 0;
      double kmx = 0.0, kmn = kInf;
      for (uint32_t b = 0; b < n; b += 32) {
        const uint32_t i = b + lane;
        Plane<W> x;
        double v = 0.0;
        bool keep = false;
        if (i < n) {
#pragma unroll
          for (int w = 0; w < W; ++w) x.w[w] = xs[w * kSmallCap + i];
          v = cs[i];
          keep = !(fabs(v) <= T);
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        __syncwarp();
        if (keep) {
          const uint32_t o = out + __popc(bal & ((1u << lane) - 1u));
#pragma unroll
          for (int w = 0; w < W; ++w) xs[w * kSmallCap + o] = x.w[w];
          cs[o] = v;
          kmx = fmax(kmx, fabs(v));
          kmn = fmin(kmn, fabs(v));
        }
        __syncwarp();
        out += __popc(bal);
      }
      g_removed += n - out;
      n = out;
      mx = warp_max_nn(kmx);
      mn = warp_min_nn(kmn);
    };
    for (int t = 0;; ++t) {
      // next touching gate at or after last + 1 (ng: the end step)
      int k = ng;
      for (int ww = (last + 1) >> 5; ww < kMaxSubGates / 32; ++ww) {
        uint32_t bits = touch[ww];
        if (ww == ((last + 1) >> 5)) bits &= ~0u << ((last + 1) & 31);
        if (bits) {
          k = min(32 * ww + __ffs(bits) - 1, ng);
          break;
        }
      }
      // gates (last, k) leave the group as it is: their truncations apply,
      // its max feeds their gmax until a threshold empties it
      if (n && last + 1 < k) {
        int jlim = k;  // gates (last, jlim) see the group's max (an emptying gate included)
        double tp = -1.0;
        for (int j0 = last + 1; j0 < k; j0 += 32) {
          const int j = j0 + (int)lane;
          const double tj = j < k ? s_tp[j] : -1.0;
          tp = fmax(tp, tj);
          const uint32_t em = __ballot_sync(0xffffffffu, j < k && mx <= tj);
          if (em && jlim == k) jlim = j0 + __ffs(em);  // emptied at gate j0 + ffs - 1
        }
        tp = warp_max(tp);
        for (int j = last + 1 + (int)lane; j < jlim; j += 32) contribute(j, mx);
        if (tp >= 0.0 && mn <= tp) truncate(tp);
      }
      if (k >= ng || n == 0) break;
      // ---- gate k: X_q on the group
      const int wq = s_wq[k];
      const uint64_t mq = s_mq[k];
      const double cosv = s_cos[k], sinv = s_sin[k], nsin = -sinv;
      for (uint32_t sl = lane; sl < 2 * kSmallCap / 4; sl += 32) reinterpret_cast<uint4*>(ht)[sl] = make_uint4(0u, 0u, 0u, 0u);
      __syncwarp();
      for (uint32_t i = lane; i < n; i += 32) {
        uint32_t h = small_hash<W>(xs, i);
        while (atomicCAS(&ht[h], 0u, i + 1) != 0u) h = (h + 1) & (2 * kSmallCap - 1);
      }
      __syncwarp();
      uint32_t added = 0;
      double gmx = 0.0;
      unsigned long long recs = 0;
      for (uint32_t b = 0; b < n; b += 32) {
        const uint32_t i = b + lane;
        bool child = false;
        Plane<W> cx;
        double cd = 0.0;
        if (i < n) {
          Plane<W> x;
#pragma unroll
          for (int w = 0; w < W; ++w) x.w[w] = xs[w * kSmallCap + i];
          Plane<W> p = x;
          p.w[wq] ^= mq;
          uint32_t h = small_hash_key<W>(p), j = 0;
          for (;;) {
            const uint32_t e = ht[h];
            if (e == 0u) break;
            bool eq = true;
#pragma unroll
            for (int w = 0; w < W; ++w) eq &= xs[w * kSmallCap + e - 1] == p.w[w];
            if (eq) {
              j = e;
              break;
            }
            h = (h + 1) & (2 * kSmallCap - 1);
          }
          const bool bit1 = (x.w[wq] & mq) != 0;
          const double c = cs[i];
          if (j) {
            if (!bit1) {  // the pair (x, x | e_q): one butterfly, by the x_q = 0 string
              double a = c, bb = cs[j - 1];
              const double d1 = __dmul_rn(sinv, a), d0 = __dmul_rn(nsin, bb);
              double v0 = __dmul_rn(a, cosv), v1 = __dmul_rn(bb, cosv);
              if (d0 != 0.0) {
                v0 = __dadd_rn(v0, d0);
                ++recs;
              }
              if (d1 != 0.0) {
                v1 = __dadd_rn(v1, d1);
                ++recs;
              }
              cs[i] = v0;
              cs[j - 1] = v1;
              gmx = fmax(gmx, fmax(fabs(v0), fabs(v1)));
              if (!(fabs(v0) <= 1.7976931348623157e308) || !(fabs(v1) <= 1.7976931348623157e308)) nonfinite = 1;
            }
          } else {  // alone: keeps c cos, its child (+sin from a Z, -sin from a Y) is a new string
            const double v = __dmul_rn(c, cosv);
            cd = __dmul_rn(bit1 ? nsin : sinv, c);
            cs[i] = v;
            gmx = fmax(gmx, fabs(v));
            if (!(fabs(v) <= 1.7976931348623157e308)) nonfinite = 1;
            if (cd != 0.0) {
              child = true;
              cx = p;
              ++recs;
              gmx = fmax(gmx, fabs(cd));
              if (!(fabs(cd) <= 1.7976931348623157e308)) nonfinite = 1;
            }
          }
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, child);
        if (child) {
          const uint32_t o = n + added + __popc(bal & ((1u << lane) - 1u));
          if (o < kSmallCap) {
#pragma unroll
            for (int w = 0; w < W; ++w) xs[w * kSmallCap + o] = cx.w[w];
            cs[o] = cd;
          }
        }
        added += __popc(bal);
      }
      __syncwarp();
      if (n + added > kSmallCap) {  // outgrew the buffer: k_branch_sublayer takes the group
        abort = true;
        break;
      }
      n += added;
      recs = __reduce_add_sync(0xffffffffu, (uint32_t)recs);  // (at most 2 per string and lane pass: far below 2^32)
      g_records += recs;
      if (recs && lane == 0) seen_local[k >> 5] |= 1u << (k & 31);
      gmx = warp_max_nn(gmx);
      if (lane == 0) contribute(k, gmx);  // gmax after gate k's apply, before its truncation
      mx = gmx;
      mn = 0.0;  // (force the truncation below)
      truncate(s_tp[k]);
      last = k;
    }
    if (abort) continue;  // nothing written: the group is untouched
    nonfinite = __any_sync(0xffffffffu, nonfinite);
    // sort by x (bitonic, padded with all-ones keys) and write out
    uint32_t P = 1;
    while (P < n) P <<= 1;
    for (uint32_t i = n + lane; i < P; i += 32) {
#pragma unroll
      for (int w = 0; w < W; ++w) xs[w * kSmallCap + i] = ~0ull;
      cs[i] = 0.0;
    }
    __syncwarp();
    for (uint32_t kk = 2; kk <= P; kk <<= 1) {
      for (uint32_t jj = kk >> 1; jj > 0; jj >>= 1) {
        for (uint32_t i = lane; i < P; i += 32) {
          const uint32_t l = i ^ jj;
          if (l > i) {
            Plane<W> a, b;
#pragma unroll
            for (int w = 0; w < W; ++w) {
              a.w[w] = xs[w * kSmallCap + i];
              b.w[w] = xs[w * kSmallCap + l];
            }
            const bool up = (i & kk) == 0;
            if (up ? plane_lt<W>(b, a) : plane_lt<W>(a, b)) {
#pragma unroll
              for (int w = 0; w < W; ++w) {
                xs[w * kSmallCap + i] = b.w[w];
                xs[w * kSmallCap + l] = a.w[w];
              }
              const double t2 = cs[i];
              cs[i] = cs[l];
              cs[l] = t2;
            }
          }
        }
        __syncwarp();
      }
    }
    unsigned long long o = 0;
    if (lane == 0) {
      o = atomicAdd(&st->bump, (unsigned long long)n);
      if (o + n > cap) {
        atomicOr(&st->err_arena, 1u);
        atomicMin(&st->err_seq, (unsigned long long)seq0);
      }
    }
    o = __shfl_sync(0xffffffffu, o, 0);
    if (o + n > cap) continue;  // the attempt faults (the host rolls back); leave the group
    for (uint32_t i = lane; i < n; i += 32) {
#pragma unroll
      for (int w = 0; w < W; ++w) ar.x[w][o + i] = xs[w * kSmallCap + i];
      ar.c[o + i] = cs[i];
    }
    if (lane == 0) {
      g.off[gid] = o;
      g.cnt[gid] = n;
      g.cap[gid] = n;
      g.gmax[gid] = n ? mx : 0.0;
      g.gmin[gid] = n ? mn : kInf;
      g.flags[gid] = nonfinite;
      spec_done[gid] = 1;
#pragma unroll
      for (int t = 0; t < kMaxSubGates / 32; ++t)
        if (seen_local[t]) atomicOr(&s_seen[t], seen_local[t]);
    }
    w_records += g_records;
    w_removed += g_removed;
    w_out += n;
    __syncwarp();
  }
  if (lane == 0) {
    if (w_records) atomicAdd(&st->records, w_records);
    if (w_removed) atomicAdd(&st->removed, w_removed);
    if (w_out) atomicAdd(&st->out_elems, w_out);
    if (w_in) atomicAdd(&st->aff_total, w_in);
  }
  __syncthreads();
  for (int k = threadIdx.x; k < ng; k += blockDim.x) {
    if (smax[k]) atomicMax(&gmax_out[k], smax[k]);
    if ((s_seen[k >> 5] >> (k & 31)) & 1u) mark_seen(st, st->seen_base + k);
  }
}

// k_branch_x: the segment / stream buffers of the per-gate path
template <int W>
constexpr size_t branch_x_smem_bytes() {
  return sizeof(BranchSmem<W>) > sizeof(SegSmem<W>) ? sizeof(BranchSmem<W>) : sizeof(SegSmem<W>);
}
// k_branch_sublayer: those, or the dense tile and its tables, whichever is larger
template <int W>
constexpr size_t branch_smem_bytes() {
  constexpr size_t a = branch_x_smem_bytes<W>();
  constexpr size_t d = kDenseSmem * sizeof(double) + sizeof(DenseTail<W>);
  return a > d ? a : d;
}
static_assert(kDenseSmem % (8 * kCta) == 0, "dense tile gathers in steps of 8 kCta");
static_assert(branch_smem_bytes<1>() >= kDenseSmem * sizeof(double) + sizeof(DenseTail<1>), "dense tail must fit");
static_assert(branch_smem_bytes<2>() >= kDenseSmem * sizeof(double) + sizeof(DenseTail<2>), "dense tail must fit");
static_assert(branch_smem_bytes<1>() >= kDenseSmem * sizeof(double) + 3 * 256 * 8, "dense tile must fit the branch buffer");
static_assert(branch_smem_bytes<2>() >= kDenseSmem * sizeof(double) + 3 * 256 * 16, "dense tile must fit the branch buffer");

// ---------------------------------------------------------------------------
// group-level reductions: live count, max |c|, min over group minima, NaN
// (truncate_now's first pass, engine.cpp:321-343, at group granularity)
// ---------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(kCta) k_reduce(GroupView<W> g, const DevStats* st, RedSlot* out,
                                                 const double* __restrict__ thr = nullptr, uint32_t rel = 0) {
  const uint32_t G = *(volatile const unsigned int*)&st->G_dev;
  const uint32_t seq_base = (uint32_t)*(volatile const unsigned long long*)&st->seq_base;
  // grid-stride, then one set of atomics per CTA (same-address atomics from
  // every warp serialise in L2)
  unsigned long long live = 0;
  double mx = 0.0, mn = __longlong_as_double(0x7ff0000000000000ll);
  uint32_t nf = 0, mc = 0;
  if (thr) {
    // deferred truncation: a group whose max is pending removal holds no live
    // string (every other value is smaller).  thr[0] bounds every slot, so
    // only groups with a max at or below it need their own slot.
    const double t0 = thr[0];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < G; i += gridDim.x * blockDim.x) {
      const uint32_t c = g.cnt[i];
      if (c) {
        live += c;
        const double gm = g.gmax[i];
        if (gm > t0 || gm > thr[pending_index(g.stamp[i], seq_base, rel)]) mx = fmax(mx, gm);
        nf |= g.flags[i] & 1u;
      }
    }
  } else {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < G; i += gridDim.x * blockDim.x) {
      const uint32_t c = g.cnt[i];
      if (c) {
        live += c;
        mx = fmax(mx, g.gmax[i]);
        mn = fmin(mn, g.gmin[i]);
        nf |= g.flags[i] & 1u;
        mc = max(mc, c);
      }
    }
  }
  mc = __reduce_max_sync(0xffffffffu, mc);
  if ((threadIdx.x & 31) == 0 && mc) atomicMax(&out->maxcnt, mc);
  live = warp_sum64(live);
  mx = warp_max(mx);
  mn = warp_min(mn);
  nf = __any_sync(0xffffffffu, nf);
  __shared__ unsigned long long sl[kWarps];
  __shared__ double smx[kWarps], smn[kWarps];
  __shared__ uint32_t snf[kWarps];
  const uint32_t w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    sl[w] = live;
    smx[w] = mx;
    smn[w] = mn;
    snf[w] = nf;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t k = 1; k < kWarps; ++k) {
      live += sl[k];
      mx = fmax(mx, smx[k]);
      mn = fmin(mn, smn[k]);
      nf |= snf[k];
    }
    if (live) atomicAdd(&out->live, live);
    atomic_max_nonneg(reinterpret_cast<double*>(&out->gmax_bits), mx);
    atomic_min_nonneg(reinterpret_cast<double*>(&out->gmin_bits), mn);
    if (nf) atomicOr(&out->nonfinite, 1u);
  }
}

// ---------------------------------------------------------------------------
// truncation: remove |c| <= T inside every group whose min |c| <= T
// (TermMap::remove_below, term_map.cpp:105-144; strict <= so exact zeros
// and -0.0 always go).  In-place streaming compaction, one CTA per group.
// ---------------------------------------------------------------------------
template <int W>
__device__ void truncate_group(GroupView<W> g, ArenaView<W> ar, uint32_t gid, double T, DevStats* st,
                               uint32_t* scan, double* rmx, double* rmn) {
  const uint32_t n = g.cnt[gid];
  const uint64_t off = g.off[gid];
  const uint32_t tid = threadIdx.x;
  uint32_t w = 0;
  double vmax = 0.0, vmin = __longlong_as_double(0x7ff0000000000000ll);
  for (uint32_t base = 0; base < n; base += kCta) {
    uint32_t p = base + tid;
    bool keep = false;
    Plane<W> k;
    double v = 0.0;
    if (p < n) {
      k = load_plane<W>(ar.x, off + p);
      v = ar.c[off + p];
      keep = !(fabs(v) <= T);
    }
    uint32_t tot;
    uint32_t o = block_excl_scan(keep ? 1u : 0u, scan, &tot);  // syncs: all reads done
    if (keep) {
      store_plane<W>(ar.x, off + w + o, k);
      ar.c[off + w + o] = v;
      vmax = fmax(vmax, fabs(v));
      vmin = fmin(vmin, fabs(v));
    }
    w += tot;
    __syncthreads();
  }
  vmax = warp_max(vmax);
  vmin = warp_min(vmin);
  if ((tid & 31) == 0) {
    rmx[tid >> 5] = vmax;
    rmn[tid >> 5] = vmin;
  }
  __syncthreads();
  if (tid == 0) {
    for (uint32_t i = 1; i < kWarps; ++i) {
      vmax = fmax(vmax, rmx[i]);
      vmin = fmin(vmin, rmn[i]);
    }
    g.cnt[gid] = w;
    g.gmax[gid] = w ? vmax : 0.0;
    g.gmin[gid] = w ? vmin : __longlong_as_double(0x7ff0000000000000ll);
    atomicAdd(&st->removed, (unsigned long long)(n - w));
  }
  __syncthreads();
}

// Per-gate epilogue (Engine::apply_gate tail, engine.cpp:309-315 and
// truncate_now, engine.cpp:318-351), device-side so no host round trip:
//   budget check on |O| after the apply -> sticky err_budget
//   [truncate] NaN/Inf -> sticky err_numerical; T = epsilon0 * gmax;
//              remove |c| <= T in every group whose min |c| <= T.
// Persistent grid-stride over groups.
template <int W>
__global__ void __launch_bounds__(kCta) k_truncate(GroupView<W> g, ArenaView<W> ar, double epsilon0,
                                                   int do_truncate, unsigned long long max_terms,
                                                   unsigned long long gate_index, RedSlot* red, RedSlot* red_next,
                                                   DevStats* st) {
  if (blockIdx.x == 0 && threadIdx.x == 0) clear_red(red_next);
  if (engine_failed(st)) return;
  const uint32_t G = *(volatile const unsigned int*)&st->G_dev;
  const unsigned long long live = *(volatile unsigned long long*)&red->live;
  if (max_terms && live > max_terms) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && atomicCAS(&st->err_budget, 0u, 1u) == 0u) {
      st->err_gate = gate_index;
      st->err_live = live;
    }
    return;
  }
  if (!do_truncate) return;
  if (*(volatile unsigned int*)&red->nonfinite) {
    if (blockIdx.x == 0 && threadIdx.x == 0 && atomicCAS(&st->err_numerical, 0u, 1u) == 0u) {
      st->err_gate = gate_index;
      st->err_live = live;
    }
    return;
  }
  const double gmax = __longlong_as_double(*(volatile long long*)&red->gmax_bits);
  const double gmin = __longlong_as_double(*(volatile long long*)&red->gmin_bits);
  const double T = epsilon0 * gmax;  // engine.cpp:345, one IEEE product
  if (blockIdx.x == 0 && threadIdx.x == 0) st->last_gmax_bits = (unsigned long long)__double_as_longlong(gmax);
  if (!(gmin <= T)) return;
  __shared__ uint32_t scan[40];
  __shared__ double rmx[kWarps], rmn[kWarps];
  for (uint32_t gid = blockIdx.x; gid < G; gid += gridDim.x) {
    if (g.cnt[gid] == 0 || !(g.gmin[gid] <= T)) continue;  // uniform per CTA
    truncate_group<W>(g, ar, gid, T, st, scan, rmx, rmn);
  }
}

// truncation at an externally supplied threshold (sharded engines: T comes
// from epsilon0 times the max over all shards)
template <int W>
__global__ void __launch_bounds__(kCta) k_truncate_T(GroupView<W> g, ArenaView<W> ar, double T, DevStats* st) {
  const uint32_t G = *(volatile const unsigned int*)&st->G_dev;
  __shared__ uint32_t scan[40];
  __shared__ double rmx[kWarps], rmn[kWarps];
  for (uint32_t gid = blockIdx.x; gid < G; gid += gridDim.x) {
    if (g.cnt[gid] == 0 || !(g.gmin[gid] <= T)) continue;  // uniform per CTA
    truncate_group<W>(g, ar, gid, T, st, scan, rmx, rmn);
  }
}

// ---------------------------------------------------------------------------
// Deferred truncation (epsilon0 > 0, per-gate cadence).  The reference
// removes |c| <= T_k = epsilon0 * gmax_k from the whole store after every gate
// k (engine.cpp:318-351).  A string that survives to gate k unchanged is
// removed at the first k whose T_k >= |c|; since an untouched group's values do
// not change, it is enough to know, per group, the largest T since the group
// was last rewritten.  thr[j] = max(T_j .. T_now) for the gates j of the
// current launch window (j = seq - window base); a group rewritten at gate j
// reads thr[j], one rewritten before the window reads thr[0].  The next gate
// that touches the group drops those strings while loading it (they act as
// absent: 0*cos + child == child, and a zero child is no record), and a flush
// compacts the rest before anything else reads the store.  The global max per
// gate skips groups whose max is pending, so T_k is exactly the reference's.
// ---------------------------------------------------------------------------
template <int W>
__global__ void __launch_bounds__(kCta) k_thresh(double epsilon0, uint32_t rel, RedSlot* red, RedSlot* red_next,
                                                 double* thr, DevStats* st) {
  if (threadIdx.x == 0) clear_red(red_next);
  if (engine_failed(st)) return;
  if (*(volatile unsigned int*)&red->nonfinite) {
    if (threadIdx.x == 0 && atomicCAS(&st->err_numerical, 0u, 1u) == 0u) {
      st->err_gate = rel;
      st->err_live = *(volatile unsigned long long*)&red->live;
    }
    return;
  }
  const double gmax = __longlong_as_double(*(volatile long long*)&red->gmax_bits);
  const double T = epsilon0 * gmax;  // engine.cpp:345, one IEEE product
  for (uint32_t j = threadIdx.x; j < rel; j += kCta) thr[j] = fmax(thr[j], T);
  if (threadIdx.x == 0) {
    st->last_gmax_bits = (unsigned long long)__double_as_longlong(gmax);
    thr[rel] = T;
    thr[rel + 1] = 0.0;  // the next gate's groups are exact when it reduces
  }
}

template <int W>
__global__ void __launch_bounds__(kCta) k_flush(GroupView<W> g, ArenaView<W> ar, const double* __restrict__ thr,
                                                uint32_t win_base, uint32_t win_len, DevStats* st) {
  const uint32_t G = *(volatile const unsigned int*)&st->G_dev;
  __shared__ uint32_t scan[40];
  __shared__ double rmx[kWarps], rmn[kWarps];
  for (uint32_t gid = blockIdx.x; gid < G; gid += gridDim.x) {
    if (g.cnt[gid] == 0) continue;
    const double P = thr[pending_index(g.stamp[gid], win_base, win_len)];
    if (!(g.gmin[gid] <= P)) continue;  // uniform per CTA
    truncate_group<W>(g, ar, gid, P, st, scan, rmx, rmn);
  }
}

// sum of c^2 over the store (Frobenius norm^2 / 2^n: conserved exactly at
// epsilon0 = 0 -- a size-independent property check, test_engine.cpp:260-304)
template <int W>
__global__ void __launch_bounds__(kCta) k_norm2(GroupView<W> g, ArenaView<W> ar, const DevStats* st, double* out) {
  const uint32_t G = *(volatile const unsigned int*)&st->G_dev;
  double acc = 0.0;
  for (uint32_t gid = blockIdx.x; gid < G; gid += gridDim.x) {
    const uint32_t n = g.cnt[gid];
    const uint64_t off = g.off[gid];
    for (uint32_t i = threadIdx.x; i < n; i += kCta) {
      const double c = ar.c[off + i];
      acc = fma(c, c, acc);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ double red[kWarps];
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (uint32_t w = 1; w < kWarps; ++w) acc += red[w];
    atomicAdd(out, acc);
  }
}

// ---------------------------------------------------------------------------
// log-binned coefficient density with a sign split (sparse_operator.cpp:
// 150-197): bin 0 holds |c/gmax| <= lower, bin bins-1 holds >= 1, the rest
// int(bins * (1 - log|x| / log lower)).  Counts are exact integers; the host
// turns them into the reference's normalized sums.  Reads 8 B per string.
// ---------------------------------------------------------------------------
constexpr int kMaxHistBins = 4096;

template <int W>
__global__ void __launch_bounds__(kCta) k_histogram(GroupView<W> g, ArenaView<W> ar, const DevStats* st, int bins,
                                                   double gmax, double lower, const double* __restrict__ edges_g,
                                                   unsigned long long* pos, unsigned long long* neg) {
  // density_histogram (sparse_operator.cpp:150-196): the bin of a string in
  // (lower, 1) is the number of host-computed edges <= |c / gmax|
  extern __shared__ unsigned int hist[];  // [2 * bins]: positive then negative, then the edges
  double* edges = reinterpret_cast<double*>(hist + 2 * ((bins + 1) & ~1));
  const int ne = bins > 1 ? bins - 1 : 1;
  for (int b = threadIdx.x; b < 2 * bins; b += kCta) hist[b] = 0;
  for (int b = threadIdx.x; b < ne; b += kCta) edges[b] = edges_g[b];
  __syncthreads();
  const uint32_t G = *(volatile const unsigned int*)&st->G_dev;
  for (uint32_t gid = blockIdx.x; gid < G; gid += gridDim.x) {
    const uint32_t n = g.cnt[gid];
    const uint64_t off = g.off[gid];
    for (uint32_t i = threadIdx.x; i < n; i += kCta) {
      const double x = ar.c[off + i] / gmax;
      const double ax = fabs(x);
      int b;
      if (ax <= lower) {
        b = 0;
      } else if (ax >= 1.0) {
        b = bins - 1;
      } else {
        int lo = 0, hi = bins - 1;  // number of edges <= ax, in [0, bins - 1]
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (edges[mid - 1] <= ax) lo = mid;
          else hi = mid - 1;
        }
        b = lo;
      }
      atomicAdd(&hist[(x < 0 ? bins : 0) + b], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < bins; b += kCta) {
    if (hist[b]) atomicAdd(&pos[b], (unsigned long long)hist[b]);
    if (hist[bins + b]) atomicAdd(&neg[b], (unsigned long long)hist[bins + b]);
  }
}

// ---------------------------------------------------------------------------
// diagonal strings (x == 0 is the smallest key of a group, so it can only be
// the first element): <0|O|0> terms (sparse_operator.cpp:32-36, 89-97)
// ---------------------------------------------------------------------------
// The per-layer readout in one launch: the group reduction of k_reduce
// (live count, max / min |c|, NaN flag, largest group) and the diagonal
// search of k_diag, a warp per group.
template <int W>
__global__ void __launch_bounds__(kCta) k_readout(GroupView<W> g, uint32_t Gp, ArenaView<W> ar, uint64_t* out_z,
                                                  double* out_c, DevStats* st, RedSlot* out) {
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t G = Gp != kKeepG ? Gp : *(volatile const unsigned int*)&st->G_dev;
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t n = i < G ? g.cnt[i] : 0u;
  unsigned long long live = 0;
  double mx = 0.0, mn = __longlong_as_double(0x7ff0000000000000ll);
  uint32_t nf = 0;
  if (n) {
    const uint64_t o = g.off[i];
    const uint32_t fl = g.flags[i];
    if (lane == 0) {
      live = n;
      mx = g.gmax[i];
      mn = g.gmin[i];
      nf = fl & 1u;
    }
    uint64_t hit = ~0ull;
    if ((fl & (kFlagUnsorted | kFlagMinFirst)) == kFlagUnsorted) {
      for (uint32_t j0 = 0; j0 < n; j0 += 32) {
        const bool z = j0 + lane < n && plane_zero<W>(load_plane<W>(ar.x, o + j0 + lane));
        const uint32_t b = __ballot_sync(0xffffffffu, z);
        if (b) {
          hit = o + j0 + __ffs(b) - 1;
          break;
        }
      }
    } else if (plane_zero<W>(load_plane<W>(ar.x, o))) {
      hit = o;
    }
    if (lane == 0 && hit != ~0ull) {
      const unsigned long long d = atomicAdd(&st->diag_count, 1ull);
#pragma unroll
      for (int k = 0; k < W; ++k) out_z[d * W + k] = g.z[k][i];
      out_c[d] = ar.c[hit];
    }
  }
  __shared__ unsigned long long sl[kWarps];
  __shared__ double smx[kWarps], smn[kWarps];
  __shared__ uint32_t snf[kWarps], smc[kWarps];
  if (lane == 0) {
    sl[w] = live;
    smx[w] = mx;
    smn[w] = mn;
    snf[w] = nf;
    smc[w] = n;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t mc = 0;
    for (uint32_t k = 0; k < kWarps; ++k) {
      if (k) {
        live += sl[k];
        mx = fmax(mx, smx[k]);
        mn = fmin(mn, smn[k]);
        nf |= snf[k];
      }
      mc = max(mc, smc[k]);
    }
    if (live) atomicAdd(&out->live, live);
    atomic_max_nonneg(reinterpret_cast<double*>(&out->gmax_bits), mx);
    atomic_min_nonneg(reinterpret_cast<double*>(&out->gmin_bits), mn);
    if (nf) atomicOr(&out->nonfinite, 1u);
    if (mc) atomicMax(&out->maxcnt, mc);
  }
}

template <int W>
__global__ void k_diag(GroupView<W> g, uint32_t G, ArenaView<W> ar, uint64_t* out_z, double* out_c,
                       DevStats* st) {
  // warp per group: a sorted group holds x = 0 first; an unsorted one
  // (kFlagUnsorted) is searched by the warp
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (i >= (G != kKeepG ? G : *(volatile const unsigned int*)&st->G_dev)) return;
  const uint32_t n = g.cnt[i];
  if (n == 0) return;
  const uint64_t o = g.off[i];
  uint64_t hit = ~0ull;
  if ((g.flags[i] & (kFlagUnsorted | kFlagMinFirst)) == kFlagUnsorted) {
    for (uint32_t j0 = 0; j0 < n; j0 += 32) {
      const bool z = j0 + lane < n && plane_zero<W>(load_plane<W>(ar.x, o + j0 + lane));
      const uint32_t b = __ballot_sync(0xffffffffu, z);
      if (b) {
        hit = o + j0 + __ffs(b) - 1;
        break;
      }
    }
  } else if (plane_zero<W>(load_plane<W>(ar.x, o))) {
    hit = o;
  }
  if (lane != 0 || hit == ~0ull) return;
  unsigned long long d = atomicAdd(&st->diag_count, 1ull);
#pragma unroll
  for (int k = 0; k < W; ++k) out_z[d * W + k] = g.z[k][i];
  out_c[d] = ar.c[hit];
}

// ---------------------------------------------------------------------------
// compaction of the arena into the other buffer (garbage collection).
// Destination offsets are the exclusive scan of the group counts (group
// order, deterministic); the copy is load-balanced over the output: each
// CTA takes kGcTile consecutive output strings and every thread finds its
// group by binary search among the groups overlapping the tile, so a few
// huge groups and many tiny ones cost the same per string.
// ---------------------------------------------------------------------------
constexpr uint32_t kGcTile = 4 * kCta;

__device__ __forceinline__ uint32_t gc_find(const unsigned long long* off, uint32_t lo, uint32_t hi,
                                            unsigned long long i) {
  // last group in [lo, hi] with off <= i
  while (lo < hi) {
    const uint32_t mid = lo + (hi - lo + 1) / 2;
    if (off[mid] <= i) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

template <int W>
__global__ void __launch_bounds__(kCta) k_gc_copy(GroupView<W> g, uint32_t G, const unsigned long long* new_off,
                                                  unsigned long long total, ArenaView<W> src, ArenaView<W> dst) {
  __shared__ uint32_t range_s[2];
  for (unsigned long long t0 = (unsigned long long)blockIdx.x * kGcTile; t0 < total;
       t0 += (unsigned long long)gridDim.x * kGcTile) {
    const unsigned long long t1 = t0 + kGcTile < total ? t0 + kGcTile : total;
    __syncthreads();
    if (threadIdx.x < 2) range_s[threadIdx.x] = gc_find(new_off, 0, G - 1, threadIdx.x ? t1 - 1 : t0);
    __syncthreads();
    const uint32_t lo = range_s[0], hi = range_s[1];
#pragma unroll
    for (uint32_t k = 0; k < kGcTile / kCta; ++k) {
      const unsigned long long i = t0 + k * kCta + threadIdx.x;
      if (i >= t1) break;
      const uint32_t gid = gc_find(new_off, lo, hi, i);
      const unsigned long long s = g.off[gid] + (i - new_off[gid]);
#pragma unroll
      for (int w = 0; w < W; ++w) dst.x[w][i] = src.x[w][s];
      dst.c[i] = src.c[s];
    }
  }
}

// after the copy: the table points into the new arena, capacity = count
template <int W>
__global__ void k_gc_finish(GroupView<W> g, uint32_t G, const unsigned long long* new_off) {
  for (uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x; gid < G; gid += gridDim.x * blockDim.x) {
    g.off[gid] = new_off[gid];
    g.cap[gid] = g.cnt[gid];
  }
}

}  // namespace ppgpu
