// pp_regroup.cuh -- rebuilding the z-grouped store after gates that move
// strings between z-groups.
//
// Used for (a) a run of Clifford gates fused into one signed permutation of
// the strings (cos = 0, |sin| = 1: every anticommuting string moves to
// I xor J with coefficient (+-sin) c, exactly -- SURVEY.md section 0 fact 6;
// a permutation never merges, so the reference's per-gate passes and the
// fused map give identical sets), and (b) any gate whose generator carries a
// Z or Y (its children change z-group).
//
// Pipeline (all passes recompute the per-string records from the source
// arena, so no record buffer is materialised):
//   insert  -- hash every record's new z-plane into an open-addressing table
//              of (fingerprint, z, count); remember the slot per record
//   scan    -- prefix sums over the table give deterministic group ids and
//              arena offsets
//   scatter -- every record goes to its group's region
//   sort    -- each group's region is sorted by x; equal keys (a parent and
//              the child landing on it, at most two per key) are summed,
//              zeros dropped (TermMap::add + remove_below semantics)
#pragma once

#include "pp_kernels.cuh"

namespace ppgpu {

constexpr uint32_t kItem = 2048;  // strings per regroup work item

struct Item {
  uint32_t g;
  uint32_t start;
  uint32_t len;
  uint32_t pad;
  unsigned long long rbase;
};

template <int W>
struct Record {
  Plane<W> x, z;
  double c;
};

// (a) fused run of Clifford gates.  Gate planes live in device memory.
template <int W>
struct CliffordProducer {
  static constexpr int kMaxRec = 1;
  const uint64_t* gx;  // [ng][W]
  const uint64_t* gz;  // [ng][W]
  const double* gsin;  // [ng], +-1
  int ng;
  uint32_t seen_base;  // window index of gate 0 (batches_sent)
  // batches_sent: bit i of acc = gate i moved a nonzero string (|c| never
  // changes along the run, so a nonzero string stays nonzero)
  static constexpr int kMarkWords = kSeenWords;
  __device__ __forceinline__ void mark(Plane<W> x, Plane<W> z, double c, unsigned long long* acc) const {
    if (c == 0.0) return;
    for (int i = 0; i < ng && i < kSeenGates; ++i) {
      Plane<W> jx, jz;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        jx.w[k] = gx[i * W + k];
        jz.w[k] = gz[i * W + k];
      }
      if (plane_parity_and<W>(x, jz) ^ plane_parity_and<W>(z, jx)) {
        const unsigned long long m = 1ull << (i & 63);
        if (!(acc[i >> 6] & m)) atomicOr(&acc[i >> 6], m);
        x = plane_xor<W>(x, jx);
        z = plane_xor<W>(z, jz);
      }
    }
  }
  __device__ void flush(const unsigned long long* acc, DevStats* st) const {
    for (int i = threadIdx.x; i < ng && i < kSeenGates; i += blockDim.x)
      if ((acc[i >> 6] >> (i & 63)) & 1ull) mark_seen(st, seen_base + i);
  }
  __device__ __forceinline__ int emit(Plane<W> x, Plane<W> z, double c, Record<W>* out, uint32_t* nrec) const {
    uint32_t moved = 0;
    for (int i = 0; i < ng; ++i) {
      Plane<W> jx, jz;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        jx.w[k] = gx[i * W + k];
        jz.w[k] = gz[i * W + k];
      }
      if (plane_parity_and<W>(x, jz) ^ plane_parity_and<W>(z, jx)) {
        int b = phase_mod4<W>(x, z, jx, jz);
        double f = b == 1 ? gsin[i] : -gsin[i];  // record_sign * sin (engine.cpp:224)
        c = __dmul_rn(f, c);                     // exact: |f| == 1
        x = plane_xor<W>(x, jx);
        z = plane_xor<W>(z, jz);
        moved += (c != 0.0);
      }
    }
    out[0].x = x;
    out[0].z = z;
    out[0].c = c;
    *nrec = moved;
    return 1;
  }
};

// (a') fused run of Clifford Z_i Z_j gates, bit-parallel.  The run's edges
// are split on the host into matchings (no shared qubit) and, inside a
// matching, into groups of equal offset d = j - i; all gates of a group act on
// disjoint sites, so one group is applied at once:
//   a  = (x ^ x >> d) & M          anticommuting edges (x_i != x_j), at bit i
//   zs = the z bit of the x-carrying site (Y there -> record sign +,
//        X -> -; engine.cpp:67-81 with the phase table)
//   factor of an edge = sign * sin = -1 iff (zs == 0) xor (sin == -1)
//   z ^= a | a << d
// Commuting Clifford rotations compose to the same signed permutation in any
// order, so regrouping the run is exact.
constexpr int kMaxZZGroups = 64;  // keeps the kernel parameter block under 4 KB
static_assert(kMaxZZGroups == kZZSeenGroups, "DevStats::zz_seen holds one entry per ZZ group");

template <int W>
struct PlaneInt;
template <>
struct PlaneInt<1> {
  using T = unsigned long long;
};
template <>
struct PlaneInt<2> {
  using T = unsigned __int128;
};

template <int W>
struct ZZGroup {
  typename PlaneInt<W>::T m;    // bit i set for every edge (i, i + d) of the group
  typename PlaneInt<W>::T neg;  // edges whose gate has sin = -1
  int d;
};

template <int W>
struct ZZRunProducer {
  static constexpr int kMaxRec = 1;
  using T = typename PlaneInt<W>::T;
  int ng;
  ZZGroup<W> grp[kMaxZZGroups];
  // batches_sent: the anticommuting edges of every group (x never changes in
  // a ZZ run, so edge (i, i + d) sends a record iff some nonzero string has
  // x_i != x_{i+d}); the host maps (group, bit) back to gates
  static constexpr int kMarkWords = 2 * kMaxZZGroups;
  __device__ __forceinline__ void mark(Plane<W> xp, Plane<W> zp, double c, unsigned long long* acc) const {
    if (c == 0.0) return;
    const T x = pack(xp);
    for (int k = 0; k < ng; ++k) {
      const T a = (x ^ (x >> grp[k].d)) & grp[k].m;
      const unsigned long long lo = (unsigned long long)a;
      if (lo & ~acc[2 * k]) atomicOr(&acc[2 * k], lo);
      if constexpr (W == 2) {
        const unsigned long long hi = (unsigned long long)(a >> 64);
        if (hi & ~acc[2 * k + 1]) atomicOr(&acc[2 * k + 1], hi);
      }
    }
  }
  __device__ void flush(const unsigned long long* acc, DevStats* st) const {
    for (int w = threadIdx.x; w < 2 * ng; w += blockDim.x)
      if (acc[w]) atomicOr(&st->zz_seen[w >> 1][w & 1], acc[w]);
  }
  __device__ __forceinline__ static T pack(const Plane<W>& p) {
    if constexpr (W == 1) return p.w[0];
    else return (T)p.w[0] | ((T)p.w[1] << 64);
  }
  __device__ __forceinline__ static Plane<W> unpack(T v) {
    Plane<W> p;
    p.w[0] = (uint64_t)v;
    if constexpr (W == 2) p.w[1] = (uint64_t)(v >> 64);
    return p;
  }
  __device__ __forceinline__ static int popc(T v) {
    if constexpr (W == 1) return __popcll(v);
    else return __popcll((uint64_t)v) + __popcll((uint64_t)(v >> 64));
  }
  __device__ __forceinline__ int emit(Plane<W> xp, Plane<W> zp, double c, Record<W>* out, uint32_t* nrec) const {
    const T x = pack(xp);
    T z = pack(zp);
    int flips = 0, moved = 0;
    for (int k = 0; k < ng; ++k) {
      const T m = grp[k].m;
      const int d = grp[k].d;
      const T a = (x ^ (x >> d)) & m;
      if (!a) continue;
      const T xi = x & m;
      const T zs = (xi & z) | (~xi & (z >> d));  // z at the x-carrying site, at bit i
      flips += popc((~zs ^ grp[k].neg) & a);
      moved += popc(a);
      z ^= a | (a << d);
    }
    out[0].x = xp;
    out[0].z = unpack(z);
    out[0].c = (flips & 1) ? -c : c;  // a product of +-1 factors: exact
    *nrec = c != 0.0 ? (uint32_t)moved : 0u;
    return 1;
  }
};

// (c) identity: regroup the store as it is (merges groups that share a z,
// e.g. after strings received from other shards were appended as groups;
// equal keys are combined by the sort pass).
template <int W>
struct IdentityProducer {
  static constexpr int kMaxRec = 1;
  static constexpr int kMarkWords = 0;
  __device__ __forceinline__ void mark(Plane<W>, Plane<W>, double, unsigned long long*) const {}
  __device__ void flush(const unsigned long long*, DevStats*) const {}
  __device__ __forceinline__ int emit(Plane<W> x, Plane<W> z, double c, Record<W>* out, uint32_t* nrec) const {
    out[0].x = x;
    out[0].z = z;
    out[0].c = c;
    *nrec = 0;
    return 1;
  }
};

// ---------------------------------------------------------------------------
// sharding (multi-GPU): owner(z) is a hash of the z-plane, so an Rx gate
// (which keeps z) never moves a string between shards; Clifford/ZZ gates do,
// and whole z-groups are evicted to their new owner after a regroup.
// ---------------------------------------------------------------------------
// Load balancing: the z-hash picks one of kBuckets virtual
// buckets and a bucket table (rebalanced from the global bucket histogram at
// every exchange, pp_sharded.cuh) maps buckets to ranks; without a table the
// owner is the hash mod the rank count.
constexpr uint32_t kBuckets = 4096;
template <int W>
__host__ __device__ __forceinline__ uint64_t shard_hash(const Plane<W>& z, uint64_t seed) {
  uint64_t h = mix64(z.w[0] ^ seed);
  if (W == 2) h = mix64(h ^ z.w[W - 1]);
  return h;
}
template <int W>
__host__ __device__ __forceinline__ uint32_t shard_owner(const Plane<W>& z, uint64_t seed, uint32_t world,
                                                         const uint16_t* bucket_rank = nullptr) {
  const uint64_t h = shard_hash<W>(z, seed);
  return bucket_rank ? (uint32_t)bucket_rank[h % kBuckets] : (uint32_t)(h % world);
}

// strings per bucket of this rank's groups (the rebalance's local histogram)
template <int W>
__global__ void k_bucket_hist(GroupView<W> g, uint32_t G, uint64_t seed, unsigned long long* hist) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G || g.cnt[i] == 0) return;
  atomicAdd(&hist[shard_hash<W>(load_plane<W>(g.z, i), seed) % kBuckets], (unsigned long long)g.cnt[i]);
}

template <int W>
__global__ void k_evict_count(GroupView<W> g, uint32_t G, uint32_t world, uint32_t rank, uint64_t seed,
                              unsigned long long* counts, const uint16_t* bucket_rank) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G || g.cnt[i] == 0) return;
  uint32_t d = shard_owner<W>(load_plane<W>(g.z, i), seed, world, bucket_rank);
  if (d != rank) atomicAdd(&counts[d], (unsigned long long)g.cnt[i]);
}

// writes every string of every group owned elsewhere as a record
// [x words, z words, coefficient bits] at its destination's cursor, then
// empties the group
template <int W>
__global__ void __launch_bounds__(kCta) k_evict_write(GroupView<W> g, ArenaView<W> ar, uint32_t world, uint32_t rank,
                                                      uint64_t seed, unsigned long long* cursor, uint64_t* out,
                                                      const uint16_t* bucket_rank) {
  const uint32_t gid = blockIdx.x;
  const uint32_t n = g.cnt[gid];
  if (n == 0) return;
  const Plane<W> z = load_plane<W>(g.z, gid);
  const uint32_t d = shard_owner<W>(z, seed, world, bucket_rank);
  if (d == rank) return;
  __shared__ unsigned long long base_s;
  if (threadIdx.x == 0) base_s = atomicAdd(&cursor[d], (unsigned long long)n);
  __syncthreads();
  const uint64_t off = g.off[gid];
  for (uint32_t i = threadIdx.x; i < n; i += kCta) {
    uint64_t* r = out + (base_s + i) * (2 * W + 1);
#pragma unroll
    for (int k = 0; k < W; ++k) {
      r[k] = ar.x[k][off + i];
      r[W + k] = z.w[k];
    }
    r[2 * W] = (uint64_t)__double_as_longlong(ar.c[off + i]);
  }
  __syncthreads();
  if (threadIdx.x == 0) g.cnt[gid] = 0;
}

// appends received records to the arena as one group per run of equal z
// (run starts flagged in `start`, group ids from an exclusive scan `gid`)
template <int W>
__global__ void k_ingest_append(const uint64_t* rec, uint64_t count, const unsigned long long* gidscan, GroupView<W> g,
                                uint32_t G0, ArenaView<W> ar, uint64_t base) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const uint64_t* r = rec + i * (2 * W + 1);
#pragma unroll
  for (int k = 0; k < W; ++k) ar.x[k][base + i] = r[k];
  ar.c[base + i] = __longlong_as_double((long long)r[2 * W]);
  bool start = i == 0;
  if (!start) {
    const uint64_t* q = rec + (i - 1) * (2 * W + 1);
#pragma unroll
    for (int k = 0; k < W; ++k) start |= q[W + k] != r[W + k];
  }
  if (start) {
    uint32_t gi = G0 + (uint32_t)gidscan[i];
#pragma unroll
    for (int k = 0; k < W; ++k) g.z[k][gi] = r[W + k];
    g.off[gi] = base + i;
    g.gmax[gi] = 0.0;
    g.gmin[gi] = 0.0;
    g.flags[gi] = 0;
    g.stamp[gi] = 0xffffffffu;
  }
}

// group sizes of the appended runs from consecutive offsets
template <int W>
__global__ void k_ingest_counts(GroupView<W> g, uint32_t G0, uint32_t nruns, uint64_t end) {
  uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nruns) return;
  const uint32_t gi = G0 + j;
  const uint64_t next = j + 1 < nruns ? g.off[gi + 1] : end;
  g.cnt[gi] = (uint32_t)(next - g.off[gi]);
  g.cap[gi] = g.cnt[gi];
}

__global__ void k_run_starts(const uint64_t* rec, uint64_t count, int words, int zoff, uint32_t* flag) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  bool start = i == 0;
  if (!start)
    for (int k = 0; k < words; ++k) start |= rec[(i - 1) * (2 * words + 1) + zoff + k] != rec[i * (2 * words + 1) + zoff + k];
  flag[i] = start ? 1u : 0u;
}

// (b) one general gate: parent scaled by cos when it anticommutes, plus the
// child (I xor J, (+-sin) c) when the increment is nonzero (engine.cpp:
// 218-245).
template <int W>
struct GateProducer {
  static constexpr int kMaxRec = 2;
  Plane<W> jx, jz;
  double cosv, sinv;
  uint32_t seen_base;  // window index of the gate (batches_sent)
  static constexpr int kMarkWords = 1;
  __device__ __forceinline__ void mark(Plane<W> x, Plane<W> z, double c, unsigned long long* acc) const {
    if (acc[0] || !(plane_parity_and<W>(x, jz) ^ plane_parity_and<W>(z, jx))) return;
    const int b = phase_mod4<W>(x, z, jx, jz);
    if (__dmul_rn(b == 1 ? sinv : -sinv, c) != 0.0) atomicOr(&acc[0], 1ull);  // emit's record condition
  }
  __device__ void flush(const unsigned long long* acc, DevStats* st) const {
    if (threadIdx.x == 0 && acc[0]) mark_seen(st, seen_base);
  }
  __device__ __forceinline__ int emit(Plane<W> x, Plane<W> z, double c, Record<W>* out, uint32_t* nrec) const {
    out[0].x = x;
    out[0].z = z;
    *nrec = 0;
    if (!(plane_parity_and<W>(x, jz) ^ plane_parity_and<W>(z, jx))) {
      out[0].c = c;
      return 1;
    }
    int b = phase_mod4<W>(x, z, jx, jz);
    out[0].c = __dmul_rn(c, cosv);
    double d = __dmul_rn(b == 1 ? sinv : -sinv, c);
    if (d == 0.0) return 1;
    out[1].x = plane_xor<W>(x, jx);
    out[1].z = plane_xor<W>(z, jz);
    out[1].c = d;
    *nrec = 1;
    return 2;
  }
};

template <int W>
struct HashTable {
  unsigned long long* fp;  // 0 = empty
  uint64_t* z[W];
  uint32_t* count;
  uint32_t* gid;
  unsigned long long mask;
};

// work items: chunks of <= kItem strings of one group
template <int W>
__global__ void k_make_items(GroupView<W> g, uint32_t G, Item* items, int maxrec, DevStats* st) {
  uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G) return;
  uint32_t n = g.cnt[i];
  if (!n) return;
  uint32_t nch = (n + kItem - 1) / kItem;
  unsigned long long base = atomicAdd(&st->items, (unsigned long long)nch);
  unsigned long long rb = atomicAdd(&st->rec_total, (unsigned long long)n * maxrec);
  for (uint32_t k = 0; k < nch; ++k) {
    Item it;
    it.g = i;
    it.start = k * kItem;
    it.len = min(kItem, n - k * kItem);
    it.pad = 0;
    it.rbase = rb + (unsigned long long)k * kItem * maxrec;
    items[base + k] = it;
  }
}

template <int W>
__device__ __forceinline__ unsigned long long z_fingerprint(const Plane<W>& z, unsigned long long seed) {
  unsigned long long f = plane_hash<W>(z, seed);
  return f ? f : 1ull;
}

// Longest probe sequence before the table counts as too small (at load
// <= 1/2 sequences stay far below this).
constexpr uint32_t kMaxProbe = 4096;

template <int W, class P>
__global__ void __launch_bounds__(kCta) k_insert(const Item* items, GroupView<W> g, ArenaView<W> src, P prod,
                                                 HashTable<W> t, uint32_t* rec_slot, unsigned long long seed,
                                                 uint32_t max_distinct, DevStats* st) {
  if (blockIdx.x >= *(volatile const unsigned long long*)&st->items) return;  // grid may be an upper bound
  const Item it = items[blockIdx.x];
  const uint64_t off = g.off[it.g] + it.start;
  const Plane<W> z = load_plane<W>(g.z, it.g);
  unsigned long long records = 0;
  __shared__ unsigned long long s_mark[P::kMarkWords > 0 ? P::kMarkWords : 1];  // batches_sent
  for (int w = threadIdx.x; w < P::kMarkWords; w += kCta) s_mark[w] = 0;
  __syncthreads();
  if constexpr (P::kMaxRec == 1) {
    // one record per string: slot counts aggregated per warp (strings of one
    // item share their old z, so a warp's records fall into few new groups)
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t i0 = 0; i0 < it.len; i0 += kCta) {
      const uint32_t i = i0 + threadIdx.x;
      uint32_t slot_out = 0xffffffffu;
      if (i < it.len) {
        Record<W> rec[1];
        uint32_t nr = 0;
        const Plane<W> xi = load_plane<W>(src.x, off + i);
        const double ci = src.c[off + i];
        const int nrec = prod.emit(xi, z, ci, rec, &nr);
        if (nr) prod.mark(xi, z, ci, s_mark);
        records += nr;
        if (nrec) {
          const unsigned long long f = z_fingerprint<W>(rec[0].z, seed);
          unsigned long long sl = f & t.mask;
          for (unsigned long long probe = 0;; ++probe) {
            unsigned long long cur = t.fp[sl];
            if (cur == 0) {
              cur = atomicCAS(&t.fp[sl], 0ull, f);
              if (cur == 0) {
                uint32_t d = atomicAdd(&st->distinct, 1u);
                if (d >= max_distinct) atomicOr(&st->overflow, 1u);
                store_plane<W>(t.z, sl, rec[0].z);
                cur = f;
              }
            }
            if (cur == f) break;
            sl = (sl + 1) & t.mask;
            // a table that is too small (the host retries with a larger one):
            // stop probing it once anyone has found out
            if ((probe & 63) == 63 && *(volatile const unsigned int*)&st->overflow) break;
            if (probe > min(t.mask, (unsigned long long)kMaxProbe)) {
              atomicOr(&st->overflow, 1u);
              break;
            }
          }
          slot_out = (uint32_t)sl;
        }
        rec_slot[it.rbase + i] = slot_out;
      }
      const uint32_t mm = __match_any_sync(0xffffffffu, slot_out);
      if (slot_out != 0xffffffffu && lane == (uint32_t)(__ffs(mm) - 1)) atomicAdd(&t.count[slot_out], __popc(mm));
    }
  } else {
  for (uint32_t i = threadIdx.x; i < it.len; i += kCta) {
    Record<W> rec[P::kMaxRec];
    uint32_t nr = 0;
    const Plane<W> xi = load_plane<W>(src.x, off + i);
    const double ci = src.c[off + i];
    int nrec = prod.emit(xi, z, ci, rec, &nr);
    if (nr) prod.mark(xi, z, ci, s_mark);
    records += nr;
#pragma unroll
    for (int r = 0; r < P::kMaxRec; ++r) {
      uint32_t slot_out = 0xffffffffu;
      if (r < nrec) {
        unsigned long long f = z_fingerprint<W>(rec[r].z, seed);
        unsigned long long s = f & t.mask;
        for (unsigned long long probe = 0;; ++probe) {
          unsigned long long cur = t.fp[s];
          if (cur == 0) {
            cur = atomicCAS(&t.fp[s], 0ull, f);
            if (cur == 0) {
              uint32_t d = atomicAdd(&st->distinct, 1u);
              if (d >= max_distinct) atomicOr(&st->overflow, 1u);
              store_plane<W>(t.z, s, rec[r].z);
              cur = f;
            }
          }
          if (cur == f) break;
          s = (s + 1) & t.mask;
          if ((probe & 63) == 63 && *(volatile const unsigned int*)&st->overflow) break;
          if (probe > min(t.mask, (unsigned long long)kMaxProbe)) {
            atomicOr(&st->overflow, 1u);
            break;
          }
        }
        atomicAdd(&t.count[s], 1u);
        slot_out = (uint32_t)s;
      }
      rec_slot[it.rbase + (unsigned long long)i * P::kMaxRec + r] = slot_out;
    }
  }
  }
  records = warp_sum64(records);
  if ((threadIdx.x & 31) == 0 && records) atomicAdd(&st->records, records);
  __syncthreads();
  prod.flush(s_mark, st);
}

// --------------------------- device-wide exclusive scan over uint32 -> u64
constexpr uint32_t kScanPer = 8;
constexpr uint32_t kScanTile = kCta * kScanPer;

__global__ void __launch_bounds__(kCta) k_scan_tiles(const uint32_t* in, unsigned long long n, int as_flag,
                                                     unsigned long long* tile_sums) {
  __shared__ unsigned long long red[kWarps];
  unsigned long long b = (unsigned long long)blockIdx.x * kScanTile;
  unsigned long long s = 0;
  for (uint32_t k = 0; k < kScanPer; ++k) {
    unsigned long long i = b + k * kCta + threadIdx.x;
    if (i < n) {
      uint32_t v = in[i];
      s += as_flag ? (v != 0) : v;
    }
  }
  s = warp_sum64(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (uint32_t w = 0; w < kWarps; ++w) t += red[w];
    tile_sums[blockIdx.x] = t;
  }
}

// single CTA: exclusive scan of tile sums in place, total at [ntiles]
__global__ void __launch_bounds__(kCta) k_scan_sums(unsigned long long* sums, unsigned long long ntiles) {
  __shared__ unsigned long long carry_s;
  __shared__ unsigned long long wsum[kWarps];
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (unsigned long long base = 0; base < ntiles; base += kCta) {
    unsigned long long i = base + threadIdx.x;
    unsigned long long v = i < ntiles ? sums[i] : 0;
    unsigned long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long nb = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= (uint32_t)o) inc += nb;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    unsigned long long wpre = 0, tot = 0;
    for (uint32_t w = 0; w < kWarps; ++w) {
      if (w < warp) wpre += wsum[w];
      tot += wsum[w];
    }
    unsigned long long carry = carry_s;
    if (i < ntiles) sums[i] = carry + wpre + inc - v;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[ntiles] = carry_s;
}

__global__ void __launch_bounds__(kCta) k_scan_apply(const uint32_t* in, unsigned long long n, int as_flag,
                                                     const unsigned long long* tile_sums, unsigned long long* out) {
  __shared__ unsigned long long wsum[kWarps];
  __shared__ unsigned long long carry_s;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry_s = tile_sums[blockIdx.x];
  __syncthreads();
  unsigned long long b = (unsigned long long)blockIdx.x * kScanTile;
  for (uint32_t k = 0; k < kScanPer; ++k) {
    unsigned long long i = b + k * kCta + threadIdx.x;
    unsigned long long v = 0;
    if (i < n) {
      uint32_t x = in[i];
      v = as_flag ? (x != 0) : x;
    }
    unsigned long long inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      unsigned long long nb = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= (uint32_t)o) inc += nb;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    unsigned long long wpre = 0, tot = 0;
    for (uint32_t w = 0; w < kWarps; ++w) {
      if (w < warp) wpre += wsum[w];
      tot += wsum[w];
    }
    unsigned long long carry = carry_s;
    if (i < n) out[i] = carry + wpre + inc - v;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + tot;
    __syncthreads();
  }
}

// new group table from the hash table (slot order => deterministic ids)
template <int W>
__global__ void k_table_emit(HashTable<W> t, const unsigned long long* gid_scan, const unsigned long long* off_scan,
                             GroupView<W> ng, uint64_t arena_base, int final_counts = 0) {
  unsigned long long s = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (s > t.mask) return;
  uint32_t c = t.count[s];
  if (!c) return;
  uint32_t gid = (uint32_t)gid_scan[s];
  t.gid[s] = gid;
#pragma unroll
  for (int k = 0; k < W; ++k) ng.z[k][gid] = t.z[k][s];
  ng.off[gid] = arena_base + off_scan[s];
  ng.cap[gid] = c;
  // scatter cursor; final_counts: the scatter takes its positions from the
  // table's slot counts (one record per string) and the group count is final
  ng.cnt[gid] = final_counts ? c : 0;
  ng.flags[gid] = 0;
  ng.stamp[gid] = 0xffffffffu;
}

template <int W, class P>
__global__ void __launch_bounds__(kCta) k_scatter(const Item* items, GroupView<W> g, ArenaView<W> src, P prod,
                                                  HashTable<W> t, const uint32_t* rec_slot, GroupView<W> ng,
                                                  ArenaView<W> dst, DevStats* st,
                                                  const unsigned long long* off_scan = nullptr) {
  if (blockIdx.x >= *(volatile const unsigned long long*)&st->items) return;
  const Item it = items[blockIdx.x];
  const uint64_t off = g.off[it.g] + it.start;
  const Plane<W> z = load_plane<W>(g.z, it.g);
  if constexpr (P::kMaxRec == 1) {
    // positions reserved per warp and new group (one atomic per group per
    // warp), straight from the table slot: the slot's record count (final
    // after k_insert) is drawn down as the cursor and its offset comes from
    // the scan -- slot verify, offset and cursor are independent loads, two
    // dependent round trips per string instead of four (slot -> group id ->
    // group offset -> cursor)
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t i0 = 0; i0 < it.len; i0 += kCta) {
      const uint32_t i = i0 + threadIdx.x;
      uint32_t sl = 0xffffffffu;
      Record<W> rec[1];
      unsigned long long so = 0;
      if (i < it.len) {
        uint32_t nr;
        const int nrec = prod.emit(load_plane<W>(src.x, off + i), z, src.c[off + i], rec, &nr);
        if (nrec) {
          sl = rec_slot[it.rbase + i];
          so = off_scan[sl];
          if (!plane_eq<W>(load_plane<W>(t.z, sl), rec[0].z)) {  // fingerprint collision
            atomicOr(&st->collision, 1u);
            sl = 0xffffffffu;
          }
        }
      }
      const uint32_t mm = __match_any_sync(0xffffffffu, sl);
      if (sl != 0xffffffffu) {
        const uint32_t leader = __ffs(mm) - 1;
        const uint32_t k = (uint32_t)__popc(mm);
        uint32_t base = 0;
        if (lane == leader) base = atomicSub(&t.count[sl], k) - k;
        base = __shfl_sync(mm, base, leader);
        const uint64_t pos = so + base + __popc(mm & ((1u << lane) - 1u));
        store_plane<W>(dst.x, pos, rec[0].x);
        dst.c[pos] = rec[0].c;
      }
    }
  } else {
  for (uint32_t i = threadIdx.x; i < it.len; i += kCta) {
    Record<W> rec[P::kMaxRec];
    uint32_t nr;
    int nrec = prod.emit(load_plane<W>(src.x, off + i), z, src.c[off + i], rec, &nr);
#pragma unroll
    for (int r = 0; r < P::kMaxRec; ++r) {
      if (r >= nrec) break;
      uint32_t s = rec_slot[it.rbase + (unsigned long long)i * P::kMaxRec + r];
      if (!plane_eq<W>(load_plane<W>(t.z, s), rec[r].z)) {  // 64-bit fingerprint collision
        atomicOr(&st->collision, 1u);
        continue;
      }
      uint32_t gid = t.gid[s];
      uint64_t pos = ng.off[gid] + atomicAdd(&ng.cnt[gid], 1u);
      store_plane<W>(dst.x, pos, rec[r].x);
      dst.c[pos] = rec[r].c;
    }
  }
  }
}

// ---------------------------------------------------------------------------
// per-group sort by x + pair combine + zero drop
// ---------------------------------------------------------------------------
constexpr uint32_t kSortSmall = 2048;

constexpr uint32_t kSortPackGroup = 256;  // groups up to this size are sorted in packs

template <int W>
struct SortSmem {
  uint64_t key[W * kSortSmall];
  double val[kSortSmall];
  uint16_t gk[kSortSmall];     // pack: group of each string (0xffff = padding)
  uint8_t em[kSortSmall];      // pack: emitted after combining
  uint32_t scan[40];
  // pack bookkeeping for one chunk of kCta consecutive groups
  uint32_t plist[kCta], pp[kCta + 1], pfirst[kCta + 1], mlist[kCta];
  uint32_t gstart[kCta + 1], estart[kCta + 1], pgid[kCta];
  uint64_t poff[kCta];
};

// bitonic sort of smem [0, npow2) (npow2 power of two, padded with max keys)
template <int W>
__device__ void smem_bitonic(uint64_t* key, double* val, uint32_t stride, uint32_t npow2) {
  for (uint32_t size = 2; size <= npow2; size <<= 1) {
    for (uint32_t j = size >> 1; j > 0; j >>= 1) {
      for (uint32_t t = threadIdx.x; t < (npow2 >> 1); t += blockDim.x) {
        uint32_t i = 2 * j * (t / j) + (t % j);
        uint32_t l = i + j;
        bool up = ((i & size) == 0);
        Plane<W> a = sk_load<W>(key, stride, i), b = sk_load<W>(key, stride, l);
        bool swap = up ? plane_lt<W>(b, a) : plane_lt<W>(a, b);
        if (swap) {
          sk_store<W>(key, stride, i, b);
          sk_store<W>(key, stride, l, a);
          double tv = val[i];
          val[i] = val[l];
          val[l] = tv;
        }
      }
      __syncthreads();
    }
  }
}

// combine adjacent equal keys of a sorted sequence, drop zeros (unless
// keep_zeros), stream to dst; accessor functions read the sorted input.
// Returns the number written; accumulates stats.  `in_key/in_val` are the
// sorted input (global or shared), `dst` the output region (may alias the
// input when writes never overtake reads, which holds for in-place use).
template <int W, class GetK, class GetV>
__device__ uint32_t combine_stream(uint32_t n, GetK getk, GetV getv, ArenaView<W> ar, uint64_t dst, int keep_zeros,
                                   uint32_t* scan, double& vmax, double& vmin, uint32_t& nonfinite,
                                   unsigned long long& removed) {
  uint32_t w = 0;
  for (uint32_t base = 0; base < n; base += kCta) {
    uint32_t p = base + threadIdx.x;
    bool e = false;
    Plane<W> k;
    double v = 0.0;
    if (p < n) {
      k = getk(p);
      bool head = (p == 0) || !plane_eq<W>(getk(p - 1), k);
      if (head) {
        v = getv(p);
        if (p + 1 < n && plane_eq<W>(getk(p + 1), k)) v = __dadd_rn(v, getv(p + 1));
        e = keep_zeros || v != 0.0;
        if (!e) ++removed;
      }
    }
    uint32_t tot;
    uint32_t o = block_excl_scan(e ? 1u : 0u, scan, &tot);
    if (e) {
      store_plane<W>(ar.x, dst + w + o, k);
      ar.c[dst + w + o] = v;
      double av = fabs(v);
      if (!(av <= 1.7976931348623157e308)) nonfinite = 1;
      vmax = fmax(vmax, av);
      vmin = fmin(vmin, av);
    }
    w += tot;
    __syncthreads();
  }
  return w;
}

template <int W>
__device__ void finish_group_stats(GroupView<W> g, uint32_t gid, uint32_t count, double vmax, double vmin,
                                   uint32_t nonfinite, unsigned long long removed, DevStats* st) {
  __shared__ double rmx[kWarps], rmn[kWarps];
  __shared__ unsigned long long rrm[kWarps];
  __shared__ uint32_t rnf[kWarps];
  vmax = warp_max(vmax);
  vmin = warp_min(vmin);
  removed = warp_sum64(removed);
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  const uint32_t tid = threadIdx.x;
  if ((tid & 31) == 0) {
    rmx[tid >> 5] = vmax;
    rmn[tid >> 5] = vmin;
    rrm[tid >> 5] = removed;
    rnf[tid >> 5] = nonfinite;
  }
  __syncthreads();
  if (tid == 0) {
    for (uint32_t i = 1; i < kWarps; ++i) {
      vmax = fmax(vmax, rmx[i]);
      vmin = fmin(vmin, rmn[i]);
      removed += rrm[i];
      nonfinite |= rnf[i];
    }
    g.cnt[gid] = count;
    g.gmax[gid] = count ? vmax : 0.0;
    g.gmin[gid] = count ? vmin : __longlong_as_double(0x7ff0000000000000ll);
    g.flags[gid] = nonfinite;
    if (removed) atomicAdd(&st->removed, removed);
  }
}

// bitonic sort of (group, x) pairs: a pack of small groups sorts in one pass
template <int W>
__device__ void smem_bitonic_pack(uint64_t* key, double* val, uint16_t* gk, uint32_t stride, uint32_t npow2) {
  for (uint32_t size = 2; size <= npow2; size <<= 1) {
    for (uint32_t j = size >> 1; j > 0; j >>= 1) {
      for (uint32_t t = threadIdx.x; t < (npow2 >> 1); t += blockDim.x) {
        const uint32_t i = 2 * j * (t / j) + (t % j);
        const uint32_t l = i + j;
        const bool up = ((i & size) == 0);
        const uint16_t ga = gk[i], gb = gk[l];
        const Plane<W> a = sk_load<W>(key, stride, i), b = sk_load<W>(key, stride, l);
        const bool b_lt_a = gb < ga || (gb == ga && plane_lt<W>(b, a));
        const bool a_lt_b = ga < gb || (ga == gb && plane_lt<W>(a, b));
        if (up ? b_lt_a : a_lt_b) {
          sk_store<W>(key, stride, i, b);
          sk_store<W>(key, stride, l, a);
          gk[i] = gb;
          gk[l] = ga;
          const double tv = val[i];
          val[i] = val[l];
          val[l] = tv;
        }
      }
      __syncthreads();
    }
  }
}

// Sorts groups of <= kSortSmall strings by x and combines equal keys in
// place.  Each CTA walks chunks of kCta consecutive groups: groups of at most
// kSortPackGroup strings are sorted together in packs of <= kSortSmall
// strings (one bitonic pass on (group, x)), larger ones one by one.
template <int W>
__global__ void __launch_bounds__(kCta) k_sort_small(GroupView<W> g, ArenaView<W> ar, int keep_zeros, DevStats* st,
                                                     int only_unsorted = 0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SortSmem<W>& sm = *reinterpret_cast<SortSmem<W>*>(smem_raw);
  const uint32_t G = *(volatile const unsigned int*)&st->distinct;
  const uint32_t tid = threadIdx.x;
  constexpr uint32_t kPer = kSortSmall / kCta;  // strings per thread in the blocked passes
  unsigned long long removed_pk = 0;
  // chunks of consecutive groups, sized so every CTA gets work when G is small
  const uint32_t chunk = max(1u, min(kCta, (G + gridDim.x - 1) / gridDim.x));
  for (uint32_t c0 = blockIdx.x * chunk; c0 < G; c0 += gridDim.x * chunk) {
    __syncthreads();
    const uint32_t gi = c0 + tid;
    const uint32_t nt =
        (tid < chunk && gi < G && sort_wanted(g.flags[gi], only_unsorted)) ? g.cnt[gi] : 0u;
    const bool small = nt > 0 && nt <= kSortPackGroup;
    const bool single = nt > kSortPackGroup && nt <= kSortSmall;
    uint32_t nsmall, tsz, nsingle;
    const uint32_t r = block_excl_scan(small ? 1u : 0u, sm.scan, &nsmall);
    const uint32_t P = block_excl_scan(small ? nt : 0u, sm.scan, &tsz);
    const uint32_t rs = block_excl_scan(single ? 1u : 0u, sm.scan, &nsingle);
    if (small) {
      sm.plist[r] = gi;
      sm.pp[r] = P;
    }
    if (single) sm.mlist[rs] = gi;
    if (tid == 0) sm.pp[nsmall] = tsz;
    __syncthreads();
    // a pack: groups whose start prefix shares one window of kSortSmall - kSortPackGroup strings
    constexpr uint32_t kWin = kSortSmall - kSortPackGroup;
    const bool start = tid < nsmall && (tid == 0 || sm.pp[tid] / kWin != sm.pp[tid - 1] / kWin);
    uint32_t npk;
    const uint32_t q = block_excl_scan(start ? 1u : 0u, sm.scan, &npk);
    if (start) sm.pfirst[q] = tid;
    if (tid == 0) sm.pfirst[npk] = nsmall;
    __syncthreads();
    for (uint32_t pj = 0; pj < npk; ++pj) {
      const uint32_t a = sm.pfirst[pj], b = sm.pfirst[pj + 1];
      const uint32_t m = b - a, base = sm.pp[a], total = sm.pp[b] - base;
      __syncthreads();
      if (tid < m) {
        const uint32_t gid = sm.plist[a + tid];
        sm.pgid[tid] = gid;
        sm.poff[tid] = g.off[gid];
        sm.gstart[tid] = sm.pp[a + tid] - base;
      }
      if (tid == 0) sm.gstart[m] = total;
      __syncthreads();
      uint32_t np2 = 1;
      while (np2 < total) np2 <<= 1;
      for (uint32_t i = tid; i < np2; i += kCta) {
        if (i < total) {
          uint32_t lo = 0, hi = m;  // group of string i
          while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) >> 1;
            if (sm.gstart[mid] <= i) lo = mid;
            else hi = mid;
          }
          const uint64_t src = sm.poff[lo] + (i - sm.gstart[lo]);
          sk_store<W>(sm.key, kSortSmall, i, load_plane<W>(ar.x, src));
          sm.val[i] = ar.c[src];
          sm.gk[i] = (uint16_t)lo;
        } else {
          sk_store<W>(sm.key, kSortSmall, i, plane_max<W>());
          sm.val[i] = 0.0;
          sm.gk[i] = 0xffff;
        }
      }
      __syncthreads();
      if (np2 > 1) smem_bitonic_pack<W>(sm.key, sm.val, sm.gk, kSortSmall, np2);
      // combine equal (group, x) neighbours (at most two per key: one
      // scaled parent and one record, or two records of one gate)
      double cv[kPer];
      uint32_t emask = 0, cnt = 0;
#pragma unroll
      for (uint32_t v = 0; v < kPer; ++v) {
        const uint32_t p = tid * kPer + v;
        cv[v] = 0.0;
        if (p < total) {
          const uint16_t k = sm.gk[p];
          const Plane<W> key = sk_load<W>(sm.key, kSortSmall, p);
          const bool head = p == 0 || sm.gk[p - 1] != k || !plane_eq<W>(sk_load<W>(sm.key, kSortSmall, p - 1), key);
          if (head) {
            double x = sm.val[p];
            if (p + 1 < total && sm.gk[p + 1] == k && plane_eq<W>(sk_load<W>(sm.key, kSortSmall, p + 1), key))
              x = __dadd_rn(x, sm.val[p + 1]);
            cv[v] = x;
            if (keep_zeros || x != 0.0) {
              emask |= 1u << v;
              ++cnt;
            } else {
              ++removed_pk;
            }
          }
        }
      }
      uint32_t etot;
      uint32_t e = block_excl_scan(cnt, sm.scan, &etot);  // barrier: all neighbour reads are done
#pragma unroll
      for (uint32_t v = 0; v < kPer; ++v) {
        const uint32_t p = tid * kPer + v;
        if (p < total) {
          sm.val[p] = cv[v];
          sm.em[p] = (emask >> v) & 1u;
          if (p == sm.gstart[sm.gk[p]]) sm.estart[sm.gk[p]] = e;  // a group's first string is a head
        }
        e += (emask >> v) & 1u;
      }
      if (tid == 0) sm.estart[m] = etot;
      __syncthreads();
      // write back each group in place (its region was fully read above)
      e -= cnt;
#pragma unroll
      for (uint32_t v = 0; v < kPer; ++v) {
        const uint32_t p = tid * kPer + v;
        if ((emask >> v) & 1u) {
          const uint16_t k = sm.gk[p];
          const uint64_t d = sm.poff[k] + (e - sm.estart[k]);
          store_plane<W>(ar.x, d, sk_load<W>(sm.key, kSortSmall, p));
          ar.c[d] = cv[v];
          ++e;
        }
      }
      // per-group statistics: one warp per group
      const uint32_t lane = tid & 31;
      for (uint32_t k = tid >> 5; k < m; k += kWarps) {
        double gx = 0.0, gn = __longlong_as_double(0x7ff0000000000000ll);
        uint32_t nf = 0;
        for (uint32_t p = sm.gstart[k] + lane; p < sm.gstart[k + 1]; p += 32) {
          if (!sm.em[p]) continue;
          const double av = fabs(sm.val[p]);
          if (!(av <= 1.7976931348623157e308)) nf = 1;
          gx = fmax(gx, av);
          gn = fmin(gn, av);
        }
        gx = warp_max(gx);
        gn = warp_min(gn);
        nf = __any_sync(0xffffffffu, nf);
        if (lane == 0) {
          const uint32_t gid = sm.pgid[k];
          const uint32_t c = sm.estart[k + 1] - sm.estart[k];
          g.cnt[gid] = c;
          g.gmax[gid] = c ? gx : 0.0;
          g.gmin[gid] = c ? gn : __longlong_as_double(0x7ff0000000000000ll);
          g.flags[gid] = nf;
        }
      }
    }
    // groups between kSortPackGroup and kSortSmall strings: one by one
    for (uint32_t mi = 0; mi < nsingle; ++mi) {
      __syncthreads();
      const uint32_t gid = sm.mlist[mi];
      const uint32_t n = g.cnt[gid];
      const uint64_t off = g.off[gid];
      uint32_t np2 = 1;
      while (np2 < n) np2 <<= 1;
      for (uint32_t i = tid; i < np2; i += kCta) {
        if (i < n) {
          sk_store<W>(sm.key, kSortSmall, i, load_plane<W>(ar.x, off + i));
          sm.val[i] = ar.c[off + i];
        } else {
          sk_store<W>(sm.key, kSortSmall, i, plane_max<W>());
          sm.val[i] = 0.0;
        }
      }
      __syncthreads();
      if (np2 > 1) smem_bitonic<W>(sm.key, sm.val, kSortSmall, np2);
      double vmax = 0.0, vmin = __longlong_as_double(0x7ff0000000000000ll);
      uint32_t nf = 0;
      unsigned long long removed = 0;
      auto getk = [&](uint32_t p) { return sk_load<W>(sm.key, kSortSmall, p); };
      auto getv = [&](uint32_t p) { return sm.val[p]; };
      uint32_t w = combine_stream<W>(n, getk, getv, ar, off, keep_zeros, sm.scan, vmax, vmin, nf, removed);
      finish_group_stats<W>(g, gid, w, vmax, vmin, nf, removed, st);
    }
  }
  removed_pk = warp_sum64(removed_pk);
  if ((tid & 31) == 0 && removed_pk) atomicAdd(&st->removed, removed_pk);
}

// two-run merge of sorted runs a=[0,na) and b=[0,nb) (global) into out,
// stable (ties: a first), one CTA, buffered through shared memory.
template <int W>
struct MergeSmem {
  uint64_t key[2][W * kBufCap];
  double val[2][kBufCap];
  uint64_t okey[W * 2 * kBufCap];
  double oval[2 * kBufCap];
  uint32_t cnt[2], pos[2], m[2];
};

template <int W>
__device__ void cta_merge_runs(MergeSmem<W>& sm, ArenaView<W> ar, uint64_t a, uint32_t na, uint64_t b, uint32_t nb,
                               ArenaView<W> out, uint64_t o) {
  const uint32_t tid = threadIdx.x;
  const uint64_t srcb[2] = {a, b};
  const uint32_t len[2] = {na, nb};
  if (tid == 0) {
    sm.cnt[0] = sm.cnt[1] = 0;
    sm.pos[0] = sm.pos[1] = 0;
  }
  __syncthreads();
  uint64_t written = 0;
  for (;;) {
    for (int s = 0; s < 2; ++s) {
      while (sm.cnt[s] < kRefill && sm.pos[s] < len[s]) {
        uint32_t take = min(kCta, len[s] - sm.pos[s]);
        if (tid < take) {
          uint64_t p = srcb[s] + sm.pos[s] + tid;
          sk_store<W>(sm.key[s], kBufCap, sm.cnt[s] + tid, load_plane<W>(ar.x, p));
          sm.val[s][sm.cnt[s] + tid] = ar.c[p];
        }
        __syncthreads();
        if (tid == 0) {
          sm.cnt[s] += take;
          sm.pos[s] += take;
        }
        __syncthreads();
      }
    }
    if (tid < 2) {
      Plane<W> kmax = plane_max<W>();
      bool bounded = false;
      for (int s = 0; s < 2; ++s) {
        if (sm.pos[s] < len[s]) {
          Plane<W> last = sk_load<W>(sm.key[s], kBufCap, sm.cnt[s] - 1);
          if (!bounded || plane_lt<W>(last, kmax)) kmax = last;
          bounded = true;
        }
      }
      sm.m[tid] = bounded ? sk_upper_bound<W>(sm.key[tid], kBufCap, sm.cnt[tid], kmax) : sm.cnt[tid];
    }
    __syncthreads();
    const uint32_t ma = sm.m[0], mb = sm.m[1];
    for (uint32_t i = tid; i < ma + mb; i += kCta) {
      bool isa = i < ma;
      uint32_t j = isa ? i : i - ma;
      Plane<W> k = sk_load<W>(sm.key[isa ? 0 : 1], kBufCap, j);
      uint32_t r = isa ? j + sk_lower_bound<W>(sm.key[1], kBufCap, mb, k)
                       : j + sk_upper_bound<W>(sm.key[0], kBufCap, ma, k);
      sk_store<W>(sm.okey, 2 * kBufCap, r, k);
      sm.oval[r] = sm.val[isa ? 0 : 1][j];
    }
    __syncthreads();
    for (uint32_t i = tid; i < ma + mb; i += kCta) {
      store_plane<W>(out.x, o + written + i, sk_load<W>(sm.okey, 2 * kBufCap, i));
      out.c[o + written + i] = sm.oval[i];
    }
    written += ma + mb;
    // shift remaining
    uint32_t rem[2] = {sm.cnt[0] - ma, sm.cnt[1] - mb};
    Plane<W> tk[2][kBufCap / kCta];
    double tv[2][kBufCap / kCta];
    for (int s = 0; s < 2; ++s)
      for (uint32_t r = 0; r < kBufCap / kCta; ++r) {
        uint32_t i = tid + r * kCta;
        if (i < rem[s]) {
          tk[s][r] = sk_load<W>(sm.key[s], kBufCap, sm.m[s] + i);
          tv[s][r] = sm.val[s][sm.m[s] + i];
        }
      }
    __syncthreads();
    for (int s = 0; s < 2; ++s)
      for (uint32_t r = 0; r < kBufCap / kCta; ++r) {
        uint32_t i = tid + r * kCta;
        if (i < rem[s]) {
          sk_store<W>(sm.key[s], kBufCap, i, tk[s][r]);
          sm.val[s][i] = tv[s][r];
        }
      }
    __syncthreads();
    bool done = rem[0] == 0 && rem[1] == 0 && sm.pos[0] >= len[0] && sm.pos[1] >= len[1];
    if (tid == 0) {
      sm.cnt[0] = rem[0];
      sm.cnt[1] = rem[1];
    }
    __syncthreads();
    if (done) break;
  }
}

// big groups (> kSortSmall): chunk bitonic sorts, then log2 merge passes
// ping-ponging between the group's region and a scratch region, then the
// combine pass back into the region.  One CTA per group.
template <int W>
__global__ void __launch_bounds__(kCta) k_sort_big(GroupView<W> g, ArenaView<W> ar, ArenaView<W> scratch,
                                                   int keep_zeros, DevStats* st, int only_unsorted = 0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const uint32_t G = *(volatile const unsigned int*)&st->distinct;
  for (uint32_t gid = blockIdx.x; gid < G; gid += gridDim.x) {
  __syncthreads();
  const uint32_t n = g.cnt[gid];
  if (n <= kSortSmall) continue;
  if (!sort_wanted(g.flags[gid], only_unsorted)) continue;
  const uint64_t off = g.off[gid];
  __shared__ unsigned long long so_s;
  if (threadIdx.x == 0) so_s = atomicAdd(&st->scratch_bump, (unsigned long long)n);
  __syncthreads();
  const uint64_t so = so_s;
  {
    SortSmem<W>& sm = *reinterpret_cast<SortSmem<W>*>(smem_raw);
    for (uint32_t c0 = 0; c0 < n; c0 += kSortSmall) {
      uint32_t len = min(kSortSmall, n - c0);
      for (uint32_t i = threadIdx.x; i < kSortSmall; i += kCta) {
        if (i < len) {
          sk_store<W>(sm.key, kSortSmall, i, load_plane<W>(ar.x, off + c0 + i));
          sm.val[i] = ar.c[off + c0 + i];
        } else {
          sk_store<W>(sm.key, kSortSmall, i, plane_max<W>());
          sm.val[i] = 0.0;
        }
      }
      __syncthreads();
      smem_bitonic<W>(sm.key, sm.val, kSortSmall, kSortSmall);
      for (uint32_t i = threadIdx.x; i < len; i += kCta) {
        store_plane<W>(ar.x, off + c0 + i, sk_load<W>(sm.key, kSortSmall, i));
        ar.c[off + c0 + i] = sm.val[i];
      }
      __syncthreads();
    }
  }
  MergeSmem<W>& mm = *reinterpret_cast<MergeSmem<W>*>(smem_raw);
  bool in_region = true;
  for (uint32_t run = kSortSmall; run < n; run <<= 1) {
    ArenaView<W> from = in_region ? ar : scratch;
    ArenaView<W> to = in_region ? scratch : ar;
    uint64_t fo = in_region ? off : so, to_o = in_region ? so : off;
    for (uint32_t s0 = 0; s0 < n; s0 += 2 * run) {
      uint32_t na = min(run, n - s0);
      uint32_t nb = (s0 + run < n) ? min(run, n - s0 - run) : 0;
      if (nb == 0) {
        for (uint32_t i = threadIdx.x; i < na; i += kCta) {
          store_plane<W>(to.x, to_o + s0 + i, load_plane<W>(from.x, fo + s0 + i));
          to.c[to_o + s0 + i] = from.c[fo + s0 + i];
        }
        __syncthreads();
      } else {
        // cta_merge_runs reads from a single arena view; both runs are in `from`
        cta_merge_runs<W>(mm, from, fo + s0, na, fo + s0 + run, nb, to, to_o + s0);
      }
    }
    in_region = !in_region;
    __syncthreads();
  }
  __shared__ uint32_t scan[40];
  double vmax = 0.0, vmin = __longlong_as_double(0x7ff0000000000000ll);
  uint32_t nf = 0;
  unsigned long long removed = 0;
  ArenaView<W> fin = in_region ? ar : scratch;
  uint64_t fo = in_region ? off : so;
  auto getk = [&](uint32_t p) { return load_plane<W>(fin.x, fo + p); };
  auto getv = [&](uint32_t p) { return fin.c[fo + p]; };
  uint32_t w = combine_stream<W>(n, getk, getv, ar, off, keep_zeros, scan, vmax, vmin, nf, removed);
  finish_group_stats<W>(g, gid, w, vmax, vmin, nf, removed, st);
  }
}

// Both exclusive scans of the regroup's slot counts (as flags: group ids;
// as values: string offsets) for a small table, in one single-CTA launch:
// each thread owns a contiguous chunk, one block scan of the chunk sums.
constexpr uint32_t kScanPairMax = 1u << 16;
constexpr uint32_t kScanPairThreads = 1024;
__global__ void __launch_bounds__(kScanPairThreads) k_scan_pair_small(const uint32_t* in, uint32_t n,
                                                                      unsigned long long* out_flag,
                                                                      unsigned long long* out_cnt, DevStats* st) {
  // a warp per contiguous segment, lanes striped (coalesced): warp totals,
  // one scan over the 32 warps, then per-chunk warp scans with a carry
  __shared__ uint32_t wf[32], wc[32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t seg = (n + 31) / 32;
  const uint32_t s0 = min(n, warp * seg), s1 = min(n, s0 + seg);
  uint32_t f = 0, c = 0;
  for (uint32_t i = s0 + lane; i < s1; i += 32) {
    const uint32_t v = in[i];
    f += v != 0;
    c += v;
  }
  f = __reduce_add_sync(0xffffffffu, f);
  c = __reduce_add_sync(0xffffffffu, c);
  if (lane == 0) {
    wf[warp] = f;
    wc[warp] = c;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t a = wf[lane], b = wc[lane];
    const uint32_t ia = warp_incl_scan(a), ib = warp_incl_scan(b);
    wf[lane] = ia - a;
    wc[lane] = ib - b;
    if (lane == 31) st->scan_total = ib;
  }
  __syncthreads();
  uint32_t bf = wf[warp], bc = wc[warp];
  for (uint32_t i0 = s0; i0 < s1; i0 += 32) {
    const uint32_t i = i0 + lane;
    const uint32_t v = i < s1 ? in[i] : 0u, fv = v != 0;
    const uint32_t ifl = warp_incl_scan(fv), icn = warp_incl_scan(v);
    if (i < s1) {
      out_flag[i] = bf + ifl - fv;
      out_cnt[i] = bc + icn - v;
    }
    bf += __shfl_sync(0xffffffffu, ifl, 31);
    bc += __shfl_sync(0xffffffffu, icn, 31);
  }
}

// Whole regroup of a small store in one CTA (a Clifford run feeding a dense
// Rx run: no x order needed).  Strings are mapped by the producer, grouped by
// their new z in a shared-memory hash table (open addressing, a state word per
// slot: empty / being written / ready), counted, given group ids and offsets
// by two block scans in slot order, scattered into the target arena, and the
// new table is filled (statistics by a warp per group, kFlagUnsorted).  The
// device takes the new group count and bump pointer (as k_regroup_commit).
constexpr uint32_t kSmallRegroupThreads = 1024;
constexpr uint32_t kSmallRegroupMax = 1024;  // strings: larger stores run faster through the multi-CTA pipeline
constexpr uint32_t small_regroup_tc(uint32_t n) {  // table slots: load <= 2/3
  uint32_t tc = 1024;
  while (tc < n + n / 2) tc <<= 1;
  return tc;
}
template <int W>
constexpr size_t small_regroup_smem(uint32_t tc, uint32_t n) {
  // table (key, state, count, offset, max / min |c| bits, non-finite per
  // slot), slot per string, group prefix
  return (size_t)tc * (8 + 12 + 8 * W + 16 + 4) + (size_t)n * 2 + 16 + (size_t)(n + 1) * 4 + 64;
}

template <int W, class P>
__global__ void __launch_bounds__(kSmallRegroupThreads) k_regroup_small(GroupView<W> gi, uint32_t Gi, ArenaView<W> ai,
                                                                        P prod, GroupView<W> go, ArenaView<W> ao,
                                                                        uint32_t n, uint32_t tc, DevStats* st,
                                                                        unsigned long long bump0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  unsigned long long* kfp = reinterpret_cast<unsigned long long*>(smem_raw);  // fingerprint of the slot's z (0: empty)
  uint64_t* key = reinterpret_cast<uint64_t*>(kfp + tc);         // [W][tc] the slot's z
  uint32_t* state = reinterpret_cast<uint32_t*>(key + W * tc);   // scatter cursor
  uint32_t* cnt = state + tc;
  uint32_t* off = cnt + tc;
  unsigned long long* smx = reinterpret_cast<unsigned long long*>(off + tc);  // max |c| bits per slot
  unsigned long long* smn = smx + tc;                                          // min |c| bits per slot
  uint32_t* snf = reinterpret_cast<uint32_t*>(smn + tc);                       // non-finite per slot
  uint16_t* slot = reinterpret_cast<uint16_t*>(snf + tc);        // per string, in flattened order
  uint32_t* gpre = reinterpret_cast<uint32_t*>(slot + ((n + 7) & ~7u));  // input group prefix (Gi + 1; Gi <= n)
  __shared__ uint32_t scr[40];
  __shared__ unsigned long long s_rec;
  __shared__ unsigned long long s_mark[P::kMarkWords > 0 ? P::kMarkWords : 1];  // batches_sent
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  for (int w = tid; w < P::kMarkWords; w += kSmallRegroupThreads) s_mark[w] = 0;
  for (uint32_t h = tid; h < tc; h += kSmallRegroupThreads) {
    kfp[h] = 0ull;
    state[h] = 0;
    cnt[h] = 0;
    smx[h] = 0ull;
    smn[h] = 0x7ff0000000000000ull;
    snf[h] = 0;
  }
  if (tid == 0) {
    s_rec = 0;
    k_reset_stats_body(st, bump0);  // as reset_stats() before a regroup
  }
  __syncthreads();
  // input group prefix (strings flattened in group order)
  {
    constexpr uint32_t kG = (kSmallRegroupMax + kSmallRegroupThreads - 1) / kSmallRegroupThreads;
    uint32_t c[kG], sum = 0;
#pragma unroll
    for (uint32_t e = 0; e < kG; ++e) {
      const uint32_t q = tid * kG + e;
      c[e] = q < Gi ? gi.cnt[q] : 0u;
      sum += c[e];
    }
    uint32_t tot;
    uint32_t p = block_excl_scan(sum, scr, &tot);
#pragma unroll
    for (uint32_t e = 0; e < kG; ++e) {
      const uint32_t q = tid * kG + e;
      if (q < Gi) gpre[q] = p;
      p += c[e];
    }
    if (tid == 0) gpre[Gi] = tot;
  }
  __syncthreads();
  auto group_of = [&](uint32_t i) -> uint32_t {  // last group with gpre <= i
    uint32_t lo = 0, hi = Gi;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (gpre[mid] <= i) lo = mid;
      else hi = mid;
    }
    return lo;
  };
  // map + insert, a thread per string
  unsigned long long rec = 0;
  for (uint32_t i = tid; i < n; i += kSmallRegroupThreads) {
    const uint32_t gg = group_of(i);
    const uint64_t a = gi.off[gg] + (i - gpre[gg]);
    Plane<W> z;
#pragma unroll
    for (int k = 0; k < W; ++k) z.w[k] = gi.z[k][gg];
    Record<W> r;
    uint32_t nrec = 0;
    const Plane<W> xa = load_plane<W>(ai.x, a);
    prod.emit(xa, z, ai.c[a], &r, &nrec);
    if (nrec) prod.mark(xa, z, ai.c[a], s_mark);
    rec += nrec;
    // slots by a 64-bit fingerprint (no waiting on another thread's key);
    // the scatter verifies the full z (a collision fails the deferred check)
    const unsigned long long fp = plane_hash<W>(r.z, 0x5eedull) | 1ull;
    uint32_t h = (uint32_t)(fp >> 40) & (tc - 1);
    for (;;) {
      const unsigned long long old = atomicCAS(&kfp[h], 0ull, fp);
      if (old == 0ull) {
#pragma unroll
        for (int k = 0; k < W; ++k) key[k * tc + h] = r.z.w[k];
        break;
      }
      if (old == fp) break;
      h = (h + 1) & (tc - 1);
    }
    atomicAdd(&cnt[h], 1u);
    slot[i] = (uint16_t)h;
    // group statistics as the strings arrive (|c| bit patterns order like
    // the values; NaN takes no part in max / min, like fmax / fmin)
    const unsigned long long ab = (unsigned long long)__double_as_longlong(r.c) & 0x7fffffffffffffffull;
    if (ab >= 0x7ff0000000000000ull) snf[h] = 1;
    if (ab <= 0x7ff0000000000000ull) {
      atomicMax(&smx[h], ab);
      atomicMin(&smn[h], ab);
    }
  }
  rec = warp_sum64(rec);
  if (lane == 0 && rec) atomicAdd(&s_rec, rec);
  __syncthreads();
  // group ids and offsets in slot order
  constexpr uint32_t kPerT = 4;  // tc <= kPerT * threads
  uint32_t used = 0, sum = 0;
#pragma unroll
  for (uint32_t e = 0; e < kPerT; ++e) {
    const uint32_t h = tid * kPerT + e;
    if (h < tc) {
      used += kfp[h] != 0ull;
      sum += cnt[h];
    }
  }
  uint32_t G, total;
  uint32_t gid = block_excl_scan(used, scr, &G);
  uint32_t o = block_excl_scan(sum, scr, &total);
#pragma unroll
  for (uint32_t e = 0; e < kPerT; ++e) {
    const uint32_t h = tid * kPerT + e;
    if (h < tc && kfp[h] != 0ull) {
      go.off[gid] = o;
      go.cnt[gid] = cnt[h];
      go.cap[gid] = cnt[h];
#pragma unroll
      for (int k = 0; k < W; ++k) go.z[k][gid] = key[k * tc + h];
      go.stamp[gid] = 0xffffffffu;
      go.gmax[gid] = __longlong_as_double((long long)smx[h]);
      go.gmin[gid] = __longlong_as_double((long long)smn[h]);
      go.flags[gid] = snf[h] | kFlagUnsorted;
      off[h] = o;
      cnt[h] = gid;  // slot -> group id from here on
      o += go.cnt[gid];
      ++gid;
    }
  }
  __syncthreads();
  for (uint32_t h = tid; h < tc; h += kSmallRegroupThreads) state[h] = 0;  // cursors (already zero; kept explicit)
  __syncthreads();
  // scatter (recomputing the producer's record; order inside a group is free)
  for (uint32_t i = tid; i < n; i += kSmallRegroupThreads) {
    const uint32_t gg = group_of(i);
    const uint64_t a = gi.off[gg] + (i - gpre[gg]);
    Plane<W> z;
#pragma unroll
    for (int k = 0; k < W; ++k) z.w[k] = gi.z[k][gg];
    Record<W> r;
    uint32_t nrec = 0;
    prod.emit(load_plane<W>(ai.x, a), z, ai.c[a], &r, &nrec);
    const uint32_t h = slot[i];
    bool same = true;
#pragma unroll
    for (int k = 0; k < W; ++k) same &= key[k * tc + h] == r.z.w[k];
    if (!same) atomicOr(&st->collision, 1u);
    const uint64_t d = off[h] + atomicAdd(&state[h], 1u);
    store_plane<W>(ao.x, d, r.x);
    ao.c[d] = r.c;
  }
  __syncthreads();
  prod.flush(s_mark, st);
  if (tid == 0) {
    st->distinct = G;
    st->scan_total = total;
    st->G_dev = G;
    st->bump = total;
    st->cliff_records += s_rec;
  }
}

// Group statistics of a regroup that skipped the sort (a Clifford run is a
// signed permutation: no equal keys to combine, no zeros): max / min |c| and
// the non-finite flag per group, marked unsorted.  Warp per group.
template <int W>
__global__ void __launch_bounds__(kCta) k_group_stats(GroupView<W> g, ArenaView<W> ar, const DevStats* st) {
  const uint32_t G = *(volatile const unsigned int*)&st->distinct;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t gid = warp; gid < G; gid += nw) {
    const uint64_t o = g.off[gid];
    const uint32_t n = g.cnt[gid];
    unsigned long long gx = 0ull, gn = 0x7ff0000000000000ull;
    uint32_t nf = 0;
    for (uint32_t j = lane; j < n; j += 32) {
      const unsigned long long ab = (unsigned long long)__double_as_longlong(ar.c[o + j]) & 0x7fffffffffffffffull;
      if (ab >= 0x7ff0000000000000ull) nf = 1;
      if (ab <= 0x7ff0000000000000ull) {
        gx = ab > gx ? ab : gx;
        gn = ab < gn ? ab : gn;
      }
    }
    gx = warp_max_bits(gx);
    gn = warp_min_bits(gn);
    nf = __any_sync(0xffffffffu, nf);
    if (lane == 0) {
      g.gmax[gid] = n ? __longlong_as_double((long long)gx) : 0.0;
      g.gmin[gid] = n ? __longlong_as_double((long long)gn) : __longlong_as_double(0x7ff0000000000000ll);
      g.flags[gid] = nf | kFlagUnsorted;
    }
  }
}

// End of a regroup whose sizes the host does not wait for: the new table's
// group count and bump pointer become the device's, and the run's records
// move aside for the next sync to account (records_sent and removed).
__global__ void k_regroup_commit(DevStats* st) {
  st->G_dev = st->distinct;
  st->bump = st->scan_total;
  st->cliff_records += st->records;
  st->records = 0;
}

__global__ void k_set_distinct(DevStats* st, unsigned int G) {
  st->distinct = G;
  st->scratch_bump = 0;
}

}  // namespace ppgpu
