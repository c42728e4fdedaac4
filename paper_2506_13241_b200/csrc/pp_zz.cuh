// pp_zz.cuh -- Z-type generators (x_J = 0: the branching Rzz of BASELINE
// config 4, Rz): branch + merge on PAIRS of z-groups.
//
// For J = (0, m) a string I = (x, z) anticommutes iff x.m is odd, and its
// child I xor J = (x, z ^ m) has the SAME x in the partner group z ^ m
// (engine.cpp:207-264 restated on the z-grouped store).  So the gate maps
// the pair {z, z ^ m} onto itself: each side's new list is the merge, by x,
// of its own strings (anticommuting ones scaled by cos) and the other
// side's anticommuting strings as children (+-sin c, sign from the phase
// B(I, J) mod 4, engine.cpp:67-81); a string present on both sides gets
// c cos + child, exactly the reference's v *= cos then v += delta.  Strings
// never leave the pair, so the gate is one pass over the store with no
// hash-and-sort regroup.  Pairs are processed in packs of small pairs per
// CTA (like the X-type packs), a missing partner group is created.
#pragma once

#include "pp_kernels.cuh"

namespace ppgpu {

// z -> group id of the current store, built per gate
template <int W>
struct ZTable {
  unsigned long long* fp;  // 0 = empty slot
  uint64_t* z[W];
  uint32_t* gid;
  unsigned long long mask;
};

template <int W>
__device__ __forceinline__ unsigned long long ztab_fp(const Plane<W>& z) {
  const unsigned long long f = plane_hash<W>(z, 0x9e3779b97f4a7c15ull);
  return f ? f : 1ull;
}

template <int W>
__global__ void k_ztab_build(GroupView<W> g, uint32_t G, ZTable<W> t) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= G) return;
  const Plane<W> z = load_plane<W>(g.z, i);
  const unsigned long long fp = ztab_fp<W>(z);
  unsigned long long slot = fp & t.mask;
  for (;;) {  // group z-planes are unique: plain linear probing
    if (atomicCAS(&t.fp[slot], 0ull, fp) == 0ull) {
#pragma unroll
      for (int k = 0; k < W; ++k) t.z[k][slot] = z.w[k];
      t.gid[slot] = i;
      return;
    }
    slot = (slot + 1) & t.mask;
  }
}

template <int W>
__device__ __forceinline__ uint32_t ztab_find(const ZTable<W>& t, const Plane<W>& z) {
  const unsigned long long fp = ztab_fp<W>(z);
  unsigned long long slot = fp & t.mask;
  for (;;) {
    const unsigned long long f = t.fp[slot];
    if (f == 0ull) return kNone;
    if (f == fp) {
      bool eq = true;
#pragma unroll
      for (int k = 0; k < W; ++k) eq &= t.z[k][slot] == z.w[k];
      if (eq) return t.gid[slot];
    }
    slot = (slot + 1) & t.mask;
  }
}

constexpr uint32_t kZSeg = 1024;  // strings per pack (both sides of all its pairs)
constexpr uint32_t kZPack = 32;   // pairs per pack
constexpr uint32_t kZLists = 2 * kZPack;

template <int W>
struct ZzSmem {
  uint64_t key[W * kZSeg];  // x planes, SoA (stride kZSeg)
  double val[kZSeg];
  uint32_t cpre[kZSeg + 4];  // exclusive prefix of "child slot" flags (anticommuting, unmatched)
  uint32_t lbv[kZSeg];       // lower bound of the string's x in the other side's list
  alignas(16) uint8_t fl[kZSeg];  // bit0 anticommutes, bit1 matched (same x on the other side)
  uint64_t okey[W * 2 * kZSeg];
  double oval[2 * kZSeg];
  alignas(16) uint8_t oemit[2 * kZSeg];
  uint16_t cpos[2 * kZSeg];
  uint32_t scan[40];
  // the pack: list j = 2 k + s is side s of pair k (side 0: the owner group)
  uint32_t np;
  uint32_t lstart[kZLists + 1];
  uint64_t lsrc[kZLists];
  double ltin[kZLists];
  uint32_t lgid[kZLists];
  uint64_t lz[W][kZLists];
  uint32_t obase[kZLists + 1];
  uint32_t ostart[kZLists + 1];
  uint32_t ocnt[kZLists], onf[kZLists];
  double omx[kZLists], omn[kZLists];
};

template <int W>
__device__ __forceinline__ uint32_t zz_list_of(const ZzSmem<W>& sm, uint32_t i) {
  uint32_t lo = 0, hi = 2 * sm.np;  // largest j with lstart[j] <= i
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (sm.lstart[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

// sign of the child of (x, z) under J = (0, jz): + if B == 1, - if B == 3
template <int W>
__device__ __forceinline__ double zz_child(const Plane<W>& x, const Plane<W>& z, const Plane<W>& jz, double sinv,
                                           double c) {
  Plane<W> zero;
#pragma unroll
  for (int k = 0; k < W; ++k) zero.w[k] = 0;
  const int b = phase_mod4<W>(x, z, zero, jz);
  return __dmul_rn(b == 1 ? sinv : -sinv, c);
}

// One pack.  Returns false when the pack holds no anticommuting string (then
// nothing is written and the caller keeps the groups as they are).
template <int W>
__device__ bool zz_segment(ZzSmem<W>& sm, ArenaView<W> ar, const Plane<W>& jz, double cosv, double sinv,
                           int keep_zeros, bool lazy, uint64_t dst, unsigned long long& records,
                           unsigned long long& removed) {
  const uint32_t tid = threadIdx.x;
  const uint32_t L = sm.lstart[2 * sm.np];
  // P1: load, deferred truncation (pending strings held as -0.0), parity
  uint32_t anti_any = 0;
  for (uint32_t i = tid; i < L; i += kCta) {
    const uint32_t j = zz_list_of<W>(sm, i);
    const uint64_t a = sm.lsrc[j] + (i - sm.lstart[j]);
    const Plane<W> x = load_plane<W>(ar.x, a);
    sk_store<W>(sm.key, kZSeg, i, x);
    double v = ar.c[a];
    const double t = sm.ltin[j];
    if (t >= 0.0 && fabs(v) <= t) v = -0.0;
    sm.val[i] = v;
    const uint8_t an = (uint8_t)plane_parity_and<W>(x, jz);
    sm.fl[i] = an;
    anti_any |= an;
  }
  if (!__syncthreads_or(anti_any)) return false;
  // P2: the same x on the other side (a match is anticommuting on both sides)
  for (uint32_t i = tid; i < L; i += kCta) {
    const uint32_t j = zz_list_of<W>(sm, i), o = j ^ 1u;
    const Plane<W> x = sk_load<W>(sm.key, kZSeg, i);
    uint32_t lo = sm.lstart[o], hi = sm.lstart[o + 1];
    const uint32_t eo = hi;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (plane_lt<W>(sk_load<W>(sm.key, kZSeg, mid), x)) lo = mid + 1;
      else hi = mid;
    }
    sm.lbv[i] = lo;
    if ((sm.fl[i] & 1u) && lo < eo && plane_eq<W>(sk_load<W>(sm.key, kZSeg, lo), x)) sm.fl[i] |= 2u;
  }
  __syncthreads();
  // P3: prefix of child slots (anticommuting and unmatched), blocked
  {
    constexpr uint32_t kV = kZSeg / kCta;
    const uint32_t fw = reinterpret_cast<const uint32_t*>(sm.fl)[tid];
    uint32_t cnt = 0;
#pragma unroll
    for (uint32_t v = 0; v < kV; ++v) {
      const uint32_t b = (fw >> (8 * v)) & 0xffu;
      cnt += (tid * kV + v < L) && (b & 1u) && !(b & 2u);
    }
    uint32_t tot;
    uint32_t e = block_excl_scan(cnt, sm.scan, &tot);
#pragma unroll
    for (uint32_t v = 0; v < kV; ++v) {
      const uint32_t i = tid * kV + v;
      sm.cpre[i] = e;
      const uint32_t b = (fw >> (8 * v)) & 0xffu;
      e += (i < L) && (b & 1u) && !(b & 2u);
    }
    if (tid == 0) sm.cpre[kZSeg] = tot;
  }
  __syncthreads();
  // P4: output list sizes = own strings + the other side's child slots
  if (tid == 0) {
    uint32_t b = 0;
    for (uint32_t j = 0; j < 2 * sm.np; ++j) {
      sm.obase[j] = b;
      const uint32_t o = j ^ 1u;
      b += (sm.lstart[j + 1] - sm.lstart[j]) + (sm.cpre[sm.lstart[o + 1]] - sm.cpre[sm.lstart[o]]);
    }
    sm.obase[2 * sm.np] = b;
  }
  __syncthreads();
  // P5: values into slots
  bool hole = false;
  for (uint32_t i = tid; i < L; i += kCta) {
    const uint32_t j = zz_list_of<W>(sm, i), o = j ^ 1u;
    const uint32_t sj = sm.lstart[j], so = sm.lstart[o];
    const uint32_t lb = sm.lbv[i];
    const uint8_t f = sm.fl[i];
    const Plane<W> x = sk_load<W>(sm.key, kZSeg, i);
    const double c = sm.val[i];
    const bool pend = lazy && is_pending(c);
    if (pend) ++removed;  // its deferred removal, counted once
    const uint32_t sp = sm.obase[j] + (i - sj) + (sm.cpre[lb] - sm.cpre[so]);
    double v;
    bool e;
    if (!(f & 1u)) {  // commutes: unchanged
      v = c;
      e = keep_zeros || v != 0.0;
    } else {
      Plane<W> zj, zo;
#pragma unroll
      for (int k = 0; k < W; ++k) {
        zj.w[k] = sm.lz[k][j];
        zo.w[k] = sm.lz[k][o];
      }
      v = __dmul_rn(c, cosv);
      if (f & 2u) {  // the other side's string at the same x sends its child here
        const double d_o = zz_child<W>(x, zo, jz, sinv, sm.val[lb]);
        if (d_o != 0.0) v = __dadd_rn(v, d_o);
      }
      e = keep_zeros || v != 0.0;
      const double d = zz_child<W>(x, zj, jz, sinv, c);
      if (d != 0.0) ++records;
      if (!(f & 2u)) {  // own child slot on the other side
        const uint32_t sc = sm.obase[o] + (lb - so) + (sm.cpre[i] - sm.cpre[sj]);
        sk_store<W>(sm.okey, 2 * kZSeg, sc, x);
        sm.oval[sc] = d;
        sm.oemit[sc] = d != 0.0;
        hole |= d == 0.0;
      }
    }
    if (!e && !pend) ++removed;
    sk_store<W>(sm.okey, 2 * kZSeg, sp, x);
    sm.oval[sp] = v;
    sm.oemit[sp] = e;
    hole |= !e;
  }
  // P6: compaction of empty slots (exact zeros), as in seg_branch
  const uint32_t s2 = sm.obase[2 * sm.np];
  constexpr uint32_t kSV = 2 * kZSeg / kCta;
  uint32_t ecnt = s2;
  if (__syncthreads_count(hole)) {
    const uint2 eb = reinterpret_cast<const uint2*>(sm.oemit)[tid];
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
  // P7: store, contiguous per list
  for (uint32_t i = tid; i < ecnt; i += kCta) {
    const uint32_t sl = dense ? i : sm.cpos[i];
    store_plane<W>(ar.x, dst + i, sk_load<W>(sm.okey, 2 * kZSeg, sl));
    ar.c[dst + i] = sm.oval[sl];
  }
  // P8: per-list output range and statistics
  const uint32_t nl = 2 * sm.np;
  if (tid <= nl) {
    const uint32_t sb = sm.obase[tid];
    uint32_t lo = 0, hi = ecnt;
    if (dense) {
      lo = sb;
    } else {
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (sm.cpos[mid] < sb) lo = mid + 1;
        else hi = mid;
      }
    }
    sm.ostart[tid] = lo;
  }
  __syncthreads();
  const uint32_t lane = tid & 31;
  for (uint32_t j = tid >> 5; j < nl; j += kWarps) {
    const uint32_t o0 = sm.ostart[j], o1 = sm.ostart[j + 1];
    unsigned long long gx = 0ull, gn = 0x7ff0000000000000ull;
    uint32_t nf = 0;
    for (uint32_t q = o0 + lane; q < o1; q += 32) {
      const unsigned long long ab =
          (unsigned long long)__double_as_longlong(sm.oval[dense ? q : sm.cpos[q]]) & 0x7fffffffffffffffull;
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
      sm.ocnt[j] = o1 - o0;
      sm.omx[j] = __longlong_as_double((long long)gx);
      sm.omn[j] = __longlong_as_double((long long)gn);
      sm.onf[j] = nf;
    }
  }
  __syncthreads();
  return true;
}

// One Z-type gate over the whole store.  Persistent CTAs take chunks of
// consecutive groups; a group owns its pair when its partner is missing or
// has a larger id.  Every pair is rewritten into fresh arena space (or left
// as it is when neither side anticommutes).  red_out: fused epilogue
// reduction (deferred truncation), taken by the writer of each pair.
template <int W>
__global__ void __launch_bounds__(kCta) k_branch_zz(GroupView<W> g, uint32_t G, ArenaView<W> ar, Plane<W> jz,
                                                     double cosv, double sinv, int keep_zeros, ZTable<W> t,
                                                     unsigned int* work, unsigned int* work_next, uint32_t seq_rel,
                                                     DevStats* st, const double* __restrict__ thr, RedSlot* red_out) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ZzSmem<W>& sm = *reinterpret_cast<ZzSmem<W>*>(smem_raw);
  const uint32_t tid = threadIdx.x;
  if (blockIdx.x == 0 && tid == 0) *work_next = 0;
  if (engine_failed(st)) return;
  const unsigned long long cap = *(volatile const unsigned long long*)&st->arena_cap;
  const uint32_t seq_base = (uint32_t)*(volatile const unsigned long long*)&st->seq_base;
  const uint32_t seq = seq_base + seq_rel;
  const uint32_t chunk = max(1u, min(kCta, (G + gridDim.x - 1) / gridDim.x));
  const bool lazy = thr != nullptr;
  const double thr0 = lazy ? thr[0] : 0.0;
  __shared__ uint32_t s_chunk;
  __shared__ uint32_t s_g[kCta], s_p[kCta], s_pp[kCta + 1], s_first[kCta + 1];
  __shared__ unsigned long long s_dst;
  unsigned long long records = 0, removed = 0, r_live = 0;
  double r_max = 0.0;
  uint32_t r_nf = 0, r_mc = 0;
  // a group's live contribution to the fused reduction, as it stands
  auto account = [&](uint32_t gi) {
    const uint32_t c = g.cnt[gi];
    if (!c) return;
    r_live += c;
    r_mc = max(r_mc, c);
    const double gm = g.gmax[gi];
    if (!lazy || gm > thr0 || gm > thr[pending_index(g.stamp[gi], seq_base, seq_rel)]) r_max = fmax(r_max, gm);
    r_nf |= g.flags[gi] & 1u;
  };
  for (;;) {
    __syncthreads();
    if (tid == 0) s_chunk = atomicAdd(work, 1u);
    __syncthreads();
    const uint32_t g0 = s_chunk * chunk;
    if (g0 >= G) break;
    // ---- owned pairs of the chunk
    const uint32_t gi = g0 + tid;
    uint32_t p = kNone, sz = 0;
    bool own = false;
    if (tid < chunk && gi < G) {
      Plane<W> z = load_plane<W>(g.z, gi);
      p = ztab_find<W>(t, plane_xor<W>(z, jz));
      own = p == kNone || gi < p;
      if (own) {
        sz = g.cnt[gi] + (p != kNone ? g.cnt[p] : 0u);
        if (g.stamp[gi] == seq) {  // done before an arena resume: account, do not redo
          if (red_out) {
            account(gi);
            if (p != kNone) account(p);
          }
          own = false;
        } else if (sz == 0) {
          own = false;
        } else if (sz > kZSeg) {
          atomicOr(&st->zz_err, 1u);  // the host's size check guarantees this cannot happen
          own = false;
        }
      }
    }
    uint32_t nown, tsz;
    const uint32_t r = block_excl_scan(own ? 1u : 0u, sm.scan, &nown);
    const uint32_t P = block_excl_scan(own ? sz : 0u, sm.scan, &tsz);
    if (own) {
      s_g[r] = gi;
      s_p[r] = p;
      s_pp[r] = P;
    }
    if (tid == 0) {
      s_pp[nown] = tsz;
      s_dst = tsz ? atomicAdd(&st->bump, 2ull * tsz) : 0ull;
      if (tsz && s_dst + 2ull * tsz > cap) {
        atomicOr(&st->err_arena, 1u);
        atomicMin(&st->err_seq, (unsigned long long)seq);
      }
    }
    __syncthreads();
    const uint64_t chunk_dst = s_dst;
    if (tsz && chunk_dst + 2ull * tsz > cap) continue;  // untouched; the host compacts and resumes
    // packs: pairs of at most kZSeg/2 strings share a pack while their start
    // prefix stays in one half segment; larger pairs go alone
    constexpr uint32_t kHalf = kZSeg / 2;
    const bool big = tid < nown && (s_pp[tid + 1] - s_pp[tid]) > kHalf;
    const bool prev_big = tid > 0 && tid < nown && (s_pp[tid] - s_pp[tid - 1]) > kHalf;
    const bool start = tid < nown && (tid % kZPack == 0 || big || prev_big || s_pp[tid] / kHalf != s_pp[tid - 1] / kHalf);
    uint32_t npk;
    const uint32_t q = block_excl_scan(start ? 1u : 0u, sm.scan, &npk);
    if (start) s_first[q] = tid;
    if (tid == 0) s_first[npk] = nown;
    __syncthreads();
    for (uint32_t pj = 0; pj < npk; ++pj) {
      const uint32_t a = s_first[pj], b = s_first[pj + 1];
      const uint32_t np = b - a;
      const uint32_t base = s_pp[a];
      __syncthreads();
      if (tid < 2 * np) {  // list tid = side (tid & 1) of pair tid >> 1
        const uint32_t k = tid >> 1, s = tid & 1u;
        const uint32_t own_g = s_g[a + k], pg = s_p[a + k];
        const uint32_t gid = s ? pg : own_g;
        const Plane<W> z0 = load_plane<W>(g.z, own_g);
        const Plane<W> zs = s ? plane_xor<W>(z0, jz) : z0;
#pragma unroll
        for (int w = 0; w < W; ++w) sm.lz[w][tid] = zs.w[w];
        sm.lgid[tid] = gid;
        const uint32_t n0 = g.cnt[own_g];
        const uint32_t off = s_pp[a + k] - base;
        sm.lstart[tid] = s ? off + n0 : off;
        if (gid != kNone) {
          sm.lsrc[tid] = g.off[gid];
          sm.ltin[tid] = lazy ? thr[pending_index(g.stamp[gid], seq_base, seq_rel)] : -1.0;
        } else {
          sm.lsrc[tid] = 0;
          sm.ltin[tid] = lazy ? 0.0 : -1.0;
        }
      }
      if (tid == 0) {
        sm.np = np;
        sm.lstart[2 * np] = s_pp[b] - base;
      }
      __syncthreads();
      const uint64_t dst = chunk_dst + 2ull * base;
      if (!zz_segment<W>(sm, ar, jz, cosv, sinv, keep_zeros, lazy, dst, records, removed)) {
        // neither side of any pair anticommutes: the groups stay as they are
        if (red_out && tid < 2 * np && sm.lgid[tid] != kNone) account(sm.lgid[tid]);
        continue;
      }
      if (tid < 2 * np) {
        const uint32_t j = tid;
        const uint32_t c = sm.ocnt[j];
        uint32_t gid = sm.lgid[j];
        if (gid == kNone && c) {  // the partner group did not exist: create it
          gid = G + atomicAdd(&st->zz_newg, 1u);
          atomicAdd(&st->G_dev, 1u);  // the epilogue kernels that follow see it
#pragma unroll
          for (int w = 0; w < W; ++w) g.z[w][gid] = sm.lz[w][j];
        }
        if (gid != kNone) {
          g.off[gid] = dst + sm.ostart[j];
          g.cnt[gid] = c;
          g.cap[gid] = c;
          g.gmax[gid] = c ? sm.omx[j] : 0.0;
          g.gmin[gid] = c ? sm.omn[j] : __longlong_as_double(0x7ff0000000000000ll);
          g.flags[gid] = sm.onf[j];
          g.stamp[gid] = seq;
          if (c) {
            r_live += c;
            r_mc = max(r_mc, c);
            r_max = fmax(r_max, sm.omx[j]);
            r_nf |= sm.onf[j];
          }
        }
      }
    }
  }
  // counters and the fused reduction
  const uint32_t rec32 = __reduce_add_sync(0xffffffffu, (uint32_t)records);
  const uint32_t rem32 = __reduce_add_sync(0xffffffffu, (uint32_t)removed);
  const uint32_t mc = __reduce_max_sync(0xffffffffu, r_mc);
  if ((tid & 31) == 0) {
    if (rec32) {
      atomicAdd(&st->records, (unsigned long long)rec32);
      mark_seen(st, st->seen_base + seq_rel);  // batches_sent: this gate sent a record
    }
    if (rem32) atomicAdd(&st->removed, (unsigned long long)rem32);
    if (mc) atomicMax(&st->zz_maxcnt, mc);
  }
  if (red_out) {
    r_live = warp_sum64(r_live);
    const unsigned long long bm = warp_max_bits((unsigned long long)__double_as_longlong(r_max));
    r_nf = __any_sync(0xffffffffu, r_nf);
    if ((tid & 31) == 0) {
      if (r_live) atomicAdd(&red_out->live, r_live);
      atomic_max_nonneg(reinterpret_cast<double*>(&red_out->gmax_bits), __longlong_as_double((long long)bm));
      if (r_nf) atomicOr(&red_out->nonfinite, 1u);
    }
  }
}

}  // namespace ppgpu
