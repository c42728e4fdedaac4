// pp_dense.cuh -- the dense Rx sublayer as its own persistent kernel.
//
// k_dense_sublayer applies a whole run of X-type gates on distinct qubits
// (epsilon0 = 0 or external truncation; SubGates::dense) to every z-group the
// dense path can take (dense_apply, pp_kernels.cuh) and leaves the rest -- a
// group resumed in the middle of a run, more than kDenseMaxK x classes, a
// block beyond kDenseMaxLog stages -- on a list for k_branch_sublayer's
// per-gate path, launched right behind it on the same stream.
//
// Against running the dense path inside k_branch_sublayer:
//  * work arrives in chunks: warp 0 claims 8 (large groups) or 32 (small
//    groups) consecutive table entries with one atomic, each lane tests one
//    entry (touched by the run? this sweep's size class?) and loads that
//    group's descriptor; the CTA then works through the chunk's queue from
//    shared memory -- one device round trip per chunk instead of four
//    dependent ones per table entry, and no barrier-bracketed iteration for
//    an entry that is skipped;
//  * the stage list comes from z alone (every gate of the run sits on its
//    own qubit, so T = z & any): no shared-memory atomics, no one-thread
//    section, two barriers.
// Reference semantics are dense_apply's (engine.cpp:207-264 per gate).
#pragma once

#include "pp_kernels.cuh"

namespace ppgpu {

constexpr uint32_t kDenseChunkBig = 8;     // table entries per claim, large-group sweep
constexpr uint32_t kDenseChunkSmall = 32;  // ... small-group sweep

template <int W>
struct DenseItem {
  Plane<W> z;
  unsigned long long off;
  double gmin;
  uint32_t gid, n, stamp, pad;
};

template <int W>
constexpr size_t dense_smem_bytes() {
  return kDenseSmem * sizeof(double) + sizeof(DenseTail<W>);
}

template <int W>
__global__ void __launch_bounds__(kCta, PP_DENSE_CTAS) k_dense_sublayer(GroupView<W> g, ArenaView<W> ar, const SubGates gates,
                                                          unsigned int* work, DevStats* st, uint32_t* left) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_touch[kMaxSubGates / 32];
  __shared__ uint32_t s_seen[kMaxSubGates / 32];
  __shared__ GroupStatsSmem gs;
  __shared__ uint32_t tscan[40];
  __shared__ DenseCtl<W> dc;
  __shared__ SubGates s_gp;
  __shared__ DenseItem<W> queue[kDenseChunkSmall];
  __shared__ uint32_t q_n, q_done;
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  if (engine_failed(st)) return;
  const uint32_t G = *(volatile const unsigned int*)&st->G_dev;
  const unsigned long long cap = *(volatile const unsigned long long*)&st->arena_cap;
  const uint32_t seq0 = (uint32_t)(*(volatile const unsigned long long*)&st->seq_base);
  if (tid < kMaxSubGates / 32) s_seen[tid] = 0;
  for (int k = tid; k < gates.ng; k += kCta) {
    s_gp.wq[k] = gates.wq[k];
    s_gp.mq[k] = gates.mq[k];
    s_gp.cosv[k] = gates.cosv[k];
    s_gp.sinv[k] = gates.sinv[k];
  }
  if (tid == 0) {
    s_gp.ng = gates.ng;
    s_gp.maxk = gates.maxk;
    s_gp.fast = gates.fast;
    dc.tpred = nullptr;
    dc.smax = nullptr;
    dc.ng = gates.ng;
    mbar_init(&dc.mbar, 1);
    dc.mphase = 0;
    dc.bulk_tiles = 0;
  }
  __syncthreads();
  const int ng = gates.ng;
  // chunk sizes: up to 8 / 32 entries per claim, fewer when the table is too
  // small to keep every CTA busy that way
  const uint32_t per_big = max(1u, min(kDenseChunkBig, G / (16u * gridDim.x)));
  const uint32_t per_small = max(1u, min(kDenseChunkSmall, G / (4u * gridDim.x)));
  const uint32_t nbig = (G + per_big - 1) / per_big;
  const uint32_t nsmall = (G + per_small - 1) / per_small;
  unsigned long long aff_elems = 0;
  bool failed = false;
  for (;;) {
    // ----- claim a chunk of table entries; queue the groups to apply
    __syncthreads();
    if (tid < 32) {
      uint32_t chunk = 0;
      if (lane == 0) chunk = atomicAdd(work, 1u);
      chunk = __shfl_sync(0xffffffffu, chunk, 0);
      const bool done = chunk >= nbig + nsmall;
      const bool bigsweep = chunk < nbig;
      const uint32_t per = bigsweep ? per_big : per_small;
      const uint32_t cand = (bigsweep ? chunk : chunk - nbig) * per + lane;
      bool take = false;
      DenseItem<W> it;
      if (!done && lane < per && cand < G) {
        it.gid = cand;
        it.n = g.cnt[cand];
        uint32_t mt = 0;
#pragma unroll
        for (int k = 0; k < W; ++k) {
          it.z.w[k] = g.z[k][cand];
          mt += __popcll(it.z.w[k] & gates.any[k]);
        }
        // large groups (a block of at least one shared-memory tile) first, so
        // the longest groups start early; the sweep follows from z alone
        take = it.n != 0 && mt != 0 && (mt >= kDenseSmemLog) == bigsweep;
        if (take) {
          it.off = g.off[cand];
          it.gmin = g.gmin[cand];
          it.stamp = g.stamp[cand];
          it.pad = 0;
        }
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, take);
      if (take) queue[__popc(bal & ((1u << lane) - 1u))] = it;
      if (lane == 0) {
        q_n = __popc(bal);
        q_done = done;
      }
    }
    __syncthreads();
    if (q_done) break;
    const uint32_t qn = q_n;
    for (uint32_t qi = 0; qi < qn && !failed; ++qi) {
      const uint32_t gid = queue[qi].gid, n = queue[qi].n;
      const uint64_t src = queue[qi].off;
      const Plane<W> z = queue[qi].z;
      const uint32_t stamp = queue[qi].stamp;
      const int k0 = (stamp - seq0 < (uint32_t)ng) ? (int)(stamp - seq0) + 1 : 0;  // resume after the stamp
      // the gates that touch this group (one ballot per warp), its touched
      // bits T = z & any and its stage list
      const int k = (int)tid;
      bool touch = false;
      int wq = 0;
      uint64_t mq = 0;
      if (k < ng) {
        wq = s_gp.wq[k];
        mq = s_gp.mq[k];
        touch = (z.w[wq] & mq) != 0;
      }
      const uint32_t tb = __ballot_sync(0xffffffffu, touch);
      __syncthreads();  // the previous group's readers of s_touch and dc are done
      if (lane == 0 && tid < kMaxSubGates) s_touch[tid >> 5] = tb;
      __syncthreads();
      uint32_t tw[kMaxSubGates / 32];
      int m = 0, klast = -1;
      bool later = false;  // a touching gate at or after k0
#pragma unroll
      for (int w = 0; w < kMaxSubGates / 32; ++w) {
        tw[w] = s_touch[w];
        m += __popc(tw[w]);
        if (tw[w]) klast = 32 * w + 31 - __clz(tw[w]);
      }
      later = klast >= k0;
      if (!later) continue;  // every touching gate is applied already (a relaunch after an arena fault)
      if (k0 > 0 || m > kDenseMaxLog) {
        // resumed in the middle of the run, or too many stages: the per-gate path
        if (tid == 0) left[atomicAdd(&st->left_n, 1u)] = gid;
        continue;
      }
      Plane<W> T;
#pragma unroll
      for (int w = 0; w < W; ++w) T.w[w] = z.w[w] & gates.any[w];
      if (touch) {
        uint32_t r = __popcll(T.w[wq] & (mq - 1));
        for (int w = 0; w < wq; ++w) r += __popcll(T.w[w]);
        uint32_t j = __popc(tw[k >> 5] & ((1u << (k & 31)) - 1u));
        for (int w = 0; w < (k >> 5); ++w) j += __popc(tw[w]);
        dc.sbit[j] = (uint8_t)r;
        dc.sgate[j] = (uint8_t)k;
        dc.scos[j] = s_gp.cosv[k];
        dc.ssin[j] = s_gp.sinv[k];
        if (r < 32) dc.tpos[r] = (uint8_t)(64 * wq + __ffsll((long long)mq) - 1);
      }
      if (tid == 0) {
        dc.T = T;
        dc.m = m;
        dc.klast = klast;
        dc.fast = (s_gp.fast && queue[qi].gmin >= kFastLive) ? 1u : 0u;
        Plane<W> F = load_plane<W>(ar.x, src);
#pragma unroll
        for (int w = 0; w < W; ++w) F.w[w] &= ~T.w[w];
        dc.F = F;
      }
      if (tid < kMaxSubGates / 32) dc.tw[tid] = tw[tid];
      __syncthreads();
      const int r = dense_apply<W>(reinterpret_cast<double*>(smem_raw), dc, gs, tscan, g, ar, s_gp, gid, n, src, s_touch,
                                   seq0, cap, st, aff_elems, s_seen);
      if (r < 0) failed = true;  // the arena is full: the host compacts and relaunches
      if (r == 0 && tid == 0) left[atomicAdd(&st->left_n, 1u)] = gid;
    }
    if (failed) break;
  }
  __syncthreads();
  // a touched group with a nonzero string sends a record through every gate
  // with sin != 0 that touches it (its vector stays nonzero through the
  // run's rotations)
  for (int k = tid; k < ng; k += kCta)
    if (((s_seen[k >> 5] >> (k & 31)) & 1u) && s_gp.sinv[k] != 0.0) mark_seen(st, st->seen_base + k);
  if (tid == 0 && aff_elems) atomicAdd(&st->aff_total, aff_elems);
  if (tid == 0 && dc.bulk_tiles) atomicAdd(&st->bulk_tiles, (unsigned long long)dc.bulk_tiles);
}

}  // namespace ppgpu
