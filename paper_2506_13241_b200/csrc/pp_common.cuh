// pp_common.cuh -- shared device helpers for the B200 Pauli-propagation engine.
//
// Keys are Pauli strings in x/z bit-planes: the
// reference's interleaved code (lo, hi) per site maps to x = lo ^ hi, z = hi.
// A plane is W uint64 words (W = 1 for n <= 64, W = 2 for n <= 128); word
// W-1 is the most significant when planes are compared as integers.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ppgpu {

constexpr uint32_t kCta = 256;         // threads per CTA for streaming kernels
constexpr uint32_t kWarps = kCta / 32;

template <int W>
struct Plane {
  uint64_t w[W];
};

template <int W>
__host__ __device__ __forceinline__ bool plane_lt(const Plane<W>& a, const Plane<W>& b) {
#pragma unroll
  for (int k = W - 1; k >= 0; --k) {
    if (a.w[k] != b.w[k]) return a.w[k] < b.w[k];
  }
  return false;
}

template <int W>
__host__ __device__ __forceinline__ bool plane_eq(const Plane<W>& a, const Plane<W>& b) {
  bool eq = true;
#pragma unroll
  for (int k = 0; k < W; ++k) eq &= (a.w[k] == b.w[k]);
  return eq;
}

template <int W>
__host__ __device__ __forceinline__ bool plane_zero(const Plane<W>& a) {
  uint64_t acc = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) acc |= a.w[k];
  return acc == 0;
}

template <int W>
__host__ __device__ __forceinline__ Plane<W> plane_xor(const Plane<W>& a, const Plane<W>& b) {
  Plane<W> r;
#pragma unroll
  for (int k = 0; k < W; ++k) r.w[k] = a.w[k] ^ b.w[k];
  return r;
}

template <int W>
__host__ __device__ __forceinline__ Plane<W> plane_max() {
  Plane<W> r;
#pragma unroll
  for (int k = 0; k < W; ++k) r.w[k] = ~uint64_t{0};
  return r;
}

template <int W>
__device__ __forceinline__ int plane_parity_and(const Plane<W>& a, const Plane<W>& b) {
  int p = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) p += __popcll(a.w[k] & b.w[k]);
  return p & 1;
}

template <int W>
__device__ __forceinline__ int plane_popc_and(const Plane<W>& a, const Plane<W>& b) {
  int p = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) p += __popcll(a.w[k] & b.w[k]);
  return p;
}

// splitmix64 finalizer; bijective on uint64.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

template <int W>
__host__ __device__ __forceinline__ uint64_t plane_hash(const Plane<W>& a, uint64_t seed) {
  uint64_t h = seed;
#pragma unroll
  for (int k = 0; k < W; ++k) h = mix64(h ^ a.w[k]);
  return h;
}

// Symplectic phase: exponent B(I, J) mod 4 of
// i in sigma_I sigma_J = i^B sigma_{I xor J}, the 4-popcount restatement of
// the reference's per-site table sum (pauli_string.cpp:25-34, 79-85):
//   B = popc(xI&zI) + popc(xJ&zJ) + 2 popc(zI&xJ) - popc((xI^xJ)&(zI^zJ)).
template <int W>
__device__ __forceinline__ int phase_mod4(const Plane<W>& xi, const Plane<W>& zi,
                                          const Plane<W>& xj, const Plane<W>& zj) {
  int b = 0;
#pragma unroll
  for (int k = 0; k < W; ++k) {
    b += __popcll(xi.w[k] & zi.w[k]) + __popcll(xj.w[k] & zj.w[k]) +
         2 * __popcll(zi.w[k] & xj.w[k]) -
         __popcll((xi.w[k] ^ xj.w[k]) & (zi.w[k] ^ zj.w[k]));
  }
  return b & 3;
}

// ---------------------------------------------------------------------------
// Block-wide scans (warp shuffles + one smem round).
// ---------------------------------------------------------------------------

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v) {
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t n = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= (uint32_t)o) v += n;
  }
  return v;
}

// Exclusive scan over the CTA; returns the exclusive prefix for this thread
// and writes the CTA total to *total.  `scratch` must hold kWarps+1 words.
// Contains __syncthreads(); call from every thread.
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* scratch, uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nw = blockDim.x >> 5;
  uint32_t inc = warp_incl_scan(v);
  __syncthreads();
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    uint32_t s = lane < nw ? scratch[lane] : 0;
    uint32_t si = warp_incl_scan(s);
    if (lane < nw) scratch[lane] = si - s;
    if (lane == nw - 1) scratch[32] = si;
  }
  __syncthreads();
  uint32_t out = scratch[warp] + inc - v;
  *total = scratch[32];
  return out;
}

// max / min over a warp of non-negative doubles (or +inf) as their bit
// patterns, which order like the values: two 32-bit REDUX steps each
__device__ __forceinline__ unsigned long long warp_max_bits(unsigned long long v) {
  const uint32_t hi = (uint32_t)(v >> 32);
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? (uint32_t)v : 0u);
  return ((unsigned long long)mh << 32) | ml;
}
__device__ __forceinline__ unsigned long long warp_min_bits(unsigned long long v) {
  const uint32_t hi = (uint32_t)(v >> 32);
  const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? (uint32_t)v : 0xffffffffu);
  return ((unsigned long long)mh << 32) | ml;
}

// the same for non-negative doubles (or +inf) held as doubles: |c| maxima and
// minima (fmax / fmin never leave a NaN in them)
__device__ __forceinline__ double warp_max_nn(double v) {
  return __longlong_as_double((long long)warp_max_bits((unsigned long long)__double_as_longlong(v)));
}
__device__ __forceinline__ double warp_min_nn(double v) {
  return __longlong_as_double((long long)warp_min_bits((unsigned long long)__double_as_longlong(v)));
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ uint64_t warp_sum64(uint64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// atomicMax on a non-negative double via its bit pattern (ordering of
// non-negative IEEE doubles matches their uint64 bit patterns).
__device__ __forceinline__ void atomic_max_nonneg(double* addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}
__device__ __forceinline__ void atomic_min_nonneg(double* addr, double v) {
  atomicMin(reinterpret_cast<unsigned long long*>(addr),
            static_cast<unsigned long long>(__double_as_longlong(v)));
}

}  // namespace ppgpu
