// scan.cuh -- multi-CTA exclusive prefix sum (reduce-then-scan) used for
// ordered stream compaction: per-tile sums, one-CTA scan of the tile sums,
// then a per-tile scan that adds the tile offset.  Three short launches; the
// data is read twice (tile sums + scan), which is cheap next to the payloads
// it places.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "pdl.cuh"

namespace vsb {

void count_launch();  // defined in hash.cu

constexpr int kScanTile = 4096;  // elements per CTA (256 threads x 16)

inline uint64_t scan_tiles(uint64_t n) { return (n + kScanTile - 1) / kScanTile; }

// v[0..16) = in[base .. base+16) (0 past n); one or four 16-B loads when the
// run is whole and aligned, element loads otherwise
template <typename T>
__device__ __forceinline__ void load16(const T* __restrict__ in, uint64_t base, uint64_t n, uint32_t v[16]) {
  const T* p = in + base;
  if (base + 16 <= n && ((uintptr_t)p & 15) == 0) {
    if constexpr (sizeof(T) == 1) {
      const uint4 q = __ldg((const uint4*)p);
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int k = 0; k < 16; ++k) v[k] = (w[k >> 2] >> (8 * (k & 3))) & 0xffu;
      return;
    } else if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint4 r = __ldg((const uint4*)p + q);
        v[4 * q] = r.x, v[4 * q + 1] = r.y, v[4 * q + 2] = r.z, v[4 * q + 3] = r.w;
      }
      return;
    }
  }
#pragma unroll
  for (int k = 0; k < 16; ++k) v[k] = base + k < n ? (uint32_t)p[k] : 0u;
}

template <typename T>
__global__ void __launch_bounds__(256) k_tile_sums(const T* __restrict__ in, uint64_t n, uint64_t* __restrict__ sums) {
  pdl_wait();
  uint32_t v[16];
  load16(in, (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * 16, n, v);
  uint64_t s = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) s += v[k];
  __shared__ uint64_t red[8];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t tot = 0;
    for (int w = 0; w < 8; ++w) tot += red[w];
    sums[blockIdx.x] = tot;
  }
}

// exclusive scan of the tile sums in place; sums[ntiles] = total
static __global__ void __launch_bounds__(1024) k_scan_tiles(uint64_t* __restrict__ sums, uint64_t ntiles) {
  pdl_wait();
  __shared__ uint64_t ws[32];
  __shared__ uint64_t carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint64_t base = 0; base < ntiles; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint64_t v = i < ntiles ? sums[i] : 0;
    uint64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = ws[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      ws[lane] = w;
    }
    __syncthreads();
    const uint64_t carry = carry_s;
    const uint64_t pre = warp ? ws[warp - 1] : 0;
    if (i < ntiles) sums[i] = carry + pre + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + ws[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) sums[ntiles] = carry_s;
}

// out[i] = exclusive prefix of in[0..i); out[n] = total (a tile's own sum
// must fit in u32: byte flags and per-block counts do).  Each thread scans
// 16 consecutive inputs; the tile-local results are staged in shared memory
// (row pitch 17 words: conflict-free) so the u64 stores leave coalesced.
template <typename T>
__global__ void __launch_bounds__(256) k_tile_scan(const T* __restrict__ in, uint64_t n,
                                                   const uint64_t* __restrict__ tile_off, uint64_t ntiles,
                                                   uint64_t* __restrict__ out) {
  pdl_wait();
  __shared__ uint32_t stage[256 * 17];
  __shared__ uint32_t ws[8];
  const uint64_t tile = (uint64_t)blockIdx.x * kScanTile;
  const uint64_t base = tile + (uint64_t)threadIdx.x * 16;
  uint32_t v[16];
  load16(in, base, n, v);
  uint32_t local = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) local += v[k];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = local;
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  uint32_t run = x - local;
  for (int w = 0; w < warp; ++w) run += ws[w];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    stage[threadIdx.x * 17 + k] = run;
    run += v[k];
  }
  __syncthreads();
  const uint64_t t0 = tile_off[blockIdx.x];
#pragma unroll 4
  for (int j = threadIdx.x; j < kScanTile; j += 256) {
    const uint64_t i = tile + j;
    if (i < n) out[i] = t0 + stage[(j >> 4) * 17 + (j & 15)];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = tile_off[ntiles];
}

// Small inputs (<= 16K elements: one round) in ONE launch: one CTA of
// 1024 threads walks the input in rounds of 16,384 (16 per thread) with a
// running carry.  Saves two launches where launch latency is the cost.
constexpr uint64_t kScanSmallMax = 1u << 14;

template <typename T>
__global__ void __launch_bounds__(1024) k_scan_small(const T* __restrict__ in, uint64_t n, uint64_t* __restrict__ out) {
  pdl_wait();
  __shared__ uint64_t ws[32];  // round totals may exceed u32 for count inputs
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t carry = 0;
  for (uint64_t round = 0; round < n; round += 1024 * 16) {
    const uint64_t base = round + (uint64_t)threadIdx.x * 16;
    uint32_t v[16];
    load16(in, base, n, v);
    uint32_t local = 0;
#pragma unroll
    for (int k = 0; k < 16; ++k) local += v[k];
    uint32_t x = local;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) ws[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = ws[lane];
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      ws[lane] = w;
    }
    __syncthreads();
    uint64_t run = carry + (warp ? ws[warp - 1] : 0u) + (x - local);
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (base + k < n) out[base + k] = run;
      run += v[k];
    }
    carry += ws[31];
    __syncthreads();  // ws is rewritten next round
  }
  if (threadIdx.x == 0) out[n] = carry;
}

// Exclusive scan of in[0..n) into out[0..n]; work holds >= scan_tiles(n)+1 u64.
template <typename T>
inline cudaError_t exclusive_scan(const T* in, uint64_t n, uint64_t* out, uint64_t* work, cudaStream_t s) {
  if (n == 0) return cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
  if (n <= kScanSmallMax) {
    { cudaError_t e = launch_pdl(k_scan_small<T>, 1, 1024, 0, s, in, n, out); vsb::count_launch(); if (e != cudaSuccess) return e; }
    return cudaGetLastError();
  }
  const uint64_t nt = scan_tiles(n);
  { cudaError_t e = launch_pdl(k_tile_sums<T>, (unsigned)nt, 256, 0, s, in, n, work); vsb::count_launch(); if (e != cudaSuccess) return e; }
  { cudaError_t e = launch_pdl(k_scan_tiles, 1, 1024, 0, s, work, nt); vsb::count_launch(); if (e != cudaSuccess) return e; }
  { cudaError_t e = launch_pdl(k_tile_scan<T>, (unsigned)nt, 256, 0, s, in, n, (const uint64_t*)work, nt, out); vsb::count_launch(); if (e != cudaSuccess) return e; }
  return cudaGetLastError();
}

}  // namespace vsb
