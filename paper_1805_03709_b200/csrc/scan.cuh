// scan.cuh -- multi-CTA exclusive prefix sum (reduce-then-scan) used for
// ordered stream compaction: per-tile sums, one-CTA scan of the tile sums,
// then a per-tile scan that adds the tile offset.  Three short launches; the
// data is read twice (tile sums + scan), which is cheap next to the payloads
// it places.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vsb {

void count_launch();  // defined in hash.cu

constexpr int kScanTile = 4096;  // elements per CTA (256 threads x 16)

inline uint64_t scan_tiles(uint64_t n) { return (n + kScanTile - 1) / kScanTile; }

template <typename T>
__global__ void __launch_bounds__(256) k_tile_sums(const T* __restrict__ in, uint64_t n, uint64_t* __restrict__ sums) {
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile;
  uint64_t s = 0;
  for (int j = threadIdx.x; j < kScanTile; j += 256) {
    const uint64_t i = base + j;
    if (i < n) s += (uint64_t)in[i];
  }
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

// out[i] = exclusive prefix of in[0..i); out[n] = total
template <typename T>
__global__ void __launch_bounds__(256) k_tile_scan(const T* __restrict__ in, uint64_t n,
                                                   const uint64_t* __restrict__ tile_off, uint64_t ntiles,
                                                   uint64_t* __restrict__ out) {
  const uint64_t base = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * 16;
  uint32_t v[16];
  uint64_t local = 0;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint64_t i = base + k;
    v[k] = i < n ? (uint32_t)in[i] : 0u;
    local += v[k];
  }
  __shared__ uint64_t ws[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = local;
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  uint64_t pre = tile_off[blockIdx.x];
  for (int w = 0; w < warp; ++w) pre += ws[w];
  uint64_t run = pre + x - local;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const uint64_t i = base + k;
    if (i < n) out[i] = run;
    run += v[k];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[n] = tile_off[ntiles];
}

// Exclusive scan of in[0..n) into out[0..n]; work holds >= scan_tiles(n)+1 u64.
template <typename T>
inline cudaError_t exclusive_scan(const T* in, uint64_t n, uint64_t* out, uint64_t* work, cudaStream_t s) {
  if (n == 0) return cudaMemsetAsync(out, 0, sizeof(uint64_t), s);
  const uint64_t nt = scan_tiles(n);
  { k_tile_sums<T><<<(unsigned)nt, 256, 0, s>>>(in, n, work); vsb::count_launch(); }
  { k_scan_tiles<<<1, 1024, 0, s>>>(work, nt); vsb::count_launch(); }
  { k_tile_scan<T><<<(unsigned)nt, 256, 0, s>>>(in, n, work, nt, out); vsb::count_launch(); }
  return cudaGetLastError();
}

}  // namespace vsb
