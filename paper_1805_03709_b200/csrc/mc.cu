// mc.cu -- Marching-Cubes-index block encoder (+ quantised TSDF, compaction).
//
// Reference: recompute_mc_block (mc_encoding.py:145-172) over the TSDF block
// layout of voxel_model.py:23-72.  For each MC block (an 8^3 block key) and
// each voxel v = (x, y, z) of it, the cube with origin v reads its 8 corners
// at v + (k&1, k>>1&1, k>>2&1); corners past the block's +x/+y/+z faces come
// from the 7 positive neighbour blocks (absent -> weight 0).  Bit k of the
// index = corner k inside (tsdf < 0); index = 0 unless all 8 corners are
// observed (weight > 0); 255 folds to 0; colour = centre voxel colour where
// index != 0 (mc_encoding.py:159-171).
//
// B200 design (one persistent CTA of 128 threads per resident slot):
//   * the 6,144-byte centre block (wire AoS layout, one contiguous row of the
//     TSDF pool) is staged into shared memory with a 1-D TMA bulk copy
//     (cp.async.bulk + mbarrier), double-buffered so the next block's copy
//     overlaps this block's compute;
//   * the 217-voxel +x/+y/+z halo is gathered with read-only loads (mostly L2
//     hits when blocks are processed in key order);
//   * inside/observed predicates are reduced to two 9x9x9 BIT grids in shared
//     memory (warp ballots for the centre, atomicOr for the halo): each cube
//     index is then 4 shifts/ands of 9-bit rows, no float work;
//   * predicates are integer tests on the IEEE bits, so the result is
//     independent of FTZ/DAZ:
//       inside   <=> 0x80000000 <  bits <= 0xFF800000   (tsdf < 0, NaN false)
//       observed <=> 0 < (int32)bits <= 0x7F800000       (weight > 0, NaN false)
//   * outputs are written with streaming stores (evict-first) so the L2 keeps
//     the TSDF rows that neighbouring blocks will read as halo.
#include <cstdint>

#include "hash_ops.cuh"
#include "scan.cuh"
#include "table.h"

namespace vsb {

constexpr int kMcThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}

__device__ __forceinline__ uint32_t inside_bit(uint32_t b) { return (b > 0x80000000u && b <= 0xFF800000u) ? 1u : 0u; }
__device__ __forceinline__ uint32_t observed_bit(uint32_t b) {
  return ((int32_t)b > 0 && b <= 0x7F800000u) ? 1u : 0u;
}

// Quantised TSDF byte (NEW; normative definition in oracle/mc_oracle.c and
// DESIGN.md A17): observed ? clamp(rint_half_even(tsdf * 127), -127, 127)
// : -128; NaN tsdf -> -128; +-inf saturate.
__device__ __forceinline__ int32_t quantise(uint32_t tb, uint32_t wb) {
  if (!observed_bit(wb)) return -128;
  const float t = __uint_as_float(tb);
  if (t != t) return -128;
  float s = __fmul_rn(t, 127.0f);
  s = fminf(fmaxf(s, -127.0f), 127.0f);
  return __float2int_rn(s);
}

// Halo item -> (neighbour c, source flat index, grid row, grid bit).
// grid rows are indexed gz*9 + gy, bit gx, with g in [0, 8].
__device__ __forceinline__ void halo_item(int i, int& c, int& flat, int& row, int& bit) {
  if (i < 64) {  // +x face: voxel (0, y, z) of neighbour (1,0,0) -> grid (8, y, z)
    const int y = i & 7, z = i >> 3;
    c = 1; flat = 8 * y + 64 * z; row = z * 9 + y; bit = 8;
  } else if (i < 128) {  // +y face: (x, 0, z) of (0,1,0) -> (x, 8, z)
    const int x = i & 7, z = (i - 64) >> 3;
    c = 2; flat = x + 64 * z; row = z * 9 + 8; bit = x;
  } else if (i < 192) {  // +z face: (x, y, 0) of (0,0,1) -> (x, y, 8)
    const int x = i & 7, y = (i - 128) >> 3;
    c = 4; flat = x + 8 * y; row = 8 * 9 + y; bit = x;
  } else if (i < 200) {  // +x+y edge: (0, 0, z) of (1,1,0) -> (8, 8, z)
    const int z = i - 192;
    c = 3; flat = 64 * z; row = z * 9 + 8; bit = 8;
  } else if (i < 208) {  // +x+z edge: (0, y, 0) of (1,0,1) -> (8, y, 8)
    const int y = i - 200;
    c = 5; flat = 8 * y; row = 8 * 9 + y; bit = 8;
  } else if (i < 216) {  // +y+z edge: (x, 0, 0) of (0,1,1) -> (x, 8, 8)
    const int x = i - 208;
    c = 6; flat = x; row = 8 * 9 + 8; bit = x;
  } else {  // corner: (0,0,0) of (1,1,1) -> (8, 8, 8)
    c = 7; flat = 0; row = 8 * 9 + 8; bit = 8;
  }
}

constexpr int kLook = kMcThreads / 8;  // blocks per batched neighbour lookup (16)

struct McSmem {
  alignas(128) uint8_t buf[2][VS_TSDF_BLOCK_BYTES];
  alignas(8) uint64_t mbar[2];
  uint32_t grid_in[2][81];
  uint32_t grid_ob[2][81];
  int32_t nb[2][kLook][8];  // neighbour rows of two lookup batches
  uint32_t cnt[2][4];
};

// Neighbour row of block `blk` for corner-block c.
template <bool kFromKeys>
__device__ __forceinline__ int32_t load_nbr(const TableView& T, const int32_t* __restrict__ keys,
                                            const int32_t* __restrict__ nbr, uint64_t blk, int c) {
  if (kFromKeys) {
    const int32_t x = keys[3 * blk] + (c & 1);
    const int32_t y = keys[3 * blk + 1] + ((c >> 1) & 1);
    const int32_t z = keys[3 * blk + 2] + ((c >> 2) & 1);
    uint32_t meta;
    return find_pos(T, x, y, z, bucket_of(T, x, y, z), &meta);
  } else {
    return __ldg(&nbr[8 * blk + c]);
  }
}

// All 128 threads resolve the 8 neighbour rows of the CTA's next kLook
// blocks at once (iterations j0 .. j0+15): one chain-walk latency per 16
// blocks instead of one per block.
template <bool kFromKeys>
__device__ __forceinline__ void lookup_batch(McSmem& sm, int buf, const TableView& T, const int32_t* keys,
                                             const int32_t* nbr, uint64_t n, uint64_t j0) {
  const int t = threadIdx.x;
  const int slot = t >> 3, c = t & 7;
  const uint64_t blk = blockIdx.x + (j0 + slot) * (uint64_t)gridDim.x;
  sm.nb[buf][slot][c] = blk < n ? load_nbr<kFromKeys>(T, keys, nbr, blk, c) : -1;
}

template <bool kFromKeys>
__global__ void __launch_bounds__(kMcThreads) k_mc_encode(TableView T, const uint8_t* __restrict__ pool,
                                                          const int32_t* __restrict__ keys,
                                                          const int32_t* __restrict__ nbr, uint64_t n,
                                                          uint32_t* __restrict__ mc_out, int8_t* __restrict__ q_out,
                                                          uint32_t* __restrict__ counts) {
  __shared__ McSmem sm;
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  const uint64_t G = gridDim.x;

  if (t == 0) {
    mbar_init(&sm.mbar[0], 1);
    mbar_init(&sm.mbar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  uint64_t blk = blockIdx.x;
  lookup_batch<kFromKeys>(sm, 0, T, keys, nbr, n, 0);
  __syncthreads();
  if (t == 0 && blk < n && sm.nb[0][0][0] >= 0) {
    mbar_arrive_expect_tx(&sm.mbar[0], VS_TSDF_BLOCK_BYTES);
    tma_load_1d(sm.buf[0], pool + (uint64_t)sm.nb[0][0][0] * VS_TSDF_BLOCK_BYTES, VS_TSDF_BLOCK_BYTES,
                &sm.mbar[0]);
  }
  uint32_t phases = 0u;  // bit s = parity of mbar[s]

  for (uint64_t j = 0; blk < n; ++j, blk += G) {
    const int s = (int)(j & 1);
    const int slot = (int)(j % kLook);
    const int bb = (int)((j / kLook) & 1);
    const uint64_t next = blk + G;
    const int32_t* nbc = sm.nb[bb][slot];
    const int32_t centre = nbc[0];
    if (slot == kLook - 1 && next < n) lookup_batch<kFromKeys>(sm, bb ^ 1, T, keys, nbr, n, j + 1);
    for (int r = t; r < 81; r += kMcThreads) {
      sm.grid_in[s][r] = 0u;
      sm.grid_ob[s][r] = 0u;
    }
    __syncthreads();  // (A) next lookups ready, grids zeroed, buf[s^1] no longer read
    if (t == 0 && next < n) {
      const int32_t nrow = (slot == kLook - 1) ? sm.nb[bb ^ 1][0][0] : sm.nb[bb][slot + 1][0];
      if (nrow >= 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive_expect_tx(&sm.mbar[s ^ 1], VS_TSDF_BLOCK_BYTES);
        tma_load_1d(sm.buf[s ^ 1], pool + (uint64_t)nrow * VS_TSDF_BLOCK_BYTES, VS_TSDF_BLOCK_BYTES,
                    &sm.mbar[s ^ 1]);
      }
    }
    uint32_t* mc_blk = mc_out ? mc_out + blk * VS_BLOCK_VOXELS : nullptr;
    int8_t* q_blk = q_out ? q_out + blk * VS_BLOCK_VOXELS : nullptr;

    if (centre < 0) {
      // absent centre: every cube's origin lives here -> all zero (:152-156)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int v = k * kMcThreads + t;
        if (mc_blk) __stcs(mc_blk + v, 0u);
        if (q_blk) __stcs((char*)q_blk + v, (char)-128);
      }
      if (counts && t == 0) counts[blk] = 0u;
      continue;
    }

    // ---- halo: 217 (tsdf, weight) pairs from the 7 positive neighbours
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int i = t + k * kMcThreads;
      if (i < 217) {
        int c, flat, row, bit;
        halo_item(i, c, flat, row, bit);
        const int32_t nrow = nbc[c];
        if (nrow >= 0) {
          const uint32_t* src = (const uint32_t*)(pool + (uint64_t)nrow * VS_TSDF_BLOCK_BYTES + 12u * flat);
          const uint32_t tb = __ldg(src), wb = __ldg(src + 1);
          if (inside_bit(tb)) atomicOr(&sm.grid_in[s][row], 1u << bit);
          if (observed_bit(wb)) atomicOr(&sm.grid_ob[s][row], 1u << bit);
        }
      }
    }

    // ---- centre: wait for the TMA copy, ballot the predicates into rows
    mbar_wait(&sm.mbar[s], (phases >> s) & 1u);
    phases ^= 1u << s;
    const uint32_t* b32 = (const uint32_t*)sm.buf[s];
    uint32_t tb[4], wb[4], rgb[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int v = k * kMcThreads + t;
      tb[k] = b32[3 * v];
      wb[k] = b32[3 * v + 1];
      rgb[k] = b32[3 * v + 2] & 0x00FFFFFFu;
      const uint32_t bin = __ballot_sync(0xffffffffu, inside_bit(tb[k]));
      const uint32_t bob = __ballot_sync(0xffffffffu, observed_bit(wb[k]));
      if (lane < 4) {
        const int r = ((k * kMcThreads + warp * 32) >> 3) + lane;  // row = y + 8z
        const int gy = r & 7, gz = r >> 3;
        atomicOr(&sm.grid_in[s][gz * 9 + gy], (bin >> (8 * lane)) & 0xFFu);
        atomicOr(&sm.grid_ob[s][gz * 9 + gy], (bob >> (8 * lane)) & 0xFFu);
      }
    }
    __syncthreads();  // (B) bit grids complete

    // ---- cube indices, cutoff, colour, quantised TSDF
    uint32_t nz = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int v = k * kMcThreads + t;
      const int x = v & 7, y = (v >> 3) & 7, z = v >> 6;
      const int r00 = z * 9 + y, r10 = r00 + 1, r01 = r00 + 9, r11 = r00 + 10;
      const uint32_t* gi = sm.grid_in[s];
      const uint32_t* go = sm.grid_ob[s];
      uint32_t idx = ((gi[r00] >> x) & 3u) | (((gi[r10] >> x) & 3u) << 2) | (((gi[r01] >> x) & 3u) << 4) |
                     (((gi[r11] >> x) & 3u) << 6);
      const uint32_t ob = ((go[r00] >> x) & 3u) | (((go[r10] >> x) & 3u) << 2) | (((go[r01] >> x) & 3u) << 4) |
                          (((go[r11] >> x) & 3u) << 6);
      if (ob != 255u || idx == 255u) idx = 0u;  // unobserved corner -> 0; cutoff 255 -> 0
      const uint32_t word = idx ? (idx | (rgb[k] << 8)) : 0u;
      if (mc_blk) __stcs(mc_blk + v, word);
      if (q_blk) __stcs((char*)q_blk + v, (char)quantise(tb[k], wb[k]));
      nz += __popc(__ballot_sync(0xffffffffu, idx != 0u));
    }
    if (counts) {
      if (lane == 0) sm.cnt[s][warp] = nz;
      __syncthreads();
      if (t == 0) counts[blk] = sm.cnt[s][0] + sm.cnt[s][1] + sm.cnt[s][2] + sm.cnt[s][3];
    }
  }
}

__global__ void k_mc_neighbors(TableView T, const int32_t* __restrict__ keys, uint64_t n,
                               int32_t* __restrict__ nbr_out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 8 * n) return;
  const uint64_t blk = i >> 3;
  const int c = (int)(i & 7);
  nbr_out[i] = load_nbr<true>(T, keys, nullptr, blk, c);
}

// One warp per MC block: ballot the non-empty cells, write them in order.
__global__ void __launch_bounds__(256) k_mc_compact(const uint32_t* __restrict__ mc, uint64_t n,
                                                    const uint64_t* __restrict__ offsets,
                                                    uint16_t* __restrict__ cell_flat, uint32_t* __restrict__ cell_mc,
                                                    uint64_t cap) {
  const uint64_t blk = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (blk >= n) return;
  uint64_t o = offsets[blk];
  const uint32_t* src = mc + blk * VS_BLOCK_VOXELS;
#pragma unroll 4
  for (int j = 0; j < 16; ++j) {
    const int v = j * 32 + lane;
    const uint32_t w = __ldcs(src + v);
    const uint32_t bal = __ballot_sync(0xffffffffu, w != 0u);
    if (w) {
      const uint64_t d = o + __popc(bal & ((1u << lane) - 1u));
      if (d < cap) {
        cell_flat[d] = (uint16_t)v;
        cell_mc[d] = w;
      }
    }
    o += __popc(bal);
  }
}

static int g_mc_grid[2] = {0, 0};

template <bool kFromKeys>
static vs_status launch_mc(const TableView& T, const uint8_t* pool, const int32_t* keys, const int32_t* nbr,
                           uint64_t n, uint8_t* mc_out, int8_t* q_out, uint32_t* counts, cudaStream_t s) {
  if (n == 0) return VS_OK;
  int& grid = g_mc_grid[kFromKeys ? 1 : 0];
  if (grid == 0) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mc_encode<kFromKeys>, kMcThreads, 0);
    if (per_sm < 1) per_sm = 1;
    grid = sms * per_sm;
  }
  const uint64_t g = n < (uint64_t)grid ? n : (uint64_t)grid;
  { ProfScope prof(1, s); k_mc_encode<kFromKeys><<<(unsigned)g, kMcThreads, 0, s>>>(T, pool, keys, nbr, n, (uint32_t*)mc_out, q_out,
                                                            counts); vsb::count_launch(); }
  VS_CK_LAUNCH("k_mc_encode");
  return VS_OK;
}

}  // namespace vsb

using namespace vsb;

extern "C" {

vs_status vs_mc_encode(const uint8_t* pool, const int32_t* nbr, uint64_t n, uint8_t* mc_out, int8_t* q_out,
                       uint32_t* counts, vs_stream_t stream) {
  if (n && (!pool || !nbr)) {
    set_error("pool/nbr must be non-NULL");
    return VS_ERR_INVALID;
  }
  if (((uintptr_t)pool & 15u) != 0) {
    set_error("pool must be 16-byte aligned (TMA bulk copy)");
    return VS_ERR_INVALID;
  }
  TableView none{};
  return launch_mc<false>(none, pool, nullptr, nbr, n, mc_out, q_out, counts, (cudaStream_t)stream);
}

vs_status vs_mc_encode_keys(const vs_table* t, const uint8_t* pool, const int32_t* keys, uint64_t n,
                            uint8_t* mc_out, int8_t* q_out, uint32_t* counts, vs_stream_t stream) {
  if (!t || (n && (!pool || !keys))) {
    set_error("table/pool/keys must be non-NULL");
    return VS_ERR_INVALID;
  }
  if (((uintptr_t)pool & 15u) != 0) {
    set_error("pool must be 16-byte aligned (TMA bulk copy)");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  return launch_mc<true>(t->view(), pool, keys, nullptr, n, mc_out, q_out, counts, (cudaStream_t)stream);
}

vs_status vs_mc_neighbors(const vs_table* t, const int32_t* keys, uint64_t n, int32_t* nbr_out,
                          vs_stream_t stream) {
  if (!t || (n && (!keys || !nbr_out))) {
    set_error("table/keys/nbr_out must be non-NULL");
    return VS_ERR_INVALID;
  }
  if (n == 0) return VS_OK;
  DeviceGuard g(t->device);
  { k_mc_neighbors<<<grid_for(8 * n, 256), 256, 0, (cudaStream_t)stream>>>(t->view(), keys, n, nbr_out); vsb::count_launch(); }
  VS_CK_LAUNCH("k_mc_neighbors");
  return VS_OK;
}

uint64_t vs_scan_workspace_bytes(uint64_t n) { return 8 * (scan_tiles(n) + 1); }

vs_status vs_mc_compact(const uint8_t* mc, const uint32_t* counts, uint64_t n, uint64_t* offsets,
                        uint16_t* cell_flat, uint32_t* cell_mc, uint64_t cell_cap, void* work_dev,
                        vs_stream_t stream) {
  if (!offsets || (n && (!mc || !counts || !work_dev))) {
    set_error("mc/counts/offsets/work must be non-NULL");
    return VS_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  VS_CK(exclusive_scan<uint32_t>(counts, n, offsets, (uint64_t*)work_dev, s));
  if (n && cell_flat && cell_mc)
    { k_mc_compact<<<grid_for(32 * n, 256), 256, 0, s>>>((const uint32_t*)mc, n, offsets, cell_flat, cell_mc,
                                                       cell_cap); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_mc_compact");
  return VS_OK;
}

}  // extern "C"
