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
#include <map>
#include <mutex>
#include <utility>

#include "faces.cuh"
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

// L2 policies (experiment knobs): in the forward sweep a TSDF
// row is first read as the halo of its -x/-y/-z neighbours and LAST as a
// centre, so centre copies may be evict-first and halo reads evict-last.
#ifndef VSB_MC_CENTRE_HINT
#define VSB_MC_CENTRE_HINT 0
#endif
#ifndef VSB_MC_HALO_HINT
#define VSB_MC_HALO_HINT 0
#endif
#ifndef VSB_MC_PROBE_HINT
#define VSB_MC_PROBE_HINT 1
#endif

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                                 uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}

__device__ __forceinline__ uint32_t ld_halo(const uint32_t* p) {
#if VSB_MC_HALO_HINT
  uint32_t v;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(policy_evict_last()));
  return v;
#else
  return __ldg(p);
#endif
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

// byte k (k < 4) = bits (k, k+1) of v: the corner pair of voxel x0 + k
__device__ __forceinline__ uint32_t pair4(uint32_t v) {
  return (v & 3u) | ((v & 6u) << 7) | ((v & 12u) << 14) | ((v & 24u) << 21);
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

// Blocks per batched neighbour lookup = blocks per work ticket (16: one find
// per thread; VSB_MC_LOOK = 8 or 4 leaves threads idle in the lookup but
// shortens a ticket, so consecutive keys are encoded closer in time).
#ifndef VSB_MC_LOOK
#define VSB_MC_LOOK 16
#endif
constexpr int kLook = VSB_MC_LOOK;
static_assert(kLook * 8 <= kMcThreads && (kLook & (kLook - 1)) == 0, "one find per thread");
#ifndef VSB_MC_STAGES
#define VSB_MC_STAGES 2
#endif
// Resident CTAs per SM the register allocation must allow (measured best:
// 10 with in-kernel hash lookups, 8 with a neighbour table; see profiles/).
#ifndef VSB_MC_MINBLOCKS_KEYS
#define VSB_MC_MINBLOCKS_KEYS 10
#endif
#ifndef VSB_MC_MINBLOCKS_NBR
#define VSB_MC_MINBLOCKS_NBR 8
#endif
constexpr int kStages = VSB_MC_STAGES;  // TMA ring depth (centre blocks in flight + 1)
constexpr int kAhead = kStages - 1;    // prefetch distance of the centre copy

struct McSmem {
  alignas(128) uint8_t buf[kStages][VS_TSDF_BLOCK_BYTES];
  alignas(8) uint64_t mbar[kStages];
  uint4 pk[2][8];  // face packs of the block's neighbours c = 1..7 (kFaces)
  uint32_t grid_in[2][81];
  uint32_t grid_ob[2][81];
  // kFaces: rows stored pre-expanded per half h: pair4(row >> 4h) (the
  // corner pairs of voxels 4h..4h+3), written once by the row's writers
  uint32_t ex_in[2][162];
  uint32_t ex_ob[2][162];
  int32_t nb[2][kLook][8];  // neighbour rows of two lookup batches
  uint32_t wsum[4];         // kCells: per-warp non-empty counts of the block
  uint32_t cbase;           // kCells: reserved start of the block's cell range
  uint32_t pair_lut[32];    // pair4 of every 5-bit row slice (VSB_MC_PAIR_LUT)
  unsigned long long tk[4]; // VSB_MC_TICKET: ticket of lookup batch k in slot k & 3
};

// Cube-index assembly through a 32-entry table of pair4 (VSB_MC_PAIR_LUT):
// entry i sits in bank i, so any mix of lane indices is conflict-free, and
// one shared load replaces pair4's eight integer ops (the scattered-halo
// encode calls it 8 times per thread and block).
#ifndef VSB_MC_PAIR_LUT
#define VSB_MC_PAIR_LUT 1
#endif

// Sweep order (experiment knob VSB_MC_REVERSE): block of sweep index i.
#ifndef VSB_MC_REVERSE
#define VSB_MC_REVERSE 0
#endif
__device__ __forceinline__ uint64_t sweep_block(uint64_t i, uint64_t n) { return VSB_MC_REVERSE ? n - 1 - i : i; }

// Work distribution.  VSB_MC_TICKET=1 (default): every lookup batch is 16
// CONSECUTIVE sweep indices claimed from a per-stream ticket counter (one
// atomicAdd per 16 blocks, claimed two batches ahead), so CTAs take work in
// sweep order as they free up: the grid-wide wavefront stays a few batches
// wide and a block's +x neighbour (97% of consecutive room keys) is read by
// the same CTA one block later.  VSB_MC_TICKET=0: static grid stride
// (iteration j of CTA c takes sweep index c + j*G); measured, the CTAs then
// drift apart by up to 1.4 ms of a 4 ms launch (profiles/r02_mc_drift.txt),
// so neighbour rows leave L2 between their halo read and their own encode.
#ifndef VSB_MC_TICKET
#define VSB_MC_TICKET 1
#endif
// next: the ticket counter; done: CTAs finished.  The last CTA to finish
// zeroes both, so the next launch on the same stream starts from 0.
struct McTickets {
  unsigned long long next, done;
};
// VSB_MC_DRIFT (measurement build): globaltimer of every CTA at iterations
// 64, 256, 640 and 1024 and at its end, read back by vs_mc_drift_read.
#ifndef VSB_MC_DRIFT
#define VSB_MC_DRIFT 0
#endif
#if VSB_MC_DRIFT
__device__ unsigned long long g_mc_drift[5][4096];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(v));
  return v;
}
#endif

// Sweep index of the CTA's j-th block (>= n: past the end); dyn: the
// launch uses tickets (large launches, see launch_mc_t).
__device__ __forceinline__ uint64_t iter_sblk(const McSmem& sm, uint32_t j, bool dyn) {
  return dyn ? (uint64_t)sm.tk[(j / kLook) & 3] * kLook + (j % kLook) : blockIdx.x + (uint64_t)j * gridDim.x;
}

// Neighbour row of block `blk` for corner-block c.
template <bool kFromKeys>
__device__ __forceinline__ int32_t load_nbr(const TableView& T, const int32_t* __restrict__ keys,
                                            const int32_t* __restrict__ nbr, uint64_t blk, int c) {
  if (kFromKeys) {
    const int32_t x = keys[3 * blk] + (c & 1);
    const int32_t y = keys[3 * blk + 1] + ((c >> 1) & 1);
    const int32_t z = keys[3 * blk + 2] + ((c >> 2) & 1);
    uint32_t meta;
    const uint32_t b = bucket_of(T, x, y, z);
#if VSB_MC_PROBE_HINT
    return find_pos(T, x, y, z, b, &meta);
#else
    return find_pos_from(T, x, y, z, b, ld_entry(T.e + b), &meta);
#endif
  } else {
    return __ldg(&nbr[8 * blk + c]);
  }
}

// All 128 threads resolve the 8 neighbour rows of the CTA's next kLook
// blocks at once (iterations j0 .. j0+15): one chain-walk latency per 16
// blocks instead of one per block.
template <bool kFromKeys, bool kDyn>
__device__ __forceinline__ void lookup_batch(McSmem& sm, int buf, const TableView& T, const int32_t* keys,
                                             const int32_t* nbr, uint64_t n, uint64_t j0, McTickets* tix) {
  const int t = threadIdx.x;
  const int slot = t >> 3, c = t & 7;
  if (slot < kLook) {
    const uint64_t sblk = iter_sblk(sm, j0 + slot, kDyn);  // sweep index
    sm.nb[buf][slot][c] = sblk < n ? load_nbr<kFromKeys>(T, keys, nbr, sweep_block(sblk, n), c) : -1;
  }
  // the ticket of the batch after next (visible after this iteration's barriers)
  if (kDyn && t == 0) sm.tk[(j0 / kLook + 2) & 3] = atomicAdd(&tix->next, 1ull);
}

// Per-thread halo items (thread t owns items t and t + 128 of 217).
struct HaloRegs {
  uint32_t tb[2], wb[2];
  int row[2];  // grid row, or -1 when the item is absent
  int bit[2];
};

// A thread's two halo items decoded once per kernel (they do not depend on
// the block): neighbour c (-1: no item), byte offset in the row, grid row/bit.
struct HaloDesc {
  int c[2];
  uint32_t off[2];
  int row[2], bit[2];
};

__device__ __forceinline__ HaloDesc halo_desc() {
  HaloDesc d;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = threadIdx.x + k * kMcThreads;
    d.c[k] = -1;
    d.off[k] = 0;
    d.row[k] = d.bit[k] = 0;
    if (i < 217) {
      int c, flat, row, bit;
      halo_item(i, c, flat, row, bit);
      d.c[k] = c;
      d.off[k] = 12u * (uint32_t)flat;  // voxel records are 12 B: (tsdf, weight) is only 4-byte aligned
      d.row[k] = row;
      d.bit[k] = bit;
    }
  }
  return d;
}

__device__ __forceinline__ void halo_prefetch(HaloRegs& h, const HaloDesc& d, const int32_t* nbc,
                                              const uint8_t* __restrict__ pool) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    h.row[k] = -1;
    if (d.c[k] >= 0) {
      const int32_t nrow = nbc[d.c[k]];
      if (nrow >= 0) {
        const uint32_t* src = (const uint32_t*)(pool + (uint64_t)nrow * VS_TSDF_BLOCK_BYTES + d.off[k]);
        h.tb[k] = ld_halo(src);
        h.wb[k] = ld_halo(src + 1);
        h.row[k] = d.row[k];
        h.bit[k] = d.bit[k];
      }
    }
  }
}

// Neighbour rows of the CTA's j-th block (j counts this CTA's blocks).
__device__ __forceinline__ const int32_t* nb_of(const McSmem& sm, uint32_t j) {
  return sm.nb[(j / kLook) & 1][j % kLook];
}

__device__ __forceinline__ void issue_centre(McSmem& sm, uint32_t j, const uint8_t* __restrict__ pool) {
  const int32_t row = nb_of(sm, j)[0];
  if (row < 0) return;
  const int b = (int)(j % kStages);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  mbar_arrive_expect_tx(&sm.mbar[b], VS_TSDF_BLOCK_BYTES);
#if VSB_MC_CENTRE_HINT
  tma_load_1d_hint(sm.buf[b], pool + (uint64_t)row * VS_TSDF_BLOCK_BYTES, VS_TSDF_BLOCK_BYTES, &sm.mbar[b],
                   policy_evict_first());
#else
  tma_load_1d(sm.buf[b], pool + (uint64_t)row * VS_TSDF_BLOCK_BYTES, VS_TSDF_BLOCK_BYTES, &sm.mbar[b]);
#endif
}


// ---- face bit-packs (halo side table).  For every TSDF pool row, the
// inside/observed predicate bits of its three LOW faces: the x = 0 face
// (bit y + 8z), the y = 0 face (bit x + 8z) and the z = 0 face (bit x + 8y),
// each as {inside lo, inside hi, observed lo, observed hi} (16 B), 48 B per
// row.  They are exactly the halo a block needs from its 7 positive
// neighbours, so an encode with packs reads seven 16-B words per block
// instead of 217 scattered 8-B voxels (~117 DRAM bursts when they miss L2).
// Packs are maintained where rows change (ingest, integration) with
// vs_mc_faces.

__device__ __forceinline__ int face_kind(int c) { return (c & 1) ? 0 : (c == 4 ? 2 : 1); }  // c: 1..7

__device__ __forceinline__ uint4 load_face(const uint8_t* __restrict__ faces, int32_t row, int c) {
  if (row < 0) return make_uint4(0u, 0u, 0u, 0u);
  return __ldg((const uint4*)(faces + (uint64_t)row * kFaceBytes) + face_kind(c));
}

__device__ __forceinline__ uint32_t bit64(uint32_t lo, uint32_t hi, int i) {
  return ((i < 32 ? lo >> i : hi >> (i - 32)) & 1u);
}
__device__ __forceinline__ uint32_t byte64(uint32_t lo, uint32_t hi, int k) {
  return ((k < 4 ? lo >> (8 * k) : hi >> (8 * (k - 4))) & 0xFFu);
}

// One warp per row (face_pack_warp, faces.cuh).
__global__ void __launch_bounds__(256) k_mc_faces(const uint8_t* __restrict__ pool, const int32_t* __restrict__ rows,
                                                  uint64_t n, uint8_t* __restrict__ faces) {
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w >= n) return;
  const int32_t row = rows ? rows[w] : (int32_t)w;
  if (row < 0) return;
  face_pack_warp(pool + (uint64_t)row * VS_TSDF_BLOCK_BYTES, faces + (uint64_t)row * kFaceBytes);
}

// Optional fused compaction (kCells): the block's non-empty
// cells are written in ascending flat index at a range reserved with ONE
// atomicAdd on a global cursor; offsets[blk] = the range start, counts[blk]
// = its length.  Each block's list is contiguous and ordered; ranges follow
// reservation order (the offsets table is the input-order view;
// vs_mc_compact gives the exact-prefix layout).  out_rows (optional): the
// MC / quantised outputs of block i go to row out_rows[i] (e.g. the MC map
// position of the block's key) instead of row i.
template <bool kFromKeys, bool kFaces, bool kCells, bool kDyn>
__global__ void __launch_bounds__(kMcThreads, kFromKeys ? VSB_MC_MINBLOCKS_KEYS : VSB_MC_MINBLOCKS_NBR) k_mc_encode(TableView T, const uint8_t* __restrict__ pool,
                                                          const uint8_t* __restrict__ faces,
                                                          const int32_t* __restrict__ keys,
                                                          const int32_t* __restrict__ nbr, uint64_t n,
                                                          const uint64_t* __restrict__ n_dev,
                                                          const int32_t* __restrict__ out_rows,
                                                          uint32_t* __restrict__ mc_out, int8_t* __restrict__ q_out,
                                                          uint32_t* __restrict__ counts,
                                                          unsigned long long* cursor, uint32_t* __restrict__ offsets,
                                                          uint16_t* __restrict__ cell_flat,
                                                          uint32_t* __restrict__ cell_mc, uint64_t cell_cap,
                                                          McTickets* tix, Entry* __restrict__ fresh_e) {
  __shared__ McSmem sm;
  if (n_dev) n = min(n, *n_dev);  // a device-produced count (no host sync in the server tick)
  const int t = threadIdx.x;
  const int lane = t & 31, warp = t >> 5;
  // the CTA's j-th block exists iff its sweep index is < n (a prefix of j);
  // each iteration evaluates the sweep index of j + 1 once (= j + kAhead)
  constexpr bool dyn = kDyn;
  static_assert(kAhead == 1, "the loop carries one look-ahead sweep index");

  if (t == 0) {
    for (int b = 0; b < kStages; ++b) mbar_init(&sm.mbar[b], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (dyn) {
      sm.tk[0] = atomicAdd(&tix->next, 1ull);
      sm.tk[1] = atomicAdd(&tix->next, 1ull);
    }
  }
  if (t < 32) sm.pair_lut[t] = pair4((uint32_t)t);  // visible after the first barrier
  if (dyn) __syncthreads();
  lookup_batch<kFromKeys, kDyn>(sm, 0, T, keys, nbr, n, 0, tix);
  __syncthreads();
  uint64_t sb = iter_sblk(sm, 0, dyn);  // sweep index of iteration j
  if (t == 0 && sb < n) issue_centre(sm, 0, pool);
  uint32_t phases = 0u;  // bit b = parity of mbar[b]
  // halo of the block processed next, loaded one iteration ahead
  const HaloDesc hd = halo_desc();
  HaloRegs hal;
  uint4 fpk = make_uint4(0u, 0u, 0u, 0u);  // kFaces: thread t < 7 holds neighbour t+1's pack, one block ahead
  if (sb < n) {
    if (kFaces) {
      if (t < 7) fpk = load_face(faces, nb_of(sm, 0)[t + 1], t + 1);
    } else {
      halo_prefetch(hal, hd, nb_of(sm, 0), pool);
    }
  }

  uint64_t sb1 = 0;  // sweep index of iteration j + 1
  for (uint32_t j = 0; sb < n; ++j, sb = sb1) {
    const uint64_t blk = sweep_block(sb, n);
#if VSB_MC_DRIFT
    if (t == 0 && blockIdx.x < 4096) {
      const int m = j == 64 ? 0 : j == 256 ? 1 : j == 640 ? 2 : j == 1024 ? 3 : -1;
      if (m >= 0) g_mc_drift[m][blockIdx.x] = gtimer();
    }
#endif
    const int s = (int)(j & 1);
    const int b = (int)(j % kStages);
    const int slot = (int)(j % kLook);
    const int32_t* nbc = nb_of(sm, j);
    const int32_t centre = nbc[0];
    // the next lookup batch must be ready before block j + kAhead is issued
    if (slot == kLook - kAhead && (dyn || blockIdx.x + (uint64_t)(j + kAhead) * gridDim.x < n))
      lookup_batch<kFromKeys, kDyn>(sm, (int)(((j / kLook) + 1) & 1), T, keys, nbr, n, (j / kLook + 1) * kLook, tix);
    if (kFaces) {
      if (t < 7) sm.pk[s][t] = fpk;  // every grid row is then written whole: no zeroing, no atomics
    } else {
      for (int r = t; r < 81; r += kMcThreads) {
        sm.grid_in[s][r] = 0u;
        sm.grid_ob[s][r] = 0u;
      }
    }
    __syncthreads();  // (A) lookups + packs ready, grids zeroed, buf[(j+kAhead)%kStages] no longer read
    sb1 = iter_sblk(sm, j + 1, dyn);  // the next batch's ticket is visible by now
    if (t == 0 && sb1 < n) issue_centre(sm, j + kAhead, pool);
    const int64_t orow = out_rows ? (int64_t)__ldg(out_rows + blk) : (int64_t)blk;  // < 0: no output row
    // the MC map entry this block's output row belongs to was created FRESH by
    // the same tick's post-less insert: settle it here (one word per block)
    if (fresh_e && t == 0 && orow >= 0) atomicAnd(&fresh_e[orow].meta, ~kFresh);
    uint32_t* mc_blk = mc_out && orow >= 0 ? mc_out + (uint64_t)orow * VS_BLOCK_VOXELS : nullptr;
    int8_t* q_blk = q_out && orow >= 0 ? q_out + (uint64_t)orow * VS_BLOCK_VOXELS : nullptr;
    const HaloRegs cur = hal;
    if (sb1 < n) {
      if (kFaces) {
        if (t < 7) fpk = load_face(faces, nb_of(sm, j + 1)[t + 1], t + 1);
      } else {
        halo_prefetch(hal, hd, nb_of(sm, j + 1), pool);
      }
    }
    if (centre < 0) {
      // absent centre: every cube's origin lives here -> all zero (:152-156)
      if (mc_blk) __stcs((uint4*)(mc_blk + 4 * t), make_uint4(0u, 0u, 0u, 0u));
      if (q_blk) __stcs((uint32_t*)(q_blk + 4 * t), 0x80808080u);
      if (kCells && t == 0) offsets[blk] = 0u;
      continue;  // counts[blk] stays 0
    }

    if (kFaces) {
      // the 17 rows on the +y / +z faces (grid rows gz*9 + 8, 72 + gy, 80)
      if (t >= 64 && t < 81) {
        uint4 lo, hi;  // the byte-source face (bits 0..7) and the bit-8 source face
        int kb, ib, row;
        if (t < 72) {  // gy = 8, gz = t - 64: y-face of (0,1,0), x-face bit (0,0,gz) of (1,1,0)
          lo = sm.pk[s][1], hi = sm.pk[s][2], kb = t - 64, ib = 8 * (t - 64), row = (t - 64) * 9 + 8;
        } else if (t < 80) {  // gz = 8, gy = t - 72: z-face of (0,0,1), x-face bit (0,gy,0) of (1,0,1)
          lo = sm.pk[s][3], hi = sm.pk[s][4], kb = t - 72, ib = t - 72, row = 72 + (t - 72);
        } else {  // gy = gz = 8: y-face byte 0 of (0,1,1), x-face bit 0 of (1,1,1)
          lo = sm.pk[s][5], hi = sm.pk[s][6], kb = 0, ib = 0, row = 80;
        }
        const uint32_t vi = byte64(lo.x, lo.y, kb) | (bit64(hi.x, hi.y, ib) << 8);
        const uint32_t vo = byte64(lo.z, lo.w, kb) | (bit64(hi.z, hi.w, ib) << 8);
        sm.ex_in[s][2 * row] = pair4(vi);
        sm.ex_in[s][2 * row + 1] = pair4(vi >> 4);
        sm.ex_ob[s][2 * row] = pair4(vo);
        sm.ex_ob[s][2 * row + 1] = pair4(vo >> 4);
      }
    }

    // ---- halo: 217 (tsdf, weight) pairs from the 7 positive neighbours,
    // loaded during the previous iteration
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      if (!kFaces && cur.row[k] >= 0) {
        if (inside_bit(cur.tb[k])) atomicOr(&sm.grid_in[s][cur.row[k]], 1u << cur.bit[k]);
        if (observed_bit(cur.wb[k])) atomicOr(&sm.grid_ob[s][cur.row[k]], 1u << cur.bit[k]);
      }
    }

    // ---- centre: wait for the TMA copy.  Thread t owns voxels 4t .. 4t+3,
    // i.e. half of row r = t/2 (row = y + 8z), x = 4h .. 4h+3 with h = t&1.
    mbar_wait(&sm.mbar[b], (phases >> b) & 1u);
    phases ^= 1u << b;
    const uint4* b128 = (const uint4*)(sm.buf[b] + 48 * t);  // 4 voxels x 12 B
    const uint4 p0 = b128[0], p1 = b128[1], p2 = b128[2];
    const uint32_t tb[4] = {p0.x, p0.w, p1.z, p2.y};
    const uint32_t wb[4] = {p0.y, p1.x, p1.w, p2.z};
    const uint32_t rgb[4] = {p0.z & 0xFFFFFFu, p1.y & 0xFFFFFFu, p2.x & 0xFFFFFFu, p2.w & 0xFFFFFFu};
    const int h = t & 1, r = t >> 1, y = r & 7, z = r >> 3, x0 = 4 * h;
    uint32_t in4 = 0, ob4 = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      in4 |= inside_bit(tb[k]) << k;
      ob4 |= observed_bit(wb[k]) << k;
    }
    // the two halves of a row meet in adjacent lanes
    uint32_t in_row = in4 << x0, ob_row = ob4 << x0;
    in_row |= __shfl_xor_sync(0xffffffffu, in_row, 1);
    ob_row |= __shfl_xor_sync(0xffffffffu, ob_row, 1);
    if (kFaces) {
      // whole rows: centre bits 0..7 + the +x neighbour's x-face bit as bit 8;
      // each lane of the pair stores its own half, pre-expanded
      const uint4 c1 = sm.pk[s][0];
      const int i = y + 8 * z;
      const uint32_t vi = in_row | (bit64(c1.x, c1.y, i) << 8);
      const uint32_t vo = ob_row | (bit64(c1.z, c1.w, i) << 8);
      sm.ex_in[s][2 * (z * 9 + y) + h] = pair4(vi >> x0);
      sm.ex_ob[s][2 * (z * 9 + y) + h] = pair4(vo >> x0);
    } else if (h == 0) {
      atomicOr(&sm.grid_in[s][z * 9 + y], in_row);
      atomicOr(&sm.grid_ob[s][z * 9 + y], ob_row);
    }
    __syncthreads();  // (B) bit grids complete

    // ---- cube indices, cutoff, colour, quantised TSDF: 4 voxels per thread
    const int r00 = z * 9 + y;
    uint32_t word[4];
    uint32_t qw = 0, nz = 0;
    // all 4 cube indices at once, one per byte: byte k of pair(v) holds bits
    // (k, k+1) of row v, so the 8 corner bits of voxel k are the 4 rows'
    // pairs stacked at bit offsets 0/2/4/6 (corner c = (c&1, c>>1&1, c>>2&1))
    uint32_t I, O;
    if (kFaces) {
      const uint32_t* ei = sm.ex_in[s] + h;
      const uint32_t* eo = sm.ex_ob[s] + h;
      I = ei[2 * r00] | (ei[2 * (r00 + 1)] << 2) | (ei[2 * (r00 + 9)] << 4) | (ei[2 * (r00 + 10)] << 6);
      O = eo[2 * r00] | (eo[2 * (r00 + 1)] << 2) | (eo[2 * (r00 + 9)] << 4) | (eo[2 * (r00 + 10)] << 6);
    } else {
      const uint32_t* gi = sm.grid_in[s];
      const uint32_t* go = sm.grid_ob[s];
#if VSB_MC_PAIR_LUT
      const uint32_t* L = sm.pair_lut;
      I = L[(gi[r00] >> x0) & 31u] | (L[(gi[r00 + 1] >> x0) & 31u] << 2) | (L[(gi[r00 + 9] >> x0) & 31u] << 4) |
          (L[(gi[r00 + 10] >> x0) & 31u] << 6);
      O = L[(go[r00] >> x0) & 31u] | (L[(go[r00 + 1] >> x0) & 31u] << 2) | (L[(go[r00 + 9] >> x0) & 31u] << 4) |
          (L[(go[r00 + 10] >> x0) & 31u] << 6);
#else
      I = pair4(gi[r00] >> x0) | (pair4(gi[r00 + 1] >> x0) << 2) | (pair4(gi[r00 + 9] >> x0) << 4) |
          (pair4(gi[r00 + 10] >> x0) << 6);
      O = pair4(go[r00] >> x0) | (pair4(go[r00 + 1] >> x0) << 2) | (pair4(go[r00 + 9] >> x0) << 4) |
          (pair4(go[r00 + 10] >> x0) << 6);
#endif
    }
    // keep a byte only where all 8 corners are observed and it is not 255
    const uint32_t keep = __vcmpeq4(O, 0xFFFFFFFFu) & ~__vcmpeq4(I, 0xFFFFFFFFu);
    const uint32_t idx4 = I & keep;
    const uint32_t nzm = __vcmpne4(idx4, 0u);
    nz = __popc(nzm) >> 3;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      word[k] = ((nzm >> (8 * k)) & 1u) ? ((idx4 >> (8 * k)) & 0xFFu) | (rgb[k] << 8) : 0u;
      qw |= ((uint32_t)quantise(tb[k], wb[k]) & 0xFFu) << (8 * k);
    }
    if (mc_blk) __stcs((uint4*)(mc_blk + 4 * t), make_uint4(word[0], word[1], word[2], word[3]));
    if (q_blk) __stcs((uint32_t*)(q_blk + 4 * t), qw);
    if (kCells) {
      // block total (warp inclusive scans, warp totals through shared memory),
      // ONE reservation, then every thread writes its non-empty voxels
      uint32_t incl = nz;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += v;
      }
      if (lane == 31) sm.wsum[warp] = incl;
      __syncthreads();  // (C)
      const uint32_t w0 = sm.wsum[0], w1 = sm.wsum[1], w2 = sm.wsum[2], w3 = sm.wsum[3];
      if (t == 0) {
        const uint32_t total = w0 + w1 + w2 + w3;
        const unsigned long long base = total ? atomicAdd(cursor, (unsigned long long)total) : 0ull;
        sm.cbase = (uint32_t)base;
        offsets[blk] = (uint32_t)base;
        if (counts) counts[blk] = total;
      }
      __syncthreads();  // (D)
      uint64_t d = (uint64_t)sm.cbase + (warp > 0 ? w0 : 0u) + (warp > 1 ? w1 : 0u) + (warp > 2 ? w2 : 0u) + incl - nz;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        if ((nzm >> (8 * k)) & 1u) {
          if (d < cell_cap) {
            __stcs(cell_flat + d, (uint16_t)(4 * t + k));
            __stcs(cell_mc + d, word[k]);
          }
          ++d;
        }
      }
    } else if (counts) {  // counts are zeroed by the launch: one reduction per warp, no barrier
      nz = __reduce_add_sync(0xffffffffu, nz);
      if (lane == 0 && nz) atomicAdd(counts + blk, nz);
    }
  }
#if VSB_MC_DRIFT
  if (t == 0 && blockIdx.x < 4096) g_mc_drift[4][blockIdx.x] = gtimer();
#endif
  if (dyn && t == 0) {
    __threadfence();  // this CTA's claims precede its "done"
    if (atomicAdd(&tix->done, 1ull) == gridDim.x - 1) {
      tix->next = 0ull;  // every CTA is past its last claim
      tix->done = 0ull;
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

static int g_mc_grid[8] = {0, 0, 0, 0, 0, 0, 0, 0};

struct McOut {
  const uint64_t* n_dev;
  const int32_t* out_rows;
  uint8_t* mc;
  int8_t* q;
  uint32_t* counts;
  unsigned long long* cursor;
  uint32_t* offsets;
  uint16_t* cell_flat;
  uint32_t* cell_mc;
  uint64_t cell_cap;
  Entry* fresh_e = nullptr;  // clear FRESH on fresh_e[out_rows[i]] (mc_encode_keys_clear)
};

// One zeroed ticket counter per (device, stream), kept for the process:
// launches on one stream run in order and the kernel's last CTA re-zeroes
// the counter, so it needs no memset per launch; launches on different
// streams never share one.  Allocated in chunks of 256 on first use (a
// synchronous cudaMalloc: make the first large encode on a stream outside
// any graph capture).
static McTickets* stream_tickets(cudaStream_t s) {
  static std::mutex mu;
  static std::map<std::pair<int, unsigned long long>, McTickets*> slots;
  static McTickets* chunk = nullptr;
  static int chunk_dev = -1, chunk_used = 256;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  // keyed by the stream's unique id, not its handle: cudaStreamPerThread is
  // one handle for a different stream on every host thread
  unsigned long long sid = 0;
  if (cudaStreamGetId(s, &sid) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  auto it = slots.find({dev, sid});
  if (it != slots.end()) return it->second;
  if (chunk_used == 256 || chunk_dev != dev) {
    McTickets* c = nullptr;
    if (cudaMalloc(&c, 256 * sizeof(McTickets)) != cudaSuccess) return nullptr;
    if (cudaMemset(c, 0, 256 * sizeof(McTickets)) != cudaSuccess) return nullptr;
    chunk = c, chunk_dev = dev, chunk_used = 0;
  }
  McTickets* t = chunk + chunk_used++;
  slots[{dev, sid}] = t;
  return t;
}

template <bool kFromKeys, bool kFaces, bool kCells>
static vs_status launch_mc_t(const TableView& T, const uint8_t* pool, const uint8_t* faces, const int32_t* keys,
                             const int32_t* nbr, uint64_t n, const McOut& o, cudaStream_t s) {
  int& grid = g_mc_grid[(kFromKeys ? 1 : 0) + (kFaces ? 2 : 0) + (kCells ? 4 : 0)];
  if (grid == 0) {
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_mc_encode<kFromKeys, kFaces, kCells, false>, kMcThreads, 0);
    if (per_sm < 1) per_sm = 1;
    grid = sms * per_sm;
  }
  const uint64_t g = n < (uint64_t)grid ? n : (uint64_t)grid;
  if (o.counts) VS_CK(cudaMemsetAsync(o.counts, 0, 4 * n, s));
  if (kCells) VS_CK(cudaMemsetAsync(o.cursor, 0, 8, s));
  // tickets only where every CTA gets several batches: a small launch (the
  // server tick's ~4k blocks) would otherwise run 16 blocks back to back in
  // few CTAs instead of 2-3 blocks in each
  McTickets* tix = nullptr;
  if (VSB_MC_TICKET && n >= (uint64_t)g * kLook * 4) {
    tix = stream_tickets(s);
    if (!tix) return VS_ERR_CUDA;
  }
  {
    ProfScope prof(1, s);
    auto kern = tix ? k_mc_encode<kFromKeys, kFaces, kCells, true> : k_mc_encode<kFromKeys, kFaces, kCells, false>;
    kern<<<(unsigned)g, kMcThreads, 0, s>>>(T, pool, faces, keys, nbr, n, o.n_dev, o.out_rows, (uint32_t*)o.mc, o.q,
                                            o.counts, o.cursor, o.offsets, o.cell_flat, o.cell_mc, o.cell_cap, tix,
                                            o.fresh_e);
    vsb::count_launch();
  }
  VS_CK_LAUNCH("k_mc_encode");
  return VS_OK;
}

template <bool kFromKeys>
static vs_status launch_mc(const TableView& T, const uint8_t* pool, const uint8_t* faces, const int32_t* keys,
                           const int32_t* nbr, uint64_t n, const McOut& o, cudaStream_t s) {
  if (n == 0) return VS_OK;
  const bool cells = o.cell_flat && o.cell_mc;
  if (faces)
    return cells ? launch_mc_t<kFromKeys, true, true>(T, pool, faces, keys, nbr, n, o, s)
                 : launch_mc_t<kFromKeys, true, false>(T, pool, faces, keys, nbr, n, o, s);
  return cells ? launch_mc_t<kFromKeys, false, true>(T, pool, faces, keys, nbr, n, o, s)
               : launch_mc_t<kFromKeys, false, false>(T, pool, faces, keys, nbr, n, o, s);
}

}  // namespace vsb

using namespace vsb;

extern "C" {

vs_status vs_mc_encode(const uint8_t* pool, const uint8_t* faces, const int32_t* nbr, uint64_t n, uint8_t* mc_out,
                       int8_t* q_out, uint32_t* counts, vs_stream_t stream) {
  if (n && (!pool || !nbr)) {
    set_error("pool/nbr must be non-NULL");
    return VS_ERR_INVALID;
  }
  if (((uintptr_t)pool & 15u) != 0) {
    set_error("pool must be 16-byte aligned (TMA bulk copy)");
    return VS_ERR_INVALID;
  }
  TableView none{};
  if (((uintptr_t)faces & 15u) != 0) {
    set_error("faces must be 16-byte aligned");
    return VS_ERR_INVALID;
  }
  McOut o{nullptr, nullptr, mc_out, q_out, counts, nullptr, nullptr, nullptr, nullptr, 0};
  return launch_mc<false>(none, pool, faces, nullptr, nbr, n, o, (cudaStream_t)stream);
}

vs_status vs_mc_encode_keys(const vs_table* t, const uint8_t* pool, const uint8_t* faces, const int32_t* keys,
                            uint64_t n, uint8_t* mc_out, int8_t* q_out, uint32_t* counts, vs_stream_t stream) {
  if (!t || (n && (!pool || !keys))) {
    set_error("table/pool/keys must be non-NULL");
    return VS_ERR_INVALID;
  }
  if (((uintptr_t)pool & 15u) != 0) {
    set_error("pool must be 16-byte aligned (TMA bulk copy)");
    return VS_ERR_INVALID;
  }
  if (((uintptr_t)faces & 15u) != 0) {
    set_error("faces must be 16-byte aligned");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  McOut o{nullptr, nullptr, mc_out, q_out, counts, nullptr, nullptr, nullptr, nullptr, 0};
  return launch_mc<true>(t->view(), pool, faces, keys, nullptr, n, o, (cudaStream_t)stream);
}

vs_status vs_mc_encode_keys_ex(const vs_table* t, const uint8_t* pool, const uint8_t* faces, const int32_t* keys,
                               uint64_t n, const uint64_t* n_dev, const int32_t* out_rows, uint8_t* mc_out,
                               int8_t* q_out, uint32_t* counts,
                               unsigned long long* cursor, uint32_t* offsets, uint16_t* cell_flat, uint32_t* cell_mc,
                               uint64_t cell_cap, vs_stream_t stream) {
  if (!t || (n && (!pool || !keys))) {
    set_error("table/pool/keys must be non-NULL");
    return VS_ERR_INVALID;
  }
  if (((uintptr_t)pool & 15u) != 0 || ((uintptr_t)faces & 15u) != 0) {
    set_error("pool and faces must be 16-byte aligned");
    return VS_ERR_INVALID;
  }
  if ((cell_flat || cell_mc) && !(cell_flat && cell_mc && cursor && offsets)) {
    set_error("compaction needs cell_flat, cell_mc, cursor and offsets");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  McOut o{n_dev, out_rows, mc_out, q_out, counts, cursor, offsets, cell_flat, cell_mc, cell_cap};
  return launch_mc<true>(t->view(), pool, faces, keys, nullptr, n, o, (cudaStream_t)stream);
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

vs_status vs_mc_faces(const uint8_t* pool, const int32_t* rows, uint64_t n, uint8_t* faces, vs_stream_t stream) {
  if (n && (!pool || !faces)) {
    set_error("pool/faces must be non-NULL");
    return VS_ERR_INVALID;
  }
  if (((uintptr_t)faces & 15u) != 0) {
    set_error("faces must be 16-byte aligned");
    return VS_ERR_INVALID;
  }
  if (n == 0) return VS_OK;
  { k_mc_faces<<<grid_for(32 * n, 256), 256, 0, (cudaStream_t)stream>>>(pool, rows, n, faces); vsb::count_launch(); }
  VS_CK_LAUNCH("k_mc_faces");
  return VS_OK;
}

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

namespace vsb {
vs_status mc_encode_keys_clear(const vs_table* t, const uint8_t* pool, const uint8_t* faces, const int32_t* keys,
                               uint64_t n, const uint64_t* n_dev, const int32_t* out_rows, uint8_t* mc_out,
                               int8_t* q_out, Entry* fresh_e, cudaStream_t s) {
  if (!t || !out_rows || (n && (!pool || !keys))) {
    set_error("table/pool/keys/out_rows must be non-NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  McOut o{n_dev, out_rows, mc_out, q_out, nullptr, nullptr, nullptr, nullptr, nullptr, 0, fresh_e};
  return launch_mc<true>(t->view(), pool, faces, keys, nullptr, n, o, s);
}
}  // namespace vsb

#if VSB_MC_DRIFT
// measurement build only: copies the drift timestamps (5 x 4096 u64) out
extern "C" int vs_mc_drift_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, vsb::g_mc_drift, sizeof(vsb::g_mc_drift)) == cudaSuccess ? 0 : 1;
}
#endif
