// shard.cu -- the block hash set sharded by key hash over the GPUs of one
// node, with the exchange done by the kernels themselves over peer memory
// (BASELINE config 5).
//
// The reference never shards (concurrent_hash.py is one in-process table);
// the owner function is free: owner(k) = fmix32(hash_key pre-modulo) mod G,
// bits independent of the local bucket hash_key(k) mod n.  Instead of the
// collective route (partition -> all-to-all counts -> all-to-all records ->
// apply -> all-to-all results -> scatter, shard.py's NCCL path), every rank
// maps every other rank's receive window (CUDA IPC over NVLink/NVSwitch) and
// one batch is eight stream-ordered kernels with no host synchronisation:
//
//   k_wpart_count  ops per owner in every warp tile (256 ops)
//   k_wpart_scan   one CTA per owner: exclusive scan over the warp tiles
//   k_wpart_push   stable placement: each op's 16-B record {x, y, z,
//                  op<<30 | input index} is STORED STRAIGHT INTO THE OWNER'S
//                  WINDOW (region of this source rank, input order kept);
//                  the last CTA publishes the per-owner counts and a release
//                  flag to every owner
//   k_wait         owner: acquire the G push flags of this epoch
//   k_shard_apply  owner: the mixed op over the concatenation of the G
//                  regions (source-major, input order inside a source) --
//                  exactly the order the collective route delivers, so the
//                  lowest-index-creates rule of duplicate inserts resolves
//                  the same way: per-op results equal a sequential replay of
//                  rank 0's batch, then rank 1's, ...
//   k_shard_post   created-flag fixup + free-list recycling (hash_ops.cuh)
//   k_shard_return owner: each result byte is stored straight back into the
//                  source's window at the op's input index; last CTA flags
//   k_wait         source: acquire the G return flags, then copy out
//
// Window reuse is safe without double buffering: a source pushes batch e+1
// only after every owner flagged the return of batch e, which each owner
// does after its last read of batch e's records.
#include <cstdio>
#include <cstring>
#include <vector>

#include "hash_ops.cuh"
#include "pdl.cuh"
#include "table.h"

namespace vsb {

constexpr int kMaxWorld = 32;
constexpr uint32_t kMaxKeys = 128;  // partition keys: (owner, bucket region) pairs
constexpr int kPartThreads = 256;
constexpr int kPartRounds = 8;
constexpr int kShardOpBlock = 128;
constexpr unsigned kReturnCtas = 148 * 4;
constexpr uint32_t kOrigMask = (1u << 30) - 1u;

// Start of every rank's IPC window: flags and counts written by the peers.
struct ShardHdr {
  unsigned long long push_flag[kMaxWorld];  // [src] epoch of src's last completed push into this window
  unsigned long long ret_flag[kMaxWorld];   // [owner] epoch of owner's last completed return into this window
  unsigned long long cnt[kMaxWorld];        // [src] records src pushed in its last push
  unsigned long long pad[kMaxWorld];
};
constexpr size_t kHdrBytes = 4096;
static_assert(sizeof(ShardHdr) <= kHdrBytes, "header");

// By-value view of the G windows for one launch.
struct ShardView {
  char* win[kMaxWorld];  // mapped base of every rank's window (own included)
  int world, rank;
  uint32_t bmax;        // per-source region capacity (records)
  uint64_t rec_off;     // byte offset of the records in a window
  uint64_t out_off;     // byte offset of the result bytes in a window
  uint64_t wmagic;      // fastmod_magic(world)
  // bucket-region order inside each (source, owner) region (VSB_SHARD_REGIONS):
  // records are partitioned by (owner, region of the owner's bucket), so the
  // owner applies them region by region -- the ops in flight touch one slice
  // of a table far larger than the L2 at a time
  uint32_t nreg;        // regions per owner (1 = input order)
  uint32_t tn;          // bucket count of the tables (equal on every rank)
  uint64_t tmagic;      // fastmod_magic(tn)
};

#ifndef VSB_SHARD_REGIONS
#define VSB_SHARD_REGIONS 1
#endif
#ifndef VSB_SHARD_REGIONS_MAX
#define VSB_SHARD_REGIONS_MAX 16
#endif

// Partition key of an op: owner * nreg + its bucket's region in the owner's
// table.  Stable placement by this key keeps, inside a source region, every
// key's ops in input order (one key = one owner, one region), so the
// sequential-replay rule of duplicate inserts is unchanged.
__device__ __forceinline__ uint32_t vowner_of(const ShardView& V, int32_t x, int32_t y, int32_t z, uint32_t o) {
  if (V.nreg <= 1) return o;
  const uint32_t b = fastmod(hash_raw(x, y, z), V.tmagic, V.tn);
  return o * V.nreg + (uint32_t)(((uint64_t)b * V.nreg) / V.tn);
}

__device__ __forceinline__ ShardHdr* hdr_of(const ShardView& V, int r) { return (ShardHdr*)V.win[r]; }
__device__ __forceinline__ int4* rec_of(const ShardView& V, int r) { return (int4*)(V.win[r] + V.rec_off); }
__device__ __forceinline__ uint8_t* out_of(const ShardView& V, int r) { return (uint8_t*)(V.win[r] + V.out_off); }

// fmix32 (MurmurHash3 finaliser) of the reference's pre-modulo hash.
__host__ __device__ __forceinline__ uint32_t owner_mix(int32_t x, int32_t y, int32_t z) {
  uint32_t h = hash_raw(x, y, z);
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}
__host__ __device__ __forceinline__ uint32_t owner_of(int32_t x, int32_t y, int32_t z, uint32_t world) {
  return owner_mix(x, y, z) % world;
}
// same, with the modulo by Lemire fastmod (M = fastmod_magic(world))
__device__ __forceinline__ uint32_t owner_fast(int32_t x, int32_t y, int32_t z, uint64_t M, uint32_t world) {
  return fastmod(owner_mix(x, y, z), M, world);
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Last CTA of a grid to arrive (threadFenceReduction pattern at system
// scope): every CTA fences its peer stores, then counts itself in.
__device__ __forceinline__ bool last_cta(unsigned int* ctr) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    last = atomicInc(ctr, gridDim.x - 1) == gridDim.x - 1;  // wraps to 0: self-resetting
  }
  __syncthreads();
  return last;
}

// ---- stable partition by owner (measured at world 1, 2^22 ops: count 14 us,
// scan 10 us, push 44 us; a single-pass decoupled look-back variant took
// 72 us and a CTA-tile count/scan/push 77 us -- the barrier-free warp tiles
// win).  Every warp owns a tile of
// 32 x kPartRounds ops and works without CTA barriers -- per-owner counts
// per warp tile, one CTA per owner scans them, and the push places every op
// at (tile offset + same-owner ops before it in the tile), input order kept.
constexpr uint32_t kWTile = 32 * kPartRounds;

// The warp's tile of keys (and op codes) is staged through warp-private
// shared memory with 16-byte coalesced loads when the tile is whole and the
// buffers 16-B aligned; lane l then takes op r*32+l of round r (stride-3
// words: bank-conflict free).
struct WarpStage {
  int32_t k[3 * kWTile];
  uint8_t op[kWTile];
};

// Stage the warp's tile into its shared buffer: 16-byte coalesced loads
// when the tile is whole and the buffers 16-B aligned, element loads (zero
// past n) otherwise.  Rounds then read their keys from shared memory, which
// keeps the kernels at 8 resident CTAs per SM.
__device__ __forceinline__ void stage_tile(const int32_t* __restrict__ keys, const uint8_t* __restrict__ ops,
                                           uint64_t n, uint64_t t0, WarpStage& S) {
  const uint32_t lane = lane_id();
  const bool whole = t0 + kWTile <= n && ((uintptr_t)keys & 15) == 0 && (!ops || ((uintptr_t)ops & 15) == 0);
  if (whole) {
    const int4* kv = (const int4*)(keys + 3 * t0);
#pragma unroll
    for (int q = 0; q < 3 * kWTile / 4 / 32; ++q) ((int4*)S.k)[q * 32 + lane] = __ldcs(kv + q * 32 + lane);
    if (ops && lane < kWTile / 16) ((int4*)S.op)[lane] = __ldcs((const int4*)(ops + t0) + lane);
  } else {
    for (uint32_t j = lane; j < 3 * kWTile; j += 32) S.k[j] = t0 * 3 + j < 3 * n ? ld_stream(keys + 3 * t0 + j) : 0;
    if (ops)
      for (uint32_t j = lane; j < kWTile; j += 32) S.op[j] = t0 + j < n ? ld_stream(ops + t0 + j) : (uint8_t)0;
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kPartThreads) k_wpart_count(const int32_t* __restrict__ keys, uint64_t n, ShardView V,
                                                              uint32_t nwt, uint32_t* __restrict__ tile_cnt) {
  pdl_wait();
  __shared__ uint32_t c[kPartThreads / 32][kMaxKeys];
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t wt = blockIdx.x * (kPartThreads / 32) + warp;
  if (wt >= nwt) return;
  const uint32_t NV = (uint32_t)V.world * V.nreg;
  for (uint32_t q = lane; q < NV; q += 32) c[warp][q] = 0;
  __syncwarp();
  __shared__ WarpStage stage[kPartThreads / 32];
  WarpStage& S = stage[warp];
  stage_tile(keys, nullptr, n, (uint64_t)wt * kWTile, S);
#pragma unroll
  for (int r = 0; r < kPartRounds; ++r) {
    const uint32_t j = r * 32 + lane;
    const uint64_t i = (uint64_t)wt * kWTile + j;
    const int32_t x = S.k[3 * j], y = S.k[3 * j + 1], z = S.k[3 * j + 2];
    const uint32_t o = i < n ? vowner_of(V, x, y, z, owner_fast(x, y, z, V.wmagic, (uint32_t)V.world)) : 0xFFFFFFFFu;
    const uint32_t m = __match_any_sync(0xFFFFFFFFu, o);
    if (o != 0xFFFFFFFFu && (int)lane == __ffs(m) - 1) c[warp][o] += __popc(m);
    __syncwarp();
  }
  for (uint32_t q = lane; q < NV; q += 32) tile_cnt[(size_t)q * nwt + wt] = c[warp][q];
}

// Start of every partition key's records inside its owner's region: the
// totals of the owner's lower bucket regions (one thread per key), and the
// per-owner record counts for the owners' headers.
__global__ void k_wpart_base(const uint32_t* __restrict__ totals, uint32_t world, uint32_t nreg,
                             uint32_t* __restrict__ base, uint32_t* __restrict__ owner_cnt) {
  pdl_wait();
  const uint32_t q = threadIdx.x;
  if (q >= world * nreg) return;
  uint32_t b = 0;
  for (uint32_t p = q - q % nreg; p < q; ++p) b += totals[p];
  base[q] = b;
  if (q % nreg == nreg - 1) owner_cnt[q / nreg] = b + totals[q];
}

// CTA o: exclusive scan of owner o's counts per GROUP of kTilesPerCta warp
// tiles (= one push CTA); the push CTA adds its warps' in-group prefix
// itself, so the scan is kTilesPerCta x shorter than a per-tile scan.
// Per chunk of 4,096 groups: coalesced loads of the tile counts, 8-lane
// shuffle sums into shared memory, then a block scan of 4 groups per thread.
constexpr uint32_t kTilesPerCta = kPartThreads / 32;
static_assert(kTilesPerCta == 8, "k_wpart_scan sums groups with 8-lane shuffles");
__global__ void __launch_bounds__(1024) k_wpart_scan(const uint32_t* __restrict__ tile_cnt, uint32_t nwt,
                                                     uint32_t* __restrict__ grp_off, uint32_t* __restrict__ totals) {
  pdl_wait();
  constexpr int kPer = 4;
  constexpr uint32_t kChunk = 1024 * kPer;  // groups per chunk
  __shared__ uint32_t gsum[kChunk];
  __shared__ uint32_t ws[32];
  const uint32_t o = blockIdx.x, lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t ngrp = (nwt + kTilesPerCta - 1) / kTilesPerCta;
  const uint32_t* in = tile_cnt + (size_t)o * nwt;
  uint32_t* out = grp_off + (size_t)o * ngrp;
  uint32_t carry = 0;
  for (uint32_t b = 0; b < ngrp; b += kChunk) {
    const uint64_t t0 = (uint64_t)b * kTilesPerCta;
#pragma unroll 8
    for (uint32_t it = 0; it < kChunk * kTilesPerCta / 1024; ++it) {
      const uint64_t t = t0 + (uint64_t)it * 1024 + threadIdx.x;
      uint32_t v = t < nwt ? in[t] : 0u;
      v += __shfl_xor_sync(0xFFFFFFFFu, v, 4);
      v += __shfl_xor_sync(0xFFFFFFFFu, v, 2);
      v += __shfl_xor_sync(0xFFFFFFFFu, v, 1);
      if ((lane & 7) == 0) gsum[(it * 1024 + threadIdx.x) >> 3] = v;
    }
    __syncthreads();
    uint32_t v[kPer], sum = 0;
#pragma unroll
    for (int k = 0; k < kPer; ++k) sum += (v[k] = gsum[threadIdx.x * kPer + k]);
    uint32_t xs = sum;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, xs, d);
      if ((int)lane >= d) xs += y;
    }
    if (lane == 31) ws[warp] = xs;
    __syncthreads();
    if (warp == 0) {
      uint32_t q = ws[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, q, d);
        if ((int)lane >= d) q += y;
      }
      ws[lane] = q;
    }
    __syncthreads();
    uint32_t run = carry + (warp ? ws[warp - 1] : 0u) + xs - sum;
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      gsum[threadIdx.x * kPer + k] = run;
      run += v[k];
    }
    carry += ws[31];
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kPer; ++k) {
      const uint32_t g = b + k * 1024 + threadIdx.x;
      if (g < ngrp) out[g] = gsum[k * 1024 + threadIdx.x];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[o] = carry;
}

__global__ void __launch_bounds__(kPartThreads) k_wpart_push(ShardView V, const int32_t* __restrict__ keys,
                                                             const uint8_t* __restrict__ ops, uint64_t n, uint32_t nwt,
                                                             const uint32_t* __restrict__ tile_cnt,
                                                             const uint32_t* __restrict__ grp_off,
                                                             const uint32_t* __restrict__ base,
                                                             const uint32_t* __restrict__ owner_cnt,
                                                             unsigned long long epoch, unsigned int* ctr) {
  pdl_wait();
  __shared__ uint32_t run[kPartThreads / 32][kMaxKeys];
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t wt = blockIdx.x * (kPartThreads / 32) + warp;
  const int G = V.world;
  const uint32_t NV = (uint32_t)G * V.nreg;  // partition keys (<= kMaxKeys)
  if (wt < nwt) {
    // tile offset = the group's offset + the tiles of earlier warps in the
    // group + the start of the key's bucket region inside its owner's region
    const uint32_t ngrp = (nwt + kTilesPerCta - 1) / kTilesPerCta;
    for (uint32_t q = lane; q < NV; q += 32) {
      uint32_t off0 = grp_off[(size_t)q * ngrp + blockIdx.x] + base[q];
      for (uint32_t w = 0; w < warp; ++w) off0 += tile_cnt[(size_t)q * nwt + blockIdx.x * kTilesPerCta + w];
      run[warp][q] = off0;
    }
    __syncwarp();
    const uint64_t t0 = (uint64_t)wt * kWTile;
    __shared__ WarpStage stage[kPartThreads / 32];
    WarpStage& S = stage[warp];
    stage_tile(keys, ops, n, t0, S);
    const size_t region = (size_t)V.rank * V.bmax;
#pragma unroll
    for (int r = 0; r < kPartRounds; ++r) {
      const uint32_t j = r * 32 + lane;
      const uint64_t i = t0 + j;
      const int32_t x = S.k[3 * j], y = S.k[3 * j + 1], z = S.k[3 * j + 2];
      const uint32_t o = i < n ? vowner_of(V, x, y, z, owner_fast(x, y, z, V.wmagic, (uint32_t)G)) : 0xFFFFFFFFu;
      const uint32_t m = __match_any_sync(0xFFFFFFFFu, o);
      if (o != 0xFFFFFFFFu) {
        const uint32_t off = run[warp][o] + __popc(m & lanemask_lt());
        int4 rec;
        rec.x = x;
        rec.y = y;
        rec.z = z;
        rec.w = (int)(((uint32_t)S.op[j] << 30) | (uint32_t)i);
        rec_of(V, o / V.nreg)[region + off] = rec;  // peer store over NVLink (local for the own rank)
      }
      __syncwarp();
      if (o != 0xFFFFFFFFu && (int)lane == __ffs(m) - 1) run[warp][o] += __popc(m);
      __syncwarp();
    }
  }
  if (last_cta(ctr) && (int)threadIdx.x < G) {
    __threadfence_system();
    ShardHdr* h = hdr_of(V, threadIdx.x);
    st_relaxed_sys(&h->cnt[V.rank], owner_cnt[threadIdx.x]);
    st_release_sys(&h->push_flag[V.rank], epoch);
  }
}

// Acquire flags[0..world) >= epoch.  Bounded: after `timeout_ns` the error
// word gets bit 1 and the kernel returns (a peer that never arrives must not
// hang the GPU).
__global__ void k_wait(const unsigned long long* flags, int world, unsigned long long epoch, unsigned int* err,
                       uint64_t timeout_ns) {
  pdl_wait();
  const int r = threadIdx.x;
  if (r >= world) return;
  const uint64_t t0 = globaltimer();
  while (ld_acquire_sys(flags + r) < epoch) {
    __nanosleep(200);
    if (globaltimer() - t0 > timeout_ns) {
      atomicOr(err, 2u);
      return;
    }
  }
}

// Routed op v (the concatenation of the G source regions, source-major):
// region r and record position p of v from the per-source counts, whose
// prefix sums every CTA keeps in shared memory.
struct Routed {
  const uint32_t* pre;  // shared [world + 1]
  int world;
  uint32_t bmax;
  __device__ __forceinline__ uint32_t total() const { return pre[world]; }
  __device__ __forceinline__ size_t pos(uint32_t v, int* region) const {
    int r = 0;
    while (r + 1 < world && pre[r + 1] <= v) ++r;
    *region = r;
    return (size_t)r * bmax + (v - pre[r]);
  }
};

// Every thread of the CTA must call it (barrier inside).  After a k_wait
// timeout (error bit 1) the regions of a peer that never arrived still hold
// its PREVIOUS batch: the routed set is then empty, so nothing stale is
// applied, fixed up or returned (vs_shard_check reports the timeout).
__device__ __forceinline__ Routed load_routed(const ShardView& V, uint32_t* spre, const unsigned int* err) {
  if (threadIdx.x == 0) {
    const ShardHdr* h = hdr_of(V, V.rank);
    const bool dead = (*(const volatile unsigned int*)err & 2u) != 0u;
    uint32_t a = 0;
    spre[0] = 0;
    for (int r = 0; r < V.world; ++r) spre[r + 1] = a += dead ? 0u : (uint32_t)h->cnt[r];
  }
  __syncthreads();
  Routed R;
  R.pre = spre;
  R.world = V.world;
  R.bmax = V.bmax;
  return R;
}

__global__ void __launch_bounds__(kShardOpBlock, 2048 / kShardOpBlock) k_shard_apply(TableView T, ShardView V, uint8_t* __restrict__ res,
                                                               int32_t* __restrict__ idx, uint32_t* __restrict__ wv,
                                                               const unsigned int* err) {
  pdl_wait();
  __shared__ uint32_t spre[kMaxWorld + 1];
  const Routed R = load_routed(V, spre, err);
  const int4* rec = rec_of(V, V.rank);
  const uint32_t total = R.total();
  int delta = 0;
#pragma unroll 1
  for (uint32_t v = blockIdx.x * kShardOpBlock + threadIdx.x; v < total; v += gridDim.x * kShardOpBlock) {
    int r;
    const int4 q = __ldcs(rec + R.pos(v, &r));
    const uint32_t b = bucket_of(T, q.x, q.y, q.z);
    const int4 pre = ld_bucket(T.e + b);
    __stcs(wv + v, (uint32_t)q.w);  // op | input index, for the post and return passes (4 B, not the record)
    delta += apply_one(T, q.x, q.y, q.z, (uint8_t)((uint32_t)q.w >> 30), v, b, pre, res, idx);
  }
  add_size_cta(T, delta);
}

// Post pass over the routed ops: 4 ops per thread per round (loads in
// flight first), created-flag fixup via the records, vacated excess entries
// back onto the free list with one warp-wide reservation per round.
__global__ void __launch_bounds__(256) k_shard_post(TableView T, ShardView V, uint8_t* __restrict__ res,
                                                    const int32_t* __restrict__ idx, const uint32_t* __restrict__ wv,
                                                    const unsigned int* err) {
  pdl_wait();
  constexpr int kOps = 4;
  __shared__ uint32_t spre[kMaxWorld + 1];
  const Routed R = load_routed(V, spre, err);
  const int4* rec = rec_of(V, V.rank);
  const uint32_t total = R.total();
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t rounds = (total + kOps * stride - 1) / (kOps * stride);  // uniform: warps stay converged
#pragma unroll 1
  for (uint32_t it = 0; it < rounds; ++it) {
    const uint32_t v0 = it * kOps * stride + blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t w[kOps];
    uint8_t rs[kOps];
    int32_t ps[kOps];
#pragma unroll
    for (int k = 0; k < kOps; ++k) {
      const uint32_t v = v0 + k * stride;
      w[k] = 0xFFFFFFFFu;
      if (v < total) {
        w[k] = wv[v];
        rs[k] = res[v];
        ps[k] = idx[v];
      }
    }
    uint32_t vac[kOps];
    int nv = 0;
#pragma unroll
    for (int k = 0; k < kOps; ++k) {
      const uint32_t v = v0 + k * stride;
      if (v >= total) continue;
      const uint32_t op = w[k] >> 30;
      if (op == 0u /*VS_OP_INSERT*/ && rs[k]) {
        post_op_t(
            T,
            [&](uint64_t m) {  // records are read only for a duplicate claim
              int rm, rv;
              const int4 p = rec[R.pos((uint32_t)m, &rm)];
              const int4 qv = rec[R.pos(v, &rv)];
              return p.x == qv.x && p.y == qv.y && p.z == qv.z;
            },
            v, 0, res, ps[k]);
      } else if (op == 2u /*VS_OP_ERASE*/ && rs[k] && ps[k] >= (int32_t)T.n) {
        vac[nv++] = (uint32_t)ps[k];
      }
    }
    push_free_many<kOps>(T, vac, nv);
  }
}

__global__ void __launch_bounds__(256) k_shard_return(ShardView V, const uint8_t* __restrict__ res,
                                                      const uint32_t* __restrict__ wv, unsigned long long epoch,
                                                      unsigned int* ctr, const unsigned int* err) {
  pdl_wait();
  __shared__ uint32_t spre[kMaxWorld + 1];
  const Routed R = load_routed(V, spre, err);
  const uint32_t total = R.total();
  const uint32_t stride = gridDim.x * blockDim.x;
#pragma unroll 1
  for (uint32_t v0 = blockIdx.x * blockDim.x + threadIdx.x; v0 < total; v0 += 4 * stride) {
    // four independent loads in flight before the stores
    uint32_t w[4];
    uint8_t b[4];
    int r[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t v = v0 + k * stride;
      if (v < total) {
        R.pos(v, &r[k]);
        w[k] = __ldcs(wv + v);
        b[k] = res[v];
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (v0 + k * stride < total) out_of(V, r[k])[w[k] & kOrigMask] = b[k];  // peer store into the source's window
  }
  // after a timeout no return flag is raised: the sources time out too
  if (last_cta(ctr) && threadIdx.x < V.world && !(*(const volatile unsigned int*)err & 2u)) {
    __threadfence_system();
    st_release_sys(&hdr_of(V, threadIdx.x)->ret_flag[V.rank], epoch);
  }
}

}  // namespace vsb

using namespace vsb;

struct vs_shard {
  vs_table* table = nullptr;
  int device = 0, rank = 0, world = 1;
  uint32_t bmax = 0;
  char* win = nullptr;  // own window (cudaMalloc, exported over CUDA IPC)
  size_t win_bytes = 0, rec_off = 0, out_off = 0;
  char* peer[kMaxWorld] = {};
  bool opened[kMaxWorld] = {};
  bool connected = false;
  // local workspace
  uint32_t* tile_cnt = nullptr;  // [world][warp tiles] ops per owner per warp tile
  uint32_t* grp_off = nullptr;   // [world][groups of kTilesPerCta tiles] exclusive offsets
  uint32_t* totals = nullptr;
  unsigned int* ctl = nullptr;  // [0] push CTA counter, [32] return CTA counter, [64] error word
  uint8_t* res = nullptr;
  int32_t* idx = nullptr;
  uint32_t* wv = nullptr;  // [world * bmax] op | input index of every routed op (written by the apply)
  unsigned long long epoch = 0;
  uint64_t timeout_ns = 20ull * 1000000000ull;

  ShardView view() const {
    ShardView v;
    memset(&v, 0, sizeof(v));
    for (int r = 0; r < world; ++r) v.win[r] = peer[r];
    v.world = world;
    v.rank = rank;
    v.bmax = bmax;
    v.rec_off = rec_off;
    v.out_off = out_off;
    v.wmagic = fastmod_magic((uint32_t)world);
    // region order pays off only when the table is far larger than the L2
    // (at world 1: 125M keys, 2^24 ops 1.50 -> 1.28 ms; 10M keys 0.33 -> 0.36 ms)
    const bool big = (uint64_t)table->cap * sizeof(Entry) >= (1ull << 30);
    const uint32_t cap_r = (uint32_t)(kMaxKeys / world < VSB_SHARD_REGIONS_MAX ? kMaxKeys / world
                                                                              : VSB_SHARD_REGIONS_MAX);
    v.nreg = VSB_SHARD_REGIONS && big ? cap_r : 1u;
    v.tn = table->n;
    v.tmagic = table->magic;
    return v;
  }
};

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

extern "C" {

vs_status vs_shard_create(vs_table* local, int rank, int world, uint64_t max_batch, vs_shard** out) {
  if (!local || !out || world < 1 || world > kMaxWorld || rank < 0 || rank >= world || max_batch < 1 ||
      max_batch > kOrigMask + 1ull || (uint64_t)world * max_batch > 0x7FFFFFFFull) {
    set_error("vs_shard_create: need 1 <= world <= 32, 0 <= rank < world, 1 <= max_batch <= 2^30, world*max_batch < 2^31");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(local->device);
  vs_shard* s = new vs_shard();
  s->table = local;
  s->device = local->device;
  s->rank = rank;
  s->world = world;
  s->bmax = (uint32_t)max_batch;
  s->rec_off = kHdrBytes;
  s->out_off = align_up(s->rec_off + (size_t)world * max_batch * sizeof(int4), 256);
  s->win_bytes = align_up(s->out_off + max_batch, 4096);
  cudaError_t e = cudaMalloc(&s->win, s->win_bytes);
  if (e == cudaSuccess) e = cudaMemset(s->win, 0, kHdrBytes);
  // warp tiles (kWTile ops) are the finest partition granularity
  const size_t nwt_max = (max_batch + kWTile - 1) / kWTile;
  if (e == cudaSuccess) e = cudaMalloc(&s->tile_cnt, (size_t)kMaxKeys * nwt_max * 4);  // (owner, region) rows
  if (e == cudaSuccess) e = cudaMalloc(&s->grp_off, (size_t)kMaxKeys * nwt_max * 4);
  if (e == cudaSuccess) e = cudaMalloc(&s->totals, 3 * kMaxKeys * 4);  // totals | base | per-owner counts
  if (e == cudaSuccess) e = cudaMalloc(&s->ctl, 128 * 4);
  if (e == cudaSuccess) e = cudaMemset(s->ctl, 0, 128 * 4);
  if (e == cudaSuccess) e = cudaMalloc(&s->res, (size_t)world * max_batch);
  if (e == cudaSuccess) e = cudaMalloc(&s->idx, (size_t)world * max_batch * 4);
  if (e == cudaSuccess) e = cudaMalloc(&s->wv, (size_t)world * max_batch * 4);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    vs_shard_destroy(s);
    return cuda_status(e, "vs_shard_create");
  }
  // load every kernel of the route now: with lazy module loading, a first
  // launch inside vs_shard_apply could wait for the device while this rank's
  // k_wait spins on peers whose launches sit behind it (one-process groups)
  {
    cudaFuncAttributes fa;
    const void* fns[] = {(const void*)k_wpart_count, (const void*)k_wpart_scan, (const void*)k_wpart_base,
                         (const void*)k_wpart_push,
                         (const void*)k_wait,        (const void*)k_shard_apply, (const void*)k_shard_post,
                         (const void*)k_shard_return};
    for (const void* f : fns)
      if (e == cudaSuccess) e = cudaFuncGetAttributes(&fa, f);
    // the staged partition kernels want 8 CTAs x 27 KB of shared memory per SM
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute((const void*)k_wpart_count, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute((const void*)k_wpart_push, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    if (e != cudaSuccess) {
      vs_shard_destroy(s);
      return cuda_status(e, "vs_shard_create (kernel load)");
    }
  }
  s->peer[rank] = s->win;
  if (world == 1) s->connected = true;
  *out = s;
  return VS_OK;
}

vs_status vs_shard_export(vs_shard* s, uint8_t handle_out[64]) {
  if (!s || !handle_out) {
    set_error("vs_shard_export: NULL argument");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(s->device);
  cudaIpcMemHandle_t h;
  VS_CK(cudaIpcGetMemHandle(&h, s->win));
  static_assert(sizeof(h) == 64, "ipc handle size");
  memcpy(handle_out, &h, 64);
  return VS_OK;
}

vs_status vs_shard_connect(vs_shard* s, const uint8_t* handles) {
  if (!s || !handles) {
    set_error("vs_shard_connect: NULL argument");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(s->device);
  for (int r = 0; r < s->world; ++r) {
    if (r == s->rank || s->opened[r]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, handles + 64 * (size_t)r, 64);
    void* p = nullptr;
    VS_CK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    s->peer[r] = (char*)p;
    s->opened[r] = true;
  }
  s->connected = true;
  return VS_OK;
}

vs_status vs_shard_connect_local(vs_shard* const* shards, int n) {
  if (!shards || n < 1) {
    set_error("vs_shard_connect_local: bad arguments");
    return VS_ERR_INVALID;
  }
  for (int i = 0; i < n; ++i) {
    if (!shards[i] || shards[i]->world != n || shards[i]->rank != i || shards[i]->device != shards[0]->device ||
        shards[i]->bmax != shards[0]->bmax) {
      set_error("vs_shard_connect_local: shards must be ranks 0..n-1 of one world on one device, same max_batch");
      return VS_ERR_INVALID;
    }
  }
  for (int i = 0; i < n; ++i) {
    for (int r = 0; r < n; ++r) shards[i]->peer[r] = shards[r]->win;
    shards[i]->connected = true;
  }
  return VS_OK;
}

vs_status vs_shard_apply(vs_shard* s, const int32_t* keys, const uint8_t* ops, uint64_t n, uint8_t* result,
                         vs_stream_t stream) {
  if (!s || !s->connected) {
    set_error("vs_shard_apply: shard not connected (vs_shard_connect)");
    return VS_ERR_INVALID;
  }
  if (n > s->bmax || (n && (!keys || !ops || !result))) {
    set_error("vs_shard_apply: n > max_batch or NULL buffer");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(s->device);
  cudaStream_t st = (cudaStream_t)stream;
  const unsigned long long ep = ++s->epoch;
  const ShardView V = s->view();
  ShardHdr* own = (ShardHdr*)s->win;
  {
    const uint32_t nwt = (uint32_t)((n + kWTile - 1) / kWTile);
    const unsigned ctas = nwt ? (nwt + kPartThreads / 32 - 1) / (kPartThreads / 32) : 1u;
    if (nwt) {
      VS_CK(launch_pdl(k_wpart_count, ctas, kPartThreads, 0, st, keys, n, V, nwt, s->tile_cnt));
      count_launch();
      VS_CK(launch_pdl(k_wpart_scan, s->world * V.nreg, 1024, 0, st, s->tile_cnt, nwt, s->grp_off, s->totals));
      count_launch();
      VS_CK(launch_pdl(k_wpart_base, 1, kMaxKeys, 0, st, s->totals, (uint32_t)s->world, V.nreg, s->totals + kMaxKeys,
                       s->totals + 2 * kMaxKeys));
      count_launch();
    } else {
      VS_CK(cudaMemsetAsync(s->totals, 0, 3 * kMaxKeys * 4, st));
    }
    VS_CK(launch_pdl(k_wpart_push, ctas, kPartThreads, 0, st, V, keys, ops, n, nwt, s->tile_cnt, s->grp_off,
                     s->totals + kMaxKeys, s->totals + 2 * kMaxKeys, ep, s->ctl));
    count_launch();
  }
  VS_CK(launch_pdl(k_wait, 1, 32, 0, st, own->push_flag, s->world, ep, s->ctl + 64, s->timeout_ns));
  count_launch();
  // incoming ~ n per rank when the keys hash evenly; the grid-stride loops
  // cover any skew
  const uint64_t hint = n + n / 8 + 4096;
  const TableView T = s->table->next_view();
  {
    ProfScope prof(0, st);
    k_shard_apply<<<grid_for(hint, kShardOpBlock), kShardOpBlock, 0, st>>>(T, V, s->res, s->idx, s->wv, s->ctl + 64);
    count_launch();
  }
  VS_CK(launch_pdl(k_shard_post, grid_for(hint, 256 * 4), 256, 0, st, T, V, s->res, s->idx, s->wv, s->ctl + 64));
  count_launch();
  // bounded grid: the last-CTA signal costs one same-address atomic per CTA
  VS_CK(launch_pdl(k_shard_return, kReturnCtas, 256, 0, st, V, s->res, s->wv, ep, s->ctl + 32, s->ctl + 64));
  count_launch();
  VS_CK(launch_pdl(k_wait, 1, 32, 0, st, own->ret_flag, s->world, ep, s->ctl + 64, s->timeout_ns));
  count_launch();
  if (n) VS_CK(cudaMemcpyAsync(result, s->win + s->out_off, n, cudaMemcpyDeviceToDevice, st));
  VS_CK_LAUNCH("vs_shard_apply");
  return VS_OK;
}

vs_status vs_shard_set_timeout_ms(vs_shard* s, uint64_t ms) {
  if (!s || ms < 1) {
    set_error("vs_shard_set_timeout_ms: bad arguments");
    return VS_ERR_INVALID;
  }
  s->timeout_ns = ms * 1000000ull;
  return VS_OK;
}

vs_status vs_shard_check(vs_shard* s) {
  if (!s) {
    set_error("vs_shard_check: NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(s->device);
  unsigned int err = 0;
  VS_CK(cudaMemcpy(&err, s->ctl + 64, 4, cudaMemcpyDeviceToHost));
  if (err & 2u) {
    set_error("vs_shard: a peer did not arrive within the timeout (collective call mismatch?)");
    return VS_ERR_CUDA;
  }
  return VS_OK;
}

vs_status vs_shard_owner(const int32_t* keys, uint64_t n, int world, int32_t* owner_out) {
  if (world < 1 || (n && (!keys || !owner_out))) {
    set_error("vs_shard_owner: bad arguments");
    return VS_ERR_INVALID;
  }
  for (uint64_t i = 0; i < n; ++i)
    owner_out[i] = (int32_t)owner_of(keys[3 * i], keys[3 * i + 1], keys[3 * i + 2], (uint32_t)world);
  return VS_OK;
}

void vs_shard_destroy(vs_shard* s) {
  if (!s) return;
  DeviceGuard g(s->device);
  for (int r = 0; r < kMaxWorld; ++r)
    if (s->opened[r]) cudaIpcCloseMemHandle(s->peer[r]);
  cudaFree(s->win);
  cudaFree(s->tile_cnt);
  cudaFree(s->grp_off);
  cudaFree(s->totals);
  cudaFree(s->ctl);
  cudaFree(s->res);
  cudaFree(s->idx);
  cudaFree(s->wv);
  delete s;
}

}  // extern "C"
