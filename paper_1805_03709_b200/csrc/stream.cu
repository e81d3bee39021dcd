// stream.cu -- per-client stream-set updates on the GPU.
//
// Reference (server.py):
//   StreamSet            :49-95   hash set + generation-order deque of NEWLY
//                                 created keys (stale entries tolerated)
//   on_tsdf_batch        :299-315 affected = ordered first-occurrence dedup of
//                                 affected_mc_blocks(k) for every updated k,
//                                 then insert_many(affected) into EVERY client
//   _attach_session      :221-249 fresh client: new set filled with
//                                 mc_map.snapshot_keys()
//   on_reset_blocks      :425-436 remove keys from every client set
// B200 design: all clients' inserts are ONE launch over a (key, client) grid;
// the per-client "created" subset (= the set difference affected \ pending_c)
// is placed into each client's FIFO ring by ONE exclusive scan over the
// C x n created flags (segment c starts at c*n), so the FIFO append order is
// the affected order, exactly the deque.append order of the reference.
#include <algorithm>
#include <cstdint>
#include <vector>

#include <cooperative_groups.h>

#include "faces.cuh"
#include "hash_ops.cuh"
#include "pdl.cuh"
#include "scan.cuh"
#include "table.h"

#ifndef VSB_FAN_SMALL
#define VSB_FAN_SMALL 1  // one-launch fan-out for n <= 4096 keys (k_multi_fan_small)
#endif
#ifndef VSB_DEDUP_MIX
#define VSB_DEDUP_MIX 1
#endif

namespace vsb {

constexpr int kMaxSets = 32;

struct SetViews {
  TableView v[kMaxSets];
};

struct FifoViews {
  int32_t* keys[kMaxSets];
  uint64_t cap[kMaxSets];
  uint64_t* tail[kMaxSets];  // device word per client (absolute tail)
};

__global__ void __launch_bounds__(256) k_multi_insert(const __grid_constant__ SetViews V,
                                                      const int32_t* __restrict__ keys, uint64_t n,
                                                      const uint64_t* __restrict__ n_dev,
                                                      uint8_t* __restrict__ created, int32_t* __restrict__ index) {
  pdl_wait();
  const int c = blockIdx.y;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const TableView& T = V.v[c];
  const uint64_t nv = n_dev && *n_dev < n ? *n_dev : n;  // keys past the device count: not inserted
  int delta = 0;
  if (i >= nv && i < n) {
    created[(uint64_t)c * n + i] = 0;
    index[(uint64_t)c * n + i] = -1;
  }
  if (i < nv) {
    const InsertResult r = insert_key(T, keys[3 * i], keys[3 * i + 1], keys[3 * i + 2], (int32_t)i);
    created[(uint64_t)c * n + i] = r.created;
    index[(uint64_t)c * n + i] = r.pos;
    delta = r.created;
  }
  add_size_cta(T, delta);
}

__global__ void k_multi_fixup(const __grid_constant__ SetViews V, const int32_t* __restrict__ keys, uint64_t n,
                              uint8_t* __restrict__ created, const int32_t* __restrict__ index) {
  pdl_wait();
  const int c = blockIdx.y;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  post_op(V.v[c], keys, i, 0, created + (uint64_t)c * n, index[(uint64_t)c * n + i]);
}

__global__ void k_fifo_append(const __grid_constant__ FifoViews F, const int32_t* __restrict__ keys, uint64_t n,
                              const uint8_t* __restrict__ created, const uint64_t* __restrict__ off) {
  pdl_wait();
  const int c = blockIdx.y;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t j = (uint64_t)c * n + i;
  if (!created[j]) return;
  const uint64_t rank = off[j] - off[(uint64_t)c * n];
  const uint64_t p = (*F.tail[c] + rank) % F.cap[c];
  int32_t* dst = F.keys[c] + 3 * p;
  dst[0] = keys[3 * i];
  dst[1] = keys[3 * i + 1];
  dst[2] = keys[3 * i + 2];
}

__global__ void k_fifo_tail(const __grid_constant__ FifoViews F, bool fifo, const uint64_t* __restrict__ off,
                            uint64_t n, int C, uint64_t* __restrict__ n_created) {
  pdl_wait();
  const int c = threadIdx.x;
  if (c >= C) return;
  const uint64_t cnt = off[(uint64_t)(c + 1) * n] - off[(uint64_t)c * n];
  if (fifo) *F.tail[c] += cnt;
  if (n_created) n_created[c] = cnt;
}

// A tick's fan-out (n <= kFanKeys affected keys) in ONE launch: one CTA per
// client runs its inserts (every thread issues the bucket loads of its keys
// before walking any chain), then -- after a CTA barrier, so every duplicate
// claim of this client is in -- the created-flag fixup, a block scan of the
// created flags in key order, the FIFO append and the tail update.  The
// multi-kernel chain above (insert -> fixup -> 3-kernel scan -> append ->
// tail) stays for large fan-outs (fresh fills).
constexpr int kFanThreads = 1024;
constexpr int kFanPer = 4;
constexpr uint32_t kFanKeys = kFanThreads * kFanPer;  // 4096 (a 512-key update tick)

__global__ void __launch_bounds__(kFanThreads) k_multi_fan_small(const __grid_constant__ SetViews V,
                                                                 const __grid_constant__ FifoViews F, bool fifo,
                                                                 const int32_t* __restrict__ keys, uint32_t n,
                                                                 const uint64_t* __restrict__ n_dev,
                                                                 uint8_t* __restrict__ created,
                                                                 uint64_t* __restrict__ n_created) {
  pdl_wait();
  __shared__ uint8_t s_cr[kFanKeys];
  __shared__ uint32_t s_warp[kFanThreads / 32];
  __shared__ uint64_t s_tail;
  const int c = blockIdx.x;
  const TableView& T = V.v[c];
  const uint32_t t = threadIdx.x;
  const uint32_t nv = n_dev && *n_dev < n ? (uint32_t)*n_dev : n;
  // ---- inserts: key i = t + k * kFanThreads (coalesced), bucket loads first
  int32_t x[kFanPer], y[kFanPer], z[kFanPer], pos[kFanPer];
  int4 pre[kFanPer];
#pragma unroll
  for (int k = 0; k < kFanPer; ++k) {
    const uint32_t i = t + k * kFanThreads;
    if (i < nv) {
      x[k] = keys[3 * i], y[k] = keys[3 * i + 1], z[k] = keys[3 * i + 2];
      pre[k] = ld_bucket(T.e + bucket_of(T, x[k], y[k], z[k]));
    }
  }
#pragma unroll
  for (int k = 0; k < kFanPer; ++k) {
    const uint32_t i = t + k * kFanThreads;
    if (i < nv) {
      const InsertResult r = insert_key(T, x[k], y[k], z[k], (int32_t)i, &pre[k]);
      s_cr[i] = r.created;
      pos[k] = r.pos;
    } else if (i < n) {
      s_cr[i] = 0;
    }
  }
  __syncthreads();  // all of this client's inserts (and duplicate claims) done
  // ---- created flags to the lowest op index among duplicates, FRESH cleared
#pragma unroll
  for (int k = 0; k < kFanPer; ++k) {
    const uint32_t i = t + k * kFanThreads;
    if (i < nv && s_cr[i]) post_op(T, keys, i, 0 /*VS_OP_INSERT*/, s_cr, pos[k]);
  }
  __syncthreads();
  // ---- exclusive scan of the flags in key order: thread t owns [4t, 4t+4)
  uint32_t own = 0;
#pragma unroll
  for (int k = 0; k < kFanPer; ++k) {
    const uint32_t i = t * kFanPer + k;
    own += i < n ? s_cr[i] : 0u;
  }
  uint32_t incl = own;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, d);
    if ((int)lane_id() >= d) incl += v;
  }
  if (lane_id() == 31) s_warp[t >> 5] = incl;
  if (t == 0) s_tail = fifo ? *F.tail[c] : 0;
  __syncthreads();
  if (t < 32) {
    uint32_t w = s_warp[t];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, w, d);
      if ((int)t >= d) w += v;
    }
    s_warp[t] = w;  // inclusive over warps
  }
  __syncthreads();
  const uint32_t total = s_warp[kFanThreads / 32 - 1];
  uint32_t rank = ((t >> 5) ? s_warp[(t >> 5) - 1] : 0u) + incl - own;
  // ---- FIFO append (deque.append order = affected order) + created flags out
#pragma unroll
  for (int k = 0; k < kFanPer; ++k) {
    const uint32_t i = t * kFanPer + k;
    if (i >= n) break;
    const uint8_t cr = s_cr[i];
    if (created) created[(uint64_t)c * n + i] = cr;
    if (cr && fifo) {
      const uint64_t p = (s_tail + rank) % F.cap[c];
      int32_t* dst = F.keys[c] + 3 * p;
      dst[0] = keys[3 * i];
      dst[1] = keys[3 * i + 1];
      dst[2] = keys[3 * i + 2];
    }
    rank += cr;
  }
  if (t == 0) {
    if (fifo) *F.tail[c] = s_tail + total;
    if (n_created) n_created[c] = total;
    if (total) {
      const uint32_t w = blockIdx.x;  // one live-key counter stripe per client CTA
      atomicAdd((unsigned long long*)&T.ctl->size[(w % kSizeStripes) * kSizeStride], (unsigned long long)total);
    }
  }
}

// ---- One stream-set tick per launch (k_stream_tick): for every client, ONE
// CLUSTER of kTickCtas CTAs (1,024 threads each) runs, back to back,
//   1. the affected dedup of the tick's updated keys (mc_encoding.py:108-115,
//      server.py:304-307: expand x8 in product((0,-1), repeat=3) order,
//      first occurrence wins) in shared memory -- every CTA computes the same
//      list (deterministic), the first CTA of the grid also writes it out;
//   2. the fan-out into its client's set (server.py:314-315): CTA r inserts
//      keys [1024r, 1024r + 1024), one per thread; the created flags are
//      ranked by a block scan plus the lower CTAs' totals (read through
//      distributed shared memory), so the FIFO append is in key order;
//   3. the client's extract_random(max_n) (concurrent_hash.py:382-402,
//      server.py:334-363): the cluster scans kTickCtas contiguous chunks per
//      round from the seeded rotating start, exchanges the chunk counts over
//      DSMEM, writes the first max_n live entries in position order and
//      removes them (spread over the cluster); vacated excess entries go
//      straight back to the free list (only this cluster touches its table,
//      and its inserts are done).
// Three launches and two grid-wide dependencies per tick become one launch.
// The fan-out keys are distinct (they come out of the dedup), so the
// created-flag fixup never resolves a duplicate across CTAs.
// VSB_TICK_PROF (measurement build): globaltimer at the phase boundaries of
// every CTA of k_stream_tick, read back by vs_tick_prof_read
#ifndef VSB_TICK_PROF
#define VSB_TICK_PROF 0
#endif
#if VSB_TICK_PROF
__device__ unsigned long long g_tick_prof[8][256];
#define TICK_MARK(m)                                                              \
  do {                                                                            \
    if (threadIdx.x == 0 && blockIdx.x < 256) {                                   \
      unsigned long long v_;                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v_));                      \
      g_tick_prof[m][blockIdx.x] = v_;                                            \
    }                                                                             \
  } while (0)
#else
#define TICK_MARK(m) \
  do {               \
  } while (0)
#endif

constexpr int kTickThreads = 1024;
constexpr int kTickCtas = 4;
constexpr uint32_t kTickMaxU = 512;
constexpr uint32_t kTickKeys = 8 * kTickMaxU;                 // 4,096 affected keys = kTickCtas x 1,024
constexpr uint32_t kTickSlots = 2 * kTickKeys;                // dedup table, load <= 0.5
constexpr int kTickPer = (int)(kTickKeys / kTickThreads);     // 4 expanded keys per thread in the dedup
constexpr int kTickScanK = 4;                                 // positions per thread per extraction round
constexpr size_t kTickSmem = 12 * (size_t)kTickKeys + 4 * (size_t)kTickSlots;  // 80 KB
static_assert(kTickKeys == (uint32_t)kTickCtas * kTickThreads, "one fan-out key per thread");

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* wsum, uint32_t* total) {
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= (uint32_t)d) incl += y;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = wsum[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= (uint32_t)d) w += y;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  *total = wsum[31];
  const uint32_t r = incl - v + (warp ? wsum[warp - 1] : 0u);
  __syncthreads();  // wsum free for the next scan
  return r;
}

__global__ void __cluster_dims__(kTickCtas, 1, 1) __launch_bounds__(kTickThreads)
    k_stream_tick(const __grid_constant__ SetViews V, const __grid_constant__ FifoViews F,
                  const __grid_constant__ FifoViews S, const int32_t* __restrict__ updated, uint32_t u,
                  uint32_t max_n, int32_t* __restrict__ aff_out, uint64_t* __restrict__ n_aff,
                  uint64_t* __restrict__ n_created, int32_t* __restrict__ keys_out, uint64_t* __restrict__ n_out) {
  pdl_wait();
  TICK_MARK(0);
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ int32_t dsm[];
  int32_t* kx = dsm;  // [kTickKeys] x, then y, then z; later the compacted keys (xyz interleaved)
  int32_t* ky = kx + kTickKeys;
  int32_t* kz = ky + kTickKeys;
  uint32_t* slot = (uint32_t*)(kz + kTickKeys);
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t wcnt[kTickScanK][32];
  __shared__ uint32_t chunk_cnt;  // read by the other CTAs of the cluster
  const int c = blockIdx.x / kTickCtas;
  const uint32_t rank = cluster.block_rank();
  const TableView& T = V.v[c];
  const uint32_t t = threadIdx.x, lane = t & 31u, warp = t >> 5;
  uint32_t total;

  // ---- 1. affected dedup (thread t owns expanded keys [4t, 4t+4): input order)
  const uint32_t m = 8 * u;
  for (uint32_t i = t; i < kTickSlots; i += kTickThreads) slot[i] = 0xFFFFFFFFu;
  int32_t x[kTickPer], y[kTickPer], z[kTickPer];
  uint32_t where[kTickPer];
#pragma unroll
  for (int k = 0; k < kTickPer; ++k) {
    const uint32_t j = t * kTickPer + k;
    if (j < m) {
      const uint32_t i = j >> 3, d = j & 7;
      x[k] = updated[3 * i] - (int32_t)((d >> 2) & 1);
      y[k] = updated[3 * i + 1] - (int32_t)((d >> 1) & 1);
      z[k] = updated[3 * i + 2] - (int32_t)(d & 1);
      kx[j] = x[k], ky[j] = y[k], kz[j] = z[k];
    }
  }
  __syncthreads();
  TICK_MARK(6);  // expanded keys loaded and staged
#pragma unroll
  for (int k = 0; k < kTickPer; ++k) {
    const uint32_t j = t * kTickPer + k;
    if (j >= m) continue;
    uint32_t h = hash_raw(x[k], y[k], z[k]);
    h ^= h >> 16;  // murmur3 finaliser: neighbouring keys share low hash bits
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
    h &= kTickSlots - 1;
    for (;;) {
      const uint32_t old = atomicCAS(&slot[h], 0xFFFFFFFFu, j);
      if (old == 0xFFFFFFFFu) break;
      if (kx[old] == x[k] && ky[old] == y[k] && kz[old] == z[k]) {
        atomicMin(&slot[h], j);
        break;
      }
      h = (h + 1) & (kTickSlots - 1);
    }
    where[k] = h;
  }
  __syncthreads();
  TICK_MARK(7);  // hash probes done
  uint32_t first = 0, cnt = 0;
#pragma unroll
  for (int k = 0; k < kTickPer; ++k) {
    const uint32_t j = t * kTickPer + k;
    if (j < m && slot[where[k]] == j) {
      first |= 1u << k;
      ++cnt;
    }
  }
  uint32_t o = block_exclusive_scan(cnt, wsum, &total);  // (every probe is done: kx.. are free now)
  int32_t* stage = kx;  // compacted affected keys, xyz interleaved
#pragma unroll
  for (int k = 0; k < kTickPer; ++k) {
    if (first & (1u << k)) {
      stage[3 * o] = x[k], stage[3 * o + 1] = y[k], stage[3 * o + 2] = z[k];
      ++o;
    }
  }
  __syncthreads();
  const uint32_t n = total;
  if (blockIdx.x == 0) {
    for (uint32_t i = t; i < 3 * n; i += kTickThreads) aff_out[i] = stage[i];
    if (t == 0 && n_aff) *n_aff = n;
  }

  TICK_MARK(1);  // dedup done
  // ---- 2. fan-out: CTA `rank` inserts key i = 1024 rank + t
  const uint32_t i = rank * kTickThreads + t;
  const uint64_t tail = *F.tail[c];  // read by every CTA before the cluster barrier below
  uint8_t cr = 0;
  if (i < n) {
    const int32_t qx = stage[3 * i], qy = stage[3 * i + 1], qz = stage[3 * i + 2];
    const InsertResult r = insert_key(T, qx, qy, qz, (int32_t)i);
    cr = r.created;
    // created flag of a distinct key: only FRESH to clear (post_op's duplicate
    // resolution cannot trigger)
    if (cr) atomicAnd(&T.e[r.pos].meta, ~kFresh);
  }
  TICK_MARK(2);  // this thread-0's insert done
  uint32_t local_total;
  const uint32_t lrank = block_exclusive_scan(cr, wsum, &local_total);
  if (t == 0) chunk_cnt = local_total;
  cluster.sync();  // chunk totals published; every insert of the cluster done; every tail read
  uint32_t lower = 0, created_total = 0;
  for (uint32_t r = 0; r < (uint32_t)kTickCtas; ++r) {
    const uint32_t v = *cluster.map_shared_rank(&chunk_cnt, r);
    lower += r < rank ? v : 0u;
    created_total += v;
  }
  if (cr) {
    int32_t* dst = F.keys[c] + 3 * ((tail + lower + lrank) % F.cap[c]);
    dst[0] = stage[3 * i], dst[1] = stage[3 * i + 1], dst[2] = stage[3 * i + 2];
  }
  if (rank == 0 && t == 0) {
    *F.tail[c] = tail + created_total;
    if (n_created) n_created[c] = created_total;
  }
  int delta = t == 0 ? (int)local_total : 0;
  cluster.sync();  // chunk_cnt is reused below
  TICK_MARK(3);  // FIFO append done

  // ---- 3. extract_random(max_n): rotating start (k_multi_extract's seed mix)
  const uint32_t cap = T.n + T.excess;
  uint64_t sd = S.cap[c] + 0x9E3779B97F4A7C15ull;
  sd = (sd ^ (sd >> 30)) * 0xBF58476D1CE4E5B9ull;
  sd = (sd ^ (sd >> 27)) * 0x94D049BB133111EBull;
  sd ^= sd >> 31;
  const uint32_t start = (uint32_t)(sd % cap);
  int32_t* out = keys_out + (uint64_t)c * max_n * 3;
  uint64_t found = 0;  // identical in every CTA of the cluster
  constexpr uint64_t kChunk = (uint64_t)kTickThreads * kTickScanK;
  for (uint64_t base = 0; base < cap && found < max_n; base += kChunk * kTickCtas) {
    const uint64_t c0 = base + rank * kChunk;
    int4 e[kTickScanK];
    bool live[kTickScanK];
    uint32_t bal[kTickScanK];
#pragma unroll
    for (int k = 0; k < kTickScanK; ++k) {
      const uint64_t q = c0 + (uint64_t)k * kTickThreads + t;
      uint64_t p = (uint64_t)start + q;
      p = p >= cap ? p - cap : p;
      live[k] = false;
      if (q < cap) {
        e[k] = ld_entry(T.e + p);
        live[k] = ((uint32_t)e[k].w & kOcc) != 0;
      }
    }
#pragma unroll
    for (int k = 0; k < kTickScanK; ++k) {
      bal[k] = __ballot_sync(0xffffffffu, live[k]);
      if (lane == 0) wcnt[k][warp] = __popc(bal[k]);
    }
    __syncthreads();
    if (t == 0) {
      uint32_t a2 = 0;
      for (int k = 0; k < kTickScanK; ++k)
        for (uint32_t w = 0; w < 32; ++w) a2 += wcnt[k][w];
      chunk_cnt = a2;
    }
    cluster.sync();  // every chunk count published
    uint64_t lo = 0, all_chunks = 0;
    for (uint32_t r = 0; r < (uint32_t)kTickCtas; ++r) {
      const uint32_t v = *cluster.map_shared_rank(&chunk_cnt, r);
      lo += r < rank ? v : 0u;
      all_chunks += v;
    }
    uint64_t before = found + lo;
#pragma unroll
    for (int k = 0; k < kTickScanK; ++k) {
      uint32_t lw = 0, all = 0;
      for (uint32_t w = 0; w < 32; ++w) {
        const uint32_t v = wcnt[k][w];
        lw += w < warp ? v : 0u;
        all += v;
      }
      if (live[k]) {
        const uint64_t d = before + lw + __popc(bal[k] & lanemask_lt());
        if (d < max_n) {
          out[3 * d] = e[k].x, out[3 * d + 1] = e[k].y, out[3 * d + 2] = e[k].z;
        }
      }
      before += all;
    }
    found += all_chunks;
    cluster.sync();  // chunk_cnt / wcnt reused by the next round
  }
  const uint64_t mn = found < max_n ? found : max_n;
  __threadfence();
  cluster.sync();  // keys_out complete (written by the whole cluster) before the removals
  TICK_MARK(4);  // extraction scan done
  for (uint64_t j = (uint64_t)rank * kTickThreads + t; j < mn; j += (uint64_t)kTickCtas * kTickThreads) {
    const int32_t p = erase_key(T, out[3 * j], out[3 * j + 1], out[3 * j + 2]);
    if (p >= 0) {
      --delta;
      if (p >= (int32_t)T.n) push_free(T, (uint32_t)p);  // every insert of this table is done
    }
  }
  add_size_cta(T, delta);
  if (rank == 0 && t == 0) n_out[c] = mn;
#if VSB_TICK_PROF
  __syncthreads();
  TICK_MARK(5);  // removals done
#endif
}

// Frustum-AABB visibility of a block (server.py:375-387): every plane
// (nx, ny, nz, d) must satisfy nx*px + ny*py + nz*pz + d >= -margin at the box
// vertex furthest along the normal.  Evaluated in double with explicitly
// rounded operations in the reference's (numpy float64) order, no FMA, so
// the decision is bit-identical to the Python predicate.
struct Frustum {
  double p[6][4];
  double margin;
  double block;
  int enabled;
};

__device__ __forceinline__ bool block_visible(const Frustum& F, int32_t kx, int32_t ky, int32_t kz) {
  const double x0 = __dmul_rn((double)kx, F.block), y0 = __dmul_rn((double)ky, F.block),
               z0 = __dmul_rn((double)kz, F.block);
  const double x1 = __dadd_rn(x0, F.block), y1 = __dadd_rn(y0, F.block), z1 = __dadd_rn(z0, F.block);
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double nx = F.p[k][0], ny = F.p[k][1], nz = F.p[k][2], d = F.p[k][3];
    const double px = nx >= 0.0 ? x1 : x0, py = ny >= 0.0 ? y1 : y0, pz = nz >= 0.0 ? z1 : z0;
    double acc = __dadd_rn(__dmul_rn(nx, px), __dmul_rn(ny, py));
    acc = __dadd_rn(acc, __dmul_rn(nz, pz));
    acc = __dadd_rn(acc, d);
    if (acc < -F.margin) return false;
  }
  return true;
}

// extract_batch / extract_matching(frustum) for several clients in ONE
// launch (concurrent_hash.py:366-402):
// one CTA per client scans live entries in position order from a seeded
// random start (wrapping), keeps the first max_n, and removes them; the
// vacated excess entries go straight back to the free list (no pops run in
// this launch, so the push cannot race a pop).
// extraction CTA shape (one CTA per client set; measured: see DESIGN §4)
#ifndef VSB_EXTRACT_ERASE_AT_SCAN
#define VSB_EXTRACT_ERASE_AT_SCAN 0  // measured: no gain over the write-out-then-erase pass (scripts/extract_ab.sh)
#endif
#ifndef VSB_EXTRACT_THREADS
#define VSB_EXTRACT_THREADS 256
#endif
#ifndef VSB_EXTRACT_K
#define VSB_EXTRACT_K 8
#endif
constexpr int kExtractThreads = VSB_EXTRACT_THREADS;
constexpr int kExtractK = VSB_EXTRACT_K;

// One CLUSTER of kExtractCtas CTAs per client set: a round scans
// kExtractCtas contiguous chunks of kExtractThreads x kExtractK positions
// (CTA r takes chunk r), every CTA ranks its live entries in position order,
// the chunk counts are exchanged through distributed shared memory, and each
// CTA writes its entries at (found so far + counts of the lower chunks +
// own rank) -- the first max_n live entries from the random start, in
// position order, exactly as one CTA scanning alone would take them.  The
// removals are then spread over the whole cluster.
constexpr int kExtractCtas = 8;

__global__ void __cluster_dims__(kExtractCtas, 1, 1) __launch_bounds__(kExtractThreads)
    k_multi_extract(const __grid_constant__ SetViews V, const __grid_constant__ FifoViews S,
                    const __grid_constant__ Frustum F, uint64_t max_n, int32_t* __restrict__ keys_out,
                    uint64_t* __restrict__ n_out) {
  pdl_wait();
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  const int c = blockIdx.x / kExtractCtas;
  const uint32_t rank = cluster.block_rank();
  const TableView& T = V.v[c];
  const uint32_t cap = T.n + T.excess;
  const uint64_t seed = S.cap[c];  // per-client seed rides in the cap slot
  uint64_t x = seed + 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  x ^= x >> 31;
  const uint32_t start = (uint32_t)(x % cap);
  int32_t* out = keys_out + (uint64_t)c * max_n * 3;
  constexpr uint32_t kWarps = kExtractThreads / 32;
  constexpr uint64_t kChunk = (uint64_t)kExtractThreads * kExtractK;
  __shared__ uint32_t wcnt[kExtractK][kWarps];
  __shared__ uint32_t chunk_cnt;  // read by the other CTAs of the cluster
  const uint32_t warp = threadIdx.x >> 5;
  uint64_t found = 0;  // identical in every CTA of the cluster
  int delta = 0;
  for (uint64_t base = 0; base < cap && found < max_n; base += kChunk * kExtractCtas) {
    const uint64_t c0 = base + rank * kChunk;
    int4 e[kExtractK];
    bool live[kExtractK];
    uint32_t pk[kExtractK];
#pragma unroll
    for (int k = 0; k < kExtractK; ++k) {
      const uint64_t q = c0 + (uint64_t)k * kExtractThreads + threadIdx.x;
      uint64_t p = (uint64_t)start + q;
      p = p >= cap ? p - cap : p;
      pk[k] = (uint32_t)p;
      live[k] = false;
      if (q < cap) {
        e[k] = ld_entry(T.e + p);
        live[k] = ((uint32_t)e[k].w & kOcc) != 0;
      }
    }
    uint32_t bal[kExtractK];
#pragma unroll
    for (int k = 0; k < kExtractK; ++k) {
      if (live[k] && F.enabled) live[k] = block_visible(F, e[k].x, e[k].y, e[k].z);
      bal[k] = __ballot_sync(0xffffffffu, live[k]);
      if (lane_id() == 0) wcnt[k][warp] = __popc(bal[k]);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t a = 0;
      for (int k = 0; k < kExtractK; ++k)
        for (uint32_t w = 0; w < kWarps; ++w) a += wcnt[k][w];
      chunk_cnt = a;
    }
    cluster.sync();  // every chunk count published
    uint64_t lower = 0, total = 0;
    for (uint32_t r = 0; r < kExtractCtas; ++r) {
      const uint32_t v = *cluster.map_shared_rank(&chunk_cnt, r);
      lower += r < rank ? v : 0u;
      total += v;
    }
    // ranks inside the chunk: (k, warp, lane) order = position order
    uint64_t o = found + lower;
#pragma unroll
    for (int k = 0; k < kExtractK; ++k) {
      uint32_t before = 0, all = 0;
      for (uint32_t w = 0; w < kWarps; ++w) {
        before += (w < warp) ? wcnt[k][w] : 0u;
        all += wcnt[k][w];
      }
      if (live[k]) {
        const uint64_t d = o + before + __popc(bal[k] & lanemask_lt());
        if (d < max_n) {
          out[3 * d] = e[k].x;
          out[3 * d + 1] = e[k].y;
          out[3 * d + 2] = e[k].z;
#if VSB_EXTRACT_ERASE_AT_SCAN
          // remove it now, from the position the scan found it at: a bucket
          // entry is its own bucket, so an unchanged, non-FRESH bucket word
          // takes the locked fast path with no chain walk; an excess entry
          // re-scans its chain under the lock (snap kLock never matches).
          // Chunks are disjoint, and a removal changes only the victim's
          // OCC and a predecessor's NEXT, so the scan of later positions
          // still sees exactly the live keys it would have seen.
          const uint32_t p = pk[k];
          const bool bucket = p < T.n;
          const uint32_t b = bucket ? p : bucket_of(T, e[k].x, e[k].y, e[k].z);
          const int32_t pos = mutate_locked(T, e[k].x, e[k].y, e[k].z, false, 0, b,
                                            bucket ? (uint32_t)e[k].w : kLock, (int32_t)p).pos;
          if (pos >= 0) {
            --delta;
            if (pos >= (int32_t)T.n) push_free(T, (uint32_t)pos);
          }
#endif
        }
      }
      o += all;
    }
    found += total;
    cluster.sync();  // chunk_cnt / wcnt reused by the next round
  }
  const uint64_t m = found < max_n ? found : max_n;
#if !VSB_EXTRACT_ERASE_AT_SCAN
  // keys_out complete (written by the whole cluster) before the removals
  __threadfence();
  cluster.sync();
  for (uint64_t j = rank * kExtractThreads + threadIdx.x; j < m; j += (uint64_t)kExtractCtas * kExtractThreads) {
    const int32_t pos = erase_key(T, out[3 * j], out[3 * j + 1], out[3 * j + 2]);
    if (pos >= 0) {
      --delta;
      if (pos >= (int32_t)T.n) push_free(T, (uint32_t)pos);
    }
  }
#endif
  add_size_cta(T, delta);
  if (rank == 0 && threadIdx.x == 0) n_out[c] = m;
}

__global__ void __launch_bounds__(256) k_multi_erase(const __grid_constant__ SetViews V,
                                                     const int32_t* __restrict__ keys, uint64_t n,
                                                     uint8_t* __restrict__ erased, int32_t* __restrict__ vacated) {
  const int c = blockIdx.y;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const TableView& T = V.v[c];
  int delta = 0;
  if (i < n) {
    const int32_t pos = erase_key(T, keys[3 * i], keys[3 * i + 1], keys[3 * i + 2]);
    if (erased) erased[(uint64_t)c * n + i] = pos >= 0;
    vacated[(uint64_t)c * n + i] = pos;
    delta = -(pos >= 0);
  }
  add_size_cta(T, delta);
}

__global__ void k_multi_recycle(const __grid_constant__ SetViews V, const int32_t* __restrict__ vacated, uint64_t n) {
  const int c = blockIdx.y;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const TableView& T = V.v[c];
  const int32_t e = vacated[(uint64_t)c * n + i];
  if (e >= (int32_t)T.n) push_free(T, (uint32_t)e);
}

// affected_mc_blocks order: itertools.product((0, -1), repeat=3) -> dx slowest
__global__ void k_expand_affected(const int32_t* __restrict__ updated, uint64_t u, int32_t* __restrict__ out) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= 8 * u) return;
  const uint64_t i = j >> 3;
  const int d = (int)(j & 7);
  out[3 * j] = updated[3 * i] - ((d >> 2) & 1);
  out[3 * j + 1] = updated[3 * i + 1] - ((d >> 1) & 1);
  out[3 * j + 2] = updated[3 * i + 2] - (d & 1);
}

// Small batches (the per-tick case: u <= 1024 updated keys, m = 8u <= 8192
// affected keys) are deduplicated by ONE CTA in shared memory: the expanded
// keys, then an open-addressing table of key indices where each slot keeps
// the LOWEST index of its key (CAS to claim, atomicMin on a key match), then
// a block scan of the first-occurrence flags in input order.  One launch and
// no scratch allocations instead of the table path's ~20 API calls.
constexpr int kDedupThreads = 1024;
constexpr int kDedupPer = 8;                                 // keys per thread
constexpr uint32_t kDedupMax = kDedupThreads * kDedupPer;    // 8192 keys
constexpr uint32_t kDedupSlots = 2 * kDedupMax;              // load <= 0.5
constexpr size_t kDedupSmem = 12 * (size_t)kDedupMax + 4 * (size_t)kDedupSlots;

__global__ void __launch_bounds__(kDedupThreads) k_dedup_small(const int32_t* __restrict__ updated, uint32_t u,
                                                               int32_t* __restrict__ out, uint64_t* __restrict__ n_dev) {
  pdl_wait();
  extern __shared__ int32_t dsm[];
  int32_t* kx = dsm;                                   // [kDedupMax] x, then y, then z
  int32_t* ky = kx + kDedupMax;
  int32_t* kz = ky + kDedupMax;
  uint32_t* slot = (uint32_t*)(kz + kDedupMax);        // [kDedupSlots] lowest key index or ~0
  __shared__ uint32_t wsum[kDedupThreads / 32];
  const uint32_t m = 8 * u, t = threadIdx.x;
  for (uint32_t i = t; i < kDedupSlots; i += kDedupThreads) slot[i] = 0xFFFFFFFFu;
  // contiguous ownership: thread t holds keys [t*8, t*8+8), so the scan below
  // runs in input order; expansion order = affected_mc_blocks (dx slowest)
  // `per` keys per thread (<= kDedupPer) so every thread of the CTA works
  const uint32_t per = (m + kDedupThreads - 1) / kDedupThreads;
  int32_t x[kDedupPer], y[kDedupPer], z[kDedupPer];
  uint32_t where[kDedupPer];
#pragma unroll
  for (int k = 0; k < kDedupPer; ++k) {
    const uint32_t j = t * per + k;
    if ((uint32_t)k < per && j < m) {
      const uint32_t i = j >> 3, d = j & 7;
      x[k] = updated[3 * i] - (int32_t)((d >> 2) & 1);
      y[k] = updated[3 * i + 1] - (int32_t)((d >> 1) & 1);
      z[k] = updated[3 * i + 2] - (int32_t)(d & 1);
      kx[j] = x[k];
      ky[j] = y[k];
      kz[j] = z[k];
    }
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kDedupPer; ++k) {
    const uint32_t j = t * per + k;
    if ((uint32_t)k >= per || j >= m) continue;
    uint32_t h = hash_raw(x[k], y[k], z[k]);
#if VSB_DEDUP_MIX
    // neighbouring keys share low hash bits; mix before masking so linear
    // probing does not cluster (murmur3 finaliser)
    h ^= h >> 16;
    h *= 0x85ebca6bu;
    h ^= h >> 13;
    h *= 0xc2b2ae35u;
    h ^= h >> 16;
#endif
    h &= kDedupSlots - 1;
    for (;;) {
      const uint32_t old = atomicCAS(&slot[h], 0xFFFFFFFFu, j);
      if (old == 0xFFFFFFFFu) break;
      if (kx[old] == x[k] && ky[old] == y[k] && kz[old] == z[k]) {
        atomicMin(&slot[h], j);
        break;
      }
      h = (h + 1) & (kDedupSlots - 1);
    }
    where[k] = h;
  }
  __syncthreads();
  uint32_t first = 0, cnt = 0;
#pragma unroll
  for (int k = 0; k < kDedupPer; ++k) {
    const uint32_t j = t * per + k;
    if ((uint32_t)k < per && j < m && slot[where[k]] == j) {
      first |= 1u << k;
      ++cnt;
    }
  }
  // block-wide exclusive scan of the per-thread counts
  const uint32_t lane = t & 31, warp = t >> 5;
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += v;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= (uint32_t)o) w += v;
    }
    wsum[lane] = w;  // inclusive over warps
  }
  __syncthreads();
  uint32_t o = incl - cnt + (warp ? wsum[warp - 1] : 0u);
  // stage the compacted keys in shared memory (the key arrays are free now:
  // every probe is done) and leave with coalesced stores -- scattered 12-B
  // stores from ONE SM were two thirds of the kernel's time
  int32_t* stage = kx;  // 3 * kDedupMax words span kx, ky, kz
#pragma unroll
  for (int k = 0; k < kDedupPer; ++k) {
    if (first & (1u << k)) {
      stage[3 * o] = x[k];
      stage[3 * o + 1] = y[k];
      stage[3 * o + 2] = z[k];
      ++o;
    }
  }
  __syncthreads();
  const uint32_t total = wsum[31];
  for (uint32_t i = t; i < 3 * total; i += kDedupThreads) out[i] = stage[i];
  if (t == 0) *n_dev = total;
}

__global__ void k_scatter_flagged(const int32_t* __restrict__ keys, uint64_t n, const uint8_t* __restrict__ flag,
                                  const uint64_t* __restrict__ off, int32_t* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  const uint64_t o = off[i];
  out[3 * o] = keys[3 * i];
  out[3 * o + 1] = keys[3 * i + 1];
  out[3 * o + 2] = keys[3 * i + 2];
}

__global__ void k_copy_u64(const uint64_t* __restrict__ src, uint64_t* __restrict__ dst) { *dst = *src; }

__global__ void k_gather_ring(const int32_t* __restrict__ ring, uint64_t cap, uint64_t head, uint64_t w,
                              int32_t* __restrict__ out) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= w) return;
  const uint64_t p = (head + j) % cap;
  out[3 * j] = ring[3 * p];
  out[3 * j + 1] = ring[3 * p + 1];
  out[3 * j + 2] = ring[3 * p + 2];
}

__global__ void k_candidates(const uint8_t* __restrict__ first, const uint8_t* __restrict__ present, uint64_t w,
                             uint8_t* __restrict__ cand) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < w) cand[j] = first[j] & present[j];
}

// position of the need-th candidate (1-based) -> *cut
__global__ void k_find_cut(const uint8_t* __restrict__ cand, const uint64_t* __restrict__ off, uint64_t w,
                           uint64_t need, uint64_t* __restrict__ cut) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < w && cand[j] && off[j] + 1 == need) *cut = j;
}

__global__ void k_clip_flags(uint8_t* __restrict__ flag, uint64_t w, uint64_t cut) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < w && j > cut) flag[j] = 0;
}

static vs_status fill_views(vs_table* const* sets, int n_sets, SetViews& V) {
  if (n_sets < 1 || n_sets > kMaxSets) {
    set_error("n_sets must be in [1, 32] per call");
    return VS_ERR_INVALID;
  }
  for (int c = 0; c < n_sets; ++c) {
    if (!sets[c]) {
      set_error("set handle is NULL");
      return VS_ERR_INVALID;
    }
    V.v[c] = sets[c]->next_view();
  }
  return VS_OK;
}

}  // namespace vsb

using namespace vsb;

extern "C" {

vs_status vs_affected_dedup(vs_table* scratch, const int32_t* updated, uint64_t u, int32_t* out_keys,
                            uint64_t* n_dev, vs_stream_t stream) {
  if (!scratch || !n_dev || (u && (!updated || !out_keys))) {
    set_error("scratch/updated/out_keys/n_dev must be non-NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(scratch->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (u == 0) {
    VS_CK(cudaMemsetAsync(n_dev, 0, 8, s));
    return VS_OK;
  }
  const uint64_t m = 8 * u;
  if (m <= kDedupMax) {
    static bool attr_set[64] = {};  // the opt-in is per device
    const int d = scratch->device;
    if (d < 0 || d >= 64 || !attr_set[d]) {
      VS_CK(cudaFuncSetAttribute(k_dedup_small, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kDedupSmem));
      if (d >= 0 && d < 64) attr_set[d] = true;
    }
    { VS_CK(launch_pdl(k_dedup_small, 1, kDedupThreads, kDedupSmem, s, updated, (uint32_t)u, out_keys, n_dev)); vsb::count_launch(); }
    VS_CK_LAUNCH("vs_affected_dedup");
    return VS_OK;
  }
  int32_t* all = nullptr;
  uint8_t* created = nullptr;
  int32_t* index = nullptr;
  uint64_t *off = nullptr, *work = nullptr;
  VS_CK(cudaMallocAsync((void**)&all, 12 * m, s));
  VS_CK(cudaMallocAsync((void**)&created, m, s));
  VS_CK(cudaMallocAsync((void**)&index, 4 * m, s));
  VS_CK(cudaMallocAsync((void**)&off, 8 * (m + 1), s));
  VS_CK(cudaMallocAsync((void**)&work, 8 * (scan_tiles(m) + 1), s));
  vs_status st = vs_table_clear(scratch, stream);
  if (st == VS_OK) {
    { k_expand_affected<<<grid_for(m, 256), 256, 0, s>>>(updated, u, all); vsb::count_launch(); }
    st = vs_table_insert(scratch, all, m, created, index, stream);
  }
  if (st == VS_OK) {
    cudaError_t e = exclusive_scan<uint8_t>(created, m, off, work, s);
    if (e != cudaSuccess) st = cuda_status(e, "exclusive_scan");
  }
  if (st == VS_OK) {
    { k_scatter_flagged<<<grid_for(m, 256), 256, 0, s>>>(all, m, created, off, out_keys); vsb::count_launch(); }
    { k_copy_u64<<<1, 1, 0, s>>>(off + m, n_dev); vsb::count_launch(); }
  }
  cudaFreeAsync(all, s);
  cudaFreeAsync(created, s);
  cudaFreeAsync(index, s);
  cudaFreeAsync(off, s);
  cudaFreeAsync(work, s);
  if (st != VS_OK) return st;
  VS_CK_LAUNCH("vs_affected_dedup");
  return VS_OK;
}

vs_status vs_stream_insert_many(vs_table* const* sets_host, int n_sets, const int32_t* keys, uint64_t n,
                                const uint64_t* n_dev, uint8_t* created, int32_t* const* fifo_keys_host,
                                const uint64_t* fifo_cap_host,
                                uint64_t* const* fifo_tail_host, uint64_t* n_created, vs_stream_t stream) {
  SetViews V;
  if (!sets_host) {
    set_error("sets is NULL");
    return VS_ERR_INVALID;
  }
  vs_status st = fill_views(sets_host, n_sets, V);
  if (st != VS_OK) return st;
  if (n >= (1ull << 31)) {
    set_error("batch too large");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(sets_host[0]->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    if (n_created) VS_CK(cudaMemsetAsync(n_created, 0, 8 * n_sets, s));
    return VS_OK;
  }
  if (!keys || !created) {
    set_error("keys/created must be non-NULL");
    return VS_ERR_INVALID;
  }
  const bool fifo = fifo_keys_host && fifo_cap_host && fifo_tail_host;
  FifoViews F{};
  if (fifo) {
    for (int c = 0; c < n_sets; ++c) {
      F.keys[c] = fifo_keys_host[c];
      F.cap[c] = fifo_cap_host[c] ? fifo_cap_host[c] : 1;
      F.tail[c] = fifo_tail_host[c];
    }
  }
  if (n <= kFanKeys && VSB_FAN_SMALL) {  // a tick: one launch, no scratch
    { VS_CK(launch_pdl(k_multi_fan_small, n_sets, kFanThreads, 0, s, V, F, fifo, keys, (uint32_t)n, n_dev, created,
                       n_created)); vsb::count_launch(); }
    VS_CK_LAUNCH("vs_stream_insert_many");
    return VS_OK;
  }
  const uint64_t total = (uint64_t)n_sets * n;
  // one stream-ordered allocation carved into the three scratch arrays
  const size_t b_index = (4 * total + 255) & ~(size_t)255, b_off = (8 * (total + 1) + 255) & ~(size_t)255;
  char* scratch_mem = nullptr;
  VS_CK(cudaMallocAsync((void**)&scratch_mem, b_index + b_off + 8 * (scan_tiles(total) + 1), s));
  int32_t* index = (int32_t*)scratch_mem;
  uint64_t* off = (uint64_t*)(scratch_mem + b_index);
  uint64_t* work = (uint64_t*)(scratch_mem + b_index + b_off);
  const dim3 grid(grid_for(n, 256), n_sets);
  // (no ProfScope here: its events would sit between the PDL-linked kernels)
  { VS_CK(launch_pdl(k_multi_insert, grid, 256, 0, s, V, keys, n, n_dev, created, index)); vsb::count_launch(); }
  { VS_CK(launch_pdl(k_multi_fixup, grid, 256, 0, s, V, keys, n, created, index)); vsb::count_launch(); }
  cudaError_t e = exclusive_scan<uint8_t>(created, total, off, work, s);
  if (e == cudaSuccess && fifo) { e = launch_pdl(k_fifo_append, grid, 256, 0, s, F, keys, n, created, off); vsb::count_launch(); }
  if (e == cudaSuccess) { e = launch_pdl(k_fifo_tail, 1, 32, 0, s, F, fifo, off, n, n_sets, n_created); vsb::count_launch(); }
  cudaFreeAsync(scratch_mem, s);
  if (e != cudaSuccess) return cuda_status(e, "vs_stream_insert_many");
  VS_CK_LAUNCH("vs_stream_insert_many");
  return VS_OK;
}

static vs_status multi_extract(vs_table* const* sets_host, int n_sets, uint64_t max_n, const uint64_t* seeds_host,
                               const Frustum& F, int32_t* keys_out, uint64_t* n_out, vs_stream_t stream) {
  SetViews V;
  if (!sets_host || !seeds_host || !n_out || (max_n && !keys_out)) {
    set_error("sets/seeds/keys_out/n_out must be non-NULL");
    return VS_ERR_INVALID;
  }
  vs_status st = fill_views(sets_host, n_sets, V);
  if (st != VS_OK) return st;
  DeviceGuard g(sets_host[0]->device);
  cudaStream_t s = (cudaStream_t)stream;
  FifoViews S{};
  for (int c = 0; c < n_sets; ++c) S.cap[c] = seeds_host[c];
  { VS_CK(launch_pdl(k_multi_extract, n_sets * kExtractCtas, kExtractThreads, 0, s, V, S, F, max_n, keys_out, n_out)); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_stream_extract");
  return VS_OK;
}

// TSDF ingest (server.py:300-303: tsdf_map.put(key, TsdfBlock.from_bytes(raw))
// per block, latest write wins): after the batched insert, the LAST op per
// position wins the claim word (epoch-tagged atomicMin of ~op), then the
// winners copy their 6,144-byte wire rows into the pool (one warp per row,
// 16-byte vector copies).

__global__ void k_put_rows(TableView T, const int32_t* __restrict__ pos, uint64_t n, const uint4* __restrict__ rows,
                           uint4* __restrict__ pool, uint8_t* __restrict__ faces) {
  const uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;
  const int32_t p = pos[i];
  if (p < 0) return;
  // the insert before this launch ran without a post pass: settle FRESH
  if (lane == 0) atomicAnd(&T.e[p].meta, ~kFresh);
  if (T.claim[p] != (T.tag | (unsigned long long)(0xFFFFFFFFu - (uint32_t)i))) return;
  const uint4* src = rows + i * (VS_TSDF_BLOCK_BYTES / 16);
  uint4* dst = pool + (uint64_t)p * (VS_TSDF_BLOCK_BYTES / 16);
#pragma unroll 4
  for (int j = lane; j < VS_TSDF_BLOCK_BYTES / 16; j += 32) dst[j] = __ldcs(src + j);
  // the encoder's halo side table for this row, from the same source bytes
  if (faces) face_pack_warp((const uint8_t*)src, faces + (uint64_t)p * kFaceBytes);
}

// MC_BATCH payload (wire.py:292-299): u32 count, then per block the key as
// <3i and its 2,048 MC bytes, gathered straight from the device MC pool.
__global__ void k_mc_pack(const int32_t* __restrict__ keys, const int32_t* __restrict__ pos, uint64_t n,
                          const uint32_t* __restrict__ pool, uint32_t* __restrict__ out) {
  const uint64_t r = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (r == 0 && lane == 0 && blockIdx.x == 0) out[0] = (uint32_t)n;
  if (r >= n) return;
  uint32_t* dst = out + 1 + r * (VS_MC_BLOCK_BYTES + 12) / 4;
  if (lane < 3) dst[lane] = (uint32_t)keys[3 * r + lane];
  const uint32_t* src = pool + (uint64_t)pos[r] * (VS_MC_BLOCK_BYTES / 4);
#pragma unroll 4
  for (int j = lane; j < VS_MC_BLOCK_BYTES / 4; j += 32) dst[3 + j] = __ldcs(src + j);
}


vs_status vs_stream_tick(vs_table* const* sets_host, int n_sets, const int32_t* updated, uint64_t u,
                         int32_t* const* fifo_keys_host, const uint64_t* fifo_cap_host,
                         uint64_t* const* fifo_tail_host, uint64_t max_extract, const uint64_t* seeds_host,
                         int32_t* affected_out, uint64_t* n_affected, uint64_t* n_created, int32_t* keys_out,
                         uint64_t* n_out, vs_stream_t stream) {
  SetViews V;
  if (!sets_host || !updated || !fifo_keys_host || !fifo_cap_host || !fifo_tail_host || !seeds_host || !affected_out ||
      !n_affected || !n_out || (max_extract && !keys_out)) {
    set_error("vs_stream_tick: sets/updated/fifos/seeds/affected_out/n_affected/n_out must be non-NULL");
    return VS_ERR_INVALID;
  }
  if (u < 1 || u > kTickMaxU || max_extract > 0xFFFFFFFFull) {
    set_error("vs_stream_tick: 1 <= u <= 512 updated keys per tick (larger updates: the separate calls)");
    return VS_ERR_INVALID;
  }
  vs_status st = fill_views(sets_host, n_sets, V);
  if (st != VS_OK) return st;
  DeviceGuard g(sets_host[0]->device);
  cudaStream_t s = (cudaStream_t)stream;
  FifoViews F{}, S{};
  for (int c = 0; c < n_sets; ++c) {
    F.keys[c] = fifo_keys_host[c];
    F.cap[c] = fifo_cap_host[c] ? fifo_cap_host[c] : 1;
    F.tail[c] = fifo_tail_host[c];
    S.cap[c] = seeds_host[c];
  }
  static bool attr_set[64] = {};  // the shared-memory opt-in is per device
  const int d = sets_host[0]->device;
  if (d < 0 || d >= 64 || !attr_set[d]) {
    VS_CK(cudaFuncSetAttribute(k_stream_tick, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kTickSmem));
    if (d >= 0 && d < 64) attr_set[d] = true;
  }
  { VS_CK(launch_pdl(k_stream_tick, n_sets * kTickCtas, kTickThreads, kTickSmem, s, V, F, S, updated, (uint32_t)u,
                     (uint32_t)max_extract, affected_out, n_affected, n_created, keys_out, n_out)); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_stream_tick");
  return VS_OK;
}

vs_status vs_stream_extract_random(vs_table* const* sets_host, int n_sets, uint64_t max_n,
                                   const uint64_t* seeds_host, int32_t* keys_out, uint64_t* n_out,
                                   vs_stream_t stream) {
  Frustum F{};
  return multi_extract(sets_host, n_sets, max_n, seeds_host, F, keys_out, n_out, stream);
}

vs_status vs_stream_extract_visible(vs_table* const* sets_host, int n_sets, uint64_t max_n,
                                    const uint64_t* seeds_host, const double* planes_host, double margin,
                                    double block_size, int32_t* keys_out, uint64_t* n_out, vs_stream_t stream) {
  if (!planes_host) {
    set_error("planes must be non-NULL");
    return VS_ERR_INVALID;
  }
  Frustum F{};
  for (int k = 0; k < 24; ++k) F.p[k / 4][k % 4] = planes_host[k];
  F.margin = margin;
  F.block = block_size;
  F.enabled = 1;
  return multi_extract(sets_host, n_sets, max_n, seeds_host, F, keys_out, n_out, stream);
}

static vs_status tsdf_put(vs_table* t, const int32_t* keys, const uint8_t* rows, uint64_t n, uint8_t* pool,
                          int32_t* index, uint8_t* faces, vs_stream_t stream, uint8_t* created_scratch = nullptr);

vs_status vs_tsdf_put(vs_table* t, const int32_t* keys, const uint8_t* rows, uint64_t n, uint8_t* pool,
                      int32_t* index, vs_stream_t stream) {
  return tsdf_put(t, keys, rows, n, pool, index, nullptr, stream);
}

// created_scratch (optional, n bytes): the insert's created flags go there
// instead of a stream-ordered allocation
static vs_status tsdf_put(vs_table* t, const int32_t* keys, const uint8_t* rows, uint64_t n, uint8_t* pool,
                          int32_t* index, uint8_t* faces, vs_stream_t stream, uint8_t* created_scratch) {
  if (!t || !index || (n && (!keys || !rows || !pool))) {
    set_error("table/keys/rows/pool/index must be non-NULL");
    return VS_ERR_INVALID;
  }
  if (((uintptr_t)rows & 15u) || ((uintptr_t)pool & 15u)) {
    set_error("rows and pool must be 16-byte aligned");
    return VS_ERR_INVALID;
  }
  if (n == 0) return VS_OK;
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* created = created_scratch;
  if (!created) VS_CK(cudaMallocAsync((void**)&created, n, s));
  // ONE insert launch that also claims each position for the latest write
  // (no created resolution: a put has no created flag), then the row copy,
  // which settles FRESH (the insert's post pass); capacity failures stay sticky
  TableView v;
  vs_status st = table_put_insert(t, keys, n, created, index, s, &v);
  if (!created_scratch) cudaFreeAsync(created, s);
  if (st != VS_OK) return st;
  { k_put_rows<<<grid_for(32 * n, 256), 256, 0, s>>>(v, index, n, (const uint4*)rows, (uint4*)pool, faces); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_tsdf_put");
  return VS_OK;
}

vs_status vs_mc_pack(const int32_t* keys, const int32_t* pos, uint64_t n, const uint8_t* mc_pool, uint8_t* out,
                     vs_stream_t stream) {
  if (!out || (n && (!keys || !pos || !mc_pool))) {
    set_error("keys/pos/mc_pool/out must be non-NULL");
    return VS_ERR_INVALID;
  }
  if (((uintptr_t)out & 3u) || ((uintptr_t)mc_pool & 3u)) {
    set_error("out and mc_pool must be 4-byte aligned");
    return VS_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  { k_mc_pack<<<grid_for(32 * (n ? n : 1), 256), 256, 0, s>>>(keys, pos, n, (const uint32_t*)mc_pool, (uint32_t*)out); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_mc_pack");
  return VS_OK;
}

vs_status vs_stream_remove_many(vs_table* const* sets_host, int n_sets, const int32_t* keys, uint64_t n,
                                uint8_t* erased, vs_stream_t stream) {
  SetViews V;
  if (!sets_host) {
    set_error("sets is NULL");
    return VS_ERR_INVALID;
  }
  vs_status st = fill_views(sets_host, n_sets, V);
  if (st != VS_OK) return st;
  if (n == 0) return VS_OK;
  if (!keys) {
    set_error("keys must be non-NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(sets_host[0]->device);
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* vacated = nullptr;
  VS_CK(cudaMallocAsync((void**)&vacated, sizeof(int32_t) * n * (uint64_t)n_sets, s));
  const dim3 grid(grid_for(n, 256), n_sets);
  { k_multi_erase<<<grid, 256, 0, s>>>(V, keys, n, erased, vacated); vsb::count_launch(); }
  { k_multi_recycle<<<grid, 256, 0, s>>>(V, vacated, n); vsb::count_launch(); }
  cudaFreeAsync(vacated, s);
  VS_CK_LAUNCH("vs_stream_remove_many");
  return VS_OK;
}

vs_status vs_stream_extract_ordered(vs_table* set, const int32_t* fifo_keys, uint64_t fifo_cap, uint64_t* head_host,
                                    uint64_t tail_host, uint64_t max_n, int32_t* keys_out, uint64_t* n_out_host,
                                    vs_table* scratch, vs_stream_t stream) {
  if (!set || !scratch || !head_host || !n_out_host || (max_n && (!fifo_keys || !keys_out))) {
    set_error("set/scratch/fifo/head/keys_out/n_out must be non-NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(set->device);
  cudaStream_t s = (cudaStream_t)stream;
  uint64_t head = *head_host, out = 0;
  *n_out_host = 0;
  if (max_n == 0 || head >= tail_host) return VS_OK;
  // window buffers sized to the scratch table (the dedup set of a window)
  const uint64_t wmax = std::max<uint64_t>(1, std::min<uint64_t>(scratch->n, 1u << 20));
  int32_t* wkeys = nullptr;
  uint8_t *first = nullptr, *present = nullptr, *cand = nullptr;
  int32_t* idx = nullptr;
  uint64_t *off = nullptr, *work = nullptr, *cut_dev = nullptr;
  VS_CK(cudaMallocAsync((void**)&wkeys, 12 * wmax, s));
  VS_CK(cudaMallocAsync((void**)&first, wmax, s));
  VS_CK(cudaMallocAsync((void**)&present, wmax, s));
  VS_CK(cudaMallocAsync((void**)&cand, wmax, s));
  VS_CK(cudaMallocAsync((void**)&idx, 4 * wmax, s));
  VS_CK(cudaMallocAsync((void**)&off, 8 * (wmax + 1), s));
  VS_CK(cudaMallocAsync((void**)&work, 8 * (scan_tiles(wmax) + 1), s));
  VS_CK(cudaMallocAsync((void**)&cut_dev, 8, s));
  vs_status st = VS_OK;
  while (st == VS_OK && out < max_n && head < tail_host) {
    const uint64_t need = max_n - out;
    uint64_t w = std::min<uint64_t>(tail_host - head, std::max<uint64_t>(need, 1024));
    w = std::min(w, wmax);
    { k_gather_ring<<<grid_for(w, 256), 256, 0, s>>>(fifo_keys, fifo_cap, head, w, wkeys); vsb::count_launch(); }
    // first occurrence inside the window (later duplicates are stale by
    // construction: the earlier entry either delivers the key or finds it gone)
    st = vs_table_clear(scratch, stream);
    if (st == VS_OK) st = vs_table_insert(scratch, wkeys, w, first, idx, stream);
    if (st == VS_OK) st = vs_table_find(set, wkeys, w, present, idx, stream);
    if (st != VS_OK) break;
    { k_candidates<<<grid_for(w, 256), 256, 0, s>>>(first, present, w, cand); vsb::count_launch(); }
    cudaError_t e = exclusive_scan<uint8_t>(cand, w, off, work, s);
    if (e != cudaSuccess) {
      st = cuda_status(e, "exclusive_scan");
      break;
    }
    uint64_t total = 0;
    if ((e = cudaMemcpyAsync(&total, off + w, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
        (e = cudaStreamSynchronize(s)) != cudaSuccess) {
      st = cuda_status(e, "extract_ordered: total");
      break;
    }
    uint64_t cut = w - 1, taken = total;
    if (total >= need) {
      { k_find_cut<<<grid_for(w, 256), 256, 0, s>>>(cand, off, w, need, cut_dev); vsb::count_launch(); }
      if ((e = cudaMemcpyAsync(&cut, cut_dev, 8, cudaMemcpyDeviceToHost, s)) != cudaSuccess ||
          (e = cudaStreamSynchronize(s)) != cudaSuccess) {
        st = cuda_status(e, "extract_ordered: cut");
        break;
      }
      taken = need;
      { k_clip_flags<<<grid_for(w, 256), 256, 0, s>>>(cand, w, cut); vsb::count_launch(); }
    }
    { k_scatter_flagged<<<grid_for(w, 256), 256, 0, s>>>(wkeys, w, cand, off, keys_out + 3 * out); vsb::count_launch(); }
    if (taken) st = vs_table_erase(set, keys_out + 3 * out, taken, nullptr, nullptr, stream);
    out += taken;
    head += cut + 1;
  }
  cudaFreeAsync(wkeys, s);
  cudaFreeAsync(first, s);
  cudaFreeAsync(present, s);
  cudaFreeAsync(cand, s);
  cudaFreeAsync(idx, s);
  cudaFreeAsync(off, s);
  cudaFreeAsync(work, s);
  cudaFreeAsync(cut_dev, s);
  cudaError_t e = cudaStreamSynchronize(s);
  if (st == VS_OK && e != cudaSuccess) st = cuda_status(e, "extract_ordered");
  *head_host = head;
  *n_out_host = out;
  return st;
}

// GpuServerCore.on_tsdf_batch (server.py:299-315) without host
// synchronisation, in ONE host call: the library issues the whole chain
// (TSDF put with latest-write-wins rows, face packs of the written rows,
// affected dedup, mc_map put, recompute into the MC / quantised pools at the
// MC map positions, fan-out into every client set) on one stream -- the
// per-call host work of the Python path was the tick's critical path.
vs_status vs_server_tick(vs_table* tsdf_map, vs_table* mc_map, vs_table* dedup_scratch, const int32_t* keys,
                         const uint8_t* rows, uint64_t u, uint8_t* tsdf_pool, uint8_t* tsdf_faces, uint8_t* mc_pool,
                         int8_t* q_pool, vs_table* const* sets_host, int n_sets, int32_t* const* fifo_keys_host,
                         const uint64_t* fifo_cap_host, uint64_t* const* fifo_tail_host, int32_t* affected_out,
                         uint64_t* n_affected, vs_stream_t stream) {
  if (!tsdf_map || !mc_map || !dedup_scratch || !affected_out || !n_affected || n_sets < 0 ||
      (n_sets > 0 && (!sets_host || !fifo_keys_host || !fifo_cap_host || !fifo_tail_host))) {
    set_error("vs_server_tick: maps/scratch/affected_out/n_affected (and the client arrays) must be non-NULL");
    return VS_ERR_INVALID;
  }
  if (u == 0) {
    cudaStream_t s = (cudaStream_t)stream;
    VS_CK(cudaMemsetAsync(n_affected, 0, 8, s));
    return VS_OK;
  }
  DeviceGuard g(tsdf_map->device);
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t m = 8 * u;
  // scratch: TSDF positions [u], MC positions [8u], created flags of the MC put [8u]
  // and of the fan-out [32 x 8u]
  const uint64_t cfan = (uint64_t)(n_sets > kMaxSets ? kMaxSets : n_sets) * m;
  const size_t b_pos = (4 * u + 255) & ~(size_t)255, b_mpos = (4 * m + 255) & ~(size_t)255,
               b_cr = (m + 255) & ~(size_t)255, b_tcr = (u + 255) & ~(size_t)255;
  const size_t need = b_pos + b_mpos + b_cr + b_tcr + (cfan ? cfan : 1);
  if (tsdf_map->tick_mem_bytes < need) {  // grow-only scratch kept on the map (stream-ordered reuse)
    if (tsdf_map->tick_mem) VS_CK(cudaFreeAsync(tsdf_map->tick_mem, s));
    tsdf_map->tick_mem = nullptr;
    tsdf_map->tick_mem_bytes = 0;
    VS_CK(cudaMallocAsync((void**)&tsdf_map->tick_mem, need, s));
    tsdf_map->tick_mem_bytes = need;
  }
  char* mem = tsdf_map->tick_mem;
  int32_t* pos = (int32_t*)mem;
  int32_t* mpos = (int32_t*)(mem + b_pos);
  uint8_t* cr = (uint8_t*)(mem + b_pos + b_mpos);
  uint8_t* tcr = (uint8_t*)(mem + b_pos + b_mpos + b_cr);
  uint8_t* cr_fan = (uint8_t*)(mem + b_pos + b_mpos + b_cr + b_tcr);
  // Two independent chains, on two streams: the TSDF put (+ face packs) on
  // `stream`, the affected dedup + MC map put (they need only the keys) on
  // a side stream; they join before the encode, which needs both.
  if (!tsdf_map->side) {
    VS_CK(cudaStreamCreateWithFlags(&tsdf_map->side, cudaStreamNonBlocking));
    VS_CK(cudaEventCreateWithFlags(&tsdf_map->ev_fork, cudaEventDisableTiming));
    VS_CK(cudaEventCreateWithFlags(&tsdf_map->ev_join, cudaEventDisableTiming));
  }
  cudaStream_t side = tsdf_map->side;
  VS_CK(cudaEventRecord(tsdf_map->ev_fork, s));
  VS_CK(cudaStreamWaitEvent(side, tsdf_map->ev_fork, 0));
  vs_status st = vs_affected_dedup(dedup_scratch, keys, u, affected_out, n_affected, (vs_stream_t)side);
  // mc_map.put positions; FRESH on the created entries is settled by the encode below
  if (st == VS_OK) st = table_insert_fresh(mc_map, affected_out, m, n_affected, cr, mpos, side);
  if (st == VS_OK) st = tsdf_put(tsdf_map, keys, rows, u, tsdf_pool, pos, tsdf_faces, stream, tcr);  // + face packs
  VS_CK(cudaEventRecord(tsdf_map->ev_join, side));
  VS_CK(cudaStreamWaitEvent(s, tsdf_map->ev_join, 0));
  if (st == VS_OK)
    st = mc_encode_keys_clear(tsdf_map, tsdf_pool, tsdf_faces, affected_out, m, n_affected, mpos, mc_pool, q_pool,
                              mc_map->view().e, s);
  for (int g0 = 0; st == VS_OK && g0 < n_sets; g0 += kMaxSets) {
    const int C = n_sets - g0 < kMaxSets ? n_sets - g0 : kMaxSets;
    st = vs_stream_insert_many(sets_host + g0, C, affected_out, m, n_affected, cr_fan, fifo_keys_host + g0,
                               fifo_cap_host + g0, fifo_tail_host + g0, nullptr, stream);
  }
  return st;
}

}  // extern "C"

#if VSB_TICK_PROF
// measurement build only: the phase timestamps (8 x 256 u64)
extern "C" int vs_tick_prof_read(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, vsb::g_tick_prof, sizeof(vsb::g_tick_prof)) == cudaSuccess ? 0 : 1;
}
#endif
