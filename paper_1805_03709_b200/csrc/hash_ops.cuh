// hash_ops.cuh -- per-op device algorithms of the block hash set/map.
//
// The algorithm is the reference's (concurrent_hash.py:127-295, §5):
// bucket entry first, collisions chained through the excess region, removal
// that never severs a reachable link.  What changes for the GPU:
//   * one thread per op, thousands of ops in flight per SM; entries are read
//     with single 16-byte L2-coherent vector loads (key + meta together);
//   * the reference's 1024 striped try-locks + seqlock versions become ONE
//     lock bit in each bucket entry's meta word (atom.or.acquire /
//     atom.exch.release), so a lock costs no extra memory traffic;
//   * readers need no version validation: chains change only by tail append
//     (published last, release) and by unlinking (victim keeps its stale NEXT,
//     like concurrent_hash.py:286-288), and unlinked excess entries are NOT
//     reused inside the launch -- they go to `retired` and rejoin the free
//     stack between launches, which removes the ABA case the seqlock guards;
//   * free-list pops are warp-aggregated (one atomic per warp, not per op).
#pragma once
#include "common.cuh"

namespace vsb {

// Pop one excess entry from the free-list stack (FreeListStack.pop,
// concurrent_hash.py:75-79), aggregated over the lanes that reach this call
// together.  Returns -1 when the stack is empty (CapacityExhausted).
__device__ __forceinline__ int64_t pop_free(const TableView& T) {
  const uint32_t m = __activemask();
  const uint32_t lane = lane_id();
  const int leader = __ffs(m) - 1;
  const int cnt = __popc(m);
  const int rank = __popc(m & lanemask_lt());
  long long old = 0;
  if ((int)lane == leader)
    old = (long long)atomicAdd((unsigned long long*)&T.ctl->free_top, (unsigned long long)(-(long long)cnt));
  old = __shfl_sync(m, old, leader);
  const long long t = old - 1 - rank;
  if (t < 0) {
    // give the failed ticket back; the stack top never rises above the
    // number of entries not yet handed out
    atomicAdd((unsigned long long*)&T.ctl->free_top, 1ull);
    return -1;
  }
  return (int64_t)T.free_stack[t];
}

// Record an unlinked excess entry for recycling after the launch.
__device__ __forceinline__ void retire(const TableView& T, uint32_t pos) {
  const uint32_t m = __activemask();
  const uint32_t lane = lane_id();
  const int leader = __ffs(m) - 1;
  const int cnt = __popc(m);
  const int rank = __popc(m & lanemask_lt());
  unsigned long long base = 0;
  if ((int)lane == leader) base = atomicAdd(&T.ctl->retired_n, (unsigned long long)cnt);
  base = __shfl_sync(m, base, leader);
  T.retired[base + rank] = pos;
}

__device__ __forceinline__ uint32_t next_pos(const TableView& T, uint32_t meta) {
  return T.n + (meta & kNext) - 1u;
}

// Lock-free retrieval (_find + _scan_chain, concurrent_hash.py:127-157).
// Returns the position or -1; *meta_out = meta of the matching entry.
__device__ __forceinline__ int32_t find_pos(const TableView& T, int32_t x, int32_t y, int32_t z,
                                            uint32_t b, uint32_t* meta_out) {
  uint32_t e = b;
#pragma unroll 1
  for (;;) {
    const int4 s = ld_entry(T.e + e);
    const uint32_t meta = (uint32_t)s.w;
    if ((meta & kOcc) && key_eq(s, x, y, z)) {
      *meta_out = meta;
      return (int32_t)e;
    }
    if (!(meta & kNext)) return -1;
    e = next_pos(T, meta);
  }
}

// A duplicate insert of a key created earlier in this launch: compete for
// the "created" flag by lowest op index (resolved by k_fixup_created).
__device__ __forceinline__ void note_duplicate(const TableView& T, int32_t pos, uint32_t meta, int32_t op) {
  if (meta & kFresh) atomicMin(&T.first_op[pos], op);
}

struct InsertResult {
  int32_t pos;   // -1 on capacity failure
  uint8_t created;
};

// _insert_pos (concurrent_hash.py:159-208): loop of non-blocking attempts;
// each retry starts with a fresh lock-free retrieval.
__device__ __forceinline__ InsertResult insert_key(const TableView& T, int32_t x, int32_t y, int32_t z,
                                                   int32_t op) {
  const uint32_t b = bucket_of(T, x, y, z);
  uint32_t* bmeta = &T.e[b].meta;
#pragma unroll 1
  for (int attempt = 0;; ++attempt) {
    uint32_t fmeta;
    int32_t pos = find_pos(T, x, y, z, b, &fmeta);
    if (pos >= 0) {
      note_duplicate(T, pos, fmeta, op);
      return {pos, 0};
    }
    const uint32_t old = atom_or_acquire(bmeta, kLock);
    if (old & kLock) {
      if (attempt > 4) __nanosleep(64);
      continue;
    }
    // --- chain lock held: re-validate (concurrent_hash.py:180-184)
    uint32_t tail = b, tail_meta = old;
    {
      const int4 s = ld_entry(T.e + b);
      if ((old & kOcc) && key_eq(s, x, y, z)) {
        atom_and_release(bmeta, ~kLock);
        note_duplicate(T, (int32_t)b, old, op);
        return {(int32_t)b, 0};
      }
      uint32_t meta = old;
      while (meta & kNext) {
        const uint32_t e = next_pos(T, meta);
        const int4 t = ld_entry(T.e + e);
        meta = (uint32_t)t.w;
        if ((meta & kOcc) && key_eq(t, x, y, z)) {
          atom_and_release(bmeta, ~kLock);
          note_duplicate(T, (int32_t)e, meta, op);
          return {(int32_t)e, 0};
        }
        tail = e;
        tail_meta = meta;
      }
    }
    if (!(old & kOcc)) {
      // claim the free bucket entry; its NEXT link is kept (:185-192)
      T.first_op[b] = op;
      st_entry(T.e + b, x, y, z, old | kLock);  // meta unchanged (still locked)
      atom_exch_release(bmeta, (old & ~kLock) | kOcc | kFresh);
      return {(int32_t)b, 1};
    }
    const int64_t ne = pop_free(T);
    if (ne < 0) {
      atom_and_release(bmeta, ~kLock);
      atomicOr(&T.ctl->error, 1u);
      return {-1, 0};
    }
    const uint32_t e = (uint32_t)ne;
    T.first_op[e] = op;
    st_entry(T.e + e, x, y, z, kOcc | kFresh);  // NEXT = 0: clears the stale offset (:200)
    const uint32_t link = e - T.n + 1u;
    if (tail == b) {
      atom_exch_release(bmeta, (old & ~(kLock | kNext)) | link);  // publish + unlock
    } else {
      st_release_u32(&T.e[tail].meta, (tail_meta & ~kNext) | link);  // publish last (:204)
      atom_and_release(bmeta, ~kLock);
    }
    return {(int32_t)e, 1};
  }
}

// remove (concurrent_hash.py:251-295).  Returns the vacated position or -1.
__device__ __forceinline__ int32_t erase_key(const TableView& T, int32_t x, int32_t y, int32_t z) {
  const uint32_t b = bucket_of(T, x, y, z);
  uint32_t* bmeta = &T.e[b].meta;
#pragma unroll 1
  for (int attempt = 0;; ++attempt) {
    uint32_t fmeta;
    if (find_pos(T, x, y, z, b, &fmeta) < 0) return -1;
    const uint32_t old = atom_or_acquire(bmeta, kLock);
    if (old & kLock) {
      if (attempt > 4) __nanosleep(64);
      continue;
    }
    const int4 s = ld_entry(T.e + b);
    if ((old & kOcc) && key_eq(s, x, y, z)) {
      // bucket case: clear occupancy only; NEXT and the chain stay (:266-275)
      atom_exch_release(bmeta, old & ~(kLock | kOcc | kFresh));
      return (int32_t)b;
    }
    uint32_t prev = b, prev_meta = old, meta = old;
    while (meta & kNext) {
      const uint32_t e = next_pos(T, meta);
      const int4 t = ld_entry(T.e + e);
      meta = (uint32_t)t.w;
      if ((meta & kOcc) && key_eq(t, x, y, z)) {
        // excess case: clear the victim but keep its stale NEXT (:280-289)
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(&T.e[e].meta),
                     "r"(meta & ~(kOcc | kFresh))
                     : "memory");
        const uint32_t vnext = meta & kNext;
        if (prev == b) {
          atom_exch_release(bmeta, (old & ~(kLock | kNext)) | vnext);
        } else {
          st_release_u32(&T.e[prev].meta, (prev_meta & ~kNext) | vnext);
          atom_and_release(bmeta, ~kLock);
        }
        retire(T, e);
        return (int32_t)e;
      }
      prev = e;
      prev_meta = meta;
    }
    // key vanished between the find and the lock; re-check (:293)
    atom_and_release(bmeta, ~kLock);
  }
}

// Warp-aggregated update of the live-key counter.  Every lane of the warp
// must call it (kernels keep out-of-range lanes alive with delta 0).
__device__ __forceinline__ void add_size(const TableView& T, int delta) {
  __syncwarp();
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) delta += __shfl_xor_sync(0xffffffffu, delta, o);
  if (lane_id() == 0 && delta != 0)
    atomicAdd(&T.ctl->size, (unsigned long long)(long long)delta);
}

}  // namespace vsb
