// hash_ops.cuh -- per-op device algorithms of the block hash set/map.
//
// The algorithm is the reference's (concurrent_hash.py:127-295, §5):
// bucket entry first, collisions chained through the excess region, removal
// that never severs a reachable link.  What changes for the GPU:
//   * one thread per op, thousands of ops in flight per SM; entries are read
//     with single 16-byte L2-coherent vector loads (key + meta together);
//   * the reference's 1024 striped try-locks + seqlock versions become ONE
//     lock bit in each bucket entry's meta word, so a lock costs no extra
//     memory traffic;
//   * readers need no version validation: chains change only by a link at
//     the head (published by one release exchange of the bucket word; the
//     tail append with VSB_HASH_HEAD_INSERT=0) and by unlinking (victim
//     keeps its stale NEXT, like
//     concurrent_hash.py:286-288), and unlinked excess entries are NOT reused
//     inside the launch -- they are recycled into the free list by a separate
//     launch, which removes the ABA case the seqlock guards;
//   * memory ordering is paid only where something is published: a claim of
//     an empty bucket is ONE 16-byte store (key + meta + unlock), lock
//     acquisition orders the re-scan through a data dependency on the lock
//     word, and release fences remain only around excess-entry links;
//   * the free-list stack is striped over kStripes counters (separate L2
//     sectors) with warp-aggregated pops; a pop fails (CapacityExhausted)
//     only after every stripe was seen empty, so exhaustion stays exact;
//   * "created" for in-batch duplicates goes to the lowest op index: a
//     duplicate marks a 1-bit-per-entry bitmap and atomicMins an epoch-tagged
//     64-bit word (no ordering, no clearing pass); creators touch neither.
#pragma once
#include "common.cuh"


// Bucket-case erases skip the re-scan when the bucket word is unchanged (1).
#ifndef VSB_HASH_ERASE_SKIP
#define VSB_HASH_ERASE_SKIP 1
#endif
// Excess-case erases validate the lookup's predecessor under the lock
// instead of re-walking the chain (1; needs a release unlock on the head
// relink, which costs what it saves: off).
#ifndef VSB_HASH_VALIDATE_PREV
#define VSB_HASH_VALIDATE_PREV 0
#endif
// New excess entries are linked at the chain head (1), which also lets an
// insert skip the locked re-scan when its bucket word is unchanged; 0 = the
// reference's tail append with a re-scan under every lock.
#ifndef VSB_HASH_ST_UNLOCK
#define VSB_HASH_ST_UNLOCK 1
#endif
// Bucket lock taken with atom.acquire (1), so the re-scan under the lock is
// ordered by the PTX memory model itself; 0 = a relaxed atom whose returned
// word feeds the re-scan's addresses (ordering by address dependency: holds
// on the hardware but is not promised by the model).  Measured on B200,
// config 2: 17.57 vs 17.57 G ops/s (scripts/ab.py, 3 alternating rounds), so
// the model-backed form is the default.
// Hardware assumption (documented, not promised by PTX): a 16-byte aligned
// st.v4 / ld.v4 of an entry is single-copy atomic on sm_100, so a lock-free
// reader that sees OCC in `meta` also sees the key stored with it.
#ifndef VSB_HASH_LOCK_ACQUIRE
#define VSB_HASH_LOCK_ACQUIRE 1
#endif
#ifndef VSB_HASH_HEAD_INSERT
#define VSB_HASH_HEAD_INSERT 1
#endif

namespace vsb {

__device__ __forceinline__ uint32_t next_pos(const TableView& T, uint32_t meta) {
  return T.n + (meta & kNext) - 1u;
}

__device__ __forceinline__ uint32_t atom_or_relaxed(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.relaxed.gpu.global.or.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ uint32_t atom_exch_relaxed(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.relaxed.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void st_relaxed_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Bucket unlock (the holder writes the whole word back).  A plain strong
// store suffices: while the lock is held no one else changes the word (a
// competing locker's OR of an already-set LOCK bit writes it unchanged, and
// L2 serialises it against the store), and the store carries the release
// ordering the link needs.  VSB_HASH_ST_UNLOCK=0 keeps exchange atomics (-1%).
__device__ __forceinline__ void unlock_release(uint32_t* p, uint32_t v) {
#if VSB_HASH_ST_UNLOCK
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#else
  atom_exch_release(p, v);
#endif
}

__device__ __forceinline__ void unlock_relaxed(uint32_t* p, uint32_t v) {
#if VSB_HASH_ST_UNLOCK
  st_relaxed_u32(p, v);
#else
  atom_exch_relaxed(p, v);
#endif
}

// Pop one excess entry (FreeListStack.pop, concurrent_hash.py:75-79) from the
// striped free list, aggregated over the lanes that reach the call together.
// Returns -1 only when every stripe is empty (CapacityExhausted).
__device__ __forceinline__ int64_t pop_free(const TableView& T) {
  uint32_t s = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % T.stripes;
#pragma unroll 1
  for (uint32_t k = 0; k < T.stripes; ++k) {
    // lanes that reconverge here may be on different stripes (they entered
    // at different times): aggregate per stripe
    const uint32_t m = __match_any_sync(__activemask(), s);
    const int leader = __ffs(m) - 1;
    const int cnt = __popc(m);
    const int rank = __popc(m & lanemask_lt());
    long long* top = T.tops + (size_t)s * kTopStride;
    long long old = 0;
    if ((int)lane_id() == leader) old = (long long)atomicAdd((unsigned long long*)top, (unsigned long long)(-(long long)cnt));
    old = __shfl_sync(m, old, leader);
    const long long t = old - 1 - rank;
    if (t >= 0) return (int64_t)T.free_stack[(size_t)s * T.stripe_cap + (size_t)t];
    // this stripe ran dry for this lane: give the ticket back, try the next
    atomicAdd((unsigned long long*)top, 1ull);
    s = (s + 1 == T.stripes) ? 0 : s + 1;
  }
  return -1;
}

// Push one vacated excess position onto the striped free list (used only by
// recycle launches, never concurrently with pops).  Warp-aggregated
// reservations; a full stripe hands the lanes on to the next stripe.
__device__ __forceinline__ void push_free(const TableView& T, uint32_t e) {
  uint32_t s = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % T.stripes;
#pragma unroll 1
  for (;;) {
    const uint32_t m = __match_any_sync(__activemask(), s);
    const int leader = __ffs(m) - 1;
    const int cnt = __popc(m);
    const int rank = __popc(m & lanemask_lt());
    long long* top = T.tops + (size_t)s * kTopStride;
    long long old = 0;
    if ((int)lane_id() == leader) old = (long long)atomicAdd((unsigned long long*)top, (unsigned long long)cnt);
    old = __shfl_sync(m, old, leader);
    const long long slot = old + rank;
    if (slot < (long long)T.stripe_cap) {
      T.free_stack[(size_t)s * T.stripe_cap + (size_t)slot] = e;
      return;
    }
    atomicAdd((unsigned long long*)top, (unsigned long long)(-1ll));  // undo the overshoot
    s = (s + 1 == T.stripes) ? 0 : s + 1;
  }
}

// Push up to kMaxPush vacated positions per lane with ONE warp-wide
// reservation (post passes).  Every lane of the warp must call it.  A stripe
// that would overflow is given back and the lane's items go one by one
// through push_free (which moves on to the next stripe).
template <int kMaxPush>
__device__ __forceinline__ void push_free_many(const TableView& T, const uint32_t (&v)[kMaxPush], int nv) {
  const uint32_t lane = lane_id();
  uint32_t incl = (uint32_t)nv;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, incl, d);
    if ((int)lane >= d) incl += y;
  }
  const uint32_t total = __shfl_sync(0xFFFFFFFFu, incl, 31);
  if (total == 0) return;
  const uint32_t s = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % T.stripes;
  long long* top = T.tops + (size_t)s * kTopStride;
  long long old = 0;
  if (lane == 0) old = (long long)atomicAdd((unsigned long long*)top, (unsigned long long)total);
  old = __shfl_sync(0xFFFFFFFFu, old, 0);
  if (old + (long long)total <= (long long)T.stripe_cap) {
    uint32_t* dst = T.free_stack + (size_t)s * T.stripe_cap + (size_t)old + (incl - (uint32_t)nv);
#pragma unroll
    for (int j = 0; j < kMaxPush; ++j)
      if (j < nv) dst[j] = v[j];
    return;
  }
  if (lane == 0) atomicAdd((unsigned long long*)top, (unsigned long long)(-(long long)total));
#pragma unroll
  for (int j = 0; j < kMaxPush; ++j)
    if (j < nv) push_free(T, v[j]);
}

// push_free_many split in two, so the caller can issue other memory work
// while lane 0's reservation atomic is in flight: push_reserve scans the
// warp's counts and issues the atomic, push_commit waits for it and stores.
struct PushRes {
  uint32_t incl, total, s;
  long long old;  // lane 0: the reservation's old top (not yet waited on)
};
__device__ __forceinline__ PushRes push_reserve(const TableView& T, int nv) {
  const uint32_t lane = lane_id();
  PushRes r;
  r.incl = (uint32_t)nv;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, r.incl, d);
    if ((int)lane >= d) r.incl += y;
  }
  r.total = __shfl_sync(0xFFFFFFFFu, r.incl, 31);
  r.s = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) % T.stripes;
  r.old = 0;
  if (r.total && lane == 0)
    r.old = (long long)atomicAdd((unsigned long long*)(T.tops + (size_t)r.s * kTopStride), (unsigned long long)r.total);
  return r;
}
template <int kMaxPush>
__device__ __forceinline__ void push_commit(const TableView& T, PushRes r, const uint32_t (&v)[kMaxPush], int nv) {
  if (r.total == 0) return;
  const long long old = __shfl_sync(0xFFFFFFFFu, r.old, 0);
  if (old + (long long)r.total <= (long long)T.stripe_cap) {
    uint32_t* dst = T.free_stack + (size_t)r.s * T.stripe_cap + (size_t)old + (r.incl - (uint32_t)nv);
#pragma unroll
    for (int j = 0; j < kMaxPush; ++j)
      if (j < nv) dst[j] = v[j];
    return;
  }
  if (lane_id() == 0) atomicAdd((unsigned long long*)(T.tops + (size_t)r.s * kTopStride), (unsigned long long)(-(long long)r.total));
#pragma unroll
  for (int j = 0; j < kMaxPush; ++j)
    if (j < nv) push_free(T, v[j]);
}

// Lock-free retrieval (_find + _scan_chain, concurrent_hash.py:127-157).
// Returns the position or -1; *meta_out = meta of the matching entry.
// ... starting from an already loaded bucket entry `s` (lets a thread
// issue the first loads of several ops before walking any of them).
__device__ __forceinline__ int32_t find_pos_from(const TableView& T, int32_t x, int32_t y, int32_t z, uint32_t b,
                                                int4 s, uint32_t* meta_out) {
  uint32_t e = b;
#pragma unroll 1
  for (;;) {
    const uint32_t meta = (uint32_t)s.w;
    if ((meta & kOcc) && key_eq(s, x, y, z)) {
      *meta_out = meta;
      return (int32_t)e;
    }
    if (!(meta & kNext)) return -1;
    e = next_pos(T, meta);
    s = ld_entry(T.e + e);
  }
}

// ... also returning the entry the walk came from (*prev_out; == b for the
// first excess entry, unset for a bucket hit)
__device__ __forceinline__ int32_t find_pos_from_p(const TableView& T, int32_t x, int32_t y, int32_t z, uint32_t b,
                                                  int4 s, uint32_t* meta_out, uint32_t* prev_out) {
  uint32_t e = b, p = b;
#pragma unroll 1
  for (;;) {
    const uint32_t meta = (uint32_t)s.w;
    if ((meta & kOcc) && key_eq(s, x, y, z)) {
      *meta_out = meta;
      *prev_out = p;
      return (int32_t)e;
    }
    if (!(meta & kNext)) return -1;
    p = e;
    e = next_pos(T, meta);
    s = ld_entry(T.e + e);
  }
}

__device__ __forceinline__ int32_t find_pos(const TableView& T, int32_t x, int32_t y, int32_t z, uint32_t b,
                                           uint32_t* meta_out) {
  return find_pos_from(T, x, y, z, b, ld_bucket(T.e + b), meta_out);  // first hop: L2 evict_last
}

// A duplicate insert of an entry created in this launch (FRESH): mark the
// entry in the L2-resident dup bitmap and compete for the "created" flag by
// lowest op index (resolved by the post launch).  Creators touch neither, so
// the common no-duplicate case costs no extra memory traffic.
__device__ __forceinline__ void claim_min(const TableView& T, int32_t pos, int32_t op) {
  atomicOr(&T.dupbits[(uint32_t)pos >> 5], 1u << ((uint32_t)pos & 31u));
  atomicMin(&T.claim[pos], T.tag | (unsigned long long)(uint32_t)op);
}

struct InsertResult {
  int32_t pos;  // -1 on capacity failure
  uint8_t created;
};

// Post pass for one op of an insert/apply batch: settle the created flag of
// a creator against in-batch duplicates (lowest op index wins), clear FRESH;
// recycle the excess entry vacated by an erase.  `same_key(m)` tells whether
// op m names the same key as op i (ops live in a flat int3 array, or in the
// routed records of a sharded batch).
template <class SameKey>
__device__ __forceinline__ void post_op_t(const TableView& T, SameKey same_key, uint64_t i, uint8_t op,
                                          uint8_t* __restrict__ result, int32_t pos) {
  if (op == 0 /*VS_OP_INSERT*/) {
    if (!result[i]) return;
    const uint32_t bit = 1u << ((uint32_t)pos & 31u);
    uint32_t* w = &T.dupbits[(uint32_t)pos >> 5];
    atomicAnd(&T.e[pos].meta, ~kFresh);
    if (!(*w & bit)) return;  // no duplicate touched this entry
    atomicAnd(w, ~bit);
    const unsigned long long c = T.claim[pos];
    if ((c & 0xFFFFFFFF00000000ull) != T.tag) return;
    const uint64_t m = (uint32_t)(c & 0xFFFFFFFFull);
    if (m < i && same_key(m)) {
      result[i] = 0;
      result[m] = 1;
    }
  } else if (op == 2 /*VS_OP_ERASE*/) {
    if (result[i] && pos >= (int32_t)T.n) push_free(T, (uint32_t)pos);
  }
}

__device__ __forceinline__ void post_op(const TableView& T, const int32_t* __restrict__ keys, uint64_t i, uint8_t op,
                                        uint8_t* __restrict__ result, int32_t pos) {
  post_op_t(
      T,
      [&](uint64_t m) {
        return keys[3 * m] == keys[3 * i] && keys[3 * m + 1] == keys[3 * i + 1] && keys[3 * m + 2] == keys[3 * i + 2];
      },
      i, op, result, pos);
}

// Locked mutation shared by inserts of absent keys and erases of present
// keys (apply_one): lock the bucket, re-scan the chain, mutate, unlock -- one
// code path for both kinds, so a warp's mixed mutations share the lock and
// re-scan latency instead of running one kind after the other.  The steps
// are insert_key's and erase_key's (concurrent_hash.py:159-208, 251-295).
// Returns {position, created} for an insert, {vacated position or -1, 0}
// for an erase.
__device__ __forceinline__ InsertResult mutate_locked(const TableView& T, int32_t x, int32_t y, int32_t z, bool ins,
                                                      int32_t op, uint32_t b, uint32_t snap, int32_t fpos = -1,
                                                      uint32_t fprev = 0, bool mixed = true, bool dup_claims = true) {
  uint32_t* bmeta = &T.e[b].meta;
#pragma unroll 1
  for (int attempt = 0;; ++attempt) {
#if VSB_HASH_LOCK_ACQUIRE
    const uint32_t old = atom_or_acquire(bmeta, kLock);
#else
    const uint32_t old = atom_or_relaxed(bmeta, kLock);
#endif
    if (old & kLock) {
      if (attempt > 4) __nanosleep(64);
      continue;
    }
    // --- chain lock held; the re-scan's first load depends on `old`
    // always 0 here, but opaque to the compiler: loads whose address adds it
    // cannot issue before the lock word came back (acquire by dependency)
    uint32_t dep;
    asm volatile("shr.u32 %0, %1, 31;" : "=r"(dep) : "r"(old));
    int32_t found = -1;
    uint32_t fmeta = 0, prev = b, prev_meta = old;  // prev: predecessor of `found`, else the tail
    // An insert whose bucket word is still exactly the one its lock-free
    // lookup started from needs no re-scan: inserts only claim the bucket
    // (OCC changes) or link at the head (NEXT changes), and an unlinked
    // position is not reused inside a launch, so an unchanged word means
    // no key entered this chain since the lookup found the key absent.
    // In a launch that also erases, a FRESH snapshot is not proof: the key
    // created in this launch can be erased (OCC and FRESH clear) and the
    // bucket re-claimed by another insert of OUR key, which restores the very
    // same word (N|OCC|FRESH) -- an ABA that would link a second copy.  A
    // non-FRESH snapshot cannot come back (a re-claim always sets FRESH), so
    // mixed launches skip only then; insert-only launches (no OCC is ever
    // cleared) keep the skip for every snapshot.
    // Likewise an erase whose key sat in the bucket entry itself: an unchanged
    // word that was not FRESH cannot have been re-claimed by another key (a
    // claim sets FRESH), so the entry still holds this key.
    const bool skip_ins = VSB_HASH_HEAD_INSERT && ins && old == snap && !(mixed && (snap & kFresh));
    const bool skip_era = VSB_HASH_ERASE_SKIP && !ins && fpos == (int32_t)b && old == snap && !(snap & kFresh);
    bool skip_ex = false;
    if (skip_era) {
      found = (int32_t)b;
      fmeta = old;
    } else if (VSB_HASH_VALIDATE_PREV && !ins && fpos >= (int32_t)T.n) {
      // excess-case erase: validate the lookup's predecessor under the lock
      // instead of re-walking the chain -- the predecessor still links to the
      // victim (an unlinked entry has OCC clear; the bucket is always the
      // head) and the victim still holds the key (positions are not reused
      // inside a launch).  Both loads are independent: one round trip.
      // both loads depend on `old`, so they issue only after the lock word
      // came back (acquire by dependency, as the re-scan's first load)
      const int4 v = ld_entry(T.e + fpos + dep);
      const uint32_t pm = fprev == b ? old : (uint32_t)ld_entry(T.e + fprev + dep).w;
      const uint32_t link = (uint32_t)fpos - T.n + 1u;
      if ((pm & kNext) == link && (fprev == b || (pm & kOcc)) && ((uint32_t)v.w & kOcc) && key_eq(v, x, y, z)) {
        found = fpos;
        fmeta = (uint32_t)v.w;
        prev = fprev;
        prev_meta = pm;
        skip_ex = true;
      }
    }
    if (!skip_ins && !skip_era && !skip_ex) {
      const int4 s = ld_entry(T.e + b + dep);
      if ((old & kOcc) && key_eq(s, x, y, z)) {
        found = (int32_t)b;
        fmeta = old;
      } else {
        uint32_t meta = old;
        while (meta & kNext) {
          const uint32_t e = next_pos(T, meta);
          const int4 t = ld_entry(T.e + e);
          meta = (uint32_t)t.w;
          if ((meta & kOcc) && key_eq(t, x, y, z)) {
            found = (int32_t)e;
            fmeta = meta;
            break;
          }
          prev = e;
          prev_meta = meta;
        }
      }
    }
    if (ins) {
      if (found >= 0) {  // inserted by another op since the lookup
        unlock_relaxed(bmeta, old);
        if (dup_claims && (fmeta & kFresh)) claim_min(T, found, op);
        return {found, 0};
      }
      if (!(old & kOcc)) {
        // claim the free bucket entry: key, OCC and unlock in ONE 16-byte
        // store; its NEXT link is kept (:185-192)
        st_entry(T.e + b, x, y, z, (old & kNext) | kOcc | kFresh);
        return {(int32_t)b, 1};
      }
      const int64_t ne = pop_free(T);
      if (ne < 0) {
        unlock_relaxed(bmeta, old);
        atomicOr(&T.ctl->error, 1u);
        return {-1, 0};
      }
      const uint32_t e = (uint32_t)ne;
      const uint32_t link = e - T.n + 1u;
#if VSB_HASH_HEAD_INSERT
      // link at the chain HEAD (right after the bucket): the new entry takes
      // the bucket's NEXT and ONE release exchange of the bucket word
      // publishes it and unlocks (the reference appends at the tail, :204;
      // lock-free readers see either the old chain or the new one)
      (void)prev_meta;
      st_entry(T.e + e, x, y, z, kOcc | kFresh | (old & kNext));
      unlock_release(bmeta, (old & ~kNext) | link);
#else
      st_entry(T.e + e, x, y, z, kOcc | kFresh);  // NEXT = 0 clears the stale offset (:200)
      if (prev == b) {
        unlock_release(bmeta, (old & ~kNext) | link);  // publish + unlock
      } else {
        st_release_u32(&T.e[prev].meta, (prev_meta & ~kNext) | link);  // publish last (:204)
        unlock_release(bmeta, old);                                  // unlock after the link
      }
#endif
      return {(int32_t)e, 1};
    }
    if (found < 0) {  // erased by another op since the lookup
      unlock_relaxed(bmeta, old);
      return {-1, 0};
    }
    if (found == (int32_t)b) {
      // bucket case: clear occupancy only; NEXT and the chain stay (:266-275)
      unlock_relaxed(bmeta, old & ~(kOcc | kFresh));
      return {found, 0};
    }
    // excess case: clear the victim but keep its stale NEXT (:280-289)
    st_relaxed_u32(&T.e[found].meta, fmeta & ~(kOcc | kFresh));
    const uint32_t vnext = fmeta & kNext;
    if (prev == b) {
      // relink + unlock, one word.  With predecessor validation the unlock
      // must be a release: the next holder of this lock validates through
      // the victim's and predecessor's OCC bits, so the OCC clear above has
      // to be visible before the chain change (a relaxed unlock let a later
      // erase see the unlinked victim still occupied and relink it again).
      if (VSB_HASH_VALIDATE_PREV)
        unlock_release(bmeta, (old & ~kNext) | vnext);
      else
        unlock_relaxed(bmeta, (old & ~kNext) | vnext);
    } else {
      st_relaxed_u32(&T.e[prev].meta, (prev_meta & ~kNext) | vnext);
      unlock_release(bmeta, old);  // unlock only after the relink
    }
    return {found, 0};
  }
}

// _insert_pos (concurrent_hash.py:159-208): a lock-free retrieval, then, if
// the key is absent, the locked claim (mutate_locked).  `pre` (optional):
// the bucket entry loaded ahead of time (a stale snapshot is harmless: every
// mutation re-validates under the lock).
// kDupClaims = false (a put: positions only, no created flag): in-batch
// duplicates claim nothing, so the caller may use the claim array itself.
template <bool kDupClaims = true>
__device__ __forceinline__ InsertResult insert_key(const TableView& T, int32_t x, int32_t y, int32_t z, int32_t op,
                                                   const int4* pre = nullptr) {
  const uint32_t b = bucket_of(T, x, y, z);
  uint32_t fmeta;
  const int4 s0 = pre ? *pre : ld_bucket(T.e + b);
  const int32_t pos = find_pos_from(T, x, y, z, b, s0, &fmeta);
  if (pos >= 0) {
    if (kDupClaims && (fmeta & kFresh)) claim_min(T, pos, op);
    return {pos, 0};
  }
  return mutate_locked(T, x, y, z, true, op, b, (uint32_t)s0.w, -1, 0, /*mixed=*/false,
                       kDupClaims);  // insert-only launches
}

// remove (concurrent_hash.py:251-295).  Returns the vacated position or -1.
// Vacated EXCESS positions are recycled by the caller's recycle launch.
__device__ __forceinline__ int32_t erase_key(const TableView& T, int32_t x, int32_t y, int32_t z,
                                            const int4* pre = nullptr) {
  const uint32_t b = bucket_of(T, x, y, z);
  uint32_t fmeta;
  const int4 s0 = pre ? *pre : ld_bucket(T.e + b);
  const int32_t fpos = find_pos_from(T, x, y, z, b, s0, &fmeta);
  if (fpos < 0) return -1;
  return mutate_locked(T, x, y, z, false, 0, b, (uint32_t)s0.w, fpos).pos;
}

// One mixed op (insert / find / erase) with its bucket entry already loaded.
// The lock-free lookup is the same walk for every kind, so it runs first for
// all lanes together (a warp with mixed kinds would otherwise walk its
// chains once per kind, one branch after the other); only inserts of absent
// keys and erases of present keys go on to mutate.  Returns the size delta.
__device__ __forceinline__ int apply_one(const TableView& T, int32_t x, int32_t y, int32_t z, uint8_t op, uint64_t i,
                                         uint32_t b, const int4& pre, uint8_t* __restrict__ result,
                                         int32_t* __restrict__ index) {
  int32_t pos;
  uint8_t res;
  int delta = 0;
  uint32_t fmeta, fprev = b;
  const int32_t fpos = find_pos_from_p(T, x, y, z, b, pre, &fmeta, &fprev);
  const bool ins = op == 0 /*VS_OP_INSERT*/, era = op == 2 /*VS_OP_ERASE*/;
  pos = fpos;
  res = !ins && fpos >= 0;  // find: found; erase: provisional
  if (ins && fpos >= 0 && (fmeta & kFresh)) claim_min(T, fpos, (int32_t)i);
  if ((ins && fpos < 0) || (era && fpos >= 0)) {
    const InsertResult r = mutate_locked(T, x, y, z, ins, (int32_t)i, b, (uint32_t)pre.w, fpos, fprev);
    pos = r.pos;
    res = ins ? r.created : (uint8_t)(r.pos >= 0);
    delta = ins ? (int)r.created : -(int)(r.pos >= 0);
  }
  __stcs(result + i, res);
  __stcs(index + i, pos);
  return delta;
}

// Warp-aggregated update of the live-key counter into one of kSizeStripes
// counters (separate 128-B lines): no CTA barrier, so a warp retires as soon
// as its own ops are done.  Every lane of the warp must call it once.
__device__ __forceinline__ void add_size_cta(const TableView& T, int delta) {
  __syncwarp();
  delta = __reduce_add_sync(0xffffffffu, delta);
  if (lane_id() == 0 && delta != 0) {
    const uint32_t w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    atomicAdd((unsigned long long*)&T.ctl->size[(w % kSizeStripes) * kSizeStride],
              (unsigned long long)(long long)delta);
  }
}

}  // namespace vsb
