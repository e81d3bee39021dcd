// common.cuh -- shared device definitions for libvsb200 (sm_100a).
//
// Entry layout (one 16-byte aligned entry per table position):
//   int32 x, y, z   the block key (full int32 range; no sentinel value exists,
//                   SURVEY.md §7.3 item 1, so all state lives in `meta`)
//   uint32 meta     bit 31 LOCK   per-bucket writer lock (bucket entries only)
//                   bit 30 OCC    occupied           (reference `_occ`, concurrent_hash.py:108)
//                   bit 29 FRESH  created in the running launch (created-flag fixup)
//                   bits 0-28 NEXT  excess offset + 1 of the next chain entry,
//                                 0 = end of chain   (reference `_next`, :109-111)
// Positions [0, n) are buckets, [n, n + excess) the excess region, exactly as
// the reference (concurrent_hash.py:104-115).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace vsb {

constexpr uint32_t kLock = 0x80000000u;
constexpr uint32_t kOcc = 0x40000000u;
constexpr uint32_t kFresh = 0x20000000u;
constexpr uint32_t kNext = 0x1FFFFFFFu;

// Spatial hash primes, concurrent_hash.py:38-40 (normative).
constexpr uint32_t kP1 = 73856093u;
constexpr uint32_t kP2 = 19349669u;
constexpr uint32_t kP3 = 83492791u;

struct __align__(16) Entry {
  int32_t x, y, z;
  uint32_t meta;
};

constexpr uint32_t kSizeStripes = 32;  // live-key counter stripes
constexpr uint32_t kSizeStride = 16;   // long longs between counter stripes (128 B)

// Device control block of one table.
struct Ctl {
  unsigned int error;  // sticky: bit 0 = capacity exhausted
  unsigned int pad;
  unsigned long long size_sum;  // scratch for vs_table_size
  long long size[kSizeStripes * kSizeStride];  // live keys = sum of the stripes (approx_size)
};

#ifndef VSB_HASH_STRIPES
#define VSB_HASH_STRIPES 128
#endif
constexpr uint32_t kMaxStripes = VSB_HASH_STRIPES;  // free-list stripes
// Fewer stripes for small excess regions: at least kStripeMinEntries entries
// per stripe, down to kMinStripes (a table that erases its whole set pushes
// into full stripes less often: config 1 0.117 -> 0.080 ms per step at 32
// stripes, config 2 unchanged at 128; profiles/r02_ab_stripes.txt).
#ifndef VSB_HASH_STRIPE_MIN_ENTRIES
#define VSB_HASH_STRIPE_MIN_ENTRIES 4096
#endif
constexpr uint32_t kStripeMinEntries = VSB_HASH_STRIPE_MIN_ENTRIES;
constexpr uint32_t kMinStripes = 32;
constexpr uint32_t kTopStride = 32;   // long longs between stripe tops (256 B)

// By-value view passed to kernels.
struct TableView {
  Entry* e;
  uint32_t* free_stack;      // [stripes * stripe_cap] absolute excess positions
  long long* tops;           // [stripes * kTopStride] entries per stripe
  unsigned long long* claim; // [cap] epoch-tagged lowest op index (created / erase dedup)
  uint32_t* dupbits;         // [cap/32] entry got a duplicate insert in this launch
  Ctl* ctl;
  uint32_t n;                // bucket_count
  uint32_t excess;
  uint32_t stripes;
  uint32_t stripe_cap;
  uint64_t magic;            // Lemire fastmod constant for n
  unsigned long long tag;    // (0xFFFFFFFF - launch epoch) << 32
};

// hash_key (concurrent_hash.py:49-59): uint32 wrapping products, XOR.
__host__ __device__ __forceinline__ uint32_t hash_raw(int32_t x, int32_t y, int32_t z) {
  return ((uint32_t)x * kP1) ^ ((uint32_t)y * kP2) ^ ((uint32_t)z * kP3);
}

__host__ __forceinline__ uint64_t fastmod_magic(uint32_t d) {
  return UINT64_C(0xFFFFFFFFFFFFFFFF) / d + 1;
}

// a mod d for 32-bit a, d (exact; Lemire et al. 2019).
__device__ __forceinline__ uint32_t fastmod(uint32_t a, uint64_t M, uint32_t d) {
  uint64_t lowbits = M * a;
  return (uint32_t)__umul64hi(lowbits, (uint64_t)d);
}

__device__ __forceinline__ uint32_t bucket_of(const TableView& T, int32_t x, int32_t y, int32_t z) {
  return fastmod(hash_raw(x, y, z), T.magic, T.n);
}

// ---- memory access helpers (L2-coherent; the table mutates inside a launch)

__device__ __forceinline__ int4 ld_entry(const Entry* p) {
  int4 v;
  asm volatile("ld.relaxed.gpu.global.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

// read-only pass over a table no kernel is mutating (stream-ordered scans)
__device__ __forceinline__ int4 ld_entry_ro(const Entry* p) { return __ldg((const int4*)p); }

// L2 eviction priority for bucket entries: every op starts at its bucket
// entry, so the bucket region (n x 16 B) is worth keeping in L2 ahead of the
// excess region and the streamed per-op inputs (VSB_HASH_L2HINT).
#ifndef VSB_HASH_L2HINT
#define VSB_HASH_L2HINT 1
#endif

__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ int4 ld_bucket(const Entry* p) {
#if VSB_HASH_L2HINT
  int4 v;
  asm volatile("ld.relaxed.gpu.global.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(policy_evict_last())
               : "memory");
  return v;
#else
  return ld_entry(p);
#endif
}

// streamed per-op inputs: read once, do not displace table lines
template <typename T>
__device__ __forceinline__ T ld_stream(const T* p) {
#if VSB_HASH_L2HINT
  return __ldcs(p);
#else
  return *p;
#endif
}

__device__ __forceinline__ void st_entry(Entry* p, int32_t x, int32_t y, int32_t z, uint32_t meta) {
  asm volatile("st.relaxed.gpu.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(x), "r"(y),
               "r"(z), "r"(meta)
               : "memory");
}

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint32_t atom_or_acquire(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.acquire.gpu.global.or.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ uint32_t atom_and_release(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.release.gpu.global.and.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ uint32_t atom_exch_release(uint32_t* p, uint32_t v) {
  uint32_t old;
  asm volatile("atom.release.gpu.global.exch.b32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ bool key_eq(const int4& s, int32_t x, int32_t y, int32_t z) {
  return s.x == x && s.y == y && s.z == z;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

inline unsigned grid_for(uint64_t n, unsigned block) {
  uint64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  return (unsigned)g;
}

}  // namespace vsb
