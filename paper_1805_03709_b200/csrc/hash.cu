// hash.cu -- batched kernels and C ABI of the block hash set/map.
//
// Reference: concurrent_hash.py (all of it).  Per-op algorithms live in
// hash_ops.cuh; this file holds the launches: one thread per op, every op
// type in one launch if wanted (vs_table_apply), followed by
//   k_post           -- gives `created` to the lowest op index among in-batch
//                       duplicates (the sequential-replay answer) and pushes
//                       the excess entries vacated by erases back onto the
//                       striped free list (FreeListStack.push,
//                       concurrent_hash.py:72-73), in one pass, so the op
//                       kernel itself needs no atomics for either.
#ifndef VSB_PDL
#define VSB_PDL 1
#endif
// k_apply launched as a programmatic dependent of the previous launch (1),
// and the post pass releasing its dependents right after its own wait (1).
#ifndef VSB_PDL_APPLY
#define VSB_PDL_APPLY 0
#endif
#ifndef VSB_POST_TRIGGER
#define VSB_POST_TRIGGER 0
#endif
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "hash_ops.cuh"
#include "pdl.cuh"
#include "table.h"

namespace vsb {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

vs_status cuda_status(cudaError_t err, const char* what) {
  g_last_error = std::string(what) + ": " + cudaGetErrorString(err);
  return VS_ERR_CUDA;
}

#ifndef VSB_HASH_BLOCK
#define VSB_HASH_BLOCK 128
#endif
constexpr int kOpBlock = VSB_HASH_BLOCK;  // threads per CTA of the op kernels

// ------------------------------------------------------- launch accounting

#ifndef VSB_PROF_RESERVE
#define VSB_PROF_RESERVE 8192
#endif
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

struct ProfRec {
  int tag;
  cudaEvent_t a, b;
};
static std::mutex g_prof_mu;
static bool g_prof_on = false;
static std::vector<cudaEvent_t> g_ev_pool;
static std::vector<ProfRec> g_prof_recs;
static uint64_t g_prof_launch0 = 0;

static cudaEvent_t take_event() {
  if (!g_ev_pool.empty()) {
    cudaEvent_t e = g_ev_pool.back();
    g_ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

ProfScope::ProfScope(int tag_, cudaStream_t s_) : tag(tag_), s(s_) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  if (!g_prof_on) return;
  cudaEvent_t a = take_event();
  cudaEventRecord(a, s);
  start = (void*)a;
}

ProfScope::~ProfScope() {
  if (!start) return;
  std::lock_guard<std::mutex> g(g_prof_mu);
  cudaEvent_t b = take_event();
  cudaEventRecord(b, s);
  g_prof_recs.push_back({tag, (cudaEvent_t)start, b});
}

// ---------------------------------------------------------------- kernels

__global__ void k_hash_keys(const int32_t* __restrict__ keys, uint64_t n, uint32_t nb,
                            uint32_t* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = hash_raw(keys[3 * i], keys[3 * i + 1], keys[3 * i + 2]) % nb;
}

// Free list: stripe s holds excess positions n + [s*C, min((s+1)*C, excess)).
__global__ void k_init_free(TableView T) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < T.excess;
       i += (uint64_t)gridDim.x * blockDim.x)
    T.free_stack[i] = T.n + (uint32_t)i;  // stripe s, slot i - s*C == i (contiguous layout)
}

__global__ void k_reset_ctl(TableView T) {
  for (uint32_t s = threadIdx.x; s < T.stripes; s += blockDim.x) {
    const long long lo = (long long)s * T.stripe_cap;
    long long c = (long long)T.excess - lo;
    if (c > (long long)T.stripe_cap) c = T.stripe_cap;
    T.tops[(size_t)s * kTopStride] = c < 0 ? 0 : c;
  }
  for (uint32_t k = threadIdx.x; k < kSizeStripes; k += blockDim.x) T.ctl->size[k * kSizeStride] = 0;
  if (threadIdx.x == 0) T.ctl->error = 0;
}

// kPut: a TSDF put (latest write wins, no created flag): duplicates claim
// nothing, and every op instead claims its position for the row copy with
// the highest op index (k_put_rows, same launch tag).
template <bool kPut>
__global__ void __launch_bounds__(kOpBlock) k_insert_t(TableView T, const int32_t* __restrict__ keys, uint64_t n,
                                                       const uint64_t* __restrict__ n_dev,
                                                       uint8_t* __restrict__ created, int32_t* __restrict__ index) {
  pdl_wait();
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t nv = n_dev && *n_dev < n ? *n_dev : n;  // ops past a device count: created 0, index -1
  int delta = 0;
  if (i >= nv && i < n) {
    created[i] = 0;
    index[i] = -1;
  }
  if (i < nv) {
    const int32_t x = keys[3 * i], y = keys[3 * i + 1], z = keys[3 * i + 2];
    const InsertResult r = insert_key<!kPut>(T, x, y, z, (int32_t)i);
    created[i] = r.created;
    index[i] = r.pos;
    delta = r.created;
    if (kPut && r.pos >= 0) atomicMin(&T.claim[r.pos], T.tag | (unsigned long long)(0xFFFFFFFFu - (uint32_t)i));
  }
  add_size_cta(T, delta);
}
#define k_insert k_insert_t<false>

__global__ void __launch_bounds__(kOpBlock) k_find(TableView T, const int32_t* __restrict__ keys, uint64_t n,
                                                   uint8_t* __restrict__ found, int32_t* __restrict__ index) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t x = keys[3 * i], y = keys[3 * i + 1], z = keys[3 * i + 2];
  uint32_t meta;
  const int32_t pos = find_pos(T, x, y, z, bucket_of(T, x, y, z), &meta);
  found[i] = pos >= 0;
  index[i] = pos;
}

// Single-pass erase for batches of DISTINCT keys (internal: extract paths).
__global__ void __launch_bounds__(kOpBlock) k_erase(TableView T, const int32_t* __restrict__ keys, uint64_t n,
                                                    const uint64_t* __restrict__ n_dev, int32_t* __restrict__ index) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n_dev) n = *n_dev < n ? *n_dev : n;
  int delta = 0;
  if (i < n) {
    const int32_t pos = erase_key(T, keys[3 * i], keys[3 * i + 1], keys[3 * i + 2]);
    index[i] = pos;
    delta = -(pos >= 0);
  }
  add_size_cta(T, delta);
}

// Duplicate removes in one batch: the lowest op index wins (sequential replay
// gives True to the first occurrence).  Phase 1 claims the key's current
// position with an epoch-tagged atomicMin (values of older batches compare
// larger, so no clearing pass is needed); phase 2 lets only winners erase.
__global__ void __launch_bounds__(kOpBlock) k_erase_claim(TableView T, const int32_t* __restrict__ keys, uint64_t n,
                                                          int32_t* __restrict__ pos_out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int32_t x = keys[3 * i], y = keys[3 * i + 1], z = keys[3 * i + 2];
  uint32_t meta;
  const int32_t pos = find_pos(T, x, y, z, bucket_of(T, x, y, z), &meta);
  pos_out[i] = pos;
  if (pos >= 0) atomicMin(&T.claim[pos], T.tag | (unsigned long long)i);
}

__global__ void __launch_bounds__(kOpBlock) k_erase_win(TableView T, const int32_t* __restrict__ keys, uint64_t n,
                                                        uint8_t* __restrict__ erased, int32_t* __restrict__ index) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int delta = 0;
  if (i < n) {
    int32_t pos = index[i];
    if (pos >= 0 && T.claim[pos] == (T.tag | (unsigned long long)i)) {
      pos = erase_key(T, keys[3 * i], keys[3 * i + 1], keys[3 * i + 2]);
    } else {
      pos = -1;
    }
    if (erased) erased[i] = pos >= 0;
    index[i] = pos;
    delta = -(pos >= 0);
  }
  add_size_cta(T, delta);
}

// Mixed batch.  Each thread owns kOpsPerThread ops (kOpBlock apart, so loads
// stay coalesced) and issues all their bucket-entry loads before walking
// any chain: more independent misses in flight per SM.
#ifndef VSB_HASH_OPS_PER_THREAD
#define VSB_HASH_OPS_PER_THREAD 1
#endif
constexpr int kOpsPerThread = VSB_HASH_OPS_PER_THREAD;

__global__ void __launch_bounds__(kOpBlock) k_apply(TableView T, const int32_t* __restrict__ keys,
                                                    const uint8_t* __restrict__ ops, uint64_t n,
                                                    uint8_t* __restrict__ result, int32_t* __restrict__ index) {
#if VSB_PDL_APPLY
  // launched as a programmatic dependent of the previous batch's post pass
  // (its launch overlaps that pass's tail): wait before touching anything
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
  const uint64_t base = (uint64_t)blockIdx.x * (kOpBlock * kOpsPerThread) + threadIdx.x;
  int32_t x[kOpsPerThread], y[kOpsPerThread], z[kOpsPerThread];
  uint8_t op[kOpsPerThread];
  uint32_t b[kOpsPerThread];
  int4 pre[kOpsPerThread];
#pragma unroll
  for (int k = 0; k < kOpsPerThread; ++k) {
    const uint64_t i = base + (uint64_t)k * kOpBlock;
    if (i < n) {
      x[k] = ld_stream(keys + 3 * i);
      y[k] = ld_stream(keys + 3 * i + 1);
      z[k] = ld_stream(keys + 3 * i + 2);
      op[k] = ld_stream(ops + i);
      b[k] = bucket_of(T, x[k], y[k], z[k]);
      pre[k] = ld_bucket(T.e + b[k]);
    }
  }
  int delta = 0;
#pragma unroll
  for (int k = 0; k < kOpsPerThread; ++k) {
    const uint64_t i = base + (uint64_t)k * kOpBlock;
    if (i < n) delta += apply_one(T, x[k], y[k], z[k], op[k], i, b[k], pre[k], result, index);
  }
  add_size_cta(T, delta);
}

static unsigned apply_grid(uint64_t n) { return grid_for(n, kOpBlock * kOpsPerThread); }

// Optional L2 persistence of the bucket region (VSB_HASH_PERSIST_L2): every
// op starts with a random bucket-entry access, so a persisting carve-out over
// the n x 16 B bucket array turns most first hops into L2 hits.
#ifndef VSB_HASH_PERSIST_L2
#define VSB_HASH_PERSIST_L2 0
#endif
static cudaError_t launch_apply(const TableView& v, const int32_t* keys, const uint8_t* ops, uint64_t n,
                                uint8_t* result, int32_t* index, cudaStream_t s) {
#if VSB_HASH_PERSIST_L2
  static size_t carve = 0;
  if (carve == 0) {
    int dev = 0, maxp = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    carve = (size_t)maxp;
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, carve);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(apply_grid(n));
  cfg.blockDim = dim3(kOpBlock);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeAccessPolicyWindow;
  attr[0].val.accessPolicyWindow.base_ptr = (void*)v.e;
  const size_t bytes = (size_t)v.n * sizeof(Entry);
  attr[0].val.accessPolicyWindow.num_bytes = bytes;
  attr[0].val.accessPolicyWindow.hitRatio = bytes > carve ? (float)carve / (float)bytes : 1.0f;
  attr[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_apply, v, keys, ops, n, result, index);
#elif VSB_PDL_APPLY
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(apply_grid(n));
  cfg.blockDim = dim3(kOpBlock);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = n >= (1u << 16);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_apply, v, keys, ops, n, result, index);
#else
  k_apply<<<apply_grid(n), kOpBlock, 0, s>>>(v, keys, ops, n, result, index);
  return cudaGetLastError();
#endif
}

// Speed-of-light probe (diagnostics): `hops` dependent random entry loads per
// thread over the whole table, k_apply's launch shape, one result byte.
__global__ void __launch_bounds__(kOpBlock) k_probe_sol(TableView T, uint64_t n, int hops, uint8_t* __restrict__ out) {
  const uint64_t i = (uint64_t)blockIdx.x * kOpBlock + threadIdx.x;
  if (i >= n) return;
  const uint32_t cap = T.n + T.excess;
  uint32_t h = (uint32_t)i * 0x9E3779B1u + 0x7F4A7C15u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 12;
  uint32_t e = h % cap;
  uint32_t acc = 0;
#pragma unroll 1
  for (int k = 0; k < hops; ++k) {
    const int4 v = k == 0 ? ld_bucket(T.e + e) : ld_entry(T.e + e);
    acc ^= (uint32_t)v.x ^ (uint32_t)v.w;
    h = h * 0x85EBCA6Bu + acc + 0x165667B1u;  // next address depends on the loaded entry
    e = h % cap;
  }
  __stcs(out + i, (uint8_t)(acc & 1u));
}

// One op of any kind on one key, then its post pass, in a single thread
// (the per-key compatibility path: BlockHashSet.insert/remove/__contains__).
__global__ void k_single(TableView T, int32_t x, int32_t y, int32_t z, uint8_t op,
                         unsigned long long* __restrict__ word, uint32_t seq) {
  int delta = 0;
  int32_t pos;
  uint32_t res;
  if (op == VS_OP_INSERT) {
    const InsertResult r = insert_key(T, x, y, z, 0);
    res = r.created;
    pos = r.pos;
    delta = r.created;
    if (r.created) atomicAnd(&T.e[r.pos].meta, ~kFresh);
  } else if (op == VS_OP_ERASE) {
    pos = erase_key(T, x, y, z);
    res = pos >= 0;
    delta = -(pos >= 0);
    if (pos >= (int32_t)T.n) push_free(T, (uint32_t)pos);  // no pops in this launch
  } else {
    uint32_t meta;
    pos = find_pos(T, x, y, z, bucket_of(T, x, y, z), &meta);
    res = pos >= 0;
  }
  if (delta) atomicAdd((unsigned long long*)&T.ctl->size[0], (unsigned long long)(long long)delta);
  // result and completion in ONE 8-byte store to mapped host memory (a single
  // PCIe write, so the host never sees one without the other):
  // bit 63 = flag, bits 32-62 = sequence number, bits 0-31 = position
  *(volatile unsigned long long*)word = ((unsigned long long)res << 63) |
                                       ((unsigned long long)(seq & 0x7FFFFFFFu) << 32) | (uint32_t)pos;
}

// Post pass after k_insert / k_apply: created flags to the lowest op index
// among in-batch duplicates (sequential replay), FRESH cleared, and the
// excess entries vacated by erases recycled -- one launch, one pass.  Each
// thread takes kPostOps ops (loads of all of them in flight first, then
// every FRESH clear and dup-bitmap load issued before any is waited on) and
// the vacated positions of a whole warp go back with one reservation.
// 64-thread CTAs x 3 ops: 0.2358 vs 0.2388 ms per config-2 step against the
// former 256 x 4 without the hoist; with the free-list reservation issued
// first (VSB_POST_HOIST=2) 0.2347; 4 consecutive ops per thread through
// three vector loads (VSB_POST_VEC, aligned arrays) 0.2341 (profiles/r02_ab_post.txt).
#ifndef VSB_POST_VEC
#define VSB_POST_VEC 1
#endif
#ifndef VSB_POST_HOIST
#define VSB_POST_HOIST 2
#endif
#ifndef VSB_POST_OPS
#define VSB_POST_OPS 4
#endif
#ifndef VSB_POST_BLOCK
#define VSB_POST_BLOCK 64
#endif
constexpr int kPostOps = VSB_POST_OPS;
constexpr int kPostBlock = VSB_POST_BLOCK;
template <bool kVec>
__global__ void __launch_bounds__(kPostBlock) k_post(TableView T, const int32_t* __restrict__ keys,
                                                     const uint8_t* __restrict__ ops, uint64_t n,
                                                     uint8_t* __restrict__ result, const int32_t* __restrict__ index) {
#if VSB_PDL
  // launched as a programmatic dependent of the op kernel: everything below
  // reads its results, so wait for its grid to complete and flush
  asm volatile("griddepcontrol.wait;" ::: "memory");
#endif
#if VSB_POST_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;");
#endif
  // kVec (4 ops per thread, 4-aligned op/result and 16-aligned index
  // arrays): a thread's ops are CONSECUTIVE and come in with three vector
  // loads; otherwise they sit kPostBlock apart (scalar, coalesced per k)
  const uint64_t base = kVec ? ((uint64_t)blockIdx.x * kPostBlock + threadIdx.x) * kPostOps
                             : (uint64_t)blockIdx.x * (kPostBlock * kPostOps) + threadIdx.x;
  constexpr uint64_t kStep = kVec ? 1 : kPostBlock;
  uint8_t op[kPostOps], res[kPostOps];
  int32_t pos[kPostOps];
  if (kVec && base + kPostOps <= n) {
    static_assert(!kVec || kPostOps == 4, "vector post loads take 4 ops per thread");
    const uint32_t ow = ops ? *(const uint32_t*)(ops + base) : 0u;  // VS_OP_INSERT == 0
    const uint32_t rw = *(const uint32_t*)(result + base);
    const int4 pw = *(const int4*)(index + base);
    const int32_t pv[4] = {pw.x, pw.y, pw.z, pw.w};
#pragma unroll
    for (int k = 0; k < kPostOps; ++k) {
      op[k] = (uint8_t)(ow >> (8 * k));
      res[k] = (uint8_t)(rw >> (8 * k));
      pos[k] = pv[k & 3];
    }
  } else {
#pragma unroll
    for (int k = 0; k < kPostOps; ++k) {
      const uint64_t i = base + (uint64_t)k * kStep;
      op[k] = 0xFF;
      if (i < n) {
        op[k] = ops ? ops[i] : (uint8_t)VS_OP_INSERT;
        res[k] = result[i];
        pos[k] = index[i];
      }
    }
  }
  uint32_t vac[kPostOps];
  int nv = 0;
#if VSB_POST_HOIST
#if VSB_POST_HOIST == 2
  // the vacated positions first: the warp's free-list reservation is in
  // flight while the FRESH clears and dup-bitmap loads below are issued
#pragma unroll
  for (int k = 0; k < kPostOps; ++k)
    if (op[k] == VS_OP_ERASE && res[k] && pos[k] >= (int32_t)T.n) vac[nv++] = (uint32_t)pos[k];
  const PushRes pr = push_reserve(T, nv);
#endif
  // every FRESH clear and dup-bitmap load of the thread's ops issued before
  // any of them is waited on (the loop below only reads the loaded words)
  uint32_t dw[kPostOps];
#pragma unroll
  for (int k = 0; k < kPostOps; ++k) {
    dw[k] = 0;
    if (op[k] == VS_OP_INSERT && res[k]) {
      atomicAnd(&T.e[pos[k]].meta, ~kFresh);
      dw[k] = __ldcg(&T.dupbits[(uint32_t)pos[k] >> 5]);
    }
  }
#if VSB_POST_HOIST == 2
  push_commit<kPostOps>(T, pr, vac, nv);
#endif
#pragma unroll
  for (int k = 0; k < kPostOps; ++k) {
    const uint64_t i = base + (uint64_t)k * kStep;
    if (op[k] == VS_OP_INSERT && res[k]) {
      const uint32_t bit = 1u << ((uint32_t)pos[k] & 31u);
      if (dw[k] & bit) {
        atomicAnd(&T.dupbits[(uint32_t)pos[k] >> 5], ~bit);
        const unsigned long long c = T.claim[pos[k]];
        if ((c & 0xFFFFFFFF00000000ull) == T.tag) {
          const uint64_t m = (uint32_t)(c & 0xFFFFFFFFull);
          if (m < i && keys[3 * m] == keys[3 * i] && keys[3 * m + 1] == keys[3 * i + 1] &&
              keys[3 * m + 2] == keys[3 * i + 2]) {
            result[i] = 0;
            result[m] = 1;
          }
        }
      }
    } else if (VSB_POST_HOIST != 2 && op[k] == VS_OP_ERASE && res[k] && pos[k] >= (int32_t)T.n) {
      vac[nv++] = (uint32_t)pos[k];
    }
  }
#else
#pragma unroll
  for (int k = 0; k < kPostOps; ++k) {
    const uint64_t i = base + (uint64_t)k * kStep;
    if (op[k] == VS_OP_INSERT && res[k]) {
      post_op(T, keys, i, VS_OP_INSERT, result, pos[k]);
    } else if (op[k] == VS_OP_ERASE && res[k] && pos[k] >= (int32_t)T.n) {
      vac[nv++] = (uint32_t)pos[k];
    }
  }
#endif
  if (VSB_POST_HOIST != 2) push_free_many<kPostOps>(T, vac, nv);
}

// k_post as a programmatic dependent launch (VSB_PDL): its launch and CTA
// setup overlap the op kernel's tail instead of following its completion.
static cudaError_t launch_post(const TableView& v, const int32_t* keys, const uint8_t* ops, uint64_t n,
                               uint8_t* result, const int32_t* index, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid_for(n, kPostBlock * kPostOps));
  cfg.blockDim = dim3(kPostBlock);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  // small batches (server-side scratch sets) gain nothing from the overlap
  attr[0].val.programmaticStreamSerializationAllowed = VSB_PDL && n >= (1u << 16);
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const bool vec = VSB_POST_VEC && kPostOps == 4 && (((uintptr_t)ops | (uintptr_t)result) & 3u) == 0 &&
                   ((uintptr_t)index & 15u) == 0;
  return vec ? cudaLaunchKernelEx(&cfg, k_post<VSB_POST_VEC != 0>, v, keys, ops, n, result, index)
             : cudaLaunchKernelEx(&cfg, k_post<false>, v, keys, ops, n, result, index);
}

// Push vacated excess positions back onto the striped free list (warp-
// aggregated reservations; a full stripe hands the lanes to the next one).
__global__ void k_recycle(TableView T, const int32_t* __restrict__ pos, const uint8_t* __restrict__ flag,
                          const uint8_t* __restrict__ ops, const uint64_t* __restrict__ n_dev, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (n_dev) n = *n_dev < n ? *n_dev : n;
  if (i >= n) return;
  const int32_t e = pos[i];
  if (e < (int32_t)T.n || (flag && !flag[i]) || (ops && ops[i] != VS_OP_ERASE)) return;
  push_free(T, (uint32_t)e);
}

// ---- ordered compaction of live entries (snapshot_keys / extract_batch)

__global__ void __launch_bounds__(256) k_chunk_count(TableView T, uint32_t cap, uint32_t* __restrict__ counts) {
  const uint64_t base = (uint64_t)blockIdx.x * kChunk;
  uint32_t c = 0;
  for (uint32_t j = threadIdx.x; j < kChunk; j += blockDim.x) {
    const uint64_t p = base + j;
    if (p < cap) c += (T.e[p].meta & kOcc) ? 1u : 0u;
  }
  __shared__ uint32_t red[8];
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane_id() == 0) red[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s = 0;
    for (int w = 0; w < 8; ++w) s += red[w];
    counts[blockIdx.x] = s;
  }
}

// Single-CTA exclusive scan of a u32 array into u64 offsets[0..n].
__global__ void __launch_bounds__(1024) k_scan_u32(const uint32_t* __restrict__ in, uint64_t n,
                                                   uint64_t* __restrict__ out) {
  __shared__ uint64_t warp_sums[32];
  __shared__ uint64_t carry_s;
  if (threadIdx.x == 0) carry_s = 0;
  __syncthreads();
  for (uint64_t base = 0; base < n; base += 1024) {
    const uint64_t i = base + threadIdx.x;
    const uint64_t v = i < n ? in[i] : 0;
    uint64_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
      const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if ((int)lane_id() >= o) x += y;
    }
    if (lane_id() == 31) warp_sums[threadIdx.x >> 5] = x;
    __syncthreads();
    if (threadIdx.x < 32) {
      uint64_t w = warp_sums[threadIdx.x];
      for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if ((int)lane_id() >= o) w += y;
      }
      warp_sums[threadIdx.x] = w;  // inclusive
    }
    __syncthreads();
    const uint64_t carry = carry_s;
    const uint64_t wpre = (threadIdx.x >> 5) ? warp_sums[(threadIdx.x >> 5) - 1] : 0;
    if (i < n) out[i] = carry + wpre + x - v;
    __syncthreads();
    if (threadIdx.x == 0) carry_s = carry + warp_sums[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[n] = carry_s;
}

__global__ void __launch_bounds__(256) k_chunk_write(TableView T, uint32_t cap, const uint64_t* __restrict__ offsets,
                                                     int32_t* __restrict__ keys_out, int32_t* __restrict__ pos_out,
                                                     uint64_t out_cap) {
  __shared__ uint32_t wcnt[8];
  const uint64_t base = (uint64_t)blockIdx.x * kChunk;
  uint64_t running = offsets[blockIdx.x];
  const uint32_t warp = threadIdx.x >> 5;
  for (uint32_t j = 0; j < kChunk; j += 256) {
    const uint64_t p = base + j + threadIdx.x;
    int4 s = make_int4(0, 0, 0, 0);
    bool occ = false;
    if (p < cap) {
      s = ld_entry(T.e + p);
      occ = ((uint32_t)s.w & kOcc) != 0;
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, occ);
    if (lane_id() == 0) wcnt[warp] = __popc(bal);
    __syncthreads();
    uint32_t before = 0, total = 0;
    for (uint32_t w = 0; w < 8; ++w) {
      const uint32_t c = wcnt[w];
      before += (w < warp) ? c : 0;
      total += c;
    }
    if (occ) {
      const uint64_t o = running + before + __popc(bal & lanemask_lt());
      if (o < out_cap) {
        if (keys_out) {
          keys_out[3 * o] = s.x;
          keys_out[3 * o + 1] = s.y;
          keys_out[3 * o + 2] = s.z;
        }
        if (pos_out) pos_out[o] = (int32_t)p;
      }
    }
    running += total;
    __syncthreads();
  }
}

__global__ void k_sum_size(Ctl* ctl) {
  long long v = threadIdx.x < kSizeStripes ? ctl->size[threadIdx.x * kSizeStride] : 0;
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (threadIdx.x == 0) ctl->size_sum = (unsigned long long)(v < 0 ? 0 : v);
}

__global__ void k_copy_total(const uint64_t* __restrict__ offsets, uint32_t nchunks, uint64_t* __restrict__ n_dev) {
  *n_dev = offsets[nchunks];
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// extract_batch selection (concurrent_hash.py:387-399): rotate the ascending
// list of live positions at a random start and take the first max_n.
__global__ void k_extract_select(TableView T, uint32_t cap, const int32_t* __restrict__ pos,
                                 const uint64_t* __restrict__ total_p, uint64_t max_n, uint64_t seed,
                                 int32_t* __restrict__ keys_out, uint64_t* __restrict__ n_out) {
  __shared__ uint64_t split_s;
  const uint64_t total = *total_p;
  const uint64_t m = total < max_n ? total : max_n;
  if (threadIdx.x == 0) {
    const uint32_t start = (uint32_t)(splitmix64(seed) % cap);
    uint64_t lo = 0, hi = total;  // first index with pos >= start (np.searchsorted)
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if ((uint32_t)pos[mid] < start) lo = mid + 1; else hi = mid;
    }
    split_s = lo;
    if (blockIdx.x == 0) *n_out = m;
  }
  __syncthreads();
  const uint64_t split = split_s;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t k = split + j;
    if (k >= total) k -= total;
    const int4 s = ld_entry(T.e + pos[k]);
    keys_out[3 * j] = s.x;
    keys_out[3 * j + 1] = s.y;
    keys_out[3 * j + 2] = s.z;
  }
}

// ---- audit (white-box invariants; tests only)

__global__ void k_audit(TableView T, uint32_t cap, uint8_t* __restrict__ reach, unsigned long long* __restrict__ out) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  // chains: mark reachable excess entries
  for (uint64_t b = tid; b < T.n; b += stride) {
    uint32_t meta = T.e[b].meta;
    uint32_t hops = 0;
    while ((meta & kNext) && hops < T.excess + 1) {
      const uint32_t e = T.n + (meta & kNext) - 1;
      if (reach[e]) atomicAdd(&out[6], 1ull);  // reached twice: chains merged
      reach[e] = 1;
      atomicAdd(&out[1], 1ull);
      meta = T.e[e].meta;
      ++hops;
    }
  }
  // live entries: unique and reachable from their own bucket
  for (uint64_t p = tid; p < cap; p += stride) {
    const Entry s = T.e[p];
    if (!(s.meta & kOcc)) continue;
    atomicAdd(&out[0], 1ull);
    const uint32_t b = bucket_of(T, s.x, s.y, s.z);
    uint32_t e = b, copies = 0, hops = 0;
    bool seen_self = false;
    for (;;) {
      const Entry c = T.e[e];
      if ((c.meta & kOcc) && c.x == s.x && c.y == s.y && c.z == s.z) {
        ++copies;
        if (e == p) seen_self = true;
      }
      if (!(c.meta & kNext) || ++hops > T.excess + 1) break;
      e = T.n + (c.meta & kNext) - 1;
    }
    if (copies != 1) atomicAdd(&out[3], 1ull);
    if (!seen_self) atomicAdd(&out[4], 1ull);
  }
}

__global__ void k_audit_free(TableView T, const uint8_t* __restrict__ reach, unsigned long long* __restrict__ out) {
  for (uint32_t s = blockIdx.x; s < T.stripes; s += gridDim.x) {
    const long long top = T.tops[(size_t)s * kTopStride];
    if (threadIdx.x == 0) atomicAdd(&out[2], (unsigned long long)(top < 0 ? 0 : top));
    for (long long j = threadIdx.x; j < top; j += blockDim.x) {
      const uint32_t e = T.free_stack[(size_t)s * T.stripe_cap + (size_t)j];
      if (e < T.n || e >= T.n + T.excess || reach[e]) atomicAdd(&out[5], 1ull);
    }
  }
}

// ------------------------------------------------------------ host helpers

void launch_recycle(const TableView& v, const int32_t* pos, const uint8_t* flag, const uint8_t* ops,
                    const uint64_t* n_dev, uint64_t n, cudaStream_t s) {
  if (n == 0) return;
  { k_recycle<<<grid_for(n, 256), 256, 0, s>>>(v, pos, flag, ops, n_dev, n); vsb::count_launch(); }
}

vs_status erase_device_count(vs_table* t, const int32_t* keys, const uint64_t* n_dev, uint64_t max_n,
                             cudaStream_t s) {
  if (max_n == 0) return VS_OK;
  int32_t* idx = nullptr;
  VS_CK(cudaMallocAsync((void**)&idx, sizeof(int32_t) * max_n, s));
  const TableView v = t->next_view();
  { k_erase<<<grid_for(max_n, kOpBlock), kOpBlock, 0, s>>>(v, keys, max_n, n_dev, idx); vsb::count_launch(); }
  launch_recycle(v, idx, nullptr, nullptr, n_dev, max_n, s);
  cudaFreeAsync(idx, s);
  VS_CK_LAUNCH("erase_device_count");
  return VS_OK;
}

static vs_status compact_live(vs_table* t, int32_t* keys_out, int32_t* pos_out, uint64_t cap_out, cudaStream_t s) {
  const TableView v = t->view();
  { k_chunk_count<<<t->nchunks, 256, 0, s>>>(v, t->cap, t->chunk_counts); vsb::count_launch(); }
  { k_scan_u32<<<1, 1024, 0, s>>>(t->chunk_counts, t->nchunks, t->chunk_offsets); vsb::count_launch(); }
  { k_chunk_write<<<t->nchunks, 256, 0, s>>>(v, t->cap, t->chunk_offsets, keys_out, pos_out, cap_out); vsb::count_launch(); }
  VS_CK_LAUNCH("compact_live");
  return VS_OK;
}

}  // namespace vsb

using namespace vsb;

// ------------------------------------------------------------------ C ABI

extern "C" {

const char* vs_last_error(void) { return g_last_error.c_str(); }
int32_t vs_abi_version(void) { return 2; }  // 2: faces argument of the MC encoders, n_dev of vs_stream_insert_many

uint64_t vs_launch_count(void) { return g_launches.load(); }

vs_status vs_profile_begin(void) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  for (auto& r : g_prof_recs) {
    g_ev_pool.push_back(r.a);
    g_ev_pool.push_back(r.b);
  }
  g_prof_recs.clear();
#if VSB_PROF_RESERVE
  // event creation inside a timed region (~2 per profiled launch) costs host
  // time on the launch path: create the region's events up front
  while (g_ev_pool.size() < (size_t)VSB_PROF_RESERVE) {
    cudaEvent_t e = nullptr;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    g_ev_pool.push_back(e);
  }
#endif
  g_prof_on = true;
  g_prof_launch0 = g_launches.load();
  return VS_OK;
}

vs_status vs_profile_end(double ms_host[4], uint64_t count_host[4], uint64_t* launches_host) {
  std::lock_guard<std::mutex> g(g_prof_mu);
  g_prof_on = false;
  for (int i = 0; i < 4; ++i) {
    if (ms_host) ms_host[i] = 0.0;
    if (count_host) count_host[i] = 0;
  }
  for (auto& r : g_prof_recs) {
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return cuda_status(e, "vs_profile_end");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    if (r.tag >= 0 && r.tag < 4) {
      if (ms_host) ms_host[r.tag] += ms;
      if (count_host) count_host[r.tag] += 1;
    }
    g_ev_pool.push_back(r.a);
    g_ev_pool.push_back(r.b);
  }
  g_prof_recs.clear();
  if (launches_host) *launches_host = g_launches.load() - g_prof_launch0;
  return VS_OK;
}

vs_status vs_hash_keys(const int32_t* keys, uint64_t n, uint32_t bucket_count, uint32_t* out, vs_stream_t stream) {
  if (bucket_count < 1) {
    set_error("bucket_count must be >= 1");
    return VS_ERR_INVALID;
  }
  if (n == 0) return VS_OK;
  { k_hash_keys<<<grid_for(n, 256), 256, 0, (cudaStream_t)stream>>>(keys, n, bucket_count, out); vsb::count_launch(); }
  VS_CK_LAUNCH("k_hash_keys");
  return VS_OK;
}

// Scratch buffers of the batched calls come from the stream-ordered
// allocator; keep freed pool memory mapped (release threshold = max) so a
// large call does not pay page mapping again after every synchronisation.
static void keep_pool_resident(int device) {
  static bool done[64] = {false};
  if (device < 0 || device >= 64 || done[device]) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done[device] = true;
}

vs_status vs_table_create(uint64_t bucket_count, uint64_t excess_capacity, int device, vs_table** out) {
  if (!out) {
    set_error("out is NULL");
    return VS_ERR_INVALID;
  }
  *out = nullptr;
  if (bucket_count < 1) {
    set_error("bucket_count must be >= 1");
    return VS_ERR_INVALID;
  }
  if (excess_capacity < 1) {
    set_error("excess_capacity must be >= 1");
    return VS_ERR_INVALID;
  }
  if (excess_capacity > kNext - 1 || bucket_count + excess_capacity >= (1ull << 31)) {
    set_error("table too large: need excess < 2^29 and bucket_count + excess < 2^31");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(device);
  keep_pool_resident(device);
  vs_table* t = new vs_table();
  t->device = device;
  t->n = (uint32_t)bucket_count;
  t->excess = (uint32_t)excess_capacity;
  t->cap = t->n + t->excess;
  {
    uint32_t st = t->excess / kStripeMinEntries;
    st = st < kMinStripes ? kMinStripes : st > kMaxStripes ? kMaxStripes : st;
    t->stripes = t->excess < st ? t->excess : st;
  }
  t->stripe_cap = (t->excess + t->stripes - 1) / t->stripes;
  t->magic = fastmod_magic(t->n);
  t->nchunks = (t->cap + kChunk - 1) / kChunk;
  cudaError_t err = cudaSuccess;
  auto A = [&](void** p, size_t bytes) {
    if (err == cudaSuccess) err = cudaMalloc(p, bytes);
  };
  A((void**)&t->e, sizeof(Entry) * (size_t)t->cap);
  A((void**)&t->free_stack, sizeof(uint32_t) * (size_t)t->stripes * t->stripe_cap);
  A((void**)&t->tops, sizeof(long long) * (size_t)t->stripes * kTopStride);
  A((void**)&t->claim, sizeof(unsigned long long) * (size_t)t->cap);
  A((void**)&t->dupbits, sizeof(uint32_t) * (size_t)(t->cap / 32 + 1));
  A((void**)&t->ctl, sizeof(Ctl));
  A((void**)&t->chunk_counts, sizeof(uint32_t) * (size_t)t->nchunks);
  A((void**)&t->chunk_offsets, sizeof(uint64_t) * ((size_t)t->nchunks + 1));
  if (err != cudaSuccess) {
    vs_table_destroy(t);
    return cuda_status(err, "vs_table_create: cudaMalloc");
  }
  vs_status st = vs_table_clear(t, nullptr);
  if (st == VS_OK) {
    cudaError_t e2 = cudaStreamSynchronize(nullptr);
    if (e2 != cudaSuccess) st = cuda_status(e2, "vs_table_create: sync");
  }
  if (st != VS_OK) {
    vs_table_destroy(t);
    return st;
  }
  *out = t;
  return VS_OK;
}

vs_status vs_table_destroy(vs_table* t) {
  if (!t) return VS_OK;
  DeviceGuard g(t->device);
  cudaFree(t->e);
  cudaFree(t->free_stack);
  cudaFree(t->tops);
  cudaFree(t->claim);
  cudaFree(t->dupbits);
  cudaFree(t->ctl);
  cudaFree(t->chunk_counts);
  cudaFree(t->chunk_offsets);
  cudaFree(t->pos_work);
  if (t->stage_host) cudaFreeHost(t->stage_host);
  if (t->side) cudaStreamDestroy(t->side);
  if (t->ev_fork) cudaEventDestroy(t->ev_fork);
  if (t->ev_join) cudaEventDestroy(t->ev_join);
  if (t->tick_mem) cudaFree(t->tick_mem);
  delete t;
  return VS_OK;
}

vs_status vs_table_info(const vs_table* t, uint64_t* nb, uint64_t* ex, uint64_t* cap) {
  if (!t) {
    set_error("table is NULL");
    return VS_ERR_INVALID;
  }
  if (nb) *nb = t->n;
  if (ex) *ex = t->excess;
  if (cap) *cap = t->cap;
  return VS_OK;
}

static vs_status check_batch(const vs_table* t, uint64_t n) {
  if (!t) {
    set_error("table is NULL");
    return VS_ERR_INVALID;
  }
  if (n >= (1ull << 31)) {
    set_error("batch too large (n must be < 2^31)");
    return VS_ERR_INVALID;
  }
  return VS_OK;
}

static vs_status table_insert(vs_table* t, const int32_t* keys, uint64_t n, const uint64_t* n_dev, uint8_t* created,
                              int32_t* index, vs_stream_t stream) {
  vs_status st = check_batch(t, n);
  if (st != VS_OK || n == 0) return st;
  if (!keys || !created || !index) {
    set_error("keys/created/index must be non-NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  const TableView v = t->next_view();
  // PDL-linked to its producer and to the post pass (no profiling events in
  // between: the bench times the mixed-op kernel, not inserts)
  { VS_CK(launch_pdl(k_insert, grid_for(n, kOpBlock), kOpBlock, 0, s, v, keys, n, n_dev, created, index)); vsb::count_launch(); }
  { VS_CK(launch_post(v, keys, nullptr, n, created, index, s)); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_table_insert");
  return VS_OK;
}

vs_status vs_table_insert(vs_table* t, const int32_t* keys, uint64_t n, uint8_t* created, int32_t* index,
                          vs_stream_t stream) {
  return table_insert(t, keys, n, nullptr, created, index, stream);
}

vs_status vs_table_insert_bounded(vs_table* t, const int32_t* keys, uint64_t n, const uint64_t* n_dev,
                                  uint8_t* created, int32_t* index, vs_stream_t stream) {
  if (!n_dev) {
    set_error("n_dev must be non-NULL");
    return VS_ERR_INVALID;
  }
  return table_insert(t, keys, n, n_dev, created, index, stream);
}

vs_status vs_table_find(vs_table* t, const int32_t* keys, uint64_t n, uint8_t* found, int32_t* index,
                        vs_stream_t stream) {
  vs_status st = check_batch(t, n);
  if (st != VS_OK || n == 0) return st;
  if (!keys || !found || !index) {
    set_error("keys/found/index must be non-NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  {
    ProfScope prof(0, s);
    { k_find<<<grid_for(n, kOpBlock), kOpBlock, 0, s>>>(t->view(), keys, n, found, index); vsb::count_launch(); }
  }
  VS_CK_LAUNCH("vs_table_find");
  return VS_OK;
}

vs_status vs_table_erase(vs_table* t, const int32_t* keys, uint64_t n, uint8_t* erased, int32_t* index,
                         vs_stream_t stream) {
  vs_status st = check_batch(t, n);
  if (st != VS_OK || n == 0) return st;
  if (!keys) {
    set_error("keys must be non-NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* idx = index;
  if (!idx) VS_CK(cudaMallocAsync((void**)&idx, sizeof(int32_t) * n, s));
  const TableView v = t->next_view();
  {
    ProfScope prof(0, s);
    { k_erase_claim<<<grid_for(n, kOpBlock), kOpBlock, 0, s>>>(v, keys, n, idx); vsb::count_launch(); }
    { k_erase_win<<<grid_for(n, kOpBlock), kOpBlock, 0, s>>>(v, keys, n, erased, idx); vsb::count_launch(); }
  }
  // vacated excess entries go back in a separate launch: pushing them from
  // k_erase_win itself was measured to leave freed entries reachable
  // (scripts/c1_loop.py: 3-5 per config-1 cycle), so it stays separate
  launch_recycle(v, idx, nullptr, nullptr, nullptr, n, s);
  if (!index) cudaFreeAsync(idx, s);
  VS_CK_LAUNCH("vs_table_erase");
  return VS_OK;
}

vs_status vs_table_apply(vs_table* t, const int32_t* keys, const uint8_t* ops, uint64_t n, uint8_t* result,
                         int32_t* index, vs_stream_t stream) {
  vs_status st = check_batch(t, n);
  if (st != VS_OK || n == 0) return st;
  if (!keys || !ops || !result || !index) {
    set_error("keys/ops/result/index must be non-NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  const TableView v = t->next_view();
  {
    ProfScope prof(0, s);
    { VS_CK(launch_apply(v, keys, ops, n, result, index, s)); vsb::count_launch(); }
  }
  { VS_CK(launch_post(v, keys, ops, n, result, index, s)); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_table_apply");
  return VS_OK;
}

vs_status vs_table_single(vs_table* t, int op, const int32_t key_host[3], uint8_t* result_host,
                           int32_t* index_host, vs_stream_t stream) {
  if (!t || !key_host || !result_host || !index_host || op < 0 || op > 2) {
    set_error("table/key/result/index must be non-NULL and op in {0,1,2}");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (!t->stage_host) {
    // mapped pinned staging: the kernel writes the result straight into host
    // memory, so a per-key call is one launch + a spin on that word
    VS_CK(cudaHostAlloc((void**)&t->stage_host, 32, cudaHostAllocMapped));
    VS_CK(cudaHostGetDevicePointer((void**)&t->stage_dev, t->stage_host, 0));
    // pinned blocks are recycled across tables: clear the result word so a
    // stale value from a previous owner can never carry this table's seq
    memset(t->stage_host, 0, 32);
    t->stage_seq = 0;
  }
  uint32_t seq = (++t->stage_seq) & 0x7FFFFFFFu;
  if (seq == 0) seq = (++t->stage_seq) & 0x7FFFFFFFu;  // 0 is the cleared word's
  volatile unsigned long long* word = (volatile unsigned long long*)t->stage_host;
  { k_single<<<1, 1, 0, s>>>(t->next_view(), key_host[0], key_host[1], key_host[2], (uint8_t)op,
                            (unsigned long long*)t->stage_dev, seq); vsb::count_launch(); }
  VS_CK(cudaGetLastError());
  // Wait by spinning on the word the kernel writes: a per-key call then
  // costs the launch and the op itself, not a stream synchronisation.  A busy
  // stream (the key queued behind long work) or a fault falls back to the
  // blocking synchronisation after ~50 us.
  const auto t0 = std::chrono::steady_clock::now();
  bool spun = false;
  while (((*word >> 32) & 0x7FFFFFFFull) != seq) {
#if defined(__x86_64__)
    __builtin_ia32_pause();
#endif
    if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(50)) {
      spun = true;
      break;
    }
  }
  if (spun) VS_CK(cudaStreamSynchronize(s));
  const unsigned long long w = *word;
  *index_host = (int32_t)(uint32_t)(w & 0xFFFFFFFFull);
  *result_host = (uint8_t)(w >> 63);
  if (op == VS_OP_INSERT && *index_host < 0) {
    unsigned int zero = 0;
    VS_CK(cudaMemcpy(&t->ctl->error, &zero, sizeof(zero), cudaMemcpyHostToDevice));
    set_error("excess list exhausted (" + std::to_string(t->excess) + " entries)");
    return VS_ERR_CAPACITY;
  }
  return VS_OK;
}

vs_status vs_table_check(vs_table* t, vs_stream_t stream) {
  if (!t) {
    set_error("table is NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  unsigned int err = 0;
  VS_CK(cudaMemcpyAsync(&err, &t->ctl->error, sizeof(err), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
  VS_CK(cudaStreamSynchronize((cudaStream_t)stream));
  if (err & 1u) {
    VS_CK(cudaMemsetAsync(&t->ctl->error, 0, sizeof(unsigned int), (cudaStream_t)stream));
    VS_CK(cudaStreamSynchronize((cudaStream_t)stream));
    set_error("excess list exhausted (" + std::to_string(t->excess) + " entries)");
    return VS_ERR_CAPACITY;
  }
  return VS_OK;
}

vs_status vs_table_size(vs_table* t, uint64_t* size_dev, uint64_t* size_host, vs_stream_t stream) {
  if (!t) {
    set_error("table is NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  { k_sum_size<<<1, 32, 0, s>>>(t->ctl); vsb::count_launch(); }
  if (size_dev) VS_CK(cudaMemcpyAsync(size_dev, &t->ctl->size_sum, 8, cudaMemcpyDeviceToDevice, s));
  if (size_host) {
    VS_CK(cudaMemcpyAsync(size_host, &t->ctl->size_sum, 8, cudaMemcpyDeviceToHost, s));
    VS_CK(cudaStreamSynchronize(s));
  }
  return VS_OK;
}

vs_status vs_table_free_count(vs_table* t, uint64_t* free_host, vs_stream_t stream) {
  if (!t || !free_host) {
    set_error("table/free_host is NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  std::vector<long long> tops((size_t)t->stripes * kTopStride);
  VS_CK(cudaMemcpyAsync(tops.data(), t->tops, sizeof(long long) * tops.size(), cudaMemcpyDeviceToHost,
                        (cudaStream_t)stream));
  VS_CK(cudaStreamSynchronize((cudaStream_t)stream));
  uint64_t sum = 0;
  for (uint32_t s = 0; s < t->stripes; ++s) {
    const long long v = tops[(size_t)s * kTopStride];
    sum += v < 0 ? 0 : (uint64_t)v;
  }
  *free_host = sum;
  return VS_OK;
}

vs_status vs_table_clear(vs_table* t, vs_stream_t stream) {
  if (!t) {
    set_error("table is NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  VS_CK(cudaMemsetAsync(t->e, 0, sizeof(Entry) * (size_t)t->cap, s));
  VS_CK(cudaMemsetAsync(t->claim, 0xFF, sizeof(unsigned long long) * (size_t)t->cap, s));
  VS_CK(cudaMemsetAsync(t->dupbits, 0, sizeof(uint32_t) * (size_t)(t->cap / 32 + 1), s));
  t->epoch = 0;
  const TableView v = t->view();
  const unsigned g_init = grid_for(t->excess, 256) < 4096 ? grid_for(t->excess, 256) : 4096;
  { k_init_free<<<g_init, 256, 0, s>>>(v); vsb::count_launch(); }
  { k_reset_ctl<<<1, 32, 0, s>>>(v); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_table_clear");
  return VS_OK;
}

vs_status vs_table_snapshot(vs_table* t, int32_t* keys_out, int32_t* index_out, uint64_t cap, uint64_t* n_dev,
                            vs_stream_t stream) {
  if (!t || !n_dev) {
    set_error("table/n_dev is NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  vs_status st = compact_live(t, keys_out, index_out, cap, s);
  if (st != VS_OK) return st;
  { k_copy_total<<<1, 1, 0, s>>>(t->chunk_offsets, t->nchunks, n_dev); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_table_snapshot");
  return VS_OK;
}

vs_status vs_table_extract(vs_table* t, uint64_t max_n, uint64_t seed, int32_t* keys_out, uint64_t* n_dev,
                           vs_stream_t stream) {
  if (!t || !n_dev) {
    set_error("table/n_dev is NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  if (max_n == 0) {
    VS_CK(cudaMemsetAsync(n_dev, 0, 8, s));
    return VS_OK;
  }
  if (!t->pos_work) VS_CK(cudaMalloc((void**)&t->pos_work, sizeof(int32_t) * (size_t)t->cap));
  vs_status st = compact_live(t, nullptr, t->pos_work, t->cap, s);
  if (st != VS_OK) return st;
  const uint64_t m = max_n < t->cap ? max_n : t->cap;
  unsigned grid = grid_for(m, 256);
  if (grid > 1184) grid = 1184;
  { k_extract_select<<<grid, 256, 0, s>>>(t->view(), t->cap, t->pos_work, t->chunk_offsets + t->nchunks, max_n, seed,
                                        keys_out, n_dev); vsb::count_launch(); }
  VS_CK_LAUNCH("k_extract_select");
  return erase_device_count(t, keys_out, n_dev, m, s);
}

vs_status vs_table_probe_sol(vs_table* t, uint64_t n, int hops, uint8_t* out, vs_stream_t stream) {
  if (!t || (n && !out) || hops < 1 || hops > 16) {
    set_error("vs_table_probe_sol: bad arguments");
    return VS_ERR_INVALID;
  }
  if (n == 0) return VS_OK;
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  const TableView v = t->view();
  {
    ProfScope prof(3, s);
    k_probe_sol<<<apply_grid(n), kOpBlock, 0, s>>>(v, n, hops, out);
    vsb::count_launch();
  }
  VS_CK_LAUNCH("vs_table_probe_sol");
  return VS_OK;
}

vs_status vs_table_audit(vs_table* t, uint64_t out_host[6], vs_stream_t stream) {
  if (!t || !out_host) {
    set_error("table/out is NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  cudaStream_t s = (cudaStream_t)stream;
  uint8_t* reach = nullptr;
  unsigned long long* out = nullptr;
  VS_CK(cudaMalloc((void**)&reach, t->cap));
  VS_CK(cudaMalloc((void**)&out, 8 * 8));
  VS_CK(cudaMemsetAsync(reach, 0, t->cap, s));
  VS_CK(cudaMemsetAsync(out, 0, 64, s));
  { k_audit<<<1184, 256, 0, s>>>(t->view(), t->cap, reach, out); vsb::count_launch(); }
  { k_audit_free<<<148, 256, 0, s>>>(t->view(), reach, out); vsb::count_launch(); }
  unsigned long long h[8];
  VS_CK(cudaMemcpyAsync(h, out, 64, cudaMemcpyDeviceToHost, s));
  VS_CK(cudaStreamSynchronize(s));
  cudaFree(reach);
  cudaFree(out);
  out_host[0] = h[0];
  out_host[1] = h[1];
  out_host[2] = h[2];
  out_host[3] = h[3];
  out_host[4] = h[4];
  out_host[5] = h[5] + h[6];
  return VS_OK;
}

}  // extern "C"

namespace vsb {
vs_status table_put_insert(vs_table* t, const int32_t* keys, uint64_t n, uint8_t* created, int32_t* index,
                           cudaStream_t s, TableView* view_out) {
  vs_status st = check_batch(t, n);
  if (st != VS_OK || n == 0) return st;
  DeviceGuard g(t->device);
  const TableView v = t->next_view();
  *view_out = v;
  { VS_CK(launch_pdl(k_insert_t<true>, grid_for(n, kOpBlock), kOpBlock, 0, s, v, keys, n, (const uint64_t*)nullptr, created, index)); vsb::count_launch(); }
  VS_CK_LAUNCH("table_put_insert");
  return VS_OK;
}

vs_status table_insert_fresh(vs_table* t, const int32_t* keys, uint64_t n, const uint64_t* n_dev, uint8_t* created,
                             int32_t* index, cudaStream_t s) {
  vs_status st = check_batch(t, n);
  if (st != VS_OK || n == 0) return st;
  DeviceGuard g(t->device);
  const TableView v = t->next_view();
  { VS_CK(launch_pdl(k_insert, grid_for(n, kOpBlock), kOpBlock, 0, s, v, keys, n, n_dev, created, index)); vsb::count_launch(); }
  VS_CK_LAUNCH("table_insert_fresh");
  return VS_OK;
}
}  // namespace vsb
