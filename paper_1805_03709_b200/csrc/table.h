// table.h -- host-side table object and shared host helpers of libvsb200.
#pragma once
#include <cstdint>
#include <string>
#include <cuda_runtime.h>

#include "common.cuh"
#include "../../include/vsb200.h"

struct vs_table {
  int device = 0;
  uint32_t n = 0, excess = 0, cap = 0;
  uint32_t stripes = 1, stripe_cap = 1;
  vsb::Entry* e = nullptr;
  uint32_t* free_stack = nullptr;
  long long* tops = nullptr;
  unsigned long long* claim = nullptr;
  uint32_t* dupbits = nullptr;
  vsb::Ctl* ctl = nullptr;
  uint64_t magic = 0;
  uint32_t epoch = 0;  // launch epoch for the claim tags
  // ordered-compaction workspace (snapshot / extract)
  uint32_t nchunks = 0;
  uint32_t* chunk_counts = nullptr;
  uint64_t* chunk_offsets = nullptr;  // nchunks + 1
  int32_t* pos_work = nullptr;        // lazily allocated, cap entries
  uint8_t* stage_host = nullptr;      // pinned staging of the single-key path (32 B)
  uint8_t* stage_dev = nullptr;
  uint32_t stage_seq = 0;             // completion sequence of the single-key path
  // side stream + fork/join events of vs_server_tick (lazily created; the
  // TSDF map's table owns them)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // vs_server_tick's scratch (positions, created flags), grow-only and kept
  // between ticks: calls on one map are stream-ordered (they mutate it)
  char* tick_mem = nullptr;
  size_t tick_mem_bytes = 0;

  // view for ONE launch; next_epoch() gives it a fresh claim tag
  vsb::TableView view() const {
    vsb::TableView v;
    v.e = e;
    v.free_stack = free_stack;
    v.tops = tops;
    v.claim = claim;
    v.dupbits = dupbits;
    v.ctl = ctl;
    v.n = n;
    v.excess = excess;
    v.stripes = stripes;
    v.stripe_cap = stripe_cap;
    v.magic = magic;
    v.tag = (unsigned long long)(0xFFFFFFFFu - epoch) << 32;
    return v;
  }
  vsb::TableView next_view() {
    ++epoch;
    if (epoch == 0xFFFFFFFFu) epoch = 1;  // tags stay ordered for 4G launches; then reset below
    return view();
  }
};

namespace vsb {

constexpr uint32_t kChunk = 4096;  // entries per CTA in ordered compaction

void set_error(const std::string& msg);
vs_status cuda_status(cudaError_t err, const char* what);

// RAII: make `dev` current for the duration of a call.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Every kernel launch of the library is counted (bench.py reports the count
// of launches inside its timed region as "gpu_launches").
void count_launch();

// Event-timed scope around the dominant kernel of a call while profiling is
// on (vs_profile_begin/end).  Tags: 0 hash op kernel, 1 MC encode, 2 reserved
// (the stream insert chain is PDL-linked, so it is not bracketed), 3 other.
struct ProfScope {
  int tag;
  cudaStream_t s;
  void* start = nullptr;
  ProfScope(int tag, cudaStream_t s);
  ~ProfScope();
};

// internal entry points shared across translation units
// Push vacated excess positions (pos[i] >= n where flag[i] and, if ops is
// given, ops[i] == VS_OP_ERASE) back onto the striped free list.
void launch_recycle(const vsb::TableView& v, const int32_t* pos, const uint8_t* flag, const uint8_t* ops,
                    const uint64_t* n_dev, uint64_t n, cudaStream_t s);
vs_status erase_device_count(vs_table* t, const int32_t* keys, const uint64_t* n_dev, uint64_t max_n,
                             cudaStream_t s);
// Insert launch WITHOUT its post pass: positions final, created flags
// provisional (in-batch duplicates unresolved), created entries left FRESH --
// the caller clears FRESH on every returned position in a later launch of
// the same chain (vs_server_tick / tsdf_put fold it into their next kernel).
vs_status table_insert_fresh(vs_table* t, const int32_t* keys, uint64_t n, const uint64_t* n_dev,
                             uint8_t* created, int32_t* index, cudaStream_t s);
// The insert of a TSDF put: positions, no created resolution, each op claims
// its position for the row copy (highest op index wins); the launch's view
// (its claim tag) goes to *view_out for k_put_rows, which also settles FRESH.
vs_status table_put_insert(vs_table* t, const int32_t* keys, uint64_t n, uint8_t* created, int32_t* index,
                           cudaStream_t s, TableView* view_out);
// vs_mc_encode_keys_ex plus: clear FRESH on entry out_rows[i] of `fresh_e`
// (the MC map whose positions are the output rows) for every encoded block.
vs_status mc_encode_keys_clear(const vs_table* t, const uint8_t* pool, const uint8_t* faces, const int32_t* keys,
                               uint64_t n, const uint64_t* n_dev, const int32_t* out_rows, uint8_t* mc_out,
                               int8_t* q_out, Entry* fresh_e, cudaStream_t s);

}  // namespace vsb

#define VS_CK(call)                                            \
  do {                                                         \
    cudaError_t _e = (call);                                   \
    if (_e != cudaSuccess) return vsb::cuda_status(_e, #call); \
  } while (0)

#define VS_CK_LAUNCH(what) VS_CK(cudaGetLastError())
