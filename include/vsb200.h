/*
 * vsb200.h -- C ABI of the B200-native SLAMCast hot path (libvsb200.so).
 *
 * This is the drop-in boundary for three pieces of the reference package
 * `voxelstream` (pure Python, /root/reference/pkg/src/voxelstream):
 *
 *   1. the concurrent block hash set / map      (concurrent_hash.py:49-491)
 *   2. the Marching-Cubes block encoder         (mc_encoding.py:83-172,
 *      TSDF block layout voxel_model.py:23-72)
 *   3. the per-client stream-set update         (server.py:49-95, 221-249,
 *      299-315, 425-436)
 *
 * Conventions
 *   - Every pointer argument is a DEVICE pointer unless its name ends in
 *     `_host`.  Keys are int32[n][3] (x, y, z), little-endian, exactly the
 *     wire layout `<3i` (wire.py:37).
 *   - Every call is asynchronous on the given CUDA stream (pass NULL for the
 *     legacy default stream) unless documented as synchronous.
 *   - All operations on ONE table must be stream-ordered (one stream, or
 *     streams ordered with events): erased excess entries are recycled into
 *     the free-list stack only between launches, which is what makes the
 *     lock-free readers inside a launch safe ("hash").
 *     Within a launch, any mix of insert / find / erase on any keys is
 *     thread-safe and keeps keys unique.
 *   - Status codes are returned, never thrown.  vs_last_error() gives a
 *     thread-local message for the last non-OK status.
 */
#ifndef VSB200_H
#define VSB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *vs_stream_t; /* == cudaStream_t */

typedef int32_t vs_status;
enum {
  VS_OK = 0,
  VS_ERR_CAPACITY = 1, /* CapacityExhausted (concurrent_hash.py:45-46,193-197) */
  VS_ERR_INVALID = 2,  /* ValueError (concurrent_hash.py:96-101)             */
  VS_ERR_CUDA = 3,     /* CUDA runtime failure                               */
  VS_ERR_OVERFLOW = 4  /* an output buffer was too small; output truncated   */
};

/* Op codes of vs_table_apply (mixed batches). */
enum { VS_OP_INSERT = 0, VS_OP_FIND = 1, VS_OP_ERASE = 2 };

/* Sizes of the data formats (voxel_model.py:23-31, mc_encoding.py:34-37). */
#define VS_BLOCK_VOXELS 512
#define VS_TSDF_BLOCK_BYTES 6144 /* 512 x {f32 tsdf, f32 weight, u8 rgb[3], u8 pad} */
#define VS_MC_BLOCK_BYTES 2048   /* 512 x {u8 index, u8 rgb[3]}                      */

const char *vs_last_error(void);
int32_t vs_abi_version(void);

/* Profiling (bench.py only).  Between begin and end, the dominant kernel of
 * every call is bracketed with CUDA events on the call's stream; end
 * synchronises those events and returns, per tag (0 hash op kernel, 1 MC
 * encode, 2 multi-set stream insert, 3 reserved), the summed kernel time in
 * ms and the number of launches, plus the number of ALL library kernel
 * launches issued in between. */
vs_status vs_profile_begin(void);
vs_status vs_profile_end(double ms_host[4], uint64_t count_host[4], uint64_t *launches_host);
/* Kernels this library has launched since it was loaded (no events: for
 * host-paced timed regions where profiling events would add host work). */
uint64_t vs_launch_count(void);

/* ---------------------------------------------------------------- hash --- */

/* hash_key (concurrent_hash.py:49-59): bucket = (x*p1 ^ y*p2 ^ z*p3) mod n,
 * products wrapping in uint32.  out[i] in [0, bucket_count). */
vs_status vs_hash_keys(const int32_t *keys, uint64_t n, uint32_t bucket_count,
                       uint32_t *out, vs_stream_t stream);

/* One table serves both BlockHashSet and BlockHashMap (the reference shares
 * _HashCore, concurrent_hash.py:85-120).  Map payloads live in caller-owned
 * arrays indexed by the returned entry position, exactly as the reference's
 * parallel `_values` list (concurrent_hash.py:112; SPEC.md "Map payloads live
 * in a parallel array indexed like entries").  Positions are stable while a
 * key is present (concurrent_hash.py:8-13).
 *
 * bucket_count >= 1, excess_capacity >= 1 (else VS_ERR_INVALID, like
 * concurrent_hash.py:96-99); bucket_count + excess_capacity < 2^31 and
 * excess_capacity < 2^29 (entry-offset field width). */
typedef struct vs_table vs_table;

vs_status vs_table_create(uint64_t bucket_count, uint64_t excess_capacity,
                          int device, vs_table **out);
vs_status vs_table_destroy(vs_table *t);
vs_status vs_table_info(const vs_table *t, uint64_t *bucket_count_host,
                        uint64_t *excess_capacity_host, uint64_t *capacity_host);

/* _insert_pos / BlockHashSet.insert / BlockHashMap.insert
 * (concurrent_hash.py:159-208, 361-364, 418-425).  created[i] = 1 for the
 * LOWEST input index among in-batch duplicates of a key that was absent
 * before the batch (= sequential replay); index[i] = entry position.  An op
 * that needed an excess entry when the free list was empty gets index -1,
 * created 0, and the table's sticky capacity flag is raised (see
 * vs_table_check).  The table is unchanged for that op. */
vs_status vs_table_insert(vs_table *t, const int32_t *keys, uint64_t n,
                          uint8_t *created, int32_t *index, vs_stream_t stream);

/* Same, for the first min(*n_dev, n) keys only (n_dev: device uint64, e.g.
 * a count produced by a previous kernel): no host synchronisation; ops past
 * the count get created 0 and index -1. */
vs_status vs_table_insert_bounded(vs_table *t, const int32_t *keys, uint64_t n, const uint64_t *n_dev,
                                  uint8_t *created, int32_t *index, vs_stream_t stream);

/* _find / __contains__ / BlockHashMap.get (concurrent_hash.py:146-157,
 * 297-298, 449-460).  Read-only.  index[i] = position or -1. */
vs_status vs_table_find(vs_table *t, const int32_t *keys, uint64_t n,
                        uint8_t *found, int32_t *index, vs_stream_t stream);

/* remove (concurrent_hash.py:251-295).  erased[i] = 1 if the key was present;
 * index[i] = the position it occupied (so map payload slots can be cleared),
 * else -1. */
vs_status vs_table_erase(vs_table *t, const int32_t *keys, uint64_t n,
                         uint8_t *erased, int32_t *index, vs_stream_t stream);

/* Mixed batch in ONE launch: ops[i] in {VS_OP_INSERT, VS_OP_FIND, VS_OP_ERASE};
 * result[i] = created / found / erased.  Per-op results equal a sequential
 * replay when no key whose membership changes in the batch appears in any
 * other op except duplicate inserts of itself; any batch
 * is safe (keys stay unique). */
vs_status vs_table_apply(vs_table *t, const int32_t *keys, const uint8_t *ops,
                         uint64_t n, uint8_t *result, int32_t *index,
                         vs_stream_t stream);

/* SYNCHRONOUS single-key op (the reference's per-key API: insert / remove /
 * __contains__, concurrent_hash.py:297-298,361-364,251-295) through pinned
 * staging: key_host[3] in, *result_host (created/found/erased) and
 * *index_host out.  An insert that finds the excess list empty returns
 * VS_ERR_CAPACITY with the table unchanged. */
vs_status vs_table_single(vs_table *t, int op, const int32_t key_host[3],
                          uint8_t *result_host, int32_t *index_host, vs_stream_t stream);

/* SYNCHRONOUS: returns VS_ERR_CAPACITY (and clears the flag) if any insert
 * since the last check hit an empty free list, else VS_OK. */
vs_status vs_table_check(vs_table *t, vs_stream_t stream);

/* approx_size (concurrent_hash.py:311-313): live-key count, device counter.
 * size_dev may be NULL; size_host (may be NULL) makes the call synchronous. */
vs_status vs_table_size(vs_table *t, uint64_t *size_dev, uint64_t *size_host,
                        vs_stream_t stream);
/* Free excess entries (len(free_stack)), synchronous. */
vs_status vs_table_free_count(vs_table *t, uint64_t *free_host, vs_stream_t stream);

/* clear (concurrent_hash.py:315-322): quiescent bulk reset. */
vs_status vs_table_clear(vs_table *t, vs_stream_t stream);

/* snapshot_keys / snapshot_items (concurrent_hash.py:300-309, 483-491):
 * live keys in ascending entry-position order.  Writes at most `cap` records;
 * *n_dev = number of live keys (may exceed cap -> VS_ERR_OVERFLOW is NOT
 * reported asynchronously; compare *n_dev with cap). index_out may be NULL. */
vs_status vs_table_snapshot(vs_table *t, int32_t *keys_out, int32_t *index_out,
                            uint64_t cap, uint64_t *n_dev, vs_stream_t stream);

/* extract_batch (concurrent_hash.py:366-402): remove and return up to max_n
 * keys, scanning occupied entries from a rotating start position derived from
 * `seed` (the reference uses random.randrange).  *n_dev = number returned. */
vs_status vs_table_extract(vs_table *t, uint64_t max_n, uint64_t seed,
                           int32_t *keys_out, uint64_t *n_dev, vs_stream_t stream);

/* Integrity check for tests (replaces the reference's white-box checks,
 * tests/test_concurrent_hash.py:113,124-126,379-383).  SYNCHRONOUS.
 * out_host[0] = live entries found by a full scan
 * out_host[1] = entries reachable from bucket chains (excess, any occupancy)
 * out_host[2] = free-list stack size
 * out_host[3] = duplicate live keys found (must be 0)
 * out_host[4] = live entries NOT reachable from their own bucket (must be 0)
 * out_host[5] = free-list entries that are also reachable (must be 0)  */
vs_status vs_table_audit(vs_table *t, uint64_t out_host[6], vs_stream_t stream);

/* Diagnostics (bench.py only): the speed of light of the op kernels' memory
 * pattern on THIS table's storage -- n threads in k_apply's launch shape,
 * each doing `hops` DEPENDENT random 16-byte entry loads (same load flavour
 * as a chain walk) and one result byte; no logic, no atomics.  out: device
 * uint8[n]. */
vs_status vs_table_probe_sol(vs_table *t, uint64_t n, int hops, uint8_t *out, vs_stream_t stream);

/* ------------------------------------------------------------ MC encode --- */

/* TSDF pool: caller-owned rows of VS_TSDF_BLOCK_BYTES in the wire layout
 * (TsdfBlock.to_bytes, voxel_model.py:55-60); row r at pool + r*6144, 16-byte
 * aligned.  nbr[i][c] = pool row of TSDF block key_i + (c&1, c>>1&1, c>>2&1)
 * or -1 if absent (c = 0 is the block itself).
 *
 * recompute_mc_block (mc_encoding.py:145-172) for n blocks:
 *   mc_out[i]  : 2048 B McBlock.to_bytes() (interleaved {index, r, g, b})
 *   q_out[i]   : 512 int8 quantised TSDF of block i (A17; NEW)
 *   counts[i]  : number of voxels with index != 0
 * Any of mc_out / q_out / counts may be NULL to skip that output.
 * faces (may be NULL): the pool's face bit-packs (vs_mc_faces), 48 B per
 * row, 16-byte aligned, current for every row a neighbour lookup can hit;
 * with them the halo of a block is seven 16-B reads instead of 217
 * scattered voxels.  Output is identical with or without. */
vs_status vs_mc_encode(const uint8_t *pool, const uint8_t *faces, const int32_t *nbr,
                       uint64_t n, uint8_t *mc_out, int8_t *q_out, uint32_t *counts,
                       vs_stream_t stream);

/* Same, but the neighbour rows come from hash lookups of keys[i] + delta in
 * `tsdf_table`, whose entry positions index `pool` (the TSDF map's parallel
 * payload array).  This is where the hash feeds the encoder. */
vs_status vs_mc_encode_keys(const vs_table *tsdf_table, const uint8_t *pool,
                            const uint8_t *faces, const int32_t *keys, uint64_t n,
                            uint8_t *mc_out, int8_t *q_out, uint32_t *counts,
                            vs_stream_t stream);

/* vs_mc_encode_keys plus three options (NEW):
 *   n_dev (may be NULL): only the first min(n, *n_dev) keys are encoded -- a
 *     device-produced count (vs_affected_dedup) needs no host sync;
 *   out_rows (may be NULL): block i's MC / quantised bytes go to row
 *     out_rows[i] of mc_out / q_out (e.g. the MC map's position of key i,
 *     so the encoder writes straight into a server's MC pool); rows < 0
 *     are skipped (e.g. an MC map insert that failed);
 *   fused compaction (cell_flat and cell_mc non-NULL): block i's
 *     non-empty cells in ascending flat index at [offsets[i], offsets[i] +
 *     counts[i]) of cell_flat / cell_mc, each range reserved with one atomic
 *     on the device counter *cursor (zeroed by the call; final value = total
 *     cells; at most cell_cap cells are written -- check *cursor <= cell_cap).
 *     Ranges follow reservation order; vs_mc_compact gives the exact-prefix
 *     layout from dense bytes. */
vs_status vs_mc_encode_keys_ex(const vs_table *tsdf_table, const uint8_t *pool,
                               const uint8_t *faces, const int32_t *keys, uint64_t n,
                               const uint64_t *n_dev, const int32_t *out_rows,
                               uint8_t *mc_out, int8_t *q_out,
                               uint32_t *counts, unsigned long long *cursor,
                               uint32_t *offsets, uint16_t *cell_flat, uint32_t *cell_mc,
                               uint64_t cell_cap, vs_stream_t stream);

/* Face bit-packs of pool rows (the halo side table of the encoder; NEW):
 * for rows[i] (or row i when rows is NULL), faces + 48*row receives the
 * inside/observed bits (the encoder's IEEE-bit predicates) of the row's
 * x = 0, y = 0 and z = 0 faces, each {inside lo, inside hi, observed lo,
 * observed hi} with bit y+8z / x+8z / x+8y.  Call it wherever rows change
 * (ingest, integration); rows < 0 are skipped. */
vs_status vs_mc_faces(const uint8_t *pool, const int32_t *rows, uint64_t n,
                      uint8_t *faces, vs_stream_t stream);

/* Neighbour table only: nbr_out[i][c] as defined above (8 batched finds). */
vs_status vs_mc_neighbors(const vs_table *tsdf_table, const int32_t *keys,
                          uint64_t n, int32_t *nbr_out, vs_stream_t stream);

/* Stream compaction of non-empty cells (NEW format):
 * offsets[0..n] = exclusive prefix of counts (offsets[n] = total);
 * cell_flat[j] = flat voxel index (x + 8y + 64z), cell_mc[j] = the 4 MC
 * bytes {index, r, g, b} as a little-endian u32; blocks in input order,
 * cells in ascending flat index.  Reads mc (dense) and counts.  Writes at
 * most cell_cap cells.  work_dev: scratch of >= vs_scan_workspace_bytes(n). */
vs_status vs_mc_compact(const uint8_t *mc, const uint32_t *counts, uint64_t n,
                        uint64_t *offsets, uint16_t *cell_flat, uint32_t *cell_mc,
                        uint64_t cell_cap, void *work_dev, vs_stream_t stream);
uint64_t vs_scan_workspace_bytes(uint64_t n);

/* ----------------------------------------------------------- stream sets --- */

/* affected_mc_blocks (mc_encoding.py:108-115) for u updated keys, with the
 * ordered first-occurrence dedup of Server.on_tsdf_batch (server.py:304-307).
 * out_keys receives <= 8u keys; *n_dev = count.  `scratch` is a table used
 * as the dedup set; it is cleared by the call. */
vs_status vs_affected_dedup(vs_table *scratch, const int32_t *updated, uint64_t u,
                            int32_t *out_keys, uint64_t *n_dev, vs_stream_t stream);

/* StreamSet.insert_many over C client sets (server.py:62-69, 314-315):
 * inserts the same n keys into every set; created[c*n + i] per client; each
 * client's newly created keys are appended, in input order, to its
 * generation-order FIFO ring (server.py:63-64).
 * fifo_keys_host[c] : device int32[fifo_cap_host[c]][3] ring of client c
 * fifo_tail_host[c] : device uint64 (absolute, monotonically increasing tail)
 * n_created         : device uint64[C] (may be NULL).
 * n_dev             : device uint64 (may be NULL): only the first
 *                     min(*n_dev, n) keys are inserted (n is then a bound),
 *                     so a count produced on the device (vs_affected_dedup)
 *                     needs no host synchronisation.
 * Fully asynchronous; up to 32 sets per call. */
vs_status vs_stream_insert_many(vs_table *const *sets_host, int n_sets,
                                const int32_t *keys, uint64_t n, const uint64_t *n_dev,
                                uint8_t *created, int32_t *const *fifo_keys_host,
                                const uint64_t *fifo_cap_host, uint64_t *const *fifo_tail_host,
                                uint64_t *n_created, vs_stream_t stream);

/* One stream-set tick in ONE launch (up to 32 client sets):
 *   affected = ordered first-occurrence dedup of affected_mc_blocks(k) over
 *              the u updated keys (mc_encoding.py:108-115, server.py:304-307)
 *              -> affected_out (device int32[8u][3]), *n_affected (device u64);
 *   insert_many(affected) into every set with the FIFO append of the created
 *              keys (server.py:314-315; fifo_* as vs_stream_insert_many),
 *              n_created[c] (device u64[C], may be NULL);
 *   extract_batch(max_extract) from every set (concurrent_hash.py:382-402,
 *              seeds_host[c] as vs_stream_extract_random) -> keys_out[c],
 *              n_out[c].
 * Equivalent to vs_affected_dedup + vs_stream_insert_many +
 * vs_stream_extract_random on the same stream; 1 <= u <= 512.  Asynchronous. */
vs_status vs_stream_tick(vs_table *const *sets_host, int n_sets, const int32_t *updated, uint64_t u,
                         int32_t *const *fifo_keys_host, const uint64_t *fifo_cap_host,
                         uint64_t *const *fifo_tail_host, uint64_t max_extract, const uint64_t *seeds_host,
                         int32_t *affected_out, uint64_t *n_affected, uint64_t *n_created,
                         int32_t *keys_out, uint64_t *n_out, vs_stream_t stream);

/* GpuServerCore.on_tsdf_batch without host synchronisation (server.py:299-315),
 * in ONE host call on `stream`: tsdf_map.put of the u wire rows (latest write
 * wins) into tsdf_pool (+ their face packs into tsdf_faces, may be NULL),
 * affected dedup -> affected_out (device int32[8u][3]) / *n_affected, mc_map
 * put of the affected keys, recompute of their MC + quantised bytes straight
 * into mc_pool / q_pool at the MC map positions, insert_many into the n_sets
 * client sets with the FIFO append (arrays as vs_stream_insert_many).  A
 * capacity failure is sticky (vs_table_check on either map).  Calls on one
 * tsdf_map must be stream-ordered (they mutate it); the call's scratch is
 * kept on tsdf_map between calls (grow-only, freed by vs_table_destroy). */
vs_status vs_server_tick(vs_table *tsdf_map, vs_table *mc_map, vs_table *dedup_scratch,
                         const int32_t *keys, const uint8_t *rows, uint64_t u,
                         uint8_t *tsdf_pool, uint8_t *tsdf_faces, uint8_t *mc_pool, int8_t *q_pool,
                         vs_table *const *sets_host, int n_sets, int32_t *const *fifo_keys_host,
                         const uint64_t *fifo_cap_host, uint64_t *const *fifo_tail_host,
                         int32_t *affected_out, uint64_t *n_affected, vs_stream_t stream);

/* extract_batch (concurrent_hash.py:366-402) on up to 32 sets in ONE launch:
 * set c scans its live entries in position order from a start position
 * derived from seeds_host[c] (wrapping), removes and returns the first max_n:
 * keys_out[c][0 .. n_out[c]) (device int32[C][max_n][3], n_out device
 * uint64[C]).  Asynchronous. */
vs_status vs_stream_extract_random(vs_table *const *sets_host, int n_sets,
                                   uint64_t max_n, const uint64_t *seeds_host,
                                   int32_t *keys_out, uint64_t *n_out, vs_stream_t stream);

/* extract_matching with the server's frustum-AABB predicate
 * (server.py:365-387, geometry.py:121-147) on up to 32 sets in one launch:
 * like vs_stream_extract_random, but only blocks whose AABB
 * [key*block_size, key*block_size + block_size] passes every plane
 * (nx*px + ny*py + nz*pz + d >= -margin at the positive vertex) are taken.
 * planes_host = double[6][4] (Frustum._planes); evaluated in IEEE double in
 * the reference's operation order (bit-identical decisions). */
vs_status vs_stream_extract_visible(vs_table *const *sets_host, int n_sets,
                                    uint64_t max_n, const uint64_t *seeds_host,
                                    const double *planes_host, double margin, double block_size,
                                    int32_t *keys_out, uint64_t *n_out, vs_stream_t stream);

/* TSDF ingest: tsdf_map.put for n wire-layout rows (server.py:300-303,
 * voxel_model.py:62-72): insert the keys into `t` (VS_ERR_CAPACITY rules of
 * vs_table_insert), then copy each row into pool + index[i]*6144 with the
 * LAST op of duplicate keys winning (sequential put order).  index[i] =
 * position (device int32[n]).  rows / pool 16-byte aligned. */
vs_status vs_tsdf_put(vs_table *t, const int32_t *keys, const uint8_t *rows, uint64_t n,
                      uint8_t *pool, int32_t *index, vs_stream_t stream);

/* MC_BATCH payload (wire.py:292-299, _pack_batch(blocks, 2048)) straight from
 * the device MC pool: out = u32 n, then n x {<3i key, 2048 MC bytes at
 * mc_pool + pos[i]*2048}; out holds 4 + 2060*n bytes (4-byte aligned). */
vs_status vs_mc_pack(const int32_t *keys, const int32_t *pos, uint64_t n,
                     const uint8_t *mc_pool, uint8_t *out, vs_stream_t stream);

/* Bulk remove of n keys from every one of n_sets tables (on_reset_blocks,
 * server.py:425-436).  erased may be NULL or device uint8[n_sets*n]. */
vs_status vs_stream_remove_many(vs_table *const *sets_host, int n_sets,
                                const int32_t *keys, uint64_t n, uint8_t *erased,
                                vs_stream_t stream);

/* extract_ordered (server.py:86-95): pop keys from the FIFO ring
 * [*head, tail), keep those whose removal from `set` succeeds, stop after
 * max_n successes.  Exact deque semantics, stale entries skipped.
 * head_host/tail_host are in/out (synchronous call). */
vs_status vs_stream_extract_ordered(vs_table *set, const int32_t *fifo_keys,
                                    uint64_t fifo_cap, uint64_t *head_host,
                                    uint64_t tail_host, uint64_t max_n,
                                    int32_t *keys_out, uint64_t *n_out_host,
                                    vs_table *scratch, vs_stream_t stream);

/* ------------------------------------------- key-hash sharded hash set --- */

/* One partition of a block hash set sharded over the `world` GPUs of a node
 * (BASELINE config 5; the reference is a single in-process
 * table, concurrent_hash.py:348-402 -- sharding is new).  owner(k) =
 * fmix32(hash_key pre-modulo, concurrent_hash.py:58) mod world.  Every rank
 * creates its shard over its local table, exports its window handle (CUDA
 * IPC, 64 bytes), gathers all ranks' handles (any out-of-band channel, e.g.
 * torch.distributed all_gather_object) and connects.  vs_shard_apply is then
 * COLLECTIVE: every rank calls it once per batch, in the same order; each
 * op is routed to its owner and the result comes back, by peer stores over
 * NVLink/NVSwitch from the kernels themselves (no host synchronisation, no
 * NCCL).  Per-op results equal a sequential replay of rank 0's batch, then
 * rank 1's, ... (A18 batches: of any order).  max_batch bounds n per call
 * (<= 2^30; world*max_batch < 2^31). */
typedef struct vs_shard vs_shard;
vs_status vs_shard_create(vs_table *local, int rank, int world, uint64_t max_batch, vs_shard **out);
void vs_shard_destroy(vs_shard *s);
vs_status vs_shard_export(vs_shard *s, uint8_t handle_out[64]);
/* handles: world x 64 bytes, rank-major (own entry ignored). */
vs_status vs_shard_connect(vs_shard *s, const uint8_t *handles);
/* All ranks of a world in ONE process on ONE device (tests and diagnostics:
 * an 8-rank node simulated on one GPU, each rank's vs_shard_apply on its own
 * stream): connects the windows directly, no IPC. */
vs_status vs_shard_connect_local(vs_shard *const *shards, int n);
/* keys device int32[n][3], ops device uint8[n] (VS_OP_*), result device
 * uint8[n] (created / found / erased).  Asynchronous on `stream`. */
vs_status vs_shard_apply(vs_shard *s, const int32_t *keys, const uint8_t *ops, uint64_t n,
                         uint8_t *result, vs_stream_t stream);
/* Bound on every device-side wait for a peer (default 20 s): a rank whose
 * peers never arrive (mismatched collective calls) gives up instead of
 * hanging the GPU, raises the shard's error flag and returns garbage. */
vs_status vs_shard_set_timeout_ms(vs_shard *s, uint64_t ms);
/* SYNCHRONOUS: VS_ERR_CUDA if a wait for a peer timed out since creation. */
vs_status vs_shard_check(vs_shard *s);
/* Host helper: owner rank of n HOST keys (the routing function). */
vs_status vs_shard_owner(const int32_t *keys, uint64_t n, int world, int32_t *owner_out);

/* ------------------------------------------------- RC-side voxel hashing --- */

/* VoxelModel.allocate_blocks / integrate_frame (voxel_model.py:105-141,
 * 165-299) on the device, bit-exact with the reference (IEEE ops in numpy's
 * order and precision; OpenBLAS FMA order for the 3x3 products).
 * params_host points to a vs_rc_params block (layout: see fusion.cu RcParams;
 * size vs_rc_params_bytes()) holding pose, intrinsics, fusion config, the
 * depth-step fractions and the sensor frustum planes.
 *   vs_rc_candidates: candidate block keys of the frame's truncation bands
 *     (_segment_block_keys, boundary-inclusive), warp-deduplicated, unordered;
 *     *n_dev = count (may exceed cap: then call again with a larger buffer).
 *   vs_rc_zero_rows: zero the pool rows of created blocks (TsdfBlock()).
 *   vs_rc_integrate: for n live blocks (keys, pool rows): frustum culling,
 *     coarse rejection, per-voxel projection and weighted update of the wire
 *     rows in place; touched[i] = 1 if any voxel of block i was updated.
 *   vs_rc_integrate_table: the same over every live block of the TSDF map
 *     `t` whose pool rows are indexed by entry slot (pool has t's capacity
 *     rows); no snapshot needed.  touched_keys_out (capacity x 3 int32)
 *     receives the touched keys in ascending slot order, *n_touched_dev
 *     their count.
 * depth: device float32[h][w]; color: device uint8[h][w][3]. */
uint64_t vs_rc_params_bytes(void);
vs_status vs_rc_candidates(const float *depth, const void *params_host, int32_t *keys_out,
                           uint64_t cap, uint64_t *n_dev, vs_stream_t stream);
vs_status vs_rc_zero_rows(const int32_t *pos, const uint8_t *created, uint64_t n,
                          uint8_t *pool, vs_stream_t stream);
vs_status vs_rc_integrate(const int32_t *keys, const int32_t *pos, uint64_t n,
                          const float *depth, const uint8_t *color, const void *params_host,
                          uint8_t *pool, uint8_t *touched, vs_stream_t stream);
vs_status vs_rc_integrate_table(const vs_table *t, const float *depth, const uint8_t *color,
                                const void *params_host, uint8_t *pool, int32_t *touched_keys_out,
                                uint64_t *n_touched_dev, vs_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* VSB200_H */
