/*
 * hash_oracle.c -- TEST INFRASTRUCTURE ONLY (the CPU oracle / CPU baseline).
 *
 * Plain-C restatement of the reference block hash set
 * (/root/reference/pkg/src/voxelstream/concurrent_hash.py), used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg as the checker.
 * Never linked into or called by the product (paper_1805_03709_b200).
 *
 * Sequential core: identical storage and decisions as the reference, so entry
 * positions are bit-exact with a sequential replay of the Python reference
 * (pinned against tests/golden/hash_seq.npz):
 *   hash_key        concurrent_hash.py:49-59
 *   storage         :104-115  (bucket region [0,n), excess [n,cap), next = 0
 *                              ends a chain, free stack preloaded range(n,cap))
 *   _scan_chain     :127-144
 *   _insert_pos     :159-208  (claim free bucket, else pop excess + append tail)
 *   remove          :251-295  (bucket: clear occ; excess: relink, push, stale next)
 *   snapshot_keys   :300-309  (ascending position)
 *   _extract        :382-402  (occupied positions rotated to a start, first
 *                              max_n removed; predicate None)
 *
 * Parallel batch mode (CPU baseline with all host threads): ops are
 * partitioned by bucket (a chain belongs to one bucket, so threads never
 * share a chain), excess pops use an atomic stack top, and erased entries
 * are pushed after the batch.  Valid for batches that follow the
 * order-independence rule of SURVEY.md §8a A18.
 */
#include <pthread.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define P1 73856093u
#define P2 19349669u
#define P3 83492791u

typedef struct {
  uint32_t n, excess, cap;
  int32_t *keys; /* cap x 3 */
  uint8_t *occ;
  uint32_t *next; /* absolute position of the next chain entry, 0 = end */
  uint32_t *stack;
  _Atomic int64_t top;
  uint64_t size;
} oh_table;

uint32_t oh_hash(int32_t x, int32_t y, int32_t z, uint32_t n) {
  uint32_t h = ((uint32_t)x * P1) ^ ((uint32_t)y * P2) ^ ((uint32_t)z * P3);
  return h % n;
}

void oh_hash_batch(const int32_t *keys, uint64_t cnt, uint32_t n, uint32_t *out) {
  for (uint64_t i = 0; i < cnt; ++i) out[i] = oh_hash(keys[3 * i], keys[3 * i + 1], keys[3 * i + 2], n);
}

static void oh_reset(oh_table *t) {
  memset(t->occ, 0, t->cap);
  memset(t->next, 0, sizeof(uint32_t) * (size_t)t->cap);
  memset(t->keys, 0, sizeof(int32_t) * 3 * (size_t)t->cap);
  for (uint32_t i = 0; i < t->excess; ++i) t->stack[i] = t->n + i;
  atomic_store(&t->top, (int64_t)t->excess);
  t->size = 0;
}

oh_table *oh_create(uint32_t n, uint32_t excess) {
  if (n < 1 || excess < 1) return NULL;
  oh_table *t = (oh_table *)calloc(1, sizeof(oh_table));
  t->n = n;
  t->excess = excess;
  t->cap = n + excess;
  t->keys = (int32_t *)malloc(sizeof(int32_t) * 3 * (size_t)t->cap);
  t->occ = (uint8_t *)malloc(t->cap);
  t->next = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)t->cap);
  t->stack = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)excess);
  if (!t->keys || !t->occ || !t->next || !t->stack) {
    free(t->keys); free(t->occ); free(t->next); free(t->stack); free(t);
    return NULL;
  }
  oh_reset(t);
  return t;
}

void oh_destroy(oh_table *t) {
  if (!t) return;
  free(t->keys); free(t->occ); free(t->next); free(t->stack); free(t);
}

void oh_clear(oh_table *t) { oh_reset(t); }
uint64_t oh_size(const oh_table *t) { return t->size; }
int64_t oh_free_count(oh_table *t) { return atomic_load(&t->top); }

static inline int keq(const oh_table *t, uint32_t e, int32_t x, int32_t y, int32_t z) {
  const int32_t *k = t->keys + 3 * (size_t)e;
  return k[0] == x && k[1] == y && k[2] == z;
}

/* _scan_chain: returns position or -1; *tail = last entry seen */
static inline int64_t scan_chain(const oh_table *t, int32_t x, int32_t y, int32_t z, uint32_t b, uint32_t *tail) {
  uint32_t e = b, last = b;
  for (;;) {
    if (t->occ[e] && keq(t, e, x, y, z)) {
      if (tail) *tail = e;
      return e;
    }
    last = e;
    e = t->next[e];
    if (e == 0) {
      if (tail) *tail = last;
      return -1;
    }
  }
}

int64_t oh_find(const oh_table *t, int32_t x, int32_t y, int32_t z) {
  return scan_chain(t, x, y, z, oh_hash(x, y, z, t->n), NULL);
}

/* returns 0 ok, 1 capacity exhausted (table unchanged) */
static int insert_one(oh_table *t, int32_t x, int32_t y, int32_t z, int64_t *pos, int *created,
                      uint32_t *retire_local, uint64_t *retire_n) {
  (void)retire_local; (void)retire_n;
  const uint32_t b = oh_hash(x, y, z, t->n);
  uint32_t tail;
  int64_t p = scan_chain(t, x, y, z, b, &tail);
  if (p >= 0) {
    *pos = p; *created = 0;
    return 0;
  }
  if (!t->occ[b]) {
    int32_t *k = t->keys + 3 * (size_t)b;
    k[0] = x; k[1] = y; k[2] = z;
    t->occ[b] = 1;
    *pos = b; *created = 1;
    return 0;
  }
  int64_t top = atomic_fetch_sub(&t->top, 1) - 1;
  if (top < 0) {
    atomic_fetch_add(&t->top, 1);
    *pos = -1; *created = 0;
    return 1;
  }
  const uint32_t e = t->stack[top];
  int32_t *k = t->keys + 3 * (size_t)e;
  k[0] = x; k[1] = y; k[2] = z;
  t->next[e] = 0; /* clear offset left stale by removal */
  t->occ[e] = 1;
  t->next[tail] = e; /* publish last */
  *pos = e; *created = 1;
  return 0;
}

/* remove; returns 1 if present.  Excess victims go to `retired` when given
 * (parallel mode), else are pushed immediately (sequential reference order). */
static int erase_one(oh_table *t, int32_t x, int32_t y, int32_t z, int64_t *pos, uint32_t *retired,
                     uint64_t *retired_n) {
  const uint32_t b = oh_hash(x, y, z, t->n);
  if (t->occ[b] && keq(t, b, x, y, z)) {
    t->occ[b] = 0; /* bucket case: keep next */
    *pos = b;
    return 1;
  }
  uint32_t prev = b, e = t->next[b];
  while (e) {
    if (t->occ[e] && keq(t, e, x, y, z)) {
      t->next[prev] = t->next[e]; /* link past the victim; victim keeps its stale next */
      t->occ[e] = 0;
      if (retired) {
        retired[(*retired_n)++] = e;
      } else {
        int64_t top = atomic_fetch_add(&t->top, 1);
        t->stack[top] = e;
      }
      *pos = e;
      return 1;
    }
    prev = e;
    e = t->next[e];
  }
  *pos = -1;
  return 0;
}

/* Sequential insert batch, stops at the first capacity failure like
 * `for k in keys: insert(k)`.  Returns the failing op index or -1. */
int64_t oh_insert_batch(oh_table *t, const int32_t *keys, uint64_t cnt, uint8_t *created, int32_t *index) {
  for (uint64_t i = 0; i < cnt; ++i) {
    int64_t pos;
    int cr;
    if (insert_one(t, keys[3 * i], keys[3 * i + 1], keys[3 * i + 2], &pos, &cr, NULL, NULL)) return (int64_t)i;
    created[i] = (uint8_t)cr;
    index[i] = (int32_t)pos;
    t->size += (uint64_t)cr;
  }
  return -1;
}

void oh_find_batch(const oh_table *t, const int32_t *keys, uint64_t cnt, uint8_t *found, int32_t *index) {
  for (uint64_t i = 0; i < cnt; ++i) {
    int64_t p = oh_find(t, keys[3 * i], keys[3 * i + 1], keys[3 * i + 2]);
    found[i] = p >= 0;
    index[i] = (int32_t)p;
  }
}

void oh_erase_batch(oh_table *t, const int32_t *keys, uint64_t cnt, uint8_t *erased, int32_t *index) {
  for (uint64_t i = 0; i < cnt; ++i) {
    int64_t pos;
    int r = erase_one(t, keys[3 * i], keys[3 * i + 1], keys[3 * i + 2], &pos, NULL, NULL);
    erased[i] = (uint8_t)r;
    index[i] = (int32_t)pos;
    t->size -= (uint64_t)r;
  }
}

/* Sequential mixed batch (op 0 insert, 1 find, 2 erase).  Returns the first
 * capacity-failing op index or -1 (the op is skipped, replay continues). */
int64_t oh_apply_batch(oh_table *t, const int32_t *keys, const uint8_t *ops, uint64_t cnt, uint8_t *result,
                       int32_t *index) {
  int64_t fail = -1;
  for (uint64_t i = 0; i < cnt; ++i) {
    const int32_t x = keys[3 * i], y = keys[3 * i + 1], z = keys[3 * i + 2];
    int64_t pos = -1;
    int r = 0;
    if (ops[i] == 0) {
      if (insert_one(t, x, y, z, &pos, &r, NULL, NULL) && fail < 0) fail = (int64_t)i;
      t->size += (uint64_t)r;
    } else if (ops[i] == 2) {
      r = erase_one(t, x, y, z, &pos, NULL, NULL);
      t->size -= (uint64_t)r;
    } else {
      pos = oh_find(t, x, y, z);
      r = pos >= 0;
    }
    result[i] = (uint8_t)r;
    index[i] = (int32_t)pos;
  }
  return fail;
}

/* ---- parallel batch (CPU baseline) ---- */

typedef struct {
  oh_table *t;
  const int32_t *keys;
  const uint8_t *ops;
  const uint32_t *bucket;
  uint64_t cnt;
  uint8_t *result;
  int32_t *index;
  int tid, nthreads;
  uint32_t *retired;
  uint64_t retired_n;
  int64_t size_delta;
  int64_t fail;
} oh_job;

static void *apply_worker(void *arg) {
  oh_job *j = (oh_job *)arg;
  oh_table *t = j->t;
  for (uint64_t i = 0; i < j->cnt; ++i) {
    if ((int)(j->bucket[i] % (uint32_t)j->nthreads) != j->tid) continue;
    const int32_t x = j->keys[3 * i], y = j->keys[3 * i + 1], z = j->keys[3 * i + 2];
    int64_t pos = -1;
    int r = 0;
    const uint8_t op = j->ops ? j->ops[i] : 0;
    if (op == 0) {
      if (insert_one(t, x, y, z, &pos, &r, NULL, NULL) && (j->fail < 0 || (int64_t)i < j->fail)) j->fail = (int64_t)i;
      j->size_delta += r;
    } else if (op == 2) {
      r = erase_one(t, x, y, z, &pos, j->retired, &j->retired_n);
      j->size_delta -= r;
    } else {
      pos = oh_find(t, x, y, z);
      r = pos >= 0;
    }
    j->result[i] = (uint8_t)r;
    j->index[i] = (int32_t)pos;
  }
  return NULL;
}

typedef struct {
  const int32_t *keys;
  uint64_t lo, hi;
  uint32_t n;
  uint32_t *out;
} hash_job;

static void *hash_worker(void *arg) {
  hash_job *h = (hash_job *)arg;
  for (uint64_t i = h->lo; i < h->hi; ++i)
    h->out[i] = oh_hash(h->keys[3 * i], h->keys[3 * i + 1], h->keys[3 * i + 2], h->n);
  return NULL;
}

/* ops may be NULL (all inserts).  Returns lowest failing op index or -1. */
int64_t oh_apply_batch_mt(oh_table *t, const int32_t *keys, const uint8_t *ops, uint64_t cnt, uint8_t *result,
                          int32_t *index, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  uint32_t *bucket = (uint32_t *)malloc(sizeof(uint32_t) * (cnt ? cnt : 1));
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  hash_job *hj = (hash_job *)malloc(sizeof(hash_job) * (size_t)nthreads);
  for (int k = 0; k < nthreads; ++k) {
    hj[k].keys = keys;
    hj[k].lo = cnt * (uint64_t)k / (uint64_t)nthreads;
    hj[k].hi = cnt * (uint64_t)(k + 1) / (uint64_t)nthreads;
    hj[k].n = t->n;
    hj[k].out = bucket;
    pthread_create(&th[k], NULL, hash_worker, &hj[k]);
  }
  for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
  oh_job *jobs = (oh_job *)calloc((size_t)nthreads, sizeof(oh_job));
  for (int k = 0; k < nthreads; ++k) {
    jobs[k].t = t; jobs[k].keys = keys; jobs[k].ops = ops; jobs[k].bucket = bucket; jobs[k].cnt = cnt;
    jobs[k].result = result; jobs[k].index = index; jobs[k].tid = k; jobs[k].nthreads = nthreads;
    jobs[k].retired = (uint32_t *)malloc(sizeof(uint32_t) * (cnt ? cnt : 1));
    jobs[k].fail = -1;
    pthread_create(&th[k], NULL, apply_worker, &jobs[k]);
  }
  int64_t fail = -1;
  for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
  /* recycle only after EVERY worker stopped popping */
  for (int k = 0; k < nthreads; ++k) {
    for (uint64_t r = 0; r < jobs[k].retired_n; ++r) {
      int64_t top = atomic_fetch_add(&t->top, 1);
      t->stack[top] = jobs[k].retired[r];
    }
    t->size += (uint64_t)jobs[k].size_delta;
    if (jobs[k].fail >= 0 && (fail < 0 || jobs[k].fail < fail)) fail = jobs[k].fail;
    free(jobs[k].retired);
  }
  free(jobs); free(hj); free(th); free(bucket);
  return fail;
}

/* snapshot_keys: live keys in ascending position order */
uint64_t oh_snapshot(const oh_table *t, int32_t *keys_out, int32_t *pos_out, uint64_t cap) {
  uint64_t m = 0;
  for (uint32_t e = 0; e < t->cap; ++e) {
    if (!t->occ[e]) continue;
    if (m < cap) {
      if (keys_out) memcpy(keys_out + 3 * m, t->keys + 3 * (size_t)e, 12);
      if (pos_out) pos_out[m] = (int32_t)e;
    }
    ++m;
  }
  return m;
}

/* raw views for white-box tests of the oracle itself */
const uint8_t *oh_occ(const oh_table *t) { return t->occ; }
const uint32_t *oh_next(const oh_table *t) { return t->next; }
const uint32_t *oh_stack(const oh_table *t) { return t->stack; }
uint32_t oh_capacity(const oh_table *t) { return t->cap; }

/* _extract (concurrent_hash.py:382-402), predicate None: the occupied
 * positions in ascending order, rotated to begin at the first one >= start
 * (the reference draws start = random.randrange(capacity)), the first max_n
 * of them removed in that order.  Returns the count; keys_out = max_n x 3.
 * The reference materialises every occupied position first; collecting the
 * first max_n and removing them afterwards takes the same keys (positions
 * never move while a key is present). */
uint64_t oh_extract(oh_table *t, uint64_t max_n, uint64_t start, int32_t *keys_out) {
  if (!max_n || !t->size) return 0;
  start %= t->cap;
  uint64_t got = 0;
  for (uint64_t k = 0; k < t->cap && got < max_n; ++k) {
    uint64_t e = start + k;
    if (e >= t->cap) e -= t->cap;
    if (t->occ[e]) {
      memcpy(keys_out + 3 * got, t->keys + 3 * e, 12);
      ++got;
    }
  }
  for (uint64_t i = 0; i < got; ++i) {
    int64_t pos;
    t->size -= (uint64_t)erase_one(t, keys_out[3 * i], keys_out[3 * i + 1], keys_out[3 * i + 2], &pos, NULL, NULL);
  }
  return got;
}
