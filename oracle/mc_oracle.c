/*
 * mc_oracle.c -- TEST INFRASTRUCTURE ONLY (the CPU oracle / CPU baseline).
 *
 * Plain-C restatement of the reference MC block encoder, used by tests/,
 * smoke() and bench.py's cpu_baseline leg; never part of the product.
 *
 *   recompute_mc_block  mc_encoding.py:145-172 (+ _corner_grids :118-142)
 *     absent centre -> all-zero block                          (:152-156)
 *     corner k of the cube at voxel (x,y,z) sits at (x+(k&1), y+(k>>1&1),
 *     z+(k>>2&1)); corners past the +faces come from the +1 neighbours;
 *     an absent neighbour contributes tsdf 0 / weight 0          (:128-142)
 *     bit k = tsdf < 0; index = 0 unless every weight > 0; 255 -> 0
 *     colour = centre voxel colour where index != 0             (:159-171)
 *   TSDF voxel layout   voxel_model.py:26-29 (f32 tsdf, f32 weight, u8 rgb[3],
 *                       u8 pad), flat index x + 8y + 64z (:31-39)
 *   McBlock.to_bytes    mc_encoding.py:69-73 ({u8 index, u8 rgb[3]} x 512)
 *
 * The compares are plain C float compares (IEEE, no fast-math, no FTZ),
 * i.e. the same predicates numpy evaluates in the reference.
 *
 * Quantised TSDF (NEW format -- no reference implementation exists,
 * SURVEY.md §8a A17; normative definition of this repo):
 *   q = observed(weight) && !isnan(tsdf)
 *         ? (int8) rint_half_even(clamp(tsdf * 127.0f, -127, 127))
 *         : -128
 * with the product computed in float32.
 *
 * Compaction (NEW format, A19): per block, the non-zero cells in ascending
 * flat index as (u16 flat, u32 {index, r, g, b}); blocks in input order.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define BLOCK_BYTES 6144

static inline void voxel(const uint8_t *pool, int32_t row, int flat, float *tsdf, float *weight) {
  if (row < 0) {
    *tsdf = 0.0f;
    *weight = 0.0f;
    return;
  }
  const uint8_t *p = pool + (size_t)row * BLOCK_BYTES + 12 * (size_t)flat;
  memcpy(tsdf, p, 4);
  memcpy(weight, p + 4, 4);
}

int8_t om_quantise(float tsdf, float weight) {
  if (!(weight > 0.0f) || isnan(tsdf)) return -128;
  float s = tsdf * 127.0f;
  if (s > 127.0f) s = 127.0f;
  if (s < -127.0f) s = -127.0f;
  return (int8_t)rintf(s);
}

void om_encode_block(const uint8_t *pool, const int32_t *nbr8, uint8_t *mc, int8_t *q, uint32_t *count) {
  uint32_t nz = 0;
  if (nbr8[0] < 0) {
    if (mc) memset(mc, 0, 2048);
    if (q) memset(q, -128, 512);
    if (count) *count = 0;
    return;
  }
  const uint8_t *centre = pool + (size_t)nbr8[0] * BLOCK_BYTES;
  for (int f = 0; f < 512; ++f) {
    const int x = f & 7, y = (f >> 3) & 7, z = f >> 6;
    unsigned index = 0;
    int all_observed = 1;
    for (int k = 0; k < 8; ++k) {
      const int cx = x + (k & 1), cy = y + ((k >> 1) & 1), cz = z + ((k >> 2) & 1);
      const int sel = (cx >> 3) | ((cy >> 3) << 1) | ((cz >> 3) << 2);
      const int ff = (cx & 7) + 8 * (cy & 7) + 64 * (cz & 7);
      float t, w;
      voxel(pool, nbr8[sel], ff, &t, &w);
      if (t < 0.0f) index |= 1u << k;
      if (!(w > 0.0f)) all_observed = 0;
    }
    if (!all_observed || index == 255u) index = 0;
    if (mc) {
      uint8_t *o = mc + 4 * f;
      o[0] = (uint8_t)index;
      if (index) {
        memcpy(o + 1, centre + 12 * f + 8, 3);
      } else {
        o[1] = o[2] = o[3] = 0;
      }
    }
    if (q) {
      float t, w;
      memcpy(&t, centre + 12 * f, 4);
      memcpy(&w, centre + 12 * f + 4, 4);
      q[f] = om_quantise(t, w);
    }
    nz += index != 0;
  }
  if (count) *count = nz;
}

typedef struct {
  const uint8_t *pool;
  const int32_t *nbr;
  uint64_t lo, hi;
  uint8_t *mc;
  int8_t *q;
  uint32_t *counts;
} om_job;

static void *encode_worker(void *arg) {
  om_job *j = (om_job *)arg;
  for (uint64_t i = j->lo; i < j->hi; ++i)
    om_encode_block(j->pool, j->nbr + 8 * i, j->mc ? j->mc + 2048 * i : NULL, j->q ? j->q + 512 * i : NULL,
                    j->counts ? j->counts + i : NULL);
  return NULL;
}

void om_encode(const uint8_t *pool, const int32_t *nbr, uint64_t n, uint8_t *mc, int8_t *q, uint32_t *counts,
               int nthreads) {
  if (nthreads < 1) nthreads = 1;
  pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
  om_job *jobs = (om_job *)malloc(sizeof(om_job) * (size_t)nthreads);
  for (int k = 0; k < nthreads; ++k) {
    jobs[k].pool = pool; jobs[k].nbr = nbr; jobs[k].mc = mc; jobs[k].q = q; jobs[k].counts = counts;
    jobs[k].lo = n * (uint64_t)k / (uint64_t)nthreads;
    jobs[k].hi = n * (uint64_t)(k + 1) / (uint64_t)nthreads;
    pthread_create(&th[k], NULL, encode_worker, &jobs[k]);
  }
  for (int k = 0; k < nthreads; ++k) pthread_join(th[k], NULL);
  free(jobs);
  free(th);
}

/* compaction of a dense MC buffer; returns total cells */
uint64_t om_compact(const uint8_t *mc, uint64_t n, uint64_t *offsets, uint16_t *cell_flat, uint32_t *cell_mc) {
  uint64_t o = 0;
  for (uint64_t i = 0; i < n; ++i) {
    offsets[i] = o;
    for (int f = 0; f < 512; ++f) {
      uint32_t w;
      memcpy(&w, mc + 2048 * i + 4 * f, 4);
      if (w) {
        if (cell_flat) cell_flat[o] = (uint16_t)f;
        if (cell_mc) cell_mc[o] = w;
        ++o;
      }
    }
  }
  offsets[n] = o;
  return o;
}
