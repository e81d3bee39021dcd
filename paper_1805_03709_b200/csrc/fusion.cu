// fusion.cu -- RC-side voxel hashing on the GPU.
//
// Reference: VoxelModel.allocate_blocks / integrate_frame
// (voxel_model.py:105-141, 165-299), geometry.py (pixel_rays :93-101,
// Frustum.intersects_aabbs :154-162, Pose.transform / inverse_transform).
//
// Bit-exact by construction: every floating-point operation is an explicit
// round-to-nearest intrinsic in the reference's numpy order and precision
// (float64 for allocation, culling and coarse rejection; float32 for the
// per-voxel projection and the weighted update), nothing is contracted.
// numpy's small matrix products go through OpenBLAS, whose order was
// measured (tests/golden):
//   (N,3)@(3,3) and (N,3)@(3,3).T : c_j = fma(a2, b2j, fma(a1, b1j, a0*b0j))
//   (N,3)@(3,)                    : fma(a2, n2, fma(a0, n0, a1*n1))
#include <cstdint>

#include "hash_ops.cuh"
#include "pdl.cuh"
#include "scan.cuh"
#include "table.h"

namespace vsb {

struct RcParams {
  double R[9];      // pose.rotation, row-major (camera -> world)
  double t[3];      // pose.translation
  float R32[9];     // pose.rotation.astype(float32)
  float t32[3];     // pose.translation.astype(float32)
  double fx, fy, cx, cy;
  int32_t width, height;
  double voxel, mu, max_weight, block;
  double tol;       // _BOUNDARY_EPS / block_size
  double one_minus_tol;
  double reach;     // truncation + block_size * sqrt(3)
  int32_t stride;   // alloc_stride
  int32_t steps;
  double ts[64];    // np.linspace(0, 1, steps)
  double planes[24];  // Frustum._planes of sensor_frustum(..., margin=block)
  double margin;
};

// ------------------------------------------------------------ allocation

// One thread per sampled pixel, walking its depth steps; a warp covers an
// 8x4 pixel tile so that neighbouring rays meet the same blocks.  A sample's
// emissions are its block key plus, within _BOUNDARY_EPS of a face, the
// face/edge/corner neighbours (_segment_block_keys).  Duplicates are dropped
// cheaply but not exhaustively (the insert dedups exactly): a thread skips a
// sample whose (key, face mask) equals its previous one, and within a warp
// only the lowest lane of each equal key (resp. key + mask) emits.
__device__ __forceinline__ void rc_sample(const RcParams& P, double r0, double r1, double d, int j, long long b[3],
                                          uint32_t& mask) {
  const double z0 = fmax(__dsub_rn(d, P.mu), P.voxel);
  const double z1 = __dadd_rn(d, P.mu);
  const double zs = __dadd_rn(z0, __dmul_rn(__dsub_rn(z1, z0), P.ts[j]));
  const double p0 = __dmul_rn(r0, zs), p1 = __dmul_rn(r1, zs), p2 = zs;  // rays * zs (ray z = 1)
  mask = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    // pose.transform: pts @ R.T + t
    const double w = __dadd_rn(__fma_rn(p2, P.R[3 * k + 2], __fma_rn(p1, P.R[3 * k + 1], __dmul_rn(p0, P.R[3 * k]))),
                               P.t[k]);
    const double g = __ddiv_rn(w, P.block);
    const double fl = floor(g);
    const double frac = __dsub_rn(g, fl);
    b[k] = (long long)fl;
    mask |= (frac < P.tol ? 1u : 0u) << (2 * k);
    mask |= (frac > P.one_minus_tol ? 2u : 0u) << (2 * k);
  }
}

constexpr int kCandStage = 256;  // >= 32 lanes x 8 emissions per step

__global__ void __launch_bounds__(256) k_rc_candidates(const float* __restrict__ depth, const __grid_constant__ RcParams P,
                                                       int32_t ws, int32_t hs, int32_t* __restrict__ out,
                                                       unsigned long long* __restrict__ count, uint64_t cap) {
  pdl_wait();
  // tile-major pixel order: warp w -> 8x4 tile, lane -> (lane & 7, lane >> 3)
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = (int)lane_id();
  const int32_t tiles_x = (ws + 7) >> 3;
  const int32_t tx = (int32_t)(warp % (uint64_t)tiles_x), ty = (int32_t)(warp / (uint64_t)tiles_x);
  const int32_t pu = tx * 8 + (lane & 7), pv = ty * 4 + (lane >> 3);
  bool valid = false;
  double r0 = 0.0, r1 = 0.0, d = 0.0;
  if (pu < ws && pv < hs) {
    const int32_t u = pu * P.stride, v = pv * P.stride;
    const float d32 = depth[(uint64_t)v * P.width + u];
    if (d32 > 0.f) {
      valid = true;
      // pixel_rays: ((u - cx) / fx, (v - cy) / fy, 1)
      r0 = __ddiv_rn(__dsub_rn((double)u, P.cx), P.fx);
      r1 = __ddiv_rn(__dsub_rn((double)v, P.cy), P.fy);
      d = (double)d32;
    }
  }
  if (__ballot_sync(0xffffffffu, valid) == 0) return;  // warp-uniform exit
  // emissions are staged per warp in shared memory and flushed with one
  // atomic reservation per kCandStage keys (one per step contended badly)
  __shared__ int32_t stage[8][3 * kCandStage];
  int32_t* buf = stage[threadIdx.x >> 5];
  int bc = 0;  // staged keys (warp-uniform)
  auto flush = [&]() {
    if (!bc) return;
    __syncwarp();
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(count, (unsigned long long)bc);
    base = __shfl_sync(0xffffffffu, base, 0);
    for (int q = lane; q < 3 * bc; q += 32)
      if (base + (unsigned long long)(q / 3) < cap) out[3 * base + q] = buf[q];
    __syncwarp();
    bc = 0;
  };
  unsigned long long last = ~0ull;
  uint32_t last_mask = 0xffffffffu;
  for (int j = 0; j < P.steps; ++j) {
    long long b[3] = {0, 0, 0};
    uint32_t mask = 0;
    if (valid) rc_sample(P, r0, r1, d, j, b, mask);
    const unsigned long long enc = ((unsigned long long)(b[0] + (1 << 20)) << 42) |
                                   ((unsigned long long)(b[1] + (1 << 20)) << 21) |
                                   (unsigned long long)(b[2] + (1 << 20));
    const bool fresh = valid && (enc != last || mask != last_mask);
    if (fresh) {
      last = enc;
      last_mask = mask;
    }
    const uint32_t fmask = __ballot_sync(0xffffffffu, fresh);
    if (!fmask) continue;
    const uint32_t same_key = __match_any_sync(0xffffffffu, fresh ? enc : ~0ull) & fmask;
    const uint32_t same_sig = same_key & __match_any_sync(0xffffffffu, fresh ? mask : 0xffffffffu);
    const bool base_leader = fresh && (__ffs(same_key) - 1) == lane;
    const bool nbr_leader = fresh && mask && (__ffs(same_sig) - 1) == lane;
    int n_emit = base_leader ? 1 : 0;
    if (nbr_leader) {
      // neighbours across the flagged faces: each axis offers {0} plus -1 (lo) and/or +1 (hi)
      const int nx = 1 + (mask & 1) + ((mask >> 1) & 1), ny = 1 + ((mask >> 2) & 1) + ((mask >> 3) & 1),
                nz = 1 + ((mask >> 4) & 1) + ((mask >> 5) & 1);
      n_emit += nx * ny * nz - 1;
    }
    // warp-local slots in the warp's shared-memory staging buffer
    int incl = n_emit;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total_w = __shfl_sync(0xffffffffu, incl, 31);
    if (bc + total_w > kCandStage) {
      flush();
    }
    int o = bc + incl - n_emit;
    auto put = [&](long long x, long long y, long long z) {
      buf[3 * o] = (int32_t)x;
      buf[3 * o + 1] = (int32_t)y;
      buf[3 * o + 2] = (int32_t)z;
      ++o;
    };
    if (base_leader) put(b[0], b[1], b[2]);
    if (nbr_leader) {
      for (int dx = -1; dx <= 1; ++dx)
        for (int dy = -1; dy <= 1; ++dy)
          for (int dz = -1; dz <= 1; ++dz) {
            if (!dx && !dy && !dz) continue;
            const int dd[3] = {dx, dy, dz};
            bool m = true;
#pragma unroll
            for (int a = 0; a < 3; ++a) m &= dd[a] == 0 || ((mask >> (2 * a + (dd[a] < 0 ? 0 : 1))) & 1u);
            if (m) put(b[0] + dx, b[1] + dy, b[2] + dz);
          }
    }
    bc += total_w;
    __syncwarp();
  }
  flush();
}

// Zero the pool rows of newly created blocks (TsdfBlock(): all zero).
__global__ void k_rc_zero_rows(const int32_t* __restrict__ pos, const uint8_t* __restrict__ created, uint64_t n,
                               uint4* __restrict__ pool) {
  pdl_wait();
  // one candidate per lane; the whole warp zeroes each created row in turn
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  const bool mine = i < n && created[i];
  uint32_t todo = __ballot_sync(0xffffffffu, mine);
  const int32_t p = mine ? pos[i] : 0;
  while (todo) {
    const int src = __ffs(todo) - 1;
    todo &= todo - 1;
    const int32_t row = __shfl_sync(0xffffffffu, p, src);
    uint4* dst = pool + (uint64_t)row * (VS_TSDF_BLOCK_BYTES / 16);
    for (int j = lane; j < VS_TSDF_BLOCK_BYTES / 16; j += 32) dst[j] = make_uint4(0, 0, 0, 0);
  }
}

// ----------------------------------------------------------------- fusion

// numpy float32 -> int32 (astype): NaN / out-of-range give INT32_MIN on x86.
__device__ __forceinline__ int32_t np_f32_to_i32(float r) {
  if (!(r >= -2147483648.0f && r < 2147483648.0f)) return INT32_MIN;
  return (int32_t)r;
}

// Block-level culling (frustum + coarse rejection): one thread per live
// block; keep[i] = 1 for blocks the per-voxel pass must visit.
__device__ __forceinline__ bool rc_block_candidate(const RcParams& P, const float* __restrict__ depth, int32_t kx,
                                                   int32_t ky, int32_t kz);

__global__ void k_rc_cull(const int32_t* __restrict__ keys, uint64_t n, const float* __restrict__ depth,
                          const __grid_constant__ RcParams P, uint8_t* __restrict__ keep) {
  pdl_wait();
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  keep[i] = rc_block_candidate(P, depth, keys[3 * i], keys[3 * i + 1], keys[3 * i + 2]);
}

// Cull over the map's entry slots; survivors are appended to `list` in
// arbitrary order (warp-aggregated), *n_list = their count.
__global__ void k_rc_cull_table(const Entry* __restrict__ e, uint32_t cap, const float* __restrict__ depth,
                                const __grid_constant__ RcParams P, uint32_t* __restrict__ list,
                                unsigned long long* __restrict__ n_list) {
  pdl_wait();
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  bool keep = false;
  if (i < cap) {
    const int4 k = ld_entry_ro(e + i);
    keep = ((uint32_t)k.w & kOcc) && rc_block_candidate(P, depth, k.x, k.y, k.z);
  }
  const uint32_t bal = __ballot_sync(0xffffffffu, keep);
  if (!bal) return;
  unsigned long long base = 0;
  if (lane_id() == 0) base = atomicAdd(n_list, (unsigned long long)__popc(bal));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (keep) list[base + __popc(bal & lanemask_lt())] = (uint32_t)i;
}

// touched slots -> their keys, ascending slot order
__global__ void k_rc_touched_keys(const uint8_t* __restrict__ touched, const uint64_t* __restrict__ off, uint32_t cap,
                                  const Entry* __restrict__ e, int32_t* __restrict__ keys_out) {
  pdl_wait();
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cap || !touched[i]) return;
  const int4 k = ld_entry_ro(e + i);
  const uint64_t o = off[i];
  keys_out[3 * o] = k.x, keys_out[3 * o + 1] = k.y, keys_out[3 * o + 2] = k.z;
}

__global__ void k_rc_gather(const uint8_t* __restrict__ keep, const uint64_t* __restrict__ off, uint64_t n,
                            uint32_t* __restrict__ list) {
  pdl_wait();
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && keep[i]) list[off[i]] = (uint32_t)i;
}

__device__ __forceinline__ bool rc_block_candidate(const RcParams& P, const float* __restrict__ depth, int32_t kx,
                                                   int32_t ky, int32_t kz) {
  // --- frustum culling (intersects_aabbs on block_aabbs, margin = block size)
  const double mn[3] = {__dmul_rn((double)kx, P.block), __dmul_rn((double)ky, P.block), __dmul_rn((double)kz, P.block)};
  const double mx[3] = {__dadd_rn(mn[0], P.block), __dadd_rn(mn[1], P.block), __dadd_rn(mn[2], P.block)};
  bool inview = true;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double* q = P.planes + 4 * k;
    const double v0 = q[0] >= 0.0 ? mx[0] : mn[0], v1 = q[1] >= 0.0 ? mx[1] : mn[1], v2 = q[2] >= 0.0 ? mx[2] : mn[2];
    const double dot = __fma_rn(v2, q[2], __fma_rn(v0, q[0], __dmul_rn(v1, q[1])));
    inview &= __dadd_rn(dot, q[3]) >= -P.margin;
  }
  if (!inview) return false;
  // --- coarse rejection of blocks far outside the truncation band
  {
    const double c[3] = {__dmul_rn((double)kx + 0.5, P.block), __dmul_rn((double)ky + 0.5, P.block),
                         __dmul_rn((double)kz + 0.5, P.block)};
    const double d0 = __dsub_rn(c[0], P.t[0]), d1 = __dsub_rn(c[1], P.t[1]), d2 = __dsub_rn(c[2], P.t[2]);
    double cc[3];
#pragma unroll
    for (int j = 0; j < 3; ++j)  // inverse_transform: (p - t) @ R
      cc[j] = __fma_rn(d2, P.R[6 + j], __fma_rn(d1, P.R[3 + j], __dmul_rn(d0, P.R[j])));
    const double cz = cc[2];
    const double cu = rint(__dadd_rn(__ddiv_rn(__dmul_rn(P.fx, cc[0]), cz), P.cx));
    const double cv = rint(__dadd_rn(__ddiv_rn(__dmul_rn(P.fy, cc[1]), cz), P.cy));
    const bool inside = cz > 0.0 && cu >= 0.0 && cu < (double)P.width && cv >= 0.0 && cv < (double)P.height;
    if (inside) {
      const float cd = depth[(uint64_t)cv * P.width + (uint64_t)cu];
      if (cd > 0.f && fabs(__dsub_rn((double)cd, cz)) > P.reach) return false;
    }
  }
  return true;
}

// Work distribution of k_rc_integrate: 1 = blocks claimed from a counter
// (balanced: blocks differ in cost -- voxels outside the image skip their
// loads), 0 = static grid stride.
#ifndef VSB_RC_TICKET
#define VSB_RC_TICKET 1
#endif

// Persistent CTAs (128 threads, 4 voxels each) walk the blocks that survived
// culling.  Per block a thread first projects its 4 voxels, then issues every
// independent load at once (depth sample + the 12-B voxel record, as three
// u32 words), then updates; the record keeps its pad byte.  `touched` is set
// per warp with a plain store (memset to 0 beforehand), so there is no CTA
// barrier between blocks.
__global__ void __launch_bounds__(128) k_rc_integrate(const int32_t* __restrict__ keys, const int32_t* __restrict__ pos,
                                                      const Entry* __restrict__ ent, const uint32_t* __restrict__ list, const uint64_t* __restrict__ n_list,
                                                      const float* __restrict__ depth, const uint8_t* __restrict__ color,
                                                      const __grid_constant__ RcParams P, uint8_t* __restrict__ pool,
                                                      uint8_t* __restrict__ touched, unsigned long long* tick) {
  pdl_wait();
  const uint64_t n_live = *n_list;
  // tick (VSB_RC_TICKET): blocks are claimed one at a time from a zeroed
  // counter, the next claim issued while the current block is processed
  __shared__ unsigned long long claim[2];
  if (tick && threadIdx.x == 0) claim[0] = atomicAdd(tick, 1ull);
  if (tick) __syncthreads();
  int cb = 0;
  const float fx = (float)P.fx, fy = (float)P.fy, cx = (float)P.cx, cy = (float)P.cy;
  const float mu = (float)P.mu, neg_mu = (float)(-P.mu), maxw = (float)P.max_weight;
  const int lx = threadIdx.x & 7, ly = (threadIdx.x >> 3) & 7, lz0 = threadIdx.x >> 6;  // f = tid + 128k: lz = lz0 + 2k
  for (uint64_t li = tick ? claim[0] : blockIdx.x; li < n_live;) {
    if (tick && threadIdx.x == 0) claim[cb ^ 1] = atomicAdd(tick, 1ull);
    const uint64_t i = list[li];
    // block source: (keys, pos) arrays, or the table's entry slots (row = slot)
    int32_t kx, ky, kz;
    uint64_t r;
    if (ent) {
      const int4 e = ld_entry_ro(ent + i);
      kx = e.x, ky = e.y, kz = e.z, r = i;
    } else {
      kx = keys[3 * i], ky = keys[3 * i + 1], kz = keys[3 * i + 2], r = (uint64_t)pos[i];
    }
    uint32_t* row = (uint32_t*)(pool + r * VS_TSDF_BLOCK_BYTES);
    // coords = ((origins + LOCAL + 0.5) * voxel).astype(float32); x, y fixed per thread
    const float c0 = __double2float_rn(__dmul_rn((double)(8ll * kx + lx) + 0.5, P.voxel));
    const float c1 = __double2float_rn(__dmul_rn((double)(8ll * ky + ly) + 0.5, P.voxel));
    const float e0 = __fsub_rn(c0, P.t32[0]), e1 = __fsub_rn(c1, P.t32[1]);
    float z[4];
    int32_t pix[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float c2 = __double2float_rn(__dmul_rn((double)(8ll * kz + lz0 + 2 * k) + 0.5, P.voxel));
      const float e2 = __fsub_rn(c2, P.t32[2]);
      float cam[3];
#pragma unroll
      for (int j = 0; j < 3; ++j)  // (coords - trans) @ rot, float32
        cam[j] = __fmaf_rn(e2, P.R32[6 + j], __fmaf_rn(e1, P.R32[3 + j], __fmul_rn(e0, P.R32[j])));
      z[k] = cam[2];
      const int32_t u = np_f32_to_i32(rintf(__fadd_rn(__fdiv_rn(__fmul_rn(fx, cam[0]), z[k]), cx)));
      const int32_t v = np_f32_to_i32(rintf(__fadd_rn(__fdiv_rn(__fmul_rn(fy, cam[1]), z[k]), cy)));
      const bool ok = z[k] > 0.f && u >= 0 && u < P.width && v >= 0 && v < P.height;
      pix[k] = ok ? v * P.width + u : -1;
    }
    float d[4];
    uint32_t r0[4], r1[4], r2[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      d[k] = 0.f;
      r0[k] = r1[k] = r2[k] = 0u;
      if (pix[k] >= 0) {
        const uint32_t* rec = row + 3 * (threadIdx.x + 128 * k);
        d[k] = depth[pix[k]];
        r0[k] = rec[0];
        r1[k] = rec[1];
        r2[k] = rec[2];
      }
    }
    bool any = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float sdf = __fsub_rn(d[k], z[k]);
      if (pix[k] < 0 || !(d[k] > 0.f && sdf >= neg_mu)) continue;
      const float obs = fminf(fmaxf(__fdiv_rn(sdf, mu), -1.0f), 1.0f);
      const uint8_t* px = color + 3 * (uint64_t)pix[k];
      const float tsdf = __uint_as_float(r0[k]), w = __uint_as_float(r1[k]);
      const float wn = __fadd_rn(w, 1.0f);
      uint32_t rgb = r2[k] & 0xff000000u;  // pad byte kept
#pragma unroll
      for (int ch = 0; ch < 3; ++ch) {
        const float old = (float)((r2[k] >> (8 * ch)) & 0xffu);
        const float cval = rintf(__fdiv_rn(__fadd_rn(__fmul_rn(old, w), (float)px[ch]), wn));
        rgb |= ((uint32_t)(uint8_t)(int)cval) << (8 * ch);
      }
      uint32_t* rec = row + 3 * (threadIdx.x + 128 * k);
      rec[0] = __float_as_uint(__fdiv_rn(__fadd_rn(__fmul_rn(tsdf, w), obs), wn));
      rec[1] = __float_as_uint(fminf(wn, maxw));
      rec[2] = rgb;
      any = true;
    }
    if (__any_sync(0xffffffffu, any) && (threadIdx.x & 31) == 0) touched[i] = 1;
    if (tick) {
      __syncthreads();  // the next claim is visible; claim[cb] is free again
      cb ^= 1;
      li = claim[cb];
    } else {
      li += gridDim.x;
    }
  }
}

}  // namespace vsb

using namespace vsb;

extern "C" {

vs_status vs_rc_candidates(const float* depth, const void* params_host, int32_t* keys_out, uint64_t cap,
                           uint64_t* n_dev, vs_stream_t stream) {
  if (!depth || !params_host || !n_dev || (cap && !keys_out)) {
    set_error("depth/params/keys_out/n_dev must be non-NULL");
    return VS_ERR_INVALID;
  }
  const RcParams& P = *(const RcParams*)params_host;
  if (P.stride < 1 || P.steps < 1 || P.steps > 64) {
    set_error("alloc_stride must be >= 1 and 1 <= steps <= 64");
    return VS_ERR_INVALID;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int32_t ws = (P.width + P.stride - 1) / P.stride, hs = (P.height + P.stride - 1) / P.stride;
  const uint64_t tiles = (uint64_t)((ws + 7) / 8) * (uint64_t)((hs + 3) / 4);
  VS_CK(cudaMemsetAsync(n_dev, 0, 8, s));
  if (tiles == 0) return VS_OK;
  { VS_CK(launch_pdl(k_rc_candidates, grid_for(32 * tiles, 256), 256, 0, s, depth, P, ws, hs, keys_out, (unsigned long long*)n_dev, cap)); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_rc_candidates");
  return VS_OK;
}

vs_status vs_rc_zero_rows(const int32_t* pos, const uint8_t* created, uint64_t n, uint8_t* pool, vs_stream_t stream) {
  if (n == 0) return VS_OK;
  if (!pos || !created || !pool) {
    set_error("pos/created/pool must be non-NULL");
    return VS_ERR_INVALID;
  }
  { VS_CK(launch_pdl(k_rc_zero_rows, grid_for(n, 256), 256, 0, (cudaStream_t)stream, pos, created, n, (uint4*)pool)); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_rc_zero_rows");
  return VS_OK;
}

}  // extern "C"

namespace vsb {
// persistent grid (all resident CTAs, capped by the block count) for k_rc_integrate
static unsigned integrate_grid(uint64_t n) {
  static int resident = 0;
  if (!resident) {
    int dev = 0, sms = 148, per_sm = 8;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_rc_integrate, 128, 0);
    resident = sms * (per_sm > 0 ? per_sm : 8);
  }
  return (unsigned)(n < (uint64_t)resident ? (n ? n : 1) : (uint64_t)resident);
}
}  // namespace vsb

extern "C" {

vs_status vs_rc_integrate(const int32_t* keys, const int32_t* pos, uint64_t n, const float* depth,
                          const uint8_t* color, const void* params_host, uint8_t* pool, uint8_t* touched,
                          vs_stream_t stream) {
  if (n == 0) return VS_OK;
  if (!keys || !pos || !depth || !color || !params_host || !pool || !touched) {
    set_error("keys/pos/depth/color/params/pool/touched must be non-NULL");
    return VS_ERR_INVALID;
  }
  const RcParams& P = *(const RcParams*)params_host;
  cudaStream_t s = (cudaStream_t)stream;
  // touched = 0 for all; the cull keeps in-view, non-rejected blocks; the
  // per-voxel kernel runs over the compacted survivors only
  uint8_t* keep = nullptr;
  uint64_t *off = nullptr, *work = nullptr;
  uint32_t* list = nullptr;
  VS_CK(cudaMallocAsync((void**)&keep, n, s));
  VS_CK(cudaMallocAsync((void**)&off, 8 * (n + 1), s));
  VS_CK(cudaMallocAsync((void**)&work, 8 * (scan_tiles(n) + 1), s));
  VS_CK(cudaMallocAsync((void**)&list, 4 * n + 16, s));
  unsigned long long* tick = VSB_RC_TICKET ? (unsigned long long*)(list + n + (n & 1)) : nullptr;
  if (tick) VS_CK(cudaMemsetAsync(tick, 0, 8, s));
  VS_CK(cudaMemsetAsync(touched, 0, n, s));
  {
    ProfScope prof(3, s);
    { VS_CK(launch_pdl(k_rc_cull, grid_for(n, 256), 256, 0, s, keys, n, depth, P, keep)); vsb::count_launch(); }
    VS_CK(exclusive_scan<uint8_t>(keep, n, off, work, s));
    { VS_CK(launch_pdl(k_rc_gather, grid_for(n, 256), 256, 0, s, keep, off, n, list)); vsb::count_launch(); }
    { VS_CK(launch_pdl(k_rc_integrate, integrate_grid(n), 128, 0, s, keys, pos, nullptr, list, off + n, depth, color, P, pool, touched, tick)); vsb::count_launch(); }
  }
  cudaFreeAsync(keep, s);
  cudaFreeAsync(off, s);
  cudaFreeAsync(work, s);
  cudaFreeAsync(list, s);
  VS_CK_LAUNCH("vs_rc_integrate");
  return VS_OK;
}

vs_status vs_rc_integrate_table(const vs_table* t, const float* depth, const uint8_t* color, const void* params_host,
                                uint8_t* pool, int32_t* touched_keys_out, uint64_t* n_touched_dev, vs_stream_t stream) {
  if (!t || !depth || !color || !params_host || !pool || !touched_keys_out || !n_touched_dev) {
    set_error("table/depth/color/params/pool/touched_keys_out/n_touched_dev must be non-NULL");
    return VS_ERR_INVALID;
  }
  DeviceGuard g(t->device);
  const RcParams& P = *(const RcParams*)params_host;
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t n = t->cap;
  // slots: cull (live + in view + not rejected) -> survivor list (any
  // order); integrate; touched slots -> scan -> keys (ascending slot order)
  uint8_t* touched = nullptr;
  uint64_t *off = nullptr, *work = nullptr;
  uint32_t* list = nullptr;
  VS_CK(cudaMallocAsync((void**)&touched, n, s));
  VS_CK(cudaMallocAsync((void**)&off, 8 * (n + 1), s));
  VS_CK(cudaMallocAsync((void**)&work, 8 * (scan_tiles(n) + 1), s));
  VS_CK(cudaMallocAsync((void**)&list, 4 * n + 16, s));
  unsigned long long* tick = VSB_RC_TICKET ? (unsigned long long*)(list + n + (n & 1)) : nullptr;
  if (tick) VS_CK(cudaMemsetAsync(tick, 0, 8, s));
  VS_CK(cudaMemsetAsync(touched, 0, n, s));
  {
    ProfScope prof(3, s);
    VS_CK(cudaMemsetAsync(off + n, 0, 8, s));
    { VS_CK(launch_pdl(k_rc_cull_table, grid_for(n, 256), 256, 0, s, t->e, t->cap, depth, P, list, (unsigned long long*)(off + n))); vsb::count_launch(); }
    { VS_CK(launch_pdl(k_rc_integrate, integrate_grid(n), 128, 0, s, nullptr, nullptr, t->e, list, off + n, depth, color, P, pool, touched, tick)); vsb::count_launch(); }
  }
  VS_CK(exclusive_scan<uint8_t>(touched, n, off, work, s));
  { VS_CK(launch_pdl(k_rc_touched_keys, grid_for(n, 256), 256, 0, s, touched, off, t->cap, t->e, touched_keys_out)); vsb::count_launch(); }
  VS_CK(cudaMemcpyAsync(n_touched_dev, off + n, 8, cudaMemcpyDeviceToDevice, s));
  cudaFreeAsync(touched, s);
  cudaFreeAsync(off, s);
  cudaFreeAsync(work, s);
  cudaFreeAsync(list, s);
  VS_CK_LAUNCH("vs_rc_integrate_table");
  return VS_OK;
}

uint64_t vs_rc_params_bytes(void) { return sizeof(RcParams); }

}  // extern "C"
