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

// One thread per (sampled pixel, depth step).  Emits the sample's block key
// (warp-deduplicated) and, for samples within _BOUNDARY_EPS of a face, the
// face/edge/corner neighbours (_segment_block_keys).
__global__ void __launch_bounds__(256) k_rc_candidates(const float* __restrict__ depth, const __grid_constant__ RcParams P,
                                                       int32_t ws, int32_t hs, int32_t* __restrict__ out,
                                                       unsigned long long* __restrict__ count, uint64_t cap) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t total = (uint64_t)ws * hs * P.steps;
  bool valid = false;
  long long b[3] = {0, 0, 0};
  bool lo[3] = {false, false, false}, hi[3] = {false, false, false};
  if (gid < total) {
    const uint64_t p = gid / P.steps;
    const int j = (int)(gid % P.steps);
    const int32_t u = (int32_t)(p % ws) * P.stride, v = (int32_t)(p / ws) * P.stride;
    const float d32 = depth[(uint64_t)v * P.width + u];
    if (d32 > 0.f) {
      valid = true;
      // pixel_rays: ((u - cx) / fx, (v - cy) / fy, 1)
      const double r0 = __ddiv_rn(__dsub_rn((double)u, P.cx), P.fx);
      const double r1 = __ddiv_rn(__dsub_rn((double)v, P.cy), P.fy);
      const double d = (double)d32;
      const double z0 = fmax(__dsub_rn(d, P.mu), P.voxel);
      const double z1 = __dadd_rn(d, P.mu);
      const double zs = __dadd_rn(z0, __dmul_rn(__dsub_rn(z1, z0), P.ts[j]));
      const double p0 = __dmul_rn(r0, zs), p1 = __dmul_rn(r1, zs), p2 = zs;  // rays * zs (ray z = 1)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        // pose.transform: pts @ R.T + t
        const double w = __dadd_rn(__fma_rn(p2, P.R[3 * k + 2], __fma_rn(p1, P.R[3 * k + 1], __dmul_rn(p0, P.R[3 * k]))),
                                   P.t[k]);
        const double g = __ddiv_rn(w, P.block);
        const double fl = floor(g);
        const double frac = __dsub_rn(g, fl);
        b[k] = (long long)fl;
        lo[k] = frac < P.tol;
        hi[k] = frac > P.one_minus_tol;
      }
    }
  }
  // base key: one emission per distinct key in the warp
  const unsigned long long enc = ((unsigned long long)(b[0] + (1 << 20)) << 42) |
                                 ((unsigned long long)(b[1] + (1 << 20)) << 21) | (unsigned long long)(b[2] + (1 << 20));
  const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
  const uint32_t same = __match_any_sync(0xffffffffu, valid ? enc : ~0ull) & vmask;
  const bool leader = valid && (__ffs(same) - 1) == (int)lane_id();
  const bool edgy = valid && (lo[0] | lo[1] | lo[2] | hi[0] | hi[1] | hi[2]);
  int n_emit = leader ? 1 : 0;
  if (edgy) {
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          if (!dx && !dy && !dz) continue;
          const int dd[3] = {dx, dy, dz};
          bool m = true;
#pragma unroll
          for (int a = 0; a < 3; ++a) m &= dd[a] == 0 || (dd[a] < 0 ? lo[a] : hi[a]);
          n_emit += m;
        }
  }
  // warp-aggregated reservation of the output slots
  int incl = n_emit;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if ((int)lane_id() >= o) incl += y;
  }
  const int total_w = __shfl_sync(0xffffffffu, incl, 31);
  unsigned long long base = 0;
  if (lane_id() == 31 && total_w) base = atomicAdd(count, (unsigned long long)total_w);
  base = __shfl_sync(0xffffffffu, base, 31);
  unsigned long long o = base + (unsigned long long)(incl - n_emit);
  auto put = [&](long long x, long long y, long long z) {
    if (o < cap) {
      out[3 * o] = (int32_t)x;
      out[3 * o + 1] = (int32_t)y;
      out[3 * o + 2] = (int32_t)z;
    }
    ++o;
  };
  if (leader) put(b[0], b[1], b[2]);
  if (edgy) {
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          if (!dx && !dy && !dz) continue;
          const int dd[3] = {dx, dy, dz};
          bool m = true;
#pragma unroll
          for (int a = 0; a < 3; ++a) m &= dd[a] == 0 || (dd[a] < 0 ? lo[a] : hi[a]);
          if (m) put(b[0] + dx, b[1] + dy, b[2] + dz);
        }
  }
}

// Zero the pool rows of newly created blocks (TsdfBlock(): all zero).
__global__ void k_rc_zero_rows(const int32_t* __restrict__ pos, const uint8_t* __restrict__ created, uint64_t n,
                               uint4* __restrict__ pool) {
  const uint64_t i = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n || !created[i]) return;
  uint4* dst = pool + (uint64_t)pos[i] * (VS_TSDF_BLOCK_BYTES / 16);
  for (int j = lane; j < VS_TSDF_BLOCK_BYTES / 16; j += 32) dst[j] = make_uint4(0, 0, 0, 0);
}

// ----------------------------------------------------------------- fusion

// numpy float32 -> int32 (astype): NaN / out-of-range give INT32_MIN on x86.
__device__ __forceinline__ int32_t np_f32_to_i32(float r) {
  if (!(r >= -2147483648.0f && r < 2147483648.0f)) return INT32_MIN;
  return (int32_t)r;
}

// One CTA (128 threads, 4 voxels each) per live block.
__global__ void __launch_bounds__(128) k_rc_integrate(const int32_t* __restrict__ keys, const int32_t* __restrict__ pos,
                                                      uint64_t n, const float* __restrict__ depth,
                                                      const uint8_t* __restrict__ color, const __grid_constant__ RcParams P,
                                                      uint8_t* __restrict__ pool, uint8_t* __restrict__ touched) {
  const uint64_t i = blockIdx.x;
  if (i >= n) return;
  const int32_t kx = keys[3 * i], ky = keys[3 * i + 1], kz = keys[3 * i + 2];
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
  if (!inview) {
    if (threadIdx.x == 0) touched[i] = 0;
    return;
  }
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
      if (cd > 0.f && fabs(__dsub_rn((double)cd, cz)) > P.reach) {
        if (threadIdx.x == 0) touched[i] = 0;
        return;
      }
    }
  }
  // --- per voxel: project, sample, weighted running average (in place)
  const float fx = (float)P.fx, fy = (float)P.fy, cx = (float)P.cx, cy = (float)P.cy;
  const float mu = (float)P.mu, neg_mu = (float)(-P.mu), maxw = (float)P.max_weight;
  uint8_t* row = pool + (uint64_t)pos[i] * VS_TSDF_BLOCK_BYTES;
  int any = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int f = threadIdx.x + 128 * k;
    const int lx = f & 7, ly = (f >> 3) & 7, lz = f >> 6;
    // coords = ((origins + LOCAL + 0.5) * voxel).astype(float32)
    const float c0 = __double2float_rn(__dmul_rn((double)(8ll * kx + lx) + 0.5, P.voxel));
    const float c1 = __double2float_rn(__dmul_rn((double)(8ll * ky + ly) + 0.5, P.voxel));
    const float c2 = __double2float_rn(__dmul_rn((double)(8ll * kz + lz) + 0.5, P.voxel));
    const float e0 = __fsub_rn(c0, P.t32[0]), e1 = __fsub_rn(c1, P.t32[1]), e2 = __fsub_rn(c2, P.t32[2]);
    float cam[3];
#pragma unroll
    for (int j = 0; j < 3; ++j)  // (coords - trans) @ rot, float32
      cam[j] = __fmaf_rn(e2, P.R32[6 + j], __fmaf_rn(e1, P.R32[3 + j], __fmul_rn(e0, P.R32[j])));
    const float z = cam[2];
    const int32_t u = np_f32_to_i32(rintf(__fadd_rn(__fdiv_rn(__fmul_rn(fx, cam[0]), z), cx)));
    const int32_t v = np_f32_to_i32(rintf(__fadd_rn(__fdiv_rn(__fmul_rn(fy, cam[1]), z), cy)));
    bool ok = z > 0.f && u >= 0 && u < P.width && v >= 0 && v < P.height;
    if (!ok) continue;
    const float d = depth[(uint64_t)v * P.width + u];
    const float sdf = __fsub_rn(d, z);
    if (!(d > 0.f && sdf >= neg_mu)) continue;
    const float obs = fminf(fmaxf(__fdiv_rn(sdf, mu), -1.0f), 1.0f);
    const uint8_t* px = color + 3 * ((uint64_t)v * P.width + u);
    float* tw = (float*)(row + 12 * f);
    uint8_t* rgb = row + 12 * f + 8;
    const float w = tw[1];
    const float wn = __fadd_rn(w, 1.0f);
    tw[0] = __fdiv_rn(__fadd_rn(__fmul_rn(tw[0], w), obs), wn);
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
      const float cval = rintf(__fdiv_rn(__fadd_rn(__fmul_rn((float)rgb[ch], w), (float)px[ch]), wn));
      rgb[ch] = (uint8_t)(int)cval;
    }
    tw[1] = fminf(wn, maxw);
    any = 1;
  }
  any = __syncthreads_or(any);
  if (threadIdx.x == 0) touched[i] = (uint8_t)any;
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
  const uint64_t total = (uint64_t)ws * hs * P.steps;
  VS_CK(cudaMemsetAsync(n_dev, 0, 8, s));
  if (total == 0) return VS_OK;
  { k_rc_candidates<<<grid_for(total, 256), 256, 0, s>>>(depth, P, ws, hs, keys_out, (unsigned long long*)n_dev, cap); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_rc_candidates");
  return VS_OK;
}

vs_status vs_rc_zero_rows(const int32_t* pos, const uint8_t* created, uint64_t n, uint8_t* pool, vs_stream_t stream) {
  if (n == 0) return VS_OK;
  if (!pos || !created || !pool) {
    set_error("pos/created/pool must be non-NULL");
    return VS_ERR_INVALID;
  }
  { k_rc_zero_rows<<<grid_for(32 * n, 256), 256, 0, (cudaStream_t)stream>>>(pos, created, n, (uint4*)pool); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_rc_zero_rows");
  return VS_OK;
}

vs_status vs_rc_integrate(const int32_t* keys, const int32_t* pos, uint64_t n, const float* depth,
                          const uint8_t* color, const void* params_host, uint8_t* pool, uint8_t* touched,
                          vs_stream_t stream) {
  if (n == 0) return VS_OK;
  if (!keys || !pos || !depth || !color || !params_host || !pool || !touched) {
    set_error("keys/pos/depth/color/params/pool/touched must be non-NULL");
    return VS_ERR_INVALID;
  }
  const RcParams& P = *(const RcParams*)params_host;
  { ProfScope prof(3, (cudaStream_t)stream); k_rc_integrate<<<(unsigned)n, 128, 0, (cudaStream_t)stream>>>(keys, pos, n, depth, color, P, pool, touched); vsb::count_launch(); }
  VS_CK_LAUNCH("vs_rc_integrate");
  return VS_OK;
}

uint64_t vs_rc_params_bytes(void) { return sizeof(RcParams); }

}  // extern "C"
