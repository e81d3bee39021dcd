// faces.cuh -- the MC encoder's IEEE-bit predicates and the face bit-pack of
// one TSDF row (the encoder's halo side table), shared by the encoder
// (mc.cu) and the TSDF ingest (stream.cu, which refreshes the packs of the
// rows it writes in the same pass).
#pragma once
#include <cstdint>

namespace vsb {

// predicates on the IEEE bits, independent of FTZ/DAZ:
//   inside   <=> 0x80000000 <  bits <= 0xFF800000   (tsdf < 0, NaN false)
//   observed <=> 0 < (int32)bits <= 0x7F800000       (weight > 0, NaN false)
// each as ONE unsigned range check (wrap-around subtraction)
__device__ __forceinline__ uint32_t inside_bit(uint32_t b) { return (b - 0x80000001u) < 0x7F800000u ? 1u : 0u; }
__device__ __forceinline__ uint32_t observed_bit(uint32_t b) { return (b - 1u) < 0x7F800000u ? 1u : 0u; }

constexpr int kFaceBytes = 48;

// Face bit-packs of one 6,144-B wire row `src` by ONE warp (every lane must
// call): the inside/observed bits of the row's x = 0 face (bit y + 8z), y = 0
// face (bit x + 8z) and z = 0 face (bit x + 8y), each as {inside lo, inside
// hi, observed lo, observed hi}, 48 B at `dst` (16-byte aligned).  Lane l
// takes bits l and l + 32 of each face.
__device__ __forceinline__ void face_pack_warp(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst) {
  const uint32_t lane = threadIdx.x & 31u;
  uint32_t word[3][4];
#pragma unroll
  for (int f = 0; f < 3; ++f) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int i = (int)lane + 32 * half;
      const int a = i & 7, b = i >> 3;
      const int flat = f == 0 ? 8 * a + 64 * b : (f == 1 ? a + 64 * b : a + 8 * b);
      const uint32_t* v = (const uint32_t*)(src + 12 * flat);
      const uint32_t in = __ballot_sync(0xFFFFFFFFu, inside_bit(__ldg(v)));
      const uint32_t ob = __ballot_sync(0xFFFFFFFFu, observed_bit(__ldg(v + 1)));
      word[f][half] = in;
      word[f][2 + half] = ob;
    }
  }
#pragma unroll
  for (int f = 0; f < 3; ++f)
    if (lane == (uint32_t)f) ((uint4*)dst)[f] = make_uint4(word[f][0], word[f][1], word[f][2], word[f][3]);
}

}  // namespace vsb
