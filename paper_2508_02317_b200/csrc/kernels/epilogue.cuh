// Shared GEMM epilogue pieces (kernels/gemm.cu, kernels/gemm2.cu).
#pragma once
#include "ptx.cuh"

namespace opx {
namespace epi {

// f[0..31] += bias[0..31] (bf16 column bias, 16-B aligned)
__device__ __forceinline__ void add_bias32(float* f, const __nv_bfloat16* b) {
  const uint4* bp = reinterpret_cast<const uint4*>(b);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 v = bp[q];
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = ptx::unpack_bf16(w[e]);
      f[q * 8 + 2 * e] += x.x;
      f[q * 8 + 2 * e + 1] += x.y;
    }
  }
}

// SwiGLU backward fused into the dact GEMM: 32 accumulator columns (dact for
// features f0 .. f0+31 of one row, rounded to bf16 exactly as the unfused path
// stored it) with the forward's gate/up (128-column interleave: gate of
// feature f at (f/128)*256 + f%128, up 128 further) -> d(gate), d(up).
__device__ __forceinline__ void swiglu_bwd32(const uint32_t* acc, const __nv_bfloat16* gu_row,
                                             __nv_bfloat16* dgu_row, int f0) {
  const int base = (f0 / 128) * 256 + (f0 % 128);
  const uint4* gp = reinterpret_cast<const uint4*>(gu_row + base);
  const uint4* up = reinterpret_cast<const uint4*>(gu_row + base + 128);
  uint4* dgp = reinterpret_cast<uint4*>(dgu_row + base);
  uint4* dup = reinterpret_cast<uint4*>(dgu_row + base + 128);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint4 gq = gp[q], uq = up[q];
    const uint32_t gv[4] = {gq.x, gq.y, gq.z, gq.w}, uv[4] = {uq.x, uq.y, uq.z, uq.w};
    uint32_t og[4], ou[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 a = ptx::unpack_bf16(
          ptx::pack_bf16(__uint_as_float(acc[q * 8 + 2 * e]), __uint_as_float(acc[q * 8 + 2 * e + 1])));
      const float2 g = ptx::unpack_bf16(gv[e]), u = ptx::unpack_bf16(uv[e]);
      const float aa[2] = {a.x, a.y}, gg[2] = {g.x, g.y}, uu[2] = {u.x, u.y};
      float dg[2], du[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float sg = 1.f / (1.f + __expf(-gg[k]));
        du[k] = aa[k] * (gg[k] * sg);
        dg[k] = aa[k] * uu[k] * sg * (1.f + gg[k] * (1.f - sg));
      }
      og[e] = ptx::pack_bf16(dg[0], dg[1]);
      ou[e] = ptx::pack_bf16(du[0], du[1]);
    }
    dgp[q] = make_uint4(og[0], og[1], og[2], og[3]);
    dup[q] = make_uint4(ou[0], ou[1], ou[2], ou[3]);
  }
}

}  // namespace epi
}  // namespace opx
