// Shared pieces of the tcgen05 attention kernels: UMMA descriptors for the
// [rows][128] bf16 tiles (two 64-column SW128 blocks), the matching smem
// swizzle, and 3-D TMA maps over the [tokens, heads, 128] Ulysses layout.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "ptx.cuh"

namespace opx {
namespace attn {

// CTA order: the grid is (tiles, heads); with band > 1 the linear block id
// walks bands of `band` heads tile-major (every head of the band at tile 0,
// then tile 1, ...), so the heaviest tiles of the LAST heads no longer start
// in the final wave (the causal tail).  band == 1 is the plain x-fastest order.
// Default band = the GQA group (its q heads share the K/V tiles; their Q/dO
// stay within L2): 7q/1kv (C1 SP4 rank shape) fwd 870 -> 930, bwd 795 -> 872
// TF/s; 28q/4kv within noise (fwd +1-3 %, bwd +-1 %); a band over all 28
// heads lost 3-4 % in the backward (Q/dO of 28 heads overflow L2).
// gridDim.y must be a multiple of band.
static __device__ __forceinline__ void cta_order(int band, int& bx, int& by) {
  if (band <= 1) {
    bx = blockIdx.x;
    by = blockIdx.y;
    return;
  }
  const int L = blockIdx.x + gridDim.x * blockIdx.y;
  const int per = band * gridDim.x;
  const int b = L / per, r = L % per;
  bx = r / band;
  by = b * band + r % band;
}
// band from the environment variable `name` (default `def`; 0 = the GQA
// group size g); a band that does not divide ny falls back to 1
static inline int cta_band(const char* name, int def, int g, int ny) {
  const char* e = getenv(name);
  int b = e ? atoi(e) : def;
  if (b == 0) b = g;
  return (b > 1 && ny % b == 0) ? b : 1;
}

static __device__ __forceinline__ uint64_t kdesc(uint32_t base, int k) {
  // K-major SW128 operand of a [128][128] tile stored as two 64-col blocks
  return ptx::umma_desc_sw128(base + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
}
static __device__ __forceinline__ uint64_t mndesc(uint32_t base, int k) {
  // MN-major SW128 operand: K rows of 128 B, the two 64-element MN chunks 16 KB apart
  return ptx::umma_desc_sw128(base + k * 2048, 16384, 1024);
}
// Packed fp32x2 ops (FFMA2 / FADD2 / FMUL2 on sm_100) and the 3-input max
// (FMNMX3): the softmax warps are issue-bound, these halve their FP work.
static __device__ __forceinline__ uint64_t f2pack(float a, float b) {
  uint64_t u;
  asm("mov.b64 %0, {%1, %2};" : "=l"(u) : "f"(a), "f"(b));
  return u;
}
static __device__ __forceinline__ void f2unpack(uint64_t u, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(u));
}
static __device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
static __device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
static __device__ __forceinline__ uint64_t fmul2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
static __device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x on the SFU, flush-to-zero (exp2f adds a denormal-range fixup per call)
static __device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// 2^x on the FMA/ALU pipes: 2^floor(x) * p(frac), p degree 3 (rel. err 8.6e-5);
// used for a fraction of the softmax exponentials to unload the SFU
static __device__ __forceinline__ float exp2_fma(float x) {
  x = fmaxf(x, -126.f);
  const float fi = floorf(x);
  const float f = x - fi;
  const float p = fmaf(fmaf(fmaf(0.07705827f, f, 0.2276545f), f, 0.69511473f), f, 1.0f);
  return __int_as_float(__float_as_int(p) + (int(fi) << 23));
}

// byte offset of 16-B chunk c (0..15) of row r in a [128][128] bf16 SW128 tile
static __device__ __forceinline__ uint32_t sw_off(int r, int c) {
  return (c >> 3) * 16384 + r * 128 + (((c & 7) ^ (r & 7)) << 4);
}


// byte offset of 16-B chunk c (0..7) of row r in a [rows][64] bf16 SW128 tile
static __device__ __forceinline__ uint32_t sw_off64(int r, int c) {
  return r * 128 + (((c & 7) ^ (r & 7)) << 4);
}

static inline PFN_cuTensorMapEncodeTiled_v12000 enc_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  return fn;
}

// [tokens, heads, 128] bf16 with token stride ld (elements) -> box {64, 1, 128}
static inline bool head_map(CUtensorMap* m, const void* base, int N, int heads, int64_t ld, int rows = 128) {
  auto enc = enc_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {128, cuuint64_t(heads), cuuint64_t(N)};
  cuuint64_t strides[2] = {256, cuuint64_t(ld) * 2};
  cuuint32_t box[3] = {64, 1, uint32_t(rows)};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}


// fp32 [tokens, heads, 128] map for bulk reduce-add of dQ: box {128, 1, rows}, no swizzle
static inline bool head_map_f32(CUtensorMap* m, const void* base, int N, int heads, int rows) {
  auto enc = enc_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {128, cuuint64_t(heads), cuuint64_t(N)};
  cuuint64_t strides[2] = {512, cuuint64_t(heads) * 512};
  cuuint32_t box[3] = {128, 1, uint32_t(rows)};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// fp32 [tokens, heads, 128] map with box {32, 1, rows}, SW128: the smem side is
// [rows][32 floats] with 16-B chunks XOR-swizzled by (row & 7), so one thread
// per row can write its 32 columns without bank conflicts (dK/dV partials).
static inline bool head_map_f32_sw(CUtensorMap* m, const void* base, int N, int heads, int rows) {
  auto enc = enc_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {128, cuuint64_t(heads), cuuint64_t(N)};
  cuuint64_t strides[2] = {512, cuuint64_t(heads) * 512};
  cuuint32_t box[3] = {32, 1, uint32_t(rows)};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace attn
}  // namespace opx
