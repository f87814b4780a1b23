// Causal packed-varlen GQA flash attention on tcgen05 (sm_100a), head_dim 128.
//
// Forward, one CTA per (128-query tile, q head):
//   warp 0      TMA producer: Q once, then K/V tiles (128 keys) into a 2-stage ring
//               (3-D tensor maps over the [tokens, heads, 128] Ulysses layout)
//   warp 1      MMA issuer (one elected lane):
//                 S_j = Q K_j^T  -> TMEM (double-buffered, 2 x 128 cols)
//                 O  += P_j V_j  -> TMEM (128 cols), P_j from smem
//               S_{j+1} is issued before waiting for P_j, so the next QK^T
//               overlaps the current softmax.
//   warps 2..5  softmax: one query row per thread (TMEM lane), masking from
//               per-token seq_start, online max with lazy rescaling (O is only
//               rescaled in TMEM when the row max grows by > 2^8), P -> bf16
//               -> 128B-swizzled smem for the PV MMA; epilogue O/l -> bf16, lse.
// Same AttnArgs contract as the mma.sync version (kernels/attention.cu).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "../runtime/kernels_api.h"
#include "ptx.cuh"

namespace opx {
namespace {

using bf16 = __nv_bfloat16;
constexpr int BM = 128, BN = 128, D = 128;
constexpr int TILE_BYTES = 128 * 128 * 2;  // 32 KB: [128 rows][128] bf16 as two 64-col SW128 blocks
constexpr int FWD_THREADS = 192;
constexpr int FWD_SMEM = 1024 + TILE_BYTES * (1 + 2 + 2 + 1) + 256;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_THRESH = 8.0f;

struct FwdParams {
  bf16* o;
  float* lse;
  int64_t ldo;
  const int* seq_start;
  int N, hq, hk, ntiles;
  float scale_log2;
};

__device__ __forceinline__ uint64_t kdesc(uint32_t base, int k) {
  // K-major SW128 operand of a [128][128] tile stored as two 64-col blocks
  return ptx::umma_desc_sw128(base + (k >> 2) * 16384 + (k & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t mndesc(uint32_t base, int k) {
  // MN-major SW128 operand: K rows of 128 B, the two 64-element MN chunks 16 KB apart
  return ptx::umma_desc_sw128(base + k * 2048, 16384, 1024);
}
// byte offset of 16-B chunk c (0..15) of row r in a [128][128] bf16 SW128 tile
__device__ __forceinline__ uint32_t sw_off(int r, int c) {
  return (c >> 3) * 16384 + r * 128 + (((c & 7) ^ (r & 7)) << 4);
}

__global__ void __launch_bounds__(FWD_THREADS, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv, const FwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK[2] = {smem + TILE_BYTES, smem + 2 * TILE_BYTES};
  uint8_t* sV[2] = {smem + 3 * TILE_BYTES, smem + 4 * TILE_BYTES};
  uint8_t* sP = smem + 5 * TILE_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 6 * TILE_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* s_empty = bars + 7;   // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* o_done = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile = p.ntiles - 1 - int(blockIdx.x);  // heavy (late) tiles first
  const int h = blockIdx.y;
  const int kh = h / (p.hq / p.hk);
  const int q0 = tile * BM;
  const int qlast = min(q0 + BM, p.N) - 1;
  const int kv0 = p.seq_start[q0] & ~(BN - 1);
  const int nkv = (qlast - kv0) / BN + 1;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tq);
    ptx::tma_prefetch(&tk);
    ptx::tma_prefetch(&tv);
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&kv_full[i], 1);
      ptx::mbar_init(&kv_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_empty[i], 128);
    }
    ptx::mbar_init(p_full, 128);
    ptx::mbar_init(o_done, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t TS[2] = {tmem, tmem + 128};
  const uint32_t TO = tmem + 256;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_expect_tx(q_full, TILE_BYTES);
      ptx::tma_load_3d(&tq, q_full, sQ, 0, h, q0);
      ptx::tma_load_3d(&tq, q_full, sQ + 16384, 64, h, q0);
      for (int j = 0; j < nkv; ++j) {
        const int st = j & 1;
        if (j >= 2) ptx::mbar_wait(&kv_empty[st], ((j >> 1) - 1) & 1);
        ptx::mbar_expect_tx(&kv_full[st], 2 * TILE_BYTES);
        const int k0 = kv0 + j * BN;
        ptx::tma_load_3d(&tk, &kv_full[st], sK[st], 0, kh, k0);
        ptx::tma_load_3d(&tk, &kv_full[st], sK[st] + 16384, 64, kh, k0);
        ptx::tma_load_3d(&tv, &kv_full[st], sV[st], 0, kh, k0);
        ptx::tma_load_3d(&tv, &kv_full[st], sV[st] + 16384, 64, kh, k0);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(BM, BN, false, false);
    constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(BM, D, false, true);
    const uint32_t q_addr = ptx::smem_u32(sQ);
    const uint32_t p_addr = ptx::smem_u32(sP);
    ptx::mbar_wait(q_full, 0);
    auto issue_pv = [&](int j) {
      ptx::mbar_wait(p_full, j & 1);
      ptx::tc_fence_after();
      if (lane == 0) {
        const uint32_t v_addr = ptx::smem_u32(sV[j & 1]);
#pragma unroll
        for (int k = 0; k < BN / 16; ++k)
          ptx::mma_bf16_ss(TO, kdesc(p_addr, k), mndesc(v_addr, k), idesc_o, (j | k) != 0);
        ptx::mma_commit(o_done);
        ptx::mma_commit(&kv_empty[j & 1]);
      }
      __syncwarp();
    };
    for (int j = 0; j < nkv; ++j) {
      const int st = j & 1;
      ptx::mbar_wait(&kv_full[st], (j >> 1) & 1);
      if (j >= 2) ptx::mbar_wait(&s_empty[st], ((j >> 1) - 1) & 1);
      ptx::tc_fence_after();
      if (lane == 0) {
        const uint32_t k_addr = ptx::smem_u32(sK[st]);
#pragma unroll
        for (int k = 0; k < D / 16; ++k)
          ptx::mma_bf16_ss(TS[st], kdesc(q_addr, k), kdesc(k_addr, k), idesc_s, k != 0);
        ptx::mma_commit(&s_full[st]);
      }
      __syncwarp();
      if (j >= 1) issue_pv(j - 1);
    }
    issue_pv(nkv - 1);
  } else {
    // ---------------- softmax warps ----------------
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int row = q0 + r;
    const bool valid_row = row < p.N;
    const int sst = valid_row ? p.seq_start[row] : 0x7fffffff;
    const uint32_t lane_off = uint32_t(quad * 32) << 16;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      const int sb = j & 1;
      ptx::mbar_wait(&s_full[sb], (j >> 1) & 1);
      ptx::tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        ptx::tmem_ld32(TS[sb] + lane_off + c * 32, v);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(v[i]);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&s_empty[sb]);
      const int kbase = kv0 + j * BN;
      const bool full_vis = kbase >= sst && kbase + BN - 1 <= row;
      float mx = -INFINITY;
      if (full_vis) {
#pragma unroll
        for (int i = 0; i < 128; ++i) {
          s[i] *= p.scale_log2;
          mx = fmaxf(mx, s[i]);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 128; ++i) {
          const int key = kbase + i;
          s[i] = (key >= sst && key <= row) ? s[i] * p.scale_log2 : -INFINITY;
          mx = fmaxf(mx, s[i]);
        }
      }
      // lazy rescale: only when the running max grows by more than 2^8
      const bool need = mx > m_used + RESCALE_THRESH || (m_used == -INFINITY && mx > -INFINITY);
      const float m_new = need ? mx : m_used;
      const float alpha = (need && m_used != -INFINITY) ? exp2f(m_used - m_new) : 1.f;
      if (j > 0) ptx::mbar_wait(o_done, (j - 1) & 1);  // PV_{j-1} done: O stable, P free
      ptx::tc_fence_after();
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          ptx::tmem_ld32(TO + lane_off + c * 32, v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
          uint32_t lo[16], hi[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            lo[i] = v[i];
            hi[i] = v[16 + i];
          }
          ptx::tmem_st16(TO + lane_off + c * 32, lo);
          ptx::tmem_st16(TO + lane_off + c * 32 + 16, hi);
        }
        ptx::tmem_wait_st();
      }
      l *= alpha;
      m_used = m_new;
      const float base = m_used == -INFINITY ? 0.f : m_used;
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float a0 = exp2f(s[c * 8 + 2 * e] - base);
          const float a1 = exp2f(s[c * 8 + 2 * e + 1] - base);
          sum += a0 + a1;
          w[e] = ptx::pack_bf16(a0, a1);
        }
        *reinterpret_cast<uint4*>(sP + sw_off(r, c)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      l += sum;
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_full);
    }
    ptx::mbar_wait(o_done, (nkv - 1) & 1);
    ptx::tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    bf16* orow = p.o + int64_t(valid_row ? row : 0) * p.ldo + int64_t(h) * D;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      ptx::tmem_ld32(TO + lane_off + c * 32, v);
      ptx::tmem_wait_ld();
      if (valid_row) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 o;
          o.x = ptx::pack_bf16(__uint_as_float(v[q * 8 + 0]) * inv, __uint_as_float(v[q * 8 + 1]) * inv);
          o.y = ptx::pack_bf16(__uint_as_float(v[q * 8 + 2]) * inv, __uint_as_float(v[q * 8 + 3]) * inv);
          o.z = ptx::pack_bf16(__uint_as_float(v[q * 8 + 4]) * inv, __uint_as_float(v[q * 8 + 5]) * inv);
          o.w = ptx::pack_bf16(__uint_as_float(v[q * 8 + 6]) * inv, __uint_as_float(v[q * 8 + 7]) * inv);
          *reinterpret_cast<uint4*>(orow + c * 32 + q * 8) = o;
        }
      }
    }
    if (valid_row) p.lse[int64_t(h) * p.N + row] = (m_used + log2f(l)) / LOG2E;
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

PFN_cuTensorMapEncodeTiled_v12000 enc_fn() {
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
bool head_map(CUtensorMap* m, const void* base, int N, int heads, int64_t ld) {
  auto enc = enc_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {128, cuuint64_t(heads), cuuint64_t(N)};
  cuuint64_t strides[2] = {256, cuuint64_t(ld) * 2};
  cuuint32_t box[3] = {64, 1, 128};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

cudaError_t k_attn_fwd_tc(const AttnArgs& a, cudaStream_t s) {
  if (a.N <= 0) return cudaSuccess;
  if (a.hq % a.hk || (a.ldq % 8) || (a.ldk % 8) || (a.ldv % 8)) return cudaErrorInvalidValue;
  CUtensorMap mq, mk, mv;
  if (!head_map(&mq, a.q, a.N, a.hq, a.ldq) || !head_map(&mk, a.k, a.N, a.hk, a.ldk) ||
      !head_map(&mv, a.v, a.N, a.hk, a.ldv))
    return cudaErrorInvalidValue;
  static bool cfg = false;
  if (!cfg) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, FWD_SMEM);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  FwdParams p;
  p.o = a.o;
  p.lse = a.lse;
  p.ldo = a.ldo;
  p.seq_start = a.seq_start;
  p.N = a.N;
  p.hq = a.hq;
  p.hk = a.hk;
  p.ntiles = (a.N + BM - 1) / BM;
  p.scale_log2 = a.scale * LOG2E;
  dim3 grid(p.ntiles, a.hq);
  ++g_kernel_launches;
  attn_fwd_tc_kernel<<<grid, FWD_THREADS, FWD_SMEM, s>>>(mq, mk, mv, p);
  return cudaGetLastError();
}



// ===========================================================================
// Backward on tcgen05.  One CTA per (128-key tile, kv head); loops over the
// q heads of the GQA group and over the 128-query tiles that can see the keys.
//   TMEM: S^T [0,128) | dP^T [128,256) | dV acc [256,384) | dK acc [384,512);
//         dQ_i (= dS K, 128 q x 128 d) reuses the S^T columns.
//   per q tile i (MMA warp):
//     S^T = K Q_i^T, dP^T = V dO_i^T                      -> s_full
//     (softmax warps: P^T = exp2(S^T*c - lse), dS^T = P^T (dP^T - delta)
//      -> bf16 SW128 smem, one key row per thread)        -> p_ready
//     dV += P^T dO_i, dK += dS^T Q_i, dQ_i = dS K          -> dq_full
//     (softmax warps read dQ_i rows from TMEM and red.add them into the fp32
//      dq accumulator)                                    -> st_free
// ===========================================================================
namespace {

constexpr int BWD_THREADS = 192;
constexpr int BWD_SMEM = 1024 + TILE_BYTES * 6 + 2 * 3 * 128 * 4 + 256;

struct BwdParams {
  const float* lse;
  const float* delta;
  float* dq_acc;
  bf16* dk;
  bf16* dv;
  int64_t lddk, lddv;
  const int* seq_start;
  const int* seq_end;
  int N, hq, hk;
  float scale, scale_log2;
};

__global__ void __launch_bounds__(BWD_THREADS, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                       const BwdParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = smem + TILE_BYTES;
  uint8_t* sQ = smem + 2 * TILE_BYTES;
  uint8_t* sO = smem + 3 * TILE_BYTES;  // dO tile
  uint8_t* sP = smem + 4 * TILE_BYTES;  // P^T [keys][q]
  uint8_t* sS = smem + 5 * TILE_BYTES;  // dS^T [keys][q]
  float* s_lse = reinterpret_cast<float*>(smem + 6 * TILE_BYTES);  // [2][128]
  float* s_dlt = s_lse + 256;                                       // [2][128]
  int* s_sst = reinterpret_cast<int*>(s_dlt + 256);                 // [2][128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_sst + 256);
  uint64_t* kv_full = bars + 0;
  uint64_t* qdo_full = bars + 1;
  uint64_t* qdo_empty = bars + 2;
  uint64_t* s_full = bars + 3;
  uint64_t* p_ready = bars + 4;
  uint64_t* dq_full = bars + 5;
  uint64_t* st_free = bars + 6;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 8);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k0 = blockIdx.x * BN;
  const int kh = blockIdx.y;
  const int G = p.hq / p.hk;
  const int klast = min(k0 + BN, p.N) - 1;
  const int qend = p.seq_end[klast];
  const int nq = (qend - k0 + BM - 1) / BM;
  const int niter = G * nq;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tq);
    ptx::tma_prefetch(&tk);
    ptx::tma_prefetch(&tv);
    ptx::tma_prefetch(&tdo);
    ptx::mbar_init(kv_full, 1);
    ptx::mbar_init(qdo_full, 1);
    ptx::mbar_init(qdo_empty, 1);
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(p_ready, 128);
    ptx::mbar_init(dq_full, 1);
    ptx::mbar_init(st_free, 128);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t TST = tmem, TDP = tmem + 128, TDV = tmem + 256, TDK = tmem + 384;

  if (warp == 0) {
    if (lane == 0) {
      ptx::mbar_expect_tx(kv_full, 2 * TILE_BYTES);
      ptx::tma_load_3d(&tk, kv_full, sK, 0, kh, k0);
      ptx::tma_load_3d(&tk, kv_full, sK + 16384, 64, kh, k0);
      ptx::tma_load_3d(&tv, kv_full, sV, 0, kh, k0);
      ptx::tma_load_3d(&tv, kv_full, sV + 16384, 64, kh, k0);
      for (int it = 0; it < niter; ++it) {
        const int h = kh * G + it / nq;
        const int q0 = k0 + (it % nq) * BM;
        if (it > 0) ptx::mbar_wait(qdo_empty, (it - 1) & 1);
        ptx::mbar_expect_tx(qdo_full, 2 * TILE_BYTES);
        ptx::tma_load_3d(&tq, qdo_full, sQ, 0, h, q0);
        ptx::tma_load_3d(&tq, qdo_full, sQ + 16384, 64, h, q0);
        ptx::tma_load_3d(&tdo, qdo_full, sO, 0, h, q0);
        ptx::tma_load_3d(&tdo, qdo_full, sO + 16384, 64, h, q0);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id_kk = ptx::idesc_bf16_f32(128, 128, false, false);
    constexpr uint32_t id_km = ptx::idesc_bf16_f32(128, 128, false, true);
    constexpr uint32_t id_mm = ptx::idesc_bf16_f32(128, 128, true, true);
    const uint32_t ak = ptx::smem_u32(sK), av = ptx::smem_u32(sV), aq = ptx::smem_u32(sQ),
                   ao = ptx::smem_u32(sO), ap = ptx::smem_u32(sP), as = ptx::smem_u32(sS);
    ptx::mbar_wait(kv_full, 0);
    for (int it = 0; it < niter; ++it) {
      ptx::mbar_wait(qdo_full, it & 1);
      if (it > 0) ptx::mbar_wait(st_free, (it - 1) & 1);
      ptx::tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k) ptx::mma_bf16_ss(TST, kdesc(ak, k), kdesc(aq, k), id_kk, k != 0);
#pragma unroll
        for (int k = 0; k < 8; ++k) ptx::mma_bf16_ss(TDP, kdesc(av, k), kdesc(ao, k), id_kk, k != 0);
        ptx::mma_commit(s_full);
      }
      __syncwarp();
      ptx::mbar_wait(p_ready, it & 1);
      ptx::tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          ptx::mma_bf16_ss(TDV, kdesc(ap, k), mndesc(ao, k), id_km, (it | k) != 0);
#pragma unroll
        for (int k = 0; k < 8; ++k)
          ptx::mma_bf16_ss(TDK, kdesc(as, k), mndesc(aq, k), id_km, (it | k) != 0);
#pragma unroll
        for (int k = 0; k < 8; ++k) ptx::mma_bf16_ss(TST, mndesc(as, k), mndesc(ak, k), id_mm, k != 0);
        ptx::mma_commit(dq_full);
        ptx::mma_commit(qdo_empty);
      }
      __syncwarp();
    }
  } else {
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int key = k0 + r;
    const uint32_t lane_off = uint32_t(quad * 32) << 16;
    for (int it = 0; it < niter; ++it) {
      const int h = kh * G + it / nq;
      const int q0 = k0 + (it % nq) * BM;
      const int buf = it & 1;
      {
        const int q = q0 + r;
        const bool ok = q < p.N;
        s_lse[buf * 128 + r] = ok ? p.lse[int64_t(h) * p.N + q] * LOG2E : INFINITY;
        s_dlt[buf * 128 + r] = ok ? p.delta[int64_t(h) * p.N + q] : 0.f;
        s_sst[buf * 128 + r] = ok ? p.seq_start[q] : 0x7fffffff;
      }
      asm volatile("bar.sync 1, 128;" ::: "memory");
      ptx::mbar_wait(s_full, it & 1);
      ptx::tc_fence_after();
      // all q columns visible for this key row?  (key <= q0, same sample)
      const bool full_vis = key <= q0 && s_sst[buf * 128 + 127] <= key && q0 + 127 < p.N &&
                            s_sst[buf * 128] <= key;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t sv[32], dv[32];
        ptx::tmem_ld32(TST + lane_off + c * 32, sv);
        ptx::tmem_ld32(TDP + lane_off + c * 32, dv);
        ptx::tmem_wait_ld();
        uint32_t pw[16], dw[16];
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float pp[2], ds[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int ql = c * 32 + i + e;
            const int q = q0 + ql;
            const bool ok = full_vis || (key <= q && key >= s_sst[buf * 128 + ql] && key < p.N);
            pp[e] = ok ? exp2f(__uint_as_float(sv[i + e]) * p.scale_log2 - s_lse[buf * 128 + ql]) : 0.f;
            ds[e] = pp[e] * (__uint_as_float(dv[i + e]) - s_dlt[buf * 128 + ql]);
          }
          pw[i / 2] = ptx::pack_bf16(pp[0], pp[1]);
          dw[i / 2] = ptx::pack_bf16(ds[0], ds[1]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int chunk = c * 4 + q;
          *reinterpret_cast<uint4*>(sP + sw_off(r, chunk)) =
              make_uint4(pw[q * 4], pw[q * 4 + 1], pw[q * 4 + 2], pw[q * 4 + 3]);
          *reinterpret_cast<uint4*>(sS + sw_off(r, chunk)) =
              make_uint4(dw[q * 4], dw[q * 4 + 1], dw[q * 4 + 2], dw[q * 4 + 3]);
        }
      }
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_ready);
      // dQ_i rows (TMEM lane r = query q0 + r) -> fp32 accumulator
      ptx::mbar_wait(dq_full, it & 1);
      ptx::tc_fence_after();
      const int q = q0 + r;
      float* dst = p.dq_acc + (int64_t(q < p.N ? q : 0) * p.hq + h) * D;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        ptx::tmem_ld32(TST + lane_off + c * 32, v);
        ptx::tmem_wait_ld();
        if (q < p.N) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            atomicAdd(reinterpret_cast<float4*>(dst + c * 32 + i),
                      make_float4(__uint_as_float(v[i]) * p.scale, __uint_as_float(v[i + 1]) * p.scale,
                                  __uint_as_float(v[i + 2]) * p.scale, __uint_as_float(v[i + 3]) * p.scale));
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(st_free);
    }
    // dK (scaled), dV rows -> bf16
    if (niter > 0) {
      const bool ok = key < p.N;
      bf16* dkr = p.dk + int64_t(ok ? key : 0) * p.lddk + int64_t(kh) * D;
      bf16* dvr = p.dv + int64_t(ok ? key : 0) * p.lddv + int64_t(kh) * D;
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        uint32_t a[32], b[32];
        ptx::tmem_ld32(TDK + lane_off + c * 32, a);
        ptx::tmem_ld32(TDV + lane_off + c * 32, b);
        ptx::tmem_wait_ld();
        if (ok) {
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 ka, va;
            uint32_t* kp = reinterpret_cast<uint32_t*>(&ka);
            uint32_t* vp = reinterpret_cast<uint32_t*>(&va);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              kp[e] = ptx::pack_bf16(__uint_as_float(a[q * 8 + 2 * e]) * p.scale,
                                     __uint_as_float(a[q * 8 + 2 * e + 1]) * p.scale);
              vp[e] = ptx::pack_bf16(__uint_as_float(b[q * 8 + 2 * e]), __uint_as_float(b[q * 8 + 2 * e + 1]));
            }
            *reinterpret_cast<uint4*>(dkr + c * 32 + q * 8) = ka;
            *reinterpret_cast<uint4*>(dvr + c * 32 + q * 8) = va;
          }
        }
      }
    }
  }
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 1) ptx::tmem_dealloc(tmem, 512);
}

// delta[h, t] = sum_d dO[t,h,d] * O[t,h,d]   (one warp per (t, h))
__global__ void delta_kernel(const bf16* __restrict__ dout, int64_t lddo, const bf16* __restrict__ o,
                             int64_t ldo, float* __restrict__ delta, int N, int hq) {
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= int64_t(N) * hq) return;
  const int tok = int(w / hq), h = int(w % hq);
  const uint2 x = *reinterpret_cast<const uint2*>(dout + int64_t(tok) * lddo + h * D + lane * 4);
  const uint2 y = *reinterpret_cast<const uint2*>(o + int64_t(tok) * ldo + h * D + lane * 4);
  const float2 x0 = ptx::unpack_bf16(x.x), x1 = ptx::unpack_bf16(x.y);
  const float2 y0 = ptx::unpack_bf16(y.x), y1 = ptx::unpack_bf16(y.y);
  float s = x0.x * y0.x + x0.y * y0.y + x1.x * y1.x + x1.y * y1.y;
#pragma unroll
  for (int off = 16; off; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
  if (lane == 0) delta[int64_t(h) * N + tok] = s;
}

}  // namespace

cudaError_t k_attn_bwd_tc(const AttnArgs& a, cudaStream_t s) {
  if (a.N <= 0) return cudaSuccess;
  if (a.hq % a.hk) return cudaErrorInvalidValue;
  CUtensorMap mq, mk, mv, mdo;
  if (!head_map(&mq, a.q, a.N, a.hq, a.ldq) || !head_map(&mk, a.k, a.N, a.hk, a.ldk) ||
      !head_map(&mv, a.v, a.N, a.hk, a.ldv) || !head_map(&mdo, a.dout, a.N, a.hq, a.lddo))
    return cudaErrorInvalidValue;
  static bool cfg = false;
  if (!cfg) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_tc_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_SMEM);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  const int64_t warps = int64_t(a.N) * a.hq;
  ++g_kernel_launches;
  delta_kernel<<<int((warps * 32 + 255) / 256), 256, 0, s>>>(a.dout, a.lddo, a.o, a.ldo, a.delta,
                                                              a.N, a.hq);
  cudaError_t e = cudaMemsetAsync(a.dq_acc, 0, size_t(a.N) * a.hq * D * sizeof(float), s);
  if (e != cudaSuccess) return e;
  BwdParams p;
  p.lse = a.lse;
  p.delta = a.delta;
  p.dq_acc = a.dq_acc;
  p.dk = a.dk;
  p.dv = a.dv;
  p.lddk = a.lddk;
  p.lddv = a.lddv;
  p.seq_start = a.seq_start;
  p.seq_end = a.seq_end;
  p.N = a.N;
  p.hq = a.hq;
  p.hk = a.hk;
  p.scale = a.scale;
  p.scale_log2 = a.scale * LOG2E;
  dim3 grid((a.N + BN - 1) / BN, a.hk);
  ++g_kernel_launches;
  attn_bwd_tc_kernel<<<grid, BWD_THREADS, BWD_SMEM, s>>>(mq, mk, mv, mdo, p);
  return cudaGetLastError();
}

}  // namespace opx
