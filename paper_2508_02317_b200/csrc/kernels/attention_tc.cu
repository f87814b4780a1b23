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
#include "attn_common.cuh"
#include "ptx.cuh"

namespace opx {
namespace {
using namespace attn;

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

__global__ void __launch_bounds__(FWD_THREADS, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv, const FwdParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-B alignment by pointer arithmetic on the __shared__ array keeps the
  // shared address space (no generic LD/ST on the hot path).
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
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

}  // namespace opx
