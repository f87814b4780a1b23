// Causal (or, for the frozen encoder, bidirectional) packed-varlen GQA flash
// attention FORWARD on tcgen05 (sm_100a), d = 128.
//
// One CTA per (pair of consecutive 128-query tiles, q head), 320 threads:
//   warp 0       TMA producer: Q0/Q1 once, K tiles (128 keys) into a 2-stage
//                ring, V into a single buffer (3-D maps over [tokens, heads, 128])
//   warp 1       MMA issuer (one elected lane), order per key tile j:
//                  S0(j+1) = Q0 K^T, S1(j+1) = Q1 K^T      (TMEM, 128 cols each)
//                  O0 += P0(j) V(j), O1 += P1(j) V(j)      (TMEM, 128 cols each)
//                so the QK^T of the next tile runs under the current softmax.
//   warps 2..5   softmax warpgroup of tile 0, warps 6..9 of tile 1: one query
//                row per thread (TMEM lane); masking from per-token seq_start;
//                lazy rescaling of O in TMEM (only when the row max grows by
//                > 2^8); a quarter of the exponentials on the FMA pipe (degree-3
//                polynomial, 8.6e-5 rel. error) to relieve MUFU; P -> bf16 ->
//                128B-swizzled smem for the PV MMA; epilogue O/l -> bf16, lse.
// The two warpgroups ping-pong against the single tensor-core pipe.
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
constexpr int FWD_THREADS = 320;
// smem: Q0 | Q1 | K[0] | K[1] | V | P0 | P1 | barriers
constexpr int FWD_SMEM = 1024 + TILE_BYTES * 7 + 256;
constexpr float LOG2E = 1.4426950408889634f;
constexpr float RESCALE_THRESH = 8.0f;
// 1/POLY_SHARE of the exponentials go to the FMA-pipe polynomial (0: none).
// Measured on B200 (C1 shapes): 1/4 -> 844 TF/s, 1/2 -> 675 TF/s: the softmax
// warps are issue-bound, not MUFU-bound, so only a small share is moved.
#ifndef OPX_FWD_POLY_SHARE
#define OPX_FWD_POLY_SHARE 4
#endif
constexpr int POLY_SHARE = OPX_FWD_POLY_SHARE;

struct FwdParams {
  bf16* o;
  float* lse;
  int64_t ldo;
  const int* seq_start;
  const int* seq_end;  // bidirectional mode only
  int N, hq, hk, npairs, causal;
  float scale_log2;
  int band;  // CTA order (attn::cta_order)
};


__global__ void __launch_bounds__(FWD_THREADS, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv, const FwdParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-B alignment by pointer arithmetic on the __shared__ array keeps the
  // shared address space (no generic LD/ST on the hot path).
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  // tile addresses by arithmetic, not by runtime-indexed arrays (those went to
  // the stack and turned the P stores into generic ST.E)
  auto sQ = [&](int i) { return smem + i * TILE_BYTES; };
  auto sK = [&](int i) { return smem + (2 + i) * TILE_BYTES; };
  uint8_t* sV = smem + 4 * TILE_BYTES;
  auto sP = [&](int i) { return smem + (5 + i) * TILE_BYTES; };
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 7 * TILE_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;
  uint64_t* v_empty = bars + 6;
  uint64_t* s_full = bars + 7;   // [2] per tile
  uint64_t* s_empty = bars + 9;  // [2]
  uint64_t* p_full = bars + 11;  // [2]
  uint64_t* o_done = bars + 13;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 16);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int bx, by;
  cta_order(p.band, bx, by);
  const int pair = p.npairs - 1 - bx;  // heavy (late) tiles first
  const int h = by;
  const int kh = h / (p.hq / p.hk);
  const int q0 = pair * 2 * BM;
  const int qlast = min(q0 + 2 * BM, p.N) - 1;
  const int kv0 = p.seq_start[q0] & ~(BN - 1);
  // last key any row of the pair sees: the row itself (causal) or the end of
  // its sample (bidirectional; seq_end is non-decreasing in the row)
  const int klast = p.causal ? qlast : p.seq_end[qlast] - 1;
  const int nkv = (klast - kv0) / BN + 1;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tq);
    ptx::tma_prefetch(&tk);
    ptx::tma_prefetch(&tv);
    ptx::mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      ptx::mbar_init(&k_full[i], 1);
      ptx::mbar_init(&k_empty[i], 1);
      ptx::mbar_init(&s_full[i], 1);
      ptx::mbar_init(&s_empty[i], 128);
      ptx::mbar_init(&p_full[i], 128);
      ptx::mbar_init(&o_done[i], 1);
    }
    ptx::mbar_init(v_full, 1);
    ptx::mbar_init(v_empty, 1);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto TS = [&](int i) { return tmem + uint32_t(i) * 128; };
  auto TO = [&](int i) { return tmem + 256 + uint32_t(i) * 128; };

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      ptx::mbar_expect_tx(q_full, 2 * TILE_BYTES);
      ptx::tma_load_3d(&tq, q_full, sQ(0), 0, h, q0);
      ptx::tma_load_3d(&tq, q_full, sQ(0) + 16384, 64, h, q0);
      ptx::tma_load_3d(&tq, q_full, sQ(1), 0, h, q0 + BM);
      ptx::tma_load_3d(&tq, q_full, sQ(1) + 16384, 64, h, q0 + BM);
      auto load_k = [&](int j) {
        const int st = j & 1;
        if (j >= 2) ptx::mbar_wait(&k_empty[st], ((j >> 1) - 1) & 1);
        ptx::mbar_expect_tx(&k_full[st], TILE_BYTES);
        ptx::tma_load_3d(&tk, &k_full[st], sK(st), 0, kh, kv0 + j * BN);
        ptx::tma_load_3d(&tk, &k_full[st], sK(st) + 16384, 64, kh, kv0 + j * BN);
      };
      load_k(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) load_k(j + 1);
        if (j >= 1) ptx::mbar_wait(v_empty, (j - 1) & 1);
        ptx::mbar_expect_tx(v_full, TILE_BYTES);
        ptx::tma_load_3d(&tv, v_full, sV, 0, kh, kv0 + j * BN);
        ptx::tma_load_3d(&tv, v_full, sV + 16384, 64, kh, kv0 + j * BN);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc_s = ptx::idesc_bf16_f32(BM, BN, false, false);
    constexpr uint32_t idesc_o = ptx::idesc_bf16_f32(BM, D, false, true);
    const uint32_t qa0 = ptx::smem_u32(sQ(0)), pa0 = ptx::smem_u32(sP(0));
    const uint32_t va = ptx::smem_u32(sV);
    ptx::mbar_wait(q_full, 0);
    auto issue_s = [&](int j) {
      const int st = j & 1;
      ptx::mbar_wait(&k_full[st], (j >> 1) & 1);
      const uint32_t ka = ptx::smem_u32(sK(st));
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (j > 0) ptx::mbar_wait(&s_empty[t], (j - 1) & 1);
        ptx::tc_fence_after();
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < D / 16; ++k)
            ptx::mma_bf16_ss(TS(t), kdesc(qa0 + uint32_t(t) * TILE_BYTES, k), kdesc(ka, k), idesc_s, k != 0);
          ptx::mma_commit(&s_full[t]);
        }
        __syncwarp();
      }
      if (lane == 0) ptx::mma_commit(&k_empty[st]);
      __syncwarp();
    };
    auto issue_pv = [&](int j) {
      ptx::mbar_wait(v_full, j & 1);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        ptx::mbar_wait(&p_full[t], j & 1);
        ptx::tc_fence_after();
        if (lane == 0) {
#pragma unroll
          for (int k = 0; k < BN / 16; ++k)
            ptx::mma_bf16_ss(TO(t), kdesc(pa0 + uint32_t(t) * TILE_BYTES, k), mndesc(va, k), idesc_o, (j | k) != 0);
          ptx::mma_commit(&o_done[t]);
        }
        __syncwarp();
      }
      if (lane == 0) ptx::mma_commit(v_empty);
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < nkv; ++j) {
      if (j + 1 < nkv) issue_s(j + 1);
      issue_pv(j);
    }
  } else {
    // ---------------- softmax warpgroups ----------------
    const int t = (warp - 2) >> 2;  // tile of this warpgroup
    const int quad = warp & 3;      // TMEM lane quadrant
    const int r = quad * 32 + lane;
    const int row = q0 + t * BM + r;
    const bool valid_row = row < p.N;
    const int sst = valid_row ? p.seq_start[row] : 0x7fffffff;
    const int kend = p.causal ? row + 1 : (valid_row ? p.seq_end[row] : 0);  // keys [sst, kend)
    const uint32_t lane_off = uint32_t(quad * 32) << 16;
    uint8_t* myP = sP(t);
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      ptx::mbar_wait(&s_full[t], j & 1);
      ptx::tc_fence_after();
      float s[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t v[32];
        ptx::tmem_ld32(TS(t) + lane_off + c * 32, v);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) s[c * 32 + i] = __uint_as_float(v[i]);
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&s_empty[t]);
      const int kbase = kv0 + j * BN;
      const bool full_vis = kbase >= sst && kbase + BN <= kend;
      // row max of the raw scores (scale > 0), 3-input max
      float mr = -INFINITY;
      if (!full_vis) {
#pragma unroll
        for (int i = 0; i < 128; ++i) {
          const int key = kbase + i;
          s[i] = (key >= sst && key < kend) ? s[i] : -INFINITY;
        }
      }
#pragma unroll
      for (int i = 0; i < 128; i += 2) mr = fmax3(mr, s[i], s[i + 1]);
      const float mx = mr * p.scale_log2;
      const bool need = mx > m_used + RESCALE_THRESH || (m_used == -INFINITY && mx > -INFINITY);
      const float m_new = need ? mx : m_used;
      const float alpha = (need && m_used != -INFINITY) ? exp2f(m_used - m_new) : 1.f;
      const float base = m_new == -INFINITY ? 0.f : m_new;
      // exponentials before waiting for the previous PV (overlap with the MMA);
      // x = s*scale - base and the row sum as packed fp32x2 ops.  Packed bf16 P
      // is written in place over s[0..63] (slot i/2 <= i)
      const uint64_t sc2 = f2pack(p.scale_log2, p.scale_log2), nb2 = f2pack(-base, -base);
      uint64_t sum2 = f2pack(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < 128; i += 2) {
        float x0, x1;
        f2unpack(ffma2(f2pack(s[i], s[i + 1]), sc2, nb2), x0, x1);
        const float a0 = (POLY_SHARE == 2 || (POLY_SHARE == 4 && (i & 7) == 6)) ? exp2_fma(x0) : ex2(x0);
        const float a1 = ex2(x1);
        sum2 = fadd2(sum2, f2pack(a0, a1));
        s[i / 2] = __uint_as_float(ptx::pack_bf16(a0, a1));
      }
      float sum_lo, sum_hi;
      f2unpack(sum2, sum_lo, sum_hi);
      const float sum = sum_lo + sum_hi;
      if (j > 0) ptx::mbar_wait(&o_done[t], (j - 1) & 1);  // PV(j-1) done: O stable, P free
      ptx::tc_fence_after();
      if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t v[32];
          ptx::tmem_ld32(TO(t) + lane_off + c * 32, v);
          ptx::tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = __float_as_uint(__uint_as_float(v[i]) * alpha);
          uint32_t lo[16], hi[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            lo[i] = v[i];
            hi[i] = v[16 + i];
          }
          ptx::tmem_st16(TO(t) + lane_off + c * 32, lo);
          ptx::tmem_st16(TO(t) + lane_off + c * 32 + 16, hi);
        }
        ptx::tmem_wait_st();
      }
      l = l * alpha + sum;
      m_used = m_new;
#pragma unroll
      for (int c = 0; c < 16; ++c)
        *reinterpret_cast<uint4*>(myP + sw_off(r, c)) =
            make_uint4(__float_as_uint(s[c * 4]), __float_as_uint(s[c * 4 + 1]),
                       __float_as_uint(s[c * 4 + 2]), __float_as_uint(s[c * 4 + 3]));
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      ptx::mbar_arrive(&p_full[t]);
    }
    ptx::mbar_wait(&o_done[t], (nkv - 1) & 1);
    ptx::tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    bf16* orow = p.o + int64_t(valid_row ? row : 0) * p.ldo + int64_t(h) * D;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t v[32];
      ptx::tmem_ld32(TO(t) + lane_off + c * 32, v);
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
  p.seq_end = a.seq_end;
  p.causal = a.causal;
  if (!a.causal && !a.seq_end) return cudaErrorInvalidValue;
  p.N = a.N;
  p.hq = a.hq;
  p.hk = a.hk;
  p.npairs = (a.N + 2 * BM - 1) / (2 * BM);
  p.scale_log2 = a.scale * LOG2E;
  p.band = cta_band("OPX_ATTN_FWD_BAND", 0, a.hq / a.hk, a.hq);
  dim3 grid(p.npairs, a.hq);
  ++g_kernel_launches;
  attn_fwd_tc_kernel<<<grid, FWD_THREADS, FWD_SMEM, s>>>(mq, mk, mv, p);
  return cudaGetLastError();
}

}  // namespace opx
