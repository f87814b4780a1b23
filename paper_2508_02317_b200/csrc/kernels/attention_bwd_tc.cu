// Causal packed-varlen GQA flash attention BACKWARD on tcgen05 (sm_100a).
//
// One CTA per (128-key tile, kv head, head split).  K and V stay in smem; the
// CTA walks its share of the q heads of the GQA group (all of them when
// kv_splits == 1) and the 64-query tiles that can see its keys
// (q in [k0, seq_end(last key))), with Q/dO in a 3-stage TMA ring.
// kv_splits > 1 shortens the CTAs (better tail balance when there are few key
// tiles, e.g. one kv head per rank under Ulysses); the per-split dK/dV
// partials are then summed by TMA bulk reduce-add into fp32 accumulators.
//
//   TMEM: S^T [0,64) | dP^T [64,128) | dQ^T [128,192) | P^T, dS^T as bf16 pairs
//         [192,224), [224,256) | dV [256,384) | dK [384,512)
//   per q tile i (MMA warp, one elected lane):
//     S^T  = K  Q_i^T    (M=128 keys, N=64 q, K=128 d)            -> s_full
//     dP^T = V  dO_i^T
//     -- softmax warps: P^T = exp2(S^T c - lse), dS^T = P^T (dP^T - delta),
//        bf16 -> TMEM (P^T, dS^T: one key row per thread) and dS -> SW128
//        smem [keys][q] -> p_ready
//     dV  += P^T  dO_i   (M=128 keys, N=128 d, K=64 q; A from TMEM)
//     dK  += dS^T Q_i    (A from TMEM)
//     dQ^T = K^T  dS^T   (M=128 d, N=64 q, K=128 keys)            -> dq_full
//     -- dQ warps (4, one per TMEM lane quadrant): dQ^T rows (one d per
//        thread, 64 q) -> fp32 smem [q][d] -> one TMA bulk reduce-add into the
//        fp32 dQ accumulator, off the softmax warps' path
// The S^T/dP^T MMAs of tile i+1 are issued as soon as the softmax warps have
// pulled S^T/dP^T(i) into registers (s_free), so they overlap the softmax of
// tile i.  dS is double-buffered in smem, so the softmax publishes tile i's
// P/dS once dV/dK(i-1) are done (kv_done) without waiting for dQ^T(i-1).
//
// What bounds it (phase stamps, tools/prof_attn_phases.py, C1 SP4 shape):
// ~3100 cycles per 64-query step; the dQ warps idle ~78 % of it and the
// softmax warps wait ~1100 cycles for S, while the MMA warp's issues block
// for ~2100 cycles (the tensor pipe queue is full): 32 MMAs of K=16 take
// ~95 cycles each instead of 48-64.  Per step the MMAs read 176 KB of smem
// (S/dP/dQ^T with N=64 read 6 KB per instruction), TMA writes 32 KB of Q/dO,
// the softmax 16 KB of dS, the dQ stage 32 KB + its bulk read 32 KB: ~290 KB
// against 128 B/clk -> a ~2270-cycle shared-memory floor.  dQ by
// red.global.add.f32 from registers (no staging) measured 1.6x slower
// (533 vs 821 TF/s); K^T / K / V as TMEM A operands would cut the MMA reads
// but the 512 TMEM columns are all in use (S^T, dP^T, dQ^T, P^T|dS^T, dV, dK).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "../runtime/gemm_api.h"
#include "../runtime/kernels_api.h"
#include "attn_common.cuh"
#include "ptx.cuh"

namespace opx {
namespace {

using bf16 = __nv_bfloat16;
using namespace attn;
constexpr int BQ = 64, BK = 128, D = 128;
// TMA, MMA, 8 softmax warps (2 per TMEM lane quadrant), 4 dQ warps (1 per quadrant)
constexpr int THREADS = 448;
constexpr int NSM = 256;       // softmax threads
constexpr int NDQ = 128;       // dQ drain threads (warps 10..13)
constexpr int DQ_T0 = 320;     // first dQ drain thread
constexpr float LOG2E = 1.4426950408889634f;
// smem map (bytes, 1024-aligned base)
// Q/dO: 3-stage ring (a stage is released only when the gradient MMAs of its
// tile complete, and the TMA refill takes ~1-2 us, so two stages starved the
// S/dP MMAs of the next tile)
constexpr int QSTAGES = 3;
constexpr int OFF_K = 0, OFF_V = 32768, OFF_Q = 65536 /*[3] x 16K*/, OFF_O = 114688 /*[3] x 16K*/,
              /* dS (bf16 [keys][q], SW128), double-buffered: tile it uses buffer it & 1 */
              OFF_S2 = 163840, OFF_S = 180224, OFF_STAGE = 196608 /*32K fp32*/, OFF_MISC = 229376;
constexpr int SMEM = 1024 + OFF_MISC + 3 * 2 * BQ * 4 + 256;
static_assert(3 * 2 * BQ * 4 + 13 * 8 + 8 <= 3 * 2 * BQ * 4 + 256, "misc region");

struct Params {
  const float* lse;
  const float* delta;
  bf16* dk;
  bf16* dv;
  int64_t lddk, lddv;
  const int* seq_start;
  const int* seq_end;
  int N, hq, hk;
  float scale, scale_log2;
  int skip_dq;  // debug: 1 = measure without the dQ reduction, 2 = without its staging too
  long long* prof;  // debug (OPX_ATTN_PROF=<cta>): clock64 stamps [64 iters][16] of one CTA
  int prof_cta;
  int band;     // CTA order (attn::cta_order)
  int splits;   // q-head splits per kv head
  int f32kv;    // dK/dV go to fp32 [N, hk, 128] through tdk/tdv (reduce-add if splits > 1)
};

__device__ __forceinline__ uint64_t kd(uint32_t base, int k, int blk) {
  return ptx::umma_desc_sw128(base + (k >> 2) * blk + (k & 3) * 32, 16, 1024);
}
__device__ __forceinline__ uint64_t md(uint32_t base, int k, int lbo) {
  return ptx::umma_desc_sw128(base + k * 2048, lbo, 1024);
}
// Phase stamps for tools/prof_attn_phases.py: build with -DOPX_ATTN_PROF_BUILD=1
// and run with OPX_ATTN_PROF=<cta>; compiled out otherwise.
#ifndef OPX_ATTN_PROF_BUILD
#define OPX_ATTN_PROF_BUILD 0
#endif
#if OPX_ATTN_PROF_BUILD
#define PROF(it, k)                                                                        \
  do {                                                                                     \
    if (p.prof && int(blockIdx.x + gridDim.x * blockIdx.y) == p.prof_cta && (it) < 64)     \
      p.prof[(it) * 16 + (k)] = clock64();                                                 \
  } while (0)
#else
#define PROF(it, k) \
  do {              \
  } while (0)
#endif
// 1/POLY_SHARE of the P exponentials on the FMA-pipe polynomial (8, 4 or 0 = none)
#ifndef OPX_BWD_POLY_SHARE
#define OPX_BWD_POLY_SHARE 0
#endif
constexpr int POLY_SHARE = OPX_BWD_POLY_SHARE;
__device__ __forceinline__ void bar_sync_softmax() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void bar_sync_dq() { asm volatile("bar.sync 2, 128;" ::: "memory"); }

__global__ void __launch_bounds__(THREADS, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tdo,
                       const __grid_constant__ CUtensorMap tdq, const __grid_constant__ CUtensorMap tdk,
                       const __grid_constant__ CUtensorMap tdv, const Params p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-B alignment by pointer arithmetic on the __shared__ array keeps the
  // shared address space (no generic LD/ST on the hot path).
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  float* s_lse = reinterpret_cast<float*>(smem + OFF_MISC);  // [2][64]
  float* s_dlt = s_lse + 2 * BQ;
  int* s_sst = reinterpret_cast<int*>(s_dlt + 2 * BQ);
  uint64_t* bars = reinterpret_cast<uint64_t*>(s_sst + 2 * BQ);
  uint64_t* kv_full = bars + 0;
  uint64_t* qdo_full = bars + 1;   // [3]
  uint64_t* qdo_empty = bars + 4;  // [3]
  uint64_t* s_full = bars + 7;
  uint64_t* p_ready = bars + 8;
  uint64_t* dq_full = bars + 9;    // [2] dQ^T(it) complete -> [it & 1] (every MMA of tile it done)
  uint64_t* dqt_free = bars + 11;  // dQ^T(it) read out of TMEM
  uint64_t* kv_done = bars + 12;   // dV/dK(it) complete: P^T/dS^T (TMEM) of tile it read
  uint64_t* s_free = bars + 13;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 14);
  float* stage = reinterpret_cast<float*>(smem + OFF_STAGE);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int bx, by;
  cta_order(p.band, bx, by);
  const int k0 = bx * BK;
  const int kh = by / p.splits, sidx = by % p.splits;
  const int G = p.hq / p.hk;
  const int hbase = kh * G + (sidx * G) / p.splits;
  const int nh = ((sidx + 1) * G) / p.splits - (sidx * G) / p.splits;
  const int klast = min(k0 + BK, p.N) - 1;
  const int qend = p.seq_end[klast];
  const int nq = (qend - k0 + BQ - 1) / BQ;
  const int niter = nh * nq;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tq);
    ptx::tma_prefetch(&tk);
    ptx::tma_prefetch(&tv);
    ptx::tma_prefetch(&tdo);
    ptx::tma_prefetch(&tdq);
    ptx::mbar_init(kv_full, 1);
    for (int i = 0; i < QSTAGES; ++i) {
      ptx::mbar_init(&qdo_full[i], 1);
      ptx::mbar_init(&qdo_empty[i], 1);
    }
    ptx::mbar_init(s_full, 1);
    ptx::mbar_init(p_ready, NSM);
    ptx::mbar_init(&dq_full[0], 1);
    ptx::mbar_init(&dq_full[1], 1);
    ptx::mbar_init(dqt_free, NDQ);
    ptx::mbar_init(kv_done, 1);
    ptx::mbar_init(s_free, NSM);
    ptx::fence_mbar_init();
  }
  if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: S^T | dP^T | dQ^T | P^T, dS^T (bf16 pairs: the A operand of the dV / dK
  // MMAs, so they read only dO / Q from smem) | dV | dK
  const uint32_t TPT = tmem + 192, TDST = tmem + 224;
  const uint32_t TST = tmem, TDP = tmem + 64, TDQ = tmem + 128,
                 TDV = tmem + 256, TDK = tmem + 384;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      ptx::mbar_expect_tx(kv_full, 4 * 16384);
      ptx::tma_load_3d(&tk, kv_full, smem + OFF_K, 0, kh, k0);
      ptx::tma_load_3d(&tk, kv_full, smem + OFF_K + 16384, 64, kh, k0);
      ptx::tma_load_3d(&tv, kv_full, smem + OFF_V, 0, kh, k0);
      ptx::tma_load_3d(&tv, kv_full, smem + OFF_V + 16384, 64, kh, k0);
      for (int it = 0; it < niter; ++it) {
        const int st = it % QSTAGES;
        const int h = hbase + it / nq;
        const int q0 = k0 + (it % nq) * BQ;
        if (it >= QSTAGES) ptx::mbar_wait(&qdo_empty[st], ((it / QSTAGES) - 1) & 1);
        ptx::mbar_expect_tx(&qdo_full[st], 4 * 8192);
        uint8_t* q = smem + OFF_Q + st * 16384;
        uint8_t* o = smem + OFF_O + st * 16384;
        ptx::tma_load_3d(&tq, &qdo_full[st], q, 0, h, q0);
        ptx::tma_load_3d(&tq, &qdo_full[st], q + 8192, 64, h, q0);
        ptx::tma_load_3d(&tdo, &qdo_full[st], o, 0, h, q0);
        ptx::tma_load_3d(&tdo, &qdo_full[st], o + 8192, 64, h, q0);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t id_s = ptx::idesc_bf16_f32(128, BQ, false, false);   // S^T, dP^T
    constexpr uint32_t id_kv = ptx::idesc_bf16_f32(128, D, false, true);    // dV, dK
    constexpr uint32_t id_q = ptx::idesc_bf16_f32(128, BQ, true, true);     // dQ^T
    const uint32_t ak = ptx::smem_u32(smem + OFF_K), av = ptx::smem_u32(smem + OFF_V);
    ptx::mbar_wait(kv_full, 0);
    // issue order: S/dP(i+1) right after P(i) is ready, then dV/dK/dQ(i), so
    // the softmax of tile i+1 overlaps the gradient MMAs of tile i.
    auto issue_sdp = [&](int it) {
      const int st = it % QSTAGES;
      const uint32_t aq = ptx::smem_u32(smem + OFF_Q + st * 16384);
      const uint32_t ao = ptx::smem_u32(smem + OFF_O + st * 16384);
      ptx::mbar_wait(&qdo_full[st], (it / QSTAGES) & 1);
      ptx::tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < D / 16; ++k)
          ptx::mma_bf16_ss(TST, kd(ak, k, 16384), kd(aq, k, 8192), id_s, k != 0);
#pragma unroll
        for (int k = 0; k < D / 16; ++k)
          ptx::mma_bf16_ss(TDP, kd(av, k, 16384), kd(ao, k, 8192), id_s, k != 0);
        ptx::mma_commit(s_full);
      }
      __syncwarp();
    };
    if (niter > 0) issue_sdp(0);
    for (int it = 0; it < niter; ++it) {
      const int qs = it % QSTAGES;          // Q/dO stage
      const uint32_t aq = ptx::smem_u32(smem + OFF_Q + qs * 16384);
      const uint32_t ao = ptx::smem_u32(smem + OFF_O + qs * 16384);
      if (it + 1 < niter) {
        ptx::mbar_wait(s_free, it & 1);  // S^T/dP^T(it) are in the softmax registers
        if (lane == 0) PROF(it, 0);
        issue_sdp(it + 1);
        if (lane == 0) PROF(it, 3);
      }
      ptx::mbar_wait(p_ready, it & 1);   // P^T/dS^T(it) in TMEM, dS(it) in smem
      if (lane == 0) PROF(it, 1);
      ptx::tc_fence_after();
      if (lane == 0) {
#pragma unroll
        for (int k = 0; k < BQ / 16; ++k)
          ptx::mma_bf16_ts(TDV, TPT + uint32_t(k) * 8, md(ao, k, 8192), id_kv, (it | k) != 0);
#pragma unroll
        for (int k = 0; k < BQ / 16; ++k)
          ptx::mma_bf16_ts(TDK, TDST + uint32_t(k) * 8, md(aq, k, 8192), id_kv, (it | k) != 0);
        ptx::mma_commit(&qdo_empty[qs]);  // release the Q/dO stage early: dQ^T does not read it
        ptx::mma_commit(kv_done);         // P^T/dS^T(it) in TMEM may be overwritten
      }
      __syncwarp();
      if (it >= 1) ptx::mbar_wait(dqt_free, (it - 1) & 1);  // dQ^T(it-1) read out of TMEM
      if (lane == 0) PROF(it, 2);
      ptx::tc_fence_after();
      if (lane == 0) {
        const uint32_t as = ptx::smem_u32(smem + ((it & 1) ? OFF_S2 : OFF_S));
#pragma unroll
        for (int k = 0; k < BK / 16; ++k)
          ptx::mma_bf16_ss(TDQ, md(ak, k, 16384), md(as, k, 8192), id_q, k != 0);
        ptx::mma_commit(&dq_full[it & 1]);
      }
      __syncwarp();
    }
  } else if (warp >= 10) {
    // ---------------- dQ drain warps ----------------
    // dQ^T(j) (thread: d row r = quad*32 + lane, all 64 q columns) -> fp32
    // staging [q][d] -> one TMA bulk reduce-add into the fp32 dQ accumulator.
    // Off the softmax warps' critical path: they only publish P/dS.
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = uint32_t(quad * 32) << 16;
    const bool dq_issuer = threadIdx.x == DQ_T0;
    for (int j = 0; j < niter; ++j) {
      const int h = hbase + j / nq;
      const int q0 = k0 + (j % nq) * BQ;
      ptx::mbar_wait(&dq_full[j & 1], (j >> 1) & 1);
      if (dq_issuer) PROF(j + 1, 8);
      ptx::tc_fence_after();
      uint32_t qa[32], qb[32];
      ptx::tmem_ld32(TDQ + lane_off, qa);
      ptx::tmem_ld32(TDQ + lane_off + 32, qb);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      ptx::mbar_arrive(dqt_free);  // the MMA warp may issue dQ^T(j+1)
      if (dq_issuer) PROF(j + 1, 11);
      if (dq_issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      bar_sync_dq();  // staging buffer free
      if (dq_issuer) PROF(j + 1, 12);
      if (p.skip_dq < 2) {
#pragma unroll
        for (int q = 0; q < 32; ++q) stage[q * D + r] = __uint_as_float(qa[q]) * p.scale;
#pragma unroll
        for (int q = 0; q < 32; ++q) stage[(32 + q) * D + r] = __uint_as_float(qb[q]) * p.scale;
      }
      ptx::fence_proxy_async();
      bar_sync_dq();
      if (dq_issuer) PROF(j + 1, 13);
      if (dq_issuer && !p.skip_dq) {
        asm volatile(
            "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                reinterpret_cast<uint64_t>(&tdq)),
            "r"(ptx::smem_u32(stage)), "r"(0), "r"(h), "r"(q0)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    }
    if (dq_issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else {
    // ---------------- softmax warps ----------------
    // warps 2..9: lane quadrant = warp & 3 (TMEM access rule), column half =
    // (warp - 2) / 4, so every quadrant is served by two warps.
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;  // key row for S^T/dP^T, d row for dQ^T
    const int c0 = half * 32;        // first of this thread's 32 q columns
    const int key = k0 + r;
    const uint32_t lane_off = uint32_t(quad * 32) << 16;
    const bool issuer = threadIdx.x == 64;
    const bool pt = issuer;  // debug stamps
    auto load_cols = [&](int it) {  // lse/delta/seq_start of tile it -> smem buffer it&1
      if (half == 0 && r < BQ) {
        const int h = hbase + it / nq;
        const int q = k0 + (it % nq) * BQ + r;
        const bool ok = q < p.N;
        const int buf = it & 1;
        s_lse[buf * BQ + r] = ok ? p.lse[int64_t(h) * p.N + q] * LOG2E : INFINITY;
        s_dlt[buf * BQ + r] = ok ? p.delta[int64_t(h) * p.N + q] : 0.f;
        s_sst[buf * BQ + r] = ok ? p.seq_start[q] : 0x7fffffff;
      }
    };
    if (niter > 0) load_cols(0);
    bar_sync_softmax();
    for (int it = 0; it < niter; ++it) {
      if (pt) PROF(it, 4);
      const int q0 = k0 + (it % nq) * BQ;
      const int buf = it & 1;
      // this thread's 32 columns of lse / delta: broadcast smem loads inside
      // the math loops (not held in registers: the kernel runs at 128 regs)
      const float* lvp = s_lse + buf * BQ + c0;
      const float* dlp = s_dlt + buf * BQ + c0;
      const int* sst = s_sst + buf * BQ;
      const bool full_vis = key <= q0 + c0 && q0 + c0 + 31 < p.N && sst[c0 + 31] <= key;
      ptx::mbar_wait(s_full, it & 1);
      if (pt) PROF(it, 5);
      ptx::tc_fence_after();
      uint32_t sv[32], dv[32];
      ptx::tmem_ld32(TST + lane_off + c0, sv);
      ptx::tmem_ld32(TDP + lane_off + c0, dv);
      ptx::tmem_wait_ld();
      ptx::tc_fence_before();
      ptx::mbar_arrive(s_free);  // the MMA warp may overwrite S^T/dP^T now
      uint32_t pw[16], dw[16];
      if (full_vis) {
        // packed fp32x2: x = s*scale - lse, dS = P (dP - delta); 1 in 4
        // exponentials on the FMA pipe
        const uint64_t sc2 = f2pack(p.scale_log2, p.scale_log2);
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          const float2 lv = *reinterpret_cast<const float2*>(lvp + i);
          const float2 dl = *reinterpret_cast<const float2*>(dlp + i);
          float x0, x1;
          f2unpack(ffma2(f2pack(__uint_as_float(sv[i]), __uint_as_float(sv[i + 1])), sc2,
                         f2pack(-lv.x, -lv.y)),
                   x0, x1);
          const bool poly = POLY_SHARE == 8 ? (i & 7) == 6 : POLY_SHARE == 4 ? (i & 3) == 2 : false;
          const float p0 = poly ? exp2_fma(x0) : ex2(x0);
          const float p1 = ex2(x1);
          const uint64_t pp = f2pack(p0, p1);
          const uint64_t dd = fadd2(f2pack(__uint_as_float(dv[i]), __uint_as_float(dv[i + 1])),
                                    f2pack(-dl.x, -dl.y));
          float d0, d1;
          f2unpack(fmul2(pp, dd), d0, d1);
          pw[i / 2] = ptx::pack_bf16(p0, p1);
          dw[i / 2] = ptx::pack_bf16(d0, d1);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 32; i += 2) {
          float pp[2];
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int q = q0 + c0 + i + e;
            const bool ok = (key <= q) & (key >= sst[c0 + i + e]) & (key < p.N);
            const float x = ex2(fmaf(__uint_as_float(sv[i + e]), p.scale_log2, -lvp[i + e]));
            pp[e] = ok ? x : 0.f;
          }
          pw[i / 2] = ptx::pack_bf16(pp[0], pp[1]);
          dw[i / 2] = ptx::pack_bf16(pp[0] * (__uint_as_float(dv[i]) - dlp[i]),
                                     pp[1] * (__uint_as_float(dv[i + 1]) - dlp[i + 1]));
        }
      }
      // the gradient MMAs of tile it-1 read P^T/dS^T (TMEM) and dS (smem):
      // wait for them, publish tile it's (P^T, dS^T: this thread's key row, its
      // 32 q columns as 16 bf16 pairs; dS also to smem for the dQ^T MMA) so the
      // MMA warp can issue its gradients at once, then drain dQ^T(it-1) while
      // dV/dK run
      if (pt) PROF(it, 6);
      // P^T/dS^T (TMEM) are free once dV/dK(it-1) are done; the dS smem
      // buffer it & 1 once dQ^T(it-2) is (the other buffer feeds dQ^T(it-1))
      if (it > 0) ptx::mbar_wait(kv_done, (it - 1) & 1);
      if (it > 1) ptx::mbar_wait(&dq_full[it & 1], ((it - 2) >> 1) & 1);
      if (pt) PROF(it, 9);
      ptx::tc_fence_after();
      ptx::tmem_st16(TPT + lane_off + uint32_t(half) * 16, pw);
      ptx::tmem_st16(TDST + lane_off + uint32_t(half) * 16, dw);
      uint8_t* sS = smem + ((it & 1) ? OFF_S2 : OFF_S);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        const int chunk = half * 4 + cc;
        *reinterpret_cast<uint4*>(sS + sw_off64(r, chunk)) =
            make_uint4(dw[cc * 4], dw[cc * 4 + 1], dw[cc * 4 + 2], dw[cc * 4 + 3]);
      }
      ptx::tmem_wait_st();
      ptx::fence_proxy_async();
      ptx::tc_fence_before();
      ptx::mbar_arrive(p_ready);
      if (pt) PROF(it, 7);
      if (it + 1 < niter) load_cols(it + 1);
      bar_sync_softmax();  // next tile's column data visible
      if (pt) PROF(it, 10);
    }
    // every MMA of the CTA is complete (dK/dV final in TMEM)
    if (niter > 0) ptx::mbar_wait(&dq_full[(niter - 1) & 1], ((niter - 1) >> 1) & 1);
    ptx::tc_fence_after();
    if (p.f32kv) {
      // ---- dK (scaled), dV -> fp32 SW128 staging [4 col chunks][128 rows][32]
      // over the free Q/dO/P/S/stage buffers, then TMA store / reduce-add.
      uint8_t* stk = smem + OFF_Q;  // [OFF_Q, OFF_STAGE): Q/dO ring + dS (the dQ warps own OFF_STAGE)
      uint8_t* stv = smem + OFF_Q + 65536;
#pragma unroll 1
      for (int c = half * 2; c < half * 2 + 2; ++c) {
        uint32_t a[32], b[32];
        ptx::tmem_ld32(TDK + lane_off + c * 32, a);
        ptx::tmem_ld32(TDV + lane_off + c * 32, b);
        ptx::tmem_wait_ld();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const uint32_t off = c * 16384 + r * 128 + (((q ^ (r & 7))) << 4);
          *reinterpret_cast<float4*>(stk + off) =
              make_float4(__uint_as_float(a[4 * q]) * p.scale, __uint_as_float(a[4 * q + 1]) * p.scale,
                          __uint_as_float(a[4 * q + 2]) * p.scale, __uint_as_float(a[4 * q + 3]) * p.scale);
          *reinterpret_cast<float4*>(stv + off) =
              make_float4(__uint_as_float(b[4 * q]), __uint_as_float(b[4 * q + 1]),
                          __uint_as_float(b[4 * q + 2]), __uint_as_float(b[4 * q + 3]));
        }
      }
      ptx::fence_proxy_async();
      bar_sync_softmax();
      if (issuer) {
        for (int c = 0; c < 4; ++c) {
          if (p.splits > 1) {
            asm volatile(
                "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(&tdk)),
                "r"(ptx::smem_u32(stk + c * 16384)), "r"(c * 32), "r"(kh), "r"(k0)
                : "memory");
            asm volatile(
                "cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(&tdv)),
                "r"(ptx::smem_u32(stv + c * 16384)), "r"(c * 32), "r"(kh), "r"(k0)
                : "memory");
          } else {
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(&tdk)),
                "r"(ptx::smem_u32(stk + c * 16384)), "r"(c * 32), "r"(kh), "r"(k0)
                : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                    reinterpret_cast<uint64_t>(&tdv)),
                "r"(ptx::smem_u32(stv + c * 16384)), "r"(c * 32), "r"(kh), "r"(k0)
                : "memory");
          }
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      }
    } else {
    // ---- dK (scaled), dV rows -> bf16 (each thread: 64 of the 128 d columns)
    const bool ok = key < p.N;
    bf16* dkr = p.dk + int64_t(ok ? key : 0) * p.lddk + int64_t(kh) * D;
    bf16* dvr = p.dv + int64_t(ok ? key : 0) * p.lddv + int64_t(kh) * D;
#pragma unroll 1
    for (int c = half * 2; c < half * 2 + 2; ++c) {
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
            const float k0f = niter ? __uint_as_float(a[q * 8 + 2 * e]) * p.scale : 0.f;
            const float k1f = niter ? __uint_as_float(a[q * 8 + 2 * e + 1]) * p.scale : 0.f;
            const float v0f = niter ? __uint_as_float(b[q * 8 + 2 * e]) : 0.f;
            const float v1f = niter ? __uint_as_float(b[q * 8 + 2 * e + 1]) : 0.f;
            kp[e] = ptx::pack_bf16(k0f, k1f);
            vp[e] = ptx::pack_bf16(v0f, v1f);
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

// dq_acc must be a dense [N, hq, 128] fp32 buffer (it is zeroed here).  With
// dk_acc/dv_acc set, dK/dV are written as dense fp32 [N, hk, 128] (and dk/dv
// are unused); kv_splits (0 = auto) then splits each GQA group across CTAs.
int attn_bwd_kv_splits(int N, int hq, int hk) {
  const int G = hq / hk;
  if (const char* e = getenv("OPX_ATTN_KV_SPLITS")) return std::max(1, std::min(G, atoi(e)));
  (void)N;
  // One q head per CTA measured best on B200 for both C1 layouts (32K tokens,
  // 7q/1kv: 437 -> 631 TFLOP/s; 28q/4kv: 600 -> 678): the causal tail of long
  // early-key tiles dominates, and the extra fp32 reduce traffic stays in L2.
  return G;
}

cudaError_t k_attn_bwd_tc(const AttnArgs& a, cudaStream_t s) {
  if (a.N <= 0) return cudaSuccess;
  if (a.hq % a.hk) return cudaErrorInvalidValue;
  const bool f32kv = a.dk_acc && a.dv_acc;
  const int splits = f32kv ? (a.kv_splits > 0 ? std::min(a.kv_splits, a.hq / a.hk)
                                              : attn_bwd_kv_splits(a.N, a.hq, a.hk))
                           : 1;
  CUtensorMap mq, mk, mv, mdo, mdq, mdk, mdv;
  if (f32kv) {
    if (!head_map_f32_sw(&mdk, a.dk_acc, a.N, a.hk, BK) || !head_map_f32_sw(&mdv, a.dv_acc, a.N, a.hk, BK))
      return cudaErrorInvalidValue;
  }
  if (!head_map(&mq, a.q, a.N, a.hq, a.ldq, BQ) || !head_map(&mk, a.k, a.N, a.hk, a.ldk, BK) ||
      !head_map(&mv, a.v, a.N, a.hk, a.ldv, BK) || !head_map(&mdo, a.dout, a.N, a.hq, a.lddo, BQ) ||
      !head_map_f32(&mdq, a.dq_acc, a.N, a.hq, BQ))
    return cudaErrorInvalidValue;
  if (!f32kv) mdk = mdv = mdq;  // unused
  static bool cfg = false;
  if (!cfg) {
    cudaError_t e = cudaFuncSetAttribute(attn_bwd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    cfg = true;
  }
  const int64_t warps = int64_t(a.N) * a.hq;
  ++g_kernel_launches;
  delta_kernel<<<int((warps * 32 + 255) / 256), 256, 0, s>>>(a.dout, a.lddo, a.o, a.ldo, a.delta, a.N, a.hq);
  cudaError_t e = cudaMemsetAsync(a.dq_acc, 0, size_t(a.N) * a.hq * D * sizeof(float), s);
  if (e != cudaSuccess) return e;
  if (f32kv && splits > 1) {
    if ((e = cudaMemsetAsync(a.dk_acc, 0, size_t(a.N) * a.hk * D * sizeof(float), s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(a.dv_acc, 0, size_t(a.N) * a.hk * D * sizeof(float), s)) != cudaSuccess) return e;
  }
  Params p;
  p.lse = a.lse;
  p.delta = a.delta;
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
  p.skip_dq = getenv("OPX_DEBUG_SKIP_DQ") ? atoi(getenv("OPX_DEBUG_SKIP_DQ")) : 0;  // 1: no reduce, 2: no stage either
  static long long* prof = nullptr;
  p.prof = nullptr;
  p.prof_cta = getenv("OPX_ATTN_PROF") ? atoi(getenv("OPX_ATTN_PROF")) : -1;
  if (p.prof_cta >= 0) {
    if (!prof) cudaMalloc(&prof, 64 * 16 * sizeof(long long));
    cudaMemsetAsync(prof, 0, 64 * 16 * sizeof(long long), s);
    p.prof = prof;
  }
  p.splits = splits;
  p.f32kv = f32kv;
  p.band = cta_band("OPX_ATTN_BAND", 0, splits, a.hk * splits);
  dim3 grid((a.N + BK - 1) / BK, a.hk * splits);
  ++g_kernel_launches;
  attn_bwd_tc_kernel<<<grid, THREADS, SMEM, s>>>(mq, mk, mv, mdo, mdq, mdk, mdv, p);
  if (p.prof) {  // debug: per-iteration phase durations (cycles) of one CTA
    long long h[64 * 16];
    cudaStreamSynchronize(s);
    cudaMemcpy(h, p.prof, sizeof h, cudaMemcpyDeviceToHost);
    double acc[16] = {};
    int n = 0;
    for (int it = 4; it < 60 && h[(it + 1) * 16 + 4]; ++it, ++n) {
      const long long* a = h + it * 16;
      const long long* b = h + (it + 1) * 16;
      acc[0] += double(b[4] - a[4]);   // iteration
      acc[1] += double(a[5] - a[4]);   // wait S
      acc[2] += double(a[6] - a[5]);   // ld + compute
      acc[3] += double(a[7] - a[6]);   // STS P/dS + arrive
      acc[4] += double(b[8] - a[7]);   // wait dQ(it)... (stamp 8 of it+1 = wait dq(it) done)
      acc[5] += double(a[9] - b[8] > 0 ? a[9] - a[7] : 0);
      acc[6] += double(a[10] - a[9]);  // load_cols + bar
      acc[7] += double(a[1] - a[0]);   // MMA: s_free -> p_ready
      acc[8] += double(a[2] - a[1]);   // MMA: wait dqt_free
      acc[9] += double(a[3] - a[0]);   // MMA: S/dP issue incl. qdo_full wait
      acc[10] += double(a[0] - a[5]);  // s_free seen by MMA - s_full seen by softmax (same it)
      acc[11] += double(b[5] - a[3]);  // S(it+1) issued -> softmax sees s_full(it+1)
      // dQ drain warps (stamps of tile it at row it+1): dq_full seen -> ld+arrive ->
      // previous reduce read done + bar -> stage written + bar; next dq_full seen
      acc[12] += double(b[11] - b[8]);
      acc[13] += double(b[12] - b[11]);
      acc[14] += double(b[13] - b[12]);
      acc[15] += double(h[(it + 2) * 16 + 8] - b[13] > 0 ? h[(it + 2) * 16 + 8] - b[13] : 0);
    }
    if (n)
      fprintf(stderr,
              "[attn_bwd prof cta %d, %d iters] iter %.0f | wait_S %.0f ld+math %.0f publish %.0f "
              "drain(wait dq %.0f, total %.0f) cols+bar %.0f | mma: s_free->p_ready %.0f wait_dqt %.0f "
              "issue_S %.0f sfull->sfree %.0f S_issue->S_seen %.0f | dq warps: ld %.0f "
              "reduce_read+bar %.0f stage %.0f idle %.0f\n",
              p.prof_cta, n, acc[0] / n, acc[1] / n, acc[2] / n, acc[3] / n, acc[4] / n, acc[5] / n,
              acc[6] / n, acc[7] / n, acc[8] / n, acc[9] / n, acc[10] / n, acc[11] / n,
              acc[12] / n, acc[13] / n, acc[14] / n, acc[15] / n);
  }
  return cudaGetLastError();
}

}  // namespace opx
