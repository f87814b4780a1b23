// Persistent warp-specialised bf16 GEMM on tcgen05 (sm_100a).
//
//   D[M,N] (op)= A[M,K] . B[N,K]^T      (bf16 in, fp32 accumulate in TMEM)
//
// Operands may be K-major or MN-major (the dgrad / wgrad forms of a linear
// layer), selected by template flags; TMA loads 128B-swizzled tiles into a
// 4-stage smem ring, one elected thread issues tcgen05.mma, and four epilogue
// warps drain a double-buffered TMEM accumulator (2 x 256 columns) while the
// next tile's MMAs run.  Epilogues fuse what follows each GEMM in the step:
// bf16/fp32 stores, the residual add, fp32 accumulation (wgrad into a grad
// buffer), and the SwiGLU gate on 128-column interleaved gate/up weights.
//
// Grouped mode (MoE experts): per-group row segments (128-aligned) with a
// per-group weight slab; either M varies per group (fwd/dgrad) or K does (wgrad).
#include <cuda.h>

#include <map>
#include <string>
#include <vector>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "../runtime/gemm_api.h"
#include "../runtime/kernels_api.h"
#include "epilogue.cuh"
#include "ptx.cuh"

namespace opx {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_STAGE_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_STAGE_BYTES = BN * BK * 2;  // 32 KB
// bf16 epilogue staging: per epilogue warp [32 rows][40] bf16, so the output
// leaves as 8 rows x 64 contiguous bytes per warp instruction instead of one
// 16-B piece of 32 different rows
constexpr int EPI_LD = 40;
constexpr int EPI_OFF = STAGES * (A_STAGE_BYTES + B_STAGE_BYTES) + 512;
constexpr int SMEM_BYTES = EPI_OFF + 4 * 32 * EPI_LD * 2 + 1024;
constexpr int NUM_THREADS = 256;

struct KParams {
  int M, N, K;
  int epi;
  void* D;
  int64_t ldd;
  const float* R;
  int64_t ldr;
  __nv_bfloat16* D2;
  int64_t ldd2;
  const __nv_bfloat16* G2;  // GEMM_EPI_SWIGLU_BWD: forward gate|up
  int64_t ldg2;
  float scale;
  // grouped
  int groups;          // 0 = plain GEMM
  int grouped_k;       // 1: K varies per group (wgrad), 0: M varies (fwd/dgrad)
  const int* g_start;  // [groups] row offset of each segment (multiple of 128)
  const int* g_rows;   // [groups] rows in each segment (padded to a multiple of 128 for grouped_k)
  int64_t g_b_rows;    // rows of B per group slab (B row coordinate offset = g * g_b_rows)
  int64_t g_d_stride;  // element offset of D between groups (grouped_k only)
  int band;            // plain GEMMs: n-blocks per raster band (L2 reuse, chosen on host)
  // GEMM_EPI_ROWMAP (grouped-M): destination of row r of group g
  __nv_bfloat16* const* rm_dst;
  const int* rm_cnt;
  const int* rm_off;
  int rm_ep;
  const __nv_bfloat16* bias;  // optional column bias
  int staged;                 // bf16 epilogue through the per-warp smem stage
};

struct TileCoord {
  int g, mb, nb, m0, k_begin, nk;
  bool valid;
};

// Tile enumeration: plain -> m fastest within an n column; grouped -> walk
// groups in order (counts come from device memory, so every role recomputes
// them identically).
__device__ __forceinline__ TileCoord tile_of(const KParams& p, int t) {
  TileCoord c{};
  const int nblk = (p.N + BN - 1) / BN;
  if (p.groups == 0) {
    // raster: bands of `band` n-blocks; m-blocks walk inside a band, n fastest
    const int mblk = (p.M + BM - 1) / BM;
    c.valid = t < mblk * nblk;
    const int per_band = p.band * mblk;
    const int b = t / per_band, r = t % per_band;
    const int bw = min(p.band, nblk - b * p.band);
    c.g = 0;
    c.mb = r / bw;
    c.nb = b * p.band + r % bw;
    c.m0 = c.mb * BM;
    c.k_begin = 0;
    c.nk = (p.K + BK - 1) / BK;
    return c;
  }
  if (!p.grouped_k) {
    for (int g = 0; g < p.groups; ++g) {
      const int rows = p.g_rows[g];
      const int mblk = (rows + BM - 1) / BM;
      const int n = mblk * nblk;
      if (t < n) {
        c.valid = true;
        c.g = g;
        c.mb = t % mblk;
        c.nb = t / mblk;
        c.m0 = p.g_start[g] + c.mb * BM;
        c.k_begin = 0;
        c.nk = (p.K + BK - 1) / BK;
        return c;
      }
      t -= n;
    }
    c.valid = false;
    return c;
  }
  // grouped_k: every group has the same (M, N) output; K = segment rows.
  const int mblk = (p.M + BM - 1) / BM;
  const int per = mblk * nblk;
  c.g = t / per;
  c.valid = c.g < p.groups;
  if (!c.valid) return c;
  const int r = t % per;
  c.mb = r % mblk;
  c.nb = r / mblk;
  c.m0 = c.mb * BM;
  c.k_begin = p.g_start[c.g];
  c.nk = p.g_rows[c.g] / BK;
  return c;
}

__device__ __forceinline__ int total_tiles(const KParams& p) {
  const int nblk = (p.N + BN - 1) / BN;
  if (p.groups == 0) return ((p.M + BM - 1) / BM) * nblk;
  if (p.grouped_k) return p.groups * ((p.M + BM - 1) / BM) * nblk;
  int n = 0;
  for (int g = 0; g < p.groups; ++g) n += ((p.g_rows[g] + BM - 1) / BM) * nblk;
  return n;
}

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const KParams p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-B alignment by pointer arithmetic on the __shared__ array keeps the
  // shared address space (no generic LD/ST on the hot path).
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 128);
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc(tmem_slot, 512);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int ntiles = total_tiles(p);

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const TileCoord c = tile_of(p, t);
        const int n0 = c.nb * BN;
        const int brow = int(c.g * p.g_b_rows);
        for (int kb = 0; kb < c.nk; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          ptx::mbar_expect_tx(&full[stage], A_STAGE_BYTES + B_STAGE_BYTES);
          uint8_t* a = sA + stage * A_STAGE_BYTES;
          uint8_t* b = sB + stage * B_STAGE_BYTES;
          const int k0 = c.k_begin + kb * BK;
          if (!A_MN) {
            ptx::tma_load_2d(&tmA, &full[stage], a, k0, c.m0);
          } else {
            ptx::tma_load_2d(&tmA, &full[stage], a, c.m0, k0);
            ptx::tma_load_2d(&tmA, &full[stage], a + 8192, c.m0 + 64, k0);
          }
          if (!B_MN) {
            ptx::tma_load_2d(&tmB, &full[stage], b, k0, brow + n0);
          } else {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              ptx::tma_load_2d(&tmB, &full[stage], b + j * 8192, n0 + 64 * j, brow + k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = ptx::idesc_bf16_f32(BM, BN, A_MN, B_MN);
    int stage = 0;
    uint32_t phase = 0;
    int local = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
      const TileCoord c = tile_of(p, t);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
      ptx::tc_fence_after();
      const uint32_t d_tmem = tmem_base + acc * BN;
      for (int kb = 0; kb < c.nk; ++kb) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        if (lane == 0) {
          const uint32_t a_addr = ptx::smem_u32(sA + stage * A_STAGE_BYTES);
          const uint32_t b_addr = ptx::smem_u32(sB + stage * B_STAGE_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            const uint64_t ad = A_MN ? ptx::umma_desc_sw128(a_addr + k * 2048, 8192, 1024)
                                     : ptx::umma_desc_sw128(a_addr + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? ptx::umma_desc_sw128(b_addr + k * 2048, 8192, 1024)
                                     : ptx::umma_desc_sw128(b_addr + k * 32, 16, 1024);
            ptx::mma_bf16_ss(d_tmem, ad, bd, idesc, (kb | k) != 0);
          }
          ptx::mma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (lane == 0) {
        if (c.nk == 0) {
          // Nothing accumulated: still hand the (stale) buffer over; the
          // epilogue writes zeros for empty K in this case.
          ptx::mbar_arrive(&tfull[acc]);
        } else {
          ptx::mma_commit(&tfull[acc]);
        }
      }
      __syncwarp();
    }
  } else if (warp >= 4) {
    // ---------------- epilogue ----------------
    const int ew = warp - 4;
    int local = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++local) {
      const TileCoord c = tile_of(p, t);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int r_local = ew * 32 + lane;
      int row = c.m0 + r_local;
      bool row_ok;
      if (p.groups && !p.grouped_k)
        row_ok = (c.mb * BM + r_local) < p.g_rows[c.g];
      else
        row_ok = row < p.M;
      const int64_t dgoff = (p.groups && p.grouped_k) ? int64_t(c.g) * p.g_d_stride : 0;
      const uint32_t tbase = tmem_base + (uint32_t(ew * 32) << 16) + acc * BN;
      const bool empty_k = c.nk == 0;

      if (p.epi == GEMM_EPI_SWIGLU_BWD) {
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld32(tbase + ch * 32, v);
          ptx::tmem_wait_ld();
          const int f0 = c.nb * BN + ch * 32;
          if (row_ok && f0 < p.N)
            epi::swiglu_bwd32(v, p.G2 + int64_t(row) * p.ldg2,
                              reinterpret_cast<__nv_bfloat16*>(p.D) + int64_t(row) * p.ldd, f0);
        }
      } else if (p.epi == GEMM_EPI_SWIGLU) {
        // Columns [0,128) of the tile are gate, [128,256) up, for features
        // nb*128 + [0,128).
#pragma unroll 1
        for (int ch = 0; ch < 4; ++ch) {
          uint32_t g[32], u[32];
          ptx::tmem_ld32(tbase + ch * 32, g);
          ptx::tmem_ld32(tbase + 128 + ch * 32, u);
          ptx::tmem_wait_ld();
          if (p.bias) {
            float bg[32], bu[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) bg[i] = __uint_as_float(g[i]), bu[i] = __uint_as_float(u[i]);
            epi::add_bias32(bg, p.bias + c.nb * BN + ch * 32);
            epi::add_bias32(bu, p.bias + c.nb * BN + 128 + ch * 32);
#pragma unroll
            for (int i = 0; i < 32; ++i) g[i] = __float_as_uint(bg[i]), u[i] = __float_as_uint(bu[i]);
          }
          const int f0 = c.nb * 128 + ch * 32;
          if (p.staged) {
            // act (and gate|up) rows out through the per-warp stage: 8 rows x
            // 64 contiguous bytes per store instruction
            if (f0 >= p.N / 2) continue;  // warp-uniform
            uint32_t pa[16], pg[16], pu[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              const float2 gf = ptx::unpack_bf16(ptx::pack_bf16(__uint_as_float(g[2 * e]), __uint_as_float(g[2 * e + 1])));
              const float2 uf = ptx::unpack_bf16(ptx::pack_bf16(__uint_as_float(u[2 * e]), __uint_as_float(u[2 * e + 1])));
              pa[e] = ptx::pack_bf16(silu(gf.x) * uf.x, silu(gf.y) * uf.y);
              pg[e] = ptx::pack_bf16(gf.x, gf.y);
              pu[e] = ptx::pack_bf16(uf.x, uf.y);
            }
            __nv_bfloat16* stg = reinterpret_cast<__nv_bfloat16*>(smem + EPI_OFF) + ew * 32 * EPI_LD;
            const int rloc0 = c.mb * BM + ew * 32, cc = (lane & 3) * 8;
            auto out = [&](const uint32_t* w, __nv_bfloat16* base, int64_t ld) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                *reinterpret_cast<uint4*>(stg + lane * EPI_LD + 8 * q) =
                    make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
              __syncwarp();
#pragma unroll
              for (int it = 0; it < 4; ++it) {
                const int rr = it * 8 + (lane >> 2);
                const bool ok = (p.groups && !p.grouped_k) ? (rloc0 + rr) < p.g_rows[c.g]
                                                           : (c.m0 + ew * 32 + rr) < p.M;
                if (ok)
                  *reinterpret_cast<uint4*>(base + int64_t(c.m0 + ew * 32 + rr) * ld + cc) =
                      *reinterpret_cast<const uint4*>(stg + rr * EPI_LD + cc);
              }
              __syncwarp();
            };
            out(pa, p.D2 + f0, p.ldd2);
            if (p.D) {
              __nv_bfloat16* gu = reinterpret_cast<__nv_bfloat16*>(p.D) + c.nb * BN + ch * 32;
              out(pg, gu, p.ldd);
              out(pu, gu + 128, p.ldd);
            }
            continue;
          }
          if (row_ok && f0 < p.N / 2) {
            __nv_bfloat16* act = p.D2 + int64_t(row) * p.ldd2 + f0;
            __nv_bfloat16* gu = p.D ? reinterpret_cast<__nv_bfloat16*>(p.D) + int64_t(row) * p.ldd +
                                          c.nb * BN + ch * 32
                                    : nullptr;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 va, vg, vu;
              uint32_t* pa = reinterpret_cast<uint32_t*>(&va);
              uint32_t* pg = reinterpret_cast<uint32_t*>(&vg);
              uint32_t* pu = reinterpret_cast<uint32_t*>(&vu);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                // round gate/up to bf16 first: the saved gu is what backward sees
                const float2 gf = ptx::unpack_bf16(ptx::pack_bf16(
                    __uint_as_float(g[q * 8 + 2 * e]), __uint_as_float(g[q * 8 + 2 * e + 1])));
                const float2 uf = ptx::unpack_bf16(ptx::pack_bf16(
                    __uint_as_float(u[q * 8 + 2 * e]), __uint_as_float(u[q * 8 + 2 * e + 1])));
                pa[e] = ptx::pack_bf16(silu(gf.x) * uf.x, silu(gf.y) * uf.y);
                pg[e] = ptx::pack_bf16(gf.x, gf.y);
                pu[e] = ptx::pack_bf16(uf.x, uf.y);
              }
              *reinterpret_cast<uint4*>(act + q * 8) = va;
              if (gu) {
                *reinterpret_cast<uint4*>(gu + q * 8) = vg;
                *reinterpret_cast<uint4*>(gu + 128 + q * 8) = vu;
              }
            }
          }
        }
      } else if ((p.epi == GEMM_EPI_BF16 || p.epi == GEMM_EPI_ROWMAP) && p.staged) {
        __nv_bfloat16* stg = reinterpret_cast<__nv_bfloat16*>(smem + EPI_OFF) + ew * 32 * EPI_LD;
        const int rloc0 = c.mb * BM + ew * 32;  // this warp's first row (within the group)
        // the 4 rows this lane stores (it * 8 + lane / 4): their destination
        // rows -- D's own, or (ROWMAP) the token owner's combine slot
        __nv_bfloat16* dst_row[4];
#pragma unroll
        for (int it = 0; it < 4; ++it) {
          const int rr = it * 8 + (lane >> 2);
          dst_row[it] = nullptr;
          const bool ok = (p.groups && !p.grouped_k) ? (rloc0 + rr) < p.g_rows[c.g] : (c.m0 + ew * 32 + rr) < p.M;
          if (!ok) continue;
          if (p.epi == GEMM_EPI_ROWMAP) {
            int rg = rloc0 + rr;
            const int* cnt = p.rm_cnt + c.g * p.rm_ep;
            int sidx = 0;
            while (sidx + 1 < p.rm_ep && rg >= cnt[sidx]) rg -= cnt[sidx++];
            dst_row[it] = p.rm_dst[sidx] + int64_t(p.rm_off[c.g * p.rm_ep + sidx] + rg) * p.ldd;
          } else {
            dst_row[it] = reinterpret_cast<__nv_bfloat16*>(p.D) + dgoff + int64_t(c.m0 + ew * 32 + rr) * p.ldd;
          }
        }
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld32(tbase + ch * 32, v);
          ptx::tmem_wait_ld();
          const int col0 = c.nb * BN + ch * 32;
          if (col0 >= p.N) continue;  // warp-uniform
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = empty_k ? 0.f : __uint_as_float(v[i]) * p.scale;
          if (p.bias) epi::add_bias32(f, p.bias + col0);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(stg + lane * EPI_LD + 8 * q) =
                make_uint4(ptx::pack_bf16(f[8 * q], f[8 * q + 1]), ptx::pack_bf16(f[8 * q + 2], f[8 * q + 3]),
                           ptx::pack_bf16(f[8 * q + 4], f[8 * q + 5]), ptx::pack_bf16(f[8 * q + 6], f[8 * q + 7]));
          __syncwarp();
          const int cc = (lane & 3) * 8, col = col0 + cc;
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int rr = it * 8 + (lane >> 2);
            if (dst_row[it] && col < p.N)
              *reinterpret_cast<uint4*>(dst_row[it] + col) = *reinterpret_cast<const uint4*>(stg + rr * EPI_LD + cc);
          }
          __syncwarp();
        }
      } else {
        // the output row: D's own, or (ROWMAP) its token owner's combine slot
        __nv_bfloat16* brow = reinterpret_cast<__nv_bfloat16*>(p.D) + dgoff + int64_t(row) * p.ldd;
        if (p.epi == GEMM_EPI_ROWMAP && row_ok) {
          int r = c.mb * BM + r_local;  // row within group c.g
          const int* cnt = p.rm_cnt + c.g * p.rm_ep;
          int s = 0;
          while (s + 1 < p.rm_ep && r >= cnt[s]) r -= cnt[s++];
          brow = p.rm_dst[s] + int64_t(p.rm_off[c.g * p.rm_ep + s] + r) * p.ldd;
        }
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld32(tbase + ch * 32, v);
          ptx::tmem_wait_ld();
          const int col0 = c.nb * BN + ch * 32;
          if (!row_ok || col0 >= p.N) continue;
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = empty_k ? 0.f : __uint_as_float(v[i]) * p.scale;
          if (p.bias) epi::add_bias32(f, p.bias + col0);
          const bool full_chunk = col0 + 32 <= p.N;
          if (p.epi == GEMM_EPI_BF16 || p.epi == GEMM_EPI_ROWMAP) {
            __nv_bfloat16* d = brow + col0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              if (!full_chunk && col0 + q * 8 >= p.N) break;
              uint4 o;
              o.x = ptx::pack_bf16(f[q * 8 + 0], f[q * 8 + 1]);
              o.y = ptx::pack_bf16(f[q * 8 + 2], f[q * 8 + 3]);
              o.z = ptx::pack_bf16(f[q * 8 + 4], f[q * 8 + 5]);
              o.w = ptx::pack_bf16(f[q * 8 + 6], f[q * 8 + 7]);
              *reinterpret_cast<uint4*>(d + q * 8) = o;
            }
          } else {
            float* d = reinterpret_cast<float*>(p.D) + dgoff + int64_t(row) * p.ldd + col0;
            const float* r = nullptr;
            if (p.epi == GEMM_EPI_F32_RESID) r = p.R + int64_t(row) * p.ldr + col0;
            if (p.epi == GEMM_EPI_F32_ACCUM) r = d;
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              if (!full_chunk && col0 + q * 4 >= p.N) break;
              float4 o = make_float4(f[q * 4 + 0], f[q * 4 + 1], f[q * 4 + 2], f[q * 4 + 3]);
              if (r) {
                const float4 rv = *reinterpret_cast<const float4*>(r + q * 4);
                o.x += rv.x;
                o.y += rv.y;
                o.z += rv.z;
                o.w += rv.w;
              }
              *reinterpret_cast<float4*>(d + q * 4) = o;
            }
          }
        }
      }
      ptx::tc_fence_before();
      ptx::mbar_arrive(&tempty[acc]);
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc(tmem_base, 512);
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;
int g_num_sms = 0;

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
  std::call_once(g_encode_once, [] {
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  return g_encode;
}

// 2-D bf16 tensor map: inner dim (contiguous) x outer dim, row stride in elements.
bool make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
              uint32_t box_inner, uint32_t box_outer) {
  auto enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides,
                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <bool A_MN, bool B_MN>
cudaError_t launch(const CUtensorMap& a, const CUtensorMap& b, const KParams& kp, int grid,
                   cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel<A_MN, B_MN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  ++g_kernel_launches;
  gemm_tc_kernel<A_MN, B_MN><<<grid, NUM_THREADS, SMEM_BYTES, s>>>(a, b, kp);
  return cudaGetLastError();
}

}  // namespace

bool gemm_make_map(void* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                   uint32_t box_inner, uint32_t box_outer) {
  return make_map(static_cast<CUtensorMap*>(map), base, inner, outer, ld, box_inner, box_outer);
}

int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

static cudaError_t gemm_run_impl(const GemmDesc& g, cudaStream_t s);

// Diagnostics (OPX_GEMM_LOG=1): per-launch CUDA events around every GEMM,
// aggregated by shape/layout/epilogue by gemm_log_dump().
namespace {
struct GemmLogEntry {
  int M, N, K, a_mn, b_mn, epi, groups;
  cudaEvent_t e0, e1;
};
std::vector<GemmLogEntry> g_gemm_log;
}  // namespace

cudaError_t gemm_run(const GemmDesc& g, cudaStream_t s) {
  static const bool log = getenv("OPX_GEMM_LOG") != nullptr;
  if (!log) return gemm_run_impl(g, s);
  GemmLogEntry e{g.M, g.N, g.K, g.a_mn, g.b_mn, g.epi, g.groups, nullptr, nullptr};
  cudaEventCreate(&e.e0);
  cudaEventCreate(&e.e1);
  cudaEventRecord(e.e0, s);
  const cudaError_t r = gemm_run_impl(g, s);
  cudaEventRecord(e.e1, s);
  g_gemm_log.push_back(e);
  return r;
}

void gemm_log_dump(const char* tag) {
  if (g_gemm_log.empty()) return;
  struct Agg {
    int n = 0;
    double ms = 0, mn = 1e30, mx = 0;
  };
  std::map<std::string, Agg> agg;
  static const bool each = getenv("OPX_GEMM_LOG")[0] == '2';
  int idx = 0;
  for (auto& e : g_gemm_log) {
    cudaEventSynchronize(e.e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e.e0, e.e1);
    char key[128];
    snprintf(key, sizeof key, "M=%d N=%d K=%d a_mn=%d b_mn=%d epi=%d groups=%d", e.M, e.N, e.K, e.a_mn,
             e.b_mn, e.epi, e.groups);
    Agg& a = agg[key];
    ++a.n;
    a.ms += ms;
    a.mn = std::min(a.mn, double(ms));
    a.mx = std::max(a.mx, double(ms));
    if (each)
      fprintf(stderr, "[gemm1 %s] #%d %s %.3f ms %.0f TF/s\n", tag, idx, key, ms,
              2.0 * e.M * e.N * e.K / ms / 1e9);
    ++idx;
    cudaEventDestroy(e.e0);
    cudaEventDestroy(e.e1);
  }
  g_gemm_log.clear();
  for (auto& kv : agg) {
    int M, N, K;
    sscanf(kv.first.c_str(), "M=%d N=%d K=%d", &M, &N, &K);
    const double mean = kv.second.ms / kv.second.n;
    fprintf(stderr, "[gemm %s] %s n=%d mean=%.3f min=%.3f max=%.3f ms  %.0f TF/s(mean) %.0f(min)\n", tag,
            kv.first.c_str(), kv.second.n, mean, kv.second.mn, kv.second.mx, 2.0 * M * N * K / mean / 1e9,
            2.0 * M * N * K / kv.second.mn / 1e9);
  }
}

static cudaError_t gemm_run_impl(const GemmDesc& g, cudaStream_t s) {
  if ((g.groups == 0 || g.grouped_k) && g.M <= 0) return cudaSuccess;
  if (g.N <= 0) return cudaSuccess;
  if (g.N % 8 != 0 || (g.epi == GEMM_EPI_SWIGLU && g.N % 256 != 0)) return cudaErrorInvalidValue;
  if (g.epi == GEMM_EPI_SWIGLU_BWD && (g.N % 128 != 0 || !g.G2 || g.groups)) return cudaErrorInvalidValue;
  if (g.epi == GEMM_EPI_SEQ2HEAD && (g.N % 128 != 0 || !g.s2h || g.groups || getenv("OPX_GEMM_1CTA")))
    return cudaErrorNotSupported;  // the fused exchange epilogue exists on the 2-CTA kernel only
  CUtensorMap ma, mb;
  const bool grouped = g.groups > 0;
  const bool gm = grouped && !g.grouped_k;  // rows of A vary per group
  const bool gk = grouped && g.grouped_k;   // K varies per group (wgrad)
  if (gk && !(g.a_mn && g.b_mn)) return cudaErrorInvalidValue;
  if (gm && g.a_mn) return cudaErrorInvalidValue;
  const uint64_t a_rows = gm ? uint64_t(g.rows_total) : uint64_t(g.M);
  const uint64_t k_ext = gk ? uint64_t(g.rows_total) : uint64_t(g.K);
  bool ok = !g.a_mn ? make_map(&ma, g.A, k_ext, a_rows, g.lda, BK, BM)
                    : make_map(&ma, g.A, uint64_t(g.M), k_ext, g.lda, 64, BK);
  if (!ok) return cudaErrorInvalidValue;
  if (!g.b_mn) {
    const uint64_t brows = gm ? uint64_t(g.groups) * uint64_t(g.N) : uint64_t(g.N);
    ok = make_map(&mb, g.B, uint64_t(g.K), brows, g.ldb, BK, BN);
  } else {
    const uint64_t krows = gm ? uint64_t(g.groups) * uint64_t(g.K) : k_ext;
    ok = make_map(&mb, g.B, uint64_t(g.N), krows, g.ldb, 64, BK);
  }
  if (!ok) return cudaErrorInvalidValue;

  KParams kp{};
  kp.M = g.M;
  kp.N = g.N;
  kp.K = g.K;
  kp.epi = g.epi;
  kp.D = g.D;
  kp.ldd = g.ldd;
  kp.R = g.R;
  kp.ldr = g.ldr;
  kp.D2 = g.D2;
  kp.ldd2 = g.ldd2;
  kp.G2 = g.G2;
  kp.ldg2 = g.ldg2;
  kp.scale = g.scale == 0.f ? 1.f : g.scale;
  kp.groups = g.groups;
  kp.grouped_k = g.grouped_k;
  kp.g_start = g.g_start;
  kp.g_rows = g.g_rows;
  kp.g_b_rows = gm ? (g.b_mn ? g.K : g.N) : 0;
  kp.g_d_stride = g.d_group_stride;

  int tiles;
  const int nblk = (g.N + BN - 1) / BN;
  kp.band = 1;
  static const bool force_1cta = getenv("OPX_GEMM_1CTA") != nullptr;
  // grouped-M (expert fwd / dgrad) on the 2-CTA kernel (device-side tile
  // lists) is opt-in: on the C2 expert shapes it measured equal (dgrad, down)
  // or slower (gate|up + SwiGLU: 0.54 vs 0.36 ms) than the 1-CTA kernel
  static const bool grouped_2cta = getenv("OPX_GEMM_GROUPED_2CTA") != nullptr;
  if (g.bias && (g.N % 32 || (g.epi != GEMM_EPI_BF16 && g.epi != GEMM_EPI_F32 &&
                              g.epi != GEMM_EPI_F32_RESID && g.epi != GEMM_EPI_SWIGLU)))
    return cudaErrorInvalidValue;
  if (g.epi == GEMM_EPI_ROWMAP && (!gm || !g.rm_dst || !g.rm_cnt || !g.rm_off))
    return cudaErrorInvalidValue;
  kp.rm_dst = g.rm_dst;
  kp.rm_cnt = g.rm_cnt;
  kp.rm_off = g.rm_off;
  kp.rm_ep = g.rm_ep;
  kp.bias = g.bias;
  {
    static const int staged = getenv("OPX_GEMM_EPI_STAGED") ? atoi(getenv("OPX_GEMM_EPI_STAGED")) : 1;
    kp.staged = staged;
  }
  if (gm && grouped_2cta && !force_1cta && g.K % BK == 0 && g.epi != GEMM_EPI_ROWMAP)
    return gemm2_run(g, 1, s);
  if (!grouped && !force_1cta) {
    // 2-CTA path: same traffic model with 256-row pair tiles and 74 pairs per wave
    const double a_bytes = double(g.M) * g.K * 2, b_blk = 256.0 * g.K * 2;
    const int mblk2 = (g.M + 255) / 256;
    // L2 budget for the resident B panel (OPX_GEMM_BUDGET_MB overrides, read per call)
    const char* be = getenv("OPX_GEMM_BUDGET_MB");
    const double budget = be ? atof(be) * 1e6 : 40e6, wave = num_sms() / 2;
    double best = 1e300;
    int band = 1;
    // candidate bands: power-of-two band widths, or (OPX_GEMM_BAND_EQUAL=1)
    // equal splits of the n-blocks for every band count -- the latter cut the
    // C1 gate|up DRAM reads 2.64 -> 2.22 GB per call but left its time and the
    // step unchanged (within +-0.5 %) and measured noisier on other shapes
    static const bool pow2 = !(getenv("OPX_GEMM_BAND_EQUAL") && atoi(getenv("OPX_GEMM_BAND_EQUAL")));
    int prev = 0;
    for (int i = 1;; ++i) {
      const int nb = pow2 ? std::min(nblk, 1 << (i - 1)) : (nblk + i - 1) / i;
      if (nb != prev) {
        prev = nb;
        const double bands = double((nblk + nb - 1) / nb);
        double b_traffic = double(nblk) * b_blk;
        if (nb * b_blk > budget) {
          const double m_per_wave = wave / nb < 1 ? 1 : wave / nb;
          b_traffic *= double(mblk2) / m_per_wave;
        }
        const double tot = a_bytes * bands + b_traffic;
        if (tot < best * 0.999) {
          best = tot;
          band = nb;
        }
      }
      if (pow2 ? nb == nblk : nb == 1) break;
    }
    return gemm2_run(g, band, s);
  }
  if (!grouped) {
    // Pick the raster band minimising a DRAM-traffic estimate: inside a band
    // the (band x 256)-row B panel should stay L2-resident while every m-block
    // streams its A panel once per band.
    const double a_bytes = double(g.M) * g.K * 2, b_blk = 256.0 * g.K * 2;
    const int mblk = (g.M + BM - 1) / BM;
    const double budget = 80e6, wave = num_sms();
    double best = 1e300;
    for (int nb = 1;; nb = nb * 2 > nblk ? nblk : nb * 2) {
      const double bands = double((nblk + nb - 1) / nb);
      double b_traffic = double(nblk) * b_blk;
      if (nb * b_blk > budget) {
        const double m_per_wave = wave / nb < 1 ? 1 : wave / nb;
        b_traffic *= double(mblk) / m_per_wave;
      }
      const double tot = a_bytes * bands + b_traffic;
      if (tot < best * 0.999) {
        best = tot;
        kp.band = nb;
      }
      if (nb == nblk) break;
    }
  }
  if (!grouped)
    tiles = ((g.M + BM - 1) / BM) * nblk;
  else if (g.grouped_k)
    tiles = g.groups * ((g.M + BM - 1) / BM) * nblk;
  else
    tiles = int((g.rows_total + BM - 1) / BM + g.groups) * nblk;  // upper bound
  int grid = tiles < num_sms() ? tiles : num_sms();
  if (grid < 1) grid = 1;
  if (!g.a_mn && !g.b_mn) return launch<false, false>(ma, mb, kp, grid, s);
  if (!g.a_mn && g.b_mn) return launch<false, true>(ma, mb, kp, grid, s);
  if (g.a_mn && !g.b_mn) return launch<true, false>(ma, mb, kp, grid, s);
  return launch<true, true>(ma, mb, kp, grid, s);
}

}  // namespace opx
