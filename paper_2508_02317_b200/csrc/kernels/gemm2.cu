// 2-CTA bf16 GEMM on tcgen05 (cta_group::2), sm_100a.
//
// A cluster of two CTAs (one TPC) computes a 256 x 256 output tile with one
// tcgen05.mma.cta_group::2 stream issued by the leader CTA: each CTA stages
// its 128 rows of A and its 128 rows (output columns) of B, so every byte
// loaded from L2 feeds twice the MMA work of the 1-CTA 128 x 256 tile
// (128 vs 85 FLOP/B) -- the 1-CTA kernel was L2->SM bandwidth bound
// (profiles/r1_c1_n1_summary.txt: 85 % L2 hit, ~14.6 TB/s L2 reads).
// Each CTA's TMEM holds its 128 accumulator rows x 256 columns (double
// buffered); its four epilogue warps drain them with the same fused
// epilogues as kernels/gemm.cu.  Grouped (MoE) GEMMs stay on the 1-CTA kernel.
//
// Tiles are handed out dynamically: the leader's producer takes tickets from a
// global counter and publishes each tile id through a small smem ring (with
// mbarriers) to its MMA warp, both CTAs' epilogues and the peer producer.  A
// static persistent schedule stalls the whole GEMM when some SMs are held by a
// concurrent kernel (the FSDP all-gather / reduce-scatter on the comm stream):
// the clusters that start late would still own 1/74 of the tiles each.  With
// tickets, late clusters just find the work already taken.
#include <cuda.h>

#include "../runtime/gemm_api.h"
#include "../runtime/kernels_api.h"
#include "../runtime/kernels_api.h"
#include "epilogue.cuh"
#include "ptx.cuh"

namespace opx {
namespace {

constexpr int BM = 128;   // rows per CTA (256 per pair)
constexpr int BNP = 256;  // output columns per pair tile
constexpr int BNC = 128;  // B rows staged per CTA
constexpr int BK = 64, STAGES = 6;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = BNC * BK * 2;  // 16 KB
constexpr int QD = 4;                    // tile-id ring depth
constexpr int Q_CONSUMERS = 1 + 1 + 4 + 4;  // peer producer, MMA, 2 x 4 epilogue warps
// fp32 epilogue staging: per epilogue warp a [32 rows][36] fp32 block, so the
// fp32 stores / residual loads go out row-contiguous (4 rows x 128 B per warp
// instruction) instead of one 16-B piece of 32 different rows
constexpr int EPI_LD = 36;
constexpr int OFF_EPI = STAGES * (A_BYTES + B_BYTES) + 512;
constexpr int SMEM = OFF_EPI + 4 * 32 * EPI_LD * 4 + 1024;
constexpr int THREADS = 256;

struct P2 {
  int M, N, K, epi, band;
  void* D;
  int64_t ldd;
  const float* R;
  int64_t ldr;
  __nv_bfloat16* D2;
  int64_t ldd2;
  const __nv_bfloat16* G2;
  int64_t ldg2;
  float scale;
  int* ctr;  // ticket counter (0 at launch; reset to 0 by the last ticket taker)
  // grouped-M (MoE experts): A/D rows of group g are g_start[g] .. +g_rows[g]
  // (128-aligned segments; a 256-row pair tile may run into the next segment,
  // those rows are computed and masked), B is slab g of a [groups*N, K]
  // (K-major) or [groups*K, N] (MN-major) stack
  int groups;
  const int* g_start;
  const int* g_rows;
  A2AArgs s2h;  // GEMM_EPI_SEQ2HEAD
  const __nv_bfloat16* bias;  // optional column bias
  int staged;                 // fp32 epilogues through the per-warp smem stage
};

__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

__device__ __forceinline__ int ntiles_of(const P2& p) {
  const int nblk = (p.N + BNP - 1) / BNP;
  if (!p.groups) return ((p.M + 2 * BM - 1) / (2 * BM)) * nblk;
  int n = 0;
  for (int g = 0; g < p.groups; ++g) n += ((p.g_rows[g] + 2 * BM - 1) / (2 * BM)) * nblk;
  return n;
}
// grouped tile t -> group, first A/D row of the pair tile, n-block
__device__ __forceinline__ void gtile_coords(const P2& p, int t, int& g, int& row0, int& nb) {
  const int nblk = (p.N + BNP - 1) / BNP;
  for (g = 0; g < p.groups; ++g) {
    const int mblk = (p.g_rows[g] + 2 * BM - 1) / (2 * BM);
    if (t < mblk * nblk) {
      row0 = p.g_start[g] + (t % mblk) * 2 * BM;
      nb = t / mblk;
      return;
    }
    t -= mblk * nblk;
  }
}
__device__ __forceinline__ void tile_coords(const P2& p, int t, int& mb, int& nb) {
  const int mblk = (p.M + 2 * BM - 1) / (2 * BM);
  const int nblk = (p.N + BNP - 1) / BNP;
  const int per_band = p.band * mblk;
  const int b = t / per_band, r = t % per_band;
  const int bw = min(p.band, nblk - b * p.band);
  mb = r / bw;
  nb = b * p.band + r % bw;
}

template <bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const P2 p) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* tq_full = tempty + 2;
  uint64_t* tq_empty = tq_full + QD;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tq_empty + QD);
  int* tile_q = reinterpret_cast<int*>(tmem_slot + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  const uint32_t rank = ptx::cluster_ctarank();
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    ptx::tma_prefetch(&tmA);
    ptx::tma_prefetch(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], 2 * 128);  // both CTAs' epilogue threads (leader's is used)
    }
    for (int s = 0; s < QD; ++s) {
      ptx::mbar_init(&tq_full[s], 1);
      ptx::mbar_init(&tq_empty[s], Q_CONSUMERS);  // leader's is used
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc_pair(tmem_slot, 512);
  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int ntiles = ntiles_of(p);
  const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;
  const int nk = (p.K + BK - 1) / BK;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs) ----------------
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int qi = 0;
      uint32_t qph = 0;
      const uint32_t peer_tq = ptx::mapa(ptx::smem_u32(tile_q), 1);
      const uint32_t peer_tqf = ptx::mapa(ptx::smem_u32(tq_full), 1);
      const uint32_t leader_tqe = ptx::mapa(ptx::smem_u32(tq_empty), 0);
      int t = cid;
      if (leader) {  // publish the first tile
        ptx::mbar_wait(&tq_empty[qi], qph ^ 1);
        tile_q[qi] = t;
        ptx::st_shared_cluster(peer_tq + 4 * qi, t);
        ptx::mbar_arrive(&tq_full[qi]);
        ptx::mbar_arrive_cluster(peer_tqf + 8 * qi);
      } else {
        ptx::mbar_wait_cluster(&tq_full[qi], qph);
        t = tile_q[qi];
        ptx::mbar_arrive_cluster(leader_tqe + 8 * qi);
      }
      if (++qi == QD) {
        qi = 0;
        qph ^= 1;
      }
      while (t < ntiles) {
        // leader: take the next ticket now, publish it after this tile's loads
        int v = 0;
        if (leader) v = atomicAdd(p.ctr, 1);
        int mb = 0, nb = 0, g = 0, row0 = 0;
        if (p.groups) gtile_coords(p, t, g, row0, nb);
        else tile_coords(p, t, mb, nb), row0 = mb * 2 * BM;
        const int m0 = row0 + int(rank) * BM;
        // grouped: B slab g sits g*N rows (K-major) / g*K k-rows (MN-major) down
        const int n0 = nb * BNP + int(rank) * BNC + (p.groups && !B_MN ? g * p.N : 0);
        const int kofs = p.groups && B_MN ? g * p.K : 0;
        for (int kb = 0; kb < nk; ++kb) {
          ptx::mbar_wait(&empty[stage], phase ^ 1);
          if (leader) ptx::mbar_expect_tx(&full[stage], 2 * (A_BYTES + B_BYTES));
          const uint32_t bar = ptx::mapa(ptx::smem_u32(&full[stage]), 0);
          uint8_t* a = sA + stage * A_BYTES;
          uint8_t* b = sB + stage * B_BYTES;
          const int k0 = kb * BK;
          if (!A_MN) {
            ptx::tma_load_2d_pair(&tmA, bar, a, k0, m0);
          } else {
            ptx::tma_load_2d_pair(&tmA, bar, a, m0, k0);
            ptx::tma_load_2d_pair(&tmA, bar, a + 8192, m0 + 64, k0);
          }
          if (!B_MN) {
            ptx::tma_load_2d_pair(&tmB, bar, b, k0, n0);
          } else {
            ptx::tma_load_2d_pair(&tmB, bar, b, n0, kofs + k0);
            ptx::tma_load_2d_pair(&tmB, bar, b + 8192, n0 + 64, kofs + k0);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (leader) {
          if (v == ntiles - 1) atomicExch(p.ctr, 0);  // last ticket overall: reset for reuse
          t = ncl + v;
          ptx::mbar_wait(&tq_empty[qi], qph ^ 1);
          tile_q[qi] = t;
          ptx::st_shared_cluster(peer_tq + 4 * qi, t);
          ptx::mbar_arrive(&tq_full[qi]);
          ptx::mbar_arrive_cluster(peer_tqf + 8 * qi);
        } else {
          ptx::mbar_wait_cluster(&tq_full[qi], qph);
          t = tile_q[qi];
          ptx::mbar_arrive_cluster(leader_tqe + 8 * qi);
        }
        if (++qi == QD) {
          qi = 0;
          qph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA only) ----------------
    if (leader) {
      constexpr uint32_t idesc = ptx::idesc_bf16_f32(2 * BM, BNP, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      int qi = 0;
      uint32_t qph = 0;
      for (;; ++local) {
        ptx::mbar_wait(&tq_full[qi], qph);
        const int t = tile_q[qi];
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&tq_empty[qi]);
        if (++qi == QD) {
          qi = 0;
          qph ^= 1;
        }
        if (t >= ntiles) break;
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        ptx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BNP;
        for (int kb = 0; kb < nk; ++kb) {
          ptx::mbar_wait(&full[stage], phase);
          ptx::tc_fence_after();
          if (lane == 0) {
            const uint32_t a_addr = ptx::smem_u32(sA + stage * A_BYTES);
            const uint32_t b_addr = ptx::smem_u32(sB + stage * B_BYTES);
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              const uint64_t ad = A_MN ? ptx::umma_desc_sw128(a_addr + k * 2048, 8192, 1024)
                                       : ptx::umma_desc_sw128(a_addr + k * 32, 16, 1024);
              const uint64_t bd = B_MN ? ptx::umma_desc_sw128(b_addr + k * 2048, 8192, 1024)
                                       : ptx::umma_desc_sw128(b_addr + k * 32, 16, 1024);
              ptx::mma_bf16_ss_pair(d_tmem, ad, bd, idesc, (kb | k) != 0);
            }
            ptx::mma_commit_pair(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (lane == 0) ptx::mma_commit_pair(&tfull[acc], 0x3);
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue (both CTAs, own 128 rows) ----------------
    const int ew = warp - 4;
    int local = 0;
    const uint32_t tempty_leader[2] = {ptx::mapa(ptx::smem_u32(&tempty[0]), 0),
                                       ptx::mapa(ptx::smem_u32(&tempty[1]), 0)};
    const uint32_t leader_tqe = ptx::mapa(ptx::smem_u32(tq_empty), 0);
    int qi = 0;
    uint32_t qph = 0;
    for (;; ++local) {
      if (leader) ptx::mbar_wait(&tq_full[qi], qph);
      else ptx::mbar_wait_cluster(&tq_full[qi], qph);
      const int t = tile_q[qi];
      __syncwarp();
      if (lane == 0) {
        if (leader) ptx::mbar_arrive(&tq_empty[qi]);
        else ptx::mbar_arrive_cluster(leader_tqe + 8 * qi);
      }
      if (++qi == QD) {
        qi = 0;
        qph ^= 1;
      }
      if (t >= ntiles) break;
      int mb = 0, nb = 0, g = 0, row0 = 0;
      if (p.groups) gtile_coords(p, t, g, row0, nb);
      else tile_coords(p, t, mb, nb), row0 = mb * 2 * BM;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      ptx::mbar_wait(&tfull[acc], acc_phase);
      ptx::tc_fence_after();
      const int row = row0 + int(rank) * BM + ew * 32 + lane;
      const bool row_ok = p.groups ? (row - p.g_start[g]) < p.g_rows[g] : row < p.M;
      const uint32_t tbase = tmem_base + (uint32_t(ew * 32) << 16) + acc * BNP;
      if (p.epi == GEMM_EPI_SWIGLU_BWD) {
#pragma unroll 1
        for (int ch = 0; ch < BNP / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld32(tbase + ch * 32, v);
          ptx::tmem_wait_ld();
          const int f0 = nb * BNP + ch * 32;
          if (row_ok && f0 < p.N)
            epi::swiglu_bwd32(v, p.G2 + int64_t(row) * p.ldg2,
                              reinterpret_cast<__nv_bfloat16*>(p.D) + int64_t(row) * p.ldd, f0);
        }
      } else if (p.epi == GEMM_EPI_SEQ2HEAD) {
        // this thread's row = local token `row` of SP rank s2h.rank; each head
        // vector of the tile goes to its owner's [rows*S, heads/sp, 128] slot
        const A2AArgs& a = p.s2h;
        const int S_loc = a.seq / a.sp;
        const int rb = row / S_loc;
        const int64_t gtok = int64_t(rb) * a.seq + int64_t(a.rank) * S_loc + (row - rb * S_loc);
        const int pos = row_ok ? a.pos[gtok] : 0;
#pragma unroll 1
        for (int hv = 0; hv < BNP / 128; ++hv) {
          const int c0 = nb * BNP + hv * 128;
          if (c0 >= p.N) break;
          int gi = 0;
          while (gi + 1 < a.ngroups && c0 >= a.g[gi + 1].col0) ++gi;
          const A2AGroup& G = a.g[gi];
          const int hh = (c0 - G.col0) >> 7;
          const int per_rank = G.heads_total / a.sp;
          const int dst = hh / per_rank, hl = hh - dst * per_rank;
          __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(G.full[dst]) +
                             (gtok * per_rank + hl) * 128;
#pragma unroll 1
          for (int ch = 0; ch < 2; ++ch) {
            uint32_t x1[32], x2[32];
            ptx::tmem_ld32(tbase + hv * 128 + ch * 32, x1);
            ptx::tmem_ld32(tbase + hv * 128 + 64 + ch * 32, x2);
            ptx::tmem_wait_ld();
            if (!row_ok) continue;
            uint32_t lo[16], hi[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) {
              // bf16 rounding where the unfused path stores qkv, then RoPE in fp32
              lo[e] = ptx::pack_bf16(__uint_as_float(x1[2 * e]) * p.scale,
                                     __uint_as_float(x1[2 * e + 1]) * p.scale);
              hi[e] = ptx::pack_bf16(__uint_as_float(x2[2 * e]) * p.scale,
                                     __uint_as_float(x2[2 * e + 1]) * p.scale);
              if (G.rope) {
                const int j = ch * 32 + 2 * e;
                const float2 a1 = ptx::unpack_bf16(lo[e]), a2 = ptx::unpack_bf16(hi[e]);
                float sn0, cs0, sn1, cs1;
                if (a.rope_tab) {
                  const float4 t = *reinterpret_cast<const float4*>(a.rope_tab + int64_t(pos) * 64 + j);
                  sn0 = t.x; cs0 = t.y; sn1 = t.z; cs1 = t.w;
                } else {
                  sincosf(float(pos) * a.inv_freq[j], &sn0, &cs0);
                  sincosf(float(pos) * a.inv_freq[j + 1], &sn1, &cs1);
                }
                lo[e] = ptx::pack_bf16(a1.x * cs0 - a2.x * sn0, a1.y * cs1 - a2.y * sn1);
                hi[e] = ptx::pack_bf16(a2.x * cs0 + a1.x * sn0, a2.y * cs1 + a1.y * sn1);
              }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              *reinterpret_cast<uint4*>(d + ch * 32 + q * 8) =
                  make_uint4(lo[4 * q], lo[4 * q + 1], lo[4 * q + 2], lo[4 * q + 3]);
              *reinterpret_cast<uint4*>(d + 64 + ch * 32 + q * 8) =
                  make_uint4(hi[4 * q], hi[4 * q + 1], hi[4 * q + 2], hi[4 * q + 3]);
            }
          }
        }
      } else if (p.epi == GEMM_EPI_SWIGLU) {
        const int grp = g;  // the group index (g is the gate chunk below)
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
            epi::add_bias32(bg, p.bias + nb * BNP + ch * 32);
            epi::add_bias32(bu, p.bias + nb * BNP + 128 + ch * 32);
#pragma unroll
            for (int i = 0; i < 32; ++i) g[i] = __float_as_uint(bg[i]), u[i] = __float_as_uint(bu[i]);
          }
          const int f0 = nb * 128 + ch * 32;
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
            __nv_bfloat16* stg = reinterpret_cast<__nv_bfloat16*>(smem + OFF_EPI) + ew * 32 * (2 * EPI_LD);
            const int rbase = row0 + int(rank) * BM + ew * 32, cc = (lane & 3) * 8;
            auto out = [&](const uint32_t* w, __nv_bfloat16* base, int64_t ld) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                *reinterpret_cast<uint4*>(stg + lane * (2 * EPI_LD) + 8 * q) =
                    make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
              __syncwarp();
#pragma unroll
              for (int it = 0; it < 4; ++it) {
                const int rr = it * 8 + (lane >> 2), r = rbase + rr;
                if (p.groups ? (r - p.g_start[grp]) < p.g_rows[grp] : r < p.M)
                  *reinterpret_cast<uint4*>(base + int64_t(r) * ld + cc) =
                      *reinterpret_cast<const uint4*>(stg + rr * (2 * EPI_LD) + cc);
              }
              __syncwarp();
            };
            out(pa, p.D2 + f0, p.ldd2);
            if (p.D) {
              __nv_bfloat16* gu = reinterpret_cast<__nv_bfloat16*>(p.D) + nb * BNP + ch * 32;
              out(pg, gu, p.ldd);
              out(pu, gu + 128, p.ldd);
            }
            continue;
          }
          if (row_ok && f0 < p.N / 2) {
            __nv_bfloat16* act = p.D2 + int64_t(row) * p.ldd2 + f0;
            __nv_bfloat16* gu = p.D ? reinterpret_cast<__nv_bfloat16*>(p.D) + int64_t(row) * p.ldd +
                                          nb * BNP + ch * 32
                                    : nullptr;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint4 va, vg, vu;
              uint32_t* pa = reinterpret_cast<uint32_t*>(&va);
              uint32_t* pg = reinterpret_cast<uint32_t*>(&vg);
              uint32_t* pu = reinterpret_cast<uint32_t*>(&vu);
#pragma unroll
              for (int e = 0; e < 4; ++e) {
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
      } else if (p.staged && p.epi == GEMM_EPI_BF16) {
        // bf16 through the same per-warp stage ([32][2 * EPI_LD] bf16): 8 rows
        // x 64 contiguous bytes per warp store instruction
        __nv_bfloat16* stg = reinterpret_cast<__nv_bfloat16*>(smem + OFF_EPI) + ew * 32 * (2 * EPI_LD);
        const int rbase = row0 + int(rank) * BM + ew * 32;
#pragma unroll 1
        for (int ch = 0; ch < BNP / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld32(tbase + ch * 32, v);
          ptx::tmem_wait_ld();
          const int col0 = nb * BNP + ch * 32;
          if (col0 >= p.N) continue;  // warp-uniform
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]) * p.scale;
          if (p.bias) epi::add_bias32(f, p.bias + col0);
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<uint4*>(stg + lane * (2 * EPI_LD) + 8 * q) =
                make_uint4(ptx::pack_bf16(f[8 * q], f[8 * q + 1]), ptx::pack_bf16(f[8 * q + 2], f[8 * q + 3]),
                           ptx::pack_bf16(f[8 * q + 4], f[8 * q + 5]), ptx::pack_bf16(f[8 * q + 6], f[8 * q + 7]));
          __syncwarp();
          const int cc = (lane & 3) * 8, col = col0 + cc;
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const int rr = it * 8 + (lane >> 2), r = rbase + rr;
            const bool ok = (p.groups ? (r - p.g_start[g]) < p.g_rows[g] : r < p.M) && col < p.N;
            if (ok)
              *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(p.D) + int64_t(r) * p.ldd + col) =
                  *reinterpret_cast<const uint4*>(stg + rr * (2 * EPI_LD) + cc);
          }
          __syncwarp();
        }
      } else if (p.staged && (p.epi == GEMM_EPI_F32 || p.epi == GEMM_EPI_F32_RESID ||
                              p.epi == GEMM_EPI_F32_ACCUM)) {
        float* stg = reinterpret_cast<float*>(smem + OFF_EPI) + ew * 32 * EPI_LD;
        const int rbase = row0 + int(rank) * BM + ew * 32;  // this warp's first row
#pragma unroll 1
        for (int ch = 0; ch < BNP / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld32(tbase + ch * 32, v);
          ptx::tmem_wait_ld();
          const int col0 = nb * BNP + ch * 32;
          if (col0 >= p.N) continue;  // warp-uniform
          // the residual / accumulated values this lane adds (4 rows x 128 B
          // per warp instruction), all 8 loads in flight before the staging
          const int c4 = (lane & 7) * 4, col = col0 + c4;
          float4 rv[8];
          bool okr[8];
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int r = rbase + it * 4 + (lane >> 3);
            okr[it] = (p.groups ? (r - p.g_start[g]) < p.g_rows[g] : r < p.M) && col < p.N;
            rv[it] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (okr[it] && p.epi != GEMM_EPI_F32)
              rv[it] = *reinterpret_cast<const float4*>(
                  p.epi == GEMM_EPI_F32_RESID ? p.R + int64_t(r) * p.ldr + col
                                              : reinterpret_cast<const float*>(p.D) + int64_t(r) * p.ldd + col);
          }
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]) * p.scale;
          if (p.bias) epi::add_bias32(f, p.bias + col0);
          // this thread's row into the staging block ...
#pragma unroll
          for (int q = 0; q < 8; ++q)
            *reinterpret_cast<float4*>(stg + lane * EPI_LD + 4 * q) =
                make_float4(f[4 * q], f[4 * q + 1], f[4 * q + 2], f[4 * q + 3]);
          __syncwarp();
          // ... and out four rows per instruction (8 lanes x 16 B per row)
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            if (!okr[it]) continue;
            const int rr = it * 4 + (lane >> 3);
            float4 o = *reinterpret_cast<const float4*>(stg + rr * EPI_LD + c4);
            o.x += rv[it].x;
            o.y += rv[it].y;
            o.z += rv[it].z;
            o.w += rv[it].w;
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(p.D) + int64_t(rbase + rr) * p.ldd + col) = o;
          }
          __syncwarp();
        }
      } else {
#pragma unroll 1
        for (int ch = 0; ch < BNP / 32; ++ch) {
          uint32_t v[32];
          ptx::tmem_ld32(tbase + ch * 32, v);
          ptx::tmem_wait_ld();
          const int col0 = nb * BNP + ch * 32;
          if (!row_ok || col0 >= p.N) continue;
          float f[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) f[i] = __uint_as_float(v[i]) * p.scale;
          if (p.bias) epi::add_bias32(f, p.bias + col0);
          const bool full_chunk = col0 + 32 <= p.N;
          if (p.epi == GEMM_EPI_BF16) {
            __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(p.D) + int64_t(row) * p.ldd + col0;
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
            float* d = reinterpret_cast<float*>(p.D) + int64_t(row) * p.ldd + col0;
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
      ptx::mbar_arrive_cluster(tempty_leader[acc]);
    }
  }

  ptx::tc_fence_before();
  ptx::cluster_sync();
  ptx::tc_fence_after();
  if (warp == 2) ptx::tmem_dealloc_pair(tmem_base, 512);
}

template <bool A_MN, bool B_MN>
cudaError_t launch2(const CUtensorMap& a, const CUtensorMap& b, const P2& p, int grid,
                    cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc2_kernel<A_MN, B_MN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  ++g_kernel_launches;
  gemm_tc2_kernel<A_MN, B_MN><<<grid, THREADS, SMEM, s>>>(a, b, p);
  return cudaGetLastError();
}

}  // namespace

// Pool of zeroed ticket counters (per device).  Each launch takes the next
// slot; kernels leave their slot at 0, so a slot is reusable once its previous
// launch has finished.  An event recorded after every launch orders the reuse:
// the launch that takes a slot again first waits for that event on its own
// stream, so more than kSlots launches in flight (no host sync, several
// streams) can never share a live counter.
static cudaError_t ticket_acquire(cudaStream_t s, int** ctr, cudaEvent_t* done) {
  constexpr int kSlots = 1024;
  static int* pool[64] = {};
  static cudaEvent_t* evs[64] = {};
  static bool used[64][kSlots] = {};
  static int next[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
  if (!pool[dev]) {
    cudaError_t e = cudaMalloc(&pool[dev], kSlots * sizeof(int));
    if (e != cudaSuccess) return e;
    if ((e = cudaMemset(pool[dev], 0, kSlots * sizeof(int))) != cudaSuccess) return e;
    evs[dev] = new cudaEvent_t[kSlots];
    for (int i = 0; i < kSlots; ++i)
      if ((e = cudaEventCreateWithFlags(&evs[dev][i], cudaEventDisableTiming)) != cudaSuccess)
        return e;
  }
  const int i = next[dev]++ % kSlots;
  if (used[dev][i]) {
    cudaError_t e = cudaStreamWaitEvent(s, evs[dev][i], 0);
    if (e != cudaSuccess) return e;
  }
  used[dev][i] = true;
  *ctr = pool[dev] + i;
  *done = evs[dev][i];
  return cudaSuccess;
}

cudaError_t gemm2_run(const GemmDesc& g, int band, cudaStream_t s) {
  const bool gm = g.groups > 0;
  if (gm && (g.grouped_k || g.a_mn)) return cudaErrorNotSupported;
  CUtensorMap ma, mb;
  const uint64_t a_rows = gm ? uint64_t(g.rows_total) : uint64_t(g.M);
  bool ok = !g.a_mn ? gemm_make_map(&ma, g.A, uint64_t(g.K), a_rows, g.lda, BK, BM)
                    : gemm_make_map(&ma, g.A, uint64_t(g.M), uint64_t(g.K), g.lda, 64, BK);
  const uint64_t nst = gm ? uint64_t(g.groups) : 1;
  ok = ok && (!g.b_mn ? gemm_make_map(&mb, g.B, uint64_t(g.K), nst * uint64_t(g.N), g.ldb, BK, BNC)
                      : gemm_make_map(&mb, g.B, uint64_t(g.N), nst * uint64_t(g.K), g.ldb, 64, BK));
  if (!ok) return cudaErrorInvalidValue;
  P2 p;
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.epi = g.epi;
  p.band = band < 1 ? 1 : band;
  p.D = g.D;
  p.ldd = g.ldd;
  p.R = g.R;
  p.ldr = g.ldr;
  p.D2 = g.D2;
  p.ldd2 = g.ldd2;
  p.G2 = g.G2;
  p.ldg2 = g.ldg2;
  p.scale = g.scale == 0.f ? 1.f : g.scale;
  p.bias = g.bias;
  {
    static const int staged = getenv("OPX_GEMM_EPI_STAGED") ? atoi(getenv("OPX_GEMM_EPI_STAGED")) : 1;
    p.staged = staged;
  }
  cudaEvent_t slot_done = nullptr;
  {
    cudaError_t e = ticket_acquire(s, &p.ctr, &slot_done);
    if (e != cudaSuccess) return e;
  }
  p.groups = g.groups;
  p.g_start = g.g_start;
  p.g_rows = g.g_rows;
  if (g.epi == GEMM_EPI_SEQ2HEAD) {
    if (!g.s2h || gm) return cudaErrorInvalidValue;
    p.s2h = *g.s2h;
  }
  // grouped: the tile count lives in device memory; idle clusters exit at once
  const int tiles = gm ? num_sms() / 2 : ((g.M + 2 * BM - 1) / (2 * BM)) * ((g.N + BNP - 1) / BNP);
  int clusters = num_sms() / 2;
  if (tiles < clusters) clusters = tiles;
  const int grid = 2 * (clusters < 1 ? 1 : clusters);
  cudaError_t e;
  if (!g.a_mn && !g.b_mn) e = launch2<false, false>(ma, mb, p, grid, s);
  else if (!g.a_mn && g.b_mn) e = launch2<false, true>(ma, mb, p, grid, s);
  else if (g.a_mn && !g.b_mn) e = launch2<true, false>(ma, mb, p, grid, s);
  else e = launch2<true, true>(ma, mb, p, grid, s);
  if (e != cudaSuccess) return e;
  return cudaEventRecord(slot_done, s);
}

}  // namespace opx
