// Causal, packed-varlen, GQA flash attention (head_dim 128), fwd + bwd.
//
// Token layout is the Ulysses "head" layout: q [N, hq, 128], k/v [N, hk, 128]
// where N = rows * S tokens of the full sequences and hq/hk are the heads this
// rank owns after the seq->head all-to-all.  Sample isolation comes from
// per-token seq_start/seq_end (derived from cu_seqlens, packing.hpp:20-31):
// key j is visible to query i iff seq_start[i] <= j <= i.
//
// This is the first (parity) implementation on warp-level mma.sync
// (m16n8k16 bf16 -> fp32) with cp.async + XOR-swizzled smem; the tcgen05/TMEM
// version replaces it behind the same AttnArgs interface.
#include <cuda_bf16.h>

#include "../runtime/kernels_api.h"
#include "ptx.cuh"

namespace opx {
namespace {

using bf16 = __nv_bfloat16;
constexpr int D = 128;
constexpr int BQ = 64, BKV = 64;
constexpr float LOG2E = 1.4426950408889634f;

// byte offset of 16-B chunk `c` of row `r` in a [rows][128] bf16 tile (256 B rows)
__device__ __forceinline__ uint32_t swz(int r, int c) { return r * 256 + ((c ^ (r & 7)) << 4); }
// [rows][64] bf16 tile (128 B rows)
__device__ __forceinline__ uint32_t swz64(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(sz)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void ldsm4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                      uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm4t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2,
                                       uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

// Load a [64 rows][128] bf16 tile (rows row0.., stride ld elements) into swizzled smem.
__device__ __forceinline__ void load_tile64(uint32_t sbase, const bf16* g, int64_t ld, int row0,
                                            int nrows) {
  // 64 rows x 16 chunks = 1024 chunks, 128 threads -> 8 each
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int idx = threadIdx.x + i * 128;
    const int r = idx >> 4, c = idx & 15;
    const int gr = row0 + r;
    const bool ok = gr < nrows;
    const bf16* src = g + int64_t(ok ? gr : 0) * ld + c * 8;
    cp_async16(sbase + swz(r, c), src, ok);
  }
}

// A fragment (16 rows x 16 k) from a swizzled [rows][128] tile at (r0, k0).
__device__ __forceinline__ void frag_a(uint32_t sbase, int r0, int k0, uint32_t (&a)[4]) {
  const int l = threadIdx.x & 31;
  const int r = r0 + (l & 7) + ((l >> 3) & 1) * 8;
  const int c = (k0 >> 3) + (l >> 4);
  ldsm4(sbase + swz(r, c), a[0], a[1], a[2], a[3]);
}
// Two B fragments (n-tiles n0, n0+8; k-step k0) from a tile stored [n][k] (non-trans).
__device__ __forceinline__ void frag_b_nk(uint32_t sbase, int n0, int k0, uint32_t& b00,
                                          uint32_t& b01, uint32_t& b10, uint32_t& b11) {
  const int l = threadIdx.x & 31;
  // matrices: (n0, k lo) (n0, k hi) (n0+8, k lo) (n0+8, k hi)
  const int r = n0 + (l & 7) + ((l >> 4) << 3);
  const int c = (k0 >> 3) + ((l >> 3) & 1);
  ldsm4(sbase + swz(r, c), b00, b01, b10, b11);
}
// Two B fragments (n-tiles n0, n0+8; k-step k0) from a tile stored [k][n] (trans).
__device__ __forceinline__ void frag_b_kn(uint32_t sbase, int n0, int k0, uint32_t& b00,
                                          uint32_t& b01, uint32_t& b10, uint32_t& b11) {
  const int l = threadIdx.x & 31;
  // matrices: (k lo, n0) (k hi, n0) (k lo, n0+8) (k hi, n0+8)
  const int r = k0 + (l & 7) + ((l >> 3) & 1) * 8;
  const int c = (n0 >> 3) + (l >> 4);
  ldsm4t(sbase + swz(r, c), b00, b01, b10, b11);
}

// ---------------------------------------------------------------------------
// forward
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) attn_fwd_kernel(const AttnArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int q0 = blockIdx.x * BQ;
  const int h = blockIdx.y;
  const int kh = h / (a.hq / a.hk);
  if (q0 >= a.N) return;
  const uint32_t sQ = ptx::smem_u32(smem);
  const uint32_t sK[2] = {sQ + 16384, sQ + 32768};
  const uint32_t sV[2] = {sQ + 49152, sQ + 65536};
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;

  const int qlast = min(q0 + BQ, a.N) - 1;
  const int kbeg = a.seq_start[q0];
  const int kb0 = kbeg & ~(BKV - 1);
  const int nkb = (qlast - kb0) / BKV + 1;

  const bf16* qg = a.q + int64_t(h) * D;
  const bf16* kg = a.k + int64_t(kh) * D;
  const bf16* vg = a.v + int64_t(kh) * D;
  load_tile64(sQ, qg, a.ldq, q0, a.N);
  load_tile64(sK[0], kg, a.ldk, kb0, a.N);
  load_tile64(sV[0], vg, a.ldv, kb0, a.N);
  cp_commit();

  const int ra = q0 + warp * 16 + g, rb = ra + 8;
  const int sa = ra < a.N ? a.seq_start[ra] : 0x7fffffff;
  const int sb = rb < a.N ? a.seq_start[rb] : 0x7fffffff;
  const float sl2 = a.scale * LOG2E;

  float m_a = -INFINITY, m_b = -INFINITY, l_a = 0.f, l_b = 0.f;
  float o[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  uint32_t qf[8][4];

  for (int it = 0; it < nkb; ++it) {
    const int buf = it & 1;
    if (it + 1 < nkb) {
      load_tile64(sK[buf ^ 1], kg, a.ldk, kb0 + (it + 1) * BKV, a.N);
      load_tile64(sV[buf ^ 1], vg, a.ldv, kb0 + (it + 1) * BKV, a.N);
      cp_commit();
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    if (it == 0) {
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) frag_a(sQ, warp * 16, ks * 16, qf[ks]);
    }
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
#pragma unroll
      for (int jp = 0; jp < 4; ++jp) {
        uint32_t b00, b01, b10, b11;
        frag_b_nk(sK[buf], jp * 16, ks * 16, b00, b01, b10, b11);
        mma16816(s[2 * jp], qf[ks], b00, b01);
        mma16816(s[2 * jp + 1], qf[ks], b10, b11);
      }
    }
    const int kbase = kb0 + it * BKV;
    float mx_a = -INFINITY, mx_b = -INFINITY;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int key = kbase + j * 8 + 2 * t + (e & 1);
        const int row = e < 2 ? ra : rb;
        const int st = e < 2 ? sa : sb;
        const bool ok = key >= st && key <= row;
        s[j][e] = ok ? s[j][e] * sl2 : -INFINITY;
      }
      mx_a = fmaxf(mx_a, fmaxf(s[j][0], s[j][1]));
      mx_b = fmaxf(mx_b, fmaxf(s[j][2], s[j][3]));
    }
#pragma unroll
    for (int o2 = 1; o2 < 4; o2 <<= 1) {
      mx_a = fmaxf(mx_a, __shfl_xor_sync(0xffffffffu, mx_a, o2));
      mx_b = fmaxf(mx_b, __shfl_xor_sync(0xffffffffu, mx_b, o2));
    }
    const float mn_a = fmaxf(m_a, mx_a), mn_b = fmaxf(m_b, mx_b);
    const float base_a = mn_a == -INFINITY ? 0.f : mn_a;
    const float base_b = mn_b == -INFINITY ? 0.f : mn_b;
    const float al_a = exp2f(m_a - base_a), al_b = exp2f(m_b - base_b);
    m_a = mn_a;
    m_b = mn_b;
    l_a *= al_a;
    l_b *= al_b;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      o[j][0] *= al_a;
      o[j][1] *= al_a;
      o[j][2] *= al_b;
      o[j][3] *= al_b;
    }
    uint32_t pa[4][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float p0 = exp2f(s[j][0] - base_a), p1 = exp2f(s[j][1] - base_a);
      const float p2 = exp2f(s[j][2] - base_b), p3 = exp2f(s[j][3] - base_b);
      l_a += p0 + p1;
      l_b += p2 + p3;
      const int kk = j >> 1, hi = j & 1;
      pa[kk][hi * 2 + 0] = ptx::pack_bf16(p0, p1);
      pa[kk][hi * 2 + 1] = ptx::pack_bf16(p2, p3);
    }
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int dn = 0; dn < 8; ++dn) {
        uint32_t b00, b01, b10, b11;
        frag_b_kn(sV[buf], dn * 16, kk * 16, b00, b01, b10, b11);
        mma16816(o[2 * dn], pa[kk], b00, b01);
        mma16816(o[2 * dn + 1], pa[kk], b10, b11);
      }
    }
    __syncthreads();
  }
  // finalize
#pragma unroll
  for (int o2 = 1; o2 < 4; o2 <<= 1) {
    l_a += __shfl_xor_sync(0xffffffffu, l_a, o2);
    l_b += __shfl_xor_sync(0xffffffffu, l_b, o2);
  }
  const float ia = l_a > 0.f ? 1.f / l_a : 0.f, ib = l_b > 0.f ? 1.f / l_b : 0.f;
  if (t == 0) {
    if (ra < a.N) a.lse[int64_t(h) * a.N + ra] = (m_a + log2f(l_a)) / LOG2E;
    if (rb < a.N) a.lse[int64_t(h) * a.N + rb] = (m_b + log2f(l_b)) / LOG2E;
  }
  // stage O through smem (reuse sQ) for 16-B coalesced stores
  uint8_t* so = smem;
  const int rla = warp * 16 + g, rlb = rla + 8;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int col = j * 8 + 2 * t;
    *reinterpret_cast<uint32_t*>(so + swz(rla, col >> 3) + (col & 7) * 2) =
        ptx::pack_bf16(o[j][0] * ia, o[j][1] * ia);
    *reinterpret_cast<uint32_t*>(so + swz(rlb, col >> 3) + (col & 7) * 2) =
        ptx::pack_bf16(o[j][2] * ib, o[j][3] * ib);
  }
  __syncthreads();
  bf16* og = a.o + int64_t(h) * D;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int idx = threadIdx.x + i * 128;
    const int r = idx >> 4, c = idx & 15;
    if (q0 + r < a.N)
      *reinterpret_cast<uint4*>(og + int64_t(q0 + r) * a.ldo + c * 8) =
          *reinterpret_cast<const uint4*>(so + swz(r, c));
  }
}

// delta[h, t] = sum_d dO[t,h,d] * O[t,h,d]
__global__ void attn_delta_kernel(const AttnArgs a) {
  const int64_t w = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= int64_t(a.N) * a.hq) return;
  const int tok = int(w / a.hq), h = int(w % a.hq);
  const uint2 x = *reinterpret_cast<const uint2*>(a.dout + int64_t(tok) * a.lddo + h * D + lane * 4);
  const uint2 y = *reinterpret_cast<const uint2*>(a.o + int64_t(tok) * a.ldo + h * D + lane * 4);
  const float2 x0 = ptx::unpack_bf16(x.x), x1 = ptx::unpack_bf16(x.y);
  const float2 y0 = ptx::unpack_bf16(y.x), y1 = ptx::unpack_bf16(y.y);
  float s = x0.x * y0.x + x0.y * y0.y + x1.x * y1.x + x1.y * y1.y;
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) a.delta[int64_t(h) * a.N + tok] = s;
}

// ---------------------------------------------------------------------------
// backward: one block per (64-key tile, kv head); loops over the q heads of
// the GQA group and the q tiles that can see the keys.  dK/dV stay in
// registers; dQ partials go to an fp32 accumulator with red.add.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(128) attn_bwd_kernel(const AttnArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int k0 = blockIdx.x * BKV;
  const int kh = blockIdx.y;
  if (k0 >= a.N) return;
  const int G = a.hq / a.hk;
  const uint32_t sK = ptx::smem_u32(smem);
  const uint32_t sV = sK + 16384;
  const uint32_t sQ = sK + 32768;
  const uint32_t sO = sK + 49152;  // dO tile
  const uint32_t sS = sK + 65536;  // dS^T [64 keys][64 q] bf16
  float* s_lse = reinterpret_cast<float*>(smem + 65536 + 8192);
  float* s_dlt = s_lse + BQ;
  int* s_sst = reinterpret_cast<int*>(s_dlt + BQ);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;

  load_tile64(sK, a.k + int64_t(kh) * D, a.ldk, k0, a.N);
  load_tile64(sV, a.v + int64_t(kh) * D, a.ldv, k0, a.N);
  cp_commit();

  const int klast = min(k0 + BKV, a.N) - 1;
  const int qend = a.seq_end[klast];  // exclusive
  const float sl2 = a.scale * LOG2E;
  const int key_a = k0 + warp * 16 + g, key_b = key_a + 8;  // rows of S^T this thread holds

  float dk[16][4], dv[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j)
#pragma unroll
    for (int e = 0; e < 4; ++e) dk[j][e] = dv[j][e] = 0.f;

  for (int gi = 0; gi < G; ++gi) {
    const int h = kh * G + gi;
    for (int q0 = k0; q0 < qend; q0 += BQ) {
      load_tile64(sQ, a.q + int64_t(h) * D, a.ldq, q0, a.N);
      load_tile64(sO, a.dout + int64_t(h) * D, a.lddo, q0, a.N);
      cp_commit();
      if (threadIdx.x < BQ) {
        const int q = q0 + threadIdx.x;
        const bool ok = q < a.N;
        s_lse[threadIdx.x] = ok ? a.lse[int64_t(h) * a.N + q] * LOG2E : INFINITY;
        s_dlt[threadIdx.x] = ok ? a.delta[int64_t(h) * a.N + q] : 0.f;
        s_sst[threadIdx.x] = ok ? a.seq_start[q] : 0x7fffffff;
      }
      cp_wait<0>();
      __syncthreads();

      // S^T = K Q^T and dP^T = V dO^T  (16 keys x 64 q per warp)
      float st[8][4], dp[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 4; ++e) st[j][e] = dp[j][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t ka[4], va[4];
        frag_a(sK, warp * 16, ks * 16, ka);
        frag_a(sV, warp * 16, ks * 16, va);
#pragma unroll
        for (int jp = 0; jp < 4; ++jp) {
          uint32_t b00, b01, b10, b11;
          frag_b_nk(sQ, jp * 16, ks * 16, b00, b01, b10, b11);
          mma16816(st[2 * jp], ka, b00, b01);
          mma16816(st[2 * jp + 1], ka, b10, b11);
          frag_b_nk(sO, jp * 16, ks * 16, b00, b01, b10, b11);
          mma16816(dp[2 * jp], va, b00, b01);
          mma16816(dp[2 * jp + 1], va, b10, b11);
        }
      }
      // P^T, dS^T
      uint32_t pa[4][4], da[4][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float p[4], ds[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int ql = j * 8 + 2 * t + (e & 1);
          const int q = q0 + ql;
          const int key = e < 2 ? key_a : key_b;
          const bool ok = key <= q && key >= s_sst[ql] && key < a.N;
          p[e] = ok ? exp2f(st[j][e] * sl2 - s_lse[ql]) : 0.f;
          ds[e] = p[e] * (dp[j][e] - s_dlt[ql]);
        }
        const int kk = j >> 1, hi = j & 1;
        pa[kk][hi * 2 + 0] = ptx::pack_bf16(p[0], p[1]);
        pa[kk][hi * 2 + 1] = ptx::pack_bf16(p[2], p[3]);
        da[kk][hi * 2 + 0] = ptx::pack_bf16(ds[0], ds[1]);
        da[kk][hi * 2 + 1] = ptx::pack_bf16(ds[2], ds[3]);
        // dS^T -> smem [key][q]
        const int kra = warp * 16 + g, krb = kra + 8;
        const int col = j * 8 + 2 * t;
        *reinterpret_cast<uint32_t*>(smem + 65536 + swz64(kra, col >> 3) + (col & 7) * 2) =
            da[kk][hi * 2 + 0];
        *reinterpret_cast<uint32_t*>(smem + 65536 + swz64(krb, col >> 3) + (col & 7) * 2) =
            da[kk][hi * 2 + 1];
      }
      // dV += P^T dO ; dK += dS^T Q
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
        for (int dn = 0; dn < 8; ++dn) {
          uint32_t b00, b01, b10, b11;
          frag_b_kn(sO, dn * 16, kk * 16, b00, b01, b10, b11);
          mma16816(dv[2 * dn], pa[kk], b00, b01);
          mma16816(dv[2 * dn + 1], pa[kk], b10, b11);
          frag_b_kn(sQ, dn * 16, kk * 16, b00, b01, b10, b11);
          mma16816(dk[2 * dn], da[kk], b00, b01);
          mma16816(dk[2 * dn + 1], da[kk], b10, b11);
        }
      }
      __syncthreads();  // dS^T complete in smem
      // dQ[q rows 16w..16w+15] = dS (16 q x 64 keys) . K (64 keys x 128), in two d halves
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        float dq[8][4];
#pragma unroll
        for (int j = 0; j < 8; ++j) dq[j][0] = dq[j][1] = dq[j][2] = dq[j][3] = 0.f;
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          // A = dS[q][key] from sdS[key][q] (trans): matrices (q lo,k lo)(q hi,k lo)(q lo,k hi)(q hi,k hi)
          uint32_t af[4];
          {
            const int r = kk * 16 + (lane & 7) + ((lane >> 4) << 3);
            const int c = ((warp * 16) >> 3) + ((lane >> 3) & 1);
            ldsm4t(sS + swz64(r, c), af[0], af[1], af[2], af[3]);
          }
#pragma unroll
          for (int dn = 0; dn < 4; ++dn) {
            uint32_t b00, b01, b10, b11;
            frag_b_kn(sK, half * 64 + dn * 16, kk * 16, b00, b01, b10, b11);
            mma16816(dq[2 * dn], af, b00, b01);
            mma16816(dq[2 * dn + 1], af, b10, b11);
          }
        }
        const int qa = q0 + warp * 16 + g, qb = qa + 8;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int col = half * 64 + j * 8 + 2 * t;
          if (qa < a.N) {
            float* p = a.dq_acc + (int64_t(qa) * a.hq + h) * D + col;
            atomicAdd(p, dq[j][0] * a.scale);
            atomicAdd(p + 1, dq[j][1] * a.scale);
          }
          if (qb < a.N) {
            float* p = a.dq_acc + (int64_t(qb) * a.hq + h) * D + col;
            atomicAdd(p, dq[j][2] * a.scale);
            atomicAdd(p + 1, dq[j][3] * a.scale);
          }
        }
      }
      __syncthreads();
    }
  }
  // write dK (scaled), dV via smem staging (reuse sQ / sO)
  uint8_t* sk = smem + 32768;
  uint8_t* sv = smem + 49152;
  const int rla = warp * 16 + g, rlb = rla + 8;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int col = j * 8 + 2 * t;
    *reinterpret_cast<uint32_t*>(sk + swz(rla, col >> 3) + (col & 7) * 2) =
        ptx::pack_bf16(dk[j][0] * a.scale, dk[j][1] * a.scale);
    *reinterpret_cast<uint32_t*>(sk + swz(rlb, col >> 3) + (col & 7) * 2) =
        ptx::pack_bf16(dk[j][2] * a.scale, dk[j][3] * a.scale);
    *reinterpret_cast<uint32_t*>(sv + swz(rla, col >> 3) + (col & 7) * 2) =
        ptx::pack_bf16(dv[j][0], dv[j][1]);
    *reinterpret_cast<uint32_t*>(sv + swz(rlb, col >> 3) + (col & 7) * 2) =
        ptx::pack_bf16(dv[j][2], dv[j][3]);
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int idx = threadIdx.x + i * 128;
    const int r = idx >> 4, c = idx & 15;
    if (k0 + r < a.N) {
      *reinterpret_cast<uint4*>(a.dk + int64_t(k0 + r) * a.lddk + kh * D + c * 8) =
          *reinterpret_cast<const uint4*>(sk + swz(r, c));
      *reinterpret_cast<uint4*>(a.dv + int64_t(k0 + r) * a.lddv + kh * D + c * 8) =
          *reinterpret_cast<const uint4*>(sv + swz(r, c));
    }
  }
}

constexpr int FWD_SMEM = 16384 * 5;
constexpr int BWD_SMEM = 65536 + 8192 + 3 * BQ * 4;

}  // namespace

cudaError_t k_attn_fwd(const AttnArgs& a, cudaStream_t s) {
  if (a.N <= 0) return cudaSuccess;
  if (a.hq % a.hk) return cudaErrorInvalidValue;
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(attn_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FWD_SMEM);
    cfg = true;
  }
  dim3 grid((a.N + BQ - 1) / BQ, a.hq);
  ++g_kernel_launches;
  attn_fwd_kernel<<<grid, 128, FWD_SMEM, s>>>(a);
  return cudaGetLastError();
}

cudaError_t k_attn_bwd(const AttnArgs& a, cudaStream_t s) {
  if (a.N <= 0) return cudaSuccess;
  if (a.hq % a.hk) return cudaErrorInvalidValue;
  static bool cfg = false;
  if (!cfg) {
    cudaFuncSetAttribute(attn_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_SMEM);
    cfg = true;
  }
  const int64_t warps = int64_t(a.N) * a.hq;
  ++g_kernel_launches;
  attn_delta_kernel<<<int((warps * 32 + 255) / 256), 256, 0, s>>>(a);
  cudaError_t e = cudaMemsetAsync(a.dq_acc, 0, size_t(a.N) * a.hq * D * sizeof(float), s);
  if (e != cudaSuccess) return e;
  dim3 grid((a.N + BKV - 1) / BKV, a.hk);
  ++g_kernel_launches;
  attn_bwd_kernel<<<grid, 128, BWD_SMEM, s>>>(a);
  return cudaGetLastError();
}

}  // namespace opx
