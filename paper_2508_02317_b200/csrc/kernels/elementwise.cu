// HBM-bound kernels of the training step: deterministic weight init, RMSNorm
// fwd/bwd, embedding gather/scatter, fused softmax-cross-entropy fwd+bwd,
// SwiGLU backward, fused AdamW, and small casts/reductions.  All are
// vectorised (16 B per thread per access) and grid-strided.
#include <algorithm>
#include <cstdint>
#include <cuda_bf16.h>

#include "../runtime/kernels_api.h"
#include "ptx.cuh"

namespace opx {
namespace {

using bf16 = __nv_bfloat16;

// ---------------------------------------------------------------------------
// Deterministic init.  Element i of a parameter with key K:
//   z_j = splitmix64(K + (2i+j) * 0xD1B54A32D192ED03), j = 0,1
//   four 24-bit draws u = z0>>40, (z0>>8)&M, z1>>40, (z1>>8)&M
//   w = fp32( double(sum(u) - 2^25) * c ),  c = std*sqrt(3)/2^24 (host-computed)
// (Irwin-Hall(4) normal approximation; exact in integer + one correctly
// rounded double multiply, so the numpy oracle reproduces it bit-for-bit.)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  uint64_t z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__device__ __forceinline__ float init_value(uint64_t key, uint64_t i, double c) {
  const uint64_t z0 = splitmix64(key + (2 * i) * 0xD1B54A32D192ED03ull);
  const uint64_t z1 = splitmix64(key + (2 * i + 1) * 0xD1B54A32D192ED03ull);
  const int64_t s = int64_t(z0 >> 40) + int64_t((z0 >> 8) & 0xFFFFFF) + int64_t(z1 >> 40) +
                    int64_t((z1 >> 8) & 0xFFFFFF) - (int64_t(1) << 25);
  return __double2float_rn(double(s) * c);
}

// Fills dst_f32[j] (and dst_bf16[j]) for physical elements j in [0, n) of a
// parameter slice whose first physical element is `phys0`.  `interleave` maps
// a [2F, H] gate|up matrix stored in 128-row interleaved blocks to the two
// logical [F, H] matrices with keys key_a (gate) and key_b (up); `experts`
// repeats that per expert slab of 2F rows.
__global__ void init_kernel(float* __restrict__ dst_f32, bf16* __restrict__ dst_bf16, int64_t n,
                            int64_t phys0, uint64_t key_a, uint64_t key_b, double c, float constant,
                            int interleave, int64_t rows_per_slab, int64_t cols) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n;
       j += int64_t(gridDim.x) * blockDim.x) {
    float w;
    if (c == 0.0) {
      w = constant;
    } else if (!interleave) {
      w = init_value(key_a, uint64_t(phys0 + j), c);
    } else {
      const int64_t p = phys0 + j;
      const int64_t row = p / cols, col = p % cols;
      const int64_t slab = row / rows_per_slab, r = row % rows_per_slab;  // rows_per_slab = 2F
      const int64_t blk = r / 256, rr = r % 256;
      const int64_t F = rows_per_slab / 2;
      const bool up = rr >= 128;
      const int64_t lrow = blk * 128 + (up ? rr - 128 : rr);
      const uint64_t li = uint64_t((slab * F + lrow) * cols + col);
      w = init_value(up ? key_b : key_a, li, c);
    }
    if (dst_f32) dst_f32[j] = w;
    if (dst_bf16) dst_bf16[j] = __float2bfloat16_rn(w);
  }
}

// ---------------------------------------------------------------------------
// RMSNorm: y = bf16(x * rsqrt(mean(x^2) + eps) * w), x fp32 residual stream.
// One 256-thread block per row; each thread keeps <= 8 float4 of the row.
// ---------------------------------------------------------------------------
constexpr int NT = 256;
constexpr int MAXV = 8;  // H <= 8192

__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x / 32, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) s += red[i];
  return s;
}

__global__ void __launch_bounds__(NT) rmsnorm_fwd_kernel(const float* __restrict__ x,
                                                         const bf16* __restrict__ w,
                                                         bf16* __restrict__ y,
                                                         float* __restrict__ rstd_out, int H,
                                                         float eps) {
  __shared__ float red[NT / 32];
  const int64_t row = blockIdx.x;
  const float4* xr = reinterpret_cast<const float4*>(x + row * H);
  const int nv = H / 4;
  float4 v[MAXV];
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int idx = threadIdx.x + i * NT;
    if (idx < nv) {
      v[i] = xr[idx];
      ss += v[i].x * v[i].x + v[i].y * v[i].y + v[i].z * v[i].z + v[i].w * v[i].w;
    }
  }
  const float tot = block_sum(ss, red);
  const float rs = rsqrtf(tot / float(H) + eps);
  if (threadIdx.x == 0 && rstd_out) rstd_out[row] = rs;
  uint2* yr = reinterpret_cast<uint2*>(y + row * H);
  const uint2* wr = reinterpret_cast<const uint2*>(w);
#pragma unroll
  for (int i = 0; i < MAXV; ++i) {
    const int idx = threadIdx.x + i * NT;
    if (idx < nv) {
      const uint2 wv = wr[idx];
      const float2 w01 = ptx::unpack_bf16(wv.x), w23 = ptx::unpack_bf16(wv.y);
      uint2 o;
      o.x = ptx::pack_bf16(v[i].x * rs * w01.x, v[i].y * rs * w01.y);
      o.y = ptx::pack_bf16(v[i].z * rs * w23.x, v[i].w * rs * w23.y);
      yr[idx] = o;
    }
  }
}

// dx_out = dres + rstd * (g - xhat * mean(g * xhat)),  g = dy * w,  xhat = x * rstd
// dw partial over the block's rows -> dw_part[blockIdx.x, H]
// V = float4s per thread (H <= NT*4*V), so registers scale with H; the next
// row's x/dy loads are issued before the current row's block reduction, which
// keeps HBM busy across the __syncthreads (the kernel was latency bound).
constexpr int BWD_ROWS = 16;
template <int V>
__global__ void __launch_bounds__(NT) rmsnorm_bwd_kernel(
    const float* __restrict__ dy, const float* __restrict__ x, const bf16* __restrict__ w,
    const float* __restrict__ rstd, const float* dres, float* dx_out,
    float* __restrict__ dw_part, int T, int H) {
  __shared__ float red[2][NT / 32];
  const int nv = H / 4;
  float4 dwacc[V], wv[V], xn[V], dn[V];
  const uint2* wr = reinterpret_cast<const uint2*>(w);
  const int r0 = blockIdx.x * BWD_ROWS;
  const int rows = min(BWD_ROWS, T - r0);
  auto load = [&](int64_t row) {
    const float4* xr = reinterpret_cast<const float4*>(x + row * H);
    const float4* gr = reinterpret_cast<const float4*>(dy + row * H);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int idx = threadIdx.x + i * NT;
      if (idx < nv) {
        xn[i] = xr[idx];
        dn[i] = gr[idx];
      }
    }
  };
#pragma unroll
  for (int i = 0; i < V; ++i) {
    dwacc[i] = make_float4(0, 0, 0, 0);
    const int idx = threadIdx.x + i * NT;
    if (idx < nv) {
      const uint2 q = wr[idx];
      const float2 a = ptx::unpack_bf16(q.x), b = ptx::unpack_bf16(q.y);
      wv[i] = make_float4(a.x, a.y, b.x, b.y);
    }
  }
  if (rows > 0) load(r0);
  for (int rr = 0; rr < rows; ++rr) {
    const int64_t row = r0 + rr;
    const float rs = rstd[row];
    float4 xh[V], g[V];
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int idx = threadIdx.x + i * NT;
      if (idx < nv) {
        const float4 xv = xn[i], dv = dn[i];
        xh[i] = make_float4(xv.x * rs, xv.y * rs, xv.z * rs, xv.w * rs);
        g[i] = make_float4(dv.x * wv[i].x, dv.y * wv[i].y, dv.z * wv[i].z, dv.w * wv[i].w);
        dot += g[i].x * xh[i].x + g[i].y * xh[i].y + g[i].z * xh[i].z + g[i].w * xh[i].w;
        dwacc[i].x += dv.x * xh[i].x;
        dwacc[i].y += dv.y * xh[i].y;
        dwacc[i].z += dv.z * xh[i].z;
        dwacc[i].w += dv.w * xh[i].w;
      }
    }
    if (rr + 1 < rows) load(row + 1);  // in flight during the reduction
    // block reduction (double-buffered scratch: one barrier per row)
#pragma unroll
    for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if ((threadIdx.x & 31) == 0) red[rr & 1][threadIdx.x / 32] = dot;
    __syncthreads();
    float tot = 0.f;
#pragma unroll
    for (int i = 0; i < NT / 32; ++i) tot += red[rr & 1][i];
    const float mean = tot / float(H);
    const float4* rr4 = dres ? reinterpret_cast<const float4*>(dres + row * H) : nullptr;
    float4* o4 = reinterpret_cast<float4*>(dx_out + row * H);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      const int idx = threadIdx.x + i * NT;
      if (idx < nv) {
        float4 o = make_float4(rs * (g[i].x - xh[i].x * mean), rs * (g[i].y - xh[i].y * mean),
                               rs * (g[i].z - xh[i].z * mean), rs * (g[i].w - xh[i].w * mean));
        if (rr4) {
          const float4 r = rr4[idx];
          o.x += r.x;
          o.y += r.y;
          o.z += r.z;
          o.w += r.w;
        }
        o4[idx] = o;
      }
    }
  }
  float4* dp = reinterpret_cast<float4*>(dw_part + int64_t(blockIdx.x) * H);
#pragma unroll
  for (int i = 0; i < V; ++i) {
    const int idx = threadIdx.x + i * NT;
    if (idx < nv) dp[idx] = dwacc[i];
  }
}

// out[c] (+)= sum_r part[r, c].  Block = 32 columns x 16 row groups: each
// thread sums every 16th row in order (4 interleaved accumulators), then the
// 16 group sums are added in order, so the result is deterministic.  (One
// thread per column walking all rows was latency-bound: 28 CTAs, ~0.2 TB/s.)
constexpr int CS_COLS = 32, CS_GROUPS = 16;
__global__ void __launch_bounds__(CS_COLS * CS_GROUPS) colsum_kernel(
    const float* __restrict__ part, int rows, int cols, void* __restrict__ out, int accumulate,
    int out_bf16) {
  __shared__ float red[CS_GROUPS][CS_COLS + 1];
  const int cx = threadIdx.x % CS_COLS, ry = threadIdx.x / CS_COLS;
  const int c = blockIdx.x * CS_COLS + cx;
  float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
  if (c < cols) {
    int r = ry;
    for (; r + 3 * CS_GROUPS < rows; r += 4 * CS_GROUPS) {
      a0 += part[int64_t(r) * cols + c];
      a1 += part[int64_t(r + CS_GROUPS) * cols + c];
      a2 += part[int64_t(r + 2 * CS_GROUPS) * cols + c];
      a3 += part[int64_t(r + 3 * CS_GROUPS) * cols + c];
    }
    for (; r < rows; r += CS_GROUPS) a0 += part[int64_t(r) * cols + c];
  }
  red[ry][cx] = (a0 + a1) + (a2 + a3);
  __syncthreads();
  if (ry != 0 || c >= cols) return;
  float s = 0.f;
#pragma unroll
  for (int g = 0; g < CS_GROUPS; ++g) s += red[g][cx];
  if (out_bf16) {
    bf16* o = static_cast<bf16*>(out);
    o[c] = __float2bfloat16(accumulate ? __bfloat162float(o[c]) + s : s);
  } else {
    float* o = static_cast<float*>(out);
    o[c] = accumulate ? o[c] + s : s;
  }
}

// ---------------------------------------------------------------------------
// Embedding
// ---------------------------------------------------------------------------
__global__ void embed_fwd_kernel(const int* __restrict__ ids, const bf16* __restrict__ E,
                                 float* __restrict__ x, int T, int H) {
  const int64_t row = blockIdx.x;
  const int id = ids[row];
  const uint4* src = reinterpret_cast<const uint4*>(E + int64_t(id) * H);
  float4* dst = reinterpret_cast<float4*>(x + row * H);
  for (int i = threadIdx.x; i < H / 8; i += blockDim.x) {
    const uint4 q = src[i];
    const float2 a = ptx::unpack_bf16(q.x), b = ptx::unpack_bf16(q.y), c = ptx::unpack_bf16(q.z),
                 d = ptx::unpack_bf16(q.w);
    dst[2 * i] = make_float4(a.x, a.y, b.x, b.y);
    dst[2 * i + 1] = make_float4(c.x, c.y, d.x, d.y);
  }
}

__global__ void embed_bwd_kernel(const int* __restrict__ ids, const float* __restrict__ dx,
                                 float* __restrict__ dE, int T, int H) {
  const int64_t row = blockIdx.x;
  const int id = ids[row];
  const float4* src = reinterpret_cast<const float4*>(dx + row * H);
  float* dst = dE + int64_t(id) * H;
  for (int i = threadIdx.x; i < H / 4; i += blockDim.x) {
    const float4 v = src[i];
    atomicAdd(reinterpret_cast<float4*>(dst) + i, v);
  }
}

// ---------------------------------------------------------------------------
// Softmax cross-entropy, fwd+bwd fused, in place on bf16 logits [T, V]:
//   loss[t] = logsumexp(z_t) - z_t[label_t]            (0 for label < 0)
//   z_t    <- (softmax(z_t) - onehot(label_t)) * inv_n  (0 row for label < 0)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(NT) ce_kernel(bf16* __restrict__ logits, int64_t ldl,
                                                const int* __restrict__ labels,
                                                float* __restrict__ loss, int V, float inv_n) {
  __shared__ float red[NT / 32];
  __shared__ float sh_m[NT / 32];
  const int64_t row = blockIdx.x;
  const int label = labels[row];
  bf16* z = logits + row * ldl;
  uint4* z8 = reinterpret_cast<uint4*>(z);
  const int nv = V / 8;
  if (label < 0) {
    for (int i = threadIdx.x; i < nv; i += NT) z8[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x == 0) loss[row] = 0.f;
    return;
  }
  // pass 1: running max / sum per thread
  float m = -INFINITY, s = 0.f;
  for (int i = threadIdx.x; i < nv; i += NT) {
    const uint4 q = z8[i];
    const uint32_t u[4] = {q.x, q.y, q.z, q.w};
    float f[8];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 t = ptx::unpack_bf16(u[e]);
      f[2 * e] = t.x;
      f[2 * e + 1] = t.y;
    }
    float lm = f[0];
#pragma unroll
    for (int e = 1; e < 8; ++e) lm = fmaxf(lm, f[e]);
    const float nm = fmaxf(m, lm);
    s *= __expf(m - nm);
#pragma unroll
    for (int e = 0; e < 8; ++e) s += __expf(f[e] - nm);
    m = nm;
  }
  // block reduce (max then rescaled sum)
  float wm = m;
#pragma unroll
  for (int o = 16; o; o >>= 1) wm = fmaxf(wm, __shfl_xor_sync(0xffffffffu, wm, o));
  const int w = threadIdx.x / 32, l = threadIdx.x & 31;
  if (l == 0) sh_m[w] = wm;
  __syncthreads();
  float gm = sh_m[0];
#pragma unroll
  for (int i = 1; i < NT / 32; ++i) gm = fmaxf(gm, sh_m[i]);
  const float tot = block_sum(s * __expf(m - gm), red);
  const float lse = gm + __logf(tot);
  if (threadIdx.x == 0) loss[row] = lse - __bfloat162float(z[label]);
  __syncthreads();  // everyone read z[label] region before overwrite
  for (int i = threadIdx.x; i < nv; i += NT) {
    const uint4 q = z8[i];
    const uint32_t u[4] = {q.x, q.y, q.z, q.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 t = ptx::unpack_bf16(u[e]);
      const int c0 = i * 8 + 2 * e;
      float g0 = __expf(t.x - lse) - (c0 == label ? 1.f : 0.f);
      float g1 = __expf(t.y - lse) - (c0 + 1 == label ? 1.f : 0.f);
      o[e] = ptx::pack_bf16(g0 * inv_n, g1 * inv_n);
    }
    z8[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

// ---------------------------------------------------------------------------
// SwiGLU backward on 128-column interleaved gate|up:
//   act = silu(g) * u ;  dg = da * u * silu'(g) ;  du = da * silu(g)
// ---------------------------------------------------------------------------
// 2-D launch: x over 16-B column chunks of one row, y over rows, so no 64-bit
// index division per element (it made the kernel instruction-bound);
// sigmoid by the MUFU reciprocal (no IEEE-division slow path).
__global__ void __launch_bounds__(NT) swiglu_bwd_kernel(const bf16* __restrict__ dact,
                                                        const bf16* __restrict__ gu,
                                                        bf16* __restrict__ dgu, int T, int F) {
  const int n8 = F / 8;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n8) return;
  const int f = c * 8;
  const int gcol = (f / 128) * 256 + f % 128;
  for (int row = blockIdx.y * blockDim.y + threadIdx.y; row < T; row += gridDim.y * blockDim.y) {
    const bf16* dr = dact + int64_t(row) * F;
    const bf16* gr = gu + int64_t(row) * 2 * F;
    bf16* orow = dgu + int64_t(row) * 2 * F;
    const uint4 da = *reinterpret_cast<const uint4*>(dr + f);
    const uint4 gq = *reinterpret_cast<const uint4*>(gr + gcol);
    const uint4 uq = *reinterpret_cast<const uint4*>(gr + gcol + 128);
    const uint32_t a[4] = {da.x, da.y, da.z, da.w}, g[4] = {gq.x, gq.y, gq.z, gq.w},
                   u[4] = {uq.x, uq.y, uq.z, uq.w};
    uint32_t og[4], ou[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 av = ptx::unpack_bf16(a[e]), gv = ptx::unpack_bf16(g[e]),
                   uv = ptx::unpack_bf16(u[e]);
      float dg[2], du[2];
      const float gg[2] = {gv.x, gv.y}, uu[2] = {uv.x, uv.y}, aa[2] = {av.x, av.y};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float sg = __fdividef(1.f, 1.f + __expf(-gg[k]));
        const float si = gg[k] * sg;
        du[k] = aa[k] * si;
        dg[k] = aa[k] * uu[k] * sg * (1.f + gg[k] * (1.f - sg));
      }
      og[e] = ptx::pack_bf16(dg[0], dg[1]);
      ou[e] = ptx::pack_bf16(du[0], du[1]);
    }
    *reinterpret_cast<uint4*>(orow + gcol) = make_uint4(og[0], og[1], og[2], og[3]);
    *reinterpret_cast<uint4*>(orow + gcol + 128) = make_uint4(ou[0], ou[1], ou[2], ou[3]);
  }
}

// ---------------------------------------------------------------------------
// AdamW (torch.optim.AdamW semantics), fp32 master/m/v/grad, bf16 param copy.
// ---------------------------------------------------------------------------
template <typename G>
__global__ void adamw_kernel(float* __restrict__ p, float* __restrict__ m, float* __restrict__ v,
                             const G* __restrict__ g, bf16* __restrict__ pb, int64_t n,
                             float lr, float b1, float b2, float eps, float wd, float bc1,
                             float bc2_sqrt) {
  const int64_t n4 = n / 4;
  const float step = lr / bc1;
  const float decay = 1.f - lr * wd;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    float4 pv = reinterpret_cast<float4*>(p)[i];
    float4 mv = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    float4 gv;
    if constexpr (sizeof(G) == 4) {
      gv = reinterpret_cast<const float4*>(g)[i];
    } else {  // bf16 gradients (layer / expert units)
      const uint2 q = reinterpret_cast<const uint2*>(g)[i];
      const float2 a = ptx::unpack_bf16(q.x), b = ptx::unpack_bf16(q.y);
      gv = make_float4(a.x, a.y, b.x, b.y);
    }
    float* pp = &pv.x;
    float* mp = &mv.x;
    float* vp = &vv.x;
    const float* gp = &gv.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      pp[e] *= decay;
      mp[e] = mp[e] + (gp[e] - mp[e]) * (1.f - b1);
      vp[e] = vp[e] * b2 + (1.f - b2) * gp[e] * gp[e];
      const float denom = sqrtf(vp[e]) / bc2_sqrt + eps;
      pp[e] -= step * mp[e] / denom;
    }
    reinterpret_cast<float4*>(p)[i] = pv;
    reinterpret_cast<float4*>(m)[i] = mv;
    reinterpret_cast<float4*>(v)[i] = vv;
    uint2 o;
    o.x = ptx::pack_bf16(pv.x, pv.y);
    o.y = ptx::pack_bf16(pv.z, pv.w);
    reinterpret_cast<uint2*>(pb)[i] = o;
  }
}

__global__ void cast_f32_bf16_kernel(const float* __restrict__ x, bf16* __restrict__ y, int64_t n) {
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(x)[i];
    uint2 o;
    o.x = ptx::pack_bf16(v.x, v.y);
    o.y = ptx::pack_bf16(v.z, v.w);
    reinterpret_cast<uint2*>(y)[i] = o;
  }
}

// gradient accumulation over micro-batches (step_graph.cpp:57,75-87): acc =
// (first ? 0 : acc) + g in fp32, g the micro-batch's fp32 or bf16 shard gradient
template <typename G>
__global__ void grad_accum_kernel(float* __restrict__ acc, const G* __restrict__ g, int64_t n,
                                  int first) {
  const int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4;
       i += int64_t(gridDim.x) * blockDim.x) {
    float4 gv;
    if constexpr (sizeof(G) == 4) {
      gv = reinterpret_cast<const float4*>(g)[i];
    } else {
      const uint2 q = reinterpret_cast<const uint2*>(g)[i];
      const float2 a = ptx::unpack_bf16(q.x), b = ptx::unpack_bf16(q.y);
      gv = make_float4(a.x, a.y, b.x, b.y);
    }
    if (!first) {
      const float4 av = reinterpret_cast<const float4*>(acc)[i];
      gv.x += av.x;
      gv.y += av.y;
      gv.z += av.z;
      gv.w += av.w;
    }
    reinterpret_cast<float4*>(acc)[i] = gv;
  }
}

// sum of a float vector (fixed order, one block) -> out[0]
__global__ void sum_kernel(const float* __restrict__ x, int64_t n, float* out) {
  __shared__ float red[NT / 32];
  float s = 0.f;
  for (int64_t i = threadIdx.x; i < n; i += NT) s += x[i];
  s = block_sum(s, red);
  if (threadIdx.x == 0) out[0] = s;
}

int grid_for(int64_t n, int per_thread = 1) {
  int64_t b = (n / per_thread + NT - 1) / NT;
  const int cap = num_sms() * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : int(b);
}

}  // namespace

cudaError_t k_init_param(float* f32, __nv_bfloat16* b16, int64_t n, int64_t phys0, uint64_t key_a,
                         uint64_t key_b, double c, float constant, int interleave,
                         int64_t rows_per_slab, int64_t cols, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  ++g_kernel_launches;
  init_kernel<<<grid_for(n), NT, 0, s>>>(f32, b16, n, phys0, key_a, key_b, c, constant,
                                         interleave, rows_per_slab, cols);
  return cudaGetLastError();
}

cudaError_t k_rmsnorm_fwd(const float* x, const __nv_bfloat16* w, __nv_bfloat16* y, float* rstd,
                          int T, int H, float eps, cudaStream_t s) {
  if (H % 4 || H > NT * 4 * MAXV) return cudaErrorInvalidValue;
  if (T <= 0) return cudaSuccess;
  ++g_kernel_launches;
  rmsnorm_fwd_kernel<<<T, NT, 0, s>>>(x, w, y, rstd, H, eps);
  return cudaGetLastError();
}

int k_rmsnorm_bwd_parts(int T) { return (T + BWD_ROWS - 1) / BWD_ROWS; }

cudaError_t k_rmsnorm_bwd(const float* dy, const float* x, const __nv_bfloat16* w,
                          const float* rstd, const float* dres, float* dx, float* dw_part,
                          void* dw, int accumulate_dw, int T, int H, cudaStream_t s, int dw_bf16) {
  if (H % 4 || H > NT * 4 * MAXV) return cudaErrorInvalidValue;
  if (T <= 0) return cudaSuccess;
  const int nb = k_rmsnorm_bwd_parts(T);
  ++g_kernel_launches;
  if (H <= NT * 4)
    rmsnorm_bwd_kernel<1><<<nb, NT, 0, s>>>(dy, x, w, rstd, dres, dx, dw_part, T, H);
  else if (H <= NT * 8)
    rmsnorm_bwd_kernel<2><<<nb, NT, 0, s>>>(dy, x, w, rstd, dres, dx, dw_part, T, H);
  else if (H <= NT * 16)
    rmsnorm_bwd_kernel<4><<<nb, NT, 0, s>>>(dy, x, w, rstd, dres, dx, dw_part, T, H);
  else
    rmsnorm_bwd_kernel<8><<<nb, NT, 0, s>>>(dy, x, w, rstd, dres, dx, dw_part, T, H);
  ++g_kernel_launches;
  colsum_kernel<<<(H + CS_COLS - 1) / CS_COLS, CS_COLS * CS_GROUPS, 0, s>>>(dw_part, nb, H, dw,
                                                                           accumulate_dw, dw_bf16);
  return cudaGetLastError();
}

cudaError_t k_embed_fwd(const int* ids, const __nv_bfloat16* E, float* x, int T, int H,
                        cudaStream_t s) {
  if (H % 8) return cudaErrorInvalidValue;
  if (T <= 0) return cudaSuccess;
  ++g_kernel_launches;
  embed_fwd_kernel<<<T, 128, 0, s>>>(ids, E, x, T, H);
  return cudaGetLastError();
}

cudaError_t k_embed_bwd(const int* ids, const float* dx, float* dE, int T, int H, cudaStream_t s) {
  if (H % 4) return cudaErrorInvalidValue;
  if (T <= 0) return cudaSuccess;
  ++g_kernel_launches;
  embed_bwd_kernel<<<T, 128, 0, s>>>(ids, dx, dE, T, H);
  return cudaGetLastError();
}

cudaError_t k_ce_fwd_bwd(__nv_bfloat16* logits, int64_t ldl, const int* labels, float* loss, int T,
                         int V, float inv_n, cudaStream_t s) {
  if (V % 8 || ldl % 8) return cudaErrorInvalidValue;
  if (T <= 0) return cudaSuccess;
  ++g_kernel_launches;
  ce_kernel<<<T, NT, 0, s>>>(logits, ldl, labels, loss, V, inv_n);
  return cudaGetLastError();
}

cudaError_t k_swiglu_bwd(const __nv_bfloat16* dact, const __nv_bfloat16* gu, __nv_bfloat16* dgu,
                         int64_t T, int F, cudaStream_t s) {
  if (F % 128) return cudaErrorInvalidValue;
  if (T <= 0) return cudaSuccess;
  ++g_kernel_launches;
  if (T > INT32_MAX) return cudaErrorInvalidValue;
  // block = bx column chunks x (NT / bx) rows, bx the widest that wastes <= 1/16 of the lanes
  const int n8 = F / 8;
  int bx = 32;
  for (int cand = NT; cand >= 32; cand /= 2)
    if ((n8 + cand - 1) / cand * cand - n8 <= n8 / 16) {
      bx = cand;
      break;
    }
  const dim3 blk(bx, NT / bx);
  const int gx = (n8 + bx - 1) / bx;
  const int64_t gy_need = (T + blk.y - 1) / blk.y;
  const int gy = int(std::min<int64_t>(gy_need, std::max(1, num_sms() * 16 / gx)));
  swiglu_bwd_kernel<<<dim3(gx, gy), blk, 0, s>>>(dact, gu, dgu, int(T), F);
  return cudaGetLastError();
}

cudaError_t k_adamw(float* p, float* m, float* v, const void* g, int g_bf16, __nv_bfloat16* pb,
                    int64_t n, float lr, float b1, float b2, float eps, float wd, int step,
                    cudaStream_t s, int blocks_per_sm) {
  if (n % 4) return cudaErrorInvalidValue;
  if (n <= 0) return cudaSuccess;
  const double bc1 = 1.0 - std::pow(double(b1), step);
  const double bc2 = 1.0 - std::pow(double(b2), step);
  // blocks_per_sm > 0 caps the grid (the optimizer overlapped with the
  // backward must leave thread slots for the compute stream's kernels: eight
  // resident 256-thread blocks per SM would take all 2048 and stall them)
  int grid = grid_for(n / 4);
  if (blocks_per_sm > 0 && grid > num_sms() * blocks_per_sm) grid = num_sms() * blocks_per_sm;
  ++g_kernel_launches;
  if (g_bf16)
    adamw_kernel<bf16><<<grid, NT, 0, s>>>(p, m, v, static_cast<const bf16*>(g), pb, n, lr, b1, b2, eps,
                                           wd, float(bc1), float(std::sqrt(bc2)));
  else
    adamw_kernel<float><<<grid, NT, 0, s>>>(p, m, v, static_cast<const float*>(g), pb, n, lr, b1, b2,
                                            eps, wd, float(bc1), float(std::sqrt(bc2)));
  return cudaGetLastError();
}

cudaError_t k_cast_f32_bf16(const float* x, __nv_bfloat16* y, int64_t n, cudaStream_t s) {
  if (n % 4) return cudaErrorInvalidValue;
  if (n <= 0) return cudaSuccess;
  ++g_kernel_launches;
  cast_f32_bf16_kernel<<<grid_for(n / 4), NT, 0, s>>>(x, y, n);
  return cudaGetLastError();
}

cudaError_t k_grad_accum(float* acc, const void* g, int g_bf16, int64_t n, int first,
                         cudaStream_t s) {
  if (n % 4) return cudaErrorInvalidValue;
  if (n <= 0) return cudaSuccess;
  ++g_kernel_launches;
  if (g_bf16)
    grad_accum_kernel<<<grid_for(n / 4), NT, 0, s>>>(acc, static_cast<const bf16*>(g), n, first);
  else
    grad_accum_kernel<<<grid_for(n / 4), NT, 0, s>>>(acc, static_cast<const float*>(g), n, first);
  return cudaGetLastError();
}

cudaError_t k_sum(const float* x, int64_t n, float* out, cudaStream_t s) {
  ++g_kernel_launches;
  sum_kernel<<<1, NT, 0, s>>>(x, n, out);
  return cudaGetLastError();
}

}  // namespace opx
