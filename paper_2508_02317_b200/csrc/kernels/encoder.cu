// Frozen omni-modal encoder glue (step_graph.cpp:141-166,
// comm.cpp:91-105): the merger's GELU, the feature scatter into the SP group
// (peer stores straight into the owning rank's feature rows: the reference's
// `scatter.<mod>` all-to-all fused with the masked scatter's addressing), the
// injection of those rows into the text embedding, and the matching zeroing of
// the embedding gradient at the replaced positions.  All HBM-bound row copies:
// 16-B vector accesses, one warp per row.
#include <cuda_bf16.h>

#include "../runtime/kernels_api.h"

namespace opx {
namespace {
using bf16 = __nv_bfloat16;

__global__ void gelu_kernel(bf16* __restrict__ x, int64_t n) {
  for (int64_t i = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) * 8; i < n;
       i += int64_t(gridDim.x) * blockDim.x * 8) {
    uint4 v = *reinterpret_cast<const uint4*>(x + i);
    bf16* e = reinterpret_cast<bf16*>(&v);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float f = __bfloat162float(e[j]);
      e[j] = __float2bfloat16_rn(0.5f * f * (1.f + erff(f * 0.70710678118654752f)));
    }
    *reinterpret_cast<uint4*>(x + i) = v;
  }
}

// feature row f -> row dst_tok[f] of rank dst_rank[f]'s feature buffer
__global__ void feat_scatter_kernel(const bf16* __restrict__ feat, int nf, int H,
                                    const int* __restrict__ dst_rank, const int* __restrict__ dst_tok,
                                    FeatPeers peers) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= nf) return;
  const uint4* s = reinterpret_cast<const uint4*>(feat + int64_t(warp) * H);
  uint4* d = reinterpret_cast<uint4*>(peers.p[dst_rank[warp]] + int64_t(dst_tok[warp]) * H);
  for (int c = lane; c < H / 8; c += 32) d[c] = s[c];
}

// x[t] = fp32(feat[t]) for the feature rows (fmask[t] != 0)
__global__ void feat_inject_kernel(float* __restrict__ x, const bf16* __restrict__ feat,
                                   const int* __restrict__ fmask, int T, int H) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= T || !fmask[t]) return;
  const uint4* s = reinterpret_cast<const uint4*>(feat + int64_t(t) * H);
  float4* d = reinterpret_cast<float4*>(x + int64_t(t) * H);
  for (int c = lane; c < H / 8; c += 32) {
    uint4 v = s[c];
    const bf16* e = reinterpret_cast<const bf16*>(&v);
    d[2 * c] = make_float4(__bfloat162float(e[0]), __bfloat162float(e[1]), __bfloat162float(e[2]),
                           __bfloat162float(e[3]));
    d[2 * c + 1] = make_float4(__bfloat162float(e[4]), __bfloat162float(e[5]),
                               __bfloat162float(e[6]), __bfloat162float(e[7]));
  }
}

__global__ void rows_zero_kernel(float* __restrict__ x, const int* __restrict__ fmask, int T, int H) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= T || !fmask[t]) return;
  float4* d = reinterpret_cast<float4*>(x + int64_t(t) * H);
  for (int c = lane; c < H / 4; c += 32) d[c] = make_float4(0.f, 0.f, 0.f, 0.f);
}

}  // namespace

cudaError_t k_gelu_bf16(__nv_bfloat16* x, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (n % 8) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  const int64_t vec = n / 8;
  const int grid = int(std::min<int64_t>((vec + 255) / 256, 148 * 16));
  gelu_kernel<<<grid, 256, 0, s>>>(x, n);
  return cudaGetLastError();
}

cudaError_t k_feat_scatter(const __nv_bfloat16* feat, int nf, int H, const int* dst_rank,
                           const int* dst_tok, const FeatPeers& peers, cudaStream_t s) {
  if (nf <= 0) return cudaSuccess;
  if (H % 8) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  feat_scatter_kernel<<<(nf + 7) / 8, 256, 0, s>>>(feat, nf, H, dst_rank, dst_tok, peers);
  return cudaGetLastError();
}

cudaError_t k_feat_inject(float* x, const __nv_bfloat16* feat, const int* fmask, int T, int H,
                          cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (H % 8) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  feat_inject_kernel<<<(T + 7) / 8, 256, 0, s>>>(x, feat, fmask, T, H);
  return cudaGetLastError();
}

cudaError_t k_rows_zero(float* x, const int* fmask, int T, int H, cudaStream_t s) {
  if (T <= 0) return cudaSuccess;
  if (H % 4) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  rows_zero_kernel<<<(T + 7) / 8, 256, 0, s>>>(x, fmask, T, H);
  return cudaGetLastError();
}

}  // namespace opx
