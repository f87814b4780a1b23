// DeepSpeed-Ulysses all-to-alls written as direct NVLink peer stores.
//
// seq->head (PAPER.md:589-603 gather_seq_scatter_heads; step_graph.cpp:224-229):
//   each rank holds rows*S/sp tokens x all heads; it writes, for every head
//   group (q / k / v), the heads owned by rank j straight into rank j's
//   [rows*S, heads/sp, 128] buffer at the tokens' global positions, applying
//   RoPE on the way (fused pack + rotary).
// head->seq (PAPER.md:604-612 gather_heads_scatter_seq; step_graph.cpp:237-239):
//   the mirror: rank j's [rows*S, heads/sp, 128] slices go back to the token
//   owners' [rows*S/sp, width] rows, optionally un-rotating (RoPE backward) and
//   reading an fp32 source (the dQ accumulator).
// With sp == 1 both degenerate to a local relayout (+ RoPE).
//
// The destination pointers are CUDA-IPC mappings of the peers' buffers; a
// release/acquire flag barrier (k_peer_barrier) orders the stores against the
// consumer kernels on the other GPUs.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "../runtime/kernels_api.h"
#include "ptx.cuh"

namespace opx {
namespace {

using bf16 = __nv_bfloat16;
// The head layout always has 128-element head vectors; a model head_dim hd < 128
// (multiple of 16) occupies the first hd elements and the rest stays zero (the
// buffers are zeroed once and never written there), so the attention kernels
// run unchanged at d = 128 with the softmax scale of hd.
constexpr int D = 128;

// Each thread moves 8 elements of the first half and the matching 8 of the
// second half of one head vector (so RoPE pairs stay in one thread).
__global__ void seq2head_kernel(const A2AArgs a) {
  const int hd = a.hd ? a.hd : D, HALF = hd / 2;
  const int per_tok = hd / 16;  // threads per head vector
  int heads = 0;
  for (int i = 0; i < a.ngroups; ++i) heads += a.g[i].heads_total;
  const int T = a.rows * (a.seq / a.sp);
  const int work = heads * per_tok;  // threads per token
  const bf16* src = reinterpret_cast<const bf16*>(a.local[0]);
  // blockDim.y tokens per block, threadIdx.x over (head, chunk) of one token:
  // no 64-bit index arithmetic (it made the kernel instruction-bound)
  for (int r = blockIdx.x * blockDim.y + threadIdx.y; r < T; r += gridDim.x * blockDim.y)
  for (int w = threadIdx.x; w < work; w += blockDim.x) {
    const int c8 = w % per_tok;
    int hh = w / per_tok;
    int gi = 0;
    while (hh >= a.g[gi].heads_total) hh -= a.g[gi++].heads_total;
    const A2AGroup& G = a.g[gi];
    const int per_rank = G.heads_total / a.sp;
    const int dst_rank = hh / per_rank, hl = hh % per_rank;
    const int S_loc = a.seq / a.sp;
    const int b = r / S_loc, p = r % S_loc;
    const int64_t gtok = int64_t(b) * a.seq + int64_t(a.rank) * S_loc + p;

    const bf16* s = src + int64_t(r) * a.local_ld + G.col0 + hh * hd + c8 * 8;
    uint4 lo = *reinterpret_cast<const uint4*>(s);
    uint4 hi = *reinterpret_cast<const uint4*>(s + HALF);
    if (G.rope) {
      const float pos = float(a.pos[gtok]);
      uint32_t* l = reinterpret_cast<uint32_t*>(&lo);
      uint32_t* h = reinterpret_cast<uint32_t*>(&hi);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 x1 = ptx::unpack_bf16(l[e]), x2 = ptx::unpack_bf16(h[e]);
        float sn0, cs0, sn1, cs1;
        if (a.rope_tab) {  // precomputed sincosf(pos * inv_freq[i]) (identical values)
          const float2* t = a.rope_tab + int64_t(a.pos[gtok]) * HALF + c8 * 8 + 2 * e;
          const float4 v = *reinterpret_cast<const float4*>(t);
          sn0 = v.x; cs0 = v.y; sn1 = v.z; cs1 = v.w;
        } else {
          sincosf(pos * a.inv_freq[c8 * 8 + 2 * e], &sn0, &cs0);
          sincosf(pos * a.inv_freq[c8 * 8 + 2 * e + 1], &sn1, &cs1);
        }
        l[e] = ptx::pack_bf16(x1.x * cs0 - x2.x * sn0, x1.y * cs1 - x2.y * sn1);
        h[e] = ptx::pack_bf16(x2.x * cs0 + x1.x * sn0, x2.y * cs1 + x1.y * sn1);
      }
    }
    bf16* d = reinterpret_cast<bf16*>(G.full[dst_rank]) + (gtok * per_rank + hl) * D + c8 * 8;
    *reinterpret_cast<uint4*>(d) = lo;
    *reinterpret_cast<uint4*>(d + HALF) = hi;
  }
}

// seq->head with TMA bulk stores (hd == 128): a CTA rotates TB consecutive
// tokens of one row into shared memory already in the destination layout
// ([group][dst rank][TB tokens][per_rank heads][128]), then one thread per
// (group, dst rank) issues a single cp.async.bulk of TB * per_rank * 256 B
// straight into that rank's buffer (the TB tokens' rows are contiguous there).
// Two staging buffers: the next chunk is rotated while the previous chunk's
// copies drain over NVLink; an issuing thread waits for its own bulk group to
// have READ the buffer before it is overwritten.
__global__ void __launch_bounds__(512) seq2head_tma_kernel(const A2AArgs a, int TB) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  int heads = 0;
  for (int i = 0; i < a.ngroups; ++i) heads += a.g[i].heads_total;
  const int S_loc = a.seq / a.sp;
  const int nchunks = a.rows * S_loc / TB;
  const int buf_elems = TB * heads * D;
  const int work = TB * heads * 8;  // 8 threads per head vector (16 + 16 elements each)
  const int ncopy = a.ngroups * a.sp;
  const bf16* src = reinterpret_cast<const bf16*>(a.local[0]);
  int it = 0;
  for (int chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x, ++it) {
    bf16* sb = reinterpret_cast<bf16*>(smem_raw) + (it & 1) * buf_elems;
    if (it >= 2) {
      // the copies that read this buffer two chunks ago must be done reading it
      if (threadIdx.x < ncopy) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      __syncthreads();
    }
    const int r0 = chunk * TB;
    for (int w = threadIdx.x; w < work; w += blockDim.x) {
      const int t = w / (heads * 8);
      const int rem = w - t * heads * 8;
      int hh = rem >> 3;
      const int c8 = rem & 7;
      int gi = 0, hbase = 0;
      while (hh >= a.g[gi].heads_total) hh -= a.g[gi].heads_total, hbase += a.g[gi++].heads_total;
      const A2AGroup& G = a.g[gi];
      const int per_rank = G.heads_total / a.sp;
      const int dst_rank = hh / per_rank, hl = hh - dst_rank * per_rank;
      const int r = r0 + t;
      const int b = r / S_loc, p = r - b * S_loc;
      const int gtok = b * a.seq + a.rank * S_loc + p;
      const bf16* sp_ = src + int64_t(r) * a.local_ld + G.col0 + hh * D + c8 * 8;
      uint4 lo = *reinterpret_cast<const uint4*>(sp_);
      uint4 hi = *reinterpret_cast<const uint4*>(sp_ + D / 2);
      if (G.rope) {
        const float2* tb = a.rope_tab + int64_t(a.pos[gtok]) * (D / 2) + c8 * 8;
        uint32_t* l = reinterpret_cast<uint32_t*>(&lo);
        uint32_t* h = reinterpret_cast<uint32_t*>(&hi);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 x1 = ptx::unpack_bf16(l[e]), x2 = ptx::unpack_bf16(h[e]);
          const float4 v = *reinterpret_cast<const float4*>(tb + 2 * e);
          l[e] = ptx::pack_bf16(x1.x * v.y - x2.x * v.x, x1.y * v.w - x2.y * v.z);
          h[e] = ptx::pack_bf16(x2.x * v.y + x1.x * v.x, x2.y * v.w + x1.y * v.z);
        }
      }
      // staging: group gi's region, dst rank's slab, token t, local head hl
      bf16* d = sb + int64_t(TB) * D * (hbase + dst_rank * per_rank) + (t * per_rank + hl) * D + c8 * 8;
      *reinterpret_cast<uint4*>(d) = lo;
      *reinterpret_cast<uint4*>(d + D / 2) = hi;
    }
    ptx::fence_proxy_async();  // generic-proxy smem writes -> visible to the bulk copies
    __syncthreads();
    if (threadIdx.x < ncopy) {
      const int gi = threadIdx.x / a.sp, j = threadIdx.x - gi * a.sp;
      int hbase = 0;
      for (int i = 0; i < gi; ++i) hbase += a.g[i].heads_total;
      const A2AGroup& G = a.g[gi];
      const int per_rank = G.heads_total / a.sp;
      const int b = r0 / S_loc, p0 = r0 - b * S_loc;
      const int64_t gtok0 = int64_t(b) * a.seq + int64_t(a.rank) * S_loc + p0;
      const bf16* s = sb + int64_t(TB) * D * (hbase + j * per_rank);
      bf16* dst = reinterpret_cast<bf16*>(G.full[j]) + gtok0 * per_rank * D;
      const uint32_t bytes = uint32_t(TB) * per_rank * D * 2;
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
                   "r"(ptx::smem_u32(s)), "r"(bytes)
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
  }
  // every copy complete (written, not only read) before the kernel ends
  if (threadIdx.x < ncopy) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

__global__ void head2seq_kernel(const A2AArgs a) {
  const int hd = a.hd ? a.hd : D, HALF = hd / 2;
  const int per_tok = hd / 16;
  int heads_loc = 0;  // heads held by this rank across groups
  for (int i = 0; i < a.ngroups; ++i) heads_loc += a.g[i].heads_total / a.sp;
  const int Ntok = a.rows * a.seq;
  const int work = heads_loc * per_tok;
  const int S_loc = a.seq / a.sp;
  for (int gt = blockIdx.x * blockDim.y + threadIdx.y; gt < Ntok; gt += gridDim.x * blockDim.y)
  for (int w = threadIdx.x; w < work; w += blockDim.x) {
    const int c8 = w % per_tok;
    int hh = w / per_tok;
    const int64_t gtok = gt;
    int gi = 0;
    while (hh >= a.g[gi].heads_total / a.sp) hh -= a.g[gi++].heads_total / a.sp;
    const A2AGroup& G = a.g[gi];
    const int per_rank = G.heads_total / a.sp;
    const int b = gt / a.seq, sp_pos = gt % a.seq;
    const int dst_rank = sp_pos / S_loc;
    const int r = b * S_loc + sp_pos % S_loc;
    float x1[8], x2[8];
    if (G.src_f32) {
      const float* s = reinterpret_cast<const float*>(G.full[0]) + (gtok * per_rank + hh) * D + c8 * 8;
      const float4 a0 = *reinterpret_cast<const float4*>(s), a1 = *reinterpret_cast<const float4*>(s + 4);
      const float4 b0 = *reinterpret_cast<const float4*>(s + HALF),
                   b1 = *reinterpret_cast<const float4*>(s + HALF + 4);
      x1[0] = a0.x; x1[1] = a0.y; x1[2] = a0.z; x1[3] = a0.w;
      x1[4] = a1.x; x1[5] = a1.y; x1[6] = a1.z; x1[7] = a1.w;
      x2[0] = b0.x; x2[1] = b0.y; x2[2] = b0.z; x2[3] = b0.w;
      x2[4] = b1.x; x2[5] = b1.y; x2[6] = b1.z; x2[7] = b1.w;
    } else {
      const bf16* s = reinterpret_cast<const bf16*>(G.full[0]) + (gtok * per_rank + hh) * D + c8 * 8;
      const uint4 lo = *reinterpret_cast<const uint4*>(s), hi = *reinterpret_cast<const uint4*>(s + HALF);
      const uint32_t* l = reinterpret_cast<const uint32_t*>(&lo);
      const uint32_t* h = reinterpret_cast<const uint32_t*>(&hi);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 u = ptx::unpack_bf16(l[e]), v = ptx::unpack_bf16(h[e]);
        x1[2 * e] = u.x; x1[2 * e + 1] = u.y; x2[2 * e] = v.x; x2[2 * e + 1] = v.y;
      }
    }
    if (G.rope) {  // inverse rotation (transpose of the forward rotary matrix)
      const float pos = float(a.pos[gtok]);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float sn, cs;
        if (a.rope_tab) {
          const float2 v = a.rope_tab[int64_t(a.pos[gtok]) * HALF + c8 * 8 + e];
          sn = v.x;
          cs = v.y;
        } else {
          sincosf(pos * a.inv_freq[c8 * 8 + e], &sn, &cs);
        }
        const float y1 = x1[e] * cs + x2[e] * sn;
        const float y2 = x2[e] * cs - x1[e] * sn;
        x1[e] = y1;
        x2[e] = y2;
      }
    }
    uint4 lo, hi;
    uint32_t* l = reinterpret_cast<uint32_t*>(&lo);
    uint32_t* h = reinterpret_cast<uint32_t*>(&hi);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      l[e] = ptx::pack_bf16(x1[2 * e], x1[2 * e + 1]);
      h[e] = ptx::pack_bf16(x2[2 * e], x2[2 * e + 1]);
    }
    const int hglob = a.rank * per_rank + hh;  // head index within the group
    bf16* d = reinterpret_cast<bf16*>(a.local[dst_rank]) + int64_t(r) * a.local_ld + G.col0 +
              hglob * hd + c8 * 8;
    *reinterpret_cast<uint4*>(d) = lo;
    *reinterpret_cast<uint4*>(d + HALF) = hi;
  }
}

__global__ void peer_barrier_kernel(uint32_t* const* peer_flags, uint32_t* my_flags, int n, int me,
                                    uint32_t epoch, int* timeout_flag) {
  const int j = threadIdx.x;
  if (j >= n) return;
  __threadfence_system();
  ptx::st_release_sys(peer_flags[j] + me, epoch);
  long long spins = 0;
  while (ptx::ld_acquire_sys(my_flags + j) < epoch) {
    if (++spins > (1ll << 31)) {  // ~seconds: report instead of hanging the box
      if (timeout_flag) atomicExch(timeout_flag, 1);
      break;
    }
  }
  __threadfence_system();
}

__global__ void rope_table_kernel(float2* tab, int npos, int half, const float* inv_freq) {
  const int64_t n = int64_t(npos) * half;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const float pos = float(i / half);
    float sn, cs;
    sincosf(pos * inv_freq[i % half], &sn, &cs);
    tab[i] = make_float2(sn, cs);
  }
}

}  // namespace

cudaError_t k_rope_table(float2* tab, int npos, int half, const float* inv_freq, cudaStream_t s) {
  if (npos <= 0) return cudaSuccess;
  ++g_kernel_launches;
  rope_table_kernel<<<num_sms() * 4, 256, 0, s>>>(tab, npos, half, inv_freq);
  return cudaGetLastError();
}

// block shape for `work` threads per token: x = work rounded to a warp
// (<= 1024), y = tokens per block so a block has ~256 threads
static dim3 a2a_block(int work) {
  const int x = std::min(1024, (work + 31) / 32 * 32);
  return dim3(x, std::max(1, 256 / x));
}

// staging tokens per chunk for the bulk-store seq->head (0 = use the
// per-thread peer-store kernel): hd 128 with a RoPE table, the chunk must not
// cross a row, two buffers of TB token rows within ~100 KB
static int seq2head_tb(const A2AArgs& a, int heads) {
  // opt-in: measured slower than the per-thread peer stores (C1 SP2 q/k/v
  // exchange 421 vs 524 GB/s)
  static const int mode = getenv("OPX_A2A_TMA") ? atoi(getenv("OPX_A2A_TMA")) : 0;
  const int hd = a.hd ? a.hd : D;
  if (!mode || hd != D || !a.rope_tab || a.ngroups * a.sp > 512) return 0;
  for (int i = 0; i < a.ngroups; ++i)
    if (a.g[i].rope && !a.rope_tab) return 0;
  const int S_loc = a.seq / a.sp;
  for (int tb = 8; tb >= 1; tb /= 2)
    if (S_loc % tb == 0 && 2 * tb * heads * D * 2 <= 100 * 1024) return tb;
  return 0;
}

cudaError_t k_a2a_seq2head(const A2AArgs& a, cudaStream_t s) {
  int heads = 0;
  for (int i = 0; i < a.ngroups; ++i) heads += a.g[i].heads_total;
  const int T = a.rows * (a.seq / a.sp);
  const int hd = a.hd ? a.hd : D;
  if (T <= 0 || heads <= 0) return cudaSuccess;
  if (const int tb = seq2head_tb(a, heads)) {
    const int smem = 2 * tb * heads * D * 2;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(seq2head_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    const int per_sm = std::max(1, std::min(4, (220 * 1024) / (smem + 1024)));
    const int blocks = std::min(T / tb, num_sms() * per_sm);
    ++g_kernel_launches;
    seq2head_tma_kernel<<<blocks, 512, smem, s>>>(a, tb);
    return cudaGetLastError();
  }
  const dim3 blk = a2a_block(heads * (hd / 16));
  const int blocks = std::min((T + int(blk.y) - 1) / int(blk.y), num_sms() * 32);
  ++g_kernel_launches;
  seq2head_kernel<<<blocks, blk, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t k_a2a_head2seq(const A2AArgs& a, cudaStream_t s) {
  int heads = 0;
  for (int i = 0; i < a.ngroups; ++i) heads += a.g[i].heads_total / a.sp;
  const int N = a.rows * a.seq;
  const int hd = a.hd ? a.hd : D;
  if (N <= 0 || heads <= 0) return cudaSuccess;
  const dim3 blk = a2a_block(heads * (hd / 16));
  const int blocks = std::min((N + int(blk.y) - 1) / int(blk.y), num_sms() * 32);
  ++g_kernel_launches;
  head2seq_kernel<<<blocks, blk, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t k_peer_barrier(uint32_t* const* peer_flags, uint32_t* my_flags, int n, int me,
                           uint32_t epoch, int* timeout_flag, cudaStream_t s) {
  ++g_kernel_launches;
  peer_barrier_kernel<<<1, 32, 0, s>>>(peer_flags, my_flags, n, me, epoch, timeout_flag);
  return cudaGetLastError();
}

}  // namespace opx
