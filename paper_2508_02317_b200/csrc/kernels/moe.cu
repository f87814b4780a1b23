// MoE expert parallelism (VeOmni EP plan; omniplan
// build_moe_block step_graph.cpp:253-293, ep_groups plan.cpp:168-182).
//
// Routing contract (bit-exact with the CPU oracle given identical inputs):
//   * router logits in fp32 with a fixed sequential K order and separately
//     rounded multiply/add (no FMA contraction);
//   * top-k on the logits (softmax is monotone), ties -> lower expert index;
//   * weights = softmax renormalised over the selected experts (Qwen3 norm_topk_prob);
//   * permutation = stable counting sort of (token, slot) pairs by expert.
// EP data movement is written as peer stores into the expert ranks' receive
// buffers (CUDA-IPC mappings), laid out as per-local-expert segments padded to
// 128 rows (so grouped-GEMM M tiles never straddle experts and wgrad K blocks
// read zeros), ordered by source rank then by the source's pair order.
#include <cstdlib>
#include <cuda_bf16.h>

#include "../runtime/kernels_api.h"
#include "ptx.cuh"

namespace opx {
namespace {

using bf16 = __nv_bfloat16;

// ---------------------------------------------------------------------------
// router logits: logits[t, e] = sum_k h[t,k] * w[e,k] in the oracle's defined
// order (oracle/model.py router_logits), so routing is bit-exact: for H a
// multiple of 128 the K range is split into 4 quarters, each summed with k
// ascending (fmul/fadd rn) by its own block (blockIdx.z), and the partials are
// combined as (p0 + p1) + (p2 + p3); otherwise one sequential sum.  Block tile:
// 32 tokens x 128 experts (256 blocks at T = 8192, two per SM), K in chunks of
// 32 staged through smem with 16-B loads; the next chunk is fetched into
// registers while the current one is consumed.
constexpr int RT = 32, RE = 128, RK = 32;
// 256 threads; thread (ty, tx): tokens ty*2 .. +1, experts tx*4 + {0..3}, 64 + tx*4 + {0..3}.
__global__ void __launch_bounds__(256, 2) router_kernel(const bf16* __restrict__ h,
                                                        const bf16* __restrict__ w,
                                                        float* __restrict__ logits_all, int T, int H,
                                                        int E, int ksplit) {
  __shared__ float sh[RK][RT + 4];
  __shared__ float sw[RK][RE + 4];
  const int t0 = blockIdx.x * RT, e0 = blockIdx.y * RE;
  // this block's K quarter (ksplit = 4) or all of K, and its partial output
  const int kb = blockIdx.z * (H / ksplit), ke = kb + H / ksplit;
  float* __restrict__ logits = logits_all + int64_t(blockIdx.z) * T * E;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  // staging: h chunk = 32 tok x 32 k = 128 x 16 B (threads 0..127),
  //          w chunk = 128 exp x 32 k = 512 x 16 B (2 per thread)
  const int hr = threadIdx.x >> 2, hc = (threadIdx.x & 3) * 8;   // h: token row, k offset
  uint4 hq = make_uint4(0, 0, 0, 0), wq[2];
  auto fetch = [&](int k0) {
    if (threadIdx.x < RT * 4) {
      const int t = t0 + hr;
      hq = t < T ? *reinterpret_cast<const uint4*>(h + int64_t(t) * H + k0 + hc) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int idx = threadIdx.x + u * 256;
      const int e = e0 + (idx >> 2);
      wq[u] = e < E ? *reinterpret_cast<const uint4*>(w + int64_t(e) * H + k0 + (idx & 3) * 8)
                    : make_uint4(0, 0, 0, 0);
    }
  };
  auto stash = [&]() {
    if (threadIdx.x < RT * 4) {
      const uint32_t v[4] = {hq.x, hq.y, hq.z, hq.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = ptx::unpack_bf16(v[q]);
        sh[hc + 2 * q][hr] = f.x;
        sh[hc + 2 * q + 1][hr] = f.y;
      }
    }
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int idx = threadIdx.x + u * 256;
      const int ee = idx >> 2, kc = (idx & 3) * 8;
      const uint32_t v[4] = {wq[u].x, wq[u].y, wq[u].z, wq[u].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float2 f = ptx::unpack_bf16(v[q]);
        sw[kc + 2 * q][ee] = f.x;
        sw[kc + 2 * q + 1][ee] = f.y;
      }
    }
  };
  float acc[2][8];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
  fetch(kb);
  for (int k0 = kb; k0 < ke; k0 += RK) {
    stash();
    __syncthreads();
    if (k0 + RK < ke) fetch(k0 + RK);  // in flight during the FMAs below
#pragma unroll 8
    for (int kk = 0; kk < RK; ++kk) {
      // this thread's experts: tx*4 + {0..3} and 64 + tx*4 + {0..3} (two
      // conflict-free 16-B loads); its tokens ty*2, ty*2 + 1 (one 8-B load)
      const float2 hv = *reinterpret_cast<const float2*>(&sh[kk][ty * 2]);
      const float4 wa = *reinterpret_cast<const float4*>(&sw[kk][tx * 4]);
      const float4 wb = *reinterpret_cast<const float4*>(&sw[kk][64 + tx * 4]);
      const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
      const float hh[2] = {hv.x, hv.y};
      // k ascending; the product of two bf16 values is exact in fp32, so the
      // fused multiply-add rounds exactly like the oracle's separate
      // multiply (exact) and add (rounded)
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = __fmaf_rn(hh[i], wv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int t = t0 + ty * 2 + i;
    if (t >= T) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int e = e0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + j - 4);
      if (e < E) logits[int64_t(t) * E + e] = acc[i][j];
    }
  }
}

// logits = (p0 + p1) + (p2 + p3) of the four K-quarter partials
__global__ void router_combine_kernel(const float* __restrict__ part, float* __restrict__ logits,
                                      int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    logits[i] = __fadd_rn(__fadd_rn(part[i], part[n + i]), __fadd_rn(part[2 * n + i], part[3 * n + i]));
}

// top-k per token (one warp per token), E <= 256, k <= 16
__global__ void topk_kernel(const float* __restrict__ logits, int T, int E, int k,
                            int* __restrict__ idx, float* __restrict__ wts) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  float v[8];
  const int per = (E + 31) / 32;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int e = lane + 32 * i;
    v[i] = (i < per && e < E) ? logits[int64_t(t) * E + e] : -INFINITY;
  }
  float sel[16];
  int seli[16];
  for (int j = 0; j < k; ++j) {
    float bv = -INFINITY;
    int bi = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = lane + 32 * i;
      if (v[i] > bv || (v[i] == bv && e < bi)) {
        bv = v[i];
        bi = e;
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) {
        bv = ov;
        bi = oi;
      }
    }
    sel[j] = bv;
    seli[j] = bi;
    if ((bi & 31) == lane) v[bi >> 5] = -INFINITY;  // remove the winner
  }
  if (lane == 0) {
    float s = 0.f;
    for (int j = 0; j < k; ++j) s += expf(sel[j] - sel[0]);
    for (int j = 0; j < k; ++j) {
      idx[int64_t(t) * k + j] = seli[j];
      wts[int64_t(t) * k + j] = expf(sel[j] - sel[0]) / s;
    }
  }
}

// ---------------------------------------------------------------------------
// stable counting sort of pairs p = t*k + j by expert idx[p]
// pass 1: per-chunk histograms; pass 2: per-expert exclusive scan over chunks
// (+ expert offsets); pass 3: each chunk assigns positions in pair order.
// ---------------------------------------------------------------------------
constexpr int CHUNK = 1024;
__global__ void hist_kernel(const int* __restrict__ idx, int P, int E, int* __restrict__ hist) {
  extern __shared__ int sh_hist[];
  for (int e = threadIdx.x; e < E; e += blockDim.x) sh_hist[e] = 0;
  __syncthreads();
  const int p0 = blockIdx.x * CHUNK;
  for (int p = p0 + threadIdx.x; p < min(p0 + CHUNK, P); p += blockDim.x)
    atomicAdd(&sh_hist[idx[p]], 1);
  __syncthreads();
  for (int e = threadIdx.x; e < E; e += blockDim.x) hist[int64_t(blockIdx.x) * E + e] = sh_hist[e];
}

// one thread per expert: chunk offsets (in place) and totals; then one block scan
__global__ void scan_kernel(int* __restrict__ hist, int nchunks, int E, int* __restrict__ counts,
                            int* __restrict__ excl) {
  const int e = threadIdx.x;
  __shared__ int tot[1024];
  if (e < E) {
    int run = 0;
    for (int c = 0; c < nchunks; ++c) {
      const int v = hist[int64_t(c) * E + e];
      hist[int64_t(c) * E + e] = run;
      run += v;
    }
    counts[e] = run;
    tot[e] = run;
  }
  __syncthreads();
  if (e == 0) {
    int run = 0;
    for (int i = 0; i < E; ++i) {
      excl[i] = run;
      run += tot[i];
    }
  }
}

__global__ void place_kernel(const int* __restrict__ idx, int P, int E, const int* __restrict__ hist,
                             const int* __restrict__ excl, int* __restrict__ pos_of_pair,
                             int* __restrict__ pair_at) {
  extern __shared__ int run[];
  for (int e = threadIdx.x; e < E; e += blockDim.x)
    run[e] = excl[e] + hist[int64_t(blockIdx.x) * E + e];
  __syncthreads();
  // one warp walks the chunk in order, 32 pairs at a time
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    const int p0 = blockIdx.x * CHUNK;
    for (int base = p0; base < min(p0 + CHUNK, P); base += 32) {
      const int p = base + lane;
      const bool ok = p < P;
      const int e = ok ? idx[p] : -1 - lane;
      const unsigned peers = __match_any_sync(0xffffffffu, e);
      const int rank_in = __popc(peers & ((1u << lane) - 1));
      const int leader = __ffs(peers) - 1;
      int basepos = 0;
      if (ok && lane == leader) basepos = run[e];
      basepos = __shfl_sync(0xffffffffu, basepos, leader);
      if (ok) {
        const int pos = basepos + rank_in;
        pos_of_pair[p] = pos;
        pair_at[pos] = p;
      }
      __syncwarp();
      if (ok && lane == leader) run[e] = basepos + __popc(peers);
      __syncwarp();
    }
  }
}

// ---------------------------------------------------------------------------
// EP layout helpers.  counts_all[s*E + e] = pairs source rank s routes to
// expert e (every EP rank holds the full matrix after the count exchange).
// Destination rank d owns experts [d*El, (d+1)*El).
// ---------------------------------------------------------------------------
struct Layout {
  int ep, E, El;
};

// One warp copies a W-element bf16 row (W % 256 == 0 for the fast path): all
// loads of the row are issued before the (possibly remote, NVLink) stores.
__device__ __forceinline__ void copy_row(bf16* __restrict__ o, const bf16* __restrict__ s, int W,
                                         int lane) {
  int c = lane * 8;
  for (; c + 7 * 256 < W; c += 8 * 256) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = *reinterpret_cast<const uint4*>(s + c + u * 256);
#pragma unroll
    for (int u = 0; u < 8; ++u) *reinterpret_cast<uint4*>(o + c + u * 256) = v[u];
  }
  for (; c < W; c += 256) *reinterpret_cast<uint4*>(o + c) = *reinterpret_cast<const uint4*>(s + c);
}

__device__ __forceinline__ int seg_len(const int* counts_all, const Layout& L, int e) {
  int n = 0;
  for (int s = 0; s < L.ep; ++s) n += counts_all[s * L.E + e];
  return n;
}

// segment starts of rank d's local experts (128-row padded), computed into smem by one warp
__device__ void seg_starts(const int* counts_all, const Layout& L, int d, int* out /*[El+1]*/) {
  if (threadIdx.x == 0) {
    int run = 0;
    for (int le = 0; le < L.El; ++le) {
      out[le] = run;
      run += (seg_len(counts_all, L, d * L.El + le) + 127) / 128 * 128;
    }
    out[L.El] = run;
  }
}

// g_start/g_rows (valid rows and 128-padded rows) of this rank's local experts
__global__ void groups_kernel(const int* __restrict__ counts_all, Layout L, int me,
                              int* __restrict__ g_start, int* __restrict__ g_rows,
                              int* __restrict__ g_rows_pad, int* __restrict__ total_rows) {
  __shared__ int st[1025];
  seg_starts(counts_all, L, me, st);
  __syncthreads();
  for (int le = threadIdx.x; le < L.El; le += blockDim.x) {
    g_start[le] = st[le];
    g_rows[le] = seg_len(counts_all, L, me * L.El + le);
    g_rows_pad[le] = st[le + 1] - st[le];
  }
  if (threadIdx.x == 0) *total_rows = st[L.El];
}

// Zero the padding rows of every local segment of a [rows, W] bf16 buffer.
__global__ void zero_pad_kernel(bf16* __restrict__ buf, int64_t ld, int W,
                                const int* __restrict__ g_start, const int* __restrict__ g_rows,
                                const int* __restrict__ g_rows_pad, int El) {
  const int le = blockIdx.y;
  if (le >= El) return;
  const int r0 = g_start[le] + g_rows[le], r1 = g_start[le] + g_rows_pad[le];
  const int n8 = W / 8;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < (r1 - r0) * n8; i += gridDim.x * blockDim.x) {
    const int r = r0 + i / n8, c = (i % n8) * 8;
    *reinterpret_cast<uint4*>(buf + int64_t(r) * ld + c) = make_uint4(0, 0, 0, 0);
  }
}

// Destination tables of the dispatch addressing, in smem (int[route_smem_ints]):
// [ep][El+1] segment starts of every destination rank, then per expert this
// rank's sorted offset (excl) and the rows earlier ranks put before ours.
// Filled by the whole block; the caller syncs.
__host__ __device__ inline int route_smem_ints(const Layout& L) { return L.ep * (L.El + 1) + 2 * L.E; }
__device__ void route_tables(const int* __restrict__ counts_all, const int* __restrict__ excl,
                             const Layout& L, int me, int* st) {
  int* sx = st + L.ep * (L.El + 1);
  int* sb = sx + L.E;
  if (threadIdx.x < L.ep) {
    const int d = threadIdx.x;
    int run = 0;
    for (int le = 0; le < L.El; ++le) {
      st[d * (L.El + 1) + le] = run;
      run += (seg_len(counts_all, L, d * L.El + le) + 127) / 128 * 128;
    }
    st[d * (L.El + 1) + L.El] = run;
  }
  for (int e = threadIdx.x; e < L.E; e += blockDim.x) {
    sx[e] = excl[e];
    int before = 0;
    for (int s = 0; s < me; ++s) before += counts_all[s * L.E + e];
    sb[e] = before;
  }
}
// receive row (on rank d, local expert le) of sorted position pos
__device__ __forceinline__ int route_row(int pos, const int* st, const Layout& L, int& d, int& le) {
  const int* sx = st + L.ep * (L.El + 1);
  const int* sb = sx + L.E;
  // expert of this sorted position: largest e with excl[e] <= pos (E <= 1024)
  int lo = 0, hi = L.E - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sx[mid] <= pos) lo = mid; else hi = mid - 1;
  }
  const int e = lo;
  d = e / L.El;
  le = e % L.El;
  return st[d * (L.El + 1) + le] + sb[e] + (pos - sx[e]);
}

// Dispatch: for every pair in this rank's sorted order, copy its token row
// (src row = pair / k, or the pair row itself when per_pair) to the expert
// rank's receive buffer.  One warp per pair, 16 B per lane.
__global__ void dispatch_kernel(const bf16* __restrict__ src, int64_t ld_src, int per_pair,
                                const int* __restrict__ pair_at, int P, int k,
                                const int* __restrict__ counts_all, const int* __restrict__ excl,
                                Layout L, int me, bf16* const* __restrict__ dst, int64_t ld_dst,
                                int W, int le_lo, int le_hi) {
  extern __shared__ int st[];
  route_tables(counts_all, excl, L, me, st);
  __syncthreads();
  const int lane = threadIdx.x & 31;
  for (int pos = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; pos < P;
       pos += (gridDim.x * blockDim.x) >> 5) {
    const int p = pair_at[pos];
    int d, le;
    const int row = route_row(pos, st, L, d, le);
    if (le < le_lo || le >= le_hi) continue;  // another phase's experts (moe_overlap)
    const bf16* s = src + int64_t(per_pair ? pos : p / k) * ld_src;
    bf16* o = dst[d] + int64_t(row) * ld_dst;
    copy_row(o, s, W, lane);
  }
}

// Combine map for GEMM_EPI_ROWMAP: for local expert le and source rank s, the
// rows of segment le that came from s (cnt) and where they go back (off: s's
// sorted offset of expert e = me*El + le): the combine's addressing as a
// table the expert GEMM epilogue reads
__global__ void combine_map_kernel(const int* __restrict__ counts_all, Layout L, int me,
                                   int* __restrict__ cnt, int* __restrict__ off) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= L.El * L.ep) return;
  const int le = i / L.ep, s = i % L.ep;
  const int e = me * L.El + le;
  const int* c = counts_all + s * L.E;
  int x = 0;
  for (int e2 = 0; e2 < e; ++e2) x += c[e2];
  cnt[i] = c[e];
  off[i] = x;
}

// Combine: every valid row of local expert segment le goes back to its source
// rank s, at s's sorted position of that pair (the combine map's tables);
// one warp per row, 16-B stores along the row (coalesced NVLink writes)
__global__ void combine_kernel(const bf16* __restrict__ src, int64_t ld_src,
                               const int* __restrict__ cnt, const int* __restrict__ off, int ep,
                               const int* __restrict__ g_start, bf16* const* __restrict__ dst,
                               int64_t ld_dst, int W, int le_lo) {
  const int lane = threadIdx.x & 31;
  const int le = le_lo + blockIdx.y;
  __shared__ int s_cnt[kMaxSp], s_off[kMaxSp];
  if (threadIdx.x < ep) {
    s_cnt[threadIdx.x] = cnt[le * ep + threadIdx.x];
    s_off[threadIdx.x] = off[le * ep + threadIdx.x];
  }
  __syncthreads();
  int n = 0;
  for (int s = 0; s < ep; ++s) n += s_cnt[s];
  for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += (gridDim.x * blockDim.x) >> 5) {
    int s = 0, o = r;
    while (o >= s_cnt[s]) o -= s_cnt[s], ++s;
    copy_row(dst[s] + int64_t(s_off[s] + o) * ld_dst, src + int64_t(g_start[le] + r) * ld_src, W, lane);
  }
}

// out[t] = resid[t] + sum_j w[t,j] * Y[pos(t,j)]  (fp32; one warp per token)
__global__ void unpermute_kernel(const bf16* __restrict__ Y, int64_t ldy, const int* __restrict__ pos_of_pair,
                                 const float* __restrict__ wts, int T, int k, int H,
                                 const float* resid, float* out) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  for (int c = lane * 4; c < H; c += 128) {
    float4 acc = resid ? *reinterpret_cast<const float4*>(resid + int64_t(t) * H + c)
                       : make_float4(0, 0, 0, 0);
    for (int j = 0; j < k; ++j) {
      const int pos = pos_of_pair[t * k + j];
      const float wj = wts ? wts[t * k + j] : 1.f;
      const uint2 q = *reinterpret_cast<const uint2*>(Y + int64_t(pos) * ldy + c);
      const float2 a = ptx::unpack_bf16(q.x), b = ptx::unpack_bf16(q.y);
      acc.x += wj * a.x;
      acc.y += wj * a.y;
      acc.z += wj * b.x;
      acc.w += wj * b.y;
    }
    *reinterpret_cast<float4*>(out + int64_t(t) * H + c) = acc;
  }
}

// backward of the weighted combine (one warp per token):
//   dYp[pos(t,j)] = bf16(w[t,j] * dx[t]);  dw[t,j] = <dx[t], Y[pos(t,j)]>
// dx[t] stays in registers (MAXC chunks of 256 columns, 8 per lane, 16-B accesses).
// ROUTE (the a2a_combine_grad fused in): the dY row of sorted position pos is
// stored straight into its expert rank's receive buffer, at the row the
// dispatch addressing gives it (peer stores over NVLink; the local share as
// plain stores), instead of into dYp for a separate dispatch pass to re-read.
template <int MAXC, bool ROUTE>
__global__ void combine_bwd_kernel(const float* __restrict__ dx, const bf16* __restrict__ Y, int64_t ldy,
                                   const int* __restrict__ pos_of_pair, const float* __restrict__ wts,
                                   int T, int k, int H, bf16* __restrict__ dYp, float* __restrict__ dw,
                                   const int* __restrict__ counts_all, const int* __restrict__ excl,
                                   Layout L, int me, bf16* const* __restrict__ dst, int64_t ld_dst,
                                   int le_lo, int le_hi) {
  extern __shared__ int st[];
  if (ROUTE) {
    route_tables(counts_all, excl, L, me, st);
    __syncthreads();
  }
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const int nc = H / 256;
  float g[MAXC][8];
#pragma unroll
  for (int i = 0; i < MAXC; ++i) {
    if (i >= nc) break;
    const float* src = dx + int64_t(t) * H + i * 256 + lane * 8;
    const float4 a = *reinterpret_cast<const float4*>(src), b = *reinterpret_cast<const float4*>(src + 4);
    g[i][0] = a.x; g[i][1] = a.y; g[i][2] = a.z; g[i][3] = a.w;
    g[i][4] = b.x; g[i][5] = b.y; g[i][6] = b.z; g[i][7] = b.w;
  }
  for (int j = 0; j < k; ++j) {
    const int pos = pos_of_pair[t * k + j];
    const float wj = wts[t * k + j];
    const bf16* yr = Y + int64_t(pos) * ldy + lane * 8;
    bf16* dr;
    if (ROUTE) {
      int d, le;
      const int row = route_row(pos, st, L, d, le);
      if (le < le_lo || le >= le_hi) continue;  // the other expert half's pair (moe_overlap)
      dr = dst[d] + int64_t(row) * ld_dst + lane * 8;
    } else {
      dr = dYp + int64_t(pos) * ldy + lane * 8;
    }
    // the whole Y row first (16 B per lane per chunk), then the stores
    uint4 yq[MAXC];
#pragma unroll
    for (int i = 0; i < MAXC; ++i)
      if (i < nc) yq[i] = *reinterpret_cast<const uint4*>(yr + i * 256);
    float dot = 0.f;
#pragma unroll
    for (int i = 0; i < MAXC; ++i) {
      if (i >= nc) break;
      const uint32_t v[4] = {yq[i].x, yq[i].y, yq[i].z, yq[i].w};
      uint32_t o[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 a = ptx::unpack_bf16(v[e]);
        dot += g[i][2 * e] * a.x + g[i][2 * e + 1] * a.y;
        o[e] = ptx::pack_bf16(wj * g[i][2 * e], wj * g[i][2 * e + 1]);
      }
      *reinterpret_cast<uint4*>(dr + i * 256) = make_uint4(o[0], o[1], o[2], o[3]);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
    if (lane == 0) dw[t * k + j] = dot;
  }
}

// router backward (renormalised softmax over the selected experts):
//   dsel_j = w_j (dw_j - sum_i w_i dw_i);  dlogits[t, idx_j] = dsel_j, else 0 (bf16)
// one warp per token: coalesced zeroing of the row, then the k scattered values
__global__ void router_bwd_kernel(const float* __restrict__ dw, const float* __restrict__ wts,
                                  const int* __restrict__ idx, int T, int k, int E,
                                  bf16* __restrict__ dlogits) {
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  bf16* row = dlogits + int64_t(t) * E;
  for (int e = lane * 2; e < E; e += 64) *reinterpret_cast<uint32_t*>(row + e) = 0u;
  float s = 0.f;
  for (int j = 0; j < k; ++j) s += wts[t * k + j] * dw[t * k + j];
  __syncwarp();
  if (lane < k)
    row[idx[t * k + lane]] = __float2bfloat16_rn(wts[t * k + lane] * (dw[t * k + lane] - s));
}

// out[i] = sum_g part[g, i]  (fixed order)
__global__ void sum_partials_kernel(const float* __restrict__ part, int G, int64_t n,
                                    void* __restrict__ out, int out_bf16) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    float acc = 0.f;
    for (int g = 0; g < G; ++g) acc += part[int64_t(g) * n + i];
    if (out_bf16) static_cast<bf16*>(out)[i] = __float2bfloat16(acc);
    else static_cast<float*>(out)[i] = acc;
  }
}

// every EP rank receives this rank's per-expert counts as row `me` of its table
__global__ void publish_counts_kernel(const int* __restrict__ counts, int* const* __restrict__ tables,
                                      int ep, int me, int E) {
  for (int i = threadIdx.x; i < ep * E; i += blockDim.x) {
    const int j = i / E, e = i % E;
    tables[j][me * E + e] = counts[e];
  }
}

// SwiGLU backward over the valid rows of every local expert segment; the
// 128-row padding of each segment is written as zeros (it feeds grouped wgrad).
__global__ void swiglu_bwd_grouped_kernel(const bf16* __restrict__ dact, const bf16* __restrict__ gu,
                                          bf16* __restrict__ dgu, const int* __restrict__ g_start,
                                          const int* __restrict__ g_rows,
                                          const int* __restrict__ g_rows_pad, int F) {
  const int le = blockIdx.y;
  const int r0 = g_start[le], nv = g_rows[le], np = g_rows_pad[le];
  const int n8 = F / 8;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < np * n8; i += gridDim.x * blockDim.x) {
    const int64_t row = r0 + i / n8;
    const int f = (i % n8) * 8;
    const int64_t gcol = int64_t(f / 128) * 256 + f % 128;
    if (i / n8 >= nv) {
      *reinterpret_cast<uint4*>(dgu + row * 2 * F + gcol) = make_uint4(0, 0, 0, 0);
      *reinterpret_cast<uint4*>(dgu + row * 2 * F + gcol + 128) = make_uint4(0, 0, 0, 0);
      continue;
    }
    const uint4 da = *reinterpret_cast<const uint4*>(dact + row * F + f);
    const uint4 gq = *reinterpret_cast<const uint4*>(gu + row * 2 * F + gcol);
    const uint4 uq = *reinterpret_cast<const uint4*>(gu + row * 2 * F + gcol + 128);
    const uint32_t a[4] = {da.x, da.y, da.z, da.w}, g[4] = {gq.x, gq.y, gq.z, gq.w},
                   u[4] = {uq.x, uq.y, uq.z, uq.w};
    uint32_t og[4], ou[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 av = ptx::unpack_bf16(a[e]), gv = ptx::unpack_bf16(g[e]), uv = ptx::unpack_bf16(u[e]);
      const float gg[2] = {gv.x, gv.y}, uu[2] = {uv.x, uv.y}, aa[2] = {av.x, av.y};
      float dg[2], du[2];
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        const float sg = __fdividef(1.f, 1.f + __expf(-gg[k]));
        du[k] = aa[k] * gg[k] * sg;
        dg[k] = aa[k] * uu[k] * sg * (1.f + gg[k] * (1.f - sg));
      }
      og[e] = ptx::pack_bf16(dg[0], dg[1]);
      ou[e] = ptx::pack_bf16(du[0], du[1]);
    }
    *reinterpret_cast<uint4*>(dgu + row * 2 * F + gcol) = make_uint4(og[0], og[1], og[2], og[3]);
    *reinterpret_cast<uint4*>(dgu + row * 2 * F + gcol + 128) = make_uint4(ou[0], ou[1], ou[2], ou[3]);
  }
}

}  // namespace

int k_moe_router_splits(int H) { return H % (4 * RK) == 0 ? 4 : 1; }

cudaError_t k_moe_router(const __nv_bfloat16* h, const __nv_bfloat16* w, float* logits, int T,
                         int H, int E, cudaStream_t s, float* partial) {
  if (H % RK || H % 8) return cudaErrorInvalidValue;
  const int ks = k_moe_router_splits(H);
  if (ks > 1 && !partial) return cudaErrorInvalidValue;
  dim3 grid((T + RT - 1) / RT, (E + RE - 1) / RE, ks);
  ++g_kernel_launches;
  router_kernel<<<grid, 256, 0, s>>>(h, w, ks > 1 ? partial : logits, T, H, E, ks);
  if (ks > 1) {
    const int64_t n = int64_t(T) * E;
    ++g_kernel_launches;
    router_combine_kernel<<<int(std::min<int64_t>((n + 255) / 256, 4096)), 256, 0, s>>>(partial, logits, n);
  }
  return cudaGetLastError();
}

cudaError_t k_moe_topk(const float* logits, int T, int E, int k, int* idx, float* wts,
                       cudaStream_t s) {
  if (E > 256 || k > 16 || k > E) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  topk_kernel<<<(T * 32 + 255) / 256, 256, 0, s>>>(logits, T, E, k, idx, wts);
  return cudaGetLastError();
}

int k_moe_sort_chunks(int P) { return (P + CHUNK - 1) / CHUNK; }

cudaError_t k_moe_sort(const int* idx, int P, int E, int* hist, int* counts, int* excl,
                       int* pos_of_pair, int* pair_at, cudaStream_t s) {
  if (E > 1024) return cudaErrorInvalidValue;
  const int nc = k_moe_sort_chunks(P);
  g_kernel_launches += 3;
  hist_kernel<<<nc, 256, E * sizeof(int), s>>>(idx, P, E, hist);
  scan_kernel<<<1, 1024, 0, s>>>(hist, nc, E, counts, excl);
  place_kernel<<<nc, 64, E * sizeof(int), s>>>(idx, P, E, hist, excl, pos_of_pair, pair_at);
  return cudaGetLastError();
}

cudaError_t k_moe_groups(const int* counts_all, int ep, int E, int me, int* g_start, int* g_rows,
                         int* g_rows_pad, int* total_rows, cudaStream_t s) {
  Layout L{ep, E, E / ep};
  if (L.El > 1024) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  groups_kernel<<<1, 128, 0, s>>>(counts_all, L, me, g_start, g_rows, g_rows_pad, total_rows);
  return cudaGetLastError();
}

cudaError_t k_moe_zero_pad(__nv_bfloat16* buf, int64_t ld, int W, const int* g_start,
                           const int* g_rows, const int* g_rows_pad, int El, cudaStream_t s) {
  dim3 grid(8, El);
  ++g_kernel_launches;
  zero_pad_kernel<<<grid, 256, 0, s>>>(buf, ld, W, g_start, g_rows, g_rows_pad, El);
  return cudaGetLastError();
}

cudaError_t k_moe_dispatch(const __nv_bfloat16* src, int64_t ld_src, int per_pair,
                           const int* pair_at, int P, int k, const int* counts_all,
                           const int* excl, int ep, int E, int me, __nv_bfloat16* const* dst,
                           int64_t ld_dst, int W, cudaStream_t s, int le_lo, int le_hi) {
  Layout L{ep, E, E / ep};
  if (le_hi < 0) le_hi = L.El;
  const int smem = (ep * (L.El + 1) + 2 * E) * int(sizeof(int));
  static const int max_blocks = getenv("OPX_A2A_BLOCKS") ? atoi(getenv("OPX_A2A_BLOCKS")) : num_sms() * 8;
  int blocks = (P * 32 + 255) / 256;
  if (blocks > max_blocks) blocks = max_blocks;
  if (blocks < 1) blocks = 1;
  ++g_kernel_launches;
  dispatch_kernel<<<blocks, 256, smem, s>>>(src, ld_src, per_pair, pair_at, P, k, counts_all,
                                            excl, L, me, dst, ld_dst, W, le_lo, le_hi);
  return cudaGetLastError();
}

cudaError_t k_moe_combine_map(const int* counts_all, int ep, int E, int me, int* cnt, int* off,
                              cudaStream_t s) {
  Layout L{ep, E, E / ep};
  const int n = L.El * ep;
  ++g_kernel_launches;
  combine_map_kernel<<<(n + 255) / 256, 256, 0, s>>>(counts_all, L, me, cnt, off);
  return cudaGetLastError();
}

cudaError_t k_moe_combine(const __nv_bfloat16* src, int64_t ld_src, const int* cnt, const int* off,
                          int ep, int El, const int* g_start, __nv_bfloat16* const* dst,
                          int64_t ld_dst, int W, int max_rows, cudaStream_t s, int le_lo, int le_n) {
  static const int max_bx = getenv("OPX_COMBINE_BX") ? atoi(getenv("OPX_COMBINE_BX")) : 64;
  int bx = (max_rows * 32 + 255) / 256 / El + 1;
  if (bx > max_bx) bx = max_bx;
  if (le_n < 0) le_n = El - le_lo;
  if (le_n <= 0) return cudaSuccess;
  dim3 grid(bx, le_n);
  ++g_kernel_launches;
  combine_kernel<<<grid, 256, 0, s>>>(src, ld_src, cnt, off, ep, g_start, dst, ld_dst, W, le_lo);
  return cudaGetLastError();
}

cudaError_t k_moe_unpermute(const __nv_bfloat16* Y, int64_t ldy, const int* pos_of_pair,
                            const float* wts, int T, int k, int H, const float* resid, float* out,
                            cudaStream_t s) {
  if (H % 128) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  unpermute_kernel<<<(T * 32 + 255) / 256, 256, 0, s>>>(Y, ldy, pos_of_pair, wts, T, k, H, resid, out);
  return cudaGetLastError();
}

cudaError_t k_moe_combine_bwd(const float* dx, const __nv_bfloat16* Y, int64_t ldy,
                              const int* pos_of_pair, const float* wts, int T, int k, int H,
                              __nv_bfloat16* dYp, float* dw, cudaStream_t s, const int* counts_all,
                              const int* excl, int ep, int E, int me, __nv_bfloat16* const* dst,
                              int64_t ld_dst, int le_lo, int le_hi) {
  if (H % 256 || H > 4096) return cudaErrorInvalidValue;
  Layout L{ep, E, ep > 0 ? E / ep : 0};
  if (le_hi < 0) le_hi = L.El;
  const bool route = dst != nullptr;
  if (route && (ep < 1 || E % ep || E > 1024)) return cudaErrorInvalidValue;
  const int smem = route ? route_smem_ints(L) * int(sizeof(int)) : 0;
  ++g_kernel_launches;
  const int blocks = (T * 32 + 255) / 256;
#define OPX_CB(C)                                                                                    \
  (route ? combine_bwd_kernel<C, true><<<blocks, 256, smem, s>>>(dx, Y, ldy, pos_of_pair, wts, T, k, H, \
                                                                  dYp, dw, counts_all, excl, L, me,   \
                                                                  dst, ld_dst, le_lo, le_hi)         \
         : combine_bwd_kernel<C, false><<<blocks, 256, 0, s>>>(dx, Y, ldy, pos_of_pair, wts, T, k, H,  \
                                                                dYp, dw, counts_all, excl, L, me, dst, \
                                                                ld_dst, 0, 0))
  if (H <= 1024)
    OPX_CB(4);
  else if (H <= 2048)
    OPX_CB(8);
  else
    OPX_CB(16);
#undef OPX_CB
  return cudaGetLastError();
}

cudaError_t k_moe_router_bwd(const float* dw, const float* wts, const int* idx, int T, int k, int E,
                             __nv_bfloat16* dlogits, cudaStream_t s) {
  if (k > 32 || E % 2) return cudaErrorInvalidValue;
  ++g_kernel_launches;
  router_bwd_kernel<<<(T * 32 + 255) / 256, 256, 0, s>>>(dw, wts, idx, T, k, E, dlogits);
  return cudaGetLastError();
}

cudaError_t k_sum_partials(const float* part, int G, int64_t n, void* out, cudaStream_t s, int out_bf16) {
  int64_t b = (n + 255) / 256;
  if (b > num_sms() * 8) b = num_sms() * 8;
  ++g_kernel_launches;
  sum_partials_kernel<<<int(b), 256, 0, s>>>(part, G, n, out, out_bf16);
  return cudaGetLastError();
}

cudaError_t k_moe_publish_counts(const int* counts, int* const* tables, int ep, int me, int E,
                                 cudaStream_t s) {
  ++g_kernel_launches;
  publish_counts_kernel<<<1, 256, 0, s>>>(counts, tables, ep, me, E);
  return cudaGetLastError();
}

cudaError_t k_moe_swiglu_bwd(const __nv_bfloat16* dact, const __nv_bfloat16* gu, __nv_bfloat16* dgu,
                             const int* g_start, const int* g_rows, const int* g_rows_pad, int El,
                             int F, int max_rows, cudaStream_t s) {
  if (F % 128) return cudaErrorInvalidValue;
  int bx = (max_rows / El * (F / 8) + 255) / 256 + 1;
  if (bx > 64) bx = 64;
  dim3 grid(bx, El);
  ++g_kernel_launches;
  swiglu_bwd_grouped_kernel<<<grid, 256, 0, s>>>(dact, gu, dgu, g_start, g_rows, g_rows_pad, F);
  return cudaGetLastError();
}

}  // namespace opx
