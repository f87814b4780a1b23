// Internal C++ launch interface of the non-GEMM kernels.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "gemm_api.h"

namespace opx {

// Number of opx kernels launched so far in this process (the executor reports
// the delta over a step as opx_step_report.launches).
extern int64_t g_kernel_launches;

// elementwise.cu
cudaError_t k_init_param(float* f32, __nv_bfloat16* b16, int64_t n, int64_t phys0, uint64_t key_a,
                         uint64_t key_b, double c, float constant, int interleave,
                         int64_t rows_per_slab, int64_t cols, cudaStream_t s);
cudaError_t k_rmsnorm_fwd(const float* x, const __nv_bfloat16* w, __nv_bfloat16* y, float* rstd,
                          int T, int H, float eps, cudaStream_t s);
int k_rmsnorm_bwd_parts(int T);
cudaError_t k_rmsnorm_bwd(const float* dy, const float* x, const __nv_bfloat16* w,
                          const float* rstd, const float* dres, float* dx, float* dw_part,
                          void* dw, int accumulate_dw, int T, int H, cudaStream_t s,
                          int dw_bf16 = 0);
cudaError_t k_embed_fwd(const int* ids, const __nv_bfloat16* E, float* x, int T, int H,
                        cudaStream_t s);
cudaError_t k_embed_bwd(const int* ids, const float* dx, float* dE, int T, int H, cudaStream_t s);
cudaError_t k_ce_fwd_bwd(__nv_bfloat16* logits, int64_t ldl, const int* labels, float* loss, int T,
                         int V, float inv_n, cudaStream_t s);
cudaError_t k_swiglu_bwd(const __nv_bfloat16* dact, const __nv_bfloat16* gu, __nv_bfloat16* dgu,
                         int64_t T, int F, cudaStream_t s);
// g: fp32 or (g_bf16) bf16 gradients
cudaError_t k_adamw(float* p, float* m, float* v, const void* g, int g_bf16, __nv_bfloat16* pb,
                    int64_t n, float lr, float b1, float b2, float eps, float wd, int step,
                    cudaStream_t s, int blocks_per_sm = 0);
cudaError_t k_cast_f32_bf16(const float* x, __nv_bfloat16* y, int64_t n, cudaStream_t s);
// acc = (first ? 0 : acc) + g (g fp32, or bf16 when g_bf16), n % 4 == 0
cudaError_t k_grad_accum(float* acc, const void* g, int g_bf16, int64_t n, int first,
                         cudaStream_t s);
cudaError_t k_sum(const float* x, int64_t n, float* out, cudaStream_t s);

// attention.cu — causal varlen GQA flash attention, head dim 128.
// q [N, hq, 128], k/v [N, hk, 128] (row strides ldq/ldk/ldv elements), o [N, hq, 128] (ldo),
// lse [hq, N] natural-log units; seq_start[t] = first token of t's sample.
struct AttnArgs {
  const __nv_bfloat16* q;
  const __nv_bfloat16* k;
  const __nv_bfloat16* v;
  __nv_bfloat16* o;
  float* lse;
  int64_t ldq, ldk, ldv, ldo;
  const int* seq_start;  // [N]
  const int* seq_end;    // [N] one past the last token of t's sample
  int N, hq, hk;
  float scale;
  // backward
  const __nv_bfloat16* dout;  // [N, hq, 128] (lddo)
  int64_t lddo;
  float* dq_acc;              // [N, hq, 128] fp32, zeroed by the caller
  __nv_bfloat16* dk;          // [N, hk, 128]
  __nv_bfloat16* dv;
  int64_t lddk, lddv;
  float* delta;               // [hq, N] scratch
  // tcgen05 backward only: fp32 dense [N, hk, 128] dK/dV outputs (replace dk/dv
  // when both set) and the number of CTAs each GQA group is split across (0 = auto)
  float* dk_acc = nullptr;
  float* dv_acc = nullptr;
  int kv_splits = 0;
  // tcgen05 forward only: 0 = bidirectional inside each sample (keys
  // [seq_start[t], seq_end[t])), the frozen encoder's attention
  int causal = 1;
};
// attention_tc.cu — the same forward on tcgen05/TMEM/TMA.
cudaError_t k_attn_fwd_tc(const AttnArgs& a, cudaStream_t s);
cudaError_t k_attn_bwd_tc(const AttnArgs& a, cudaStream_t s);
int attn_bwd_kv_splits(int N, int hq, int hk);

// a2a.cu — Ulysses all-to-all over peer memory with fused RoPE.
constexpr int kMaxSp = 8;
struct A2AGroup {
  int heads_total;                 // heads of this type across the sp group
  int col0;                        // first column (in elements) of this type in the local row
  int rope;                        // 1: apply RoPE (seq->head) / inverse RoPE (head->seq)
  int src_f32;                     // head->seq only: source is fp32 (dq accumulator)
  void* full[kMaxSp];              // seq->head: per-rank destination [m*S, heads/sp, 128]
                                   // head->seq: this rank's source   (only full[0] used)
};
struct A2AArgs {
  int sp, rank;                    // sp group size and this rank's position in it
  int rows, seq;                   // rows (sequences) per rank, full sequence length S
  int ngroups;
  A2AGroup g[3];
  void* local[kMaxSp];             // seq->head: this rank's source (local[0]);
                                   // head->seq: per-rank destination [rows*S/sp, width]
  int64_t local_ld;                // row stride (elements) of the local [tokens, width] buffers
  const int* pos;                  // [rows*S] position ids (global token index)
  const float* inv_freq;           // [hd/2]
  int hd = 0;                      // model head_dim (0 = 128); <= 128, multiple of 16
  const float2* rope_tab = nullptr;  // optional [positions][hd/2] (sin, cos) table
};
// (sin, cos)(pos * inv_freq[i]) for pos < npos, i < half: the a2a kernels' RoPE
// table (computed with the same sincosf, so results are unchanged)
cudaError_t k_rope_table(float2* tab, int npos, int half, const float* inv_freq, cudaStream_t s);
cudaError_t k_a2a_seq2head(const A2AArgs& a, cudaStream_t s);
cudaError_t k_a2a_head2seq(const A2AArgs& a, cudaStream_t s);
// encoder.cu — frozen encoder glue: GELU in place on bf16,
// feature rows -> the owning SP rank's feature buffer (peer stores), feature
// rows -> the fp32 embedding output, and zeroing of the replaced rows' grads.
struct FeatPeers {
  __nv_bfloat16* p[kMaxSp];
};
cudaError_t k_gelu_bf16(__nv_bfloat16* x, int64_t n, cudaStream_t s);
cudaError_t k_feat_scatter(const __nv_bfloat16* feat, int nf, int H, const int* dst_rank,
                           const int* dst_tok, const FeatPeers& peers, cudaStream_t s);
cudaError_t k_feat_inject(float* x, const __nv_bfloat16* feat, const int* fmask, int T, int H,
                          cudaStream_t s);
cudaError_t k_rows_zero(float* x, const int* fmask, int T, int H, cudaStream_t s);
// Peer barrier: signal every peer then wait until every peer reached `epoch`.
cudaError_t k_peer_barrier(uint32_t* const* peer_flags, uint32_t* my_flags, int n, int me,
                           uint32_t epoch, int* timeout_flag, cudaStream_t s);

}  // namespace opx

namespace opx {
// moe.cu — routing, permutation and EP exchange (see the file header).
// K-quarter count of the router's defined summation order (4 when H % 128 == 0)
int k_moe_router_splits(int H);
// partial: [splits][T][E] fp32 scratch (required when splits > 1)
cudaError_t k_moe_router(const __nv_bfloat16* h, const __nv_bfloat16* w, float* logits, int T,
                         int H, int E, cudaStream_t s, float* partial = nullptr);
cudaError_t k_moe_topk(const float* logits, int T, int E, int k, int* idx, float* wts,
                       cudaStream_t s);
int k_moe_sort_chunks(int P);
cudaError_t k_moe_sort(const int* idx, int P, int E, int* hist, int* counts, int* excl,
                       int* pos_of_pair, int* pair_at, cudaStream_t s);
cudaError_t k_moe_groups(const int* counts_all, int ep, int E, int me, int* g_start, int* g_rows,
                         int* g_rows_pad, int* total_rows, cudaStream_t s);
cudaError_t k_moe_zero_pad(__nv_bfloat16* buf, int64_t ld, int W, const int* g_start,
                           const int* g_rows, const int* g_rows_pad, int El, cudaStream_t s);
cudaError_t k_moe_dispatch(const __nv_bfloat16* src, int64_t ld_src, int per_pair,
                           const int* pair_at, int P, int k, const int* counts_all,
                           const int* excl, int ep, int E, int me, __nv_bfloat16* const* dst,
                           int64_t ld_dst, int W, cudaStream_t s, int le_lo = 0, int le_hi = -1);
// rows of local expert segments [le_lo, le_lo+le_n) back to their source ranks
// (one warp per row) at the combine map's offsets
cudaError_t k_moe_combine(const __nv_bfloat16* src, int64_t ld_src, const int* cnt, const int* off,
                          int ep, int El, const int* g_start, __nv_bfloat16* const* dst,
                          int64_t ld_dst, int W, int max_rows, cudaStream_t s, int le_lo = 0,
                          int le_n = -1);
// [El][ep] row counts / destination offsets of the combine (GEMM_EPI_ROWMAP / k_moe_combine)
cudaError_t k_moe_combine_map(const int* counts_all, int ep, int E, int me, int* cnt, int* off,
                              cudaStream_t s);
cudaError_t k_moe_unpermute(const __nv_bfloat16* Y, int64_t ldy, const int* pos_of_pair,
                            const float* wts, int T, int k, int H, const float* resid, float* out,
                            cudaStream_t s);
// dst != nullptr: the dY rows go straight to the expert ranks' receive buffers
// (the a2a_combine_grad fused in, k_moe_dispatch's addressing) instead of dYp;
// then only pairs of local experts [le_lo, le_hi) are processed (dw included)
cudaError_t k_moe_combine_bwd(const float* dx, const __nv_bfloat16* Y, int64_t ldy,
                              const int* pos_of_pair, const float* wts, int T, int k, int H,
                              __nv_bfloat16* dYp, float* dw, cudaStream_t s,
                              const int* counts_all = nullptr, const int* excl = nullptr, int ep = 0,
                              int E = 0, int me = 0, __nv_bfloat16* const* dst = nullptr,
                              int64_t ld_dst = 0, int le_lo = 0, int le_hi = -1);
cudaError_t k_moe_publish_counts(const int* counts, int* const* tables, int ep, int me, int E,
                                 cudaStream_t s);
cudaError_t k_moe_swiglu_bwd(const __nv_bfloat16* dact, const __nv_bfloat16* gu, __nv_bfloat16* dgu,
                             const int* g_start, const int* g_rows, const int* g_rows_pad, int El,
                             int F, int max_rows, cudaStream_t s);
cudaError_t k_sum_partials(const float* part, int G, int64_t n, void* out, cudaStream_t s,
                           int out_bf16 = 0);
cudaError_t k_moe_router_bwd(const float* dw, const float* wts, const int* idx, int T, int k, int E,
                             __nv_bfloat16* dlogits, cudaStream_t s);
}  // namespace opx
