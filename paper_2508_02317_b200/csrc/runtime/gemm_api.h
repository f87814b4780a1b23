// Internal C++ interface to the tcgen05 GEMM (kernels/gemm.cu).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace opx {

struct A2AArgs;  // kernels_api.h

enum GemmEpi : int {
  GEMM_EPI_BF16 = 0,       // D(bf16) = acc*scale
  GEMM_EPI_F32 = 1,        // D(f32)  = acc*scale
  GEMM_EPI_F32_RESID = 2,  // D(f32)  = R + acc*scale   (R may alias D)
  GEMM_EPI_F32_ACCUM = 3,  // D(f32) += acc*scale
  GEMM_EPI_SWIGLU = 4,     // D2(bf16)[., N/2] = silu(gate)*up; D (optional) = bf16 gate|up
  // acc = dact[., N] (N = F); G2 = the forward's bf16 gate|up [., 2N] (128-col
  // interleave); D(bf16)[., 2N] = d(gate)|d(up) of silu(gate)*up, same layout
  GEMM_EPI_SWIGLU_BWD = 5,
  // Ulysses seq->head fused into the epilogue (async_ulysses, step_graph.cpp:
  // 217-241): every 128-column head vector of a row goes, rounded to bf16 and
  // RoPE'd per its group, straight to the owning SP rank's head-layout buffer
  // over NVLink (the k_a2a_seq2head addressing); D is unused.  head_dim 128,
  // plain (non-grouped) GEMMs on the 2-CTA kernel only.
  GEMM_EPI_SEQ2HEAD = 6,
  // grouped-M (expert) GEMMs: bf16 row r of group g goes to peer rank s's
  // buffer rm_dst[s] at row rm_off[g*ep+s] + (r - sum of rm_cnt[g*ep+0..s-1])
  // -- the MoE combine (rows back to their token owners' sorted positions,
  // step_graph.cpp:253-293) fused into the expert GEMM as NVLink peer stores
  GEMM_EPI_ROWMAP = 7,
};

// D[M,N] = A . B^T with
//   A: !a_mn -> stored [M rows, K cols] (lda) ;  a_mn -> stored [K rows, M cols] (lda)
//   B: !b_mn -> stored [N rows, K cols] (ldb) ;  b_mn -> stored [K rows, N cols] (ldb)
// Grouped (MoE) forms:
//   groups>0, grouped_k=0: A rows are 128-aligned segments g_start[g]..+g_rows[g] of a
//     buffer with rows_total rows; B is a stack of `groups` slabs ([N,K] or [K,N]);
//     D rows follow A rows.
//   groups>0, grouped_k=1: K of group g = rows g_start[g]..+g_rows[g] (g_rows multiple
//     of 64, zero padded) of A ([rows_total, M], a_mn) and B ([rows_total, N], b_mn);
//     D of group g at D + g*d_group_stride.
struct GemmDesc {
  int M = 0, N = 0, K = 0;
  const __nv_bfloat16* A = nullptr;
  int64_t lda = 0;
  bool a_mn = false;
  const __nv_bfloat16* B = nullptr;
  int64_t ldb = 0;
  bool b_mn = false;
  int epi = GEMM_EPI_BF16;
  void* D = nullptr;
  int64_t ldd = 0;
  const float* R = nullptr;
  int64_t ldr = 0;
  __nv_bfloat16* D2 = nullptr;
  int64_t ldd2 = 0;
  const __nv_bfloat16* G2 = nullptr;  // GEMM_EPI_SWIGLU_BWD input
  int64_t ldg2 = 0;
  float scale = 1.f;
  int groups = 0;
  int grouped_k = 0;
  const int* g_start = nullptr;
  const int* g_rows = nullptr;
  int64_t rows_total = 0;
  int64_t d_group_stride = 0;
  const A2AArgs* s2h = nullptr;  // GEMM_EPI_SEQ2HEAD routing (copied at launch)
  // optional bf16 column bias [N] (BF16 / F32 / F32_RESID / SWIGLU epilogues;
  // SWIGLU: in the 128-column gate|up interleave of B's rows), added to the
  // accumulator before rounding / activation
  const __nv_bfloat16* bias = nullptr;
  // GEMM_EPI_ROWMAP: device array [rm_ep] of destination bases; per-group
  // tables [groups][rm_ep] of row counts and destination row offsets
  __nv_bfloat16* const* rm_dst = nullptr;
  const int* rm_cnt = nullptr;
  const int* rm_off = nullptr;
  int rm_ep = 1;
};

cudaError_t gemm_run(const GemmDesc& g, cudaStream_t s);
// OPX_GEMM_LOG diagnostics: print per-shape GEMM times recorded since the last dump.
void gemm_log_dump(const char* tag);
// 2-CTA (cta_group::2, 256x256 per CTA pair) path for plain GEMMs; gemm_run
// dispatches to it unless OPX_GEMM_1CTA is set.
cudaError_t gemm2_run(const GemmDesc& g, int band, cudaStream_t s);
// 2-D bf16 TMA map (inner contiguous dim, outer dim, row stride in elements), SW128.
bool gemm_make_map(void* map, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                   uint32_t box_inner, uint32_t box_outer);
int num_sms();

}  // namespace opx
