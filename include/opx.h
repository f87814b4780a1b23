/*
 * opx — C ABI of the B200-native FSDP + Ulysses-SP + EP training step.
 *
 * The reference (omniplan, /root/reference/proj) exposes this path only as a
 * C++ model: build_step_graph -> simulate -> report (step_graph.hpp:59-60,
 * simulator.hpp:57-62) behind the ParallelPlan API (plan.hpp:26-107) and the
 * JSON config schema (config_io.hpp:24-50).  opx keeps that API surface and
 * executes the step on B200s instead of simulating it.  Every entry point is
 * plain C: pointers, sizes, JSON strings; no C++ types or exceptions cross.
 *
 * Return codes mirror the reference CLI exit codes (cli.hpp:15-19) where one
 * exists: 0 ok, 2 config error, 3 invalid plan, plus 6 CUDA/NCCL error,
 * 7 parity failure, 8 peer timeout, 9 bad argument.  Details of the last
 * failure on the calling thread: opx_last_error().
 */
#ifndef OPX_H
#define OPX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OPX_OK 0
#define OPX_ERR_CONFIG 2
#define OPX_ERR_PLAN 3
#define OPX_ERR_CUDA 6
#define OPX_ERR_PARITY 7
#define OPX_ERR_TIMEOUT 8
#define OPX_ERR_ARG 9

const char* opx_last_error(void);
const char* opx_version(void);

/* ------------------------------------------------------------------------
 * Plan layer (host only)
 * ------------------------------------------------------------------------ */

/* Replaces omniplan::validate (plan.hpp:68-69, plan.cpp:19-83) behind
 * parse_cluster/model/workload (config_io.cpp:52-151).  plan_json holds the
 * ParallelPlan fields (to_json keys, config_io.cpp:248-262); dp_shard may be
 * omitted and is derived as world/(dp_replicate*sp) like cli.cpp:46-65.
 * Returns 0 if valid, 3 if violations (written to out_codes as lines
 * "code<TAB>message", reference codes unchanged), 2 on config errors. */
int opx_plan_validate(const char* cluster_json, const char* model_json,
                      const char* workload_json, const char* plan_json, char* out_codes,
                      size_t cap);

/* Resolves a valid plan into a JSON document: label (plan_label, plan.cpp:149-159),
 * mesh + groups (plan_mesh/groups_along/ep_groups, plan.cpp:161-182,
 * mesh.cpp:71-105), expert sharding (plan.cpp:85-93), module plans
 * (plan.cpp:95-107), parameter accounting (specs.cpp:36-107) and per-rank
 * collective volumes (comm.cpp:8-105). */
int opx_plan_resolve(const char* cluster_json, const char* model_json,
                     const char* workload_json, const char* plan_json, char* out_json,
                     size_t cap);

/* ------------------------------------------------------------------------
 * Step executor: the real counterpart of build_step_graph + simulate + report.
 * One handle per rank (process/GPU).
 * ------------------------------------------------------------------------ */
typedef struct opx_step opx_step;

/* Measured StepReport (simulator.hpp:43-50), device-timed on this rank.  The
 * reference's fields keep their meaning, computed as report() does
 * (simulator.cpp:106-131) but on measured CUDA-event intervals of this rank's
 * streams instead of simulated ones.  The interval-based fields (comm_s,
 * comm_wait_s, exposed_comm, phase breakdown) need exec "trace" (default on). */
typedef struct {
  double step_time_s;   /* first kernel -> optimizer end, CUDA events */
  double fwd_s, bwd_s, opt_s;  /* summed over micro-batches; opt_s = tail after the backward */
  double comm_wait_s;   /* seconds of comm intervals not covered by compute (simulator.cpp:71-104) */
  double loss;          /* global mean token loss (all-reduced) */
  double tokens;        /* tokens processed by this rank this step (all micro-batches) */
  double n_valid;       /* global count of supervised tokens */
  int64_t launches;     /* opx kernels launched during the step */
  double enqueue_s;     /* host wall time spent enqueueing the step (launch-bound if ~step_time_s) */
  int64_t kept_layers;  /* layers whose activations stay resident (no full recompute) */
  /* ---- StepReport (simulator.hpp:43-50) */
  double throughput;    /* global_batch*seq_len / (step_time_s*world), tokens/s/GPU (simulator.cpp:113-115) */
  double mfu;           /* throughput * model_flops_per_token / cluster.gpu.peak_flops (:116-117) */
  double exposed_comm;  /* comm_wait_s / step_time_s (:118) */
  double model_flops_per_token;  /* flops_per_token(model, seq_len) (specs.cpp:93-107) */
  double comm_s;        /* summed duration of the comm nodes */
  int64_t accum_steps;  /* micro-batches in the step: global_batch/(dp_width*micro_batch) */
} opx_step_report;

/* 128-byte NCCL unique id for the world communicator (rank 0 creates it). */
int opx_nccl_unique_id(void* out128);

/* exec_json: {"seed":.., "lr":.., "betas":[..], "eps":.., "weight_decay":..,
 *             "rope_theta":.., "rms_eps":.., "ce_chunk":.., "trace":bool} */
int opx_step_create(const char* cluster_json, const char* model_json,
                    const char* workload_json, const char* plan_json, const char* exec_json,
                    int rank, int local_device, const void* nccl_id128, opx_step** out);
/* CUDA-IPC handles of this rank's peer-visible buffers (opaque bytes). */
int opx_step_ipc_export(opx_step* st, void* out, size_t cap, size_t* len);
/* All ranks' exports concatenated in rank order (world * len bytes). */
int opx_step_ipc_import(opx_step* st, const void* all, size_t len_per_rank);
int opx_step_init_weights(opx_step* st, uint64_t seed);
/* Host arrays for THIS rank: ids/labels of its local tokens (rows x S/sp,
 * row-major), positions of ALL rows*S tokens of its sequences (position
 * within sample), cu_seqlens over those rows*S tokens (packing.hpp:28
 * convention), and the global supervised-token count.  With gradient
 * accumulation (global_batch = k*dp_width*micro_batch, step_graph.cpp:57)
 * "rows" is k*micro_batch: micro-batch j is rows [j*m, (j+1)*m) of the
 * arrays, and n_valid counts all k micro-batches of all ranks. */
int opx_step_load_batch(opx_step* st, const int32_t* ids, const int32_t* labels,
                        const int32_t* positions, const int32_t* cu_seqlens, int n_cu,
                        int64_t n_valid_global);
/* Frozen omni-modal encoder inputs (step_graph.cpp:141-166):
 * the n_items image items placed in THIS rank's micro-batch rows, sorted by
 * (row, position): rows[j] (0-based within the micro-batch), positions[j] =
 * first of its tokens_per_item placeholder tokens in that row, and bf16
 * patches [n_items, 4*tokens_per_item, patch_width].  Each SP rank encodes
 * items j % sp == its SP index and stores the features to the ranks owning
 * the placeholder positions.  Call after opx_step_load_batch, before run. */
int opx_step_load_images(opx_step* st, const void* pixels_bf16, int n_items, const int32_t* rows,
                         const int32_t* positions);
int opx_step_run(opx_step* st, opx_step_report* rep);
/* FSDP flat-shard checkpoint: every unit's fp32 master /
 * exp_avg / exp_avg_sq shards in the executor's chunked layout plus a
 * manifest; replaces the reference's on-disk step state that `omniplan
 * reshard` plans move between world sizes (reshard.cpp:20-56, cli.cpp:422-496).
 * Collective in spirit: every rank calls it; synchronise ranks around it. */
int opx_step_save(opx_step* st, const char* dir);
/* Loads a checkpoint saved with the same shard counts (reshard it first with
 * paper_2508_02317_b200/checkpoint.py otherwise); bf16 params = round(master). */
int opx_step_load(opx_step* st, const char* dir);
/* Copies a named tensor to host. Names: "param:<name>", "grad:<name>",
 * "master:<name>", "exp_avg:<name>", "exp_avg_sq:<name>", "loss_rows".
 * <name> follows HF naming ("model.layers.0.self_attn.q_proj.weight"). Only
 * the part this rank owns is returned for sharded tensors (see opx_step_tensor_info). */
int opx_step_get(opx_step* st, const char* name, void* host_dst, size_t bytes);
/* Describes a named tensor: numel, and the [begin,end) element interval of the
 * flattened logical tensor held by this rank. */
int opx_step_tensor_info(opx_step* st, const char* name, int64_t* numel, int64_t* begin,
                         int64_t* end);
/* The last step's report as to_json(StepReport) (report.cpp:117-128):
 * {"step_time_s","throughput_tokens_per_s_per_gpu","mfu","exposed_comm_fraction",
 *  "model_flops_per_token","phase_breakdown":{phase:{"compute_s","comm_s"}}}
 * with phase names from step_graph.cpp (fwd.layer<i>, bwd.layer<i>, fwd.head,
 * bwd.head, encoder, optimizer).  len receives strlen; cap must exceed it. */
int opx_step_report_json(opx_step* st, char* out_json, size_t cap, size_t* len);
/* exposed_comm_seconds (simulator.cpp:71-104; replaces its private helper,
 * used by report() at simulator.cpp:118): seconds of the comm intervals
 * [comm_start[i], comm_end[i]) that no compute interval covers.  Intervals may
 * overlap or nest (several streams).  Host-only, no GPU; the step's
 * exposed_comm / comm_wait_s are this over its measured node intervals. */
double opx_exposed_comm_seconds(const double* compute_start, const double* compute_end,
                                int64_t n_compute, const double* comm_start,
                                const double* comm_end, int64_t n_comm);
/* Chrome trace of the last step in simulator.cpp:133-151's schema. */
int opx_step_trace(opx_step* st, char* out_json, size_t cap, size_t* len);
int opx_step_destroy(opx_step* st);

/* ------------------------------------------------------------------------
 * Kernel-level entry points (device pointers, cudaStream_t as void*).
 * ------------------------------------------------------------------------ */
/* D = A . B^T (see csrc/runtime/gemm_api.h for layouts and epilogues).
 * epi 5 (SwiGLU backward): acc = dact [M, N]; D2/ldd2 pass the forward's bf16
 * gate|up [M, 2N] (input); D receives d(gate)|d(up) [M, 2N] in the same layout. */
int opx_gemm(int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B,
             int64_t ldb, int b_mn, int epi, void* D, int64_t ldd, const float* R, int64_t ldr,
             void* D2, int64_t ldd2, float scale, void* stream);
int opx_gemm_grouped(int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B,
                     int64_t ldb, int b_mn, int epi, void* D, int64_t ldd, void* D2,
                     int64_t ldd2, int groups, int grouped_k, const int* g_start,
                     const int* g_rows, int64_t rows_total, int64_t d_group_stride,
                     void* stream);
int opx_rmsnorm_fwd(const float* x, const void* w, void* y, float* rstd, int T, int H, float eps,
                    void* stream);
int opx_rmsnorm_bwd(const float* dy, const float* x, const void* w, const float* rstd,
                    const float* dres, float* dx, float* dw_part, float* dw, int T, int H,
                    void* stream);
int opx_rmsnorm_bwd_parts(int T);
int opx_ce_fwd_bwd(void* logits, int64_t ldl, const int32_t* labels, float* loss, int T, int V,
                   float inv_n, void* stream);
int opx_swiglu_bwd(const void* dact, const void* gu, void* dgu, int64_t T, int F, void* stream);
int opx_adamw(float* p, float* m, float* v, const float* g, void* pb, int64_t n, float lr,
              float b1, float b2, float eps, float wd, int step, void* stream);
int opx_embed_fwd(const int32_t* ids, const void* E, float* x, int T, int H, void* stream);
int opx_embed_bwd(const int32_t* ids, const float* dx, float* dE, int T, int H, void* stream);
int opx_init_param(float* f32, void* b16, int64_t n, int64_t phys0, uint64_t key_a,
                   uint64_t key_b, double c, float constant, int interleave,
                   int64_t rows_per_slab, int64_t cols, void* stream);
uint64_t opx_param_key(const char* name, uint64_t seed);
/* Causal varlen GQA attention (tcgen05/TMEM), head_dim 128, layouts in kernels_api.h. */
int opx_attn_fwd_tc(const void* q, const void* k, const void* v, void* o, float* lse,
                    int64_t ldq, int64_t ldk, int64_t ldv, int64_t ldo, const int32_t* seq_start,
                    const int32_t* seq_end, int N, int hq, int hk, float scale, void* stream);
/* Bidirectional varlen attention (keys [seq_start[t], seq_end[t])), the frozen
 * encoder's self-attention (step_graph.cpp:141-166). */
int opx_attn_fwd_bidir_tc(const void* q, const void* k, const void* v, void* o, float* lse,
                          int64_t ldq, int64_t ldk, int64_t ldv, int64_t ldo,
                          const int32_t* seq_start, const int32_t* seq_end, int N, int hq, int hk,
                          float scale, void* stream);
int opx_attn_bwd_tc(const void* q, const void* k, const void* v, const void* o, const float* lse,
                    const void* dout, float* dq_acc, void* dk, void* dv, float* delta,
                    int64_t ld_q, int64_t ld_kv, const int32_t* seq_start, const int32_t* seq_end,
                    int N, int hq, int hk, float scale, void* stream);
/* Same backward with fp32 dense [N, hk, 128] dK/dV outputs; each GQA group is
 * split across kv_splits CTAs (0 = automatic) whose partials are summed by TMA
 * bulk reduce-add.  This is the form the training step uses. */
int opx_attn_bwd_tc_f32kv(const void* q, const void* k, const void* v, const void* o,
                          const float* lse, const void* dout, float* dq_acc, float* dk_acc,
                          float* dv_acc, float* delta, int64_t ld_q, int64_t ld_kv,
                          const int32_t* seq_start, const int32_t* seq_end, int N, int hq, int hk,
                          float scale, int kv_splits, void* stream);
/* Sequence packing (packing.cpp:10-83 pack + padding_ratio): first fit of
 * samples (ids may be NULL -> 0..n-1) toward `target` tokens; policy 0 = first
 * fit decreasing (ties by ascending id), 1 = arrival order.  Writes
 * {"rows":[{"capacity","entries":[[id,offset,length],..],"boundaries":[..]}],
 *  "padding_ratio":x}; an over-length sample returns 2 (PackError's message). */
int opx_pack(const int64_t* ids, const int64_t* lengths, int64_t n, int64_t target, int policy,
             char* out_json, size_t cap);
/* Reshard copy plan for one flat parameter (reshard.cpp:20-56 make_plan):
 * rank r of a layout owns [min(r*c, numel), min((r+1)*c, numel)) with
 * c = ceil(numel/parts) when align == 0 (the reference) or
 * c = round_up(numel, align*parts)/parts (the executor's FSDP units, align 64).
 * Writes {"numel","src_chunk","dst_chunk","ops":[[src_rank,src_off,dst_rank,dst_off,len],..]}
 * ordered by (dst_rank, dst_offset); verified like reshard.cpp:58-110. */
int opx_reshard_plan(int64_t numel, int64_t src_parts, int64_t src_align, int64_t dst_parts,
                     int64_t dst_align, char* out_json, size_t cap);
/* Single-rank Ulysses relayout (sp == 1 path) with RoPE, for testing. */
int opx_rope_pack(const void* qkv, int64_t ld, void* q_full, void* k_full, void* v_full,
                  int hq, int hk, int rows, int S, const int32_t* pos, const float* inv_freq,
                  void* stream);

/* Ulysses exchanges as NVLink peer stores (kernels/a2a.cu), the kernels
 * behind VeOmni's gather_seq_scatter_heads / gather_heads_scatter_seq
 * (step_graph.cpp:224-239 a2a_q/k/v, a2a_out).
 * seq2head: this SP rank's [rows*S/sp, (hq+2hk)*hd] q|k|v rows (row stride ld)
 * go to every rank j's [rows*S, h/sp, 128] head-layout buffers q_dst[j],
 * k_dst[j], v_dst[j] (device pointers, host arrays of sp entries; peers via
 * CUDA IPC or peer access), RoPE on q/k when pos (global position ids [rows*S])
 * and inv_freq ([hd/2]) are given.  head2seq: this rank's [rows*S, hq/sp, 128]
 * attention output back to the token owners' [rows*S/sp, hq*hd] rows dst[j]. */
int opx_ulysses_seq2head(const void* qkv, int64_t ld, void* const* q_dst, void* const* k_dst,
                         void* const* v_dst, int sp, int rank, int rows, int S, int hq, int hk,
                         int hd, const int32_t* pos, const float* inv_freq, void* stream);
int opx_ulysses_head2seq(const void* o_heads, void* const* dst, int64_t ld, int sp, int rank,
                         int rows, int S, int hq, int hd, void* stream);

/* MoE routing (moe.cu): fp32 router logits with a fixed sequential K order, each
 * step one rounding of acc + h*w (the bf16 x bf16 product is exact), top-k with lower-index tie break, weights =
 * softmax renormalised over the selected experts (Qwen3 norm_topk_prob). */
int opx_moe_route(const void* h, const void* w_router, int T, int H, int E, int k,
                  float* logits, int32_t* topk_idx, float* topk_w, void* stream);
/* Stable counting sort of the T*k (token, slot) pairs by expert: pos_of_pair[p]
 * is the sorted position of pair p = t*k + j, pair_at[pos] its inverse,
 * counts/excl the per-expert counts and exclusive offsets.  hist needs
 * opx_moe_sort_chunks(P) * E ints of scratch. */
int opx_moe_sort_chunks(int P);
int opx_moe_sort(const int32_t* topk_idx, int P, int E, int32_t* hist, int32_t* counts,
                 int32_t* excl, int32_t* pos_of_pair, int32_t* pair_at, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* OPX_H */
