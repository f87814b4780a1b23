// The training-step executor behind opx_step_* (the measured counterpart of
// omniplan's build_step_graph + simulate, step_graph.cpp:441-448 /
// simulator.cpp:14-65).
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <map>
#include <string>
#include <vector>

#include "../host/plan.hpp"
#include "kernels_api.h"
#include "opx.h"

namespace opx {

using bf16 = __nv_bfloat16;

struct ExecCfg {
  uint64_t seed = 2508;
  float lr = 1e-4f, b1 = 0.9f, b2 = 0.95f, eps = 1e-8f, wd = 0.1f;
  double rope_theta = 1e6;
  float rms_eps = 1e-6f;
  int64_t ce_chunk = 8192;
  bool trace = true;  // node events for the report (exposed comm, phases) and the chrome trace
  // recompute=full: keep the attention activations of as many dense layers as
  // free HBM allows (their backward recomputes only gate|up)
  bool selective_recompute = true;
  // bf16 gradients for layer / expert units (the reference's memory model,
  // memory.cpp; halves gradient HBM and reduce-scatter bytes)
  bool bf16_grads = true;
};

// One parameter inside an FSDP flat unit.  `phys_name` is the name exposed by
// opx_step_get; `interleave` marks a [2F, H] gate|up matrix stored as 128-row
// interleaved blocks (logical names key_a = gate, key_b = up).
struct Param {
  std::string name;
  int64_t off = 0, numel = 0;
  std::vector<int64_t> shape;
  bool ones = false;
  int interleave = 0;
  std::string key_a, key_b;
  int64_t rows_per_slab = 0, cols = 0;
  int64_t logical_offset = 0;  // element offset of this slab in the logical tensor (experts)
  int64_t logical_numel = 0;   // numel of the logical tensor (0: same as numel)
};

// FSDP unit: a flat parameter buffer sharded over `P` ranks with the
// reference's ceil-chunk convention (reshard.cpp:11-18) applied to the
// numel padded to a multiple of 64*P.
struct Unit {
  std::string name;
  std::vector<Param> params;
  int64_t numel = 0, padded = 0, shard = 0;
  int P = 1, idx = 0;          // shard-group size and this rank's index in it
  ncclComm_t comm = nullptr;   // shard group
  ncclComm_t rep_comm = nullptr;  // HSDP replicate group (nullptr if none)
  float *master = nullptr, *m = nullptr, *v = nullptr;
  // gradients: fp32, or bf16 when gbf (layer and expert units: halves their
  // memory and reduce-scatter bytes; the head keeps fp32 for its scatter-add
  // embedding gradient and chunk-accumulated LM-head gradient)
  void* gshard = nullptr;
  bool gbf = false;
  size_t gbytes() const { return gbf ? 2 : 4; }
  void* gat(void* base, int64_t off) const { return static_cast<char*>(base) + off * int64_t(gbytes()); }
  // gradient accumulation (accum_steps > 1): fp32 sum of the micro-batches'
  // shard gradients; AdamW and the HSDP all-reduce read it after the last one
  float* gacc = nullptr;
  bf16* pshard = nullptr;
  bf16* full = nullptr;        // gathered params (alias of pshard when P == 1)
  void* gfull = nullptr;       // full-layout grads (alias of gshard when P == 1)
  const Param* find(const std::string& n) const {
    for (auto& p : params)
      if (p.name == n) return &p;
    return nullptr;
  }
};

// One measured node: name / phase follow step_graph.cpp (a16); tid is the
// stream it ran on (0 compute, 1 FSDP comm, 2 optimizer, 3/4 MoE side
// streams); comm marks the reference's collective nodes (NCCL gathers and
// reduce-scatters, Ulysses and EP exchanges incl. their flag barriers);
// span marks an enclosing interval that is not a busy node of its own.
struct TraceEv {
  std::string name, phase;
  int tid;
  cudaEvent_t a, b;
  bool comm = false, span = false;
  std::string fused;  // names of the reference nodes a fused exchange stands for
};

class Step {
 public:
  ~Step();
  int create(const Cluster& c, const Model& m, const Workload& w, const Plan& p, const ExecCfg& ex,
             int rank, int device, const void* nccl_id);
  int ipc_export(void* out, size_t cap, size_t* len);
  int ipc_import(const void* all, size_t len_per_rank);
  int init_weights(uint64_t seed);
  int load_batch(const int32_t* ids, const int32_t* labels, const int32_t* pos, const int32_t* cu,
                 int n_cu, int64_t n_valid);
  // frozen encoder inputs (step_encoder.cpp): bf16 patches [n, 4*tpi, pd] of
  // the n items placed in this rank's micro-batch rows, sorted by (row, pos)
  int load_images(const uint16_t* pixels, int n, const int32_t* row, const int32_t* pos);
  int run(opx_step_report* rep);
  int save(const std::string& dir);  // checkpoint.cpp
  int load(const std::string& dir);
  int get(const std::string& name, void* dst, size_t bytes);
  int info(const std::string& name, int64_t* numel, int64_t* b, int64_t* e);
  std::string trace_json();
  // to_json(StepReport) keys (report.cpp:117-128) of the last step
  std::string report_json();

 private:
  // ---- configuration
  Cluster c_;
  Model m_;
  Workload w_;
  Plan p_;
  Arch a_;
  ExecCfg ex_;
  int rank_ = 0, world_ = 1, dev_ = 0;
  int rep_i_ = 0, shard_i_ = 0, sp_i_ = 0;
  std::vector<int64_t> sp_members_, shard_members_, rep_members_;
  int rows_ = 1, S_ = 1, S_loc_ = 1, T_ = 1, Ntok_ = 1;
  bool relay_ = false;  // head-layout relayout needed (sp > 1 or head_dim < 128)
  int H_ = 0, d_ = 128, hq_ = 0, hk_ = 0, hql_ = 0, hkl_ = 0, Wqkv_ = 0, F_ = 0, V_ = 0;
  int step_count_ = 0;
  int64_t n_valid_ = 1;
  // gradient accumulation (step_graph.cpp:57): micro-batches per step, the
  // one being executed, and its trace suffix (".m<k>", step_graph.cpp:133-135)
  int accum_ = 1, mb_ = 0;
  bool last_mb() const { return mb_ == accum_ - 1; }
  std::string mtag() const { return ".m" + std::to_string(mb_); }
  // final gradient of a unit's shard for this micro-batch is ready on stream s:
  // accumulate, and on the last micro-batch HSDP all-reduce + AdamW
  int unit_grad_ready(Unit& u, cudaStream_t s, const std::string& name, int layer);
  int64_t bytes_alloc_ = 0;

  // ---- streams, comms, events
  cudaStream_t cs_ = nullptr, ms_ = nullptr;
  // optimizer stream: each unit's AdamW runs as soon as its gradient is final
  // (after its reduce-scatter), overlapping the rest of the backward
  cudaStream_t os_ = nullptr;
  int opt_unit(Unit& u, cudaStream_t after, const std::string& name);
  ncclComm_t world_comm_ = nullptr, shard_comm_ = nullptr, rep_comm_ = nullptr,
             shard_comm_head_ = nullptr;
  cudaEvent_t ev_start_ = nullptr, ev_fwd_ = nullptr, ev_bwd_ = nullptr, ev_end_ = nullptr;
  std::vector<cudaEvent_t> ev_mb_;  // [2*accum]: forward end / backward end of each micro-batch
  std::vector<cudaEvent_t> ev_ag_, ev_use_done_, ev_grad_done_, ev_rs_done_;
  cudaEvent_t ev_head_ag_ = nullptr, ev_head_rs_ = nullptr;
  std::vector<TraceEv> trace_;
  std::vector<cudaEvent_t> ev_pool_;
  size_t ev_next_ = 0;

  // ---- parameters
  std::vector<Unit> units_;  // [0] head, [1+l] layer l
  std::vector<bf16*> gslot_;     // gathered-param slots (P > 1)
  std::vector<void*> gradslot_;  // full-grad slots (P > 1; bf16 when ExecCfg::bf16_grads)
  int nslots_ = 2;

  // ---- peer-visible arena (Ulysses exchanges)
  char* arena_ = nullptr;
  size_t arena_bytes_ = 0;
  std::vector<char*> peer_arena_;  // by world rank
  std::vector<cudaIpcMemHandle_t> opened_;
  size_t off_flags_ = 0, off_do_[2] = {0, 0}, off_dqkv_[2] = {0, 0};
  // q/k/v (head layout) and o (token layout) exchange buffers: slots 0..1 are
  // the double buffer used by recomputed layers; with recompute=none layer l
  // keeps its own slot 2+l until its backward.
  std::vector<size_t> off_q_, off_k_, off_v_, off_o_;
  uint32_t** d_peer_flags_ = nullptr;  // device array [sp] of peer flag pointers
  int* d_timeout_ = nullptr;
  int* d_agree_ = nullptr;  // scratch of the setup-time agreement reductions (allocated before any collective)
  uint32_t epoch_ = 0;
  int xq_ = 0, xo_ = 0, xdo_ = 0, xd_ = 0;  // double-buffer selectors

  // ---- batch
  // d_* point at the current micro-batch inside the *_all_ arrays (accum_ of each)
  int32_t *d_ids_ = nullptr, *d_labels_ = nullptr, *d_pos_ = nullptr, *d_sstart_ = nullptr,
          *d_send_ = nullptr;
  int32_t *d_ids_all_ = nullptr, *d_labels_all_ = nullptr, *d_pos_all_ = nullptr,
          *d_sstart_all_ = nullptr, *d_send_all_ = nullptr;
  void bind_micro(int mb) {
    mb_ = mb;
    d_ids_ = d_ids_all_ + int64_t(mb) * T_;
    d_labels_ = d_labels_all_ + int64_t(mb) * T_;
    d_pos_ = d_pos_all_ + int64_t(mb) * Ntok_;
    d_sstart_ = d_sstart_all_ + int64_t(mb) * Ntok_;
    d_send_ = d_send_all_ + int64_t(mb) * Ntok_;
  }
  float* d_inv_freq_ = nullptr;

  // ---- activations
  // Per-layer forward activations needed by the backward.  recompute=full
  // (plan.hpp:32 default) keeps one scratch set and recomputes each layer in
  // the backward; recompute=none keeps a set per layer (dense layers).
  struct Acts {
    bf16 *h = nullptr, *h2 = nullptr, *gu = nullptr, *act = nullptr, *ofull = nullptr;
    float *x2 = nullptr, *r1 = nullptr, *r2 = nullptr, *lse = nullptr;
  };
  Acts scratch_;
  std::vector<Acts> saved_;
  bool save_acts_ = false;
  // recompute=none keeps every layer's forward activations; MoE layers keep
  // the attention activations, their routing and the combined expert outputs
  // and only re-run dispatch + gate|up in the backward (moe_bwd).
  // per-layer: 0 = recompute the whole layer, 1 = attention state kept (the
  // backward recomputes the norms, the output projection and gate|up, not
  // q/k/v nor attention), 2 = everything kept
  std::vector<int> keep_mode_;
  bool keeps_acts(int l) const { return keep_mode_[size_t(l)] >= 1; }
  bool keeps_mlp(int l) const { return keep_mode_[size_t(l)] == 2; }
  // saved activations of layer l; a mode-1 layer keeps only its attention
  // state (q/k/v/o slot, lse, head-layout output) and borrows the scratch
  // buffers for everything its backward recomputes
  void bind_layer(int l) {
    bind(saved_[size_t(l)]);
    if (!keeps_mlp(l)) {
      h_ = scratch_.h;
      h2_ = scratch_.h2;
      x2_ = scratch_.x2;
      r1_ = scratch_.r1;
      r2_ = scratch_.r2;
      gu_ = scratch_.gu;
      act_ = scratch_.act;
    }
  }
  void bind(const Acts& a) {
    h_ = a.h;
    h2_ = a.h2;
    gu_ = a.gu;
    act_ = a.act;
    ofull_ = a.ofull;
    x2_ = a.x2;
    r1_ = a.r1;
    r2_ = a.r2;
    lse_ = a.lse;
  }
  int next_rslot() {
    xq_ ^= 1;
    return xq_;
  }
  bool store_gu_ = false;
  std::vector<float*> x_saved_;  // layer inputs [L+1][T,H] fp32 (x_saved_[L] = final)
  float2* d_rope_ = nullptr;  // [S][d/2] (sin, cos)
  bool rope_tab_ok_ = true;   // every position id of the batch is < S
  bf16 *h_ = nullptr, *qkv_ = nullptr, *ofull_ = nullptr, *h2_ = nullptr, *gu_ = nullptr,
       *act_ = nullptr;
  float *x2_ = nullptr, *r1_ = nullptr, *r2_ = nullptr, *lse_ = nullptr;
  // backward scratch
  float *dx_ = nullptr, *dtmp_ = nullptr, *dq_acc_ = nullptr, *delta_ = nullptr,
        *dw_part_ = nullptr;
  bf16 *dxb_ = nullptr, *dact_ = nullptr, *dgu_ = nullptr;
  float *dk_ = nullptr, *dv_ = nullptr;  // fp32 dK/dV (split-GQA reduce-add)
  // head
  bf16 *hf_ = nullptr, *logits_ = nullptr;
  float *rf_ = nullptr, *dhf_ = nullptr, *loss_rows_ = nullptr, *loss_sum_ = nullptr;

  // ---- helpers
  template <class T>
  T* alloc(size_t n, bool zero = true);
  std::vector<void*> allocs_;
  cudaEvent_t ev();
  void mark(const std::string& name, const std::string& phase, int tid, cudaEvent_t a,
            cudaEvent_t b, const char* fused = nullptr);
  // measured StepReport of the last step (simulator.cpp:106-131 on real intervals)
  opx_step_report last_{};
  std::map<std::string, std::pair<double, double>> phases_;  // phase -> (compute_s, comm_s)
  void measure_nodes(opx_step_report* r);
  int build_units();
  int alloc_acts();
  int gather(Unit& u, int slot, cudaEvent_t wait_ev);
  bf16* q_full(int b) { return reinterpret_cast<bf16*>(arena_ + off_q_[b]); }
  bf16* k_full(int b) { return reinterpret_cast<bf16*>(arena_ + off_k_[b]); }
  bf16* v_full(int b) { return reinterpret_cast<bf16*>(arena_ + off_v_[b]); }
  bf16* o_loc(int b) { return reinterpret_cast<bf16*>(arena_ + off_o_[b]); }
  bf16* do_full(int b) { return reinterpret_cast<bf16*>(arena_ + off_do_[b]); }
  bf16* dqkv_loc(int b) { return reinterpret_cast<bf16*>(arena_ + off_dqkv_[b]); }
  char* peer(int sp_j, size_t off) {
    return (sp_j == sp_i_ ? arena_ : peer_arena_[size_t(sp_members_[size_t(sp_j)])]) + off;
  }
  int barrier_sp(cudaStream_t s);
  // async_ulysses: the seq->head exchanges ride in the producing GEMM's
  // epilogue (GEMM_EPI_SEQ2HEAD; head_dim 128 only, else the exchange kernel)
  bool async_s2h() const { return p_.async_ulysses && d_ == 128; }
  // layer pieces
  int layer_fwd(int l, const Unit& u, const float* x_in, float* x_out, int slot);
  int layer_bwd(int l, Unit& u, void* grads);
  int head_fwd_bwd(Unit& u, float* grads);
  // ---- frozen omni-modal encoder (step_encoder.cpp)
  struct Enc {
    bool on = false;
    std::string name;
    int He = 0, L = 0, heads = 0, d = 0, F = 0, pd = 0, tpi = 0;
    // FSDP units of the frozen module (plan.cpp:95-107 shards every module):
    // [0] patch embed, [1 + i] block i (params: norm1 | qkv | qkv bias | proj |
    // proj bias | norm2 | gate_up | gate_up bias (128-interleaved like the
    // weight) | down | down bias), [L + 1] merger (ln_q | mlp.0 | bias | mlp.2 |
    // bias).  Each rank keeps its bf16 shard only (no optimizer state); the
    // forward all-gathers unit i + 2 into slot i % 2 while unit i computes.
    static constexpr int kBlk = 10;
    std::vector<Unit> units;
    bf16* slot[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> ev_ag, ev_use;
    const bf16* wp(int unit, int param) const {
      const Unit& u = units[size_t(unit)];
      return u.full + u.params[size_t(param)].off;
    }
    // Qwen2.5-VL geometry: g x g patches per item, windows of window_merge^2
    // merge units, full-attention blocks, 2-D RoPE (sin, cos) per patch of an
    // item in window order [P][d/2]
    int g = 0, window_merge = 4;
    std::vector<char> fullatt;
    std::vector<int> worder;  // merge units in window order (get_window_index)
    std::vector<int> wlens;   // window lengths in patches
    double rope_theta = 1e4;
    float2* rope = nullptr;
    int cap = 0, n_loc = 0, n_all = 0;  // items: buffer capacity, encoded here, in the micro-batch
    bf16 *pix = nullptr, *h = nullptr, *qkv = nullptr, *q = nullptr, *k = nullptr, *v = nullptr,
         *o = nullptr, *o2 = nullptr, *act = nullptr, *y1 = nullptr, *feat = nullptr;
    float *x = nullptr, *rstd = nullptr, *lse = nullptr;
    // per patch row: item span (full attention), window span, RoPE row (i % P)
    int *st = nullptr, *en = nullptr, *wst = nullptr, *wen = nullptr, *rpos = nullptr,
        *dst_rank = nullptr, *dst_tok = nullptr;
    std::vector<void*> bufs;  // item-sized buffers (re-allocated when cap grows)
  } enc_;
  int* d_fmask_ = nullptr;  // [T] local tokens replaced by encoder features
  size_t off_feat_ = 0;     // arena: [T, H] bf16 feature rows written by the SP peers
  int enc_setup();
  int enc_alloc(int items);
  int enc_init_weights(uint64_t seed);
  int enc_forward();  // encoder fwd + scatter into the SP group + inject (cs_)
  // ---- MoE / expert parallelism (step_moe.cpp)
  bool moe_ = false;
  int E_ = 0, topk_ = 0, Fe_ = 0, El_ = 0, ep_ = 1, ep_i_ = 0, De_ = 1;
  std::vector<int64_t> ep_members_;
  ncclComm_t expert_comm_ = nullptr;
  std::vector<Unit> expert_units_;  // [layer]; empty params for dense layers
  bf16* eslot_ = nullptr;           // expert gather buffer (De > 1)
  void* egrad_slot_ = nullptr;      // expert full-grad buffer (De > 1)
  int64_t cap_rows_ = 0;            // receive-buffer rows (worst case)
  size_t off_flags_ep_ = 0, off_xrecv_ = 0, off_dyrecv_ = 0, off_dxback_ = 0;
  // routing state + the peer-written count table and combine buffer: slot 0 is
  // scratch (recomputed layers), slot 1 + l belongs to MoE layer l under recompute=none
  struct MoeRoute {
    float* wts = nullptr;
    int *idx = nullptr, *pos = nullptr, *pairat = nullptr, *cnt = nullptr, *excl = nullptr,
        *g_start = nullptr, *g_rows = nullptr, *g_rows_pad = nullptr, *g_total = nullptr;
  };
  std::vector<MoeRoute> routes_;        // [slot]
  std::vector<size_t> off_counts_s_;    // [slot]
  std::vector<size_t> off_yback_s_;     // [slot]
  int rslot_ = 0;
  void moe_bind(int l);                 // select slot 1+l (l >= 0) or scratch (l < 0)
  int* counts_cur() { return reinterpret_cast<int*>(arena_ + off_counts_s_[size_t(rslot_)]); }
  bf16* yback_cur() { return reinterpret_cast<bf16*>(arena_ + off_yback_s_[size_t(rslot_)]); }
  int** count_tab_cur() { return d_count_tables_ + size_t(rslot_) * kMaxSp; }
  bf16** yback_tab_cur() { return d_yback_peers_ + size_t(rslot_) * kMaxSp; }
  uint32_t** d_ep_flags_ = nullptr;
  // recompute=none MoE backward: the token re-send of layer l runs on xs_ with
  // its own barrier flags while the compute stream finishes the layer above
  cudaStream_t xs_ = nullptr;
  size_t off_flags_ep2_ = 0;
  uint32_t** d_ep_flags2_ = nullptr;
  uint32_t epoch_ep2_ = 0;
  // moe_overlap: the second expert half of the forward runs on xs2_ with its own
  // barrier flag set
  cudaStream_t xs2_ = nullptr;
  size_t off_flags_ep3_ = 0;
  uint32_t** d_ep_flags3_ = nullptr;
  uint32_t epoch_ep3_ = 0;
  int barrier_ep3(cudaStream_t s);
  std::vector<cudaEvent_t> ev_redisp_;  // [layer]
  int moe_redispatch(int l);            // issue on xs_ after the caller's cs_ point
  int next_moe_below(int l) const {
    for (int j = l - 1; j >= 0; --j)
      if (a_.is_moe_layer(j)) return j;
    return -1;
  }
  int** d_count_tables_ = nullptr;
  bf16** d_xrecv_peers_ = nullptr;  // [1 + L][kMaxSp]: slot 0 shared, 1 + l kept by layer l
  // recompute=none: layers whose dispatched tokens stay in their own arena
  // slot until the backward (no re-send on xs_), chosen by free HBM at setup
  std::vector<size_t> off_xrecv_l_;  // [L], 0 = uses the shared buffer
  bool keeps_x(int l) const { return l >= 0 && size_t(l) < off_xrecv_l_.size() && off_xrecv_l_[size_t(l)]; }
  bf16* xrecv_of(int l) { return reinterpret_cast<bf16*>(arena_ + (keeps_x(l) ? off_xrecv_l_[size_t(l)] : off_xrecv_)); }
  bf16** xrecv_peers_of(int l) { return d_xrecv_peers_ + (keeps_x(l) ? size_t(1 + l) * kMaxSp : 0); }
  // ... and, while HBM allows, their gate|up pre-activations and SwiGLU output
  // (the backward then skips the gate|up recompute)
  std::vector<bf16*> gu_l_, act_l_;  // [L]
  bool keeps_gu(int l) const { return l >= 0 && size_t(l) < gu_l_.size() && gu_l_[size_t(l)]; }
  bf16** d_yback_peers_ = nullptr;
  bf16** d_dyrecv_peers_ = nullptr;
  bf16** d_dxback_peers_ = nullptr;
  uint32_t epoch_ep_ = 0;
  bool in_recompute_ = false;       // layer_fwd called from layer_bwd
  std::vector<int*> route_idx_;     // [layer] forward top-k indices (T*k), for parity checks
  float *r_logits_ = nullptr, *r_wts_ = nullptr, *r_dw_ = nullptr, *r_logits_part_ = nullptr;
  int *r_idx_ = nullptr, *r_pos_ = nullptr, *r_pairat_ = nullptr, *r_cnt_ = nullptr,
      *r_excl_ = nullptr, *r_hist_ = nullptr, *g_start_ = nullptr, *g_rows_ = nullptr,
      *g_rows_pad_ = nullptr, *g_total_ = nullptr;
  float* wr_part_ = nullptr;          // split-K partials of the router wgrad
  int *rm_cnt_ = nullptr, *rm_off_ = nullptr;  // [El][ep] combine map (GEMM_EPI_ROWMAP)
  int* wr_gs_ = nullptr;              // chunk starts / rows for the split
  int* wr_gr_ = nullptr;
  int wr_split_ = 1;
  bf16 *gu_e_ = nullptr, *act_e_ = nullptr, *y_e_ = nullptr, *dact_e_ = nullptr, *dgu_e_ = nullptr,
       *dx_e_ = nullptr, *dyp_ = nullptr, *dlogits_ = nullptr;
  char* ep_peer(int j, size_t off) {
    return (j == ep_i_ ? arena_ : peer_arena_[size_t(ep_members_[size_t(j)])]) + off;
  }
  int moe_setup_groups();      // in create(), before build_units
  int moe_build_units();       // expert units
  int moe_arena(size_t* off);   // reserve arena regions (advances *off); ranks agree on the layout
  int moe_alloc();             // local scratch
  int moe_import();            // peer tables after ipc import
  int barrier_ep(cudaStream_t s);
  int moe_fwd(int l, const Unit& u, const Unit& eu, const float* x2, float* x_out);
  int moe_bwd(int l, const Unit& u, Unit& eu, void* G, void* Ge, float* dh2);
  struct CkptUnit {
    std::string name;
    Unit* u;
  };
  std::vector<CkptUnit> ckpt_units();
  int check(cudaError_t e, const char* what);
  int nccl(ncclResult_t r, const char* what);
};

template <class T>
T* Step::alloc(size_t n, bool zero) {
  void* p = nullptr;
  const size_t bytes = (n * sizeof(T) > 256 ? n * sizeof(T) : 256);
  if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
  if (zero) cudaMemset(p, 0, bytes);
  allocs_.push_back(p);
  bytes_alloc_ += int64_t(bytes);
  return static_cast<T*>(p);
}

}  // namespace opx
