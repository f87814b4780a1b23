// Training-step executor: one instance per rank (process / GPU).
//
// Executes, with real kernels and collectives, the per-layer schedule that
// omniplan's GraphBuilder only models (step_graph.cpp:75-409):
//   fwd:  AG(layer) on the comm stream, prefetched one layer ahead
//         (issue_gather, :179-189) -> norm -> QKV GEMM -> seq->head a2a (+RoPE)
//         -> attention -> head->seq a2a -> out GEMM(+residual) -> norm ->
//         gate|up GEMM(+SwiGLU) -> down GEMM(+residual)
//   head: final norm -> LM-head GEMM -> fused CE fwd/bwd (chunked) -> dgrad/wgrad
//   bwd:  per layer (high to low) full recompute of the layer (recompute=full,
//         plan.hpp:32), the mirrored GEMMs, the four backward Ulysses
//         exchanges the reference model omits (test_simulator.cpp:205), grad
//         reduce-scatter on the comm stream (:351-354) + HSDP all-reduce (:356-364)
//   opt:  fused AdamW on the local fp32 shard (:392-409).
// Node names and phases follow step_graph.cpp so measured traces line up with
// the simulated ones.
#include <chrono>
#include "step.h"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <sstream>

#include "common.h"
#include "json.hpp"

namespace opx {

namespace {
constexpr int64_t kAlign = 64;
int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
}  // namespace

int Step::check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return OPX_OK;
  return cuda_fail(e, what);
}
int Step::nccl(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return OPX_OK;
  set_error(std::string(what) + ": " + ncclGetErrorString(r));
  return OPX_ERR_CUDA;
}

#define TRY(x)                  \
  do {                          \
    int rc_ = (x);              \
    if (rc_ != OPX_OK) return rc_; \
  } while (0)
#define CU(x) TRY(check((x), #x))
#define NC(x) TRY(nccl((x), #x))

cudaEvent_t Step::ev() {
  if (ev_next_ == ev_pool_.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ev_pool_.push_back(e);
  }
  return ev_pool_[ev_next_++];
}

void Step::mark(const std::string& name, const std::string& phase, int tid, cudaEvent_t a,
                cudaEvent_t b, const char* fused) {
  TraceEv t{name, phase, tid, a, b};
  // the reference's collective nodes: FSDP/HSDP NCCL ops on the comm stream,
  // the Ulysses / EP exchanges (and their flag barriers) on the compute
  // stream, the encoder feature scatter (step_graph.cpp:150-160, 215-247, 265-283)
  // (an exchange over a group of one rank is a local relayout, not a
  // collective: the reference emits no node for it, step_graph.cpp add_collective)
  auto starts = [&](const char* p) { return name.rfind(p, 0) == 0; };
  auto has = [&](const char* p) { return name.find(p) != std::string::npos; };
  const bool ep_x = has(".a2a_dispatch") || has(".a2a_combine") || has(".a2a_counts") ||
                    has(".a2a_redispatch");
  const bool a2a = has(".a2a_") && (ep_x ? ep_ > 1 : has(".a2a_wait") ? (p_.sp > 1 || ep_ > 1)
                                                                       : p_.sp > 1);
  t.comm = tid == 1 || a2a || (starts("scatter.") && p_.sp > 1) || starts("fwd.ag.") || starts("bwd.ag.") ||
           starts("bwd.rs.") || starts("bwd.ar.");
  if (fused) t.fused = fused;
  trace_.push_back(std::move(t));
}

Step::~Step() {
  if (cs_) cudaStreamSynchronize(cs_);
  if (ms_) cudaStreamSynchronize(ms_);
  if (os_) cudaStreamSynchronize(os_);
  if (xs_) cudaStreamSynchronize(xs_);
  if (xs2_) cudaStreamSynchronize(xs2_);
  for (size_t r = 0; r < peer_arena_.size(); ++r)
    if (peer_arena_[r] && peer_arena_[r] != arena_) cudaIpcCloseMemHandle(peer_arena_[r]);
  for (void* p : allocs_) cudaFree(p);
  for (auto e : ev_pool_) cudaEventDestroy(e);
  for (auto* v : {&ev_ag_, &ev_use_done_, &ev_grad_done_, &ev_rs_done_})
    for (auto e : *v) cudaEventDestroy(e);
  for (auto e : {ev_start_, ev_fwd_, ev_bwd_, ev_end_, ev_head_ag_, ev_head_rs_})
    if (e) cudaEventDestroy(e);
  for (auto e : ev_mb_)
    if (e) cudaEventDestroy(e);
  for (auto* v : {&enc_.ev_ag, &enc_.ev_use})
    for (auto e : *v)
      if (e) cudaEventDestroy(e);
  if (expert_comm_) ncclCommDestroy(expert_comm_);
  if (rep_comm_) ncclCommDestroy(rep_comm_);
  if (shard_comm_) ncclCommDestroy(shard_comm_);
  if (shard_comm_head_) ncclCommDestroy(shard_comm_head_);
  if (world_comm_) ncclCommDestroy(world_comm_);
  if (cs_) cudaStreamDestroy(cs_);
  if (ms_) cudaStreamDestroy(ms_);
  if (os_) cudaStreamDestroy(os_);
  if (xs_) cudaStreamDestroy(xs_);
  if (xs2_) cudaStreamDestroy(xs2_);
  for (auto e : ev_redisp_)
    if (e) cudaEventDestroy(e);
}

int Step::opt_unit(Unit& u, cudaStream_t after, const std::string& name) {
  if (u.params.empty()) return OPX_OK;
  cudaEvent_t ready = ev();
  CU(cudaEventRecord(ready, after));
  CU(cudaStreamWaitEvent(os_, ready, 0));
  const bool acc = accum_ > 1;  // AdamW reads the fp32 micro-batch sum
  // OPX_ADAMW_OVERLAP_BLOCKS caps the grid of the units updated while the
  // backward still runs (blocks per SM; the exposed head update keeps the
  // whole GPU).  Off by default: capping at 1-2 blocks per SM measured slower
  // (C2/EP4 176-184K vs 190K tokens/s, C1 1 GPU equal) -- the longer AdamW
  // overlaps more of the backward's HBM-bound kernels
  static const int overlap_bps =
      getenv("OPX_ADAMW_OVERLAP_BLOCKS") ? atoi(getenv("OPX_ADAMW_OVERLAP_BLOCKS")) : 0;
  const int bps = &u == &units_[0] ? 0 : overlap_bps;
  CU(k_adamw(u.master, u.m, u.v, acc ? static_cast<void*>(u.gacc) : u.gshard, acc ? 0 : u.gbf,
             u.pshard, u.shard, ex_.lr, ex_.b1, ex_.b2, ex_.eps, ex_.wd, step_count_, os_, bps));
  if (ex_.trace) {
    cudaEvent_t done = ev();
    CU(cudaEventRecord(done, os_));
    mark(name, "optimizer", 2, ready, done);
  }
  return OPX_OK;
}

// ---------------------------------------------------------------------------
// setup
// ---------------------------------------------------------------------------
int Step::create(const Cluster& c, const Model& m, const Workload& w, const Plan& p,
                 const ExecCfg& ex, int rank, int device, const void* nccl_id) {
  c_ = c;
  m_ = m;
  w_ = w;
  p_ = p;
  ex_ = ex;
  rank_ = rank;
  world_ = int(p.world());
  dev_ = device;
  const Module* f = m.foundation();
  if (!f || !f->arch) {
    set_error("model has no foundation arch");
    return OPX_ERR_CONFIG;
  }
  a_ = *f->arch;
  if (a_.head_dim > 128 || a_.head_dim % 16 || a_.hidden % 128 || a_.ffn % 128) {
    set_error("executor requires head_dim <= 128 (multiple of 16) and hidden, ffn multiples of 128");
    return OPX_ERR_CONFIG;
  }
  d_ = int(a_.head_dim);
  // attention runs on 128-wide zero-padded head vectors; a relayout between the
  // local [T, heads*d] rows and the head layout is needed for SP or d < 128
  relay_ = p.sp > 1 || d_ != 128;
  if (p.sp > kMaxSp) {
    set_error("sp > 8 is not supported (one NVSwitch domain)");
    return OPX_ERR_CONFIG;
  }
  CU(cudaSetDevice(device));
  // compute and comm streams at the highest priority, the optimizer stream at
  // the lowest: its HBM-bound AdamW blocks only fill SMs the step leaves idle
  int prio_lo = 0, prio_hi = 0;
  CU(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  CU(cudaStreamCreateWithPriority(&cs_, cudaStreamNonBlocking, prio_hi));
  CU(cudaStreamCreateWithPriority(&ms_, cudaStreamNonBlocking, prio_hi));
  CU(cudaStreamCreateWithPriority(&os_, cudaStreamNonBlocking, prio_lo));
  for (cudaEvent_t* e : {&ev_start_, &ev_fwd_, &ev_bwd_, &ev_end_, &ev_head_ag_, &ev_head_rs_})
    CU(cudaEventCreate(e));

  // mesh coordinates (plan_mesh: dp_replicate x dp_shard x sp, row-major)
  const int sp = int(p.sp), sh = int(p.dp_shard);
  sp_i_ = rank % sp;
  shard_i_ = (rank / sp) % sh;
  rep_i_ = rank / (sp * sh);
  for (int j = 0; j < sp; ++j) sp_members_.push_back((rep_i_ * sh + shard_i_) * sp + j);
  for (int j = 0; j < sh * sp; ++j) shard_members_.push_back(int64_t(rep_i_) * sh * sp + j);
  for (int j = 0; j < int(p.dp_replicate); ++j)
    rep_members_.push_back(int64_t(j) * sh * sp + shard_i_ * sp + sp_i_);

  d_agree_ = alloc<int>(4);
  if (!d_agree_) return cuda_fail(cudaErrorMemoryAllocation, "setup scratch");
  if (world_ > 1) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    // Per-layer FSDP/HSDP/EP collectives run on the comm stream beside the
    // compute kernels: cap the SMs NCCL takes (OPX_NCCL_MAX_CTAS, default 8) so
    // the overlapped GEMMs (dynamic tile tickets) keep most of the GPU.
    ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
    {
      const char* e = getenv("OPX_NCCL_MAX_CTAS");
      const int mx = e ? atoi(e) : 8;
      if (mx > 0) {
        cfg.maxCTAs = mx;
        cfg.minCTAs = std::min(mx, 4);
      }
    }
    // The head unit's gather (first in the step) and reduce-scatter (last)
    // are exposed, so they use an uncapped communicator.
    NC(ncclCommInitRank(&world_comm_, world_, id, rank_));
    if (sh * sp > 1) {
      NC(ncclCommSplit(world_comm_, rep_i_, rank_, &shard_comm_, &cfg));
      NC(ncclCommSplit(world_comm_, rep_i_, rank_, &shard_comm_head_, nullptr));
    }
    if (p.dp_replicate > 1)
      NC(ncclCommSplit(world_comm_, shard_i_ * sp + sp_i_, rank_, &rep_comm_, &cfg));
    else
      NC(ncclCommSplit(world_comm_, NCCL_SPLIT_NOCOLOR, rank_, &rep_comm_, &cfg));
  }

  // gradient accumulation: global_batch = accum * dp_width * micro_batch
  // (step_graph.cpp:57; validate's batch_divisibility guarantees the division)
  accum_ = int(w.global_batch / (p.dp_width() * p.micro_batch));
  if (accum_ < 1) {
    set_error("global_batch must be a positive multiple of dp_replicate*dp_shard*micro_batch");
    return OPX_ERR_CONFIG;
  }
  ev_mb_.resize(size_t(2 * accum_));
  for (auto& e : ev_mb_) CU(cudaEventCreate(&e));
  rows_ = int(p.micro_batch);
  S_ = int(w.seq_len);
  S_loc_ = S_ / sp;
  T_ = rows_ * S_loc_;
  Ntok_ = rows_ * S_;
  H_ = int(a_.hidden);
  hq_ = int(a_.heads);
  hk_ = int(a_.kv_heads);
  hql_ = hq_ / sp;
  hkl_ = hk_ / sp;
  Wqkv_ = (hq_ + 2 * hk_) * d_;
  F_ = int(a_.ffn);
  V_ = int(a_.vocab);
  nslots_ = int(std::max<int64_t>(p.prefetch_depth, 0)) + 1;
  if (nslots_ < 2) nslots_ = 2;
  if (a_.moe) {
    if (a_.moe->experts % 64) {
      set_error("MoE executor requires num_experts % 64 == 0");
      return OPX_ERR_CONFIG;
    }
    TRY(moe_setup_groups());
  }
  TRY(build_units());
  if (shard_comm_head_) units_[0].comm = shard_comm_head_;
  TRY(enc_setup());
  TRY(alloc_acts());
  return OPX_OK;
}

int Step::build_units() {
  const int P = int(p_.shard_degree());
  const int my = shard_i_ * int(p_.sp) + sp_i_;
  auto finish = [&](Unit& u) -> int {
    u.P = P;
    u.idx = my;
    u.comm = shard_comm_;
    u.rep_comm = p_.dp_replicate > 1 ? rep_comm_ : nullptr;
    u.padded = round_up(u.numel, kAlign * P);
    u.shard = u.padded / P;
    u.master = alloc<float>(size_t(u.shard));
    u.m = alloc<float>(size_t(u.shard));
    u.v = alloc<float>(size_t(u.shard));
    u.gshard = u.gbf ? static_cast<void*>(alloc<bf16>(size_t(u.shard)))
                     : static_cast<void*>(alloc<float>(size_t(u.shard)));
    u.pshard = alloc<bf16>(size_t(u.shard));
    if (accum_ > 1) {
      u.gacc = alloc<float>(size_t(u.shard), false);
      if (!u.gacc) {
        set_error("out of device memory for gradient accumulation shards");
        return OPX_ERR_CUDA;
      }
    }
    if (!u.master || !u.m || !u.v || !u.gshard || !u.pshard) {
      set_error("out of device memory for parameter shards");
      return OPX_ERR_CUDA;
    }
    if (P == 1) {
      u.full = u.pshard;
      u.gfull = u.gshard;
    }
    return OPX_OK;
  };
  auto add = [](Unit& u, const std::string& name, std::vector<int64_t> shape, bool ones,
                int interleave = 0, const std::string& ka = "", const std::string& kb = "") {
    Param q;
    q.name = name;
    q.shape = shape;
    q.numel = 1;
    for (auto s : shape) q.numel *= s;
    q.off = u.numel;
    q.ones = ones;
    q.interleave = interleave;
    q.key_a = ka.empty() ? name : ka;
    q.key_b = kb;
    if (interleave) {
      q.rows_per_slab = shape[shape.size() - 2];
      q.cols = shape.back();
    }
    u.numel += round_up(q.numel, 128);
    u.params.push_back(q);
  };
  const int64_t H = H_, V = V_, F = F_;
  units_.clear();
  {
    Unit u;
    u.name = "head";
    add(u, "model.embed_tokens.weight", {V, H}, false);
    add(u, "model.norm.weight", {H}, true);
    add(u, "lm_head.weight", {V, H}, false);
    TRY(finish(u));
    units_.push_back(std::move(u));
  }
  for (int l = 0; l < a_.layers; ++l) {
    Unit u;
    const std::string p = "model.layers." + std::to_string(l) + ".";
    u.name = "layer" + std::to_string(l);
    u.gbf = ex_.bf16_grads;
    add(u, p + "input_layernorm.weight", {H}, true);
    add(u, p + "self_attn.q_proj.weight", {int64_t(hq_) * d_, H}, false);
    add(u, p + "self_attn.k_proj.weight", {int64_t(hk_) * d_, H}, false);
    add(u, p + "self_attn.v_proj.weight", {int64_t(hk_) * d_, H}, false);
    add(u, p + "self_attn.o_proj.weight", {H, int64_t(hq_) * d_}, false);
    add(u, p + "post_attention_layernorm.weight", {H}, true);
    if (a_.is_moe_layer(l)) {
      add(u, p + "mlp.gate.weight", {int64_t(a_.moe->experts), H}, false);
    } else {
      add(u, p + "mlp.gate_up_proj.weight", {2 * F, H}, false, 1, p + "mlp.gate_proj.weight",
          p + "mlp.up_proj.weight");
      add(u, p + "mlp.down_proj.weight", {H, F}, false);
    }
    TRY(finish(u));
    units_.push_back(std::move(u));
  }
  if (P > 1) {
    int64_t mx = 0;
    for (size_t i = 1; i < units_.size(); ++i) mx = std::max(mx, units_[i].padded);
    for (int s = 0; s < nslots_; ++s) {
      gslot_.push_back(alloc<bf16>(size_t(mx), false));
      if (!gslot_.back()) return cuda_fail(cudaErrorMemoryAllocation, "gather slots");
    }
    for (int s = 0; s < 2; ++s) {
      gradslot_.push_back(ex_.bf16_grads ? static_cast<void*>(alloc<bf16>(size_t(mx)))
                                         : static_cast<void*>(alloc<float>(size_t(mx))));
      if (!gradslot_.back()) return cuda_fail(cudaErrorMemoryAllocation, "grad slots");
    }
    Unit& hu = units_[0];
    hu.full = alloc<bf16>(size_t(hu.padded), false);
    hu.gfull = alloc<float>(size_t(hu.padded));
    if (!hu.full || !hu.gfull) return cuda_fail(cudaErrorMemoryAllocation, "head gather");
  }
  if (moe_) TRY(moe_build_units());
  const int L = int(a_.layers);
  ev_ag_.resize(size_t(L));
  ev_use_done_.resize(size_t(L));
  ev_grad_done_.resize(size_t(L));
  ev_rs_done_.resize(size_t(L));
  for (auto* v : {&ev_ag_, &ev_use_done_, &ev_grad_done_, &ev_rs_done_})
    for (auto& e : *v) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return OPX_OK;
}

int Step::alloc_acts() {
  const size_t T = size_t(T_), H = size_t(H_), N = size_t(Ntok_);
  // peer-visible arena: flags + the Ulysses exchange buffers (double-buffered)
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += round_up(int64_t(bytes), 256);
    return o;
  };
  off_flags_ = take(64 * sizeof(uint32_t));
  const int L = int(a_.layers);
  save_acts_ = !p_.recompute_full;
  keep_mode_.assign(size_t(L), save_acts_ ? 2 : 0);
  if (!save_acts_ && ex_.selective_recompute && !moe_) {
    // bytes one attention-kept layer adds: its q/k/v/o exchange slot, the
    // sp>1 head-layout output and lse
    const size_t per_layer =
        round_up(int64_t(N * size_t(hql_) * 256), 256) + 2 * round_up(int64_t(N * size_t(hkl_) * 256), 256) +
        round_up(int64_t(T * size_t(hq_) * 256), 256) + (relay_ ? N * size_t(hql_) * 256 : 0) +
        N * size_t(hql_) * 4 + 4 * 256;
    // everything else this function and the step still allocate
    const size_t F = size_t(F_), V = size_t(V_);
    const size_t chunk = size_t(std::min<int64_t>(ex_.ce_chunk, T_));
    const size_t fixed =
        2 * (N * size_t(hql_) * 256 + 2 * N * size_t(hkl_) * 256 + T * size_t(hq_) * 256) +  // 2 slots
        2 * (N * size_t(hql_) * 256 + T * size_t(Wqkv_) * 2) +                               // dO, dqkv
        size_t(L + 1) * T * H * 4 +                                                           // x_saved
        per_layer + T * H * 12 + T * 8 + T * 2 * F * 2 + T * F * 2 +                         // scratch acts
        T * size_t(Wqkv_) * 2 + 2 * T * H * 4 + T * H * 2 + T * F * 2 + T * 2 * F * 2 +    // qkv, dx, dtmp, dxb, dact, dgu
        N * size_t(hql_) * 128 * 4 + 2 * N * size_t(hkl_) * 128 * 4 + N * size_t(hql_) * 4 +  // dq, dk, dv, delta
        size_t(k_rmsnorm_bwd_parts(T_)) * H * 4 + T * H * 2 + T * H * 4 + chunk * V * 2;    // dw_part, hf, dhf, logits
    size_t free_b = 0, total_b = 0;
    CU(cudaMemGetInfo(&free_b, &total_b));
    const size_t margin = size_t(6) << 30;  // NCCL, CUDA context growth, allocator slack
    int K = 0;
    size_t budget = free_b > fixed + margin ? free_b - fixed - margin : 0;
    K = int(std::min<size_t>(size_t(L), budget / per_layer));
    for (int l = L - K; l < L; ++l) keep_mode_[size_t(l)] = 1;  // the backward starts at the top
    budget -= size_t(K) * per_layer;
    // what is left upgrades layers to keeping everything (no gate|up recompute)
    const size_t mlp_extra = T * H * 8 + T * 8 + T * size_t(2 * F_) * 2 + T * size_t(F_) * 2 + 8 * 256;
    for (int l = L - 1; l >= L - K && budget >= mlp_extra; --l) {
      keep_mode_[size_t(l)] = 2;
      budget -= mlp_extra;
    }
  }
  const int xslots = 2 + L;
  for (int b = 0; b < xslots; ++b) {
    if (b >= 2 && !keeps_acts(b - 2)) {
      off_q_.push_back(0);
      off_k_.push_back(0);
      off_v_.push_back(0);
      off_o_.push_back(0);
      continue;
    }
    off_q_.push_back(take(N * size_t(hql_) * 128 * 2));
    off_k_.push_back(take(N * size_t(hkl_) * 128 * 2));
    off_v_.push_back(take(N * size_t(hkl_) * 128 * 2));
    off_o_.push_back(take(T * size_t(hq_) * 128 * 2));
  }
  for (int b = 0; b < 2; ++b) {
    off_do_[b] = take(N * size_t(hql_) * 128 * 2);
    off_dqkv_[b] = take(T * size_t(Wqkv_) * 2);
  }
  if (moe_) TRY(moe_arena(&off));
  if (enc_.on) off_feat_ = take(T * H * 2);
  arena_bytes_ = off;
  if (cudaMalloc(&arena_, arena_bytes_) != cudaSuccess) {
    set_error("out of device memory for the peer arena (" + std::to_string(arena_bytes_ >> 20) +
              " MiB)" + (save_acts_ ? "; recompute=none does not fit, use recompute=full" : ""));
    return OPX_ERR_CUDA;
  }
  CU(cudaMemset(arena_, 0, arena_bytes_));
  allocs_.push_back(arena_);
  bytes_alloc_ += int64_t(arena_bytes_);
  peer_arena_.assign(size_t(world_), nullptr);
  peer_arena_[size_t(rank_)] = arena_;
  d_peer_flags_ = alloc<uint32_t*>(kMaxSp);
  d_timeout_ = alloc<int>(1);

  for (int l = 0; l <= L; ++l) x_saved_.push_back(alloc<float>(T * H, false));
  auto make_acts = [&](Acts& a, bool dense_mlp, bool lean = false) -> bool {
    if (lean) {  // mode 1: attention state only
      a.ofull = relay_ ? alloc<bf16>(N * size_t(hql_) * 128, false) : nullptr;
      a.lse = alloc<float>(N * size_t(hql_), false);
      return a.lse && (!relay_ || a.ofull);
    }
    a.h = alloc<bf16>(T * H, false);
    a.ofull = relay_ ? alloc<bf16>(N * size_t(hql_) * 128, false) : nullptr;
    a.lse = alloc<float>(N * size_t(hql_), false);
    a.x2 = alloc<float>(T * H, false);
    a.r1 = alloc<float>(T, false);
    a.r2 = alloc<float>(T, false);
    a.h2 = alloc<bf16>(T * H, false);
    a.gu = dense_mlp ? alloc<bf16>(T * size_t(2 * F_), false) : nullptr;
    a.act = dense_mlp ? alloc<bf16>(T * size_t(F_), false) : nullptr;
    return a.h && a.lse && a.x2 && a.h2 && (!dense_mlp || (a.gu && a.act)) &&
           (!relay_ || a.ofull);
  };
  bool any_dense = false;
  for (int l = 0; l < L; ++l) any_dense = any_dense || !a_.is_moe_layer(l);
  if (!make_acts(scratch_, any_dense)) return cuda_fail(cudaErrorMemoryAllocation, "activations");
  saved_.assign(size_t(L), Acts{});
  for (int l = 0; l < L; ++l)
    if (keeps_acts(l) && !make_acts(saved_[size_t(l)], keeps_mlp(l) && !a_.is_moe_layer(l),
                                    keep_mode_[size_t(l)] == 1)) {
      set_error("out of device memory for recompute=none activations (layer " +
                std::to_string(l) + "); use recompute=full");
      return OPX_ERR_CUDA;
    }
  bind(scratch_);
  qkv_ = alloc<bf16>(T * size_t(Wqkv_), false);
  dx_ = alloc<float>(T * H, false);
  dtmp_ = alloc<float>(T * H, false);
  dxb_ = alloc<bf16>(T * H, false);
  dact_ = alloc<bf16>(T * size_t(F_), false);
  dgu_ = alloc<bf16>(T * size_t(2 * F_), false);
  dq_acc_ = alloc<float>(N * size_t(hql_) * 128, false);
  dk_ = alloc<float>(N * size_t(hkl_) * 128, false);
  dv_ = alloc<float>(N * size_t(hkl_) * 128, false);
  delta_ = alloc<float>(N * size_t(hql_), false);
  dw_part_ = alloc<float>(size_t(k_rmsnorm_bwd_parts(T_)) * H, false);
  hf_ = alloc<bf16>(T * H, false);
  rf_ = alloc<float>(T, false);
  dhf_ = alloc<float>(T * H, false);
  const int64_t chunk = std::min<int64_t>(ex_.ce_chunk, T_);
  logits_ = alloc<bf16>(size_t(chunk) * size_t(V_), false);
  const size_t A = size_t(accum_);
  loss_rows_ = alloc<float>(T * A);
  loss_sum_ = alloc<float>(4);
  d_ids_all_ = alloc<int32_t>(T * A);
  d_labels_all_ = alloc<int32_t>(T * A);
  d_pos_all_ = alloc<int32_t>(N * A);
  d_sstart_all_ = alloc<int32_t>(N * A);
  d_send_all_ = alloc<int32_t>(N * A);
  bind_micro(0);
  d_inv_freq_ = alloc<float>(64);
  for (void* q : {(void*)h_, (void*)logits_, (void*)dq_acc_, (void*)d_inv_freq_, (void*)x2_})
    if (!q) return cuda_fail(cudaErrorMemoryAllocation, "activations");
  std::vector<float> inv(64);
  for (int i = 0; i < 64; ++i)  // RoPE over head_dim d: theta^(-2i/d), i < d/2
    inv[size_t(i)] = i < d_ / 2 ? float(1.0 / std::pow(ex_.rope_theta, double(2 * i) / double(d_))) : 0.f;
  CU(cudaMemcpy(d_inv_freq_, inv.data(), 64 * sizeof(float), cudaMemcpyHostToDevice));
  // RoPE (sin, cos) per position id (< S) and frequency, once: the exchange
  // kernels read it instead of evaluating sincosf per element
  d_rope_ = alloc<float2>(size_t(S_) * size_t(d_ / 2), false);
  if (!d_rope_) return cuda_fail(cudaErrorMemoryAllocation, "rope table");
  CU(k_rope_table(d_rope_, S_, d_ / 2, d_inv_freq_, cs_));
  CU(cudaStreamSynchronize(cs_));
  if (moe_) TRY(moe_alloc());
  if (p_.sp == 1) {  // no peers: flags point at ourselves
    uint32_t* f = reinterpret_cast<uint32_t*>(arena_ + off_flags_);
    CU(cudaMemcpy(d_peer_flags_, &f, sizeof(f), cudaMemcpyHostToDevice));
  }
  return OPX_OK;
}

// Export = the arena's CUDA-IPC handle + its byte size.  Peers store into
// each other's arenas at locally computed offsets, so import refuses a peer
// whose arena layout (size) differs from ours.
int Step::ipc_export(void* out, size_t cap, size_t* len) {
  const size_t need = sizeof(cudaIpcMemHandle_t) + sizeof(uint64_t);
  if (cap < need) {
    set_error("ipc export buffer too small");
    return OPX_ERR_ARG;
  }
  cudaIpcMemHandle_t h;
  CU(cudaIpcGetMemHandle(&h, arena_));
  const uint64_t bytes = arena_bytes_;
  std::memcpy(out, &h, sizeof(h));
  std::memcpy(static_cast<char*>(out) + sizeof(h), &bytes, sizeof(bytes));
  *len = need;
  return OPX_OK;
}

int Step::ipc_import(const void* all, size_t len) {
  if (len != sizeof(cudaIpcMemHandle_t) + sizeof(uint64_t)) {
    set_error("ipc import: unexpected handle size");
    return OPX_ERR_ARG;
  }
  const char* base = static_cast<const char*>(all);
  // The SP group (Ulysses) and the EP group (dispatch/combine) exchange
  // through peer memory.
  std::vector<int64_t> peers = sp_members_;
  for (int64_t r : ep_members_)
    if (std::find(peers.begin(), peers.end(), r) == peers.end()) peers.push_back(r);
  for (int64_t r : peers) {
    if (r == rank_ || peer_arena_[size_t(r)]) continue;
    cudaIpcMemHandle_t h;
    uint64_t bytes = 0;
    std::memcpy(&h, base + size_t(r) * len, sizeof(h));
    std::memcpy(&bytes, base + size_t(r) * len + sizeof(h), sizeof(bytes));
    if (bytes != arena_bytes_) {
      set_error("ipc import: rank " + std::to_string(r) + " has a " + std::to_string(bytes) +
                "-byte peer arena, this rank " + std::to_string(arena_bytes_) +
                " (layouts differ; peer stores would land at wrong offsets)");
      return OPX_ERR_CONFIG;
    }
    void* p = nullptr;
    CU(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    peer_arena_[size_t(r)] = static_cast<char*>(p);
  }
  std::vector<uint32_t*> flags(size_t(kMaxSp), nullptr);
  for (int j = 0; j < int(p_.sp); ++j)
    flags[size_t(j)] = reinterpret_cast<uint32_t*>(peer(j, off_flags_));
  CU(cudaMemcpy(d_peer_flags_, flags.data(), kMaxSp * sizeof(uint32_t*), cudaMemcpyHostToDevice));
  if (moe_) TRY(moe_import());
  return OPX_OK;
}

int Step::init_weights(uint64_t seed) {
  const double c = 0.02 * std::sqrt(3.0) / 16777216.0;
  std::vector<Unit*> all;
  for (Unit& u : units_) all.push_back(&u);
  for (Unit& u : expert_units_)
    if (!u.params.empty()) all.push_back(&u);
  for (Unit* up : all) {
    Unit& u = *up;
    const int64_t sb = int64_t(u.idx) * u.shard, se = sb + u.shard;
    CU(cudaMemsetAsync(u.master, 0, size_t(u.shard) * 4, cs_));
    CU(cudaMemsetAsync(u.pshard, 0, size_t(u.shard) * 2, cs_));
    CU(cudaMemsetAsync(u.m, 0, size_t(u.shard) * 4, cs_));
    CU(cudaMemsetAsync(u.v, 0, size_t(u.shard) * 4, cs_));
    CU(cudaMemsetAsync(u.gshard, 0, size_t(u.shard) * u.gbytes(), cs_));
    for (const Param& q : u.params) {
      const int64_t lo = std::max(sb, q.off), hi = std::min(se, q.off + q.numel);
      if (hi <= lo) continue;
      const uint64_t ka = param_key(q.key_a, seed);
      const uint64_t kb = q.key_b.empty() ? 0 : param_key(q.key_b, seed);
      CU(k_init_param(u.master + (lo - sb), u.pshard + (lo - sb), hi - lo,
                      lo - q.off + q.logical_offset, ka, kb,
                      q.ones ? 0.0 : c, 1.0f, q.interleave, q.rows_per_slab, q.cols, cs_));
    }
  }
  step_count_ = 0;
  TRY(enc_init_weights(seed));
  CU(cudaStreamSynchronize(cs_));
  return OPX_OK;
}

int Step::load_batch(const int32_t* ids, const int32_t* labels, const int32_t* pos,
                     const int32_t* cu, int n_cu, int64_t n_valid) {
  // accum_ micro-batches of rows_ rows each, back to back
  const int64_t Nall = int64_t(Ntok_) * accum_;
  if (n_cu < 2 || cu[0] != 0 || cu[n_cu - 1] != Nall) {
    set_error("cu_seqlens must start at 0 and end at rows*seq_len (packing.hpp:28)");
    return OPX_ERR_ARG;
  }
  if (enc_.on && accum_ > 1) {
    set_error("a frozen encoder module with gradient accumulation is not supported");
    return OPX_ERR_CONFIG;
  }
  // per token: start / end of its sample, relative to its micro-batch
  std::vector<int32_t> st(static_cast<size_t>(Nall)), en(static_cast<size_t>(Nall));
  for (int i = 0; i + 1 < n_cu; ++i) {
    if (cu[i + 1] <= cu[i]) {
      set_error("cu_seqlens must be strictly increasing");
      return OPX_ERR_ARG;
    }
    if (cu[i] / S_ != (cu[i + 1] - 1) / S_) {
      set_error("a packed sample crosses a row boundary");
      return OPX_ERR_ARG;
    }
    const int32_t base = cu[i] / Ntok_ * Ntok_;
    for (int t = cu[i]; t < cu[i + 1]; ++t) {
      st[size_t(t)] = cu[i] - base;
      en[size_t(t)] = cu[i + 1] - base;
    }
  }
  n_valid_ = std::max<int64_t>(n_valid, 1);
  const size_t TA = size_t(T_) * size_t(accum_);
  CU(cudaMemcpyAsync(d_ids_all_, ids, TA * 4, cudaMemcpyHostToDevice, cs_));
  CU(cudaMemcpyAsync(d_labels_all_, labels, TA * 4, cudaMemcpyHostToDevice, cs_));
  // the RoPE table covers position ids [0, S); other ids use per-element sincosf
  rope_tab_ok_ = true;
  for (int64_t i = 0; i < Nall; ++i)
    if (pos[i] < 0 || pos[i] >= S_) {
      rope_tab_ok_ = false;
      break;
    }
  CU(cudaMemcpyAsync(d_pos_all_, pos, size_t(Nall) * 4, cudaMemcpyHostToDevice, cs_));
  CU(cudaMemcpyAsync(d_sstart_all_, st.data(), size_t(Nall) * 4, cudaMemcpyHostToDevice, cs_));
  CU(cudaMemcpyAsync(d_send_all_, en.data(), size_t(Nall) * 4, cudaMemcpyHostToDevice, cs_));
  CU(cudaStreamSynchronize(cs_));
  return OPX_OK;
}

// ---------------------------------------------------------------------------
// collectives
// ---------------------------------------------------------------------------
int Step::gather(Unit& u, int slot, cudaEvent_t wait_ev) {
  if (u.P == 1) return OPX_OK;
  if (wait_ev) CU(cudaStreamWaitEvent(ms_, wait_ev, 0));
  bf16* dst = slot < 0 ? u.full : gslot_[size_t(slot)];
  u.full = dst;
  NC(ncclAllGather(u.pshard, dst, size_t(u.shard), ncclBfloat16, u.comm, ms_));
  return OPX_OK;
}

int Step::barrier_sp(cudaStream_t s) {
  if (p_.sp == 1) return OPX_OK;
  ++epoch_;
  CU(k_peer_barrier(d_peer_flags_, reinterpret_cast<uint32_t*>(arena_ + off_flags_), int(p_.sp),
                    sp_i_, epoch_, d_timeout_, s));
  return OPX_OK;
}

// ---------------------------------------------------------------------------
// one layer
// ---------------------------------------------------------------------------
namespace {
// timing experiments only: OPX_DEBUG_NO_A2A skips the Ulysses exchanges (wrong numerics)
bool dbg_no_a2a() {
  static const bool v = getenv("OPX_DEBUG_NO_A2A") != nullptr;
  return v;
}
struct LayerW {
  const bf16 *ln1, *qkv, *o, *ln2, *gu, *down;
};
LayerW layer_w(const Unit& u, const bf16* base) {
  LayerW w;
  w.ln1 = base + u.params[0].off;
  w.qkv = base + u.params[1].off;
  w.o = base + u.params[4].off;
  w.ln2 = base + u.params[5].off;
  w.gu = u.params.size() > 7 ? base + u.params[6].off : nullptr;
  w.down = u.params.size() > 7 ? base + u.params[7].off : nullptr;
  return w;
}
GemmDesc gd(int M, int N, int K, const bf16* A, int64_t lda, bool amn, const bf16* B, int64_t ldb,
            bool bmn, int epi, void* D, int64_t ldd) {
  GemmDesc g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.A = A;
  g.lda = lda;
  g.a_mn = amn;
  g.B = B;
  g.ldb = ldb;
  g.b_mn = bmn;
  g.epi = epi;
  g.D = D;
  g.ldd = ldd;
  return g;
}
}  // namespace

int Step::layer_fwd(int l, const Unit& u, const float* x_in, float* x_out, int slot) {
  const LayerW W = layer_w(u, u.full);
  const int T = T_, H = H_, F = F_;
  const std::string pre = "fwd.layer" + std::to_string(l) + mtag();
  const std::string ph = "fwd.layer" + std::to_string(l);
  const bool tr = ex_.trace;
  cudaEvent_t e0 = tr ? ev() : nullptr, e1 = nullptr;
  if (tr) cudaEventRecord(e0, cs_);
  CU(k_rmsnorm_fwd(x_in, W.ln1, h_, r1_, T, H, ex_.rms_eps, cs_));
  const int qb = slot, ob = slot;
  // async_ulysses (step_graph.cpp:217-241): the seq->head exchange runs inside
  // the QKV GEMM's epilogue (peer stores tile by tile, overlapping the
  // mainloop of the other tiles) instead of as a kernel after it
  const bool fused = async_s2h();
  if (!fused) {
    CU(gemm_run(gd(T, Wqkv_, H, h_, H, false, W.qkv, H, false, GEMM_EPI_BF16, qkv_, Wqkv_), cs_));
    if (tr) {
      e1 = ev();
      cudaEventRecord(e1, cs_);
      mark(pre + ".qkv_proj", ph, 0, e0, e1);
      e0 = e1;
    }
  }
  {
    A2AArgs a{};
    a.sp = int(p_.sp);
    a.rank = sp_i_;
    a.rows = rows_;
    a.seq = S_;
    a.ngroups = 3;
    a.g[0].heads_total = hq_;
    a.g[0].col0 = 0;
    a.g[0].rope = 1;
    a.g[1].heads_total = hk_;
    a.g[1].col0 = hq_ * d_;
    a.g[1].rope = 1;
    a.g[2].heads_total = hk_;
    a.g[2].col0 = (hq_ + hk_) * d_;
    a.g[2].rope = 0;
    for (int j = 0; j < int(p_.sp); ++j) {
      a.g[0].full[j] = peer(j, off_q_[qb]);
      a.g[1].full[j] = peer(j, off_k_[qb]);
      a.g[2].full[j] = peer(j, off_v_[qb]);
    }
    a.local[0] = qkv_;
    a.local_ld = Wqkv_;
    a.pos = d_pos_;
    a.inv_freq = d_inv_freq_;
    a.hd = d_;
    a.rope_tab = rope_tab_ok_ ? d_rope_ : nullptr;
    if (fused) {
      GemmDesc g = gd(T, Wqkv_, H, h_, H, false, W.qkv, H, false, GEMM_EPI_SEQ2HEAD, nullptr, 0);
      g.s2h = &a;
      CU(gemm_run(g, cs_));
      if (tr) {  // one node: projection + the exchange it carries
        e1 = ev();
        cudaEventRecord(e1, cs_);
        mark(pre + ".qkv_proj", ph, 0, e0, e1, "qkv_proj,a2a_q,a2a_k,a2a_v");
        e0 = e1;
      }
    } else {
      if (!dbg_no_a2a()) CU(k_a2a_seq2head(a, cs_));
      // the exchange kernel and the flag barrier are traced apart, so the
      // node's NVLink rate is the kernel's own (the wait absorbs rank skew)
      if (tr) {
        e1 = ev();
        cudaEventRecord(e1, cs_);
        mark(pre + ".a2a_qkv", ph, 0, e0, e1, "a2a_q,a2a_k,a2a_v");
        e0 = e1;
      }
    }
    TRY(barrier_sp(cs_));
    if (tr && p_.sp > 1) {
      e1 = ev();
      cudaEventRecord(e1, cs_);
      mark(pre + ".a2a_wait", ph, 0, e0, e1);
      e0 = e1;
    }
  }
  bf16* attn_out = relay_ ? ofull_ : o_loc(ob);
  {
    AttnArgs a{};
    a.q = q_full(qb);
    a.k = k_full(qb);
    a.v = v_full(qb);
    a.o = attn_out;
    a.lse = lse_;
    a.ldq = hql_ * 128;
    a.ldk = a.ldv = hkl_ * 128;
    a.ldo = hql_ * 128;
    a.seq_start = d_sstart_;
    a.seq_end = d_send_;
    a.N = Ntok_;
    a.hq = hql_;
    a.hk = hkl_;
    a.scale = 1.0f / std::sqrt(float(d_));
    CU(k_attn_fwd_tc(a, cs_));
  }
  if (tr) {
    e1 = ev();
    cudaEventRecord(e1, cs_);
    mark(pre + ".attn_core", ph, 0, e0, e1);
    e0 = e1;
  }
  if (relay_) {
    A2AArgs a{};
    a.sp = int(p_.sp);
    a.rank = sp_i_;
    a.rows = rows_;
    a.seq = S_;
    a.ngroups = 1;
    a.g[0].heads_total = hq_;
    a.g[0].full[0] = ofull_;
    for (int j = 0; j < int(p_.sp); ++j) a.local[j] = peer(j, off_o_[ob]);
    a.local_ld = hq_ * d_;
    a.pos = d_pos_;
    a.inv_freq = d_inv_freq_;
    a.hd = d_;
    a.rope_tab = rope_tab_ok_ ? d_rope_ : nullptr;
    if (!dbg_no_a2a()) CU(k_a2a_head2seq(a, cs_));
    if (tr) {
      e1 = ev();
      cudaEventRecord(e1, cs_);
      mark(pre + ".a2a_out", ph, 0, e0, e1);
      e0 = e1;
    }
    TRY(barrier_sp(cs_));
    if (tr && p_.sp > 1) {
      e1 = ev();
      cudaEventRecord(e1, cs_);
      mark(pre + ".a2a_wait", ph, 0, e0, e1);
      e0 = e1;
    }
  }
  {
    GemmDesc g = gd(T, H, hq_ * d_, o_loc(ob), hq_ * d_, false, W.o, hq_ * d_, false,
                    GEMM_EPI_F32_RESID, x2_, H);
    g.R = x_in;
    g.ldr = H;
    CU(gemm_run(g, cs_));
  }
  if (tr) {
    e1 = ev();
    cudaEventRecord(e1, cs_);
    mark(pre + ".out_proj", ph, 0, e0, e1);
    e0 = e1;
  }
  CU(k_rmsnorm_fwd(x2_, W.ln2, h2_, r2_, T, H, ex_.rms_eps, cs_));
  if (a_.is_moe_layer(l)) {
    TRY(moe_fwd(l, u, expert_units_[size_t(l)], x2_, x_out));
    if (tr) {
      e1 = ev();
      cudaEventRecord(e1, cs_);
      mark(pre + ".moe", ph, 0, e0, e1);
    }
    return OPX_OK;
  }
  {
    // gate|up pre-activations are only needed by the backward (recompute pass)
    GemmDesc g = gd(T, 2 * F, H, h2_, H, false, W.gu, H, false, GEMM_EPI_SWIGLU,
                    store_gu_ ? gu_ : nullptr, 2 * F);
    g.D2 = act_;
    g.ldd2 = F;
    CU(gemm_run(g, cs_));
  }
  {
    GemmDesc g = gd(T, H, F, act_, F, false, W.down, F, false, GEMM_EPI_F32_RESID, x_out, H);
    g.R = x2_;
    g.ldr = H;
    CU(gemm_run(g, cs_));
  }
  if (tr) {
    e1 = ev();
    cudaEventRecord(e1, cs_);
    mark(pre + ".mlp", ph, 0, e0, e1);
  }
  return OPX_OK;
}

int Step::layer_bwd(int l, Unit& u, void* G) {
  const int T = T_, H = H_, F = F_, Q = hq_ * d_;
  const LayerW W = layer_w(u, u.full);
  const bool tr = ex_.trace;
  const std::string pre = "bwd.layer" + std::to_string(l) + mtag();
  const std::string ph = "bwd.layer" + std::to_string(l);
  cudaEvent_t e0 = tr ? ev() : nullptr, e1 = nullptr;
  if (tr) cudaEventRecord(e0, cs_);
  // full recompute of the layer (recompute=full); x_out goes to scratch
  int qb, ob;
  if (keeps_acts(l)) {  // this layer's forward activations are resident
    bind_layer(l);
    qb = ob = 2 + l;
    if (!keeps_mlp(l) && !a_.is_moe_layer(l)) {
      // attention-kept layer: recompute ln1 (h, for the qkv weight gradient),
      // the output projection + residual (x2), ln2 (h2) and gate|up + SwiGLU
      CU(k_rmsnorm_fwd(x_saved_[size_t(l)], W.ln1, h_, r1_, T, H, ex_.rms_eps, cs_));
      {
        GemmDesc g = gd(T, H, hq_ * d_, o_loc(ob), hq_ * d_, false, W.o, hq_ * d_, false,
                        GEMM_EPI_F32_RESID, x2_, H);
        g.R = x_saved_[size_t(l)];
        g.ldr = H;
        CU(gemm_run(g, cs_));
      }
      CU(k_rmsnorm_fwd(x2_, W.ln2, h2_, r2_, T, H, ex_.rms_eps, cs_));
      GemmDesc g = gd(T, 2 * F, H, h2_, H, false, W.gu, H, false, GEMM_EPI_SWIGLU, gu_, 2 * F);
      g.D2 = act_;
      g.ldd2 = F;
      CU(gemm_run(g, cs_));
    }
  } else {
    bind(scratch_);
    qb = ob = next_rslot();
    in_recompute_ = true;
    store_gu_ = true;
    const int rc_fwd = layer_fwd(l, u, x_saved_[size_t(l)], dtmp_, qb);
    in_recompute_ = false;
    store_gu_ = false;
    TRY(rc_fwd);
  }
  if (tr) {
    e1 = ev();
    cudaEventRecord(e1, cs_);
    mark(pre + ".recompute", ph, 0, e0, e1);
    e0 = e1;
  }
  void* g_ln1 = u.gat(G, u.params[0].off);
  void* g_qkv = u.gat(G, u.params[1].off);
  void* g_o = u.gat(G, u.params[4].off);
  void* g_ln2 = u.gat(G, u.params[5].off);
  void* g_gu = u.params.size() > 7 ? u.gat(G, u.params[6].off) : nullptr;
  void* g_down = u.params.size() > 7 ? u.gat(G, u.params[7].off) : nullptr;
  const int EPI_G = u.gbf ? GEMM_EPI_BF16 : GEMM_EPI_F32;  // weight-gradient epilogue

  // ---- MLP (dense) or MoE block
  if (a_.is_moe_layer(l)) {
    Unit& eu = expert_units_[size_t(l)];
    TRY(moe_bwd(l, u, eu, G, eu.gfull, dtmp_));
    CU(k_rmsnorm_bwd(dtmp_, x2_, W.ln2, r2_, dx_, dx_, dw_part_, g_ln2, 0, T, H, cs_, u.gbf));
  } else {
    // per-GEMM sub-nodes when tracing (mlp.*), so the profile separates the
    // dgrad/wgrad GEMMs from the elementwise work
    auto sub = [&](const char* name) {
      if (!tr) return;
      e1 = ev();
      cudaEventRecord(e1, cs_);
      mark(pre + ".mlp." + name, ph, 0, e0, e1);
      e0 = e1;
    };
    CU(k_cast_f32_bf16(dx_, dxb_, int64_t(T) * H, cs_));
    // (GEMM_EPI_SWIGLU_BWD fuses the next kernel into this GEMM's epilogue, but
    // its sigmoid/expf work made the epilogue outlast the mainloop: 172 ms vs
    // 89 + 32 ms unfused per C1 step on one GPU, so the step keeps them apart)
    CU(gemm_run(gd(T, F, H, dxb_, H, false, W.down, F, true, GEMM_EPI_BF16, dact_, F), cs_));
    sub("dgrad_down");
    CU(gemm_run(gd(H, F, T, dxb_, H, true, act_, F, true, EPI_G, g_down, F), cs_));
    sub("wgrad_down");
    CU(k_swiglu_bwd(dact_, gu_, dgu_, T, F, cs_));
    sub("swiglu_bwd");
    CU(gemm_run(gd(T, H, 2 * F, dgu_, 2 * F, false, W.gu, H, true, GEMM_EPI_F32, dtmp_, H), cs_));
    sub("dgrad_gu");
    CU(gemm_run(gd(2 * F, H, T, dgu_, 2 * F, true, h2_, H, true, EPI_G, g_gu, H), cs_));
    sub("wgrad_gu");
    CU(k_rmsnorm_bwd(dtmp_, x2_, W.ln2, r2_, dx_, dx_, dw_part_, g_ln2, 0, T, H, cs_, u.gbf));
    sub("rmsnorm_bwd");
  }
  if (tr && a_.is_moe_layer(l)) {
    e1 = ev();
    cudaEventRecord(e1, cs_);
    mark(pre + ".moe", ph, 0, e0, e1);
    e0 = e1;
  }
  // ---- attention output projection
  CU(k_cast_f32_bf16(dx_, dxb_, int64_t(T) * H, cs_));
  const int db = xdo_;
  xdo_ ^= 1;
  bf16* do_loc = relay_ ? ofull_ + 0 : do_full(db);  // see below when relaying
  bf16* do_scratch = nullptr;
  if (relay_) {
    // ofull_ still holds the attention output needed by attn_bwd: use dact_
    // (dead after the MLP backward, >= T*hq*128 elements) as the local dO.
    do_scratch = dact_;
    do_loc = do_scratch;
  }
  A2AArgs a_do{};
  if (relay_) {
    a_do.sp = int(p_.sp);
    a_do.rank = sp_i_;
    a_do.rows = rows_;
    a_do.seq = S_;
    a_do.ngroups = 1;
    a_do.g[0].heads_total = hq_;
    for (int j = 0; j < int(p_.sp); ++j) a_do.g[0].full[j] = peer(j, off_do_[db]);
    a_do.local[0] = do_loc;
    a_do.local_ld = Q;
    a_do.pos = d_pos_;
    a_do.inv_freq = d_inv_freq_;
    a_do.hd = d_;
    a_do.rope_tab = rope_tab_ok_ ? d_rope_ : nullptr;
  }
  const bool fused_do = relay_ && async_s2h();
  if (fused_do) {  // async_ulysses: dO goes to its head owners from the dgrad epilogue
    GemmDesc g = gd(T, Q, H, dxb_, H, false, W.o, Q, true, GEMM_EPI_SEQ2HEAD, nullptr, 0);
    g.s2h = &a_do;
    CU(gemm_run(g, cs_));
  } else {
    CU(gemm_run(gd(T, Q, H, dxb_, H, false, W.o, Q, true, GEMM_EPI_BF16, do_loc, Q), cs_));
  }
  CU(gemm_run(gd(H, Q, T, dxb_, H, true, o_loc(ob), Q, true, EPI_G, g_o, Q), cs_));
  if (tr) {
    e1 = ev();
    cudaEventRecord(e1, cs_);
    mark(pre + ".out_proj", ph, 0, e0, e1, fused_do ? "out_proj,a2a_do" : nullptr);
    e0 = e1;
  }
  if (relay_) {
    if (!fused_do && !dbg_no_a2a()) CU(k_a2a_seq2head(a_do, cs_));
    if (tr) {
      e1 = ev();
      cudaEventRecord(e1, cs_);
      if (!fused_do) mark(pre + ".a2a_do", ph, 0, e0, e1);
      e0 = e1;
    }
    TRY(barrier_sp(cs_));
    if (tr && p_.sp > 1) {
      e1 = ev();
      cudaEventRecord(e1, cs_);
      mark(pre + ".a2a_wait", ph, 0, e0, e1);
      e0 = e1;
    }
  }
  // ---- attention core
  {
    AttnArgs a{};
    a.q = q_full(qb);
    a.k = k_full(qb);
    a.v = v_full(qb);
    a.o = relay_ ? ofull_ : o_loc(ob);
    a.lse = lse_;
    a.ldq = hql_ * 128;
    a.ldk = a.ldv = hkl_ * 128;
    a.ldo = hql_ * 128;
    a.seq_start = d_sstart_;
    a.seq_end = d_send_;
    a.N = Ntok_;
    a.hq = hql_;
    a.hk = hkl_;
    a.scale = 1.0f / std::sqrt(float(d_));
    a.dout = do_full(db);
    a.lddo = hql_ * 128;
    a.dq_acc = dq_acc_;
    a.dk_acc = dk_;
    a.dv_acc = dv_;
    a.delta = delta_;
    CU(k_attn_bwd_tc(a, cs_));
  }
  if (tr) {
    e1 = ev();
    cudaEventRecord(e1, cs_);
    mark(pre + ".attn_core", ph, 0, e0, e1);
    e0 = e1;
  }
  // ---- head->seq for dq (fp32, un-rotate), dk (un-rotate), dv
  const int xb = xd_;
  xd_ ^= 1;
  {
    A2AArgs a{};
    a.sp = int(p_.sp);
    a.rank = sp_i_;
    a.rows = rows_;
    a.seq = S_;
    a.ngroups = 3;
    a.g[0] = A2AGroup{hq_, 0, 1, 1, {dq_acc_}};
    a.g[1] = A2AGroup{hk_, hq_ * d_, 1, 1, {dk_}};
    a.g[2] = A2AGroup{hk_, (hq_ + hk_) * d_, 0, 1, {dv_}};
    for (int j = 0; j < int(p_.sp); ++j) a.local[j] = peer(j, off_dqkv_[xb]);
    a.local_ld = Wqkv_;
    a.pos = d_pos_;
    a.inv_freq = d_inv_freq_;
    a.hd = d_;
    a.rope_tab = rope_tab_ok_ ? d_rope_ : nullptr;
    if (!dbg_no_a2a()) CU(k_a2a_head2seq(a, cs_));
    if (tr) {
      e1 = ev();
      cudaEventRecord(e1, cs_);
      mark(pre + ".a2a_dqkv", ph, 0, e0, e1, "a2a_dq,a2a_dk,a2a_dv");
      e0 = e1;
    }
    TRY(barrier_sp(cs_));
    if (tr && p_.sp > 1) {
      e1 = ev();
      cudaEventRecord(e1, cs_);
      mark(pre + ".a2a_wait", ph, 0, e0, e1);
      e0 = e1;
    }
  }
  bf16* dqkv = dqkv_loc(xb);
  CU(gemm_run(gd(T, H, Wqkv_, dqkv, Wqkv_, false, W.qkv, H, true, GEMM_EPI_F32, dtmp_, H), cs_));
  CU(gemm_run(gd(Wqkv_, H, T, dqkv, Wqkv_, true, h_, H, true, EPI_G, g_qkv, H), cs_));
  CU(k_rmsnorm_bwd(dtmp_, x_saved_[size_t(l)], W.ln1, r1_, dx_, dx_, dw_part_, g_ln1, 0, T, H,
                   cs_, u.gbf));
  if (tr) {
    e1 = ev();
    cudaEventRecord(e1, cs_);
    mark(pre + ".qkv_proj", ph, 0, e0, e1);
  }
  return OPX_OK;
}

int Step::head_fwd_bwd(Unit& u, float* G) {
  const int T = T_, H = H_, V = V_;
  const bf16* W_norm = u.full + u.params[1].off;
  const bf16* W_head = u.full + u.params[2].off;
  float* g_norm = G + u.params[1].off;
  float* g_head = G + u.params[2].off;
  const float* xf = x_saved_.back();
  const bool tr = ex_.trace;
  // the loss is computed chunk by chunk with the backward of each chunk right
  // behind its forward: the logits GEMM + CE of a chunk are fwd.head nodes,
  // its dgrad / wgrad GEMMs (and the final norm's backward) bwd.head nodes
  cudaEvent_t e0 = tr ? ev() : nullptr;
  if (tr) cudaEventRecord(e0, cs_);
  auto node = [&](const char* name) {
    if (!tr) return;
    cudaEvent_t e1 = ev();
    cudaEventRecord(e1, cs_);
    mark(std::string(name) + mtag(), name, 0, e0, e1);
    e0 = e1;
  };
  CU(k_rmsnorm_fwd(xf, W_norm, hf_, rf_, T, H, ex_.rms_eps, cs_));
  const int C = int(std::min<int64_t>(ex_.ce_chunk, T));
  for (int c0 = 0; c0 < T; c0 += C) {
    const int n = std::min(C, T - c0);
    CU(gemm_run(gd(n, V, H, hf_ + int64_t(c0) * H, H, false, W_head, H, false, GEMM_EPI_BF16,
                   logits_, V),
                cs_));
    CU(k_ce_fwd_bwd(logits_, V, d_labels_ + c0, loss_rows_ + int64_t(mb_) * T + c0, n, V,
                    1.0f / float(n_valid_), cs_));
    node("fwd.head");
    CU(gemm_run(gd(n, H, V, logits_, V, false, W_head, H, true, GEMM_EPI_F32,
                   dhf_ + int64_t(c0) * H, H),
                cs_));
    CU(gemm_run(gd(V, H, n, logits_, V, true, hf_ + int64_t(c0) * H, H, true,
                   c0 == 0 ? GEMM_EPI_F32 : GEMM_EPI_F32_ACCUM, g_head, H),
                cs_));
    node("bwd.head");
  }
  CU(k_rmsnorm_bwd(dhf_, xf, W_norm, rf_, nullptr, dx_, dw_part_, g_norm, 0, T, H, cs_));
  node("bwd.head");
  return OPX_OK;
}

// ---------------------------------------------------------------------------
// the step
// ---------------------------------------------------------------------------
int Step::unit_grad_ready(Unit& u, cudaStream_t s, const std::string& name, int layer) {
  if (u.params.empty()) return OPX_OK;
  const ncclDataType_t gdt = u.gbf ? ncclBfloat16 : ncclFloat;
  void* g = u.gshard;
  if (accum_ > 1) {
    CU(k_grad_accum(u.gacc, u.gshard, u.gbf, u.shard, mb_ == 0, s));
    if (!last_mb()) return OPX_OK;
    g = u.gacc;
  }
  if (u.rep_comm) {
    // HSDP: replicas all-reduce the (accumulated) shard gradient on the last
    // micro-batch only (step_graph.cpp:356-364)
    const bool tr = ex_.trace;
    cudaEvent_t a = tr ? ev() : nullptr;
    if (tr) cudaEventRecord(a, s);
    NC(ncclAllReduce(g, g, size_t(u.shard), accum_ > 1 ? ncclFloat : gdt, ncclSum, u.rep_comm, s));
    if (tr) {
      cudaEvent_t b = ev();
      cudaEventRecord(b, s);
      mark("bwd.ar." + name + mtag(), layer < 0 ? "bwd.head" : "bwd.layer" + std::to_string(layer),
           s == ms_ ? 1 : 0, a, b);
    }
  }
  return opt_unit(u, s, "opt." + name);
}

int Step::run(opx_step_report* rep) {
  const int L = int(a_.layers);
  const bool tr = ex_.trace;
  trace_.clear();
  ev_next_ = 0;
  ++step_count_;
  const int64_t launches0 = g_kernel_launches;
  const auto host_t0 = std::chrono::steady_clock::now();
  CU(cudaMemsetAsync(d_timeout_, 0, sizeof(int), cs_));
  CU(cudaEventRecord(ev_start_, cs_));
  CU(cudaStreamWaitEvent(ms_, ev_start_, 0));
  Unit& hu = units_[0];
  const int P = hu.P;

  // the head's parameters are gathered once and stay resident for every
  // micro-batch (its gradient is reduce-scattered per micro-batch)
  bind_micro(0);
  if (P > 1) {
    cudaEvent_t a = tr ? ev() : nullptr;
    if (tr) cudaEventRecord(a, ms_);
    TRY(gather(hu, -1, nullptr));
    CU(cudaEventRecord(ev_head_ag_, ms_));
    if (tr) mark("fwd.ag.head" + mtag(), "fwd.head", 1, a, ev_head_ag_);
    CU(cudaStreamWaitEvent(cs_, ev_head_ag_, 0));
  }

  auto issue_gather = [&](int l, bool bwd) -> int {
    Unit& u = units_[size_t(1 + l)];
    if (u.P == 1) return OPX_OK;
    const int slot = l % nslots_;
    // the slot was last used by layer l + nslots (bwd) or l - nslots (fwd);
    // across micro-batches the gather queues behind the previous micro-batch's
    // reduce-scatters on ms_, which each waited for their layer's backward
    const int prev = bwd ? l + nslots_ : l - nslots_;
    cudaEvent_t wait = (prev >= 0 && prev < L) ? ev_use_done_[size_t(prev)] : nullptr;
    cudaEvent_t a = tr ? ev() : nullptr;
    if (wait) CU(cudaStreamWaitEvent(ms_, wait, 0));
    if (tr) cudaEventRecord(a, ms_);
    TRY(gather(u, slot, nullptr));
    CU(cudaEventRecord(ev_ag_[size_t(l)], ms_));
    if (tr)
      mark(std::string(bwd ? "bwd" : "fwd") + ".ag.layer" + std::to_string(l) + mtag(),
           std::string(bwd ? "bwd" : "fwd") + ".layer" + std::to_string(l), 1, a,
           ev_ag_[size_t(l)]);
    return OPX_OK;
  };

  for (int mb = 0; mb < accum_; ++mb) {
    bind_micro(mb);
    // ---------------- forward ----------------
    // embedding grad region is scatter-added: zero it
    CU(cudaMemsetAsync(hu.gat(hu.gfull, hu.params[0].off), 0, size_t(hu.params[0].numel) * 4, cs_));
    CU(k_embed_fwd(d_ids_, hu.full + hu.params[0].off, x_saved_[0], T_, H_, cs_));
    TRY(enc_forward());  // frozen encoder: features replace the placeholder embeddings

    for (int l = 0; l < std::min(L, nslots_ - 1); ++l) TRY(issue_gather(l, false));
    for (int l = 0; l < L; ++l) {
      Unit& u = units_[size_t(1 + l)];
      if (u.P > 1) CU(cudaStreamWaitEvent(cs_, ev_ag_[size_t(l)], 0));
      if (l + nslots_ - 1 < L) TRY(issue_gather(l + nslots_ - 1, false));
      int slot;
      if (keeps_acts(l)) {
        bind_layer(l);
        slot = 2 + l;
        store_gu_ = keeps_mlp(l);
      } else {
        bind(scratch_);
        slot = next_rslot();
        store_gu_ = false;
      }
      if (moe_ && a_.is_moe_layer(l) && De_ > 1) {
        Unit& eu = expert_units_[size_t(l)];
        eu.full = eslot_;
        NC(ncclAllGather(eu.pshard, eslot_, size_t(eu.shard), ncclBfloat16, eu.comm, cs_));
      }
      TRY(layer_fwd(l, u, x_saved_[size_t(l)], x_saved_[size_t(l + 1)], slot));
      store_gu_ = false;
      CU(cudaEventRecord(ev_use_done_[size_t(l)], cs_));
    }
    CU(cudaEventRecord(ev_mb_[size_t(2 * mb)], cs_));

    if (moe_ && save_acts_) {
      // the top MoE layer's token re-send can start now, overlapping the head:
      // every peer passed that layer's forward combine barrier, so its expert
      // GEMMs no longer read the receive buffer
      const int lt = next_moe_below(L);
      if (lt >= 0) {
        cudaEvent_t e = ev();
        CU(cudaEventRecord(e, cs_));
        CU(cudaStreamWaitEvent(xs_, e, 0));
        TRY(moe_redispatch(lt));
      }
    }
    // ---------------- head (fwd + CE + bwd) ----------------
    TRY(head_fwd_bwd(hu, static_cast<float*>(hu.gfull)));  // the head keeps fp32 grads

    // ---------------- backward ----------------
    // layers L-nslots .. L-1 are still resident in their slots from the forward
    const int resident_from = std::max(0, L - nslots_);
    for (int l = L - 1; l >= 0; --l) {
      Unit& u = units_[size_t(1 + l)];
      if (u.P > 1) {
        if (l < resident_from) CU(cudaStreamWaitEvent(cs_, ev_ag_[size_t(l)], 0));
        // prefetch the next (lower) layer that is not resident
        const int nxt = l - 1;
        if (nxt >= 0 && nxt < resident_from) {
          // only issue once per layer: when l is the first layer above nxt
          TRY(issue_gather(nxt, true));
        }
        u.full = gslot_[size_t(l % nslots_)];
        u.gfull = gradslot_[size_t(l % 2)];
        if (l + 2 < L) CU(cudaStreamWaitEvent(cs_, ev_rs_done_[size_t(l + 2)], 0));
      }
      if (moe_ && a_.is_moe_layer(l) && De_ > 1) {
        Unit& eu = expert_units_[size_t(l)];
        eu.full = eslot_;
        eu.gfull = egrad_slot_;
        NC(ncclAllGather(eu.pshard, eslot_, size_t(eu.shard), ncclBfloat16, eu.comm, cs_));
      }
      TRY(layer_bwd(l, u, u.gfull));
      if (moe_ && a_.is_moe_layer(l)) {
        // expert grads: sum over the ranks holding the same experts, then replicas
        Unit& eu = expert_units_[size_t(l)];
        if (eu.P > 1) {
          if (eu.padded > eu.numel)
            CU(cudaMemsetAsync(eu.gat(eu.gfull, eu.numel), 0,
                               size_t(eu.padded - eu.numel) * eu.gbytes(), cs_));
          NC(ncclReduceScatter(eu.gfull, eu.gshard, size_t(eu.shard),
                               eu.gbf ? ncclBfloat16 : ncclFloat, ncclSum, eu.comm, cs_));
        }
        TRY(unit_grad_ready(eu, cs_, "experts.layer" + std::to_string(l), l));
      }
      CU(cudaEventRecord(ev_use_done_[size_t(l)], cs_));
      if (u.P > 1 || u.rep_comm) {
        CU(cudaEventRecord(ev_grad_done_[size_t(l)], cs_));
        CU(cudaStreamWaitEvent(ms_, ev_grad_done_[size_t(l)], 0));
        if (u.P > 1) {
          cudaEvent_t a = tr ? ev() : nullptr;
          if (tr) cudaEventRecord(a, ms_);
          if (u.padded > u.numel)
            CU(cudaMemsetAsync(u.gat(u.gfull, u.numel), 0, size_t(u.padded - u.numel) * u.gbytes(),
                               ms_));
          NC(ncclReduceScatter(u.gfull, u.gshard, size_t(u.shard), u.gbf ? ncclBfloat16 : ncclFloat,
                               ncclSum, u.comm, ms_));
          if (tr) {
            cudaEvent_t b = ev();
            cudaEventRecord(b, ms_);
            mark("bwd.rs.layer" + std::to_string(l) + mtag(), "bwd.layer" + std::to_string(l), 1,
                 a, b);
          }
        }
        TRY(unit_grad_ready(u, ms_, "layer" + std::to_string(l), l));
        CU(cudaEventRecord(ev_rs_done_[size_t(l)], ms_));
      } else {
        TRY(unit_grad_ready(u, cs_, "layer" + std::to_string(l), l));
      }
    }
    if (enc_.on && enc_.n_all) CU(k_rows_zero(dx_, d_fmask_, T_, H_, cs_));
    CU(k_embed_bwd(d_ids_, dx_, static_cast<float*>(hu.gfull) + hu.params[0].off, T_, H_, cs_));
    if (P > 1 || hu.rep_comm) {
      CU(cudaEventRecord(ev_head_rs_, cs_));
      CU(cudaStreamWaitEvent(ms_, ev_head_rs_, 0));
      if (P > 1) {
        cudaEvent_t a = tr ? ev() : nullptr;
        if (tr) cudaEventRecord(a, ms_);
        if (hu.padded > hu.numel)
          CU(cudaMemsetAsync(hu.gat(hu.gfull, hu.numel), 0, size_t(hu.padded - hu.numel) * 4, ms_));
        NC(ncclReduceScatter(hu.gfull, hu.gshard, size_t(hu.shard), ncclFloat, ncclSum, hu.comm,
                             ms_));
        if (tr) {
          cudaEvent_t b = ev();
          cudaEventRecord(b, ms_);
          mark("bwd.rs.head" + mtag(), "bwd.head", 1, a, b);
        }
      }
      TRY(unit_grad_ready(hu, ms_, "head", -1));
    } else {
      TRY(unit_grad_ready(hu, cs_, "head", -1));
    }
    // join the comm stream (and the MoE side stream): the next micro-batch
    // reuses the gradient slots, exchange buffers and routing state
    cudaEvent_t join = ev();
    CU(cudaEventRecord(join, ms_));
    CU(cudaStreamWaitEvent(cs_, join, 0));
    if (xs_) {
      cudaEvent_t xj = ev();
      CU(cudaEventRecord(xj, xs_));
      CU(cudaStreamWaitEvent(cs_, xj, 0));
    }
    CU(cudaEventRecord(ev_mb_[size_t(2 * mb + 1)], cs_));
  }
  CU(cudaEventRecord(ev_bwd_, cs_));

  // ---------------- optimizer ----------------
  // every unit's AdamW was issued on os_ as soon as its gradient was final;
  // the step ends when the last one (the head, whose embedding gradient
  // completes last) is done
  cudaEvent_t opt_join = ev();
  CU(cudaEventRecord(opt_join, os_));
  CU(cudaStreamWaitEvent(cs_, opt_join, 0));
  CU(cudaEventRecord(ev_end_, cs_));
  if (tr) {
    mark("optimizer", "optimizer", 0, ev_bwd_, ev_end_);
    trace_.back().span = true;  // the exposed tail; the opt.* nodes are the busy intervals
  }

  // loss: local sum -> world all-reduce (reporting only, off the timed path)
  CU(k_sum(loss_rows_, int64_t(T_) * accum_, loss_sum_, cs_));
  if (world_comm_) NC(ncclAllReduce(loss_sum_, loss_sum_, 1, ncclFloat, ncclSum, world_comm_, cs_));
  const double enqueue_s =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - host_t0).count();
  float loss = 0.f;
  int timeout = 0;
  CU(cudaMemcpyAsync(&loss, loss_sum_, 4, cudaMemcpyDeviceToHost, cs_));
  CU(cudaMemcpyAsync(&timeout, d_timeout_, 4, cudaMemcpyDeviceToHost, cs_));
  CU(cudaStreamSynchronize(cs_));
  if (getenv("OPX_GEMM_LOG")) gemm_log_dump(("rank" + std::to_string(rank_)).c_str());
  if (timeout) {
    set_error("peer barrier timed out (a peer rank stalled)");
    return OPX_ERR_TIMEOUT;
  }
  float t_all = 0, t_opt = 0;
  CU(cudaEventElapsedTime(&t_all, ev_start_, ev_end_));
  CU(cudaEventElapsedTime(&t_opt, ev_bwd_, ev_end_));
  double t_fwd = 0, t_bwd = 0;
  for (int mb = 0; mb < accum_; ++mb) {
    float f = 0, b = 0;
    CU(cudaEventElapsedTime(&f, mb ? ev_mb_[size_t(2 * mb - 1)] : ev_start_, ev_mb_[size_t(2 * mb)]));
    CU(cudaEventElapsedTime(&b, ev_mb_[size_t(2 * mb)], ev_mb_[size_t(2 * mb + 1)]));
    t_fwd += f;
    t_bwd += b;
  }
  opx_step_report& r = last_;
  std::memset(&r, 0, sizeof(r));
  r.step_time_s = t_all * 1e-3;
  r.fwd_s = t_fwd * 1e-3;
  r.bwd_s = t_bwd * 1e-3;
  r.opt_s = t_opt * 1e-3;
  r.loss = double(loss) / double(n_valid_);
  r.tokens = double(T_) * accum_;
  r.n_valid = double(n_valid_);
  r.launches = g_kernel_launches - launches0 - 1;  // minus the loss reduction
  r.enqueue_s = enqueue_s;
  for (int m : keep_mode_) r.kept_layers += m >= 1;
  r.accum_steps = accum_;
  // simulator.cpp:111-118 on the measured step time
  r.throughput = double(w_.global_batch) * double(w_.seq_len) / (r.step_time_s * double(world_));
  r.model_flops_per_token = flops_per_token_ref(m_, w_.seq_len);
  r.mfu = c_.peak_flops > 0 ? r.throughput * r.model_flops_per_token / c_.peak_flops : 0.0;
  measure_nodes(&r);
  if (rep) *rep = r;
  return OPX_OK;
}

void Step::measure_nodes(opx_step_report* r) {
  // exposed_comm_seconds (simulator.cpp:71-104) and the phase breakdown
  // (:120-129) over this rank's measured node intervals
  phases_.clear();
  std::vector<std::pair<double, double>> compute, comm;
  for (auto& t : trace_) {
    if (t.span) continue;
    float s = 0, e = 0;
    if (cudaEventElapsedTime(&s, ev_start_, t.a) != cudaSuccess) continue;
    if (cudaEventElapsedTime(&e, ev_start_, t.b) != cudaSuccess) continue;
    const double a = s * 1e-3, b = e * 1e-3;
    (t.comm ? comm : compute).push_back({a, b});
    auto& ph = phases_[t.phase];
    (t.comm ? ph.second : ph.first) += b - a;
    if (t.comm) r->comm_s += b - a;
  }
  cudaGetLastError();
  const double exposed = exposed_comm_seconds(compute, comm);
  r->comm_wait_s = exposed;
  r->exposed_comm = r->step_time_s > 0 ? exposed / r->step_time_s : 0.0;
}

std::string Step::report_json() {
  nlohmann::json ph = nlohmann::json::object();
  for (const auto& [name, c] : phases_) ph[name] = {{"compute_s", c.first}, {"comm_s", c.second}};
  nlohmann::json j{{"step_time_s", last_.step_time_s},
                   {"throughput_tokens_per_s_per_gpu", last_.throughput},
                   {"mfu", last_.mfu},
                   {"exposed_comm_fraction", last_.exposed_comm},
                   {"model_flops_per_token", last_.model_flops_per_token},
                   {"phase_breakdown", std::move(ph)}};
  return j.dump();
}

// ---------------------------------------------------------------------------
// inspection
// ---------------------------------------------------------------------------
int Step::info(const std::string& full, int64_t* numel, int64_t* b, int64_t* e) {
  const size_t colon = full.find(':');
  const std::string name = colon == std::string::npos ? full : full.substr(colon + 1);
  std::vector<const Unit*> all;
  for (const Unit& u : units_) all.push_back(&u);
  for (const Unit& u : expert_units_) all.push_back(&u);
  for (const Unit* up : all) {
    const Unit& u = *up;
    const Param* q = u.find(name);
    if (!q) continue;
    const int64_t sb = int64_t(u.idx) * u.shard, se = sb + u.shard;
    const int64_t lo = std::max(sb, q->off), hi = std::min(se, q->off + q->numel);
    *numel = q->logical_numel ? q->logical_numel : q->numel;
    *b = std::min(std::max<int64_t>(lo - q->off, 0), q->numel);
    *e = std::max(*b, std::min<int64_t>(hi - q->off, q->numel));
    *b += q->logical_offset;
    *e += q->logical_offset;
    return OPX_OK;
  }
  set_error("unknown tensor '" + name + "'");
  return OPX_ERR_ARG;
}

int Step::get(const std::string& full, void* dst, size_t bytes) {
  if (full.rfind("route:", 0) == 0) {  // forward top-k indices of MoE layer l (this rank's accum*T*k)
    const int l = std::atoi(full.c_str() + 6);
    if (l < 0 || l >= int(route_idx_.size()) || !route_idx_[size_t(l)] ||
        bytes != size_t(T_) * size_t(topk_) * size_t(accum_) * 4) {
      set_error("route: bad layer or size");
      return OPX_ERR_ARG;
    }
    CU(cudaMemcpy(dst, route_idx_[size_t(l)], bytes, cudaMemcpyDeviceToHost));
    return OPX_OK;
  }
  if (full == "features") {  // [T, H] feature rows received from the encoder (bf16 -> fp32)
    if (!enc_.on || bytes != size_t(T_) * size_t(H_) * 4) {
      set_error("features: no encoder or size mismatch");
      return OPX_ERR_ARG;
    }
    std::vector<uint16_t> h(size_t(T_) * size_t(H_));
    CU(cudaMemcpy(h.data(), arena_ + off_feat_, h.size() * 2, cudaMemcpyDeviceToHost));
    float* o = static_cast<float*>(dst);
    for (size_t i = 0; i < h.size(); ++i) {
      const uint32_t w = uint32_t(h[i]) << 16;
      std::memcpy(&o[i], &w, 4);
    }
    return OPX_OK;
  }
  if (full == "loss_rows") {
    if (bytes != size_t(T_) * size_t(accum_) * 4) {
      set_error("loss_rows: size mismatch");
      return OPX_ERR_ARG;
    }
    CU(cudaMemcpy(dst, loss_rows_, bytes, cudaMemcpyDeviceToHost));
    return OPX_OK;
  }
  const size_t colon = full.find(':');
  if (colon == std::string::npos) {
    set_error("tensor names are kind:name");
    return OPX_ERR_ARG;
  }
  const std::string kind = full.substr(0, colon), name = full.substr(colon + 1);
  std::vector<const Unit*> all;
  for (const Unit& u : units_) all.push_back(&u);
  for (const Unit& u : expert_units_) all.push_back(&u);
  for (const Unit* up : all) {
    const Unit& u = *up;
    const Param* q = u.find(name);
    if (!q) continue;
    const int64_t sb = int64_t(u.idx) * u.shard;
    int64_t n, b, e;
    TRY(info(full, &n, &b, &e));
    const int64_t cnt = e - b, src0 = q->off + (b - q->logical_offset) - sb;
    if (kind == "param") {
      if (bytes != size_t(cnt) * 2) {
        set_error("size mismatch for " + full);
        return OPX_ERR_ARG;
      }
      if (cnt) CU(cudaMemcpy(dst, u.pshard + src0, bytes, cudaMemcpyDeviceToHost));
      return OPX_OK;
    }
    if (bytes != size_t(cnt) * 4) {
      set_error("size mismatch for " + full);
      return OPX_ERR_ARG;
    }
    if (kind == "grad" && accum_ > 1) {  // the step's gradient: the micro-batch sum
      if (cnt) CU(cudaMemcpy(dst, u.gacc + src0, bytes, cudaMemcpyDeviceToHost));
      return OPX_OK;
    }
    if (kind == "grad" && u.gbf) {  // bf16 gradients are returned widened to fp32
      std::vector<uint16_t> h(static_cast<size_t>(cnt));
      if (cnt) CU(cudaMemcpy(h.data(), static_cast<const bf16*>(u.gshard) + src0, size_t(cnt) * 2,
                             cudaMemcpyDeviceToHost));
      float* o = static_cast<float*>(dst);
      for (int64_t i = 0; i < cnt; ++i) {
        const uint32_t w = uint32_t(h[size_t(i)]) << 16;
        std::memcpy(&o[i], &w, 4);
      }
      return OPX_OK;
    }
    const float* src = kind == "master" ? u.master
                       : kind == "grad" ? static_cast<const float*>(u.gshard)
                       : kind == "exp_avg" ? u.m
                       : kind == "exp_avg_sq" ? u.v
                                              : nullptr;
    if (!src) {
      set_error("unknown tensor kind '" + kind + "'");
      return OPX_ERR_ARG;
    }
    if (cnt) CU(cudaMemcpy(dst, src + src0, bytes, cudaMemcpyDeviceToHost));
    return OPX_OK;
  }
  set_error("unknown tensor '" + name + "'");
  return OPX_ERR_ARG;
}

std::string Step::trace_json() {
  nlohmann::json evs = nlohmann::json::array();
  for (auto& t : trace_) {
    float s = 0, e = 0;
    if (cudaEventElapsedTime(&s, ev_start_, t.a) != cudaSuccess) continue;
    if (cudaEventElapsedTime(&e, ev_start_, t.b) != cudaSuccess) continue;
    nlohmann::json args{{"phase", t.phase}};
    if (!t.fused.empty()) args["fused"] = t.fused;
    if (t.span) args["span"] = true;
    evs.push_back({{"name", t.name},
                   {"cat", t.comm ? "comm" : "compute"},
                   {"ph", "X"},
                   {"ts", double(s) * 1e3},
                   {"dur", double(e - s) * 1e3},
                   {"pid", rank_},
                   {"tid", t.tid},
                   {"args", args}});
  }
  nlohmann::json j{{"traceEvents", evs}, {"displayTimeUnit", "ms"}};
  return j.dump();
}

}  // namespace opx

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
using namespace opx;

struct opx_step {
  Step impl;
};

extern "C" {

int opx_nccl_unique_id(void* out128) {
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) {
    set_error(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    return OPX_ERR_CUDA;
  }
  std::memcpy(out128, &id, sizeof(id));
  return OPX_OK;
}

int opx_step_create(const char* cj, const char* mj, const char* wj, const char* pj,
                    const char* ej, int rank, int device, const void* nccl_id, opx_step** out) {
  *out = nullptr;
  Cluster c;
  Model m;
  Workload w;
  Plan p;
  ExecCfg ex;
  try {
    c = parse_cluster_json(cj ? cj : "");
    m = parse_model_json(mj ? mj : "");
    w = parse_workload_json(wj ? wj : "");
    p = parse_plan_json(pj ? pj : "{}");
    if (p.dp_shard < 0) p.dp_shard = c.world() / std::max<int64_t>(1, p.dp_replicate * p.sp);
    nlohmann::json e = nlohmann::json::parse(ej && *ej ? ej : "{}");
    ex.seed = e.value("seed", ex.seed);
    ex.lr = e.value("lr", ex.lr);
    if (e.contains("betas")) {
      ex.b1 = e["betas"][0].get<float>();
      ex.b2 = e["betas"][1].get<float>();
    }
    ex.eps = e.value("eps", ex.eps);
    ex.wd = e.value("weight_decay", ex.wd);
    ex.rope_theta = e.value("rope_theta", ex.rope_theta);
    ex.rms_eps = e.value("rms_eps", ex.rms_eps);
    ex.ce_chunk = e.value("ce_chunk", ex.ce_chunk);
    ex.trace = e.value("trace", true);
    ex.selective_recompute = e.value("selective_recompute", true);
    ex.bf16_grads = e.value("bf16_grads", true);
  } catch (const std::exception& e) {
    set_error(e.what());
    return OPX_ERR_CONFIG;
  }
  auto v = validate_plan(p, c, m, w);
  if (!v.empty()) {
    std::string s;
    for (auto& x : v) s += x.code + " ";
    set_error("plan invalid: " + s);
    return OPX_ERR_PLAN;
  }
  auto* st = new opx_step;
  int rc = st->impl.create(c, m, w, p, ex, rank, device, nccl_id);
  if (rc != OPX_OK) {
    delete st;
    return rc;
  }
  *out = st;
  return OPX_OK;
}

int opx_step_ipc_export(opx_step* st, void* out, size_t cap, size_t* len) {
  return st->impl.ipc_export(out, cap, len);
}
int opx_step_ipc_import(opx_step* st, const void* all, size_t len) {
  return st->impl.ipc_import(all, len);
}
int opx_step_init_weights(opx_step* st, uint64_t seed) { return st->impl.init_weights(seed); }
int opx_step_load_batch(opx_step* st, const int32_t* ids, const int32_t* labels,
                        const int32_t* positions, const int32_t* cu, int n_cu, int64_t n_valid) {
  return st->impl.load_batch(ids, labels, positions, cu, n_cu, n_valid);
}
int opx_step_load_images(opx_step* st, const void* pixels_bf16, int n_items, const int32_t* rows,
                         const int32_t* positions) {
  if (n_items < 0 || (n_items > 0 && (!pixels_bf16 || !rows || !positions))) {
    set_error("opx_step_load_images: bad arguments");
    return OPX_ERR_ARG;
  }
  return st->impl.load_images(static_cast<const uint16_t*>(pixels_bf16), n_items, rows, positions);
}
int opx_step_run(opx_step* st, opx_step_report* rep) { return st->impl.run(rep); }
int opx_step_save(opx_step* st, const char* dir) { return st->impl.save(dir ? dir : ""); }
int opx_step_load(opx_step* st, const char* dir) { return st->impl.load(dir ? dir : ""); }
int opx_step_get(opx_step* st, const char* name, void* dst, size_t bytes) {
  return st->impl.get(name, dst, bytes);
}
int opx_step_tensor_info(opx_step* st, const char* name, int64_t* numel, int64_t* b, int64_t* e) {
  return st->impl.info(name, numel, b, e);
}
int opx_step_report_json(opx_step* st, char* out, size_t cap, size_t* len) {
  const std::string s = st->impl.report_json();
  *len = s.size();
  if (!out || cap <= s.size()) {
    set_error("report buffer too small");
    return OPX_ERR_ARG;
  }
  std::memcpy(out, s.data(), s.size());
  out[s.size()] = 0;
  return OPX_OK;
}
int opx_step_trace(opx_step* st, char* out, size_t cap, size_t* len) {
  const std::string s = st->impl.trace_json();
  *len = s.size();
  if (!out || cap <= s.size()) {
    set_error("trace buffer too small");
    return OPX_ERR_ARG;
  }
  std::memcpy(out, s.data(), s.size());
  out[s.size()] = 0;
  return OPX_OK;
}
int opx_step_destroy(opx_step* st) {
  delete st;
  return OPX_OK;
}

}  // extern "C"
