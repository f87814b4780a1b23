// MoE / expert-parallel part of the step executor.
//
// Placement follows the reference plan API: EP groups are consecutive
// ep-chunks of each (dp_shard x sp) group (ep_groups, plan.cpp:168-182); rank
// e of an EP group owns experts [e*E/ep, (e+1)*E/ep) (Shard(0) of the stacked
// expert weights), each FSDP-sharded over the strided group
// of the (dp_shard*sp)/ep ranks with the same EP position
// (resolve_expert_sharding, plan.cpp:85-93).  Per MoE layer the forward runs
// router -> top-k -> stable permutation -> count exchange -> dispatch (peer
// stores) -> grouped gate|up GEMM with SwiGLU epilogue -> grouped down GEMM ->
// combine (peer stores) -> weighted unpermute + residual, the modeled
// a2a_dispatch / experts / a2a_combine nodes of build_moe_block
// (step_graph.cpp:253-293); the backward mirrors it (a2a_combine_grad,
// experts, a2a_dispatch_grad) and adds the router gradient.
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "common.h"
#include "step.h"

namespace opx {

#define TRY(x)                     \
  do {                             \
    int rc_ = (x);                 \
    if (rc_ != OPX_OK) return rc_; \
  } while (0)
#define CU(x) TRY(check((x), #x))
#define NC(x) TRY(nccl((x), #x))

namespace {
int64_t rup(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
}  // namespace

int Step::moe_setup_groups() {
  const Moe& m = *a_.moe;
  moe_ = true;
  E_ = int(m.experts);
  topk_ = int(m.top_k);
  Fe_ = int(m.ffn);
  ep_ = int(p_.ep);
  El_ = E_ / ep_;
  const int P = int(p_.shard_degree());
  De_ = P / ep_;
  if (Fe_ % 128 || E_ > 256 || topk_ > 16) {
    set_error("MoE executor requires expert_ffn_dim % 128 == 0, num_experts <= 256, top_k <= 16");
    return OPX_ERR_CONFIG;
  }
  if (ep_ > kMaxSp) {
    set_error("ep > 8 is not supported (one NVSwitch domain)");
    return OPX_ERR_CONFIG;
  }
  const int ms = shard_i_ * int(p_.sp) + sp_i_;  // index in the shard group
  const int g = ms / ep_;
  ep_i_ = ms % ep_;
  ep_members_.clear();
  for (int j = 0; j < ep_; ++j) ep_members_.push_back(shard_members_[size_t(g * ep_ + j)]);
  if (world_comm_)
    NC(ncclCommSplit(world_comm_, De_ > 1 ? rep_i_ * ep_ + ep_i_ : NCCL_SPLIT_NOCOLOR, rank_,
                     &expert_comm_, nullptr));
  return OPX_OK;
}

int Step::moe_build_units() {
  const int64_t H = H_, Fe = Fe_, El = El_, E = E_;
  const int ms = shard_i_ * int(p_.sp) + sp_i_;
  expert_units_.assign(size_t(a_.layers), Unit{});
  int64_t mx = 0;
  for (int l = 0; l < a_.layers; ++l) {
    if (!a_.is_moe_layer(l)) continue;
    Unit& u = expert_units_[size_t(l)];
    const std::string p = "model.layers." + std::to_string(l) + ".mlp.experts.";
    u.name = "layer" + std::to_string(l) + ".experts";
    Param gu;
    gu.name = p + "gate_up_proj";
    gu.shape = {El, 2 * Fe, H};
    gu.numel = El * 2 * Fe * H;
    gu.off = 0;
    gu.interleave = 1;
    gu.key_a = p + "gate_proj";
    gu.key_b = p + "up_proj";
    gu.rows_per_slab = 2 * Fe;
    gu.cols = H;
    gu.logical_offset = int64_t(ep_i_) * gu.numel;
    gu.logical_numel = E * 2 * Fe * H;
    Param dn;
    dn.name = p + "down_proj";
    dn.shape = {El, H, Fe};
    dn.numel = El * H * Fe;
    dn.off = rup(gu.numel, 128);
    dn.key_a = dn.name;
    dn.logical_offset = int64_t(ep_i_) * dn.numel;
    dn.logical_numel = E * H * Fe;
    u.params = {gu, dn};
    u.numel = dn.off + rup(dn.numel, 128);
    u.P = De_;
    u.idx = ms / ep_;
    u.comm = expert_comm_;
    u.rep_comm = p_.dp_replicate > 1 ? rep_comm_ : nullptr;
    u.padded = rup(u.numel, 64 * int64_t(De_));
    u.shard = u.padded / De_;
    u.master = alloc<float>(size_t(u.shard));
    u.m = alloc<float>(size_t(u.shard));
    u.v = alloc<float>(size_t(u.shard));
    u.gbf = ex_.bf16_grads;
    u.gshard = u.gbf ? static_cast<void*>(alloc<bf16>(size_t(u.shard)))
                     : static_cast<void*>(alloc<float>(size_t(u.shard)));
    u.pshard = alloc<bf16>(size_t(u.shard));
    if (accum_ > 1 && !(u.gacc = alloc<float>(size_t(u.shard), false))) {
      set_error("out of device memory for expert gradient accumulation shards");
      return OPX_ERR_CUDA;
    }
    if (!u.master || !u.m || !u.v || !u.gshard || !u.pshard) {
      set_error("out of device memory for expert shards");
      return OPX_ERR_CUDA;
    }
    if (De_ == 1) {
      u.full = u.pshard;
      u.gfull = u.gshard;
    }
    mx = std::max(mx, u.padded);
  }
  if (De_ > 1 && mx > 0) {
    eslot_ = alloc<bf16>(size_t(mx), false);
    egrad_slot_ = ex_.bf16_grads ? static_cast<void*>(alloc<bf16>(size_t(mx)))
                                 : static_cast<void*>(alloc<float>(size_t(mx)));
    if (!eslot_ || !egrad_slot_) return cuda_fail(cudaErrorMemoryAllocation, "expert slots");
  }
  return OPX_OK;
}

int Step::moe_arena(size_t* off_io) {
  size_t off = *off_io;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += size_t(rup(int64_t(bytes), 256));
    return o;
  };
  const size_t H = size_t(H_), P = size_t(T_) * size_t(topk_);
  cap_rows_ = int64_t(P) * ep_ + int64_t(El_) * 128;
  off_flags_ep_ = take(64 * sizeof(uint32_t));
  off_flags_ep2_ = take(64 * sizeof(uint32_t));
  off_flags_ep3_ = take(64 * sizeof(uint32_t));
  const int L = int(a_.layers);
  const int nslots = save_acts_ ? 1 + L : 1;
  off_counts_s_.assign(size_t(nslots), 0);
  off_yback_s_.assign(size_t(nslots), 0);
  for (int sl = 0; sl < nslots; ++sl) {
    if (sl > 0 && !a_.is_moe_layer(sl - 1)) continue;
    off_counts_s_[size_t(sl)] = take(size_t(ep_) * size_t(E_) * sizeof(int));
    off_yback_s_[size_t(sl)] = take(P * H * 2);
  }
  off_xrecv_ = take(size_t(cap_rows_) * H * 2);
  off_dyrecv_ = take(size_t(cap_rows_) * H * 2);
  off_dxback_ = take(P * H * 2);
  // recompute=none with EP: give the top MoE layers their own dispatch buffer
  // (worst-case rows) while HBM allows, so their backward needs no token
  // re-send (OPX_MOE_KEEP_X_MARGIN_GB of headroom kept for the rest)
  off_xrecv_l_.assign(size_t(L), 0);
  if (save_acts_ && ep_ > 1) {
    int K = 0;
    size_t free_b = 0, total_b = 0;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      const char* e = getenv("OPX_MOE_KEEP_X_MARGIN_GB");
      const size_t margin = size_t(e ? atof(e) : 48.0) << 30;
      const size_t per = size_t(rup(int64_t(size_t(cap_rows_) * H * 2), 256));
      const size_t budget = free_b > off + margin ? free_b - off - margin : 0;
      K = int(std::min<size_t>(size_t(L), budget / per));
    }
    if (const char* e = getenv("OPX_MOE_KEEP_X_MAX")) K = std::min(K, std::max(0, atoi(e)));
    // Every rank must agree on K: peers store into each other's kept slots at
    // locally computed offsets.  Every rank always joins the min-reduction
    // (a local failure above contributes 0), and a failed collective is an
    // error, never a silent K = 0 that would diverge from the peers' layout.
    if (world_comm_) {
      CU(cudaMemcpy(d_agree_, &K, sizeof(int), cudaMemcpyHostToDevice));
      NC(ncclAllReduce(d_agree_, d_agree_, 1, ncclInt32, ncclMin, world_comm_, cs_));
      CU(cudaStreamSynchronize(cs_));
      CU(cudaMemcpy(&K, d_agree_, sizeof(int), cudaMemcpyDeviceToHost));
    }
    for (int l = L - 1; l >= 0 && K > 0; --l) {
      if (!a_.is_moe_layer(l)) continue;
      off_xrecv_l_[size_t(l)] = take(size_t(cap_rows_) * H * 2);
      --K;
    }
  }
  *off_io = off;
  return OPX_OK;
}

int Step::moe_alloc() {
  const size_t T = size_t(T_), P = T * size_t(topk_), cap = size_t(cap_rows_);
  const size_t E = size_t(E_), H = size_t(H_), Fe = size_t(Fe_);
  r_logits_ = alloc<float>(T * E, false);
  if (k_moe_router_splits(H_) > 1 &&
      !(r_logits_part_ = alloc<float>(size_t(k_moe_router_splits(H_)) * T * E, false)))
    return cuda_fail(cudaErrorMemoryAllocation, "router partials");
  r_dw_ = alloc<float>(P, false);
  r_hist_ = alloc<int>(size_t(k_moe_sort_chunks(int(P))) * E);
  routes_.assign(off_counts_s_.size(), MoeRoute{});
  for (size_t sl = 0; sl < routes_.size(); ++sl) {
    if (sl > 0 && !a_.is_moe_layer(int(sl) - 1)) continue;
    MoeRoute& r = routes_[sl];
    r.wts = alloc<float>(P, false);
    r.idx = alloc<int>(P, false);
    r.pos = alloc<int>(P, false);
    r.pairat = alloc<int>(P, false);
    r.cnt = alloc<int>(E);
    r.excl = alloc<int>(E);
    r.g_start = alloc<int>(size_t(El_));
    r.g_rows = alloc<int>(size_t(El_));
    r.g_rows_pad = alloc<int>(size_t(El_));
    r.g_total = alloc<int>(1);
    if (!r.wts || !r.idx || !r.pos || !r.pairat || !r.cnt || !r.excl || !r.g_start || !r.g_rows ||
        !r.g_rows_pad || !r.g_total)
      return cuda_fail(cudaErrorMemoryAllocation, "MoE routing state");
  }
  moe_bind(-1);
  gu_e_ = alloc<bf16>(cap * 2 * Fe, false);
  act_e_ = alloc<bf16>(cap * Fe);
  y_e_ = alloc<bf16>(cap * H, false);
  rm_cnt_ = alloc<int>(size_t(El_) * size_t(ep_));
  rm_off_ = alloc<int>(size_t(El_) * size_t(ep_));
  if (!rm_cnt_ || !rm_off_) return cuda_fail(cudaErrorMemoryAllocation, "MoE combine map");
  dact_e_ = alloc<bf16>(cap * Fe, false);
  dgu_e_ = alloc<bf16>(cap * 2 * Fe);
  dx_e_ = alloc<bf16>(cap * H, false);
  dyp_ = alloc<bf16>(P * H, false);
  dlogits_ = alloc<bf16>(T * E, false);
  d_ep_flags_ = alloc<uint32_t*>(kMaxSp);
  d_ep_flags2_ = alloc<uint32_t*>(kMaxSp);
  d_ep_flags3_ = alloc<uint32_t*>(kMaxSp);
  if (p_.moe_overlap && ep_ > 1) {
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(cudaStreamCreateWithPriority(&xs2_, cudaStreamNonBlocking, hi));
  }
  if (save_acts_) {
    int lo = 0, hi = 0;
    CU(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(cudaStreamCreateWithPriority(&xs_, cudaStreamNonBlocking, hi));
    ev_redisp_.assign(size_t(a_.layers), nullptr);
    for (auto& e : ev_redisp_) CU(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  d_count_tables_ = alloc<int*>(kMaxSp * routes_.size());
  d_xrecv_peers_ = alloc<bf16*>(kMaxSp * (1 + size_t(a_.layers)));
  d_yback_peers_ = alloc<bf16*>(kMaxSp * routes_.size());
  d_dyrecv_peers_ = alloc<bf16*>(kMaxSp);
  d_dxback_peers_ = alloc<bf16*>(kMaxSp);
  for (void* q : {(void*)gu_e_, (void*)act_e_, (void*)y_e_, (void*)dact_e_, (void*)dgu_e_,
                  (void*)dx_e_, (void*)dyp_, (void*)d_dxback_peers_})
    if (!q) return cuda_fail(cudaErrorMemoryAllocation, "MoE scratch");
  // router wgrad dWr[E, H] = dlogits^T h2 has only E x H / 256^2 output tiles
  // and K = T: split K into chunks (grouped-K GEMM) and reduce the partials.
  wr_split_ = 16;
  while (wr_split_ > 1 && (T / size_t(wr_split_)) < 256) wr_split_ /= 2;
  {
    const int chunk = int((T + size_t(wr_split_) - 1) / size_t(wr_split_) + 63) / 64 * 64;
    std::vector<int> gs(static_cast<size_t>(wr_split_)), gr(static_cast<size_t>(wr_split_));
    for (int g = 0; g < wr_split_; ++g) {
      gs[size_t(g)] = g * chunk;
      gr[size_t(g)] = chunk;
    }
    wr_gs_ = alloc<int>(size_t(wr_split_));
    wr_gr_ = alloc<int>(size_t(wr_split_));
    wr_part_ = alloc<float>(size_t(wr_split_) * E * H, false);
    if (!wr_gs_ || !wr_gr_ || !wr_part_) return cuda_fail(cudaErrorMemoryAllocation, "router split");
    CU(cudaMemcpy(wr_gs_, gs.data(), gs.size() * 4, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(wr_gr_, gr.data(), gr.size() * 4, cudaMemcpyHostToDevice));
  }
  route_idx_.assign(size_t(a_.layers), nullptr);
  for (int l = 0; l < a_.layers; ++l)
    if (a_.is_moe_layer(l)) route_idx_[size_t(l)] = alloc<int>(P * size_t(accum_), false);
  // kept-token layers (top first) also keep gate|up + SwiGLU while HBM leaves
  // OPX_MOE_KEEP_GU_MARGIN_GB of headroom (a local choice: no peer sees them)
  gu_l_.assign(size_t(a_.layers), nullptr);
  act_l_.assign(size_t(a_.layers), nullptr);
  {
    size_t free_b = 0, total_b = 0;
    const char* e = getenv("OPX_MOE_KEEP_GU_MARGIN_GB");
    const size_t margin = size_t(e ? atof(e) : 16.0) << 30;
    const size_t per = cap * 3 * Fe * 2 + 1024;
    if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
      size_t budget = free_b > margin ? free_b - margin : 0;
      for (int l = a_.layers - 1; l >= 0 && budget >= per; --l) {
        if (!keeps_x(l)) continue;
        gu_l_[size_t(l)] = alloc<bf16>(cap * 2 * Fe, false);
        act_l_[size_t(l)] = alloc<bf16>(cap * Fe);
        if (!gu_l_[size_t(l)] || !act_l_[size_t(l)]) return cuda_fail(cudaErrorMemoryAllocation, "MoE kept gate|up");
        budget -= per;
      }
    }
  }
  if (ep_ == 1) TRY(moe_import());
  return OPX_OK;
}

void Step::moe_bind(int l) {
  rslot_ = l >= 0 ? 1 + l : 0;
  const MoeRoute& r = routes_[size_t(rslot_)];
  r_wts_ = r.wts;
  r_idx_ = r.idx;
  r_pos_ = r.pos;
  r_pairat_ = r.pairat;
  r_cnt_ = r.cnt;
  r_excl_ = r.excl;
  g_start_ = r.g_start;
  g_rows_ = r.g_rows;
  g_rows_pad_ = r.g_rows_pad;
  g_total_ = r.g_total;
}

int Step::moe_import() {
  const size_t ns = routes_.size();
  std::vector<void*> fl(kMaxSp, nullptr), fl2(kMaxSp, nullptr), fl3(kMaxSp, nullptr),
      ct(kMaxSp * ns, nullptr),
      xr(kMaxSp * (1 + size_t(a_.layers)), nullptr),
      yb(kMaxSp * ns, nullptr), dy(kMaxSp, nullptr), dx(kMaxSp, nullptr);
  for (int j = 0; j < ep_; ++j) {
    fl[size_t(j)] = ep_peer(j, off_flags_ep_);
    fl2[size_t(j)] = ep_peer(j, off_flags_ep2_);
    fl3[size_t(j)] = ep_peer(j, off_flags_ep3_);
    for (size_t sl = 0; sl < ns; ++sl) {
      ct[sl * kMaxSp + size_t(j)] = ep_peer(j, off_counts_s_[sl]);
      yb[sl * kMaxSp + size_t(j)] = ep_peer(j, off_yback_s_[sl]);
    }
    xr[size_t(j)] = ep_peer(j, off_xrecv_);
    for (int l = 0; l < a_.layers; ++l)
      if (keeps_x(l)) xr[size_t(1 + l) * kMaxSp + size_t(j)] = ep_peer(j, off_xrecv_l_[size_t(l)]);
    dy[size_t(j)] = ep_peer(j, off_dyrecv_);
    dx[size_t(j)] = ep_peer(j, off_dxback_);
  }
  const size_t b = kMaxSp * sizeof(void*);
  CU(cudaMemcpy(d_ep_flags_, fl.data(), b, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_ep_flags2_, fl2.data(), b, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_ep_flags3_, fl3.data(), b, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_count_tables_, ct.data(), b * ns, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_xrecv_peers_, xr.data(), b * (1 + size_t(a_.layers)), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_yback_peers_, yb.data(), b * ns, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_dyrecv_peers_, dy.data(), b, cudaMemcpyHostToDevice));
  CU(cudaMemcpy(d_dxback_peers_, dx.data(), b, cudaMemcpyHostToDevice));
  return OPX_OK;
}

int Step::moe_redispatch(int l) {
  if (l < 0 || !xs_ || !keeps_acts(l) || !a_.is_moe_layer(l) || keeps_x(l)) return OPX_OK;
  const MoeRoute& r = routes_[size_t(1 + l)];
  const int* counts = reinterpret_cast<const int*>(arena_ + off_counts_s_[size_t(1 + l)]);
  const int P = T_ * topk_;
  cudaEvent_t a = ex_.trace ? ev() : nullptr;
  if (a) cudaEventRecord(a, xs_);
  CU(k_moe_dispatch(saved_[size_t(l)].h2, H_, 0, r.pairat, P, topk_, counts, r.excl, ep_, E_,
                    ep_i_, d_xrecv_peers_, H_, H_, xs_));
  if (ep_ > 1) {
    ++epoch_ep2_;
    CU(k_peer_barrier(d_ep_flags2_, reinterpret_cast<uint32_t*>(arena_ + off_flags_ep2_), ep_, ep_i_,
                      epoch_ep2_, d_timeout_, xs_));
  }
  CU(cudaEventRecord(ev_redisp_[size_t(l)], xs_));
  if (a) {
    cudaEvent_t b = ev();
    cudaEventRecord(b, xs_);
    mark("bwd.layer" + std::to_string(l) + mtag() + ".a2a_redispatch", "bwd.layer" + std::to_string(l), 3,
         a, b);
  }
  return OPX_OK;
}

int Step::barrier_ep3(cudaStream_t s) {
  if (ep_ == 1) return OPX_OK;
  ++epoch_ep3_;
  CU(k_peer_barrier(d_ep_flags3_, reinterpret_cast<uint32_t*>(arena_ + off_flags_ep3_), ep_, ep_i_,
                    epoch_ep3_, d_timeout_, s));
  return OPX_OK;
}

int Step::barrier_ep(cudaStream_t s) {
  if (ep_ == 1) return OPX_OK;
  ++epoch_ep_;
  CU(k_peer_barrier(d_ep_flags_, reinterpret_cast<uint32_t*>(arena_ + off_flags_ep_), ep_, ep_i_,
                    epoch_ep_, d_timeout_, s));
  return OPX_OK;
}

namespace {
GemmDesc grouped(int M, int N, int K, const bf16* A, int64_t lda, bool amn, const bf16* B,
                 int64_t ldb, bool bmn, int epi, void* D, int64_t ldd, int groups, int gk,
                 const int* gs, const int* gr, int64_t rows_total, int64_t dstride) {
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
  g.groups = groups;
  g.grouped_k = gk;
  g.g_start = gs;
  g.g_rows = gr;
  g.rows_total = rows_total;
  g.d_group_stride = dstride;
  return g;
}
// moe_overlap: the two expert halves' GEMMs run concurrently on their two
// streams (disjoint rows of every buffer; the ticketed GEMMs share the SMs);
// OPX_MOE_SERIAL_HALVES=1 orders half B's GEMMs after half A's (round 1)
// The combine / dX return ride in the expert GEMM epilogues (GEMM_EPI_ROWMAP:
// rows peer-stored to their token owners through the per-warp stage, 8 rows x
// 64 contiguous bytes per store instruction): C2/EP4 192K vs 188K tokens/s for
// the separate warp-per-row combine kernel (OPX_MOE_FUSED_COMBINE=0).  Without
// the staging (one 16-B store of 32 different rows per instruction) the fused
// form had measured 143K.
bool moe_fused_combine() {
  static const bool v = !getenv("OPX_MOE_FUSED_COMBINE") || atoi(getenv("OPX_MOE_FUSED_COMBINE"));
  return v;
}
// the a2a_combine_grad (dY rows to the expert ranks) fused into the combine
// backward: each dY row is peer-stored to its receive row as it is computed,
// instead of written locally and re-read by a dispatch pass.  Measured:
// C2 slice 1 GPU 122.5K vs 121.2K tokens/s (combine_bwd + dispatch 3.8 -> 2.5 ms);
// C2/EP4 with moe_overlap, one fused pass over all pairs: 192.8K vs 196.2K
// (the per-half dispatch on two streams let half B's expert backward start
// earlier), hence the per-half fused passes there.  OPX_MOE_FUSED_DY=0
// restores the separate dispatch.
int moe_fused_dy_mode() {
  static const int v = getenv("OPX_MOE_FUSED_DY") ? atoi(getenv("OPX_MOE_FUSED_DY")) : -1;
  return v;
}
bool moe_serial_halves() {
  static const bool v = getenv("OPX_MOE_SERIAL_HALVES") && atoi(getenv("OPX_MOE_SERIAL_HALVES"));
  return v;
}
}  // namespace

int Step::moe_fwd(int l, const Unit& u, const Unit& eu, const float* x2, float* x_out) {
  const std::string pre = std::string(in_recompute_ ? "bwd" : "fwd") + ".layer" + std::to_string(l) + mtag() + ".";
  const std::string ph = std::string(in_recompute_ ? "bwd" : "fwd") + ".layer" + std::to_string(l);
  cudaEvent_t e0 = nullptr;
  auto mk = [&](const char* name, const char* fused = nullptr) {
    if (!ex_.trace) return;
    cudaEvent_t e1 = ev();
    cudaEventRecord(e1, cs_);
    if (e0) mark(pre + name, ph, 0, e0, e1, fused);
    e0 = e1;
  };
  mk("");
  moe_bind(keeps_acts(l) ? l : -1);
  const int T = T_, H = H_, E = E_, k = topk_, Fe = Fe_, P = T_ * topk_;
  const bf16* Wr = u.full + u.params[6].off;
  const bf16* Wgu = eu.full + eu.params[0].off;
  const bf16* Wd = eu.full + eu.params[1].off;
  int* counts_all = counts_cur();
  const int xl = in_recompute_ ? -1 : l;  // a kept layer's own dispatch buffer
  bf16* xrecv = xrecv_of(xl);
  bf16 *gu_sv = gu_e_, *act_sv = act_e_;
  const bool kg = !in_recompute_ && keeps_gu(l);  // store this layer's gate|up + SwiGLU
  if (kg) {
    gu_e_ = gu_l_[size_t(l)];
    act_e_ = act_l_[size_t(l)];
  }
  bf16** xpeers = xrecv_peers_of(xl);
  bf16* yback = yback_cur();
  CU(k_moe_router(h2_, Wr, r_logits_, T, H, E, cs_, r_logits_part_));
  CU(k_moe_topk(r_logits_, T, E, k, r_idx_, r_wts_, cs_));
  if (!in_recompute_ && route_idx_[size_t(l)])
    CU(cudaMemcpyAsync(route_idx_[size_t(l)] + int64_t(mb_) * P, r_idx_, size_t(P) * sizeof(int),
                       cudaMemcpyDeviceToDevice, cs_));
  CU(k_moe_sort(r_idx_, P, E, r_hist_, r_cnt_, r_excl_, r_pos_, r_pairat_, cs_));
  mk("router");
  CU(k_moe_publish_counts(r_cnt_, count_tab_cur(), ep_, ep_i_, E, cs_));
  TRY(barrier_ep(cs_));
  CU(k_moe_groups(counts_all, ep_, E, ep_i_, g_start_, g_rows_, g_rows_pad_, g_total_, cs_));
  CU(k_moe_combine_map(counts_all, ep_, E, ep_i_, rm_cnt_, rm_off_, cs_));
  mk("a2a_counts");
  // down projection of experts [lo, lo + n), then the a2a_combine: every row
  // back to its token owner's combine buffer (or, fused, from the GEMM's
  // epilogue straight away)
  const bool fusedc = moe_fused_combine();
  auto down = [&](int lo, int n, cudaStream_t st) -> int {
    GemmDesc g = grouped(0, H, Fe, act_e_, Fe, false, Wd + int64_t(lo) * H * Fe, Fe, false,
                         fusedc ? GEMM_EPI_ROWMAP : GEMM_EPI_BF16, y_e_, H, n, 0, g_start_ + lo,
                         g_rows_ + lo, cap_rows_, 0);
    g.rm_dst = yback_tab_cur();
    g.rm_cnt = rm_cnt_ + int64_t(lo) * ep_;
    g.rm_off = rm_off_ + int64_t(lo) * ep_;
    g.rm_ep = ep_;
    CU(gemm_run(g, st));
    return OPX_OK;
  };
  auto combine = [&](int lo, int n, cudaStream_t st) -> int {
    if (!fusedc)
      CU(k_moe_combine(y_e_, H, rm_cnt_, rm_off_, ep_, El_, g_start_, yback_tab_cur(), H, H,
                       int(cap_rows_), st, lo, n));
    return OPX_OK;
  };
  const char* fused_tag = fusedc ? "experts,a2a_combine" : nullptr;
  // experts [lo, hi) of every rank: dispatch -> barrier -> gate|up + SwiGLU ->
  // down -> combine -> barrier, on stream st with barrier flag set `fs`
  auto phase = [&](int lo, int hi, cudaStream_t st, int fs, bool marks) -> int {
    CU(k_moe_dispatch(h2_, H, 0, r_pairat_, P, k, counts_all, r_excl_, ep_, E, ep_i_,
                      xpeers, H, H, st, lo, hi));
    if (marks) mk("a2a_dispatch");
    TRY(fs ? barrier_ep3(st) : barrier_ep(st));
    if (marks) mk("a2a_wait");
    const int n = hi - lo;
    CU(k_moe_zero_pad(xrecv, H, H, g_start_ + lo, g_rows_ + lo, g_rows_pad_ + lo, n, st));
    {
      // gate|up pre-activations are only needed by the backward (recompute pass)
      GemmDesc g = grouped(0, 2 * Fe, H, xrecv, H, false, Wgu + int64_t(lo) * 2 * Fe * H, H, false,
                           GEMM_EPI_SWIGLU, (in_recompute_ || kg) ? gu_e_ : nullptr, 2 * Fe, n, 0,
                           g_start_ + lo, g_rows_ + lo, cap_rows_, 0);
      g.D2 = act_e_;
      g.ldd2 = Fe;
      CU(gemm_run(g, st));
    }
    CU(k_moe_zero_pad(act_e_, Fe, Fe, g_start_ + lo, g_rows_ + lo, g_rows_pad_ + lo, n, st));
    TRY(down(lo, n, st));
    if (marks) mk("experts", fused_tag);
    TRY(combine(lo, n, st));
    if (marks && !fusedc) mk("a2a_combine");
    TRY(fs ? barrier_ep3(st) : barrier_ep(st));
    if (marks) mk("a2a_wait");
    return OPX_OK;
  };
  if (p_.moe_overlap && ep_ > 1 && El_ >= 2 && xs2_) {
    // moe_overlap (plan.hpp): two expert halves pipelined on two streams so the
    // second half's dispatch overlaps the first half's GEMMs and the first
    // half's combine overlaps the second half's GEMMs (expert GEMMs of the two
    // halves are serialised with an event)
    const int h = El_ / 2;
    cudaEvent_t ready = ev(), gemm_a = ev(), done_b = ev();
    CU(cudaEventRecord(ready, cs_));
    CU(cudaStreamWaitEvent(xs2_, ready, 0));
    // half B: dispatch, then its GEMMs after half A's
    CU(k_moe_dispatch(h2_, H, 0, r_pairat_, P, k, counts_all, r_excl_, ep_, E, ep_i_,
                      xpeers, H, H, xs2_, h, El_));
    TRY(barrier_ep3(xs2_));
    // half A on the compute stream
    CU(k_moe_dispatch(h2_, H, 0, r_pairat_, P, k, counts_all, r_excl_, ep_, E, ep_i_,
                      xpeers, H, H, cs_, 0, h));
    mk("a2a_dispatch");
    TRY(barrier_ep(cs_));
    mk("a2a_wait");
    auto experts = [&](int lo, int hi, cudaStream_t st) -> int {
      const int n = hi - lo;
      CU(k_moe_zero_pad(xrecv, H, H, g_start_ + lo, g_rows_ + lo, g_rows_pad_ + lo, n, st));
      GemmDesc g = grouped(0, 2 * Fe, H, xrecv, H, false, Wgu + int64_t(lo) * 2 * Fe * H, H, false,
                           GEMM_EPI_SWIGLU, (in_recompute_ || kg) ? gu_e_ : nullptr, 2 * Fe, n, 0,
                           g_start_ + lo, g_rows_ + lo, cap_rows_, 0);
      g.D2 = act_e_;
      g.ldd2 = Fe;
      CU(gemm_run(g, st));
      CU(k_moe_zero_pad(act_e_, Fe, Fe, g_start_ + lo, g_rows_ + lo, g_rows_pad_ + lo, n, st));
      return down(lo, n, st);
    };
    TRY(experts(0, h, cs_));
    CU(cudaEventRecord(gemm_a, cs_));
    mk("experts", fused_tag);
    if (moe_serial_halves()) CU(cudaStreamWaitEvent(xs2_, gemm_a, 0));
    TRY(experts(h, El_, xs2_));
    TRY(combine(h, El_ - h, xs2_));
    TRY(barrier_ep3(xs2_));
    CU(cudaEventRecord(done_b, xs2_));
    TRY(combine(0, h, cs_));
    if (!fusedc) mk("a2a_combine");
    TRY(barrier_ep(cs_));
    CU(cudaStreamWaitEvent(cs_, done_b, 0));
    // the compute stream now waits for half B: its expert GEMMs, combine and barrier
    mk("experts_b");
  } else {
    TRY(phase(0, El_, cs_, 0, true));
  }
  CU(k_moe_unpermute(yback, H, r_pos_, r_wts_, T, k, H, x2, x_out, cs_));
  mk("unpermute");
  gu_e_ = gu_sv;
  act_e_ = act_sv;
  return OPX_OK;
}

int Step::moe_bwd(int l, const Unit& u, Unit& eu, void* G, void* Ge, float* dh2) {
  const std::string pre = "bwd.layer" + std::to_string(l) + mtag() + ".";
  const std::string ph = "bwd.layer" + std::to_string(l);
  cudaEvent_t e0 = nullptr;
  auto mk = [&](const char* name, const char* fused = nullptr) {
    if (!ex_.trace) return;
    cudaEvent_t e1 = ev();
    cudaEventRecord(e1, cs_);
    if (e0) mark(pre + name, ph, 0, e0, e1, fused);
    e0 = e1;
  };
  mk("");
  const bool kept = keeps_acts(l);
  moe_bind(kept ? l : -1);
  const int T = T_, H = H_, E = E_, k = topk_, Fe = Fe_, P = T_ * topk_;
  const bf16* Wr = u.full + u.params[6].off;
  const bf16* Wgu = eu.full + eu.params[0].off;
  const bf16* Wd = eu.full + eu.params[1].off;
  int* counts_all = counts_cur();
  bf16* xrecv = xrecv_of(kept ? l : -1);
  bf16* yback = yback_cur();
  bf16* dyrecv = reinterpret_cast<bf16*>(arena_ + off_dyrecv_);
  bf16* dxback = reinterpret_cast<bf16*>(arena_ + off_dxback_);
  bf16 *gu_sv = gu_e_, *act_sv = act_e_;
  if (kept && keeps_gu(l)) {  // gate|up and SwiGLU kept from the forward
    gu_e_ = gu_l_[size_t(l)];
    act_e_ = act_l_[size_t(l)];
  } else if (kept) {
    // selective recompute: routing and combined outputs are resident; the
    // tokens were re-sent on xs_ (moe_redispatch, overlapping the layer above);
    // redo gate|up, storing the pre-activations for the SwiGLU backward
    if (!keeps_x(l)) {
      CU(cudaStreamWaitEvent(cs_, ev_redisp_[size_t(l)], 0));
      mk("a2a_redispatch_wait");
    }
    CU(k_moe_zero_pad(xrecv, H, H, g_start_, g_rows_, g_rows_pad_, El_, cs_));
    GemmDesc g = grouped(0, 2 * Fe, H, xrecv, H, false, Wgu, H, false, GEMM_EPI_SWIGLU, gu_e_,
                         2 * Fe, El_, 0, g_start_, g_rows_, cap_rows_, 0);
    g.D2 = act_e_;
    g.ldd2 = Fe;
    CU(gemm_run(g, cs_));
    CU(k_moe_zero_pad(act_e_, Fe, Fe, g_start_, g_rows_, g_rows_pad_, El_, cs_));
    mk("gate_up_recompute");
  }
  CU(k_moe_combine_map(counts_all, ep_, E, ep_i_, rm_cnt_, rm_off_, cs_));
  const bool fusedc = moe_fused_combine();
  auto dx_return = [&](int lo, int n, cudaStream_t st) -> int {
    if (!fusedc)
      CU(k_moe_combine(dx_e_, H, rm_cnt_, rm_off_, ep_, El_, g_start_, d_dxback_peers_, H, H,
                       int(cap_rows_), st, lo, n));
    return OPX_OK;
  };
  // weighted combine backward: per-pair output grads and router-weight grads;
  // a2a_combine_grad: pair grads travel to the expert ranks (same layout as
  // dispatch) -- fused: stored there straight from the combine backward
  const bool overlap = p_.moe_overlap && ep_ > 1 && El_ >= 2 && xs2_;
  const bool fdy = moe_fused_dy_mode() != 0;
  // fused: local experts [lo, hi) of every rank (moe_overlap issues the halves
  // on two streams, half B first)
  auto combine_bwd_to = [&](int lo, int hi, cudaStream_t st) -> int {
    CU(k_moe_combine_bwd(dx_, yback, H, r_pos_, r_wts_, T, k, H, nullptr, r_dw_, st, counts_all,
                         r_excl_, ep_, E, ep_i_, d_dyrecv_peers_, H, lo, hi));
    return OPX_OK;
  };
  if (fdy && !overlap) {
    TRY(combine_bwd_to(0, El_, cs_));
    mk("combine_bwd", "combine_bwd,a2a_combine_grad");
  } else if (!fdy) {
    CU(k_moe_combine_bwd(dx_, yback, H, r_pos_, r_wts_, T, k, H, dyp_, r_dw_, cs_));
    mk("combine_bwd");
  }
  // experts [lo, hi): zero-pad, dgrad/wgrad of down, SwiGLU backward,
  // dgrad/wgrad of gate|up (wgrad K = 128-padded segment rows)
  auto experts_bwd = [&](int lo, int hi, cudaStream_t st) -> int {
    const int n = hi - lo;
    const int64_t gs_d = int64_t(H) * Fe, gs_gu = int64_t(2) * Fe * H;  // slab sizes
    const int epi_w = eu.gbf ? GEMM_EPI_BF16 : GEMM_EPI_F32;
    CU(k_moe_zero_pad(dyrecv, H, H, g_start_ + lo, g_rows_ + lo, g_rows_pad_ + lo, n, st));
    CU(gemm_run(grouped(0, Fe, H, dyrecv, H, false, Wd + lo * gs_d, Fe, true, GEMM_EPI_BF16, dact_e_,
                        Fe, n, 0, g_start_ + lo, g_rows_ + lo, cap_rows_, 0),
                st));
    CU(gemm_run(grouped(H, Fe, 0, dyrecv, H, true, act_e_, Fe, true, epi_w,
                        eu.gat(Ge, eu.params[1].off + lo * gs_d), Fe, n, 1, g_start_ + lo,
                        g_rows_pad_ + lo, cap_rows_, gs_d),
                st));
    CU(k_moe_swiglu_bwd(dact_e_, gu_e_, dgu_e_, g_start_ + lo, g_rows_ + lo, g_rows_pad_ + lo, n, Fe,
                        int(cap_rows_), st));
    {
      // dX rows (fused: straight from the epilogue) back to their token owners
      GemmDesc g = grouped(0, H, 2 * Fe, dgu_e_, 2 * Fe, false, Wgu + lo * gs_gu, H, true,
                           fusedc ? GEMM_EPI_ROWMAP : GEMM_EPI_BF16, dx_e_, H, n, 0, g_start_ + lo,
                           g_rows_ + lo, cap_rows_, 0);
      g.rm_dst = d_dxback_peers_;
      g.rm_cnt = rm_cnt_ + int64_t(lo) * ep_;
      g.rm_off = rm_off_ + int64_t(lo) * ep_;
      g.rm_ep = ep_;
      CU(gemm_run(g, st));
    }
    CU(gemm_run(grouped(2 * Fe, H, 0, dgu_e_, 2 * Fe, true, xrecv, H, true, epi_w,
                        eu.gat(Ge, eu.params[0].off + lo * gs_gu), H, n, 1, g_start_ + lo,
                        g_rows_pad_ + lo, cap_rows_, gs_gu),
                st));
    return OPX_OK;
  };
  if (overlap) {
    // moe_overlap: the second expert half's dY dispatch overlaps the first
    // half's expert backward, and the first half's dX combine the second's
    const int h = El_ / 2;
    cudaEvent_t ready = ev(), done_a = ev(), done_b = ev();
    CU(cudaEventRecord(ready, cs_));
    CU(cudaStreamWaitEvent(xs2_, ready, 0));
    if (fdy)
      TRY(combine_bwd_to(h, El_, xs2_));
    else
      CU(k_moe_dispatch(dyp_, H, 1, r_pairat_, P, k, counts_all, r_excl_, ep_, E, ep_i_,
                        d_dyrecv_peers_, H, H, xs2_, h, El_));
    TRY(barrier_ep3(xs2_));
    if (fdy) {
      TRY(combine_bwd_to(0, h, cs_));
      mk("combine_bwd", "combine_bwd,a2a_combine_grad");
    } else {
      CU(k_moe_dispatch(dyp_, H, 1, r_pairat_, P, k, counts_all, r_excl_, ep_, E, ep_i_,
                        d_dyrecv_peers_, H, H, cs_, 0, h));
      mk("a2a_combine_grad");
    }
    TRY(barrier_ep(cs_));
    mk("a2a_wait");
    TRY(experts_bwd(0, h, cs_));
    CU(cudaEventRecord(done_a, cs_));
    mk("experts", fusedc ? "experts,a2a_dispatch_grad" : nullptr);
    if (moe_serial_halves()) CU(cudaStreamWaitEvent(xs2_, done_a, 0));
    TRY(experts_bwd(h, El_, xs2_));
    TRY(dx_return(h, El_ - h, xs2_));
    TRY(barrier_ep3(xs2_));
    CU(cudaEventRecord(done_b, xs2_));
    TRY(dx_return(0, h, cs_));
    if (!fusedc) mk("a2a_dispatch_grad");
    TRY(barrier_ep(cs_));
    CU(cudaStreamWaitEvent(cs_, done_b, 0));
    mk("experts_b");  // half B's expert backward, dX combine and barrier
  } else {
    if (!fdy) {
      CU(k_moe_dispatch(dyp_, H, 1, r_pairat_, P, k, counts_all, r_excl_, ep_, E, ep_i_,
                        d_dyrecv_peers_, H, H, cs_));
      mk("a2a_combine_grad");
    }
    TRY(barrier_ep(cs_));
    mk("a2a_wait");
    // a2a_dispatch_grad: input grads travel back to the token owners
    TRY(experts_bwd(0, El_, cs_));
    mk("experts", fusedc ? "experts,a2a_dispatch_grad" : nullptr);
    TRY(dx_return(0, El_, cs_));
    if (!fusedc) mk("a2a_dispatch_grad");
    TRY(barrier_ep(cs_));
    mk("a2a_wait");
  }
  CU(k_moe_unpermute(dxback, H, r_pos_, nullptr, T, k, H, nullptr, dh2, cs_));
  // router: renormalised-softmax backward, then dh2 += dlogits . Wr, dWr = dlogits^T h2
  CU(k_moe_router_bwd(r_dw_, r_wts_, r_idx_, T, k, E, dlogits_, cs_));
  {
    GemmDesc g;
    g.M = T;
    g.N = H;
    g.K = E;
    g.A = dlogits_;
    g.lda = E;
    g.B = Wr;
    g.ldb = H;
    g.b_mn = true;
    g.epi = GEMM_EPI_F32_RESID;
    g.D = dh2;
    g.ldd = H;
    g.R = dh2;
    g.ldr = H;
    CU(gemm_run(g, cs_));
  }
  CU(gemm_run(grouped(E, H, 0, dlogits_, E, true, h2_, H, true, GEMM_EPI_F32, wr_part_, H,
                      wr_split_, 1, wr_gs_, wr_gr_, T, int64_t(E) * H),
              cs_));
  CU(k_sum_partials(wr_part_, wr_split_, int64_t(E) * H, u.gat(G, u.params[6].off), cs_, u.gbf));
  mk("router");
  if (kept) {
    // every peer passed the dispatch_grad barrier above, so all of them are done
    // with their receive buffers for this layer: re-send the next MoE layer's tokens
    const int ln = next_moe_below(l);
    if (ln >= 0) {
      cudaEvent_t e = ev();
      CU(cudaEventRecord(e, cs_));
      CU(cudaStreamWaitEvent(xs_, e, 0));
      TRY(moe_redispatch(ln));
    }
  }
  gu_e_ = gu_sv;
  act_e_ = act_sv;
  return OPX_OK;
}

}  // namespace opx
