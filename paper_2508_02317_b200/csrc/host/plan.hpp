// Host-side parallel-plan layer of the opx executor.
//
// This is the drop-in half of the boundary: the value types, validation codes,
// mesh/group derivation and work accounting that omniplan's planner exposes
// (reference: proj/include/omniplan/{specs,mesh,plan,comm}.hpp), restated so the
// executor can consume the same JSON configs and refuse the same plans.  Nothing
// here touches the GPU.
//
//   reference symbol                         -> here
//   specs.hpp:48-62   TransformerSpec         -> opx::Arch
//   specs.hpp:39-44   MoeSpec                 -> opx::Moe
//   specs.hpp:68-84   ModuleSpec/ModelSpec    -> opx::Module / opx::Model
//   specs.hpp:88-95   WorkloadSpec            -> opx::Workload
//   specs.hpp:15-35   Gpu/Link/ClusterSpec    -> opx::Cluster
//   plan.hpp:26-46    ParallelPlan            -> opx::Plan
//   plan.hpp:68-69    validate                -> opx::validate_plan
//   plan.hpp:75       resolve_expert_sharding -> opx::expert_sharding
//   plan.hpp:101,105  plan_mesh / ep_groups   -> opx::plan_mesh / opx::ep_groups
//   mesh.hpp:35-43    groups_along            -> opx::groups_along
//   specs.cpp:93-107  flops_per_token         -> opx::flops_per_token_ref
//   comm.cpp:8-105    *_volume                -> opx::vol_*
#pragma once

#include <cstdint>
#include <exception>
#include <map>
#include <optional>
#include <string>
#include <vector>

namespace opx {

using i64 = std::int64_t;

struct Cluster {
  i64 num_nodes = 1, gpus_per_node = 1;
  double peak_flops = 0, hbm_bytes = 0;
  double intra_bw = 0, inter_bw = 0, intra_lat = 0, inter_lat = 0;
  i64 world() const { return num_nodes * gpus_per_node; }
};

struct Moe {
  i64 experts = 1, top_k = 1, ffn = 1, stride = 1;
};

struct Arch {
  i64 layers = 0, hidden = 0, heads = 1, kv_heads = 1, head_dim = 1, ffn = 1, vocab = 0;
  std::optional<Moe> moe;
  // Vision encoders (Qwen2.5-VL; optional arch keys the reference ignores):
  // window side in 2x2 merge units, full-attention blocks (default: every 8th
  // and the last), 2-D RoPE base
  i64 window_merge = 4;
  std::optional<std::vector<i64>> fullatt_blocks;
  double rope_theta = 10000.0;
  bool is_moe_layer(i64 l) const { return moe && (l + 1) % moe->stride == 0; }
  i64 q_width() const { return heads * head_dim; }
  i64 kv_width() const { return kv_heads * head_dim; }
};

enum class ModuleKind { encoder, foundation, decoder };

struct Module {
  std::string name;
  ModuleKind kind = ModuleKind::encoder;
  std::optional<Arch> arch;
  std::optional<i64> raw_params;
  bool trainable = false;
  i64 tokens_per_item = 0;
};

struct Model {
  std::vector<Module> modules;
  i64 dtype_bytes = 2;
  const Module* foundation() const;
};

struct Workload {
  i64 seq_len = 1, micro_batch = 1, global_batch = 1;
  std::map<std::string, double> mix;
  double fraction(const std::string& name) const {
    auto it = mix.find(name);
    return it == mix.end() ? 0.0 : it->second;
  }
};

struct Plan {
  i64 dp_replicate = 1, dp_shard = 1, sp = 1, ep = 1, micro_batch = 1;
  bool recompute_full = true;
  bool offload_optimizer = false, offload_activations = false;
  bool async_ulysses = false, moe_overlap = false;
  i64 prefetch_depth = 1;
  double moe_imbalance = 1.0;
  i64 tp = 1, pp = 1;
  i64 world() const { return dp_replicate * dp_shard * sp; }
  i64 shard_degree() const { return dp_shard * sp; }
  i64 dp_width() const { return dp_replicate * dp_shard; }
};

struct Violation {
  std::string code, message;
};

// ---- parameter accounting (specs.cpp:13-55) --------------------------------
struct LayerParams {
  i64 qkv = 0;      // Wq, Wk, Wv + attention norm
  i64 out = 0;      // Wo
  i64 mlp = 0;      // dense gated MLP + mlp norm (only the norm on MoE layers)
  bool moe = false;
  i64 router = 0;
  i64 experts_total = 0, experts_active = 0;
  i64 total() const { return qkv + out + mlp + router + experts_total; }
  i64 active() const { return qkv + out + mlp + router + experts_active; }
  double gathered(i64 ep) const {
    return double(qkv + out + mlp + router) + double(experts_total) / double(ep);
  }
};
LayerParams layer_params(const Arch& a, i64 layer);
i64 head_params(const Arch& a);
i64 arch_params(const Arch& a, bool active_only);
i64 module_params(const Module& m, bool active_only);
double flops_per_token_ref(const Model& m, i64 seq_len);

std::vector<std::string> check_cluster(const Cluster& c);
std::vector<std::string> check_arch(const Arch& a);
std::vector<std::string> check_model(const Model& m);
std::vector<std::string> check_workload(const Workload& w);

// ---- mesh ------------------------------------------------------------------
struct MeshDim {
  std::string name;
  i64 size = 1;
};
struct Mesh {
  std::vector<MeshDim> dims;
  i64 world = 1;
  int index_of(const std::string& n) const;
};
struct Group {
  std::vector<std::string> dims;
  std::vector<i64> members;
};
Mesh make_mesh(const std::vector<MeshDim>& dims, i64 world);  // throws std::invalid_argument
std::vector<i64> coord_of(const Mesh& m, i64 rank);
i64 rank_of(const Mesh& m, const std::vector<i64>& coord);
std::vector<Group> groups_along(const Mesh& m, const std::vector<std::string>& names);

// ---- plan ------------------------------------------------------------------
std::vector<Violation> validate_plan(const Plan& p, const Cluster& c, const Model& m,
                                     const Workload& w);
struct ExpertSharding {
  i64 experts_per_rank = 0, per_expert_fsdp_degree = 0;
};
ExpertSharding expert_sharding(const Plan& p, const Arch& a);
Mesh plan_mesh(const Plan& p);
std::vector<Group> ep_groups(const Plan& p);
std::string plan_label(const Plan& p);

// The group of `rank` along the given mesh dims (helper for the executor).
Group group_of(const std::vector<Group>& gs, i64 rank);

// ---- communication volumes (comm.cpp) ---------------------------------------
enum class Coll { all_gather, reduce_scatter, all_reduce, all_to_all };
double vol_collective(Coll k, double full_bytes, i64 group);
double vol_ulysses(const Plan& p, const Arch& a, const Workload& w, i64 dtype_bytes);
double vol_fsdp_step(const Plan& p, i64 module_params, i64 dtype_bytes);
double vol_hsdp(const Plan& p, i64 module_params, i64 dtype_bytes);
double vol_ep_dispatch(const Plan& p, const Arch& a, i64 tokens_local, i64 dtype_bytes);

// ---- FSDP flat-shard convention (reshard.hpp:15-24 owned_interval) ----------
struct Interval {
  i64 begin = 0, end = 0;
};
Interval owned_interval(i64 numel, i64 parts, i64 rank);

// ---- reshard copy plans (reshard.cpp:20-56 make_plan, :58-110 verify) -------
// Rank r of a layout owns [min(r*c, n), min((r+1)*c, n)).  chunk = 0 means the
// reference's c = ceil(n / parts); the executor's FSDP units use
// c = round_up(n, align*parts) / parts (flat buffers padded for aligned
// collectives), so a checkpoint shard is "chunk c of the logical numel" and
// the same interval-intersection plan moves it between world sizes.
struct CopyOp {
  i64 src_rank = 0, src_offset = 0, dst_rank = 0, dst_offset = 0, len = 0;
};
i64 layout_chunk(i64 numel, i64 parts, i64 align);  // align 0 -> ceil(n/parts)
Interval chunk_interval(i64 numel, i64 chunk, i64 rank);
std::vector<CopyOp> reshard_plan(i64 numel, i64 src_parts, i64 src_chunk, i64 dst_parts,
                                 i64 dst_chunk);
std::vector<std::string> reshard_verify(const std::vector<CopyOp>& ops, i64 numel);

// ---- JSON config I/O (config_io.cpp:52-151, 248-262) -----------------------
// All parse functions throw opx::ConfigError with a path-qualified message.
struct ConfigError : std::exception {
  std::string msg;
  explicit ConfigError(std::string m) : msg(std::move(m)) {}
  const char* what() const noexcept override { return msg.c_str(); }
};
Cluster parse_cluster_json(const std::string& text);
Model parse_model_json(const std::string& text);
Workload parse_workload_json(const std::string& text);
Plan parse_plan_json(const std::string& text);  // PlanFlags-shaped object, defaults as plan.hpp
std::string plan_to_json(const Plan& p);

}  // namespace opx
