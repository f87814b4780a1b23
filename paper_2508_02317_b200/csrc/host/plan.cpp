// Host plan layer: accounting, mesh, validation, volumes and config parsing.
// Semantics follow omniplan (file:line cited per function); the code is an
// independent restatement organised around what the executor needs.
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <stdexcept>

#include "json.hpp"

namespace opx {

using nlohmann::json;

// ---------------------------------------------------------------------------
// Parameter accounting.  specs.cpp:36-50 (layer_shape), :52-55 (head), :93-107.
// Bias-free blocks: q,k,v,o projections, two RMSNorm vectors, gated MLP
// (3*H*ffn) or E experts of 3*H*ffn_e plus an H*E router on MoE layers.
// ---------------------------------------------------------------------------
LayerParams layer_params(const Arch& a, i64 layer) {
  LayerParams p;
  p.qkv = a.hidden * (a.q_width() + 2 * a.kv_width()) + a.hidden;
  p.out = a.hidden * a.q_width();
  if (a.is_moe_layer(layer)) {
    p.moe = true;
    p.router = a.hidden * a.moe->experts;
    p.experts_total = a.moe->experts * 3 * a.hidden * a.moe->ffn;
    p.experts_active = 3 * a.hidden * a.moe->ffn * a.moe->top_k;
    p.mlp = a.hidden;
  } else {
    p.mlp = 3 * a.hidden * a.ffn + a.hidden;
  }
  return p;
}

i64 head_params(const Arch& a) { return 2 * a.vocab * a.hidden + a.hidden; }

i64 arch_params(const Arch& a, bool active_only) {
  i64 n = head_params(a);
  for (i64 l = 0; l < a.layers; ++l) {
    LayerParams p = layer_params(a, l);
    n += active_only ? p.active() : p.total();
  }
  return n;
}

i64 module_params(const Module& m, bool active_only) {
  if (m.arch) return arch_params(*m.arch, active_only);
  return m.raw_params.value_or(0);
}

const Module* Model::foundation() const {
  for (auto& m : modules)
    if (m.kind == ModuleKind::foundation) return &m;
  return nullptr;
}

double flops_per_token_ref(const Model& model, i64 S) {
  double f = 0;
  for (const Module& m : model.modules) {
    f += (m.trainable ? 6.0 : 2.0) * double(module_params(m, true));
    if (m.kind == ModuleKind::foundation && m.arch)
      f += (m.trainable ? 3.0 : 1.0) * 2.0 * double(m.arch->layers) * double(m.arch->hidden) *
           double(S);
  }
  return f;
}

// specs.cpp:109-213
std::vector<std::string> check_cluster(const Cluster& c) {
  std::vector<std::string> out;
  if (c.num_nodes < 1 || c.gpus_per_node < 1) out.push_back("cluster world must be at least 1 device");
  if (!(c.peak_flops > 0)) out.push_back("gpu.peak_flops must be > 0");
  if (!(c.hbm_bytes > 0)) out.push_back("gpu.hbm_bytes must be > 0");
  if (!(c.intra_bw > 0 && c.inter_bw > 0 && c.intra_lat > 0 && c.inter_lat > 0))
    out.push_back("link bandwidths and latencies must be > 0");
  if (c.intra_bw < c.inter_bw) out.push_back("intra_node_bw must be >= inter_node_bw");
  return out;
}

std::vector<std::string> check_arch(const Arch& a) {
  std::vector<std::string> out;
  if (a.layers < 0) out.push_back("layers must be >= 0");
  if (std::min({a.hidden, a.heads, a.head_dim, a.ffn, a.vocab, a.kv_heads}) < 1)
    out.push_back("transformer dimensions must be >= 1");
  if (a.heads * a.head_dim != a.hidden) out.push_back("heads * head_dim must equal hidden");
  if (a.kv_heads > 0 && a.heads % a.kv_heads) out.push_back("kv_heads must divide heads");
  if (a.moe) {
    if (a.moe->top_k < 1 || a.moe->top_k > a.moe->experts)
      out.push_back("moe top_k must satisfy 1 <= top_k <= num_experts");
    if (a.moe->stride < 1) out.push_back("moe_layer_stride must be >= 1");
    if (a.moe->ffn < 1) out.push_back("expert_ffn_dim must be >= 1");
  }
  return out;
}

std::vector<std::string> check_model(const Model& m) {
  std::vector<std::string> out;
  int n_found = 0;
  for (const Module& mod : m.modules) {
    n_found += mod.kind == ModuleKind::foundation;
    const std::string tag = "module '" + mod.name + "': ";
    if (mod.arch.has_value() == mod.raw_params.has_value())
      out.push_back(tag + "exactly one of arch / raw_param_count must be set");
    if (mod.tokens_per_item < 0) out.push_back(tag + "tokens_per_item must be >= 0");
    if (mod.arch)
      for (auto& s : check_arch(*mod.arch)) out.push_back(tag + s);
  }
  if (n_found != 1) out.push_back("model must contain exactly one foundation module");
  if (m.dtype_bytes != 1 && m.dtype_bytes != 2 && m.dtype_bytes != 4)
    out.push_back("param_dtype_bytes must be 1, 2 or 4");
  return out;
}

std::vector<std::string> check_workload(const Workload& w) {
  std::vector<std::string> out;
  if (w.seq_len < 1) out.push_back("seq_len must be >= 1");
  if (w.micro_batch < 1) out.push_back("micro_batch must be >= 1");
  if (w.global_batch < w.micro_batch) out.push_back("global_batch must be >= micro_batch");
  if (!w.mix.empty()) {
    double s = 0;
    for (auto& [k, v] : w.mix) {
      if (v < 0) out.push_back("modality fraction for '" + k + "' must be >= 0");
      s += v;
    }
    if (std::fabs(s - 1.0) > 1e-9) out.push_back("modality fractions must sum to 1");
  }
  return out;
}

// ---------------------------------------------------------------------------
// Mesh: row-major, last dimension fastest (mesh.cpp:21-105).
// ---------------------------------------------------------------------------
int Mesh::index_of(const std::string& n) const {
  for (size_t i = 0; i < dims.size(); ++i)
    if (dims[i].name == n) return int(i);
  return -1;
}

Mesh make_mesh(const std::vector<MeshDim>& dims, i64 world) {
  i64 prod = 1;
  for (size_t i = 0; i < dims.size(); ++i) {
    if (dims[i].size < 1) throw std::invalid_argument("mesh dim '" + dims[i].name + "' has size < 1");
    for (size_t j = 0; j < i; ++j)
      if (dims[j].name == dims[i].name)
        throw std::invalid_argument("duplicate mesh dim name '" + dims[i].name + "'");
    prod *= dims[i].size;
  }
  if (prod != world)
    throw std::invalid_argument("mesh dim sizes multiply to " + std::to_string(prod) +
                                ", expected world size " + std::to_string(world));
  return Mesh{dims, world};
}

std::vector<i64> coord_of(const Mesh& m, i64 rank) {
  if (rank < 0 || rank >= m.world) throw std::out_of_range("rank outside mesh");
  std::vector<i64> c(m.dims.size());
  for (size_t i = m.dims.size(); i-- > 0;) {
    c[i] = rank % m.dims[i].size;
    rank /= m.dims[i].size;
  }
  return c;
}

i64 rank_of(const Mesh& m, const std::vector<i64>& c) {
  if (c.size() != m.dims.size()) throw std::invalid_argument("coordinate arity does not match mesh");
  i64 r = 0;
  for (size_t i = 0; i < c.size(); ++i) {
    if (c[i] < 0 || c[i] >= m.dims[i].size) throw std::out_of_range("coordinate out of range");
    r = r * m.dims[i].size + c[i];
  }
  return r;
}

std::vector<Group> groups_along(const Mesh& m, const std::vector<std::string>& names) {
  std::vector<char> sel(m.dims.size(), 0);
  for (auto& n : names) {
    int i = m.index_of(n);
    if (i < 0) throw std::invalid_argument("unknown mesh dim '" + n + "'");
    sel[size_t(i)] = 1;
  }
  // A group = ranks agreeing on every unselected coordinate.  Enumerate the
  // unselected "base" coordinates in rank order and expand each into its
  // members; members come out ascending because selected coords are walked
  // in row-major order.
  std::vector<Group> out;
  std::vector<char> seen(size_t(m.world), 0);
  for (i64 r = 0; r < m.world; ++r) {
    if (seen[size_t(r)]) continue;
    Group g;
    g.dims = names;
    auto base = coord_of(m, r);
    for (i64 q = r; q < m.world; ++q) {
      auto c = coord_of(m, q);
      bool same = true;
      for (size_t i = 0; i < c.size() && same; ++i) same = sel[i] || c[i] == base[i];
      if (same) {
        g.members.push_back(q);
        seen[size_t(q)] = 1;
      }
    }
    out.push_back(std::move(g));
  }
  return out;  // ordered by lowest member by construction
}

Group group_of(const std::vector<Group>& gs, i64 rank) {
  for (auto& g : gs)
    if (std::find(g.members.begin(), g.members.end(), rank) != g.members.end()) return g;
  throw std::invalid_argument("rank not in any group");
}

// ---------------------------------------------------------------------------
// Plan validation with the reference's stable codes (plan.cpp:19-83).
// ---------------------------------------------------------------------------
std::vector<Violation> validate_plan(const Plan& p, const Cluster& c, const Model& m,
                                     const Workload& w) {
  std::vector<Violation> v;
  auto add = [&](const char* code, std::string msg) { v.push_back({code, std::move(msg)}); };
  auto s = [](i64 x) { return std::to_string(x); };
  if (std::min({p.dp_replicate, p.dp_shard, p.sp, p.ep, p.micro_batch}) < 1) {
    add("size_positive", "all plan sizes must be >= 1");
    return v;
  }
  if (p.tp != 1 || p.pp != 1)
    add("tp_pp_unsupported", "tensor/pipeline parallel sizing is not supported; tp and pp must be 1");
  if (p.world() != c.world())
    add("world_product", "dp_replicate*dp_shard*sp = " + s(p.world()) +
                             " does not equal world size " + s(c.world()));
  for (const Module& mod : m.modules) {
    if (!mod.arch) continue;
    const Arch& a = *mod.arch;
    if (mod.kind == ModuleKind::foundation && p.sp > 1) {
      if (a.heads % p.sp)
        add("head_divisibility", "module '" + mod.name + "': heads " + s(a.heads) +
                                     " not divisible by sp " + s(p.sp));
      if (a.kv_heads % p.sp)
        add("kv_head_divisibility", "module '" + mod.name + "': kv_heads " + s(a.kv_heads) +
                                        " not divisible by sp " + s(p.sp));
    }
    if (a.moe && a.moe->experts % p.ep)
      add("expert_divisibility", "module '" + mod.name + "': num_experts " +
                                     s(a.moe->experts) + " not divisible by ep " + s(p.ep));
  }
  if (w.seq_len % p.sp)
    add("seq_divisibility", "seq_len " + s(w.seq_len) + " not divisible by sp " + s(p.sp));
  if (p.shard_degree() % p.ep)
    add("ep_factorization",
        "ep " + s(p.ep) + " does not divide dp_shard*sp = " + s(p.shard_degree()));
  const i64 unit = p.dp_width() * p.micro_batch;
  if (w.global_batch % unit)
    add("batch_divisibility", "global_batch " + s(w.global_batch) +
                                  " not divisible by dp_replicate*dp_shard*micro_batch = " +
                                  s(unit));
  return v;
}

ExpertSharding expert_sharding(const Plan& p, const Arch& a) {
  if (!a.moe) throw std::invalid_argument("expert_sharding called on a dense module");
  return {a.moe->experts / p.ep, p.shard_degree() / p.ep};
}

Mesh plan_mesh(const Plan& p) {
  return make_mesh({{"dp_replicate", p.dp_replicate}, {"dp_shard", p.dp_shard}, {"sp", p.sp}},
                   p.world());
}

std::vector<Group> ep_groups(const Plan& p) {
  std::vector<Group> out;
  for (const Group& flat : groups_along(plan_mesh(p), {"dp_shard", "sp"}))
    for (size_t b = 0; b + size_t(p.ep) <= flat.members.size(); b += size_t(p.ep)) {
      Group g;
      g.dims = {"ep"};
      g.members.assign(flat.members.begin() + long(b), flat.members.begin() + long(b + p.ep));
      out.push_back(std::move(g));
    }
  return out;
}

std::string plan_label(const Plan& p) {
  std::string l = p.dp_replicate > 1 ? "HSDP" + std::to_string(p.dp_replicate) : "FSDP";
  if (p.sp > 1 || p.ep > 1) l += "+SP" + std::to_string(p.sp);
  if (p.ep > 1) l += "+EP" + std::to_string(p.ep);
  return l;
}

// ---------------------------------------------------------------------------
// Volumes: ring accounting per rank (comm.cpp:8-89).
// ---------------------------------------------------------------------------
double vol_collective(Coll k, double full, i64 g) {
  if (g <= 1 || full <= 0) return 0;
  const double f = double(g - 1) / double(g);
  return (k == Coll::all_reduce ? 2.0 : 1.0) * full * f;
}

double vol_ulysses(const Plan& p, const Arch& a, const Workload& w, i64 b) {
  if (p.sp <= 1) return 0;
  const double width = 2.0 * double(a.hidden) + 2.0 * double(a.kv_width());
  const double T = double(p.micro_batch) * double(w.seq_len) / double(p.sp);
  return width * T * double(b) * double(p.sp - 1) / double(p.sp);
}

double vol_fsdp_step(const Plan& p, i64 n, i64 b) {
  return 3.0 * vol_collective(Coll::all_gather, double(n) * double(b), p.shard_degree());
}

double vol_hsdp(const Plan& p, i64 n, i64 b) {
  if (p.dp_replicate <= 1) return 0;
  return vol_collective(Coll::all_reduce, double(n) * double(b) / double(p.shard_degree()),
                        p.dp_replicate);
}

double vol_ep_dispatch(const Plan& p, const Arch& a, i64 T, i64 b) {
  if (p.ep <= 1 || !a.moe) return 0;
  const double payload = double(T) * double(a.moe->top_k) * double(a.hidden) * double(b);
  return 2.0 * payload * double(p.ep - 1) / double(p.ep) * p.moe_imbalance;
}

Interval owned_interval(i64 n, i64 parts, i64 r) {
  if (r < 0 || r >= parts) throw std::out_of_range("rank outside [0, parts)");
  const i64 c = (n + parts - 1) / parts;
  return {std::min(r * c, n), std::min((r + 1) * c, n)};
}

i64 layout_chunk(i64 n, i64 parts, i64 align) {
  if (parts <= 0) throw std::invalid_argument("parts must be positive");
  if (align <= 0) return (n + parts - 1) / parts;
  const i64 q = align * parts;
  return (n + q - 1) / q * q / parts;
}

Interval chunk_interval(i64 n, i64 c, i64 r) { return {std::min(r * c, n), std::min((r + 1) * c, n)}; }

// Interval intersection of every destination shard with every source shard,
// ordered by (dst_rank, dst_offset) like make_plan (reshard.cpp:20-56).
std::vector<CopyOp> reshard_plan(i64 n, i64 sp, i64 sc, i64 dp, i64 dc) {
  if (sp <= 0 || dp <= 0) throw std::invalid_argument("parts must be positive");
  if (sc * sp < n || dc * dp < n) throw std::invalid_argument("layout does not cover numel");
  std::vector<CopyOp> ops;
  for (i64 d = 0; d < dp; ++d) {
    const Interval di = chunk_interval(n, dc, d);
    if (di.end <= di.begin) continue;
    for (i64 s = 0; s < sp; ++s) {
      const Interval si = chunk_interval(n, sc, s);
      const i64 lo = std::max(di.begin, si.begin), hi = std::min(di.end, si.end);
      if (lo < hi) ops.push_back({s, lo - si.begin, d, lo - di.begin, hi - lo});
    }
  }
  return ops;
}

// Same checks as verify (reshard.cpp:58-110): positive lengths, total == numel,
// every destination rank written contiguously from 0 with no gap or overlap.
std::vector<std::string> reshard_verify(const std::vector<CopyOp>& ops, i64 n) {
  std::vector<std::string> v;
  i64 total = 0, max_dst = -1;
  for (auto& o : ops) {
    total += o.len;
    max_dst = std::max(max_dst, o.dst_rank);
    if (o.len <= 0) v.push_back("non-positive copy length in op for dst rank " + std::to_string(o.dst_rank));
  }
  if (total != n) v.push_back("copy lengths sum to " + std::to_string(total) + ", expected " + std::to_string(n));
  std::vector<std::vector<Interval>> per(size_t(max_dst + 1));
  for (auto& o : ops)
    if (o.len > 0) per[size_t(o.dst_rank)].push_back({o.dst_offset, o.dst_offset + o.len});
  i64 covered = 0;
  for (size_t d = 0; d < per.size(); ++d) {
    auto& iv = per[d];
    std::sort(iv.begin(), iv.end(), [](const Interval& a, const Interval& b) { return a.begin < b.begin; });
    i64 cur = 0;
    for (auto& i : iv) {
      if (i.begin < cur) v.push_back("overlapping writes on dst rank " + std::to_string(d));
      else if (i.begin > cur) v.push_back("coverage gap on dst rank " + std::to_string(d));
      cur = std::max(cur, i.end);
    }
    covered += cur;
  }
  if (covered != n && total == n) v.push_back("destination coverage is " + std::to_string(covered));
  return v;
}

// ---------------------------------------------------------------------------
// JSON configs: same field names as config_io.cpp:52-151.
// ---------------------------------------------------------------------------
namespace {

[[noreturn]] void cfg_fail(const std::string& ctx, const std::string& what) {
  throw ConfigError(ctx.empty() ? what : ctx + ": " + what);
}

json parse_text(const std::string& text, const char* ctx) {
  try {
    return json::parse(text);
  } catch (const std::exception& e) {
    cfg_fail(ctx, std::string("JSON parse error: ") + e.what());
  }
}

void need(const json& j, std::initializer_list<const char*> keys, const std::string& ctx) {
  if (!j.is_object()) cfg_fail(ctx, "expected a JSON object");
  for (const char* k : keys)
    if (!j.contains(k)) cfg_fail(ctx, std::string("missing required field '") + k + "'");
}

void ok_or_fail(const std::vector<std::string>& probs, const std::string& ctx) {
  if (probs.empty()) return;
  std::string s;
  for (size_t i = 0; i < probs.size(); ++i) s += (i ? "; " : "") + probs[i];
  cfg_fail(ctx, s);
}

template <class T>
T get(const json& j, const char* k, const std::string& ctx) {
  try {
    return j.at(k).get<T>();
  } catch (const std::exception& e) {
    cfg_fail(ctx, std::string("field '") + k + "': " + e.what());
  }
}

Arch arch_from(const json& j, const std::string& ctx) {
  need(j, {"layers", "hidden", "heads", "kv_heads", "head_dim", "ffn_dim", "vocab"}, ctx);
  Arch a;
  a.layers = get<i64>(j, "layers", ctx);
  a.hidden = get<i64>(j, "hidden", ctx);
  a.heads = get<i64>(j, "heads", ctx);
  a.kv_heads = get<i64>(j, "kv_heads", ctx);
  a.head_dim = get<i64>(j, "head_dim", ctx);
  a.ffn = get<i64>(j, "ffn_dim", ctx);
  a.vocab = get<i64>(j, "vocab", ctx);
  a.window_merge = j.value("window_merge", i64{4});
  if (j.contains("fullatt_blocks")) a.fullatt_blocks = get<std::vector<i64>>(j, "fullatt_blocks", ctx);
  a.rope_theta = j.value("rope_theta", 10000.0);
  if (j.contains("moe")) {
    const json& mj = j.at("moe");
    need(mj, {"num_experts", "top_k", "expert_ffn_dim"}, ctx + ".moe");
    Moe m;
    m.experts = get<i64>(mj, "num_experts", ctx);
    m.top_k = get<i64>(mj, "top_k", ctx);
    m.ffn = get<i64>(mj, "expert_ffn_dim", ctx);
    m.stride = mj.value("moe_layer_stride", i64{1});
    a.moe = m;
  }
  return a;
}

}  // namespace

Cluster parse_cluster_json(const std::string& text) {
  json j = parse_text(text, "cluster");
  need(j, {"num_nodes", "gpus_per_node", "gpu", "link"}, "cluster");
  need(j.at("gpu"), {"peak_flops", "hbm_bytes"}, "cluster.gpu");
  need(j.at("link"), {"intra_node_bw", "inter_node_bw", "intra_latency", "inter_latency"},
       "cluster.link");
  Cluster c;
  c.num_nodes = get<i64>(j, "num_nodes", "cluster");
  c.gpus_per_node = get<i64>(j, "gpus_per_node", "cluster");
  c.peak_flops = get<double>(j.at("gpu"), "peak_flops", "cluster.gpu");
  c.hbm_bytes = get<double>(j.at("gpu"), "hbm_bytes", "cluster.gpu");
  const json& l = j.at("link");
  c.intra_bw = get<double>(l, "intra_node_bw", "cluster.link");
  c.inter_bw = get<double>(l, "inter_node_bw", "cluster.link");
  c.intra_lat = get<double>(l, "intra_latency", "cluster.link");
  c.inter_lat = get<double>(l, "inter_latency", "cluster.link");
  ok_or_fail(check_cluster(c), "cluster");
  return c;
}

Model parse_model_json(const std::string& text) {
  json j = parse_text(text, "model");
  need(j, {"modules"}, "model");
  Model m;
  m.dtype_bytes = j.value("param_dtype_bytes", i64{2});
  for (const json& mj : j.at("modules")) {
    need(mj, {"name", "kind"}, "model.modules[]");
    Module mod;
    mod.name = mj.at("name").get<std::string>();
    const std::string ctx = "model.modules['" + mod.name + "']";
    const std::string kind = mj.at("kind").get<std::string>();
    if (kind == "encoder") mod.kind = ModuleKind::encoder;
    else if (kind == "foundation") mod.kind = ModuleKind::foundation;
    else if (kind == "decoder") mod.kind = ModuleKind::decoder;
    else cfg_fail(ctx, "unknown module kind '" + kind + "'");
    mod.trainable = mj.value("trainable", false);
    mod.tokens_per_item = mj.value("tokens_per_item", i64{0});
    if (mj.contains("arch")) mod.arch = arch_from(mj.at("arch"), ctx + ".arch");
    if (mj.contains("raw_param_count")) mod.raw_params = mj.at("raw_param_count").get<i64>();
    m.modules.push_back(std::move(mod));
  }
  ok_or_fail(check_model(m), "model");
  if (!m.foundation()->arch) cfg_fail("model", "the foundation module requires an arch");
  return m;
}

Workload parse_workload_json(const std::string& text) {
  json j = parse_text(text, "workload");
  need(j, {"seq_len", "micro_batch", "global_batch"}, "workload");
  Workload w;
  w.seq_len = get<i64>(j, "seq_len", "workload");
  w.micro_batch = get<i64>(j, "micro_batch", "workload");
  w.global_batch = get<i64>(j, "global_batch", "workload");
  if (j.contains("modality_mix"))
    for (auto& [k, v] : j.at("modality_mix").items()) w.mix[k] = v.get<double>();
  ok_or_fail(check_workload(w), "workload");
  return w;
}

// Plan objects use the to_json(ParallelPlan) keys (config_io.cpp:248-262) and
// the CLI flag defaults (plan.hpp:26-46); dp_shard may be omitted and is then
// derived as world / (dp_replicate * sp) by the caller.
Plan parse_plan_json(const std::string& text) {
  json j = parse_text(text, "plan");
  if (!j.is_object()) cfg_fail("plan", "expected a JSON object");
  Plan p;
  p.dp_replicate = j.value("dp_replicate", i64{1});
  p.dp_shard = j.value("dp_shard", i64{-1});
  p.sp = j.value("sp", i64{1});
  p.ep = j.value("ep", i64{1});
  p.micro_batch = j.value("micro_batch", i64{1});
  const std::string rc = j.value("recompute", std::string("full"));
  if (rc != "full" && rc != "none") cfg_fail("plan", "recompute must be 'full' or 'none'");
  p.recompute_full = rc == "full";
  p.offload_optimizer = j.value("offload_optimizer", false);
  p.offload_activations = j.value("offload_activations", false);
  p.async_ulysses = j.value("async_ulysses", false);
  p.moe_overlap = j.value("moe_overlap", false);
  p.prefetch_depth = j.value("fsdp_prefetch_depth", i64{1});
  p.moe_imbalance = j.value("moe_imbalance", 1.0);
  p.tp = j.value("tp", i64{1});
  p.pp = j.value("pp", i64{1});
  return p;
}

std::string plan_to_json(const Plan& p) {
  json j{{"dp_replicate", p.dp_replicate},
         {"dp_shard", p.dp_shard},
         {"sp", p.sp},
         {"ep", p.ep},
         {"micro_batch", p.micro_batch},
         {"recompute", p.recompute_full ? "full" : "none"},
         {"offload_optimizer", p.offload_optimizer},
         {"offload_activations", p.offload_activations},
         {"async_ulysses", p.async_ulysses},
         {"moe_overlap", p.moe_overlap},
         {"fsdp_prefetch_depth", p.prefetch_depth},
         {"moe_imbalance", p.moe_imbalance},
         {"label", plan_label(p)}};
  return j.dump();
}

}  // namespace opx
