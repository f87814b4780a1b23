// TEST INFRASTRUCTURE ONLY: a C shim over the compiled reference planner
// (omniplan, /root/reference/proj/src, built by oracle/Makefile into
// oracle/_ref/libomniplan_ref.so).  tests/test_plan_ref.py uses it to check
// libopx's plan layer (validation codes, mesh groups, FLOPs, volumes) against
// the reference itself on random instances.  Never linked into libopx.
#include <cstring>
#include <sstream>
#include <string>

#include "json.hpp"
#include "omniplan/comm.hpp"
#include "omniplan/config_io.hpp"
#include "omniplan/packing.hpp"
#include "omniplan/plan.hpp"
#include "omniplan/reshard.hpp"
#include "omniplan/simulator.hpp"
#include "omniplan/step_graph.hpp"

using namespace omniplan;
using nlohmann::json;

namespace {

int out(const std::string& s, char* buf, size_t cap) {
  if (s.size() + 1 > cap) return 9;
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return 0;
}

ParallelPlan plan_from(const json& j, std::int64_t world) {
  ParallelPlan p;
  p.dp_replicate = j.value("dp_replicate", std::int64_t{1});
  p.sp = j.value("sp", std::int64_t{1});
  p.ep = j.value("ep", std::int64_t{1});
  p.micro_batch = j.value("micro_batch", std::int64_t{1});
  std::int64_t sh = j.value("dp_shard", std::int64_t{-1});
  if (sh < 0) sh = p.dp_replicate * p.sp > 0 ? world / (p.dp_replicate * p.sp) : 0;
  p.dp_shard = sh;
  p.recompute = j.value("recompute", std::string("full")) == "none" ? RecomputeMode::none
                                                                    : RecomputeMode::full;
  p.async_ulysses = j.value("async_ulysses", false);
  p.moe_overlap = j.value("moe_overlap", false);
  p.fsdp_prefetch_depth = j.value("fsdp_prefetch_depth", std::int64_t{1});
  p.moe_imbalance = j.value("moe_imbalance", 1.0);
  p.tp = j.value("tp", std::int64_t{1});
  p.pp = j.value("pp", std::int64_t{1});
  return p;
}

json groups(const std::vector<Group>& gs) {
  json a = json::array();
  for (auto& g : gs) a.push_back(g.members);
  return a;
}

}  // namespace

extern "C" {

int ref_resolve(const char* cj, const char* mj, const char* wj, const char* pj, char* buf,
                size_t cap) {
  try {
    ClusterSpec c = parse_cluster(json::parse(cj));
    ModelSpec m = parse_model(json::parse(mj));
    WorkloadSpec w = parse_workload(json::parse(wj));
    ParallelPlan p = plan_from(json::parse(pj), c.world_size());
    json r;
    json codes = json::array();
    for (auto& v : validate(p, c, m, w)) codes.push_back(v.code);
    r["violations"] = codes;
    r["flops_per_token"] = flops_per_token(m, w.seq_len);
    const auto& f = *m.foundation().arch;
    if (codes.empty()) {
      Mesh mesh = plan_mesh(p);
      r["label"] = plan_label(p);
      r["groups"] = {{"sp", groups(groups_along(mesh, {"sp"}))},
                     {"shard", groups(groups_along(mesh, {"dp_shard", "sp"}))},
                     {"replicate", groups(groups_along(mesh, {"dp_replicate"}))},
                     {"ep", groups(ep_groups(p))}};
      if (f.moe) {
        auto es = resolve_expert_sharding(p, f);
        r["expert_sharding"] = {{"experts_per_rank", es.experts_per_rank},
                                {"per_expert_fsdp_degree", es.per_expert_fsdp_degree}};
      }
      std::int64_t total = 0;
      for (auto& mod : m.modules) total += module_param_count(mod);
      const std::int64_t b = m.param_dtype_bytes;
      const std::int64_t T = p.micro_batch * w.seq_len / p.sp;
      r["volumes"] = {{"ulysses_per_layer", ulysses_attention_volume(p, f, w, b)},
                      {"fsdp_step", fsdp_step_volume(p, total, b)},
                      {"hsdp", hsdp_allreduce_volume(p, total, b)},
                      {"ep_dispatch_per_moe_layer", ep_dispatch_volume(p, f, T, b)}};
      json layers = json::array();
      for (std::int64_t l = 0; l < f.layers; ++l) {
        auto s = layer_shape(f, l);
        layers.push_back({{"qkv", s.qkv_params}, {"out", s.out_params}, {"mlp", s.mlp_params},
                          {"moe", s.is_moe}, {"router", s.router_params},
                          {"experts_total", s.expert_params_total},
                          {"experts_active", s.expert_params_active},
                          {"gathered", s.gathered(p.ep)}});
      }
      r["layers"] = layers;
      r["head_params"] = head_param_count(f);
      json mods = json::array();
      for (auto& mp : resolve_module_plans(p, m))
        mods.push_back({{"module_name", mp.module_name}, {"fsdp", mp.fsdp},
                        {"participates_in_sp", mp.participates_in_sp},
                        {"expert_placement", mp.expert_placement}});
      r["module_plans"] = mods;
    }
    return out(r.dump(), buf, cap);
  } catch (const std::exception& e) {
    return out(std::string("{\"error\": ") + json(e.what()).dump() + "}", buf, cap) ? 9 : 2;
  }
}

// The reference's own CPU path for one step: build_step_graph + simulate +
// report (step_graph.cpp:441-448, simulator.cpp:14-131).  Returns the
// StepReport keys plus graph statistics and the wall time of the call.
int ref_simulate(const char* cj, const char* mj, const char* wj, const char* pj, char* buf,
                 size_t cap) {
  try {
    ClusterSpec c = parse_cluster(json::parse(cj));
    ModelSpec m = parse_model(json::parse(mj));
    WorkloadSpec w = parse_workload(json::parse(wj));
    ParallelPlan p = plan_from(json::parse(pj), c.world_size());
    StepGraph g = build_step_graph(p, m, c, w);
    SimOptions so;
    so.compute_efficiency = json::parse(pj).value("compute_efficiency", so.compute_efficiency);
    Timeline tl = simulate(g, p, c, so);
    StepReport rep = report(tl, g, p, m, c, w);
    json r{{"step_time_s", rep.step_time},
           {"throughput_tokens_per_s_per_gpu", rep.throughput},
           {"mfu", rep.mfu},
           {"exposed_comm_fraction", rep.exposed_comm},
           {"nodes", g.nodes.size()},
           {"collectives", g.collective_count()},
           {"all_to_all", g.collective_count(CollectiveKind::all_to_all)},
           {"all_gather", g.collective_count(CollectiveKind::all_gather)},
           {"reduce_scatter", g.collective_count(CollectiveKind::reduce_scatter)},
           {"all_reduce", g.collective_count(CollectiveKind::all_reduce)}};
    json names = json::array();
    json nodes = json::array();
    for (auto& n : g.nodes) {
      names.push_back(n.name);
      nodes.push_back({{"name", n.name},
                       {"kind", n.kind == NodeKind::compute ? "compute" : "collective"},
                       {"flops", n.flops},
                       {"bytes", n.bytes}});
    }
    r["node_names"] = names;
    r["nodes"] = nodes;
    return out(r.dump(), buf, cap);
  } catch (const std::exception& e) {
    return out(std::string("{\"error\": ") + json(e.what()).dump() + "}", buf, cap) ? 9 : 2;
  }
}

// The reference's packer (packing.cpp:10-50): policy 0 FFD, 1 arrival.
int ref_pack(const long long* lengths, long long n, long long target, int policy, char* buf,
             size_t cap) {
  try {
    std::vector<Sample> v;
    for (long long i = 0; i < n; ++i) v.push_back(Sample{i, lengths[i]});
    auto rows = pack(v, target, policy == 1 ? PackPolicy::first_fit_arrival
                                            : PackPolicy::first_fit_decreasing);
    json rj = json::array();
    for (auto& r : rows) {
      json e = json::array();
      for (auto& x : r.entries) e.push_back({x.id, x.offset, x.length});
      rj.push_back({{"capacity", r.capacity}, {"entries", e}, {"boundaries", r.boundaries}});
    }
    return out(json{{"rows", rj}, {"padding_ratio", padding_ratio(rows)}}.dump(), buf, cap);
  } catch (const PackError& e) {
    return out(std::string("{\"error\": ") + json(e.what()).dump() + ", \"sample\": " +
                   std::to_string(e.sample_id) + "}", buf, cap) ? 9 : 2;
  } catch (const std::exception& e) {
    return out(std::string("{\"error\": ") + json(e.what()).dump() + "}", buf, cap) ? 9 : 2;
  }
}

// The reference's reshard copy plan (reshard.cpp:20-56) for ceil-chunk layouts.
int ref_reshard_plan(long long numel, long long src_parts, long long dst_parts, char* buf,
                     size_t cap) {
  try {
    ReshardPlan p = make_plan(ShardLayout{"p", numel, src_parts}, ShardLayout{"p", numel, dst_parts});
    json ops = json::array();
    for (auto& o : p.ops) ops.push_back({o.src_rank, o.src_offset, o.dst_rank, o.dst_offset, o.len});
    json r{{"numel", p.numel}, {"ops", ops}, {"violations", verify(p, numel)}};
    return out(r.dump(), buf, cap);
  } catch (const std::exception& e) {
    return out(std::string("{\"error\": ") + json(e.what()).dump() + "}", buf, cap) ? 9 : 2;
  }
}

// the reference's report() (simulator.cpp:108-130) on a one-device timeline of
// n intervals (chan 0 = compute, 1 = comm): exposed comm in seconds
int ref_exposed_comm(const double* start, const double* end, const int* chan, long long n,
                     double makespan, double* exposed_s) {
  StepGraph g;
  Timeline tl;
  tl.world = 1;
  tl.makespan = makespan;
  for (long long i = 0; i < n; ++i) {
    OpNode nd;
    nd.id = i;
    nd.kind = chan[i] ? NodeKind::collective : NodeKind::compute;
    nd.name = "n" + std::to_string(i);
    nd.phase = "p";
    g.nodes.push_back(nd);
    tl.events.push_back(TimelineEvent{0, chan[i], start[i], end[i], i});
    tl.node_start.push_back(start[i]);
    tl.node_end.push_back(end[i]);
  }
  ParallelPlan p;
  ModelSpec m;
  ClusterSpec c;
  c.gpu.peak_flops = 1.0;
  WorkloadSpec w;
  const StepReport r = report(tl, g, p, m, c, w);
  *exposed_s = r.exposed_comm * makespan;
  return 0;
}

}  // extern "C"
