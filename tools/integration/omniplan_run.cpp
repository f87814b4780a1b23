// `omniplan run`: the reference's `simulate` flow (cli.cpp:239-289
// cmd_simulate) with the simulation replaced by execution through opx's C ABI
// -- INTEGRATION.md section 1 as a real translation unit.  It is compiled
// against the reference's own headers (/root/reference/proj/include) and links
// the reference library built from its sources by oracle/Makefile
// (oracle/_ref/libomniplan_ref.so) next to libopx.so, so both sides of the
// boundary meet in one binary:
//   * configs are parsed by the reference's parse_* (config_io.cpp:52-151);
//   * the plan is validated by the reference's validate (plan.cpp:19-83) AND by
//     opx_plan_validate -- the codes must agree;
//   * the reference simulates the step (build_step_graph -> simulate -> report);
//   * unless --plan-only, opx executes the same plan on GPU 0 (single rank) and
//     the measured numbers are serialised by the reference's own
//     to_json(StepReport) (report.cpp:117-128).
// Test infrastructure: built and run by tests/test_integration_cpp.py.
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "omniplan/config_io.hpp"
#include "omniplan/plan.hpp"
#include "omniplan/report.hpp"
#include "omniplan/simulator.hpp"
#include "omniplan/step_graph.hpp"
#include "opx.h"

using namespace omniplan;

namespace {

std::string slurp(const std::string& p) {
  std::ifstream f(p);
  std::stringstream ss;
  ss << f.rdbuf();
  return ss.str();
}

// cli.cpp:46-65 plan_from_flags (cli.cpp is not part of the linked library)
ParallelPlan plan_from_args(int argc, char** argv, const ClusterSpec& c, const WorkloadSpec& w) {
  ParallelPlan p;
  p.micro_batch = w.micro_batch;
  for (int i = 4; i < argc; ++i) {
    const std::string a = argv[i];
    auto num = [&](std::int64_t& v) { v = std::stoll(argv[++i]); };
    if (a == "--sp") num(p.sp);
    else if (a == "--ep") num(p.ep);
    else if (a == "--dp-replicate") num(p.dp_replicate);
    else if (a == "--micro-batch") num(p.micro_batch);
    else if (a == "--recompute") p.recompute = std::string(argv[++i]) == "none" ? RecomputeMode::none : RecomputeMode::full;
    else if (a == "--async-ulysses") p.async_ulysses = true;
    else if (a == "--moe-overlap") p.moe_overlap = true;
  }
  if (p.dp_replicate * p.sp > 0 && c.world_size() % (p.dp_replicate * p.sp) == 0)
    p.dp_shard = c.world_size() / (p.dp_replicate * p.sp);
  return p;
}

bool has(int argc, char** argv, const char* flag) {
  for (int i = 4; i < argc; ++i)
    if (!std::strcmp(argv[i], flag)) return true;
  return false;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s cluster.json model.json workload.json [--sp N] [--ep N] "
                         "[--dp-replicate N] [--recompute full|none] [--async-ulysses] "
                         "[--moe-overlap] [--plan-only] [--steps K]\n", argv[0]);
    return 2;
  }
  const std::string cj = slurp(argv[1]), mj = slurp(argv[2]), wj = slurp(argv[3]);
  ClusterSpec cluster;
  ModelSpec model;
  WorkloadSpec workload;
  try {
    cluster = parse_cluster(nlohmann::json::parse(cj));
    model = parse_model(nlohmann::json::parse(mj));
    workload = parse_workload(nlohmann::json::parse(wj));
  } catch (const std::exception& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 2;
  }
  const ParallelPlan plan = plan_from_args(argc, argv, cluster, workload);
  const std::string pj = to_json(plan).dump();

  // both validators on the same plan: identical codes, identical order
  std::vector<std::string> ref_codes;
  for (const auto& v : validate(plan, cluster, model, workload)) ref_codes.push_back(v.code);
  std::vector<char> buf(1 << 16);
  const int vrc = opx_plan_validate(cj.c_str(), mj.c_str(), wj.c_str(), pj.c_str(), buf.data(), buf.size());
  std::vector<std::string> opx_codes;
  {
    std::stringstream ss(buf.data());
    std::string line;
    while (std::getline(ss, line))
      if (!line.empty()) opx_codes.push_back(line.substr(0, line.find('\t')));
  }
  nlohmann::json out;
  out["plan"] = nlohmann::json::parse(pj);
  out["validate"] = {{"reference", ref_codes}, {"opx", opx_codes}, {"opx_rc", vrc}};
  if (ref_codes != opx_codes) {
    std::printf("%s\n", out.dump().c_str());
    std::fprintf(stderr, "validator mismatch\n");
    return 7;
  }
  if (!ref_codes.empty()) {
    std::printf("%s\n", out.dump().c_str());
    return 3;  // cli.hpp kExitPlanInvalid
  }
  const StepGraph graph = build_step_graph(plan, model, cluster, workload);
  const Timeline tl = simulate(graph, plan, cluster);
  out["simulated"] = to_json(report(tl, graph, plan, model, cluster, workload));
  if (has(argc, argv, "--plan-only") || cluster.world_size() != 1) {
    std::printf("%s\n", out.dump().c_str());
    return 0;
  }

  // ---- execute on GPU 0 through the C ABI
  int steps = 1;
  for (int i = 4; i + 1 < argc; ++i)
    if (!std::strcmp(argv[i], "--steps")) steps = std::atoi(argv[i + 1]);
  opx_step* st = nullptr;
  char nid[128] = {};
  int rc = opx_step_create(cj.c_str(), mj.c_str(), wj.c_str(), pj.c_str(), "{}", 0, 0, nid, &st);
  if (rc) {
    std::fprintf(stderr, "opx_step_create: %s\n", opx_last_error());
    return rc;
  }
  std::vector<char> blob(4096);
  size_t len = 0;
  if ((rc = opx_step_ipc_export(st, blob.data(), blob.size(), &len)) ||
      (rc = opx_step_ipc_import(st, blob.data(), len)) || (rc = opx_step_init_weights(st, 2508))) {
    std::fprintf(stderr, "setup: %s\n", opx_last_error());
    return rc;
  }
  // synthetic batch: global_batch rows of seq_len tokens, one sample per row
  const std::int64_t S = workload.seq_len, rows = workload.global_batch;
  const auto& arch = *model.foundation().arch;
  std::vector<int32_t> ids(size_t(rows * S)), labels(size_t(rows * S)), pos(size_t(rows * S)),
      cu(size_t(rows + 1));
  std::uint64_t x = 2508;
  std::int64_t n_valid = 0;
  for (std::int64_t r = 0; r < rows; ++r) {
    cu[size_t(r)] = int32_t(r * S);
    for (std::int64_t t = 0; t < S; ++t) {
      x = x * 6364136223846793005ull + 1442695040888963407ull;
      ids[size_t(r * S + t)] = int32_t((x >> 33) % std::uint64_t(arch.vocab));
      pos[size_t(r * S + t)] = int32_t(t);
    }
    for (std::int64_t t = 0; t < S; ++t) {
      const bool last = t + 1 == S;
      labels[size_t(r * S + t)] = last ? -100 : ids[size_t(r * S + t + 1)];
      n_valid += !last;
    }
  }
  cu[size_t(rows)] = int32_t(rows * S);
  opx_step_report rep{};
  for (int s = 0; s < steps && !rc; ++s) {
    rc = opx_step_load_batch(st, ids.data(), labels.data(), pos.data(), cu.data(), int(rows + 1), n_valid);
    if (!rc) rc = opx_step_run(st, &rep);
  }
  if (rc) {
    std::fprintf(stderr, "run: %s\n", opx_last_error());
    return rc;
  }
  // the measured report in the reference's own StepReport / to_json
  StepReport r;
  r.step_time = rep.step_time_s;
  r.throughput = rep.throughput;
  r.mfu = rep.mfu;
  r.exposed_comm = rep.exposed_comm;
  r.model_flops_per_token = rep.model_flops_per_token;
  std::vector<char> js(1 << 20);
  if (!opx_step_report_json(st, js.data(), js.size(), &len)) {
    const auto j = nlohmann::json::parse(js.data());
    for (auto it = j["phase_breakdown"].begin(); it != j["phase_breakdown"].end(); ++it)
      r.phase_breakdown[it.key()] = PhaseCost{it.value()["compute_s"].get<double>(),
                                              it.value()["comm_s"].get<double>()};
  }
  out["measured"] = to_json(r);
  out["loss"] = rep.loss;
  opx_step_destroy(st);
  std::printf("%s\n", out.dump().c_str());
  return 0;
}
