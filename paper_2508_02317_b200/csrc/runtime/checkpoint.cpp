// FSDP flat-shard checkpoints.
//
// Every unit (head, one per layer, one expert unit per MoE layer and EP
// position) is saved as the shards the executor already holds: rank `idx` of
// a unit with `parts` shards owns elements chunk_interval(numel, chunk, idx) of
// the logical flat parameter, chunk = layout_chunk(numel, parts, 64) (the
// 64*P-padded flat buffers, plan.hpp).  A shard file holds that interval of
// the fp32 master weights, then exp_avg, then exp_avg_sq.  Because the layout
// is "chunk c of the logical numel", the reference's interval-intersection
// copy plan (reshard.cpp:20-56, restated as opx::reshard_plan) moves a
// checkpoint between world sizes; paper_2508_02317_b200/checkpoint.py applies
// it.  bf16 parameters are not stored: they are the bf16 rounding of master.
//
//   <dir>/manifest.json               step, align, units[{name, numel, parts, chunk}]
//   <dir>/<unit>/shard<idx>.bin       3 x (end-begin) fp32
//
// Only the first HSDP replica writes (replicas hold identical shards); global
// rank 0 writes the manifest.  The caller synchronises ranks around save/load.
#include <filesystem>
#include <fstream>

#include "common.h"
#include "json.hpp"
#include "step.h"

namespace opx {

#define TRY(x)                     \
  do {                             \
    int rc_ = (x);                 \
    if (rc_ != OPX_OK) return rc_; \
  } while (0)
#define CU(x) TRY(check((x), #x))

namespace {
constexpr int64_t kAlign = 64;

std::string expert_name(int l, int e, int ep) {
  return "layer" + std::to_string(l) + ".experts.ep" + std::to_string(e) + "of" + std::to_string(ep);
}
}  // namespace

std::vector<Step::CkptUnit> Step::ckpt_units() {
  std::vector<CkptUnit> v;
  for (Unit& u : units_) v.push_back({u.name, &u});
  for (size_t l = 0; l < expert_units_.size(); ++l)
    if (!expert_units_[l].params.empty())
      v.push_back({expert_name(int(l), ep_i_, ep_), &expert_units_[l]});
  return v;
}

int Step::save(const std::string& dir) {
  namespace fs = std::filesystem;
  CU(cudaStreamSynchronize(cs_));
  CU(cudaStreamSynchronize(os_));
  try {
    fs::create_directories(dir);
    if (rank_ == 0) {
      nlohmann::json m;
      m["format"] = "opx-fsdp-shards-1";
      m["step"] = step_count_;
      m["align"] = kAlign;
      nlohmann::json units = nlohmann::json::array();
      for (Unit& u : units_)
        units.push_back({{"name", u.name}, {"numel", u.numel}, {"parts", u.P},
                         {"chunk", u.shard}});
      for (size_t l = 0; l < expert_units_.size(); ++l) {
        const Unit& u = expert_units_[l];
        if (u.params.empty()) continue;
        for (int e = 0; e < ep_; ++e)
          units.push_back({{"name", expert_name(int(l), e, ep_)}, {"numel", u.numel},
                           {"parts", u.P}, {"chunk", u.shard}});
      }
      m["units"] = units;
      m["plan"] = {{"dp_replicate", p_.dp_replicate}, {"dp_shard", p_.dp_shard}, {"sp", p_.sp},
                   {"ep", p_.ep}};
      std::ofstream(fs::path(dir) / "manifest.json") << m.dump(1);
    }
    if (rep_i_ != 0) return OPX_OK;
    for (auto& cu : ckpt_units()) {
      Unit& u = *cu.u;
      const Interval iv = chunk_interval(u.numel, u.shard, u.idx);
      const int64_t n = std::max<int64_t>(0, iv.end - iv.begin);
      std::vector<float> host(size_t(3 * n));
      if (n > 0) {
        CU(cudaMemcpy(host.data(), u.master, size_t(n) * 4, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(host.data() + n, u.m, size_t(n) * 4, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(host.data() + 2 * n, u.v, size_t(n) * 4, cudaMemcpyDeviceToHost));
      }
      const fs::path d = fs::path(dir) / cu.name;
      fs::create_directories(d);
      std::ofstream f(d / ("shard" + std::to_string(u.idx) + ".bin"), std::ios::binary);
      f.write(reinterpret_cast<const char*>(host.data()), std::streamsize(host.size() * 4));
      if (!f) throw std::runtime_error("write failed: " + (d / "shard").string());
    }
  } catch (const std::exception& e) {
    set_error(std::string("checkpoint save: ") + e.what());
    return OPX_ERR_ARG;
  }
  return OPX_OK;
}

int Step::load(const std::string& dir) {
  namespace fs = std::filesystem;
  CU(cudaStreamSynchronize(cs_));
  CU(cudaStreamSynchronize(os_));
  try {
    nlohmann::json m;
    {
      std::ifstream f(fs::path(dir) / "manifest.json");
      if (!f) throw std::runtime_error("no manifest.json in " + dir);
      f >> m;
    }
    std::map<std::string, nlohmann::json> by_name;
    for (auto& u : m.at("units")) by_name[u.at("name").get<std::string>()] = u;
    for (auto& cu : ckpt_units()) {
      Unit& u = *cu.u;
      auto it = by_name.find(cu.name);
      if (it == by_name.end()) throw std::runtime_error("unit " + cu.name + " not in checkpoint");
      const auto& j = it->second;
      if (j.at("numel").get<int64_t>() != u.numel)
        throw std::runtime_error("unit " + cu.name + ": numel differs from the model");
      if (j.at("parts").get<int64_t>() != u.P || j.at("chunk").get<int64_t>() != u.shard)
        throw std::runtime_error("unit " + cu.name + " saved with " +
                                 std::to_string(j.at("parts").get<int64_t>()) +
                                 " shards, this plan has " + std::to_string(u.P) +
                                 ": reshard the checkpoint first (checkpoint.py)");
      const Interval iv = chunk_interval(u.numel, u.shard, u.idx);
      const int64_t n = std::max<int64_t>(0, iv.end - iv.begin);
      std::vector<float> host(size_t(3 * n));
      std::ifstream f(fs::path(dir) / cu.name / ("shard" + std::to_string(u.idx) + ".bin"),
                      std::ios::binary);
      f.read(reinterpret_cast<char*>(host.data()), std::streamsize(host.size() * 4));
      if (!f || f.gcount() != std::streamsize(host.size() * 4))
        throw std::runtime_error("short shard file for " + cu.name);
      // padding past the logical numel stays zero
      CU(cudaMemset(u.master, 0, size_t(u.shard) * 4));
      CU(cudaMemset(u.m, 0, size_t(u.shard) * 4));
      CU(cudaMemset(u.v, 0, size_t(u.shard) * 4));
      if (n > 0) {
        CU(cudaMemcpy(u.master, host.data(), size_t(n) * 4, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(u.m, host.data() + n, size_t(n) * 4, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(u.v, host.data() + 2 * n, size_t(n) * 4, cudaMemcpyHostToDevice));
      }
      CU(k_cast_f32_bf16(u.master, u.pshard, u.shard, cs_));
    }
    step_count_ = m.at("step").get<int>();
    CU(cudaStreamSynchronize(cs_));
  } catch (const std::exception& e) {
    set_error(std::string("checkpoint load: ") + e.what());
    return OPX_ERR_ARG;
  }
  return OPX_OK;
}

}  // namespace opx
