// C-ABI: error plumbing, plan-layer entry points and kernel-level wrappers.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>

#include "../host/packing.hpp"
#include "../host/plan.hpp"
#include "common.h"
#include "json.hpp"
#include "kernels_api.h"
#include "opx.h"

namespace opx {
thread_local std::string g_last_error;
int64_t g_kernel_launches = 0;
void set_error(const std::string& s) { g_last_error = s; }

int cuda_fail(cudaError_t e, const char* what) {
  set_error(std::string(what) + ": " + cudaGetErrorString(e));
  return OPX_ERR_CUDA;
}

uint64_t fnv1a64(const char* s) {
  uint64_t h = 0xcbf29ce484222325ull;
  for (; *s; ++s) {
    h ^= uint8_t(*s);
    h *= 0x100000001b3ull;
  }
  return h;
}

// simulator.cpp:71-104: comm intervals sorted by start, each walked against
// the compute intervals (sorted by start) that overlap it; a compute interval
// nested inside one already passed leaves the cursor where it is
double exposed_comm_seconds(std::vector<std::pair<double, double>>& compute,
                            std::vector<std::pair<double, double>>& comm) {
  std::sort(compute.begin(), compute.end());
  std::sort(comm.begin(), comm.end());
  double exposed = 0;
  size_t ci = 0;
  for (const auto& [start, end] : comm) {
    double cur = start;
    while (ci < compute.size() && compute[ci].second <= cur) ++ci;
    for (size_t j = ci; cur < end; ++j) {
      if (j >= compute.size() || compute[j].first >= end) {
        exposed += end - cur;
        break;
      }
      if (compute[j].first > cur) exposed += compute[j].first - cur;
      cur = std::max(cur, compute[j].second);
    }
  }
  return exposed;
}

uint64_t param_key(const std::string& name, uint64_t seed) {
  return fnv1a64(name.c_str()) ^ (seed * 0x9E3779B97F4A7C15ull);
}

namespace {

int copy_out(const std::string& s, char* out, size_t cap) {
  if (!out || cap == 0) return OPX_OK;
  const size_t n = s.size() < cap - 1 ? s.size() : cap - 1;
  std::memcpy(out, s.data(), n);
  out[n] = 0;
  if (s.size() >= cap) {
    set_error("output buffer too small: need " + std::to_string(s.size() + 1));
    return OPX_ERR_ARG;
  }
  return OPX_OK;
}

struct Loaded {
  Cluster c;
  Model m;
  Workload w;
  Plan p;
};

// Parses the four JSON documents; derives dp_shard when absent (cli.cpp:46-65).
int load_all(const char* cj, const char* mj, const char* wj, const char* pj, Loaded& L) {
  try {
    L.c = parse_cluster_json(cj ? cj : "");
    L.m = parse_model_json(mj ? mj : "");
    L.w = parse_workload_json(wj ? wj : "");
    L.p = parse_plan_json(pj ? pj : "{}");
    // cross_validate (config_io.cpp:179-193)
    for (auto& [name, f] : L.w.mix) {
      (void)f;
      if (name == "text") continue;
      bool found = false;
      for (auto& mod : L.m.modules) found = found || mod.name == name;
      if (!found) throw ConfigError("workload: modality_mix entry '" + name + "' names no model module");
    }
    if (L.p.dp_shard < 0) {
      const i64 denom = L.p.dp_replicate * L.p.sp;
      L.p.dp_shard = denom > 0 && L.c.world() % denom == 0 ? L.c.world() / denom : 0;
    }
  } catch (const ConfigError& e) {
    set_error(e.what());
    return OPX_ERR_CONFIG;
  } catch (const std::exception& e) {
    set_error(std::string("config: ") + e.what());
    return OPX_ERR_CONFIG;
  }
  return OPX_OK;
}

}  // namespace
}  // namespace opx

using namespace opx;
using nlohmann::json;

extern "C" {

const char* opx_last_error(void) { return g_last_error.c_str(); }
const char* opx_version(void) { return "opx 0.1 (sm_100a)"; }

int opx_plan_validate(const char* cj, const char* mj, const char* wj, const char* pj,
                      char* out_codes, size_t cap) {
  Loaded L;
  if (int rc = load_all(cj, mj, wj, pj, L)) return rc;
  auto v = validate_plan(L.p, L.c, L.m, L.w);
  std::string s;
  for (auto& x : v) s += x.code + "\t" + x.message + "\n";
  if (int rc = copy_out(s, out_codes, cap)) return rc;
  if (!v.empty()) {
    set_error("plan invalid: " + v.front().code);
    return OPX_ERR_PLAN;
  }
  return OPX_OK;
}

int opx_plan_resolve(const char* cj, const char* mj, const char* wj, const char* pj,
                     char* out_json, size_t cap) {
  Loaded L;
  if (int rc = load_all(cj, mj, wj, pj, L)) return rc;
  auto v = validate_plan(L.p, L.c, L.m, L.w);
  if (!v.empty()) {
    std::string s;
    for (auto& x : v) s += x.code + "\t" + x.message + "\n";
    copy_out(s, out_json, cap);
    set_error("plan invalid: " + v.front().code);
    return OPX_ERR_PLAN;
  }
  try {
    const Plan& p = L.p;
    const Module* f = L.m.foundation();
    const Arch& a = *f->arch;
    Mesh mesh = plan_mesh(p);
    auto grp = [](const std::vector<Group>& gs) {
      json arr = json::array();
      for (auto& g : gs) arr.push_back(g.members);
      return arr;
    };
    json j;
    j["label"] = plan_label(p);
    j["plan"] = json::parse(plan_to_json(p));
    j["world"] = p.world();
    json dims = json::array();
    for (auto& d : mesh.dims) dims.push_back({{"name", d.name}, {"size", d.size}});
    j["mesh"] = dims;
    j["groups"] = {{"sp", grp(groups_along(mesh, {"sp"}))},
                   {"shard", grp(groups_along(mesh, {"dp_shard", "sp"}))},
                   {"replicate", grp(groups_along(mesh, {"dp_replicate"}))},
                   {"ep", grp(ep_groups(p))}};
    if (a.moe) {
      auto es = expert_sharding(p, a);
      j["expert_sharding"] = {{"experts_per_rank", es.experts_per_rank},
                              {"per_expert_fsdp_degree", es.per_expert_fsdp_degree}};
    }
    json mods = json::array();
    for (auto& mod : L.m.modules)
      mods.push_back({{"module_name", mod.name},
                      {"fsdp", true},
                      {"participates_in_sp", mod.kind == ModuleKind::foundation},
                      {"expert_placement", bool(mod.arch && mod.arch->moe)},
                      {"params", module_params(mod, false)},
                      {"active_params", module_params(mod, true)}});
    j["module_plans"] = mods;
    json layers = json::array();
    for (i64 l = 0; l < a.layers; ++l) {
      auto lp = layer_params(a, l);
      layers.push_back({{"qkv", lp.qkv},
                        {"out", lp.out},
                        {"mlp", lp.mlp},
                        {"moe", lp.moe},
                        {"router", lp.router},
                        {"experts_total", lp.experts_total},
                        {"experts_active", lp.experts_active},
                        {"gathered", lp.gathered(p.ep)}});
    }
    j["layers"] = layers;
    j["head_params"] = head_params(a);
    j["flops_per_token"] = flops_per_token_ref(L.m, L.w.seq_len);
    const i64 b = L.m.dtype_bytes;
    const i64 T = p.micro_batch * L.w.seq_len / p.sp;
    i64 total = 0;
    for (auto& mod : L.m.modules) total += module_params(mod, false);
    j["volumes"] = {{"ulysses_per_layer", vol_ulysses(p, a, L.w, b)},
                    {"fsdp_step", vol_fsdp_step(p, total, b)},
                    {"hsdp", vol_hsdp(p, total, b)},
                    {"ep_dispatch_per_moe_layer", vol_ep_dispatch(p, a, T, b)}};
    j["local_tokens"] = T;
    return copy_out(j.dump(), out_json, cap);
  } catch (const std::exception& e) {
    set_error(std::string("resolve: ") + e.what());
    return OPX_ERR_CONFIG;
  }
}

int opx_gemm(int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B,
             int64_t ldb, int b_mn, int epi, void* D, int64_t ldd, const float* R, int64_t ldr,
             void* D2, int64_t ldd2, float scale, void* stream) {
  GemmDesc g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.A = static_cast<const __nv_bfloat16*>(A);
  g.lda = lda;
  g.a_mn = a_mn;
  g.B = static_cast<const __nv_bfloat16*>(B);
  g.ldb = ldb;
  g.b_mn = b_mn;
  g.epi = epi;
  g.D = D;
  g.ldd = ldd;
  g.R = R;
  g.ldr = ldr;
  if (epi == GEMM_EPI_SWIGLU_BWD) {  // D2/ldd2 carry the forward gate|up (an input)
    g.G2 = static_cast<const __nv_bfloat16*>(D2);
    g.ldg2 = ldd2;
  } else {
    g.D2 = static_cast<__nv_bfloat16*>(D2);
    g.ldd2 = ldd2;
  }
  g.scale = scale;
  cudaError_t e = gemm_run(g, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? OPX_OK : cuda_fail(e, "opx_gemm");
}

int opx_gemm_grouped(int M, int N, int K, const void* A, int64_t lda, int a_mn, const void* B,
                     int64_t ldb, int b_mn, int epi, void* D, int64_t ldd, void* D2,
                     int64_t ldd2, int groups, int grouped_k, const int* g_start,
                     const int* g_rows, int64_t rows_total, int64_t d_group_stride,
                     void* stream) {
  GemmDesc g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.A = static_cast<const __nv_bfloat16*>(A);
  g.lda = lda;
  g.a_mn = a_mn;
  g.B = static_cast<const __nv_bfloat16*>(B);
  g.ldb = ldb;
  g.b_mn = b_mn;
  g.epi = epi;
  g.D = D;
  g.ldd = ldd;
  g.D2 = static_cast<__nv_bfloat16*>(D2);
  g.ldd2 = ldd2;
  g.groups = groups;
  g.grouped_k = grouped_k;
  g.g_start = g_start;
  g.g_rows = g_rows;
  g.rows_total = rows_total;
  g.d_group_stride = d_group_stride;
  cudaError_t e = gemm_run(g, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? OPX_OK : cuda_fail(e, "opx_gemm_grouped");
}

#define OPX_CALL(expr, what)                        \
  do {                                              \
    cudaError_t e_ = (expr);                        \
    return e_ == cudaSuccess ? OPX_OK : cuda_fail(e_, what); \
  } while (0)

int opx_rmsnorm_fwd(const float* x, const void* w, void* y, float* rstd, int T, int H, float eps,
                    void* stream) {
  OPX_CALL(k_rmsnorm_fwd(x, static_cast<const __nv_bfloat16*>(w), static_cast<__nv_bfloat16*>(y),
                         rstd, T, H, eps, static_cast<cudaStream_t>(stream)),
           "opx_rmsnorm_fwd");
}
int opx_rmsnorm_bwd(const float* dy, const float* x, const void* w, const float* rstd,
                    const float* dres, float* dx, float* dw_part, float* dw, int T, int H,
                    void* stream) {
  OPX_CALL(k_rmsnorm_bwd(dy, x, static_cast<const __nv_bfloat16*>(w), rstd, dres, dx, dw_part, dw,
                         0, T, H, static_cast<cudaStream_t>(stream)),
           "opx_rmsnorm_bwd");
}
int opx_rmsnorm_bwd_parts(int T) { return k_rmsnorm_bwd_parts(T); }
int opx_ce_fwd_bwd(void* logits, int64_t ldl, const int32_t* labels, float* loss, int T, int V,
                   float inv_n, void* stream) {
  OPX_CALL(k_ce_fwd_bwd(static_cast<__nv_bfloat16*>(logits), ldl, labels, loss, T, V, inv_n,
                        static_cast<cudaStream_t>(stream)),
           "opx_ce_fwd_bwd");
}
int opx_swiglu_bwd(const void* dact, const void* gu, void* dgu, int64_t T, int F, void* stream) {
  OPX_CALL(k_swiglu_bwd(static_cast<const __nv_bfloat16*>(dact),
                        static_cast<const __nv_bfloat16*>(gu), static_cast<__nv_bfloat16*>(dgu), T,
                        F, static_cast<cudaStream_t>(stream)),
           "opx_swiglu_bwd");
}
int opx_adamw(float* p, float* m, float* v, const float* g, void* pb, int64_t n, float lr,
              float b1, float b2, float eps, float wd, int step, void* stream) {
  OPX_CALL(k_adamw(p, m, v, g, 0, static_cast<__nv_bfloat16*>(pb), n, lr, b1, b2, eps, wd, step,
                   static_cast<cudaStream_t>(stream)),
           "opx_adamw");
}
int opx_embed_fwd(const int32_t* ids, const void* E, float* x, int T, int H, void* stream) {
  OPX_CALL(k_embed_fwd(ids, static_cast<const __nv_bfloat16*>(E), x, T, H,
                       static_cast<cudaStream_t>(stream)),
           "opx_embed_fwd");
}
int opx_embed_bwd(const int32_t* ids, const float* dx, float* dE, int T, int H, void* stream) {
  OPX_CALL(k_embed_bwd(ids, dx, dE, T, H, static_cast<cudaStream_t>(stream)), "opx_embed_bwd");
}
int opx_init_param(float* f32, void* b16, int64_t n, int64_t phys0, uint64_t key_a,
                   uint64_t key_b, double c, float constant, int interleave,
                   int64_t rows_per_slab, int64_t cols, void* stream) {
  OPX_CALL(k_init_param(f32, static_cast<__nv_bfloat16*>(b16), n, phys0, key_a, key_b, c,
                        constant, interleave, rows_per_slab, cols,
                        static_cast<cudaStream_t>(stream)),
           "opx_init_param");
}
uint64_t opx_param_key(const char* name, uint64_t seed) { return param_key(name, seed); }

int opx_attn_fwd_tc(const void* q, const void* k, const void* v, void* o, float* lse,
                    int64_t ldq, int64_t ldk, int64_t ldv, int64_t ldo, const int32_t* seq_start,
                    const int32_t* seq_end, int N, int hq, int hk, float scale, void* stream) {
  AttnArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.k = static_cast<const __nv_bfloat16*>(k);
  a.v = static_cast<const __nv_bfloat16*>(v);
  a.o = static_cast<__nv_bfloat16*>(o);
  a.lse = lse;
  a.ldq = ldq;
  a.ldk = ldk;
  a.ldv = ldv;
  a.ldo = ldo;
  a.seq_start = seq_start;
  a.seq_end = seq_end;
  a.N = N;
  a.hq = hq;
  a.hk = hk;
  a.scale = scale;
  OPX_CALL(k_attn_fwd_tc(a, static_cast<cudaStream_t>(stream)), "opx_attn_fwd_tc");
}

int opx_attn_fwd_bidir_tc(const void* q, const void* k, const void* v, void* o, float* lse,
                          int64_t ldq, int64_t ldk, int64_t ldv, int64_t ldo,
                          const int32_t* seq_start, const int32_t* seq_end, int N, int hq, int hk,
                          float scale, void* stream) {
  AttnArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.k = static_cast<const __nv_bfloat16*>(k);
  a.v = static_cast<const __nv_bfloat16*>(v);
  a.o = static_cast<__nv_bfloat16*>(o);
  a.lse = lse;
  a.ldq = ldq;
  a.ldk = ldk;
  a.ldv = ldv;
  a.ldo = ldo;
  a.seq_start = seq_start;
  a.seq_end = seq_end;
  a.N = N;
  a.hq = hq;
  a.hk = hk;
  a.scale = scale;
  a.causal = 0;
  OPX_CALL(k_attn_fwd_tc(a, static_cast<cudaStream_t>(stream)), "opx_attn_fwd_bidir_tc");
}

int opx_attn_bwd_tc(const void* q, const void* k, const void* v, const void* o, const float* lse,
                 const void* dout, float* dq_acc, void* dk, void* dv, float* delta,
                 int64_t ld_q, int64_t ld_kv, const int32_t* seq_start, const int32_t* seq_end,
                 int N, int hq, int hk, float scale, void* stream) {
  AttnArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.k = static_cast<const __nv_bfloat16*>(k);
  a.v = static_cast<const __nv_bfloat16*>(v);
  a.o = static_cast<__nv_bfloat16*>(const_cast<void*>(o));
  a.lse = const_cast<float*>(lse);
  a.ldq = ld_q;
  a.ldk = ld_kv;
  a.ldv = ld_kv;
  a.ldo = ld_q;
  a.seq_start = seq_start;
  a.seq_end = seq_end;
  a.N = N;
  a.hq = hq;
  a.hk = hk;
  a.scale = scale;
  a.dout = static_cast<const __nv_bfloat16*>(dout);
  a.lddo = ld_q;
  a.dq_acc = dq_acc;
  a.dk = static_cast<__nv_bfloat16*>(dk);
  a.dv = static_cast<__nv_bfloat16*>(dv);
  a.lddk = ld_kv;
  a.lddv = ld_kv;
  a.delta = delta;
  OPX_CALL(k_attn_bwd_tc(a, static_cast<cudaStream_t>(stream)), "opx_attn_bwd_tc");
}

double opx_exposed_comm_seconds(const double* compute_start, const double* compute_end,
                                int64_t n_compute, const double* comm_start,
                                const double* comm_end, int64_t n_comm) {
  std::vector<std::pair<double, double>> compute, comm;
  for (int64_t i = 0; i < n_compute; ++i) compute.push_back({compute_start[i], compute_end[i]});
  for (int64_t i = 0; i < n_comm; ++i) comm.push_back({comm_start[i], comm_end[i]});
  return opx::exposed_comm_seconds(compute, comm);
}

int opx_pack(const int64_t* ids, const int64_t* lengths, int64_t n, int64_t target, int policy,
             char* out_json, size_t cap) {
  try {
    std::vector<opx::PackSample> v(size_t(n > 0 ? n : 0));
    for (int64_t i = 0; i < n; ++i) v[size_t(i)] = {ids ? ids[i] : i, lengths[i]};
    const auto rows = opx::pack(v, target, policy == 1 ? opx::PackPolicy::first_fit_arrival
                                                       : opx::PackPolicy::first_fit_decreasing);
    nlohmann::json j;
    nlohmann::json rj = nlohmann::json::array();
    for (const auto& r : rows) {
      nlohmann::json e = nlohmann::json::array();
      for (const auto& x : r.entries) e.push_back({x.id, x.offset, x.length});
      rj.push_back({{"capacity", r.capacity}, {"entries", e}, {"boundaries", r.boundaries}});
    }
    j["rows"] = rj;
    j["padding_ratio"] = opx::padding_ratio(rows);
    const std::string s = j.dump();
    if (s.size() + 1 > cap) {
      opx::set_error("pack output buffer too small (need " + std::to_string(s.size() + 1) + ")");
      return OPX_ERR_ARG;
    }
    std::memcpy(out_json, s.c_str(), s.size() + 1);
    return OPX_OK;
  } catch (const opx::PackError& e) {
    opx::set_error(e.what());
    return OPX_ERR_CONFIG;
  } catch (const std::exception& e) {
    opx::set_error(e.what());
    return OPX_ERR_ARG;
  }
}

int opx_reshard_plan(int64_t numel, int64_t src_parts, int64_t src_align, int64_t dst_parts,
                     int64_t dst_align, char* out_json, size_t cap) {
  try {
    const int64_t sc = opx::layout_chunk(numel, src_parts, src_align);
    const int64_t dc = opx::layout_chunk(numel, dst_parts, dst_align);
    const auto ops = opx::reshard_plan(numel, src_parts, sc, dst_parts, dc);
    const auto bad = opx::reshard_verify(ops, numel);
    if (!bad.empty()) {
      opx::set_error("reshard plan invalid: " + bad[0]);
      return OPX_ERR_ARG;
    }
    std::string s = "{\"numel\":" + std::to_string(numel) + ",\"src_chunk\":" + std::to_string(sc) +
                    ",\"dst_chunk\":" + std::to_string(dc) + ",\"ops\":[";
    for (size_t i = 0; i < ops.size(); ++i) {
      const auto& o = ops[i];
      s += (i ? ",[" : "[") + std::to_string(o.src_rank) + "," + std::to_string(o.src_offset) + "," +
           std::to_string(o.dst_rank) + "," + std::to_string(o.dst_offset) + "," +
           std::to_string(o.len) + "]";
    }
    s += "]}";
    if (s.size() + 1 > cap) {
      opx::set_error("reshard plan buffer too small");
      return OPX_ERR_ARG;
    }
    std::memcpy(out_json, s.c_str(), s.size() + 1);
    return OPX_OK;
  } catch (const std::exception& e) {
    opx::set_error(e.what());
    return OPX_ERR_ARG;
  }
}

int opx_attn_bwd_tc_f32kv(const void* q, const void* k, const void* v, const void* o,
                          const float* lse, const void* dout, float* dq_acc, float* dk_acc,
                          float* dv_acc, float* delta, int64_t ld_q, int64_t ld_kv,
                          const int32_t* seq_start, const int32_t* seq_end, int N, int hq, int hk,
                          float scale, int kv_splits, void* stream) {
  AttnArgs a{};
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.k = static_cast<const __nv_bfloat16*>(k);
  a.v = static_cast<const __nv_bfloat16*>(v);
  a.o = static_cast<__nv_bfloat16*>(const_cast<void*>(o));
  a.lse = const_cast<float*>(lse);
  a.ldq = ld_q;
  a.ldk = ld_kv;
  a.ldv = ld_kv;
  a.ldo = ld_q;
  a.seq_start = seq_start;
  a.seq_end = seq_end;
  a.N = N;
  a.hq = hq;
  a.hk = hk;
  a.scale = scale;
  a.dout = static_cast<const __nv_bfloat16*>(dout);
  a.lddo = ld_q;
  a.dq_acc = dq_acc;
  a.dk_acc = dk_acc;
  a.dv_acc = dv_acc;
  a.kv_splits = kv_splits;
  a.delta = delta;
  OPX_CALL(k_attn_bwd_tc(a, static_cast<cudaStream_t>(stream)), "opx_attn_bwd_tc_f32kv");
}

int opx_rope_pack(const void* qkv, int64_t ld, void* q_full, void* k_full, void* v_full, int hq,
                  int hk, int rows, int S, const int32_t* pos, const float* inv_freq,
                  void* stream) {
  A2AArgs a{};
  a.sp = 1;
  a.rank = 0;
  a.rows = rows;
  a.seq = S;
  a.ngroups = 3;
  a.g[0] = A2AGroup{hq, 0, 1, 0, {q_full}};
  a.g[1] = A2AGroup{hk, hq * 128, 1, 0, {k_full}};
  a.g[2] = A2AGroup{hk, (hq + hk) * 128, 0, 0, {v_full}};
  a.local[0] = const_cast<void*>(qkv);
  a.local_ld = ld;
  a.pos = pos;
  a.inv_freq = inv_freq;
  OPX_CALL(k_a2a_seq2head(a, static_cast<cudaStream_t>(stream)), "opx_rope_pack");
}

int opx_ulysses_seq2head(const void* qkv, int64_t ld, void* const* q_dst, void* const* k_dst,
                         void* const* v_dst, int sp, int rank, int rows, int S, int hq, int hk,
                         int hd, const int32_t* pos, const float* inv_freq, void* stream) {
  if (sp < 1 || sp > kMaxSp || rank < 0 || rank >= sp || hq % sp || hk % sp || S % sp) {
    set_error("opx_ulysses_seq2head: bad sp/rank/head split");
    return OPX_ERR_ARG;
  }
  A2AArgs a{};
  a.sp = sp;
  a.rank = rank;
  a.rows = rows;
  a.seq = S;
  a.ngroups = 3;
  a.g[0] = A2AGroup{hq, 0, pos ? 1 : 0, 0, {}};
  a.g[1] = A2AGroup{hk, hq * hd, pos ? 1 : 0, 0, {}};
  a.g[2] = A2AGroup{hk, (hq + hk) * hd, 0, 0, {}};
  for (int j = 0; j < sp; ++j) {
    a.g[0].full[j] = q_dst[j];
    a.g[1].full[j] = k_dst[j];
    a.g[2].full[j] = v_dst[j];
  }
  a.local[0] = const_cast<void*>(qkv);
  a.local_ld = ld;
  a.pos = pos;
  a.inv_freq = inv_freq;
  a.hd = hd;
  OPX_CALL(k_a2a_seq2head(a, static_cast<cudaStream_t>(stream)), "opx_ulysses_seq2head");
}

int opx_ulysses_head2seq(const void* o_heads, void* const* dst, int64_t ld, int sp, int rank,
                         int rows, int S, int hq, int hd, void* stream) {
  if (sp < 1 || sp > kMaxSp || rank < 0 || rank >= sp || hq % sp || S % sp) {
    set_error("opx_ulysses_head2seq: bad sp/rank/head split");
    return OPX_ERR_ARG;
  }
  A2AArgs a{};
  a.sp = sp;
  a.rank = rank;
  a.rows = rows;
  a.seq = S;
  a.ngroups = 1;
  a.g[0].heads_total = hq;
  a.g[0].full[0] = const_cast<void*>(o_heads);
  for (int j = 0; j < sp; ++j) a.local[j] = dst[j];
  a.local_ld = ld;
  a.hd = hd;
  OPX_CALL(k_a2a_head2seq(a, static_cast<cudaStream_t>(stream)), "opx_ulysses_head2seq");
}

int opx_moe_route(const void* h, const void* w, int T, int H, int E, int k, float* logits,
                  int32_t* idx, float* wts, void* stream) {
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  float* part = nullptr;
  if (k_moe_router_splits(H) > 1) {
    cudaError_t e = cudaMallocAsync(&part, size_t(k_moe_router_splits(H)) * T * E * sizeof(float), s);
    if (e != cudaSuccess) return cuda_fail(e, "opx_moe_route scratch");
  }
  cudaError_t e = k_moe_router(static_cast<const __nv_bfloat16*>(h),
                               static_cast<const __nv_bfloat16*>(w), logits, T, H, E, s, part);
  if (part) cudaFreeAsync(part, s);
  if (e != cudaSuccess) return cuda_fail(e, "opx_moe_route");
  OPX_CALL(k_moe_topk(logits, T, E, k, idx, wts, s), "opx_moe_route");
}
int opx_moe_sort_chunks(int P) { return k_moe_sort_chunks(P); }
int opx_moe_sort(const int32_t* idx, int P, int E, int32_t* hist, int32_t* counts, int32_t* excl,
                 int32_t* pos, int32_t* pair_at, void* stream) {
  OPX_CALL(k_moe_sort(idx, P, E, hist, counts, excl, pos, pair_at, static_cast<cudaStream_t>(stream)),
           "opx_moe_sort");
}

}  // extern "C"
