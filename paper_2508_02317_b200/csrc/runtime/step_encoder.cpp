// Frozen omni-modal encoder inside the step.
//
// Reference: step_graph.cpp:141-166 build_encoders — per micro-batch an
// `encoder.<mod>` compute node over this rank's share of the modality tokens
// (no backward node when the module is frozen) and a `scatter.<mod>`
// all_to_all of the features into the SP group (comm.cpp:91-105); the module
// fields come from specs.hpp:66-75 (name, kind, arch, trainable,
// tokens_per_item).  The encoder math is HF transformers' Qwen2.5-VL vision
// tower (modeling_qwen2_5_vl.py:345-518: biases, 2-D RoPE, windowed and
// full-attention blocks, 2x2 patch merger), restated in oracle/encoder.py and
// pinned against the HF module there.
//
// B200 mapping: the items of a micro-batch are dealt round-robin to the SP
// ranks (item j -> rank j % sp; every rank then encodes mix_fraction x its
// share of the tokens, step_graph.cpp:147), each rank runs the ViT over its
// patches with the backbone's kernels (tcgen05 GEMMs with bias / SwiGLU
// epilogues, bidirectional tcgen05 attention on 128-padded heads through the
// seq->head relayout kernel, which also applies the 2-D RoPE from a per-patch
// (sin, cos) table).  Windows cost nothing extra: the host uploads each
// item's patches already in window order (get_window_index's permutation),
// windowed blocks see per-window [seq_start, seq_end) spans, full-attention
// blocks per-item spans, and the merger's rows are stored straight into the
// feature buffer of the SP rank that owns each placeholder position in the
// inverse order (NVLink peer stores into the CUDA-IPC arena: the
// all-to-all, the un-permutation and the masked scatter's addressing in one
// pass).  After an SP barrier every rank overwrites its placeholder
// embeddings with the received rows; the backward zeroes their gradient rows
// before the embedding scatter-add (the features are frozen).  The frozen
// weights are FSDP-sharded like every module (plan.cpp:95-107): each rank
// keeps a bf16 shard of every unit (patch embed, each block, the merger; no
// gradient or optimizer state) and the forward all-gathers unit i + 2 into a
// double-buffered slot on the comm stream while unit i computes.
#include <algorithm>
#include <cmath>
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
int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }
GemmDesc egd(int M, int N, int K, const bf16* A, int64_t lda, const bf16* B, int64_t ldb, int epi,
             void* D, int64_t ldd) {
  GemmDesc g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.A = A;
  g.lda = lda;
  g.a_mn = false;
  g.B = B;
  g.ldb = ldb;
  g.b_mn = false;
  g.epi = epi;
  g.D = D;
  g.ldd = ldd;
  return g;
}
}  // namespace

int Step::enc_setup() {
  const Module* em = nullptr;
  for (const Module& m : m_.modules)
    if (m.kind == ModuleKind::encoder && m.arch) {
      em = &m;
      break;
    }
  if (!em) return OPX_OK;
  if (em->trainable) {
    set_error("encoder '" + em->name + "': only frozen (trainable=false) encoders are executed");
    return OPX_ERR_CONFIG;
  }
  const Arch& ea = *em->arch;
  Enc& e = enc_;
  e.on = true;
  e.name = em->name;
  e.He = int(ea.hidden);
  e.L = int(ea.layers);
  e.heads = int(ea.heads);
  e.d = int(ea.head_dim);
  e.F = int(ea.ffn);
  e.pd = int(ea.vocab);  // an encoder's "vocab" is its patch width
  e.tpi = int(em->tokens_per_item);
  e.g = int(std::lround(std::sqrt(4.0 * e.tpi)));
  e.window_merge = int(ea.window_merge);
  e.rope_theta = ea.rope_theta;
  if (ea.kv_heads != ea.heads || e.d > 128 || e.d % 16 || e.He % 128 || e.F % 128 || e.pd % 8 ||
      e.tpi <= 0 || e.tpi > S_loc_ || e.g * e.g != 4 * e.tpi || e.g % 2 || e.window_merge < 1) {
    set_error("encoder requires kv_heads == heads, head_dim <= 128 (multiple of 16), hidden and ffn "
              "multiples of 128, patch width (arch.vocab) a multiple of 8, 0 < tokens_per_item <= "
              "seq/sp with 4*tokens_per_item a square of even side, window_merge >= 1");
    return OPX_ERR_CONFIG;
  }
  // full-attention blocks: the arch's list, else Qwen2.5-VL's every 8th + the last
  e.fullatt.assign(size_t(e.L), 0);
  if (ea.fullatt_blocks) {
    for (i64 b : *ea.fullatt_blocks)
      if (b >= 0 && b < e.L) e.fullatt[size_t(b)] = 1;
  } else {
    for (int i = 0; i < e.L; ++i) e.fullatt[size_t(i)] = (i + 1) % 8 == 0 || i == e.L - 1;
  }
  // window order of the merge units (get_window_index, padding windows dropped)
  {
    const int lg = e.g / 2, wm = e.window_merge;
    const int nw = (lg + wm - lg % wm) / wm;
    e.worder.clear();
    e.wlens.clear();
    for (int wh = 0; wh < nw; ++wh)
      for (int ww = 0; ww < nw; ++ww) {
        int n = 0;
        for (int i = 0; i < wm; ++i)
          for (int j = 0; j < wm; ++j) {
            const int uh = wh * wm + i, uw = ww * wm + j;
            if (uh < lg && uw < lg) {
              e.worder.push_back(uh * lg + uw);
              ++n;
            }
          }
        if (n) e.wlens.push_back(4 * n);
      }
  }
  const int64_t He = e.He, Wq = int64_t(e.heads) * e.d, F = e.F;
  // units and their params (HF names; init keys), sharded like the backbone's
  auto add = [](Unit& u, const std::string& name, int64_t n, bool ones, int interleave = 0,
                const std::string& kb = "", int64_t rows = 0, int64_t cols = 0) {
    Param q;
    q.name = q.key_a = name;
    q.key_b = kb;
    q.numel = n;
    q.shape = {n};
    q.off = u.numel;
    q.ones = ones;
    q.interleave = interleave;
    q.rows_per_slab = rows;
    q.cols = cols;
    u.numel += round_up(n, 128);
    u.params.push_back(q);
  };
  const std::string V = "visual.";
  e.units.assign(size_t(e.L) + 2, Unit{});
  add(e.units[0], V + "patch_embed.proj.weight", He * e.pd, false);
  for (int i = 0; i < e.L; ++i) {
    Unit& u = e.units[size_t(1 + i)];
    const std::string p = V + "blocks." + std::to_string(i) + ".";
    add(u, p + "norm1.weight", He, true);
    add(u, p + "attn.qkv.weight", 3 * Wq * He, false);
    add(u, p + "attn.qkv.bias", 3 * Wq, false);
    add(u, p + "attn.proj.weight", He * Wq, false);
    add(u, p + "attn.proj.bias", He, false);
    add(u, p + "norm2.weight", He, true);
    add(u, p + "mlp.gate_proj.weight", 2 * F * He, false, 1, p + "mlp.up_proj.weight", 2 * F, He);
    add(u, p + "mlp.gate_proj.bias", 2 * F, false, 1, p + "mlp.up_proj.bias", 2 * F, 1);
    add(u, p + "mlp.down_proj.weight", He * F, false);
    add(u, p + "mlp.down_proj.bias", He, false);
  }
  {
    Unit& u = e.units.back();
    add(u, V + "merger.ln_q.weight", He, true);
    add(u, V + "merger.mlp.0.weight", 16 * He * He, false);
    add(u, V + "merger.mlp.0.bias", 4 * He, false);
    add(u, V + "merger.mlp.2.weight", int64_t(H_) * 4 * He, false);
    add(u, V + "merger.mlp.2.bias", H_, false);
  }
  const int nsh = int(p_.shard_degree());
  const int my = shard_i_ * int(p_.sp) + sp_i_;
  int64_t mx = 0;
  for (Unit& u : e.units) {
    u.name = "encoder";
    u.P = nsh;
    u.idx = my;
    u.comm = shard_comm_;
    u.padded = round_up(u.numel, 64 * int64_t(nsh));
    u.shard = u.padded / nsh;
    u.pshard = alloc<bf16>(size_t(u.shard));
    if (!u.pshard) return cuda_fail(cudaErrorMemoryAllocation, "encoder weight shards");
    if (nsh == 1) u.full = u.pshard;
    mx = std::max(mx, u.padded);
  }
  if (nsh > 1) {
    for (auto& sl : e.slot)
      if (!(sl = alloc<bf16>(size_t(mx), false)))
        return cuda_fail(cudaErrorMemoryAllocation, "encoder gather slots");
    e.ev_ag.resize(e.units.size());
    e.ev_use.resize(e.units.size());
    for (auto* v : {&e.ev_ag, &e.ev_use})
      for (auto& ev : *v) CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  }
  d_fmask_ = alloc<int>(size_t(T_));
  // 2-D RoPE table of one item's patches in window order: pair (j, j + d/2)
  // turns by hpos * inv[j] (j < d/4) or wpos * inv[j - d/4] (rot_pos_emb,
  // apply_rotary_pos_emb_vision); sin/cos of the fp32 angle in double
  const int P = 4 * e.tpi, hd2 = e.d / 2, hd4 = e.d / 4;
  e.rope = alloc<float2>(size_t(P) * hd2, false);
  if (!d_fmask_ || !e.rope) return cuda_fail(cudaErrorMemoryAllocation, "encoder buffers");
  std::vector<float> inv(static_cast<size_t>(hd4));
  for (int i = 0; i < hd4; ++i)
    inv[size_t(i)] = float(1.0 / std::pow(e.rope_theta, double(2 * i) / double(hd2)));
  std::vector<float2> tab(size_t(P) * hd2);
  for (int r = 0; r < P; ++r) {
    const int patch = e.worder[size_t(r / 4)] * 4 + r % 4;  // processor-order patch of row r
    const int unit = patch / 4, sub = patch % 4;
    const int hp = (unit / (e.g / 2)) * 2 + sub / 2, wp = (unit % (e.g / 2)) * 2 + sub % 2;
    for (int j = 0; j < hd2; ++j) {
      const float ang = j < hd4 ? float(hp) * inv[size_t(j)] : float(wp) * inv[size_t(j - hd4)];
      tab[size_t(r) * hd2 + j] = make_float2(float(std::sin(double(ang))), float(std::cos(double(ang))));
    }
  }
  CU(cudaMemcpy(e.rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
  return OPX_OK;
}

int Step::enc_init_weights(uint64_t seed) {
  if (!enc_.on) return OPX_OK;
  // each rank fills its shard of every unit (same counter-based init as the
  // backbone: values depend on (name, logical index) only, oracle/encoder.py)
  const double c = 0.02 * std::sqrt(3.0) / 16777216.0;
  for (Unit& u : enc_.units) {
    const int64_t sb = int64_t(u.idx) * u.shard, se = sb + u.shard;
    CU(cudaMemsetAsync(u.pshard, 0, size_t(u.shard) * 2, cs_));
    for (const Param& q : u.params) {
      const int64_t lo = std::max(sb, q.off), hi = std::min(se, q.off + q.numel);
      if (hi <= lo) continue;
      const uint64_t ka = param_key(q.key_a, seed);
      const uint64_t kb = q.key_b.empty() ? 0 : param_key(q.key_b, seed);
      CU(k_init_param(nullptr, u.pshard + (lo - sb), hi - lo, lo - q.off, ka, kb, q.ones ? 0.0 : c,
                      1.0f, q.interleave, q.rows_per_slab, q.cols, cs_));
    }
  }
  return OPX_OK;
}

int Step::enc_alloc(int items) {
  Enc& e = enc_;
  if (items <= e.cap) return OPX_OK;
  CU(cudaStreamSynchronize(cs_));
  for (void* p : e.bufs) {
    cudaFree(p);
    allocs_.erase(std::remove(allocs_.begin(), allocs_.end(), p), allocs_.end());
  }
  e.bufs.clear();
  const size_t Np = size_t(items) * 4 * size_t(e.tpi), He = size_t(e.He);
  const size_t Wq = size_t(e.heads) * size_t(e.d);
  auto a = [&](auto*& ptr, size_t n) {
    using T = std::remove_reference_t<decltype(*ptr)>;
    ptr = alloc<T>(n);  // zeroed: the 128-padded head lanes (d < 128) must read 0
    e.bufs.push_back(ptr);
    return ptr != nullptr;
  };
  bool ok = a(e.pix, Np * size_t(e.pd)) && a(e.x, Np * He) && a(e.rstd, Np) &&
            a(e.lse, Np * size_t(e.heads)) && a(e.h, Np * He) &&
            a(e.qkv, Np * 3 * Wq) && a(e.q, Np * size_t(e.heads) * 128) &&
            a(e.k, Np * size_t(e.heads) * 128) && a(e.v, Np * size_t(e.heads) * 128) &&
            a(e.o, Np * size_t(e.heads) * 128) && a(e.o2, Np * Wq) && a(e.act, Np * size_t(e.F)) &&
            a(e.y1, Np * He) && a(e.feat, Np / 4 * size_t(H_)) && a(e.st, Np) && a(e.en, Np) &&
            a(e.wst, Np) && a(e.wen, Np) && a(e.rpos, Np) && a(e.dst_rank, Np / 4) &&
            a(e.dst_tok, Np / 4);
  if (!ok) return cuda_fail(cudaErrorMemoryAllocation, "encoder activations");
  e.cap = items;
  return OPX_OK;
}

int Step::load_images(const uint16_t* pixels, int n, const int32_t* row, const int32_t* pos) {
  if (!enc_.on) {
    set_error("the model has no encoder module with an arch");
    return OPX_ERR_CONFIG;
  }
  Enc& e = enc_;
  const int sp = int(p_.sp), tpi = e.tpi, P = 4 * tpi;
  std::vector<int32_t> mask(size_t(T_), 0);
  std::vector<int> mine;
  for (int j = 0; j < n; ++j) {
    if (row[j] < 0 || row[j] >= rows_ || pos[j] < 0 || pos[j] + tpi > S_ ||
        (j > 0 && (row[j] < row[j - 1] || (row[j] == row[j - 1] && pos[j] < pos[j - 1] + tpi)))) {
      set_error("image items must lie inside their row, sorted by (row, pos), without overlap");
      return OPX_ERR_ARG;
    }
    for (int t = 0; t < tpi; ++t) {
      const int s = pos[j] + t;
      if (s / S_loc_ == sp_i_) mask[size_t(row[j]) * S_loc_ + s % S_loc_] = 1;
    }
    if (j % sp == sp_i_) mine.push_back(j);
  }
  e.n_all = n;
  e.n_loc = int(mine.size());
  CU(cudaMemcpyAsync(d_fmask_, mask.data(), size_t(T_) * 4, cudaMemcpyHostToDevice, cs_));
  if (e.n_loc == 0) return OPX_OK;
  TRY(enc_alloc(e.n_loc));
  // patches are staged in window order (merge unit worder[m] becomes unit m);
  // merger row m of an item is the feature of its placeholder token worder[m]
  const size_t patch_elems = size_t(e.pd), item_elems = size_t(P) * patch_elems;
  std::vector<uint16_t> px(size_t(e.n_loc) * item_elems);
  const size_t NpL = size_t(e.n_loc) * P;
  std::vector<int32_t> st(NpL), en(NpL), wst(NpL), wen(NpL), rp(NpL), dr(size_t(e.n_loc) * tpi),
      dt(size_t(e.n_loc) * tpi);
  for (int k = 0; k < e.n_loc; ++k) {
    const int j = mine[size_t(k)];
    for (int m = 0; m < P / 4; ++m)
      std::memcpy(px.data() + size_t(k) * item_elems + size_t(m) * 4 * patch_elems,
                  pixels + size_t(j) * item_elems + size_t(e.worder[size_t(m)]) * 4 * patch_elems,
                  4 * patch_elems * 2);
    int w0 = 0;
    for (int len : e.wlens) {
      for (int i = 0; i < len; ++i) {
        wst[size_t(k) * P + w0 + i] = k * P + w0;
        wen[size_t(k) * P + w0 + i] = k * P + w0 + len;
      }
      w0 += len;
    }
    for (int i = 0; i < P; ++i) {
      st[size_t(k) * P + i] = k * P;
      en[size_t(k) * P + i] = (k + 1) * P;
      rp[size_t(k) * P + i] = i;
    }
    for (int m = 0; m < tpi; ++m) {
      const int s = pos[j] + e.worder[size_t(m)];
      dr[size_t(k) * tpi + m] = s / S_loc_;
      dt[size_t(k) * tpi + m] = row[j] * S_loc_ + s % S_loc_;
    }
  }
  CU(cudaMemcpyAsync(e.pix, px.data(), px.size() * 2, cudaMemcpyHostToDevice, cs_));
  CU(cudaMemcpyAsync(e.st, st.data(), st.size() * 4, cudaMemcpyHostToDevice, cs_));
  CU(cudaMemcpyAsync(e.en, en.data(), en.size() * 4, cudaMemcpyHostToDevice, cs_));
  CU(cudaMemcpyAsync(e.wst, wst.data(), wst.size() * 4, cudaMemcpyHostToDevice, cs_));
  CU(cudaMemcpyAsync(e.wen, wen.data(), wen.size() * 4, cudaMemcpyHostToDevice, cs_));
  CU(cudaMemcpyAsync(e.rpos, rp.data(), rp.size() * 4, cudaMemcpyHostToDevice, cs_));
  CU(cudaMemcpyAsync(e.dst_rank, dr.data(), dr.size() * 4, cudaMemcpyHostToDevice, cs_));
  CU(cudaMemcpyAsync(e.dst_tok, dt.data(), dt.size() * 4, cudaMemcpyHostToDevice, cs_));
  CU(cudaStreamSynchronize(cs_));
  return OPX_OK;
}

int Step::enc_forward() {
  Enc& e = enc_;
  if (!e.on) return OPX_OK;
  const bool tr = ex_.trace;
  cudaEvent_t e0 = tr ? ev() : nullptr, e1 = nullptr;
  if (tr) cudaEventRecord(e0, cs_);
  const int Np = e.n_loc * 4 * e.tpi, He = e.He, Wq = e.heads * e.d, F = e.F, nf = e.n_loc * e.tpi;
  const int64_t ldh = int64_t(e.heads) * 128;  // 128-padded head layout
  const int U = int(e.units.size());
  const bool sharded = e.units[0].P > 1;
  // FSDP: the unit gathers are collectives of the shard group, so every rank
  // runs them whether or not it encodes items this step (one unit ahead)
  auto gather = [&](int i) -> int {
    Unit& u = e.units[size_t(i)];
    u.full = e.slot[i % 2];
    if (i >= 2) CU(cudaStreamWaitEvent(ms_, e.ev_use[size_t(i - 2)], 0));
    cudaEvent_t a = tr ? ev() : nullptr;
    if (tr) cudaEventRecord(a, ms_);
    NC(ncclAllGather(u.pshard, u.full, size_t(u.shard), ncclBfloat16, u.comm, ms_));
    CU(cudaEventRecord(e.ev_ag[size_t(i)], ms_));
    if (tr) mark("fwd.ag.encoder." + e.name + ".u" + std::to_string(i) + mtag(), "encoder", 1, a,
                 e.ev_ag[size_t(i)]);
    return OPX_OK;
  };
  auto use = [&](int i) -> int {  // unit i's weights are needed on cs_ from here
    if (!sharded) return OPX_OK;
    CU(cudaStreamWaitEvent(cs_, e.ev_ag[size_t(i)], 0));
    return OPX_OK;
  };
  auto done = [&](int i) -> int {  // unit i's compute is enqueued: its slot can be refilled
    if (!sharded) return OPX_OK;
    CU(cudaEventRecord(e.ev_use[size_t(i)], cs_));
    if (i + 2 < U) TRY(gather(i + 2));
    return OPX_OK;
  };
  if (sharded) {
    CU(cudaEventRecord(e.ev_use[0], cs_));  // the slots' previous readers (last step) are done
    CU(cudaStreamWaitEvent(ms_, e.ev_use[0], 0));
    TRY(gather(0));
    if (U > 1) TRY(gather(1));
  }
  const bool run = Np > 0;
  TRY(use(0));
  if (run)
    CU(gemm_run(egd(Np, He, e.pd, e.pix, e.pd, e.wp(0, 0), e.pd, GEMM_EPI_F32, e.x, He), cs_));
  TRY(done(0));
  for (int i = 0; i < e.L; ++i) {
    const int ui = 1 + i;
    TRY(use(ui));
    if (run) {
      CU(k_rmsnorm_fwd(e.x, e.wp(ui, 0), e.h, e.rstd, Np, He, ex_.rms_eps, cs_));
      {
        GemmDesc g = egd(Np, 3 * Wq, He, e.h, He, e.wp(ui, 1), He, GEMM_EPI_BF16, e.qkv, 3 * Wq);
        g.bias = e.wp(ui, 2);
        CU(gemm_run(g, cs_));
      }
      {
        // [Np, 3, heads*d] -> [Np, heads, 128] q / k / v with the 2-D RoPE on
        // q and k (sp = 1 relayout; table row = patch row within its item)
        A2AArgs a{};
        a.sp = 1;
        a.rank = 0;
        a.rows = 1;
        a.seq = Np;
        a.ngroups = 3;
        bf16* dst[3] = {e.q, e.k, e.v};
        for (int g = 0; g < 3; ++g) {
          a.g[g].heads_total = e.heads;
          a.g[g].col0 = g * Wq;
          a.g[g].rope = g < 2;
          a.g[g].full[0] = dst[g];
        }
        a.local[0] = e.qkv;
        a.local_ld = 3 * Wq;
        a.hd = e.d;
        a.pos = e.rpos;
        a.rope_tab = e.rope;
        CU(k_a2a_seq2head(a, cs_));
      }
      {
        AttnArgs a{};
        a.q = e.q;
        a.k = e.k;
        a.v = e.v;
        a.o = e.o;
        a.lse = e.lse;  // not kept: the encoder has no backward
        a.ldq = a.ldk = a.ldv = ldh;
        a.ldo = ldh;
        const bool full = e.fullatt[size_t(i)];
        a.seq_start = full ? e.st : e.wst;
        a.seq_end = full ? e.en : e.wen;
        a.N = Np;
        a.hq = a.hk = e.heads;
        a.scale = 1.0f / std::sqrt(float(e.d));
        a.causal = 0;
        CU(k_attn_fwd_tc(a, cs_));
      }
      const bf16* o2 = e.o;
      int64_t ldo2 = ldh;
      if (e.d != 128) {
        A2AArgs a{};
        a.sp = 1;
        a.rank = 0;
        a.rows = 1;
        a.seq = Np;
        a.ngroups = 1;
        a.g[0].heads_total = e.heads;
        a.g[0].full[0] = e.o;
        a.local[0] = e.o2;
        a.local_ld = Wq;
        a.hd = e.d;
        CU(k_a2a_head2seq(a, cs_));
        o2 = e.o2;
        ldo2 = Wq;
      }
      {
        GemmDesc g = egd(Np, He, Wq, o2, ldo2, e.wp(ui, 3), Wq, GEMM_EPI_F32_RESID, e.x, He);
        g.R = e.x;
        g.ldr = He;
        g.bias = e.wp(ui, 4);
        CU(gemm_run(g, cs_));
      }
      CU(k_rmsnorm_fwd(e.x, e.wp(ui, 5), e.h, e.rstd, Np, He, ex_.rms_eps, cs_));
      {
        GemmDesc g = egd(Np, 2 * F, He, e.h, He, e.wp(ui, 6), He, GEMM_EPI_SWIGLU, nullptr, 2 * F);
        g.D2 = e.act;
        g.ldd2 = F;
        g.bias = e.wp(ui, 7);
        CU(gemm_run(g, cs_));
      }
      {
        GemmDesc g = egd(Np, He, F, e.act, F, e.wp(ui, 8), F, GEMM_EPI_F32_RESID, e.x, He);
        g.R = e.x;
        g.ldr = He;
        g.bias = e.wp(ui, 9);
        CU(gemm_run(g, cs_));
      }
    }
    TRY(done(ui));
  }
  // merger: rmsnorm_q, 2x2 merge (4 consecutive patches = one [4 He] row), MLP with GELU
  const int um = U - 1;
  TRY(use(um));
  if (run) {
    CU(k_rmsnorm_fwd(e.x, e.wp(um, 0), e.h, e.rstd, Np, He, ex_.rms_eps, cs_));
    {
      GemmDesc g = egd(Np / 4, 4 * He, 4 * He, e.h, 4 * He, e.wp(um, 1), 4 * He, GEMM_EPI_BF16, e.y1,
                       4 * He);
      g.bias = e.wp(um, 2);
      CU(gemm_run(g, cs_));
    }
    CU(k_gelu_bf16(e.y1, int64_t(Np / 4) * 4 * He, cs_));
    {
      GemmDesc g = egd(nf, H_, 4 * He, e.y1, 4 * He, e.wp(um, 3), 4 * He, GEMM_EPI_BF16, e.feat, H_);
      g.bias = e.wp(um, 4);
      CU(gemm_run(g, cs_));
    }
  }
  TRY(done(um));
  if (e.n_all == 0) return OPX_OK;  // no image in this SP group's rows: no scatter
  if (tr) {
    e1 = ev();
    cudaEventRecord(e1, cs_);
    mark("encoder." + e.name + mtag(), "encoder", 0, e0, e1);
    e0 = e1;
  }
  // scatter.<mod>: feature rows -> the owning SP rank's feature buffer (rows
  // in window order; dst_tok holds each row's placeholder token)
  FeatPeers fp{};
  for (int j = 0; j < int(p_.sp); ++j) fp.p[j] = reinterpret_cast<bf16*>(peer(j, off_feat_));
  CU(k_feat_scatter(e.feat, nf, H_, e.dst_rank, e.dst_tok, fp, cs_));
  TRY(barrier_sp(cs_));
  CU(k_feat_inject(x_saved_[0], reinterpret_cast<const bf16*>(arena_ + off_feat_), d_fmask_, T_, H_,
                   cs_));
  if (tr) {
    e1 = ev();
    cudaEventRecord(e1, cs_);
    mark("scatter." + e.name + mtag(), "encoder", 0, e0, e1);
  }
  return OPX_OK;
}

}  // namespace opx
