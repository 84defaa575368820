// models.hpp -- builders of the all-in-one training-step function
// for the BASELINE.json configs: a BERT MLM encoder (C1 tiny fp32 / C2 base /
// C4 large) and a GPT-2 causal LM (C3 medium / C5 XL).  Pure graph
// construction over the reference IR: forward ops are emitted with
// tb::Graph, the backward by tb::autodiff, then the fusion pass and the
// optimizer (SGD, or Adam with the fused bf16 param copy), optionally ZeRO-1
// partitioned (reduce_scatter -> sharded update -> all_gather).
//
// Parameters live in ONE flat f32 master buffer (and, under AutoCast, one flat
// bf16 copy); every weight is a `view` of it.  That single segment is what makes
// the optimizer one multi-tensor launch and the ZeRO collectives one bucket each.
#pragma once

#include <cmath>
#include <sstream>

#include "graph.hpp"

namespace tb {

struct ModelCfg {
  std::string kind = "bert";  // bert | gpt2
  int64_t L = 2, H = 128, A = 2, F = 512, V = 1024, S = 128, B = 8;
  int64_t max_pos = 0;      // 0 -> bert: 512, gpt2: S
  std::string dtype = "f32";  // activation / compute dtype: f32 | bf16
  double p = 0.0;           // dropout
  std::string opt = "sgd";  // sgd | adam
  double lr = 0.01, beta1 = 0.9, beta2 = 0.999, eps = 1e-6;
  int64_t seed_w = 42, seed_d = 1234, seed_drop = 7;
  int64_t world = 1;        // ZeRO-1 data-parallel ranks
  double ln_eps = 1e-12;
  int fuse = 1;             // run the fusion pass
  int save_deriv = 1;       // act linears save act'(u) for the backward instead of u
  double bucket_mb = 25.0;  // ZeRO gradient bucket size (f32 MB; 0: one bucket per segment)
  int zero = 0;             // force the ZeRO data plane at world 1 (identity collectives)
  int rules = 1;            // rule-based fusion of elementwise runs (ew_closure)
  std::string disable_patterns;  // comma list of FusionPattern names switched off
  int flash = 1;            // bf16 attention lse mode: 1 for S > 128, 2 always, 0 never (stored-P path)
  bool zero_on() const { return world > 1 || zero; }
  int64_t vocab_pad() const { return ((V + 63) / 64) * 64; }
  int64_t T() const { return B * S; }
  int64_t positions() const { return max_pos ? max_pos : (kind == "bert" ? std::max<int64_t>(512, S) : S); }
};

inline ModelCfg parse_cfg(const std::string& s) {
  ModelCfg c;
  std::istringstream is(s);
  std::string kv;
  while (std::getline(is, kv, ';')) {
    auto eq = kv.find('=');
    if (eq == std::string::npos) continue;
    std::string k = kv.substr(0, eq), v = kv.substr(eq + 1);
    auto I = [&] { return std::stoll(v); };
    auto D = [&] { return std::stod(v); };
    if (k == "kind") c.kind = v;
    else if (k == "L") c.L = I();
    else if (k == "H") c.H = I();
    else if (k == "A") c.A = I();
    else if (k == "F") c.F = I();
    else if (k == "V") c.V = I();
    else if (k == "S") c.S = I();
    else if (k == "B") c.B = I();
    else if (k == "max_pos") c.max_pos = I();
    else if (k == "dtype") c.dtype = v;
    else if (k == "p") c.p = D();
    else if (k == "opt") c.opt = v;
    else if (k == "lr") c.lr = D();
    else if (k == "beta1") c.beta1 = D();
    else if (k == "beta2") c.beta2 = D();
    else if (k == "eps") c.eps = D();
    else if (k == "seed_w") c.seed_w = I();
    else if (k == "seed_d") c.seed_d = I();
    else if (k == "seed_drop") c.seed_drop = I();
    else if (k == "world") c.world = I();
    else if (k == "ln_eps") c.ln_eps = D();
    else if (k == "fuse") c.fuse = int(I());
    else if (k == "save_deriv") c.save_deriv = int(I());
    else if (k == "bucket_mb") c.bucket_mb = D();
    else if (k == "zero") c.zero = int(I());
    else if (k == "flash") c.flash = int(I());
    else if (k == "rules") c.rules = int(I());
    else if (k == "disable_patterns") c.disable_patterns = v;
    else throw Error("unknown model config key '" + k + "'");
  }
  if (c.H % c.A) throw TypeError("H must be divisible by A");
  return c;
}

/// the `disable_patterns` key: FusionPattern names (graph.hpp) switched off
inline std::set<std::string> disabled_patterns(const ModelCfg& c) {
  std::set<std::string> off;
  std::istringstream ps(c.disable_patterns);
  std::string n;
  while (std::getline(ps, n, ',')) {
    if (n.empty()) continue;
    bool known = false;
    for (auto& fp : b200_patterns()) known = known || n == fp.name;
    if (!known) throw RegistryError("disable_patterns: no fusion pattern " + n);
    off.insert(n);
  }
  return off;
}

enum class Init { Uniform, Ones, Zeros };
struct ParamSeg {
  std::string name;
  std::vector<int64_t> shape;
  int64_t offset, numel;
  Init init;
};

struct TrainStep {
  ModelCfg cfg;
  FunctionPtr fn;
  int64_t P = 0;      // real parameter count
  int64_t P_pad = 0;  // padded to a multiple of world (ZeRO shards)
  std::vector<ParamSeg> segs;
  // function parameter roles (indices into fn->params)
  int i_ids = -1, i_labels = -1, i_pos = -1, i_type = -1, i_params = -1, i_p16 = -1, i_m = -1, i_v = -1,
      i_step = -1, i_rng = -1;
  std::vector<std::pair<int, int>> state_binding;  // (ret index, param index): in-place state update
  FusionStats fusion;
  // ZeRO: gradient / parameter buckets (flat offset, numel) covering [0, P_pad);
  // rank r owns slice r (ceil(numel / world) elements) of every bucket, and
  // its shard state is the concatenation of those slices in bucket order
  std::vector<std::pair<int64_t, int64_t>> buckets;
  int64_t shard_n = 0;
  int rule_closures = 0;  // ew_closure groups made by finalize_graph
  int64_t shard() const { return shard_n ? shard_n : P_pad / cfg.world; }
};

class ParamTable {
 public:
  // every segment starts on a 64-element (128 B for bf16) boundary so each
  // weight view is a legal TMA base for the tcgen05 GEMM
  void add(const std::string& name, std::vector<int64_t> shape, Init init) {
    int64_t n = 1;
    for (auto d : shape) n *= d;
    total_ = (total_ + 63) / 64 * 64;
    segs_.push_back({name, shape, total_, n, init});
    total_ += n;
  }
  const std::vector<ParamSeg>& segs() const { return segs_; }
  int64_t total() const { return total_; }
  const ParamSeg& get(const std::string& n) const {
    for (auto& s : segs_)
      if (s.name == n) return s;
    throw Error("no parameter " + n);
  }

 private:
  std::vector<ParamSeg> segs_;
  int64_t total_ = 0;
};

inline ParamTable param_table(const ModelCfg& c) {
  ParamTable t;
  const int64_t H = c.H, F = c.F, Vp = c.vocab_pad();
  const auto U = Init::Uniform, O = Init::Ones, Z = Init::Zeros;
  t.add("word_emb", {Vp, H}, U);
  t.add("pos_emb", {c.positions(), H}, U);
  if (c.kind == "bert") {
    t.add("type_emb", {2, H}, U);
    t.add("emb_ln.g", {H}, O);
    t.add("emb_ln.b", {H}, Z);
  }
  for (int64_t l = 0; l < c.L; ++l) {
    const std::string p = "layer" + std::to_string(l) + ".";
    if (c.kind == "gpt2") {
      t.add(p + "ln1.g", {H}, O);
      t.add(p + "ln1.b", {H}, Z);
    }
    t.add(p + "qkv.w", {H, 3 * H}, U);
    t.add(p + "qkv.b", {3 * H}, Z);
    t.add(p + "proj.w", {H, H}, U);
    t.add(p + "proj.b", {H}, Z);
    if (c.kind == "bert") {
      t.add(p + "ln1.g", {H}, O);
      t.add(p + "ln1.b", {H}, Z);
    } else {
      t.add(p + "ln2.g", {H}, O);
      t.add(p + "ln2.b", {H}, Z);
    }
    t.add(p + "ffn1.w", {H, F}, U);
    t.add(p + "ffn1.b", {F}, Z);
    t.add(p + "ffn2.w", {F, H}, U);
    t.add(p + "ffn2.b", {H}, Z);
    if (c.kind == "bert") {
      t.add(p + "ln2.g", {H}, O);
      t.add(p + "ln2.b", {H}, Z);
    }
  }
  if (c.kind == "bert") {
    t.add("mlm.dense.w", {H, H}, U);
    t.add("mlm.dense.b", {H}, Z);
    t.add("mlm.ln.g", {H}, O);
    t.add("mlm.ln.b", {H}, Z);
    t.add("mlm.dec.b", {Vp}, Z);
  } else {
    t.add("lnf.g", {H}, O);
    t.add("lnf.b", {H}, Z);
  }
  return t;
}

/// horizontal_fuse_collectives.  The per-parameter
/// collectives of partition_zero are merged into buckets
/// BEFORE the shard layout is fixed (a rank's shard is a function of the
/// bucket table, so merging afterwards would move elements between ranks):
/// consecutive cut candidates (parameter segment starts, 64-element aligned)
/// are merged greedily until a bucket holds >= bucket_elems; bucket_elems <= 0
/// keeps one bucket per segment (no fusion).  Returns (offset, numel) buckets
/// tiling [0, P).
inline std::vector<std::pair<int64_t, int64_t>> hfuse_buckets(const std::vector<int64_t>& starts, int64_t P,
                                                              int64_t bucket_elems) {
  std::vector<std::pair<int64_t, int64_t>> out;
  int64_t a = 0;
  for (int64_t c : starts) {
    if (c <= a || c >= P) continue;
    if (c - a >= std::max<int64_t>(bucket_elems, 1)) {
      out.push_back({a, c - a});
      a = c;
    }
  }
  if (P > a) out.push_back({a, P - a});
  return out;
}

/// rank r's ZeRO shard of a flat [P_pad] vector: slice r of every bucket
/// (zero padded to ceil(numel / world)), in bucket order -- what
/// reduce_scatter delivers and all_gather reassembles.
inline std::vector<float> shard_of(const TrainStep& ts, const std::vector<float>& full, int64_t rank) {
  if (ts.buckets.empty()) return full;
  const int64_t W = ts.cfg.world;
  std::vector<float> out;
  out.reserve(size_t(ts.shard()));
  for (auto [o, n] : ts.buckets) {
    const int64_t sh = (n + W - 1) / W;
    for (int64_t j = 0; j < sh; ++j) {
      const int64_t k = rank * sh + j;
      out.push_back(k < n ? full[size_t(o + k)] : 0.0f);
    }
  }
  return out;
}

/// Build the training step.  Inputs: ids, labels, pos_ids (+ type_ids for
/// BERT), params (f32 master, sharded under ZeRO), [p16 (half copy, full)],
/// [m, v (sharded), step].  Outputs: (loss, new states...) with in-place
/// bindings back onto the state inputs.
inline TrainStep build_train_step(const ModelCfg& c) {
  TrainStep ts;
  ts.cfg = c;
  ParamTable tab = param_table(c);
  ts.segs = tab.segs();
  ts.P = tab.total();
  ts.P_pad = ((ts.P + 64 * c.world - 1) / (64 * c.world)) * (64 * c.world);  // 128 B-aligned shards
  const bool amp = c.dtype != "f32";
  const DType act = dtype_from(c.dtype);
  const int64_t T = c.T(), H = c.H, Vp = c.vocab_pad();
  const bool adam = c.opt == "adam";
  const bool zero = c.zero_on();
  if (zero) {
    std::vector<int64_t> starts;
    for (auto& sg : ts.segs) starts.push_back(sg.offset);
    ts.buckets = hfuse_buckets(starts, ts.P_pad, int64_t(c.bucket_mb * 1e6 / 4.0));
    for (auto [o, n] : ts.buckets) ts.shard_n += (n + c.world - 1) / c.world;
  }

  Graph g;
  auto P = [&](const std::string& n, TensorType t) {
    auto v = g.param(n, t);
    return int(g.params().size() - 1);
  };
  ts.i_ids = P("ids", {kI32, {T}});
  ts.i_labels = P("labels", {kI32, {T}});
  ts.i_pos = P("pos_ids", {kI32, {T}});
  if (c.kind == "bert") ts.i_type = P("type_ids", {kI32, {T}});
  const int64_t pstate = zero ? ts.shard() : ts.P_pad;
  ts.i_params = P("params", {kF32, {pstate}});
  // the compute copy: full under AutoCast; under ZeRO the rank keeps its
  // SHARD of it and the step all-gathers the full copy first (f32 steps
  // gather the master shard itself)
  if (amp) ts.i_p16 = P("p16", {act, {zero ? ts.shard() : ts.P_pad}});
  if (adam) {
    ts.i_m = P("m", {kF32, {pstate}});
    ts.i_v = P("v", {kF32, {pstate}});
    ts.i_step = P("step", {kF32, {1}});
  }
  // dropout step counter (f32[1] state, +1 per step): the Philox counter's
  // 4th word, so the dropout masks change every step (device and oracle alike)
  if (c.p > 0.0) ts.i_rng = P("rng_step", {kF32, {1}});
  auto par = [&](int i) { return g.params()[i]; };
  VarPtr rng_next = c.p > 0.0 ? g.op("add_scalar", {par(ts.i_rng)}, {{"value", 1.0}}, "rng") : nullptr;
  VarPtr ids = par(ts.i_ids), labels = par(ts.i_labels), pos_ids = par(ts.i_pos);
  VarPtr wsrc = amp ? par(ts.i_p16) : par(ts.i_params);
  if (zero) {
    // ZeRO-1 all-gather of the compute copy, one collective per bucket at the
    // top of the step: the forward's first layers wait only for their own
    // bucket, the rest of the gather overlaps the forward (comm stream)
    VarPtr src = wsrc;
    std::vector<VarPtr> full;
    int64_t so = 0;
    for (auto [o, n] : ts.buckets) {
      const int64_t sh = (n + c.world - 1) / c.world;
      VarPtr v = g.op("view", {src}, {{"offset", so}, {"shape", std::to_string(sh)}}, "psh");
      full.push_back(g.op("all_gather", {v}, {{"world", c.world}, {"shape", std::to_string(n)}}, "pag"));
      so += sh;
    }
    wsrc = full.size() == 1 ? full[0] : g.op("concat", full, {}, "pfull");
  }

  std::vector<Leaf> leaves;
  std::map<std::string, VarPtr> W;
  for (auto& s : ts.segs) {
    auto v = g.op("view", {wsrc}, {{"offset", s.offset}, {"shape", opreg::shape_attr(s.shape)}}, "w");
    W[s.name] = v;
    leaves.push_back({v, s.offset, s.numel});
  }
  int64_t salt = 1;
  auto drop_attrs = [&](AttrMap a = {}) {
    a["p"] = c.p;
    a["seed"] = c.seed_drop;
    a["salt"] = salt++;
    return a;
  };
  auto linear = [&](VarPtr x, const std::string& w, const std::string& b, const std::string& actf = "none",
                    int tw = 0) {
    AttrMap a{{"act", actf}};
    if (tw) a["tw"] = std::int64_t(1);
    // the forward epilogue saves act'(u) (not u): the backward's dgrad epilogue
    // then multiplies by it instead of re-evaluating the derivative
    if (actf == "gelu" || actf == "relu") {
      a["save_preact"] = std::int64_t(1);
      if (c.save_deriv) a["save"] = std::string("grad");
    }
    VarPtr y = g.op("linear", {x, W[w], W[b]}, a);
    return y->ty.is_tuple() ? g.get(y, 0) : y;
  };
  AttrMap attn_attrs{{"heads", c.A}, {"seq", c.S}, {"causal", std::int64_t(c.kind == "gpt2")}};
  // bf16, head dim 64: lse mode keeps only the per-row log-sum-exp for the
  // backward (P recomputed there, not stored), plus the dropout keep bits.
  // S > 128 always (flash kernels); at S <= 128 the stored-P persistent path
  // is faster (BERT-base 6.16k vs 6.12k samples/s with lse mode there: the
  // backward's QK^T recompute costs more than the P traffic it saves), so
  // lse mode there is opt-in (flash=2) -- it raises the no-remat max batch
  // 3242 -> 3554 and leaves the remat max batch at 8714
  const bool flash = c.dtype == "bf16" && c.H / c.A == 64 && c.S % 8 == 0 &&
                     ((c.flash == 1 && c.S > 128) || c.flash == 2);
  if (flash) attn_attrs["lse"] = std::int64_t(1);
  if (c.p > 0.0 && c.dtype == "bf16" && c.H / c.A == 64 && c.S % 8 == 0 && (flash || c.S <= 128))
    attn_attrs["save_mask"] = std::int64_t(1);
  // residual LayerNorms save their dropout keep bits for the backward (no Philox re-run)
  auto ln_attrs = [&]() {
    AttrMap a{{"eps", c.ln_eps}};
    if (c.p > 0.0 && c.H % 8 == 0 && (c.T() * c.H) % 32 == 0) a["save_mask"] = std::int64_t(1);
    return a;
  };

  // ---- embeddings
  VarPtr h;
  if (c.kind == "bert") {
    VarPtr type_ids = par(ts.i_type);
    VarPtr e;
    if (c.dtype == "bf16") {  // one fused gather-and-add kernel (same roundings)
      e = g.op("embedding_sum", {ids, pos_ids, type_ids, W["word_emb"], W["pos_emb"], W["type_emb"]});
    } else {
      e = g.op("add", {g.op("embedding", {ids, W["word_emb"]}), g.op("embedding", {pos_ids, W["pos_emb"]})});
      e = g.op("add", {e, g.op("embedding", {type_ids, W["type_emb"]})});
    }
    VarPtr ln = g.op("layer_norm", {e, W["emb_ln.g"], W["emb_ln.b"]}, {{"eps", c.ln_eps}});
    h = g.get(ln, 0);
    if (c.p > 0) h = g.op("dropout", {h}, drop_attrs());
  } else {
    h = g.op("add", {g.op("embedding", {ids, W["word_emb"]}), g.op("embedding", {pos_ids, W["pos_emb"]})});
    if (c.p > 0) h = g.op("dropout", {h}, drop_attrs());
  }
  // ---- encoder / decoder blocks
  for (int64_t l = 0; l < c.L; ++l) {
    const std::string p = "layer" + std::to_string(l) + ".";
    if (c.kind == "bert") {  // post-LN
      VarPtr qkv = linear(h, p + "qkv.w", p + "qkv.b");
      VarPtr at = g.op("attention", {qkv}, drop_attrs(attn_attrs));
      VarPtr ao = linear(g.get(at, 0), p + "proj.w", p + "proj.b");
      VarPtr l1 = g.op("add_layer_norm", {ao, h, W[p + "ln1.g"], W[p + "ln1.b"]}, drop_attrs(ln_attrs()));
      VarPtr h1 = g.get(l1, 0);
      VarPtr f = linear(h1, p + "ffn1.w", p + "ffn1.b", "gelu");
      VarPtr f2 = linear(f, p + "ffn2.w", p + "ffn2.b");
      VarPtr l2 = g.op("add_layer_norm", {f2, h1, W[p + "ln2.g"], W[p + "ln2.b"]}, drop_attrs(ln_attrs()));
      h = g.get(l2, 0);
    } else {  // GPT-2 pre-LN: h = h + drop(attn(ln1(h))); h = h + drop(mlp(ln2(h)))
      VarPtr x1 = g.get(g.op("layer_norm", {h, W[p + "ln1.g"], W[p + "ln1.b"]}, {{"eps", 1e-5}}), 0);
      VarPtr qkv = linear(x1, p + "qkv.w", p + "qkv.b");
      VarPtr at = g.op("attention", {qkv}, drop_attrs(attn_attrs));
      VarPtr ao = linear(g.get(at, 0), p + "proj.w", p + "proj.b");
      if (c.p > 0) ao = g.op("dropout", {ao}, drop_attrs());
      h = g.op("add", {ao, h});
      VarPtr x2 = g.get(g.op("layer_norm", {h, W[p + "ln2.g"], W[p + "ln2.b"]}, {{"eps", 1e-5}}), 0);
      VarPtr f = linear(x2, p + "ffn1.w", p + "ffn1.b", "gelu");
      VarPtr f2 = linear(f, p + "ffn2.w", p + "ffn2.b");
      if (c.p > 0) f2 = g.op("dropout", {f2}, drop_attrs());
      h = g.op("add", {f2, h});
    }
  }
  // ---- LM head (tied decoder: logits = x . word_emb^T, all positions as HF computes)
  VarPtr x;
  if (c.kind == "bert") {
    VarPtr t = linear(h, "mlm.dense.w", "mlm.dense.b", "gelu");
    x = g.get(g.op("layer_norm", {t, W["mlm.ln.g"], W["mlm.ln.b"]}, {{"eps", c.ln_eps}}), 0);
  } else {
    x = g.get(g.op("layer_norm", {h, W["lnf.g"], W["lnf.b"]}, {{"eps", 1e-5}}), 0);
  }
  VarPtr logits;
  if (c.kind == "bert") {
    logits = linear(x, "word_emb", "mlm.dec.b", "none", /*tw=*/1);
  } else {
    logits = g.op("matmul_t", {x, W["word_emb"]}, {{"tb", std::int64_t(1)}});
  }
  VarPtr ce = g.op("cross_entropy", {logits, labels},
                   {{"classes", c.V}, {"ignore_index", std::int64_t(-100)}, {"grad", std::int64_t(1)}});
  VarPtr loss = g.get(ce, 0, "loss");

  // ---- backward (autodiff) -> flat f32 gradient [P]
  // gaps between aligned segments and the tail up to P_pad get zero gradients
  // (SPEC.md:513,566 zero-padded shards)
  GradResult gr = autodiff(g, loss, leaves, ts.P_pad, /*make_flat=*/!zero);
  VarPtr grad = gr.flat_grad;
  if (grad && numel(grad->ty.tensor()) != ts.P_pad)
    throw Error("build_train_step: flat gradient has " + std::to_string(numel(grad->ty.tensor())) +
                " elements, expected P_pad " + std::to_string(ts.P_pad));

  // ---- optimizer (+ ZeRO-1)
  std::vector<VarPtr> rets{loss};
  const std::string full_shape = std::to_string(ts.P_pad);
  VarPtr gsh = grad;
  if (zero) {
    // one sum-reduce-scatter per bucket over the
    // bucket's own gradient pieces -- so in the IR each collective depends
    // only on its bucket and overlap_schedule can start it as soon as those
    // pieces exist; the shard is the concatenation of the bucket shards
    std::vector<VarPtr> shards;
    size_t pi = 0;
    for (auto [o, n] : ts.buckets) {
      std::vector<VarPtr> pieces;
      while (pi < gr.parts.size() && gr.parts[pi].first < o + n) {
        if (gr.parts[pi].first < o) throw Error("ZeRO: a gradient piece straddles a bucket boundary");
        pieces.push_back(gr.parts[pi++].second);
      }
      VarPtr gb = pieces.size() == 1 ? pieces[0] : g.op("concat", pieces, {}, "gbkt");
      if (numel(gb->ty.tensor()) != n) throw Error("ZeRO: bucket pieces do not tile the bucket");
      shards.push_back(g.op("reduce_scatter", {gb}, {{"world", c.world}}, "gsh"));
    }
    gsh = shards.size() == 1 ? shards[0] : g.op("concat", shards, {}, "gshard");
  }
  if (!adam) {
    // mean over ranks folded into the step size: lr / N
    VarPtr np = g.op("sgd_update", {par(ts.i_params), gsh}, {{"lr", c.lr / double(c.world)}});
    rets.push_back(np);
    ts.state_binding.push_back({1, ts.i_params});
    if (amp) {  // refresh the compute copy (its shard under ZeRO: gathered next step)
      VarPtr nh = g.op("convert", {np}, {{"to", c.dtype}});
      rets.push_back(nh);
      ts.state_binding.push_back({2, ts.i_p16});
    }
  } else {
    VarPtr step = par(ts.i_step);
    VarPtr step1 = g.op("add_scalar", {step}, {{"value", 1.0}});
    AttrMap aa{{"lr", c.lr}, {"beta1", c.beta1}, {"beta2", c.beta2}, {"eps", c.eps},
               {"grad_scale", 1.0 / double(c.world)}, {"half", c.dtype}};
    VarPtr up = g.op("adam_update_ex", {par(ts.i_params), gsh, par(ts.i_m), par(ts.i_v), step1}, aa);
    VarPtr np = g.get(up, 0), nm = g.get(up, 1), nv = g.get(up, 2), nh = g.get(up, 3);
    rets.insert(rets.end(), {np, nm, nv, step1});
    ts.state_binding.push_back({1, ts.i_params});
    ts.state_binding.push_back({2, ts.i_m});
    ts.state_binding.push_back({3, ts.i_v});
    ts.state_binding.push_back({4, ts.i_step});
    if (amp) {  // the bf16 compute copy (its shard under ZeRO: gathered next step)
      rets.push_back(nh);
      ts.state_binding.push_back({5, ts.i_p16});
    }
  }
  if (rng_next) {
    rets.push_back(rng_next);
    ts.state_binding.push_back({int(rets.size()) - 1, ts.i_rng});
  }
  FunctionPtr raw = g.finish(rets);
  LetSeq seq = ir::flatten(*raw);
  ts.fusion = fuse(seq, c.fuse != 0, disabled_patterns(c));
  ts.fn = ir::make_fn(raw->name, raw->params, seq);
  return ts;
}

/// trainc::Rng (tensor.hpp:145-176) init: weights uniform(-0.02, 0.02) in
/// segment order from seed_w; LayerNorm gamma 1, biases/beta 0.
inline std::vector<float> init_params(const TrainStep& ts) {
  std::vector<float> p(size_t(ts.P_pad), 0.0f);
  Rng rng(static_cast<uint64_t>(ts.cfg.seed_w));
  for (auto& s : ts.segs) {
    for (int64_t i = 0; i < s.numel; ++i) {
      float v = 0.0f;
      if (s.init == Init::Uniform) v = rng.uniform(-0.02f, 0.02f);
      else if (s.init == Init::Ones) v = 1.0f;
      p[size_t(s.offset + i)] = v;
    }
  }
  // vocabulary padding rows of the word embedding stay zero (never indexed)
  for (auto& s : ts.segs)
    if (s.name == "word_emb")
      for (int64_t r = ts.cfg.V; r < ts.cfg.vocab_pad(); ++r)
        for (int64_t j = 0; j < ts.cfg.H; ++j) p[size_t(s.offset + r * ts.cfg.H + j)] = 0.0f;
  return p;
}

inline uint16_t bf16_bits(float f) {
  uint32_t x;
  std::memcpy(&x, &f, 4);
  if ((x & 0x7fffffffu) > 0x7f800000u) return uint16_t((x >> 16) | 0x40u);
  x += 0x7fffu + ((x >> 16) & 1u);
  return uint16_t(x >> 16);
}

}  // namespace tb
