// autocast.hpp -- the AutoCast mixed-precision pass (PAPER.md
// §3.1.2, Fig. 3) over the reference IR, moved to bf16.
//
//  Policy       per base op: Low (compute in the low dtype, bf16 by default),
//               F32 (numerically sensitive: statistics, losses, optimizer), or
//               Follow (adopt the inputs' dtype when uniform, else f32).  Total:
//               an op without an entry is an error, never a silent default.
//  autocast     forward walk of the let sequence: resolves every Call's
//               precision, records one cast site per (producer, consumer, arg)
//               whose dtype differs, and re-infers output types through the
//               registry's type relations with the cast-to input types.
//  place_casts  the exclusive/shared decision: a producer
//               value needed in dtype d by k consumers gets one exclusive cast
//               per fusion-capable consumer (emitted immediately before it, so
//               the fusion rules can take it into that consumer's closure) and
//               one shared cast for the rest (emitted after the producer); with
//               no fusion-capable consumer, exactly one shared cast.
//  fusion query "fusion-capable" is answered by the rule table of the fusion
//               module: Elemwise/Injective/Reduction
//               consumers absorb an elementwise predecessor; Opaque ops (GEMMs,
//               attention, collectives, optimizer) do not.
//
// Casts are emitted as the reference's `cast` when the target is f16/f32 and as
// `convert` (ext_ops.hpp) for bf16.  Parameters (master weights) keep their
// f32 type; the optimizer is F32 policy, so it reads and writes f32 only.
#pragma once

#include <cstdio>
#include <cstdlib>
#include <map>
#include <set>
#include <string>
#include <vector>

#include "graph.hpp"

namespace tb {

/// F32Math: the op computes in f32 but its b200 kernel loads low-precision
/// inputs and widens them in registers -- the cast-up lives inside the
/// consumer's kernel.  Activation-shaped f32 inputs next to a low one are cast
/// down (the b200 kernels read one activation storage dtype); statistics,
/// gamma and beta keep theirs.
enum class Prec { Low, F32, Follow, F32Math };

struct PrecisionPolicy {
  DType low = kBF16;
  std::map<std::string, Prec> by_op;
  Prec of(const std::string& base) const {
    auto it = by_op.find(base);
    if (it == by_op.end()) throw Error("autocast: precision policy has no entry for op '" + base + "'");
    return it->second;
  }
};

/// SPEC.md:322 default, extended to the b200 ops: contractions Low; reductions,
/// normalisation statistics, softmax, losses, optimizer F32; the rest Follow.
inline PrecisionPolicy default_policy(DType low = kBF16) {
  PrecisionPolicy p;
  p.low = low;
  for (const char* o : {"matmul", "matmul_t", "linear", "matmul_dact", "matmul_pair", "batch_matmul",
                        "attention", "attention_dx"})
    p.by_op[o] = Prec::Low;
  for (const char* o : {"sum", "mean", "mse", "softmax", "softmax_dx", "layer_norm", "add_layer_norm", "layer_norm_dx",
                        "cross_entropy", "sgd_update", "adam_update", "adam_update_ex", "colsum", "embedding_dx",
                        "allreduce", "reduce_scatter", "all_gather", "reduce_scatter_batched", "all_gather_batched",
                        "concat", "view", "shard"})
    p.by_op[o] = Prec::F32;
  for (const char* o : {"add", "sub", "mul", "div", "neg", "tanh", "relu", "gtz", "tanh_dx", "bcast", "transpose",
                        "reshape", "gelu", "gelu_dx", "dropout", "embedding", "embedding_sum", "add_scalar", "fill"})
    p.by_op[o] = Prec::Follow;
  return p;
}

/// The policy the b200 step uses: default_policy with the normalisation,
/// softmax, loss and column-sum ops as F32Math (their kernels read bf16 and
/// accumulate in f32: k_ln_fwd16 / k_ln_bwd16 / k_attn_* / k_ce_row / k_colsum).
inline PrecisionPolicy b200_policy() {
  PrecisionPolicy p = default_policy(kBF16);
  for (const char* o : {"layer_norm", "add_layer_norm", "layer_norm_dx", "softmax", "softmax_dx", "cross_entropy",
                        "colsum", "embedding_dx"})
    p.by_op[o] = Prec::F32Math;
  // gathers from the bf16 compute copy of the tables (like the hand-built
  // step's embedding_sum): the table cast is a parameter cast, folded into
  // the optimizer's bf16 copy by +fold
  for (const char* o : {"embedding", "embedding_sum"}) p.by_op[o] = Prec::Low;
  return p;
}

inline PrecisionPolicy all_f32_policy() {
  PrecisionPolicy p = default_policy();
  for (auto& kv : p.by_op) kv.second = Prec::F32;
  return p;
}

inline bool is_float(DType d) { return d == kF32 || d == kF16 || d == kBF16; }

/// The fusion module's rule table: can `base` take an elementwise
/// predecessor (a cast) into its closure?
inline bool absorbs_elementwise_predecessor(const std::string& base) {
  if (base == "cast" || base == "convert") return true;
  const auto cat = opreg::registry().base(base).category;
  return cat == opreg::OpCategory::Elemwise || cat == opreg::OpCategory::Injective ||
         cat == opreg::OpCategory::Reduction;
}

struct CastSite {
  const ir::Var* producer;
  size_t consumer;  // let index
  size_t arg;
  DType to;
};

enum class Placement { Auto, AllShared };

struct CastReport {
  int sites = 0;
  int casts = 0;
  int exclusive = 0;
  int shared = 0;
  int low_ops = 0;           // Calls resolved to the low dtype
  int f32_violations = 0;    // F32-policy Calls left with a non-f32 float input (must be 0)
  int standalone_casts = 0;  // casts of computed values the fusion rules cannot take into a closure
  int param_casts = 0;       // casts of function parameters (the b200 step keeps these as the
                             // bf16 compute copy written by the fused optimizer update)
};

inline std::string dtype_token(DType d) {
  return d == kF32 ? "f32" : d == kF16 ? "f16" : d == kBF16 ? "bf16" : "i32";
}

/// Apply the policy to an all-f32 typed ANF function.
inline FunctionPtr autocast(const ir::FunctionIR& fn, const PrecisionPolicy& pol, CastReport* rep = nullptr,
                            Placement placement = Placement::Auto) {
  LetSeq seq = ir::flatten(fn);
  CastReport r;
  // ---- phase 1: resolve precisions, collect sites, re-infer types ----------
  std::map<const ir::Var*, Type> ty;  // new types of params and lets
  for (auto& p : fn.params) ty[p.get()] = p->ty;
  std::vector<CastSite> sites;
  std::vector<Type> let_ty(seq.lets.size());
  std::vector<std::string> let_base(seq.lets.size());
  for (size_t i = 0; i < seq.lets.size(); ++i) {
    const auto& b = seq.lets[i];
    const auto& e = b.value;
    if (e->kind == ExprKind::TupleGet) {
      const Type& t = ty.at(e->args.at(0)->var.get());
      let_ty[i] = t.tuple().fields.at(size_t(e->index));
      ty[b.var.get()] = let_ty[i];
      continue;
    }
    if (e->kind != ExprKind::Call) throw Error("autocast: unsupported let kind (expects calls and tuple_get)");
    const std::string base = base_name(e->op);
    let_base[i] = base;
    std::vector<Type> in;
    for (auto& a : e->args) {
      if (a->kind != ExprKind::VarRef) throw Error("autocast: expects ANF var arguments");
      in.push_back(ty.at(a->var.get()));
    }
    if (base != "cast" && base != "convert") {
      const Prec pr = pol.of(base);
      DType target = kF32;
      if (pr == Prec::F32Math) {
        // the b200 kernels read all activation-shaped inputs (those shaped like
        // a low-precision input) in one storage dtype and widen on load; the
        // statistics / gamma / beta keep their own dtype
        std::set<std::vector<int64_t>> low_shapes;
        for (auto& t : in)
          if (t.is_tensor() && t.tensor().dtype == pol.low) low_shapes.insert(t.tensor().shape);
        // f32 accumulators by contract (embedding_dx's base gradient)
        static const std::map<std::string, std::set<size_t>> pinned_f32 = {{"embedding_dx", {2}}};
        auto pin = pinned_f32.find(base);
        for (size_t k = 0; k < in.size(); ++k) {
          if (!in[k].is_tensor() || in[k].tensor().dtype != kF32 || !low_shapes.count(in[k].tensor().shape)) continue;
          if (pin != pinned_f32.end() && pin->second.count(k)) continue;
          sites.push_back({e->args[k]->var.get(), i, k, pol.low});
          auto t = in[k].tensor();
          t.dtype = pol.low;
          in[k] = Type(t);
        }
        let_ty[i] = opreg::registry().type_rel_of(e->op)(in, e->call_attrs);
        ty[b.var.get()] = let_ty[i];
        continue;
      } else if (pr == Prec::Low) {
        target = pol.low;
      }
      else if (pr == Prec::Follow) {
        std::set<DType> ds;
        for (auto& t : in)
          if (t.is_tensor() && is_float(t.tensor().dtype)) ds.insert(t.tensor().dtype);
        target = ds.size() == 1 ? *ds.begin() : kF32;
      }
      if (target == pol.low && target != kF32 && pr == Prec::Low) ++r.low_ops;
      for (size_t k = 0; k < in.size(); ++k) {
        if (!in[k].is_tensor() || !is_float(in[k].tensor().dtype) || in[k].tensor().dtype == target) continue;
        sites.push_back({e->args[k]->var.get(), i, k, target});
        auto t = in[k].tensor();
        t.dtype = target;
        in[k] = Type(t);
      }
    }
    let_ty[i] = opreg::registry().type_rel_of(e->op)(in, e->call_attrs);
    ty[b.var.get()] = let_ty[i];
  }
  r.sites = int(sites.size());

  // ---- phase 2: place casts (exclusive / shared) ----------------------------
  struct Group {
    std::vector<size_t> consumers;  // distinct let indices, ascending
  };
  std::map<std::pair<const ir::Var*, DType>, Group> groups;
  std::vector<std::pair<const ir::Var*, DType>> order;  // first-seen order (deterministic)
  for (auto& s : sites) {
    auto key = std::make_pair(s.producer, s.to);
    if (!groups.count(key)) order.push_back(key);
    auto& g = groups[key];
    if (g.consumers.empty() || g.consumers.back() != s.consumer) g.consumers.push_back(s.consumer);
  }
  // exclusive: one cast per fusion-capable consumer (with k == 1 this is the
  // single cast); everything else shares one cast per (producer, dtype)
  std::set<std::pair<size_t, std::pair<const ir::Var*, DType>>> exclusive_at;
  std::set<std::pair<const ir::Var*, DType>> needs_shared;
  for (auto& key : order)
    for (size_t c : groups[key].consumers) {
      if (placement == Placement::Auto && absorbs_elementwise_predecessor(let_base[c])) exclusive_at.insert({c, key});
      else needs_shared.insert(key);
    }

  // rebuild with fresh vars (the input function is left untouched)
  std::map<const ir::Var*, VarPtr> nv;
  for (auto& p : fn.params) nv[p.get()] = p;
  std::map<std::pair<const ir::Var*, DType>, VarPtr> shared_var;
  LetSeq out;
  int serial = 0;
  auto emit_cast = [&](const ir::Var* src, DType to) {
    const VarPtr& sv = nv.at(src);
    auto t = sv->ty.tensor();
    t.dtype = to;
    auto call = ir::call(to == kBF16 ? "convert" : "cast", {ir::var_ref(sv)}, AttrMap{{"to", dtype_token(to)}});
    call->ty = Type(t);
    auto v = ir::make_var(sv->id + "_" + dtype_token(to) + std::to_string(serial++), Type(t));
    out.lets.push_back({v, call});
    ++r.casts;
    return v;
  };
  auto emit_shared_of = [&](const ir::Var* producer) {
    for (auto& key : order)
      if (key.first == producer && needs_shared.count(key)) {
        shared_var[key] = emit_cast(producer, key.second);
        ++r.shared;
      }
  };
  for (auto& p : fn.params) emit_shared_of(p.get());
  for (size_t i = 0; i < seq.lets.size(); ++i) {
    const auto& b = seq.lets[i];
    const auto& e = b.value;
    std::vector<ExprPtr> args;
    std::map<std::pair<const ir::Var*, DType>, VarPtr> mine;  // this consumer's exclusive casts
    for (size_t k = 0; k < e->args.size(); ++k) {
      const ir::Var* pv = e->args[k]->var.get();
      VarPtr use = nv.at(pv);
      for (auto& st : sites) {
        if (st.consumer != i || st.arg != k) continue;
        auto key = std::make_pair(pv, st.to);
        if (mine.count(key)) {
          use = mine[key];  // same producer at another arg: one cast per consumer
        } else if (exclusive_at.count({i, key})) {
          use = mine[key] = emit_cast(pv, st.to);  // immediately before its consumer
          ++r.exclusive;
        } else {
          use = shared_var.at(key);
        }
      }
      args.push_back(ir::var_ref(use));
    }
    ExprPtr ne;
    if (e->kind == ExprKind::TupleGet) ne = ir::tuple_get(args.at(0), e->index);
    else ne = ir::call(e->op, args, e->call_attrs);
    ne->ty = let_ty[i];
    auto v = ir::make_var(b.var->id, let_ty[i], b.var->attrs);
    nv[b.var.get()] = v;
    out.lets.push_back({v, ne});
    emit_shared_of(b.var.get());
  }
  if (seq.ret && seq.ret->kind == ExprKind::Tuple) {
    std::vector<ExprPtr> xs;
    TupleType tt;
    for (auto& a : seq.ret->args) {
      const VarPtr& v = nv.at(a->var.get());
      xs.push_back(ir::var_ref(v));
      tt.fields.push_back(v->ty.tensor());
    }
    out.ret = ir::tuple(xs);
    out.ret->ty = tt;
  } else {
    throw Error("autocast: expects a tuple return");
  }

  // ---- post-pass checks and the fusion-rule cast census ----------------------
  std::map<const ir::Var*, std::vector<std::string>> consumers_of;
  std::map<const ir::Var*, std::string> producer_base;
  for (auto& b : out.lets) {
    if (b.value->kind != ExprKind::Call) continue;
    producer_base[b.var.get()] = base_name(b.value->op);
    for (auto& a : b.value->args) consumers_of[a->var.get()].push_back(base_name(b.value->op));
  }
  for (auto& b : out.lets) {
    if (b.value->kind != ExprKind::Call) continue;
    const std::string base = base_name(b.value->op);
    if (base == "cast" || base == "convert") {
      const auto& cs = consumers_of[b.var.get()];
      const ir::Var* src = b.value->args[0]->var.get();
      const bool into_consumer = cs.size() == 1 && absorbs_elementwise_predecessor(cs[0]);
      const bool into_producer = producer_base.count(src) &&
                                 opreg::registry().base(producer_base[src]).category == opreg::OpCategory::Elemwise;
      bool is_param = false;  // a parameter, or a view of one (the flat weight buffer's slices)
      for (auto& p : fn.params) is_param |= p.get() == src;
      if (!is_param && producer_base.count(src) && producer_base[src] == "view") is_param = true;
      if (is_param) ++r.param_casts;
      else if (!into_consumer && !into_producer) {
        ++r.standalone_casts;
        if (std::getenv("TB_AUTOCAST_DEBUG"))
          std::fprintf(stderr, "standalone cast of %%%s (%s) -> %zu consumers (%s...)\n", src->id.c_str(),
                       producer_base.count(src) ? producer_base[src].c_str() : "param", cs.size(),
                       cs.empty() ? "" : cs[0].c_str());
      }
      continue;
    }
    if (pol.of(base) != Prec::F32) continue;
    for (auto& a : b.value->args) {
      const Type& t = a->var->ty;
      if (t.is_tensor() && is_float(t.tensor().dtype) && t.tensor().dtype != kF32) ++r.f32_violations;
    }
  }
  if (rep) *rep = r;
  return ir::make_fn(fn.name, fn.params, out);
}

/// After AutoCast: fold the per-step parameter casts into the optimizer's
/// compute copy.  Every `convert(view(params){offset,shape}) -> bf16` becomes
/// `view(p16){offset,shape}` of a new bf16 [P] state parameter, and the
/// optimizer (`adam_update_ex`) emits that copy (half=bf16) as a new state
/// output bound to p16.  p16 = bf16_rne(params) holds at step entry (the
/// initialiser and the previous step's Adam both round the same master
/// weights), so the result is bit-identical to the AutoCast'd step with the
/// convert launches gone -- the structure of the hand-built bf16 graph.
/// Returns the new function; *i_p16 and state_binding are updated.  World 1,
/// Adam only (returns the input when there is nothing to fold).
inline FunctionPtr fold_param_casts(const ir::FunctionIR& fn, int i_params, int64_t P_pad, int* i_p16,
                                    std::vector<std::pair<int, int>>& state_binding, int* folded = nullptr) {
  LetSeq seq = ir::flatten(fn);
  const ir::Var* params = fn.params.at(size_t(i_params)).get();
  std::map<const ir::Var*, const ExprPtr*> view_of;  // let var -> its view(params) call
  for (auto& b : seq.lets)
    if (b.value->kind == ExprKind::Call && base_name(b.value->op) == "view" &&
        b.value->args.at(0)->var.get() == params)
      view_of[b.var.get()] = &b.value;
  size_t adam = seq.lets.size();
  for (size_t i = 0; i < seq.lets.size(); ++i)
    if (seq.lets[i].value->kind == ExprKind::Call && base_name(seq.lets[i].value->op) == "adam_update_ex") adam = i;
  int n = 0;
  for (auto& b : seq.lets)
    if (b.value->kind == ExprKind::Call && base_name(b.value->op) == "convert" &&
        ir::attr_string(b.value->call_attrs, "to", "") == "bf16" && view_of.count(b.value->args.at(0)->var.get()))
      ++n;
  if (folded) *folded = n;
  if (n == 0 || adam == seq.lets.size()) return ir::make_fn(fn.name, fn.params, seq);

  std::vector<VarPtr> ps = fn.params;
  auto p16 = ir::make_var("p16", Type(TensorType{kBF16, {P_pad}}));
  ps.push_back(p16);
  *i_p16 = int(ps.size()) - 1;
  LetSeq out;
  VarPtr copy;
  for (size_t i = 0; i < seq.lets.size(); ++i) {
    auto b = seq.lets[i];
    const auto& e = b.value;
    if (e->kind == ExprKind::Call && base_name(e->op) == "convert" &&
        ir::attr_string(e->call_attrs, "to", "") == "bf16" && view_of.count(e->args.at(0)->var.get())) {
      const ExprPtr& vcall = *view_of[e->args[0]->var.get()];
      auto nv = ir::call(vcall->op, {ir::var_ref(p16)}, vcall->call_attrs);
      std::vector<Type> in{p16->ty};
      nv->ty = opreg::registry().type_rel_of(vcall->op)(in, vcall->call_attrs);
      out.lets.push_back({b.var, nv});
      continue;
    }
    if (i == adam) {
      AttrMap a = e->call_attrs;
      a["half"] = std::string("bf16");
      auto ne = ir::call(e->op, e->args, a);
      std::vector<Type> in;
      for (auto& x : e->args) in.push_back(x->var->ty);
      ne->ty = opreg::registry().type_rel_of(e->op)(in, a);
      auto v = ir::make_var(b.var->id, ne->ty, b.var->attrs);
      out.lets.push_back({v, ne});
      // later tuple_gets of the optimizer refer to the new var
      for (size_t j = i + 1; j < seq.lets.size(); ++j) {
        auto& ej = seq.lets[j].value;
        if (ej->kind == ExprKind::TupleGet && ej->args[0]->var.get() == b.var.get()) {
          auto g = ir::tuple_get(ir::var_ref(v), ej->index);
          g->ty = ne->ty.tuple().fields.at(size_t(ej->index));
          seq.lets[j].value = g;
          seq.lets[j].var->ty = g->ty;
        }
      }
      auto g = ir::tuple_get(ir::var_ref(v), 3);
      g->ty = ne->ty.tuple().fields.at(3);
      copy = ir::make_var("p16_next", g->ty);
      out.lets.push_back({copy, g});
      continue;
    }
    out.lets.push_back(b);
  }
  std::vector<ExprPtr> xs = seq.ret->args;
  xs.push_back(ir::var_ref(copy));
  TupleType tt;
  for (auto& x : xs) tt.fields.push_back(x->var->ty.tensor());
  out.ret = ir::tuple(xs);
  out.ret->ty = tt;
  state_binding.push_back({int(xs.size()) - 1, *i_p16});
  return ir::make_fn(fn.name, ps, out);
}

/// The session key `autocast=<policy>[+fold][+fuse]`, parsed in ONE place for
/// the device session (capi.cpp) and the oracle interpreter (oracle/interp.cpp)
/// so both build the same graph.  Unknown policies and unknown '+' tokens are
/// errors (never a silent all-f32 fallback).
struct AutocastKey {
  std::string policy;  // "b200" | "default" | "f32"
  bool fold = false;   // fold_param_casts
  bool fuse = false;   // fusion re-run on the bf16 graph
};

inline PrecisionPolicy policy_by_name(const std::string& pn) {
  if (pn == "b200") return b200_policy();
  if (pn == "default") return default_policy();
  if (pn == "f32") return all_f32_policy();
  throw Error("autocast: unknown policy '" + pn + "' (b200 | default | f32)");
}

inline AutocastKey parse_autocast_key(const std::string& key) {
  AutocastKey k;
  std::vector<std::string> parts;
  size_t a = 0;
  while (true) {
    size_t b = key.find('+', a);
    parts.push_back(key.substr(a, b == std::string::npos ? std::string::npos : b - a));
    if (b == std::string::npos) break;
    a = b + 1;
  }
  k.policy = parts[0];
  (void)policy_by_name(k.policy);  // validates
  for (size_t i = 1; i < parts.size(); ++i) {
    if (parts[i] == "fold") k.fold = true;
    else if (parts[i] == "fuse") k.fuse = true;
    else throw Error("autocast: unknown key token '+" + parts[i] + "' in '" + key + "'");
  }
  return k;
}

}  // namespace tb
