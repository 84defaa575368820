// graph.hpp -- typed ANF construction, reverse-mode autodiff and the peephole
// fusion pass, all over the reference IR (ir.hpp) and registry (opreg.hpp).
//
//  Graph      incremental ANF emitter on top of ir::AnfBuilder (ir.hpp:265-313)
//             that runs each op's type relation as it is emitted, so every Var
//             carries its TensorType/TupleType immediately.
//  autodiff   SPEC.md:217-279: reverse traversal of the let sequence, one
//             adjoint rule per base op, fan-out accumulation as an explicit
//             `add` chain in deterministic reverse-traversal order.  Leaves are
//             `view`s of a flat parameter buffer; their gradients are emitted as
//             one flat `concat` in offset order (the buffer the optimizer and the
//             ZeRO reduce-scatter consume as a single segment).
//  fuse       SPEC.md:346-422 restricted to the patterns the b200 kernels
//             implement: dact into the producing dgrad GEMM epilogue, residual
//             gradient sums into layer_norm_dx, tied-embedding accumulation into
//             embedding_dx; then dead-let elimination.
#pragma once

#include <algorithm>
#include <functional>
#include <map>
#include <set>
#include <unordered_map>

#include "ext_ops.hpp"

namespace tb {

using ir::ExprKind;
using ir::ExprPtr;
using ir::FunctionPtr;
using ir::LetBinding;
using ir::LetSeq;
using ir::VarPtr;

inline AttrMap attrs_merge(AttrMap a, const AttrMap& b) {
  for (auto& [k, v] : b) a[k] = v;
  return a;
}

class Graph {
 public:
  explicit Graph(std::string name = "train_step") : name_(std::move(name)), ab_("t") {}

  VarPtr param(const std::string& id, TensorType ty, AttrMap attrs = {}) {
    auto v = ir::make_var(id, Type(ty), std::move(attrs));
    ab_.reserve(id);
    params_.push_back(v);
    return v;
  }

  /// Emit `op(args...)` as a let; the type relation runs now.
  VarPtr op(const std::string& name, const std::vector<VarPtr>& args, AttrMap attrs = {},
            const std::string& hint = "") {
    std::vector<ExprPtr> xs;
    std::vector<Type> tys;
    for (auto& a : args) {
      if (!a) throw Error("internal: null argument to " + name);
      xs.push_back(ir::var_ref(a));
      tys.push_back(a->ty);
    }
    const auto& base = opreg::registry().base_of(name);
    if (base.arity >= 0 && int(args.size()) != base.arity)
      throw TypeError(name + ": expects " + std::to_string(base.arity) + " args, got " +
                      std::to_string(args.size()));
    Type out = opreg::registry().type_rel_of(name)(tys, attrs);
    auto call = ir::call(name, std::move(xs), std::move(attrs));
    call->ty = out;
    auto v = ab_.emit(call, hint.empty() ? "t" : hint);
    v->ty = out;
    return v;
  }

  VarPtr get(const VarPtr& tup, int i, const std::string& hint = "") {
    if (!tup->ty.is_tuple()) throw TypeError("tuple_get on non-tuple %" + tup->id);
    auto e = ir::tuple_get(ir::var_ref(tup), i);
    Type t = tup->ty.tuple().fields.at(i);
    e->ty = t;
    auto v = ab_.emit(e, hint.empty() ? "t" : hint);
    v->ty = t;
    return v;
  }

  LetSeq& seq() { return ab_.seq(); }
  const std::vector<VarPtr>& params() const { return params_; }

  FunctionPtr finish(const std::vector<VarPtr>& rets) {
    LetSeq s = ab_.seq();
    std::vector<ExprPtr> xs;
    TupleType tt;
    for (auto& r : rets) {
      xs.push_back(ir::var_ref(r));
      tt.fields.push_back(r->ty.tensor());
    }
    s.ret = ir::tuple(xs);
    s.ret->ty = tt;
    return ir::make_fn(name_, params_, s);
  }

 private:
  std::string name_;
  ir::AnfBuilder ab_;
  std::vector<VarPtr> params_;
};

inline const std::string& call_op(const LetBinding& b) { return b.value->op; }
inline VarPtr arg_var(const ExprPtr& call, size_t i) {
  const auto& a = call->args.at(i);
  return a->kind == ExprKind::VarRef ? a->var : nullptr;
}

// ------------------------------------------------------------------ autodiff

/// A differentiable leaf: a `view` of a flat parameter buffer, with the offset
/// of its master (f32) segment in the gradient buffer.
struct Leaf {
  VarPtr view;
  int64_t offset;  // element offset in the flat master buffer
  int64_t numel;
};

struct AdjointCtx {
  Graph& g;
  const LetBinding& let;
  std::vector<VarPtr> dout;  // per output field (tensor ops: size 1); null = no grad
};
using Adjoint = std::function<std::vector<VarPtr>(AdjointCtx&)>;  // grad per input (null = none)

inline std::map<std::string, Adjoint>& adjoints() {
  static std::map<std::string, Adjoint> m;
  return m;
}

inline AttrMap pick(const AttrMap& a, std::initializer_list<const char*> keys) {
  AttrMap r;
  for (auto* k : keys)
    if (a.count(k)) r[k] = a.at(k);
  return r;
}

/// Gradient of an elementwise input whose shape may be broadcast (trailing
/// dims, opreg.hpp:75-87): reduce over the broadcast dims.
inline VarPtr unbroadcast(Graph& g, const VarPtr& grad, const TensorType& target) {
  const auto& gt = grad->ty.tensor();
  if (gt.shape == target.shape) return grad;
  // only the bias-style case [.., N] -> [N] is needed by the models
  if (target.rank() == 1 && target.shape[0] == gt.shape.back()) {
    VarPtr s = g.op("colsum", {grad});
    if (target.dtype != kF32) s = g.op("convert", {s}, {{"to", std::string(dtype_str(target.dtype))}});
    return s;
  }
  if (numel(target) == numel(gt))
    return g.op("reshape", {grad}, {{"shape", opreg::shape_attr(target.shape)}});
  throw NonDifferentiable("unbroadcast from " + type_str(gt) + " to " + type_str(target));
}

inline void register_default_adjoints() {
  auto& A = adjoints();
  if (!A.empty()) return;
  // --- reference base ops ---
  A["add"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    auto a = arg_var(c.let.value, 0), b = arg_var(c.let.value, 1);
    return {a ? unbroadcast(c.g, c.dout[0], a->ty.tensor()) : nullptr,
            b ? unbroadcast(c.g, c.dout[0], b->ty.tensor()) : nullptr};
  };
  A["sub"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    auto b = arg_var(c.let.value, 1);
    return {c.dout[0], b ? c.g.op("neg", {unbroadcast(c.g, c.dout[0], b->ty.tensor())}) : nullptr};
  };
  A["mul"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    auto a = arg_var(c.let.value, 0), b = arg_var(c.let.value, 1);
    return {b ? unbroadcast(c.g, c.g.op("mul", {c.dout[0], b}), a->ty.tensor()) : nullptr,
            a ? unbroadcast(c.g, c.g.op("mul", {c.dout[0], a}), b->ty.tensor()) : nullptr};
  };
  A["neg"] = [](AdjointCtx& c) -> std::vector<VarPtr> { return {c.g.op("neg", {c.dout[0]})}; };
  // tanh: NeedsY, dx = tanh_dx(y, dy) = dy * (1 - y^2) -- not the paper's 1-2y
  A["tanh"] = [](AdjointCtx& c) -> std::vector<VarPtr> { return {c.g.op("tanh_dx", {c.let.var, c.dout[0]})}; };
  // relu: NeedsX, subgradient 0 at the kink via gtz
  A["relu"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    return {c.g.op("mul", {c.dout[0], c.g.op("gtz", {arg_var(c.let.value, 0)})})};
  };
  A["gelu"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    return {c.g.op("gelu_dx", {arg_var(c.let.value, 0), c.dout[0]})};
  };
  // matmul: dA = dY B^T, dB = A^T dY with the transposes absorbed
  A["matmul"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    auto a = arg_var(c.let.value, 0), b = arg_var(c.let.value, 1);
    return {c.g.op("matmul_t", {c.dout[0], b}, {{"tb", std::int64_t(1)}}),
            c.g.op("matmul_t", {a, c.dout[0]}, {{"ta", std::int64_t(1)}})};
  };
  // matmul_t (ta = 0): C = A op(B); dA = dC op(B)^T, dB = (A^T dC) or (dC^T A), f32
  A["matmul_t"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    const auto& at = c.let.value->call_attrs;
    if (ir::attr_int(at, "ta", 0) || ir::attr_double(at, "alpha", 1.0) != 1.0)
      throw NonDifferentiable("matmul_t adjoint supports ta=0, alpha=1");
    const int tb = int(ir::attr_int(at, "tb", 0));
    auto a = arg_var(c.let.value, 0), b = arg_var(c.let.value, 1);
    VarPtr dy = c.dout[0];
    VarPtr da = c.g.op("matmul_t", {dy, b}, {{"tb", std::int64_t(tb ? 0 : 1)}});
    VarPtr db = tb ? c.g.op("matmul_t", {dy, a}, {{"ta", std::int64_t(1)}, {"out", std::string("f32")}})
                   : c.g.op("matmul_t", {a, dy}, {{"ta", std::int64_t(1)}, {"out", std::string("f32")}});
    return {da, db};
  };
  A["convert"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    auto a = arg_var(c.let.value, 0);
    return {c.g.op("convert", {c.dout[0]}, {{"to", std::string(dtype_str(a->ty.tensor().dtype))}})};
  };
  A["reshape"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    auto a = arg_var(c.let.value, 0);
    return {c.g.op("reshape", {c.dout[0]}, {{"shape", opreg::shape_attr(a->ty.tensor().shape)}})};
  };
  A["dropout"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    return {c.g.op("dropout", {c.dout[0]}, pick(c.let.value->call_attrs, {"p", "seed", "salt"}))};
  };
  // --- extension ops ---
  // linear: du = dy * act'(u); dx = du W^T; dW = x^T du (f32, the master grad);
  // db = colsum(du).  Needs u (save_preact) for relu/gelu, y for tanh.
  A["linear"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    const auto& at = c.let.value->call_attrs;
    const std::string act = ir::attr_string(at, "act", "none");
    const int tw = int(ir::attr_int(at, "tw", 0));
    auto x = arg_var(c.let.value, 0), w = arg_var(c.let.value, 1);
    VarPtr dy = c.dout[0];
    if (!dy) return {nullptr, nullptr, nullptr};
    VarPtr du = dy;
    if (act != "none") {
      if (act == "tanh") {
        VarPtr y = c.let.var->ty.is_tuple() ? c.g.get(c.let.var, 0) : c.let.var;
        du = c.g.op("tanh_dx", {y, dy});
      } else {
        if (!c.let.var->ty.is_tuple()) throw NonDifferentiable("linear(act=" + act + ") needs save_preact=1");
        VarPtr u = c.g.get(c.let.var, 1);
        if (ir::attr_string(at, "save", "preact") == "grad")  // u already holds act'(pre-activation)
          du = c.g.op("mul", {dy, u});
        else
          du = act == "gelu" ? c.g.op("gelu_dx", {u, dy}) : c.g.op("mul", {dy, c.g.op("gtz", {u})});
      }
    }
    VarPtr dx = c.g.op("matmul_t", {du, w}, {{"tb", std::int64_t(tw ? 0 : 1)}});
    VarPtr dw = tw ? c.g.op("matmul_t", {du, x}, {{"ta", std::int64_t(1)}, {"out", std::string("f32")}})
                   : c.g.op("matmul_t", {x, du}, {{"ta", std::int64_t(1)}, {"out", std::string("f32")}});
    VarPtr db = c.g.op("colsum", {du});
    return {dx, dw, db};
  };
  A["attention"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    if (!c.dout[0]) return {nullptr};
    auto qkv = arg_var(c.let.value, 0);
    if (ir::attr_int(c.let.value->call_attrs, "lse", 0)) {  // flash: P recomputed from (ctx, lse)
      std::vector<VarPtr> args{qkv, c.g.get(c.let.var, 0), c.g.get(c.let.var, 1), c.dout[0]};
      if (c.let.var->ty.tuple().fields.size() > 2) args.push_back(c.g.get(c.let.var, 2));
      return {c.g.op("attention_dx", args, c.let.value->call_attrs)};
    }
    VarPtr probs = c.g.get(c.let.var, 1);
    std::vector<VarPtr> args{qkv, probs, c.dout[0]};
    if (c.let.var->ty.tuple().fields.size() > 2) args.push_back(c.g.get(c.let.var, 2));  // saved keep bits
    return {c.g.op("attention_dx", args, c.let.value->call_attrs)};
  };
  A["layer_norm"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    if (!c.dout[0]) return {nullptr, nullptr, nullptr};
    auto x = arg_var(c.let.value, 0), gm = arg_var(c.let.value, 1);
    auto t = c.g.op("layer_norm_dx", {x, gm, c.g.get(c.let.var, 1), c.g.get(c.let.var, 2), c.dout[0]});
    return {c.g.get(t, 0), c.g.get(t, 1), c.g.get(t, 2)};
  };
  A["add_layer_norm"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    if (!c.dout[0]) return {nullptr, nullptr, nullptr, nullptr};
    auto gm = arg_var(c.let.value, 2);
    const auto& at = c.let.value->call_attrs;
    std::vector<VarPtr> args{c.g.get(c.let.var, 1), gm, c.g.get(c.let.var, 2), c.g.get(c.let.var, 3), c.dout[0]};
    AttrMap la = pick(at, {"p", "seed", "salt"});
    if (c.let.var->ty.is_tuple() && c.let.var->ty.tuple().fields.size() > 4) {  // saved keep bits
      args.push_back(c.g.get(c.let.var, 4));
      la["mask_in"] = std::int64_t(1);
    }
    auto t = c.g.op("layer_norm_dx", args, la);
    VarPtr ds = c.g.get(t, 0);
    VarPtr dx = ir::attr_double(at, "p", 0.0) > 0.0 ? c.g.get(t, 3) : ds;
    return {dx, ds, c.g.get(t, 1), c.g.get(t, 2)};
  };
  A["embedding_sum"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    const size_t n = c.let.value->args.size() / 2;
    std::vector<VarPtr> g(2 * n, nullptr);
    if (!c.dout[0]) return g;
    for (size_t k = 0; k < n; ++k) {
      auto ids = arg_var(c.let.value, k), tab = arg_var(c.let.value, n + k);
      g[n + k] = c.g.op("embedding_dx", {ids, c.dout[0]}, {{"rows", tab->ty.tensor().shape[0]}});
    }
    return g;
  };
  A["embedding"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    auto ids = arg_var(c.let.value, 0), tab = arg_var(c.let.value, 1);
    return {nullptr, c.g.op("embedding_dx", {ids, c.dout[0]}, {{"rows", tab->ty.tensor().shape[0]}})};
  };
  // monolithic CE adjoint: dlogits is the op's second output; the
  // loss is the function's final output so d loss = 1.
  A["cross_entropy"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
    if (!c.let.var->ty.is_tuple()) throw NonDifferentiable("cross_entropy needs grad=1");
    return {c.g.get(c.let.var, 1), nullptr};
  };
}

/// dependency_report: per forward op, which forward tensors
/// its ADJOINT retains -- its inputs x (by argument position) and its output y
/// (for a tuple op: any field) -- read off the lets the adjoint emitted.
/// tanh keeps only y (NeedsY), matmul both inputs, add nothing (NeedsNeither).
struct DepEntry {
  int let = -1;              // forward let index
  std::string op;
  std::vector<int> inputs;   // argument positions the adjoint reads
  bool output = false;       // y (or a field of it) read by the adjoint
};

struct GradResult {
  VarPtr flat_grad;             // f32 [P] in leaf-offset order (null with make_flat=false)
  std::vector<std::pair<int64_t, VarPtr>> parts;  // (flat offset, f32 piece): leaf grads and zero gaps
  size_t n_forward = 0;         // lets before the backward
  std::vector<DepEntry> deps;   // dependency_report, forward order
};

/// Reverse-mode AD of `loss` w.r.t. the leaves (which must tile [0, P) of the
/// flat master buffer).  Appends the backward lets to `g` and returns the flat
/// gradient var.
inline GradResult autodiff(Graph& g, const VarPtr& loss, std::vector<Leaf> leaves, int64_t P,
                           bool make_flat = true) {
  register_default_adjoints();
  LetSeq fwd = g.seq();  // snapshot of the forward lets
  std::unordered_map<const ir::Var*, VarPtr> grad;
  std::map<std::pair<const ir::Var*, int>, VarPtr> tgrad;
  std::unordered_map<const ir::Var*, size_t> index;
  for (size_t i = 0; i < fwd.lets.size(); ++i) index[fwd.lets[i].var.get()] = i;

  auto accumulate = [&](const VarPtr& v, const VarPtr& d) {
    if (!d) return;
    auto it = grad.find(v.get());
    if (it == grad.end()) {
      grad[v.get()] = d;
    } else {
      VarPtr a = it->second, b = d;
      if (a->ty.tensor().dtype != b->ty.tensor().dtype)
        b = g.op("convert", {b}, {{"to", std::string(dtype_str(a->ty.tensor().dtype))}});
      it->second = g.op("add", {a, b});
    }
  };

  // seed: the loss must come from cross_entropy(grad=1) via tuple_get 0
  {
    auto it = index.find(loss.get());
    if (it == index.end()) throw Error("autodiff: loss is not a let of this graph");
    const auto& lb = fwd.lets[it->second];
    if (lb.value->kind != ExprKind::TupleGet)
      throw NonDifferentiable("autodiff: loss must be tuple_get(cross_entropy(..., grad=1), 0)");
    auto src = lb.value->args[0]->var;
    tgrad[{src.get(), 0}] = loss;  // placeholder: d loss = 1 (consumed by the CE adjoint)
  }

  std::vector<DepEntry> deps_rev;
  for (size_t ii = fwd.lets.size(); ii-- > 0;) {
    const LetBinding& lb = fwd.lets[ii];
    const ExprPtr& e = lb.value;
    if (e->kind == ExprKind::TupleGet) {
      auto it = grad.find(lb.var.get());
      if (it != grad.end()) {
        auto key = std::make_pair(e->args[0]->var.get(), e->index);
        auto jt = tgrad.find(key);
        if (jt == tgrad.end()) tgrad[key] = it->second;
        else jt->second = g.op("add", {jt->second, it->second});
      }
      continue;
    }
    if (e->kind != ExprKind::Call) continue;
    if (e->op == "view") continue;  // leaves: handled below
    std::vector<VarPtr> dout;
    bool any = false;
    if (lb.var->ty.is_tuple()) {
      for (size_t k = 0; k < lb.var->ty.tuple().fields.size(); ++k) {
        auto jt = tgrad.find({lb.var.get(), int(k)});
        dout.push_back(jt == tgrad.end() ? nullptr : jt->second);
        any = any || jt != tgrad.end();
      }
    } else {
      auto it = grad.find(lb.var.get());
      dout.push_back(it == grad.end() ? nullptr : it->second);
      any = it != grad.end();
    }
    if (!any) continue;
    auto rule = adjoints().find(e->op);
    if (rule == adjoints().end()) throw NonDifferentiable("no adjoint registered for op " + e->op);
    AdjointCtx ctx{g, lb, dout};
    const size_t mark = g.seq().lets.size();
    auto dins = rule->second(ctx);
    {  // dependency_report: what this adjoint's lets read from the forward
      DepEntry de;
      de.let = int(ii);
      de.op = e->op;
      std::set<const ir::Var*> read;
      for (size_t k = mark; k < g.seq().lets.size(); ++k)
        for (auto& a : g.seq().lets[k].value->args)
          if (a->kind == ExprKind::VarRef) read.insert(a->var.get());
      for (size_t k = 0; k < e->args.size(); ++k)
        if (e->args[k]->kind == ExprKind::VarRef && read.count(e->args[k]->var.get())) de.inputs.push_back(int(k));
      de.output = read.count(lb.var.get()) > 0;
      deps_rev.push_back(de);
    }
    for (size_t j = 0; j < dins.size() && j < e->args.size(); ++j) {
      auto av = arg_var(e, j);
      if (av && dins[j]) accumulate(av, dins[j]);
    }
  }

  // leaf gradients -> one flat f32 buffer in offset order
  std::sort(leaves.begin(), leaves.end(), [](const Leaf& a, const Leaf& b) { return a.offset < b.offset; });
  std::vector<VarPtr> parts;
  std::vector<std::pair<int64_t, VarPtr>> placed;
  int64_t pos = 0;
  auto zeros = [&](int64_t n) {
    return g.op("fill", {}, {{"shape", std::to_string(n)}, {"dtype", std::string("f32")}, {"value", 0.0}});
  };
  for (auto& lf : leaves) {
    if (lf.offset < pos) throw Error("autodiff: parameter leaves overlap");
    if (lf.offset > pos) {  // alignment gap
      parts.push_back(zeros(lf.offset - pos));
      placed.push_back({pos, parts.back()});
      pos = lf.offset;
    }
    auto it = grad.find(lf.view.get());
    if (it == grad.end()) throw NonDifferentiable("no gradient reaches parameter %" + lf.view->id);
    VarPtr d = it->second;
    if (d->ty.tensor().dtype != kF32) d = g.op("convert", {d}, {{"to", std::string("f32")}});
    if (numel(d->ty.tensor()) != lf.numel)
      throw Error("autodiff: gradient of %" + lf.view->id + " has " + std::to_string(numel(d->ty.tensor())) +
                  " elements, the parameter " + std::to_string(lf.numel));
    parts.push_back(d);
    placed.push_back({pos, d});
    pos += lf.numel;
  }
  if (pos > P) throw Error("autodiff: leaves exceed the flat buffer");
  if (pos < P) {
    parts.push_back(zeros(P - pos));
    placed.push_back({pos, parts.back()});
  }
  GradResult r;
  if (make_flat) r.flat_grad = g.op("concat", parts, {}, "grad");
  r.parts = std::move(placed);
  r.n_forward = fwd.lets.size();
  r.deps.assign(deps_rev.rbegin(), deps_rev.rend());
  return r;
}

/// materialization_set: the forward tensors a training
/// graph's backward reads -- the union of what the adjoints retained
/// (dependency_report): every forward op input they read and every output
/// (or output field) they read.  Empty for an inference-only graph.
inline std::set<const ir::Var*> materialization_set(const LetSeq& fwd, const GradResult& gr) {
  std::set<const ir::Var*> m;
  for (auto& d : gr.deps) {
    const auto& b = fwd.lets.at(size_t(d.let));
    for (int k : d.inputs)
      if (b.value->args.at(size_t(k))->kind == ExprKind::VarRef) m.insert(b.value->args[size_t(k)]->var.get());
    if (d.output) m.insert(b.var.get());
  }
  return m;
}

// ---------------------------------------------------------- rule fusion
/// Rule-based fusion: after the pattern rewrites,
/// maximal runs of consecutive Elemwise lets of one element count (inputs of
/// that size or [1] scalars, float) become one multi-output `ew_closure`
/// (SPEC.md:359-362): its inputs are the values the run reads from outside,
/// its outputs every member value used after the run -- so forward tensors the
/// backward needs (the materialization set) escape as outputs instead of
/// blocking fusion.  A consecutive run contracts to a node without creating a
/// cycle.  Groups are capped at 16 ops (and 8 inputs / 8 outputs); a run of
/// one op stays a bare op.  The closure's program rounds every member's result
/// to its dtype, so values are bit-identical to the unfused ops.
inline std::string base_name(const std::string& op);

struct RuleFuseStats {
  int closures = 0, fused_ops = 0;
};

inline bool rule_fusible_op(const std::string& base) {
  static const std::set<std::string> ops = {"add",  "sub",  "mul",  "div",  "tanh_dx", "gelu_dx", "neg",
                                            "tanh", "relu", "gtz",  "gelu", "convert", "cast",    "add_scalar"};
  return ops.count(base) > 0;
}

inline RuleFuseStats rule_fuse(LetSeq& s, int max_group = 16) {
  RuleFuseStats st;
  const int n = int(s.lets.size());
  auto is_fl = [](DType d) { return d == kF32 || d == kF16 || d == kBF16; };
  auto elig = [&](int i, int64_t& cnt) {
    const auto& b = s.lets[size_t(i)];
    if (b.value->kind != ExprKind::Call || !b.var->ty.is_tensor()) return false;
    if (!rule_fusible_op(base_name(b.value->op))) return false;
    const auto& o = b.var->ty.tensor();
    if (!is_fl(o.dtype)) return false;
    cnt = numel(o);
    for (auto& a : b.value->args) {
      if (a->kind != ExprKind::VarRef || !a->var->ty.is_tensor()) return false;
      const auto& t = a->var->ty.tensor();
      if (!is_fl(t.dtype) || (numel(t) != cnt && numel(t) != 1)) return false;
    }
    return true;
  };
  // uses after position i of each var (and returned vars)
  std::unordered_map<const ir::Var*, int> last_use;
  for (int i = 0; i < n; ++i)
    for (auto& a : s.lets[size_t(i)].value->args)
      if (a->kind == ExprKind::VarRef) last_use[a->var.get()] = i;
  std::set<const ir::Var*> returned;
  if (s.ret) {
    if (s.ret->kind == ExprKind::VarRef) returned.insert(s.ret->var.get());
    for (auto& a : s.ret->args)
      if (a->kind == ExprKind::VarRef) returned.insert(a->var.get());
  }
  LetSeq out;
  out.ret = s.ret;
  auto emit_group = [&](int g0, int g1) {  // lets [g0, g1)
    if (g1 - g0 < 2) {
      for (int i = g0; i < g1; ++i) out.lets.push_back(s.lets[size_t(i)]);
      return;
    }
    std::map<const ir::Var*, int> reg;
    std::vector<VarPtr> ins;
    std::set<const ir::Var*> members;
    for (int i = g0; i < g1; ++i) members.insert(s.lets[size_t(i)].var.get());
    for (int i = g0; i < g1; ++i)
      for (auto& a : s.lets[size_t(i)].value->args)
        if (!members.count(a->var.get()) && !reg.count(a->var.get())) {
          reg[a->var.get()] = int(ins.size());
          ins.push_back(a->var);
        }
    std::vector<int> outm;  // member indices used after the run
    for (int i = g0; i < g1; ++i) {
      const ir::Var* v = s.lets[size_t(i)].var.get();
      auto it = last_use.find(v);
      if (returned.count(v) || (it != last_use.end() && it->second >= g1)) outm.push_back(i);
    }
    if (ins.size() > 8 || outm.size() > 8 || outm.empty()) {
      for (int i = g0; i < g1; ++i) out.lets.push_back(s.lets[size_t(i)]);
      return;
    }
    std::string prog, outs, otypes;
    int next = int(ins.size());
    for (int i = g0; i < g1; ++i) {
      const auto& b = s.lets[size_t(i)];
      std::string base = base_name(b.value->op);
      const int ra = reg.at(b.value->args[0]->var.get());
      const int rb = b.value->args.size() > 1 ? reg.at(b.value->args[1]->var.get()) : ra;
      double imm = 0.0;
      if (base == "convert" || base == "cast") base = "copy";
      if (base == "add_scalar") imm = ir::attr_double(b.value->call_attrs, "value", 0.0);
      char buf[96];
      std::snprintf(buf, sizeof buf, "%s %d %d %d %d %.9g;", base.c_str(), next, ra, rb,
                    dtype_code(b.var->ty.tensor().dtype), imm);
      prog += buf;
      reg[b.var.get()] = next++;
    }
    for (size_t k = 0; k < outm.size(); ++k) {
      const auto& b = s.lets[size_t(outm[k])];
      outs += (k ? "," : "") + std::to_string(reg.at(b.var.get()));
      const auto& t = b.var->ty.tensor();
      otypes += (k ? ";" : "") + std::string(dtype_str(t.dtype)) + ":" + opreg::shape_attr(t.shape);
    }
    AttrMap at{{"prog", prog}, {"outs", outs}, {"otypes", otypes}};
    std::vector<ExprPtr> xs;
    std::vector<Type> tys;
    for (auto& v : ins) {
      xs.push_back(ir::var_ref(v));
      tys.push_back(v->ty);
    }
    auto call = ir::call("ew_closure", std::move(xs), at);
    call->ty = opreg::registry().type_rel_of("ew_closure")(tys, at);
    if (outm.size() == 1) {
      out.lets.push_back({s.lets[size_t(outm[0])].var, call});  // the member's var now names the closure
    } else {
      auto cv = ir::make_var(s.lets[size_t(g0)].var->id + "_clo", call->ty);
      out.lets.push_back({cv, call});
      for (size_t k = 0; k < outm.size(); ++k) {
        const auto& b = s.lets[size_t(outm[k])];
        auto g = ir::tuple_get(ir::var_ref(cv), int(k));
        g->ty = b.var->ty;
        out.lets.push_back({b.var, g});
      }
    }
    ++st.closures;
    st.fused_ops += g1 - g0;
  };
  int g0 = -1;
  int64_t gcnt = 0;
  for (int i = 0; i < n; ++i) {
    int64_t cnt = 0;
    const bool e = elig(i, cnt);
    if (g0 >= 0 && e && cnt == gcnt && i - g0 < max_group) continue;
    if (g0 >= 0) emit_group(g0, i);
    g0 = -1;
    if (e) {
      g0 = i;
      gcnt = cnt;
    } else {
      out.lets.push_back(s.lets[size_t(i)]);
    }
  }
  if (g0 >= 0) emit_group(g0, n);
  s = std::move(out);
  return st;
}

// -------------------------------------------------------------------- fusion

struct UseInfo {
  std::unordered_map<const ir::Var*, int> count;
  std::set<const ir::Var*> returned;
};

inline UseInfo count_uses(const LetSeq& s) {
  UseInfo u;
  for (auto& b : s.lets)
    for (auto& a : b.value->args)
      if (a->kind == ExprKind::VarRef) u.count[a->var.get()]++;
  if (s.ret)
    for (auto& a : s.ret->args)
      if (a->kind == ExprKind::VarRef) {
        u.count[a->var.get()]++;
        u.returned.insert(a->var.get());
      }
  return u;
}

struct FusionStats {
  int dact = 0, ln_dy2 = 0, emb_base = 0, ln_bias = 0, pairs = 0, ce_mask = 0, dead = 0, ln_drop = 0;
  std::map<std::string, int> by_pattern;  // matches per FusionPattern name
};

/// The b200 dialect's fusion patterns: a name, a
/// priority (applied in descending order where roots coincide), the root op
/// the rooted DAG template starts from, and the template.  Each rewrite lands
/// on a hand-written b200 fused kernel (the paper's "GEMM + activation"
/// library-pattern analog).  `disable_patterns` (model cfg key) switches
/// patterns off by name.
struct FusionPattern {
  const char* name;
  int priority;
  const char* root;
  const char* tmpl;
};
inline const std::vector<FusionPattern>& b200_patterns() {
  static const std::vector<FusionPattern> p = {
      {"b200.dgrad_gelu_epilogue", 30, "gelu_dx", "gelu_dx(u, matmul_t(a, b)) -> matmul_dact(a, b, u){act=gelu}"},
      {"b200.dgrad_saved_deriv_epilogue", 29, "mul", "mul(matmul_t(a, b), d) -> matmul_dact(a, b, d){act=deriv}"},
      {"b200.ln_post_dropout", 28, "dropout", "dropout(layer_norm(x, g, b).0) -> layer_norm{post_dropout}.0"},
      {"b200.ln_dx_in_dropout", 27, "layer_norm_dx", "layer_norm_dx(.., dropout(dy)) -> layer_norm_dx{in_p}(.., dy)"},
      {"b200.ln_dx_residual_dy2", 26, "layer_norm_dx", "layer_norm_dx(.., add(a, b)) -> layer_norm_dx(.., a, b)"},
      {"b200.ln_dx_bias_grad", 25, "colsum", "colsum(layer_norm_dx(..).k) -> layer_norm_dx{bias_grad}.last"},
      {"b200.ce_masked_colsum", 24, "colsum", "colsum(cross_entropy(x, l).1) -> colsum(dlogits, l){ignore_index}"},
      {"b200.tied_embedding_base", 23, "add", "add(embedding_dx(ids, dy), X) -> embedding_dx(ids, dy, X)"},
      {"b200.attention_saved_mask", 22, "attention_dx",
       "attention_dx(qkv, attention(qkv).1, dctx) -> attention{save_mask}, attention_dx(.., attention.2)"},
      {"b200.embedding_sum", 21, "add", "add(embedding(i, T) | embedding_sum(..), embedding(j, U)) -> embedding_sum(.., j, .., U)"},
      {"b200.dgrad_wgrad_pair", 20, "matmul_t", "matmul_t(dY, W) ~ matmul_t(X, dY){ta} -> matmul_pair"},
  };
  return p;
}

/// b200.attention_saved_mask: a bf16 attention forward with dropout (S <= 128,
/// head dim 64, stored P) whose backward regenerates the keep bits instead
/// stores them (save_mask: 4 i32 words per query row) and its attention_dx
/// reads them -- what the hand-built bf16 step asks for directly; AutoCast
/// output reaches it through this rewrite (the all-f32 model's attention keeps
/// no mask).  Same Philox bits either way, so the result is bit-identical.
inline int attach_attention_masks(LetSeq& s) {
  std::unordered_map<const ir::Var*, size_t> def;
  for (size_t i = 0; i < s.lets.size(); ++i) def[s.lets[i].var.get()] = i;
  const DType bf16 = dtype_from("bf16");
  std::map<size_t, VarPtr> mask_of;                 // attention let -> its mask var
  std::map<size_t, std::vector<LetBinding>> after;  // get-lets inserted after an attention
  int n = 0;
  for (size_t j = 0; j < s.lets.size(); ++j) {
    auto& bd = s.lets[j];
    if (bd.value->kind != ExprKind::Call || bd.value->op != "attention_dx" || bd.value->args.size() != 3 ||
        bd.value->call_attrs.count("save_mask") || bd.value->call_attrs.count("lse") ||
        bd.value->args[1]->kind != ExprKind::VarRef)
      continue;
    auto pit = def.find(bd.value->args[1]->var.get());
    if (pit == def.end()) continue;
    auto& gl = s.lets[pit->second];
    if (gl.value->kind != ExprKind::TupleGet || gl.value->index != 1 || gl.value->args[0]->kind != ExprKind::VarRef)
      continue;
    auto ait = def.find(gl.value->args[0]->var.get());
    if (ait == def.end()) continue;
    auto& al = s.lets[ait->second];
    if (al.value->kind != ExprKind::Call || al.value->op != "attention" || al.value->call_attrs.count("lse") ||
        al.value->args.size() != 1 || al.value->args[0]->kind != ExprKind::VarRef)
      continue;
    const AttrMap& at = al.value->call_attrs;
    const int64_t S = ir::attr_int(at, "seq", 0), A = ir::attr_int(at, "heads", 0);
    const TensorType q = al.value->args[0]->var->ty.tensor();
    if (ir::attr_double(at, "p", 0.0) <= 0.0 || S <= 0 || S > 128 || S % 8 || A <= 0 || q.dtype != bf16 ||
        q.shape.empty() || q.shape.back() != 3 * 64 * A)
      continue;
    VarPtr mv;
    auto mit = mask_of.find(ait->second);
    if (mit != mask_of.end()) {
      mv = mit->second;
    } else {
      if (at.count("save_mask")) continue;  // already storing bits, but not visible through a get: leave it
      AttrMap na = at;
      na["save_mask"] = std::int64_t(1);
      const Type nt = opreg::registry().type_rel_of("attention")({al.value->args[0]->var->ty}, na);
      al.value->call_attrs = na;
      al.value->ty = nt;
      al.var->ty = nt;
      const int k = int(nt.tuple().fields.size()) - 1;
      mv = ir::make_var(al.var->id + "_mask", Type(nt.tuple().fields[size_t(k)]));
      auto g = ir::tuple_get(ir::var_ref(al.var), k);
      g->ty = mv->ty;
      after[ait->second].push_back({mv, g});
      mask_of[ait->second] = mv;
    }
    bd.value->args.push_back(ir::var_ref(mv));
    bd.value->call_attrs["save_mask"] = std::int64_t(1);
    ++n;
  }
  if (!n) return 0;
  LetSeq out;
  out.ret = s.ret;
  for (size_t k = 0; k < s.lets.size(); ++k) {
    out.lets.push_back(s.lets[k]);
    auto it = after.find(k);
    if (it != after.end()) out.lets.insert(out.lets.end(), it->second.begin(), it->second.end());
  }
  s = std::move(out);
  return n;
}

/// Horizontal fusion (SPEC.md:533-540 applied to GEMMs): a weight-gradient
/// matmul_t and the nearest bf16 GEMM sharing an operand with it within
/// `window` lets (the linear's data gradient -- matmul_t or matmul_dact on the
/// same dY) become one matmul_pair: one persistent launch whose tiles fill the
/// SMs the small weight-gradient GEMM leaves idle.  The pair is placed at the
/// later member (every argument of both is defined by then); the earlier
/// member must have no use before that point.  Both become tuple_gets.
inline int fuse_gemm_pairs(LetSeq& s, int window = 6) {
  const int n = int(s.lets.size());
  auto is_gemm = [](const ExprPtr& e) {
    return e->kind == ExprKind::Call && (e->op == "matmul_t" || e->op == "matmul_dact");
  };
  const DType bf16 = dtype_from("bf16");
  auto bf16_operands = [&](const ExprPtr& e) {
    for (int k = 0; k < 2; ++k)
      if (e->args[k]->kind != ExprKind::VarRef || e->args[k]->var->ty.tensor().dtype != bf16) return false;
    return true;
  };
  auto uses = [&](int k, const ir::Var* v) {
    for (auto& a : s.lets[k].value->args)
      if (a->kind == ExprKind::VarRef && a->var.get() == v) return true;
    return false;
  };
  std::vector<char> used(n, 0), drop(n, 0);
  std::map<int, std::vector<LetBinding>> at_pos;  // replacement lets for position hi
  int n_pairs = 0;
  for (int j = 0; j < n; ++j) {
    auto& b2 = s.lets[j];
    if (used[j] || !is_gemm(b2.value) || b2.value->op != "matmul_t" || !bf16_operands(b2.value)) continue;
    if (ir::attr_string(b2.value->call_attrs, "out", "") != "f32") continue;  // weight gradients only
    for (int d = 1; d <= window; ++d) {
      int cand[2] = {j - d, j + d};
      int i = -1;
      for (int c : cand) {
        if (c < 0 || c >= n || used[c]) continue;
        auto& b1 = s.lets[c];
        if (!is_gemm(b1.value) || !bf16_operands(b1.value) || b1.var->ty.is_tuple()) continue;
        if (b1.value->op == "matmul_t" && ir::attr_string(b1.value->call_attrs, "out", "") == "f32") continue;
        bool share = false;
        for (auto& a2 : b2.value->args)
          for (auto& a1 : b1.value->args)
            if (a1->kind == ExprKind::VarRef && a2->kind == ExprKind::VarRef && a1->var == a2->var) share = true;
        if (!share) continue;
        const int lo = std::min(c, j), hi = std::max(c, j);
        bool free_between = true;
        for (int k = lo + 1; k <= hi && free_between; ++k)
          if (uses(k, s.lets[lo].var.get())) free_between = false;
        if (!free_between) continue;
        i = c;
        break;
      }
      if (i < 0) continue;
      auto& b1 = s.lets[i];
      AttrMap at;
      const auto& a1 = b1.value->call_attrs;
      const auto& a2 = b2.value->call_attrs;
      const bool dact = b1.value->op == "matmul_dact";
      at["n0"] = std::int64_t(dact ? 3 : 2);
      at["ta0"] = ir::attr_int(a1, "ta", 0);
      at["tb0"] = ir::attr_int(a1, "tb", 0);
      at["alpha0"] = ir::attr_double(a1, "alpha", 1.0);
      if (dact) at["act0"] = ir::attr_string(a1, "act", "none");
      if (a1.count("out")) at["out0"] = ir::attr_string(a1, "out", "");
      at["ta1"] = ir::attr_int(a2, "ta", 0);
      at["tb1"] = ir::attr_int(a2, "tb", 0);
      at["alpha1"] = ir::attr_double(a2, "alpha", 1.0);
      at["out1"] = ir::attr_string(a2, "out", "");
      std::vector<ExprPtr> args(b1.value->args.begin(), b1.value->args.end());
      args.insert(args.end(), b2.value->args.begin(), b2.value->args.end());
      auto call = ir::call("matmul_pair", args, at);
      TupleType tt{{b1.var->ty.tensor(), b2.var->ty.tensor()}};
      call->ty = tt;
      auto pv = ir::make_var(b1.var->id + "_pair", tt);
      auto g0 = ir::tuple_get(ir::var_ref(pv), 0);
      g0->ty = b1.var->ty;
      auto g1 = ir::tuple_get(ir::var_ref(pv), 1);
      g1->ty = b2.var->ty;
      const int lo = std::min(i, j), hi = std::max(i, j);
      at_pos[hi] = {LetBinding{pv, call}, LetBinding{b1.var, g0}, LetBinding{b2.var, g1}};
      drop[lo] = 1;
      used[i] = used[j] = 1;
      ++n_pairs;
      break;
    }
  }
  LetSeq out;
  out.ret = s.ret;
  for (int k = 0; k < n; ++k) {
    if (drop[k]) continue;
    auto it = at_pos.find(k);
    if (it == at_pos.end()) out.lets.push_back(s.lets[k]);
    else out.lets.insert(out.lets.end(), it->second.begin(), it->second.end());
  }
  s = std::move(out);
  return n_pairs;
}

/// Pattern fusion + dead-let elimination.  Each rewrite needs the absorbed
/// producer to have exactly one use (SPEC.md:381-388 materialization rule).
inline FusionStats fuse(LetSeq& s, bool patterns = true, const std::set<std::string>& disabled = {}) {
  FusionStats st;
  for (auto& fp : b200_patterns()) {
    if (!opreg::registry().has_base(fp.root)) throw RegistryError(std::string("pattern root op unknown: ") + fp.root);
    st.by_pattern[fp.name] = 0;
  }
  auto on = [&](const char* name) { return !disabled.count(name); };
  UseInfo u = count_uses(s);
  std::unordered_map<const ir::Var*, size_t> def;
  for (size_t i = 0; i < s.lets.size(); ++i) def[s.lets[i].var.get()] = i;
  std::set<size_t> removed;
  auto producer = [&](const VarPtr& v) -> LetBinding* {
    if (!v) return nullptr;
    auto it = def.find(v.get());
    if (it == def.end() || removed.count(it->second)) return nullptr;
    auto& b = s.lets[it->second];
    return b.value->kind == ExprKind::Call ? &b : nullptr;
  };
  auto single = [&](const VarPtr& v) { return u.count[v.get()] == 1 && !u.returned.count(v.get()); };

  for (size_t i = 0; patterns && i < s.lets.size(); ++i) {
    auto& b = s.lets[i];
    if (b.value->kind != ExprKind::Call) continue;
    const std::string op = b.value->op;
    // 0. add(embedding(i, T) | embedding_sum(ids.., tables..), embedding(j, U))
    //    -> embedding_sum(ids.., j, tables.., U): the gathers and the add chain
    //    in one kernel, each sum rounded to the tables' 16-bit dtype exactly as
    //    the chain rounds it (IEEE addition commutes, so either add operand
    //    order gives the same bits)
    if (op == "add" && on("b200.embedding_sum") && b.value->args.size() == 2) {
      auto a0 = arg_var(b.value, 0), a1 = arg_var(b.value, 1);
      auto* p0 = producer(a0);
      auto* p1 = producer(a1);
      auto is_emb = [](LetBinding* p) { return p && p->value->op == "embedding" && p->value->args.size() == 2; };
      auto is_sum = [](LetBinding* p) { return p && p->value->op == "embedding_sum"; };
      LetBinding *acc = nullptr, *one = nullptr;
      VarPtr va, vo;
      if ((is_emb(p0) || is_sum(p0)) && is_emb(p1)) acc = p0, one = p1, va = a0, vo = a1;
      else if (is_emb(p0) && is_sum(p1)) acc = p1, one = p0, va = a1, vo = a0;
      const DType ty = b.value->ty.tensor().dtype;
      if (acc && single(va) && single(vo) && (ty == dtype_from("bf16") || ty == dtype_from("f16")) &&
          acc->value->ty.tensor().dtype == ty && one->value->ty.tensor().dtype == ty &&
          !acc->value->call_attrs.size() && !one->value->call_attrs.size()) {
        std::vector<ExprPtr> ids, tabs;
        if (is_sum(acc)) {
          const size_t n = acc->value->args.size() / 2;
          for (size_t k = 0; k < n; ++k) ids.push_back(acc->value->args[k]), tabs.push_back(acc->value->args[n + k]);
        } else {
          ids.push_back(acc->value->args[0]);
          tabs.push_back(acc->value->args[1]);
        }
        ids.push_back(one->value->args[0]);
        tabs.push_back(one->value->args[1]);
        bool same = true;
        for (auto& t : tabs) same = same && t->ty.tensor().dtype == ty;
        if (same) {
          std::vector<ExprPtr> xs = ids;
          xs.insert(xs.end(), tabs.begin(), tabs.end());
          auto call = ir::call("embedding_sum", std::move(xs), AttrMap{});
          call->ty = b.value->ty;
          b.value = call;
          removed.insert(def[va.get()]);
          removed.insert(def[vo.get()]);
          ++st.by_pattern["b200.embedding_sum"];
          continue;
        }
      }
    }
    // 1. gelu_dx(u, matmul_t(a, b)) -> matmul_dact(a, b, u)   (dact in the dgrad epilogue)
    if (op == "gelu_dx" && on("b200.dgrad_gelu_epilogue")) {
      auto src = arg_var(b.value, 1);
      auto* p = producer(src);
      if (p && p->value->op == "matmul_t" && single(src) && ir::attr_double(p->value->call_attrs, "alpha", 1.0) == 1.0 &&
          !p->value->call_attrs.count("out")) {
        AttrMap at = pick(p->value->call_attrs, {"ta", "tb"});
        at["act"] = std::string("gelu");
        auto call = ir::call("matmul_dact", {p->value->args[0], p->value->args[1], b.value->args[0]}, at);
        call->ty = b.value->ty;
        b.value = call;
        removed.insert(def[src.get()]);
        ++st.dact;
        ++st.by_pattern["b200.dgrad_gelu_epilogue"];
        continue;
      }
    }
    // 1b. mul(matmul_t(a, b), d) with d = act'(u) saved by linear(save=grad)
    //     -> matmul_dact(a, b, d, act=deriv)   (same shape, no broadcast)
    if (op == "mul" && b.value->args.size() == 2 && on("b200.dgrad_saved_deriv_epilogue")) {
      bool done = false;
      for (int side = 0; side < 2 && !done; ++side) {
        auto src = arg_var(b.value, side), other = arg_var(b.value, 1 - side);
        auto* p = producer(src);
        if (!p || !other || p->value->op != "matmul_t" || !single(src) ||
            ir::attr_double(p->value->call_attrs, "alpha", 1.0) != 1.0 || p->value->call_attrs.count("out"))
          continue;
        if (src->ty.is_tuple() || other->ty.is_tuple() || b.var->ty.is_tuple()) continue;
        const auto &ts = src->ty.tensor(), &to = other->ty.tensor(), &tr = b.var->ty.tensor();
        if (ts.shape != to.shape || ts.dtype != to.dtype || tr.shape != ts.shape || tr.dtype != ts.dtype) continue;
        AttrMap at = pick(p->value->call_attrs, {"ta", "tb"});
        at["act"] = std::string("deriv");
        auto call = ir::call("matmul_dact", {p->value->args[0], p->value->args[1], b.value->args[1 - side]}, at);
        call->ty = b.value->ty;
        b.value = call;
        removed.insert(def[src.get()]);
        ++st.dact;
        ++st.by_pattern["b200.dgrad_saved_deriv_epilogue"];
        done = true;
      }
      if (done) continue;
    }
    // 6a. dropout(get(layer_norm(x, g, b), 0)) -> layer_norm {post_dropout} (16-bit):
    //     the LN kernel applies the output dropout (same roundings, one pass)
    if (op == "dropout" && b.value->args.size() == 1 && on("b200.ln_post_dropout")) {
      auto src = arg_var(b.value, 0);
      auto it = src ? def.find(src.get()) : def.end();
      if (it != def.end() && !removed.count(it->second) && s.lets[it->second].value->kind == ExprKind::TupleGet &&
          single(src) && s.lets[it->second].value->index == 0) {
        auto& gl = s.lets[it->second];
        auto tv = gl.value->args[0]->kind == ExprKind::VarRef ? gl.value->args[0]->var : nullptr;
        auto* lp = producer(tv);
        const auto& ty = b.var->ty;
        if (lp && lp->value->op == "layer_norm" && !lp->value->call_attrs.count("post_dropout") && !ty.is_tuple() &&
            (ty.tensor().dtype == kBF16 || ty.tensor().dtype == kF16) && ty.tensor().shape.back() % 8 == 0) {
          for (const char* k : {"p", "seed", "salt"})
            if (b.value->call_attrs.count(k)) lp->value->call_attrs[k] = b.value->call_attrs.at(k);
          lp->value->call_attrs["post_dropout"] = std::int64_t(1);
          auto e = ir::tuple_get(ir::var_ref(tv), 0);
          e->ty = b.value->ty;
          b.value = e;
          removed.insert(it->second);  // the old get is now unused
          ++st.ln_drop;
          ++st.by_pattern["b200.ln_post_dropout"];
          continue;
        }
      }
    }
    // 6b. layer_norm_dx(s, g, m, r, dropout(dy)) -> layer_norm_dx {in_p, in_seed, in_salt}
    if (op == "layer_norm_dx" && b.value->args.size() == 5 && !b.value->call_attrs.count("in_p") &&
        on("b200.ln_dx_in_dropout")) {
      auto src = arg_var(b.value, 4);
      auto* p = producer(src);
      const auto& ty = src ? src->ty : b.var->ty;
      if (p && p->value->op == "dropout" && single(src) && !ty.is_tuple() &&
          (ty.tensor().dtype == kBF16 || ty.tensor().dtype == kF16) && ty.tensor().shape.back() % 8 == 0) {
        AttrMap at = b.value->call_attrs;
        at["in_p"] = ir::attr_double(p->value->call_attrs, "p", 0.0);
        at["in_seed"] = ir::attr_int(p->value->call_attrs, "seed", 0);
        at["in_salt"] = ir::attr_int(p->value->call_attrs, "salt", 0);
        auto call = ir::call("layer_norm_dx", {b.value->args[0], b.value->args[1], b.value->args[2],
                                               b.value->args[3], p->value->args[0]}, at);
        call->ty = b.value->ty;
        b.value = call;
        removed.insert(def[src.get()]);
        ++st.ln_drop;
        ++st.by_pattern["b200.ln_dx_in_dropout"];
        continue;
      }
    }
    // 2. layer_norm_dx(s, g, m, r, add(a, b)) -> layer_norm_dx(s, g, m, r, a, b)
    const size_t lnm = op == "layer_norm_dx" && ir::attr_int(b.value->call_attrs, "mask_in", 0) ? 1 : 0;
    if (op == "layer_norm_dx" && b.value->args.size() == 5 + lnm && on("b200.ln_dx_residual_dy2")) {
      auto src = arg_var(b.value, 4);
      auto* p = producer(src);
      if (p && p->value->op == "add" && single(src)) {
        auto a = arg_var(p->value, 0), c = arg_var(p->value, 1);
        if (a && c && a->ty == src->ty && c->ty == src->ty) {
          std::vector<ExprPtr> nargs{b.value->args[0], b.value->args[1], b.value->args[2], b.value->args[3],
                                     p->value->args[0], p->value->args[1]};
          if (lnm) nargs.push_back(b.value->args[5]);  // the mask stays last
          auto call = ir::call("layer_norm_dx", nargs, b.value->call_attrs);
          call->ty = b.value->ty;
          b.value = call;
          removed.insert(def[src.get()]);
          ++st.ln_dy2;
          ++st.by_pattern["b200.ln_dx_residual_dy2"];
          continue;
        }
      }
    }
    // 4. colsum(get(layer_norm_dx(...), k)), k = the gradient leaving the
    //    LayerNorm (dx when p > 0, else ds) -> an extra f32 [H] output of
    //    layer_norm_dx (attr bias_grad): the bias gradient of the linear that
    //    fed the LayerNorm, summed in the same row order, with no extra pass
    if (op == "colsum" && on("b200.ln_dx_bias_grad")) {
      auto src = arg_var(b.value, 0);
      auto it = src ? def.find(src.get()) : def.end();
      if (it != def.end() && !removed.count(it->second) && s.lets[it->second].value->kind == ExprKind::TupleGet) {
        auto& gl = s.lets[it->second];
        auto tv = gl.value->args[0]->kind == ExprKind::VarRef ? gl.value->args[0]->var : nullptr;
        auto* lp = producer(tv);
        if (lp && lp->value->op == "layer_norm_dx" && !lp->value->call_attrs.count("bias_grad")) {
          const bool has_dx = ir::attr_double(lp->value->call_attrs, "p", 0.0) > 0.0;
          if (gl.value->index == (has_dx ? 3 : 0)) {
            lp->value->call_attrs["bias_grad"] = std::int64_t(1);
            TupleType tt = lp->var->ty.tuple();
            tt.fields.push_back(b.value->ty.tensor());
            lp->var->ty = tt;
            lp->value->ty = tt;
            auto e = ir::tuple_get(ir::var_ref(lp->var), int(tt.fields.size()) - 1);
            e->ty = b.value->ty;
            b.value = e;
            ++st.ln_bias;
            ++st.by_pattern["b200.ln_dx_bias_grad"];
            continue;
          }
        }
      }
    }
    // 5. colsum(get(cross_entropy(logits, labels), 1)) -> colsum(dlogits, labels):
    //    rows with label == ignore_index are exact zeros of dlogits, skip them
    if (op == "colsum" && b.value->args.size() == 1 && on("b200.ce_masked_colsum")) {
      auto src = arg_var(b.value, 0);
      auto it = src ? def.find(src.get()) : def.end();
      if (it != def.end() && s.lets[it->second].value->kind == ExprKind::TupleGet &&
          s.lets[it->second].value->index == 1) {
        auto& gl = s.lets[it->second];
        auto tv = gl.value->args[0]->kind == ExprKind::VarRef ? gl.value->args[0]->var : nullptr;
        auto* cp = producer(tv);
        if (cp && cp->value->op == "cross_entropy" && cp->value->args.size() == 2) {
          AttrMap at = b.value->call_attrs;
          at["ignore_index"] = ir::attr_int(cp->value->call_attrs, "ignore_index", -100);
          auto call = ir::call("colsum", {b.value->args[0], cp->value->args[1]}, at);
          call->ty = b.value->ty;
          b.value = call;
          ++st.ce_mask;
          ++st.by_pattern["b200.ce_masked_colsum"];
          continue;
        }
      }
    }
    // 3. add(embedding_dx(ids, dy), X) -> embedding_dx(ids, dy, X)  (tied embeddings)
    if (op == "add" && on("b200.tied_embedding_base")) {
      for (int side = 0; side < 2; ++side) {
        auto src = arg_var(b.value, side), other = arg_var(b.value, 1 - side);
        auto* p = producer(src);
        if (p && other && p->value->op == "embedding_dx" && p->value->args.size() == 2 && single(src) &&
            other->ty == src->ty) {
          auto call = ir::call("embedding_dx", {p->value->args[0], p->value->args[1], b.value->args[1 - side]},
                               p->value->call_attrs);
          call->ty = b.value->ty;
          b.value = call;
          removed.insert(def[src.get()]);
          ++st.emb_base;
          ++st.by_pattern["b200.tied_embedding_base"];
          break;
        }
      }
    }
  }
  LetSeq out;
  for (size_t i = 0; i < s.lets.size(); ++i)
    if (!removed.count(i)) out.lets.push_back(s.lets[i]);
  out.ret = s.ret;
  // dead-let elimination (everything here is pure except collectives/shard)
  bool changed = true;
  while (changed) {
    changed = false;
    UseInfo uu = count_uses(out);
    LetSeq keep;
    keep.ret = out.ret;
    for (auto& b : out.lets) {
      bool pure = b.value->kind != ExprKind::Call || opreg::registry().base_of(b.value->op).pure;
      if (pure && uu.count[b.var.get()] == 0) {
        ++st.dead;
        changed = true;
        continue;
      }
      keep.lets.push_back(b);
    }
    out = std::move(keep);
  }
  s = std::move(out);
  if (patterns && on("b200.attention_saved_mask"))
    st.by_pattern["b200.attention_saved_mask"] = attach_attention_masks(s);
  if (patterns && on("b200.dgrad_wgrad_pair")) st.pairs = fuse_gemm_pairs(s);
  st.by_pattern["b200.dgrad_wgrad_pair"] = st.pairs;
  return st;
}

/// dispatch_pass (opreg.hpp:740-766) works on Dataflow form; this applies the
/// same OpRegistry::resolve decision in place on ANF so the execution order
/// chosen by memsched is untouched.
inline void dispatch_anf(LetSeq& s, const opreg::DispatchConfig& cfg) {
  for (auto& b : s.lets) {
    if (b.value->kind != ExprKind::Call || b.value->op.find('.') != std::string::npos) continue;
    try {
      b.value->op = opreg::registry().resolve(b.value->op, cfg).full_name();
    } catch (const UnimplementedOp& e) {
      std::string shapes;
      for (auto& a : b.value->args) shapes += (shapes.empty() ? "" : ", ") + (a->var ? type_str(a->var->ty) : "?");
      throw UnimplementedOp(std::string(e.what()) + " (inputs: " + shapes + ")");
    }
  }
}

inline std::string base_name(const std::string& op) {
  auto d = op.find('.');
  return d == std::string::npos ? op : op.substr(d + 1);
}

}  // namespace tb
