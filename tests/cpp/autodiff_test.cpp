// autodiff_test.cpp -- CPU checks of the autodiff pass (host/graph.hpp) against
// dependency_report's known answers (tanh -> {y}, matmul ->
// both inputs, add -> {}), the fan-out accumulation chain, the memory property
// of NeedsY vs NeedsBoth (liveness of tanh's input), and determinism (two
// autodiff runs print byte-identical text).  Built and run by
// tests/test_autodiff.py (needs the reference headers; no device).
#include <cstdio>
#include <string>

#include "memsched.hpp"
#include "text_ext.hpp"

using namespace tb;

static int fails = 0;
#define CHECK(c, ...)                                            \
  do {                                                           \
    if (!(c)) {                                                  \
      std::printf("FAIL %s:%d %s: ", __FILE__, __LINE__, #c);    \
      std::printf(__VA_ARGS__);                                  \
      std::printf("\n");                                         \
      ++fails;                                                   \
    }                                                            \
  } while (0)

struct Built {
  FunctionPtr fn;
  size_t n_forward = 0;
  std::vector<DepEntry> deps;
  std::string u;  // id of tanh's input
};

// MLP step: u = x W1; t = tanh(u); [fan-out: y = add(t, t)]; logits = y W2;
// (loss, dlogits) = cross_entropy(logits, labels); flat gradient of [W1 | W2].
static Built build_mlp(bool fan_out) {
  const int64_t B = 4, D = 8, C = 16;
  Graph g;
  auto x = g.param("x", TensorType{kF32, {B, D}});
  auto labels = g.param("labels", TensorType{kI32, {B}});
  auto params = g.param("params", TensorType{kF32, {D * D + D * C}});
  auto w1 = g.op("view", {params}, {{"offset", std::int64_t(0)}, {"shape", std::string("8,8")}}, "w");
  auto w2 = g.op("view", {params}, {{"offset", D * D}, {"shape", std::string("8,16")}}, "w");
  auto u = g.op("matmul", {x, w1}, {}, "u");
  auto t = g.op("tanh", {u}, {}, "t");
  auto y = fan_out ? g.op("add", {t, t}, {}, "y") : t;
  auto logits = g.op("matmul", {y, w2}, {}, "logits");
  auto ce = g.op("cross_entropy", {logits, labels}, {{"classes", C}, {"grad", std::int64_t(1)}});
  auto loss = g.get(ce, 0, "loss");
  Built r;
  GradResult gr = autodiff(g, loss, {{w1, 0, D * D}, {w2, D * D, D * C}}, D * D + D * C);
  r.n_forward = gr.n_forward;
  r.deps = gr.deps;
  r.u = u->id;
  r.fn = g.finish({loss, gr.flat_grad});
  return r;
}

static const DepEntry* find(const Built& b, const std::string& op, int nth = 0) {
  for (auto& e : b.deps)
    if (e.op == op && nth-- == 0) return &e;
  return nullptr;
}

static int last_use_of(const ir::FunctionIR& fn, const std::string& id) {
  auto seq = ir::flatten(fn);
  int last = -1;
  for (size_t i = 0; i < seq.lets.size(); ++i)
    for (auto& a : seq.lets[i].value->args)
      if (a->kind == ExprKind::VarRef && a->var->id == id) last = int(i);
  return last;
}

int main() {
  ensure_registered({});

  // --- dependency_report known answers
  Built b = build_mlp(false);
  const DepEntry* th = find(b, "tanh");
  CHECK(th && th->inputs.empty() && th->output, "tanh must retain only y");
  const DepEntry* mm = find(b, "matmul", 0);
  CHECK(mm && mm->inputs.size() == 2 && mm->inputs[0] == 0 && mm->inputs[1] == 1,
        "matmul must retain both inputs");
  Built bf = build_mlp(true);
  const DepEntry* ad = find(bf, "add");
  CHECK(ad && ad->inputs.empty(), "add must retain nothing (NeedsNeither)");

  // --- fan-out: t feeds add twice; its gradient is one `add` of
  // the two incoming contributions (deterministic reverse order), then tanh_dx
  {
    auto seq = ir::flatten(*bf.fn);
    int adds_bwd = 0, tdx = 0;
    for (size_t i = bf.n_forward; i < seq.lets.size(); ++i) {
      const auto& e = seq.lets[i].value;
      if (e->kind != ExprKind::Call) continue;
      if (e->op == "add") ++adds_bwd;
      if (e->op == "tanh_dx") {
        ++tdx;
        // its dy argument is the accumulated add of the fan-out contributions
        const auto& dy = e->args.at(1)->var;
        bool from_add = false;
        for (size_t k = bf.n_forward; k < i; ++k)
          if (seq.lets[k].var.get() == dy.get() && seq.lets[k].value->op == "add") from_add = true;
        CHECK(from_add, "tanh_dx must consume the accumulated fan-out gradient");
      }
    }
    CHECK(adds_bwd == 1 && tdx == 1, "fan-out: %d backward adds, %d tanh_dx", adds_bwd, tdx);
  }

  // --- memory property: NeedsY keeps tanh's input u out of
  // the backward; a NeedsBoth adjoint (dx = dy * (1 - tanh(x)^2) recomputed
  // from x) extends u's liveness into the backward.
  {
    const int last_y = last_use_of(*b.fn, b.u);
    auto saved = adjoints()["tanh"];
    adjoints()["tanh"] = [](AdjointCtx& c) -> std::vector<VarPtr> {
      auto x = arg_var(c.let.value, 0);
      auto t = c.g.op("tanh", {x});
      return {c.g.op("tanh_dx", {t, c.dout[0]})};
    };
    Built both = build_mlp(false);
    adjoints()["tanh"] = saved;
    const int last_both = last_use_of(*both.fn, both.u);
    CHECK(last_y < int(b.n_forward), "NeedsY: u must die in the forward (last use %d, forward %zu)", last_y,
          b.n_forward);
    CHECK(last_both >= int(both.n_forward), "NeedsBoth: u must live into the backward (%d)", last_both);
    CHECK(last_y < last_both, "liveness of u must shrink: %d vs %d", last_y, last_both);
    // and so does the planner's peak
    auto p_y = peak_memory(*b.fn), p_both = peak_memory(*both.fn);
    CHECK(p_y.peak <= p_both.peak, "peak %lld vs %lld", (long long)p_y.peak, (long long)p_both.peak);
  }

  // --- materialization_set: tanh's y is in it (NeedsY), its
  // input u is not; it is exactly the forward tensors the backward lets read;
  // an inference-only graph has none
  {
    const int64_t B = 4, D = 8, C = 16;
    Graph g;
    auto x = g.param("x", TensorType{kF32, {B, D}});
    auto labels = g.param("labels", TensorType{kI32, {B}});
    auto params = g.param("params", TensorType{kF32, {D * D + D * C}});
    auto w1 = g.op("view", {params}, {{"offset", std::int64_t(0)}, {"shape", std::string("8,8")}}, "w");
    auto w2 = g.op("view", {params}, {{"offset", D * D}, {"shape", std::string("8,16")}}, "w");
    auto u = g.op("matmul", {x, w1}, {}, "u");
    auto t = g.op("tanh", {u}, {}, "t");
    auto logits = g.op("matmul", {t, w2}, {}, "logits");
    auto ce = g.op("cross_entropy", {logits, labels}, {{"classes", C}, {"grad", std::int64_t(1)}});
    auto loss = g.get(ce, 0, "loss");
    LetSeq fwd = g.seq();
    GradResult gr = autodiff(g, loss, {{w1, 0, D * D}, {w2, D * D, D * C}}, D * D + D * C);
    auto ms = materialization_set(fwd, gr);
    CHECK(ms.count(t.get()) && !ms.count(u.get()), "tanh: y materialized, x not");
    CHECK(ms.count(x.get()) && ms.count(w1.get()) && ms.count(w2.get()), "matmul inputs materialized");
    // dynamic check: exactly the forward vars the backward lets reference
    std::set<const ir::Var*> fwdv, read;
    for (auto& b : fwd.lets) fwdv.insert(b.var.get());
    for (auto& p : {x, labels, params}) fwdv.insert(p.get());
    auto all = g.seq();
    for (size_t i = fwd.lets.size(); i < all.lets.size(); ++i)
      for (auto& a : all.lets[i].value->args)
        if (a->kind == ExprKind::VarRef && fwdv.count(a->var.get())) read.insert(a->var.get());
    for (auto* v : ms) CHECK(read.count(v), "materialized var %s is read by the backward", v->id.c_str());
    GradResult none;
    CHECK(materialization_set(fwd, none).empty(), "inference-only graph: empty set");
  }

  // --- determinism: two runs, byte-identical text
  {
    std::string t1 = print_text_ext(*build_mlp(true).fn), t2 = print_text_ext(*build_mlp(true).fn);
    CHECK(t1 == t2, "autodiff text differs between runs");
  }

  if (fails) {
    std::printf("%d failures\n", fails);
    return 1;
  }
  std::printf("autodiff spec examples OK\n");
  return 0;
}
