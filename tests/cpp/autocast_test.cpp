// autocast_test.cpp -- CPU checks of the AutoCast pass (host/autocast.hpp)
// against the SPEC.md:296-326 examples and invariants.  Built and run by
// tests/test_autocast.py (needs the reference headers; no device).
#include <cstdio>
#include <cstdlib>
#include <string>

#include "autocast.hpp"
#include "models.hpp"

using namespace tb;

static int fails = 0;
#define CHECK(c, ...)                                   \
  do {                                                  \
    if (!(c)) {                                         \
      std::printf("FAIL %s:%d %s: ", __FILE__, __LINE__, #c); \
      std::printf(__VA_ARGS__);                         \
      std::printf("\n");                                \
      ++fails;                                          \
    }                                                   \
  } while (0)

static TensorType f32(std::vector<int64_t> s) { return TensorType{kF32, s}; }

static int count_op(const ir::FunctionIR& fn, const std::string& base) {
  int n = 0;
  for (auto& b : ir::flatten(fn).lets)
    if (b.value->kind == ExprKind::Call && base_name(b.value->op) == base) ++n;
  return n;
}

static DType ret_dtype(const ir::FunctionIR& fn, size_t i) {
  return ir::flatten(fn).ret->args.at(i)->var->ty.tensor().dtype;
}

int main() {
  ensure_registered({});
  const auto pol = default_policy();

  {  // single matmul(x, w) -> cast(x), cast(w), matmul in bf16
    Graph g("mm");
    auto x = g.param("x", f32({4, 8}));
    auto w = g.param("w", f32({8, 16}));
    auto y = g.op("matmul", {x, w});
    auto fn = g.finish({y});
    CastReport r;
    auto out = autocast(*fn, pol, &r);
    CHECK(r.casts == 2 && r.sites == 2, "casts %d sites %d", r.casts, r.sites);
    CHECK(count_op(*out, "convert") == 2, "converts %d", count_op(*out, "convert"));
    CHECK(ret_dtype(*out, 0) == kBF16, "matmul output not bf16");
    CHECK(fn->params[0]->ty.tensor().dtype == kF32, "params must stay f32");
    CHECK(ret_dtype(*fn, 0) == kF32, "input function modified");
    std::printf("single_matmul casts=%d\n", r.casts);
  }
  {  // all-F32 policy -> identity (zero casts)
    Graph g("mlp");
    auto x = g.param("x", f32({4, 8}));
    auto w = g.param("w", f32({8, 8}));
    auto h = g.op("relu", {g.op("matmul", {x, w})});
    auto l = g.op("mean", {h});
    auto fn = g.finish({l});
    CastReport r;
    auto out = autocast(*fn, all_f32_policy(), &r);
    CHECK(r.casts == 0 && r.sites == 0, "casts %d", r.casts);
    CHECK(ir::flatten(*out).lets.size() == ir::flatten(*fn).lets.size(), "let count changed");
    std::printf("all_f32 casts=%d\n", r.casts);
  }
  {  // softmax after a bf16 matmul: cast-up before the F32 op
    Graph g("sm");
    auto x = g.param("x", f32({4, 8}));
    auto w = g.param("w", f32({8, 16}));
    auto s = g.op("softmax", {g.op("matmul", {x, w})});
    auto fn = g.finish({s});
    CastReport r;
    auto out = autocast(*fn, pol, &r);
    CHECK(r.f32_violations == 0, "violations %d", r.f32_violations);
    CHECK(ret_dtype(*out, 0) == kF32, "softmax output not f32");
    CHECK(r.casts == 3, "casts %d", r.casts);
    std::printf("softmax casts=%d\n", r.casts);
  }
  // Fig. 3 topology: one producer whose value two consumers need in another dtype
  auto fig3 = [&](bool fusable, Placement pl, CastReport* r) {
    Graph g("fig3");
    auto x = g.param("x", f32({4, 8}));
    auto w = g.param("w", f32({8, 8}));
    auto b = g.param("b", f32({4, 8}));
    VarPtr c1, c2;
    if (fusable) {  // bf16 producer, two elementwise consumers computing in f32
      auto p = g.op("matmul", {x, w});
      c1 = g.op("add", {p, b});
      c2 = g.op("mul", {p, b});
    } else {  // f32 producer, two GEMM (opaque) consumers computing in bf16
      auto p = g.op("add", {x, b});
      c1 = g.op("matmul", {p, w});
      c2 = g.op("matmul", {p, w});
    }
    return autocast(*g.finish({c1, c2}), pol, r, pl);
  };
  {
    CastReport a, s;
    fig3(true, Placement::Auto, &a);
    fig3(true, Placement::AllShared, &s);
    // the producer's value feeds two fusable consumers: 2 exclusive casts, all in closures
    CHECK(a.exclusive == 2 && a.standalone_casts == 0, "excl %d standalone %d", a.exclusive, a.standalone_casts);
    CHECK(s.shared >= 1 && s.standalone_casts >= 1, "shared placement standalone %d", s.standalone_casts);
    CHECK(a.standalone_casts <= s.standalone_casts, "minimality bound");
    std::printf("fig3_fusable exclusive=%d standalone=%d shared_placement_standalone=%d\n", a.exclusive,
                a.standalone_casts, s.standalone_casts);
    CastReport o;
    fig3(false, Placement::Auto, &o);
    // opaque consumers: exactly one shared cast of the producer (x, w casts aside)
    CHECK(o.exclusive == 0, "exclusive %d", o.exclusive);
    std::printf("fig3_opaque shared=%d casts=%d standalone=%d\n", o.shared, o.casts, o.standalone_casts);
  }
  {  // policy missing an op -> error
    Graph g("m");
    auto x = g.param("x", f32({4, 8}));
    auto fn = g.finish({g.op("tanh", {x})});
    PrecisionPolicy p = pol;
    p.by_op.erase("tanh");
    bool threw = false;
    try {
      autocast(*fn, p);
    } catch (const Error& e) {
      threw = std::string(e.what()).find("no entry for op 'tanh'") != std::string::npos;
    }
    CHECK(threw, "missing-op policy accepted");
  }
  {  // cast round trip: bf16(f32(v)) == bf16(v) for bf16-representable v
    for (uint32_t h = 0; h < 65536; h += 7) {
      uint32_t u = h << 16;
      float f;
      std::memcpy(&f, &u, 4);
      if (f != f) continue;
      CHECK(bf16_bits(f) == uint16_t(h), "bf16 round trip %u", h);
    }
  }
  for (const char* cfg : {"kind=bert;L=2;H=128;A=2;F=512;V=1024;S=128;B=8;dtype=f32;opt=adam",
                          "kind=bert;L=2;H=128;A=2;F=512;V=1024;S=128;B=8;dtype=f32;opt=sgd"}) {
    // the whole f32 training step (forward + autodiff backward + optimizer)
    auto ts = build_train_step(parse_cfg(cfg));
    CastReport r;
    auto out = autocast(*ts.fn, pol, &r);
    CHECK(r.f32_violations == 0, "violations %d", r.f32_violations);
    CHECK(r.low_ops > 0 && r.casts > 0, "low %d casts %d", r.low_ops, r.casts);
    // master weights and optimizer state stay f32; the optimizer reads f32 only
    for (auto& p : out->params)
      if (p->id == "params" || p->id == "m" || p->id == "v") CHECK(p->ty.tensor().dtype == kF32, "%s", p->id.c_str());
    for (auto& b : ir::flatten(*out).lets) {
      if (b.value->kind != ExprKind::Call) continue;
      const std::string base = base_name(b.value->op);
      if (base == "sgd_update" || base == "adam_update" || base == "adam_update_ex")
        for (auto& a : b.value->args)
          if (is_float(a->var->ty.tensor().dtype)) CHECK(a->var->ty.tensor().dtype == kF32, "optimizer input");
      if (base == "linear" || base == "matmul_t" || base == "batch_matmul" || base == "attention")
        for (auto& a : b.value->args)
          if (is_float(a->var->ty.tensor().dtype)) CHECK(a->var->ty.tensor().dtype == kBF16, "%s input", base.c_str());
    }
    std::printf("train_step %s default_policy lets=%zu low_ops=%d sites=%d casts=%d exclusive=%d shared=%d "
                "param_casts=%d standalone=%d\n",
                parse_cfg(cfg).opt.c_str(), ir::flatten(*out).lets.size(), r.low_ops, r.sites, r.casts, r.exclusive,
                r.shared, r.param_casts, r.standalone_casts);
    // the b200 policy: normalisation/softmax/loss kernels widen bf16 on load
    CastReport rb;
    auto outb = autocast(*ts.fn, b200_policy(), &rb);
    CHECK(rb.f32_violations == 0, "b200 violations %d", rb.f32_violations);
    CHECK(rb.casts < r.casts, "b200 policy should need fewer casts (%d vs %d)", rb.casts, r.casts);
    std::printf("train_step %s b200_policy low_ops=%d sites=%d casts=%d exclusive=%d shared=%d param_casts=%d "
                "standalone=%d\n",
                parse_cfg(cfg).opt.c_str(), rb.low_ops, rb.sites, rb.casts, rb.exclusive, rb.shared, rb.param_casts,
                rb.standalone_casts);
  }
  std::printf(fails ? "FAILED %d\n" : "OK\n", fails);
  return fails ? 1 : 0;
}
