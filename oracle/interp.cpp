// interp.cpp -- the reference ANF interpreter, "the universal oracle"
// (SPEC.md:636), over the CPU restatement of exec_base (oracle.c).
// TEST INFRASTRUCTURE: loaded only by tests/, smoke() and bench.py's CPU legs.
//
// It builds the SAME training-step graph as the product (paper_2303_04759_b200/
// host/models.hpp: forward + autodiff + fusion, un-dispatched) and evaluates it
// let by let with host tensors -- f32 storage, half types rounded after every
// op -- so a whole-step GPU result can be compared against it on identical
// inputs, parameters and dropout masks.
#include <cstring>
#include <memory>

#include "models.hpp"
#include "oracle.h"

namespace {

using namespace tb;

struct HVal {
  std::vector<std::shared_ptr<std::vector<uint32_t>>> fields;  // 4-byte slots: f32 bits or i32
  std::vector<TensorType> types;
};

thread_local std::string g_err;

struct Interp {
  TrainStep ts;
  std::vector<std::shared_ptr<std::vector<uint32_t>>> state;  // one per fn param
  double last_loss = 0;
};

orc_tensor odesc(std::vector<uint32_t>& buf, const TensorType& t) {
  orc_tensor d{};
  d.ptr = buf.data();
  d.dtype = dtype_code(t.dtype);
  d.rank = t.rank();
  for (int i = 0; i < t.rank(); ++i) d.shape[i] = t.shape[i];
  return d;
}

std::vector<orc_attr> oattrs(const AttrMap& m, std::vector<std::string>& keep) {
  keep.reserve(2 * m.size() + 2);
  std::vector<orc_attr> out;
  for (auto& [k, v] : m) {
    orc_attr a{};
    keep.push_back(k);
    a.key = keep.back().c_str();
    if (auto* i = std::get_if<std::int64_t>(&v)) {
      a.kind = 0;
      a.i = *i;
    } else if (auto* d = std::get_if<double>(&v)) {
      a.kind = 1;
      a.d = *d;
    } else {
      a.kind = 2;
      keep.push_back(std::get<std::string>(v));
      a.s = keep.back().c_str();
    }
    out.push_back(a);
  }
  return out;
}

void run_step(Interp& I) {
  const ir::FunctionIR& fn = *I.ts.fn;
  auto seq = ir::flatten(fn);
  std::unordered_map<const ir::Var*, HVal> env;
  for (size_t p = 0; p < fn.params.size(); ++p)
    env[fn.params[p].get()] = HVal{{I.state[p]}, {fn.params[p]->ty.tensor()}};
  for (auto& b : seq.lets) {
    const auto& e = b.value;
    if (e->kind == ExprKind::TupleGet) {
      const HVal& t = env.at(e->args[0]->var.get());
      env[b.var.get()] = HVal{{t.fields.at(e->index)}, {t.types.at(e->index)}};
      continue;
    }
    std::vector<TensorType> otys;
    if (b.var->ty.is_tuple()) otys = b.var->ty.tuple().fields;
    else otys = {b.var->ty.tensor()};
    HVal out;
    for (auto& t : otys) {
      out.fields.push_back(std::make_shared<std::vector<uint32_t>>(size_t(numel(t)), 0u));
      out.types.push_back(t);
    }
    std::vector<orc_tensor> ins, outs;
    for (auto& a : e->args) {
      HVal& v = env.at(a->var.get());
      ins.push_back(odesc(*v.fields[0], v.types[0]));
    }
    for (size_t k = 0; k < otys.size(); ++k) outs.push_back(odesc(*out.fields[k], otys[k]));
    std::vector<std::string> keep;
    auto at = oattrs(e->call_attrs, keep);
    const std::string base = base_name(e->op);
    if (orc_exec(base.c_str(), ins.data(), int(ins.size()), outs.data(), int(outs.size()), at.data(),
                 int(at.size())) != 0)
      throw Error("oracle " + base + ": " + orc_last_error());
    env[b.var.get()] = std::move(out);
  }
  // returns -> state bindings; loss
  const HVal& loss = env.at(seq.ret->args.at(0)->var.get());
  float lv;
  std::memcpy(&lv, loss.fields[0]->data(), 4);
  I.last_loss = lv;
  for (auto& [rj, pi] : I.ts.state_binding) {
    const HVal& v = env.at(seq.ret->args.at(rj)->var.get());
    *I.state[pi] = *v.fields[0];
  }
}

}  // namespace

extern "C" {

const char* orc_interp_last_error(void) { return g_err.c_str(); }

/// Same cfg string as tb_session_create (model keys only).
void* orc_interp_create(const char* cfg) {
  try {
    ensure_registered({});
    auto I = std::make_unique<Interp>();
    I->ts = build_train_step(parse_cfg(cfg ? cfg : ""));
    const auto& ps = I->ts.fn->params;
    for (auto& p : ps) I->state.push_back(std::make_shared<std::vector<uint32_t>>(size_t(numel(p->ty.tensor())), 0u));
    // params / half copy from the shared initialiser; m, v, step = 0
    std::vector<float> p = init_params(I->ts);
    std::memcpy(I->state[I->ts.i_params]->data(), p.data(), p.size() * 4);
    if (I->ts.i_p16 >= 0)
      for (size_t i = 0; i < p.size(); ++i) {
        float q = orc_quantize_bf16(p[i]);
        std::memcpy(&(*I->state[I->ts.i_p16])[i], &q, 4);
      }
    const int64_t T = I->ts.cfg.T();
    for (int64_t t = 0; t < T; ++t) (*I->state[I->ts.i_pos])[t] = uint32_t(t % I->ts.cfg.S);
    return I.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void orc_interp_destroy(void* h) { delete static_cast<Interp*>(h); }

int orc_interp_step(void* h, const int32_t* ids, const int32_t* labels, float* loss) {
  try {
    auto* I = static_cast<Interp*>(h);
    const int64_t T = I->ts.cfg.T();
    std::memcpy(I->state[I->ts.i_ids]->data(), ids, size_t(T) * 4);
    std::memcpy(I->state[I->ts.i_labels]->data(), labels, size_t(T) * 4);
    run_step(*I);
    *loss = float(I->last_loss);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

/// copy function parameter `name` (f32 slots / i32) to host
int orc_interp_read(void* h, const char* name, void* dst, int64_t nelem) {
  auto* I = static_cast<Interp*>(h);
  const auto& ps = I->ts.fn->params;
  for (size_t i = 0; i < ps.size(); ++i)
    if (ps[i]->id == name) {
      int64_t n = std::min<int64_t>(nelem, int64_t(I->state[i]->size()));
      std::memcpy(dst, I->state[i]->data(), size_t(n) * 4);
      return 0;
    }
  g_err = std::string("no parameter ") + name;
  return 1;
}

}  // extern "C"
