#include <sstream>
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

#include "memsched.hpp"
#include "pipeline.hpp"
#include "oracle.h"

namespace {

using namespace tb;

struct HVal {
  std::vector<std::shared_ptr<std::vector<uint32_t>>> fields;  // 4-byte slots: f32 bits or i32
  std::vector<TensorType> types;
};

thread_local std::string g_err;
// the dropout step of the step being interpreted (rng_step state after its
// increment), or -1 for a graph without dropout
thread_local int64_t g_rng_step = -1;

struct Interp {
  TrainStep ts;
  std::vector<std::shared_ptr<std::vector<uint32_t>>> state;  // one per fn param
  double last_loss = 0;
  std::vector<uint32_t> last_grad;  // the optimizer's gradient input of the last step (f32 slots)
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

using Env = std::unordered_map<const ir::Var*, HVal>;

// kind: 0 reduce_scatter (sum), 1 all_gather, 2 allreduce (sum); f32 slots
using CollFn = int (*)(int kind, const float* in, int64_t in_n, float* out, int64_t out_n, int world, int rank);

bool is_collective(const std::string& base) {
  return base == "reduce_scatter" || base == "all_gather" || base == "allreduce";
}
int coll_kind(const std::string& base) { return base == "reduce_scatter" ? 0 : base == "all_gather" ? 1 : 2; }

Env init_env(const Interp& I) {
  Env env;
  const ir::FunctionIR& fn = *I.ts.fn;
  for (size_t p = 0; p < fn.params.size(); ++p)
    env[fn.params[p].get()] = HVal{{I.state[p]}, {fn.params[p]->ty.tensor()}};
  return env;
}

HVal alloc_out(const ir::LetBinding& b) {
  std::vector<TensorType> otys;
  if (b.var->ty.is_tuple()) otys = b.var->ty.tuple().fields;
  else otys = {b.var->ty.tensor()};
  HVal out;
  for (auto& t : otys) {
    out.fields.push_back(std::make_shared<std::vector<uint32_t>>(size_t(numel(t)), 0u));
    out.types.push_back(t);
  }
  return out;
}

// one let on one rank (everything except collectives with world > 1)
void exec_let(Env& env, const ir::LetBinding& b) {
  const auto& e = b.value;
  if (e->kind == ExprKind::TupleGet) {
    const HVal& t = env.at(e->args[0]->var.get());
    env[b.var.get()] = HVal{{t.fields.at(e->index)}, {t.types.at(e->index)}};
    return;
  }
  HVal out = alloc_out(b);
  std::vector<orc_tensor> ins, outs;
  for (auto& a : e->args) {
    HVal& v = env.at(a->var.get());
    ins.push_back(odesc(*v.fields[0], v.types[0]));
  }
  for (size_t k = 0; k < out.fields.size(); ++k) outs.push_back(odesc(*out.fields[k], out.types[k]));
  std::vector<std::string> keep;
  AttrMap am = e->call_attrs;
  if (g_rng_step >= 0) am["rng_step"] = std::int64_t(g_rng_step);  // Philox counter word 3
  auto at = oattrs(am, keep);
  const std::string base = base_name(e->op);
  if (orc_exec(base.c_str(), ins.data(), int(ins.size()), outs.data(), int(outs.size()), at.data(),
               int(at.size())) != 0)
    throw Error("oracle " + base + ": " + orc_last_error());
  env[b.var.get()] = std::move(out);
}

void finish_step(Interp& I, Env& env, const ir::LetSeq& seq) {
  const HVal& loss = env.at(seq.ret->args.at(0)->var.get());
  float lv;
  std::memcpy(&lv, loss.fields[0]->data(), 4);
  I.last_loss = lv;
  for (auto& [rj, pi] : I.ts.state_binding) {
    const HVal& v = env.at(seq.ret->args.at(rj)->var.get());
    *I.state[pi] = *v.fields[0];
  }
}

/// single rank; collectives with world > 1 go through `coll` (e.g. gloo from
/// Python) -- without it the oracle refuses them like exec_base does.
int64_t next_rng_step(const Interp& I) {
  if (I.ts.i_rng < 0) return -1;
  float v;
  std::memcpy(&v, I.state[size_t(I.ts.i_rng)]->data(), 4);
  return int64_t(v + 1.0f);  // the step's add_scalar(rng_step, 1)
}

void run_step(Interp& I, CollFn coll = nullptr, int rank = 0) {
  auto seq = ir::flatten(*I.ts.fn);
  Env env = init_env(I);
  g_rng_step = next_rng_step(I);
  for (auto& b : seq.lets) {
    const auto& e = b.value;
    if (e->kind == ExprKind::Call && is_collective(base_name(e->op)) &&
        ir::attr_int(e->call_attrs, "world", 1) > 1 && coll) {
      HVal out = alloc_out(b);
      HVal& in = env.at(e->args[0]->var.get());
      const int world = int(ir::attr_int(e->call_attrs, "world", 1));
      if (coll(coll_kind(base_name(e->op)), reinterpret_cast<const float*>(in.fields[0]->data()),
               int64_t(in.fields[0]->size()), reinterpret_cast<float*>(out.fields[0]->data()),
               int64_t(out.fields[0]->size()), world, rank))
        throw ProtocolError("collective callback failed at %" + b.var->id);
      env[b.var.get()] = std::move(out);
      continue;
    }
    if (e->kind == ExprKind::Call) {
      const std::string base = base_name(e->op);
      if (base == "sgd_update" || base == "adam_update" || base == "adam_update_ex")
        I.last_grad = *env.at(e->args.at(1)->var.get()).fields[0];
    }
    exec_let(env, b);
  }
  finish_step(I, env, seq);
}

/// The deterministic in-process bus: ranks execute the same
/// let sequence in lockstep; a collective is a barrier where the bus reduces in
/// fixed rank order 0..n-1 (so the simulation is bit-reproducible); a
/// mismatched op across ranks raises ProtocolError.
void run_world_step(std::vector<Interp>& R) {
  const int N = int(R.size());
  g_rng_step = next_rng_step(R[0]);
  auto seq = ir::flatten(*R[0].ts.fn);
  std::vector<ir::LetSeq> seqs;
  for (auto& I : R) seqs.push_back(ir::flatten(*I.ts.fn));
  std::vector<Env> env;
  for (auto& I : R) env.push_back(init_env(I));
  for (size_t li = 0; li < seq.lets.size(); ++li) {
    const auto& b = seq.lets[li];
    const auto& e = b.value;
    for (int r = 1; r < N; ++r) {
      const auto& br = seqs[r].lets.at(li);
      if (br.value->kind != e->kind || br.value->op != e->op)
        throw ProtocolError("bus: rank " + std::to_string(r) + " issued a different op at let " + std::to_string(li));
    }
    if (e->kind == ExprKind::Call && is_collective(base_name(e->op))) {
      const std::string base = base_name(e->op);
      // every rank built its own graph: look each rank's vars up in its own let
      std::vector<const float*> in(N);
      for (int r = 0; r < N; ++r)
        in[r] = reinterpret_cast<const float*>(
            env[r].at(seqs[r].lets[li].value->args[0]->var.get()).fields[0]->data());
      const int64_t in_n = int64_t(env[0].at(e->args[0]->var.get()).fields[0]->size());
      for (int r = 0; r < N; ++r) {
        HVal out = alloc_out(seqs[r].lets[li]);
        float* o = reinterpret_cast<float*>(out.fields[0]->data());
        const int64_t out_n = int64_t(out.fields[0]->size());
        if (base == "reduce_scatter") {  // shard r of the rank-ordered sum (zero padded)
          for (int64_t k = 0; k < out_n; ++k) {
            const int64_t g = int64_t(r) * out_n + k;
            float acc = 0.0f;
            for (int q = 0; q < N; ++q) acc += g < in_n ? in[q][g] : 0.0f;
            o[k] = acc;
          }
        } else if (base == "all_gather") {  // concat of shards, truncated
          for (int64_t k = 0; k < out_n; ++k) o[k] = in[k / in_n][k % in_n];
        } else {  // allreduce
          for (int64_t k = 0; k < out_n; ++k) {
            float acc = 0.0f;
            for (int q = 0; q < N; ++q) acc += in[q][k];
            o[k] = acc;
          }
        }
        env[r][seqs[r].lets[li].var.get()] = std::move(out);
      }
      continue;
    }
    for (int r = 0; r < N; ++r) exec_let(env[r], seqs[r].lets[li]);
  }
  for (int r = 0; r < N; ++r) finish_step(R[r], env[r], seqs[r]);
}

std::unique_ptr<Interp> make_interp(const std::string& cfg, int rank) {
  ensure_registered({});
  auto I = std::make_unique<Interp>();
  // optional "autocast=<policy>" key: interpret the AutoCast'd f32 step
  std::string model, amp, kv;
  int64_t budget = 0;
  int sched = 0, remat_chain = 1;
  std::istringstream is(cfg);
  while (std::getline(is, kv, ';')) {
    if (kv.rfind("autocast=", 0) == 0) amp = kv.substr(9);
    else if (kv.rfind("budget=", 0) == 0) budget = std::stoll(kv.substr(7));
    else if (kv.rfind("schedule=", 0) == 0) sched = std::stoi(kv.substr(9));
    else if (kv.rfind("remat_chain=", 0) == 0) remat_chain = std::stoi(kv.substr(12));
    else if (!kv.empty()) model += kv + ";";
  }
  I->ts = build_train_step(parse_cfg(model));
  if (!amp.empty()) apply_autocast(I->ts, amp);  // same parser and phases as the session
  finalize_graph(I->ts);  // rule-based fusion, as the session does
  // the memsched phases in the session's order (capi.cpp prepare): the
  // interpreter then executes the scheduled / rematerialised let sequence
  if (sched) I->ts.fn = ir::make_fn(I->ts.fn->name, I->ts.fn->params, schedule(*I->ts.fn, I->ts.state_binding));
  if (budget > 0) I->ts.fn = rematerialize(*I->ts.fn, budget, I->ts.state_binding, false, remat_chain != 0).first;
  const auto& ps = I->ts.fn->params;
  for (auto& p : ps) I->state.push_back(std::make_shared<std::vector<uint32_t>>(size_t(numel(p->ty.tensor())), 0u));
  // params (this rank's shard under ZeRO) / half copy from the shared
  // initialiser; m, v, step = 0
  std::vector<float> p = shard_of(I->ts, init_params(I->ts), rank);  // ZeRO: slice `rank` of every bucket
  if (int64_t(p.size()) != int64_t(I->state[I->ts.i_params]->size())) throw Error("interp: shard size mismatch");
  std::memcpy(I->state[I->ts.i_params]->data(), p.data(), p.size() * 4);
  if (I->ts.i_p16 >= 0) {
    const DType cd = I->ts.fn->params[I->ts.i_p16]->ty.tensor().dtype;
    for (size_t i = 0; i < p.size(); ++i) {
      float q = cd == kBF16 ? orc_quantize_bf16(p[i]) : cd == kF16 ? orc_quantize_f16(p[i]) : p[i];
      std::memcpy(&(*I->state[I->ts.i_p16])[i], &q, 4);
    }
  }
  const int64_t T = I->ts.cfg.T();
  for (int64_t t = 0; t < T; ++t) (*I->state[I->ts.i_pos])[t] = uint32_t(t % I->ts.cfg.S);
  return I;
}

}  // namespace

extern "C" {

const char* orc_interp_last_error(void) { return g_err.c_str(); }

/// Same cfg string as tb_session_create (model keys only).
void* orc_interp_create(const char* cfg) {
  try {
    return make_interp(cfg ? cfg : "", 0).release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

/// one rank of a world (cfg carries world=N): params = shard `rank`
void* orc_interp_create_rank(const char* cfg, int rank) {
  try {
    return make_interp(cfg ? cfg : "", rank).release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void orc_interp_destroy(void* h) { delete static_cast<Interp*>(h); }

/// coll: optional collective callback for world > 1 (NULL: refuse, as exec_base)
int orc_interp_step_coll(void* h, const int32_t* ids, const int32_t* labels, float* loss, CollFn coll, int rank) {
  try {
    auto* I = static_cast<Interp*>(h);
    const int64_t T = I->ts.cfg.T();
    std::memcpy(I->state[I->ts.i_ids]->data(), ids, size_t(T) * 4);
    std::memcpy(I->state[I->ts.i_labels]->data(), labels, size_t(T) * 4);
    run_step(*I, coll, rank);
    *loss = float(I->last_loss);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

int orc_interp_step(void* h, const int32_t* ids, const int32_t* labels, float* loss) {
  return orc_interp_step_coll(h, ids, labels, loss, nullptr, 0);
}

/// lockstep world of N ranks on the in-process bus
struct WorldH {
  std::vector<Interp> ranks;
};

void* orc_world_create(const char* cfg, int n) {
  try {
    auto w = std::make_unique<WorldH>();
    for (int r = 0; r < n; ++r) w->ranks.push_back(std::move(*make_interp(cfg ? cfg : "", r)));
    return w.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void orc_world_destroy(void* h) { delete static_cast<WorldH*>(h); }

/// ids/labels: N consecutive per-rank batches of T tokens; losses: N floats
int orc_world_step(void* h, const int32_t* ids, const int32_t* labels, float* losses) {
  try {
    auto* w = static_cast<WorldH*>(h);
    const int64_t T = w->ranks[0].ts.cfg.T();
    for (size_t r = 0; r < w->ranks.size(); ++r) {
      auto& I = w->ranks[r];
      std::memcpy(I.state[I.ts.i_ids]->data(), ids + r * T, size_t(T) * 4);
      std::memcpy(I.state[I.ts.i_labels]->data(), labels + r * T, size_t(T) * 4);
    }
    run_world_step(w->ranks);
    for (size_t r = 0; r < w->ranks.size(); ++r) losses[r] = float(w->ranks[r].last_loss);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}

void* orc_world_rank(void* h, int r) { return &static_cast<WorldH*>(h)->ranks.at(size_t(r)); }

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

/// overwrite function parameter `name` (f32 slots / i32) from host memory
int orc_interp_write(void* h, const char* name, const void* src, int64_t nelem) {
  auto* I = static_cast<Interp*>(h);
  const auto& ps = I->ts.fn->params;
  for (size_t i = 0; i < ps.size(); ++i)
    if (ps[i]->id == name) {
      if (nelem != int64_t(I->state[i]->size())) {
        g_err = std::string("write ") + name + ": size mismatch";
        return 1;
      }
      std::memcpy(I->state[i]->data(), src, size_t(nelem) * 4);
      return 0;
    }
  g_err = std::string("no parameter ") + name;
  return 1;
}

/// the flat gradient the optimizer consumed in the last step (before any
/// ZeRO grad_scale), f32; returns its element count when dst is NULL
int64_t orc_interp_read_grad(void* h, float* dst, int64_t nelem) {
  auto* I = static_cast<Interp*>(h);
  const int64_t n = int64_t(I->last_grad.size());
  if (dst) std::memcpy(dst, I->last_grad.data(), size_t(std::min(n, nelem)) * 4);
  return n;
}

}  // extern "C"
