// capi.cpp -- libtrainc_b200.so: the C entry points of the b200 training-step
// runtime (graph build -> autodiff -> fusion -> memsched -> dispatch -> device
// VM), used by bench.py / tests / __graft_entry__ through ctypes.  This is the
// host side "above the C ABI": C++ over the reference's IR/registry, calling
// libtcb200.so for every kernel.
#include <chrono>
#include <cstring>
#include <memory>
#include <sstream>

#include "distpar.hpp"
#include "pipeline.hpp"
#include "text_ext.hpp"
#include "tnsr.hpp"
#include "trainc_b200.h"
#include "vm.hpp"

namespace tb {

static thread_local std::string g_err;

struct Session {
  ModelCfg cfg;
  TrainStep ts;
  FunctionPtr fn;  // dispatched, scheduled (and rematerialised) step
  DeviceVM vm;
  void* stream = nullptr;
  int device = 0;
  int rank = 0;
  int32_t* h_ids = nullptr;  // pinned staging
  int32_t* h_labels = nullptr;
  float* h_loss = nullptr;
  RematPlan remat;
  int64_t budget = 0;
  double compile_ms = 0;
  std::string text;
};

static std::string print_fn(const ir::FunctionIR& fn) {
  std::ostringstream os;
  os << "fn " << fn.name << "(";
  for (size_t i = 0; i < fn.params.size(); ++i)
    os << (i ? ", " : "") << "%" << fn.params[i]->id << ": " << type_str(fn.params[i]->ty);
  os << ") {\n";
  auto seq = ir::flatten(fn);
  for (auto& b : seq.lets) {
    os << "  let %" << b.var->id << " = ";
    if (b.value->kind == ExprKind::TupleGet) {
      os << "%" << b.value->args[0]->var->id << "." << b.value->index;
    } else {
      os << b.value->op << "(";
      for (size_t i = 0; i < b.value->args.size(); ++i)
        os << (i ? ", " : "") << "%" << b.value->args[i]->var->id;
      os << ")";
      if (!b.value->call_attrs.empty()) {
        os << " @{";
        bool first = true;
        for (auto& [k, v] : b.value->call_attrs) {
          os << (first ? "" : ", ") << k << "=";
          first = false;
          if (auto* i = std::get_if<std::int64_t>(&v)) os << *i;
          else if (auto* d = std::get_if<double>(&v)) os << *d;
          else os << std::get<std::string>(v);
        }
        os << "}";
      }
    }
    os << " : " << type_str(b.var->ty) << ";\n";
  }
  os << "  (";
  if (seq.ret)
    for (size_t i = 0; i < seq.ret->args.size(); ++i) os << (i ? ", " : "") << "%" << seq.ret->args[i]->var->id;
  os << ")\n}\n";
  return os.str();
}

}  // namespace tb

using namespace tb;

#define TB_TRY(...)                          \
  try {                                      \
    __VA_ARGS__;                             \
    return 0;                                \
  } catch (const std::exception& e) {        \
    g_err = e.what();                        \
    return 1;                                \
  }

extern "C" {

const char* tb_last_error(void) { return g_err.c_str(); }

/// cfg: "kind=bert;L=12;H=768;..." plus optional runtime keys
///   budget=<bytes>  rematerialise the step under this memory budget
///   schedule=1      p-c list scheduling
///   rank=<r>        ZeRO rank (with world=<n>)
// graph pipeline shared by the device session and the CPU-only inspection
// entry points: build -> autodiff/fusion -> [schedule] -> [remat] -> dispatch
static void prepare(Session& s, const char* cfg_c) {
  ensure_registered(split_ws(tcb_supported_ops()));
  std::string model, all = cfg_c ? cfg_c : "";
  std::istringstream is(all);
  std::string kv;
  int do_schedule = 0;
  int remat_chain = 1;  // remat: depth-2 chains through tuple producers (memsched.hpp)
  std::string amp;
  while (std::getline(is, kv, ';')) {
    if (kv.rfind("budget=", 0) == 0) s.budget = std::stoll(kv.substr(7));
    else if (kv.rfind("schedule=", 0) == 0) do_schedule = std::stoi(kv.substr(9));
    else if (kv.rfind("autocast=", 0) == 0) amp = kv.substr(9);
    else if (kv.rfind("remat_chain=", 0) == 0) remat_chain = std::stoi(kv.substr(12));
    else if (kv.rfind("rank=", 0) == 0) s.rank = std::stoi(kv.substr(5));
    else if (!kv.empty()) model += kv + ";";
  }
  s.cfg = parse_cfg(model);
  s.ts = build_train_step(s.cfg);
  FunctionPtr fn = s.ts.fn;
  if (!amp.empty()) {  // graph-generation pass: AutoCast the all-f32 step (SPEC.md:721 phase order)
    apply_autocast(s.ts, amp);
    fn = s.ts.fn;
  }
  s.ts.fn = fn;
  finalize_graph(s.ts);  // rule-based fusion (ew_closure)
  fn = s.ts.fn;
  if (do_schedule) fn = ir::make_fn(fn->name, fn->params, schedule(*fn, s.ts.state_binding));
  // ZeRO: overlap_schedule -- every collective starts as soon
  // as its bucket exists (the VM runs them on its comm stream)
  if (s.cfg.zero_on()) fn = ir::make_fn(fn->name, fn->params, hoist_collectives(ir::flatten(*fn)));
  if (s.budget > 0) {
    auto [rf, plan] = rematerialize(*fn, s.budget, s.ts.state_binding, false, remat_chain != 0);
    fn = rf;
    s.remat = plan;
  }
  // dispatch (opreg.hpp:740-766 semantics) to the b200 dialect on "cuda"
  LetSeq seq = ir::flatten(*fn);
  opreg::DispatchConfig dc;
  dc.device = "cuda";
  dc.enabled_dialects = {"b200"};
  dispatch_anf(seq, dc);
  s.fn = ir::make_fn(fn->name, fn->params, seq);
}

/// CPU-only: build the step graph and its memory plan without a device.
/// out: P, P_pad, lets, planner_peak, arena_plan_bytes, state_bytes, fused_dact,
/// fused_ln_dy2, fused_emb, dead, remat_replays, peak_before_remat, peak_after_remat,
/// fused_ln_bias, fused_pairs
int tb_graph_info(const char* cfg, int64_t* out, int n) {
  TB_TRY({
    Session s;
    prepare(s, cfg);
    Layout L = build_layout(*s.fn, s.ts.state_binding);
    MemProfile mp = peak_memory(L);
    ArenaPlan ap = plan_arena(L);
    int64_t v[] = {s.ts.P, s.ts.P_pad, L.n, mp.peak, ap.size, mp.state_bytes, s.ts.fusion.dact, s.ts.fusion.ln_dy2,
                   s.ts.fusion.emb_base, s.ts.fusion.dead, s.remat.replays, s.remat.peak_before, s.remat.peak_after,
                   s.ts.fusion.ln_bias, s.ts.fusion.pairs};
    for (int i = 0; i < n && i < int(sizeof v / sizeof v[0]); ++i) out[i] = v[i];
  });
}

static thread_local std::string g_text;
const char* tb_graph_text(const char* cfg, const char* what) {
  try {
    Session s;
    prepare(s, cfg);
    std::string w = what ? what : "";
    if (w == "mem") {
      auto mp = peak_memory(build_layout(*s.fn, s.ts.state_binding));
      std::ostringstream os;
      os << "index,live_bytes\n";
      for (size_t i = 0; i < mp.curve.size(); ++i) os << i << "," << mp.curve[i] << "\n";
      g_text = os.str();
    } else if (w == "remat") {  // the remat plan of cfg (needs budget=): one split per line
      std::ostringstream os;
      os << "replays " << s.remat.replays << "\npeak_before " << s.remat.peak_before << "\npeak_after "
         << s.remat.peak_after << "\n";
      for (auto& sp : s.remat.splits)
        os << "split " << sp.victim << " " << sp.evict_index << " " << sp.replay_before << "\n";
      g_text = os.str();
    } else if (w == "fusion") {  // pattern census: "name priority root matches"
      std::ostringstream os;
      for (auto& fp : b200_patterns())
        os << fp.name << " " << fp.priority << " " << fp.root << " " << s.ts.fusion.by_pattern[fp.name] << "\n";
      os << "rule.ew_closure 0 - " << s.ts.rule_closures << "\n";
      g_text = os.str();
    } else if (w == "buckets") {  // ZeRO buckets: "offset numel shard" per line
      std::ostringstream os;
      for (auto [o, n] : s.ts.buckets) os << o << " " << n << " " << (n + s.cfg.world - 1) / s.cfg.world << "\n";
      g_text = os.str();
    } else if (w == "timeline") {  // two-stream cost simulation of the step (distpar.hpp)
      Timeline t = timeline(ir::flatten(*s.fn));
      std::ostringstream os;
      os << "serial " << t.serial << "\noverlap " << t.overlap << "\nevents " << t.events << "\ncollectives "
         << t.collectives << "\n";
      g_text = os.str();
    } else if (w == "segments") {  // flat parameter layout: "name offset numel" per line
      std::ostringstream os;
      for (auto& g : s.ts.segs) os << g.name << " " << g.offset << " " << g.numel << "\n";
      g_text = os.str();
    } else if (w == "text") {
      g_text = print_text_ext(*s.fn);  // the reference's text IR (text.hpp) + bf16/i32 tokens
    } else {
      g_text = print_fn(*s.fn);
    }
  } catch (const std::exception& e) {
    g_err = e.what();
    g_text.clear();
  }
  return g_text.c_str();
}

void* tb_session_create(const char* cfg_c, int device) {
  try {
    auto t0 = std::chrono::steady_clock::now();
    auto s = std::make_unique<Session>();
    s->device = device;
    prepare(*s, cfg_c);
    s->vm.set_device(device);
    s->vm.set_world(int(s->cfg.world));
    s->vm.compile(s->fn, s->ts.state_binding);
    tcb_check(tcb_stream_create(&s->stream), "stream");
    const int64_t T = s->cfg.T();
    tcb_check(tcb_host_alloc(reinterpret_cast<void**>(&s->h_ids), uint64_t(T) * 4), "pinned");
    tcb_check(tcb_host_alloc(reinterpret_cast<void**>(&s->h_labels), uint64_t(T) * 4), "pinned");
    tcb_check(tcb_host_alloc(reinterpret_cast<void**>(&s->h_loss), 64), "pinned");
    // constant inputs: position ids (t mod S) and token types (0)
    std::vector<int32_t> pos(static_cast<size_t>(T)), typ(static_cast<size_t>(T), 0);
    for (int64_t t = 0; t < T; ++t) pos[size_t(t)] = int32_t(t % s->cfg.S);
    tcb_check(tcb_memcpy(s->vm.param_ptr(s->ts.i_pos), pos.data(), uint64_t(T) * 4, 0, nullptr), "pos");
    if (s->ts.i_type >= 0)
      tcb_check(tcb_memcpy(s->vm.param_ptr(s->ts.i_type), typ.data(), uint64_t(T) * 4, 0, nullptr), "type");
    tcb_check(tcb_device_sync(), "sync");
    s->compile_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    return s.release();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void tb_session_destroy(void* h) {
  auto* s = static_cast<Session*>(h);
  if (!s) return;
  if (s->stream) tcb_stream_destroy(s->stream);
  if (s->h_ids) tcb_host_free(s->h_ids);
  if (s->h_labels) tcb_host_free(s->h_labels);
  if (s->h_loss) tcb_host_free(s->h_loss);
  delete s;
}

/// out[0..]: P, P_pad, T, arena_bytes, state_bytes, planner_peak, instructions,
/// kernels_per_step, lets, fused_dact, fused_ln_dy2, fused_emb, dead, remat_replays,
/// peak_before_remat, compile_us, shard
int tb_session_info(void* h, int64_t* out, int n) {
  TB_TRY({
    auto* s = static_cast<Session*>(h);
    const auto& st = s->vm.stats();
    int64_t v[] = {s->ts.P, s->ts.P_pad, s->cfg.T(), st.arena_bytes, st.state_bytes, st.planner_peak,
                   st.instructions, st.kernels, st.lets, s->ts.fusion.dact, s->ts.fusion.ln_dy2,
                   s->ts.fusion.emb_base, s->ts.fusion.dead, s->remat.replays, s->remat.peak_before,
                   int64_t(s->compile_ms * 1000), s->ts.shard()};
    for (int i = 0; i < n && i < int(sizeof v / sizeof v[0]); ++i) out[i] = v[i];
  });
}

int tb_session_init_params(void* h) {
  TB_TRY({
    auto* s = static_cast<Session*>(h);
    // the rank's ZeRO shard (slice `rank` of every bucket), or all of it
    std::vector<float> p = shard_of(s->ts, init_params(s->ts), s->rank);
    const int64_t sh = int64_t(p.size());
    tcb_check(tcb_memcpy(s->vm.param_ptr(s->ts.i_params), p.data(), uint64_t(sh) * 4, 0, nullptr), "params");
    if (s->ts.i_p16 >= 0) {
      const DType cd = s->ts.fn->params[s->ts.i_p16]->ty.tensor().dtype;
      if (cd == kF32) {
        tcb_check(tcb_memcpy(s->vm.param_ptr(s->ts.i_p16), p.data(), uint64_t(p.size()) * 4, 0, nullptr), "pcopy");
      } else {
        if (cd != kBF16) throw Error("init_params: unsupported compute-copy dtype");
        std::vector<uint16_t> h16(p.size());
        for (size_t i = 0; i < p.size(); ++i) h16[i] = bf16_bits(p[i]);
        tcb_check(tcb_memcpy(s->vm.param_ptr(s->ts.i_p16), h16.data(), uint64_t(h16.size()) * 2, 0, nullptr), "p16");
      }
    }
    if (s->ts.i_m >= 0) {
      tcb_check(tcb_memset(s->vm.param_ptr(s->ts.i_m), 0, uint64_t(sh) * 4, nullptr), "m");
      tcb_check(tcb_memset(s->vm.param_ptr(s->ts.i_v), 0, uint64_t(sh) * 4, nullptr), "v");
      tcb_check(tcb_memset(s->vm.param_ptr(s->ts.i_step), 0, 4, nullptr), "step");
    }
    tcb_check(tcb_device_sync(), "sync");
  });
}

/// Synthetic MLM batch: ids = Rng(seed).below(V); 15% of the
/// positions (Rng.below(100) < 15) carry their id as label, the rest -100.
int tb_synthetic_batch(int64_t T, int64_t V, int64_t seed, int32_t* ids, int32_t* labels, int causal_lm) {
  TB_TRY({
    Rng r(static_cast<uint64_t>(seed));
    for (int64_t t = 0; t < T; ++t) ids[t] = int32_t(r.below(uint32_t(V)));
    for (int64_t t = 0; t < T; ++t) {
      if (causal_lm) labels[t] = (t + 1 < T) ? ids[t + 1] : -100;
      else labels[t] = r.below(100) < 15 ? ids[t] : -100;
    }
  });
}

/// Copy a batch from host memory into the step's input buffers (H2D on the
/// session stream, through the pinned staging buffers).
int tb_session_set_batch(void* h, const int32_t* ids, const int32_t* labels) {
  TB_TRY({
    auto* s = static_cast<Session*>(h);
    const int64_t T = s->cfg.T();
    if (ids != s->h_ids) std::memcpy(s->h_ids, ids, size_t(T) * 4);
    if (labels != s->h_labels) std::memcpy(s->h_labels, labels, size_t(T) * 4);
    tcb_check(tcb_memcpy(s->vm.param_ptr(s->ts.i_ids), s->h_ids, uint64_t(T) * 4, 0, s->stream), "ids");
    tcb_check(tcb_memcpy(s->vm.param_ptr(s->ts.i_labels), s->h_labels, uint64_t(T) * 4, 0, s->stream), "labels");
  });
}

/// pinned staging pointers (so callers can fill them without an extra copy)
int32_t* tb_session_ids_buffer(void* h) { return static_cast<Session*>(h)->h_ids; }
int32_t* tb_session_labels_buffer(void* h) { return static_cast<Session*>(h)->h_labels; }

int tb_session_step(void* h, int use_graph) {
  TB_TRY({
    auto* s = static_cast<Session*>(h);
    s->vm.run(s->stream, use_graph != 0);
  });
}

/// enqueue the D2H read of the loss; *out valid after tb_session_sync
int tb_session_fetch_loss(void* h) {
  TB_TRY({
    auto* s = static_cast<Session*>(h);
    auto seq = ir::flatten(s->vm.fn());
    const ir::Var* lv = seq.ret->args.at(0)->var.get();
    tcb_check(tcb_memcpy(s->h_loss, s->vm.ptr_of(lv), 4, 1, s->stream), "loss");
  });
}
float tb_session_loss_value(void* h) { return static_cast<Session*>(h)->h_loss[0]; }

int tb_session_sync(void* h) { TB_TRY(tcb_check(tcb_stream_sync(static_cast<Session*>(h)->stream), "sync")); }

void* tb_session_stream(void* h) { return static_cast<Session*>(h)->stream; }

/// device pointer / byte size of function parameter `name` (ids, labels,
/// params, p16, m, v, step, ...)
int tb_session_param(void* h, const char* name, void** ptr, int64_t* bytes) {
  TB_TRY({
    auto* s = static_cast<Session*>(h);
    const auto& ps = s->vm.fn().params;
    for (size_t i = 0; i < ps.size(); ++i)
      if (ps[i]->id == name) {
        *ptr = s->vm.param_ptr(int(i));
        *bytes = nbytes(ps[i]->ty);
        return 0;
      }
    throw Error(std::string("no parameter ") + name);
  });
}

/// offsets/shapes of the flat parameter segments: "name offset numel\n"
const char* tb_session_segments(void* h) {
  auto* s = static_cast<Session*>(h);
  std::ostringstream os;
  for (auto& g : s->ts.segs) os << g.name << " " << g.offset << " " << g.numel << "\n";
  s->text = os.str();
  return s->text.c_str();
}

/// "ir": the dispatched step function; "bytecode": VM disassembly;
/// "mem": liveness/peak CSV (index,live_bytes,op) as `trainc inspect --mem`
const char* tb_session_text(void* h, const char* what) {
  auto* s = static_cast<Session*>(h);
  std::string w = what ? what : "";
  if (w == "ir") s->text = print_fn(s->vm.fn());
  else if (w == "bytecode") s->text = s->vm.disasm();
  else if (w == "mem") {
    auto mp = peak_memory(s->vm.layout());
    auto seq = ir::flatten(s->vm.fn());
    std::ostringstream os;
    os << "index,live_bytes,op\n";
    for (size_t i = 0; i < mp.curve.size() && i < seq.lets.size(); ++i)
      os << i << "," << mp.curve[i] << ","
         << (seq.lets[i].value->kind == ExprKind::Call ? seq.lets[i].value->op : "tuple_get") << "\n";
    s->text = os.str();
  } else s->text = "";
  return s->text.c_str();
}

/// vm.profile: `repeats` eager steps with CUDA events around
/// every instruction; CSV idx,op,let,median_us,bytes_in,bytes_out,kernels.
const char* tb_session_profile(void* h, int repeats) { return tb_session_profile_inner(h, repeats, 1); }

/// ... with every launch instruction run `inner` times back to back between
/// its events (per-launch mean: no event round trip per launch).  Advances the
/// session's training state `inner` updates per profiled step.
const char* tb_session_profile_inner(void* h, int repeats, int inner) {
  auto* s = static_cast<Session*>(h);
  try {
    s->text = s->vm.profile(s->stream, repeats, inner);
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
  return s->text.c_str();
}

int tb_session_set_comm(void* h, void* comm) {
  TB_TRY(static_cast<Session*>(h)->vm.set_comm(comm));
}

/// Parse text IR (text_ext.hpp: the reference's format plus bf16/i32
/// parameter tokens), re-infer every type, and print it again.  Returns NULL
/// with tb_last_error() on a parse or type error.
const char* tb_text_reprint(const char* text) {
  try {
    ensure_registered(split_ws(tcb_supported_ops()));
    ir::ModuleIR m = parse_text_ext(text ? text : "");
    if (m.functions.size() != 1) throw Error("tb_text_reprint: expects one function");
    g_text = print_text_ext(*m.functions[0].second);
    return g_text.c_str();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

/// CPU-only memsched on one text-IR function (text.hpp
/// syntax + bf16/i32 parameter tokens).  transient_inputs: function inputs die
/// at their last use (the accounting of SPEC.md's examples) instead of living
/// throughout (the device VM).  what:
///   "liveness"  one line per var field: "id field unit def last bytes" (unit =
///               root storage unit; aliases share their source's unit)
///   "curve"     "peak <bytes> <index>" then "i <live bytes>" per let
///   "schedule"  p-c list schedule: "peak_before B", "peak_after B",
///               "order id id ...", then the scheduled function's text
///   "remat"     rematerialise under `budget`: "replays N", "peak_before B",
///               "peak_after B", "split victim evict_index replay_before" per
///               split, then the transformed function's text
/// Returns NULL (tb_last_error) on parse/type errors or BudgetInfeasible.
const char* tb_memsched_text(const char* text, const char* what, int64_t budget, int transient_inputs) {
  try {
    ensure_registered(split_ws(tcb_supported_ops()));
    ir::ModuleIR m = parse_text_ext(text ? text : "");
    if (m.functions.size() != 1) throw Error("tb_memsched_text: expects one function");
    FunctionPtr fn = m.functions[0].second;
    const bool tr = transient_inputs != 0;
    const std::string w = what ? what : "";
    std::ostringstream os;
    if (w == "liveness") {
      Layout L = build_layout(*fn, {}, true, tr);
      auto line = [&](const ir::Var* v) {
        const auto& rs = L.refs.at(v);
        for (size_t k = 0; k < rs.size(); ++k) {
          int u = L.root(rs[k].unit).first;
          os << v->id << " " << k << " " << u << " " << L.units[u].def << " " << L.units[u].last << " "
             << rs[k].bytes << "\n";
        }
      };
      for (auto& p : fn->params) line(p.get());
      for (auto& b : ir::flatten(*fn).lets) line(b.var.get());
    } else if (w == "curve") {
      MemProfile mp = peak_memory(*fn, {}, tr);
      os << "peak " << mp.peak << " " << mp.peak_index << "\n";
      for (size_t i = 0; i < mp.curve.size(); ++i) os << i << " " << mp.curve[i] << "\n";
    } else if (w == "schedule") {
      LetSeq sq = schedule(*fn, {}, tr);
      FunctionPtr f2 = ir::make_fn(fn->name, fn->params, sq);
      os << "peak_before " << peak_memory(*fn, {}, tr).peak << "\n";
      os << "peak_after " << peak_memory(*f2, {}, tr).peak << "\n";
      os << "order";
      for (auto& b : sq.lets) os << " " << b.var->id;
      os << "\n" << print_text_ext(*f2);
    } else if (w == "overlap") {  // hoist_collectives + timeline: per let "id stream start end wait"
      LetSeq h = hoist_collectives(ir::flatten(*fn));
      Timeline t = timeline(h);
      os << "serial " << t.serial << "\noverlap " << t.overlap << "\nevents " << t.events << "\n";
      for (size_t i = 0; i < h.lets.size(); ++i) {
        const auto& e = t.ops[i];
        os << "op " << h.lets[i].var->id << " " << e.stream << " " << e.start << " " << e.end << " "
           << (e.wait_on >= 0 ? h.lets[size_t(e.wait_on)].var->id : std::string("-")) << "\n";
      }
    } else if (w == "remat") {
      auto [f2, plan] = rematerialize(*fn, budget, {}, tr);
      os << "replays " << plan.replays << "\npeak_before " << plan.peak_before << "\npeak_after "
         << plan.peak_after << "\n";
      for (auto& sp : plan.splits)
        os << "split " << sp.victim << " " << sp.evict_index << " " << sp.replay_before << "\n";
      os << print_text_ext(*f2);
    } else {
      throw Error("tb_memsched_text: unknown query '" + w + "'");
    }
    g_text = os.str();
    return g_text.c_str();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

/// backends::derive_priorities (backends.hpp:387-419) over vm.profile-style
/// latency samples, one per line "dialect op shape_class median_us"; returns
/// "dialect.op priority" lines (lower median -> higher priority).
const char* tb_derive_priorities(const char* samples) {
  try {
    std::vector<backends::LatencySample> v;
    std::istringstream is(samples ? samples : "");
    std::string line;
    while (std::getline(is, line)) {
      std::istringstream ls(line);
      backends::LatencySample x;
      if (ls >> x.dialect >> x.op >> x.shape_class >> x.median_us) v.push_back(x);
    }
    auto t = backends::derive_priorities(v);
    std::ostringstream os;
    for (auto& [k, pr] : t.priorities) os << k << " " << pr << "\n";
    g_text = os.str();
    return g_text.c_str();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

/// CPU-only: run the AutoCast pass (host/autocast.hpp) on the all-f32 training
/// step of `cfg` under policy "default", "b200" or "f32", with
/// placement "auto" (exclusive/shared) or "shared".  out: sites, casts,
/// exclusive, shared, low_ops, f32_violations, standalone_casts, param_casts, lets
int tb_autocast_info(const char* cfg, const char* policy, const char* placement, int64_t* out, int n) {
  TB_TRY({
    ensure_registered(split_ws(tcb_supported_ops()));
    ModelCfg c = parse_cfg(cfg ? cfg : "");
    if (c.dtype != "f32") throw Error("autocast: expects the all-f32 step (dtype=f32)");
    TrainStep ts = build_train_step(c);
    const PrecisionPolicy pol = policy_by_name(policy ? policy : "default");
    const std::string pl = placement ? placement : "auto";
    CastReport r;
    FunctionPtr fn = autocast(*ts.fn, pol, &r, pl == "shared" ? Placement::AllShared : Placement::Auto);
    int64_t v[] = {r.sites, r.casts, r.exclusive, r.shared, r.low_ops, r.f32_violations, r.standalone_casts,
                   r.param_casts, int64_t(ir::flatten(*fn).lets.size())};
    for (int i = 0; i < n && i < int(sizeof v / sizeof v[0]); ++i) out[i] = v[i];
  });
}

/// KernelCache::clear (backends.hpp:356-361) plus the plans (and their device
/// scratch) behind it.  Only valid while no session is alive: a live VM holds
/// plan handles.
int tb_cache_clear(void) {
  TB_TRY({
    std::lock_guard<std::mutex> g(PlanTable::global().mu);
    for (auto& kv : PlanTable::global().plans)
      if (kv.second) tcb_plan_destroy(kv.second);
    PlanTable::global().plans.clear();
    backends::KernelCache::global().clear();
  });
}

/// KernelCache counters (backends.hpp:363-368): compiles, hits, size
int tb_cache_stats(int64_t* out3) {
  TB_TRY({
    auto& c = backends::KernelCache::global();
    out3[0] = int64_t(c.compiles());
    out3[1] = int64_t(c.hits());
    out3[2] = int64_t(c.size());
  });
}

// --- TNSR tensor files (tensor.hpp:76-139; host/tnsr.hpp) -------------------

/// Write `data` (host memory, stored element bytes) as a TNSR file.
/// code: 0 f32, 1 f16 (the reference's), 2 bf16, 3 i32 (extension).
int tb_tnsr_save(const char* path, const void* data, int code, int rank, const int64_t* shape) {
  TB_TRY({
    tnsr::Header h;
    h.code = code;
    tnsr::code_bytes(code);
    if (rank < 0) throw Error("bad tensor file header");
    h.shape.assign(shape, shape + rank);
    tnsr::save(path, h, data);
  });
}

/// Header of a TNSR file: *code, *rank, shape[0..min(rank, cap)).
int tb_tnsr_header(const char* path, int* code, int* rank, int64_t* shape, int cap) {
  TB_TRY({
    tnsr::Header h = tnsr::load_header(path);
    *code = h.code;
    *rank = int(h.shape.size());
    for (int i = 0; i < cap && i < int(h.shape.size()); ++i) shape[i] = h.shape[size_t(i)];
  });
}

/// Read the data section of a TNSR file into host memory (bytes must match).
int tb_tnsr_load(const char* path, void* data, int64_t bytes) {
  TB_TRY(tnsr::load(path, data, bytes));
}

static const ir::Var& session_param(Session* s, const char* name, int* index) {
  const auto& ps = s->vm.fn().params;
  for (size_t i = 0; i < ps.size(); ++i)
    if (ps[i]->id == name) {
      *index = int(i);
      return *ps[i];
    }
  throw Error(std::string("no parameter ") + name);
}

/// Checkpoint one device-resident step parameter (params, p16, m, v, step, ...)
/// to a TNSR file: stream-ordered D2H on the session stream, then the write.
int tb_session_save_param(void* h, const char* name, const char* path) {
  TB_TRY({
    auto* s = static_cast<Session*>(h);
    int idx = 0;
    const auto& v = session_param(s, name, &idx);
    const auto& tt = v.ty.tensor();
    std::vector<char> buf(size_t(nbytes(tt)));
    tcb_check(tcb_memcpy(buf.data(), s->vm.param_ptr(idx), uint64_t(buf.size()), 1, s->stream), "d2h");
    tcb_check(tcb_stream_sync(s->stream), "sync");
    tnsr::Header hd;
    hd.code = int(tt.dtype);
    hd.shape = tt.shape;
    tnsr::save(path, hd, buf.data());
  });
}

/// Restore a step parameter from a TNSR file written for the same graph: the
/// dtype code and shape must equal the parameter's (no implicit conversion).
int tb_session_load_param(void* h, const char* name, const char* path) {
  TB_TRY({
    auto* s = static_cast<Session*>(h);
    int idx = 0;
    const auto& v = session_param(s, name, &idx);
    const auto& tt = v.ty.tensor();
    tnsr::Header hd = tnsr::load_header(path);
    if (hd.code != int(tt.dtype) || hd.shape != tt.shape)
      throw TypeError(std::string("TNSR file ") + path + " does not match parameter " + name);
    std::vector<char> buf(size_t(nbytes(tt)));
    tnsr::load(path, buf.data(), int64_t(buf.size()));
    tcb_check(tcb_memcpy(s->vm.param_ptr(idx), buf.data(), uint64_t(buf.size()), 0, s->stream), "h2d");
    tcb_check(tcb_stream_sync(s->stream), "sync");
  });
}

}  // extern "C"
