// vm.hpp -- the device VM on libtcb200.
//
// compile():  ANF (dispatched to b200.*) -> bytecode.  One storage unit per
//             value (memsched.hpp Layout); static arena offsets from the
//             liveness plan replace the spec's runtime StoragePool (pow2 slabs)
//             -- every AllocStorage/Free is resolved at compile time, so a step
//             performs no allocation.  Each Invoke resolves its launch plan
//             through the reference's KernelCache (backends.hpp:338-383) keyed
//             per SPEC.md:596-600; aliases (view / reshape / tuple_get / elided
//             concat) emit nothing; collectives become NCCL instructions.
// run():      enqueue every instruction on the compute stream; the first run
//             is captured into a CUDA graph and later steps replay it
//             (capture on first run, replay after).
#pragma once

#include <cstdio>

#include "memsched.hpp"
#include "tcb200.h"
#include "trainc/backends.hpp"

namespace tb {

inline void tcb_check(int rc, const std::string& what) {
  if (rc == TCB_OK) return;
  std::string m = what + ": " + tcb_last_error();
  if (rc == TCB_ERR_UNIMPLEMENTED) throw UnimplementedOp(m);
  if (rc == TCB_ERR_TYPE) throw TypeError(m);
  if (rc == TCB_ERR_PROTOCOL) throw ProtocolError(m);
  throw Error(m);
}

inline tcb_tensor desc(void* ptr, const TensorType& t) {
  tcb_tensor d{};
  d.ptr = ptr;
  d.dtype = dtype_code(t.dtype);
  d.rank = t.rank();
  for (int i = 0; i < t.rank(); ++i) d.shape[i] = t.shape[i];
  return d;
}

/// KernelCacheKey: dialect op, input shapes + dtypes,
/// attributes (the closure-hash slot carries the attribute string), plus the
/// device the plan was compiled for (plans hold read-only device data).
inline std::string cache_key(const std::string& op, const std::vector<TensorType>& in,
                             const std::vector<TensorType>& out, const AttrMap& attrs, int device = 0) {
  std::string k = "dev" + std::to_string(device) + "|" + op + "|";
  for (auto& t : in) k += type_str(t) + ",";
  k += "->";
  for (auto& t : out) k += type_str(t) + ",";
  k += "|";
  for (auto& [a, v] : attrs) {
    k += a + "=";
    if (auto* i = std::get_if<std::int64_t>(&v)) k += std::to_string(*i);
    else if (auto* d = std::get_if<double>(&v)) {
      char buf[64];
      std::snprintf(buf, sizeof buf, "%.17g", *d);
      k += buf;
    } else k += std::get<std::string>(v);
    k += ";";
  }
  return k;
}

inline std::vector<tcb_attr> to_tcb_attrs(const AttrMap& m, std::vector<std::string>& keep) {
  std::vector<tcb_attr> out;
  keep.reserve(keep.size() + 2 * m.size());
  for (auto& [k, v] : m) {
    tcb_attr a{};
    keep.push_back(k);
    a.key = keep.back().c_str();
    if (auto* i = std::get_if<std::int64_t>(&v)) {
      a.kind = TCB_ATTR_INT;
      a.i = *i;
    } else if (auto* d = std::get_if<double>(&v)) {
      a.kind = TCB_ATTR_FLOAT;
      a.d = *d;
    } else {
      a.kind = TCB_ATTR_STR;
      keep.push_back(std::get<std::string>(v));
      a.s = keep.back().c_str();
    }
    out.push_back(a);
  }
  return out;
}

/// Process-wide plan table behind backends::KernelCache: the cache owns the
/// Kernel entries (key, compile/hit counters, last-writer-wins), this table owns
/// the tcb_plan each key compiled to.  Plans are immutable and shared.
struct PlanTable {
  std::mutex mu;
  std::map<std::string, tcb_plan> plans;
  static PlanTable& global() {
    static PlanTable t;
    return t;
  }
};

inline tcb_plan get_plan(const std::string& op, const std::vector<TensorType>& in, const std::vector<TensorType>& out,
                         const AttrMap& attrs, int device = 0) {
  const std::string key = cache_key(op, in, out, attrs, device);
  backends::KernelCache::global().get(key, [&]() -> backends::KernelPtr {
    std::vector<tcb_tensor> di, dout;
    for (auto& t : in) di.push_back(desc(nullptr, t));
    for (auto& t : out) dout.push_back(desc(nullptr, t));
    std::vector<std::string> keep;
    auto at = to_tcb_attrs(attrs, keep);
    tcb_plan p = nullptr;
    tcb_check(tcb_plan_create(op.c_str(), di.data(), int(di.size()), dout.data(), int(dout.size()), at.data(),
                              int(at.size()), nullptr, &p),
              "compile " + op);
    {
      // a plan already published under this key may be held by a running VM:
      // it is never destroyed -- a concurrent duplicate compile is dropped
      // (the KernelCache entry itself stays last-writer-wins, backends.hpp:335-337)
      std::lock_guard<std::mutex> g(PlanTable::global().mu);
      auto& slot = PlanTable::global().plans[key];
      if (slot) tcb_plan_destroy(p);
      else slot = p;
    }
    auto k = std::make_shared<backends::Kernel>();
    k->key = key;
    k->exec = [key](const TensorList&) -> TensorList {
      throw Error("b200 kernel " + key + " executes on device buffers; use the device VM");
    };
    return k;
  });
  std::lock_guard<std::mutex> g(PlanTable::global().mu);
  return PlanTable::global().plans.at(key);
}

enum class OpKind { Launch, ReduceScatter, AllGather, AllReduce, Copy };

struct Instr {
  OpKind kind = OpKind::Launch;
  std::string op;     // dialect op name
  int let = -1;
  tcb_plan plan = nullptr;
  std::vector<tcb_tensor> in, out;
  int64_t copy_bytes = 0;
  int nkernels = 0;
};

struct VMStats {
  int64_t arena_bytes = 0, state_bytes = 0, planner_peak = 0, workspace_bytes = 0;
  int instructions = 0, kernels = 0, lets = 0;
  int kernels_static = 0;  // sum of the plans' kernel counts (before fold deferral)
};

class DeviceVM {
 public:
  DeviceVM() = default;
  DeviceVM(const DeviceVM&) = delete;
  ~DeviceVM() { release(); }

  /// fn: dispatched ANF.  state_binding: (ret index, param index).
  void compile(FunctionPtr fn, std::vector<std::pair<int, int>> state_binding, void* comm = nullptr) {
    release();
    fn_ = fn;
    sb_ = std::move(state_binding);
    comm_ = comm;
    seq_ = ir::flatten(*fn_);
    layout_ = build_layout(*fn_, sb_);
    arena_ = plan_arena(layout_);
    auto mp = peak_memory(layout_);
    stats_ = {};
    stats_.planner_peak = mp.peak;
    stats_.arena_bytes = arena_.size;
    stats_.lets = int(seq_.lets.size());
    // device memory: the arena (activations) + one buffer per parameter
    void* base = nullptr;
    tcb_check(tcb_init(device_, uint64_t(std::max<int64_t>(arena_.size, 256)), &base), "tcb_init");
    arena_base_ = static_cast<char*>(base);
    param_ptr_.assign(fn_->params.size(), nullptr);
    int64_t state = 0;
    for (size_t p = 0; p < fn_->params.size(); ++p) state += (nbytes(fn_->params[p]->ty) + 255) / 256 * 256;
    void* sbase = nullptr;
    tcb_check(tcb_init(device_, uint64_t(std::max<int64_t>(state, 256)), &sbase), "tcb_init(state)");
    state_base_ = static_cast<char*>(sbase);
    int64_t off = 0;
    for (size_t p = 0; p < fn_->params.size(); ++p) {
      param_ptr_[p] = state_base_ + off;
      off += (nbytes(fn_->params[p]->ty) + 255) / 256 * 256;
    }
    stats_.state_bytes = state;
    tcb_check(tcb_memset(state_base_, 0, uint64_t(std::max<int64_t>(state, 256)), nullptr), "memset state");
    emit_bytecode();
  }

  char* ptr_of(const ir::Var* v, int field = 0) const {
    const Ref& r = layout_.refs.at(v).at(field);
    auto [root, sub] = layout_.root(r.unit);
    const Unit& u = layout_.units[root];
    char* base = u.param >= 0 ? static_cast<char*>(param_ptr_[u.param]) : arena_base_ + arena_.offset[root];
    return base + sub + r.off;
  }
  void* param_ptr(int p) const { return param_ptr_.at(p); }
  const ir::FunctionIR& fn() const { return *fn_; }

  /// enqueue one step on `stream`; use_graph: capture once, then replay
  void run(void* stream, bool use_graph) {
    // deferred partial-sum folds for this step's enqueue (pool allocated here,
    // outside capture); enqueue flushes them before the optimizer
    if (has_collectives_ && !comm_ && world_ > 1)
      throw ProtocolError("device VM: a world-" + std::to_string(world_) +
                          " step needs a communicator (set_comm) before it runs");
    if (fold_defer_ && !fold_ctx_) tcb_check(tcb_fold_ctx_create(fold_pool_bytes(), &fold_ctx_), "fold context");
    tcb_check(tcb_fold_use(fold_defer_ ? fold_ctx_ : nullptr), "fold use");
    struct Off {
      ~Off() { tcb_fold_use(nullptr); }
    } off;
    uint64_t d0 = 0, l0 = 0, d1 = 0, l1 = 0;
    tcb_check(tcb_fold_counters(&d0, &l0), "fold counters");
    if (use_graph) {
      if (!graph_) {
        tcb_check(tcb_graph_capture_begin(stream), "graph capture");
        enqueue(stream);
        tcb_check(tcb_graph_capture_end(stream, &graph_), "graph capture end");
        tcb_check(tcb_fold_counters(&d1, &l1), "fold counters");
        stats_.kernels = int(stats_.kernels_static - int64_t(d1 - d0) + int64_t(l1 - l0));
      }
      tcb_check(tcb_graph_launch(graph_, stream), "graph launch");
    } else {
      enqueue(stream);
      tcb_check(tcb_fold_counters(&d1, &l1), "fold counters");
      stats_.kernels = int(stats_.kernels_static - int64_t(d1 - d0) + int64_t(l1 - l0));
    }
  }
  static uint64_t fold_pool_bytes() {
    const char* e = std::getenv("TCB_FOLD_POOL_MB");
    return uint64_t(e ? std::atoll(e) : 256) << 20;
  }
  void set_fold_defer(bool on) { fold_defer_ = on; }

  void set_comm(void* c) {
    comm_ = c;
    if (graph_) {
      tcb_graph_destroy(graph_);
      graph_ = nullptr;
    }
  }
  void set_device(int d) { device_ = d; }
  void set_world(int w) { world_ = w; }
  const VMStats& stats() const { return stats_; }
  const Layout& layout() const { return layout_; }
  const std::vector<Instr>& code() const { return code_; }

  /// disassembly: one instruction per line, `idx: OPCODE args`
  std::string disasm() const {
    std::string s;
    for (size_t i = 0; i < code_.size(); ++i) {
      const Instr& x = code_[i];
      const char* k = x.kind == OpKind::Launch ? "Invoke" : x.kind == OpKind::Copy ? "Move" : "Collective";
      s += std::to_string(i) + ": " + k + " " + x.op + " let=" + std::to_string(x.let) + " in=[";
      for (auto& t : x.in) s += std::to_string(static_cast<const char*>(t.ptr) - arena_base_) + ",";
      s += "] out=[";
      for (auto& t : x.out) s += std::to_string(static_cast<const char*>(t.ptr) - arena_base_) + ",";
      s += "]\n";
    }
    return s;
  }

 private:
  void emit_bytecode() {
    code_.clear();
    rng_ptr_ = nullptr;
    for (size_t p = 0; p < fn_->params.size(); ++p)
      if (fn_->params[p]->id == "rng_step") rng_ptr_ = param_ptr_[p];
    std::set<int> copy_concat(layout_.concat_copy.begin(), layout_.concat_copy.end());
    for (size_t i = 0; i < seq_.lets.size(); ++i) {
      const auto& b = seq_.lets[i];
      if (b.value->kind != ExprKind::Call) continue;
      const std::string base = base_name(b.value->op);
      if ((base == "view" || base == "reshape")) continue;
      if (base == "concat" && !copy_concat.count(int(i))) continue;
      Instr ins;
      ins.op = b.value->op;
      ins.let = int(i);
      std::vector<TensorType> tin, tout;
      for (auto& a : b.value->args) {
        const auto& t = a->var->ty.tensor();
        tin.push_back(t);
        ins.in.push_back(desc(ptr_of(a->var.get()), t));
      }
      if (b.var->ty.is_tuple()) {
        const auto& f = b.var->ty.tuple().fields;
        for (size_t k = 0; k < f.size(); ++k) {
          tout.push_back(f[k]);
          ins.out.push_back(desc(ptr_of(b.var.get(), int(k)), f[k]));
        }
      } else {
        tout.push_back(b.var->ty.tensor());
        ins.out.push_back(desc(ptr_of(b.var.get()), b.var->ty.tensor()));
      }
      // dropout sites read the step's rng_step state as a trailing launch input
      // (plan attr rng_in=1): their Philox masks change every step
      AttrMap pattrs = b.value->call_attrs;
      if (rng_ptr_ && (pattrs.count("seed") || pattrs.count("in_seed")) &&
          (ir::attr_double(pattrs, "p", 0.0) > 0.0 || ir::attr_double(pattrs, "in_p", 0.0) > 0.0)) {
        pattrs["rng_in"] = std::int64_t(1);
        TensorType rt{kF32, {1}};
        tin.push_back(rt);
        ins.in.push_back(desc(rng_ptr_, rt));
      }
      if (base == "reduce_scatter") ins.kind = OpKind::ReduceScatter;
      else if (base == "all_gather") ins.kind = OpKind::AllGather;
      else if (base == "allreduce") ins.kind = OpKind::AllReduce;
      else {
        ins.plan = get_plan(b.value->op, tin, tout, pattrs, device_);
        ins.nkernels = tcb_plan_num_kernels(ins.plan);
      }
      if (ins.kind != OpKind::Launch) ins.nkernels = 1;
      stats_.kernels += ins.nkernels;
      stats_.kernels_static += ins.nkernels;
      code_.push_back(std::move(ins));
    }
    // returned values bound to a state param but not written in place: copy back
    if (seq_.ret) {
      for (auto& [rj, pi] : sb_) {
        auto& a = seq_.ret->args.at(rj);
        char* src = ptr_of(a->var.get());
        char* dst = static_cast<char*>(param_ptr_[pi]);
        if (src == dst) continue;
        Instr c;
        c.kind = OpKind::Copy;
        c.op = "copy_back";
        c.copy_bytes = nbytes(a->var->ty);
        c.in.push_back(desc(src, a->var->ty.tensor()));
        c.out.push_back(desc(dst, a->var->ty.tensor()));
        code_.push_back(c);
      }
    }
    stats_.instructions = int(code_.size());
    // one launch workspace for the whole (stream-ordered) step: the largest
    // any plan asks for (plans own no mutable device memory)
    uint64_t ws = 0;
    for (auto& x : code_) {
      if (!x.plan) continue;
      uint64_t b = 0;
      tcb_check(tcb_plan_workspace_bytes(x.plan, &b), "workspace size");
      ws = std::max(ws, b);
    }
    if (ws) {
      void* w = nullptr;
      tcb_check(tcb_init(device_, ws, &w), "tcb_init(workspace)");
      ws_ = w;
      ws_bytes_ = ws;
    }
    stats_.workspace_bytes = int64_t(ws);
    for (auto& x : code_)
      if (x.kind == OpKind::ReduceScatter || x.kind == OpKind::AllGather || x.kind == OpKind::AllReduce)
        has_collectives_ = true;
  }

  static DType code_dtype(int c) {
    return c == TCB_F32 ? kF32 : c == TCB_BF16 ? dtype_from("bf16") : c == TCB_I32 ? kI32 : kF16;
  }

  static bool is_optimizer(const std::string& op) {
    return op == "adam_update" || op == "adam_update_ex" || op == "sgd_update";
  }
  // vm.profile: events around every main-stream instruction
  // and every fold flush of an eager step
  struct ProfMark {
    int instr;  // index into code_, -1: a deferred-fold flush
    void *e0, *e1;
  };
  std::vector<ProfMark>* prof_ = nullptr;
  int prof_inner_ = 1;
  std::vector<void*> prof_events_;
  size_t prof_used_ = 0;
  void* prof_rec(void* stream) {
    if (prof_used_ >= prof_events_.size()) {
      void* e = nullptr;
      tcb_check(tcb_event_create(&e), "event");
      prof_events_.push_back(e);
    }
    void* e = prof_events_[prof_used_++];
    tcb_check(tcb_event_record(e, stream), "event record");
    return e;
  }
  void flush_folds(void* stream) {
    void* e0 = prof_ ? prof_rec(stream) : nullptr;
    tcb_check(tcb_fold_flush(stream), "fold flush");
    if (prof_) prof_->push_back({-1, e0, prof_rec(stream)});
  }

 public:
  /// vm.profile: `repeats` eager steps with CUDA events around every
  /// instruction; one CSV row per instruction (and per deferred-fold flush):
  /// idx,op,let,median_us,bytes_in,bytes_out,kernels.  Compile time is not in
  /// here (it happened at session creation: the one-time bucket).  inner > 1:
  /// each launch instruction runs `inner` times back to back between its
  /// events and its time is the mean -- the in-stream cost of a launch without
  /// the event round trip, the way the graph replay sees it.  It leaves the
  /// session's training state advanced `inner` optimizer updates per step
  /// (profile on a session whose state does not matter).
  std::string profile(void* stream, int repeats, int inner = 1) {
    prof_inner_ = std::max(1, inner);
    struct InnerOff {
      DeviceVM* v;
      ~InnerOff() { v->prof_inner_ = 1; }
    } inner_off{this};
    std::vector<std::vector<float>> times;
    std::vector<ProfMark> marks;
    std::vector<ProfMark> first;
    for (int r = 0; r < std::max(1, repeats); ++r) {
      marks.clear();
      prof_used_ = 0;
      prof_ = &marks;
      struct Off {
        DeviceVM* v;
        ~Off() { v->prof_ = nullptr; }
      } off{this};
      run(stream, false);
      tcb_check(tcb_stream_sync(stream), "sync");
      if (r == 0) {
        first = marks;
        times.assign(marks.size(), {});
      }
      if (marks.size() != first.size()) throw Error("profile: instruction stream changed between repeats");
      for (size_t i = 0; i < marks.size(); ++i) {
        float ms = 0;
        tcb_check(tcb_event_elapsed_ms(marks[i].e0, marks[i].e1, &ms), "elapsed");
        const bool launch = marks[i].instr >= 0 && code_[size_t(marks[i].instr)].kind == OpKind::Launch;
        times[i].push_back(launch ? ms / float(prof_inner_) : ms);
      }
    }
    std::string out = "idx,op,let,median_us,bytes_in,bytes_out,kernels,shapes\n";
    auto shp = [](const std::vector<tcb_tensor>& ts) {
      std::string r;
      for (size_t i = 0; i < ts.size(); ++i) {
        if (i) r += ";";
        for (int d = 0; d < ts[i].rank; ++d) r += (d ? "x" : "") + std::to_string(ts[i].shape[d]);
      }
      return r;
    };
    for (size_t i = 0; i < first.size(); ++i) {
      auto v = times[i];
      std::sort(v.begin(), v.end());
      const double med = 1000.0 * v[v.size() / 2];
      const int k = first[i].instr;
      int64_t bi = 0, bo = 0;
      std::string op = "fold_flush";
      int let = -1, nk = 1;
      std::string shapes;
      if (k >= 0) {
        const Instr& x = code_[size_t(k)];
        shapes = shp(x.in) + ">" + shp(x.out);
        for (auto& t : x.in) bi += nbytes_desc(t);
        for (auto& t : x.out) bo += nbytes_desc(t);
        op = x.op;
        let = x.let;
        nk = x.nkernels;
      }
      char buf[256];
      std::snprintf(buf, sizeof buf, "%zu,%s,%d,%.3f,%lld,%lld,%d,", i, op.c_str(), let, med, (long long)bi,
                    (long long)bo, nk);
      out += buf + shapes + "\n";
    }
    return out;
  }

 private:
  void enqueue(void* stream) {
    for (size_t xi = 0; xi < code_.size(); ++xi) {
      auto& x = code_[xi];
      if (x.kind != OpKind::Launch || is_optimizer(x.op)) flush_folds(stream);
      if (x.kind == OpKind::ReduceScatter || x.kind == OpKind::AllGather || x.kind == OpKind::AllReduce) {
        enqueue_collective(x, stream);
        continue;
      }
      wait_comm_hazards(x, stream);
      void* pe0 = prof_ ? prof_rec(stream) : nullptr;
      switch (x.kind) {
        case OpKind::Launch:
          // vm.profile with inner > 1 relaunches each instruction back to back
          // (data-independent timing; in-place ops see their own outputs)
          for (int rep = 0; rep < (prof_ ? prof_inner_ : 1); ++rep)
            tcb_check(tcb_launch_ws(x.plan, x.in.data(), int(x.in.size()), x.out.data(), int(x.out.size()), ws_,
                                    ws_bytes_, stream),
                      x.op);
          break;
        case OpKind::ReduceScatter:
          tcb_check(tcb_reduce_scatter(comm_, x.in.data(), int(x.in.size()), &x.out[0], stream), x.op);
          break;
        case OpKind::AllGather:
          tcb_check(tcb_all_gather(comm_, &x.in[0], x.out.data(), int(x.out.size()), stream), x.op);
          break;
        case OpKind::AllReduce:
          tcb_check(tcb_memcpy(x.out[0].ptr, x.in[0].ptr, uint64_t(nbytes_desc(x.in[0])), 2, stream), x.op);
          tcb_check(tcb_all_reduce(comm_, &x.out[0], stream), x.op);
          break;
        case OpKind::Copy:
          tcb_check(tcb_memcpy(x.out[0].ptr, x.in[0].ptr, uint64_t(x.copy_bytes), 2, stream), "copy_back");
          break;
      }
      if (prof_) prof_->push_back({int(xi), pe0, prof_rec(stream)});
    }
    flush_folds(stream);
    if (!inflight_.empty()) {  // join: the step ends when the last collective is done
      tcb_check(tcb_stream_wait_event(stream, inflight_.back().done), "stream wait");
      ++comm_waits_;
      inflight_.clear();
    }
    comm_ev_used_ = 0;
  }

  // ---- the comm stream (distpar overlap_schedule) ----
  // Collectives run on their own stream: each one waits for everything the
  // compute stream enqueued before it (its inputs were hoisted right behind
  // their producers by hoist_collectives), and a compute instruction waits on
  // the latest in-flight collective whose buffers it touches (RAW on the
  // collective's output, WAR on its input's arena space): one signal/wait
  // pair per cross-stream edge.
  struct Inflight {
    void* done;
    std::vector<std::pair<const char*, const char*>> ranges;
  };
  std::vector<Inflight> inflight_;
  void* comm_stream_ = nullptr;
  std::vector<void*> comm_ev_;
  size_t comm_ev_used_ = 0;
  int comm_waits_ = 0;
  void* comm_event() {
    if (comm_ev_used_ >= comm_ev_.size()) {
      void* e = nullptr;
      tcb_check(tcb_event_create(&e), "event");
      comm_ev_.push_back(e);
    }
    return comm_ev_[comm_ev_used_++];
  }
  static std::pair<const char*, const char*> range_of(const tcb_tensor& t) {
    const char* a = static_cast<const char*>(t.ptr);
    return {a, a + nbytes_desc(t)};
  }
  void enqueue_collective(Instr& x, void* stream) {
    flush_folds(stream);  // deferred gradient folds of this bucket land first
    if (!comm_stream_) tcb_check(tcb_stream_create(&comm_stream_), "comm stream");
    void* go = comm_event();
    tcb_check(tcb_event_record(go, stream), "event record");
    tcb_check(tcb_stream_wait_event(comm_stream_, go), "stream wait");
    void* pe0 = prof_ ? prof_rec(comm_stream_) : nullptr;
    switch (x.kind) {
      case OpKind::ReduceScatter:
        tcb_check(tcb_reduce_scatter(comm_, x.in.data(), int(x.in.size()), &x.out[0], comm_stream_), x.op);
        break;
      case OpKind::AllGather:
        tcb_check(tcb_all_gather(comm_, &x.in[0], x.out.data(), int(x.out.size()), comm_stream_), x.op);
        break;
      default:
        tcb_check(tcb_memcpy(x.out[0].ptr, x.in[0].ptr, uint64_t(nbytes_desc(x.in[0])), 2, comm_stream_), x.op);
        tcb_check(tcb_all_reduce(comm_, &x.out[0], comm_stream_), x.op);
        break;
    }
    if (prof_) prof_->push_back({int(&x - code_.data()), pe0, prof_rec(comm_stream_)});
    Inflight f;
    f.done = comm_event();
    tcb_check(tcb_event_record(f.done, comm_stream_), "event record");
    for (auto& t : x.in) f.ranges.push_back(range_of(t));
    for (auto& t : x.out) f.ranges.push_back(range_of(t));
    inflight_.push_back(std::move(f));
  }
  void wait_comm_hazards(const Instr& x, void* stream) {
    if (inflight_.empty()) return;
    int last = -1;
    for (int k = int(inflight_.size()) - 1; k >= 0 && last < 0; --k)
      for (auto& r : inflight_[size_t(k)].ranges) {
        bool hit = false;
        for (auto* ts : {&x.in, &x.out})
          for (auto& t : *ts) {
            auto q = range_of(t);
            if (q.first < r.second && r.first < q.second) hit = true;
          }
        if (hit) {
          last = k;
          break;
        }
      }
    if (last < 0) return;
    tcb_check(tcb_stream_wait_event(stream, inflight_[size_t(last)].done), "stream wait");
    ++comm_waits_;
    inflight_.erase(inflight_.begin(), inflight_.begin() + last + 1);  // the comm stream is FIFO
  }

  static int64_t nbytes_desc(const tcb_tensor& t) {
    int64_t n = 1;
    for (int i = 0; i < t.rank; ++i) n *= t.shape[i];
    return n * (t.dtype == TCB_F32 || t.dtype == TCB_I32 ? 4 : t.dtype == TCB_U8 ? 1 : 2);
  }

  void release() {
    for (void* e : prof_events_) tcb_event_destroy(e);
    prof_events_.clear();
    for (void* e : comm_ev_) tcb_event_destroy(e);
    comm_ev_.clear();
    if (comm_stream_) tcb_stream_destroy(comm_stream_);
    comm_stream_ = nullptr;
    inflight_.clear();
    if (graph_) tcb_graph_destroy(graph_);
    graph_ = nullptr;
    if (arena_base_) tcb_free_arena(arena_base_);
    if (state_base_) tcb_free_arena(state_base_);
    if (ws_) tcb_free_arena(ws_);
    if (fold_ctx_) tcb_fold_ctx_destroy(fold_ctx_);
    arena_base_ = state_base_ = nullptr;
    ws_ = fold_ctx_ = nullptr;
    ws_bytes_ = 0;
    has_collectives_ = false;
    code_.clear();
  }

  int device_ = 0;
  // TCB_FOLD_DEFER=0 folds every partial sum in place (A/B and debugging)
  bool fold_defer_ = !(std::getenv("TCB_FOLD_DEFER") && std::atoi(std::getenv("TCB_FOLD_DEFER")) == 0);
  FunctionPtr fn_;
  LetSeq seq_;
  std::vector<std::pair<int, int>> sb_;
  Layout layout_;
  ArenaPlan arena_;
  char* arena_base_ = nullptr;
  char* state_base_ = nullptr;
  std::vector<void*> param_ptr_;
  std::vector<Instr> code_;
  void* graph_ = nullptr;
  void* comm_ = nullptr;
  void* ws_ = nullptr;        // launch workspace of the compute stream
  uint64_t ws_bytes_ = 0;
  void* fold_ctx_ = nullptr;  // this VM's deferred-fold pool
  bool has_collectives_ = false;
  int world_ = 1;
  void* rng_ptr_ = nullptr;   // the rng_step state (dropout step counter)
  VMStats stats_;
};

}  // namespace tb
