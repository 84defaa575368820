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
/// attributes (the closure-hash slot carries the attribute string).
inline std::string cache_key(const std::string& op, const std::vector<TensorType>& in,
                             const std::vector<TensorType>& out, const AttrMap& attrs) {
  std::string k = op + "|";
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
                         const AttrMap& attrs) {
  const std::string key = cache_key(op, in, out, attrs);
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
      std::lock_guard<std::mutex> g(PlanTable::global().mu);
      auto& slot = PlanTable::global().plans[key];
      if (slot) tcb_plan_destroy(slot);  // last writer wins (backends.hpp:335-337)
      slot = p;
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
  int64_t arena_bytes = 0, state_bytes = 0, planner_peak = 0;
  int instructions = 0, kernels = 0, lets = 0;
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
    if (use_graph) {
      if (!graph_) {
        tcb_check(tcb_graph_capture_begin(stream), "graph capture");
        enqueue(stream);
        tcb_check(tcb_graph_capture_end(stream, &graph_), "graph capture end");
      }
      tcb_check(tcb_graph_launch(graph_, stream), "graph launch");
    } else {
      enqueue(stream);
    }
  }

  void set_comm(void* c) {
    comm_ = c;
    for (auto& ins : code_)
      (void)ins;
    if (graph_) {
      tcb_graph_destroy(graph_);
      graph_ = nullptr;
    }
  }
  void set_device(int d) { device_ = d; }
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
      if (base == "reduce_scatter") ins.kind = OpKind::ReduceScatter;
      else if (base == "all_gather") ins.kind = OpKind::AllGather;
      else if (base == "allreduce") ins.kind = OpKind::AllReduce;
      else {
        ins.plan = get_plan(b.value->op, tin, tout, b.value->call_attrs);
        ins.nkernels = tcb_plan_num_kernels(ins.plan);
      }
      if (ins.kind != OpKind::Launch) ins.nkernels = 1;
      stats_.kernels += ins.nkernels;
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
  }

  void enqueue(void* stream) {
    for (auto& x : code_) {
      switch (x.kind) {
        case OpKind::Launch:
          tcb_check(tcb_launch(x.plan, x.in.data(), int(x.in.size()), x.out.data(), int(x.out.size()), stream),
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
    }
  }

  static int64_t nbytes_desc(const tcb_tensor& t) {
    int64_t n = 1;
    for (int i = 0; i < t.rank; ++i) n *= t.shape[i];
    return n * (t.dtype == TCB_F32 || t.dtype == TCB_I32 ? 4 : t.dtype == TCB_U8 ? 1 : 2);
  }

  void release() {
    if (graph_) tcb_graph_destroy(graph_);
    graph_ = nullptr;
    if (arena_base_) tcb_free_arena(arena_base_);
    if (state_base_) tcb_free_arena(state_base_);
    arena_base_ = state_base_ = nullptr;
    code_.clear();
  }

  int device_ = 0;
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
  VMStats stats_;
};

}  // namespace tb
