// memsched.hpp -- execution-order optimisation on ANF:
// exact liveness over storage units, the peak-memory curve, the p-c greedy
// list scheduler and budgeted rematerialisation by liveness splitting.
//
// Storage model (shared with the device VM, so the planner's numbers are the
// VM's numbers): every tensor-valued let owns a storage unit, except
//   view / reshape / tuple_get   aliases of their source (0 bytes),
//   concat                       its inputs are placed inside its output
//                                ("concat elision"), so the output unit is live
//                                from the first input's definition,
//   state-bound outputs          written in place into the state parameter they
//                                update (optimizer p/m/v, step, half copy).
// A unit is live on [def, last use]; parameters are live throughout.  The op at
// index i needs its inputs and outputs live at i.
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <map>
#include <numeric>
#include <unordered_map>

#include "graph.hpp"

namespace tb {

struct Unit {
  int64_t bytes = 0;
  int def = 0, last = 0;
  int parent = -1;        // concat elision: placed inside parent at sub_off
  int64_t sub_off = 0;
  int param = -1;         // >= 0: a function parameter (persistent state / input)
  int producer = -1;      // let index that writes it (-1 for params)
  bool pinned = true;     // params: live over the whole function
};

struct Ref {
  int unit = -1;
  int64_t off = 0;   // byte offset inside the unit
  int64_t bytes = 0;
};

struct Layout {
  std::vector<Unit> units;
  std::unordered_map<const ir::Var*, std::vector<Ref>> refs;  // per tensor field
  std::vector<int> concat_copy;  // lets whose concat could not be fully elided
  int n = 0;                     // number of lets
  // root unit of u (following concat parents) and the byte offset inside it
  std::pair<int, int64_t> root(int u) const {
    int64_t off = 0;
    while (units[u].parent >= 0) {
      off += units[u].sub_off;
      u = units[u].parent;
    }
    return {u, off};
  }
};

/// the returned expressions of a let sequence: a tuple's fields or one var
inline std::vector<ExprPtr> ret_exprs(const LetSeq& seq) {
  if (!seq.ret) return {};
  if (seq.ret->kind == ExprKind::Tuple) return seq.ret->args;
  return {seq.ret};
}

inline bool inplace_safe(const std::string& base, int in_idx, int out_idx) {
  if (base == "adam_update" || base == "adam_update_ex")
    return (out_idx == 0 && in_idx == 0) || (out_idx == 1 && in_idx == 2) || (out_idx == 2 && in_idx == 3);
  if (base == "sgd_update") return in_idx == 0 && out_idx == 0;
  if (base == "add_scalar") return in_idx == 0 && out_idx == 0;
  if (base == "embedding_dx") return in_idx == 2 && out_idx == 0;  // base + scatter
  if (base == "cross_entropy") return in_idx == 0 && out_idx == 1;  // logits -> dlogits (k_ce_row)
  return false;
}

/// state_binding: (ret index, param index) pairs; params listed are written in
/// place when liveness allows (otherwise the VM copies back after the step).
///
/// transient_inputs: the accounting of SPEC.md's memsched EXAMPLES (:454-458,
/// "predecessor freed after each step"), where a function input that is not
/// bound state occupies memory only until its last use; the default is the
/// invariant of SPEC.md:431 ("params ... live over the whole function"), which
/// is also what the device VM does (inputs are persistent buffers).
inline Layout build_layout(const ir::FunctionIR& fn, const std::vector<std::pair<int, int>>& state_binding,
                           bool elide_concat = true, bool transient_inputs = false) {
  Layout L;
  auto seq = ir::flatten(fn);
  L.n = int(seq.lets.size());
  auto new_unit = [&](int64_t bytes, int def, int producer, int param = -1) {
    Unit u;
    u.bytes = bytes;
    u.def = def;
    u.last = def;
    u.producer = producer;
    u.param = param;
    L.units.push_back(u);
    return int(L.units.size()) - 1;
  };
  for (size_t p = 0; p < fn.params.size(); ++p) {
    int u = new_unit(nbytes(fn.params[p]->ty), -1, -1, int(p));
    L.units[u].last = L.n;
    L.refs[fn.params[p].get()] = {Ref{u, 0, L.units[u].bytes}};
  }
  // returned var -> param it must be written into
  std::unordered_map<const ir::Var*, int> bind;
  std::unordered_map<const ir::Var*, int> ret_index;
  if (seq.ret && seq.ret->kind == ExprKind::Tuple) {
    for (size_t j = 0; j < seq.ret->args.size(); ++j) {
      auto& a = seq.ret->args[j];
      if (a->kind == ExprKind::VarRef) ret_index[a->var.get()] = int(j);
    }
    for (auto& [rj, pi] : state_binding)
      if (rj < int(seq.ret->args.size()) && seq.ret->args[rj]->kind == ExprKind::VarRef)
        bind[seq.ret->args[rj]->var.get()] = pi;
  }
  // last use of every var; for params the alias-aware last use (views of a
  // param are reads of it) comes from an unbound dry run of this function
  std::unordered_map<const ir::Var*, int> last_use;
  for (int i = 0; i < L.n; ++i)
    for (auto& a : seq.lets[i].value->args)
      if (a->kind == ExprKind::VarRef) last_use[a->var.get()] = i;
  if (!state_binding.empty()) {
    Layout dry = build_layout(fn, {}, elide_concat);
    for (auto& u : dry.units)
      if (u.param >= 0) {
        int l = -1;
        for (int i = 0; i < dry.n; ++i)
          for (auto& a : seq.lets[i].value->args)
            if (a->kind == ExprKind::VarRef)
              for (auto& r : dry.refs.at(a->var.get()))
                if (dry.root(r.unit).first == int(&u - dry.units.data())) l = i;
        last_use[fn.params[u.param].get()] = l;
      }
  }
  // a field var (tuple_get) that is returned/bound: find it through tuple_gets
  std::unordered_map<const ir::Var*, std::map<int, const ir::Var*>> tuple_fields;
  for (auto& b : seq.lets)
    if (b.value->kind == ExprKind::TupleGet)
      tuple_fields[b.value->args[0]->var.get()][b.value->index] = b.var.get();

  auto try_bind = [&](const ir::Var* out_var, int let_i, const ir::ExprPtr& call, int out_idx) -> int {
    auto it = bind.find(out_var);
    if (it == bind.end()) return -1;
    int pi = it->second;
    const ir::Var* pv = fn.params[pi].get();
    auto lu = last_use.find(pv);
    int lastp = lu == last_use.end() ? -1 : lu->second;
    if (lastp > let_i) return -1;
    if (lastp == let_i) {
      bool ok = false;
      for (size_t k = 0; k < call->args.size(); ++k)
        if (call->args[k]->kind == ExprKind::VarRef && call->args[k]->var.get() == pv)
          ok = inplace_safe(base_name(call->op), int(k), out_idx);
      if (!ok) return -1;
    }
    return L.refs[pv][0].unit;
  };

  // number of vars referring to each unit (aliases block plain in-place reuse)
  std::vector<int> unit_refs(L.units.size(), 1);
  auto note = [&](int u) {
    if (int(unit_refs.size()) <= u) unit_refs.resize(u + 1, 0);
    unit_refs[u]++;
  };

  for (int i = 0; i < L.n; ++i) {
    const auto& b = seq.lets[i];
    const auto& e = b.value;
    auto arg_refs = [&](size_t k) -> const std::vector<Ref>& { return L.refs.at(e->args[k]->var.get()); };
    if (e->kind == ExprKind::TupleGet) {
      L.refs[b.var.get()] = {L.refs.at(e->args[0]->var.get()).at(e->index)};
      note(L.refs[b.var.get()][0].unit);
      continue;
    }
    if (e->kind != ExprKind::Call) throw Error("memsched: unsupported let kind");
    const std::string base = base_name(e->op);
    if (base == "view") {
      Ref r = arg_refs(0)[0];
      const auto& src = e->args[0]->var->ty.tensor();
      r.off += ir::attr_int(e->call_attrs, "offset", 0) * dtype_bytes(src.dtype);
      r.bytes = nbytes(b.var->ty);
      L.refs[b.var.get()] = {r};
      note(r.unit);
      continue;
    }
    if (base == "reshape") {
      L.refs[b.var.get()] = {arg_refs(0)[0]};
      note(arg_refs(0)[0].unit);
      continue;
    }
    if (base == "concat") {
      int u = new_unit(nbytes(b.var->ty), i, i);
      int64_t off = 0;
      bool all = true;
      for (size_t k = 0; k < e->args.size(); ++k) {
        const Ref& r = arg_refs(k)[0];
        Unit& cu = L.units[r.unit];
        bool ok = elide_concat && r.off == 0 && r.bytes == cu.bytes && cu.param < 0 && cu.parent < 0 &&
                  cu.producer >= 0 && last_use[e->args[k]->var.get()] == i;
        // the producer must produce exactly this unit (not a tuple field shared elsewhere)
        if (ok) {
          cu.parent = u;
          cu.sub_off = off;
          L.units[u].def = std::min(L.units[u].def, cu.def);
        } else {
          all = false;
        }
        off += r.bytes;
      }
      if (!all) L.concat_copy.push_back(i);
      L.refs[b.var.get()] = {Ref{u, 0, L.units[u].bytes}};
      note(u);
      continue;
    }
    // ordinary op: one unit per output field, or in place into a bound param
    std::vector<Ref> outs;
    if (b.var->ty.is_tuple()) {
      const auto& fields = b.var->ty.tuple().fields;
      auto tf = tuple_fields.find(b.var.get());
      std::set<int> taken;  // input units already handed to an earlier field
      for (size_t k = 0; k < fields.size(); ++k) {
        int pu = -1;
        const ir::Var* fv = (tf != tuple_fields.end() && tf->second.count(int(k))) ? tf->second.at(int(k)) : nullptr;
        if (fv) pu = try_bind(fv, i, e, int(k));
        // plain in-place reuse for a field (same rules as single-output ops)
        if (pu < 0 && !(fv && bind.count(fv))) {
          for (size_t a = 0; a < e->args.size() && pu < 0; ++a) {
            if (e->args[a]->kind != ExprKind::VarRef || !inplace_safe(base, int(a), int(k))) continue;
            const ir::Var* av = e->args[a]->var.get();
            const auto& rs = L.refs.at(av);
            if (rs.size() != 1) continue;
            const Ref& r = rs[0];
            const Unit& cu = L.units[r.unit];
            if (cu.param < 0 && cu.parent < 0 && r.off == 0 && r.bytes == cu.bytes && cu.bytes == nbytes(fields[k]) &&
                unit_refs[r.unit] == 1 && last_use[av] == i && !ret_index.count(av) && !taken.count(r.unit))
              pu = r.unit;
          }
          if (pu >= 0) taken.insert(pu);
        }
        if (pu >= 0) outs.push_back(Ref{pu, 0, nbytes(fields[k])});
        else {
          int u = new_unit(nbytes(fields[k]), i, i);
          outs.push_back(Ref{u, 0, L.units[u].bytes});
        }
      }
    } else {
      int pu = try_bind(b.var.get(), i, e, 0);
      // plain in-place reuse: an in-place-safe input whose whole, unaliased
      // activation unit dies at this op hands its storage to the output
      if (pu < 0 && !bind.count(b.var.get())) {
        for (size_t k = 0; k < e->args.size() && pu < 0; ++k) {
          if (e->args[k]->kind != ExprKind::VarRef || !inplace_safe(base, int(k), 0)) continue;
          const ir::Var* av = e->args[k]->var.get();
          const auto& rs = L.refs.at(av);
          if (rs.size() != 1) continue;
          const Ref& r = rs[0];
          const Unit& cu = L.units[r.unit];
          if (cu.param < 0 && cu.parent < 0 && r.off == 0 && r.bytes == cu.bytes && cu.bytes == nbytes(b.var->ty) &&
              unit_refs[r.unit] == 1 && last_use[av] == i && !ret_index.count(av))
            pu = r.unit;
        }
      }
      if (pu >= 0) outs.push_back(Ref{pu, 0, nbytes(b.var->ty)});
      else {
        int u = new_unit(nbytes(b.var->ty), i, i);
        outs.push_back(Ref{u, 0, L.units[u].bytes});
      }
    }
    L.refs[b.var.get()] = outs;
    for (auto& r : outs) {
      if (int(unit_refs.size()) <= r.unit) unit_refs.resize(r.unit + 1, 0);
      unit_refs[r.unit]++;
    }
  }
  // uses extend lifetimes
  for (int i = 0; i < L.n; ++i)
    for (auto& a : seq.lets[i].value->args)
      if (a->kind == ExprKind::VarRef)
        for (auto& r : L.refs.at(a->var.get())) L.units[r.unit].last = std::max(L.units[r.unit].last, i);
  for (auto& a : ret_exprs(seq))
    if (a->kind == ExprKind::VarRef)
      for (auto& r : L.refs.at(a->var.get())) L.units[r.unit].last = L.n;
  // concat children: the parent covers them
  for (size_t u = 0; u < L.units.size(); ++u) {
    if (L.units[u].parent < 0) continue;
    auto [root, off] = L.root(int(u));
    (void)off;
    L.units[root].def = std::min(L.units[root].def, L.units[u].def);
    L.units[root].last = std::max(L.units[root].last, L.units[u].last);
  }
  if (transient_inputs) {
    std::set<int> bound;
    for (auto& [rj, pi] : state_binding) bound.insert(pi);
    std::vector<int> lastp(L.units.size(), -1);
    for (int i = 0; i < L.n; ++i)
      for (auto& a : seq.lets[i].value->args)
        if (a->kind == ExprKind::VarRef)
          for (auto& r : L.refs.at(a->var.get())) {
            int ru = L.root(r.unit).first;
            lastp[ru] = std::max(lastp[ru], i);
          }
    for (auto& a : ret_exprs(seq))
      if (a->kind == ExprKind::VarRef)
        for (auto& r : L.refs.at(a->var.get())) lastp[L.root(r.unit).first] = L.n;
    for (size_t u = 0; u < L.units.size(); ++u) {
      Unit& x = L.units[u];
      if (x.param < 0 || bound.count(x.param)) continue;
      x.pinned = false;
      x.def = 0;
      x.last = std::max(lastp[u], 0);
    }
  }
  return L;
}

// ------------------------------------------------------------ peak memory
struct MemProfile {
  std::vector<int64_t> curve;  // bytes live at each let index
  int64_t peak = 0;
  int peak_index = -1;
  int64_t state_bytes = 0;     // parameters (live throughout)
};

/// a tensor occupies its bytes from its producing op through
/// its last use; op i needs inputs + outputs live at i.
inline MemProfile peak_memory(const Layout& L) {
  MemProfile m;
  m.curve.assign(std::max(L.n, 1), 0);
  for (size_t u = 0; u < L.units.size(); ++u) {
    const Unit& x = L.units[u];
    if (x.parent >= 0) continue;
    if (x.param >= 0 && x.pinned) {
      m.state_bytes += x.bytes;
      for (auto& c : m.curve) c += x.bytes;
      continue;
    }
    for (int i = std::max(0, x.def); i <= std::min(x.last, L.n - 1); ++i) m.curve[i] += x.bytes;
  }
  for (int i = 0; i < int(m.curve.size()); ++i)
    if (m.curve[i] > m.peak) {
      m.peak = m.curve[i];
      m.peak_index = i;
    }
  return m;
}

inline MemProfile peak_memory(const ir::FunctionIR& fn, const std::vector<std::pair<int, int>>& sb = {},
                             bool transient_inputs = false) {
  return peak_memory(build_layout(fn, sb, true, transient_inputs));
}

// ----------------------------------------------------------- arena plan
struct ArenaPlan {
  std::vector<int64_t> offset;  // per unit (-1: not in the arena)
  int64_t size = 0;             // high-water mark
};

/// Static offsets for every non-parameter root unit: walk the let order, free
/// units after their last use, place new units best-fit into freed gaps
/// (address-ordered free list), else at the top.  Deterministic.
inline ArenaPlan plan_arena(const Layout& L, int64_t align = 256) {
  ArenaPlan P;
  P.offset.assign(L.units.size(), -1);
  std::vector<std::vector<int>> starts(L.n + 1), ends(L.n + 2);
  for (size_t u = 0; u < L.units.size(); ++u) {
    const Unit& x = L.units[u];
    if (x.parent >= 0 || x.param >= 0 || x.bytes == 0) continue;
    starts[std::max(0, x.def)].push_back(int(u));
    ends[std::min(x.last, L.n) + 1].push_back(int(u));
  }
  std::map<int64_t, int64_t> free_;  // offset -> size
  int64_t top = 0;
  auto rnd = [&](int64_t b) { return (b + align - 1) / align * align; };
  auto release = [&](int u) {
    int64_t off = P.offset[u], sz = rnd(L.units[u].bytes);
    auto it = free_.emplace(off, sz).first;
    auto nx = std::next(it);
    if (nx != free_.end() && it->first + it->second == nx->first) {
      it->second += nx->second;
      free_.erase(nx);
    }
    if (it != free_.begin()) {
      auto pv = std::prev(it);
      if (pv->first + pv->second == it->first) {
        pv->second += it->second;
        free_.erase(it);
        it = pv;
      }
    }
    if (it->first + it->second == top) {
      top = it->first;
      free_.erase(it);
    }
  };
  for (int i = 0; i <= L.n; ++i) {
    for (int u : ends[i]) release(u);
    auto& st = starts[std::min(i, L.n)];
    if (i < L.n) {
      std::vector<int> us = st;
      std::sort(us.begin(), us.end(), [&](int a, int b) {
        return L.units[a].bytes != L.units[b].bytes ? L.units[a].bytes > L.units[b].bytes : a < b;
      });
      for (int u : us) {
        int64_t sz = rnd(L.units[u].bytes);
        auto best = free_.end();
        for (auto it = free_.begin(); it != free_.end(); ++it)
          if (it->second >= sz && (best == free_.end() || it->second < best->second)) best = it;
        if (best != free_.end()) {
          P.offset[u] = best->first;
          int64_t rem = best->second - sz, noff = best->first + sz;
          free_.erase(best);
          if (rem > 0) free_.emplace(noff, rem);
        } else {
          P.offset[u] = top;
          top += sz;
        }
        P.size = std::max(P.size, top);
      }
    }
  }
  return P;
}

// ---------------------------------------------------------------- cost model
/// Per-op cost for scheduling / remat scores: GEMM-shaped ops
/// m*n*k, attention its two batched products, everything else the element
/// count of its largest operand -- CostModel::op_cost (opreg.hpp:536-559)
/// extended to the closure-like extension ops it would throw on.
inline double op_cost(const ir::ExprPtr& call) {
  const std::string base = base_name(call->op);
  auto T = [&](size_t i) { return call->args.at(i)->var->ty.tensor(); };
  if (base == "matmul") return double(T(0).shape[0]) * T(0).shape[1] * T(1).shape[1];
  if (base == "linear" || base == "matmul_t" || base == "matmul_dact") {
    const auto& a = T(0);
    double k = a.shape[ir::attr_int(call->call_attrs, "ta", 0) ? 0 : 1];
    return double(numel(a)) / k * k * double(numel(T(1))) / k;
  }
  if (base == "matmul_pair") {
    const int n0 = int(ir::attr_int(call->call_attrs, "n0", 2));
    const auto &a0 = T(0), &b0 = T(1), &a1 = T(size_t(n0)), &b1 = T(size_t(n0) + 1);
    double k0 = a0.shape[ir::attr_int(call->call_attrs, "ta0", 0) ? 0 : 1];
    double k1 = a1.shape[ir::attr_int(call->call_attrs, "ta1", 0) ? 0 : 1];
    return double(numel(a0)) * double(numel(b0)) / k0 + double(numel(a1)) * double(numel(b1)) / k1;
  }
  if (base == "attention" || base == "attention_dx") {
    const auto& q = T(0);
    double S = double(ir::attr_int(call->call_attrs, "seq", q.shape[0]));
    return 2.0 * double(q.shape[0]) * S * double(q.shape[1] / 3);
  }
  double n = 1;
  for (auto& a : call->args)
    if (a->kind == ExprKind::VarRef && a->var->ty.is_tensor()) n = std::max(n, double(numel(a->var->ty.tensor())));
  if (call->ty.is_tensor()) n = std::max(n, double(numel(call->ty.tensor())));
  return n;
}

// ------------------------------------------------------------------ schedule
/// p - c greedy list scheduling: among ready lets pick the
/// one with minimum (bytes produced - bytes freed), ties by original order.
inline LetSeq schedule(const ir::FunctionIR& fn, const std::vector<std::pair<int, int>>& sb = {},
                       bool transient_inputs = false) {
  Layout L = build_layout(fn, sb, true, transient_inputs);
  LetSeq seq = ir::flatten(fn);
  const int n = int(seq.lets.size());
  std::unordered_map<const ir::Var*, int> def;
  for (int i = 0; i < n; ++i) def[seq.lets[i].var.get()] = i;
  std::vector<std::vector<int>> deps(n), users(n);
  for (int i = 0; i < n; ++i)
    for (auto& a : seq.lets[i].value->args)
      if (a->kind == ExprKind::VarRef && def.count(a->var.get())) {
        int d = def[a->var.get()];
        deps[i].push_back(d);
        users[d].push_back(i);
      }
  // remaining uses per root unit
  auto roots_of = [&](const ir::Var* v) {
    std::vector<int> r;
    for (auto& ref : L.refs.at(v)) r.push_back(L.root(ref.unit).first);
    return r;
  };
  std::vector<int> remaining(L.units.size(), 0);
  for (int i = 0; i < n; ++i)
    for (auto& a : seq.lets[i].value->args)
      if (a->kind == ExprKind::VarRef)
        for (int u : roots_of(a->var.get())) remaining[u]++;
  std::vector<char> pinned(L.units.size(), 0);
  for (size_t u = 0; u < L.units.size(); ++u)
    if ((L.units[u].param >= 0 && L.units[u].pinned) || L.units[u].last >= n) pinned[u] = 1;
  std::vector<int> indeg(n);
  for (int i = 0; i < n; ++i) indeg[i] = int(deps[i].size());
  std::vector<int> ready;
  for (int i = 0; i < n; ++i)
    if (!indeg[i]) ready.push_back(i);
  std::vector<char> produced(L.units.size(), 0);
  LetSeq out;
  out.ret = seq.ret;
  while (!ready.empty()) {
    int best = -1;
    double best_score = 0;
    for (int i : ready) {
      const auto& b = seq.lets[i];
      double p = 0, c = 0;
      for (auto& r : L.refs.at(b.var.get())) {
        int u = L.root(r.unit).first;
        if (!produced[u] && L.units[u].param < 0) p += double(L.units[u].bytes);
      }
      std::unordered_map<int, int> cnt;
      for (auto& a : b.value->args)
        if (a->kind == ExprKind::VarRef)
          for (int u : roots_of(a->var.get())) cnt[u]++;
      for (auto& [u, k] : cnt)
        if (!pinned[u] && remaining[u] == k) c += double(L.units[u].bytes);
      double sc = p - c;
      if (best < 0 || sc < best_score || (sc == best_score && i < best)) {
        best = i;
        best_score = sc;
      }
    }
    ready.erase(std::find(ready.begin(), ready.end(), best));
    const auto& b = seq.lets[best];
    for (auto& r : L.refs.at(b.var.get())) produced[L.root(r.unit).first] = 1;
    for (auto& a : b.value->args)
      if (a->kind == ExprKind::VarRef)
        for (int u : roots_of(a->var.get())) remaining[u]--;
    out.lets.push_back(b);
    for (int j : users[best])
      if (--indeg[j] == 0) ready.push_back(j);
  }
  if (int(out.lets.size()) != n) throw Error("schedule: cycle detected");
  return out;
}

// -------------------------------------------------------------- rematerialize
struct RematSplit {
  std::string victim;  // var id evicted
  int evict_index;     // evicted after this position (in the output order)
  int replay_before;   // position of the first use it was replayed for
};
struct RematPlan {
  std::vector<RematSplit> splits;
  int replays = 0;     // replayed ops ("overhead")
  int64_t peak_before = 0, peak_after = 0;
};

inline bool replayable(const ir::ExprPtr& e) {
  if (e->kind != ExprKind::Call) return false;
  const std::string base = base_name(e->op);
  if (is_alias_op(base) || base == "fill") return false;
  const auto& bop = opreg::registry().base_of(e->op);
  return bop.pure && !bop.collective;
}

/// Budgeted rematerialisation: simulate the live set in
/// order; wherever the projected bytes (live + this op's new outputs) exceed
/// the budget, evict the live, not-currently-needed, replayable tensor with the
/// minimum score cost(producer) * remaining_uses / bytes (ties: larger, then
/// earlier), and replay its producer right before its next use (liveness
/// split).  Replay inputs must be live there; depth-1 victims only (the spec
/// allows <= 3; deeper chains are not evicted).  Throws BudgetInfeasible when
/// the floor (state + max single-op working set) exceeds the budget.
/// tuple_chains: a dead input that is a FIELD of a replayable tuple producer
/// (a LayerNorm output feeding a linear, as in pre-LN GPT-2) may be re-created
/// by replaying that producer whole (depth-2 chain through a twin get-let).
inline std::pair<FunctionPtr, RematPlan> rematerialize(const ir::FunctionIR& fn, int64_t budget,
                                                        const std::vector<std::pair<int, int>>& sb = {},
                                                        bool transient_inputs = false, bool tuple_chains = true) {
  RematPlan plan;
  auto cur = std::make_shared<ir::FunctionIR>(fn);
  for (int iter = 0; iter < 100000; ++iter) {
    Layout L = build_layout(*cur, sb, true, transient_inputs);
    MemProfile mp = peak_memory(L);
    if (iter == 0) plan.peak_before = mp.peak;
    plan.peak_after = mp.peak;
    if (mp.peak <= budget) return {cur, plan};
    LetSeq seq = ir::flatten(*cur);
    const int n = int(seq.lets.size());
    const int i = mp.peak_index;
    // floor: state + inputs/outputs of op i
    int64_t floor_i = mp.state_bytes;
    std::set<int> needed;
    for (auto& r : L.refs.at(seq.lets[i].var.get())) needed.insert(L.root(r.unit).first);
    for (auto& a : seq.lets[i].value->args)
      if (a->kind == ExprKind::VarRef)
        for (auto& r : L.refs.at(a->var.get())) needed.insert(L.root(r.unit).first);
    for (int u : needed)
      if (L.units[u].param < 0 || !L.units[u].pinned) floor_i += L.units[u].bytes;
    // candidates: units live across i, not used at i, produced by a replayable
    // single-output op whose inputs are params or still live at the next use
    std::unordered_map<const ir::Var*, int> def;
    for (int k = 0; k < n; ++k) def[seq.lets[k].var.get()] = k;
    int best_u = -1, best_next = -1;
    // depth-2 chain entries: a dead input of the replayed producer, re-created
    // by replaying ITS producer let `prod` (a tuple producer when the input is
    // a field of it: `field` >= 0, re-read through a twin get-let)
    struct ChainEnt {
      const ir::Var* dead;
      int prod;
      int field;
    };
    std::vector<ChainEnt> best_chain;
    double best_score = std::numeric_limits<double>::infinity();
    for (size_t u = 0; u < L.units.size(); ++u) {
      const Unit& x = L.units[u];
      if (x.param >= 0 || x.parent >= 0 || x.producer < 0 || x.def >= i || x.last <= i || x.last >= n) continue;
      if (needed.count(int(u))) continue;
      const auto& pe = seq.lets[x.producer].value;
      // tuple producers are replayed whole (every field recomputed; field uses
      // after the split are redirected to the replay, see below)
      if (!replayable(pe)) continue;
      // next use after i
      int next = -1, uses_after = 0;
      for (int k = i + 1; k < n; ++k)
        for (auto& a : seq.lets[k].value->args)
          if (a->kind == ExprKind::VarRef)
            for (auto& r : L.refs.at(a->var.get()))
              if (L.root(r.unit).first == int(u)) {
                if (next < 0) next = k;
                ++uses_after;
              }
      if (next < 0) continue;
      // replay inputs must be live at `next` (params, or units whose last >=
      // next); an input that is dead there may itself be replayed first when
      // its producer is a single-output replayable op whose inputs are live
      // (a depth-2 chain; SPEC.md:485 allows up to 3)
      bool ok = true;
      double cost = op_cost(pe);
      std::vector<ChainEnt> chain;
      for (auto& a : pe->args) {
        if (a->kind != ExprKind::VarRef || !ok) continue;
        bool dead = false;
        for (auto& r : L.refs.at(a->var.get())) {
          const Unit& iu = L.units[L.root(r.unit).first];
          if ((iu.param < 0 || !iu.pinned) && iu.last < next) dead = true;
        }
        if (!dead) continue;
        auto dit = def.find(a->var.get());
        if (dit == def.end()) {
          ok = false;
          continue;
        }
        int prod = dit->second, field = -1;
        if (seq.lets[prod].value->kind == ExprKind::TupleGet && tuple_chains) {  // a field of a tuple producer
          const auto& tg = seq.lets[prod].value;
          auto tit = tg->args[0]->kind == ExprKind::VarRef ? def.find(tg->args[0]->var.get()) : def.end();
          if (tit == def.end()) {
            ok = false;
            continue;
          }
          field = int(tg->index);
          prod = tit->second;
        }
        const auto& p2 = seq.lets[prod];
        if (p2.value->kind != ExprKind::Call || (field < 0 && p2.var->ty.is_tuple()) || !replayable(p2.value)) {
          ok = false;
          continue;
        }
        for (auto& a2 : p2.value->args) {
          if (a2->kind != ExprKind::VarRef) continue;
          for (auto& r2 : L.refs.at(a2->var.get())) {
            const Unit& iu2 = L.units[L.root(r2.unit).first];
            if ((iu2.param < 0 || !iu2.pinned) && iu2.last < next) ok = false;
          }
        }
        if (ok) {
          chain.push_back({a->var.get(), prod, field});
          cost += op_cost(p2.value);
        }
      }
      if (!ok) continue;
      double score = cost * uses_after / double(std::max<int64_t>(1, x.bytes));
      if (score < best_score) {
        best_score = score;
        best_u = int(u);
        best_next = next;
        best_chain = chain;
      }
    }
    if (best_u < 0 && std::getenv("TB_REMAT_DEBUG")) {  // why nothing is evictable here
      std::fprintf(stderr, "remat: peak %lld at %d (%s), floor %lld, budget %lld\n", (long long)mp.peak, i,
                   seq.lets[i].value->op.c_str(), (long long)floor_i, (long long)budget);
      for (size_t u = 0; u < L.units.size(); ++u) {
        const Unit& x = L.units[u];
        if (x.param >= 0 || x.parent >= 0 || x.def >= i || x.last <= i || x.bytes < (int64_t(256) << 20)) continue;
        const char* why = needed.count(int(u)) ? "needed" : x.producer < 0 ? "no producer"
                          : !replayable(seq.lets[x.producer].value) ? "not replayable" : "inputs dead / no next";
        std::fprintf(stderr, "  unit %zu %lld MB def %d last %d %s: %s\n", u, (long long)(x.bytes >> 20), x.def,
                     x.last, x.producer >= 0 ? seq.lets[x.producer].value->op.c_str() : "-", why);
      }
    }
    if (best_u < 0) {
      if (floor_i > budget)
        throw BudgetInfeasible("remat: floor " + std::to_string(floor_i) + " B exceeds budget " + std::to_string(budget));
      throw BudgetInfeasible("remat: no evictable tensor at index " + std::to_string(i));
    }
    // liveness split: clone the producer right before best_next, rename uses >= best_next
    const int prod = L.units[best_u].producer;
    const auto& pb = seq.lets[prod];
    auto nv = ir::make_var(pb.var->id + "_r" + std::to_string(plan.replays), pb.var->ty, pb.var->attrs);
    auto ne = std::make_shared<ir::Expr>(*pb.value);
    ne->serial = ir::detail::next_serial();
    // depth-2 chain: replay the dead inputs' producers first, feed the replay
    std::vector<std::pair<ir::VarPtr, ir::ExprPtr>> chain_lets;
    for (auto& ce_ : best_chain) {
      const auto& cb = seq.lets[ce_.prod];
      auto cv2 = ir::make_var(cb.var->id + "_r" + std::to_string(plan.replays), cb.var->ty, cb.var->attrs);
      auto ce = std::make_shared<ir::Expr>(*cb.value);
      ce->serial = ir::detail::next_serial();
      chain_lets.push_back({cv2, ce});
      ir::VarPtr feed = cv2;
      if (ce_.field >= 0) {  // twin get-let of the replayed tuple's field
        const Type ft = cb.var->ty.tuple().fields.at(size_t(ce_.field));
        auto gv = ir::make_var(ce_.dead->id + "_r" + std::to_string(plan.replays), ft, ce_.dead->attrs);
        auto ge = ir::tuple_get(ir::var_ref(cv2), ce_.field);
        ge->ty = ft;
        chain_lets.push_back({gv, ge});
        feed = gv;
      }
      for (auto& a : ne->args)
        if (a->kind == ExprKind::VarRef && a->var.get() == ce_.dead) a = ir::var_ref(feed);
      plan.replays++;
    }
    const ir::Var* old = pb.var.get();
    // a tuple producer's fields are read through get-lets; those defined before
    // the split whose vars are used after it get a twin on the replay
    std::unordered_map<const ir::Var*, ir::VarPtr> twin;
    std::vector<std::pair<ir::VarPtr, ir::ExprPtr>> twin_lets;
    if (pb.var->ty.is_tuple())
      for (int k = 0; k < best_next; ++k) {
        const auto& g = seq.lets[k];
        if (g.value->kind != ExprKind::TupleGet || g.value->args[0]->kind != ExprKind::VarRef ||
            g.value->args[0]->var.get() != old)
          continue;
        auto tv = ir::make_var(g.var->id + "_r" + std::to_string(plan.replays), g.var->ty, g.var->attrs);
        auto te = ir::tuple_get(ir::var_ref(nv), g.value->index);
        te->ty = g.value->ty;
        twin[g.var.get()] = tv;
        twin_lets.push_back({tv, te});
      }
    LetSeq out;
    out.ret = seq.ret;
    for (int k = 0; k < n; ++k) {
      if (k == best_next) {
        for (auto& c : chain_lets) out.lets.push_back({c.first, c.second});
        out.lets.push_back({nv, ne});
        for (auto& t : twin_lets) out.lets.push_back({t.first, t.second});
      }
      auto b = seq.lets[k];
      if (k >= best_next) {
        bool touched = false;
        auto e2 = std::make_shared<ir::Expr>(*b.value);
        for (auto& a : e2->args) {
          if (a->kind != ExprKind::VarRef) continue;
          if (a->var.get() == old) {
            a = ir::var_ref(nv);
            touched = true;
          } else if (auto it = twin.find(a->var.get()); it != twin.end()) {
            a = ir::var_ref(it->second);
            touched = true;
          }
        }
        if (touched) b.value = e2;
      }
      out.lets.push_back(b);
    }
    // returned vars are never victims (last < n), so ret is unchanged
    plan.splits.push_back({pb.var->id, i, best_next});
    plan.replays++;
    cur = ir::make_fn(cur->name, cur->params, out);
  }
  throw BudgetInfeasible("remat: iteration limit");
}

}  // namespace tb
