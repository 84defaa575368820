// distpar.hpp -- the overlap half of distpar for the ZeRO-1
// step that models.hpp builds (partition_zero + horizontal_fuse_collectives
// live there, because the shard layout is a function of the bucket table).
//
//  hoist_collectives  list scheduling that starts every collective as early as
//                     its inputs allow: a collective -- and the alias lets
//                     (view / concat) that exist only to feed it -- is emitted
//                     right after its last dependency; everything else keeps
//                     its order.  Dependence-preserving; values unchanged.
//  stream_of          Comm for collectives, Compute for everything else.
//  timeline           the two-stream cost simulation: per-op costs from the
//                     memsched cost table (op_cost), comm = alpha + beta * bytes
//                     (alpha = 1000, beta = 1 cost units); a
//                     consumer on the other stream waits on the latest
//                     producer it reads there -- one signal/wait pair per
//                     cross-stream edge -- and the makespan is compared with
//                     the serialized sum.
// The device VM (vm.hpp) executes exactly this assignment: collectives on its
// comm stream, an event wait wherever the timeline has a cross-stream edge.
#pragma once

#include <algorithm>
#include <set>
#include <unordered_map>
#include <vector>

#include "memsched.hpp"

namespace tb {

inline bool is_collective_op(const std::string& base) {
  return base == "reduce_scatter" || base == "all_gather" || base == "allreduce" ||
         base == "reduce_scatter_batched" || base == "all_gather_batched";
}

enum class Stream { Compute = 0, Comm = 1 };

inline Stream stream_of(const LetBinding& b) {
  return b.value->kind == ExprKind::Call && is_collective_op(base_name(b.value->op)) ? Stream::Comm
                                                                                    : Stream::Compute;
}

/// lets whose value only feeds collectives through alias ops (the bucket
/// views / concats): they move with their collective
inline std::vector<char> collective_feeders(const LetSeq& s) {
  const int n = int(s.lets.size());
  std::unordered_map<const ir::Var*, int> def;
  for (int i = 0; i < n; ++i) def[s.lets[i].var.get()] = i;
  std::vector<std::vector<int>> users(n);
  for (int i = 0; i < n; ++i)
    for (auto& a : s.lets[i].value->args)
      if (a->kind == ExprKind::VarRef && def.count(a->var.get())) users[def[a->var.get()]].push_back(i);
  std::set<const ir::Var*> returned;
  for (auto& a : ret_exprs(s))
    if (a->kind == ExprKind::VarRef) returned.insert(a->var.get());
  std::vector<char> hoist(n, 0);
  for (int i = n - 1; i >= 0; --i) {
    const auto& b = s.lets[i];
    if (stream_of(b) == Stream::Comm) {
      hoist[i] = 1;
      continue;
    }
    if (b.value->kind != ExprKind::Call) continue;
    const std::string base = base_name(b.value->op);
    if (base != "view" && base != "concat" && base != "reshape") continue;
    if (users[i].empty() || returned.count(b.var.get())) continue;
    bool all = true;
    for (int u : users[i]) all = all && hoist[u];
    hoist[i] = all;
  }
  return hoist;
}

inline LetSeq hoist_collectives(const LetSeq& s) {
  const int n = int(s.lets.size());
  std::unordered_map<const ir::Var*, int> def;
  for (int i = 0; i < n; ++i) def[s.lets[i].var.get()] = i;
  std::vector<std::vector<int>> deps(n);
  for (int i = 0; i < n; ++i)
    for (auto& a : s.lets[i].value->args)
      if (a->kind == ExprKind::VarRef && def.count(a->var.get())) deps[i].push_back(def[a->var.get()]);
  const std::vector<char> hoist = collective_feeders(s);
  std::vector<char> done(n, 0);
  LetSeq out;
  out.ret = s.ret;
  auto ready = [&](int i) {
    for (int d : deps[i])
      if (!done[d]) return false;
    return true;
  };
  auto emit = [&](int i) {
    out.lets.push_back(s.lets[i]);
    done[i] = 1;
  };
  auto drain = [&]() {  // every pending hoistable let whose inputs exist, in original order
    bool more = true;
    while (more) {
      more = false;
      for (int i = 0; i < n; ++i)
        if (hoist[i] && !done[i] && ready(i)) {
          emit(i);
          more = true;
        }
    }
  };
  drain();
  for (int i = 0; i < n; ++i) {
    if (hoist[i]) continue;
    if (!ready(i)) throw Error("hoist_collectives: dependence order violated");
    emit(i);
    drain();
  }
  if (int(out.lets.size()) != n) throw Error("hoist_collectives: unscheduled lets");
  return out;
}

struct TimelineEntry {
  int stream = 0;
  double start = 0, end = 0;
  int wait_on = -1;  // let index (in this order) of the cross-stream producer waited on, -1: none
};
struct Timeline {
  std::vector<TimelineEntry> ops;
  double serial = 0, overlap = 0;
  int events = 0, collectives = 0;
};

/// comm cost of a collective: alpha + beta * payload bytes
inline double comm_cost(const LetBinding& b, double alpha, double beta) {
  int64_t bytes = 0;
  for (auto& a : b.value->args)
    if (a->kind == ExprKind::VarRef && a->var->ty.is_tensor()) bytes = std::max(bytes, nbytes(a->var->ty));
  if (b.var->ty.is_tensor()) bytes = std::max(bytes, nbytes(b.var->ty));
  return alpha + beta * double(bytes);
}

inline Timeline timeline(const LetSeq& s, double alpha = 1000.0, double beta = 1.0) {
  const int n = int(s.lets.size());
  std::unordered_map<const ir::Var*, int> def;
  for (int i = 0; i < n; ++i) def[s.lets[i].var.get()] = i;
  Timeline t;
  t.ops.resize(size_t(n));
  double free_at[2] = {0, 0};
  for (int i = 0; i < n; ++i) {
    const auto& b = s.lets[i];
    const int st = int(stream_of(b));
    double cost = 0;
    if (b.value->kind == ExprKind::Call) {
      const std::string base = base_name(b.value->op);
      if (st == 1) {
        cost = comm_cost(b, alpha, beta);
        ++t.collectives;
      } else if (!is_alias_op(base)) {
        cost = op_cost(b.value);
      }
    }
    double start = free_at[st];
    int wait = -1;
    for (auto& a : b.value->args) {
      if (a->kind != ExprKind::VarRef) continue;
      auto it = def.find(a->var.get());
      if (it == def.end()) continue;
      const TimelineEntry& p = t.ops[size_t(it->second)];
      start = std::max(start, p.end);
      if (p.stream != st && (wait < 0 || t.ops[size_t(wait)].end < p.end)) wait = it->second;
    }
    // a wait is needed only if the stream's own order does not already cover it
    if (wait >= 0) {
      bool covered = false;
      for (int k = i - 1; k >= 0; --k)
        if (t.ops[size_t(k)].stream == st && t.ops[size_t(k)].wait_on >= wait &&
            t.ops[size_t(t.ops[size_t(k)].wait_on)].stream != st) {
          covered = true;
          break;
        }
      if (!covered) ++t.events;
    }
    t.ops[size_t(i)] = {st, start, start + cost, wait};
    free_at[st] = start + cost;
    t.serial += cost;
  }
  t.overlap = std::max(free_at[0], free_at[1]);
  return t;
}

}  // namespace tb
