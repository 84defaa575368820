// pipeline.hpp -- the graph-generation phases shared by the device session
// (capi.cpp) and the CPU oracle interpreter (oracle/interp.cpp), so a session
// key builds the same step graph on both sides (SPEC.md:719-722 phase order:
// autodiff -> [autocast] -> fusion -> memsched -> dispatch).
#pragma once

#include "autocast.hpp"
#include "models.hpp"

namespace tb {

/// AutoCast the all-f32 training step in place per `autocast=<key>`
/// (parse_autocast_key): the pass, then optionally fold_param_casts (the
/// parameter converts become the optimizer's bf16 compute copy) and a fusion
/// re-run on the bf16 graph.
inline void apply_autocast(TrainStep& ts, const std::string& key) {
  const AutocastKey k = parse_autocast_key(key);
  if (ts.cfg.dtype != "f32") throw Error("autocast: expects the all-f32 step (dtype=f32)");
  ts.fn = autocast(*ts.fn, policy_by_name(k.policy));
  if (k.fold) {
    if (ts.cfg.world != 1 || ts.cfg.opt != "adam") throw Error("autocast +fold: world 1 Adam steps only");
    ts.fn = fold_param_casts(*ts.fn, ts.i_params, ts.P_pad, &ts.i_p16, ts.state_binding);
  }
  if (k.fuse) {
    LetSeq fs = ir::flatten(*ts.fn);
    fuse(fs, ts.cfg.fuse != 0, disabled_patterns(ts.cfg));
    ts.fn = ir::make_fn(ts.fn->name, ts.fn->params, fs);
  }
}

/// The last graph-generation phase (after AutoCast, before memsched and
/// dispatch): rule-based fusion of elementwise runs into ew_closures
/// (graph.hpp rule_fuse; key rules=0 disables it).
inline RuleFuseStats finalize_graph(TrainStep& ts) {
  RuleFuseStats st;
  if (!ts.cfg.fuse || !ts.cfg.rules) return st;
  LetSeq s = ir::flatten(*ts.fn);
  st = rule_fuse(s);
  ts.fn = ir::make_fn(ts.fn->name, ts.fn->params, s);
  ts.rule_closures = st.closures;
  return st;
}

}  // namespace tb
