// text_ext.hpp -- the reference's text IR (text.hpp) for b200 step graphs.
//
// The reference printer names every non-f32 dtype "f16" (dtype_name,
// dtype.hpp:51-53) and its parser knows only f32/f16 (text.hpp:424-432), so a
// bf16 step or an i32 index parameter would be mislabelled silently.  Only
// parameter types are spelled in the text (let types are re-inferred), so the
// extension is confined to the fn header:
//   print: the reference printer, then the header's parameter dtype tokens are
//          rewritten from the true types (bf16, i32);
//   parse: bf16/i32 parameter tokens are read into a side table and replaced
//          by f32 for the reference parser; the parameters are then retyped
//          and every let re-inferred through the registry (infer_types,
//          opreg.hpp:719-735).
// Tuple fields print as `%t .0` (see print_text_ext).  Otherwise, for
// all-f32/f16 functions, both directions are exactly the reference's.
#pragma once

#include <map>
#include <regex>
#include <string>

#include "trainc/text.hpp"
#include "ext_ops.hpp"

namespace tb {

inline std::string ext_dtype_token(DType d) {
  return d == kF32 ? "f32" : d == kF16 ? "f16" : d == kBF16 ? "bf16" : d == kI32 ? "i32" : "?";
}

inline std::string print_text_ext(const ir::FunctionIR& fn) {
  std::string s = ir::print_text(fn);
  const size_t eol = s.find('\n');
  std::string head = s.substr(0, eol);
  for (auto& p : fn.params) {
    if (!p->ty.is_tensor()) continue;
    const DType d = p->ty.tensor().dtype;
    if (d == kF32 || d == kF16) continue;
    const std::string from = "%" + p->id + ": f16[", to = "%" + p->id + ": " + ext_dtype_token(d) + "[";
    const size_t at = head.find(from);
    if (at == std::string::npos) throw Error("print_text_ext: parameter %" + p->id + " not found in header");
    head.replace(at, from.size(), to);
  }
  std::string body = eol == std::string::npos ? "" : s.substr(eol);
  // tuple fields: the reference prints `%t.0`, which its own lexer reads back
  // as one identifier (idents may contain '.', text.hpp:207-220); a space
  // before the dot makes it the Dot token its parser expects (text.hpp:453-459)
  static const std::regex field(R"((%[A-Za-z_][A-Za-z0-9_]*)\.([0-9]+))");
  body = std::regex_replace(body, field, "$1 .$2");
  return head + body;
}

/// The reference parser creates a fresh Var object per `%id` occurrence; the
/// passes here (memsched, the VM) identify values by Var pointer, so every
/// reference is relinked to its definition (param or let) by id.
inline void relink_vars(ir::FunctionIR& fn) {
  std::unordered_map<std::string, VarPtr> def;
  for (auto& p : fn.params) def[p->id] = p;
  auto seq = ir::flatten(fn);
  std::function<void(const ExprPtr&)> fix = [&](const ExprPtr& e) {
    if (!e) return;
    if (e->kind == ExprKind::VarRef) {
      auto it = def.find(e->var->id);
      if (it == def.end()) throw Error("text: %" + e->var->id + " used before its definition");
      e->var = it->second;
      return;
    }
    for (auto& a : e->args) fix(a);
  };
  for (auto& b : seq.lets) {
    fix(b.value);
    def[b.var->id] = b.var;
  }
  fix(seq.ret);
}

inline ir::ModuleIR parse_text_ext(const std::string& src) {
  std::map<std::string, DType> ext;  // param id -> dtype outside the reference format
  static const std::regex tok(R"(%([A-Za-z0-9_.]+): (bf16|i32)\[)");
  std::string out;
  size_t last = 0;
  for (auto it = std::sregex_iterator(src.begin(), src.end(), tok); it != std::sregex_iterator(); ++it) {
    const auto& m = *it;
    ext[m[1].str()] = m[2].str() == "bf16" ? kBF16 : kI32;
    out += src.substr(last, size_t(m.position(0)) - last) + "%" + m[1].str() + ": f32[";
    last = size_t(m.position(0) + m.length(0));
  }
  out += src.substr(last);
  ir::ModuleIR mod = ir::parse_text(out);
  for (auto& [name, fn] : mod.functions) {
    for (auto& p : fn->params) {
      auto e = ext.find(p->id);
      if (e == ext.end()) continue;
      auto t = p->ty.tensor();
      t.dtype = e->second;
      p->ty = Type(t);
    }
    relink_vars(*fn);
    ir::infer_types(*fn);
  }
  return mod;
}

}  // namespace tb
