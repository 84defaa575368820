// ext_ops.hpp -- the b200 backend's additions to the reference operator
// registry, made ONLY through its public API (no reference header is edited):
//
//  * extension base ops the transformer configs need, each
//    with a type relation: OpRegistry::register_base_op (opreg.hpp:141-144)
//  * the `b200` dialect: one DialectOp{"b200", base, 20, {"cuda"}} per base op
//    libtcb200 implements: OpRegistry::register_dialect_op (opreg.hpp:146-152)
//  * two extra dtype codes, carried in the reference's DType byte
//    (dtype.hpp:45 is `enum class DType : uint8_t`): BF16 = 2, I32 = 3.
//    Byte sizes and names for them come from tb::nbytes / tb::dtype_str, not
//    from dtype_width / dtype_name (which only know F32/F16).
#pragma once

#include <cstring>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include "trainc/opreg.hpp"

namespace tb {

using namespace trainc;
using ir::AttrMap;
using opreg::BaseOp;
using opreg::DialectOp;
using opreg::OpCategory;
using opreg::OpRegistry;

inline constexpr DType kF32 = DType::F32;
inline constexpr DType kF16 = DType::F16;
inline constexpr DType kBF16 = static_cast<DType>(2);
inline constexpr DType kI32 = static_cast<DType>(3);

inline int dtype_code(DType d) { return static_cast<int>(d); }  // == TCB_* codes
inline int dtype_bytes(DType d) { return d == kF32 || d == kI32 ? 4 : 2; }
inline const char* dtype_str(DType d) {
  switch (static_cast<int>(d)) {
    case 0: return "f32";
    case 1: return "f16";
    case 2: return "bf16";
    case 3: return "i32";
  }
  return "?";
}
inline DType dtype_from(const std::string& s) {
  if (s == "f32") return kF32;
  if (s == "f16") return kF16;
  if (s == "bf16") return kBF16;
  if (s == "i32") return kI32;
  throw TypeError("unknown dtype '" + s + "'");
}
inline bool is_half(DType d) { return d == kF16 || d == kBF16; }

inline int64_t numel(const TensorType& t) {
  int64_t n = 1;
  for (auto d : t.shape) n *= d;
  return n;
}
inline int64_t nbytes(const TensorType& t) { return numel(t) * dtype_bytes(t.dtype); }
inline int64_t nbytes(const Type& t) {
  if (t.is_tensor()) return nbytes(t.tensor());
  if (t.is_tuple()) {
    int64_t s = 0;
    for (auto& f : t.tuple().fields) s += nbytes(f);
    return s;
  }
  return 0;
}
inline std::string type_str(const TensorType& t) {
  std::string s = dtype_str(t.dtype);
  s += '[';
  for (size_t i = 0; i < t.shape.size(); ++i) s += (i ? "," : "") + std::to_string(t.shape[i]);
  return s + ']';
}
inline std::string type_str(const Type& t) {
  if (t.is_tensor()) return type_str(t.tensor());
  if (!t.is_tuple()) return "?";
  std::string s = "(";
  for (size_t i = 0; i < t.tuple().fields.size(); ++i) s += (i ? ", " : "") + type_str(t.tuple().fields[i]);
  return s + ")";
}

namespace rel {
inline TensorType T(const Type& t, const std::string& op) { return opreg::rel::expect_tensor(t, op); }
inline void need_rank(const TensorType& t, int r, const std::string& op) {
  if (t.rank() != r) throw TypeError(op + ": expected rank " + std::to_string(r) + ", got " + type_str(t));
}
inline void need_float(const TensorType& t, const std::string& op) {
  if (t.dtype == kI32) throw TypeError(op + ": float tensor required");
}
inline int64_t a_int(const AttrMap& a, const char* k, int64_t d) { return ir::attr_int(a, k, d); }
// output dtype attr "out" (default: fallback)
inline DType out_dtype(const AttrMap& a, DType fallback) {
  std::string s = ir::attr_string(a, "out", "");
  return s.empty() ? fallback : dtype_from(s);
}
}  // namespace rel

// GEMM shape rule shared by linear / matmul_t / matmul_dact
inline std::vector<int64_t> gemm_shape(const TensorType& a, const TensorType& b, int ta, int tb,
                                       const std::string& op) {
  rel::need_rank(a, 2, op);
  rel::need_rank(b, 2, op);
  int64_t M = ta ? a.shape[1] : a.shape[0];
  int64_t K = ta ? a.shape[0] : a.shape[1];
  int64_t Kb = tb ? b.shape[1] : b.shape[0];
  int64_t N = tb ? b.shape[0] : b.shape[1];
  if (K != Kb) throw TypeError(op + ": inner dimensions disagree (" + type_str(a) + " x " + type_str(b) + ")");
  if (a.dtype != b.dtype) throw TypeError(op + ": dtype mismatch without explicit cast");
  return {M, N};
}

inline void register_extension_ops(OpRegistry& r) {
  using V = std::vector<Type>;
  auto reg = [&](const char* name, int arity, OpCategory cat, opreg::TypeRel rel, bool pure = true) {
    if (r.has_base(name)) return;
    BaseOp b;
    b.name = name;
    b.arity = arity;
    b.category = cat;
    b.type_rel = std::move(rel);
    b.pure = pure;
    r.register_base_op(std::move(b));
  };
  const auto E = OpCategory::Elemwise, I = OpCategory::Injective, R = OpCategory::Reduction,
             O = OpCategory::Opaque;

  // cast to any of f32 / f16 / bf16 (the reference `cast` only knows f16/f32)
  reg("convert", 1, E, [](const V& in, const AttrMap& a) -> Type {
    auto t = rel::T(in[0], "convert");
    t.dtype = dtype_from(ir::attr_string(a, "to", "f32"));
    return t;
  });
  // zero-copy slice of the flattened input
  reg("view", 1, I, [](const V& in, const AttrMap& a) -> Type {
    auto t = rel::T(in[0], "view");
    TensorType o{t.dtype, opreg::parse_shape_attr(ir::attr_string(a, "shape"))};
    int64_t off = ir::attr_int(a, "offset", 0);
    if (off < 0 || off + numel(o) > numel(t)) throw TypeError("view: slice out of range");
    return o;
  });
  // flat 1-D concatenation (horizontal buffer fusion; elided by the VM)
  reg("concat", -1, I, [](const V& in, const AttrMap&) -> Type {
    if (in.empty()) throw TypeError("concat: no inputs");
    auto t0 = rel::T(in[0], "concat");
    int64_t n = 0;
    for (auto& x : in) {
      auto t = rel::T(x, "concat");
      if (t.dtype != t0.dtype) throw TypeError("concat: dtype mismatch");
      n += numel(t);
    }
    return TensorType{t0.dtype, {n}};
  });
  // act(x . W + b); tw: W stored [N, K]; save_preact: also return u = x.W + b
  reg("linear", 3, O, [](const V& in, const AttrMap& a) -> Type {
    auto x = rel::T(in[0], "linear"), w = rel::T(in[1], "linear"), b = rel::T(in[2], "linear");
    auto mn = gemm_shape(x, w, 0, int(rel::a_int(a, "tw", 0)), "linear");
    if (numel(b) != mn[1]) throw TypeError("linear: bias must have N elements");
    TensorType y{x.dtype, mn};
    if (rel::a_int(a, "save_preact", 0)) return TupleType{{y, y}};
    return y;
  });
  // alpha * op(A) op(B), out dtype attr
  reg("matmul_t", 2, O, [](const V& in, const AttrMap& a) -> Type {
    auto x = rel::T(in[0], "matmul_t"), y = rel::T(in[1], "matmul_t");
    auto mn = gemm_shape(x, y, int(rel::a_int(a, "ta", 0)), int(rel::a_int(a, "tb", 0)), "matmul_t");
    return TensorType{rel::out_dtype(a, x.dtype), mn};
  });
  // (op(A) op(B)) * act'(aux)
  reg("matmul_dact", 3, O, [](const V& in, const AttrMap& a) -> Type {
    auto x = rel::T(in[0], "matmul_dact"), y = rel::T(in[1], "matmul_dact"), u = rel::T(in[2], "matmul_dact");
    auto mn = gemm_shape(x, y, int(rel::a_int(a, "ta", 0)), int(rel::a_int(a, "tb", 0)), "matmul_dact");
    if (u.shape != mn) throw TypeError("matmul_dact: aux shape must equal the product's");
    return TensorType{x.dtype, mn};
  });
  // matmul_pair(a0, b0 [, aux0], a1, b1) {n0, ta0, tb0, alpha0, act0, out0, ta1, tb1, alpha1, out1}
  //   -> (matmul_t / matmul_dact of problem 0, matmul_t of problem 1): two
  //   independent GEMMs in one launch (horizontal fusion of a linear's
  //   data- and weight-gradient, which share dY)
  reg("matmul_pair", -1, O, [](const V& in, const AttrMap& a) -> Type {
    const int n0 = int(rel::a_int(a, "n0", 2));
    if ((n0 != 2 && n0 != 3) || int(in.size()) != n0 + 2) throw TypeError("matmul_pair: (a0, b0 [, aux0], a1, b1)");
    auto x0 = rel::T(in[0], "matmul_pair"), y0 = rel::T(in[1], "matmul_pair");
    auto x1 = rel::T(in[n0], "matmul_pair"), y1 = rel::T(in[n0 + 1], "matmul_pair");
    auto mn0 = gemm_shape(x0, y0, int(rel::a_int(a, "ta0", 0)), int(rel::a_int(a, "tb0", 0)), "matmul_pair");
    auto mn1 = gemm_shape(x1, y1, int(rel::a_int(a, "ta1", 0)), int(rel::a_int(a, "tb1", 0)), "matmul_pair");
    if (n0 == 3 && rel::T(in[2], "matmul_pair").shape != mn0) throw TypeError("matmul_pair: aux0 shape");
    auto od = [&](const char* k, DType d) {
      auto it = a.find(k);
      return it == a.end() ? d : dtype_from(ir::attr_string(a, k, ""));
    };
    return TupleType{{TensorType{od("out0", x0.dtype), mn0}, TensorType{od("out1", x1.dtype), mn1}}};
  });
  reg("batch_matmul", 2, O, [](const V& in, const AttrMap& a) -> Type {
    auto x = rel::T(in[0], "batch_matmul"), y = rel::T(in[1], "batch_matmul");
    rel::need_rank(x, 3, "batch_matmul");
    rel::need_rank(y, 3, "batch_matmul");
    int ta = int(rel::a_int(a, "ta", 0)), tb = int(rel::a_int(a, "tb", 0));
    if (x.shape[0] != y.shape[0]) throw TypeError("batch_matmul: batch mismatch");
    int64_t M = ta ? x.shape[2] : x.shape[1], K = ta ? x.shape[1] : x.shape[2];
    int64_t Kb = tb ? y.shape[2] : y.shape[1], N = tb ? y.shape[1] : y.shape[2];
    if (K != Kb) throw TypeError("batch_matmul: inner dimensions disagree");
    return TensorType{rel::out_dtype(a, x.dtype), {x.shape[0], M, N}};
  });
  // attention(qkv [T, 3H]) -> (ctx [T, H], probs [B*A*S, S])
  reg("attention", 1, O, [](const V& in, const AttrMap& a) -> Type {
    auto q = rel::T(in[0], "attention");
    rel::need_rank(q, 2, "attention");
    int64_t H = q.shape[1] / 3, A = rel::a_int(a, "heads", 1), S = rel::a_int(a, "seq", q.shape[0]);
    if (q.shape[1] % 3 || H % A || q.shape[0] % S) throw TypeError("attention: bad qkv/heads/seq");
    int64_t B = q.shape[0] / S;
    if (rel::a_int(a, "lse", 0)) {
      // lse=1 (flash): (ctx, per-row log-sum-exp f32 [B*A*S] [, keep bits,
      // ceil(S/32) i32 words per query row])
      TupleType t{{TensorType{q.dtype, {q.shape[0], H}}, TensorType{kF32, {B * A * S}}}};
      if (rel::a_int(a, "save_mask", 0) && ir::attr_double(a, "p", 0.0) > 0.0)
        t.fields.push_back(TensorType{kI32, {B * A * S * ((S + 31) / 32)}});
      return t;
    }
    TupleType t{{TensorType{q.dtype, {q.shape[0], H}}, TensorType{q.dtype, {B * A * S, S}}}};
    // save_mask (p > 0): the dropout keep bits, 4 i32 words per query row (S <= 128)
    if (rel::a_int(a, "save_mask", 0) && ir::attr_double(a, "p", 0.0) > 0.0) {
      if (S > 128) throw TypeError("attention: save_mask needs seq <= 128");
      t.fields.push_back(TensorType{kI32, {B * A * S * 4}});
    }
    return t;
  });
  // attention_dx(qkv, probs, dctx [, saved keep bits]) -> dqkv
  // lse=1: attention_dx(qkv, ctx, lse, dctx [, keep bits]) -> dqkv
  reg("attention_dx", -1, O, [](const V& in, const AttrMap& a) -> Type {
    if (rel::a_int(a, "lse", 0)) {
      if (in.size() != 4 && in.size() != 5) throw TypeError("attention_dx lse=1: (qkv, ctx, lse, dctx [, mask])");
      return rel::T(in[0], "attention_dx");
    }
    if (in.size() != 3 && in.size() != 4) throw TypeError("attention_dx: (qkv, probs, dctx [, mask])");
    return rel::T(in[0], "attention_dx");
  });
  // layer_norm(x, gamma, beta) -> (y, mean f32[T], rstd f32[T])
  reg("layer_norm", 3, O, [](const V& in, const AttrMap&) -> Type {
    auto x = rel::T(in[0], "layer_norm");
    int64_t H = x.shape.back(), Tn = numel(x) / H;
    if (numel(rel::T(in[1], "layer_norm")) != H) throw TypeError("layer_norm: gamma size");
    return TupleType{{x, TensorType{kF32, {Tn}}, TensorType{kF32, {Tn}}}};
  });
  // add_layer_norm(x, r, gamma, beta) -> (y, s = dropout(x) + r, mean, rstd)
  //   [, keep bits as i32 [T*H/32] (byte i = elements 8i..8i+7) with save_mask and p > 0]
  reg("add_layer_norm", 4, O, [](const V& in, const AttrMap& a) -> Type {
    auto x = rel::T(in[0], "add_layer_norm"), r = rel::T(in[1], "add_layer_norm");
    if (!(x == r)) throw TypeError("add_layer_norm: x and residual differ");
    int64_t H = x.shape.back(), Tn = numel(x) / H;
    TupleType t{{x, x, TensorType{kF32, {Tn}}, TensorType{kF32, {Tn}}}};
    if (rel::a_int(a, "save_mask", 0) && ir::attr_double(a, "p", 0.0) > 0.0) {
      if (H % 8 || numel(x) % 32) throw TypeError("add_layer_norm: save_mask needs H % 8 == 0, T*H % 32 == 0");
      t.fields.push_back(TensorType{kI32, {numel(x) / 32}});
    }
    return t;
  });
  // layer_norm_dx(s, gamma, mean, rstd, dy [, dy2]) -> (ds, dgamma, dbeta [, dx if p > 0]
  //   [, dbias = column sums of the outgoing gradient if bias_grad])
  //   (mask_in: a last input holds add_layer_norm's saved keep bits)
  reg("layer_norm_dx", -1, O, [](const V& in, const AttrMap& a) -> Type {
    const size_t nm = rel::a_int(a, "mask_in", 0) ? 1 : 0;
    if (in.size() != 5 + nm && in.size() != 6 + nm) throw TypeError("layer_norm_dx: 5 or 6 inputs (+ mask)");
    auto s = rel::T(in[0], "layer_norm_dx");
    TensorType g{kF32, {s.shape.back()}};
    TupleType t{{s, g, g}};
    if (ir::attr_double(a, "p", 0.0) > 0.0) t.fields.push_back(s);
    if (ir::attr_int(a, "bias_grad", 0)) t.fields.push_back(g);
    return t;
  });
  reg("gelu", 1, E, [](const V& in, const AttrMap&) -> Type { return rel::T(in[0], "gelu"); });
  reg("gelu_dx", 2, E, [](const V& in, const AttrMap&) -> Type { return rel::T(in[1], "gelu_dx"); });
  reg("dropout", 1, E, [](const V& in, const AttrMap&) -> Type { return rel::T(in[0], "dropout"); });
  reg("softmax", 1, O, [](const V& in, const AttrMap&) -> Type { return rel::T(in[0], "softmax"); });
  reg("softmax_dx", 2, O, [](const V& in, const AttrMap&) -> Type { return rel::T(in[0], "softmax_dx"); });
  // embedding(ids i32[...], table[V, H]) -> [..., H]
  reg("embedding", 2, I, [](const V& in, const AttrMap& a) -> Type {
    auto ids = rel::T(in[0], "embedding"), tab = rel::T(in[1], "embedding");
    if (ids.dtype != kI32) throw TypeError("embedding: ids must be i32");
    rel::need_rank(tab, 2, "embedding");
    auto shape = ids.shape;
    shape.push_back(tab.shape[1]);
    return TensorType{rel::out_dtype(a, tab.dtype), shape};
  });
  // embedding_sum(ids_0..ids_{n-1}, table_0..table_{n-1}) -> [..., H]: the
  // rounded chain (e_0 + e_1) + e_2 ... of n embedding lookups
  reg("embedding_sum", -1, I, [](const V& in, const AttrMap&) -> Type {
    const size_t n = in.size() / 2;
    if (in.size() != 2 * n || n < 2 || n > 4) throw TypeError("embedding_sum: (ids.., tables..), 2 to 4 tables");
    auto ids = rel::T(in[0], "embedding_sum"), tab = rel::T(in[n], "embedding_sum");
    rel::need_rank(tab, 2, "embedding_sum");
    for (size_t k = 0; k < n; ++k) {
      auto ik = rel::T(in[k], "embedding_sum"), tk = rel::T(in[n + k], "embedding_sum");
      if (ik.dtype != kI32 || !(ik == ids)) throw TypeError("embedding_sum: ids must be i32 of one shape");
      rel::need_rank(tk, 2, "embedding_sum");
      if (tk.shape[1] != tab.shape[1] || tk.dtype != tab.dtype) throw TypeError("embedding_sum: tables differ");
    }
    auto shape = ids.shape;
    shape.push_back(tab.shape[1]);
    return TensorType{tab.dtype, shape};
  });
  // embedding_dx(ids, dy [, base]) {rows} -> f32 [rows, H]
  reg("embedding_dx", -1, O, [](const V& in, const AttrMap& a) -> Type {
    if (in.size() != 2 && in.size() != 3) throw TypeError("embedding_dx: 2 or 3 inputs");
    auto dy = rel::T(in[1], "embedding_dx");
    return TensorType{kF32, {rel::a_int(a, "rows", 1), dy.shape.back()}};
  });
  // cross_entropy(logits [T, Vp], labels i32[T]) -> loss f32[1] (grad=0) or (loss, dlogits)
  reg("cross_entropy", 2, O, [](const V& in, const AttrMap& a) -> Type {
    auto x = rel::T(in[0], "cross_entropy"), l = rel::T(in[1], "cross_entropy");
    rel::need_rank(x, 2, "cross_entropy");
    if (l.dtype != kI32 || numel(l) != x.shape[0]) throw TypeError("cross_entropy: labels must be i32[T]");
    TensorType loss{kF32, {1}};
    if (rel::a_int(a, "grad", 0)) return TupleType{{loss, x}};
    return loss;
  });
  // adam_update_ex(p, g, m, v, step) -> (p, m, v, p_half)
  reg("adam_update_ex", 5, O, [](const V& in, const AttrMap& a) -> Type {
    auto p = rel::T(in[0], "adam_update_ex");
    for (int i = 0; i < 4; ++i)
      if (!(rel::T(in[i], "adam_update_ex") == p) || p.dtype != kF32)
        throw TypeError("adam_update_ex: master params/states must be f32 of one shape");
    TensorType h{dtype_from(ir::attr_string(a, "half", "bf16")), p.shape};
    return TupleType{{p, p, p, h}};
  });
  // rule-fused elementwise group (graph.hpp rule_fuse): inputs -> the group's
  // externally used values; otypes = "dtype:d0,d1;dtype:..." one per output
  reg("ew_closure", -1, O, [](const V& in, const AttrMap& a) -> Type {
    if (in.empty()) throw TypeError("ew_closure: no inputs");
    std::vector<TensorType> outs;
    std::string spec = ir::attr_string(a, "otypes", ""), item;
    size_t pos = 0;
    while (pos <= spec.size()) {
      size_t e = spec.find(';', pos);
      item = spec.substr(pos, e == std::string::npos ? std::string::npos : e - pos);
      if (!item.empty()) {
        const size_t c = item.find(':');
        if (c == std::string::npos) throw TypeError("ew_closure: bad otypes");
        outs.push_back(TensorType{dtype_from(item.substr(0, c)), opreg::parse_shape_attr(item.substr(c + 1))});
      }
      if (e == std::string::npos) break;
      pos = e + 1;
    }
    if (outs.empty()) throw TypeError("ew_closure: no outputs");
    if (outs.size() == 1) return outs[0];
    return TupleType{outs};
  });
  // x + value (a scalar attribute): the optimizer step counter
  reg("add_scalar", 1, E, [](const V& in, const AttrMap&) -> Type { return rel::T(in[0], "add_scalar"); });
  // constant fill (zero gradients of alignment gaps / pads)
  reg("fill", 0, E, [](const V&, const AttrMap& a) -> Type {
    return TensorType{dtype_from(ir::attr_string(a, "dtype", "f32")), opreg::parse_shape_attr(ir::attr_string(a, "shape"))};
  });
  // f32 column sums over all leading dims (bias gradients)
  // colsum(x [, labels]) {ignore_index}: f32 column sums over all leading dims;
  // with labels, rows whose label is ignore_index are skipped (they are exact
  // zeros in the cross-entropy gradient this feeds the decoder bias from)
  reg("colsum", -1, R, [](const V& in, const AttrMap&) -> Type {
    if (in.size() != 1 && in.size() != 2) throw TypeError("colsum: (x [, labels])");
    auto x = rel::T(in[0], "colsum");
    if (in.size() == 2) {
      auto l = rel::T(in[1], "colsum");
      if (l.dtype != kI32 || numel(l) * x.shape.back() != numel(x)) throw TypeError("colsum: labels i32 [rows]");
    }
    return TensorType{kF32, {x.shape.back()}};
  });
}

// Ops the VM executes itself (no kernel): arena aliases and collectives.
inline bool is_alias_op(const std::string& base) {
  return base == "view" || base == "reshape" || base == "concat";
}

/// Register the b200 dialect for every base op in `ops` (the list libtcb200
/// reports through tcb_supported_ops) plus the collectives, which the VM routes
/// to NCCL.  Priority 20 beats opt (12) and ref (5); device gate "cuda".
inline void register_b200_dialect(OpRegistry& r, const std::vector<std::string>& ops) {
  static const char* kCollectives[] = {"allreduce", "reduce_scatter", "all_gather", "shard",
                                       "reduce_scatter_batched", "all_gather_batched"};
  auto add = [&](const std::string& op) {
    if (!r.has_base(op) || r.find_dialect("b200." + op)) return;
    DialectOp d;
    d.dialect = "b200";
    d.base = op;
    d.priority = 20;
    d.device_gate = {"cuda"};
    r.register_dialect_op(std::move(d));
  };
  for (auto& op : ops) add(op);
  for (auto* c : kCollectives) add(c);
}

/// Process-wide registration before any compile (the registry is "built once,
/// then read-only").  Idempotent and additive: the registry is
/// a process-unique object shared by every library that includes opreg.hpp
/// (its static is emitted as a unique symbol), so a CPU-only user (the oracle
/// interpreter, which registers no dialect) and the device runtime can load in
/// either order.
inline void ensure_registered(const std::vector<std::string>& b200_ops) {
  static std::mutex mu;
  std::lock_guard<std::mutex> g(mu);
  register_extension_ops(opreg::registry());
  register_b200_dialect(opreg::registry(), b200_ops);
}

inline std::vector<std::string> split_ws(const std::string& s) {
  std::vector<std::string> out;
  std::istringstream is(s);
  std::string w;
  while (is >> w) out.push_back(w);
  return out;
}

}  // namespace tb
