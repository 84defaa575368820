// k_transformer.cu -- the memory-bound transformer ops the reference lacks
// (SURVEY.md §2.4 / §8a A15): softmax / softmax_dx (layer_norm and
// layer_norm_dx live in k_layernorm*.cu), the attention fwd/bwd closures (tcgen05
// GEMMs on strided head views + row softmax), embedding gather / deterministic
// scatter-add, and the fused cross-entropy loss + gradient.
//
// Row kernels use one warp per row with 16-byte vector loads when the row length
// allows, f32 statistics and warp-shuffle reductions; the oracle (oracle.c) has
// the same formulas with sequential sums (tolerance-checked, not bit-exact).
#include "k_rowops.cuh"

namespace tcb {

// ------------------------------------------------------------------ softmax
// rows of length C; v = x*scale (causal: -inf for col > row % Sq); P = softmax;
// optional Pd = dropout(P) (index = row*C + col).  One warp per row.
constexpr int SM_MAXV = 32;  // up to 32 values per lane: C <= 1024

// 4 consecutive elements (vector access when the row is 4-element aligned)
template <typename T>
__device__ __forceinline__ void ld4(const T* p, int64_t i, int64_t lim, bool vec, float* f) {
  if (vec) {
    if constexpr (sizeof(T) == 4) {
      float4 a = *reinterpret_cast<const float4*>(p + i);
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    } else {
      uint2 q = *reinterpret_cast<const uint2*>(p + i);
      const T* h = reinterpret_cast<const T*>(&q);
#pragma unroll
      for (int k = 0; k < 4; ++k) f[k] = to_f(h[k]);
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k) f[k] = i + k < lim ? to_f(p[i + k]) : 0.0f;
  }
}
template <typename T>
__device__ __forceinline__ void st4(T* p, int64_t i, int64_t lim, bool vec, const float* f) {
  if (vec) {
    if constexpr (sizeof(T) == 4) {
      *reinterpret_cast<float4*>(p + i) = make_float4(f[0], f[1], f[2], f[3]);
    } else {
      uint2 q;
      T* h = reinterpret_cast<T*>(&q);
#pragma unroll
      for (int k = 0; k < 4; ++k) h[k] = from_f<T>(f[k]);
      *reinterpret_cast<uint2*>(p + i) = q;
    }
  } else {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i + k < lim) p[i + k] = from_f<T>(f[k]);
  }
}

// One warp per row; lane owns NQ quads of 4 adjacent columns (C <= 128*NQ),
// so the row lives in registers and one Philox call covers a quad's 4 keep bits.
template <typename TI, typename TO, int NQ>
__global__ void __launch_bounds__(256) k_softmax(const TI* __restrict__ x, TO* __restrict__ P,
                                                 TO* __restrict__ Pd, int64_t rows, int C, int Sq,
                                                 float scale, int causal, DropCfg d, bool vec) {
  TCB_PDL_ENTRY();
  drop_resolve(d);
  constexpr int RW = NQ == 1 ? 4 : NQ == 2 ? 2 : 1;  // rows per warp, loads batched
  const int lane = threadIdx.x & 31;
  const int64_t row0 = (blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5)) * RW;
  if (row0 >= rows) return;
  float v[RW][NQ][4];
#pragma unroll
  for (int q = 0; q < RW; ++q)
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      const int j0 = (c * 32 + lane) * 4;
      const int64_t base = (row0 + q) * C;
      if (row0 + q < rows && j0 < C) ld4(x, base + j0, base + C, vec, v[q][c]);
    }
  float m[RW], sum[RW];
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    const int qi = int((row0 + q) % Sq);
    m[q] = -INFINITY;
#pragma unroll
    for (int c = 0; c < NQ; ++c)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int j = (c * 32 + lane) * 4 + k;
        float t = (j < C) ? v[q][c][k] * scale : -INFINITY;
        if (causal && j > qi) t = -INFINITY;
        v[q][c][k] = t;
        m[q] = fmaxf(m[q], t);
      }
  }
#pragma unroll
  for (int q = 0; q < RW; ++q) m[q] = warp_max(m[q]);
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    sum[q] = 0.0f;
#pragma unroll
    for (int c = 0; c < NQ; ++c)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        v[q][c][k] = v[q][c][k] == -INFINITY ? 0.0f : expf(v[q][c][k] - m[q]);
        sum[q] += v[q][c][k];
      }
  }
#pragma unroll
  for (int q = 0; q < RW; ++q) sum[q] = warp_sum(sum[q]);
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    if (row0 + q >= rows) break;
    const int64_t base = (row0 + q) * C, lim = base + C;
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      const int j0 = (c * 32 + lane) * 4;
      if (j0 >= C) continue;
      float o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = to_f(from_f<TO>(v[q][c][k] / sum[q]));
      st4(P, base + j0, lim, vec, o);
      if (Pd) {
        const uint32_t bits = dropout_bits4(d, uint64_t(base + j0));
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = ((bits >> k) & 1u) ? o[k] * d.scale : 0.0f;
        st4(Pd, base + j0, lim, vec, o);
      }
    }
  }
}

// dS = P * (dP - rowdot(P, dP)) * scale with dP = dropout(dPd); optional Pd out
template <typename TP, typename TG, typename TO, int NQ>
__global__ void __launch_bounds__(256) k_softmax_bwd(const TP* __restrict__ P, const TG* __restrict__ dPd,
                                                     TO* __restrict__ dS, TO* __restrict__ Pd_o, int64_t rows,
                                                     int C, float scale, DropCfg d, bool vec) {
  TCB_PDL_ENTRY();
  drop_resolve(d);
  constexpr int RW = NQ == 1 ? 4 : NQ == 2 ? 2 : 1;
  const int lane = threadIdx.x & 31;
  const int64_t row0 = (blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5)) * RW;
  if (row0 >= rows) return;
  float pv[RW][NQ][4], dp[RW][NQ][4];
#pragma unroll
  for (int q = 0; q < RW; ++q)
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      const int j0 = (c * 32 + lane) * 4;
      const int64_t base = (row0 + q) * C;
#pragma unroll
      for (int k = 0; k < 4; ++k) pv[q][c][k] = dp[q][c][k] = 0.0f;
      if (row0 + q < rows && j0 < C) {
        ld4(P, base + j0, base + C, vec, pv[q][c]);
        ld4(dPd, base + j0, base + C, vec, dp[q][c]);
      }
    }
  float dot[RW];
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    dot[q] = 0.0f;
    const int64_t base = (row0 + q) * C;
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      const int j0 = (c * 32 + lane) * 4;
      if (row0 + q >= rows || j0 >= C) continue;
      const uint32_t bits = dropout_bits4(d, uint64_t(base + j0));
      float pdv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const bool keep = (bits >> k) & 1u;
        dp[q][c][k] = keep ? dp[q][c][k] * d.scale : 0.0f;
        pdv[k] = keep ? pv[q][c][k] * d.scale : 0.0f;
        dot[q] += pv[q][c][k] * dp[q][c][k];
      }
      if (Pd_o) st4(Pd_o, base + j0, base + C, vec, pdv);
    }
  }
#pragma unroll
  for (int q = 0; q < RW; ++q) dot[q] = warp_sum(dot[q]);
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    if (row0 + q >= rows) break;
    const int64_t base = (row0 + q) * C;
#pragma unroll
    for (int c = 0; c < NQ; ++c) {
      const int j0 = (c * 32 + lane) * 4;
      if (j0 >= C) continue;
      float o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = pv[q][c][k] * (dp[q][c][k] - dot[q]) * scale;
      st4(dS, base + j0, base + C, vec, o);
    }
  }
}

// NQ = ceil(C / 128) in {1, 2, 4, 8}
template <typename Fn>
static void dispatch_nq(int C, Fn&& f) {
  const int nq = (C + 127) / 128;
  if (nq <= 1) f(std::integral_constant<int, 1>{});
  else if (nq <= 2) f(std::integral_constant<int, 2>{});
  else if (nq <= 4) f(std::integral_constant<int, 4>{});
  else if (nq <= 8) f(std::integral_constant<int, 8>{});
  else fail(TCB_ERR_UNIMPLEMENTED, "softmax: row length > 1024 unsupported");
}

// grid for the softmax kernels: 8 warps per CTA, RW(NQ) rows per warp
template <int NQ>
static unsigned sm_grid(int64_t rows) {
  constexpr int RW = NQ == 1 ? 4 : NQ == 2 ? 2 : 1;
  return unsigned((rows + 8 * RW - 1) / (8 * RW));
}

template <typename Fn>
static void dispatch2(int a, int b, Fn&& f) {
  dispatch_float(a, [&](auto* pa) { dispatch_float(b, [&](auto* pb) { f(pa, pb); }); });
}

static void b_softmax(Plan& p) {
  check_arity(p, 1, 1, 1, 2);
  const Spec& X = p.in[0];
  const int C = int(X.dim(-1));
  require(C <= SM_MAXV * 32, "softmax: row length > 1024 unsupported");
  const int64_t rows = X.numel() / C;
  const int Sq = X.rank >= 2 ? int(X.dim(-2)) : 1;
  const float scale = float(p.attrs.f("scale", 1.0));
  const int causal = int(p.attrs.i("causal", 0));
  const DropCfg d = drop_cfg(p.attrs);
  dispatch2(X.dtype, p.out[0].dtype, [&](auto* pa, auto* pb) {
   using TI = std::remove_pointer_t<decltype(pa)>;
   using TO = std::remove_pointer_t<decltype(pb)>;
   dispatch_nq(C, [&](auto nq) {
    constexpr int NQ = decltype(nq)::value;
    const bool pd = p.out.size() > 1;
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      const bool vec = C % 4 == 0 && reinterpret_cast<uintptr_t>(in[0].ptr) % 16 == 0 &&
                       reinterpret_cast<uintptr_t>(out[0].ptr) % 16 == 0 &&
                       (!pd || reinterpret_cast<uintptr_t>(out[1].ptr) % 16 == 0);
      launch_k(k_softmax<TI, TO, NQ>, sm_grid<NQ>(rows), 256, 0, s, 
          (const TI*)in[0].ptr, (TO*)out[0].ptr, pd ? (TO*)out[1].ptr : nullptr, rows, C, Sq, scale, causal, with_step(d), vec);
    };
   });
  });
}
TCB_REGISTER("softmax", b_softmax);

static void b_softmax_dx(Plan& p) {
  check_arity(p, 2, 2, 1, 1);
  const Spec& Y = p.in[0];
  const int C = int(Y.dim(-1));
  require(C <= SM_MAXV * 32, "softmax_dx: row length > 1024 unsupported");
  const int64_t rows = Y.numel() / C;
  const float scale = float(p.attrs.f("scale", 1.0));
  DropCfg d;  // no dropout on the standalone op
  const int dg = p.in[1].dtype;
  dispatch2(Y.dtype, p.out[0].dtype, [&](auto* pa, auto* pb) {
    using TP = std::remove_pointer_t<decltype(pa)>;
    using TO = std::remove_pointer_t<decltype(pb)>;
    dispatch_float(dg, [&](auto* pg) {
     using TG = std::remove_pointer_t<decltype(pg)>;
     dispatch_nq(C, [&](auto nq) {
      constexpr int NQ = decltype(nq)::value;
      p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
        const bool vec = C % 4 == 0 && reinterpret_cast<uintptr_t>(in[0].ptr) % 16 == 0 &&
                         reinterpret_cast<uintptr_t>(in[1].ptr) % 16 == 0 &&
                         reinterpret_cast<uintptr_t>(out[0].ptr) % 16 == 0;
        launch_k(k_softmax_bwd<TP, TG, TO, NQ>, sm_grid<NQ>(rows), 256, 0, s, 
            (const TP*)in[0].ptr, (const TG*)in[1].ptr, (TO*)out[0].ptr, nullptr, rows, C, scale, d, vec);
      };
     });
    });
  });
}
TCB_REGISTER("softmax_dx", b_softmax_dx);

// ---------------------------------------------------------------- attention
// qkv [T, 3H] with T = B*S; heads A, dh = H/A.  Head (b, h) of Q/K/V is a
// strided [S, dh] view (row stride 3H) -- consumed directly by the GEMM tensor
// maps, no head split/merge copies.
struct AttnGeom {
  int64_t B, S, A, H, dh, Z;
  float scale;
  int causal;
  DropCfg d;
  int dt;
  bool exact;
};

static AttnGeom attn_geom(const Plan& p, bool any_len = false) {
  const Spec& X = p.in[0];
  require(X.rank == 2 && X.shape[1] % 3 == 0, p.op + ": qkv must be [T, 3H]");
  AttnGeom g;
  g.H = X.shape[1] / 3;
  g.A = p.attrs.i("heads", 1);
  g.S = p.attrs.i("seq", X.shape[0]);
  require(g.A >= 1 && g.H % g.A == 0, p.op + ": heads must divide H");
  require(g.S >= 1 && X.shape[0] % g.S == 0, p.op + ": seq must divide T");
  require(any_len || g.S <= SM_MAXV * 32, p.op + ": seq > 1024 unsupported");
  g.B = X.shape[0] / g.S;
  g.dh = g.H / g.A;
  g.Z = g.B * g.A;
  g.scale = float(p.attrs.f("scale", 1.0 / std::sqrt(double(g.dh))));
  g.causal = int(p.attrs.i("causal", 0));
  g.d = drop_cfg(p.attrs);
  g.dt = X.dtype;
  g.exact = X.dtype == TCB_F32 || p.attrs.i("exact", 0) != 0;
  return g;
}

// operand view of part `part` (0 q, 1 k, 2 v) of qkv for batch z = (b, h)
static GemmOperand qkv_view(const AttnGeom& g, const void* qkv, int part) {
  GemmOperand o;
  o.ptr = static_cast<const char*>(qkv) + size_t(part) * g.H * dtype_bytes(g.dt);
  o.ld = 3 * g.H;
  o.s1 = g.S * 3 * g.H;
  o.s2 = g.dh;
  o.dtype = g.dt;
  return o;
}
static GemmOperand sq_view(const AttnGeom& g, const void* p, int dt) {  // [Z, S, S]
  GemmOperand o;
  o.ptr = p;
  o.ld = g.S;
  o.s1 = g.A * g.S * g.S;
  o.s2 = g.S * g.S;
  o.dtype = dt;
  return o;
}
static GemmOperand ctx_view(const AttnGeom& g, const void* p) {  // [T, H] head views
  GemmOperand o;
  o.ptr = p;
  o.ld = g.H;
  o.s1 = g.S * g.H;
  o.s2 = g.dh;
  o.dtype = g.dt;
  return o;
}
static GemmArgs attn_gemm(const AttnGeom& g, int64_t M, int64_t N, int64_t K, GemmOperand a, int ta,
                          GemmOperand b, int tb) {
  GemmArgs r;
  r.M = M;
  r.N = N;
  r.K = K;
  r.Z = g.Z;
  r.Z2 = g.A;
  r.a = a;
  r.b = b;
  r.ta = ta;
  r.tb = tb;
  return r;
}
static void set_c(GemmArgs& r, void* c, int64_t ld, int64_t s1, int64_t s2, int dt) {
  r.c = c;
  r.ldc = ld;
  r.c_s1 = s1;
  r.c_s2 = s2;
  r.c_dtype = dt;
}

// attention(qkv) {lse=1} -> (ctx [T,H], lse f32 [Z*S] [, keep bits i32 [Z*S*ceil(S/32)]]):
// the flash kernels of k_flash.cu (any S % 8 == 0, head dim 64, bf16)
static void b_attention_lse(Plan& p) {
  check_arity(p, 1, 1, 2, 3);
  const AttnGeom g = attn_geom(p, true);
  if (!flash_ok(g.dt, g.S, g.H, g.A) || g.exact)
    fail(TCB_ERR_UNIMPLEMENTED, "attention lse=1: needs bf16, head dim 64, seq % 8 == 0");
  require(p.out[0].numel() == g.B * g.S * g.H && p.out[0].dtype == g.dt, "attention: ctx must be [T, H]");
  require(p.out[1].numel() == g.Z * g.S && p.out[1].dtype == TCB_F32, "attention lse=1: lse must be f32 [B*A*S]");
  const bool save_mask = p.out.size() > 2;
  const int64_t nw = (g.S + 31) / 32;
  if (save_mask)
    require(g.d.p > 0.0f && p.out[2].numel() * dtype_bytes(p.out[2].dtype) >= g.Z * g.S * nw * 4,
            "attention: save_mask needs p > 0 and ceil(S/32) words per query row");
  // S <= 128: the persistent per-head kernels (k_attention.cu) in lse mode --
  // measured faster there than the flash grid; longer sequences: flash
  const bool persistent = attn_fused_ok(g.dt, g.S, g.H, g.A, g.exact) && !p.attrs.i("flash_kernel", 0);
  p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    DropCfg d = with_step(g.d);
    if (save_mask) d.mask_out = static_cast<uint8_t*>(out[2].ptr);
    if (persistent)
      launch_attn_fwd(in[0].ptr, out[0].ptr, nullptr, g.B, g.S, g.H, g.A, g.scale, g.causal, d, s, nullptr,
                      static_cast<float*>(out[1].ptr));
    else
      launch_flash_fwd(in[0].ptr, out[0].ptr, static_cast<float*>(out[1].ptr), g.B, g.S, g.H, g.A, g.scale,
                       g.causal, d, s);
  };
}

// attention_dx(qkv, ctx, lse, dctx [, keep bits]) {lse=1} -> dqkv
static void b_attention_dx_lse(Plan& p) {
  check_arity(p, 4, 5, 1, 1);
  const AttnGeom g = attn_geom(p, true);
  if (!flash_ok(g.dt, g.S, g.H, g.A) || g.exact)
    fail(TCB_ERR_UNIMPLEMENTED, "attention_dx lse=1: needs bf16, head dim 64, seq % 8 == 0");
  require(p.in[1].numel() == g.B * g.S * g.H && p.in[1].dtype == g.dt, "attention_dx: ctx must be [T, H]");
  require(p.in[2].numel() == g.Z * g.S && p.in[2].dtype == TCB_F32, "attention_dx: lse must be f32 [B*A*S]");
  require(p.in[3].numel() == g.B * g.S * g.H && p.in[3].dtype == g.dt, "attention_dx: dctx must be [T, H]");
  require(p.out[0].numel() == p.in[0].numel(), "attention_dx: dqkv must be [T, 3H]");
  const bool mask_in = p.in.size() > 4;
  const int64_t nt = (g.S + 127) / 128;
  const size_t dq = p.ws_take(nt > 1 ? size_t(g.B * g.S * g.H) * sizeof(float) : 0);
  p.nkernels = nt > 1 ? 2 : 1;  // (+ a memset node) the dQ f32 -> bf16 store
  const bool persistent = attn_fused_ok(g.dt, g.S, g.H, g.A, g.exact) && !p.attrs.i("flash_kernel", 0);
  p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    DropCfg d = with_step(g.d);
    if (mask_in) d.mask_in = static_cast<const uint8_t*>(in[4].ptr);
    if (persistent) {
      launch_attn_bwd(in[0].ptr, nullptr, in[3].ptr, out[0].ptr, g.B, g.S, g.H, g.A, g.scale, g.causal, d, s,
                      static_cast<const float*>(in[2].ptr));
      return;
    }
    launch_flash_bwd(in[0].ptr, in[1].ptr, static_cast<const float*>(in[2].ptr), in[3].ptr, out[0].ptr,
                     nt > 1 ? static_cast<float*>(ws_at(dq)) : nullptr, g.B, g.S, g.H, g.A, g.scale, g.causal, d, s);
  };
}

// attention(qkv) -> (ctx [T,H], probs [Z*S, S])
static void b_attention(Plan& p) {
  if (p.attrs.i("lse", 0)) return b_attention_lse(p);
  check_arity(p, 1, 1, 2, 3);
  const AttnGeom g = attn_geom(p);
  require(p.out[0].numel() == g.B * g.S * g.H, "attention: ctx must be [T, H]");
  require(p.out[1].numel() == g.Z * g.S * g.S, "attention: probs must be [B*A*S, S]");
  // save_mask: a third output keeps the dropout bits, 4 words per query row
  const bool save_mask = p.out.size() > 2;
  const bool fused = attn_fused_ok(g.dt, g.S, g.H, g.A, g.exact) && !p.attrs.i("unfused", 0);
  if (save_mask) {
    if (!fused) fail(TCB_ERR_UNIMPLEMENTED, "attention: save_mask needs the fused kernel");
    require(g.d.p > 0.0f && p.out[2].numel() * dtype_bytes(p.out[2].dtype) >= g.Z * g.S * 16,
            "attention: save_mask needs p > 0 and a Z*S*4-word mask");
  }
  if (fused) {
    void* trace = reinterpret_cast<void*>(p.attrs.i("tc_trace", 0));  // tooling only
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      DropCfg d = with_step(g.d);
      if (save_mask) d.mask_out = static_cast<uint8_t*>(out[2].ptr);
      launch_attn_fwd(in[0].ptr, out[0].ptr, out[1].ptr, g.B, g.S, g.H, g.A, g.scale, g.causal, d, s, trace);
    };
    return;
  }
  const size_t nsq = size_t(g.Z) * g.S * g.S;
  const size_t scores = p.ws_take(nsq * 4);
  const size_t pd = p.ws_take(g.d.p > 0.0f ? nsq * dtype_bytes(g.dt) : 0);
  p.nkernels = 3;
  dispatch_float(g.dt, [&](auto* tp) {
    using T = std::remove_pointer_t<decltype(tp)>;
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      // 1. scores = scale * Q K^T (f32)
      GemmArgs q = attn_gemm(g, g.S, g.S, g.dh, qkv_view(g, in[0].ptr, 0), 0, qkv_view(g, in[0].ptr, 1), 1);
      q.alpha = g.scale;
      set_c(q, ws_at(scores), g.S, g.A * g.S * g.S, g.S * g.S, TCB_F32);
      launch_gemm(q, g.exact, s);
      // 2. P = softmax(scores) (+ dropout copy)
      const int64_t rows = g.Z * g.S;
      T* Pd = g.d.p > 0.0f ? (T*)ws_at(pd) : nullptr;
      dispatch_nq(int(g.S), [&](auto nq) {
        launch_k(k_softmax<float, T, decltype(nq)::value>, sm_grid<decltype(nq)::value>(rows), 256, 0, s, 
            (const float*)ws_at(scores), (T*)out[1].ptr, Pd, rows, int(g.S), int(g.S), 1.0f, g.causal, with_step(g.d),
            g.S % 4 == 0 && reinterpret_cast<uintptr_t>(out[1].ptr) % 16 == 0);
      });
      // 3. ctx = Pd V
      GemmArgs c = attn_gemm(g, g.S, g.dh, g.S, sq_view(g, Pd ? (const void*)Pd : out[1].ptr, g.dt), 0,
                             qkv_view(g, in[0].ptr, 2), 0);
      set_c(c, out[0].ptr, g.H, g.S * g.H, g.dh, g.dt);
      launch_gemm(c, g.exact, s);
    };
  });
}
TCB_REGISTER("attention", b_attention);

// attention_dx(qkv, probs, dctx) -> dqkv [T, 3H]
static void b_attention_dx(Plan& p) {
  if (p.attrs.i("lse", 0)) return b_attention_dx_lse(p);
  check_arity(p, 3, 4, 1, 1);
  const AttnGeom g = attn_geom(p);
  require(p.out[0].numel() == p.in[0].numel(), "attention_dx: dqkv must be [T, 3H]");
  const bool mask_in = p.in.size() > 3;  // the forward's saved keep bits
  const bool fused = attn_fused_ok(g.dt, g.S, g.H, g.A, g.exact) && !p.attrs.i("unfused", 0);
  if (mask_in && !fused) fail(TCB_ERR_UNIMPLEMENTED, "attention_dx: a saved mask needs the fused kernel");
  if (fused) {
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      DropCfg d = with_step(g.d);
      if (mask_in) d.mask_in = static_cast<const uint8_t*>(in[3].ptr);
      launch_attn_bwd(in[0].ptr, in[1].ptr, in[2].ptr, out[0].ptr, g.B, g.S, g.H, g.A, g.scale, g.causal, d, s);
    };
    return;
  }
  const size_t nsq = size_t(g.Z) * g.S * g.S;
  const size_t dpd = p.ws_take(nsq * 4);
  const size_t ds = p.ws_take(nsq * dtype_bytes(g.dt));
  const size_t pd = p.ws_take(g.d.p > 0.0f ? nsq * dtype_bytes(g.dt) : 0);
  p.nkernels = 5;
  dispatch_float(g.dt, [&](auto* tp) {
    using T = std::remove_pointer_t<decltype(tp)>;
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      const void* qkv = in[0].ptr;
      // 1. dPd = dctx V^T (f32)
      GemmArgs a = attn_gemm(g, g.S, g.S, g.dh, ctx_view(g, in[2].ptr), 0, qkv_view(g, qkv, 2), 1);
      set_c(a, ws_at(dpd), g.S, g.A * g.S * g.S, g.S * g.S, TCB_F32);
      launch_gemm(a, g.exact, s);
      // 2. dS = P (dP - rowdot) * scale ; Pd
      const int64_t rows = g.Z * g.S;
      T* Pd = g.d.p > 0.0f ? (T*)ws_at(pd) : nullptr;
      dispatch_nq(int(g.S), [&](auto nq) {
        launch_k(k_softmax_bwd<T, float, T, decltype(nq)::value>, sm_grid<decltype(nq)::value>(rows), 256, 0, s, 
            (const T*)in[1].ptr, (const float*)ws_at(dpd), (T*)ws_at(ds), Pd, rows, int(g.S), g.scale, with_step(g.d),
            g.S % 4 == 0 && reinterpret_cast<uintptr_t>(in[1].ptr) % 16 == 0);
      });
      char* dq = static_cast<char*>(out[0].ptr);
      const size_t part = size_t(g.H) * dtype_bytes(g.dt);
      // 3. dQ = dS K
      GemmArgs b = attn_gemm(g, g.S, g.dh, g.S, sq_view(g, ws_at(ds), g.dt), 0, qkv_view(g, qkv, 1), 0);
      set_c(b, dq, 3 * g.H, g.S * 3 * g.H, g.dh, g.dt);
      launch_gemm(b, g.exact, s);
      // 4. dK = dS^T Q
      GemmArgs c = attn_gemm(g, g.S, g.dh, g.S, sq_view(g, ws_at(ds), g.dt), 1, qkv_view(g, qkv, 0), 0);
      set_c(c, dq + part, 3 * g.H, g.S * 3 * g.H, g.dh, g.dt);
      launch_gemm(c, g.exact, s);
      // 5. dV = Pd^T dctx
      GemmArgs v = attn_gemm(g, g.S, g.dh, g.S, sq_view(g, Pd ? (const void*)Pd : in[1].ptr, g.dt), 1,
                             ctx_view(g, in[2].ptr), 0);
      set_c(v, dq + 2 * part, 3 * g.H, g.S * 3 * g.H, g.dh, g.dt);
      launch_gemm(v, g.exact, s);
    };
  });
}
TCB_REGISTER("attention_dx", b_attention_dx);

// ---------------------------------------------------------------- embedding
template <typename TT, typename TO>
__global__ void k_embed(const int32_t* __restrict__ ids, const TT* __restrict__ table, TO* __restrict__ out,
                        int64_t T, int64_t H, int64_t V, int* __restrict__ err) {
  TCB_PDL_ENTRY();
  const int64_t t = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= T) return;
  const int32_t id = ids[t];
  if (id < 0 || id >= V) {
    if (lane == 0) atomicExch(err, 1);
    return;
  }
  for (int64_t j = lane; j < H; j += 32) out[t * H + j] = from_f<TO>(to_f(table[int64_t(id) * H + j]));
}

static void b_embedding(Plan& p) {
  check_arity(p, 2, 2, 1, 1);
  require(p.in[0].dtype == TCB_I32, "embedding: ids must be i32");
  require(p.in[1].rank == 2, "embedding: table must be rank 2");
  const int64_t T = p.in[0].numel(), V = p.in[1].shape[0], H = p.in[1].shape[1];
  require(p.out[0].numel() == T * H, "embedding: output must be [T, H]");
  auto err = std::make_shared<Scratch>(4);
  TCB_CUDA(cudaMemset(err->p, 0, 4));
  dispatch2(p.in[1].dtype, p.out[0].dtype, [&](auto* pa, auto* pb) {
    using TT = std::remove_pointer_t<decltype(pa)>;
    using TO = std::remove_pointer_t<decltype(pb)>;
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      launch_k(k_embed<TT, TO>, unsigned((T + 7) / 8), 256, 0, s, (const int32_t*)in[0].ptr, (const TT*)in[1].ptr,
                                                             (TO*)out[0].ptr, T, H, V, (int*)err->p);
    };
  });
}
TCB_REGISTER("embedding", b_embedding);

// embedding_sum(ids_0..ids_{n-1}, table_0..table_{n-1}) = (e_0 + e_1) + e_2 ...
// with the sum rounded to the tables' dtype after every add -- exactly the
// embedding / add chain it replaces (BERT: word + position + token type), one
// warp per token, 16-byte row chunks.
struct EmbSumArgs {
  const int32_t* ids[4];
  const void* tab[4];
  int64_t V[4];
  int n;
};
template <typename T>
__global__ void __launch_bounds__(256) k_embed_sum(const EmbSumArgs a, T* __restrict__ out, int64_t Tn, int64_t H,
                                                   int* __restrict__ err, bool vec) {
  TCB_PDL_ENTRY();
  const int64_t t = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (t >= Tn) return;
  int64_t row[4];
  for (int k = 0; k < a.n; ++k) {
    const int32_t id = a.ids[k][t];
    if (id < 0 || id >= a.V[k]) {
      if (lane == 0) atomicExch(err, 1);
      return;
    }
    row[k] = int64_t(id) * H;
  }
  if (vec) {
    for (int64_t c = lane; c < H / 8; c += 32) {
      float acc[8];
      unpack8<T>(*reinterpret_cast<const uint4*>(static_cast<const T*>(a.tab[0]) + row[0] + c * 8), acc);
      for (int k = 1; k < a.n; ++k) {
        float f[8];
        unpack8<T>(*reinterpret_cast<const uint4*>(static_cast<const T*>(a.tab[k]) + row[k] + c * 8), f);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc[e] = to_f(from_f<T>(__fadd_rn(acc[e], f[e])));
      }
      *reinterpret_cast<uint4*>(out + t * H + c * 8) = pack8<T>(acc);
    }
  } else {
    for (int64_t j = lane; j < H; j += 32) {
      float acc = to_f(static_cast<const T*>(a.tab[0])[row[0] + j]);
      for (int k = 1; k < a.n; ++k) acc = to_f(from_f<T>(__fadd_rn(acc, to_f(static_cast<const T*>(a.tab[k])[row[k] + j]))));
      out[t * H + j] = from_f<T>(acc);
    }
  }
}

static void b_embedding_sum(Plan& p) {
  const int n = int(p.in.size()) / 2;
  require(int(p.in.size()) == 2 * n && n >= 2 && n <= 4, "embedding_sum: (ids_0.., table_0..), 2 to 4 tables");
  check_arity(p, 2 * n, 2 * n, 1, 1);
  const int64_t Tn = p.in[0].numel(), H = p.in[n].shape[1];
  const int dt = p.in[n].dtype;
  for (int k = 0; k < n; ++k) {
    require(p.in[k].dtype == TCB_I32 && p.in[k].numel() == Tn, "embedding_sum: ids must be i32 of one shape");
    require(p.in[n + k].rank == 2 && p.in[n + k].shape[1] == H && p.in[n + k].dtype == dt,
            "embedding_sum: tables must be [V_k, H] of one dtype");
  }
  require(p.out[0].dtype == dt && p.out[0].numel() == Tn * H, "embedding_sum: output is [T, H] in the tables' dtype");
  require(dt == TCB_BF16 || dt == TCB_F16, "embedding_sum: 16-bit tables");
  auto err = std::make_shared<Scratch>(4);
  TCB_CUDA(cudaMemset(err->p, 0, 4));
  std::vector<int64_t> V(n);
  for (int k = 0; k < n; ++k) V[k] = p.in[n + k].shape[0];
  auto launch = [=](auto* tp, const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    using T = std::remove_pointer_t<decltype(tp)>;
    EmbSumArgs a{};
    a.n = n;
    bool vec = H % 8 == 0 && reinterpret_cast<uintptr_t>(out[0].ptr) % 16 == 0;
    for (int k = 0; k < n; ++k) {
      a.ids[k] = static_cast<const int32_t*>(in[k].ptr);
      a.tab[k] = in[n + k].ptr;
      a.V[k] = V[k];
      vec = vec && reinterpret_cast<uintptr_t>(in[n + k].ptr) % 16 == 0;
    }
    launch_k(k_embed_sum<T>, unsigned((Tn + 7) / 8), 256, 0, s, a, static_cast<T*>(out[0].ptr), Tn, H, (int*)err->p,
             vec);
  };
  p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    if (dt == TCB_BF16) launch(static_cast<__nv_bfloat16*>(nullptr), in, out, s);
    else launch(static_cast<__half*>(nullptr), in, out, s);
  };
}
TCB_REGISTER("embedding_sum", b_embedding_sum);

// Deterministic scatter-add: the tokens are stably sorted by id (LSD radix
// sort, 8-bit digits, ties in ascending t), then every chunk of <= EMB_CHUNK
// equal ids accumulates its rows in ascending t onto base -- the oracle's
// order exactly for segments of <= EMB_CHUNK rows, so f32 results are
// bit-identical; longer segments fold their chunk sums in chunk order.
// O(T) work per pass (the earlier pairwise rank was O(T^2): 0.56 s per launch
// at T = 1.1M tokens, the remat max batch).
constexpr int RDX_TILE = 2048;  // keys per block: 8 warps x 8 rounds x 32 lanes
constexpr int RDX_WARPS = 8, RDX_ROUNDS = RDX_TILE / (RDX_WARPS * 32);

// per-tile histogram of digit (key >> shift) & 255 -> counts[digit][tile]
__global__ void __launch_bounds__(256) k_radix_count(const int32_t* __restrict__ keys, int64_t T, int shift,
                                                     int32_t* __restrict__ counts, int ntiles) {
  TCB_PDL_ENTRY();
  __shared__ int32_t h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t t0 = int64_t(blockIdx.x) * RDX_TILE;
  for (int e = threadIdx.x; e < RDX_TILE; e += 256)
    if (t0 + e < T) atomicAdd(&h[(keys[t0 + e] >> shift) & 255], 1);
  __syncthreads();
  counts[int64_t(threadIdx.x) * ntiles + blockIdx.x] = h[threadIdx.x];
}

// exclusive scan of n counts in place (digit-major, tile-minor): one block
__global__ void __launch_bounds__(1024) k_radix_scan(int32_t* __restrict__ c, int64_t n) {
  TCB_PDL_ENTRY();
  __shared__ int32_t part[1024];
  const int64_t per = (n + 1023) / 1024, lo = threadIdx.x * per, hi = lo + per < n ? lo + per : n;
  int32_t sum = 0;
  for (int64_t i = lo; i < hi; ++i) sum += c[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 1; off < 1024; off <<= 1) {  // inclusive Hillis-Steele over the thread sums
    const int32_t v = threadIdx.x >= unsigned(off) ? part[threadIdx.x - off] : 0;
    __syncthreads();
    part[threadIdx.x] += v;
    __syncthreads();
  }
  int32_t run = threadIdx.x ? part[threadIdx.x - 1] : 0;
  for (int64_t i = lo; i < hi; ++i) {
    const int32_t v = c[i];
    c[i] = run;
    run += v;
  }
}

// stable scatter of one tile: element e = warp * 256 + round * 32 + lane (t
// order); its rank among equal digits of the tile = equal digits in earlier
// warps + earlier rounds of its warp + lower lanes of its round
__global__ void __launch_bounds__(256) k_radix_scatter(const int32_t* __restrict__ kin,
                                                       const int32_t* __restrict__ vin, int32_t* __restrict__ kout,
                                                       int32_t* __restrict__ vout, int64_t T, int shift,
                                                       const int32_t* __restrict__ offs, int ntiles) {
  TCB_PDL_ENTRY();
  __shared__ int32_t wc[RDX_WARPS][256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RDX_WARPS * 256; i += 256) (&wc[0][0])[i] = 0;
  __syncthreads();
  const int64_t t0 = int64_t(blockIdx.x) * RDX_TILE;
  const uint32_t lt = (1u << lane) - 1u;
  int32_t key[RDX_ROUNDS], val[RDX_ROUNDS], rk[RDX_ROUNDS];
#pragma unroll
  for (int r = 0; r < RDX_ROUNDS; ++r) {
    const int64_t t = t0 + w * (RDX_ROUNDS * 32) + r * 32 + lane;
    const bool ok = t < T;
    key[r] = ok ? kin[t] : 0;
    val[r] = ok ? (vin ? vin[t] : int32_t(t)) : 0;
    const int d = ok ? (key[r] >> shift) & 255 : 256 + lane;  // tail lanes: unique non-digits
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    rk[r] = ok ? wc[w][d] + __popc(peers & lt) : 0;
    __syncwarp();
    if (ok && (peers & lt) == 0) wc[w][d] += __popc(peers);  // lowest lane of the group
    __syncwarp();
  }
  __syncthreads();
  {  // exclusive prefix over the warps, per digit (thread = digit)
    int32_t run = 0;
    for (int ww = 0; ww < RDX_WARPS; ++ww) {
      const int32_t v = wc[ww][threadIdx.x];
      wc[ww][threadIdx.x] = run;
      run += v;
    }
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < RDX_ROUNDS; ++r) {
    const int64_t t = t0 + w * (RDX_ROUNDS * 32) + r * 32 + lane;
    if (t >= T) continue;
    const int d = (key[r] >> shift) & 255;
    const int64_t pos = int64_t(offs[int64_t(d) * ntiles + blockIdx.x]) + wc[w][d] + rk[r];
    kout[pos] = key[r];
    vout[pos] = val[r];
  }
}

// Small inputs (T <= RDX_SMALL): every digit pass of the same stable sort in
// one CTA through shared memory -- one launch instead of three per pass.
// Element e = warp * (R * 32) + round * 32 + lane (t order), R = ceil(T / 1024).
constexpr int RDX_SMALL = 8192, RDX_SW = 32;  // keys, warps
constexpr int RDX_SMALL_SMEM = (4 * RDX_SMALL + RDX_SW * 256) * 4;  // 160 KB
__global__ void __launch_bounds__(1024) k_radix_sort_small(const int32_t* __restrict__ ids, int T, int passes,
                                                           int32_t* __restrict__ kout, int32_t* __restrict__ vout) {
  TCB_PDL_ENTRY();
  extern __shared__ int32_t sm[];
  int32_t* kA = sm;
  int32_t* vA = kA + RDX_SMALL;
  int32_t* kB = vA + RDX_SMALL;
  int32_t* vB = kB + RDX_SMALL;
  int32_t* wc = vB + RDX_SMALL;  // [RDX_SW][256]
  __shared__ int32_t base[256];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int R = (T + 1023) / 1024;
  const uint32_t lt = (1u << lane) - 1u;
  for (int i = threadIdx.x; i < T; i += 1024) {
    kA[i] = ids[i];
    vA[i] = i;
  }
  for (int ps = 0; ps < passes; ++ps) {
    const int shift = 8 * ps;
    for (int i = threadIdx.x; i < RDX_SW * 256; i += 1024) wc[i] = 0;
    __syncthreads();
    int32_t rk[RDX_SMALL / 1024];
#pragma unroll
    for (int r = 0; r < RDX_SMALL / 1024; ++r) {
      if (r >= R) break;
      const int e = w * (R * 32) + r * 32 + lane;
      const bool ok = e < T;
      const int d = ok ? (kA[e] >> shift) & 255 : 256 + lane;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      rk[r] = ok ? wc[w * 256 + d] + __popc(peers & lt) : 0;
      __syncwarp();
      if (ok && (peers & lt) == 0) wc[w * 256 + d] += __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    if (threadIdx.x < 256) {  // digit totals -> exclusive prefix over the warps
      const int d = threadIdx.x;
      int32_t run = 0;
      for (int ww = 0; ww < RDX_SW; ++ww) {
        const int32_t v = wc[ww * 256 + d];
        wc[ww * 256 + d] = run;
        run += v;
      }
      base[d] = run;
    }
    __syncthreads();
    if (threadIdx.x < 32) {  // exclusive scan of the 256 digit totals (one warp, 8 per lane)
      int32_t v[8], sum = 0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        v[k] = base[lane * 8 + k];
        sum += v[k];
      }
      int32_t inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      int32_t run = inc - sum;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        base[lane * 8 + k] = run;
        run += v[k];
      }
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < RDX_SMALL / 1024; ++r) {
      if (r >= R) break;
      const int e = w * (R * 32) + r * 32 + lane;
      if (e >= T) continue;
      const int d = (kA[e] >> shift) & 255;
      const int pos = base[d] + wc[w * 256 + d] + rk[r];
      kB[pos] = kA[e];
      vB[pos] = vA[e];
    }
    __syncthreads();
    int32_t* t;
    t = kA, kA = kB, kB = t;
    t = vA, vA = vB, vB = t;
  }
  for (int i = threadIdx.x; i < T; i += 1024) {
    kout[i] = kA[i];
    vout[i] = vA[i];
  }
}

// segment bounds by id from the sorted ids: start[id] = first position,
// end[id] = one past the last (only ids that occur are written and read)
__global__ void __launch_bounds__(256) k_embed_segments(const int32_t* __restrict__ sid, int64_t T,
                                                        int32_t* __restrict__ start, int32_t* __restrict__ end) {
  TCB_PDL_ENTRY();
  for (int64_t p = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; p < T; p += int64_t(gridDim.x) * blockDim.x) {
    const int32_t id = sid[p];
    if (p == 0 || sid[p - 1] != id) start[id] = int32_t(p);
    if (p + 1 == T || sid[p + 1] != id) end[id] = int32_t(p + 1);
  }
}

constexpr int EMB_CHUNK = 128;  // rows per partial sum of a long segment

// Segments longer than EMB_CHUNK are summed chunk by chunk (each chunk in
// ascending t into part[chunk_start]) and folded here in chunk order onto
// base: deterministic; for segments <= EMB_CHUNK rows k_embed_accum writes the
// oracle's exact sequential sum directly.
// The block's sorted positions (pos = blockIdx.x + k * gridDim.x) are
// screened 256 at a time by all threads at once (one round of id / segment
// loads instead of a dependent chain per position); the positions that have
// work are listed in shared memory and then processed column-parallel.
// mode 0 (accumulate): chunk starts (pos - head) % EMB_CHUNK == 0;
// mode 1 (fold): heads of segments longer than EMB_CHUNK.
template <int MODE>
__device__ __forceinline__ int embed_screen(const int32_t* __restrict__ sid, const int32_t* __restrict__ start,
                                            const int32_t* __restrict__ send, int64_t T, int64_t k0,
                                            int64_t* list) {
  __shared__ int n;
  if (threadIdx.x == 0) n = 0;
  __syncthreads();
  const int64_t pos = int64_t(blockIdx.x) + (k0 + threadIdx.x) * gridDim.x;
  if (pos < T) {
    const int32_t id = sid[pos];
    const int64_t head = start[id];
    const int32_t len = send[id] - int32_t(head);
    const bool work = MODE == 0 ? (pos - head) % EMB_CHUNK == 0 : (pos == head && len > EMB_CHUNK);
    if (work) list[atomicAdd(&n, 1)] = pos;
  }
  __syncthreads();
  const int m = n;  // list order is arbitrary: every listed position writes its own rows
  __syncthreads();
  return m;
}

__global__ void __launch_bounds__(256) k_embed_fold(const int32_t* __restrict__ sid,
                                                    const int32_t* __restrict__ start,
                                                    const int32_t* __restrict__ end,
                                                    const float* __restrict__ part, float* __restrict__ out,
                                                    int64_t T, int64_t H) {
  TCB_PDL_ENTRY();
  __shared__ int64_t list[256];
  const int64_t j = int64_t(blockIdx.y) * blockDim.x + threadIdx.x;
  const int64_t per = (T - blockIdx.x + gridDim.x - 1) / gridDim.x;  // positions of this block
  for (int64_t k0 = 0; k0 < per; k0 += 256) {
    const int m = embed_screen<1>(sid, start, end, T, k0, list);
    for (int w = 0; w < m; ++w) {
      const int64_t pos = list[w];
      if (j >= H) continue;
      const int32_t id = sid[pos];
      const int32_t len = end[id] - int32_t(pos);
      float acc = out[int64_t(id) * H + j];
      for (int64_t c = pos; c < pos + len; c += EMB_CHUNK) acc = __fadd_rn(acc, part[c * H + j]);
      out[int64_t(id) * H + j] = acc;
    }
    __syncthreads();  // the list is rewritten by the next screen
  }
}

// block (positions, column tile): for each sorted position `pos` that starts a
// chunk of a segment of equal ids, each thread accumulates one column over the
// chunk in ascending t (loads batched 16 deep; the adds keep the oracle's
// order).  Column-parallel, so one id covering every token (token-type ids) is
// 256x wider than a warp.
template <typename TD>
__global__ void __launch_bounds__(256) k_embed_accum(const int32_t* __restrict__ sid,
                                                     const int32_t* __restrict__ sorted,
                                                     const int32_t* __restrict__ start,
                                                     const int32_t* __restrict__ send,
                                                     const TD* __restrict__ dy, float* __restrict__ out,
                                                     float* __restrict__ part, int64_t T, int64_t H) {
  TCB_PDL_ENTRY();
  __shared__ int64_t list[256];
  const int64_t j = int64_t(blockIdx.y) * blockDim.x + threadIdx.x;
  const int64_t per = (T - blockIdx.x + gridDim.x - 1) / gridDim.x;  // positions of this block
  for (int64_t k0 = 0; k0 < per; k0 += 256) {
    const int m = embed_screen<0>(sid, start, send, T, k0, list);
    for (int w = 0; w < m; ++w) {
      const int64_t pos = list[w];
      if (j >= H) continue;
      const int32_t id = sid[pos];
      const int64_t head = start[id];
      const int32_t len = send[id] - int32_t(head);
      const bool single = len <= EMB_CHUNK;
      const int64_t end = (head + len) < (pos + EMB_CHUNK) ? (head + len) : (pos + EMB_CHUNK);
      float acc = single ? out[int64_t(id) * H + j] : 0.0f;
      int64_t q = pos;
      for (; q + 16 <= end; q += 16) {
        float v[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) v[k] = to_f(dy[int64_t(sorted[q + k]) * H + j]);
#pragma unroll
        for (int k = 0; k < 16; ++k) acc = __fadd_rn(acc, v[k]);
      }
      for (; q + 4 <= end; q += 4) {
        float v0 = to_f(dy[int64_t(sorted[q]) * H + j]);
        float v1 = to_f(dy[int64_t(sorted[q + 1]) * H + j]);
        float v2 = to_f(dy[int64_t(sorted[q + 2]) * H + j]);
        float v3 = to_f(dy[int64_t(sorted[q + 3]) * H + j]);
        acc = __fadd_rn(__fadd_rn(__fadd_rn(__fadd_rn(acc, v0), v1), v2), v3);
      }
      for (; q < end; ++q) acc = __fadd_rn(acc, to_f(dy[int64_t(sorted[q]) * H + j]));
      if (single) out[int64_t(id) * H + j] = acc;
      else part[pos * H + j] = acc;
    }
    __syncthreads();  // the list is rewritten by the next screen
  }
}

static void b_embedding_dx(Plan& p) {
  check_arity(p, 2, 3, 1, 1);
  require(p.in[0].dtype == TCB_I32, "embedding_dx: ids must be i32");
  require(p.out[0].dtype == TCB_F32 && p.out[0].rank == 2, "embedding_dx: output is f32 [V, H]");
  const int64_t T = p.in[0].numel(), V = p.out[0].shape[0], H = p.out[0].shape[1];
  require(p.in[1].numel() == T * H, "embedding_dx: dy must be [T, H]");
  require(T < (int64_t(1) << 31) && V < (int64_t(1) << 31), "embedding_dx: T and V must fit in int32");
  const bool has_base = p.in.size() > 2;
  if (has_base) require(p.in[2].dtype == TCB_F32 && p.in[2].numel() == V * H, "embedding_dx: base is f32 [V,H]");
  // radix passes over the id bits (ids are in [0, V))
  int bits = 1;
  while ((int64_t(1) << bits) < V) ++bits;
  const int passes = (bits + 7) / 8;
  const int ntiles = int((T + RDX_TILE - 1) / RDX_TILE);
  // key/value double buffers, digit counts, per-id segment bounds
  const size_t kv = p.ws_take(size_t(T) * 16);
  const size_t cnt = p.ws_take(size_t(256) * ntiles * 4);
  const size_t seg = p.ws_take(size_t(V) * 8);
  // chunk partials of long segments (launch workspace)
  const size_t part = p.ws_take(size_t(T) * H * 4);
  p.nkernels = (T <= RDX_SMALL ? 1 : 3 * passes) + 3;  // sort (one CTA, or count/scan/scatter per pass), segments, accumulate, fold
  if (T <= RDX_SMALL) {
    static std::once_flag once;
    std::call_once(once, [] {
      TCB_CUDA(cudaFuncSetAttribute(k_radix_sort_small, cudaFuncAttributeMaxDynamicSharedMemorySize, RDX_SMALL_SMEM));
    });
  }
  dispatch_float(p.in[1].dtype, [&](auto* tp) {
    using TD = std::remove_pointer_t<decltype(tp)>;
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      const size_t nb = size_t(V) * H * 4;
      if (has_base) {
        if (in[2].ptr != out[0].ptr) TCB_CUDA(cudaMemcpyAsync(out[0].ptr, in[2].ptr, nb, cudaMemcpyDeviceToDevice, s));
      } else {
        TCB_CUDA(cudaMemsetAsync(out[0].ptr, 0, nb, s));
      }
      int32_t* k0 = (int32_t*)ws_at(kv);
      int32_t* v0 = k0 + T;
      int32_t* k1 = v0 + T;
      int32_t* v1 = k1 + T;
      int32_t* counts = (int32_t*)ws_at(cnt);
      int32_t* start = (int32_t*)ws_at(seg);
      int32_t* send = start + V;
      const int32_t* kin = (const int32_t*)in[0].ptr;
      const int32_t* vin = nullptr;  // pass 0: values are the token indices
      if (T <= RDX_SMALL) {
        launch_k(k_radix_sort_small, 1u, 1024, RDX_SMALL_SMEM, s, kin, int(T), passes, k1, v1);
        kin = k1;
        vin = v1;
      }
      for (int ps = 0; T > RDX_SMALL && ps < passes; ++ps) {
        int32_t* ko = (ps & 1) ? k0 : k1;
        int32_t* vo = (ps & 1) ? v0 : v1;
        launch_k(k_radix_count, unsigned(ntiles), 256, 0, s, kin, T, 8 * ps, counts, ntiles);
        launch_k(k_radix_scan, 1u, 1024, 0, s, counts, int64_t(256) * ntiles);
        launch_k(k_radix_scatter, unsigned(ntiles), 256, 0, s, kin, vin, ko, vo, T, 8 * ps, (const int32_t*)counts,
                 ntiles);
        kin = ko;
        vin = vo;
      }
      const int32_t* sid = kin;      // ids in sorted order
      const int32_t* srt = vin;      // their token indices
      launch_k(k_embed_segments, grid_for(T, 256), 256, 0, s, sid, T, start, send);
      // persistent-ish grids: ~8 CTAs per SM in total over the column tiles
      const int64_t ct = (H + 255) / 256;
      const int64_t gx = std::max<int64_t>(1, std::min<int64_t>(T, (kNumSMs * 8 + ct - 1) / ct));
      const dim3 g2{unsigned(gx), unsigned(ct)};
      launch_k(k_embed_accum<TD>, g2, 256, 0, s, sid, srt, (const int32_t*)start, (const int32_t*)send,
               (const TD*)in[1].ptr, (float*)out[0].ptr, (float*)ws_at(part), T, H);
      launch_k(k_embed_fold, g2, 256, 0, s, sid, (const int32_t*)start, (const int32_t*)send,
               (const float*)ws_at(part), (float*)out[0].ptr, T, H);
    };
  });
}
TCB_REGISTER("embedding_dx", b_embedding_dx);

// ------------------------------------------------------------ cross entropy
// (logits [T, Vp], labels [T]) -> (loss f32[1], dlogits [T, Vp])
__global__ void k_ce_count(const int32_t* __restrict__ labels, int64_t T, int64_t ign, float* __restrict__ inv_n) {
  TCB_PDL_ENTRY();
  __shared__ int part[32];
  int c = 0;
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) c += labels[t] != ign;
  for (int m = 16; m; m >>= 1) c += __shfl_xor_sync(0xffffffffu, c, m);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) n += part[w];
    inv_n[0] = n ? 1.0f / float(n) : 0.0f;
  }
}

template <typename T>
// dx may alias x (the planner runs cross_entropy in place, logits -> dlogits):
// every element is read by the thread that later overwrites it, and the label
// logit is read before the block barrier that precedes any write
__global__ void __launch_bounds__(512) k_ce_row(const T* x, const int32_t* __restrict__ labels,
                                                T* dx, float* __restrict__ row_loss,
                                                const float* __restrict__ inv_n_p, int64_t Vp, int64_t V,
                                                int64_t ign, float gscale, int* __restrict__ err, bool vec) {
  TCB_PDL_ENTRY();
  __shared__ float sm[32], ss[32];
  const int64_t t = blockIdx.x;
  const int32_t lab = labels[t];
  const T* xr = x + t * Vp;
  T* dr = dx ? dx + t * Vp : nullptr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lab == ign) {  // no loss, zero gradient row (16-byte stores when aligned)
    if (dr) {
      if (vec) {
        constexpr int EPV = 16 / sizeof(T);  // elements per 16-byte store
        for (int64_t c = threadIdx.x; c < Vp / EPV; c += blockDim.x)
          reinterpret_cast<uint4*>(dr)[c] = make_uint4(0, 0, 0, 0);
      } else {
        for (int64_t j = threadIdx.x; j < Vp; j += blockDim.x) dr[j] = from_f<T>(0.0f);
      }
    }
    if (threadIdx.x == 0) row_loss[t] = 0.0f;
    return;
  }
  if (lab < 0 || lab >= V) {
    if (threadIdx.x == 0) atomicExch(err, 1);
    return;
  }
  const float xlab = threadIdx.x == 0 ? to_f(xr[lab]) : 0.0f;  // before any thread may overwrite it
  // pass 1: online max / sum
  float m = -INFINITY, s = 0.0f;
  const int64_t nch = V / 8;
  for (int64_t c = threadIdx.x; c < (vec ? nch : 0); c += blockDim.x) {
    float f[8];
    Vec8<T>::load(xr + c * 8, f);
    float lm = f[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) lm = fmaxf(lm, f[k]);
    if (lm > m) {
      s *= expf(m - lm);
      m = lm;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += expf(f[k] - m);
  }
  for (int64_t j = (vec ? nch * 8 : 0) + threadIdx.x; j < V; j += blockDim.x) {
    float f = to_f(xr[j]);
    if (f > m) {
      s *= expf(m - f);
      m = f;
    }
    s += expf(f - m);
  }
  // combine (m, s) across the block
  float wm = warp_max(m);
  s = s * (m == -INFINITY ? 0.0f : expf(m - wm));
  s = warp_sum(s);
  if (lane == 0) {
    sm[warp] = wm;
    ss[warp] = s;
  }
  __syncthreads();
  float M = -INFINITY;
  for (int w = 0; w < nw; ++w) M = fmaxf(M, sm[w]);
  float S = 0.0f;
  for (int w = 0; w < nw; ++w) S += ss[w] * expf(sm[w] - M);
  const float lse = M + logf(S);
  if (threadIdx.x == 0) row_loss[t] = lse - xlab;
  if (!dr) return;
  // pass 2: gradient
  const float inv_s = 1.0f / S;
  const float k = gscale * inv_n_p[0];
  for (int64_t c = threadIdx.x; c < (vec ? Vp / 8 : 0); c += blockDim.x) {
    float f[8];
    Vec8<T>::load(xr + c * 8, f);
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int64_t j = c * 8 + q;
      float v = j < V ? expf(f[q] - M) * inv_s : 0.0f;
      if (j == lab) v -= 1.0f;
      f[q] = v * k;
    }
    Vec8<T>::store(dr + c * 8, f);
  }
  for (int64_t j = (vec ? (Vp / 8) * 8 : 0) + threadIdx.x; j < Vp; j += blockDim.x) {
    float v = j < V ? expf(to_f(xr[j]) - M) * inv_s : 0.0f;
    if (j == lab) v -= 1.0f;
    dr[j] = from_f<T>(v * k);
  }
}

__global__ void k_ce_final(const float* __restrict__ row_loss, const float* __restrict__ inv_n, int64_t T,
                           float* __restrict__ loss) {
  TCB_PDL_ENTRY();
  __shared__ float part[32];
  float a = 0.0f;
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) a += row_loss[t];
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    float s = 0.0f;
    for (int w = 0; w < int(blockDim.x >> 5); ++w) s += part[w];
    loss[0] = s * inv_n[0];
  }
}

static void b_cross_entropy(Plan& p) {
  check_arity(p, 2, 2, 1, 2);
  const Spec& X = p.in[0];
  require(X.rank == 2, "cross_entropy: logits must be [T, V]");
  require(p.in[1].dtype == TCB_I32 && p.in[1].numel() == X.shape[0], "cross_entropy: labels must be i32 [T]");
  require(p.out[0].dtype == TCB_F32 && p.out[0].numel() == 1, "cross_entropy: loss is f32[1]");
  const int64_t T = X.shape[0], Vp = X.shape[1];
  const int64_t V = p.attrs.i("classes", Vp);
  require(V >= 1 && V <= Vp, "cross_entropy: classes must be in [1, Vp]");
  const int64_t ign = p.attrs.i("ignore_index", -100);
  const float gscale = float(p.attrs.f("grad_scale", 1.0));
  const bool grad = p.out.size() > 1;
  if (grad) require(same_shape(p.out[1], X) && p.out[1].dtype == X.dtype, "cross_entropy: dlogits like logits");
  const size_t ws = p.ws_take(size_t(T + 4) * 4);
  auto err = std::make_shared<Scratch>(4);  // sticky error flag (label out of range), write-only
  TCB_CUDA(cudaMemset(err->p, 0, 4));
  p.nkernels = 3;
  dispatch_float(X.dtype, [&](auto* tp) {
    using T_ = std::remove_pointer_t<decltype(tp)>;
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      float* inv_n = (float*)ws_at(ws);
      float* rows = inv_n + 4;
      const bool vec = Vp % 8 == 0 && reinterpret_cast<uintptr_t>(in[0].ptr) % 16 == 0 &&
                       (!grad || reinterpret_cast<uintptr_t>(out[1].ptr) % 16 == 0);
      launch_k(k_ce_count, 1, 1024, 0, s, (const int32_t*)in[1].ptr, T, ign, inv_n);
      launch_k(k_ce_row<T_>, unsigned(T), 512, 0, s, (const T_*)in[0].ptr, (const int32_t*)in[1].ptr,
                                                grad ? (T_*)out[1].ptr : nullptr, rows, inv_n, Vp, V, ign,
                                                gscale, (int*)err->p, vec);
      launch_k(k_ce_final, 1, 1024, 0, s, rows, inv_n, T, (float*)out[0].ptr);
    };
  });
}
TCB_REGISTER("cross_entropy", b_cross_entropy);

}  // namespace tcb
