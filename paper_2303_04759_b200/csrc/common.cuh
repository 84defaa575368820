// common.cuh -- shared plumbing of libtcb200 (the b200 dialect kernels).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <type_traits>
#include <map>
#include <memory>
#include <mutex>
#include <cmath>
#include <type_traits>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tcb200.h"

namespace tcb {

constexpr int kNumSMs = 148;

// ------------------------------------------------------------------ errors
struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& m) { throw Status(code, m); }
inline void require(bool c, const std::string& m) {
  if (!c) fail(TCB_ERR_TYPE, m);
}
#define TCB_CUDA(x)                                                                   \
  do {                                                                                \
    cudaError_t e_ = (x);                                                             \
    if (e_ != cudaSuccess)                                                            \
      ::tcb::fail(TCB_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

// ------------------------------------------------------------------ tensors
struct Spec {
  int dtype = TCB_F32;
  int rank = 0;
  int64_t shape[TCB_MAX_RANK] = {0};
  int64_t numel() const {
    int64_t n = 1;
    for (int i = 0; i < rank; ++i) n *= shape[i];
    return n;
  }
  int64_t dim(int i) const { return shape[i < 0 ? rank + i : i]; }
};

inline int dtype_bytes(int d) { return d == TCB_F32 || d == TCB_I32 ? 4 : d == TCB_U8 ? 1 : 2; }
inline const char* dtype_name(int d) {
  switch (d) {
    case TCB_F32: return "f32";
    case TCB_F16: return "f16";
    case TCB_BF16: return "bf16";
    case TCB_I32: return "i32";
    case TCB_U8: return "u8";
  }
  return "?";
}
inline bool is_float(int d) { return d == TCB_F32 || d == TCB_F16 || d == TCB_BF16; }

// ------------------------------------------------------------------ attrs
struct Attrs {
  std::map<std::string, tcb_attr> m;
  std::vector<std::string> strs;  // storage
  double f(const char* k, double d) const {
    auto it = m.find(k);
    if (it == m.end()) return d;
    return it->second.kind == TCB_ATTR_FLOAT ? it->second.d
           : it->second.kind == TCB_ATTR_INT ? double(it->second.i)
                                             : d;
  }
  int64_t i(const char* k, int64_t d) const {
    auto it = m.find(k);
    if (it == m.end()) return d;
    return it->second.kind == TCB_ATTR_INT ? it->second.i
           : it->second.kind == TCB_ATTR_FLOAT ? int64_t(it->second.d)
                                               : d;
  }
  std::string s(const char* k, const std::string& d) const {
    auto it = m.find(k);
    if (it == m.end() || it->second.kind != TCB_ATTR_STR || !it->second.s) return d;
    return it->second.s;
  }
};

// --------------------------------------------------------------- device math
__device__ __forceinline__ float ld_f(const float* p, int64_t i) { return p[i]; }
__device__ __forceinline__ float ld_f(const __half* p, int64_t i) { return __half2float(p[i]); }
__device__ __forceinline__ float ld_f(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}
__device__ __forceinline__ void st_f(float* p, int64_t i, float v) { p[i] = v; }
__device__ __forceinline__ void st_f(__half* p, int64_t i, float v) { p[i] = __float2half_rn(v); }
__device__ __forceinline__ void st_f(__nv_bfloat16* p, int64_t i, float v) {
  p[i] = __float2bfloat16_rn(v);
}
template <typename T>
__device__ __forceinline__ T from_f(float v);
template <>
__device__ __forceinline__ float from_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ __half from_f<__half>(float v) { return __float2half_rn(v); }
template <>
__device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__half v) { return __half2float(v); }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }

// erf-based GELU and its derivative (match oracle.c gelu_f / gelu_grad_f)
__device__ __forceinline__ float gelu_f(float x) {
  return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f));
}
__device__ __forceinline__ float gelu_grad_f(float x) {
  float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752f));
  float pdf = expf(-0.5f * x * x) * 0.39894228040143268f;
  return __fadd_rn(cdf, __fmul_rn(x, pdf));
}

// Packed f32x2 arithmetic (sm_100 FADD2 / FMUL2 / FFMA2): one instruction per
// element pair, each lane IEEE round-to-nearest like the scalar op, so results
// are bit-identical to the scalar code while issue-bound row kernels halve
// their FP instruction count.
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 splat2(float a) { return make_float2(a, a); }
// a 32-bit word of two 16-bit floats <-> float2 (bf16: shifts; f16: cvt)
__device__ __forceinline__ float2 bf2_to_f2(uint32_t w) {
  return make_float2(__uint_as_float(w << 16), __uint_as_float(w & 0xffff0000u));
}

// GEMM-epilogue GELU / GELU' on the MUFU path: Phi(x) from the
// Abramowitz-Stegun 7.1.26 erfc (|err| <= 1.5e-7, with ex2.approx / rcp.approx
// adding a few ulp) sharing one exponential exp(-x^2/2) with the pdf term.
// ~14 instructions instead of ~35 for erff/expf; the bf16 results differ from
// the oracle's erff in a handful of last-bit roundings (tolerance-checked).
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void fast_phi(float x, float& phi, float& e) {
  const float ax = fabsf(x);
  e = ex2_approx(x * x * -0.72134752044448170f);                   // exp(-x^2/2)
  const float t = rcp_approx(fmaf(0.23164188f, ax, 1.0f));         // 1/(1 + p z), z = |x|/sqrt(2)
  float poly = fmaf(t, 1.061405429f, -1.453152027f);
  poly = fmaf(t, poly, 1.421413741f);
  poly = fmaf(t, poly, -0.284496736f);
  poly = fmaf(t, poly, 0.254829592f);
  const float half_erfc = 0.5f * (poly * t) * e;                  // 0.5 erfc(z)
  phi = x >= 0.0f ? 1.0f - half_erfc : half_erfc;
}
// fast_phi on an element pair with f32x2 arithmetic (same operations, same
// order per lane as fast_phi -> bit-identical results, half the FP issue slots)
__device__ __forceinline__ void fast_phi2(float2 x, float2& phi, float2& e) {
  const float2 ax = make_float2(fabsf(x.x), fabsf(x.y));
  const float2 q = mul2(mul2(x, x), splat2(-0.72134752044448170f));
  e = make_float2(ex2_approx(q.x), ex2_approx(q.y));
  const float2 den = fma2(splat2(0.23164188f), ax, splat2(1.0f));
  const float2 t = make_float2(rcp_approx(den.x), rcp_approx(den.y));
  float2 poly = fma2(t, splat2(1.061405429f), splat2(-1.453152027f));
  poly = fma2(t, poly, splat2(1.421413741f));
  poly = fma2(t, poly, splat2(-0.284496736f));
  poly = fma2(t, poly, splat2(0.254829592f));
  const float2 he = mul2(mul2(splat2(0.5f), mul2(poly, t)), e);
  const float2 one_m = add2(splat2(1.0f), make_float2(-he.x, -he.y));
  phi = make_float2(x.x >= 0.0f ? one_m.x : he.x, x.y >= 0.0f ? one_m.y : he.y);
}
__device__ __forceinline__ float fast_gelu(float x) {
  float phi, e;
  fast_phi(x, phi, e);
  return x * phi;
}
__device__ __forceinline__ float fast_gelu_grad(float x) {
  float phi, e;
  fast_phi(x, phi, e);
  return fmaf(x * 0.39894228040143268f, e, phi);
}

// ACT_DERIV: the aux operand already holds act'(u) (a forward epilogue saved
// the derivative instead of the pre-activation), so act'(aux) = aux
enum Act { ACT_NONE = 0, ACT_RELU = 1, ACT_TANH = 2, ACT_GELU = 3, ACT_DERIV = 4 };
inline int parse_act(const std::string& s) {
  if (s.empty() || s == "none") return ACT_NONE;
  if (s == "deriv") return ACT_DERIV;
  if (s == "relu") return ACT_RELU;
  if (s == "tanh") return ACT_TANH;
  if (s == "gelu") return ACT_GELU;
  fail(TCB_ERR_TYPE, "unknown activation '" + s + "'");
}
__device__ __forceinline__ float act_f(int act, float v) {
  switch (act) {
    case ACT_RELU: return v > 0.0f ? v : 0.0f;
    case ACT_TANH: return tanhf(v);
    case ACT_GELU: return gelu_f(v);
    default: return v;
  }
}
// act'(u) from the pre-activation u (what a save_grad epilogue stores)
__device__ __forceinline__ float deriv_of_preact(int act, float u) {
  switch (act) {
    case ACT_RELU: return u > 0.0f ? 1.0f : 0.0f;
    case ACT_TANH: {
      const float y = tanhf(u);
      return __fsub_rn(1.0f, __fmul_rn(y, y));
    }
    case ACT_GELU: return gelu_grad_f(u);
    default: return 1.0f;
  }
}
__device__ __forceinline__ float dact_f(int act, float aux) {
  switch (act) {
    case ACT_RELU: return aux > 0.0f ? 1.0f : 0.0f;
    case ACT_TANH: return __fsub_rn(1.0f, __fmul_rn(aux, aux));
    case ACT_GELU: return gelu_grad_f(aux);
    case ACT_DERIV: return aux;
    default: return 1.0f;
  }
}

// Philox4x32-10 keep decision, identical to oracle.c orc_dropout_keep.
__device__ __forceinline__ void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t lo0 = 0xD2511F53u * c[0];
    uint32_t hi0 = __umulhi(0xD2511F53u, c[0]);
    uint32_t lo1 = 0xCD9E8D57u * c[2];
    uint32_t hi1 = __umulhi(0xCD9E8D57u, c[2]);
    uint32_t n0 = hi1 ^ c[1] ^ k0;
    uint32_t n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0;
    c[1] = lo1;
    c[2] = n2;
    c[3] = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
}
struct DropCfg {
  float p = 0.0f, scale = 1.0f;
  uint64_t seed = 0, salt = 0;
  // keep iff the 16-bit draw h >= thr.  h * 2^-16 is exact in f32, so this is
  // the oracle's float(h) * (1/65536) >= p exactly, with thr = ceil(p * 65536)
  uint32_t thr = 0;
  // optional saved keep bits, one byte per 8 consecutive elements (bit k =
  // element 8i+k): a forward site writes them, its backward reads them
  // instead of re-running Philox (add_layer_norm save_mask / layer_norm_dx mask_in)
  uint8_t* mask_out = nullptr;
  const uint8_t* mask_in = nullptr;
  // Philox counter word 3: the training step's dropout step (rng_step state,
  // f32, incremented once per step), so masks differ from step to step.
  // Read on the device once per kernel (drop_resolve, after griddepcontrol.wait)
  uint32_t step = 0;
  const float* step_ptr = nullptr;
};
__device__ __forceinline__ void drop_resolve(DropCfg& d) {
  if (d.step_ptr) d.step = uint32_t(*d.step_ptr);
}
// 8 keep bits for indices (q*8 .. q*8+7): one Philox call, 16 bits per element
// (identical to oracle.c orc_dropout_keep); integer compares: the high half of
// word w is >= thr iff w >= thr << 16
__device__ __forceinline__ uint32_t dropout_bits8q(const DropCfg& d, uint64_t q) {
  uint32_t c[4] = {uint32_t(q), uint32_t(d.salt), uint32_t(d.salt >> 32), d.step};
  philox4x32_10(c, uint32_t(d.seed), uint32_t(d.seed >> 32));
  uint32_t bits = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    bits |= ((c[k] & 0xFFFFu) >= d.thr ? 1u : 0u) << (2 * k);
    bits |= ((c[k] >> 16) >= d.thr ? 1u : 0u) << (2 * k + 1);
  }
  return bits;
}
__device__ __forceinline__ bool dropout_keep(const DropCfg& d, uint64_t idx) {
  if (d.p <= 0.0f) return true;
  return (dropout_bits8q(d, idx >> 3) >> (idx & 7)) & 1u;
}
// keep bits of the 4 elements i0 .. i0+3 (one call when they share an 8-group)
__device__ __forceinline__ uint32_t dropout_bits4(const DropCfg& d, uint64_t i0) {
  if (d.p <= 0.0f) return 0xFu;
  if ((i0 & 7) <= 4) return (dropout_bits8q(d, i0 >> 3) >> (i0 & 7)) & 0xFu;
  uint32_t b = 0;
  for (int k = 0; k < 4; ++k) b |= uint32_t(dropout_keep(d, i0 + k)) << k;
  return b;
}
// the rng_step input of the launch in progress (tcb_launch appends it when the
// plan was created with rng_in=1); nullptr: step 0
const float*& launch_rng();
inline DropCfg with_step(DropCfg d) {
  d.step_ptr = launch_rng();
  return d;
}
inline DropCfg drop_cfg(const Attrs& a) {
  DropCfg d;
  d.p = float(a.f("p", 0.0));
  d.scale = d.p > 0.0f ? 1.0f / (1.0f - d.p) : 1.0f;
  d.seed = uint64_t(a.i("seed", 0));
  d.thr = d.p > 0.0f ? uint32_t(std::ceil(double(d.p) * 65536.0)) : 0u;
  d.salt = uint64_t(a.i("salt", 0));
  return d;
}

inline int grid_for(int64_t n, int block, int max_blocks = kNumSMs * 8) {
  int64_t g = (n + block - 1) / block;
  if (g > max_blocks) g = max_blocks;
  if (g < 1) g = 1;
  return int(g);
}

// dtype dispatch helper: calls f((T*)nullptr) with the storage type
template <typename Fn>
void dispatch_float(int dtype, Fn&& f) {
  switch (dtype) {
    case TCB_F32: f((float*)nullptr); return;
    case TCB_F16: f((__half*)nullptr); return;
    case TCB_BF16: f((__nv_bfloat16*)nullptr); return;
  }
  fail(TCB_ERR_TYPE, std::string("unsupported dtype ") + dtype_name(dtype));
}

// Device allocation owned by a plan: only for READ-ONLY plan data (schedule
// tables) -- mutable scratch comes from the launch workspace (Plan::ws_take).
struct Scratch {
  void* p = nullptr;
  explicit Scratch(size_t bytes) { TCB_CUDA(cudaMalloc(&p, bytes ? bytes : 16)); }
  ~Scratch() {
    if (p) cudaFree(p);
  }
};

// ------------------------------------------------ programmatic dependent launch
// Every b200 kernel is launched with programmatic stream serialization: the
// next kernel in the stream may be scheduled as soon as all CTAs of the
// current one have started (launch_dependents), so its launch latency and
// prologue overlap our tail.  Correctness: every kernel executes
// griddepcontrol.wait (which returns once the preceding grid has completed
// and flushed) before it touches global memory; since every kernel waits,
// completion order stays transitive along the stream.  TCB_PDL=0 disables.
#define TCB_PDL_ENTRY()                                          \
  do {                                                           \
    asm volatile("griddepcontrol.wait;" ::: "memory");           \
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); \
  } while (0)
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Profiling knob (never set in tests / the bench): TCB_SKIP_FOLDS=1 drops the
// deterministic partial-sum folds (LN dgamma/dbeta, bias colsums, K-slice
// reductions) to bound what merging them could save.  Outputs are then wrong.
inline bool skip_folds() {
  static const bool v = std::getenv("TCB_SKIP_FOLDS") && std::atoi(std::getenv("TCB_SKIP_FOLDS"));
  return v;
}
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("TCB_PDL");
    return !(e && e[0] == '0');
  }();
  return on;
}
// fills a launch attribute slot with PDL; returns the number of attributes used
inline int pdl_attr(cudaLaunchAttribute* a) {
  if (!pdl_enabled()) return 0;
  a->id = cudaLaunchAttributeProgrammaticStreamSerialization;
  a->val.programmaticStreamSerializationAllowed = 1;
  return 1;
}
template <typename... KP, typename... Args>
inline void launch_k(void (*kern)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  cfg.attrs = at;
  cfg.numAttrs = pdl_attr(at);
  TCB_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// ------------------------------------------------------------------ plans
using RunFn = std::function<void(const tcb_tensor* in, tcb_tensor* out, cudaStream_t s)>;

struct Plan {
  std::string op;  // base op
  std::string key;
  std::vector<Spec> in, out;
  Attrs attrs;
  RunFn run;
  int nkernels = 1;
  // Mutable device scratch is NOT owned by the plan (plans are shared through
  // the process-wide KernelCache by VMs that may run concurrently): a builder
  // reserves a byte range of the per-launch WORKSPACE with ws_take() and the
  // run function addresses it with ws_at(offset).  The caller of the launch
  // (a VM) supplies one workspace for its whole stream (tcb_launch_ws).
  size_t ws_bytes = 0;
  size_t ws_take(size_t bytes) {
    const size_t off = (ws_bytes + 255) & ~size_t(255);
    ws_bytes = off + ((bytes + 255) & ~size_t(255));
    return off;
  }
};

// the workspace of the launch in progress on this thread (set by tcb_launch_ws)
char*& launch_ws();
inline void* ws_at(size_t off) {
  char* b = launch_ws();
  if (!b) fail(TCB_ERR_ARG, "launch without a workspace for a plan that needs one");
  return b + off;
}

using Builder = void (*)(Plan&);
void register_builder(const char* op, Builder b);
struct AutoReg {
  AutoReg(const char* op, Builder b) { register_builder(op, b); }
};
#define TCB_CAT2(a, b) a##b
#define TCB_CAT(a, b) TCB_CAT2(a, b)
#define TCB_REGISTER(op, fn) static ::tcb::AutoReg TCB_CAT(_tcb_reg_, __COUNTER__)(op, fn)

inline void check_arity(const Plan& p, int nin_min, int nin_max, int nout_min, int nout_max) {
  int ni = int(p.in.size()), no = int(p.out.size());
  if (ni < nin_min || ni > nin_max || no < nout_min || no > nout_max)
    fail(TCB_ERR_TYPE, "b200." + p.op + ": wrong number of inputs/outputs (" + std::to_string(ni) +
                           ", " + std::to_string(no) + ")");
}
inline bool same_shape(const Spec& a, const Spec& b) {
  if (a.rank != b.rank) return false;
  for (int i = 0; i < a.rank; ++i)
    if (a.shape[i] != b.shape[i]) return false;
  return true;
}

}  // namespace tcb
