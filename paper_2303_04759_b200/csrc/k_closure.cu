// k_closure.cu -- b200.ew_closure: one kernel for a rule-fused group of
// elementwise ops (fusion module; SURVEY.md §8a A5
// "fused-elementwise kernels generated per rule-fusion closure").
//
// The closure body is a register program built by the host fusion pass
// (host/graph.hpp rule_fuse): inputs are registers 0..nin-1 (loaded from their
// storage dtype; [1]-element inputs broadcast), every instruction writes one
// new register and rounds it to that instruction's dtype -- exactly the
// rounding the separate exec_base kernels apply to their outputs -- and the
// closure's outputs are registers stored in their dtypes.  Compiled with
// -fmad=false with the same *_rn arithmetic as k_elementwise.cu, so a closure
// is bit-identical to running its ops one by one (tanh/gelu: device libm).
#include <sstream>

#include "common.cuh"

namespace tcb {

enum CloOp : uint8_t { C_ADD, C_SUB, C_MUL, C_DIV, C_TANH_DX, C_GELU_DX, C_NEG, C_TANH, C_RELU, C_GTZ, C_GELU,
                       C_COPY, C_ADDS };
constexpr int CLO_MAX_INS = 16, CLO_MAX_IN = 8, CLO_MAX_OUT = 8;

struct CloIns {
  uint8_t op, dst, a, b;
  int dt;      // rounding dtype of the result
  float imm;   // add_scalar value
};
struct CloProg {
  int nins, nin, nout;
  CloIns ins[CLO_MAX_INS];
  const void* in[CLO_MAX_IN];
  int in_dt[CLO_MAX_IN];
  int64_t in_n[CLO_MAX_IN];  // 1: broadcast scalar
  void* out[CLO_MAX_OUT];
  int out_dt[CLO_MAX_OUT];
  uint8_t out_reg[CLO_MAX_OUT];
};

__device__ __forceinline__ float clo_ld(const void* p, int dt, int64_t i) {
  if (dt == TCB_F32) return static_cast<const float*>(p)[i];
  if (dt == TCB_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  return __half2float(static_cast<const __half*>(p)[i]);
}
__device__ __forceinline__ float clo_round(int dt, float v) {
  if (dt == TCB_BF16) return __bfloat162float(__float2bfloat16_rn(v));
  if (dt == TCB_F16) return __half2float(__float2half_rn(v));
  return v;
}
__device__ __forceinline__ void clo_st(void* p, int dt, int64_t i, float v) {
  if (dt == TCB_F32) static_cast<float*>(p)[i] = v;
  else if (dt == TCB_BF16) static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else static_cast<__half*>(p)[i] = __float2half_rn(v);
}

__global__ void __launch_bounds__(256) k_ew_closure(const __grid_constant__ CloProg P, int64_t n) {
  TCB_PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float r[CLO_MAX_IN + CLO_MAX_INS];
#pragma unroll
    for (int k = 0; k < CLO_MAX_IN; ++k)
      if (k < P.nin) r[k] = clo_ld(P.in[k], P.in_dt[k], P.in_n[k] == 1 ? 0 : i);
#pragma unroll
    for (int k = 0; k < CLO_MAX_INS; ++k) {
      if (k >= P.nins) break;
      const CloIns& c = P.ins[k];
      const float x = r[c.a], y = r[c.b];
      float v;
      switch (c.op) {
        case C_ADD: v = __fadd_rn(x, y); break;
        case C_SUB: v = __fsub_rn(x, y); break;
        case C_MUL: v = __fmul_rn(x, y); break;
        case C_DIV: v = __fdiv_rn(x, y); break;
        case C_TANH_DX: v = __fmul_rn(y, __fsub_rn(1.0f, __fmul_rn(x, x))); break;
        case C_GELU_DX: v = __fmul_rn(y, gelu_grad_f(x)); break;
        case C_NEG: v = -x; break;
        case C_TANH: v = tanhf(x); break;
        case C_RELU: v = x > 0.0f ? x : 0.0f; break;
        case C_GTZ: v = x > 0.0f ? 1.0f : 0.0f; break;
        case C_GELU: v = gelu_f(x); break;
        case C_ADDS: v = __fadd_rn(x, c.imm); break;
        default: v = x; break;  // C_COPY: convert / cast (the rounding is the op)
      }
      r[c.dst] = clo_round(c.dt, v);
    }
#pragma unroll
    for (int k = 0; k < CLO_MAX_OUT; ++k)
      if (k < P.nout) clo_st(P.out[k], P.out_dt[k], i, r[P.out_reg[k]]);
  }
}

static uint8_t clo_opcode(const std::string& s) {
  static const std::map<std::string, uint8_t> m = {
      {"add", C_ADD},   {"sub", C_SUB},   {"mul", C_MUL},         {"div", C_DIV},   {"tanh_dx", C_TANH_DX},
      {"gelu_dx", C_GELU_DX}, {"neg", C_NEG}, {"tanh", C_TANH}, {"relu", C_RELU}, {"gtz", C_GTZ},
      {"gelu", C_GELU}, {"copy", C_COPY}, {"add_scalar", C_ADDS}};
  auto it = m.find(s);
  if (it == m.end()) fail(TCB_ERR_UNIMPLEMENTED, "ew_closure: no closure opcode " + s);
  return it->second;
}

// ew_closure(inputs..) {prog="op dst a b dt imm;...", outs="reg,reg,.."} -> outputs
static void b_ew_closure(Plan& p) {
  const int nin = int(p.in.size()), nout = int(p.out.size());
  require(nin >= 1 && nin <= CLO_MAX_IN && nout >= 1 && nout <= CLO_MAX_OUT, "ew_closure: 1-8 inputs and outputs");
  const int64_t n = p.out[0].numel();
  CloProg P{};
  P.nin = nin;
  P.nout = nout;
  for (int k = 0; k < nin; ++k) {
    require(is_float(p.in[k].dtype), "ew_closure: float inputs only");
    require(p.in[k].numel() == n || p.in[k].numel() == 1, "ew_closure: inputs are same-size or scalars");
    P.in_dt[k] = p.in[k].dtype;
    P.in_n[k] = p.in[k].numel();
  }
  for (int k = 0; k < nout; ++k) {
    require(p.out[k].numel() == n && is_float(p.out[k].dtype), "ew_closure: outputs are same-size floats");
    P.out_dt[k] = p.out[k].dtype;
  }
  std::istringstream is(p.attrs.s("prog", ""));
  std::string ins;
  while (std::getline(is, ins, ';')) {
    if (ins.empty()) continue;
    require(P.nins < CLO_MAX_INS, "ew_closure: more than 16 instructions");
    std::istringstream f(ins);
    std::string op;
    int dst, a, b, dt;
    float imm;
    if (!(f >> op >> dst >> a >> b >> dt >> imm)) fail(TCB_ERR_TYPE, "ew_closure: bad instruction '" + ins + "'");
    const int limit = nin + P.nins;
    require(dst == limit && a >= 0 && a < limit && b >= 0 && b < limit, "ew_closure: registers out of order");
    P.ins[P.nins++] = CloIns{clo_opcode(op), uint8_t(dst), uint8_t(a), uint8_t(b), dt, imm};
  }
  std::istringstream os(p.attrs.s("outs", ""));
  std::string reg;
  int k = 0;
  while (std::getline(os, reg, ',')) {
    require(k < nout, "ew_closure: more output registers than outputs");
    const int rg = std::stoi(reg);
    require(rg >= 0 && rg < nin + P.nins, "ew_closure: output register out of range");
    P.out_reg[k++] = uint8_t(rg);
  }
  require(k == nout, "ew_closure: one output register per output");
  p.run = [P, n, nin, nout](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) mutable {
    for (int i = 0; i < nin; ++i) P.in[i] = in[i].ptr;
    for (int i = 0; i < nout; ++i) P.out[i] = out[i].ptr;
    launch_k(k_ew_closure, grid_for(n, 256), 256, 0, s, P, n);
  };
}
TCB_REGISTER("ew_closure", b_ew_closure);

}  // namespace tcb
