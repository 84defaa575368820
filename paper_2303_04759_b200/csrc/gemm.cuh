// gemm.cuh -- the GEMM problem description shared by the exact SIMT kernel
// (k_gemm_exact.cu) and the tcgen05 tensor-core kernel (k_gemm_tc.cu).
//
// C[z](m,n) = epi( alpha * sum_k A[z](m,k) * B[z](k,n) )
//   A[z](m,k) = ta ? A[off_a(z) + k*lda + m] : A[off_a(z) + m*lda + k]
//   B[z](k,n) = tb ? B[off_b(z) + n*ldb + k] : B[off_b(z) + k*ldb + n]
//   off_x(z) = (z / Z2) * x_s1 + (z % Z2) * x_s2      (two-level batch: (b, head))
// epilogue (in this order, f32):
//   v = alpha*acc; v += bias[n]; v *= act'(aux(m,n)); aux_out(m,n) = v; v = act(v)
// then one round-to-nearest-even store into C's dtype.  This covers matmul
// (backends.hpp:143-155), matmul_add_act (backends.hpp:311-324) and the
// extension GEMMs (linear, matmul_t, matmul_dact, batch_matmul, attention).
#pragma once
#include "common.cuh"

namespace tcb {

struct GemmOperand {
  const void* ptr = nullptr;
  int64_t ld = 0, s1 = 0, s2 = 0;
  int dtype = TCB_F32;
};

struct GemmArgs {
  int64_t M = 0, N = 0, K = 0;
  int64_t Z = 1, Z2 = 1;
  int ta = 0, tb = 0;
  GemmOperand a, b;
  void* c = nullptr;
  int64_t ldc = 0, c_s1 = 0, c_s2 = 0;
  int c_dtype = TCB_F32;
  float alpha = 1.0f;
  const void* bias = nullptr;  // [N], dtype bias_dtype
  int bias_dtype = TCB_F32;
  int act = ACT_NONE;          // forward activation
  int dact = ACT_NONE;         // multiply by act'(aux)
  const void* aux = nullptr;   // same layout as C (ldc, batch strides), aux_dtype
  int aux_dtype = TCB_F32;
  void* aux_out = nullptr;     // pre-activation store, same layout/dtype as C
  int save_grad = 0;           // aux_out holds act'(pre-activation) instead (consumed with ACT_DERIV)
  int force_bn = 0, force_cg = 0;  // tcgen05 tile override (tests / tuning); 0 = cost model
  void* trace = nullptr;           // optional per-CTA timeline buffer (16 x u64 per CTA, tooling)
  int no_tma_epi = 0;              // force the direct-store epilogue (tooling)
  int generic_epi = 0;             // force the runtime-dispatched epilogue (parity tests of the variants)
  const int* sched = nullptr;      // device LPT schedule of a pair launch (gemm_pair_schedule)
  int sched_rounds = 0;
  int wsplit = 1;                  // > 1: c is a [wsplit][M][N] f32 workspace of K-slice partials
};

struct TcChoice {
  int bn, cg;
};
// plan-owned state of a prepared GEMM (none needed today)
struct GemmWs {};

// Launch helpers (defined in the .cu files)
void launch_gemm_exact(const GemmArgs& g, cudaStream_t s);
// returns false when the tensor-core path cannot take this problem
bool gemm_tc_supported(const GemmArgs& g, std::string* why);
void launch_gemm_tc(const GemmArgs& g, cudaStream_t s);
// two independent problems in one persistent launch (same tile shape)
void launch_gemm_tc_pair(const GemmArgs& g0, const GemmArgs& g1, cudaStream_t s);
// host-side longest-processing-time unit schedule for a pair launch
std::vector<int> gemm_pair_schedule(const GemmArgs& g0, const GemmArgs& g1, int* rounds);
// K slices for problem idx of a pair (1 = none); partials then need
// launch_wsplit_reduce into the real output
int gemm_pair_wsplit(GemmArgs g0, GemmArgs g1, int idx);
bool gemm_wsplit_ok(const GemmArgs& g, int S);
void launch_wsplit_reduce(const float* ws, float* out, int64_t n, int S, cudaStream_t s);
// cost-model choice of tile shape / CTA pairing for a problem
TcChoice gemm_tc_choose(const GemmArgs& g);
// plan-time: freeze the tile choice (no-op for the exact kernel).
void gemm_prepare(GemmArgs& g, bool exact, GemmWs& keep);

// Fused short-sequence attention (k_attention.cu): bf16, head dim 64, S <= 128
bool attn_fused_ok(int dt, int64_t S, int64_t H, int64_t A, bool exact);
// lse != nullptr: lse mode (no P stored / loaded; per-row log-sum-exp written / read)
void launch_attn_fwd(const void* qkv, void* ctx, void* probs, int64_t B, int64_t S, int64_t H, int64_t A, float scale,
                     int causal, const DropCfg& d, cudaStream_t s, void* trace = nullptr, float* lse = nullptr);
void launch_attn_bwd(const void* qkv, const void* probs, const void* dctx, void* dqkv, int64_t B, int64_t S, int64_t H,
                     int64_t A, float scale, int causal, const DropCfg& d, cudaStream_t s, const float* lse = nullptr);

// Flash attention (k_flash.cu): any seq % 8 == 0, head dim 64, bf16; saves lse
bool flash_ok(int dt, int64_t S, int64_t H, int64_t A);
void launch_flash_fwd(const void* qkv, void* ctx, float* lse, int64_t B, int64_t S, int64_t H, int64_t A,
                      float scale, int causal, const DropCfg& d, cudaStream_t s);
void launch_flash_bwd(const void* qkv, const void* ctx, const float* lse, const void* dctx, void* dqkv,
                      float* dq_ws, int64_t B, int64_t S, int64_t H, int64_t A, float scale, int causal,
                      const DropCfg& d, cudaStream_t s);

// Picks the kernel: tcgen05 for f16/bf16 operands unless exact is requested or
// the shape is unsupported (then the exact SIMT kernel; never a CPU path).
inline void launch_gemm(const GemmArgs& g, bool exact, cudaStream_t s) {
  if (!exact && gemm_tc_supported(g, nullptr)) launch_gemm_tc(g, s);
  else launch_gemm_exact(g, s);
}

}  // namespace tcb
