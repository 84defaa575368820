// k_gemm_exact.cu -- the exact SIMT GEMM: one thread per output element,
// acc += a*b with k ascending using __fmul_rn/__fadd_rn (no FMA), exactly the
// order and roundings of matmul_ref (backends.hpp:143-155).  f32 results are
// therefore BIT-IDENTICAL to the reference; it is the b200 kernel for the fp32
// configuration (SURVEY.md §7.3 hard part 3: TF32 tensor cores miss 1e-4) and
// the parity anchor for the tensor-core path.  Operands are staged through
// shared memory in 32-wide k tiles (coalesced for either major-ness).
#include "gemm.cuh"

namespace tcb {

__device__ __forceinline__ float ld_g(const void* p, int dt, int64_t i) {
  if (dt == TCB_F32) return static_cast<const float*>(p)[i];
  if (dt == TCB_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  return __half2float(static_cast<const __half*>(p)[i]);
}
__device__ __forceinline__ void st_g(void* p, int dt, int64_t i, float v) {
  if (dt == TCB_F32) static_cast<float*>(p)[i] = v;
  else if (dt == TCB_BF16) static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else static_cast<__half*>(p)[i] = __float2half_rn(v);
}

constexpr int XT = 16;  // output tile XT x XT, one thread per output
constexpr int KT = 32;

__global__ void __launch_bounds__(XT* XT) k_gemm_exact(GemmArgs g) {
  TCB_PDL_ENTRY();
  __shared__ float sa[XT][KT + 1];  // [m][k]
  __shared__ float sb[KT][XT + 1];  // [k][n]
  const int64_t z = blockIdx.z;
  const int64_t zb = z / g.Z2, zr = z % g.Z2;
  const int64_t offa = zb * g.a.s1 + zr * g.a.s2;
  const int64_t offb = zb * g.b.s1 + zr * g.b.s2;
  const int64_t offc = zb * g.c_s1 + zr * g.c_s2;
  const int tx = threadIdx.x % XT, ty = threadIdx.x / XT;
  const int64_t m0 = int64_t(blockIdx.y) * XT, n0 = int64_t(blockIdx.x) * XT;
  const int64_t m = m0 + ty, n = n0 + tx;
  float acc = 0.0f;
  for (int64_t k0 = 0; k0 < g.K; k0 += KT) {
    // load A tile [XT m][KT k] and B tile [KT k][XT n]
    for (int idx = threadIdx.x; idx < XT * KT; idx += XT * XT) {
      int mi, ki;
      if (g.ta) { mi = idx % XT; ki = idx / XT; }  // contiguous along m
      else { ki = idx % KT; mi = idx / KT; }       // contiguous along k
      int64_t gm = m0 + mi, gk = k0 + ki;
      float v = 0.0f;
      if (gm < g.M && gk < g.K)
        v = ld_g(g.a.ptr, g.a.dtype, offa + (g.ta ? gk * g.a.ld + gm : gm * g.a.ld + gk));
      sa[mi][ki] = v;
      int ni, kj;
      if (g.tb) { kj = idx % KT; ni = idx / KT; }
      else { ni = idx % XT; kj = idx / XT; }
      int64_t gn = n0 + ni, gk2 = k0 + kj;
      float w = 0.0f;
      if (gn < g.N && gk2 < g.K)
        w = ld_g(g.b.ptr, g.b.dtype, offb + (g.tb ? gn * g.b.ld + gk2 : gk2 * g.b.ld + gn));
      sb[kj][ni] = w;
    }
    __syncthreads();
    const int kend = int(g.K - k0 < KT ? g.K - k0 : KT);
    for (int kk = 0; kk < kend; ++kk) acc = __fadd_rn(acc, __fmul_rn(sa[ty][kk], sb[kk][tx]));
    __syncthreads();
  }
  if (m >= g.M || n >= g.N) return;
  float v = g.alpha == 1.0f ? acc : __fmul_rn(acc, g.alpha);
  if (g.bias) v = __fadd_rn(v, ld_g(g.bias, g.bias_dtype, n));
  const int64_t ci = offc + m * g.ldc + n;
  if (g.dact != ACT_NONE) v = __fmul_rn(v, dact_f(g.dact, ld_g(g.aux, g.aux_dtype, ci)));
  if (g.aux_out) st_g(g.aux_out, g.c_dtype, ci, g.save_grad ? deriv_of_preact(g.act, v) : v);
  if (g.act != ACT_NONE) v = act_f(g.act, v);
  st_g(g.c, g.c_dtype, ci, v);
}

void launch_gemm_exact(const GemmArgs& g, cudaStream_t s) {
  dim3 grid(unsigned((g.N + XT - 1) / XT), unsigned((g.M + XT - 1) / XT), unsigned(g.Z));
  launch_k(k_gemm_exact, grid, XT * XT, 0, s, g);
}

}  // namespace tcb
