// k_optim.cu -- fused optimizer updates over flat parameter buffers.
//
//  sgd_update      backends.hpp:216-221  p - lr*g (float lr, no FMA): bit-exact.
//  adam_update     backends.hpp:222-243  per-element double math with bias
//                  corrections 1 - beta^t (t read from the step tensor):
//                  B200's FP64 rate makes this free next to the 28 B/param of
//                  HBM traffic, so the update is bit-exact up to the ulp of the
//                  device pow() in the bias corrections.
//  adam_update_ex  the same + grad_scale (the ZeRO 1/N mean fold)
//                  + the bf16/f16 copy of the new parameter as a 4th output
//                  (AutoCast's param cast fused into the producer).
// The VM lays all parameters (and grads, m, v) out as single flat segments, so
// one launch updates the whole model -- horizontal fusion of the per-param
// updates, i.e. a multi-tensor optimizer.
// Updates may be in place (out ptr == in ptr): each element is read before it is
// written by the same thread.
#include "common.cuh"

namespace tcb {

__global__ void k_sgd(const float* __restrict__ p, const float* __restrict__ g, float* pn, int64_t n,
                      float lr) {
  TCB_PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    pn[i] = __fsub_rn(p[i], __fmul_rn(lr, g[i]));
}

static void b_sgd(Plan& p) {
  check_arity(p, 2, 2, 1, 1);
  require(p.in[0].dtype == TCB_F32 && p.in[1].dtype == TCB_F32,
          "sgd_update: master params/grads must be f32");
  require(same_shape(p.in[0], p.in[1]), "sgd_update: param/grad shape mismatch");
  const int64_t n = p.in[0].numel();
  const float lr = float(p.attrs.f("lr", 0.0));
  p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    launch_k(k_sgd, grid_for(n, 256), 256, 0, s, (const float*)in[0].ptr, (const float*)in[1].ptr,
                                            (float*)out[0].ptr, n, lr);
  };
}
TCB_REGISTER("sgd_update", b_sgd);

struct AdamCfg {
  double lr, b1, b2, eps, gs;
};

// f64 update like the oracle, with the per-step constants folded: mhat / vhat
// multiply by precomputed 1/bc (lr/bc1 for the numerator), leaving one divide
// and one square root per element (the oracle's three divides cost the kernel
// its HBM roofline).  m, v are bit-identical to the oracle's; p differs only
// when the f64 update sits within ~1e-16 of an f32 rounding boundary.
struct AdamStep {
  double lr_bc1, rbc2;
};
template <typename TH>
__device__ __forceinline__ void adam_elem(const AdamCfg& c, const AdamStep& k, float p, float g, float m, float v,
                                          float& po, float& mo, float& vo, TH* half, int64_t i) {
  double gd = g;
  if (c.gs != 1.0) gd = __dmul_rn(gd, c.gs);
  double mi = __dadd_rn(__dmul_rn(c.b1, double(m)), __dmul_rn(__dsub_rn(1.0, c.b1), gd));
  double vi = __dadd_rn(__dmul_rn(c.b2, double(v)), __dmul_rn(__dmul_rn(__dsub_rn(1.0, c.b2), gd), gd));
  const double denom = __dadd_rn(__dsqrt_rn(__dmul_rn(vi, k.rbc2)), c.eps);
  const double upd = __ddiv_rn(__dmul_rn(k.lr_bc1, mi), denom);
  float pn = float(__dsub_rn(double(p), upd));
  po = pn;
  mo = float(mi);
  vo = float(vi);
  if (half) half[i] = from_f<TH>(pn);
}

template <typename TH>
__global__ void __launch_bounds__(256) k_adam(const float* __restrict__ p, const float* __restrict__ g,
                                              const float* __restrict__ m, const float* __restrict__ v,
                                              const float* __restrict__ step, float* po, float* mo,
                                              float* vo, TH* half, int64_t n, AdamCfg c) {
  TCB_PDL_ENTRY();
  const double t = double(step[0]);
  const double bc1 = __dsub_rn(1.0, pow(c.b1, t));
  const double bc2 = __dsub_rn(1.0, pow(c.b2, t));
  const AdamStep k{c.lr / bc1, 1.0 / bc2};
  const int64_t nv = n / 4;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < nv; q += stride) {
    float4 P = reinterpret_cast<const float4*>(p)[q];
    float4 G = reinterpret_cast<const float4*>(g)[q];
    float4 M = reinterpret_cast<const float4*>(m)[q];
    float4 V = reinterpret_cast<const float4*>(v)[q];
    float4 PO, MO, VO;
    adam_elem(c, k, P.x, G.x, M.x, V.x, PO.x, MO.x, VO.x, (TH*)nullptr, 0);
    adam_elem(c, k, P.y, G.y, M.y, V.y, PO.y, MO.y, VO.y, (TH*)nullptr, 0);
    adam_elem(c, k, P.z, G.z, M.z, V.z, PO.z, MO.z, VO.z, (TH*)nullptr, 0);
    adam_elem(c, k, P.w, G.w, M.w, V.w, PO.w, MO.w, VO.w, (TH*)nullptr, 0);
    if (half) {  // the low-precision copy as one 8- (16-bit) or 16-byte (f32) store
      if constexpr (sizeof(TH) == 2) {
        TH h4[4] = {from_f<TH>(PO.x), from_f<TH>(PO.y), from_f<TH>(PO.z), from_f<TH>(PO.w)};
        reinterpret_cast<uint2*>(half)[q] = *reinterpret_cast<const uint2*>(h4);
      } else {
        reinterpret_cast<float4*>(half)[q] = PO;
      }
    }
    reinterpret_cast<float4*>(po)[q] = PO;
    reinterpret_cast<float4*>(mo)[q] = MO;
    reinterpret_cast<float4*>(vo)[q] = VO;
  }
  for (int64_t i = nv * 4 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride)
    adam_elem(c, k, p[i], g[i], m[i], v[i], po[i], mo[i], vo[i], half, i);
}

static void b_adam(Plan& p) {
  check_arity(p, 5, 5, 3, 4);
  for (int i = 0; i < 4; ++i) {
    require(p.in[i].dtype == TCB_F32, "adam_update: master params/states must be f32");
    require(same_shape(p.in[i], p.in[0]), "adam_update: shape mismatch");
  }
  require(p.in[4].numel() == 1 && p.in[4].dtype == TCB_F32, "adam_update: step must be an f32 scalar");
  AdamCfg c{p.attrs.f("lr", 1e-3), p.attrs.f("beta1", 0.9), p.attrs.f("beta2", 0.999),
            p.attrs.f("eps", 1e-8), p.attrs.f("grad_scale", 1.0)};
  const int64_t n = p.in[0].numel();
  const int hd = p.out.size() > 3 ? p.out[3].dtype : -1;
  if (hd >= 0) require(is_float(hd), "adam_update_ex: 4th output must be a float copy");
  p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    for (int i = 0; i < 4; ++i)
      if (reinterpret_cast<uintptr_t>(in[i].ptr) % 16 || (i < 3 && reinterpret_cast<uintptr_t>(out[i].ptr) % 16))
        fail(TCB_ERR_ARG, "adam_update: buffers must be 16-byte aligned");
    if (hd >= 0 && reinterpret_cast<uintptr_t>(out[3].ptr) % 16)
      fail(TCB_ERR_ARG, "adam_update_ex: the parameter copy must be 16-byte aligned");
    const int bs = 256;
    const int grid = grid_for((n + 3) / 4, bs, kNumSMs * 4);
    if (hd == TCB_BF16)
      launch_k(k_adam<__nv_bfloat16>, grid, bs, 0, s, 
          (const float*)in[0].ptr, (const float*)in[1].ptr, (const float*)in[2].ptr,
          (const float*)in[3].ptr, (const float*)in[4].ptr, (float*)out[0].ptr, (float*)out[1].ptr,
          (float*)out[2].ptr, (__nv_bfloat16*)out[3].ptr, n, c);
    else if (hd == TCB_F16)
      launch_k(k_adam<__half>, grid, bs, 0, s, (const float*)in[0].ptr, (const float*)in[1].ptr,
                                          (const float*)in[2].ptr, (const float*)in[3].ptr,
                                          (const float*)in[4].ptr, (float*)out[0].ptr,
                                          (float*)out[1].ptr, (float*)out[2].ptr,
                                          (__half*)out[3].ptr, n, c);
    else
      launch_k(k_adam<float>, grid, bs, 0, s, (const float*)in[0].ptr, (const float*)in[1].ptr,
                                         (const float*)in[2].ptr, (const float*)in[3].ptr,
                                         (const float*)in[4].ptr, (float*)out[0].ptr,
                                         (float*)out[1].ptr, (float*)out[2].ptr,
                                         hd == TCB_F32 ? (float*)out[3].ptr : nullptr, n, c);
  };
}
TCB_REGISTER("adam_update", b_adam);
TCB_REGISTER("adam_update_ex", b_adam);

}  // namespace tcb
