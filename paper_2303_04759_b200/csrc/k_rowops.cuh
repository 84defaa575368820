// k_rowops.cuh -- shared row-kernel helpers of the transformer ops (k_layernorm.cu,
// k_layernorm_dx.cu, k_transformer.cu): warp reductions, 8-wide vector
// load/store and pack/unpack, the H-chunk dispatch, dropout keep bits.
#pragma once
#include "gemm.cuh"
#include "fold.cuh"

namespace tcb {

// ---------------------------------------------------------------- utilities
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int m = 16; m; m >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, m));
  return v;
}


// 8 consecutive elements <-> floats
template <typename T>
struct Vec8;
template <>
struct Vec8<__nv_bfloat16> {
  static __device__ __forceinline__ void load(const __nv_bfloat16* p, float* f) {
    uint4 q = *reinterpret_cast<const uint4*>(p);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __bfloat1622float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  static __device__ __forceinline__ void store(__nv_bfloat16* p, const float* f) {
    uint4 q;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = q;
  }
};
template <>
struct Vec8<__half> {
  static __device__ __forceinline__ void load(const __half* p, float* f) {
    uint4 q = *reinterpret_cast<const uint4*>(p);
    const __half2* h = reinterpret_cast<const __half2*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float2 t = __half22float2(h[i]);
      f[2 * i] = t.x;
      f[2 * i + 1] = t.y;
    }
  }
  static __device__ __forceinline__ void store(__half* p, const float* f) {
    uint4 q;
    __half2* h = reinterpret_cast<__half2*>(&q);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2half2_rn(f[2 * i], f[2 * i + 1]);
    *reinterpret_cast<uint4*>(p) = q;
  }
};
template <>
struct Vec8<float> {
  static __device__ __forceinline__ void load(const float* p, float* f) {
    float4 a = *reinterpret_cast<const float4*>(p), b = *reinterpret_cast<const float4*>(p + 4);
    f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
    f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
  }
  static __device__ __forceinline__ void store(float* p, const float* f) {
    *reinterpret_cast<float4*>(p) = make_float4(f[0], f[1], f[2], f[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(f[4], f[5], f[6], f[7]);
  }
};

// load/store 8 elements starting at i (vector path when aligned, else scalar)
template <typename T>
__device__ __forceinline__ void ld8(const T* p, int64_t i, int64_t n, bool vec, float* f) {
  if (vec) {
    Vec8<T>::load(p + i, f);
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = i + k < n ? to_f(p[i + k]) : 0.0f;
  }
}
template <typename T>
__device__ __forceinline__ void st8(T* p, int64_t i, int64_t n, bool vec, const float* f) {
  if (vec) {
    Vec8<T>::store(p + i, f);
  } else {
#pragma unroll
    for (int k = 0; k < 8; ++k)
      if (i + k < n) p[i + k] = from_f<T>(f[k]);
  }
}

constexpr int LN_MAXC = 8;  // up to 8 chunks of 8 per lane: H <= 2048

// calls f(std::integral_constant<int, NC>) with NC = ceil(H / 256)
template <typename Fn>
static void dispatch_nc(int H, Fn&& f) {
  switch ((H + 255) / 256) {
    case 1: f(std::integral_constant<int, 1>{}); return;
    case 2: f(std::integral_constant<int, 2>{}); return;
    case 3: f(std::integral_constant<int, 3>{}); return;
    case 4: f(std::integral_constant<int, 4>{}); return;
    case 5: f(std::integral_constant<int, 5>{}); return;
    case 6: f(std::integral_constant<int, 6>{}); return;
    case 7: f(std::integral_constant<int, 7>{}); return;
    case 8: f(std::integral_constant<int, 8>{}); return;
  }
  fail(TCB_ERR_UNIMPLEMENTED, "layer norm: hidden size > 2048 unsupported");
}

// keep bits for elements i .. i+7 (two Philox calls when i is 4-aligned)
__device__ __forceinline__ uint32_t drop_bits8(const DropCfg& d, uint64_t i) {
  if (d.p <= 0.0f) return 0xFFu;
  if ((i & 7) == 0) return dropout_bits8q(d, i >> 3);
  uint32_t b = 0;
  for (int k = 0; k < 8; ++k) b |= uint32_t(dropout_keep(d, i + k)) << k;
  return b;
}

template <typename T>
__device__ __forceinline__ void unpack8(const uint4& q, float* f) {
  const T* h = reinterpret_cast<const T*>(&q);
#pragma unroll
  for (int k = 0; k < 8; ++k) f[k] = to_f(h[k]);
}
template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b) {
  if constexpr (std::is_same<T, __nv_bfloat16>::value) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  } else {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
}
template <typename T>
__device__ __forceinline__ uint4 pack8(const float* f) {
  return make_uint4(pack2<T>(f[0], f[1]), pack2<T>(f[2], f[3]), pack2<T>(f[4], f[5]), pack2<T>(f[6], f[7]));
}
// 8 packed 16-bit values <-> 4 float2 (element pairs for the f32x2 ops)
template <typename T>
__device__ __forceinline__ void unpack8x2(const uint4& q, float2* f) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&q);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    if constexpr (std::is_same<T, __nv_bfloat16>::value) f[k] = bf2_to_f2(w[k]);
    else f[k] = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
  }
}
template <typename T>
__device__ __forceinline__ uint4 pack8x2(const float2* f) {
  return make_uint4(pack2<T>(f[0].x, f[0].y), pack2<T>(f[1].x, f[1].y), pack2<T>(f[2].x, f[2].y),
                    pack2<T>(f[3].x, f[3].y));
}
// keep-mask select of a pair: (bit k ? t.x : 0, bit k+1 ? t.y : 0)
__device__ __forceinline__ float2 keep2(uint32_t bits, int k, float2 t) {
  return make_float2(((bits >> k) & 1u) ? t.x : 0.0f, ((bits >> (k + 1)) & 1u) ? t.y : 0.0f);
}
// per-column f32 parameters staged in smem once per CTA (gamma [, beta]): one
// 16-byte load per thread, all in flight together (H % 8 == 0, 16-byte aligned)
template <typename T, bool GF>
__device__ __forceinline__ void stage_params(const void* g, const void* b, float* sg, float* sb, int H) {
  const int n8 = H / 8, n = b ? 2 * n8 : n8;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    const bool isb = i >= n8;
    const int c = isb ? i - n8 : i;
    float4* dst = reinterpret_cast<float4*>((isb ? sb : sg) + c * 8);
    if constexpr (GF) {
      const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(isb ? b : g) + c * 8);
      const float4 u = __ldg(src), v = __ldg(src + 1);
      dst[0] = u;
      dst[1] = v;
    } else {
      float f[8];
      unpack8<T>(__ldg(reinterpret_cast<const uint4*>(static_cast<const T*>(isb ? b : g) + c * 8)), f);
      dst[0] = make_float4(f[0], f[1], f[2], f[3]);
      dst[1] = make_float4(f[4], f[5], f[6], f[7]);
    }
  }
}
__device__ __forceinline__ void lds8x2(const float* p, float2* f) {
  const float4 a = reinterpret_cast<const float4*>(p)[0], b = reinterpret_cast<const float4*>(p)[1];
  f[0] = make_float2(a.x, a.y); f[1] = make_float2(a.z, a.w);
  f[2] = make_float2(b.x, b.y); f[3] = make_float2(b.z, b.w);
}

}  // namespace tcb
