// k_layernorm.cu -- layer_norm / add_layer_norm (+ fused residual dropout) forward
// (SURVEY.md §2.4 / §8a A15).  Split from k_transformer.cu so the ~90 kernel
// instantiations (dtype x H-chunks x gamma dtype x full rows) compile in parallel.
#include "k_rowops.cuh"

namespace tcb {

// ------------------------------------------------------------ layer norm fwd
// y = LN(s) where s = x (layer_norm) or s = round(dropout(x) + r) (add_layer_norm)
// NC: 8-element chunks per lane (H <= 256*NC), so the row stays in registers
// with no dead predicated slots.
template <typename T, int NC>
__global__ void __launch_bounds__(256) k_ln_fwd(const T* __restrict__ x, const T* __restrict__ r,
                                                const float* __restrict__ gamma_f,
                                                const T* __restrict__ gamma_t, const float* __restrict__ beta_f,
                                                const T* __restrict__ beta_t, T* __restrict__ y,
                                                T* __restrict__ s_out, float* __restrict__ mean_o,
                                                float* __restrict__ rstd_o, int64_t rows, int H, float eps,
                                                DropCfg d, bool vec) {
  TCB_PDL_ENTRY();
  drop_resolve(d);
  // RW rows per warp, every global load of both rows issued before the first
  // reduction so enough bytes are in flight to cover DRAM latency
  constexpr int RW = NC <= 2 ? 2 : 1;
  const int lane = threadIdx.x & 31;
  const int64_t row0 = (blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5)) * RW;
  if (row0 >= rows) return;
  const int nch = (H + 7) / 8;
  float v[RW][NC][8], rr[RW][NC][8];
#pragma unroll
  for (int q = 0; q < RW; ++q)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int64_t row = row0 + q;
      const int ch = lane + c * 32;
      if (row < rows && ch < nch) {
        const int64_t i = row * H + ch * 8;
        ld8(x, i, (row + 1) * int64_t(H), vec, v[q][c]);
        if (r) ld8(r, i, (row + 1) * int64_t(H), vec, rr[q][c]);
      }
    }
  float sum[RW];
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    sum[q] = 0.0f;
    const int64_t row = row0 + q;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ch = lane + c * 32;
      if (row < rows && ch < nch) {
        const int64_t i = row * H + ch * 8;
        if (r) {
          const uint32_t bits = drop_bits8(d, uint64_t(i));
          if (d.mask_out && (i & 7) == 0) d.mask_out[i >> 3] = uint8_t(bits);
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            float xv = ((bits >> k) & 1u) ? __fmul_rn(v[q][c][k], d.scale) : 0.0f;
            v[q][c][k] = to_f(from_f<T>(__fadd_rn(xv, rr[q][c][k])));  // s rounded to storage dtype
          }
          st8(s_out, i, (row + 1) * int64_t(H), vec, v[q][c]);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (ch * 8 + k < H) sum[q] += v[q][c][k];
      }
    }
  }
  const float inv = 1.0f / float(H);
  float mean[RW], sq[RW];
#pragma unroll
  for (int q = 0; q < RW; ++q) mean[q] = warp_sum(sum[q]) * inv;
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    sq[q] = 0.0f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ch = lane + c * 32;
      if (ch < nch) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (ch * 8 + k < H) {
            float dd = v[q][c][k] - mean[q];
            sq[q] += dd * dd;
          }
      }
    }
  }
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    const int64_t row = row0 + q;
    if (row >= rows) break;
    const float rstd = 1.0f / sqrtf(warp_sum(sq[q]) * inv + eps);
    if (lane == 0) {
      mean_o[row] = mean[q];
      rstd_o[row] = rstd;
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ch = lane + c * 32;
      if (ch < nch) {
        float o[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int j = ch * 8 + k;
          if (j < H) {
            float g = gamma_f ? __ldg(gamma_f + j) : to_f(gamma_t[j]);
            float b = beta_f ? __ldg(beta_f + j) : to_f(beta_t[j]);
            o[k] = (v[q][c][k] - mean[q]) * rstd * g + b;
          } else {
            o[k] = 0.0f;
          }
        }
        st8(y, row * H + ch * 8, (row + 1) * int64_t(H), vec, o);
      }
    }
  }
}

// 16-bit vector fast path (bf16/f16, H % 8 == 0, 16-byte rows): two rows per
// warp with every load of both rows issued up front and kept packed (8
// elements per uint4), so a 2-CTA/SM wave holds all BERT-base rows in flight.
// The path is instruction-bound (one wave, ~13 warps/SM), so: gamma / beta as
// 16-byte vectors, paired f32->16-bit conversions, y = fma(fma(s, rstd,
// -mean*rstd), g, b), and FULL (H == NC*256) drops the per-chunk guards.
template <typename T, int NC, bool GF, bool FULL>
__global__ void __launch_bounds__(256) k_ln_fwd16(const T* __restrict__ x, const T* __restrict__ r,
                                                  const void* __restrict__ gamma, const void* __restrict__ beta,
                                                  T* __restrict__ y, T* __restrict__ s_out, float* __restrict__ mean_o,
                                                  float* __restrict__ rstd_o, int64_t rows, int H, float eps,
                                                  DropCfg d) {
  TCB_PDL_ENTRY();
  drop_resolve(d);
  constexpr int RW = 2;
  __shared__ __align__(16) float sg[NC * 256], sb[NC * 256];
  const int lane = threadIdx.x & 31;
  const int64_t row0 = (blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5)) * RW;
  const int nch = FULL ? NC * 32 : H / 8;
  uint4 xq[RW][NC], rq[RW][NC];
#pragma unroll
  for (int q = 0; q < RW; ++q)
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ch = lane + c * 32;
      if (row0 + q < rows && (FULL || ch < nch)) {
        const int64_t i = (row0 + q) * H + ch * 8;
        xq[q][c] = __ldg(reinterpret_cast<const uint4*>(x + i));
        if (r) rq[q][c] = __ldg(reinterpret_cast<const uint4*>(r + i));
      }
    }
  stage_params<T, GF>(gamma, beta, sg, sb, H);
  __syncthreads();
  const float inv = 1.0f / float(H);
  const float2 sc2 = splat2(d.scale);
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    const int64_t row = row0 + q;
    if (row >= rows) break;
    float2 v[NC][4];
    float2 sum2 = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ch = lane + c * 32;
      if (FULL || ch < nch) {
        unpack8x2<T>(xq[q][c], v[c]);
        if (r) {
          const int64_t i = row * H + ch * 8;
          float2 rv[4];
          unpack8x2<T>(rq[q][c], rv);
          const uint32_t bits = d.p > 0.0f ? dropout_bits8q(d, uint64_t(i) >> 3) : 0xFFu;
          if (d.mask_out) d.mask_out[i >> 3] = uint8_t(bits);
          float2 sv[4];
#pragma unroll
          for (int k = 0; k < 4; ++k) sv[k] = add2(keep2(bits, 2 * k, mul2(v[c][k], sc2)), rv[k]);
          const uint4 w = pack8x2<T>(sv);  // s in the storage dtype
          unpack8x2<T>(w, v[c]);
          *reinterpret_cast<uint4*>(s_out + i) = w;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) sum2 = add2(sum2, v[c][k]);
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) v[c][k] = make_float2(0.0f, 0.0f);
      }
    }
    const float mean = warp_sum(sum2.x + sum2.y) * inv;
    const float2 nm2 = splat2(-mean);
    float2 sq2 = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (FULL || lane + c * 32 < nch)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const float2 dd = add2(v[c][k], nm2);
          sq2 = fma2(dd, dd, sq2);
        }
    const float rstd = 1.0f / sqrtf(warp_sum(sq2.x + sq2.y) * inv + eps);
    const float2 rs2 = splat2(rstd), nmr2 = splat2(-mean * rstd);
    if (lane == 0) {
      mean_o[row] = mean;
      rstd_o[row] = rstd;
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ch = lane + c * 32;
      if (FULL || ch < nch) {
        float2 g[4], b[4], o[4];
        lds8x2(sg + ch * 8, g);
        lds8x2(sb + ch * 8, b);
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = fma2(fma2(v[c][k], rs2, nmr2), g[k], b[k]);
        uint4 w = pack8x2<T>(o);
        if (!r && d.p > 0.0f) {  // post_dropout: dropout(LN(x)) as the separate op rounds it
          const uint32_t bits = dropout_bits8q(d, uint64_t(row * H + ch * 8) >> 3);
          unpack8x2<T>(w, o);
#pragma unroll
          for (int k = 0; k < 4; ++k) o[k] = keep2(bits, 2 * k, mul2(o[k], sc2));
          w = pack8x2<T>(o);
        }
        *reinterpret_cast<uint4*>(y + row * H + ch * 8) = w;
      }
    }
  }
}

static void build_ln_fwd(Plan& p, bool residual) {
  if (residual) check_arity(p, 4, 4, 4, 5);
  else check_arity(p, 3, 3, 3, 3);
  // add_layer_norm save_mask: a 5th output holds the residual-branch keep bits
  const bool save_mask = residual && p.out.size() == 5;
  const Spec& X = p.in[0];
  const int H = int(X.dim(-1));
  const int64_t rows = X.numel() / H;
  require(H <= LN_MAXC * 8 * 32, p.op + ": hidden size > 2048 unsupported");
  const Spec& G = p.in[residual ? 2 : 1];
  require(G.numel() == H, p.op + ": gamma must have H elements");
  require(G.dtype == TCB_F32 || G.dtype == X.dtype, p.op + ": gamma dtype");
  const bool gf = G.dtype == TCB_F32;
  const float eps = float(p.attrs.f("eps", 1e-12));
  DropCfg d0 = drop_cfg(p.attrs);
  // plain layer_norm: dropout on the OUTPUT only with attr post_dropout (16-bit path)
  const bool post_drop = !residual && p.attrs.i("post_dropout", 0) != 0 && d0.p > 0.0f;
  if (!residual && !post_drop) d0 = DropCfg{};
  if (post_drop) require(X.dtype != TCB_F32 && H % 8 == 0, p.op + ": post_dropout needs a 16-bit input, H % 8 == 0");
  if (save_mask)
    require(H % 8 == 0 && d0.p > 0.0f && p.out[4].numel() * dtype_bytes(p.out[4].dtype) * 8 >= X.numel(),
            p.op + ": save_mask needs p > 0, H % 8 == 0 and a T*H/8-byte mask output");
  dispatch_float(X.dtype, [&](auto* tp) {
   using T = std::remove_pointer_t<decltype(tp)>;
   dispatch_nc(H, [&](auto nc) {
    constexpr int NC = decltype(nc)::value;
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      DropCfg d = with_step(d0);
      if (save_mask) d.mask_out = static_cast<uint8_t*>(out[4].ptr);
      const int gi = residual ? 2 : 1;
      bool vec = (H % 8 == 0);
      for (int i = 0; i < (residual ? 2 : 1); ++i) vec = vec && reinterpret_cast<uintptr_t>(in[i].ptr) % 16 == 0;
      vec = vec && reinterpret_cast<uintptr_t>(out[0].ptr) % 16 == 0;
      if (residual) vec = vec && reinterpret_cast<uintptr_t>(out[1].ptr) % 16 == 0;
      if constexpr (sizeof(T) == 2) {
        // parameter vectors need 16-byte alignment too
        for (int i = gi; i < gi + 2; ++i) vec = vec && reinterpret_cast<uintptr_t>(in[i].ptr) % 16 == 0;
        if (vec) {
          const bool full = H == NC * 256;
          auto kern = gf ? (full ? k_ln_fwd16<T, NC, true, true> : k_ln_fwd16<T, NC, true, false>)
                         : (full ? k_ln_fwd16<T, NC, false, true> : k_ln_fwd16<T, NC, false, false>);
          launch_k(kern, unsigned((rows + 15) / 16), 256, 0, s, (const T*)in[0].ptr,
                   residual ? (const T*)in[1].ptr : nullptr, (const void*)in[gi].ptr, (const void*)in[gi + 1].ptr,
                   (T*)out[0].ptr, residual ? (T*)out[1].ptr : nullptr, (float*)out[residual ? 2 : 1].ptr,
                   (float*)out[residual ? 3 : 2].ptr, rows, H, eps, d);
          return;
        }
      }
      if (post_drop) fail(TCB_ERR_UNIMPLEMENTED, p.op + ": post_dropout needs aligned 16-bit rows");
      constexpr int RW = NC <= 2 ? 2 : 1;
      launch_k(k_ln_fwd<T, NC>, unsigned((rows + 8 * RW - 1) / (8 * RW)), 256, 0, s, 
          (const T*)in[0].ptr, residual ? (const T*)in[1].ptr : nullptr,
          gf ? (const float*)in[gi].ptr : nullptr, gf ? nullptr : (const T*)in[gi].ptr,
          gf ? (const float*)in[gi + 1].ptr : nullptr, gf ? nullptr : (const T*)in[gi + 1].ptr,
          (T*)out[0].ptr, residual ? (T*)out[1].ptr : nullptr, (float*)out[residual ? 2 : 1].ptr,
          (float*)out[residual ? 3 : 2].ptr, rows, H, eps, d, vec);
    };
   });
  });
}
static void b_layer_norm(Plan& p) { build_ln_fwd(p, false); }
static void b_add_layer_norm(Plan& p) { build_ln_fwd(p, true); }
TCB_REGISTER("layer_norm", b_layer_norm);
TCB_REGISTER("add_layer_norm", b_add_layer_norm);

}  // namespace tcb
