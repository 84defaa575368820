// k_layernorm_dx.cu -- layer_norm_dx (+ fused dy fan-in, dropout and bias
// gradient) backward.  Split from k_transformer.cu
// for parallel compilation.
#include "k_rowops.cuh"

namespace tcb {

// ------------------------------------------------------------ layer norm bwd
// dy += dy2 (fused fan-out accumulation); ds = rstd*(g - mean(g) - xh*mean(g*xh));
// dx = dropout(ds);
// per-CTA partial column sums of dy*xh and dy -> ws, then k_colsum finalises.
constexpr int LNB_ROWS = 16;  // rows per CTA (8 warps x 2 rows)

template <typename T, int NC>
__global__ void __launch_bounds__(256) k_ln_bwd(const T* __restrict__ sx, const float* __restrict__ gamma_f,
                                                const T* __restrict__ gamma_t, const float* __restrict__ mean,
                                                const float* __restrict__ rstd, const T* __restrict__ dy,
                                                const T* __restrict__ dy2, T* __restrict__ ds_o,
                                                T* __restrict__ dx_o, float* __restrict__ ws, int nparts,
                                                int64_t rows, int H, DropCfg d, bool vec) {
  TCB_PDL_ENTRY();
  drop_resolve(d);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nch = (H + 7) / 8;
  // per-warp dgamma/dbeta partials live in smem (not registers), laid out
  // [warp][2][k][chunk] so a warp's accesses are bank-conflict free
  extern __shared__ float red[];
  constexpr int CP = NC * 32;  // chunk pitch
  float* pg = red + (warp * 3 + 0) * 8 * CP;
  float* pb = red + (warp * 3 + 1) * 8 * CP;
  float* pz = red + (warp * 3 + 2) * 8 * CP;  // bias grad: column sums of the outgoing gradient
#pragma unroll
  for (int c = 0; c < NC; ++c)
#pragma unroll
    for (int k = 0; k < 8; ++k) pg[k * CP + c * 32 + lane] = pb[k * CP + c * 32 + lane] = pz[k * CP + c * 32 + lane] = 0.0f;
  const float inv = 1.0f / float(H);
  for (int rr = 0; rr < LNB_ROWS / 8; ++rr) {
    const int64_t row = int64_t(blockIdx.x) * LNB_ROWS + warp * (LNB_ROWS / 8) + rr;
    if (row >= rows) break;
    const float mu = mean[row], rs = rstd[row];
    float xh[NC][8], g[NC][8];
    float c1 = 0.0f, c2 = 0.0f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ch = lane + c * 32;
      if (ch < nch) {
        const int64_t i = row * H + ch * 8;
        float sv[8], dv[8];
        ld8(sx, i, (row + 1) * int64_t(H), vec, sv);
        ld8(dy, i, (row + 1) * int64_t(H), vec, dv);
        if (dy2) {
          float d2[8];
          ld8(dy2, i, (row + 1) * int64_t(H), vec, d2);
#pragma unroll
          for (int k = 0; k < 8; ++k) dv[k] = __fadd_rn(dv[k], d2[k]);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int j = ch * 8 + k;
          if (j < H) {
            float gm = gamma_f ? gamma_f[j] : to_f(gamma_t[j]);
            xh[c][k] = (sv[k] - mu) * rs;
            g[c][k] = dv[k] * gm;
            c1 += g[c][k] * xh[c][k];
            c2 += g[c][k];
            pg[k * CP + c * 32 + lane] += dv[k] * xh[c][k];
            pb[k * CP + c * 32 + lane] += dv[k];
          } else {
            xh[c][k] = g[c][k] = 0.0f;
          }
        }
      }
    }
    c1 = warp_sum(c1) * inv;
    c2 = warp_sum(c2) * inv;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ch = lane + c * 32;
      if (ch < nch) {
        const int64_t i = row * H + ch * 8;
        float o[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = rs * (g[c][k] - c2 - xh[c][k] * c1);
        st8(ds_o, i, (row + 1) * int64_t(H), vec, o);
        if (dx_o) {
          const uint32_t bits = d.mask_in ? uint32_t(d.mask_in[i >> 3]) : drop_bits8(d, uint64_t(i));
#pragma unroll
          for (int k = 0; k < 8; ++k) o[k] = ((bits >> k) & 1u) ? o[k] * d.scale : 0.0f;
          st8(dx_o, i, (row + 1) * int64_t(H), vec, o);
        }
        if (nparts > 2) {
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (ch * 8 + k < H) pz[k * CP + c * 32 + lane] += to_f(from_f<T>(o[k]));
        }
      }
    }
  }
  // CTA partials: fold the 8 warps' smem rows, then one row of ws per CTA
  __syncthreads();
  for (int j = threadIdx.x; j < H; j += blockDim.x) {
    const int off = (j & 7) * CP + (j >> 3);
    for (int a = 0; a < nparts; ++a) {
      float acc = 0.0f;
      for (int w = 0; w < 8; ++w) acc += red[(w * 3 + a) * 8 * CP + off];
      ws[(int64_t(blockIdx.x) * nparts + a) * H + j] = acc;
    }
  }
}

// 16-bit vector fast path: both rows' loads issued up front (packed). Pass 1
// walks chunk-major over the two rows, so each column's dgamma / dbeta partial
// (the two rows' sum) is complete in registers and stored once to the warp's
// smem row [warp][part][H] (no read-modify-write); pass 2 recomputes xh and g
// from the packed loads, writes ds / dx and the bias-grad partial likewise.
// The 8 warp rows fold per CTA (16-byte smem reads) into one ws row per part.
template <typename T, int NC, bool GF, bool FULL>
__global__ void __launch_bounds__(256, NC <= 3 ? 2 : 1) k_ln_bwd16(const T* __restrict__ sx, const void* __restrict__ gamma,
                                                  const float* __restrict__ mean, const float* __restrict__ rstd,
                                                  const T* __restrict__ dy, const T* __restrict__ dy2,
                                                  T* __restrict__ ds_o, T* __restrict__ dx_o, float* __restrict__ ws,
                                                  int nparts, int64_t rows, int H, DropCfg d, DropCfg din) {
  TCB_PDL_ENTRY();
  drop_resolve(d);
  drop_resolve(din);
  constexpr int RW = LNB_ROWS / 8;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nch = FULL ? NC * 32 : H / 8;
  extern __shared__ __align__(16) float red[];  // [8 warps][3 parts][H], then gamma (f32) [H]
  float* prow = red + warp * 3 * H;
  float* sg = red + 8 * 3 * H;
  const int64_t row0 = int64_t(blockIdx.x) * LNB_ROWS + warp * RW;
  uint4 sq[RW][NC], dq[RW][NC], d2q[RW][NC];
  float2 rs2[RW], nmr2[RW];
  bool live[RW];
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    live[q] = row0 + q < rows;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int ch = lane + c * 32;
      if (live[q] && (FULL || ch < nch)) {
        const int64_t i = (row0 + q) * H + ch * 8;
        sq[q][c] = __ldg(reinterpret_cast<const uint4*>(sx + i));
        dq[q][c] = __ldg(reinterpret_cast<const uint4*>(dy + i));
        if (dy2) d2q[q][c] = __ldg(reinterpret_cast<const uint4*>(dy2 + i));
      }
    }
    const float mu = live[q] ? mean[row0 + q] : 0.0f, rs = live[q] ? rstd[row0 + q] : 0.0f;
    rs2[q] = splat2(rs);
    nmr2[q] = splat2(-mu * rs);
  }
  stage_params<T, GF>(gamma, nullptr, sg, nullptr, H);
  __syncthreads();
  // in_dropout (the output dropout of a plain layer_norm folded in): the incoming
  // gradient is the separate dropout op's result, round(keep ? dy * scale : 0)
  uint32_t inb[RW][NC];
  if (din.p > 0.0f) {
#pragma unroll
    for (int q = 0; q < RW; ++q)
#pragma unroll
      for (int c = 0; c < NC; ++c)
        inb[q][c] = live[q] ? dropout_bits8q(din, uint64_t((row0 + q) * H + (lane + c * 32) * 8) >> 3) : 0u;
  }
  const float2 isc2 = splat2(din.scale);
  // xh = s*rs - mu*rs, dv = dy + dy2 and g = dv * gamma of chunk c of row q (pairs)
  auto load_row = [&](int q, int c, const float2* gm, float2* xh, float2* dv, float2* g) {
    float2 sv[4];
    unpack8x2<T>(sq[q][c], sv);
    unpack8x2<T>(dq[q][c], dv);
    if (din.p > 0.0f) {
#pragma unroll
      for (int k = 0; k < 4; ++k) dv[k] = keep2(inb[q][c], 2 * k, mul2(dv[k], isc2));
      const uint4 w = pack8x2<T>(dv);
      unpack8x2<T>(w, dv);
    }
    if (dy2) {
      float2 d2[4];
      unpack8x2<T>(d2q[q][c], d2);
#pragma unroll
      for (int k = 0; k < 4; ++k) dv[k] = add2(dv[k], d2[k]);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      xh[k] = fma2(sv[k], rs2[q], nmr2[q]);
      g[k] = mul2(dv[k], gm[k]);
    }
  };
  const float inv = 1.0f / float(H);
  float2 c1[RW], c2[RW];
#pragma unroll
  for (int q = 0; q < RW; ++q) c1[q] = c2[q] = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ch = lane + c * 32;
    if (!(FULL || ch < nch)) continue;
    float2 gm[4], pg[4], pb[4];
    lds8x2(sg + ch * 8, gm);
#pragma unroll
    for (int k = 0; k < 4; ++k) pg[k] = pb[k] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      if (!live[q]) break;
      float2 xh[4], dv[4], g[4];
      load_row(q, c, gm, xh, dv, g);
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        c1[q] = fma2(g[k], xh[k], c1[q]);
        c2[q] = add2(c2[q], g[k]);
        pg[k] = fma2(dv[k], xh[k], pg[k]);
        pb[k] = add2(pb[k], dv[k]);
      }
    }
    float4* o0 = reinterpret_cast<float4*>(prow + ch * 8);
    float4* o1 = reinterpret_cast<float4*>(prow + H + ch * 8);
    o0[0] = make_float4(pg[0].x, pg[0].y, pg[1].x, pg[1].y);
    o0[1] = make_float4(pg[2].x, pg[2].y, pg[3].x, pg[3].y);
    o1[0] = make_float4(pb[0].x, pb[0].y, pb[1].x, pb[1].y);
    o1[1] = make_float4(pb[2].x, pb[2].y, pb[3].x, pb[3].y);
  }
  // o = rs * (g - c2 - xh * c1) = fma(rs, g, fma(xh, -rs*c1, -rs*c2))
  float2 a1[RW], a0[RW];
#pragma unroll
  for (int q = 0; q < RW; ++q) {
    const float m1 = warp_sum(c1[q].x + c1[q].y) * inv, m2 = warp_sum(c2[q].x + c2[q].y) * inv;
    a1[q] = splat2(-rs2[q].x * m1);
    a0[q] = splat2(-rs2[q].x * m2);
  }
  const float2 sc2 = splat2(d.scale);
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    const int ch = lane + c * 32;
    if (!(FULL || ch < nch)) continue;
    float2 gm[4], pz[4];
    lds8x2(sg + ch * 8, gm);
#pragma unroll
    for (int k = 0; k < 4; ++k) pz[k] = make_float2(0.0f, 0.0f);
#pragma unroll
    for (int q = 0; q < RW; ++q) {
      if (!live[q]) break;
      float2 xh[4], dv[4], g[4], o[4];
      load_row(q, c, gm, xh, dv, g);
      const int64_t i = (row0 + q) * H + ch * 8;
#pragma unroll
      for (int k = 0; k < 4; ++k) o[k] = fma2(rs2[q], g[k], fma2(xh[k], a1[q], a0[q]));
      uint4 w = pack8x2<T>(o);
      *reinterpret_cast<uint4*>(ds_o + i) = w;
      if (dx_o) {
        const uint32_t bits = d.mask_in ? uint32_t(d.mask_in[i >> 3])
                              : d.p > 0.0f ? dropout_bits8q(d, uint64_t(i) >> 3) : 0xFFu;
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = keep2(bits, 2 * k, mul2(o[k], sc2));
        w = pack8x2<T>(o);
        *reinterpret_cast<uint4*>(dx_o + i) = w;
      }
      if (nparts > 2) {  // bias grad: the outgoing gradient as stored
        float2 f[4];
        unpack8x2<T>(w, f);
#pragma unroll
        for (int k = 0; k < 4; ++k) pz[k] = add2(pz[k], f[k]);
      }
    }
    if (nparts > 2) {
      float4* o2 = reinterpret_cast<float4*>(prow + 2 * H + ch * 8);
      o2[0] = make_float4(pz[0].x, pz[0].y, pz[1].x, pz[1].y);
      o2[1] = make_float4(pz[2].x, pz[2].y, pz[3].x, pz[3].y);
    }
  }
  // warps whose rows are all past the end contribute zeros
  if (!live[0]) {
    for (int j = lane * 4; j < 3 * H; j += 128) *reinterpret_cast<float4*>(prow + j) = make_float4(0, 0, 0, 0);
  }
  __syncthreads();
  for (int j = threadIdx.x * 4; j < H; j += blockDim.x * 4) {
    for (int a = 0; a < nparts; ++a) {
      float4 acc = make_float4(0, 0, 0, 0);
#pragma unroll
      for (int w = 0; w < 8; ++w) {
        const float4 t = *reinterpret_cast<const float4*>(red + (w * 3 + a) * H + j);
        acc.x += t.x; acc.y += t.y; acc.z += t.z; acc.w += t.w;
      }
      *reinterpret_cast<float4*>(ws + (int64_t(blockIdx.x) * nparts + a) * H + j) = acc;
    }
  }
}

// sum the per-CTA partials in fixed order -> dgamma, dbeta (f32): block = 32
// columns x 8 warps; warp w folds partial rows w, w+8, ...; smem combines.
// fold the per-CTA partial rows ws[k][a][j] (k < nblk, a < np) in fixed order:
// block = 32 columns x 32 warps, warp w sums rows w, w+32, ... (loads
// unrolled), then warp a folds the 32 warp sums of part a in warp order
__global__ void __launch_bounds__(1024) k_ln_colsum(const float* __restrict__ ws, float* __restrict__ dg,
                                                    float* __restrict__ db, float* __restrict__ dbias, int nblk,
                                                    int H) {
  TCB_PDL_ENTRY();
  __shared__ float ra[3][32][33];
  const int np = dbias ? 3 : 2;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j = blockIdx.x * 32 + lane;
  float acc[3] = {0.0f, 0.0f, 0.0f};
  if (j < H) {
#pragma unroll 4
    for (int k = warp; k < nblk; k += 32) {
#pragma unroll
      for (int a = 0; a < 3; ++a)
        if (a < np) acc[a] += ws[(int64_t(k) * np + a) * H + j];
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) ra[a][warp][lane] = acc[a];
  __syncthreads();
  if (warp < np && j < H) {
    float t = 0.0f;
#pragma unroll 8
    for (int w = 0; w < 32; ++w) t += ra[warp][w][lane];
    (warp == 0 ? dg : warp == 1 ? db : dbias)[j] = t;
  }
}

static void b_layer_norm_dx(Plan& p) {
  // mask_in: the last input holds the forward's saved keep bits
  const bool mask_in = p.attrs.i("mask_in", 0) != 0;
  check_arity(p, 5 + int(mask_in), 6 + int(mask_in), 3, 5);
  const Spec& S = p.in[0];
  const int H = int(S.dim(-1));
  const int64_t rows = S.numel() / H;
  require(H <= LN_MAXC * 8 * 32, "layer_norm_dx: hidden size > 2048 unsupported");
  require(p.out[1].dtype == TCB_F32 && p.out[2].dtype == TCB_F32, "layer_norm_dx: dgamma/dbeta are f32");
  const bool gf = p.in[1].dtype == TCB_F32;
  const DropCfg d0 = drop_cfg(p.attrs);
  // in_p / in_seed / in_salt: the forward layer_norm's post_dropout, applied to dy
  DropCfg din;
  din.p = float(p.attrs.f("in_p", 0.0));
  din.scale = din.p > 0.0f ? 1.0f / (1.0f - din.p) : 1.0f;
  din.seed = uint64_t(p.attrs.i("in_seed", 0));
  din.salt = uint64_t(p.attrs.i("in_salt", 0));
  din.thr = din.p > 0.0f ? uint32_t(std::ceil(double(din.p) * 65536.0)) : 0u;
  const bool bias = p.attrs.i("bias_grad", 0) != 0;
  const bool has_res = int(p.in.size()) - int(mask_in) > 5, has_dx = int(p.out.size()) - int(bias) > 3;
  const int nin = int(p.in.size());
  if (mask_in) require(H % 8 == 0, "layer_norm_dx: mask_in needs H % 8 == 0");
  // the kernels read every activation-shaped input (dy, x, the residual dy2) as S's dtype
  for (int i = 1; i < nin - int(mask_in); ++i)
    if (p.in[i].numel() == S.numel())
      require(p.in[i].dtype == S.dtype, "layer_norm_dx: activation-shaped inputs must share one dtype");
  const int di = has_dx ? 4 : 3;  // index of the fused bias-grad output
  require(int(p.out.size()) - int(bias) >= 3, "layer_norm_dx: outputs (ds, dg, db [, dx] [, dbias])");
  if (bias) require(p.out[di].dtype == TCB_F32 && p.out[di].numel() == H, "layer_norm_dx: dbias is f32 [H]");
  const int np = bias ? 3 : 2;
  const int nblk = int((rows + LNB_ROWS - 1) / LNB_ROWS);
  const size_t ws = p.ws_take(size_t(nblk) * np * H * sizeof(float));
  const int ncs = (H + 255) / 256;
  const size_t smem = size_t(8) * 3 * 8 * 32 * ncs * sizeof(float) + size_t(H) * sizeof(float);  // partials + gamma
  p.nkernels = 2;
  dispatch_float(S.dtype, [&](auto* tp) {
   using T = std::remove_pointer_t<decltype(tp)>;
   dispatch_nc(H, [&](auto nc) {
    constexpr int NC = decltype(nc)::value;
    static std::once_flag once;
    std::call_once(once, [] {
      constexpr int sm = 8 * 3 * 8 * 32 * NC * 4 + NC * 256 * 4;
      TCB_CUDA(cudaFuncSetAttribute(k_ln_bwd<T, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      if constexpr (sizeof(T) == 2) {
        TCB_CUDA(cudaFuncSetAttribute(k_ln_bwd16<T, NC, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        TCB_CUDA(cudaFuncSetAttribute(k_ln_bwd16<T, NC, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        TCB_CUDA(cudaFuncSetAttribute(k_ln_bwd16<T, NC, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        TCB_CUDA(cudaFuncSetAttribute(k_ln_bwd16<T, NC, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      }
    });
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      DropCfg d = with_step(d0);
      if (mask_in) d.mask_in = static_cast<const uint8_t*>(in[nin - 1].ptr);
      bool vec = H % 8 == 0;
      for (int i : {0, 4}) vec = vec && reinterpret_cast<uintptr_t>(in[i].ptr) % 16 == 0;
      if (has_res) vec = vec && reinterpret_cast<uintptr_t>(in[5].ptr) % 16 == 0;
      vec = vec && reinterpret_cast<uintptr_t>(out[0].ptr) % 16 == 0;
      if (has_dx) vec = vec && reinterpret_cast<uintptr_t>(out[3].ptr) % 16 == 0;
      const float* gfp = gf ? (const float*)in[1].ptr : nullptr;
      const T* gtp = gf ? nullptr : (const T*)in[1].ptr;
      const T* d2 = has_res ? (const T*)in[5].ptr : nullptr;
      T* dxp = has_dx ? (T*)out[3].ptr : nullptr;
      bool fast = false;
      if constexpr (sizeof(T) == 2) fast = vec && reinterpret_cast<uintptr_t>(in[1].ptr) % 16 == 0;
      // deferred fold: this instance's partials go to its own buffer, folded at the flush
      float* dws = fold_deferring() ? fold_scratch(out[1].ptr, 0, size_t(nblk) * np * H * sizeof(float)) : nullptr;
      float* wsp = dws ? dws : (float*)ws_at(ws);
      if (din.p > 0.0f && (!fast || has_res))
        fail(TCB_ERR_UNIMPLEMENTED, "layer_norm_dx: in_p needs the 16-bit path and a single dy");
      if (fast) {
        if constexpr (sizeof(T) == 2) {
          const bool full = H == NC * 256;
          auto kern = gf ? (full ? k_ln_bwd16<T, NC, true, true> : k_ln_bwd16<T, NC, true, false>)
                         : (full ? k_ln_bwd16<T, NC, false, true> : k_ln_bwd16<T, NC, false, false>);
          launch_k(kern, nblk, 256, smem, s, (const T*)in[0].ptr, (const void*)in[1].ptr, (const float*)in[2].ptr,
                   (const float*)in[3].ptr, (const T*)in[4].ptr, d2, (T*)out[0].ptr, dxp, wsp, np, rows, H,
                   d, with_step(din));
        }
      } else {
        launch_k(k_ln_bwd<T, NC>, nblk, 256, smem, s, (const T*)in[0].ptr, gfp, gtp, (const float*)in[2].ptr,
                 (const float*)in[3].ptr, (const T*)in[4].ptr, d2, (T*)out[0].ptr, dxp, wsp, np, rows, H, d,
                 vec);
      }
      if (dws) {
        float* dst[3] = {(float*)out[1].ptr, (float*)out[2].ptr, bias ? (float*)out[di].ptr : nullptr};
        for (int a = 0; a < np; ++a) fold_defer(FoldJob{dws + size_t(a) * H, int64_t(np) * H, nblk, H, dst[a], 1.0f});
        fold_op_deferred();
        return;
      }
      if (!skip_folds()) launch_k(k_ln_colsum, (H + 31) / 32, 1024, 0, s, (const float*)ws_at(ws), (float*)out[1].ptr, (float*)out[2].ptr,
               bias ? (float*)out[di].ptr : nullptr, nblk, H);
    };
   });
  });
}
TCB_REGISTER("layer_norm_dx", b_layer_norm_dx);

}  // namespace tcb
