// k_reduce.cu -- b200 kernels for sum / mean (backends.hpp:95-141) and mse
// (backends.hpp:205-214).
//
// Two strategies:
//  * exact: one thread per output slot accumulates its reduced elements in
//    row-major order -- the same order as the reference's flat scan, so f32/f16
//    results are bit-identical to exec_base.  Used for the reference dtypes.
//  * fast: warp-per-column-tile tree reduction for bf16 activations (the AMP
//    extension; bias gradients of [T, N] GEMM outputs), deterministic but in a
//    different association order (tolerance-checked).
#include "common.cuh"
#include "fold.cuh"

namespace tcb {

struct RedGeom {
  int rank;
  int64_t shape[TCB_MAX_RANK];
  int reduced[TCB_MAX_RANK];
  int64_t count;  // elements per slot
};

static RedGeom red_geom(const Spec& x, const std::string& axes_s) {
  RedGeom g{};
  g.rank = x.rank;
  for (int i = 0; i < x.rank; ++i) g.shape[i] = x.shape[i];
  if (axes_s.empty()) {
    for (int i = 0; i < x.rank; ++i) g.reduced[i] = 1;
  } else {
    size_t pos = 0;
    while (pos < axes_s.size()) {
      size_t c = axes_s.find(',', pos);
      if (c == std::string::npos) c = axes_s.size();
      int a = std::stoi(axes_s.substr(pos, c - pos));
      if (a < 0 || a >= x.rank) fail(TCB_ERR_TYPE, "reduction axis out of range: " + axes_s);
      g.reduced[a] = 1;
      pos = c + 1;
    }
  }
  g.count = 1;
  for (int i = 0; i < x.rank; ++i)
    if (g.reduced[i]) g.count *= x.shape[i];
  return g;
}

// exact: thread per output slot; walk reduced coordinates in row-major order
template <typename T, typename TO>
__global__ void k_reduce_exact(const T* __restrict__ x, TO* __restrict__ o, int64_t nslots, RedGeom g,
                               int mean) {
  TCB_PDL_ENTRY();
  int64_t slot = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (slot >= nslots) return;
  // base offset of this slot (kept dims), strides of all dims
  int64_t stride[TCB_MAX_RANK];
  int64_t s = 1;
  for (int d = g.rank - 1; d >= 0; --d) {
    stride[d] = s;
    s *= g.shape[d];
  }
  int64_t base = 0, rem = slot;
  for (int d = g.rank - 1; d >= 0; --d) {
    if (g.reduced[d]) continue;
    int64_t q = rem / g.shape[d];
    base += (rem - q * g.shape[d]) * stride[d];
    rem = q;
  }
  float acc = 0.0f;
  for (int64_t r = 0; r < g.count; ++r) {
    int64_t off = 0, rr = r;
    for (int d = g.rank - 1; d >= 0; --d) {
      if (!g.reduced[d]) continue;
      int64_t q = rr / g.shape[d];
      off += (rr - q * g.shape[d]) * stride[d];
      rr = q;
    }
    acc = __fadd_rn(acc, to_f(x[base + off]));
  }
  if (mean) acc = __fmul_rn(acc, 1.0f / float(g.count));
  o[slot] = from_f<TO>(acc);
}

// fast: x viewed as [outer, red, inner]; block = 32 inner columns x 8 warps
template <typename T, typename TO>
__global__ void k_reduce_cols(const T* __restrict__ x, TO* __restrict__ o, int64_t outer, int64_t red,
                              int64_t inner, float scale) {
  TCB_PDL_ENTRY();
  __shared__ float part[8][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t tiles_per_outer = (inner + 31) / 32;
  const int64_t ob = blockIdx.x / tiles_per_outer;
  const int64_t col = (blockIdx.x % tiles_per_outer) * 32 + lane;
  float acc = 0.0f;
  if (col < inner) {
    const T* px = x + ob * red * inner + col;
    for (int64_t r = warp; r < red; r += 8) acc += to_f(px[r * inner]);
  }
  part[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && col < inner) {
    float t = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += part[w][lane];
    o[ob * inner + col] = from_f<TO>(t * scale);
  }
}

// fast: inner == 1, one warp per row
template <typename T, typename TO>
__global__ void k_reduce_rows(const T* __restrict__ x, TO* __restrict__ o, int64_t rows, int64_t red,
                              float scale) {
  TCB_PDL_ENTRY();
  const int64_t row = blockIdx.x * int64_t(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float acc = 0.0f;
  for (int64_t j = lane; j < red; j += 32) acc += to_f(x[row * red + j]);
#pragma unroll
  for (int m = 16; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if (lane == 0) o[row] = from_f<TO>(acc * scale);
}

static void build_reduce(Plan& p, int mean) {
  check_arity(p, 1, 1, 1, 1);
  const Spec& X = p.in[0];
  require(is_float(X.dtype), p.op + ": float dtypes only");
  RedGeom g = red_geom(X, p.attrs.s("axes", ""));
  const int64_t nslots = p.out[0].numel();
  require(nslots * g.count == X.numel(), p.op + ": output shape mismatch");
  // contiguous reduced block?
  int first = -1, last = -1;
  for (int i = 0; i < X.rank; ++i)
    if (g.reduced[i]) {
      if (first < 0) first = i;
      last = i;
    }
  bool contiguous = first >= 0;
  for (int i = first; contiguous && i <= last; ++i) contiguous = g.reduced[i];
  const bool exact = X.dtype != TCB_BF16 || p.attrs.i("exact", 0) != 0 || !contiguous;
  const int dto = p.out[0].dtype;
  dispatch_float(X.dtype, [&](auto* tp) {
    using T = std::remove_pointer_t<decltype(tp)>;
    dispatch_float(dto, [&](auto* op_) {
      using TO = std::remove_pointer_t<decltype(op_)>;
      if (exact) {
        p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
          launch_k(k_reduce_exact<T, TO>, unsigned((nslots + 127) / 128), 128, 0, s, 
              (const T*)in[0].ptr, (TO*)out[0].ptr, nslots, g, mean);
        };
        return;
      }
      int64_t outer = 1, red = 1, inner = 1;
      for (int i = 0; i < first; ++i) outer *= X.shape[i];
      for (int i = first; i <= last; ++i) red *= X.shape[i];
      for (int i = last + 1; i < X.rank; ++i) inner *= X.shape[i];
      const float scale = mean ? 1.0f / float(red) : 1.0f;
      if (inner == 1) {
        p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
          launch_k(k_reduce_rows<T, TO>, unsigned((outer + 7) / 8), 256, 0, s, (const T*)in[0].ptr,
                                                                          (TO*)out[0].ptr, outer, red, scale);
        };
      } else {
        const int64_t blocks = outer * ((inner + 31) / 32);
        p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
          launch_k(k_reduce_cols<T, TO>, unsigned(blocks), 256, 0, s, (const T*)in[0].ptr, (TO*)out[0].ptr,
                                                                  outer, red, inner, scale);
        };
      }
    });
  });
}
static void b_sum(Plan& p) { build_reduce(p, 0); }
static void b_mean(Plan& p) { build_reduce(p, 1); }
TCB_REGISTER("sum", b_sum);
TCB_REGISTER("mean", b_mean);

// Split-row column sums of x [R, C] (C % 8 == 0, 16-byte rows): block (cx, cy)
// covers 256 columns x CS_ROWS rows; each lane owns 8 adjacent columns (one
// 16-byte load per row), the 8 warps interleave rows, smem folds the warps and
// the block writes one partial row; k_colsum_final adds the partials in chunk
// order.  Deterministic; fills the machine at any R.
constexpr int CS_ROWS = 64;  // rows per block: 8 per warp, all loads in flight at once

template <typename T>
__global__ void __launch_bounds__(256) k_colsum_partial(const T* __restrict__ x, float* __restrict__ part,
                                                        int64_t R, int64_t C, const int32_t* __restrict__ lab,
                                                        int32_t ign) {
  TCB_PDL_ENTRY();
  __shared__ float red[8][256 + 4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = int64_t(blockIdx.x) * 256 + lane * 8;
  const int64_t r0 = int64_t(blockIdx.y) * CS_ROWS;
  const int64_t r1 = r0 + CS_ROWS < R ? r0 + CS_ROWS : R;
  float acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0f;
  if (c0 < C) {
    constexpr int RPW = CS_ROWS / 8;
    if constexpr (sizeof(T) == 2) {
      uint4 q[RPW];
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        const int64_t r = r0 + warp + 8 * i;
        // rows labelled ignore_index are skipped (exact zeros of a CE gradient)
        q[i] = (r < r1 && !(lab && lab[r] == ign)) ? *reinterpret_cast<const uint4*>(x + r * C + c0)
                                                   : make_uint4(0, 0, 0, 0);
      }
      // packed: two columns per f32x2 add (same per-column order, same bits)
      float2 a2[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) a2[k] = make_float2(0.0f, 0.0f);
#pragma unroll
      for (int i = 0; i < RPW; ++i) {
        const uint32_t w[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          float2 f;
          if constexpr (std::is_same<T, __nv_bfloat16>::value)
            f = make_float2(__uint_as_float(w[k] << 16), __uint_as_float(w[k] & 0xffff0000u));
          else
            f = __half22float2(*reinterpret_cast<const __half2*>(&w[k]));
          a2[k] = add2(a2[k], f);
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) acc[2 * k] = a2[k].x, acc[2 * k + 1] = a2[k].y;
    } else {
      for (int64_t r = r0 + warp; r < r1; r += 8) {
        if (lab && lab[r] == ign) continue;
        float4 a = *reinterpret_cast<const float4*>(x + r * C + c0);
        float4 b = *reinterpret_cast<const float4*>(x + r * C + c0 + 4);
        acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
        acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
      }
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) red[warp][lane * 8 + k] = acc[k];
  __syncthreads();
  const int64_t c = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (c < C) {
    float s = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
    part[int64_t(blockIdx.y) * C + c] = s;
  }
}

// Labelled variant (decoder bias gradient of the MLM head): most rows carry
// ignore_index and are exact zeros, so a block covers a long row range (rpc
// rows) and each warp walks its rows loading only the labelled ones -- few,
// large blocks keep the partial buffer (and the final fold) small.
template <typename T>
__global__ void __launch_bounds__(256) k_colsum_partial_masked(const T* __restrict__ x, float* __restrict__ part,
                                                               int64_t R, int64_t C, int64_t rpc,
                                                               const int32_t* __restrict__ lab, int32_t ign) {
  TCB_PDL_ENTRY();
  __shared__ float red[8][256 + 4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = int64_t(blockIdx.x) * 256 + lane * 8;
  const int64_t r0 = int64_t(blockIdx.y) * rpc;
  const int64_t r1 = r0 + rpc < R ? r0 + rpc : R;
  float acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = 0.0f;
  if (c0 < C) {
    for (int64_t r = r0 + warp; r < r1; r += 8) {
      if (__ldg(lab + r) == ign) continue;  // warp-uniform: one row per warp
      float f[8];
      if constexpr (sizeof(T) == 2) {
        const uint4 q = *reinterpret_cast<const uint4*>(x + r * C + c0);
        const T* h = reinterpret_cast<const T*>(&q);
#pragma unroll
        for (int k = 0; k < 8; ++k) f[k] = to_f(h[k]);
      } else {
        const float4 a = *reinterpret_cast<const float4*>(x + r * C + c0);
        const float4 b = *reinterpret_cast<const float4*>(x + r * C + c0 + 4);
        f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc[k] += f[k];
    }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) red[warp][lane * 8 + k] = acc[k];
  __syncthreads();
  const int64_t c = int64_t(blockIdx.x) * 256 + threadIdx.x;
  if (c < C) {
    float s = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
    part[int64_t(blockIdx.y) * C + c] = s;
  }
}

// block = 32 columns x 32 warps; warp w sums partial rows w, w+32, ... (loads
// unrolled 4 deep), then warp 0 adds the 32 warp sums in order: deterministic
__global__ void __launch_bounds__(1024) k_colsum_final(const float* __restrict__ part, float* __restrict__ out,
                                                       int64_t nchunk, int64_t C, float scale) {
  TCB_PDL_ENTRY();
  __shared__ float red[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c = int64_t(blockIdx.x) * 32 + lane;
  float s = 0.0f;
  if (c < C) {
#pragma unroll 4
    for (int64_t k = warp; k < nchunk; k += 32) s += part[k * C + c];
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && c < C) {
    float t = 0.0f;
#pragma unroll 8
    for (int w = 0; w < 32; ++w) t += red[w][lane];
    out[c] = t * scale;
  }
}

// colsum: f32 column sums over all leading dims (bias gradients of [T, N]
// GEMM outputs); exact row order for f32 input, split-row tree otherwise.
// With a labels input, rows labelled ignore_index are not read on the split-row
// path (they are exact zeros of the CE gradient); the other paths add those
// zeros, which leaves every sum unchanged.
static void b_colsum(Plan& p) {
  check_arity(p, 1, 2, 1, 1);
  const bool masked = p.in.size() > 1;
  if (masked) require(p.in[1].dtype == TCB_I32, "colsum: labels must be i32");
  const int32_t ign = int32_t(p.attrs.i("ignore_index", -100));
  const Spec& X = p.in[0];
  require(is_float(X.dtype), "colsum: float input");
  require(p.out[0].dtype == TCB_F32, "colsum: output is f32");
  const int64_t C = X.dim(-1), R = X.numel() / C;
  require(p.out[0].numel() == C, "colsum: output must have the last dim's size");
  RedGeom g{};
  g.rank = 2;
  g.shape[0] = R;
  g.shape[1] = C;
  g.reduced[0] = 1;
  g.count = R;
  const bool exact = X.dtype == TCB_F32 || p.attrs.i("exact", 0) != 0;
  dispatch_float(X.dtype, [&](auto* tp) {
    using T = std::remove_pointer_t<decltype(tp)>;
    if (exact) {
      p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
        launch_k(k_reduce_exact<T, float>, unsigned((C + 127) / 128), 128, 0, s, (const T*)in[0].ptr,
                                                                           (float*)out[0].ptr, C, g, 0);
      };
    } else if (C % 8 == 0) {
      // masked: ~8 blocks per SM in total, each over rpc rows (a multiple of 8)
      const int64_t cblocks = (C + 255) / 256;
      int64_t rpc = CS_ROWS;
      if (masked) {
        const int64_t want = std::max<int64_t>(1, (kNumSMs * 8 + cblocks - 1) / cblocks);
        rpc = std::max<int64_t>(CS_ROWS, (((R + want - 1) / want) + 7) / 8 * 8);
      }
      const int64_t nchunk = (R + rpc - 1) / rpc;
      const size_t ws = p.ws_take(size_t(nchunk) * C * 4);
      p.nkernels = 2;
      p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
        if (reinterpret_cast<uintptr_t>(in[0].ptr) % 16) fail(TCB_ERR_ARG, "colsum: input not 16-byte aligned");
        const dim3 grid{unsigned(cblocks), unsigned(nchunk)};
        float* dws = fold_deferring() ? fold_scratch(out[0].ptr, 0, size_t(nchunk) * C * 4) : nullptr;
        float* wsp = dws ? dws : (float*)ws_at(ws);
        if (masked)
          launch_k(k_colsum_partial_masked<T>, grid, 256, 0, s, (const T*)in[0].ptr, wsp, R, C, rpc,
                   (const int32_t*)in[1].ptr, ign);
        else
          launch_k(k_colsum_partial<T>, grid, 256, 0, s, (const T*)in[0].ptr, wsp, R, C,
                   (const int32_t*)nullptr, ign);
        if (dws) {
          fold_defer(FoldJob{dws, C, int(nchunk), int(C), (float*)out[0].ptr, 1.0f});
          fold_op_deferred();
          return;
        }
        if (!skip_folds()) launch_k(k_colsum_final, unsigned((C + 31) / 32), 1024, 0, s, (const float*)ws_at(ws), (float*)out[0].ptr, nchunk, C,
                                                                  1.0f);
      };
    } else {
      p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
        launch_k(k_reduce_cols<T, float>, unsigned((C + 31) / 32), 256, 0, s, (const T*)in[0].ptr,
                                                                        (float*)out[0].ptr, 1, R, C, 1.0f);
      };
    }
  });
}
TCB_REGISTER("colsum", b_colsum);

// mse: sequential f32 sum of squared differences, then acc / numel (a divide)
template <typename T>
__global__ void k_mse_exact(const T* __restrict__ a, const T* __restrict__ b, float* o, int64_t n) {
  TCB_PDL_ENTRY();
  float acc = 0.0f;
  for (int64_t i = 0; i < n; ++i) {
    float d = __fsub_rn(to_f(a[i]), to_f(b[i]));
    acc = __fadd_rn(acc, __fmul_rn(d, d));
  }
  o[0] = __fdiv_rn(acc, float(n));
}
template <typename T>
__global__ void k_mse_block(const T* __restrict__ a, const T* __restrict__ b, float* o, int64_t n) {
  TCB_PDL_ENTRY();
  __shared__ float part[32];
  float acc = 0.0f;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    float d = to_f(a[i]) - to_f(b[i]);
    acc += d * d;
  }
  for (int m = 16; m; m >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, m);
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.0f;
    for (int w = 0; w < int(blockDim.x / 32); ++w) t += part[w];
    o[0] = t / float(n);
  }
}
static void b_mse(Plan& p) {
  check_arity(p, 2, 2, 1, 1);
  require(same_shape(p.in[0], p.in[1]), "mse: prediction/label shape mismatch");
  require(p.in[0].dtype == p.in[1].dtype, "mse: dtype mismatch without explicit cast");
  require(p.out[0].dtype == TCB_F32 && p.out[0].numel() == 1, "mse: output is f32[1]");
  const int64_t n = p.in[0].numel();
  dispatch_float(p.in[0].dtype, [&](auto* tp) {
    using T = std::remove_pointer_t<decltype(tp)>;
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      if (n <= (1 << 16))
        launch_k(k_mse_exact<T>, 1, 1, 0, s, (const T*)in[0].ptr, (const T*)in[1].ptr, (float*)out[0].ptr, n);
      else
        launch_k(k_mse_block<T>, 1, 1024, 0, s, (const T*)in[0].ptr, (const T*)in[1].ptr, (float*)out[0].ptr, n);
    };
  });
}
TCB_REGISTER("mse", b_mse);

}  // namespace tcb
