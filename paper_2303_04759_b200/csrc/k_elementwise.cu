// k_elementwise.cu -- b200 kernels for the reference's elementwise / layout ops
// (backends.hpp:67-93,168-202) and the gelu / dropout / convert / view / concat
// extensions.
//
// Semantics are exec_base's: f32 compute, one round-to-nearest-even store into
// the output dtype.  This file is compiled with -fmad=false and uses the *_rn
// intrinsics, so results are bit-identical to the CPU oracle (tanh/gelu aside:
// device tanhf/erff differ from glibc by ulps).
#include "common.cuh"

namespace tcb {

enum BinOp { B_ADD, B_SUB, B_MUL, B_DIV, B_TANH_DX, B_GELU_DX };

__device__ __forceinline__ float ld_any(const void* p, int dt, int64_t i) {
  if (dt == TCB_F32) return static_cast<const float*>(p)[i];
  if (dt == TCB_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  return __half2float(static_cast<const __half*>(p)[i]);
}
__device__ __forceinline__ void st_any(void* p, int dt, int64_t i, float v) {
  if (dt == TCB_F32) static_cast<float*>(p)[i] = v;
  else if (dt == TCB_BF16) static_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(v);
  else static_cast<__half*>(p)[i] = __float2half_rn(v);
}

template <int OP>
__device__ __forceinline__ float binop(float x, float y) {
  if (OP == B_ADD) return __fadd_rn(x, y);
  if (OP == B_SUB) return __fsub_rn(x, y);
  if (OP == B_MUL) return __fmul_rn(x, y);
  if (OP == B_DIV) return __fdiv_rn(x, y);
  if (OP == B_TANH_DX) return __fmul_rn(y, __fsub_rn(1.0f, __fmul_rn(x, x)));  // (y, dy)
  return __fmul_rn(y, gelu_grad_f(x));                                          // (x, dy)
}

// BcastIndex (backends.hpp:30-57) on the device: per-operand strides over the
// output's dims, 0 for broadcast dims.
struct BC {
  int rank;
  int64_t shape[TCB_MAX_RANK];
  int64_t sa[TCB_MAX_RANK];
  int64_t sb[TCB_MAX_RANK];
};

static void bc_strides(const Spec& out, const Spec& in, int64_t* s) {
  for (int i = 0; i < TCB_MAX_RANK; ++i) s[i] = 0;
  int64_t stride = 1;
  for (int i = 0; i < in.rank; ++i) {
    int id = in.rank - 1 - i, od = out.rank - 1 - i;
    s[od] = in.shape[id] == 1 ? 0 : stride;
    stride *= in.shape[id];
  }
}

template <int OP>
__global__ void k_binary_bc(const void* __restrict__ a, int dta, const void* __restrict__ b, int dtb,
                            void* __restrict__ o, int dto, int64_t n, BC bc) {
  TCB_PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t ia = 0, ib = 0, rem = i;
    for (int d = bc.rank - 1; d >= 0; --d) {
      int64_t q = rem / bc.shape[d];
      int64_t r = rem - q * bc.shape[d];
      ia += r * bc.sa[d];
      ib += r * bc.sb[d];
      rem = q;
    }
    st_any(o, dto, i, binop<OP>(ld_any(a, dta, ia), ld_any(b, dtb, ib)));
  }
}

// same-shape, same-dtype fast path: 8 elements per thread per iteration
template <int OP, typename T>
__global__ void k_binary_same(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ o,
                              int64_t n) {
  TCB_PDL_ENTRY();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride)
    o[i] = from_f<T>(binop<OP>(to_f(a[i]), to_f(b[i])));
}

// scalar-b or row-vector-b (trailing-dim broadcast of a [C] vector)
template <int OP, typename T>
__global__ void k_binary_row(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ o,
                             int64_t n, int64_t cols, int b_first) {
  TCB_PDL_ENTRY();
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    float x = to_f(a[i]), y = to_f(b[i % cols]);
    o[i] = from_f<T>(b_first ? binop<OP>(y, x) : binop<OP>(x, y));
  }
}

template <int OP>
static void build_binary(Plan& p) {
  check_arity(p, 2, 2, 1, 1);
  const Spec &A = p.in[0], &B = p.in[1], &O = p.out[0];
  require(is_float(A.dtype) && is_float(B.dtype) && is_float(O.dtype), p.op + ": float dtypes only");
  const int64_t n = O.numel();
  // trailing-dim broadcast check (rel::elemwise_binary / broadcast_shape, opreg.hpp:75-87)
  for (const Spec* s : {&A, &B}) {
    require(s->rank <= O.rank, p.op + ": input rank exceeds output rank");
    for (int i = 0; i < s->rank; ++i) {
      int64_t d = s->shape[s->rank - 1 - i], od = O.shape[O.rank - 1 - i];
      require(d == od || d == 1, p.op + ": shapes are not broadcast-compatible");
    }
  }
  const bool same = same_shape(A, O) && same_shape(B, O) && A.dtype == O.dtype && B.dtype == O.dtype;
  if (same) {
    dispatch_float(O.dtype, [&](auto* tp) {
      using T = std::remove_pointer_t<decltype(tp)>;
      p.run = [n](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
        launch_k(k_binary_same<OP, T>, grid_for(n, 256), 256, 0, s, 
            (const T*)in[0].ptr, (const T*)in[1].ptr, (T*)out[0].ptr, n);
      };
    });
    return;
  }
  // b (or a) is a trailing row vector / scalar of the same dtype
  auto is_row = [&](const Spec& v) {
    int64_t c = v.numel();
    if (c == 1) return true;
    if (v.rank > O.rank) return false;
    int64_t tail = 1;
    for (int i = 0; i < v.rank; ++i) tail *= O.shape[O.rank - 1 - i];
    if (tail != c) return false;
    for (int i = 0; i < v.rank; ++i)
      if (v.shape[v.rank - 1 - i] != O.shape[O.rank - 1 - i]) return false;
    return true;
  };
  if (A.dtype == O.dtype && B.dtype == O.dtype && same_shape(A, O) && is_row(B)) {
    const int64_t cols = B.numel();
    dispatch_float(O.dtype, [&](auto* tp) {
      using T = std::remove_pointer_t<decltype(tp)>;
      p.run = [n, cols](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
        launch_k(k_binary_row<OP, T>, grid_for(n, 256), 256, 0, s, 
            (const T*)in[0].ptr, (const T*)in[1].ptr, (T*)out[0].ptr, n, cols, 0);
      };
    });
    return;
  }
  if (A.dtype == O.dtype && B.dtype == O.dtype && same_shape(B, O) && is_row(A)) {
    const int64_t cols = A.numel();
    dispatch_float(O.dtype, [&](auto* tp) {
      using T = std::remove_pointer_t<decltype(tp)>;
      p.run = [n, cols](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
        launch_k(k_binary_row<OP, T>, grid_for(n, 256), 256, 0, s, 
            (const T*)in[1].ptr, (const T*)in[0].ptr, (T*)out[0].ptr, n, cols, 1);
      };
    });
    return;
  }
  BC bc{};
  bc.rank = O.rank;
  for (int i = 0; i < O.rank; ++i) bc.shape[i] = O.shape[i];
  bc_strides(O, A, bc.sa);
  bc_strides(O, B, bc.sb);
  const int dta = A.dtype, dtb = B.dtype, dto = O.dtype;
  p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    launch_k(k_binary_bc<OP>, grid_for(n, 256), 256, 0, s, in[0].ptr, dta, in[1].ptr, dtb, out[0].ptr, dto,
                                                       n, bc);
  };
}

static void b_add(Plan& p) { build_binary<B_ADD>(p); }
static void b_sub(Plan& p) { build_binary<B_SUB>(p); }
static void b_mul(Plan& p) { build_binary<B_MUL>(p); }
static void b_div(Plan& p) { build_binary<B_DIV>(p); }
static void b_tanh_dx(Plan& p) { build_binary<B_TANH_DX>(p); }
static void b_gelu_dx(Plan& p) { build_binary<B_GELU_DX>(p); }
TCB_REGISTER("add", b_add);
TCB_REGISTER("sub", b_sub);
TCB_REGISTER("mul", b_mul);
TCB_REGISTER("div", b_div);
TCB_REGISTER("tanh_dx", b_tanh_dx);
TCB_REGISTER("gelu_dx", b_gelu_dx);

// ------------------------------------------------------------------- unary
enum UnOp { U_NEG, U_TANH, U_RELU, U_GTZ, U_GELU, U_COPY };

template <int OP>
__device__ __forceinline__ float unop(float x) {
  if (OP == U_NEG) return -x;
  if (OP == U_TANH) return tanhf(x);
  if (OP == U_RELU) return x > 0.0f ? x : 0.0f;
  if (OP == U_GTZ) return x > 0.0f ? 1.0f : 0.0f;
  if (OP == U_GELU) return gelu_f(x);
  return x;
}

template <int OP>
__global__ void k_unary(const void* __restrict__ a, int dta, void* __restrict__ o, int dto, int64_t n) {
  TCB_PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    st_any(o, dto, i, unop<OP>(ld_any(a, dta, i)));
}

template <int OP>
static void build_unary(Plan& p) {
  check_arity(p, 1, 1, 1, 1);
  require(is_float(p.in[0].dtype) && is_float(p.out[0].dtype), p.op + ": float dtypes only");
  require(p.in[0].numel() == p.out[0].numel(), p.op + ": shape mismatch");
  const int64_t n = p.out[0].numel();
  const int dta = p.in[0].dtype, dto = p.out[0].dtype;
  p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    launch_k(k_unary<OP>, grid_for(n, 256), 256, 0, s, in[0].ptr, dta, out[0].ptr, dto, n);
  };
}
static void b_neg(Plan& p) { build_unary<U_NEG>(p); }
static void b_tanh(Plan& p) { build_unary<U_TANH>(p); }
static void b_relu(Plan& p) { build_unary<U_RELU>(p); }
static void b_gtz(Plan& p) { build_unary<U_GTZ>(p); }
static void b_gelu(Plan& p) { build_unary<U_GELU>(p); }
static void b_cast(Plan& p) { build_unary<U_COPY>(p); }  // cast / convert: round into out dtype
TCB_REGISTER("neg", b_neg);
TCB_REGISTER("tanh", b_tanh);
TCB_REGISTER("relu", b_relu);
TCB_REGISTER("gtz", b_gtz);
TCB_REGISTER("gelu", b_gelu);
TCB_REGISTER("cast", b_cast);
TCB_REGISTER("convert", b_cast);

// ------------------------------------------------------------------- bcast
__global__ void k_bcast(const void* __restrict__ a, int dta, void* __restrict__ o, int dto, int64_t n,
                        BC bc) {
  TCB_PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    int64_t ia = 0, rem = i;
    for (int d = bc.rank - 1; d >= 0; --d) {
      int64_t q = rem / bc.shape[d];
      ia += (rem - q * bc.shape[d]) * bc.sa[d];
      rem = q;
    }
    st_any(o, dto, i, ld_any(a, dta, ia));
  }
}
static void b_bcast(Plan& p) {
  check_arity(p, 1, 1, 1, 1);
  require(is_float(p.in[0].dtype), "bcast: float dtypes only");
  BC bc{};
  bc.rank = p.out[0].rank;
  for (int i = 0; i < bc.rank; ++i) bc.shape[i] = p.out[0].shape[i];
  bc_strides(p.out[0], p.in[0], bc.sa);
  const int64_t n = p.out[0].numel();
  const int dta = p.in[0].dtype, dto = p.out[0].dtype;
  p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    launch_k(k_bcast, grid_for(n, 256), 256, 0, s, in[0].ptr, dta, out[0].ptr, dto, n, bc);
  };
}
TCB_REGISTER("bcast", b_bcast);

// --------------------------------------------------------------- transpose
// 32x32 smem tile, +1 padding (no bank conflicts); raw element copy.
template <typename W>
__global__ void k_transpose(const W* __restrict__ in, W* __restrict__ out, int64_t R, int64_t C) {
  TCB_PDL_ENTRY();
  __shared__ W tile[32][33];
  int64_t c0 = int64_t(blockIdx.x) * 32, r0 = int64_t(blockIdx.y) * 32;
  for (int k = threadIdx.y; k < 32; k += 8) {
    int64_t r = r0 + k, c = c0 + threadIdx.x;
    if (r < R && c < C) tile[k][threadIdx.x] = in[r * C + c];
  }
  __syncthreads();
  for (int k = threadIdx.y; k < 32; k += 8) {
    int64_t c = c0 + k, r = r0 + threadIdx.x;
    if (r < R && c < C) out[c * R + r] = tile[threadIdx.x][k];
  }
}
static void b_transpose(Plan& p) {
  check_arity(p, 1, 1, 1, 1);
  require(p.in[0].rank == 2, "transpose: rank-2 input required");
  const int64_t R = p.in[0].shape[0], C = p.in[0].shape[1];
  const int w = dtype_bytes(p.in[0].dtype);
  require(p.out[0].dtype == p.in[0].dtype, "transpose: dtype mismatch");
  dim3 grid(unsigned((C + 31) / 32), unsigned((R + 31) / 32)), block(32, 8);
  p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    if (w == 4)
      launch_k(k_transpose<uint32_t>, grid, block, 0, s, (const uint32_t*)in[0].ptr, (uint32_t*)out[0].ptr, R, C);
    else if (w == 2)
      launch_k(k_transpose<uint16_t>, grid, block, 0, s, (const uint16_t*)in[0].ptr, (uint16_t*)out[0].ptr, R, C);
    else
      launch_k(k_transpose<uint8_t>, grid, block, 0, s, (const uint8_t*)in[0].ptr, (uint8_t*)out[0].ptr, R, C);
  };
}
TCB_REGISTER("transpose", b_transpose);

// ---------------------------------------------------------- reshape / view
// Copies; the device VM elides both as arena aliases (zero-copy) and only
// launches these for standalone use.
static void b_reshape(Plan& p) {
  check_arity(p, 1, 1, 1, 1);
  require(p.in[0].numel() == p.out[0].numel(), "reshape: element count mismatch");
  const size_t nb = size_t(p.out[0].numel()) * dtype_bytes(p.out[0].dtype);
  p.nkernels = 0;
  p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    TCB_CUDA(cudaMemcpyAsync(out[0].ptr, in[0].ptr, nb, cudaMemcpyDeviceToDevice, s));
  };
}
TCB_REGISTER("reshape", b_reshape);

static void b_view(Plan& p) {
  check_arity(p, 1, 1, 1, 1);
  const int64_t off = p.attrs.i("offset", 0);
  require(off >= 0 && off + p.out[0].numel() <= p.in[0].numel(), "view: slice out of range");
  require(p.in[0].dtype == p.out[0].dtype, "view: dtype mismatch");
  const int w = dtype_bytes(p.out[0].dtype);
  const size_t nb = size_t(p.out[0].numel()) * w;
  p.nkernels = 0;
  p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    TCB_CUDA(cudaMemcpyAsync(out[0].ptr, (const char*)in[0].ptr + off * w, nb,
                             cudaMemcpyDeviceToDevice, s));
  };
}
TCB_REGISTER("view", b_view);

static void b_concat(Plan& p) {
  require(p.in.size() >= 1 && p.out.size() == 1, "concat: arity");
  int64_t tot = 0;
  for (auto& s : p.in) {
    require(s.dtype == p.out[0].dtype, "concat: dtype mismatch");
    tot += s.numel();
  }
  require(tot == p.out[0].numel(), "concat: element count mismatch");
  std::vector<size_t> nb;
  for (auto& s : p.in) nb.push_back(size_t(s.numel()) * dtype_bytes(s.dtype));
  p.nkernels = 0;
  p.run = [nb](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
    char* dst = (char*)out[0].ptr;
    for (size_t i = 0; i < nb.size(); ++i) {
      if (in[i].ptr != dst) TCB_CUDA(cudaMemcpyAsync(dst, in[i].ptr, nb[i], cudaMemcpyDeviceToDevice, s));
      dst += nb[i];
    }
  };
}
TCB_REGISTER("concat", b_concat);

// ----------------------------------------------------------------- dropout
// one Philox call yields the keep bits for 8 consecutive elements
template <typename T>
__global__ void k_dropout(const T* __restrict__ x, T* __restrict__ y, int64_t n, DropCfg d) {
  TCB_PDL_ENTRY();
  drop_resolve(d);
  const int64_t nq = (n + 7) / 8;
  for (int64_t q = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; q < nq;
       q += int64_t(gridDim.x) * blockDim.x) {
    uint32_t bits = d.p > 0.0f ? dropout_bits8q(d, uint64_t(q)) : 0xFFu;
#pragma unroll
    for (int w = 0; w < 8; ++w) {
      int64_t i = q * 8 + w;
      if (i < n) y[i] = from_f<T>(((bits >> w) & 1u) ? __fmul_rn(to_f(x[i]), d.scale) : 0.0f);
    }
  }
}
static void b_dropout(Plan& p) {
  check_arity(p, 1, 1, 1, 1);
  require(p.in[0].dtype == p.out[0].dtype, "dropout: dtype mismatch");
  const int64_t n = p.out[0].numel();
  const DropCfg d = drop_cfg(p.attrs);
  dispatch_float(p.out[0].dtype, [&](auto* tp) {
    using T = std::remove_pointer_t<decltype(tp)>;
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      launch_k(k_dropout<T>, grid_for((n + 7) / 8, 256), 256, 0, s, (const T*)in[0].ptr, (T*)out[0].ptr, n, with_step(d));
    };
  });
}
TCB_REGISTER("dropout", b_dropout);

// --------------------------------------------------------- add_scalar / fill
template <typename T>
__global__ void k_add_scalar(const T* __restrict__ x, T* __restrict__ y, int64_t n, float v) {
  TCB_PDL_ENTRY();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = from_f<T>(__fadd_rn(to_f(x[i]), v));
}
static void b_add_scalar(Plan& p) {
  check_arity(p, 1, 1, 1, 1);
  require(p.in[0].dtype == p.out[0].dtype && same_shape(p.in[0], p.out[0]), "add_scalar: shape/dtype");
  const int64_t n = p.out[0].numel();
  const float v = float(p.attrs.f("value", 0.0));
  dispatch_float(p.out[0].dtype, [&](auto* tp) {
    using T = std::remove_pointer_t<decltype(tp)>;
    p.run = [=](const tcb_tensor* in, tcb_tensor* out, cudaStream_t s) {
      launch_k(k_add_scalar<T>, grid_for(n, 256), 256, 0, s, (const T*)in[0].ptr, (T*)out[0].ptr, n, v);
    };
  });
}
TCB_REGISTER("add_scalar", b_add_scalar);

template <typename T>
__global__ void k_fill(T* __restrict__ y, int64_t n, float v) {
  TCB_PDL_ENTRY();
  const T t = from_f<T>(v);
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = t;
}
static void b_fill(Plan& p) {
  check_arity(p, 0, 0, 1, 1);
  const int64_t n = p.out[0].numel();
  const float v = float(p.attrs.f("value", 0.0));
  dispatch_float(p.out[0].dtype, [&](auto* tp) {
    using T = std::remove_pointer_t<decltype(tp)>;
    p.run = [=](const tcb_tensor*, tcb_tensor* out, cudaStream_t s) {
      launch_k(k_fill<T>, grid_for(n, 256), 256, 0, s, (T*)out[0].ptr, n, v);
    };
  });
}
TCB_REGISTER("fill", b_fill);

}  // namespace tcb
