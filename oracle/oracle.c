/* oracle.c -- CPU restatement of the reference `ref` kernels plus the
 * transformer extension ops (TEST INFRASTRUCTURE, see oracle.h).
 *
 * Reference file:line citations are into /root/reference/proj/include/trainc/.
 * Must be compiled with -ffp-contract=off -O2 (no -ffast-math, no -march).
 */
#include "oracle.h"

#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

static int fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  return 1;
}

const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- rounding */

/* fp16.hpp:14-45 float_to_half_bits, restated. */
uint16_t orc_float_to_half_bits(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t exp = (x >> 23) & 0xffu;
  uint32_t man = x & 0x7fffffu;
  if (exp == 0xffu) {
    if (man == 0) return (uint16_t)(sign | 0x7c00u);
    uint32_t payload = man >> 13;
    if (payload == 0) payload = 1;
    return (uint16_t)(sign | 0x7c00u | payload);
  }
  int e = (int)exp - 127 + 15;
  if (e >= 31) return (uint16_t)(sign | 0x7c00u);
  if (e <= 0) {
    if (e < -11) return (uint16_t)sign;
    uint32_t m = man | 0x800000u;
    int shift = 14 - e;
    uint32_t half = m >> shift;
    uint32_t rem = m & ((1u << shift) - 1u);
    uint32_t threshold = 1u << (shift - 1);
    if (rem > threshold || (rem == threshold && (half & 1u))) half++;
    return (uint16_t)(sign | half);
  }
  uint32_t half = sign | ((uint32_t)e << 10) | (man >> 13);
  uint32_t rem = man & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (half & 1u))) half++;
  return (uint16_t)half;
}

/* fp16.hpp:47-70 half_bits_to_float, restated. */
float orc_half_bits_to_float(uint16_t h) {
  uint32_t sign = (uint32_t)(h & 0x8000u) << 16;
  uint32_t exp = (h >> 10) & 0x1fu;
  uint32_t man = h & 0x3ffu;
  uint32_t out;
  if (exp == 0x1fu) {
    out = sign | 0x7f800000u | (man << 13);
  } else if (exp == 0) {
    if (man == 0) {
      out = sign;
    } else {
      int shift = 0;
      while (!(man & 0x400u)) {
        man <<= 1;
        ++shift;
      }
      man &= 0x3ffu;
      out = sign | ((uint32_t)(113 - shift) << 23) | (man << 13);
    }
  } else {
    out = sign | ((exp - 15 + 127) << 23) | (man << 13);
  }
  float f;
  memcpy(&f, &out, 4);
  return f;
}

/* fp16.hpp:74-76 */
float orc_quantize_f16(float f) { return orc_half_bits_to_float(orc_float_to_half_bits(f)); }

/* bf16 extension: IEEE round-to-nearest-even on the top 16 bits, the same
 * contract as __float2bfloat16_rn on the device; NaN stays a quiet NaN. */
uint16_t orc_float_to_bf16_bits(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  if ((x & 0x7fffffffu) > 0x7f800000u) return (uint16_t)((x >> 16) | 0x40u);
  uint32_t lsb = (x >> 16) & 1u;
  x += 0x7fffu + lsb;
  return (uint16_t)(x >> 16);
}

float orc_bf16_bits_to_float(uint16_t h) {
  uint32_t x = (uint32_t)h << 16;
  float f;
  memcpy(&f, &x, 4);
  return f;
}

float orc_quantize_bf16(float f) { return orc_bf16_bits_to_float(orc_float_to_bf16_bits(f)); }

/* round_if_f16 (backends.hpp:59-61) generalised to the half types. */
static inline float rnd(int dtype, float v) {
  if (dtype == ORC_F16) return orc_quantize_f16(v);
  if (dtype == ORC_BF16) return orc_quantize_bf16(v);
  return v;
}

static void round_all(const orc_tensor* t, int64_t n) {
  if (t->dtype != ORC_F16 && t->dtype != ORC_BF16) return;
  float* p = (float*)t->ptr;
  for (int64_t i = 0; i < n; ++i) p[i] = rnd(t->dtype, p[i]);
}

/* ------------------------------------------------------------------ philox */
/* Philox4x32-10 (Salmon et al., SC'11), the counter-based generator used by
 * every dropout site on both CPU and GPU.  One call
 * covers 8 elements: element i of a site draws 16-bit lane (i & 7) of
 * philox(counter = {i >> 3, salt_lo, salt_hi, 0}, key = {seed_lo, seed_hi})
 * (low half of word (i&7)>>1 for even i, high half for odd); keep iff
 * h * 2^-16 >= p. */
static void philox4x32_10(uint32_t c[4], uint32_t k0, uint32_t k1) {
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
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

/* Counter word 3 is the training step's dropout step (the step graph's
 * rng_step state, incremented once per step; attr "rng_step" of the op being
 * executed), so masks differ from step to step; 0 outside a step. */
static __thread uint32_t g_rng_step;

int orc_dropout_keep_step(uint64_t seed, uint64_t salt, uint64_t index, float p, uint32_t step) {
  if (p <= 0.0f) return 1;
  uint32_t c[4] = {(uint32_t)(index >> 3), (uint32_t)salt, (uint32_t)(salt >> 32), step};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint32_t w = c[(index & 7) >> 1];
  uint32_t h = (index & 1) ? (w >> 16) : (w & 0xFFFFu);
  float u = (float)h * (1.0f / 65536.0f);
  return u >= p;
}

int orc_dropout_keep(uint64_t seed, uint64_t salt, uint64_t index, float p) {
  if (p <= 0.0f) return 1;
  uint32_t c[4] = {(uint32_t)(index >> 3), (uint32_t)salt, (uint32_t)(salt >> 32), g_rng_step};
  philox4x32_10(c, (uint32_t)seed, (uint32_t)(seed >> 32));
  uint32_t w = c[(index & 7) >> 1];
  uint32_t h = (index & 1) ? (w >> 16) : (w & 0xFFFFu);
  float u = (float)h * (1.0f / 65536.0f);
  return u >= p;
}

/* --------------------------------------------------------------------- rng */
/* std::mt19937 (MT19937, 32-bit) restated so the synthetic data matches
 * trainc::Rng bit for bit (tensor.hpp:145-176). */
struct orc_rng_ {
  uint32_t mt[624];
  int idx;
};

orc_rng* orc_rng_new(uint64_t seed) {
  orc_rng* r = (orc_rng*)malloc(sizeof(orc_rng));
  uint32_t s = (uint32_t)(seed ^ (seed >> 32)); /* tensor.hpp:147 */
  r->mt[0] = s;
  for (int i = 1; i < 624; ++i)
    r->mt[i] = 1812433253u * (r->mt[i - 1] ^ (r->mt[i - 1] >> 30)) + (uint32_t)i;
  r->idx = 624;
  return r;
}

void orc_rng_free(orc_rng* r) { free(r); }

uint32_t orc_rng_next_u32(orc_rng* r) {
  if (r->idx >= 624) {
    for (int i = 0; i < 624; ++i) {
      uint32_t y = (r->mt[i] & 0x80000000u) | (r->mt[(i + 1) % 624] & 0x7fffffffu);
      uint32_t v = r->mt[(i + 397) % 624] ^ (y >> 1);
      if (y & 1u) v ^= 0x9908b0dfu;
      r->mt[i] = v;
    }
    r->idx = 0;
  }
  uint32_t y = r->mt[r->idx++];
  y ^= y >> 11;
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= y >> 18;
  return y;
}

/* tensor.hpp:150-156: uniform() = float((gen() >> 8) * 2^-24) computed in double */
float orc_rng_uniform(orc_rng* r, float lo, float hi) {
  float u = (float)((double)(orc_rng_next_u32(r) >> 8) * (1.0 / 16777216.0));
  return lo + (hi - lo) * u;
}

/* tensor.hpp:163-165 */
uint32_t orc_rng_below(orc_rng* r, uint32_t n) { return n ? orc_rng_next_u32(r) % n : 0; }

void orc_rng_fill_uniform(orc_rng* r, float* out, int64_t n, float lo, float hi) {
  for (int64_t i = 0; i < n; ++i) out[i] = orc_rng_uniform(r, lo, hi);
}

void orc_rng_fill_below(orc_rng* r, int32_t* out, int64_t n, uint32_t bound) {
  for (int64_t i = 0; i < n; ++i) out[i] = (int32_t)orc_rng_below(r, bound);
}

/* ------------------------------------------------------------------- attrs */
static const orc_attr* find_attr(const orc_attr* a, int na, const char* k) {
  for (int i = 0; i < na; ++i)
    if (strcmp(a[i].key, k) == 0) return &a[i];
  return NULL;
}
/* ir.hpp:34-40 attr_int: doubles truncate */
static int64_t aint(const orc_attr* a, int na, const char* k, int64_t dflt) {
  const orc_attr* x = find_attr(a, na, k);
  if (!x) return dflt;
  if (x->kind == 0) return x->i;
  if (x->kind == 1) return (int64_t)x->d;
  return dflt;
}
/* ir.hpp:42-48 attr_double */
static double adbl(const orc_attr* a, int na, const char* k, double dflt) {
  const orc_attr* x = find_attr(a, na, k);
  if (!x) return dflt;
  if (x->kind == 1) return x->d;
  if (x->kind == 0) return (double)x->i;
  return dflt;
}
static const char* astr(const orc_attr* a, int na, const char* k, const char* dflt) {
  const orc_attr* x = find_attr(a, na, k);
  if (!x || x->kind != 2) return dflt;
  return x->s;
}

static int64_t numel(const orc_tensor* t) {
  int64_t n = 1;
  for (int i = 0; i < t->rank; ++i) n *= t->shape[i];
  return n;
}
static inline float* F(const orc_tensor* t) { return (float*)t->ptr; }

/* --------------------------------------------------------------- broadcast */
/* BcastIndex (backends.hpp:30-57): maps a row-major flat index over `out` to a
 * flat index over `in`, aligning trailing dims and pinning size-1 dims. */
typedef struct {
  int rank;
  int64_t out_shape[8];
  int64_t in_strides[8];
} bcast_t;

static void bcast_init(bcast_t* b, const orc_tensor* out, const orc_tensor* in) {
  b->rank = out->rank;
  int64_t stride = 1;
  for (int i = 0; i < 8; ++i) b->in_strides[i] = 0;
  for (int i = 0; i < out->rank; ++i) b->out_shape[i] = out->shape[i];
  for (int i = 0; i < in->rank; ++i) {
    int in_dim = in->rank - 1 - i;
    int out_dim = out->rank - 1 - i;
    b->in_strides[out_dim] = (in->shape[in_dim] == 1) ? 0 : stride;
    stride *= in->shape[in_dim];
  }
}

static int64_t bcast_map(const bcast_t* b, int64_t out_flat) {
  int64_t in_flat = 0;
  for (int i = b->rank; i-- > 0;) {
    int64_t d = b->out_shape[i];
    in_flat += (out_flat % d) * b->in_strides[i];
    out_flat /= d;
  }
  return in_flat;
}

/* ------------------------------------------------------------ elementwise */
enum { OP_ADD, OP_SUB, OP_MUL, OP_DIV, OP_TANH_DX };

/* elemwise_binary (backends.hpp:67-85).  The reference has four loops (same
 * shape / scalar b / scalar a / BcastIndex); they compute identical values, so
 * the restatement uses the general mapping. */
static int elemwise_binary(int op, const orc_tensor* a, const orc_tensor* b, orc_tensor* out) {
  bcast_t ia, ib;
  bcast_init(&ia, out, a);
  bcast_init(&ib, out, b);
  const float* A = F(a);
  const float* B = F(b);
  float* O = F(out);
  int64_t n = numel(out);
  for (int64_t i = 0; i < n; ++i) {
    float x = A[bcast_map(&ia, i)], y = B[bcast_map(&ib, i)], r;
    switch (op) {
      case OP_ADD: r = x + y; break;
      case OP_SUB: r = x - y; break;
      case OP_MUL: r = x * y; break;
      case OP_DIV: r = x / y; break;
      default: r = y * (1.0f - x * x); break; /* tanh_dx(y, dy), backends.hpp:172-173 */
    }
    O[i] = rnd(out->dtype, r);
  }
  return 0;
}

static inline float gelu_f(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }
static inline float gelu_grad_f(float x) {
  float cdf = 0.5f * (1.0f + erff(x * 0.70710678118654752f));
  float pdf = expf(-0.5f * x * x) * 0.39894228040143268f;
  return cdf + x * pdf;
}

/* elemwise_unary (backends.hpp:87-93) with ops from backends.hpp:174-177 plus
 * the gelu extension. */
static int elemwise_unary(const char* op, const orc_tensor* a, orc_tensor* out) {
  const float* A = F(a);
  float* O = F(out);
  int64_t n = numel(out);
  for (int64_t i = 0; i < n; ++i) {
    float x = A[i], r;
    if (!strcmp(op, "neg")) r = -x;
    else if (!strcmp(op, "tanh")) r = tanhf(x);
    else if (!strcmp(op, "relu")) r = x > 0.0f ? x : 0.0f;
    else if (!strcmp(op, "gtz")) r = x > 0.0f ? 1.0f : 0.0f;
    else if (!strcmp(op, "gelu")) r = gelu_f(x);
    else return fail("no unary op %s", op);
    O[i] = rnd(out->dtype, r);
  }
  return 0;
}

/* ---------------------------------------------------------------- reduce */
/* detail::reduce (backends.hpp:95-141): row-major scan of the input,
 * accumulating each element into its output slot; mean multiplies by
 * 1.0f/count (not a divide). */
static int reduce_op(const orc_tensor* x, orc_tensor* out, const char* axes_s, int mean) {
  int reduced[8] = {0};
  if (!axes_s || !*axes_s) {
    for (int i = 0; i < x->rank; ++i) reduced[i] = 1;
  } else {
    const char* p = axes_s;
    while (*p) {
      int a = atoi(p);
      if (a < 0 || a >= x->rank) return fail("reduction axis out of range: %s", axes_s);
      reduced[a] = 1;
      while (*p && *p != ',') ++p;
      if (*p == ',') ++p;
    }
  }
  int64_t out_stride[8] = {0};
  int64_t stride = 1;
  for (int i = x->rank; i-- > 0;) {
    if (!reduced[i]) {
      out_stride[i] = stride;
      stride *= x->shape[i];
    }
  }
  int64_t count = 1;
  for (int i = 0; i < x->rank; ++i)
    if (reduced[i]) count *= x->shape[i];
  float* O = F(out);
  int64_t on = numel(out);
  for (int64_t i = 0; i < on; ++i) O[i] = 0.0f;
  const float* X = F(x);
  int64_t n = numel(x);
  for (int64_t flat = 0; flat < n; ++flat) {
    int64_t o = 0, rem = flat;
    for (int i = x->rank; i-- > 0;) {
      int64_t d = x->shape[i];
      o += (rem % d) * out_stride[i];
      rem /= d;
    }
    O[o] += X[flat];
  }
  if (mean) {
    float inv = 1.0f / (float)count;
    for (int64_t i = 0; i < on; ++i) O[i] *= inv;
  }
  round_all(out, on);
  return 0;
}

/* ------------------------------------------------------------------ gemm */
/* matmul_ref (backends.hpp:143-155): per output, acc = 0; acc += a*b with k
 * ascending (two roundings per step -- no FMA).  ta/tb read the operands
 * transposed (the extension that absorbs `transpose`). */
static void gemm_acc(const float* A, const float* B, float* C, int64_t M, int64_t N, int64_t K,
                     int ta, int tb, float alpha) {
  /* Evaluated in matmul_blocked's loop order (backends.hpp:280-304, tile 32):
   * each C[i][j] still accumulates a*b in ascending k from 0.0f, so the bits
   * equal matmul_ref's i-j-k loop (the opt/ref equivalence the reference relies
   * on) -- only the memory access pattern differs. */
  const float* Ar = A;
  const float* Br = B;
  float* At = NULL;
  float* Bt = NULL;
  if (ta) { /* materialise A as [M, K] */
    At = (float*)malloc(sizeof(float) * (size_t)(M * K));
    for (int64_t k = 0; k < K; ++k)
      for (int64_t i = 0; i < M; ++i) At[i * K + k] = A[k * M + i];
    Ar = At;
  }
  if (tb) { /* materialise B as [K, N] */
    Bt = (float*)malloc(sizeof(float) * (size_t)(K * N));
    for (int64_t j = 0; j < N; ++j)
      for (int64_t k = 0; k < K; ++k) Bt[k * N + j] = B[j * K + k];
    Br = Bt;
  }
  for (int64_t i = 0; i < M * N; ++i) C[i] = 0.0f;
  const int64_t tile = 32;
  for (int64_t i0 = 0; i0 < M; i0 += tile) {
    const int64_t imax = i0 + tile < M ? i0 + tile : M;
    for (int64_t k0 = 0; k0 < K; k0 += tile) {
      const int64_t kmax = k0 + tile < K ? k0 + tile : K;
      for (int64_t j0 = 0; j0 < N; j0 += 256) {
        const int64_t jmax = j0 + 256 < N ? j0 + 256 : N;
        for (int64_t i = i0; i < imax; ++i) {
          float* crow = C + i * N;
          for (int64_t kk = k0; kk < kmax; ++kk) {
            const float aik = Ar[i * K + kk];
            const float* brow = Br + kk * N;
            for (int64_t j = j0; j < jmax; ++j) crow[j] += aik * brow[j];
          }
        }
      }
    }
  }
  if (alpha != 1.0f)
    for (int64_t i = 0; i < M * N; ++i) C[i] *= alpha;
  free(At);
  free(Bt);
}

enum { ACT_NONE = 0, ACT_RELU = 1, ACT_TANH = 2, ACT_GELU = 3, ACT_DERIV = 4 };
static int parse_act(const char* s) {
  if (!s || !*s || !strcmp(s, "none")) return ACT_NONE;
  if (!strcmp(s, "relu")) return ACT_RELU;
  if (!strcmp(s, "tanh")) return ACT_TANH;
  if (!strcmp(s, "gelu")) return ACT_GELU;
  if (!strcmp(s, "deriv")) return ACT_DERIV;
  return -1;
}
static inline float act_f(int act, float v) {
  switch (act) {
    case ACT_RELU: return v > 0.0f ? v : 0.0f;
    case ACT_TANH: return tanhf(v);
    case ACT_GELU: return gelu_f(v);
    default: return v;
  }
}
/* linear: act(x . W + bias) -- matmul_add_act (backends.hpp:311-324) with the
 * gelu extension; one rounding at the end; tw reads W stored [N,K].  u (may be
 * NULL) receives the rounded pre-activation, or with save_grad the rounded
 * derivative act'(pre-activation). */
static void linear_fwd(const orc_tensor* x, const orc_tensor* w, const orc_tensor* bias, orc_tensor* y,
                       orc_tensor* u, int act, int tw, int save_grad);
/* derivative given the saved aux value: pre-activation u for relu/gelu, the
 * output y for tanh (tanh_dx semantics, backends.hpp:172-173). */
static inline float dact_f(int act, float aux) {
  switch (act) {
    case ACT_RELU: return aux > 0.0f ? 1.0f : 0.0f;
    case ACT_TANH: return 1.0f - aux * aux;
    case ACT_GELU: return gelu_grad_f(aux);
    case ACT_DERIV: return aux; /* aux already holds act'(u) (linear save=grad) */
    default: return 1.0f;
  }
}
/* act'(u) from the pre-activation: what linear(save=grad) stores as u */
static inline float deriv_of_preact(int act, float u) {
  switch (act) {
    case ACT_RELU: return u > 0.0f ? 1.0f : 0.0f;
    case ACT_TANH: { float y = tanhf(u); return 1.0f - y * y; }
    case ACT_GELU: return gelu_grad_f(u);
    default: return 1.0f;
  }
}

static void linear_fwd(const orc_tensor* x, const orc_tensor* w, const orc_tensor* bias, orc_tensor* y,
                       orc_tensor* u, int act, int tw, int save_grad) {
  int64_t M = x->shape[0], K = x->shape[1];
  int64_t N = tw ? w->shape[0] : w->shape[1];
  gemm_acc(F(x), F(w), F(y), M, N, K, 0, tw, 1.0f);
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < N; ++j) {
      float v = F(y)[i * N + j] + F(bias)[j];
      if (u) F(u)[i * N + j] = rnd(u->dtype, save_grad ? deriv_of_preact(act, v) : v);
      F(y)[i * N + j] = rnd(y->dtype, act_f(act, v));
    }
}

/* ------------------------------------------------------------- attention */
typedef struct {
  int64_t B, S, A, H, dh;
  float scale, p;
  uint64_t seed, salt;
  int causal, dt;
} attn_t;

static void attn_heads(const orc_tensor* qkv, attn_t* at, const orc_attr* a, int na) {
  int64_t T = qkv->shape[0];
  at->H = qkv->shape[1] / 3;
  at->A = aint(a, na, "heads", 1);
  at->S = aint(a, na, "seq", T);
  at->B = T / at->S;
  at->dh = at->H / at->A;
  at->scale = (float)adbl(a, na, "scale", 1.0 / sqrt((double)at->dh));
  at->p = (float)adbl(a, na, "p", 0.0);
  at->seed = (uint64_t)aint(a, na, "seed", 0);
  at->salt = (uint64_t)aint(a, na, "salt", 0);
  at->causal = (int)aint(a, na, "causal", 0);
  at->dt = qkv->dtype;
}

/* Fused attention forward (extension op).  Rounding points
 * mirror the b200 pipeline: scores f32, P and dropout(P) and ctx rounded to the
 * activation dtype. */
/* mask (may be NULL): the dropout keep bits, word (z*S + i)*4 + (j >> 5), bit j & 31 */
static int attention_fwd(const orc_tensor* qkv, orc_tensor* ctx, orc_tensor* probs, orc_tensor* mask,
                         const orc_attr* a, int na) {
  attn_t at;
  attn_heads(qkv, &at, a, na);
  const int64_t S = at.S, dh = at.dh, H = at.H, H3 = 3 * at.H;
  const float* X = F(qkv);
  float* C = F(ctx);
  float* P = F(probs);
  float* s = (float*)malloc(sizeof(float) * S);
  float* pd = (float*)malloc(sizeof(float) * S * S);
  const float sp = at.p > 0.0f ? 1.0f / (1.0f - at.p) : 1.0f;
  for (int64_t b = 0; b < at.B; ++b)
    for (int64_t h = 0; h < at.A; ++h) {
      const int64_t z = b * at.A + h;
      for (int64_t i = 0; i < S; ++i) {
        float m = -INFINITY;
        for (int64_t j = 0; j < S; ++j) {
          float acc = 0.0f;
          for (int64_t d = 0; d < dh; ++d)
            acc += X[(b * S + i) * H3 + h * dh + d] * X[(b * S + j) * H3 + H + h * dh + d];
          float v = acc * at.scale;
          if (at.causal && j > i) v = -INFINITY;
          s[j] = v;
          if (v > m) m = v;
        }
        float sum = 0.0f;
        for (int64_t j = 0; j < S; ++j) {
          s[j] = expf(s[j] - m);
          sum += s[j];
        }
        for (int64_t j = 0; j < S; ++j) {
          float pv = rnd(at.dt, s[j] / sum);
          P[(z * S + i) * S + j] = pv;
          uint64_t idx = (uint64_t)((z * S + i) * S + j);
          const int keep = orc_dropout_keep(at.seed, at.salt, idx, at.p);
          if (mask) {
            uint32_t* mw = (uint32_t*)mask->ptr + (z * S + i) * 4 + (j >> 5);
            if ((j & 31) == 0) *mw = 0xffffffffu;
            if (!keep) *mw &= ~(1u << (j & 31));
          }
          float dv = keep ? pv * sp : 0.0f;
          pd[i * S + j] = rnd(at.dt, dv);
        }
      }
      for (int64_t i = 0; i < S; ++i)
        for (int64_t d = 0; d < dh; ++d) {
          float acc = 0.0f;
          for (int64_t j = 0; j < S; ++j) acc += pd[i * S + j] * X[(b * S + j) * H3 + 2 * H + h * dh + d];
          C[(b * S + i) * H + h * dh + d] = rnd(at.dt, acc);
        }
    }
  free(s);
  free(pd);
  return 0;
}

static int attention_bwd(const orc_tensor* qkv, const orc_tensor* probs, const orc_tensor* dctx,
                         const orc_tensor* mask, orc_tensor* dqkv, const orc_attr* a, int na) {
  attn_t at;
  attn_heads(qkv, &at, a, na);
  const int64_t S = at.S, dh = at.dh, H = at.H, H3 = 3 * at.H;
  const float* X = F(qkv);
  const float* P = F(probs);
  const float* dC = F(dctx);
  float* dX = F(dqkv);
  float* ds = (float*)malloc(sizeof(float) * S * S);
  float* pd = (float*)malloc(sizeof(float) * S * S);
  float* dp = (float*)malloc(sizeof(float) * S);
  const float sp = at.p > 0.0f ? 1.0f / (1.0f - at.p) : 1.0f;
  for (int64_t b = 0; b < at.B; ++b)
    for (int64_t h = 0; h < at.A; ++h) {
      const int64_t z = b * at.A + h;
      for (int64_t i = 0; i < S; ++i) {
        float rowdot = 0.0f;
        for (int64_t j = 0; j < S; ++j) {
          float acc = 0.0f;
          for (int64_t d = 0; d < dh; ++d)
            acc += dC[(b * S + i) * H + h * dh + d] * X[(b * S + j) * H3 + 2 * H + h * dh + d];
          uint64_t idx = (uint64_t)((z * S + i) * S + j);
          int keep = mask ? (int)((((const uint32_t*)mask->ptr)[(z * S + i) * 4 + (j >> 5)] >> (j & 31)) & 1u)
                          : orc_dropout_keep(at.seed, at.salt, idx, at.p);
          float pv = P[(z * S + i) * S + j];
          dp[j] = keep ? acc * sp : 0.0f;
          pd[i * S + j] = rnd(at.dt, keep ? pv * sp : 0.0f);
          rowdot += pv * dp[j];
        }
        for (int64_t j = 0; j < S; ++j) {
          float pv = P[(z * S + i) * S + j];
          ds[i * S + j] = rnd(at.dt, pv * (dp[j] - rowdot) * at.scale);
        }
      }
      for (int64_t i = 0; i < S; ++i)
        for (int64_t d = 0; d < dh; ++d) {
          float acc = 0.0f;
          for (int64_t j = 0; j < S; ++j) acc += ds[i * S + j] * X[(b * S + j) * H3 + H + h * dh + d];
          dX[(b * S + i) * H3 + h * dh + d] = rnd(at.dt, acc);
        }
      for (int64_t j = 0; j < S; ++j)
        for (int64_t d = 0; d < dh; ++d) {
          float acck = 0.0f, accv = 0.0f;
          for (int64_t i = 0; i < S; ++i) {
            acck += ds[i * S + j] * X[(b * S + i) * H3 + h * dh + d];
            accv += pd[i * S + j] * dC[(b * S + i) * H + h * dh + d];
          }
          dX[(b * S + j) * H3 + H + h * dh + d] = rnd(at.dt, acck);
          dX[(b * S + j) * H3 + 2 * H + h * dh + d] = rnd(at.dt, accv);
        }
    }
  free(ds);
  free(pd);
  free(dp);
  return 0;
}

/* attention lse=1 (the flash kernels): exact f32 softmax P (no intermediate
 * rounding), Pd = P keep / (1-p), ctx = round(Pd V); the second output is the
 * per-row log-sum-exp of the scaled scores, lse = log sum_j exp(scale s_j)
 * (causal: j <= i).  Keep bits of (z, i, j): Philox index (z*S + i)*S + j;
 * mask (may be NULL): ceil(S/32) words per query row, word (z*S+i)*nw + j/32. */
static int attention_fwd_lse(const orc_tensor* qkv, orc_tensor* ctx, orc_tensor* lse_t, orc_tensor* mask,
                             const orc_attr* a, int na) {
  attn_t at;
  attn_heads(qkv, &at, a, na);
  const int64_t S = at.S, dh = at.dh, H = at.H, H3 = 3 * at.H, nw = (S + 31) / 32;
  const float* X = F(qkv);
  float* C = F(ctx);
  float* L = F(lse_t);
  float* s = (float*)malloc(sizeof(float) * S);
  float* pd = (float*)malloc(sizeof(float) * S * S);
  const float sp = at.p > 0.0f ? 1.0f / (1.0f - at.p) : 1.0f;
  for (int64_t b = 0; b < at.B; ++b)
    for (int64_t h = 0; h < at.A; ++h) {
      const int64_t z = b * at.A + h;
      for (int64_t i = 0; i < S; ++i) {
        float m = -INFINITY;
        for (int64_t j = 0; j < S; ++j) {
          float acc = 0.0f;
          for (int64_t d = 0; d < dh; ++d)
            acc += X[(b * S + i) * H3 + h * dh + d] * X[(b * S + j) * H3 + H + h * dh + d];
          float v = acc * at.scale;
          if (at.causal && j > i) v = -INFINITY;
          s[j] = v;
          if (v > m) m = v;
        }
        float sum = 0.0f;
        for (int64_t j = 0; j < S; ++j) {
          s[j] = expf(s[j] - m);
          sum += s[j];
        }
        L[z * S + i] = m + logf(sum);
        for (int64_t j = 0; j < S; ++j) {
          const int keep = orc_dropout_keep(at.seed, at.salt, (uint64_t)((z * S + i) * S + j), at.p);
          if (mask) {
            uint32_t* mw = (uint32_t*)mask->ptr + (z * S + i) * nw + (j >> 5);
            if ((j & 31) == 0) *mw = 0xffffffffu;
            if (!keep) *mw &= ~(1u << (j & 31));
          }
          pd[i * S + j] = keep ? s[j] / sum * sp : 0.0f;
        }
      }
      for (int64_t i = 0; i < S; ++i)
        for (int64_t d = 0; d < dh; ++d) {
          float acc = 0.0f;
          for (int64_t j = 0; j < S; ++j) acc += pd[i * S + j] * X[(b * S + j) * H3 + 2 * H + h * dh + d];
          C[(b * S + i) * H + h * dh + d] = rnd(at.dt, acc);
        }
    }
  free(s);
  free(pd);
  return 0;
}

/* attention_dx lse=1 (qkv, ctx, lse, dctx [, mask]) -> dqkv: P recomputed
 * from the scores and lse, D_i = sum_d dO O (O = the stored ctx), dP = keep
 * (dO . V_j) / (1-p), dS = round(P (dP - D) scale), Pd = round(P keep / (1-p))
 * (the MMA operands are activation-dtype tiles); dQ = dS K, dK = dS^T Q,
 * dV = Pd^T dO, each rounded once. */
static int attention_bwd_lse(const orc_tensor* qkv, const orc_tensor* ctx, const orc_tensor* lse_t,
                             const orc_tensor* dctx, const orc_tensor* mask, orc_tensor* dqkv, const orc_attr* a,
                             int na) {
  attn_t at;
  attn_heads(qkv, &at, a, na);
  const int64_t S = at.S, dh = at.dh, H = at.H, H3 = 3 * at.H, nw = (S + 31) / 32;
  const float* X = F(qkv);
  const float* O = F(ctx);
  const float* L = F(lse_t);
  const float* dC = F(dctx);
  float* dX = F(dqkv);
  float* ds = (float*)malloc(sizeof(float) * S * S);
  float* pd = (float*)malloc(sizeof(float) * S * S);
  const float sp = at.p > 0.0f ? 1.0f / (1.0f - at.p) : 1.0f;
  for (int64_t b = 0; b < at.B; ++b)
    for (int64_t h = 0; h < at.A; ++h) {
      const int64_t z = b * at.A + h;
      for (int64_t i = 0; i < S; ++i) {
        float D = 0.0f;
        for (int64_t d = 0; d < dh; ++d) D += dC[(b * S + i) * H + h * dh + d] * O[(b * S + i) * H + h * dh + d];
        for (int64_t j = 0; j < S; ++j) {
          float acc = 0.0f, dpd = 0.0f;
          for (int64_t d = 0; d < dh; ++d) {
            acc += X[(b * S + i) * H3 + h * dh + d] * X[(b * S + j) * H3 + H + h * dh + d];
            dpd += dC[(b * S + i) * H + h * dh + d] * X[(b * S + j) * H3 + 2 * H + h * dh + d];
          }
          const int valid = !(at.causal && j > i);
          const float p = valid ? expf(acc * at.scale - L[z * S + i]) : 0.0f;
          const uint64_t idx = (uint64_t)((z * S + i) * S + j);
          const int keep = mask ? (int)((((const uint32_t*)mask->ptr)[(z * S + i) * nw + (j >> 5)] >> (j & 31)) & 1u)
                                : orc_dropout_keep(at.seed, at.salt, idx, at.p);
          const float dp = keep ? dpd * sp : 0.0f;
          ds[i * S + j] = rnd(at.dt, p * (dp - D) * at.scale);
          pd[i * S + j] = rnd(at.dt, keep ? p * sp : 0.0f);
        }
      }
      for (int64_t i = 0; i < S; ++i)
        for (int64_t d = 0; d < dh; ++d) {
          float acc = 0.0f;
          for (int64_t j = 0; j < S; ++j) acc += ds[i * S + j] * X[(b * S + j) * H3 + H + h * dh + d];
          dX[(b * S + i) * H3 + h * dh + d] = rnd(at.dt, acc);
        }
      for (int64_t j = 0; j < S; ++j)
        for (int64_t d = 0; d < dh; ++d) {
          float acck = 0.0f, accv = 0.0f;
          for (int64_t i = 0; i < S; ++i) {
            acck += ds[i * S + j] * X[(b * S + i) * H3 + h * dh + d];
            accv += pd[i * S + j] * dC[(b * S + i) * H + h * dh + d];
          }
          dX[(b * S + j) * H3 + H + h * dh + d] = rnd(at.dt, acck);
          dX[(b * S + j) * H3 + 2 * H + h * dh + d] = rnd(at.dt, accv);
        }
    }
  free(ds);
  free(pd);
  return 0;
}

/* ------------------------------------------------------------- layernorm */
/* Row statistics: left-to-right f32 sums; mean = sum * (1/H); two-pass
 * variance; rstd = 1/sqrtf(var + eps). */
static void ln_row(const float* x, int64_t H, float eps, float* mean_o, float* rstd_o) {
  const float inv = 1.0f / (float)H;
  float sum = 0.0f;
  for (int64_t j = 0; j < H; ++j) sum += x[j];
  float mean = sum * inv;
  float sq = 0.0f;
  for (int64_t j = 0; j < H; ++j) {
    float d = x[j] - mean;
    sq += d * d;
  }
  *mean_o = mean;
  *rstd_o = 1.0f / sqrtf(sq * inv + eps);
}

/* mask (may be NULL): add_layer_norm save_mask -- the residual-branch keep
 * bits, byte i holding elements 8i..8i+7 (bit k = element 8i+k) */
static int layer_norm_fwd(const orc_tensor* x, const orc_tensor* r, const orc_tensor* g,
                          const orc_tensor* bta, orc_tensor* y, orc_tensor* s_out,
                          orc_tensor* mean_t, orc_tensor* rstd_t, orc_tensor* mask, const orc_attr* a, int na) {
  const int64_t H = x->shape[x->rank - 1];
  const int64_t T = numel(x) / H;
  const float eps = (float)adbl(a, na, "eps", 1e-12);
  const float p = (float)adbl(a, na, "p", 0.0);
  const uint64_t seed = (uint64_t)aint(a, na, "seed", 0), salt = (uint64_t)aint(a, na, "salt", 0);
  const float sp = p > 0.0f ? 1.0f / (1.0f - p) : 1.0f;
  const int post_drop = !r && p > 0.0f && aint(a, na, "post_dropout", 0);
  float* row = (float*)malloc(sizeof(float) * H);
  const float* X = F(x);
  for (int64_t t = 0; t < T; ++t) {
    for (int64_t j = 0; j < H; ++j) {
      float v = X[t * H + j];
      if (r) {
        uint64_t idx = (uint64_t)(t * H + j);
        const int keep = orc_dropout_keep(seed, salt, idx, p);
        if (mask) {
          uint8_t* mb = (uint8_t*)mask->ptr;
          if ((idx & 7) == 0) mb[idx >> 3] = 0;
          mb[idx >> 3] |= (uint8_t)(keep << (idx & 7));
        }
        v = (keep ? v * sp : 0.0f) + F(r)[t * H + j];
        v = rnd(x->dtype, v);
        F(s_out)[t * H + j] = v;
      }
      row[j] = v;
    }
    float mean, rstd;
    ln_row(row, H, eps, &mean, &rstd);
    F(mean_t)[t] = mean;
    F(rstd_t)[t] = rstd;
    for (int64_t j = 0; j < H; ++j) {
      float o = rnd(y->dtype, (row[j] - mean) * rstd * F(g)[j] + F(bta)[j]);
      if (post_drop) /* layer_norm post_dropout = the dropout op on the rounded output */
        o = rnd(y->dtype, orc_dropout_keep(seed, salt, (uint64_t)(t * H + j), p) ? o * sp : 0.0f);
      F(y)[t * H + j] = o;
    }
  }
  free(row);
  return 0;
}

/* layer_norm_dx(s, gamma, mean, rstd, dy [, dy2]) -> (ds, dgamma, dbeta [, dx]).
 * dy2 is a second incoming gradient summed into dy first (fan-out accumulation
 * of the residual stream fused into the backward). */
static int layer_norm_bwd(const orc_tensor* const* in, int nin, orc_tensor* out, int nout,
                          const orc_attr* a, int na) {
  const orc_tensor *s = in[0], *g = in[1], *mean_t = in[2], *rstd_t = in[3], *dy = in[4];
  const orc_tensor* dy2 = nin > 5 ? in[5] : NULL;
  const int64_t H = s->shape[s->rank - 1];
  const int64_t T = numel(s) / H;
  const float p = (float)adbl(a, na, "p", 0.0);
  const uint64_t seed = (uint64_t)aint(a, na, "seed", 0), salt = (uint64_t)aint(a, na, "salt", 0);
  const float sp = p > 0.0f ? 1.0f / (1.0f - p) : 1.0f;
  const float inv = 1.0f / (float)H;
  /* in_p: the forward layer_norm's post_dropout folded in -- dy is first the
   * dropout op's output round(keep ? dy * scale : 0) */
  const float in_p = (float)adbl(a, na, "in_p", 0.0);
  const uint64_t in_seed = (uint64_t)aint(a, na, "in_seed", 0), in_salt = (uint64_t)aint(a, na, "in_salt", 0);
  const float in_sp = in_p > 0.0f ? 1.0f / (1.0f - in_p) : 1.0f;
#define LN_DY(t, j)                                                                                     \
  (in_p > 0.0f ? rnd(dy->dtype, orc_dropout_keep(in_seed, in_salt, (uint64_t)((t) * H + (j)), in_p)    \
                                     ? F(dy)[(t) * H + (j)] * in_sp : 0.0f)                          \
               : F(dy)[(t) * H + (j)])
  float* dg = F(&out[1]);
  float* db = F(&out[2]);
  /* bias_grad: column sums (row order) of the outgoing gradient as stored --
   * exactly colsum() of that output, fused (host/graph.hpp pattern 4) */
  const int bias_grad = (int)aint(a, na, "bias_grad", 0);
  const int has_dx = nout - bias_grad > 3;
  float* dbias = bias_grad ? F(&out[has_dx ? 4 : 3]) : NULL;
  const orc_tensor* gout = has_dx ? &out[3] : &out[0];
  for (int64_t j = 0; j < H; ++j) dg[j] = db[j] = 0.0f;
  if (dbias)
    for (int64_t j = 0; j < H; ++j) dbias[j] = 0.0f;
  for (int64_t t = 0; t < T; ++t) {
    const float mean = F(mean_t)[t], rstd = F(rstd_t)[t];
    float c1 = 0.0f, c2 = 0.0f;
    for (int64_t j = 0; j < H; ++j) {
      float xh = (F(s)[t * H + j] - mean) * rstd;
      float dyv = LN_DY(t, j);
      if (dy2) dyv += F(dy2)[t * H + j];
      float gg = dyv * F(g)[j];
      c1 += gg * xh;
      c2 += gg;
    }
    c1 *= inv;
    c2 *= inv;
    for (int64_t j = 0; j < H; ++j) {
      float xh = (F(s)[t * H + j] - mean) * rstd;
      float dyv = LN_DY(t, j);
      if (dy2) dyv += F(dy2)[t * H + j];
      float gg = dyv * F(g)[j];
      float dsv = rstd * (gg - c2 - xh * c1);
      F(&out[0])[t * H + j] = rnd(out[0].dtype, dsv);
      if (has_dx) {
        uint64_t idx = (uint64_t)(t * H + j);
        F(&out[3])[t * H + j] =
            rnd(out[3].dtype, (in[6] ? (((const uint8_t*)in[6]->ptr)[idx >> 3] >> (idx & 7)) & 1
                                      : orc_dropout_keep(seed, salt, idx, p))
                                  ? dsv * sp : 0.0f);
      }
      dg[j] += dyv * xh;
      db[j] += dyv;
      if (dbias) dbias[j] += F(gout)[t * H + j];
    }
  }
  return 0;
#undef LN_DY
}

/* ----------------------------------------------------------- cross entropy */
/* cross_entropy(logits[T,Vp], labels[T]) -> (loss f32[1], dlogits[T,Vp]).
 * Rows with label == ignore_index contribute nothing; columns >= classes are
 * padding (zero gradient).  loss = sum_t (lse_t - x[t,label]) / n_valid and
 * dlogits = (softmax - onehot) * grad_scale / n_valid: the fused forward +
 * monolithic adjoint ("monolithic" mode). */
static int cross_entropy(const orc_tensor* logits, const orc_tensor* labels, orc_tensor* loss,
                         orc_tensor* dlog, const orc_attr* a, int na) {
  const int64_t T = logits->shape[0], Vp = logits->shape[1];
  const int64_t V = aint(a, na, "classes", Vp);
  const int64_t ign = aint(a, na, "ignore_index", -100);
  const float gscale = (float)adbl(a, na, "grad_scale", 1.0);
  const float* X = F(logits);
  const int32_t* L = (const int32_t*)labels->ptr;
  int64_t nvalid = 0;
  for (int64_t t = 0; t < T; ++t)
    if (L[t] != ign) ++nvalid;
  const float inv_n = nvalid ? 1.0f / (float)nvalid : 0.0f;
  float total = 0.0f;
  for (int64_t t = 0; t < T; ++t) {
    const float* x = X + t * Vp;
    float* d = dlog ? F(dlog) + t * Vp : NULL;
    if (L[t] == ign) {
      if (d)
        for (int64_t j = 0; j < Vp; ++j) d[j] = 0.0f;
      continue;
    }
    if (L[t] < 0 || L[t] >= V) return fail("cross_entropy: label %d out of range", L[t]);
    float m = -INFINITY;
    for (int64_t j = 0; j < V; ++j)
      if (x[j] > m) m = x[j];
    float sum = 0.0f;
    for (int64_t j = 0; j < V; ++j) sum += expf(x[j] - m);
    float lse = m + logf(sum);
    total += lse - x[L[t]];
    if (d) {
      const float inv_sum = 1.0f / sum;
      for (int64_t j = 0; j < Vp; ++j) {
        float v = j < V ? expf(x[j] - m) * inv_sum : 0.0f;
        if (j == L[t]) v -= 1.0f;
        d[j] = rnd(dlog->dtype, v * (gscale * inv_n));
      }
    }
  }
  F(loss)[0] = total * inv_n;
  return 0;
}

/* ------------------------------------------------------------------- adam */
/* adam_update (backends.hpp:222-243): double-precision math per element with
 * bias corrections 1 - beta^t, t read from the step tensor.  The _ex variant
 * scales the gradient by grad_scale (ZeRO 1/N mean) and emits the
 * bf16 copy of the updated parameter as a 4th output (fused AutoCast cast). */
static int adam(const orc_tensor* const* in, orc_tensor* out, int nout, const orc_attr* a,
                int na) {
  const double lr = adbl(a, na, "lr", 1e-3);
  const double b1 = adbl(a, na, "beta1", 0.9);
  const double b2 = adbl(a, na, "beta2", 0.999);
  const double eps = adbl(a, na, "eps", 1e-8);
  const double gs = adbl(a, na, "grad_scale", 1.0);
  const double t = F(in[4])[0];
  const double bc1 = 1.0 - pow(b1, t);
  const double bc2 = 1.0 - pow(b2, t);
  const int64_t n = numel(in[0]);
  for (int64_t i = 0; i < n; ++i) {
    double g = F(in[1])[i];
    if (gs != 1.0) g *= gs;
    double mi = b1 * F(in[2])[i] + (1.0 - b1) * g;
    double vi = b2 * F(in[3])[i] + (1.0 - b2) * g * g;
    double mhat = mi / bc1;
    double vhat = vi / bc2;
    float pn = (float)(F(in[0])[i] - lr * mhat / (sqrt(vhat) + eps));
    F(&out[0])[i] = pn;
    F(&out[1])[i] = (float)mi;
    F(&out[2])[i] = (float)vi;
    if (nout > 3) F(&out[3])[i] = rnd(out[3].dtype, pn);
  }
  return 0;
}

/* ew_closure: a rule-fused elementwise group (host/graph.hpp rule_fuse).
 * Registers 0..nin-1 are the inputs ([1]-element inputs broadcast); each
 * instruction "op dst a b dtype imm" computes one exec_base elementwise op in
 * f32 and rounds to its dtype (backends.hpp:59-61, :67-93) -- the same value
 * the op would store unfused; outs = the output registers. */
static int ew_closure(const orc_tensor* in, int nin, orc_tensor* out, int nout, const orc_attr* a, int na) {
  const char* prog = astr(a, na, "prog", "");
  const char* outs = astr(a, na, "outs", "");
  enum { MAXI = 16 };
  char opn[MAXI][16];
  int dst[MAXI], ra[MAXI], rb[MAXI], dt[MAXI], ni = 0, oreg[8], no = 0;
  float imm[MAXI];
  const char* q = prog;
  while (*q && ni < MAXI) {
    int used = 0;
    if (sscanf(q, "%15s %d %d %d %d %f%n", opn[ni], &dst[ni], &ra[ni], &rb[ni], &dt[ni], &imm[ni], &used) != 6)
      return fail("ew_closure: bad program");
    ++ni;
    q += used;
    while (*q == ';' || *q == ' ') ++q;
  }
  q = outs;
  while (*q && no < 8) {
    oreg[no++] = (int)strtol(q, (char**)&q, 10);
    while (*q == ',') ++q;
  }
  if (no != nout) return fail("ew_closure: %d output registers for %d outputs", no, nout);
  const int64_t n = numel(&out[0]);
  float r[8 + MAXI];
  for (int64_t i = 0; i < n; ++i) {
    for (int k = 0; k < nin; ++k) r[k] = F(&in[k])[numel(&in[k]) == 1 ? 0 : i];
    for (int k = 0; k < ni; ++k) {
      const float x = r[ra[k]], y = r[rb[k]];
      float v;
      const char* o = opn[k];
      if (!strcmp(o, "add")) v = x + y;
      else if (!strcmp(o, "sub")) v = x - y;
      else if (!strcmp(o, "mul")) v = x * y;
      else if (!strcmp(o, "div")) v = x / y;
      else if (!strcmp(o, "tanh_dx")) v = y * (1.0f - x * x);
      else if (!strcmp(o, "gelu_dx")) v = y * gelu_grad_f(x);
      else if (!strcmp(o, "neg")) v = -x;
      else if (!strcmp(o, "tanh")) v = tanhf(x);
      else if (!strcmp(o, "relu")) v = x > 0.0f ? x : 0.0f;
      else if (!strcmp(o, "gtz")) v = x > 0.0f ? 1.0f : 0.0f;
      else if (!strcmp(o, "gelu")) v = gelu_f(x);
      else if (!strcmp(o, "add_scalar")) v = x + imm[k];
      else if (!strcmp(o, "copy")) v = x;
      else return fail("ew_closure: no op %s", o);
      r[dst[k]] = rnd(dt[k], v);
    }
    for (int k = 0; k < nout; ++k) F(&out[k])[i] = rnd(out[k].dtype, r[oreg[k]]);
  }
  return 0;
}

/* --------------------------------------------------------------- dispatch */
#define NEED(ni, no)                                                              \
  do {                                                                            \
    if (nin < (ni) || nout < (no)) return fail("%s: expects %d inputs, %d outputs", op, ni, no); \
  } while (0)

int orc_exec(const char* op, const orc_tensor* in, int nin, orc_tensor* out, int nout,
             const orc_attr* attrs, int na) {
  g_err[0] = 0;
  const orc_attr* A = attrs;
  g_rng_step = (uint32_t)aint(A, na, "rng_step", 0);
  /* exec_base if-chain, backends.hpp:168-273 */
  if (!strcmp(op, "add")) { NEED(2, 1); return elemwise_binary(OP_ADD, &in[0], &in[1], &out[0]); }
  if (!strcmp(op, "sub")) { NEED(2, 1); return elemwise_binary(OP_SUB, &in[0], &in[1], &out[0]); }
  if (!strcmp(op, "mul")) { NEED(2, 1); return elemwise_binary(OP_MUL, &in[0], &in[1], &out[0]); }
  if (!strcmp(op, "div")) { NEED(2, 1); return elemwise_binary(OP_DIV, &in[0], &in[1], &out[0]); }
  if (!strcmp(op, "tanh_dx")) { NEED(2, 1); return elemwise_binary(OP_TANH_DX, &in[0], &in[1], &out[0]); }
  if (!strcmp(op, "neg") || !strcmp(op, "tanh") || !strcmp(op, "relu") || !strcmp(op, "gtz") ||
      !strcmp(op, "gelu")) {
    NEED(1, 1);
    return elemwise_unary(op, &in[0], &out[0]);
  }
  if (!strcmp(op, "gelu_dx")) { /* (x, dy) -> dy * gelu'(x) */
    NEED(2, 1);
    int64_t n = numel(&out[0]);
    for (int64_t i = 0; i < n; ++i)
      F(&out[0])[i] = rnd(out[0].dtype, F(&in[1])[i] * gelu_grad_f(F(&in[0])[i]));
    return 0;
  }
  /* cast (backends.hpp:178-183) and its bf16 extension `convert` */
  if (!strcmp(op, "cast") || !strcmp(op, "convert")) {
    NEED(1, 1);
    int64_t n = numel(&out[0]);
    for (int64_t i = 0; i < n; ++i) F(&out[0])[i] = rnd(out[0].dtype, F(&in[0])[i]);
    return 0;
  }
  if (!strcmp(op, "bcast")) { /* backends.hpp:184-190 */
    NEED(1, 1);
    bcast_t bi;
    bcast_init(&bi, &out[0], &in[0]);
    int64_t n = numel(&out[0]);
    for (int64_t i = 0; i < n; ++i) F(&out[0])[i] = rnd(out[0].dtype, F(&in[0])[bcast_map(&bi, i)]);
    return 0;
  }
  if (!strcmp(op, "transpose")) { /* backends.hpp:191-197 */
    NEED(1, 1);
    int64_t r = in[0].shape[0], c = in[0].shape[1];
    for (int64_t i = 0; i < r; ++i)
      for (int64_t j = 0; j < c; ++j) F(&out[0])[j * r + i] = F(&in[0])[i * c + j];
    return 0;
  }
  if (!strcmp(op, "reshape")) { /* backends.hpp:198-202 */
    NEED(1, 1);
    memcpy(out[0].ptr, in[0].ptr, sizeof(float) * numel(&out[0]));
    return 0;
  }
  if (!strcmp(op, "view")) { /* zero-copy slice extension: out = flat(in)[offset:offset+numel] */
    NEED(1, 1);
    int64_t off = aint(A, na, "offset", 0);
    size_t w = in[0].dtype == ORC_U8 ? 1 : 4;
    memcpy(out[0].ptr, (char*)in[0].ptr + off * w, w * numel(&out[0]));
    return 0;
  }
  if (!strcmp(op, "concat")) { /* flat concatenation of flattened inputs */
    NEED(1, 1);
    char* dst = (char*)out[0].ptr;
    for (int i = 0; i < nin; ++i) {
      size_t nb = 4 * (size_t)numel(&in[i]);
      memcpy(dst, in[i].ptr, nb);
      dst += nb;
    }
    return 0;
  }
  if (!strcmp(op, "sum")) { NEED(1, 1); return reduce_op(&in[0], &out[0], astr(A, na, "axes", ""), 0); }
  if (!strcmp(op, "mean")) { NEED(1, 1); return reduce_op(&in[0], &out[0], astr(A, na, "axes", ""), 1); }
  if (!strcmp(op, "add_scalar")) { /* x + value, one rounding */
    NEED(1, 1);
    float v = (float)adbl(A, na, "value", 0.0);
    int64_t n = numel(&out[0]);
    for (int64_t i = 0; i < n; ++i) F(&out[0])[i] = rnd(out[0].dtype, F(&in[0])[i] + v);
    return 0;
  }
  if (!strcmp(op, "fill")) {
    if (nout < 1) return fail("fill: one output");
    float v = (float)adbl(A, na, "value", 0.0);
    int64_t n = numel(&out[0]);
    for (int64_t i = 0; i < n; ++i) F(&out[0])[i] = rnd(out[0].dtype, v);
    return 0;
  }
  if (!strcmp(op, "colsum")) { /* bias gradient: f32 column sums over all leading dims, rows ascending;
                                  with labels, rows labelled ignore_index are skipped */
    NEED(1, 1);
    int64_t C = in[0].shape[in[0].rank - 1], R = numel(&in[0]) / C;
    const int32_t* lab = nin > 1 ? (const int32_t*)in[1].ptr : NULL;
    const int64_t ign = aint(A, na, "ignore_index", -100);
    for (int64_t j = 0; j < C; ++j) F(&out[0])[j] = 0.0f;
    for (int64_t r = 0; r < R; ++r) {
      if (lab && lab[r] == ign) continue;
      for (int64_t j = 0; j < C; ++j) F(&out[0])[j] += F(&in[0])[r * C + j];
    }
    return 0;
  }
  if (!strcmp(op, "mse")) { /* backends.hpp:205-214: sequential acc, then a divide */
    NEED(2, 1);
    float acc = 0.0f;
    int64_t n = numel(&in[0]);
    for (int64_t i = 0; i < n; ++i) {
      float d = F(&in[0])[i] - F(&in[1])[i];
      acc += d * d;
    }
    F(&out[0])[0] = acc / (float)n;
    return 0;
  }
  if (!strcmp(op, "matmul")) { /* backends.hpp:143-155,215 */
    NEED(2, 1);
    gemm_acc(F(&in[0]), F(&in[1]), F(&out[0]), in[0].shape[0], in[1].shape[1], in[0].shape[1], 0, 0, 1.0f);
    round_all(&out[0], numel(&out[0]));
    return 0;
  }
  if (!strcmp(op, "matmul_t")) { /* C = alpha * op(A) op(B), one rounding at the end */
    NEED(2, 1);
    int ta = (int)aint(A, na, "ta", 0), tb = (int)aint(A, na, "tb", 0);
    int64_t M = ta ? in[0].shape[1] : in[0].shape[0];
    int64_t K = ta ? in[0].shape[0] : in[0].shape[1];
    int64_t N = tb ? in[1].shape[0] : in[1].shape[1];
    gemm_acc(F(&in[0]), F(&in[1]), F(&out[0]), M, N, K, ta, tb, (float)adbl(A, na, "alpha", 1.0));
    round_all(&out[0], numel(&out[0]));
    return 0;
  }
  if (!strcmp(op, "batch_matmul")) {
    NEED(2, 1);
    int ta = (int)aint(A, na, "ta", 0), tb = (int)aint(A, na, "tb", 0);
    int64_t Z = in[0].shape[0];
    int64_t M = ta ? in[0].shape[2] : in[0].shape[1];
    int64_t K = ta ? in[0].shape[1] : in[0].shape[2];
    int64_t N = tb ? in[1].shape[1] : in[1].shape[2];
    for (int64_t z = 0; z < Z; ++z)
      gemm_acc(F(&in[0]) + z * M * K, F(&in[1]) + z * K * N, F(&out[0]) + z * M * N, M, N, K, ta, tb,
               (float)adbl(A, na, "alpha", 1.0));
    round_all(&out[0], numel(&out[0]));
    return 0;
  }
  /* linear: act(x . W + bias) -- matmul_add_act (backends.hpp:311-324) with the
   * gelu extension; one rounding at the end; tw reads W stored [N,K].
   * Outputs (y) or (y, u) where u is the rounded pre-activation, or with
   * save=grad the rounded derivative act'(pre-activation). */
  if (!strcmp(op, "linear")) {
    NEED(3, 1);
    int act = parse_act(astr(A, na, "act", "none"));
    if (act < 0) return fail("linear: bad act");
    const int save_grad = !strcmp(astr(A, na, "save", "preact"), "grad");
    linear_fwd(&in[0], &in[1], &in[2], &out[0], nout > 1 ? &out[1] : NULL, act, (int)aint(A, na, "tw", 0),
               save_grad);
    return 0;
  }
  /* embedding_sum(ids.., tables..): gathers added in table order, each sum
   * rounded to the tables' dtype (= the embedding / add chain it replaces) */
  if (!strcmp(op, "embedding_sum")) {
    const int n = nin / 2;
    if (nin != 2 * n || n < 2 || nout != 1) return fail("embedding_sum: (ids.., tables..) -> 1 output");
    const int64_t Tn = numel(&in[0]), H = in[n].shape[1];
    for (int64_t t = 0; t < Tn; ++t)
      for (int64_t j = 0; j < H; ++j) {
        float acc = F(&in[n])[(int64_t)((const int32_t*)in[0].ptr)[t] * H + j];
        for (int k = 1; k < n; ++k)
          acc = rnd(out[0].dtype, acc + F(&in[n + k])[(int64_t)((const int32_t*)in[k].ptr)[t] * H + j]);
        F(&out[0])[t * H + j] = rnd(out[0].dtype, acc);
      }
    return 0;
  }
  /* matmul_pair(a0, b0 [, aux0], a1, b1): problem 0 is matmul_t (n0 = 2) or
   * matmul_dact (n0 = 3), problem 1 matmul_t -- the same arithmetic as the two
   * separate ops (horizontal fusion only changes the launch). */
  if (!strcmp(op, "matmul_pair")) {
    const int n0 = (int)aint(A, na, "n0", 2);
    if (nin != n0 + 2 || nout != 2) return fail("matmul_pair: expects %d inputs, 2 outputs", n0 + 2);
    for (int p = 0; p < 2; ++p) {
      char kt[8], kb[8], kal[8];
      snprintf(kt, sizeof kt, "ta%d", p);
      snprintf(kb, sizeof kb, "tb%d", p);
      snprintf(kal, sizeof kal, "alpha%d", p);
      const orc_tensor* a0 = &in[p ? n0 : 0];
      const orc_tensor* b0 = &in[p ? n0 + 1 : 1];
      int ta = (int)aint(A, na, kt, 0), tb = (int)aint(A, na, kb, 0);
      int64_t M = ta ? a0->shape[1] : a0->shape[0];
      int64_t K = ta ? a0->shape[0] : a0->shape[1];
      int64_t N = tb ? b0->shape[0] : b0->shape[1];
      gemm_acc(F(a0), F(b0), F(&out[p]), M, N, K, ta, tb, (float)adbl(A, na, kal, 1.0));
      if (p == 0 && n0 == 3) {
        int act = parse_act(astr(A, na, "act0", "none"));
        for (int64_t i = 0; i < M * N; ++i)
          F(&out[0])[i] = rnd(out[0].dtype, F(&out[0])[i] * dact_f(act, F(&in[2])[i]));
      } else {
        round_all(&out[p], M * N);
      }
    }
    return 0;
  }
  /* matmul_dact(a, b, aux): (op(a) op(b)) * act'(aux) -- a backward GEMM with the
   * activation derivative fused into its epilogue. */
  if (!strcmp(op, "matmul_dact")) {
    NEED(3, 1);
    int act = parse_act(astr(A, na, "act", "none"));
    int ta = (int)aint(A, na, "ta", 0), tb = (int)aint(A, na, "tb", 0);
    int64_t M = ta ? in[0].shape[1] : in[0].shape[0];
    int64_t K = ta ? in[0].shape[0] : in[0].shape[1];
    int64_t N = tb ? in[1].shape[0] : in[1].shape[1];
    gemm_acc(F(&in[0]), F(&in[1]), F(&out[0]), M, N, K, ta, tb, 1.0f);
    int64_t n = M * N;
    for (int64_t i = 0; i < n; ++i)
      F(&out[0])[i] = rnd(out[0].dtype, F(&out[0])[i] * dact_f(act, F(&in[2])[i]));
    return 0;
  }
  if (!strcmp(op, "sgd_update")) { /* backends.hpp:216-221 */
    NEED(2, 1);
    float lr = (float)adbl(A, na, "lr", 0.0);
    int64_t n = numel(&out[0]);
    for (int64_t i = 0; i < n; ++i) F(&out[0])[i] = F(&in[0])[i] - lr * F(&in[1])[i];
    return 0;
  }
  if (!strcmp(op, "adam_update") || !strcmp(op, "adam_update_ex")) {
    NEED(5, 3);
    const orc_tensor* ins[5] = {&in[0], &in[1], &in[2], &in[3], &in[4]};
    return adam(ins, out, nout, A, na);
  }
  if (!strcmp(op, "dropout")) {
    NEED(1, 1);
    float p = (float)adbl(A, na, "p", 0.0);
    uint64_t seed = (uint64_t)aint(A, na, "seed", 0), salt = (uint64_t)aint(A, na, "salt", 0);
    float sp = p > 0.0f ? 1.0f / (1.0f - p) : 1.0f;
    int64_t n = numel(&out[0]);
    for (int64_t i = 0; i < n; ++i)
      F(&out[0])[i] = rnd(out[0].dtype, orc_dropout_keep(seed, salt, (uint64_t)i, p) ? F(&in[0])[i] * sp : 0.0f);
    return 0;
  }
  if (!strcmp(op, "softmax")) { /* rows of the last axis; scale then optional causal mask */
    NEED(1, 1);
    float scale = (float)adbl(A, na, "scale", 1.0);
    int causal = (int)aint(A, na, "causal", 0);
    int64_t C = in[0].shape[in[0].rank - 1], R = numel(&in[0]) / C;
    int64_t Sq = in[0].rank >= 2 ? in[0].shape[in[0].rank - 2] : 1;
    for (int64_t r = 0; r < R; ++r) {
      const float* x = F(&in[0]) + r * C;
      float* y = F(&out[0]) + r * C;
      int64_t qi = r % Sq;
      float m = -INFINITY;
      for (int64_t j = 0; j < C; ++j) {
        float v = (causal && j > qi) ? -INFINITY : x[j] * scale;
        y[j] = v;
        if (v > m) m = v;
      }
      float sum = 0.0f;
      for (int64_t j = 0; j < C; ++j) {
        y[j] = expf(y[j] - m);
        sum += y[j];
      }
      for (int64_t j = 0; j < C; ++j) y[j] = rnd(out[0].dtype, y[j] / sum);
    }
    return 0;
  }
  if (!strcmp(op, "softmax_dx")) { /* (y, dy) -> scale * y * (dy - sum(y*dy)) */
    NEED(2, 1);
    float scale = (float)adbl(A, na, "scale", 1.0);
    int64_t C = in[0].shape[in[0].rank - 1], R = numel(&in[0]) / C;
    for (int64_t r = 0; r < R; ++r) {
      const float* y = F(&in[0]) + r * C;
      const float* dy = F(&in[1]) + r * C;
      float dot = 0.0f;
      for (int64_t j = 0; j < C; ++j) dot += y[j] * dy[j];
      for (int64_t j = 0; j < C; ++j) F(&out[0])[r * C + j] = rnd(out[0].dtype, y[j] * (dy[j] - dot) * scale);
    }
    return 0;
  }
  if (!strcmp(op, "ew_closure")) return ew_closure(in, nin, out, nout, A, na);
  if (!strcmp(op, "attention") && aint(A, na, "lse", 0)) {
    NEED(1, 2);
    return attention_fwd_lse(&in[0], &out[0], &out[1], nout > 2 ? &out[2] : NULL, A, na);
  }
  if (!strcmp(op, "attention_dx") && aint(A, na, "lse", 0)) {
    NEED(4, 1);
    return attention_bwd_lse(&in[0], &in[1], &in[2], &in[3], nin > 4 ? &in[4] : NULL, &out[0], A, na);
  }
  if (!strcmp(op, "attention")) {
    NEED(1, 2);
    return attention_fwd(&in[0], &out[0], &out[1], nout > 2 ? &out[2] : NULL, A, na);
  }
  if (!strcmp(op, "attention_dx")) {
    NEED(3, 1);
    return attention_bwd(&in[0], &in[1], &in[2], nin > 3 ? &in[3] : NULL, &out[0], A, na);
  }
  if (!strcmp(op, "layer_norm")) {
    NEED(3, 3);
    return layer_norm_fwd(&in[0], NULL, &in[1], &in[2], &out[0], NULL, &out[1], &out[2], NULL, A, na);
  }
  if (!strcmp(op, "add_layer_norm")) {
    NEED(4, 4);
    return layer_norm_fwd(&in[0], &in[1], &in[2], &in[3], &out[0], &out[1], &out[2], &out[3], nout > 4 ? &out[4] : NULL,
                          A, na);
  }
  if (!strcmp(op, "layer_norm_dx")) {
    NEED(5, 3);
    /* mask_in: the last input is add_layer_norm's saved keep bits */
    const int mask_in = (int)aint(A, na, "mask_in", 0) != 0;
    const int nd = nin - mask_in;
    const orc_tensor* ins[7] = {&in[0], &in[1], &in[2], &in[3], &in[4], nd > 5 ? &in[5] : NULL,
                                mask_in ? &in[nin - 1] : NULL};
    return layer_norm_bwd(ins, nd, out, nout, A, na);
  }
  if (!strcmp(op, "embedding")) { /* out[t,:] = table[ids[t],:] */
    NEED(2, 1);
    const int32_t* ids = (const int32_t*)in[0].ptr;
    int64_t T = numel(&in[0]), V = in[1].shape[0], H = in[1].shape[1];
    for (int64_t t = 0; t < T; ++t) {
      if (ids[t] < 0 || ids[t] >= V) return fail("embedding: id %d out of range", ids[t]);
      for (int64_t j = 0; j < H; ++j) F(&out[0])[t * H + j] = rnd(out[0].dtype, F(&in[1])[ids[t] * H + j]);
    }
    return 0;
  }
  if (!strcmp(op, "embedding_dx")) { /* (ids, dy [, base]) -> base + scatter_add, t ascending */
    NEED(2, 1);
    const int32_t* ids = (const int32_t*)in[0].ptr;
    int64_t T = numel(&in[0]), V = out[0].shape[0], H = out[0].shape[1];
    if (nin > 2) memcpy(out[0].ptr, in[2].ptr, sizeof(float) * V * H);
    else memset(out[0].ptr, 0, sizeof(float) * V * H);
    for (int64_t t = 0; t < T; ++t)
      for (int64_t j = 0; j < H; ++j) F(&out[0])[ids[t] * H + j] += F(&in[1])[t * H + j];
    return 0;
  }
  if (!strcmp(op, "cross_entropy")) {
    NEED(2, 1);
    return cross_entropy(&in[0], &in[1], &out[0], nout > 1 ? &out[1] : NULL, A, na);
  }
  /* collectives at world == 1 (backends.hpp:245-273) */
  if (!strcmp(op, "allreduce") || !strcmp(op, "reduce_scatter") || !strcmp(op, "all_gather") ||
      !strcmp(op, "shard") || !strcmp(op, "reduce_scatter_batched") ||
      !strcmp(op, "all_gather_batched")) {
    int64_t world = aint(A, na, "world", 1);
    if (world != 1)
      return fail("collective op %s requires the simulation bus (world=%lld)", op, (long long)world);
    if (!strcmp(op, "reduce_scatter_batched") || !strcmp(op, "all_gather_batched")) {
      for (int i = 0; i < nin && i < nout; ++i) {
        int64_t n = numel(&out[i]), m = numel(&in[i]);
        for (int64_t j = 0; j < n && j < m; ++j) F(&out[i])[j] = F(&in[i])[j];
      }
      return 0;
    }
    int64_t n = numel(&out[0]), m = numel(&in[0]);
    for (int64_t j = 0; j < n; ++j) F(&out[0])[j] = j < m ? F(&in[0])[j] : 0.0f;
    return 0;
  }
  return fail("no ref kernel for op %s", op);
}
