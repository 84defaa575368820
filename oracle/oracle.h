/* oracle.h -- CPU restatement of the reference kernels (TEST INFRASTRUCTURE).
 *
 * This library is the parity checker for libtcb200.so.  It is NOT part of the
 * product: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.
 *
 * Semantics follow /root/reference/proj/include/trainc/backends.hpp (the `ref`
 * dialect, "the bit-level ground truth"): f32 compute, fixed left-to-right
 * accumulation, half types emulated as f32 storage rounded to nearest-even
 * after every op (backends.hpp:59-61).  Each function in oracle.c cites the
 * reference line it restates.  Extension ops (transformer ops the reference
 * lacks) follow the same conventions; their parity is pinned by
 * finite differences and torch CPU (tests/test_oracle_*), not by the reference.
 *
 * Build with -ffp-contract=off (contraction changes matmul bits).
 */
#ifndef TRAINC_ORACLE_H_
#define TRAINC_ORACLE_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* same layout as tcb_tensor (include/tcb200.h); ptr is HOST memory:
 * float* for f32/f16/bf16 (emulated, values on the half grid), int32_t* for
 * i32, uint8_t* for u8. */
typedef struct {
  void* ptr;
  int32_t dtype;
  int32_t rank;
  int64_t shape[8];
  int64_t stride[8];
} orc_tensor;

typedef struct {
  const char* key;
  int32_t kind; /* 0 int, 1 float, 2 string */
  int64_t i;
  double d;
  const char* s;
} orc_attr;

enum { ORC_F32 = 0, ORC_F16 = 1, ORC_BF16 = 2, ORC_I32 = 3, ORC_U8 = 4 };

/* Execute base op `op` (no dialect prefix).  Outputs are preallocated by the
 * caller with the shapes the type relation gives.  Returns 0 or non-zero with
 * orc_last_error() set. */
int orc_exec(const char* op, const orc_tensor* in, int nin, orc_tensor* out, int nout,
             const orc_attr* attrs, int nattr);
const char* orc_last_error(void);

/* rounding helpers (fp16.hpp:14-76 restated; bf16 is the extension) */
uint16_t orc_float_to_half_bits(float f);
float orc_half_bits_to_float(uint16_t h);
float orc_quantize_f16(float f);
uint16_t orc_float_to_bf16_bits(float f);
float orc_bf16_bits_to_float(uint16_t h);
float orc_quantize_bf16(float f);

/* Philox4x32-10 keep-mask draw used by dropout: 1 = keep. */
int orc_dropout_keep_step(uint64_t seed, uint64_t salt, uint64_t index, float p, uint32_t step);
int orc_dropout_keep(uint64_t seed, uint64_t salt, uint64_t index, float p);

/* mt19937-backed generator restating Rng (tensor.hpp:145-176) so synthetic
 * data is byte-identical to what the reference would generate. */
typedef struct orc_rng_ orc_rng;
orc_rng* orc_rng_new(uint64_t seed);
void orc_rng_free(orc_rng* r);
uint32_t orc_rng_next_u32(orc_rng* r);
float orc_rng_uniform(orc_rng* r, float lo, float hi);
uint32_t orc_rng_below(orc_rng* r, uint32_t n);
void orc_rng_fill_uniform(orc_rng* r, float* out, int64_t n, float lo, float hi);
void orc_rng_fill_below(orc_rng* r, int32_t* out, int64_t n, uint32_t bound);

#ifdef __cplusplus
}
#endif
#endif
