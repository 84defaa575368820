// fold.cuh -- deferred partial-sum folds.
//
// Several backward ops reduce over the token dimension in two deterministic
// stages: a wide kernel writes per-block partial rows, a small kernel folds the
// rows in fixed order (LayerNorm dgamma / dbeta / fused bias grad, bias-grad
// colsums).  The folded vectors are only read by the optimizer, so inside a
// training step the VM turns deferral on: each such op writes its partials to
// a buffer owned by that op instance (keyed by its output pointer) and queues a
// FoldJob; tcb_fold_flush() then folds every queued job in ONE launch before the
// optimizer (and tcb_launch flushes early if any launch reads a pending
// output).  The sums and their order are exactly those of the per-op fold
// kernels, so results are bit-identical with deferral on or off.
#pragma once
#include "common.cuh"

namespace tcb {

// out[c] = scale * sum_{r < nrows} src[r * ld + c] for c < ncols, rows added
// in the per-op kernels' order (32 interleaved warp sums, then warp order)
struct FoldJob {
  const float* src;
  int64_t ld;
  int nrows;
  int ncols;
  float* out;
  float scale;
};

struct FoldCtx;
FoldCtx* fold_ctx_create(size_t pool_bytes);  // outside stream capture
void fold_ctx_destroy(FoldCtx* c);
void fold_use(FoldCtx* c);  // this thread's deferral uses c (nullptr: off)
bool fold_deferring();
// deferral on/off; on allocates (once, eagerly) a pool of pool_bytes for the
// per-instance partial buffers.  Must be called outside stream capture.
void fold_set(bool on, size_t pool_bytes);
// per-op-instance partial buffer carved from the pool (nullptr: not deferring
// or the pool is exhausted -- the op then folds in place)
float* fold_scratch(const void* key, int tag, size_t bytes);
void fold_defer(const FoldJob& j);
// one per op instance whose fold kernel was deferred (launch accounting)
void fold_op_deferred();
void fold_counters(uint64_t* ops, uint64_t* launches);
void fold_flush(cudaStream_t s);
// flush now if any of [ptr, ptr + bytes) is a pending job's output
void fold_flush_if_reads(const void* ptr, size_t bytes, cudaStream_t s);

}  // namespace tcb
