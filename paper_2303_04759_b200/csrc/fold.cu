// fold.cu -- deferred partial-sum folds (see fold.cuh).
#include <map>
#include <utility>
#include <vector>

#include "fold.cuh"

namespace tcb {

// A pool of per-op-instance partial buffers.  One context per launch context
// (the device VM owns one; its slots die with it), so sessions never share
// slots and a later session cannot be handed a smaller slot of an earlier one.
struct FoldCtx {
  std::unique_ptr<Scratch> pool;
  size_t pool_bytes = 0, used = 0;
  std::map<std::pair<const void*, int>, std::pair<size_t, size_t>> slots;  // (key, tag) -> (offset, bytes)
};

namespace {
struct FoldState {
  bool on = false;
  FoldCtx* ctx = nullptr;  // active context (a VM's, or `own` for tcb_fold_defer)
  FoldCtx own;
  std::vector<FoldJob> jobs;
  uint64_t ops_deferred = 0, flush_launches = 0;  // cumulative (launch accounting)
};
// per thread: one VM (rank) per thread may run concurrently,
// each with its own queue and context on its own device
FoldState& st() {
  thread_local FoldState s;
  return s;
}
}  // namespace

bool fold_deferring() { return st().on; }

float* fold_scratch(const void* key, int tag, size_t bytes) {
  FoldState& s = st();
  if (!s.on || !s.ctx || !s.ctx->pool) return nullptr;
  FoldCtx& c = *s.ctx;
  bytes = (bytes + 255) & ~size_t(255);
  auto it = c.slots.find({key, tag});
  if (it != c.slots.end() && it->second.second >= bytes)
    return reinterpret_cast<float*>(static_cast<char*>(c.pool->p) + it->second.first);
  // new key, or a larger request than the slot holds: carve a fresh region
  if (c.used + bytes > c.pool_bytes) return nullptr;  // pool exhausted: the op folds in place
  c.slots[{key, tag}] = {c.used, bytes};
  float* p = reinterpret_cast<float*>(static_cast<char*>(c.pool->p) + c.used);
  c.used += bytes;
  return p;
}

FoldCtx* fold_ctx_create(size_t pool_bytes) {
  auto* c = new FoldCtx;
  if (pool_bytes) {
    c->pool = std::make_unique<Scratch>(pool_bytes);
    c->pool_bytes = pool_bytes;
  }
  return c;
}
void fold_ctx_destroy(FoldCtx* c) {
  FoldState& s = st();
  if (s.ctx == c) {
    s.ctx = nullptr;
    s.on = false;
  }
  delete c;
}
void fold_use(FoldCtx* c) {
  FoldState& s = st();
  s.ctx = c;
  s.on = c && c->pool;
}

void fold_defer(const FoldJob& j) {
  // an identical job already queued (the same plan relaunched on the same
  // buffers, e.g. vm.profile's repeated launches) folds the same partials
  // into the same output: once is enough
  for (const FoldJob& q : st().jobs)
    if (q.src == j.src && q.out == j.out && q.ld == j.ld && q.nrows == j.nrows && q.ncols == j.ncols &&
        q.scale == j.scale)
      return;
  st().jobs.push_back(j);
}
void fold_op_deferred() { ++st().ops_deferred; }
void fold_counters(uint64_t* ops, uint64_t* launches) {
  *ops = st().ops_deferred;
  *launches = st().flush_launches;
}

constexpr int FOLD_MAXJ = 192;  // kernel parameters: ~8.5 KB of the 32 KB limit
constexpr int FOLD_COLS = 128;  // columns per block: 32 lanes x float4
struct FoldTable {
  FoldJob job[FOLD_MAXJ];
  int ub[FOLD_MAXJ + 1];  // first column block of each job (prefix sums)
  int n;
};

// Same sums, same order as k_ln_colsum / k_colsum_final (so deferral is
// bit-identical): phase w = 0..31 sums rows w, w+32, ... in increasing order,
// then the 32 phase sums are added in phase order.  A block covers 128 columns
// (a float4 per lane); warp v owns phases 4v..4v+3, so all of a thread's row
// loads of one round are independent and in flight together.
__global__ void __launch_bounds__(256) k_fold_multi(const __grid_constant__ FoldTable T) {
  TCB_PDL_ENTRY();
  __shared__ float4 red[32][32];  // [phase][lane]
  const int b = blockIdx.x;
  int j = 0;
  while (j + 1 < T.n && T.ub[j + 1] <= b) ++j;
  const FoldJob& J = T.job[j];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t c0 = int64_t(b - T.ub[j]) * FOLD_COLS + lane * 4;
  const bool vec = (J.ncols % 4 == 0) && (J.ld % 4 == 0) && (reinterpret_cast<uintptr_t>(J.src) % 16 == 0);
  float4 s[4];
#pragma unroll
  for (int p = 0; p < 4; ++p) s[p] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
  if (c0 < J.ncols) {
    for (int r = 0; r < J.nrows; r += 32) {
      float4 x[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const int k = r + warp * 4 + p;
        x[p] = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        if (k < J.nrows) {
          const float* q = J.src + int64_t(k) * J.ld + c0;
          if (vec) {
            x[p] = *reinterpret_cast<const float4*>(q);
          } else {
            x[p].x = q[0];
            if (c0 + 1 < J.ncols) x[p].y = q[1];
            if (c0 + 2 < J.ncols) x[p].z = q[2];
            if (c0 + 3 < J.ncols) x[p].w = q[3];
          }
        }
      }
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        if (r + warp * 4 + p < J.nrows) {
          s[p].x += x[p].x;
          s[p].y += x[p].y;
          s[p].z += x[p].z;
          s[p].w += x[p].w;
        }
      }
    }
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) red[warp * 4 + p][lane] = s[p];
  __syncthreads();
  if (warp == 0 && c0 < J.ncols) {
    float4 t = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll 8
    for (int w = 0; w < 32; ++w) {
      const float4 v = red[w][lane];
      t.x += v.x;
      t.y += v.y;
      t.z += v.z;
      t.w += v.w;
    }
    const float sc = J.scale;
    float* o = J.out + c0;
    o[0] = sc == 1.0f ? t.x : t.x * sc;
    if (c0 + 1 < J.ncols) o[1] = sc == 1.0f ? t.y : t.y * sc;
    if (c0 + 2 < J.ncols) o[2] = sc == 1.0f ? t.z : t.z * sc;
    if (c0 + 3 < J.ncols) o[3] = sc == 1.0f ? t.w : t.w * sc;
  }
}

void fold_flush(cudaStream_t s) {
  FoldState& S = st();
  size_t i = 0;
  while (i < S.jobs.size()) {
    FoldTable T{};
    int units = 0;
    T.n = 0;
    for (; i < S.jobs.size() && T.n < FOLD_MAXJ; ++i) {
      T.job[T.n] = S.jobs[i];
      T.ub[T.n] = units;
      units += (S.jobs[i].ncols + FOLD_COLS - 1) / FOLD_COLS;
      ++T.n;
    }
    T.ub[T.n] = units;
    if (units) {
      launch_k(k_fold_multi, unsigned(units), 256, 0, s, T);
      ++S.flush_launches;
    }
  }
  S.jobs.clear();
}

void fold_flush_if_reads(const void* ptr, size_t bytes, cudaStream_t s) {
  FoldState& S = st();
  if (S.jobs.empty() || !ptr) return;
  const char* a = static_cast<const char*>(ptr);
  for (const FoldJob& j : S.jobs) {
    const char* o = reinterpret_cast<const char*>(j.out);
    if (a < o + size_t(j.ncols) * sizeof(float) && o < a + bytes) {
      fold_flush(s);
      return;
    }
  }
}

void fold_set(bool on, size_t pool_bytes) {
  FoldState& s = st();
  FoldCtx& c = s.own;
  if (on && pool_bytes && (!c.pool || c.pool_bytes < pool_bytes)) {
    c.pool.reset();
    c.slots.clear();
    c.used = 0;
    c.pool = std::make_unique<Scratch>(pool_bytes);
    c.pool_bytes = pool_bytes;
  }
  s.ctx = &c;
  s.on = on && c.pool != nullptr;
}

}  // namespace tcb
