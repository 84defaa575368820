// k_attention.cu -- fused multi-head attention for short sequences (S <= 128,
// head dim 64): one CTA per (batch, head), everything on-chip.
//
// Forward  (oracle.c attention_fwd):
//   TMA Q, K, V head tiles straight out of qkv [T, 3H] (no split copies)
//   S  = Q K^T                 tcgen05.mma 128x128x64 -> TMEM
//   P  = softmax(scale * S)    16 warps: a (query row = TMEM lane, 32-key
//                              quarter) per thread, quarters combined in smem
//   probs <- P (bf16)          swizzled smem tile -> TMA store (saved for bwd)
//   Pd = dropout(P)            Philox keep bits, same indices as k_softmax
//   O  = Pd V                  tcgen05.mma 128x64x128 (Pd = K-major A from
//                              smem, V = MN-major B) -> TMEM -> TMA store ctx
// Backward (oracle.c attention_bwd):
//   dPd = dO V^T  -> TMEM;  per row: dP = keep*dPd/(1-p), rowdot = P.dP,
//   dS = P (dP - rowdot) scale (bf16 smem), Pd in place of P;
//   dV = Pd^T dO, dQ = dS K, dK = dS^T Q: the transposed operands are the same
//   smem tiles read through MN-major UMMA descriptors; dQ/dK/dV -> TMA stores
//   into dqkv.
// Scores/P never touch HBM except the bf16 P the backward needs: per head the
// forward moves 48 KB in + 16 KB ctx + 32 KB probs, the backward 96 KB in +
// 48 KB out.
#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace tcb {

constexpr int AT_S = 128;         // query / key tile (sequence padded to 128)
constexpr int AT_D = 64;          // head dim (one SWIZZLE_128B row)
constexpr int AT_TILE = 16384;    // 128 rows x 128 B
constexpr int AT_THREADS = 256;   // backward: 8 warps, 2 per TMEM lane quarter, one per 64-key half
constexpr int AT_FWD_THREADS = 512;  // forward: 16 warps, 4 per lane quarter, one per 32-key quarter

struct AttnArgs {
  int S, H, A, dh, causal, Z;
  unsigned long long* trace;
  float scale;
  DropCfg d;
  // lse mode (attention lse=1): the forward writes the per-row log-sum-exp
  // instead of storing P; the backward recomputes P = 2^(S log2e scale - lse
  // log2e) from a QK^T MMA instead of loading it
  float* lse_out;
  const float* lse_in;
  int nw;  // saved keep-bit words per query row: 4 (stored-P mode), ceil(S/32) (lse mode)
};

// byte offset of granule g (8 bf16) of row r in a [128 rows x 128 B] SW128 tile
__device__ __forceinline__ uint32_t sw128(int r, int g) { return uint32_t(r * 128 + ((g ^ (r & 7)) << 4)); }

__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

__device__ __forceinline__ void tma_load_3(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1,
                                           int c2) {
  tma_load_4d<1>(dst, map, smem_u32(bar), c0, c1, c2, 0);
}

// keep bits for 64 row elements j0 .. j0+63 of flat index base + j (base, j0 % 8 == 0)
__device__ __forceinline__ void keep_bits64(const DropCfg& d, uint64_t base, int j0, int S, uint32_t (&kb)[2]) {
  kb[0] = kb[1] = 0xffffffffu;
  if (d.p <= 0.0f) return;
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    if (j0 + g * 8 < S) {
      const uint32_t b = dropout_bits8q(d, ((base + j0) >> 3) + g);
      kb[g >> 2] = (kb[g >> 2] & ~(0xffu << ((g & 3) * 8))) | (b << ((g & 3) * 8));
    }
  }
}
// keep bits for 32 row elements j0 .. j0+31 of flat index base + j (base, j0 % 8 == 0)
__device__ __forceinline__ uint32_t keep_bits32(const DropCfg& d, uint64_t base, int j0, int S) {
  uint32_t kb = 0xffffffffu;
  if (d.p <= 0.0f) return kb;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    if (j0 + g * 8 < S) {
      const uint32_t b = dropout_bits8q(d, ((base + j0) >> 3) + g);
      kb = (kb & ~(0xffu << (g * 8))) | (b << (g * 8));
    }
  }
  return kb;
}
// e^x on the MUFU path (ex2.approx; -inf -> 0); the oracle's expf differs by a few ulp
__device__ __forceinline__ float fast_exp(float x) { return ex2_approx(x * 1.4426950408889634f); }

// ------------------------------------------------------------------ forward
// Thread layout: warp w owns TMEM lane quarter q = w % 4 (query rows 32q..+31)
// and key quarter cq = w / 4 (columns 32cq..+31, half of one SW128 P tile); the
// four quarters of a row combine max / sum through smem.
__global__ void __launch_bounds__(AT_FWD_THREADS) k_attn_fwd(const __grid_constant__ CUtensorMap m_qkv,
                                                             const __grid_constant__ CUtensorMap m_probs,
                                                             const __grid_constant__ CUtensorMap m_ctx,
                                                             const AttnArgs a) {
  // Persistent over heads z = blockIdx.x, +gridDim.x, ...: the Q/K/V tiles of
  // the next head stream in (TMA, second buffer) while this head's softmax and
  // PV product run; ctx / probs leave through asynchronous TMA stores.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQKV = sm;                        // 2 buffers x (Q, K, V)
  uint8_t* sP = sm + 6 * AT_TILE;            // 2 tiles: keys 0-63, 64-127 (probs, stored)
  uint8_t* sPd = sm + 8 * AT_TILE;           // 2 tiles: dropout(P), the PV operand (p > 0)
  float* red = reinterpret_cast<float*>(sm + 10 * AT_TILE);  // [2 stats][4 quarters][128 rows]
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 1024);  // load[2], mma1, mma2
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, cq = warp >> 2;
  const int row = q * 32 + lane;  // query row = TMEM lane
  const int j0 = cq * 32;         // this thread's key columns
  const int Z = gridDim.x > 0 ? a.Z : 0;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&m_qkv)) : "memory");
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc1<256>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tslot;
  pdl_wait();
  pdl_trigger();
  DropCfg dd = a.d;
  drop_resolve(dd);

  auto issue_load = [&](int zz, int buf) {
    const int bb = zz / a.A, hh = zz % a.A;
    uint8_t* dst = sQKV + buf * 3 * AT_TILE;
    mbar_expect_tx(&bar[buf], 3 * AT_TILE);
    tma_load_3(dst, &m_qkv, &bar[buf], hh * AT_D, 0, bb);
    tma_load_3(dst + AT_TILE, &m_qkv, &bar[buf], a.H + hh * AT_D, 0, bb);
    tma_load_3(dst + 2 * AT_TILE, &m_qkv, &bar[buf], 2 * a.H + hh * AT_D, 0, bb);
  };
  if (tid == 0 && int(blockIdx.x) < Z) issue_load(blockIdx.x, 0);
  const uint32_t trow = tm + (uint32_t(q * 32) << 16);
  int it = 0;
  unsigned long long* tr = a.trace ? a.trace + blockIdx.x * 8 : nullptr;
  auto T = [&](int k) {
    if (tr && tid == 0 && it == 1) tr[k] = gtimer();
  };
  for (int z = blockIdx.x; z < Z; z += gridDim.x, ++it) {
    T(0);
    const int buf = it & 1;
    const int b = z / a.A, h = z % a.A;
    uint8_t* sQ = sQKV + buf * 3 * AT_TILE;
    uint8_t* sK = sQ + AT_TILE;
    uint8_t* sV = sQ + 2 * AT_TILE;
    if (tid == 0) {
      const int zn = z + int(gridDim.x);
      if (zn < Z) {
        // the other buffer last held head it-1: its MMAs are complete and its
        // Q tile (ctx staging) has been read by that head's store
        bulk_wait_read<0>();
        issue_load(zn, buf ^ 1);
      }
      mbar_wait(&bar[buf], (it >> 1) & 1);
      T(1);
      tc_fence_after();
      constexpr uint32_t id1 = umma_idesc(128, 128, true, false, false);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        tc_mma<1>(tm, umma_desc(smem_u32(sQ) + k * 32, 16, 1024), umma_desc(smem_u32(sK) + k * 32, 16, 1024), id1,
                  k ? 1u : 0u);
      tc_commit<1>(&bar[2]);
    }
    // dropout keep bits overlap the QK^T MMA (and are saved for the backward)
    const uint32_t kb = keep_bits32(dd, (uint64_t(z) * a.S + row) * a.S, j0, a.S);
    if (dd.mask_out && row < a.S && cq < a.nw)
      reinterpret_cast<uint32_t*>(dd.mask_out)[(uint64_t(z) * a.S + row) * a.nw + cq] = kb;
    mbar_wait(&bar[2], it & 1);
    tc_fence_after();
    T(2);

    // ---- softmax over this thread's 32 scores
    float v[32];
    {
      uint32_t r[32];
      TMEM_LD32(trow + j0, r);
      tmem_wait_ld();
#pragma unroll
      for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
    }
    // scores scaled into the log2 domain: p = 2^(s*scale*log2e - max)
    const float sl2 = a.scale * 1.4426950408889634f;
    const int lim = a.causal ? min(a.S, row + 1) : a.S;  // valid key columns of this row
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float t = j0 + j < lim ? v[j] * sl2 : -INFINITY;
      v[j] = t;
      mx = fmaxf(mx, t);
    }
    red[cq * 128 + row] = mx;
    // the previous head's probs store must have read sP before it is rewritten
    if (tid == 0) bulk_wait_read<0>();
    __syncthreads();
    mx = fmaxf(fmaxf(red[row], red[128 + row]), fmaxf(red[256 + row], red[384 + row]));
    float sum = 0.0f;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      v[j] = ex2_approx(v[j] - mx);  // ex2(-inf) = 0 for masked columns
      sum += v[j];
    }
    red[512 + cq * 128 + row] = sum;
    __syncthreads();
    const float inv =
        row < a.S ? 1.0f / ((red[512 + row] + red[640 + row]) + (red[768 + row] + red[896 + row])) : 0.0f;
    uint8_t* tileP = sP + (cq >> 1) * AT_TILE;
    const int g0 = (cq & 1) * 4;  // this quarter's first 16-byte granule in the tile row
    // P rounded to bf16 (the stored probs) = this quarter of the K-major A tile
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint4 w;
      w.x = pack_bf2(v[g * 8 + 0] * inv, v[g * 8 + 1] * inv);
      w.y = pack_bf2(v[g * 8 + 2] * inv, v[g * 8 + 3] * inv);
      w.z = pack_bf2(v[g * 8 + 4] * inv, v[g * 8 + 5] * inv);
      w.w = pack_bf2(v[g * 8 + 6] * inv, v[g * 8 + 7] * inv);
      *reinterpret_cast<uint4*>(tileP + sw128(row, g0 + g)) = w;
      v[g * 8 + 0] = bf_lo(w.x), v[g * 8 + 1] = bf_hi(w.x), v[g * 8 + 2] = bf_lo(w.y), v[g * 8 + 3] = bf_hi(w.y);
      v[g * 8 + 4] = bf_lo(w.z), v[g * 8 + 5] = bf_hi(w.z), v[g * 8 + 6] = bf_lo(w.w), v[g * 8 + 7] = bf_hi(w.w);
    }
    fence_proxy_async();
    __syncthreads();
    T(3);
    if (a.lse_out) {  // lse mode: no P store; the row's log-sum-exp instead
      if (cq == 0 && row < a.S) {
        const float tot = (red[512 + row] + red[640 + row]) + (red[768 + row] + red[896 + row]);
        a.lse_out[uint64_t(z) * a.S + row] = (mx + __log2f(tot)) * 0.6931471805599453f;
      }
    } else if (tid == 0) {
      // P is read only by this layer's backward: evict-first in L2
      tma_store_4d_evict_first(&m_probs, sP, 0, 0, z, 0);
      if (a.S > 64) tma_store_4d_evict_first(&m_probs, sP + AT_TILE, 64, 0, z, 0);
      bulk_commit();
    }
    uint8_t* sA = sP;
    if (dd.p > 0.0f) {
      // Pd = bf16(P * keep / (1-p)) into its own tile: the probs store keeps reading sP
      sA = sPd;
      uint8_t* tileD = sPd + (cq >> 1) * AT_TILE;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float pd[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int j = g * 8 + e;
          pd[e] = ((kb >> j) & 1u) ? v[j] * dd.scale : 0.0f;
        }
        uint4 w;
        w.x = pack_bf2(pd[0], pd[1]);
        w.y = pack_bf2(pd[2], pd[3]);
        w.z = pack_bf2(pd[4], pd[5]);
        w.w = pack_bf2(pd[6], pd[7]);
        *reinterpret_cast<uint4*>(tileD + sw128(row, g0 + g)) = w;
      }
      fence_proxy_async();
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      constexpr uint32_t id2 = umma_idesc(128, 64, true, false, true);
#pragma unroll
      for (int k = 0; k < 8; ++k)
          tc_mma<1>(tm + 128, umma_desc(smem_u32(sA) + (k >> 2) * AT_TILE + (k & 3) * 32, 16, 1024),
                  umma_desc(smem_u32(sV) + k * 2048, AT_TILE, 1024), id2, k ? 1u : 0u);
      tc_commit<1>(&bar[3]);
    }
    mbar_wait(&bar[3], it & 1);
    tc_fence_after();
    T(4);
    // ---- ctx row, this thread's 16 head-dim columns -> bf16 -> staging (this
    // head's Q tile, no longer needed) -> TMA store
    {
      uint32_t r[16];
      TMEM_LD16(trow + 128 + cq * 16, r);
      tmem_wait_ld();
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        uint4 w;
        w.x = pack_bf2(__uint_as_float(r[g * 8 + 0]), __uint_as_float(r[g * 8 + 1]));
        w.y = pack_bf2(__uint_as_float(r[g * 8 + 2]), __uint_as_float(r[g * 8 + 3]));
        w.z = pack_bf2(__uint_as_float(r[g * 8 + 4]), __uint_as_float(r[g * 8 + 5]));
        w.w = pack_bf2(__uint_as_float(r[g * 8 + 6]), __uint_as_float(r[g * 8 + 7]));
        *reinterpret_cast<uint4*>(sQ + sw128(row, cq * 2 + g)) = w;
      }
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tma_store_4d(&m_ctx, sQ, h * AT_D, 0, b, 0);
      bulk_commit();
    }
    T(5);
  }
  if (tid == 0) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free1<256>(tm);
  }
}

// ----------------------------------------------------------------- backward
__global__ void __launch_bounds__(AT_THREADS) k_attn_bwd(const __grid_constant__ CUtensorMap m_qkv,
                                                         const __grid_constant__ CUtensorMap m_probs,
                                                         const __grid_constant__ CUtensorMap m_dctx,
                                                         const __grid_constant__ CUtensorMap m_dqkv,
                                                         const AttnArgs a) {
  // Persistent over heads like the forward: buffer set it&1 holds this head's
  // inputs (Q, K, V, dO, P) while the next head's stream into the other set.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sIn = sm;                         // 2 x [Q, K, V, dO, P(2 tiles)]
  uint8_t* sS = sm + 12 * AT_TILE;           // 2 tiles: dS
  float* red = reinterpret_cast<float*>(sm + 14 * AT_TILE);  // [2 halves][128 rows]
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 256);   // load[2], mma1, mma2
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 4);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, hf = warp >> 2;
  const int row = q * 32 + lane;
  const int j0 = hf * 64;
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc1<512>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tm = *tslot;
  pdl_wait();
  pdl_trigger();
  DropCfg dd = a.d;
  drop_resolve(dd);

  auto issue_load = [&](int zz, int buf) {
    const int bb = zz / a.A, hh = zz % a.A;
    uint8_t* d = sIn + buf * 6 * AT_TILE;
    mbar_expect_tx(&bar[buf], (a.lse_in ? 4 : 6) * AT_TILE);
    tma_load_3(d, &m_qkv, &bar[buf], hh * AT_D, 0, bb);
    tma_load_3(d + AT_TILE, &m_qkv, &bar[buf], a.H + hh * AT_D, 0, bb);
    tma_load_3(d + 2 * AT_TILE, &m_qkv, &bar[buf], 2 * a.H + hh * AT_D, 0, bb);
    tma_load_3(d + 3 * AT_TILE, &m_dctx, &bar[buf], hh * AT_D, 0, bb);
    if (!a.lse_in) {  // lse mode: P is recomputed from a QK^T MMA, not loaded
      tma_load_3(d + 4 * AT_TILE, &m_probs, &bar[buf], 0, 0, zz);
      tma_load_3(d + 5 * AT_TILE, &m_probs, &bar[buf], 64, 0, zz);
    }
  };
  if (tid == 0 && int(blockIdx.x) < a.Z) issue_load(blockIdx.x, 0);
  int it = 0;
  for (int z = blockIdx.x; z < a.Z; z += gridDim.x, ++it) {
  const int buf = it & 1;
  const int b = z / a.A, h = z % a.A;
  uint8_t* sQ = sIn + buf * 6 * AT_TILE;
  uint8_t* sK = sQ + AT_TILE;
  uint8_t* sV = sQ + 2 * AT_TILE;
  uint8_t* sO = sQ + 3 * AT_TILE;   // dO
  uint8_t* sP = sQ + 4 * AT_TILE;   // 2 tiles: P, then Pd in place
  if (tid == 0) {
    const int zn = z + int(gridDim.x);
    if (zn < a.Z) {
      bulk_wait_read<0>();  // head it-1's output stores have read the other set
      issue_load(zn, buf ^ 1);
    }
    mbar_wait(&bar[buf], (it >> 1) & 1);
    tc_fence_after();
    // dPd = dO V^T  (A = dO K-major, B = V K-major: [key][dh])
    constexpr uint32_t id1 = umma_idesc(128, 128, true, false, false);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      tc_mma<1>(tm, umma_desc(smem_u32(sO) + k * 32, 16, 1024), umma_desc(smem_u32(sV) + k * 32, 16, 1024), id1,
                k ? 1u : 0u);
    if (a.lse_in) {  // S = Q K^T -> TMEM columns 256..383 (P recomputed from it and lse)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        tc_mma<1>(tm + 256, umma_desc(smem_u32(sQ) + k * 32, 16, 1024),
                  umma_desc(smem_u32(sK) + k * 32, 16, 1024), id1, k ? 1u : 0u);
    }
    tc_commit<1>(&bar[2]);
  }
  uint32_t kb[2];
  if (dd.mask_in) {  // the forward's saved keep bits (no Philox re-run)
    const uint32_t* mw = reinterpret_cast<const uint32_t*>(dd.mask_in) + (uint64_t(z) * a.S + row) * a.nw + 2 * hf;
    kb[0] = row < a.S && 2 * hf < a.nw ? mw[0] : 0xffffffffu;
    kb[1] = row < a.S && 2 * hf + 1 < a.nw ? mw[1] : 0xffffffffu;
  } else {
    keep_bits64(dd, (uint64_t(z) * a.S + row) * a.S, j0, a.S, kb);
  }
  const float sd = dd.p > 0.0f ? dd.scale : 1.0f;
  mbar_wait(&bar[2], it & 1);
  tc_fence_after();

  const uint32_t trow = tm + (uint32_t(q * 32) << 16) + j0;
  uint8_t* tileP = sP + hf * AT_TILE;
  uint8_t* tileS = sS + hf * AT_TILE;
  // pass 1: rowdot = sum_j P_j * dP_j (this half), combined through smem
  float dp[64];
  float rowdot = 0.0f;
  const float lse2 = (a.lse_in && row < a.S) ? a.lse_in[uint64_t(z) * a.S + row] * 1.4426950408889634f : 0.0f;
  const float sl2 = a.scale * 1.4426950408889634f;
  const int lim = row >= a.S ? 0 : a.causal ? min(a.S, row + 1) : a.S;
#pragma unroll
  for (int c = 0; c < 2; ++c) {
    uint32_t r[32];
    TMEM_LD32(trow + c * 32, r);
    if (a.lse_in) {  // P = 2^(s*scale*log2e - lse*log2e), rounded to bf16 into the P tile
      uint32_t rs[32];
      TMEM_LD32(trow + 256 + c * 32, rs);
      tmem_wait_ld();
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float pf[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int col = j0 + c * 32 + g * 8 + e;
          pf[e] = col < lim ? ex2_approx(__uint_as_float(rs[g * 8 + e]) * sl2 - lse2) : 0.0f;
        }
        uint4 w;
        w.x = pack_bf2(pf[0], pf[1]);
        w.y = pack_bf2(pf[2], pf[3]);
        w.z = pack_bf2(pf[4], pf[5]);
        w.w = pack_bf2(pf[6], pf[7]);
        *reinterpret_cast<uint4*>(tileP + sw128(row, c * 4 + g)) = w;
      }
    }
    tmem_wait_ld();
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint4 w = *reinterpret_cast<const uint4*>(tileP + sw128(row, c * 4 + g));
      const float p[8] = {bf_lo(w.x), bf_hi(w.x), bf_lo(w.y), bf_hi(w.y), bf_lo(w.z), bf_hi(w.z), bf_lo(w.w), bf_hi(w.w)};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int j = c * 32 + g * 8 + e;
        const bool keep = (kb[j >> 5] >> (j & 31)) & 1u;
        dp[j] = keep ? __uint_as_float(r[g * 8 + e]) * sd : 0.0f;
        rowdot += p[e] * dp[j];
      }
    }
  }
  red[hf * 128 + row] = rowdot;
  __syncthreads();
  rowdot = red[row] + red[128 + row];
  // pass 2: dS = P (dP - rowdot) scale -> sS; Pd -> sP (in place)
#pragma unroll
  for (int g = 0; g < 8; ++g) {
    uint8_t* pp = tileP + sw128(row, g);
    const uint4 w = *reinterpret_cast<const uint4*>(pp);
    const float p[8] = {bf_lo(w.x), bf_hi(w.x), bf_lo(w.y), bf_hi(w.y), bf_lo(w.z), bf_hi(w.z), bf_lo(w.w), bf_hi(w.w)};
    float ds[8], pd[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int j = g * 8 + e;
      const bool keep = (kb[j >> 5] >> (j & 31)) & 1u;
      pd[e] = keep ? p[e] * sd : 0.0f;
      ds[e] = p[e] * (dp[j] - rowdot) * a.scale;
    }
    uint4 o;
    o.x = pack_bf2(ds[0], ds[1]);
    o.y = pack_bf2(ds[2], ds[3]);
    o.z = pack_bf2(ds[4], ds[5]);
    o.w = pack_bf2(ds[6], ds[7]);
    *reinterpret_cast<uint4*>(tileS + sw128(row, g)) = o;
    if (dd.p > 0.0f) {
      o.x = pack_bf2(pd[0], pd[1]);
      o.y = pack_bf2(pd[2], pd[3]);
      o.z = pack_bf2(pd[4], pd[5]);
      o.w = pack_bf2(pd[6], pd[7]);
      *reinterpret_cast<uint4*>(pp) = o;
    }
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tc_fence_after();
    // M = 128 over two 64-wide MN chunks of a [K=128 rows][128 B] tile pair: LBO = tile
    constexpr uint32_t id_mm = umma_idesc(128, 64, true, true, true);   // A MN-major, B MN-major
    constexpr uint32_t id_km = umma_idesc(128, 64, true, false, true);  // A K-major, B MN-major
#pragma unroll
    for (int k = 0; k < 8; ++k)  // dV = Pd^T dO -> cols 128..191
      tc_mma<1>(tm + 128, umma_desc(smem_u32(sP) + k * 2048, AT_TILE, 1024),
                umma_desc(smem_u32(sO) + k * 2048, AT_TILE, 1024), id_mm, k ? 1u : 0u);
#pragma unroll
    for (int k = 0; k < 8; ++k)  // dQ = dS K -> cols 0..63
      tc_mma<1>(tm, umma_desc(smem_u32(sS) + (k >> 2) * AT_TILE + (k & 3) * 32, 16, 1024),
                umma_desc(smem_u32(sK) + k * 2048, AT_TILE, 1024), id_km, k ? 1u : 0u);
#pragma unroll
    for (int k = 0; k < 8; ++k)  // dK = dS^T Q -> cols 64..127
      tc_mma<1>(tm + 64, umma_desc(smem_u32(sS) + k * 2048, AT_TILE, 1024),
                umma_desc(smem_u32(sQ) + k * 2048, AT_TILE, 1024), id_mm, k ? 1u : 0u);
    tc_commit<1>(&bar[3]);
  }
  mbar_wait(&bar[3], it & 1);
  tc_fence_after();
  // dQ (query row), dK, dV (key row = TMEM lane): this thread's 32 head-dim
  // columns of each -> bf16 staging in sQ / sK / sV
  uint8_t* stage[3] = {sQ, sK, sV};
  const uint32_t col[3] = {0, 64, 128};
  const uint32_t tbase = tm + (uint32_t(q * 32) << 16) + hf * 32;
#pragma unroll
  for (int t = 0; t < 3; ++t) {
    uint32_t r[32];
    TMEM_LD32(tbase + col[t], r);
    tmem_wait_ld();
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      uint4 w;
      w.x = pack_bf2(__uint_as_float(r[g * 8 + 0]), __uint_as_float(r[g * 8 + 1]));
      w.y = pack_bf2(__uint_as_float(r[g * 8 + 2]), __uint_as_float(r[g * 8 + 3]));
      w.z = pack_bf2(__uint_as_float(r[g * 8 + 4]), __uint_as_float(r[g * 8 + 5]));
      w.w = pack_bf2(__uint_as_float(r[g * 8 + 6]), __uint_as_float(r[g * 8 + 7]));
      *reinterpret_cast<uint4*>(stage[t] + sw128(row, hf * 4 + g)) = w;
    }
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tma_store_4d(&m_dqkv, sQ, h * AT_D, 0, b, 0);
    tma_store_4d(&m_dqkv, sK, a.H + h * AT_D, 0, b, 0);
    tma_store_4d(&m_dqkv, sV, 2 * a.H + h * AT_D, 0, b, 0);
    bulk_commit();
  }
  tc_fence_before();
  __syncthreads();
  }
  if (tid == 0) bulk_wait_all();
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free1<512>(tm);
  }
}

// ------------------------------------------------------------------ host
constexpr int AT_FWD_SMEM = 1024 + 10 * AT_TILE + 4096 + 64;
constexpr int AT_BWD_SMEM = 1024 + 14 * AT_TILE + 1024 + 64;

bool attn_fused_ok(int dt, int64_t S, int64_t H, int64_t A, bool exact) {
  return !exact && dt == TCB_BF16 && A > 0 && H % A == 0 && H / A == AT_D && S >= 8 && S <= AT_S && S % 8 == 0;
}

// [rows=S per batch] x [cols] bf16 family -> 3-D map {cols, S, B}, box {64, 128}
static CUtensorMap seq_map(const void* p, int64_t cols, int64_t S, int64_t B) {
  return encode4(p, TCB_BF16, cols, S, B, 1, cols, S * cols, S * cols * B, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
}

void launch_attn_fwd(const void* qkv, void* ctx, void* probs, int64_t B, int64_t S, int64_t H, int64_t A, float scale,
                     int causal, const DropCfg& d, cudaStream_t s, void* trace, float* lse) {
  static std::once_flag once;
  std::call_once(once, [] {
    TCB_CUDA(cudaFuncSetAttribute(k_attn_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, AT_FWD_SMEM));
  });
  const CUtensorMap mq = seq_map(qkv, 3 * H, S, B);
  const CUtensorMap mc = seq_map(ctx, H, S, B);
  // lse mode: no probs tensor (the map is never used; point it at ctx)
  const CUtensorMap mp = lse ? mc : encode4(probs, TCB_BF16, S, S, B * A, 1, S, S * S, S * S * B * A, 64, 128,
                                            CU_TENSOR_MAP_SWIZZLE_128B);
  AttnArgs a{int(S), int(H), int(A), int(H / A), causal, int(B * A), static_cast<unsigned long long*>(trace), scale, d,
             lse, nullptr, lse ? int((S + 31) / 32) : 4};
  const int grid = int(B * A < kNumSMs ? B * A : kNumSMs);
  launch_k(k_attn_fwd, unsigned(grid), AT_FWD_THREADS, AT_FWD_SMEM, s, mq, mp, mc, a);
  TCB_CUDA(cudaGetLastError());
}

void launch_attn_bwd(const void* qkv, const void* probs, const void* dctx, void* dqkv, int64_t B, int64_t S, int64_t H,
                     int64_t A, float scale, int causal, const DropCfg& d, cudaStream_t s, const float* lse) {
  static std::once_flag once;
  std::call_once(once, [] {
    TCB_CUDA(cudaFuncSetAttribute(k_attn_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, AT_BWD_SMEM));
  });
  const CUtensorMap mq = seq_map(qkv, 3 * H, S, B);
  const CUtensorMap mo = seq_map(dctx, H, S, B);
  const CUtensorMap md = seq_map(dqkv, 3 * H, S, B);
  const CUtensorMap mp = lse ? mo : encode4(probs, TCB_BF16, S, S, B * A, 1, S, S * S, S * S * B * A, 64, 128,
                                            CU_TENSOR_MAP_SWIZZLE_128B);
  AttnArgs a{int(S), int(H), int(A), int(H / A), causal, int(B * A), nullptr, scale, d, nullptr, lse,
             lse ? int((S + 31) / 32) : 4};
  const int grid = int(B * A < kNumSMs ? B * A : kNumSMs);
  launch_k(k_attn_bwd, unsigned(grid), AT_THREADS, AT_BWD_SMEM, s, mq, mp, mo, md, a);
  TCB_CUDA(cudaGetLastError());
}

}  // namespace tcb
