// k_flash.cu -- fused attention for any sequence length (S % 8 == 0, head dim
// 64, bf16), tcgen05 + TMA, saving only the per-row log-sum-exp for the
// backward (attention lse=1; the S<=128 kernels in k_attention.cu store P).
//
// Forward: one CTA per (head z, 128-query tile).  For every 128-key tile j:
// S = Q K_j^T (tcgen05 -> TMEM), online softmax in the log2 domain (running
// max m and sum l per row; the 4 threads of a row combine through smem),
// dropout applied to the un-normalised p, O = alpha O + Pd V_j accumulated in
// TMEM (alpha = 2^(m_old - m_new) rescales O in TMEM between the MMAs).  At
// the end ctx = O / l (bf16, TMA store) and lse = (m + log2 l) ln 2.  With
// S <= 128 there is one key tile: K/V are single-buffered and the CTA fits
// twice per SM (occupancy), longer sequences double-buffer K/V.
//
// Backward (FlashAttention-2 order): one CTA per (head z, 128-key tile); for
// every query tile i: S = Q_i K^T and dPd = dO_i V^T (TMEM), P = 2^(S log2e
// scale - lse_i log2e) recomputed, D_i = rowsum(dO_i * O_i), dS = P (dP - D_i)
// scale, then dV += Pd^T dO_i, dK += dS^T Q_i (TMEM accumulators across i)
// and dQ_i = dS K (one tile: stored; several: f32 atomics into a workspace,
// converted to bf16 by a last kernel).
#include "common.cuh"
#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace tcb {

namespace {
constexpr int FA_D = 64;           // head dim (one SWIZZLE_128B row)
constexpr int FA_TILE = 16384;     // 128 rows x 128 B
constexpr int FA_FWD_THREADS = 512;
constexpr int FA_BWD_THREADS = 256;

struct FlashArgs {
  int S, H, A, Z, causal, nt;  // nt = ceil(S / 128)
  float scale;
  DropCfg d;
  int nw;                      // saved-mask words per query row (ceil(S / 32))
  float* lse;                  // [Z * S]
  float* dq;                   // backward, nt > 1: f32 [B*S, H] accumulator
};

__device__ __forceinline__ uint32_t sw128(int r, int g) { return uint32_t(r * 128 + ((g ^ (r & 7)) << 4)); }
__device__ __forceinline__ uint32_t pack_bf2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
__device__ __forceinline__ void ld3(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  tma_load_4d<1>(dst, map, smem_u32(bar), c0, c1, c2, 0);
}
#define TMEM_ST16(taddr, r)                                                                            \
  asm volatile(                                                                                        \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14," \
      "%15,%16};" ::"r"(taddr),                                                                        \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), \
      "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])                \
      : "memory")
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// keep bits of 32 keys c0 .. c0+31 (c0 % 8 == 0) of flat row base (0 beyond S)
__device__ __forceinline__ uint32_t keep32(const DropCfg& d, uint64_t base, int c0, int S) {
  uint32_t kb = 0xffffffffu;
  if (d.p <= 0.0f) return kb;
#pragma unroll
  for (int g = 0; g < 4; ++g)
    if (c0 + g * 8 < S) {
      const uint32_t b = dropout_bits8q(d, ((base + uint64_t(c0)) >> 3) + g);
      kb = (kb & ~(0xffu << (g * 8))) | (b << (g * 8));
    }
  return kb;
}
}  // namespace

// ------------------------------------------------------------------ forward
template <int NBUF>
__global__ void __launch_bounds__(FA_FWD_THREADS) k_flash_fwd(const __grid_constant__ CUtensorMap m_qkv,
                                                              const __grid_constant__ CUtensorMap m_ctx,
                                                              const FlashArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sK = sm + FA_TILE;                    // NBUF tiles
  uint8_t* sV = sK + NBUF * FA_TILE;             // NBUF tiles
  uint8_t* sP = sV + NBUF * FA_TILE;             // 2 tiles: keys 0-63, 64-127 (dropout applied)
  float* red = reinterpret_cast<float*>(sP + 2 * FA_TILE);  // [2][4][128]
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 1024);  // q, kv[NBUF], s, pv
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 8);
  uint64_t* bq = &bar[0];
  uint64_t* bkv = &bar[1];
  uint64_t* bs = &bar[1 + NBUF];
  uint64_t* bpv = &bar[2 + NBUF];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, cq = warp >> 2;
  const int row = q * 32 + lane;
  const int z = blockIdx.x / a.nt, qt = blockIdx.x % a.nt;
  const int b = z / a.A, h = z % a.A;
  const int qi = qt * 128 + row;  // query row in the sequence
  const int nkv = a.causal ? qt + 1 : a.nt;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&m_qkv)) : "memory");
    for (int i = 0; i < 3 + NBUF; ++i) mbar_init(&bar[i], 1);
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

  auto load_kv = [&](int j, int buf) {
    mbar_expect_tx(&bkv[buf], 2 * FA_TILE);
    ld3(sK + buf * FA_TILE, &m_qkv, &bkv[buf], a.H + h * FA_D, j * 128, b);
    ld3(sV + buf * FA_TILE, &m_qkv, &bkv[buf], 2 * a.H + h * FA_D, j * 128, b);
  };
  if (tid == 0) {
    mbar_expect_tx(bq, FA_TILE);
    ld3(sQ, &m_qkv, bq, h * FA_D, qt * 128, b);
    for (int j = 0; j < NBUF && j < nkv; ++j) load_kv(j, j);
  }
  const uint32_t trow = tm + (uint32_t(q * 32) << 16);
  const float sl2 = a.scale * 1.4426950408889634f;
  const bool row_ok = qi < a.S;
  const int lim = !row_ok ? 0 : a.causal ? min(a.S, qi + 1) : a.S;  // valid key columns
  const uint64_t mbase = (uint64_t(z) * a.S + uint64_t(qi)) * uint64_t(a.S);
  float m = -INFINITY, l = 0.0f;

  for (int j = 0; j < nkv; ++j) {
    const int buf = NBUF == 1 ? 0 : (j & 1);
    if (tid == 0) {
      if (j == 0) mbar_wait(bq, 0);
      if (NBUF == 1 && j > 0) {  // single K/V buffer: reload once PV(j-1) has read V
        mbar_wait(bpv, (j - 1) & 1);
        load_kv(j, 0);
      }
      mbar_wait(&bkv[buf], NBUF == 1 ? (j & 1) : ((j >> 1) & 1));
      tc_fence_after();
      constexpr uint32_t id1 = umma_idesc(128, 128, true, false, false);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        tc_mma<1>(tm, umma_desc(smem_u32(sQ) + k * 32, 16, 1024),
                  umma_desc(smem_u32(sK + buf * FA_TILE) + k * 32, 16, 1024), id1, k ? 1u : 0u);
      tc_commit<1>(bs);
      if (NBUF == 2 && j > 0 && j + 1 < nkv) {  // buffer of tile j-1 -> tile j+1 once PV(j-1) is done
        mbar_wait(bpv, (j - 1) & 1);
        load_kv(j + 1, buf ^ 1);
      }
    }
    const int c0 = j * 128 + cq * 32;  // this thread's first key column
    const uint32_t kb = row_ok ? keep32(dd, mbase, c0, a.S) : 0u;
    if (dd.mask_out && row_ok && (c0 >> 5) < a.nw)
      reinterpret_cast<uint32_t*>(dd.mask_out)[(uint64_t(z) * a.S + qi) * a.nw + (c0 >> 5)] = kb;
    mbar_wait(bs, j & 1);
    tc_fence_after();
    float v[32];
    {
      uint32_t r[32];
      TMEM_LD32(trow + cq * 32, r);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 32; ++e) v[e] = c0 + e < lim ? __uint_as_float(r[e]) * sl2 : -INFINITY;
    }
    float mx = -INFINITY;
#pragma unroll
    for (int e = 0; e < 32; ++e) mx = fmaxf(mx, v[e]);
    red[cq * 128 + row] = mx;
    __syncthreads();
    mx = fmaxf(fmaxf(red[row], red[128 + row]), fmaxf(red[256 + row], red[384 + row]));
    const float mn = fmaxf(m, mx);
    const float mu = mn == -INFINITY ? 0.0f : mn;  // fully masked so far: no shift
    const float alpha = ex2_approx(m - mu);        // 0 on the first tile (m = -inf)
    float qs = 0.0f;
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      v[e] = ex2_approx(v[e] - mu);
      qs += v[e];
    }
    red[512 + cq * 128 + row] = qs;
    // PV(j-1) must be done before P is rewritten and O rescaled
    if (j > 0) {
      mbar_wait(bpv, (j - 1) & 1);
      tc_fence_after();
    }
    __syncthreads();
    l = l * alpha + ((red[512 + row] + red[640 + row]) + (red[768 + row] + red[896 + row]));
    m = mn;
    uint8_t* tileP = sP + (cq >> 1) * FA_TILE;
    const int g0 = (cq & 1) * 4;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      float pd[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int jj = g * 8 + e;
        pd[e] = ((kb >> jj) & 1u) ? v[jj] * dd.scale : 0.0f;
      }
      uint4 w;
      w.x = pack_bf2(pd[0], pd[1]);
      w.y = pack_bf2(pd[2], pd[3]);
      w.z = pack_bf2(pd[4], pd[5]);
      w.w = pack_bf2(pd[6], pd[7]);
      *reinterpret_cast<uint4*>(tileP + sw128(row, g0 + g)) = w;
    }
    // O *= alpha (this thread's 16 of the row's 64 columns); tcgen05.ld/st are
    // warp-collective, so the skip test must be warp-uniform
    if (j > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
      uint32_t r[16];
      TMEM_LD16(trow + 128 + cq * 16, r);
      tmem_wait_ld();
#pragma unroll
      for (int e = 0; e < 16; ++e) r[e] = __float_as_uint(__uint_as_float(r[e]) * alpha);
      TMEM_ST16(trow + 128 + cq * 16, r);
      tmem_wait_st();
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      constexpr uint32_t id2 = umma_idesc(128, 64, true, false, true);
#pragma unroll
      for (int k = 0; k < 8; ++k)
        tc_mma<1>(tm + 128, umma_desc(smem_u32(sP) + (k >> 2) * FA_TILE + (k & 3) * 32, 16, 1024),
                  umma_desc(smem_u32(sV + buf * FA_TILE) + k * 2048, FA_TILE, 1024), id2,
                  (j > 0 || k > 0) ? 1u : 0u);
      tc_commit<1>(bpv);
    }
  }
  mbar_wait(bpv, (nkv - 1) & 1);
  tc_fence_after();
  {  // ctx = O / l -> bf16 -> staging in sQ -> TMA store (rows >= S clipped)
    const float inv = row_ok && l > 0.0f ? 1.0f / l : 0.0f;
    uint32_t r[16];
    TMEM_LD16(trow + 128 + cq * 16, r);
    tmem_wait_ld();
#pragma unroll
    for (int g = 0; g < 2; ++g) {
      uint4 w;
      w.x = pack_bf2(__uint_as_float(r[g * 8 + 0]) * inv, __uint_as_float(r[g * 8 + 1]) * inv);
      w.y = pack_bf2(__uint_as_float(r[g * 8 + 2]) * inv, __uint_as_float(r[g * 8 + 3]) * inv);
      w.z = pack_bf2(__uint_as_float(r[g * 8 + 4]) * inv, __uint_as_float(r[g * 8 + 5]) * inv);
      w.w = pack_bf2(__uint_as_float(r[g * 8 + 6]) * inv, __uint_as_float(r[g * 8 + 7]) * inv);
      *reinterpret_cast<uint4*>(sQ + sw128(row, cq * 2 + g)) = w;
    }
  }
  if (cq == 0 && row_ok) a.lse[uint64_t(z) * a.S + qi] = (m + __log2f(l)) * 0.6931471805599453f;
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tma_store_4d(&m_ctx, sQ, h * FA_D, qt * 128, b, 0);
    bulk_commit();
    bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free1<256>(tm);
  }
}

// ----------------------------------------------------------------- backward
__global__ void __launch_bounds__(FA_BWD_THREADS) k_flash_bwd(const __grid_constant__ CUtensorMap m_qkv,
                                                              const __grid_constant__ CUtensorMap m_ctx,
                                                              const __grid_constant__ CUtensorMap m_dctx,
                                                              const __grid_constant__ CUtensorMap m_dqkv,
                                                              const FlashArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm;
  uint8_t* sV = sm + FA_TILE;
  uint8_t* sIn = sm + 2 * FA_TILE;      // 2 x [Q, dO, O]
  uint8_t* sS = sIn + 6 * FA_TILE;      // 2 tiles: dS [q rows x keys]
  uint8_t* sPd = sS + 2 * FA_TILE;      // 2 tiles: Pd
  float* red = reinterpret_cast<float*>(sPd + 2 * FA_TILE);  // [2][128]
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + 256);    // kv, in[2], s, mm
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 8);
  uint64_t* bkv = &bar[0];
  uint64_t* bin = &bar[1];
  uint64_t* bs = &bar[3];
  uint64_t* bmm = &bar[4];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = warp & 3, hf = warp >> 2;
  const int row = q * 32 + lane;
  const int z = blockIdx.x / a.nt, kt = blockIdx.x % a.nt;
  const int b = z / a.A, h = z % a.A;
  const int qlo = a.causal ? kt : 0;
  const int nq = a.nt - qlo;
  if (tid == 0) {
    for (int i = 0; i < 5; ++i) mbar_init(&bar[i], 1);
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
  auto load_in = [&](int i, int buf) {
    const int qq = qlo + i;
    uint8_t* d = sIn + buf * 3 * FA_TILE;
    mbar_expect_tx(&bin[buf], 3 * FA_TILE);
    ld3(d, &m_qkv, &bin[buf], h * FA_D, qq * 128, b);
    ld3(d + FA_TILE, &m_dctx, &bin[buf], h * FA_D, qq * 128, b);
    ld3(d + 2 * FA_TILE, &m_ctx, &bin[buf], h * FA_D, qq * 128, b);
  };
  if (tid == 0) {
    mbar_expect_tx(bkv, 2 * FA_TILE);
    ld3(sK, &m_qkv, bkv, a.H + h * FA_D, kt * 128, b);
    ld3(sV, &m_qkv, bkv, 2 * a.H + h * FA_D, kt * 128, b);
    load_in(0, 0);
    if (nq > 1) load_in(1, 1);
  }
  const float sl2 = a.scale * 1.4426950408889634f;
  const float sd = dd.p > 0.0f ? dd.scale : 1.0f;
  const int kr = kt * 128 + hf * 64;  // this thread's first key column
  const uint32_t tS = tm, tP = tm + 128, tdV = tm + 256, tdK = tm + 320, tdQ = tm + 384;
  const uint32_t lrow = uint32_t(q * 32) << 16;

  for (int i = 0; i < nq; ++i) {
    const int buf = i & 1;
    const int qt = qlo + i;
    const int qi = qt * 128 + row;
    const bool row_ok = qi < a.S;
    uint8_t* sQ = sIn + buf * 3 * FA_TILE;
    uint8_t* sdO = sQ + FA_TILE;
    uint8_t* sO = sQ + 2 * FA_TILE;
    if (tid == 0) {
      if (i == 0) mbar_wait(bkv, 0);
      mbar_wait(&bin[buf], (i >> 1) & 1);
      tc_fence_after();
      constexpr uint32_t id1 = umma_idesc(128, 128, true, false, false);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        tc_mma<1>(tS, umma_desc(smem_u32(sQ) + k * 32, 16, 1024), umma_desc(smem_u32(sK) + k * 32, 16, 1024), id1,
                  k ? 1u : 0u);
#pragma unroll
      for (int k = 0; k < 4; ++k)
        tc_mma<1>(tP, umma_desc(smem_u32(sdO) + k * 32, 16, 1024), umma_desc(smem_u32(sV) + k * 32, 16, 1024),
                  id1, k ? 1u : 0u);
      tc_commit<1>(bs);
    }
    // meanwhile: D_i = rowsum(dO * O) (this thread's half of the head dim),
    // lse_i, and the keep bits of this thread's 64 keys
    if (i == 0) mbar_wait(&bin[0], 0);
    else mbar_wait(&bin[buf], (i >> 1) & 1);
    float dsum = 0.0f;
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      const uint4 x = *reinterpret_cast<const uint4*>(sdO + sw128(row, hf * 4 + g));
      const uint4 o = *reinterpret_cast<const uint4*>(sO + sw128(row, hf * 4 + g));
      dsum += bf_lo(x.x) * bf_lo(o.x) + bf_hi(x.x) * bf_hi(o.x) + bf_lo(x.y) * bf_lo(o.y) + bf_hi(x.y) * bf_hi(o.y) +
              bf_lo(x.z) * bf_lo(o.z) + bf_hi(x.z) * bf_hi(o.z) + bf_lo(x.w) * bf_lo(o.w) + bf_hi(x.w) * bf_hi(o.w);
    }
    const float lse2 = row_ok ? a.lse[uint64_t(z) * a.S + qi] * 1.4426950408889634f : 0.0f;
    const uint64_t mbase = (uint64_t(z) * a.S + uint64_t(qi)) * uint64_t(a.S);
    uint32_t kb[2] = {0u, 0u};
    if (row_ok) {
      if (dd.mask_in) {
        const uint32_t* mw = reinterpret_cast<const uint32_t*>(dd.mask_in) + (uint64_t(z) * a.S + qi) * a.nw;
        kb[0] = (kr >> 5) < a.nw ? mw[kr >> 5] : 0u;
        kb[1] = ((kr >> 5) + 1) < a.nw ? mw[(kr >> 5) + 1] : 0u;
      } else {
        kb[0] = keep32(dd, mbase, kr, a.S);
        kb[1] = keep32(dd, mbase, kr + 32, a.S);
      }
    }
    const int lim = !row_ok ? 0 : a.causal ? min(a.S, qi + 1) : a.S;
    red[hf * 128 + row] = dsum;
    // the previous tile's MMAs read sS / sPd: done before they are rewritten
    if (i > 0) {
      mbar_wait(bmm, (i - 1) & 1);
      tc_fence_after();
    }
    __syncthreads();
    const float D = red[row] + red[128 + row];
    mbar_wait(bs, i & 1);
    tc_fence_after();
    uint8_t* tileS = sS + hf * FA_TILE;
    uint8_t* tileP = sPd + hf * FA_TILE;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t rs[32], rp[32];
      TMEM_LD32(tS + lrow + hf * 64 + c * 32, rs);
      TMEM_LD32(tP + lrow + hf * 64 + c * 32, rp);
      tmem_wait_ld();
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        float ds[8], pd[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int jj = c * 32 + g * 8 + e;
          const bool valid = kr + jj < lim;
          const float p = valid ? ex2_approx(__uint_as_float(rs[g * 8 + e]) * sl2 - lse2) : 0.0f;
          const bool keep = (kb[jj >> 5] >> (jj & 31)) & 1u;
          const float dp = keep ? __uint_as_float(rp[g * 8 + e]) * sd : 0.0f;
          ds[e] = p * (dp - D) * a.scale;
          pd[e] = keep ? p * sd : 0.0f;
        }
        uint4 w;
        w.x = pack_bf2(ds[0], ds[1]);
        w.y = pack_bf2(ds[2], ds[3]);
        w.z = pack_bf2(ds[4], ds[5]);
        w.w = pack_bf2(ds[6], ds[7]);
        *reinterpret_cast<uint4*>(tileS + sw128(row, c * 4 + g)) = w;
        w.x = pack_bf2(pd[0], pd[1]);
        w.y = pack_bf2(pd[2], pd[3]);
        w.z = pack_bf2(pd[4], pd[5]);
        w.w = pack_bf2(pd[6], pd[7]);
        *reinterpret_cast<uint4*>(tileP + sw128(row, c * 4 + g)) = w;
      }
    }
    fence_proxy_async();
    tc_fence_before();
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      constexpr uint32_t id_mm = umma_idesc(128, 64, true, true, true);   // A MN-major, B MN-major
      constexpr uint32_t id_km = umma_idesc(128, 64, true, false, true);  // A K-major, B MN-major
#pragma unroll
      for (int k = 0; k < 8; ++k)  // dV += Pd^T dO
        tc_mma<1>(tdV, umma_desc(smem_u32(sPd) + k * 2048, FA_TILE, 1024),
                  umma_desc(smem_u32(sdO) + k * 2048, FA_TILE, 1024), id_mm, (i > 0 || k > 0) ? 1u : 0u);
#pragma unroll
      for (int k = 0; k < 8; ++k)  // dK += dS^T Q
        tc_mma<1>(tdK, umma_desc(smem_u32(sS) + k * 2048, FA_TILE, 1024),
                  umma_desc(smem_u32(sQ) + k * 2048, FA_TILE, 1024), id_mm, (i > 0 || k > 0) ? 1u : 0u);
#pragma unroll
      for (int k = 0; k < 8; ++k)  // dQ = dS K
        tc_mma<1>(tdQ, umma_desc(smem_u32(sS) + (k >> 2) * FA_TILE + (k & 3) * 32, 16, 1024),
                  umma_desc(smem_u32(sK) + k * 2048, FA_TILE, 1024), id_km, k ? 1u : 0u);
      tc_commit<1>(bmm);
    }
    mbar_wait(bmm, i & 1);
    tc_fence_after();
    {  // dQ rows of this query tile: this thread's 32 of 64 columns
      uint32_t r[32];
      TMEM_LD32(tdQ + lrow + hf * 32, r);
      tmem_wait_ld();
      if (a.nt == 1) {  // the only key tile: dQ is final -> bf16 staging in sQ -> TMA store
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint4 w;
          w.x = pack_bf2(__uint_as_float(r[g * 8 + 0]), __uint_as_float(r[g * 8 + 1]));
          w.y = pack_bf2(__uint_as_float(r[g * 8 + 2]), __uint_as_float(r[g * 8 + 3]));
          w.z = pack_bf2(__uint_as_float(r[g * 8 + 4]), __uint_as_float(r[g * 8 + 5]));
          w.w = pack_bf2(__uint_as_float(r[g * 8 + 6]), __uint_as_float(r[g * 8 + 7]));
          *reinterpret_cast<uint4*>(sQ + sw128(row, hf * 4 + g)) = w;
        }
      } else if (row_ok) {
        float* dst = a.dq + (uint64_t(b) * a.S + qi) * a.H + h * FA_D + hf * 32;
#pragma unroll
        for (int e = 0; e < 32; e += 4)
          atomicAdd(reinterpret_cast<float4*>(dst + e),
                    make_float4(__uint_as_float(r[e]), __uint_as_float(r[e + 1]), __uint_as_float(r[e + 2]),
                                __uint_as_float(r[e + 3])));
      }
    }
    if (a.nt == 1) {
      fence_proxy_async();
      __syncthreads();
      if (tid == 0) {
        tma_store_4d(&m_dqkv, sQ, h * FA_D, qt * 128, b, 0);
        bulk_commit();
      }
    }
    __syncthreads();
    if (tid == 0 && i + 2 < nq) {  // this buffer's tiles are consumed: prefetch tile i+2
      bulk_wait_read<0>();
      load_in(i + 2, buf);
    }
  }
  // dK, dV (key row = TMEM lane): bf16 -> staging in sK / sV -> TMA store
  {
    uint8_t* stage[2] = {sK, sV};
    const uint32_t col[2] = {320, 256};
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      uint32_t r[32];
      TMEM_LD32(tm + lrow + col[t] + hf * 32, r);
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
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  if (tid == 0) {
    tma_store_4d(&m_dqkv, sK, a.H + h * FA_D, kt * 128, b, 0);
    tma_store_4d(&m_dqkv, sV, 2 * a.H + h * FA_D, kt * 128, b, 0);
    bulk_commit();
    bulk_wait_all();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_free1<512>(tm);
  }
}

// dQ accumulator (f32 [B*S, H]) -> the Q columns of dqkv (bf16 [B*S, 3H])
__global__ void k_flash_dq_store(const float* __restrict__ dq, __nv_bfloat16* __restrict__ dqkv, int64_t rows,
                                 int H) {
  TCB_PDL_ENTRY();
  const int64_t n4 = rows * H / 4;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = reinterpret_cast<const float4*>(dq)[i];
    const int64_t e = i * 4, r = e / H, c = e % H;
    uint2 w;
    w.x = pack_bf2(v.x, v.y);
    w.y = pack_bf2(v.z, v.w);
    *reinterpret_cast<uint2*>(dqkv + r * 3 * H + c) = w;
  }
}

// ------------------------------------------------------------------ host
static CUtensorMap fa_map(const void* p, int64_t cols, int64_t S, int64_t B) {
  return encode4(p, TCB_BF16, cols, S, B, 1, cols, S * cols, S * cols * B, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
}
constexpr int fa_fwd_smem(int nbuf) { return 1024 + (1 + 2 * nbuf + 2) * FA_TILE + 4096 + 128; }
constexpr int FA_BWD_SMEM = 1024 + 12 * FA_TILE + 1024 + 128;

bool flash_ok(int dt, int64_t S, int64_t H, int64_t A) {
  return dt == TCB_BF16 && A > 0 && H % A == 0 && H / A == FA_D && S >= 8 && S % 8 == 0 && S <= 16384;
}

void launch_flash_fwd(const void* qkv, void* ctx, float* lse, int64_t B, int64_t S, int64_t H, int64_t A,
                      float scale, int causal, const DropCfg& d, cudaStream_t s) {
  const int nt = int((S + 127) / 128);
  FlashArgs a{int(S), int(H), int(A), int(B * A), causal, nt, scale, d, int((S + 31) / 32), lse, nullptr};
  const CUtensorMap mq = fa_map(qkv, 3 * H, S, B), mc = fa_map(ctx, H, S, B);
  const unsigned grid = unsigned(B * A * nt);
  if (nt == 1) {
    static std::once_flag once;
    std::call_once(once, [] {
      TCB_CUDA(cudaFuncSetAttribute(k_flash_fwd<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, fa_fwd_smem(1)));
    });
    launch_k(k_flash_fwd<1>, grid, FA_FWD_THREADS, fa_fwd_smem(1), s, mq, mc, a);
  } else {
    static std::once_flag once;
    std::call_once(once, [] {
      TCB_CUDA(cudaFuncSetAttribute(k_flash_fwd<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, fa_fwd_smem(2)));
    });
    launch_k(k_flash_fwd<2>, grid, FA_FWD_THREADS, fa_fwd_smem(2), s, mq, mc, a);
  }
}

void launch_flash_bwd(const void* qkv, const void* ctx, const float* lse, const void* dctx, void* dqkv,
                      float* dq_ws, int64_t B, int64_t S, int64_t H, int64_t A, float scale, int causal,
                      const DropCfg& d, cudaStream_t s) {
  static std::once_flag once;
  std::call_once(once, [] {
    TCB_CUDA(cudaFuncSetAttribute(k_flash_bwd, cudaFuncAttributeMaxDynamicSharedMemorySize, FA_BWD_SMEM));
  });
  const int nt = int((S + 127) / 128);
  FlashArgs a{int(S), int(H), int(A), int(B * A), causal, nt, scale, d, int((S + 31) / 32),
              const_cast<float*>(lse), dq_ws};
  const CUtensorMap mq = fa_map(qkv, 3 * H, S, B), mc = fa_map(ctx, H, S, B), mo = fa_map(dctx, H, S, B),
                    md = fa_map(dqkv, 3 * H, S, B);
  if (nt > 1) TCB_CUDA(cudaMemsetAsync(dq_ws, 0, size_t(B * S * H) * sizeof(float), s));
  launch_k(k_flash_bwd, unsigned(B * A * nt), FA_BWD_THREADS, FA_BWD_SMEM, s, mq, mc, mo, md, a);
  if (nt > 1)
    launch_k(k_flash_dq_store, unsigned(grid_for(B * S * H / 4, 256)), 256, 0, s, (const float*)dq_ws,
             (__nv_bfloat16*)dqkv, int64_t(B * S), int(H));
}

}  // namespace tcb
