// k_gemm_tc.cu -- bf16/f16 tensor-core GEMM for sm_100a: tcgen05.mma with the
// accumulator in TMEM, operands staged by TMA (SWIZZLE_128B), warp-specialised,
// persistent, optionally on a CTA pair (cta_group::2).
//
//   warp 0      TMA producer (one lane): A/B k-blocks into a STAGES-deep smem
//               ring, mbarrier full/empty handshake
//   warp 1      MMA issuer (one lane, leader CTA only): tcgen05.mma kind::f16,
//               (128*CG) x BN x 16 per instruction, fp32 accumulate in TMEM;
//               tcgen05.commit frees smem stages / publishes finished tiles
//   warp 2      TMEM allocator (2 x BN columns: double-buffered accumulator)
//   warps 4-11  epilogue: tcgen05.ld 32x32b.x32 -> alpha, bias, act'(aux),
//               pre-activation, act -> bf16/f32 into a swizzled smem box ->
//               TMA store (cp.async.bulk.tensor, bulk_group); the act'(aux)
//               operand arrives by TMA too, one chunk ahead
//
// CG = 2: a cluster of two CTAs on one TPC computes a 256 x BN tile with
// M=256 MMAs issued by the leader.  Each CTA loads its own 128 rows of A and
// half (BN/2 rows) of B, so every byte a CTA stages feeds twice the MMA work of
// the 1-CTA kernel (smem/L2 traffic per FLOP halves).  Both CTAs' TMA bytes
// land on the leader's full barrier; MMA commits are multicast to both CTAs;
// both epilogues release the accumulator on the leader's tmem-empty barrier.
//
// Operands may be K-major or MN-major (A: ta, B: tb), which absorbs the
// reference's `transpose` ops into the TMA/UMMA descriptors.
// Batched problems (attention heads, batch_matmul) use 4-D tensor maps
// {inner, outer, z2, z1}, so every batch gets exact zero-filled tails.
#include "gemm.cuh"
#include "tc_ptx.cuh"

namespace tcb {

constexpr int TC_BM = 128;  // accumulator rows per CTA
constexpr int TC_BK = 64;   // 64 bf16 = 128 B = one SWIZZLE_128B atom row
// epilogue warps per CTA by launch class (alternating whole-step A/Bs decide;
// tools/probe_gemm.py in isolation for the per-kernel numbers): 12 for plain /
// bias / f32 stores (step 4.92 -> 4.87 ms vs 8 over 6 rounds, though 8 is a
// little faster in isolation: plain 21.7 vs 22.8 us; both beat 16), 12 for the
// GELU forward epilogues (27.7 vs 28.3 us at 16), 16 (4 per TMEM lane quarter)
// for act'(aux) (24.9 us; slower at 12 and 8)
constexpr int TC_EPI_WARPS = 16;                      // the default (heaviest) count
#ifndef TC_EPW_LIGHT
#define TC_EPW_LIGHT 12
#endif
#ifndef TC_EPW_HEAVY
#define TC_EPW_HEAVY 12
#endif
#ifndef TC_EPW_AUX
#define TC_EPW_AUX 16
#endif
template <int EPW>
constexpr int tc_threads() { return 128 + 32 * EPW; }  // warps 0-3: TMA, MMA, TMEM, spare
constexpr int TC_EW = 16;                             // epilogue chunk width (columns)
constexpr int TC_SLOT = 32 * TC_EW * 4;               // per-warp output slot: f32 box or (y, u) 16-bit boxes
// output staging slots per warp: one (the operand ring gets the smem: +1 stage);
// the act'(aux) kernels, epilogue-bound, keep two so stores overlap
template <bool AUX>
constexpr int out_ring() { return AUX ? 2 : 1; }

template <int BN, int CG, bool AUX, int EPW = TC_EPI_WARPS>
struct TcCfg {
  static constexpr int B_ROWS = BN / CG;  // B rows (N) staged by each CTA
  // MN-major B arrives in 64-column boxes; a 96-row half (BN=192 pair) takes two,
  // the second over-fetching 32 columns the MMA never reads
  static constexpr int B_CHUNKS = (B_ROWS + 63) / 64;
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;
  static constexpr int B_BYTES = B_CHUNKS * 64 * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int EPI_BYTES =
      EPW * out_ring<AUX>() * TC_SLOT;
  static constexpr int BIAS_BYTES = EPW * ((BN / TC_EW + EPW / 4 - 1) / (EPW / 4)) * TC_EW * 4;
  static constexpr int BAR_BYTES = 1024;
  static constexpr int BUDGET = 227 * 1024 - 1024 - BAR_BYTES - EPI_BYTES - BIAS_BYTES;
  static constexpr int STAGES = BUDGET / STAGE_BYTES > 8 ? 8 : BUDGET / STAGE_BYTES;
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;
  static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + BIAS_BYTES + BAR_BYTES;
  static_assert(STAGES >= 2, "smem budget");
  static_assert(CG == 1 || (BN / 2) % 16 == 0, "cta pair splits B");
};

struct TcProb {
  int64_t M, N, K, Z, Z2;
  int ta, tb;
  int m_blocks, n_blocks, k_blocks;  // m_blocks counts (128*CG)-row blocks
  int64_t num_tiles;
  int kps;  // k-blocks per unit (a K slice with wsplit > 1, else the whole K)
  // > 1: the problem's K is cut into wsplit slices run as separate units; unit
  // (s, tile) accumulates k-blocks [s*kps, +kps) and stores its f32 partial tile
  // to slice s of a [wsplit][M][N] workspace (C map Z2 = wsplit), which a fixed-
  // order reduction kernel sums afterwards (deterministic)
  int wsplit;
  uint32_t idesc;
  // epilogue
  void* c;
  int64_t ldc, c_s1, c_s2;
  int c_dtype;
  float alpha;
  const void* bias;
  int bias_dtype;
  int act, dact;
  const void* aux;
  int aux_dtype;
  void* aux_out;
  int save_grad;  // aux_out = act'(pre-activation)
  int tma_epi;   // 1: smem + TMA-store epilogue (tensor maps valid); 0: direct stores
  int generic_epi;  // 1: never a compile-time epilogue variant (tests)
  int c_vec_ok;  // direct path: 16-byte aligned rows
};
// One launch runs one or two GEMM problems with the same tile shape (a
// "grouped" launch: the backward's data-gradient and weight-gradient GEMMs of a
// linear share dY and run side by side, filling the SMs the small weight
// gradient leaves idle).  Units [0, pr[0].num_tiles) belong to problem 0.
struct TcParams {
  TcProb pr[2];
  int nprob;
  int64_t num_units;
  // optional static schedule: cluster c runs units sched[c], sched[c + n_cl],
  // ... up to the first -1 (longest-processing-time balanced on the host);
  // without it cluster c runs units c, c + n_cl, ...
  const int* sched;
  int sched_rounds;
  unsigned long long* trace;  // optional per-CTA timeline (tools/probe_gemm.py --trace)
};
__device__ __forceinline__ int64_t unit_at(const TcParams& P, int64_t cl, int64_t ncl, int64_t i) {
  if (P.sched) return i < P.sched_rounds ? int64_t(__ldg(P.sched + i * ncl + cl)) : -1;
  const int64_t u = cl + i * ncl;
  return u < P.num_units ? u : -1;
}
__device__ __forceinline__ int unit_prob(const TcParams& P, int64_t u) {
  return (P.nprob > 1 && u >= P.pr[0].num_tiles) ? 1 : 0;
}
// compile-time epilogue variants (see finish_fast in the kernel)
enum EpiKind { EK_GENERIC = 0, EK_PLAIN = 1, EK_BIAS = 2, EK_GELU_SAVE = 3, EK_DERIV = 4, EK_F32 = 5 };
template <bool AUX>
__device__ __forceinline__ int epi_kind(const TcProb& Q) {
  if (!Q.tma_epi || Q.alpha != 1.0f || Q.generic_epi) return EK_GENERIC;
  if (Q.c_dtype == TCB_F32)  // weight gradients (and their K-slice partials)
    return (!Q.bias && Q.act == ACT_NONE && Q.dact == ACT_NONE && !Q.aux_out) ? EK_F32 : EK_GENERIC;
  if (Q.c_dtype != TCB_BF16) return EK_GENERIC;
  if (Q.dact != ACT_NONE)
    return (AUX && Q.dact == ACT_DERIV && Q.aux_dtype == TCB_BF16 && !Q.bias && Q.act == ACT_NONE && !Q.aux_out)
               ? EK_DERIV
               : EK_GENERIC;
  if (Q.save_grad) return (Q.act == ACT_GELU && Q.bias && Q.aux_out) ? EK_GELU_SAVE : EK_GENERIC;
  if (Q.act != ACT_NONE || Q.aux_out) return EK_GENERIC;
  return Q.bias ? EK_BIAS : EK_PLAIN;
}


__device__ __forceinline__ float ld_e(const void* p, int dt, int64_t i) {
  if (dt == TCB_F32) return static_cast<const float*>(p)[i];
  if (dt == TCB_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  return __half2float(static_cast<const __half*>(p)[i]);
}

__device__ __forceinline__ void decode_tile(const TcProb& P, int64_t t, int& z, int& mb, int& nb) {
  const int64_t per_z = int64_t(P.m_blocks) * P.n_blocks;
  z = int(t / per_z);
  int64_t r = t - int64_t(z) * per_z;
  mb = int(r / P.n_blocks);
  nb = int(r - int64_t(mb) * P.n_blocks);
}

// ------------------------------------------------------------ epilogue math
// The epilogue works on boxes of 32 rows (one TMEM lane quarter, lane = row)
// x TC_EW columns.
template <int W>
__device__ __forceinline__ void apply_act(int act, float (&v)[W]) {
  switch (act) {
    case ACT_RELU:
#pragma unroll
      for (int j = 0; j < W; ++j) v[j] = v[j] > 0.0f ? v[j] : 0.0f;
      break;
    case ACT_TANH:
#pragma unroll
      for (int j = 0; j < W; ++j) v[j] = tanhf(v[j]);
      break;
    case ACT_GELU:
#pragma unroll
      for (int j = 0; j < W; j += 2) {
        const float2 x = make_float2(v[j], v[j + 1]);
        float2 phi, e;
        fast_phi2(x, phi, e);
        const float2 y = mul2(x, phi);
        v[j] = y.x;
        v[j + 1] = y.y;
      }
      break;
    default:
      break;
  }
}
template <int W>
__device__ __forceinline__ void apply_dact(int act, float (&v)[W], const float (&a)[W]) {
  switch (act) {
    case ACT_RELU:
#pragma unroll
      for (int j = 0; j < W; ++j) v[j] *= a[j] > 0.0f ? 1.0f : 0.0f;
      break;
    case ACT_TANH:
#pragma unroll
      for (int j = 0; j < W; ++j) v[j] *= __fsub_rn(1.0f, __fmul_rn(a[j], a[j]));
      break;
    case ACT_GELU:
#pragma unroll
      for (int j = 0; j < W; j += 2) {
        const float2 x = make_float2(a[j], a[j + 1]);
        float2 phi, e;
        fast_phi2(x, phi, e);
        const float2 g = fma2(mul2(x, splat2(0.39894228040143268f)), e, phi);
        const float2 r = mul2(make_float2(v[j], v[j + 1]), g);
        v[j] = r.x;
        v[j + 1] = r.y;
      }
      break;
    case ACT_DERIV:
#pragma unroll
      for (int j = 0; j < W; j += 2) {
        const float2 r = mul2(make_float2(v[j], v[j + 1]), make_float2(a[j], a[j + 1]));
        v[j] = r.x;
        v[j + 1] = r.y;
      }
      break;
    default:
      break;
  }
}
// y = act(v) in place and d = act'(v) (save_grad epilogue); GELU shares one
// Phi / exp evaluation between the two
template <int W>
__device__ __forceinline__ void act_and_deriv(int act, float (&v)[W], float (&d)[W]) {
  if (act == ACT_GELU) {
#pragma unroll
    for (int j = 0; j < W; j += 2) {
      const float2 x = make_float2(v[j], v[j + 1]);
      float2 phi, e;
      fast_phi2(x, phi, e);
      const float2 g = fma2(mul2(x, splat2(0.39894228040143268f)), e, phi);
      const float2 y = mul2(x, phi);
      d[j] = g.x;
      d[j + 1] = g.y;
      v[j] = y.x;
      v[j + 1] = y.y;
    }
    return;
  }
#pragma unroll
  for (int j = 0; j < W; ++j) {
    if (act == ACT_TANH) {
      v[j] = tanhf(v[j]);
      d[j] = __fsub_rn(1.0f, __fmul_rn(v[j], v[j]));
    } else if (act == ACT_RELU) {
      d[j] = v[j] > 0.0f ? 1.0f : 0.0f;
      v[j] = v[j] > 0.0f ? v[j] : 0.0f;
    } else {
      d[j] = 1.0f;
    }
  }
}

__device__ __forceinline__ uint32_t pack2(float a, float b, int dt) {
  if (dt == TCB_BF16) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
  }
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void unpack2(uint32_t w, int dt, float& a, float& b) {
  if (dt == TCB_BF16) {
    a = __uint_as_float(w << 16);
    b = __uint_as_float(w & 0xffff0000u);
  } else {
    float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w));
    a = f.x;
    b = f.y;
  }
}
// Staging boxes: one row per lane, 16-byte granules XOR-swizzled exactly as
// TMA's SWIZZLE_{32,64,128}B (granule ^= row bits above the row size), so
// the st.shared are bank-conflict free and the TMA store un-swizzles.
template <int W>
struct Box {
  static constexpr int ROW16 = W * 2;  // bytes per row, 16-bit elements
  static constexpr int ROW32 = W * 4;  // bytes per row, f32
  static __device__ __forceinline__ int sw(int row, int g, int row_bytes) {
    // granule index bits [4, 4+log2(row_bytes/16)) ^= address bits [7, ...)
    const int ng = row_bytes / 16;
    return (g ^ ((row * row_bytes >> 7) & (ng - 1)));
  }
};
template <int W, typename H>
__device__ __forceinline__ void stage_row16(uint8_t* box, int lane, const float (&v)[W]) {
  constexpr int RB = W * 2;
#pragma unroll
  for (int g = 0; g < RB / 16; ++g) {
    uint4 q;
    if constexpr (std::is_same<H, __nv_bfloat16>::value) {
      q.x = pack2(v[8 * g], v[8 * g + 1], TCB_BF16);
      q.y = pack2(v[8 * g + 2], v[8 * g + 3], TCB_BF16);
      q.z = pack2(v[8 * g + 4], v[8 * g + 5], TCB_BF16);
      q.w = pack2(v[8 * g + 6], v[8 * g + 7], TCB_BF16);
    } else {
      q.x = pack2(v[8 * g], v[8 * g + 1], TCB_F16);
      q.y = pack2(v[8 * g + 2], v[8 * g + 3], TCB_F16);
      q.z = pack2(v[8 * g + 4], v[8 * g + 5], TCB_F16);
      q.w = pack2(v[8 * g + 6], v[8 * g + 7], TCB_F16);
    }
    *reinterpret_cast<uint4*>(box + lane * RB + (Box<W>::sw(lane, g, RB) << 4)) = q;
  }
}
// one uniform dtype branch per row (the 16-bit packs are then single-path)
template <int W>
__device__ __forceinline__ void stage_row(uint8_t* box, int lane, int dt, const float (&v)[W]) {
  if (dt == TCB_F32) {
    constexpr int RB = W * 4;
#pragma unroll
    for (int g = 0; g < RB / 16; ++g) {
      float4 q = make_float4(v[4 * g], v[4 * g + 1], v[4 * g + 2], v[4 * g + 3]);
      *reinterpret_cast<float4*>(box + lane * RB + (Box<W>::sw(lane, g, RB) << 4)) = q;
    }
  } else if (dt == TCB_BF16) {
    stage_row16<W, __nv_bfloat16>(box, lane, v);
  } else {
    stage_row16<W, __half>(box, lane, v);
  }
}

// Direct-store fallback (C or aux not TMA-able): W consecutive values of one
// row, scalar stores with a tail guard.
template <int W>
__device__ __forceinline__ void store_row(void* dst, int dt, int64_t base, const float (&v)[W], int nvalid) {
#pragma unroll
  for (int j = 0; j < W; ++j) {
    if (j < nvalid) {
      if (dt == TCB_F32) static_cast<float*>(dst)[base + j] = v[j];
      else if (dt == TCB_BF16) static_cast<__nv_bfloat16*>(dst)[base + j] = __float2bfloat16_rn(v[j]);
      else static_cast<__half*>(dst)[base + j] = __float2half_rn(v[j]);
    }
  }
}

struct EpiMaps {
  CUtensorMap c, u;
};

template <int BN, int CG, bool AUX, int EPW>
__global__ void __launch_bounds__(tc_threads<EPW>(), 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA0, const __grid_constant__ CUtensorMap tmB0,
              const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmB1,
              const __grid_constant__ EpiMaps EM0, const __grid_constant__ EpiMaps EM1, const TcParams P) {
  using C = TcCfg<BN, CG, AUX, EPW>;
  constexpr int W = TC_EW;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint8_t* sEpi = smem + C::STAGES * C::STAGE_BYTES;        // epilogue warps x 2 output slots
  constexpr int OUT_RING = out_ring<AUX>();
  float* sBias = reinterpret_cast<float*>(sEpi + EPW * OUT_RING * TC_SLOT);  // per-warp bias columns
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sBias) + C::BIAS_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  // the warp index broadcast from lane 0: the compiler then treats it (and the
  // tile coordinates derived from it) as warp-uniform, so TMA / tcgen05 issue
  // takes uniform registers directly instead of a per-lane R2UR loop
  const int warp = __shfl_sync(0xffffffffu, int(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  constexpr bool clustered = CG == 2;
  const uint32_t crank = clustered ? cluster_ctarank() : 0;
  const uint32_t rank = crank % CG;          // position in the CTA pair
  const uint32_t lead = crank - rank;        // the pair leader's cluster rank
  const int64_t cl_id = blockIdx.x / CG, n_cl = gridDim.x / CG;
  const uint16_t mcast = uint16_t(3u << lead);
  unsigned long long* tr = P.trace ? P.trace + blockIdx.x * 16 : nullptr;
  if (tr && threadIdx.x == 0) tr[0] = gtimer();

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA0)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB0)) : "memory");
    if (P.nprob > 1) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA1)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB1)) : "memory");
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], CG * EPW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    if constexpr (CG == 2) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  if (clustered) cluster_sync();
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // everything above (barriers, TMEM, descriptor prefetch) overlapped the
  // previous kernel's tail; from here on we read its outputs
  pdl_wait();
  pdl_trigger();
  if (tr && threadIdx.x == 0) tr[1] = gtimer();

  if (warp == 0) {
    // ===================== TMA producer (both CTAs) =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t ui = 0, u; (u = unit_at(P, cl_id, n_cl, ui)) >= 0; ++ui) {
        const int prob = unit_prob(P, u);
        const TcProb& Q = P.pr[prob];
        const CUtensorMap* mA = prob ? &tmA1 : &tmA0;
        const CUtensorMap* mB = prob ? &tmB1 : &tmB0;
        const int64_t t = u - (prob ? P.pr[0].num_tiles : 0);
        int z, mb, nb;
        decode_tile(Q, t, z, mb, nb);
        const int kb0 = (Q.wsplit > 1 ? z : 0) * Q.kps;
        const int kb1 = min(kb0 + Q.kps, Q.k_blocks);
        if (Q.wsplit > 1) z = 0;  // z is the K slice, not a batch index
        const int z1 = int(z / Q.Z2), z2 = int(z % Q.Z2);
        const int m0 = mb * (TC_BM * CG) + int(rank) * TC_BM;
        const int n0 = nb * BN + int(rank) * C::B_ROWS;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          // both CTAs' bytes complete on the leader's barrier
          const uint32_t fb = CG == 2 ? mapa(smem_u32(&full[stage]), lead) : smem_u32(&full[stage]);
          if (rank == 0)
            mbar_expect_tx(&full[stage], CG * (C::A_BYTES + (Q.tb ? C::B_ROWS * TC_BK * 2 : C::B_BYTES)));
          uint8_t* a_dst = sA + stage * C::A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          const int k0 = kb * TC_BK;
          if (!Q.ta) {
            tma_load_4d<CG>(a_dst, mA, fb, k0, m0, z2, z1);
          } else {
#pragma unroll
            for (int c = 0; c < TC_BM / 64; ++c) tma_load_4d<CG>(a_dst + c * 8192, mA, fb, m0 + c * 64, k0, z2, z1);
          }
          if (Q.tb) {
            tma_load_4d<CG>(b_dst, mB, fb, k0, n0, z2, z1);
          } else {
#pragma unroll
            for (int c = 0; c < C::B_CHUNKS; ++c)
              tma_load_4d<CG>(b_dst + c * 8192, mB, fb, n0 + c * 64, k0, z2, z1);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    if (lane == 0 && rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t ui = 0, u; (u = unit_at(P, cl_id, n_cl, ui)) >= 0; ++ui) {
        const int prob = unit_prob(P, u);
        const TcProb& Q = P.pr[prob];
        int kb0 = 0;
        if (Q.wsplit > 1) {
          int z, mb, nb;
          decode_tile(Q, u - (prob ? P.pr[0].num_tiles : 0), z, mb, nb);
          kb0 = z * Q.kps;
        }
        const int kb1 = min(kb0 + Q.kps, Q.k_blocks);
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + uint32_t(acc * BN);
        // descriptors of stage 0; stage s and k-step k only move the start
        // address field (bits 0-13, 16-byte units): + s * stage bytes / 16 and
        // + k * (K-major: 32 B -> 2, MN-major: 16 k-rows x 128 B -> 128)
        // LBO = 8 KB between 64-wide MN chunks, SBO = 1 KB between 8-row atoms.
        const uint64_t a_desc0 = Q.ta ? umma_desc(smem_u32(sA), 8192, 1024) : umma_desc(smem_u32(sA), 16, 1024);
        const uint64_t b_desc0 = Q.tb ? umma_desc(smem_u32(sB), 16, 1024) : umma_desc(smem_u32(sB), 8192, 1024);
        const uint32_t a_step = Q.ta ? 128u : 2u, b_step = Q.tb ? 2u : 128u;
        const uint32_t idesc = Q.idesc;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (tr && ui == 0 && kb == kb0) tr[2] = gtimer();
          const uint64_t ad0 = a_desc0 + uint64_t(stage * (C::A_BYTES >> 4));
          const uint64_t bd0 = b_desc0 + uint64_t(stage * (C::B_BYTES >> 4));
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k)
            tc_mma<CG>(tmem_d, ad0 + uint64_t(k * a_step), bd0 + uint64_t(k * b_step), idesc,
                       (kb > kb0 || k) ? 1u : 0u);
          tc_commit<CG>(&empty[stage], mcast);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit<CG>(&tfull[acc], mcast);
        if (tr) {
          tr[3] = gtimer();
          if (ui < 3) tr[12 + ui] = tr[3];
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue (EPW warps, both CTAs) =====================
    // warp w may only touch TMEM lanes 32*(w%4)..+31 (its 32 rows); the warps
    // sharing a lane quarter take every TC_EPI_SPLIT-th W-column chunk
    constexpr int NCH = BN / W;
    constexpr int SPLIT = EPW / 4;
    constexpr int CPW = (NCH + SPLIT - 1) / SPLIT;  // chunks per warp per tile (max)
    const int ew = warp - 4;
    const int q = warp & 3;
    const int sub = ew >> 2;
    uint8_t* slots = sEpi + ew * OUT_RING * TC_SLOT;
    float* wbias = sBias + ew * CPW * W;
    const uint32_t tempty_addr0 = CG == 2 ? mapa(smem_u32(&tempty[0]), lead) : smem_u32(&tempty[0]);
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t sidx = 0;    // output slot ring
    // act'(aux) loads: each lane reads its row's 16 16-bit values straight
    // from global (2 x 16 B, read-only path; the fast path prefetches the next
    // chunk's into registers).  The earlier per-warp TMA box ring (three 1 KB
    // boxes in flight, mbarrier per box) cost 48 KB of shared memory and was
    // slower: act'(aux) dgrad 27.5 -> 24.9 us with direct loads.
    auto aux_ld = [&](const TcProb& Qa, int64_t mm, int64_t cof, int64_t nn, uint4& x0, uint4& x1) {
      if (mm < Qa.M && nn + W <= Qa.N) {
        const uint4* src = reinterpret_cast<const uint4*>(static_cast<const uint16_t*>(Qa.aux) + cof + mm * Qa.ldc + nn);
        x0 = __ldg(src);
        x1 = __ldg(src + 1);
      } else {
        x0 = x1 = make_uint4(0, 0, 0, 0);
        if (mm < Qa.M) {
          uint16_t* h = reinterpret_cast<uint16_t*>(&x0);
          for (int j = 0; j < W && nn + j < Qa.N; ++j)
            h[j] = static_cast<const uint16_t*>(Qa.aux)[cof + mm * Qa.ldc + nn + j];  // x0, x1 contiguous
        }
      }
    };
    auto aux_unpack = [&](int dt, const uint4& x0, const uint4& x1, float (&a)[W]) {
      const uint32_t w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
#pragma unroll
      for (int k = 0; k < 8; ++k) unpack2(w[k], dt, a[2 * k], a[2 * k + 1]);
    };

    for (int64_t ui = 0, u; (u = unit_at(P, cl_id, n_cl, ui)) >= 0; ++ui) {
      const int prob = unit_prob(P, u);
      const TcProb& Q = P.pr[prob];
      const EpiMaps& EM = prob ? EM1 : EM0;
      const bool has_aux = AUX && Q.tma_epi && Q.dact != ACT_NONE;
      const int64_t t = u - (prob ? P.pr[0].num_tiles : 0);
      int z, mb, nb;
      decode_tile(Q, t, z, mb, nb);
      const int z1 = Q.wsplit > 1 ? 0 : int(z / Q.Z2), z2 = Q.wsplit > 1 ? z : int(z % Q.Z2);
      const int64_t coff = int64_t(z1) * Q.c_s1 + int64_t(z2) * Q.c_s2;
      const int mrow0 = mb * (TC_BM * CG) + int(rank) * TC_BM + q * 32;  // this warp's 32-row box
      // per-tile TMA-store operands broadcast from lane 0 once (warp-uniform:
      // the stores issue from uniform registers, no per-lane R2UR loop)
      const int un0 = __shfl_sync(0xffffffffu, int(nb) * BN, 0), sy = __shfl_sync(0xffffffffu, mrow0, 0);
      const int sz2 = __shfl_sync(0xffffffffu, z2, 0), sz1 = __shfl_sync(0xffffffffu, z1, 0);
      const CUtensorMap* mc = uniform_ptr(&EM.c);
      const CUtensorMap* mu = uniform_ptr(&EM.u);
      const int64_t m = int64_t(mrow0) + lane;
      // finishes one W-column chunk: v holds the f32 accumulator row segment
      auto finish = [&](float (&v)[W], int ci, int64_t n0) {
        if (Q.alpha != 1.0f) {
#pragma unroll
          for (int j = 0; j < W; ++j) v[j] *= Q.alpha;
        }
        if (Q.bias) {
          const float4* bb = reinterpret_cast<const float4*>(wbias + ci * W);
#pragma unroll
          for (int j = 0; j < W / 4; ++j) {
            const float4 b4 = bb[j];
            const float2 lo = add2(make_float2(v[4 * j], v[4 * j + 1]), make_float2(b4.x, b4.y));
            const float2 hi = add2(make_float2(v[4 * j + 2], v[4 * j + 3]), make_float2(b4.z, b4.w));
            v[4 * j] = lo.x;
            v[4 * j + 1] = lo.y;
            v[4 * j + 2] = hi.x;
            v[4 * j + 3] = hi.y;
          }
        }
        if (Q.tma_epi) {
          if (has_aux) {
            uint4 x0, x1;
            aux_ld(Q, m, coff, n0, x0, x1);
            float a[W];
            aux_unpack(Q.aux_dtype, x0, x1, a);
            apply_dact<W>(Q.dact, v, a);
          }
          uint8_t* slot = slots + sidx * TC_SLOT;
          if (lane == 0) bulk_wait_read<OUT_RING - 1>();  // the store that last used this slot has read it
          __syncwarp();
          if (Q.save_grad) {
            float dv[W];
            act_and_deriv<W>(Q.act, v, dv);
            stage_row<W>(slot + TC_SLOT / 2, lane, Q.c_dtype, dv);
          } else {
            if (Q.aux_out) stage_row<W>(slot + TC_SLOT / 2, lane, Q.c_dtype, v);
            apply_act<W>(Q.act, v);
          }
          stage_row<W>(slot, lane, Q.c_dtype, v);
          fence_proxy_async();
          const int sx = un0 + (sub + ci * SPLIT) * W;  // = n0, from uniform values
          if (lane == 0) {
            tma_store_4d(mc, slot, sx, sy, sz2, sz1);
            if (Q.aux_out) tma_store_4d(mu, slot + TC_SLOT / 2, sx, sy, sz2, sz1);
            bulk_commit();
          }
          if (++sidx == OUT_RING) sidx = 0;
        } else if (m < Q.M) {
          const int nvalid = int(Q.N - n0 < W ? Q.N - n0 : W);
          const int64_t base = coff + m * Q.ldc + n0;
          if (Q.dact != ACT_NONE) {
            float a[W];
#pragma unroll
            for (int j = 0; j < W; ++j) a[j] = j < nvalid ? ld_e(Q.aux, Q.aux_dtype, base + j) : 0.0f;
            apply_dact<W>(Q.dact, v, a);
          }
          if (Q.save_grad) {
            float dv[W];
            act_and_deriv<W>(Q.act, v, dv);
            store_row<W>(Q.aux_out, Q.c_dtype, base, dv, nvalid);
          } else {
            if (Q.aux_out) store_row<W>(Q.aux_out, Q.c_dtype, base, v, nvalid);
            apply_act<W>(Q.act, v);
          }
          store_row<W>(Q.c, Q.c_dtype, base, v, nvalid);
        }
      };
      // The step's hot epilogues with every choice fixed at compile time (TMA
      // path, bf16 output, alpha 1): no per-chunk branches on the problem's
      // fields, constant-folded activation / dtype switches.
      //   EK_BIAS: + bias;  EK_GELU_SAVE: + bias, y = GELU(u) and GELU'(u)
      //   stored (FFN1 forward);  EK_DERIV: * act'(aux) (prefetched registers)
      //   (FFN2 backward data gradient);  EK_F32: plain f32 output (weight
      //   gradients, K-slice partials).  Anything else: `finish` above.
      uint4 pa0 = make_uint4(0, 0, 0, 0), pa1 = pa0;  // prefetched act'(aux) of the current chunk
      auto finish_fast = [&](auto kind, float (&v)[W], int ci, int64_t n0) {
        constexpr int K = decltype(kind)::value;
        if constexpr (K == EK_BIAS || K == EK_GELU_SAVE) {
          const float4* bb = reinterpret_cast<const float4*>(wbias + ci * W);
#pragma unroll
          for (int j = 0; j < W / 4; ++j) {
            const float4 b4 = bb[j];
            const float2 lo = add2(make_float2(v[4 * j], v[4 * j + 1]), make_float2(b4.x, b4.y));
            const float2 hi = add2(make_float2(v[4 * j + 2], v[4 * j + 3]), make_float2(b4.z, b4.w));
            v[4 * j] = lo.x;
            v[4 * j + 1] = lo.y;
            v[4 * j + 2] = hi.x;
            v[4 * j + 3] = hi.y;
          }
        }
        if constexpr (K == EK_DERIV && AUX) {
          float a[W];
          aux_unpack(TCB_BF16, pa0, pa1, a);
          apply_dact<W>(ACT_DERIV, v, a);
        }
        uint8_t* slot = slots + sidx * TC_SLOT;
        if (lane == 0) bulk_wait_read<OUT_RING - 1>();
        __syncwarp();
        if constexpr (K == EK_GELU_SAVE) {
          float dv[W];
          act_and_deriv<W>(ACT_GELU, v, dv);
          stage_row16<W, __nv_bfloat16>(slot + TC_SLOT / 2, lane, dv);
        }
        if constexpr (K == EK_F32) stage_row<W>(slot, lane, TCB_F32, v);
        else stage_row16<W, __nv_bfloat16>(slot, lane, v);
        fence_proxy_async();
        const int sx = un0 + (sub + ci * SPLIT) * W;  // = n0, from uniform values
        if constexpr (K == EK_GELU_SAVE) {
          if (lane == 0) {
            tma_store_4d(mc, slot, sx, sy, sz2, sz1);
            tma_store_4d_evict_first(mu, slot + TC_SLOT / 2, sx, sy, sz2, sz1);  // GELU'(u): read in the backward
            bulk_commit();
          }
        } else if (lane == 0) {
          tma_store_4d(mc, slot, sx, sy, sz2, sz1);
          bulk_commit();
        }
        if (++sidx == OUT_RING) sidx = 0;
      };
      auto load_bias = [&]() {
        // this warp's bias columns for the tile -> smem (read back as broadcasts)
        __syncwarp();
        for (int i = lane; i < CPW * W; i += 32) {
          const int c = sub + (i / W) * SPLIT;
          const int64_t n = int64_t(nb) * BN + int64_t(c) * W + (i % W);
          wbias[i] = (c < NCH && n < Q.N) ? ld_e(Q.bias, Q.bias_dtype, n) : 0.0f;
        }
        __syncwarp();
      };
      if (Q.bias) load_bias();
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (tr && ew == 0 && ui == 0) tr[4] = gtimer();
      if (tr && ew == 0 && lane == 0 && ui >= 1 && ui < 3) tr[8 + 2 * (ui - 1)] = gtimer();
      auto chunks = [&](auto kind) {
        constexpr int K = decltype(kind)::value;
        constexpr bool PF = K == EK_DERIV && AUX;
        if (PF) aux_ld(Q, m, coff, int64_t(nb) * BN + sub * W, pa0, pa1);  // the first chunk's act'(aux)
#pragma unroll 1
        for (int c = sub, ci = 0; c < NCH; c += SPLIT, ++ci) {
          const int64_t n0 = int64_t(nb) * BN + c * W;
          if (n0 >= Q.N) continue;
          uint4 na0, na1;  // prefetch: the next chunk's act'(aux) while this one runs
          if (PF) {
            if (c + SPLIT < NCH) aux_ld(Q, m, coff, n0 + SPLIT * W, na0, na1);
            else na0 = na1 = make_uint4(0, 0, 0, 0);
          }
          uint32_t r[W];
          const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN + c * W);
          if constexpr (W == 16) TMEM_LD16(taddr, r);
          else TMEM_LD32(taddr, r);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          float v[W];
#pragma unroll
          for (int j = 0; j < W; ++j) v[j] = __uint_as_float(r[j]);
          if constexpr (K == EK_GENERIC) finish(v, ci, n0);
          else finish_fast(kind, v, ci, n0);
          if (PF) pa0 = na0, pa1 = na1;
        }
      };
      switch (epi_kind<AUX>(Q)) {
        case EK_BIAS: chunks(std::integral_constant<int, EK_BIAS>{}); break;
        case EK_GELU_SAVE: chunks(std::integral_constant<int, EK_GELU_SAVE>{}); break;
        case EK_DERIV: chunks(std::integral_constant<int, EK_DERIV>{}); break;
        case EK_PLAIN: chunks(std::integral_constant<int, EK_PLAIN>{}); break;
        case EK_F32: chunks(std::integral_constant<int, EK_F32>{}); break;
        default: chunks(std::integral_constant<int, EK_GENERIC>{}); break;
      }
      if (tr && ew == 0 && lane == 0 && ui == 0) tr[6] = gtimer();
      if (tr && ew == 0 && lane == 0 && ui >= 1 && ui < 3) tr[9 + 2 * (ui - 1)] = gtimer();
      // release the accumulator to the (leader's) MMA warp
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster(tempty_addr0 + acc * 8);
        else mbar_arrive(&tempty[acc]);
      }
      if (tr && ew == 0 && lane == 0 && ui == 0) tr[7] = gtimer();
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait_all();
    if (tr && lane == 0) atomicMax(&tr[5], gtimer());
  }
  tc_fence_before();
  if (clustered) cluster_sync();
  else __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    if constexpr (CG == 2)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS));
  }
}

// operand -> 4-D map, box {64, box_outer}, SWIZZLE_128B
static CUtensorMap make_map(const GemmOperand& o, int64_t inner, int64_t outer, int64_t Z2, int64_t Z1,
                            uint32_t box_outer) {
  return encode4(o.ptr, o.dtype, inner, outer, Z2, Z1, o.ld, o.s2, o.s1, 64, box_outer, CU_TENSOR_MAP_SWIZZLE_128B);
}

bool gemm_tc_supported(const GemmArgs& g, std::string* why) {
  auto no = [&](const char* w) {
    if (why) *why = w;
    return false;
  };
  if (!((g.a.dtype == TCB_BF16 && g.b.dtype == TCB_BF16) || (g.a.dtype == TCB_F16 && g.b.dtype == TCB_F16)))
    return no("operands must both be bf16 or f16");
  for (const GemmOperand* o : {&g.a, &g.b}) {
    if ((o->ld * 2) % 16) return no("leading dimension must be a multiple of 8 elements");
    if ((o->s1 * 2) % 16 || (o->s2 * 2) % 16) return no("batch strides must be 16-byte multiples");
    if (o->ptr && reinterpret_cast<uintptr_t>(o->ptr) % 16) return no("operand not 16-byte aligned");
  }
  if (g.M > (int64_t(1) << 31) || g.N > (int64_t(1) << 31) || g.K > (int64_t(1) << 31))
    return no("dimension too large");
  return true;
}

// Can C / aux_out / aux go through TMA boxes?  (16-byte aligned bases and
// strides; aux only 16-bit)
static bool epi_tma_ok(const GemmArgs& g) {
  const int es = dtype_bytes(g.c_dtype);
  auto al = [](const void* p) { return reinterpret_cast<uintptr_t>(p) % 16 == 0; };
  if (!al(g.c) || (g.ldc * es) % 16 || (g.c_s1 * es) % 16 || (g.c_s2 * es) % 16) return false;
  if (g.aux_out && !al(g.aux_out)) return false;
  if (g.aux_out && g.c_dtype == TCB_F32) return false;  // y + u must fit one slot
  if (g.dact != ACT_NONE) {
    if (g.aux_dtype == TCB_F32 || !al(g.aux)) return false;
    const int ea = dtype_bytes(g.aux_dtype);
    if ((g.ldc * ea) % 16 || (g.c_s1 * ea) % 16 || (g.c_s2 * ea) % 16) return false;
  }
  return true;
}

// one problem's kernel parameters and tensor maps for tile shape (BN, CG)
template <int BN, int CG, bool AUX>
static void fill_prob(const GemmArgs& g, TcProb& P, CUtensorMap& ta, CUtensorMap& tb, EpiMaps& em) {
  using C = TcCfg<BN, CG, AUX>;
  P.M = g.M;
  P.N = g.N;
  P.K = g.K;
  P.Z = g.Z;
  P.Z2 = g.Z2;
  P.ta = g.ta;
  P.tb = g.tb;
  P.m_blocks = int((g.M + TC_BM * CG - 1) / (TC_BM * CG));
  P.n_blocks = int((g.N + BN - 1) / BN);
  P.k_blocks = int((g.K + TC_BK - 1) / TC_BK);
  P.wsplit = g.wsplit > 1 ? g.wsplit : 1;
  P.num_tiles = int64_t(P.m_blocks) * P.n_blocks * g.Z * P.wsplit;
  P.kps = (P.k_blocks + P.wsplit - 1) / P.wsplit;
  P.idesc = umma_idesc(TC_BM * CG, BN, g.a.dtype == TCB_BF16, g.ta != 0, g.tb == 0);
  P.c = g.c;
  P.ldc = g.ldc;
  P.c_s1 = g.c_s1;
  P.c_s2 = P.wsplit > 1 ? g.M * g.ldc : g.c_s2;  // workspace slices
  P.c_dtype = g.c_dtype;
  P.alpha = g.alpha;
  P.bias = g.bias;
  P.bias_dtype = g.bias_dtype;
  P.act = g.act;
  P.dact = g.dact;
  P.aux = g.aux;
  P.aux_dtype = g.aux_dtype;
  P.aux_out = g.aux_out;
  P.save_grad = g.aux_out ? g.save_grad : 0;
  const int es = dtype_bytes(g.c_dtype);
  P.c_vec_ok = (reinterpret_cast<uintptr_t>(g.c) % 16 == 0) && ((g.ldc * es) % 16 == 0) &&
               ((g.c_s1 * es) % 16 == 0) && ((g.c_s2 * es) % 16 == 0) &&
               (!g.aux_out || reinterpret_cast<uintptr_t>(g.aux_out) % 16 == 0);
  P.tma_epi = epi_tma_ok(g) && (g.dact == ACT_NONE || AUX) && !g.no_tma_epi;
  P.generic_epi = g.generic_epi;
  const int64_t Z1 = (g.Z + g.Z2 - 1) / g.Z2;
  ta = g.ta ? make_map(g.a, g.M, g.K, g.Z2, Z1, 64) : make_map(g.a, g.K, g.M, g.Z2, Z1, TC_BM);
  tb = g.tb ? make_map(g.b, g.K, g.N, g.Z2, Z1, C::B_ROWS) : make_map(g.b, g.N, g.K, g.Z2, Z1, 64);
  std::memset(&em, 0, sizeof(em));
  if (P.tma_epi) {
    // boxes of 32 rows x TC_EW columns, swizzled by their row size (see stage_row)
    auto sw = [](int row_bytes) {
      return row_bytes == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
             : row_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                               : CU_TENSOR_MAP_SWIZZLE_32B;
    };
    const CUtensorMapSwizzle csw = sw(TC_EW * dtype_bytes(g.c_dtype));
    if (P.wsplit > 1)
      em.c = encode4(g.c, g.c_dtype, g.N, g.M, P.wsplit, 1, g.ldc, g.M * g.ldc, 0, TC_EW, 32, csw);
    else
      em.c = encode4(g.c, g.c_dtype, g.N, g.M, g.Z2, Z1, g.ldc, g.c_s2, g.c_s1, TC_EW, 32, csw);
    if (g.aux_out) em.u = encode4(g.aux_out, g.c_dtype, g.N, g.M, g.Z2, Z1, g.ldc, g.c_s2, g.c_s1, TC_EW, 32, csw);
  }
}

// launch n (1 or 2) problems with one tile shape in a single persistent grid
template <int BN, int CG, bool AUX, int EPW>
static void launch_cfg(const GemmArgs* gs, int n, cudaStream_t s) {
  using C = TcCfg<BN, CG, AUX, EPW>;
  static std::once_flag once;
  std::call_once(once, [] {
    TCB_CUDA(cudaFuncSetAttribute(k_gemm_tc<BN, CG, AUX, EPW>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  });
  TcParams P{};
  P.nprob = n;
  P.trace = reinterpret_cast<unsigned long long*>(gs[0].trace);
  CUtensorMap ta[2], tb[2];
  EpiMaps em[2];
  for (int i = 0; i < n; ++i) fill_prob<BN, CG, AUX>(gs[i], P.pr[i], ta[i], tb[i], em[i]);
  if (n == 1) {
    ta[1] = ta[0];
    tb[1] = tb[0];
    em[1] = em[0];
  }
  P.num_units = P.pr[0].num_tiles + (n > 1 ? P.pr[1].num_tiles : 0);
  P.sched = gs[0].sched;
  P.sched_rounds = gs[0].sched_rounds;
  const int64_t units = P.num_units * CG;
  int grid = int(units < kNumSMs ? units : kNumSMs);
  grid = (grid / CG) * CG;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(unsigned(grid));
  cfg.blockDim = dim3(tc_threads<EPW>());
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1 + pdl_attr(&attr[1]);
  TCB_CUDA(cudaLaunchKernelEx(&cfg, k_gemm_tc<BN, CG, AUX, EPW>, ta[0], tb[0], ta[1], tb[1], em[0], em[1], P));
}

// Tile configuration by a wave-quantised cost model (calibrated on the
// BERT-base shapes, profiles/r01_gemm_tile_sweep.jsonl):
//   time ~ rounds * (kps + K_FIX) * BN / eff(CG, BN)
// rounds = ceil(units / concurrent units), a CTA pair is one unit of 74;
// K_FIX k-blocks model the per-unit fill/drain; eff(.) is the relative
// mainloop throughput per SM of each tile shape.
static int stage_bytes(int bn, int cg) { return TC_BM * TC_BK * 2 + ((bn / cg + 63) / 64) * 64 * TC_BK * 2; }
static int stages_of(int bn, int cg) {
  const int cpw = (bn / TC_EW + TC_EPI_WARPS / 4 - 1) / (TC_EPI_WARPS / 4);
  const int budget = 227 * 1024 - 1024 - 1024 - TC_EPI_WARPS * out_ring<false>() * TC_SLOT - TC_EPI_WARPS * cpw * TC_EW * 4;
  return std::min(8, budget / stage_bytes(bn, cg));
}
static TcChoice choose(const GemmArgs& g) {
  if (g.force_bn) return {g.force_bn, g.force_cg ? g.force_cg : 1};
  struct Cand {
    int bn, cg;
    double eff;
  };
  const Cand cands[] = {{256, 2, 1.0}, {192, 2, 0.85}, {128, 2, 0.6}, {256, 1, 0.75}, {192, 1, 0.7}, {128, 1, 0.55}};
  const int64_t kblocks = (g.K + TC_BK - 1) / TC_BK;
  constexpr double K_FIX = 6.0;
  TcChoice best{128, 1};
  double best_cost = 1e30;
  for (const Cand& c : cands) {
    if (c.bn > 128 && g.N <= 128) continue;
    if (c.cg == 2 && g.M <= 128) continue;  // the pair's second CTA would only see padding
    const int64_t mb = (g.M + 128 * c.cg - 1) / (128 * c.cg);
    const int64_t nb = (g.N + c.bn - 1) / c.bn;
    const int64_t tiles = mb * nb * g.Z;
    const int64_t conc = kNumSMs / c.cg;
    const double rounds = double((tiles + conc - 1) / conc);
    const double cost = rounds * (double(kblocks) + K_FIX) * double(c.bn) / c.eff;
    if (cost < best_cost * 0.97) {
      best_cost = cost;
      best = {c.bn, c.cg};
    }
  }
  return best;
}

TcChoice gemm_tc_choose(const GemmArgs& g) { return choose(g); }

void gemm_prepare(GemmArgs& g, bool exact, GemmWs& keep) {
  (void)keep;
  if (exact || !gemm_tc_supported(g, nullptr)) return;
  const TcChoice c = choose(g);
  g.force_bn = c.bn;
  g.force_cg = c.cg;
}

static void dispatch_tc(const GemmArgs* gs, int n, const TcChoice& c, cudaStream_t s) {
  bool aux = false, light = true;
  for (int i = 0; i < n; ++i) {
    aux = aux || gs[i].dact != ACT_NONE;
    // plain / bias / f32 stores: no activation, no second output
    light = light && gs[i].act == ACT_NONE && !gs[i].aux_out;
  }
#define TC_CASE(BN_, CG_)                                  \
  if (c.bn == BN_ && c.cg == CG_) {                        \
    if (aux) launch_cfg<BN_, CG_, true, TC_EPW_AUX>(gs, n, s);     \
    else if (light) launch_cfg<BN_, CG_, false, TC_EPW_LIGHT>(gs, n, s); \
    else launch_cfg<BN_, CG_, false, TC_EPW_HEAVY>(gs, n, s);        \
    return;                                                \
  }
  TC_CASE(256, 2)
  TC_CASE(192, 2)
  TC_CASE(128, 2)
  TC_CASE(256, 1)
  TC_CASE(192, 1)
  TC_CASE(128, 1)
#undef TC_CASE
  fail(TCB_ERR_TYPE, "tcgen05 gemm: unsupported forced tile config");
}

void launch_gemm_tc(const GemmArgs& g, cudaStream_t s) {
  std::string why;
  if (!gemm_tc_supported(g, &why)) fail(TCB_ERR_UNIMPLEMENTED, "tcgen05 gemm: " + why);
  dispatch_tc(&g, 1, choose(g), s);
}

// Two independent problems in one grid (same tile shape); the
// problem with more k-blocks per tile goes first.
static TcChoice pair_choice(const GemmArgs& g0, const GemmArgs& g1) {
  TcChoice c{g0.force_bn ? g0.force_bn : 256, g0.force_cg ? g0.force_cg : 2};
  if (c.cg == 2 && (g0.M <= 128 || g1.M <= 128)) c.cg = 1;
  return c;
}
void launch_gemm_tc_pair(const GemmArgs& g0, const GemmArgs& g1, cudaStream_t s) {
  std::string why;
  for (const GemmArgs* g : {&g0, &g1})
    if (!gemm_tc_supported(*g, &why)) fail(TCB_ERR_UNIMPLEMENTED, "tcgen05 gemm pair: " + why);
  const TcChoice c = pair_choice(g0, g1);
  const bool swap = g1.K > g0.K;
  GemmArgs gs[2] = {swap ? g1 : g0, swap ? g0 : g1};
  gs[0].sched = g0.sched;
  gs[0].sched_rounds = g0.sched_rounds;
  dispatch_tc(gs, 2, c, s);
}

// Longest-processing-time schedule for a pair launch: unit cost = its k-blocks
// plus an epilogue weight (GELU / act' epilogues cost more), every unit goes to
// the least-loaded cluster, largest first.  Returns the [rounds][clusters]
// table (-1 = done) the kernel walks; deterministic (ties by index).
static std::vector<int> lpt_table(const GemmArgs& g0, const GemmArgs& g1, int* rounds, double* max_load) {
  const TcChoice c = pair_choice(g0, g1);
  const bool swap = g1.K > g0.K;
  const GemmArgs* gs[2] = {swap ? &g1 : &g0, swap ? &g0 : &g1};
  std::vector<std::pair<double, int>> units;
  int64_t base = 0;
  for (const GemmArgs* g : gs) {
    const int ws = g->wsplit > 1 ? g->wsplit : 1;
    const int64_t tiles = ((g->M + 128 * c.cg - 1) / (128 * c.cg)) * ((g->N + c.bn - 1) / c.bn) * g->Z * ws;
    const int64_t kbt = (g->K + TC_BK - 1) / TC_BK;
    const double kb = double((kbt + ws - 1) / ws);
    const double epi = (g->dact != ACT_NONE || g->act == ACT_GELU) ? 6.0 : 2.0;
    for (int64_t t = 0; t < tiles; ++t) units.push_back({kb + epi, int(base + t)});
    base += tiles;
  }
  const int64_t total = int64_t(units.size()) * c.cg;
  int grid = int(total < kNumSMs ? total : kNumSMs);
  grid = (grid / c.cg) * c.cg;
  const int ncl = grid / c.cg;
  std::stable_sort(units.begin(), units.end(), [](auto& a, auto& b) { return a.first > b.first; });
  std::vector<double> load(ncl, 0.0);
  std::vector<std::vector<int>> lists(ncl);
  for (auto& [cost, u] : units) {
    int best = 0;
    for (int k = 1; k < ncl; ++k)
      if (load[k] < load[best]) best = k;
    load[best] += cost;
    lists[best].push_back(u);
  }
  int r = 0;
  for (auto& l : lists) r = std::max(r, int(l.size()));
  std::vector<int> table(size_t(r) * ncl, -1);
  for (int k = 0; k < ncl; ++k)
    for (size_t i = 0; i < lists[k].size(); ++i) table[i * ncl + k] = lists[k][i];
  *rounds = r;
  if (max_load) *max_load = *std::max_element(load.begin(), load.end());
  return table;
}
std::vector<int> gemm_pair_schedule(const GemmArgs& g0, const GemmArgs& g1, int* rounds) {
  return lpt_table(g0, g1, rounds, nullptr);
}

// K slices for problem `idx` of a pair (a weight gradient whose few long tiles
// bound the launch): the S in {1, 2, 4, 8} minimising the LPT makespan plus
// the slice reduction (its launch and (S+1) f32 passes over M x N, in k-block
// units of ~0.34 us).  Only plain f32 outputs with no epilogue work qualify.
bool gemm_wsplit_ok(const GemmArgs& g, int S) {
  const int64_t kbt = (g.K + TC_BK - 1) / TC_BK;
  const int64_t kps = (kbt + S - 1) / S;
  return S >= 1 && S <= 16 && (S - 1) * kps < kbt && g.c_dtype == TCB_F32 && !g.bias && g.act == ACT_NONE &&
         g.dact == ACT_NONE && !g.aux_out && g.Z == 1 && g.ldc == g.N && g.alpha == 1.0f;
}
int gemm_pair_wsplit(GemmArgs g0, GemmArgs g1, int idx) {
  GemmArgs& g = idx ? g1 : g0;
  const int64_t kbt = (g.K + TC_BK - 1) / TC_BK;
  if (!gemm_wsplit_ok(g, 1) || kbt < 16) return 1;
  int best_s = 1;
  double best = 1e30;
  for (int S : {1, 2, 4, 8}) {
    if (kbt / S < 4 || !gemm_wsplit_ok(g, S)) break;
    g.wsplit = S;
    int r = 0;
    double ml = 0.0;
    lpt_table(g0, g1, &r, &ml);
    const double red = S > 1 ? (2.0 + double(S + 1) * double(g.M * g.N) * 4.0 / 5e6) / 0.34 : 0.0;
    if (ml + red < best * 0.95) {
      best = ml + red;
      best_s = S;
    }
  }
  return best_s;
}

// out = sum_s ws[s] in slice order (deterministic), float4 vectorised
__global__ void k_wsplit_reduce(const float* __restrict__ ws, float* __restrict__ out, int64_t n, int S) {
  TCB_PDL_ENTRY();
  const int64_t n4 = n / 4, stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n4; i += stride) {
    float4 acc = reinterpret_cast<const float4*>(ws)[i];
    for (int s = 1; s < S; ++s) {
      const float4 v = reinterpret_cast<const float4*>(ws + s * n)[i];
      acc.x += v.x;
      acc.y += v.y;
      acc.z += v.z;
      acc.w += v.w;
    }
    reinterpret_cast<float4*>(out)[i] = acc;
  }
  for (int64_t i = n4 * 4 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    float acc = ws[i];
    for (int s = 1; s < S; ++s) acc += ws[s * n + i];
    out[i] = acc;
  }
}
void launch_wsplit_reduce(const float* ws, float* out, int64_t n, int S, cudaStream_t s) {
  if (!skip_folds()) launch_k(k_wsplit_reduce, grid_for((n + 3) / 4, 256, kNumSMs * 4), 256, 0, s, ws, out, n, S);
}

}  // namespace tcb
