// k_gemm_tc.cu -- bf16/f16 tensor-core GEMM for sm_100a: tcgen05.mma with the
// accumulator in TMEM, operands staged by TMA (SWIZZLE_128B), warp-specialised
// and persistent.
//
//   warp 0      TMA producer (one elected lane): A/B k-blocks into a STAGES-deep
//               smem ring, mbarrier full/empty handshake
//   warp 1      MMA issuer (one lane): tcgen05.mma.cta_group::1.kind::f16,
//               128 x BN x 16 per instruction, fp32 accumulate in TMEM;
//               tcgen05.commit frees smem stages / publishes finished tiles
//   warp 2      TMEM allocator (2 x BN columns: double-buffered accumulator)
//   warps 4-7   epilogue: tcgen05.ld 32x32b.x32 -> alpha, bias, act'(aux),
//               pre-activation store, act -> one rounding into C's dtype
//
// Operands may be K-major or MN-major (A: ta, B: tb), which absorbs the
// reference's `transpose` ops into the TMA/UMMA descriptors.
// Batched problems (attention heads, batch_matmul) use 4-D tensor maps
// {inner, outer, z2, z1}, so every batch gets exact zero-filled tails.
#include <cuda.h>

#include <mutex>

#include "gemm.cuh"

namespace tcb {

constexpr int TC_BM = 128;
constexpr int TC_BK = 64;  // 64 bf16 = 128 B = one SWIZZLE_128B atom row

template <int BN>
struct TcCfg {
  static constexpr int STAGES = BN == 256 ? 4 : BN == 192 ? 5 : 6;
  static constexpr int A_BYTES = TC_BM * TC_BK * 2;  // 16 KB
  static constexpr int B_BYTES = BN * TC_BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = 2 * BN <= 256 ? 256 : 512;  // power of two >= 2 accumulators
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
};

struct TcParams {
  int64_t M, N, K, Z, Z2;
  int ta, tb;
  int m_blocks, n_blocks, k_blocks;
  int64_t num_tiles;
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
  int c_vec_ok;  // 16-byte aligned rows
};

// ------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
// UMMA shared-memory descriptor, SWIZZLE_128B, version 1 (sm_100)
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= uint64_t((saddr & 0x3FFFFu) >> 4);
  d |= uint64_t((lbo >> 4) & 0x3FFFu) << 16;
  d |= uint64_t((sbo >> 4) & 0x3FFFu) << 32;
  d |= 1ull << 46;
  d |= 2ull << 61;
  return d;
}

#define TMEM_LD32(taddr, r)                                                                     \
  asm volatile(                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"  \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"        \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),     \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), \
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),           \
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),           \
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])            \
      : "r"(taddr))

__device__ __forceinline__ float ld_e(const void* p, int dt, int64_t i) {
  if (dt == TCB_F32) return static_cast<const float*>(p)[i];
  if (dt == TCB_BF16) return __bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]);
  return __half2float(static_cast<const __half*>(p)[i]);
}

__device__ __forceinline__ void decode_tile(const TcParams& P, int64_t t, int& z, int& mb, int& nb) {
  const int64_t per_z = int64_t(P.m_blocks) * P.n_blocks;
  z = int(t / per_z);
  int64_t r = t - int64_t(z) * per_z;
  mb = int(r / P.n_blocks);
  nb = int(r - int64_t(mb) * P.n_blocks);
}

// Store 32 consecutive f32 values of one row into dst (dtype dt).  Every loop
// is unrolled with compile-time indices so v[] stays in registers (a runtime
// trip count here made ptxas spill the whole array to local memory).
__device__ __forceinline__ void store_row32(void* dst, int dt, int64_t base, const float (&v)[32], bool vec,
                                            int nvalid) {
  if (dt == TCB_F32) {
    float* o = static_cast<float*>(dst) + base;
    if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(o + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) o[j] = v[j];
    }
  } else if (dt == TCB_BF16) {
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(dst) + base;
    if (vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 8) {
        uint4 q;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[j], v[j + 1]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(v[j + 2], v[j + 3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[j + 4], v[j + 5]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(v[j + 6], v[j + 7]);
        q.x = *reinterpret_cast<uint32_t*>(&h0);
        q.y = *reinterpret_cast<uint32_t*>(&h1);
        q.z = *reinterpret_cast<uint32_t*>(&h2);
        q.w = *reinterpret_cast<uint32_t*>(&h3);
        *reinterpret_cast<uint4*>(o + j) = q;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) o[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    __half* o = static_cast<__half*>(dst) + base;
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) o[j] = __float2half_rn(v[j]);
  }
}

// 32 consecutive output columns of one row: epilogue + store
__device__ __forceinline__ void epi_store32(const TcParams& P, const uint32_t (&r)[32], int64_t m, int64_t n0,
                                            int64_t coff) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * P.alpha;
  const int64_t base = coff + m * P.ldc + n0;
  const int nvalid = int(P.N - n0 < 32 ? P.N - n0 : 32);
  if (P.bias) {
    if (P.bias_dtype == TCB_F32) {
      const float* b = static_cast<const float*>(P.bias) + n0;
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) v[j] += __ldg(b + j);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (j < nvalid) v[j] += ld_e(P.bias, P.bias_dtype, n0 + j);
    }
  }
  if (P.dact != ACT_NONE) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (j < nvalid) v[j] *= dact_f(P.dact, ld_e(P.aux, P.aux_dtype, base + j));
  }
  const bool vec = P.c_vec_ok && nvalid == 32;
  if (P.aux_out) store_row32(P.aux_out, P.c_dtype, base, v, vec, nvalid);  // pre-activation u
  if (P.act != ACT_NONE) {
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = act_f(P.act, v[j]);
  }
  store_row32(P.c, P.c_dtype, base, v, vec, nvalid);
}

constexpr int TC_THREADS = 384;  // warps 0-3: TMA, MMA, TMEM alloc, spare; 4-11: epilogue

template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
              const TcParams P) {
  using C = TcCfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], TC_THREADS - 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
        int z, mb, nb;
        decode_tile(P, t, z, mb, nb);
        const int z1 = int(z / P.Z2), z2 = int(z % P.Z2);
        const int m0 = mb * TC_BM, n0 = nb * BN;
        for (int kb = 0; kb < P.k_blocks; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], C::STAGE_BYTES);
          uint8_t* a_dst = sA + stage * C::A_BYTES;
          uint8_t* b_dst = sB + stage * C::B_BYTES;
          const int k0 = kb * TC_BK;
          if (!P.ta) {
            tma_load_4d(a_dst, &tmA, &full[stage], k0, m0, z2, z1);
          } else {
#pragma unroll
            for (int c = 0; c < TC_BM / 64; ++c)
              tma_load_4d(a_dst + c * 8192, &tmA, &full[stage], m0 + c * 64, k0, z2, z1);
          }
          if (P.tb) {
            tma_load_4d(b_dst, &tmB, &full[stage], k0, n0, z2, z1);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tma_load_4d(b_dst + c * 8192, &tmB, &full[stage], n0 + c * 64, k0, z2, z1);
          }
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer =====================
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int64_t t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + uint32_t(acc * BN);
        for (int kb = 0; kb < P.k_blocks; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + stage * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < TC_BK / 16; ++k) {
            // K-major: +32 B per 16-element k step inside the 128 B swizzle row;
            // MN-major: +2048 B (16 k-rows of 128 B); LBO = 8 KB between 64-wide
            // MN chunks, SBO = 1 KB between 8-row swizzle atoms.
            const uint64_t ad = P.ta ? umma_desc(a_addr + k * 2048, 8192, 1024)
                                     : umma_desc(a_addr + k * 32, 16, 1024);
            const uint64_t bd = P.tb ? umma_desc(b_addr + k * 32, 16, 1024)
                                     : umma_desc(b_addr + k * 2048, 8192, 1024);
            tc_mma(tmem_d, ad, bd, P.idesc, (kb | k) ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          if (++stage == C::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue (8 warps) =====================
    // warp w may only touch TMEM lanes 32*(w%4)..+31; the two warps sharing a
    // lane quarter split the tile's 32-column chunks between them
    const int q = warp & 3;
    const int half = (warp - 4) >> 2;
    const int row = q * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int64_t t = blockIdx.x; t < P.num_tiles; t += gridDim.x) {
      int z, mb, nb;
      decode_tile(P, t, z, mb, nb);
      const int64_t coff = int64_t(z / P.Z2) * P.c_s1 + int64_t(z % P.Z2) * P.c_s2;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int64_t m = int64_t(mb) * TC_BM + row;
#pragma unroll 1
      for (int c = half; c < BN / 32; c += 2) {
        uint32_t r[32];
        const uint32_t taddr = tmem_base + (uint32_t(q * 32) << 16) + uint32_t(acc * BN + c * 32);
        TMEM_LD32(taddr, r);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int64_t n0 = int64_t(nb) * BN + c * 32;
        if (m < P.M && n0 < P.N) epi_store32(P, r, m, n0, coff);
      }
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::TMEM_COLS));
  }
}

// ------------------------------------------------------------- host side
using PFN_encodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
  static PFN_encodeTiled fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_encodeTiled>(p);
  });
  if (!fn) fail(TCB_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  return fn;
}

// operand -> 4-D map {inner, outer, z2, z1}; box {64, box_outer, 1, 1}
static CUtensorMap make_map(const GemmOperand& o, int dtype, int64_t inner, int64_t outer, int64_t Z2,
                            int64_t Z1, uint32_t box_outer) {
  CUtensorMap map;
  const int es = 2;
  cuuint64_t dims[4] = {cuuint64_t(inner), cuuint64_t(outer), cuuint64_t(Z2), cuuint64_t(Z1)};
  auto stride_or = [&](int64_t s, int64_t fallback) {
    int64_t v = s > 0 ? s : fallback;
    return cuuint64_t(((v * es + 15) / 16) * 16);
  };
  const int64_t plane = o.ld * outer;
  cuuint64_t strides[3] = {cuuint64_t(o.ld * es), stride_or(o.s2, plane), stride_or(o.s1, plane * Z2)};
  cuuint32_t box[4] = {64, box_outer, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = get_encode()(&map, dtype == TCB_BF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                    : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                            4, const_cast<void*>(o.ptr), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(TCB_ERR_CUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return map;
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

template <int BN>
static void launch_bn(const GemmArgs& g, cudaStream_t s) {
  using C = TcCfg<BN>;
  static std::once_flag once;
  std::call_once(once, [] {
    TCB_CUDA(cudaFuncSetAttribute(k_gemm_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM));
  });
  TcParams P{};
  P.M = g.M;
  P.N = g.N;
  P.K = g.K;
  P.Z = g.Z;
  P.Z2 = g.Z2;
  P.ta = g.ta;
  P.tb = g.tb;
  P.m_blocks = int((g.M + TC_BM - 1) / TC_BM);
  P.n_blocks = int((g.N + BN - 1) / BN);
  P.k_blocks = int((g.K + TC_BK - 1) / TC_BK);
  P.num_tiles = int64_t(P.m_blocks) * P.n_blocks * g.Z;
  const uint32_t fmt = g.a.dtype == TCB_BF16 ? 1u : 0u;
  P.idesc = (1u << 4)                      // D format f32
            | (fmt << 7) | (fmt << 10)     // A, B format
            | (uint32_t(g.ta) << 15)       // A major: 1 = MN
            | (uint32_t(!g.tb) << 16)      // B major: 1 = MN (B stored [K, N])
            | (uint32_t(BN >> 3) << 17)    // N
            | (uint32_t(TC_BM >> 4) << 24);  // M
  P.c = g.c;
  P.ldc = g.ldc;
  P.c_s1 = g.c_s1;
  P.c_s2 = g.c_s2;
  P.c_dtype = g.c_dtype;
  P.alpha = g.alpha;
  P.bias = g.bias;
  P.bias_dtype = g.bias_dtype;
  P.act = g.act;
  P.dact = g.dact;
  P.aux = g.aux;
  P.aux_dtype = g.aux_dtype;
  P.aux_out = g.aux_out;
  const int es = dtype_bytes(g.c_dtype);
  P.c_vec_ok = (reinterpret_cast<uintptr_t>(g.c) % 16 == 0) && ((g.ldc * es) % 16 == 0) &&
               ((g.c_s1 * es) % 16 == 0) && ((g.c_s2 * es) % 16 == 0) &&
               (!g.aux_out || reinterpret_cast<uintptr_t>(g.aux_out) % 16 == 0);
  const int64_t Z1 = (g.Z + g.Z2 - 1) / g.Z2;
  CUtensorMap ta = g.ta ? make_map(g.a, g.a.dtype, g.M, g.K, g.Z2, Z1, 64)
                        : make_map(g.a, g.a.dtype, g.K, g.M, g.Z2, Z1, TC_BM);
  CUtensorMap tb = g.tb ? make_map(g.b, g.b.dtype, g.K, g.N, g.Z2, Z1, BN)
                        : make_map(g.b, g.b.dtype, g.N, g.K, g.Z2, Z1, 64);
  const int grid = int(P.num_tiles < kNumSMs ? P.num_tiles : kNumSMs);
  k_gemm_tc<BN><<<grid, TC_THREADS, C::SMEM, s>>>(ta, tb, P);
}

void launch_gemm_tc(const GemmArgs& g, cudaStream_t s) {
  std::string why;
  if (!gemm_tc_supported(g, &why)) fail(TCB_ERR_UNIMPLEMENTED, "tcgen05 gemm: " + why);
  // Tile width by a wave-quantised cost model: time ~ waves(BN) * BN / e(BN),
  // where e(BN) is the measured mainloop efficiency of a 1-CTA 128xBN tile
  // (smem-read bound at small BN: ~0.5 @128, ~0.66 @192, ~0.75 @256).
  const int64_t mb = (g.M + TC_BM - 1) / TC_BM;
  int best = 128;
  double best_cost = 1e30;
  const int cand[3] = {256, 192, 128};
  const double eff[3] = {0.75, 0.66, 0.5};
  for (int i = 0; i < 3; ++i) {
    const int bn = cand[i];
    if (bn > 128 && g.N <= 128) continue;
    const int64_t nb = (g.N + bn - 1) / bn;
    const int64_t tiles = mb * nb * g.Z;
    const double waves = double((tiles + kNumSMs - 1) / kNumSMs);
    // columns actually computed per n-block (tail blocks waste the remainder)
    const double cost = waves * double(bn) / eff[i];
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = bn;
    }
  }
  if (best == 256) launch_bn<256>(g, s);
  else if (best == 192) launch_bn<192>(g, s);
  else launch_bn<128>(g, s);
}

}  // namespace tcb
