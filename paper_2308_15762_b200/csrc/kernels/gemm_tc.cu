// bf16 GEMM on the 5th-generation tensor cores (sm_100a): tcgen05.mma with
// fp32 accumulators in TMEM, operands staged by TMA with 128-byte swizzle,
// warp-specialised persistent CTAs.
//
//   warp 0      TMA producer (one lane): STAGES-deep smem ring, full/empty mbarriers
//   warp 1      MMA issuer (one lane): 4 x tcgen05.mma (K=16) per 64-wide K block
//   warp 2      TMEM owner: allocates 512 columns = two 128x256 fp32 accumulators
//   warps 4-7   epilogue: tcgen05.ld -> fused op (bias / residual / GELU /
//               dGELU / fp32 accumulate) -> global; TMEM buffer released to MMA
// Two accumulators let the epilogue of tile i overlap the MMAs of tile i+1.
//
// Operand majorness is a template parameter: K-major tiles are TMA boxes of
// {64 K, rows}; MN-major tiles are {64 MN, 64 K} boxes, one per 64-wide MN chunk,
// described to the MMA with the canonical SW128 MN-major descriptor
// (LBO = chunk stride, SBO = 8-row group stride).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>

#include "kernels/gemm.cuh"

namespace wpk {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int CHUNK_BYTES = 64 * BK * 2;  // one 64(MN) x 64(K) SW128 box, 8 KB
constexpr int NUM_THREADS = 256;
constexpr int TMEM_COLS = 512;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;

struct Params {
  int M, N, K, nb1, nb2;
  int tiles_m, tiles_n, num_tiles, k_blocks;
  int vec_ok;
  Epilogue epi;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// 32 lanes x 32 consecutive fp32 columns: thread i gets row (lane base + i).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bits.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(lbo_bytes >> 4) << 16) |
         (static_cast<uint64_t>(sbo_bytes >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__device__ __forceinline__ void decode_tile(const Params& p, int t, int& m_blk, int& n_blk, int& z1, int& z2) {
  m_blk = t % p.tiles_m;
  int r = t / p.tiles_m;
  n_blk = r % p.tiles_n;
  const int z = r / p.tiles_n;
  z1 = z % p.nb1;
  z2 = z / p.nb1;
}

__device__ __forceinline__ float load_elem(const void* base, int dtype, int64_t off) {
  return dtype == kF32 ? static_cast<const float*>(base)[off]
                       : __bfloat162float(static_cast<const __nv_bfloat16*>(base)[off]);
}

__device__ __forceinline__ void store_elem(void* base, int dtype, int64_t off, float v) {
  if (dtype == kF32) static_cast<float*>(base)[off] = v;
  else static_cast<__nv_bfloat16*>(base)[off] = __float2bfloat16_rn(v);
}

// Epilogue for one row segment of 32 columns starting at (row, col0).
__device__ __forceinline__ void epilogue_chunk(const Params& p, const float* acc, int row, int col0,
                                               int64_t zoff) {
  const Epilogue& e = p.epi;
  const int64_t base = zoff + static_cast<int64_t>(row) * e.ldc + col0;
  const int ncols = min(32, p.N - col0);
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = acc[i] * e.alpha;
  if (e.bias) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < ncols) v[i] += e.bias[col0 + i];
  }
  const bool vec = p.vec_ok && ncols == 32;
  if (e.mode == kEpiAccum) {  // fp32 C
    float* c = static_cast<float*>(e.c) + base;
    if (vec) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) {
        float4 o = *reinterpret_cast<float4*>(c + i);
        o.x += v[i];
        o.y += v[i + 1];
        o.z += v[i + 2];
        o.w += v[i + 3];
        *reinterpret_cast<float4*>(c + i) = o;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < ncols) c[i] += v[i];
    }
    return;
  }
  if (e.mode == kEpiResidual) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < ncols) v[i] += load_elem(e.resid, e.c_dtype, base + i);
  } else if (e.mode == kEpiGelu) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      if (i < ncols) {
        // GELU of the pre-activation as stored, so backward sees the same value.
        const float pre = e.c_dtype == kF32 ? v[i] : __bfloat162float(__float2bfloat16_rn(v[i]));
        store_elem(e.aux, e.c_dtype, base + i, pre);
        v[i] = gelu_f(pre);
      }
    }
  } else if (e.mode == kEpiDGelu) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (i < ncols) v[i] *= gelu_grad_f(load_elem(e.aux, e.c_dtype, base + i));
  }
  if (e.c_dtype == kBF16) {
    __nv_bfloat16* c = static_cast<__nv_bfloat16*>(e.c) + base;
    if (vec) {
#pragma unroll
      for (int i = 0; i < 32; i += 8) {
        uint4 pk;
        __nv_bfloat162 h0 = __floats2bfloat162_rn(v[i], v[i + 1]);
        __nv_bfloat162 h1 = __floats2bfloat162_rn(v[i + 2], v[i + 3]);
        __nv_bfloat162 h2 = __floats2bfloat162_rn(v[i + 4], v[i + 5]);
        __nv_bfloat162 h3 = __floats2bfloat162_rn(v[i + 6], v[i + 7]);
        pk.x = *reinterpret_cast<uint32_t*>(&h0);
        pk.y = *reinterpret_cast<uint32_t*>(&h1);
        pk.z = *reinterpret_cast<uint32_t*>(&h2);
        pk.w = *reinterpret_cast<uint32_t*>(&h3);
        *reinterpret_cast<uint4*>(c + i) = pk;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < ncols) c[i] = __float2bfloat16_rn(v[i]);
    }
  } else {
    float* c = static_cast<float*>(e.c) + base;
    if (vec) {
#pragma unroll
      for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(c + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i < ncols) c[i] = v[i];
    }
  }
}

template <bool A_MN, bool B_MN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty_bar = full_bar + STAGES;
  uint64_t* tfull_bar = empty_bar + STAGES;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;      // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------------------------------------------------------- TMA
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int mb, nb, z1, z2;
        decode_tile(p, t, mb, nb, z1, z2);
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(&full_bar[stage], STAGE_BYTES);
          if (!A_MN) {
            tma_load_4d(&map_a, &full_bar[stage], sa, kb * BK, mb * BM, z1, z2);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_4d(&map_a, &full_bar[stage], sa + j * CHUNK_BYTES, mb * BM + j * 64, kb * BK, z1, z2);
          }
          if (!B_MN) {
            tma_load_4d(&map_b, &full_bar[stage], sb, kb * BK, nb * BN, z1, z2);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j)
              tma_load_4d(&map_b, &full_bar[stage], sb + j * CHUNK_BYTES, nb * BN + j * 64, kb * BK, z1, z2);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------------- MMA
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(A_MN) << 15) |
                                 (uint32_t(B_MN) << 16) | (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < p.k_blocks; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: +32 B per K=16 step inside the 128 B swizzle row.
            // MN-major: +16 rows x 128 B per K=16 step (two 8-row groups).
            const uint64_t ad = A_MN ? make_desc(sa + k * 2048, CHUNK_BYTES, 1024) : make_desc(sa + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? make_desc(sb + k * 2048, CHUNK_BYTES, 1024) : make_desc(sb + k * 32, 16, 1024);
            tc_mma(tmem_d, ad, bd, idesc, (kb | k) != 0);
          }
          tc_commit(&empty_bar[stage]);  // smem slot free once these MMAs retire
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc_commit(&tfull_bar[acc]);  // accumulator ready for the epilogue
      }
    }
  } else if (warp >= 4) {
    // -------------------------------------------------------------- epilogue
    const int ew = warp & 3;  // TMEM lane quarter this warp may access
    int local = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x, ++local) {
      int mb, nb, z1, z2;
      decode_tile(p, t, mb, nb, z1, z2);
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = mb * BM + ew * 32 + lane;
      const int64_t zoff = static_cast<int64_t>(z1) * p.epi.c_b1 + static_cast<int64_t>(z2) * p.epi.c_b2;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * BN;
      const int col_end = min(BN, p.N - nb * BN);
      for (int c = 0; c < col_end; c += 32) {
        float v[32];
        tmem_ld32(taddr + c, v);  // warp-collective: every lane participates
        if (row < p.M) epilogue_chunk(p, v, row, nb * BN + c, zoff);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
    }
  }

  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// ------------------------------------------------------------------ host side

PFN_cuTensorMapEncodeTiled_v12000 get_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* ptr = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess) {
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
  });
  if (!fn) throw std::runtime_error("cuTensorMapEncodeTiled unavailable");
  return fn;
}

// 4-D bf16 map {inner, outer, nb1, nb2}; box {64, box_outer, 1, 1}, SW128.
CUtensorMap make_map(const Operand& op, int64_t inner, int64_t outer, int nb1, int nb2, int box_outer) {
  CUtensorMap m;
  const int64_t es = 2;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer),
                        static_cast<cuuint64_t>(nb1), static_cast<cuuint64_t>(nb2)};
  auto fix = [](int64_t bytes) { return static_cast<cuuint64_t>(bytes <= 0 ? 16 : ((bytes + 15) / 16) * 16); };
  cuuint64_t strides[3] = {fix(op.ld * es), fix(nb1 > 1 ? op.b1 * es : op.ld * es * outer),
                           fix(nb2 > 1 ? op.b2 * es : op.ld * es * outer)};
  cuuint32_t box[4] = {64, static_cast<cuuint32_t>(box_outer), 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  if ((reinterpret_cast<uintptr_t>(op.ptr) & 15) || (op.ld * es) % 16 || (nb1 > 1 && (op.b1 * es) % 16) ||
      (nb2 > 1 && (op.b2 * es) % 16)) {
    throw std::runtime_error("gemm_tc: operand pointer/strides must be 16-byte aligned");
  }
  CUresult r = get_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(op.ptr), dims, strides, box,
                             estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
  return m;
}

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  }
  return n;
}

template <bool A_MN, bool B_MN>
void launch(const GemmProblem& g, const Params& p, cudaStream_t s) {
  auto* k = gemm_tc_kernel<A_MN, B_MN>;
  static uint64_t attr_done = 0;  // one bit per CUDA device
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_done >> (dev & 63) & 1)) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    attr_done |= 1ull << (dev & 63);
  }
  const CUtensorMap ma = A_MN ? make_map(g.A, g.M, g.K, g.nb1, g.nb2, 64) : make_map(g.A, g.K, g.M, g.nb1, g.nb2, BM);
  const CUtensorMap mbm = B_MN ? make_map(g.B, g.N, g.K, g.nb1, g.nb2, 64) : make_map(g.B, g.K, g.N, g.nb1, g.nb2, BN);
  const int grid = std::min(p.num_tiles, num_sms());
  k<<<grid, NUM_THREADS, SMEM_BYTES, s>>>(ma, mbm, p);
}

}  // namespace

int gemm_tc(const GemmProblem& g, cudaStream_t s) {  // declared in gemm.cuh
  if (g.in_dtype != kBF16) throw std::runtime_error("gemm_tc: inputs must be bf16");
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return 0;
  Params p{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.nb1 = g.nb1;
  p.nb2 = g.nb2;
  p.tiles_m = (g.M + BM - 1) / BM;
  p.tiles_n = (g.N + BN - 1) / BN;
  p.num_tiles = p.tiles_m * p.tiles_n * g.nb1 * g.nb2;
  p.k_blocks = (g.K + BK - 1) / BK;
  p.epi = g.epi;
  const int es = g.epi.c_dtype == kF32 ? 4 : 2;
  auto al = [&](const void* q) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  p.vec_ok = (g.epi.ldc * es) % 16 == 0 && (g.epi.c_b1 * es) % 16 == 0 && (g.epi.c_b2 * es) % 16 == 0 &&
             al(g.epi.c) && al(g.epi.resid) && al(g.epi.aux);
  if (!g.A.mn_major && !g.B.mn_major) launch<false, false>(g, p, s);
  else if (!g.A.mn_major && g.B.mn_major) launch<false, true>(g, p, s);
  else if (g.A.mn_major && !g.B.mn_major) launch<true, false>(g, p, s);
  else launch<true, true>(g, p, s);
  return 1;
}

}  // namespace wpk
