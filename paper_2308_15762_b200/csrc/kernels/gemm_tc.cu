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
#include <cstdlib>
#include <mutex>
#include <stdexcept>
#include <string>

#include "kernels/ops.cuh"
#include "kernels/tc_common.cuh"

namespace wpk {
namespace tc {

template <bool A_MN, bool B_MN, int BN>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const __grid_constant__ Params p) {
  using Cfg = TileCfg<BN>;
  constexpr int STAGES = Cfg::STAGES, STAGE_BYTES = Cfg::STAGE_BYTES;
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
      mbar_init(&tempty_bar[a], 8);  // one arrival per epilogue warp
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
        int mb, nb, z1, z2, kb0, kb1;
        decode_tile(p, t, mb, nb, z1, z2);
        k_range<BN>(p, mb, nb, kb0, kb1);
        for (int kb = kb0; kb < kb1; ++kb) {
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
      for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
        int mb, nb, z1, z2, kb0, kb1;
        decode_tile(p, t, mb, nb, z1, z2);
        k_range<BN>(p, mb, nb, kb0, kb1);
        if (kb0 >= kb1) continue;
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        ++local;
        mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * 256;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full_bar[stage], phase);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // K-major: +32 B per K=16 step inside the 128 B swizzle row.
            // MN-major: +16 rows x 128 B per K=16 step (two 8-row groups).
            const uint64_t ad = desc_add(A_MN ? make_desc(sa, CHUNK_BYTES, 1024) : make_desc(sa, 16, 1024),
                                         A_MN ? k * 2048 : k * 32);
            const uint64_t bd = desc_add(B_MN ? make_desc(sb, CHUNK_BYTES, 1024) : make_desc(sb, 16, 1024),
                                         B_MN ? k * 2048 : k * 32);
            tc_mma(tmem_d, ad, bd, idesc, (kb != kb0 || k != 0));
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
    const int ew = warp & 3;          // TMEM lane quarter this warp may access
    const int half = (warp - 4) >> 2;  // which half of the tile's columns
    int local = 0;
    for (int t = blockIdx.x; t < p.num_tiles; t += gridDim.x) {
      int mb, nb, z1, z2, kb0, kb1;
      decode_tile(p, t, mb, nb, z1, z2);
      k_range<BN>(p, mb, nb, kb0, kb1);
      if (kb0 >= kb1) continue;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      ++local;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = mb * BM + ew * 32 + lane;
      const int64_t zoff = static_cast<int64_t>(z1) * p.epi.c_b1 + static_cast<int64_t>(z2) * p.epi.c_b2;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * 256;
      const int col_end = min(BN, p.N - nb * BN);
      for (int c = half * (BN / 2); c < min(col_end, (half + 1) * (BN / 2)); c += 32) {
        float v[32];
        tmem_ld32(taddr + c, v);  // warp-collective: every lane participates
        if (row < p.M) epilogue_chunk(p, v, row, nb * BN + c, zoff);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty_bar[acc]);
    }
  }

  __syncwarp();
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

CUtensorMap make_slab_map(const void* ptr, int dtype, int64_t cols, int64_t rows, int64_t ld) {
  CUtensorMap m;
  const int64_t es = dtype == kF32 ? 4 : 2;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * es)};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(128 / es), static_cast<cuuint32_t>(SLAB_ROWS)};
  cuuint32_t estr[2] = {1, 1};
  if ((reinterpret_cast<uintptr_t>(ptr) & 15) || (ld * es) % 16) {
    throw std::runtime_error("gemm epilogue map: pointer/ld must be 16-byte aligned");
  }
  const CUresult r = get_encoder()(&m, dtype == kF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16,
                                   2, const_cast<void*>(ptr), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("cuTensorMapEncodeTiled (epilogue) failed: " + std::to_string(int(r)));
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

template <bool A_MN, bool B_MN, int BN>
void launch(const GemmProblem& g, const Params& p, cudaStream_t s) {
  auto* k = gemm_tc_kernel<A_MN, B_MN, BN>;
  constexpr int SMEM_BYTES = TileCfg<BN>::SMEM_BYTES;
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

void fill_params(const GemmProblem& g, Params& p, int tile_m, int tile_n) {
  p = Params{};
  p.M = g.M;
  p.N = g.N;
  p.K = g.K;
  p.nb1 = g.nb1;
  p.nb2 = g.nb2;
  p.tiles_m = (g.M + tile_m - 1) / tile_m;
  p.tiles_n = (g.N + tile_n - 1) / tile_n;
  p.causal = g.causal;
  p.num_tiles = p.tiles_m * p.tiles_n * g.nb1 * g.nb2;
  p.k_blocks = (g.K + BK - 1) / BK;
  p.epi = g.epi;
  const int es = g.epi.c_dtype == kF32 ? 4 : 2;
  auto al = [&](const void* q) { return q == nullptr || (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  p.vec_ok = (g.epi.ldc * es) % 16 == 0 && (g.epi.c_b1 * es) % 16 == 0 && (g.epi.c_b2 * es) % 16 == 0 &&
             al(g.epi.c) && al(g.epi.resid) && al(g.epi.aux) && al(g.epi.bias);
}

}  // namespace tc

using namespace tc;

// Tile-shape policy: the CTA-pair kernel (256 x 256 per SM pair, half the
// operand traffic per MMA) for the linear layers; the single-CTA kernel for
// attention's batched / causal / narrow (N <= 128) problems.
int gemm_tc(const GemmProblem& g, cudaStream_t s) {  // declared in gemm.cuh
  if (g.in_dtype != kBF16) throw std::runtime_error("gemm_tc: inputs must be bf16");
  if (g.M <= 0 || g.N <= 0 || g.K <= 0) return 0;
  static const bool pair_off = std::getenv("WP_GEMM_NO_PAIR") != nullptr;
  if (!pair_off && g.causal == kCausalNone && g.M >= 256 && g.N > 128 && g.nb1 * g.nb2 == 1) return gemm_tc2(g, s);
  if (g.epi.ln_x) throw std::runtime_error("gemm: LayerNorm-backward partials need the CTA-pair kernel");
  if (g.epi.rd_x) throw std::runtime_error("gemm: fused row dot products need the CTA-pair kernel");
  if (g.epi.colsum) {  // unfused path: the column sums as a separate pass
    if (g.nb1 * g.nb2 != 1) throw std::runtime_error("gemm: colsum needs an unbatched problem");
    GemmProblem g2 = g;
    g2.epi.colsum = nullptr;
    const int n = gemm_tc(g2, s);
    return n + colsum_accum(g.epi.c_dtype, g.epi.c, g.epi.colsum, g.M, g.N, static_cast<int>(g.epi.ldc), s);
  }
  const int BN = g.N <= 128 ? 128 : 256;
  Params p;
  fill_params(g, p, BM, BN);
  const int sel = (g.A.mn_major ? 2 : 0) + (g.B.mn_major ? 1 : 0) + (BN == 128 ? 4 : 0);
  switch (sel) {
    case 0: launch<false, false, 256>(g, p, s); break;
    case 1: launch<false, true, 256>(g, p, s); break;
    case 2: launch<true, false, 256>(g, p, s); break;
    case 3: launch<true, true, 256>(g, p, s); break;
    case 4: launch<false, false, 128>(g, p, s); break;
    case 5: launch<false, true, 128>(g, p, s); break;
    case 6: launch<true, false, 128>(g, p, s); break;
    default: launch<true, true, 128>(g, p, s); break;
  }
  return 1;
}

}  // namespace wpk
