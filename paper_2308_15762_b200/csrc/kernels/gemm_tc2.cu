// bf16 GEMM on a CTA pair (tcgen05.mma.cta_group::2): one 256 x 256 output
// tile per SM pair of a 2-CTA cluster.  Each CTA stages its own 128 rows of A
// and its own 128 columns of B (TMA .cta_group::2, bytes counted on the
// leader's barrier); the leader's single MMA thread issues M=256, N=256,
// K=16 instructions that read both CTAs' shared memory and accumulate rows
// 0-127 into the leader's TMEM and rows 128-255 into the peer's.  Per SM and
// K block that is 32 KB of operand traffic for 128x256x64 MACs -- two thirds
// of the 1-CTA 128 x 256 tile's 48 KB -- which is what lets the tensor pipe
// stay fed from L2.
//
//   warp 0      TMA producer (both CTAs): 6-stage ring of 32 KB stages
//   warp 1      MMA issuer (leader only): commits multicast to both CTAs
//   warp 2      TMEM owner (cta_group::2 alloc/dealloc in both CTAs)
//   warps 4-11  epilogue (both CTAs): own TMEM rows -> fused op -> global;
//               release the accumulator on the leader's barrier (16 arrivals)
//
// Epilogue (TE=true, every aligned problem): each epilogue warp owns a 32-row
// x 128-column block of its CTA's 128 x 256 accumulator and moves it through
// two 4 KB SW128 smem slabs (32 rows x 128 bytes): tcgen05.ld -> bias / GELU
// / dGELU / residual in registers -> slab -> one TMA bulk tensor store per
// slab (fp32 gradient accumulation uses the TMA reduce-add store, so C is
// never read by the SM).  Residual and GELU-input tiles arrive by TMA into the
// same slab.  Global traffic is then whole 128-byte rows per request instead
// of one row per lane; the ring drops to 5 stages to make room (64 KB slabs).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

#include "kernels/tc_common.cuh"

namespace wpk {
namespace tc {
namespace {

constexpr int PBN = 256;           // pair tile N
constexpr int HALF_N = PBN / 2;    // columns staged per CTA
constexpr int PM = 2 * BM;         // pair tile M
constexpr int P_STAGE_BYTES = A_BYTES + HALF_N * BK * 2;  // 32 KB
constexpr int EPI_WARPS = 8;
constexpr int STG_BYTES = EPI_WARPS * 2 * SLAB_BYTES;  // 64 KB of epilogue slabs

template <bool TE>
struct PairCfg {
  static constexpr int STAGES = TE ? 5 : 6;
  static constexpr int SMEM_BYTES = STAGES * P_STAGE_BYTES + (TE ? STG_BYTES : 0) + 1024 + 512;
};

// One slab of the TMA epilogue: CPC accumulator columns (64 bf16 / 32 fp32)
// of the warp's 32 rows starting at (row0, gcol); see the file header.
template <int CPC>
__device__ __forceinline__ void epi_slab(const Params& p, const CUtensorMap* map_c, const CUtensorMap* map_x,
                                         uint8_t* slabs, uint64_t* sbar, uint32_t& sphase, int& buf, uint32_t taddr,
                                         int gcol, int row0, int lane, const float* bias, bool prefetched = false) {
  const Epilogue& e = p.epi;
  const int mode = e.mode;
  constexpr int dt = CPC == 32 ? kF32 : kBF16;
  const bool needs_in = mode == kEpiResidual || mode == kEpiDGelu;
  uint8_t* sb = slabs + buf * SLAB_BYTES;
  const bool ln = CPC == 64 && e.ln_x != nullptr;  // LayerNorm-backward partials (store mode, bf16 C)
  const bool rd = CPC == 64 && e.rd_x != nullptr;  // row dot products with rd_x (store mode, bf16 C)
  const bool aux2 = ln || rd;                      // a second input slab, loaded into xb
  const int xb = buf ^ 1;                          // the LN input slab (buf flips below)
  uint8_t* sx = slabs + xb * SLAB_BYTES;
  // prefetched: the input slab was loaded (into slab `buf`) by the caller a
  // tile ahead, after the slabs' previous stores had read them
  if (lane == 0 && !prefetched) {
    // the slab(s) about to be written must have been read out by earlier stores
    if (mode == kEpiGelu || aux2) bulk_wait_read<0>();
    else bulk_wait_read<1>();
  }
  __syncwarp();
  if (needs_in && lane == 0 && !prefetched) {
    mbar_expect_tx(&sbar[buf], SLAB_BYTES);
    tma_load_2d(map_x, &sbar[buf], sb, gcol, row0);
  }
  if (aux2 && lane == 0) {
    mbar_expect_tx(&sbar[xb], SLAB_BYTES);
    tma_load_2d(map_x, &sbar[xb], sx, gcol, row0);
  }
  float v[CPC];
  tmem_ld32(taddr, v);
  if constexpr (CPC == 64) tmem_ld32(taddr + 32, v + 32);
  // alpha / bias with packed f32x2 arithmetic (the epilogue warps share
  // their sub-partitions with the MMA issuer: fewer issue slots here keep
  // the tensor pipe fed); no work at all for alpha = 1 without a bias.
  const float2 al2 = make_float2(e.alpha, e.alpha);
  if (bias && gcol + CPC <= p.N) {
#pragma unroll
    for (int i = 0; i < CPC; i += 4) {
      const float4 b4 = *reinterpret_cast<const float4*>(bias + gcol + i);
      const float2 r0 = smx::ffma2(make_float2(v[i], v[i + 1]), al2, make_float2(b4.x, b4.y));
      const float2 r1 = smx::ffma2(make_float2(v[i + 2], v[i + 3]), al2, make_float2(b4.z, b4.w));
      v[i] = r0.x, v[i + 1] = r0.y, v[i + 2] = r1.x, v[i + 3] = r1.y;
    }
  } else if (bias) {
#pragma unroll
    for (int i = 0; i < CPC; ++i) v[i] = v[i] * e.alpha + (gcol + i < p.N ? bias[gcol + i] : 0.f);
  } else if (e.alpha != 1.f) {
#pragma unroll
    for (int i = 0; i < CPC; i += 2) {
      const float2 r = smx::fmul2(make_float2(v[i], v[i + 1]), al2);
      v[i] = r.x, v[i + 1] = r.y;
    }
  }
  if (needs_in) {
    mbar_wait(&sbar[buf], (sphase >> buf) & 1);
    sphase ^= 1u << buf;
    float x[CPC];
    if constexpr (CPC == 32) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const float4 f = *reinterpret_cast<const float4*>(sb + slab_off(lane, q));
        x[4 * q] = f.x, x[4 * q + 1] = f.y, x[4 * q + 2] = f.z, x[4 * q + 3] = f.w;
      }
    } else {
      slab_get_bf16(sb, lane, x);
    }
    if (mode == kEpiResidual) {
#pragma unroll
      for (int i = 0; i < CPC; i += 2) {
        const float2 r = smx::fadd2(make_float2(v[i], v[i + 1]), make_float2(x[i], x[i + 1]));
        v[i] = r.x, v[i + 1] = r.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < CPC; i += 2) {
        const float2 gg = gelu_grad_fast2(make_float2(x[i], x[i + 1]));
        const float2 r = smx::fmul2(make_float2(v[i], v[i + 1]), gg);
        v[i] = r.x, v[i + 1] = r.y;
      }
    }
  }
  auto put = [&](uint8_t* slab) {
    if constexpr (CPC == 32) slab_put_f32(slab, lane, v);
    else slab_put_bf16(slab, lane, v);
  };
  if (mode == kEpiGelu) {
    uint8_t* sg = slabs + (buf ^ 1) * SLAB_BYTES;
    // GELU of the stored (bf16-rounded) pre-activation: round once, packed,
    // and store the packed words as they are.
    if constexpr (CPC == 64) {
      uint32_t pk[CPC / 2];
#pragma unroll
      for (int i = 0; i < CPC; i += 2) {
        const __nv_bfloat162 h = __floats2bfloat162_rn(v[i], v[i + 1]);
        pk[i / 2] = *reinterpret_cast<const uint32_t*>(&h);
        const float2 f = __bfloat1622float2(h);
        v[i] = f.x, v[i + 1] = f.y;
      }
      slab_put_bf16_packed(sb, lane, pk);
    } else {
#pragma unroll
      for (int i = 0; i < CPC; ++i) v[i] = round_to(dt, v[i]);
      put(sb);
    }
#pragma unroll
    for (int i = 0; i < CPC; i += 2) {
      const float2 r = gelu_fast2(make_float2(v[i], v[i + 1]));
      v[i] = r.x, v[i + 1] = r.y;
    }
    put(sg);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      tma_store_2d(map_x, sb, gcol, row0);
      tma_store_2d(map_c, sg, gcol, row0);
      bulk_commit();
    }
  } else {
    put(sb);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (mode == kEpiAccum) tma_reduce_add_2d(map_c, sb, gcol, row0);
      else tma_store_2d(map_c, sb, gcol, row0);
      bulk_commit();
    }
    buf ^= 1;
  }
  if (ln) {
    // LayerNorm-backward partials of this slab (v = dLN, still intact):
    // per-row sums of g = dLN * w and g * xhat, and dw's column sums of
    // dLN * xhat (db is the colsum below).
    mbar_wait(&sbar[xb], (sphase >> xb) & 1);
    sphase ^= 1u << xb;
    float xv[CPC];
    slab_get_bf16(sx, lane, xv);
    const int row = row0 + lane;
    const bool valid = row < p.M;
    const float mu = valid ? e.ln_mean[row] : 0.f, rs = valid ? e.ln_rstd[row] : 0.f;
    float sg = 0.f, sgx = 0.f;
#pragma unroll
    for (int i = 0; i < CPC; ++i) {
      const float wv = gcol + i < p.N ? e.ln_w[gcol + i] : 0.f;
      const float xh = (xv[i] - mu) * rs;
      const float g = v[i] * wv;
      sg += g;
      sgx += g * xh;
      xv[i] = valid ? v[i] * xh : 0.f;  // dw term
    }
    if (valid) {
      atomicAdd(e.ln_rows + 2 * row, sg);
      atomicAdd(e.ln_rows + 2 * row + 1, sgx);
    }
#pragma unroll
    for (int q = 0; q < CPC / 32; ++q) {
      float* w = xv + 32 * q;
#pragma unroll
      for (int sh = 16; sh >= 1; sh >>= 1) {
        const bool up = (lane & sh) != 0;
#pragma unroll
        for (int i = 0; i < sh; ++i) {
          const float send = up ? w[i] : w[i + sh];
          const float keep = up ? w[i + sh] : w[i];
          w[i] = keep + __shfl_xor_sync(0xffffffffu, send, sh);
        }
      }
      const int col = gcol + 32 * q + lane;
      if (col < p.N) atomicAdd(e.ln_dw + col, w[0]);
    }
  }
  if (rd) {
    mbar_wait(&sbar[xb], (sphase >> xb) & 1);
    sphase ^= 1u << xb;
    float xv[CPC];
    slab_get_bf16(sx, lane, xv);
    const int row = row0 + lane;
    if (row < p.M && gcol < p.N) {
      // dot of the bf16-rounded row with x: packed rounding and FFMA2 into
      // two independent pair accumulators
      float2 acc2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int i = 0; i < CPC; i += 2) {
        const float2 rv = __bfloat1622float2(__floats2bfloat162_rn(v[i], v[i + 1]));
        acc2[(i >> 1) & 1] = smx::ffma2(rv, make_float2(xv[i], xv[i + 1]), acc2[(i >> 1) & 1]);
      }
      const float acc = (acc2[0].x + acc2[0].y) + (acc2[1].x + acc2[1].y);
      const int64_t ngrp = p.N / e.rd_group;
      atomicAdd(e.rd_out + (row / e.rd_seq * ngrp + gcol / e.rd_group) * e.rd_seq + row % e.rd_seq, acc);
    }
  }
  if (e.colsum && CPC == 64 && mode != kEpiGelu) {
    // Column sums of the bf16 C just staged (the stored values, which are
    // what the next GEMMs and the reference's rounding points see): lane l
    // reads columns 2l, 2l+1 down the slab's 32 rows (one 128-byte row per
    // warp load, conflict-free) -- half the instructions of the butterfly
    // below; rows past M skipped.
    __syncwarp();
    const int rows = min(32, p.M - row0);
    float2 cs = make_float2(0.f, 0.f);
#pragma unroll 8
    for (int r = 0; r < rows; ++r) {
      const uint32_t u = *reinterpret_cast<const uint32_t*>(sb + slab_off(r, lane >> 2) + (lane & 3) * 4);
      cs = smx::fadd2(cs, __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u)));
    }
    const int col = gcol + 2 * lane;
    if (col < p.N) atomicAdd(e.colsum + col, cs.x);
    if (col + 1 < p.N) atomicAdd(e.colsum + col + 1, cs.y);
  } else if (e.colsum) {
    // Column sums of this slab's 32 rows (one per lane): a transposing
    // butterfly leaves column (32q + lane) in v[32q] after 31 shuffles per 32
    // columns, then one atomic per column per warp (rows past M masked).
    if (row0 + lane >= p.M)
#pragma unroll
      for (int i = 0; i < CPC; ++i) v[i] = 0.f;
#pragma unroll
    for (int q = 0; q < CPC / 32; ++q) {
      float* w = v + 32 * q;
#pragma unroll
      for (int sh = 16; sh >= 1; sh >>= 1) {
        const bool up = (lane & sh) != 0;
#pragma unroll
        for (int i = 0; i < sh; ++i) {
          const float send = up ? w[i] : w[i + sh];
          const float keep = up ? w[i + sh] : w[i];
          w[i] = keep + __shfl_xor_sync(0xffffffffu, send, sh);
        }
      }
      const int col = gcol + 32 * q + lane;
      if (col < p.N) atomicAdd(e.colsum + col, w[0]);
    }
  }
}

template <bool A_MN, bool B_MN, bool TE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(NUM_THREADS, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                    const __grid_constant__ CUtensorMap map_c, const __grid_constant__ CUtensorMap map_x,
                    const __grid_constant__ Params p) {
  constexpr int P_STAGES = PairCfg<TE>::STAGES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* stg = smem + P_STAGES * P_STAGE_BYTES;  // epilogue slabs (TE)
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(stg + (TE ? STG_BYTES : 0));
  uint64_t* empty_bar = full_bar + P_STAGES;
  uint64_t* tfull_bar = empty_bar + P_STAGES;  // [2]
  uint64_t* tempty_bar = tfull_bar + 2;        // [2]
  uint64_t* slab_bar = tempty_bar + 2;         // [EPI_WARPS][2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(slab_bar + 2 * EPI_WARPS);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < P_STAGES; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull_bar[a], 1);
      mbar_init(&tempty_bar[a], 16);  // 8 epilogue warps x 2 CTAs (leader's copy is used)
    }
    for (int i = 0; i < 2 * EPI_WARPS; ++i) mbar_init(&slab_bar[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised before any remote arrive / TMA
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int u = pair; u < p.num_tiles * p.k_split; u += npairs) {
        int mb, nb, z1 = 0, z2 = 0;
        decode_tile_grouped(p, u / p.k_split, mb, nb);
        const int kb0 = (u % p.k_split) * p.kb_per, kb1 = min(p.k_blocks, kb0 + p.kb_per);
        const int row0 = mb * PM + static_cast<int>(rank) * BM;
        const int col0 = nb * PBN + static_cast<int>(rank) * HALF_N;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t* sa = smem + stage * P_STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          if (leader) mbar_expect_tx(&full_bar[stage], 2 * P_STAGE_BYTES);
          if (!A_MN) {
            tma_load_4d_pair(&map_a, &full_bar[stage], sa, kb * BK, row0, z1, z2);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j)
              tma_load_4d_pair(&map_a, &full_bar[stage], sa + j * CHUNK_BYTES, row0 + j * 64, kb * BK, z1, z2);
          }
          if (!B_MN) {
            tma_load_4d_pair(&map_b, &full_bar[stage], sb, kb * BK, col0, z1, z2);
          } else {
#pragma unroll
            for (int j = 0; j < HALF_N / 64; ++j)
              tma_load_4d_pair(&map_b, &full_bar[stage], sb + j * CHUNK_BYTES, col0 + j * 64, kb * BK, z1, z2);
          }
          if (++stage == P_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // The whole warp walks the loop with warp-uniform state (shared-memory
      // base from the extern array, TMEM base broadcast, stage / phase from
      // an induction counter, vote-based barrier waits) and one elected lane
      // issues: the compiler then keeps the descriptors in uniform registers
      // and the MMAs go out back to back (see elect_one).
      const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint32_t sbase = (smem_u32(smem_raw) + 1023u) & ~1023u;
      if (sbase != smem_u32(smem)) __trap();  // shared-space and generic alignment must agree
      constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(A_MN) << 15) |
                                 (uint32_t(B_MN) << 16) | (uint32_t(PBN >> 3) << 17) | (uint32_t(PM >> 4) << 24);
      int it = 0;  // k-blocks consumed (all tiles): stage = it % P_STAGES
      int local = 0;
      for (int u = pair; u < p.num_tiles * p.k_split; u += npairs, ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (local >> 1) & 1;
        mbar_wait_warp(&tempty_bar[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tbase + acc * PBN;
        const int kb0 = (u % p.k_split) * p.kb_per, kb1 = min(p.k_blocks, kb0 + p.kb_per);
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int stage = it % P_STAGES;
          mbar_wait_warp(&full_bar[stage], (it / P_STAGES) & 1);
          tc_fence_after();
          const uint32_t sa = sbase + stage * P_STAGE_BYTES;
          const uint32_t sb = sa + A_BYTES;
          const uint64_t ad0 = A_MN ? make_desc(sa, CHUNK_BYTES, 1024) : make_desc(sa, 16, 1024);
          const uint64_t bd0 = B_MN ? make_desc(sb, CHUNK_BYTES, 1024) : make_desc(sb, 16, 1024);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            if (elect_one())
              tc_mma_pair(tmem_d, desc_add(ad0, A_MN ? k * 2048 : k * 32), desc_add(bd0, B_MN ? k * 2048 : k * 32),
                          idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          if (elect_one()) tc_commit_pair(&empty_bar[stage]);  // frees this stage in both CTAs
          __syncwarp();
        }
        if (elect_one()) tc_commit_pair(&tfull_bar[acc]);  // both halves of the accumulator ready
        __syncwarp();
      }
    }
  } else if (warp >= 4 && TE) {
    const int ew = warp & 3;
    const int half = (warp - 4) >> 2;
    const bool f32 = p.epi.mode == kEpiAccum || p.epi.c_dtype == kF32;
    const int cpc = f32 ? 32 : 64;  // columns per slab
    uint8_t* slabs = stg + (warp - 4) * 2 * SLAB_BYTES;
    uint64_t* sbar = slab_bar + (warp - 4) * 2;
    uint32_t sphase = 0;
    int buf = 0;
    int local = 0;
    // dGELU with a bf16 C: the warp's two 64-column pre-activation slabs of a
    // tile are loaded one tile ahead (once the previous tile's stores have
    // read the slabs), so their latency hides behind the mainloop -- what
    // the short-K FC2 data gradients (K = hidden) need; the residual mode
    // measured better without it.
    const bool pre = p.epi.mode == kEpiDGelu && !f32 && !p.epi.ln_x && !p.epi.rd_x;
    auto prefetch = [&](int u) {
      int mb, nb;
      decode_tile_grouped(p, u / p.k_split, mb, nb);
      const int row0 = mb * PM + static_cast<int>(rank) * BM + ew * 32;
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int gcol = nb * PBN + half * (PBN / 2) + i * 64;
        if (gcol >= p.N) break;
        mbar_expect_tx(&sbar[i], SLAB_BYTES);
        tma_load_2d(&map_x, &sbar[i], slabs + i * SLAB_BYTES, gcol, row0);
      }
    };
    if (pre && lane == 0 && pair < p.num_tiles * p.k_split) prefetch(pair);
    for (int u = pair; u < p.num_tiles * p.k_split; u += npairs, ++local) {
      int mb, nb;
      decode_tile_grouped(p, u / p.k_split, mb, nb);
      const float* bias = u % p.k_split == 0 ? p.epi.bias : nullptr;  // split-K: bias once
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row0 = mb * PM + static_cast<int>(rank) * BM + ew * 32;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * PBN;
      for (int c = half * (PBN / 2), i = 0; c < (half + 1) * (PBN / 2); c += cpc, ++i) {
        const int gcol = nb * PBN + c;
        if (gcol >= p.N) break;
        if (pre) buf = i;
        if (f32) epi_slab<32>(p, &map_c, &map_x, slabs, sbar, sphase, buf, taddr + c, gcol, row0, lane, bias);
        else epi_slab<64>(p, &map_c, &map_x, slabs, sbar, sphase, buf, taddr + c, gcol, row0, lane, bias, pre);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&tempty_bar[acc], 0);
      if (pre && lane == 0 && u + npairs < p.num_tiles * p.k_split) {
        bulk_wait_read<0>();  // this tile's stores have read both slabs
        prefetch(u + npairs);
      }
    }
    if (lane == 0) bulk_wait<0>();
  } else if (warp >= 4) {
    const int ew = warp & 3;
    const int half = (warp - 4) >> 2;
    int local = 0;
    for (int t = pair; t < p.num_tiles; t += npairs, ++local) {
      int mb, nb, z1, z2;
      decode_tile_grouped(p, t, mb, nb);
        z1 = z2 = 0;
      const int acc = local & 1;
      const uint32_t acc_phase = (local >> 1) & 1;
      mbar_wait(&tfull_bar[acc], acc_phase);
      tc_fence_after();
      const int row = mb * PM + static_cast<int>(rank) * BM + ew * 32 + lane;
      const int64_t zoff = static_cast<int64_t>(z1) * p.epi.c_b1 + static_cast<int64_t>(z2) * p.epi.c_b2;
      const uint32_t taddr = tmem_base + (static_cast<uint32_t>(ew * 32) << 16) + acc * PBN;
      const int col_end = min(PBN, p.N - nb * PBN);
      for (int c = half * (PBN / 2); c < min(col_end, (half + 1) * (PBN / 2)); c += 32) {
        float v[32];
        tmem_ld32(taddr + c, v);
        if (row < p.M) epilogue_chunk(p, v, row, nb * PBN + c, zoff);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(&tempty_bar[acc], 0);
    }
  }

  tc_fence_before();
  __syncwarp();
  cluster_sync();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

template <bool A_MN, bool B_MN, bool TE>
void launch_pair(const GemmProblem& g, const Params& p, cudaStream_t s) {
  auto* k = gemm_tc2_kernel<A_MN, B_MN, TE>;
  constexpr int SMEM = PairCfg<TE>::SMEM_BYTES;
  static uint64_t attr_done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_done >> (dev & 63) & 1)) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    attr_done |= 1ull << (dev & 63);
  }
  const CUtensorMap ma = A_MN ? make_map(g.A, g.M, g.K, g.nb1, g.nb2, 64) : make_map(g.A, g.K, g.M, g.nb1, g.nb2, BM);
  const CUtensorMap mb =
      B_MN ? make_map(g.B, g.N, g.K, g.nb1, g.nb2, 64) : make_map(g.B, g.K, g.N, g.nb1, g.nb2, HALF_N);
  CUtensorMap mc{}, mx{};
  if (TE) {
    const Epilogue& e = g.epi;
    const int dt = e.mode == kEpiAccum ? kF32 : e.c_dtype;
    mc = make_slab_map(e.c, dt, g.N, g.M, e.ldc);
    const void* x = e.mode == kEpiResidual ? e.resid
                    : (e.mode == kEpiGelu || e.mode == kEpiDGelu) ? e.aux
                    : e.ln_x                                      ? e.ln_x
                                                                  : e.rd_x;
    mx = x ? make_slab_map(x, dt, g.N, g.M, e.ldc) : mc;
  }
  const int pairs = std::min(p.num_tiles * std::max(1, p.k_split), num_sms() / 2);
  k<<<2 * pairs, NUM_THREADS, SMEM, s>>>(ma, mb, mc, mx, p);
}

}  // namespace

int gemm_tc2(const GemmProblem& g, cudaStream_t s) {
  Params p;
  fill_params(g, p, PM, PBN);
  static const int gm_env = std::getenv("WP_GEMM_GROUP_M") ? std::atoi(std::getenv("WP_GEMM_GROUP_M")) : 8;
  p.group_m = std::max(1, std::min(gm_env, p.tiles_m));
  static const bool te_off = std::getenv("WP_GEMM_NO_TMA_EPI") != nullptr;  // A/B switch for profiling
  const bool te = p.vec_ok && !te_off;
  if (g.epi.ln_x && (!te || g.epi.mode != kEpiStore || g.epi.c_dtype != kBF16)) {
    throw std::runtime_error("gemm: LayerNorm-backward partials need the TMA epilogue, store mode and a bf16 C");
  }
  if (g.epi.rd_x && (!te || g.epi.mode != kEpiStore || g.epi.c_dtype != kBF16 || g.epi.ln_x || g.epi.rd_group % 64 ||
                     g.N % g.epi.rd_group || g.epi.rd_seq <= 0)) {
    throw std::runtime_error("gemm: fused row dot products need the TMA epilogue, store mode, a bf16 C, no LN "
                             "partials and 64-column-aligned groups");
  }
  // Split-K for the fp32 gradient accumulation (the TMA reduce-add epilogue
  // makes partial tiles commutative): a 2-way split when it fills the last
  // wave of SM pairs better; 3-4 ways only for long K ranges (>= 64 blocks)
  // and a clearly better last wave (shorter ranges lose more to pipeline
  // fill and fp32 reduce traffic than the wave gains).
  p.k_split = 1;
  p.kb_per = p.k_blocks;
  static const bool split_off = std::getenv("WP_GEMM_NO_SPLITK") != nullptr;
  if (te && !split_off && g.epi.mode == kEpiAccum) {
    const int pairs = num_sms() / 2;
    double best = 0.0;
    for (int s = 1; s <= 4 && p.k_blocks / s >= (s <= 2 ? 32 : 64); ++s) {
      const int per = (p.k_blocks + s - 1) / s, parts = (p.k_blocks + per - 1) / per;
      const int64_t units = int64_t(p.num_tiles) * parts;
      const double eff = double(units) / (double((units + pairs - 1) / pairs) * pairs);
      if (eff > best + (s <= 2 ? 0.02 : 0.06)) {
        best = eff;
        p.k_split = parts;
        p.kb_per = per;
      }
    }
  }
  const int sel = (g.A.mn_major ? 2 : 0) + (g.B.mn_major ? 1 : 0) + (te ? 4 : 0);
  switch (sel) {
    case 0: launch_pair<false, false, false>(g, p, s); break;
    case 1: launch_pair<false, true, false>(g, p, s); break;
    case 2: launch_pair<true, false, false>(g, p, s); break;
    case 3: launch_pair<true, true, false>(g, p, s); break;
    case 4: launch_pair<false, false, true>(g, p, s); break;
    case 5: launch_pair<false, true, true>(g, p, s); break;
    case 6: launch_pair<true, false, true>(g, p, s); break;
    default: launch_pair<true, true, true>(g, p, s); break;
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("gemm_tc2 launch: ") + cudaGetErrorString(e));
  return 1;
}

}  // namespace tc
}  // namespace wpk
