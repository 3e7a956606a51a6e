// Shared pieces of the tcgen05 GEMM kernels (1-CTA gemm_tc.cu, CTA-pair
// gemm_tc2.cu): PTX wrappers for mbarrier / TMA / tcgen05, the SW128 smem
// descriptor, tile decoding and the fused epilogue.
#pragma once

#include "kernels/softmax_math.cuh"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <cstdint>

#include "kernels/gemm.cuh"

namespace wpk {
namespace tc {

constexpr int BM = 128, BK = 64;
constexpr int A_BYTES = BM * BK * 2;      // 16 KB
constexpr int CHUNK_BYTES = 64 * BK * 2;  // one 64(MN) x 64(K) SW128 box, 8 KB
constexpr int NUM_THREADS = 384;  // warps 0-3 control, 4-11 epilogue (two column halves)
constexpr int TMEM_COLS = 512;

// Tile width N: 256 for the linear layers, 128 when N <= 128 (attention's
// head dimension) so no MMA column is spent on zero padding.
template <int BN>
struct TileCfg {
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN == 256 ? 4 : 6;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;
};

struct Params {
  int M, N, K, nb1, nb2;
  int tiles_m, tiles_n, num_tiles, k_blocks;
  int vec_ok;
  int causal;  // kCausal* (gemm.cuh): per-tile skip / K range inside each s x s block
  int group_m;  // CTA-pair kernel: tiles are rastered in groups of group_m M-blocks (L2 reuse)
  int k_split, kb_per;  // CTA-pair kernel, fp32 accumulation: K split into k_split ranges of kb_per blocks
  Epilogue epi;
};

// K-block range [kb0, kb1) of output tile (m_blk, n_blk); empty = skip tile.
template <int BN>
__device__ __forceinline__ void k_range(const Params& p, int m_blk, int n_blk, int& kb0, int& kb1) {
  kb0 = 0;
  kb1 = p.k_blocks;
  if (p.causal == kCausalSkipUpper) {
    if (n_blk * BN > m_blk * BM + BM - 1) kb1 = 0;  // every key after every query
  } else if (p.causal == kCausalKUpToRow) {
    kb1 = min(kb1, (m_blk * BM + BM + BK - 1) / BK);
  } else if (p.causal == kCausalKFromRow) {
    kb0 = (m_blk * BM) / BK;
  }
}

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

__device__ __forceinline__ bool mbar_try(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ uint64_t global_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Watchdog of every pipeline wait: a barrier that has not flipped after
// kMbarTimeoutNs means a protocol bug (a missing arrive / commit), not a
// slow producer -- trap so the launch fails with an error instead of
// spinning forever and wedging the GPU.
constexpr uint64_t kMbarTimeoutNs = 10ull * 1000 * 1000 * 1000;

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (mbar_try(a, parity)) return;
  const uint64_t t0 = global_ns();
  for (uint32_t n = 1;; ++n) {
    if (mbar_try(a, parity)) return;
    if ((n & 1023u) == 0 && global_ns() - t0 > kMbarTimeoutNs) __trap();
  }
}

// mbar_wait for a whole converged warp with a warp-uniform exit (vote), so
// the compiler keeps the issuer's loop state in uniform registers.
__device__ __forceinline__ void mbar_wait_warp(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  if (__all_sync(0xffffffffu, mbar_try(a, parity))) return;
  const uint64_t t0 = global_ns();
  for (uint32_t n = 1;; ++n) {
    if (__all_sync(0xffffffffu, mbar_try(a, parity))) return;
    if ((n & 1023u) == 0 && global_ns() - t0 > kMbarTimeoutNs) __trap();
  }
}

__device__ __forceinline__ void tma_load_4d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                            int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
      "[%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// L2 prefetch of a 4D TMA box (no shared memory, no completion).
__device__ __forceinline__ void tma_prefetch_4d(const CUtensorMap* map, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3)
               : "memory");
}

// Plain bulk copy global -> shared (16-byte aligned, size a multiple of 16),
// completion counted on `bar` (expect_tx the bytes first).
__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar))
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

// tmem_ld32 without the wait: several loads in flight, then tmem_wait_ld().
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Shared-memory matrix descriptor, SWIZZLE_128B, sm_100 version bits.
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo_bytes, uint32_t sbo_bytes) {
  return static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4) | (static_cast<uint64_t>(lbo_bytes >> 4) << 16) |
         (static_cast<uint64_t>(sbo_bytes >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

// Descriptor of the same layout `bytes` further on (start-address field only;
// offsets stay inside shared memory, so the 14-bit field never carries).
__device__ __forceinline__ uint64_t desc_add(uint64_t desc, uint32_t bytes) { return desc + (bytes >> 4); }

// Grouped raster (single batch element): consecutive tile ids walk the
// group_m M-blocks of a group fastest, then N, then the next group, so the
// tiles in flight at once (one per SM pair) share a few A and B panels that
// stay in L2 instead of streaming every A panel from DRAM once per N-block.
__device__ __forceinline__ void decode_tile_grouped(const Params& p, int t, int& m_blk, int& n_blk) {
  const int per_group = p.group_m * p.tiles_n;
  const int g = t / per_group, first = g * p.group_m;
  const int gm = min(p.tiles_m - first, p.group_m);
  const int r = t - g * per_group;
  m_blk = first + r % gm;
  n_blk = r / gm;
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

// 8 contiguous elements of C-typed memory <-> floats (16 B bf16 / 32 B fp32).
__device__ __forceinline__ void ld8(const void* base, int dtype, int64_t off, float* v) {
  if (dtype == kF32) {
    const float4 a = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + off);
    const float4 b = *reinterpret_cast<const float4*>(static_cast<const float*>(base) + off + 4);
    v[0] = a.x, v[1] = a.y, v[2] = a.z, v[3] = a.w, v[4] = b.x, v[5] = b.y, v[6] = b.z, v[7] = b.w;
  } else {
    const uint4 u = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(base) + off);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[2 * i] = f.x, v[2 * i + 1] = f.y;
    }
  }
}

__device__ __forceinline__ void st8(void* base, int dtype, int64_t off, const float* v) {
  if (dtype == kF32) {
    float* c = static_cast<float*>(base) + off;
    *reinterpret_cast<float4*>(c) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(c + 4) = make_float4(v[4], v[5], v[6], v[7]);
  } else {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(base) + off) = u;
  }
}

// GELU (tanh form) on the MUFU tanh: the tensor-core path runs in bf16 mode,
// whose 2^-9 storage rounding dominates tanh.approx's ~2^-11 error.
__device__ __forceinline__ float tanh_fast(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float gelu_fast(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  return 0.5f * x * (1.0f + tanh_fast(k0 * fmaf(k1 * x, x * x, x)));
}
__device__ __forceinline__ float gelu_grad_fast(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float x2 = x * x;
  const float t = tanh_fast(k0 * fmaf(k1 * x, x2, x));
  return 0.5f * (1.0f + t) + 0.5f * x * (1.0f - t * t) * k0 * fmaf(3.0f * k1, x2, 1.0f);
}

// The same two on a pair of columns with packed f32x2 arithmetic (FFMA2 /
// FMUL2 / FADD2: half the FP32 issue slots of the scalar forms, which share
// the SM sub-partition with the MMA issuer in the GEMM epilogue).
__device__ __forceinline__ float2 gelu_fast2(float2 x) {
  using namespace smx;
  const float2 k0 = make_float2(0.7978845608028654f, 0.7978845608028654f), k1 = make_float2(0.044715f, 0.044715f);
  const float2 c = ffma2(fmul2(k1, x), fmul2(x, x), x);
  const float2 d = fmul2(k0, c);
  const float2 t = make_float2(tanh_fast(d.x), tanh_fast(d.y));
  return fmul2(fmul2(make_float2(0.5f, 0.5f), x), fadd2(make_float2(1.0f, 1.0f), t));
}
__device__ __forceinline__ float2 gelu_grad_fast2(float2 x) {
  using namespace smx;
  const float2 k0 = make_float2(0.7978845608028654f, 0.7978845608028654f), k1 = make_float2(0.044715f, 0.044715f);
  const float2 one = make_float2(1.0f, 1.0f), half = make_float2(0.5f, 0.5f);
  const float2 x2 = fmul2(x, x);
  const float2 d = fmul2(k0, ffma2(fmul2(k1, x), x2, x));
  const float2 t = make_float2(tanh_fast(d.x), tanh_fast(d.y));
  const float2 omt2 = ffma2(make_float2(-t.x, -t.y), t, one);                       // 1 - t^2
  const float2 s = ffma2(make_float2(3.0f * 0.044715f, 3.0f * 0.044715f), x2, one);  // 1 + 3 k1 x^2
  const float2 q = fmul2(fmul2(fmul2(fmul2(half, x), omt2), k0), s);
  return ffma2(half, fadd2(one, t), q);
}

__device__ __forceinline__ float round_to(int dtype, float x) {
  return dtype == kF32 ? x : __bfloat162float(__float2bfloat16_rn(x));
}

// Epilogue of one row segment of 32 accumulator columns at (row, col0).
// Full, aligned segments move 8 elements per access; ragged tails go scalar.
__device__ __forceinline__ void epilogue_chunk(const Params& p, const float* acc, int row, int col0,
                                               int64_t zoff) {
  const Epilogue& e = p.epi;
  const int64_t base = zoff + static_cast<int64_t>(row) * e.ldc + col0;
  const int ncols = min(32, p.N - col0);
  const int dt = e.mode == kEpiAccum ? kF32 : e.c_dtype;
  if (p.vec_ok && ncols == 32) {
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      float v[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = acc[8 * g + i] * e.alpha;
      if (e.bias) {
        const float4 b0 = *reinterpret_cast<const float4*>(e.bias + col0 + 8 * g);
        const float4 b1 = *reinterpret_cast<const float4*>(e.bias + col0 + 8 * g + 4);
        v[0] += b0.x, v[1] += b0.y, v[2] += b0.z, v[3] += b0.w, v[4] += b1.x, v[5] += b1.y, v[6] += b1.z,
            v[7] += b1.w;
      }
      const int64_t off = base + 8 * g;
      if (e.mode == kEpiAccum) {
        float o[8];
        ld8(e.c, kF32, off, o);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] += o[i];
      } else if (e.mode == kEpiResidual) {
        float r[8];
        ld8(e.resid, dt, off, r);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] += r[i];
      } else if (e.mode == kEpiGelu) {
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = round_to(dt, v[i]);  // GELU of the stored pre-activation
        st8(e.aux, dt, off, v);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = gelu_fast(v[i]);
      } else if (e.mode == kEpiDGelu) {
        float u[8];
        ld8(e.aux, dt, off, u);
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] *= gelu_grad_fast(u[i]);
      }
      st8(e.c, dt, off, v);
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i >= ncols) continue;
    const int64_t off = base + i;
    float v = acc[i] * e.alpha + (e.bias ? e.bias[col0 + i] : 0.f);
    if (e.mode == kEpiAccum) {
      static_cast<float*>(e.c)[off] += v;
      continue;
    }
    if (e.mode == kEpiResidual) {
      v += load_elem(e.resid, dt, off);
    } else if (e.mode == kEpiGelu) {
      v = round_to(dt, v);
      store_elem(e.aux, dt, off, v);
      v = gelu_fast(v);
    } else if (e.mode == kEpiDGelu) {
      v *= gelu_grad_fast(load_elem(e.aux, dt, off));
    }
    store_elem(e.c, dt, off, v);
  }
}

// --- CTA-pair (cta_group::2) variants -------------------------------------
// TMA load whose completion is counted on the pair leader's mbarrier (the
// peer bit of the shared::cluster barrier address cleared).
constexpr uint32_t kPeerBitMask = 0xFEFFFFFFu;

__device__ __forceinline__ void tma_load_4d_pair(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                                 int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar) & kPeerBitMask)
      : "memory");
}

__device__ __forceinline__ void tc_mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// One lane of a converged warp (elect.sync).  The MMA issuers run their
// loops in the whole warp with warp-uniform operands (shared-memory base and
// TMEM base broadcast with __shfl_sync), so the compiler keeps descriptors in
// uniform registers and issues tcgen05.mma back to back -- about 2 SASS
// instructions per MMA instead of ~10 (ELECT / R2UR per operand) from a
// single-lane branch; the issuer shares its SM sub-partition with epilogue /
// softmax warps, so its issue slots are what keeps the tensor pipe fed.
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "elect.sync _|p, 0xffffffff;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}

// Arrive on the barrier at the same offset in both CTAs of the pair.
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .b16 m;\n"
      "mov.b16 m, 3;\n"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Arrive on the barrier at `bar`'s offset in cluster CTA `rank`.
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t rank) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(rank));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}

// --- TMA epilogue: registers -> swizzled smem slab -> bulk tensor store ----
// A slab is 32 rows x 128 bytes (64 bf16 or 32 fp32 columns) in the SW128
// layout: 16-byte chunk c of row r at r*128 + ((c ^ (r & 7)) << 4), so a warp
// writing one chunk per lane (one row per lane) hits every bank exactly 4x.
constexpr int SLAB_ROWS = 32;
constexpr int SLAB_BYTES = SLAB_ROWS * 128;  // 4 KB

__device__ __forceinline__ uint32_t slab_off(int r, int c) { return r * 128 + ((c ^ (r & 7)) << 4); }

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
// global += smem (fp32 add performed at L2; the gradient-accumulation epilogue).
__device__ __forceinline__ void tma_reduce_add_2d(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.reduce.async.bulk.tensor.2d.global.shared::cta.add.tile.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(smem_u32(src))
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// One lane's row of a slab: 8 chunks of 16 bytes.
__device__ __forceinline__ void slab_put_bf16(uint8_t* slab, int r, const float* v /*64*/) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    uint4 u;
    __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(v[8 * c + 2 * i], v[8 * c + 2 * i + 1]);
    *reinterpret_cast<uint4*>(slab + slab_off(r, c)) = u;
  }
}
// Same with the row already packed as bf16x2 (32 words).
__device__ __forceinline__ void slab_put_bf16_packed(uint8_t* slab, int r, const uint32_t* pk /*32*/) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    *reinterpret_cast<uint4*>(slab + slab_off(r, c)) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
}
__device__ __forceinline__ void slab_get_bf16(const uint8_t* slab, int r, float* v /*64*/) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const uint4 u = *reinterpret_cast<const uint4*>(slab + slab_off(r, c));
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(h[i]);
      v[8 * c + 2 * i] = f.x, v[8 * c + 2 * i + 1] = f.y;
    }
  }
}
__device__ __forceinline__ void slab_put_f32(uint8_t* slab, int r, const float* v /*32*/) {
#pragma unroll
  for (int c = 0; c < 8; ++c)
    *reinterpret_cast<float4*>(slab + slab_off(r, c)) = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encoder();
// 2-D map over a row-major [rows, cols] matrix (leading dimension ld
// elements) with a {128 bytes, 32 rows} box and SW128: the epilogue slab.
CUtensorMap make_slab_map(const void* ptr, int dtype, int64_t cols, int64_t rows, int64_t ld);
CUtensorMap make_map(const Operand& op, int64_t inner, int64_t outer, int nb1, int nb2, int box_outer);
int num_sms();
void fill_params(const GemmProblem& g, Params& p, int tile_m, int tile_n);
int gemm_tc2(const GemmProblem& g, cudaStream_t s);  // CTA-pair kernel, 256 x 256 tiles

}  // namespace tc
}  // namespace wpk
