// Flash attention forward on the 5th-gen tensor cores (sm_100a).
//
// One CTA per (128-query tile, head, sequence).  Q stays in shared memory;
// K/V tiles of 128 keys stream through a 2-stage TMA ring.  Per KV tile:
//   MMA warp   S_j = Q K_j^T  (M=128, N=128, K=D)  -> TMEM (double-buffered)
//   softmax    4 warps, one query row per thread: tcgen05.ld the row of S_j,
//              online max/sum in the log2 domain with *lazy* rescaling (the
//              running max only moves when it grows by more than 2^8, so the
//              O rescale through TMEM is rare), P_j -> bf16 -> shared memory
//              in the SW128 K-major layout the MMA reads
//   MMA warp   O += P_j V_j   (M=128, N=D, K=128; A = P from smem, B = V tile
//              MN-major) accumulated in TMEM
// The QK^T of tile j+1 overlaps the softmax of tile j.  Causal: tiles past
// the diagonal are never loaded; the diagonal tile is masked in registers.
// Epilogue: O / l -> bf16 ctx row, lse2 = m + log2(l) for the backward.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <stdexcept>
#include <string>

#include "kernels/attention.cuh"
#include "kernels/tc_common.cuh"

namespace wpk {
namespace {

using namespace tc;

constexpr int QT = 128;                 // queries per CTA
constexpr int KT = 128;                 // keys per tile
constexpr int ATOM = 128 * 64 * 2;      // one SW128 K-major atom: 128 rows x 64 bf16 = 16 KB
constexpr int FA_THREADS = 256;
constexpr uint32_t kSCol0 = 0, kSCol1 = 128, kOCol = 256;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

template <int D>
struct FaCfg {
  static constexpr int Q_BYTES = QT * D * 2;
  static constexpr int KV_BYTES = KT * D * 2;  // one K or V tile
  static constexpr int P_BYTES = QT * KT * 2;
  static constexpr int SMEM = Q_BYTES + 4 * KV_BYTES + P_BYTES + 1024 + 256;
};

struct FaParams {
  int seq, heads, n_q_tiles, causal;
  float scale_log2;
  __nv_bfloat16* ctx;
  int ld_ctx;
  float* lse2;
};

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])),
      "r"(__float_as_uint(v[11])), "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])),
      "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])),
      "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
      "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])),
      "r"(__float_as_uint(v[23])), "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])),
      "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])),
      "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31])));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tma_load_attn(const CUtensorMap* map, uint64_t* bar, void* dst, int d0, int head,
                                              int row, int b) {
  tma_load_4d(map, bar, dst, d0, head, row, b);
}

// Byte offset of the 16-byte chunk `c` (8 bf16) of row `r` in an SW128
// K-major tile made of 128-row atoms of 64 elements.
__device__ __forceinline__ uint32_t swz(int r, int c) {
  const int atom = c >> 3, cc = c & 7;
  return atom * ATOM + (r >> 3) * 1024 + (r & 7) * 128 + ((cc ^ (r & 7)) << 4);
}

template <int D>
__global__ void __launch_bounds__(FA_THREADS, 1)
    flash_fwd_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                     const __grid_constant__ CUtensorMap map_v, const __grid_constant__ FaParams p) {
  using Cfg = FaCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Cfg::Q_BYTES;       // [2] stages
  uint8_t* sV = sK + 2 * Cfg::KV_BYTES;  // [2] stages
  uint8_t* sP = sV + 2 * Cfg::KV_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + Cfg::P_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* s_empty = bars + 7;   // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* o_done = bars + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 12);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // Heavy (late) query tiles first for causal load balance.
  const int qi = p.n_q_tiles - 1 - static_cast<int>(blockIdx.x % p.n_q_tiles);
  const int head = static_cast<int>((blockIdx.x / p.n_q_tiles) % p.heads);
  const int b = static_cast<int>(blockIdx.x / (p.n_q_tiles * p.heads));
  const int n_kv = p.causal ? qi + 1 : p.seq / KT;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_q)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_k)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_v)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], 4);
    }
    mbar_init(p_full, 4);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------- TMA
      mbar_expect_tx(q_full, Cfg::Q_BYTES);
#pragma unroll
      for (int a = 0; a < D / 64; ++a) tma_load_attn(&map_q, q_full, sQ + a * ATOM, a * 64, head, qi * QT, b);
      for (int j = 0; j < n_kv; ++j) {
        const int st = j & 1;
        mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], 2 * Cfg::KV_BYTES);
#pragma unroll
        for (int a = 0; a < D / 64; ++a) {
          tma_load_attn(&map_k, &kv_full[st], sK + st * Cfg::KV_BYTES + a * ATOM, a * 64, head, j * KT, b);
          tma_load_attn(&map_v, &kv_full[st], sV + st * Cfg::KV_BYTES + a * ATOM, a * 64, head, j * KT, b);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------------------- MMA
      // S: M=128, N=128, A=Q K-major, B=K K-major.  PV: M=128, N=D, A=P K-major, B=V MN-major.
      constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(KT >> 3) << 17) |
                                   (uint32_t(QT >> 4) << 24);
      constexpr uint32_t idesc_pv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(D >> 3) << 17) |
                                    (uint32_t(QT >> 4) << 24);
      const uint32_t q_addr = smem_u32(sQ);
      auto issue_s = [&](int j) {
        const int st = j & 1;
        const uint32_t k_addr = smem_u32(sK + st * Cfg::KV_BYTES);
        const uint32_t dcol = tmem + (st ? kSCol1 : kSCol0);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * ATOM + (k & 3) * 32;
          tc_mma(dcol, make_desc(q_addr + off, 16, 1024), make_desc(k_addr + off, 16, 1024), idesc_s, k != 0);
        }
        tc_commit(&s_full[st]);
      };
      mbar_wait(q_full, 0);
      mbar_wait(&kv_full[0], 0);
      tc_fence_after();
      issue_s(0);
      for (int j = 0; j < n_kv; ++j) {
        if (j + 1 < n_kv) {
          const int st = (j + 1) & 1;
          mbar_wait(&kv_full[st], ((j + 1) >> 1) & 1);
          if (j >= 1) mbar_wait(&s_empty[st], ((j - 1) >> 1) & 1);
          tc_fence_after();
          issue_s(j + 1);
        }
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        const uint32_t p_addr = smem_u32(sP);
        const uint32_t v_addr = smem_u32(sV + (j & 1) * Cfg::KV_BYTES);
#pragma unroll
        for (int k = 0; k < KT / 16; ++k) {
          const uint64_t ad = make_desc(p_addr + (k >> 2) * ATOM + (k & 3) * 32, 16, 1024);
          const uint64_t bd = make_desc(v_addr + k * 2048, ATOM, 1024);
          tc_mma(tmem + kOCol, ad, bd, idesc_pv, (j | k) != 0);
        }
        tc_commit(&kv_empty[j & 1]);
        tc_commit(o_done);
      }
    }
  } else if (warp >= 4) {
    // ---------------------------------------------------------- softmax
    const int ew = warp & 3;
    const int r = ew * 32 + lane;         // query row within the tile
    const int q = qi * QT + r;            // query position
    const uint32_t lane_base = static_cast<uint32_t>(ew * 32) << 16;
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kv; ++j) {
      const int st = j & 1;
      mbar_wait(&s_full[st], (j >> 1) & 1);
      tc_fence_after();
      float s[KT];
#pragma unroll
      for (int c = 0; c < KT; c += 32) tmem_ld32(tmem + lane_base + (st ? kSCol1 : kSCol0) + c, s + c);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[st]);
      const bool diag = p.causal && j == qi;
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < KT; ++c) {
        s[c] = (diag && c > r) ? -INFINITY : s[c] * p.scale_log2;
        mx = fmaxf(mx, s[c]);
      }
      float alpha = 1.f;
      if (mx > m_used + kRescaleThreshold) {
        alpha = ex2(m_used - mx);  // 0 on the first tile
        m_used = mx;
        l *= alpha;
      }
      float sum = 0.f;
#pragma unroll
      for (int c = 0; c < KT; ++c) {
        s[c] = ex2(s[c] - m_used);
        sum += s[c];
      }
      l += sum;
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);  // PV_{j-1} done: O settled, P buffer free
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
          for (int c = 0; c < D; c += 32) {
            float o[32];
            tmem_ld32(tmem + lane_base + kOCol + c, o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tmem_st32(tmem + lane_base + kOCol + c, o);
          }
        }
      }
      // P row -> bf16 -> SW128 K-major smem (2 atoms of 64 keys).
#pragma unroll
      for (int c = 0; c < KT / 8; ++c) {
        uint4 u;
        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) h2[i] = __floats2bfloat162_rn(s[8 * c + 2 * i], s[8 * c + 2 * i + 1]);
        *reinterpret_cast<uint4*>(sP + swz(r, c)) = u;
      }
      fence_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
    }
    mbar_wait(o_done, (n_kv - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    __nv_bfloat16* out = p.ctx + (static_cast<int64_t>(b) * p.seq + q) * p.ld_ctx + head * D;
#pragma unroll
    for (int c = 0; c < D; c += 32) {
      float o[32];
      tmem_ld32(tmem + lane_base + kOCol + c, o);
#pragma unroll
      for (int g = 0; g < 32; g += 8) {
        uint4 u;
        __nv_bfloat162* h2 = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int i = 0; i < 4; ++i) h2[i] = __floats2bfloat162_rn(o[g + 2 * i] * inv, o[g + 2 * i + 1] * inv);
        *reinterpret_cast<uint4*>(out + c + g) = u;
      }
    }
    p.lse2[(static_cast<int64_t>(b) * p.heads + head) * p.seq + q] = m_used + __log2f(l);
  }

  tc_fence_before();
  __syncwarp();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// {D, heads, seq, mbs} view of one of Q / K / V inside qkv; box {64, 1, 128, 1}.
CUtensorMap attn_map(const void* base, const AttnShape& s) {
  CUtensorMap m;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(s.head_dim), static_cast<cuuint64_t>(s.heads),
                        static_cast<cuuint64_t>(s.seq), static_cast<cuuint64_t>(s.mbs)};
  const uint64_t ld = 3ull * s.hidden * 2;
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(s.head_dim) * 2, ld, ld * s.seq};
  cuuint32_t box[4] = {64, 1, 128, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = get_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                                   box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("attention tensor map: " + std::to_string(int(r)));
  return m;
}

template <int D>
void launch_fwd(const AttnShape& s, const void* qkv, void* ctx, float* lse2, cudaStream_t stream) {
  auto* k = flash_fwd_kernel<D>;
  static uint64_t attr_done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_done >> (dev & 63) & 1)) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, FaCfg<D>::SMEM);
    attr_done |= 1ull << (dev & 63);
  }
  const auto* base = static_cast<const __nv_bfloat16*>(qkv);
  const CUtensorMap mq = attn_map(base, s), mk = attn_map(base + s.hidden, s), mv = attn_map(base + 2 * s.hidden, s);
  FaParams p;
  p.seq = s.seq;
  p.heads = s.heads;
  p.n_q_tiles = s.seq / QT;
  p.causal = s.causal;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  p.ctx = static_cast<__nv_bfloat16*>(ctx);
  p.ld_ctx = s.hidden;
  p.lse2 = lse2;
  const int grid = p.n_q_tiles * s.heads * s.mbs;
  k<<<grid, FA_THREADS, FaCfg<D>::SMEM, stream>>>(mq, mk, mv, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("flash_attn_fwd: ") + cudaGetErrorString(e));
}

}  // namespace

int flash_attn_fwd(const AttnShape& s, const void* qkv, void* ctx, float* lse2, cudaStream_t stream) {
  if (s.seq % 128 || (s.head_dim != 64 && s.head_dim != 128)) {
    throw std::runtime_error("flash_attn_fwd: needs seq % 128 == 0 and head_dim in {64, 128}");
  }
  if (s.head_dim == 128) launch_fwd<128>(s, qkv, ctx, lse2, stream);
  else launch_fwd<64>(s, qkv, ctx, lse2, stream);
  return 1;
}

}  // namespace wpk
