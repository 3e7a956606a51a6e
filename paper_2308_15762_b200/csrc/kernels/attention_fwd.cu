// Flash attention forward on the 5th-gen tensor cores (sm_100a).
//
// One CTA per (pair of adjacent 128-query tiles 2i, 2i+1; head; sequence),
// heavy pairs first.  Both query tiles share every K / V tile, streamed by
// TMA through a 3-slot ring of single tiles (K_0, V_0, K_1, V_1, ...).  Two
// softmax warpgroups (warps 4-7: tile A = 2i, warps 8-11: tile B = 2i+1)
// hold a whole 128-wide S row per thread in registers: setmaxnreg moves the
// register file from the control warpgroup (40) to them (232).
// ping-pong on the tensor core, which the single MMA thread feeds in the
// order  S_A(j+1), S_B(j+1), PV_A(j), PV_B(j):
//   S_x(j)  = Q_x K_j^T   (M=128, N=128, K=D)  -> TMEM S_x
//   PV_x(j) : O_x += P_x(j) V_j  (M=128, N=D, K=128; P from smem)  -> TMEM O_x
// so while one warpgroup turns S into P (online max/sum in the log2 domain,
// lazy O rescale only when the running max grows by more than 2^8) the
// tensor core works on the other's products.  A warpgroup overlaps its own
// exponentials of step j+1 with the PV of step j; only the P store waits.
// Causal: key tiles past a query tile's diagonal are neither loaded nor
// multiplied; the diagonal tile is masked in registers.
// Epilogue: O / l -> bf16 ctx rows, lse2 = m + log2(l) for the backward.
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

constexpr int QT = 128;                 // queries per tile
constexpr int KT = 128;                 // keys per tile
constexpr int ATOM = 128 * 64 * 2;      // one SW128 K-major atom: 128 rows x 64 bf16 = 16 KB
constexpr int FA_THREADS = 384;         // w0 TMA, w1 TMEM + MMA, w4-7 softmax A, w8-11 softmax B
constexpr int NK = 2, NV = 2;           // K / V tile slots
constexpr int RING = NK + NV;

// Ring tile t: K_j = 2j, V_j = 2j+1.  K tiles cycle NK slots, V tiles NV
// slots (P lives in TMEM, so shared memory holds Q and NK + NV K/V tiles).
__device__ __forceinline__ int ring_slot(int t) { return (t & 1) ? NK + (t >> 1) % NV : (t >> 1) % NK; }
__device__ __forceinline__ int ring_use(int t) { return (t & 1) ? (t >> 1) / NV : (t >> 1) / NK; }
constexpr float kRescaleThreshold = 8.0f;  // log2 units

template <int D>
struct FaCfg {
  static constexpr int TILE = 128 * D * 2;  // one Q, K or V tile
  static constexpr int P_BYTES = QT * KT * 2;
  static constexpr int SMEM = 2 * TILE + RING * TILE + 1024 + 512;  // P lives in TMEM
  __device__ static constexpr uint32_t col_s(int x) { return x ? 128u : 0u; }
  __device__ static constexpr uint32_t col_o(int x) { return x ? 256u + D : 256u; }
};

struct FaParams {
  int batch, seq, heads, n_q_tiles, n_pairs, causal;
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

// 128 consecutive fp32 TMEM columns of this warp's 32 lanes: four x32 loads
// in flight, one wait.
__device__ __forceinline__ void tmem_ld32x4(uint32_t taddr, float* v) {
  uint32_t* u = reinterpret_cast<uint32_t*>(v);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(u[32 * q + 0]), "=r"(u[32 * q + 1]), "=r"(u[32 * q + 2]), "=r"(u[32 * q + 3]),
          "=r"(u[32 * q + 4]), "=r"(u[32 * q + 5]), "=r"(u[32 * q + 6]), "=r"(u[32 * q + 7]),
          "=r"(u[32 * q + 8]), "=r"(u[32 * q + 9]), "=r"(u[32 * q + 10]), "=r"(u[32 * q + 11]),
          "=r"(u[32 * q + 12]), "=r"(u[32 * q + 13]), "=r"(u[32 * q + 14]), "=r"(u[32 * q + 15]),
          "=r"(u[32 * q + 16]), "=r"(u[32 * q + 17]), "=r"(u[32 * q + 18]), "=r"(u[32 * q + 19]),
          "=r"(u[32 * q + 20]), "=r"(u[32 * q + 21]), "=r"(u[32 * q + 22]), "=r"(u[32 * q + 23]),
          "=r"(u[32 * q + 24]), "=r"(u[32 * q + 25]), "=r"(u[32 * q + 26]), "=r"(u[32 * q + 27]),
          "=r"(u[32 * q + 28]), "=r"(u[32 * q + 29]), "=r"(u[32 * q + 30]), "=r"(u[32 * q + 31])
        : "r"(taddr + 32 * q));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

#ifdef WP_FA_TRACE
// Debug timeline of CTA 0 (build with -DWP_FA_TRACE): clock64 per (event,
// warpgroup, step) in a static smem table, copied out at the end.
__device__ unsigned long long g_fa_trace[16 * 2 * 32];
#define FA_TRACE(ev, x, j)                                                                        \
  do {                                                                                            \
    if (blockIdx.x == 0 && (j) < 32) g_fa_trace[((ev) * 2 + (x)) * 32 + (j)] = clock64();          \
  } while (0)
#else
#define FA_TRACE(ev, x, j) \
  do {                     \
  } while (0)
#endif

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

// O += P V with P read from tensor memory (A operand, K-major: lane = query,
// 32-bit column j = keys 2j, 2j+1 as bf16x2) -- P never touches shared memory.
__device__ __forceinline__ void tc_mma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

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
  uint8_t* sQ = smem;                     // [2] tiles
  uint8_t* sR = sQ + 2 * Cfg::TILE;       // [RING] K/V slots
  uint64_t* bars = reinterpret_cast<uint64_t*>(sR + RING * Cfg::TILE);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;           // [RING]
  uint64_t* kv_empty = kv_full + RING;    // [RING]
  uint64_t* s_full = kv_empty + RING;     // [2]
  uint64_t* s_empty = s_full + 2;         // [2]
  uint64_t* p_full = s_empty + 2;         // [2]
  uint64_t* o_done = p_full + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  // Heavy (late) query-tile pairs first for causal load balance.
  // Heaviest-first (LPT) order: the last query-tile pair (longest causal key
  // range) of every (batch, head) launches first.
  const int bh = p.batch * p.heads;
  const int pi = p.n_pairs - 1 - static_cast<int>(blockIdx.x / bh);
  const int head = static_cast<int>(blockIdx.x % bh % p.heads);
  const int b = static_cast<int>(blockIdx.x % bh / p.heads);
  const int qt[2] = {2 * pi, 2 * pi + 1};
  const bool has_b = qt[1] < p.n_q_tiles;
  const int n_all = p.seq / KT;
  const int nkv[2] = {p.causal ? qt[0] + 1 : n_all, has_b ? (p.causal ? qt[1] + 1 : n_all) : 0};
  const int n_max = max(nkv[0], nkv[1]);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_q)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_k)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_v)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < RING; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&s_full[x], 1);
      mbar_init(&s_empty[x], 4);
      mbar_init(&p_full[x], 4);
      mbar_init(&o_done[x], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------------- TMA
      mbar_expect_tx(q_full, (has_b ? 2 : 1) * Cfg::TILE);
      for (int x = 0; x < (has_b ? 2 : 1); ++x)
#pragma unroll
        for (int a = 0; a < D / 64; ++a)
          tma_load_4d(&map_q, q_full, sQ + x * Cfg::TILE + a * ATOM, a * 64, head, qt[x] * QT, b);
      auto load = [&](int t) {
        const int slot = ring_slot(t), use = ring_use(t);
        if (use > 0) mbar_wait(&kv_empty[slot], (use - 1) & 1);
        mbar_expect_tx(&kv_full[slot], Cfg::TILE);
        const CUtensorMap* m = (t & 1) ? &map_v : &map_k;
#pragma unroll
        for (int a = 0; a < D / 64; ++a)
          tma_load_4d(m, &kv_full[slot], sR + slot * Cfg::TILE + a * ATOM, a * 64, head, (t >> 1) * KT, b);
      };
      // In consumption order: K_0, V_0, K_1, V_1, ... (S(j+1) is issued right
      // after PV(j)); each load waits only for its own slot.
      for (int t = 0; t < 2 * n_max; ++t) load(t);
    } else if (warp == 1 && lane == 0) {
      // ------------------------------------------------------------- MMA
      // S: M=128, N=128, A=Q K-major, B=K K-major.  PV: M=128, N=D, A=P K-major, B=V MN-major.
      constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(KT >> 3) << 17) |
                                   (uint32_t(QT >> 4) << 24);
      constexpr uint32_t idesc_pv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(D >> 3) << 17) |
                                    (uint32_t(QT >> 4) << 24);
      auto tile_ready = [&](int t) -> uint32_t {  // waits for ring tile t, returns its smem address
        const int slot = ring_slot(t);
        mbar_wait(&kv_full[slot], ring_use(t) & 1);
        tc_fence_after();
        return smem_u32(sR + slot * Cfg::TILE);
      };
      auto free_tile = [&](int t) { tc_commit(&kv_empty[ring_slot(t)]); };
      auto issue_s = [&](int x, int j) {
        FA_TRACE(8, x, j);
        // S_x(j) overwrites P_x(j-1): in order after PV_x(j-1), which read it.
        const uint32_t k_addr = tile_ready(2 * j);
        const uint32_t q_addr = smem_u32(sQ + x * Cfg::TILE);
        FA_TRACE(10, x, j);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * ATOM + (k & 3) * 32;
          tc_mma(tmem + Cfg::col_s(x), make_desc(q_addr + off, 16, 1024), make_desc(k_addr + off, 16, 1024),
                 idesc_s, k != 0);
        }
        tc_commit(&s_full[x]);
        FA_TRACE(1, x, j);
      };
      auto issue_pv = [&](int x, int j) {
        FA_TRACE(9, x, j);
        mbar_wait(&p_full[x], j & 1);
        tc_fence_after();
        const uint32_t v_addr = tile_ready(2 * j + 1);
        FA_TRACE(11, x, j);
#pragma unroll
        for (int k = 0; k < KT / 16; ++k) {
          const uint64_t bd = make_desc(v_addr + k * 2048, ATOM, 1024);
          tc_mma_ts(tmem + Cfg::col_o(x), tmem + Cfg::col_s(x) + k * 8, bd, idesc_pv, (j | k) != 0);
        }
        tc_commit(&o_done[x]);
        FA_TRACE(2, x, j);
      };
      mbar_wait(q_full, 0);
      if (nkv[0] > 0) {
        issue_s(0, 0);
        if (nkv[1] == 0) free_tile(0);
      }
      if (nkv[1] > 0) {
        issue_s(1, 0);
        free_tile(0);
      }
      // Per step: PV_x(j) then S_x(j+1) for each warpgroup (S_x(j+1) reuses
      // P_x(j)'s columns); the other warpgroup's softmax overlaps both.
      for (int j = 0; j < n_max; ++j) {
        for (int x = 0; x < 2; ++x) {
          if (j >= nkv[x]) continue;
          issue_pv(x, j);
          if (x == 1 || j >= nkv[1]) free_tile(2 * j + 1);
          if (j + 1 < nkv[x]) {
            issue_s(x, j + 1);
            if (x == 1 || j + 1 >= nkv[1]) free_tile(2 * (j + 1));
          }
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 224;");
    // ---------------------------------------------------------- softmax
    const int x = (warp - 4) >> 2;  // 0: tile A, 1: tile B
    const int n_kv = nkv[x];
    if (n_kv > 0) {
      const int ew = warp & 3;
      const int r = ew * 32 + lane;         // query row within the tile
      const int q = qt[x] * QT + r;         // query position
      const uint32_t lane_base = static_cast<uint32_t>(ew * 32) << 16;
      const uint32_t s_col = tmem + lane_base + Cfg::col_s(x);
      const uint32_t o_col = tmem + lane_base + Cfg::col_o(x);
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kv; ++j) {
        if (lane == 0 && (warp & 3) == 0) FA_TRACE(3, x, j);
        mbar_wait(&s_full[x], j & 1);
        tc_fence_after();
        if (lane == 0 && (warp & 3) == 0) FA_TRACE(4, x, j);
        // The whole S row in registers (4 loads, one wait), then S_x is free
        // for the next QK^T at once.
        float sv[KT];
        tmem_ld32x4(s_col, sv);
        if (p.causal && j == qt[x]) {  // diagonal tile: keys after the query masked
#pragma unroll
          for (int c = 0; c < KT; ++c) sv[c] = c > r ? -INFINITY : sv[c];
        }
        float mx = sv[0];
#pragma unroll
        for (int c = 1; c < KT; ++c) mx = fmaxf(mx, sv[c]);
        mx *= p.scale_log2;
        float alpha = 1.f;
        if (mx > m_used + kRescaleThreshold) {
          alpha = ex2(m_used - mx);  // 0 on the first tile
          m_used = mx;
          l *= alpha;
        }
        float sum = 0.f;
        const float mb = m_used;
#pragma unroll
        for (int c = 0; c < KT; ++c) {
          sv[c] = ex2(fmaf(sv[c], p.scale_log2, -mb));
          sum += sv[c];
        }
        l += sum;
        if (j > 0) {
          if (lane == 0 && (warp & 3) == 0) FA_TRACE(5, x, j);
          mbar_wait(&o_done[x], (j - 1) & 1);  // PV_x(j-1) done: O settled, P buffer free
          tc_fence_after();
          if (lane == 0 && (warp & 3) == 0) FA_TRACE(6, x, j);
        }
        // P row -> bf16x2 -> TMEM over this row's S columns (A operand of PV).
#pragma unroll
        for (int q = 0; q < KT / 32; ++q) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(sv[32 * q + 2 * i], sv[32 * q + 2 * i + 1]);
            pk[i] = *reinterpret_cast<uint32_t*>(&h2);
          }
          tmem_st16(s_col + 16 * q, pk);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        // Lazy rescale of O (before PV_x(j) is issued; S registers are dead).
        if (j > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll 1
          for (int c = 0; c < D; c += 32) {
            float o[32];
            tmem_ld32(o_col + c, o);
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] *= alpha;
            tmem_st32(o_col + c, o);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[x]);
        if (lane == 0 && (warp & 3) == 0) FA_TRACE(7, x, j);
      }
      mbar_wait(&o_done[x], (n_kv - 1) & 1);
      tc_fence_after();
      const float inv = 1.f / l;
      __nv_bfloat16* out = p.ctx + (static_cast<int64_t>(b) * p.seq + q) * p.ld_ctx + head * D;
#pragma unroll
      for (int c = 0; c < D; c += 32) {
        float o[32];
        tmem_ld32(o_col + c, o);
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
  }

  tc_fence_before();
  __syncwarp();
  __syncthreads();
  if (warp == 1) {
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
  p.batch = s.mbs;
  p.seq = s.seq;
  p.heads = s.heads;
  p.n_q_tiles = s.seq / QT;
  p.n_pairs = (p.n_q_tiles + 1) / 2;
  p.causal = s.causal;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(D));
  p.ctx = static_cast<__nv_bfloat16*>(ctx);
  p.ld_ctx = s.hidden;
  p.lse2 = lse2;
  const int grid = p.n_pairs * s.heads * s.mbs;
  k<<<grid, FA_THREADS, FaCfg<D>::SMEM, stream>>>(mq, mk, mv, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k);
    throw std::runtime_error(std::string("flash_attn_fwd: ") + cudaGetErrorString(e) + " (regs " +
                             std::to_string(fa.numRegs) + ", max threads " + std::to_string(fa.maxThreadsPerBlock) +
                             ", smem " + std::to_string(FaCfg<D>::SMEM) + " + " + std::to_string(fa.sharedSizeBytes) +
                             ")");
  }
}

}  // namespace

#ifdef WP_FA_TRACE
}  // namespace wpk
extern "C" int wp_debug_fa_trace(unsigned long long* out, int cap) {
  using namespace wpk;
  const int n = cap < 16 * 2 * 32 ? cap : 16 * 2 * 32;
  cudaMemcpyFromSymbol(out, g_fa_trace, n * sizeof(unsigned long long));
  return n;
}
namespace wpk {
#endif

int flash_attn_fwd(const AttnShape& s, const void* qkv, void* ctx, float* lse2, cudaStream_t stream) {
  if (s.seq % 128 || (s.head_dim != 64 && s.head_dim != 128)) {
    throw std::runtime_error("flash_attn_fwd: needs seq % 128 == 0 and head_dim in {64, 128}");
  }
  if (s.head_dim == 128) launch_fwd<128>(s, qkv, ctx, lse2, stream);
  else launch_fwd<64>(s, qkv, ctx, lse2, stream);
  return 1;
}

}  // namespace wpk
