// Flash attention forward on the 5th-gen tensor cores (sm_100a).
//
// Persistent CTAs (one per SM) walk work items = (pair of adjacent 128-query
// tiles 2i, 2i+1; head; sequence), heaviest causal pairs first, in snake
// order across CTAs.  Both query tiles of an item share every K / V tile,
// streamed by TMA through a FIFO ring (K_0, V_0, K_1, V_1, ...) that runs on
// across items; Q is double-buffered per item, so the next item's Q, K_0 and
// first S products land while the current item finishes -- only the first
// item of a CTA pays the load latency.  Two softmax warpgroups (warps 4-7:
// tile A = 2i, warps 8-11: tile B = 2i+1) hold a whole 128-wide S row per
// thread in registers (setmaxnreg: 72 for the control warps, 216 for them; 4x32x72 + 8x32x216
// = the 168 x 384 registers the CTA is launched with).
// The single MMA thread issues, per key tile j,
//   S_x(j)  = Q_x K_j^T   (M=128, N=128, K=D)  -> TMEM S_x
//   PV_x(j) : O_x += P_x(j) V_j  (M=128, N=D, K=128; P_x from TMEM)  -> TMEM O_x
// D = 128 (TMEM full: S_A, S_B, O_A, O_B): P_x(j) is written over S_x(j), so
// the order is PV_A(j), S_A(j+1), PV_B(j), S_B(j+1) and one warpgroup's
// softmax overlaps the other's products.  D = 64: P_x has its own columns,
// so S_x(j+1) is issued as soon as the softmax has S_x(j) in registers and
// the next S is ready when the softmax finishes (S_A(j+1), S_B(j+1),
// PV_A(j), PV_B(j)).  Softmax: online max / sum in the log2 domain with lazy
// O rescale (only when the running max grows by more than 2^8), FMNMX3 row
// max, packed FFMA2 / FADD2 arithmetic, part of the 2^x on the FMA pipe by a
// polynomial (ex2_poly2) to relieve the SFU.  Causal: key tiles past a query
// tile's diagonal are neither loaded nor multiplied; the diagonal tile is
// masked in registers.  Epilogue: O / l -> bf16 into the item's own Q tile
// (free once its last S is done) -> per-warp TMA stores of 32 coalesced rows;
// lse2 = m + log2(l) for the backward.  It overlaps the next item's first S
// products; the Q buffer returns to the loader when the store has read it.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

#include "kernels/attention.cuh"
#include "kernels/softmax_math.cuh"
#include "kernels/tc_common.cuh"

namespace wpk {
namespace {

using namespace tc;
using namespace smx;

constexpr int QT = 128;                 // queries per tile
constexpr int KT = 128;                 // keys per tile
constexpr int ATOM = 128 * 64 * 2;      // one SW128 K-major atom: 128 rows x 64 bf16 = 16 KB
constexpr int FA_THREADS = 384;         // w0 TMA, w1 TMEM + MMA, w4-7 softmax A, w8-11 softmax B
constexpr float kRescaleThreshold = 8.0f;  // log2 units

// Shared memory: Q double-buffered across work items (item parity), K / V
// in one FIFO ring of RING tiles in consumption order K_0, V_0, K_1, V_1 ...
// (tile t in slot t % RING, continuing across items).  D = 128: 4 Q + 3 ring
// tiles = 224 KB; D = 64: 4 Q + 6 ring tiles = 160 KB.
// TMEM (512 columns): S_A, S_B (128 each), O_A, O_B (D each) and, at D = 64,
// P_A / P_B in their own 64 columns (bf16x2) so S_x(j+1) may overwrite S_x(j)
// as soon as the softmax has it in registers; at D = 128 there is no room and
// P_x(j) is written over S_x(j) (S_x(j+1) waits for PV_x(j) to read it).
template <int D>
struct FaCfg {
  static constexpr int TILE = 128 * D * 2;  // one Q, K or V tile
  static constexpr int RING = D == 128 ? 3 : 6;
  static constexpr bool PSEP = D == 64;
  static constexpr int SMEM = 4 * TILE + RING * TILE + 1024 + 512;
  __device__ static constexpr uint32_t col_s(int x) { return x ? 128u : 0u; }
  __device__ static constexpr uint32_t col_o(int x) { return x ? 256u + D : 256u; }
  __device__ static constexpr uint32_t col_p(int x) { return PSEP ? 256u + 2 * D + 64u * x : col_s(x); }
};

struct FaParams {
  int batch, seq, heads, n_q_tiles, n_pairs, causal, n_items;
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

// POLY: of every 8 column pairs of an S row, this many take the polynomial
// 2^x (3 = 37.5 % at both D: measured best with 2, ahead of 0 and of 4-5,
// which cost more FMA-pipe issue than they save on the SFU).
// WP_FA_POLY=n (0, 2-5) overrides for A/B.
constexpr int kFaPolyD128 = 3, kFaPolyD64 = 3;

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile("cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%1, %2, %3, %4}], [%5];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(src))
               : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Byte offset of the 16-byte chunk `c` (8 bf16) of row `r` in an SW128
// K-major tile made of 128-row atoms of 64 elements.
__device__ __forceinline__ uint32_t swz(int r, int c) {
  const int atom = c >> 3, cc = c & 7;
  return atom * ATOM + (r >> 3) * 1024 + (r & 7) * 128 + ((cc ^ (r & 7)) << 4);
}

// Work item w (heaviest first: the last query-tile pair of every (batch,
// head), then the one before, ...) -> its coordinates and key-tile counts.
struct FaItem {
  int b, head, qt0, has_b, nkv0, nkv1, n_max;
};
__device__ __forceinline__ FaItem fa_item(const FaParams& p, int w) {
  const int bh = p.batch * p.heads;
  FaItem it;
  const int pi = p.n_pairs - 1 - w / bh;
  it.head = w % bh % p.heads;
  it.b = w % bh / p.heads;
  it.qt0 = 2 * pi;
  it.has_b = it.qt0 + 1 < p.n_q_tiles;
  const int n_all = p.seq / KT;
  it.nkv0 = p.causal ? it.qt0 + 1 : n_all;
  it.nkv1 = it.has_b ? (p.causal ? it.qt0 + 2 : n_all) : 0;
  it.n_max = max(it.nkv0, it.nkv1);
  return it;
}
// Persistent CTAs take the heaviest-first item list in snake order (round k
// runs CTAs 0..G-1 on even k, G-1..0 on odd k), which evens out the per-CTA
// totals of the causal pairs' 2, 4, 6, ... key tiles.
__device__ __forceinline__ int fa_item_index(int k) {
  const int G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  return k * G + ((k & 1) ? G - 1 - c : c);
}

template <int D, int POLY>
__global__ void __launch_bounds__(FA_THREADS, 1)
    flash_fwd_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                     const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_o,
                     const __grid_constant__ FaParams p) {
  using Cfg = FaCfg<D>;
  constexpr int RING = Cfg::RING;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                     // [2 items][2 tiles]
  uint8_t* sR = sQ + 4 * Cfg::TILE;       // [RING] K/V slots
  uint64_t* bars = reinterpret_cast<uint64_t*>(sR + RING * Cfg::TILE);
  uint64_t* q_full = bars + 0;            // [2] per Q buffer
  uint64_t* q_empty = bars + 2;           // [2] last S + the 8 softmax warps' O stores out of it
  uint64_t* kv_full = bars + 4;           // [RING]
  uint64_t* kv_empty = kv_full + RING;    // [RING]
  uint64_t* s_full = kv_empty + RING;     // [2]
  uint64_t* s_empty = s_full + 2;         // [2] (PSEP: S_x read into registers)
  uint64_t* p_full = s_empty + 2;         // [2]
  uint64_t* o_done = p_full + 2;          // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_done + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_q)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_k)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_v)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_o)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int x = 0; x < 2; ++x) {
      mbar_init(&q_full[x], 1);
      mbar_init(&q_empty[x], 9);
      mbar_init(&s_full[x], 1);
      mbar_init(&s_empty[x], 4);
      mbar_init(&p_full[x], 4);
      mbar_init(&o_done[x], 1);
    }
    for (int s = 0; s < RING; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
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
    asm volatile("setmaxnreg.dec.sync.aligned.u32 72;");
    if (warp == 0 && lane == 0) {
      // ------------------------------------------------------------- TMA
      // Q of item kq into buffer kq & 1, once item kq-2 is done with it
      // (its last S, and its O rows staged there and stored).
      auto load_q = [&](int kq) {
        const int wq = fa_item_index(kq);
        if (wq >= p.n_items) return;
        const FaItem iq = fa_item(p, wq);
        const int qb = kq & 1;
        if (kq >= 2) mbar_wait(&q_empty[qb], ((kq - 2) >> 1) & 1);
        mbar_expect_tx(&q_full[qb], (iq.has_b ? 2 : 1) * Cfg::TILE);
        for (int x = 0; x < (iq.has_b ? 2 : 1); ++x)
#pragma unroll
          for (int a = 0; a < D / 64; ++a)
            tma_load_4d(&map_q, &q_full[qb], sQ + (2 * qb + x) * Cfg::TILE + a * ATOM, a * 64, iq.head,
                        (iq.qt0 + x) * QT, iq.b);
      };
      int t0 = 0;  // ring tiles loaded so far (all items)
      load_q(0);
      for (int k = 0;; ++k) {
        const int w = fa_item_index(k);
        if (w >= p.n_items) break;
        const FaItem it = fa_item(p, w);
        // In consumption order K_0, V_0, K_1, V_1, ...; each load waits only
        // for its own slot (FIFO: tile t reuses the slot of tile t - RING).
        // The next item's Q goes out a few tiles into this one.
        const int tq = min(3, 2 * it.n_max - 1);
        for (int t = 0; t < 2 * it.n_max; ++t) {
          const int g = t0 + t, slot = g % RING, use = g / RING;
          if (use > 0) mbar_wait(&kv_empty[slot], (use - 1) & 1);
          mbar_expect_tx(&kv_full[slot], Cfg::TILE);
          const CUtensorMap* m = (t & 1) ? &map_v : &map_k;
#pragma unroll
          for (int a = 0; a < D / 64; ++a)
            tma_load_4d(m, &kv_full[slot], sR + slot * Cfg::TILE + a * ATOM, a * 64, it.head, (t >> 1) * KT, it.b);
          if (t == tq) load_q(k + 1);
        }
        t0 += 2 * it.n_max;
      }
    } else if (warp == 1) {
      // ------------------------------------------------------------- MMA
      // The whole warp walks the issue loop with warp-uniform state and one
      // elected lane issues (see elect_one): uniform-register descriptors,
      // back-to-back MMAs, few issue slots taken from the softmax warps
      // that share this sub-partition.
      const uint32_t tb = __shfl_sync(0xffffffffu, tmem, 0);
      const uint32_t sQa = (smem_u32(smem_raw) + 1023u) & ~1023u;
      const uint32_t sRa = sQa + 4 * Cfg::TILE;
      if (sQa != smem_u32(sQ)) __trap();  // shared-space and generic alignment must agree
      // S: M=128, N=128, A=Q K-major, B=K K-major.  PV: M=128, N=D, A=P (TMEM), B=V MN-major.
      constexpr uint32_t idesc_s = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(KT >> 3) << 17) |
                                   (uint32_t(QT >> 4) << 24);
      constexpr uint32_t idesc_pv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(D >> 3) << 17) |
                                    (uint32_t(QT >> 4) << 24);
      int t0 = 0;              // ring tiles consumed before this item
      int ns[2] = {0, 0};      // S_x issued (all items)
      int npv[2] = {0, 0};     // PV_x issued (all items)
      auto tile_ready = [&](int g) -> uint32_t {  // waits for ring tile g, returns its smem address
        const int slot = g % RING;
        mbar_wait_warp(&kv_full[slot], (g / RING) & 1);
        tc_fence_after();
        return sRa + slot * Cfg::TILE;
      };
      auto free_tile = [&](int g) {
        if (elect_one()) tc_commit(&kv_empty[g % RING]);
        __syncwarp();
      };
      for (int k = 0;; ++k) {
        const int w = fa_item_index(k);
        if (w >= p.n_items) break;
        const FaItem it = fa_item(p, w);
        const int qb = k & 1;
        const int nkv[2] = {it.nkv0, it.nkv1};
        mbar_wait_warp(&q_full[qb], (k >> 1) & 1);
        tc_fence_after();
        auto issue_s = [&](int x, int j) {
          // PSEP: S_x(j) may overwrite S_x(j-1) once the softmax has it in
          // registers; otherwise it follows PV_x(j-1) (which read P_x(j-1)
          // from these columns) in issue order.
          FA_TRACE(8, x, ns[x]);
          if (Cfg::PSEP && ns[x] > 0) {
            mbar_wait_warp(&s_empty[x], (ns[x] - 1) & 1);
            tc_fence_after();
          }
          const uint32_t k_addr = tile_ready(t0 + 2 * j);
          const uint32_t q_addr = sQa + (2 * qb + x) * Cfg::TILE;
          FA_TRACE(10, x, ns[x]);
          const uint64_t qd = make_desc(q_addr, 16, 1024), kd = make_desc(k_addr, 16, 1024);
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * ATOM + (kk & 3) * 32;
            if (elect_one()) tc_mma(tb + Cfg::col_s(x), desc_add(qd, off), desc_add(kd, off), idesc_s, kk != 0);
          }
          if (elect_one()) tc_commit(&s_full[x]);
          __syncwarp();
          FA_TRACE(1, x, ns[x]);
          ++ns[x];
        };
        auto issue_pv = [&](int x, int j) {
          FA_TRACE(9, x, npv[x]);
          mbar_wait_warp(&p_full[x], npv[x] & 1);
          tc_fence_after();
          const uint32_t v_addr = tile_ready(t0 + 2 * j + 1);
          FA_TRACE(11, x, npv[x]);
          const uint64_t vd = make_desc(v_addr, ATOM, 1024);
#pragma unroll
          for (int kk = 0; kk < KT / 16; ++kk) {
            if (elect_one())
              tc_mma_ts(tb + Cfg::col_o(x), tb + Cfg::col_p(x) + kk * 8, desc_add(vd, kk * 2048), idesc_pv,
                        (j | kk) != 0);
          }
          if (elect_one()) tc_commit(&o_done[x]);
          __syncwarp();
          FA_TRACE(2, x, npv[x]);
          ++npv[x];
        };
        // K_j is freed after its last S (S_B(j), or S_A(j) past B's range),
        // V_j after its last PV; Q after the item's last S.
        auto last_s = [&](int x, int j) { return x == 1 || j >= nkv[1]; };
        if (nkv[0] > 0) {
          issue_s(0, 0);
          if (last_s(0, 0)) free_tile(t0);
        }
        if (nkv[1] > 0) {
          issue_s(1, 0);
          free_tile(t0);
        }
        for (int j = 0; j < it.n_max; ++j) {
          if constexpr (Cfg::PSEP) {
            // S_x(j+1) as soon as the softmax read S_x(j), then the PVs.
            for (int x = 0; x < 2; ++x)
              if (j + 1 < nkv[x]) {
                issue_s(x, j + 1);
                if (last_s(x, j + 1)) free_tile(t0 + 2 * (j + 1));
              }
            for (int x = 0; x < 2; ++x)
              if (j < nkv[x]) {
                issue_pv(x, j);
                if (last_s(x, j)) free_tile(t0 + 2 * j + 1);
              }
          } else {
            // PV_x(j) then S_x(j+1) (over P_x(j)'s columns) per warpgroup; the
            // other warpgroup's softmax overlaps both.
            for (int x = 0; x < 2; ++x) {
              if (j >= nkv[x]) continue;
              issue_pv(x, j);
              if (last_s(x, j)) free_tile(t0 + 2 * j + 1);
              if (j + 1 < nkv[x]) {
                issue_s(x, j + 1);
                if (last_s(x, j + 1)) free_tile(t0 + 2 * (j + 1));
              }
            }
          }
          if (j + 2 == it.n_max || it.n_max == 1) {  // every S of the item issued
            if (elect_one()) tc_commit(&q_empty[qb]);
            __syncwarp();
          }
        }
        t0 += 2 * it.n_max;
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 216;");
    // ---------------------------------------------------------- softmax
    const int x = (warp - 4) >> 2;  // 0: tile A, 1: tile B
    const int ew = warp & 3;
    const int r = ew * 32 + lane;  // query row within the tile
    const uint32_t lane_base = static_cast<uint32_t>(ew * 32) << 16;
    const uint32_t s_col = tmem + lane_base + Cfg::col_s(x);
    const uint32_t p_col = tmem + lane_base + Cfg::col_p(x);
    const uint32_t o_col = tmem + lane_base + Cfg::col_o(x);
    int n = 0;  // tiles of this warpgroup so far (all items): barrier phases
    int pending = -1;  // Q buffer whose O store is in flight (released once its smem read is done)
    auto release = [&]() {
      if (pending >= 0 && lane == 0) {
        bulk_wait_read<0>();
        mbar_arrive(&q_empty[pending]);
      }
      pending = -1;
    };
    for (int k = 0;; ++k) {
      const int w = fa_item_index(k);
      if (w >= p.n_items) break;
      const FaItem it = fa_item(p, w);
      const int qb = k & 1;
      const int n_kv = x ? it.nkv1 : it.nkv0;
      if (n_kv == 0) {
        release();
        if (lane == 0) mbar_arrive(&q_empty[qb]);
        continue;
      }
      const int qt = it.qt0 + x;
      const int q = qt * QT + r;  // query position
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kv; ++j, ++n) {
        if (lane == 0 && ew == 0) FA_TRACE(3, x, n);
        mbar_wait(&s_full[x], n & 1);
        tc_fence_after();
        if (lane == 0 && ew == 0) FA_TRACE(4, x, n);
        // The whole S row in registers (4 loads, one wait).
        float sv[KT];
        tmem_ld32x4(s_col, sv);
        if constexpr (Cfg::PSEP) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_empty[x]);  // S_x(j+1) may overwrite these columns
        }
        if (p.causal && j == qt) {  // diagonal tile: keys after the query masked
#pragma unroll
          for (int c = 0; c < KT; ++c) sv[c] = c > r ? -INFINITY : sv[c];
        }
        // Row max: four independent 3-input max chains (FMNMX3).
        float m4[4] = {sv[0], sv[1], sv[2], sv[3]};
#pragma unroll
        for (int c = 4; c + 8 <= KT; c += 8) {
#pragma unroll
          for (int u = 0; u < 4; ++u) m4[u] = fmax3(m4[u], sv[c + u], sv[c + 4 + u]);
        }
        // columns KT-4 .. KT-1 close the chains
        float mx = fmax3(fmax3(m4[0], m4[1], sv[KT - 4]), fmax3(m4[2], m4[3], sv[KT - 3]),
                         fmaxf(sv[KT - 2], sv[KT - 1]));
        mx *= p.scale_log2;
        float alpha = 1.f;
        if (mx > m_used + kRescaleThreshold) {
          alpha = ex2(m_used - mx);  // 0 on the first tile
          m_used = mx;
          l *= alpha;
        }
        // P = 2^(s*scale - m): packed scale, POLY of every 8 pairs on
        // the FMA pipe, the rest on the SFU; four packed partial sums.
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(-m_used, -m_used);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < KT; c += 2) {
          float2 e = ffma2(make_float2(sv[c], sv[c + 1]), sc2, nm2);
          if (((c >> 1) & 7) < POLY) {
            e = ex2_poly2(e);
          } else {
            e.x = ex2(e.x);
            e.y = ex2(e.y);
          }
          sv[c] = e.x;
          sv[c + 1] = e.y;
          acc[(c >> 1) & 3] = fadd2(acc[(c >> 1) & 3], e);
        }
        const float2 s01 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        l += s01.x + s01.y;
        if (j > 0) {
          if (lane == 0 && ew == 0) FA_TRACE(5, x, n);
          mbar_wait(&o_done[x], (n - 1) & 1);  // PV_x(j-1) done: O settled, P buffer free
          tc_fence_after();
          if (lane == 0 && ew == 0) FA_TRACE(6, x, n);
        }
        // P row -> bf16x2 -> TMEM (A operand of PV).
#pragma unroll
        for (int qq = 0; qq < KT / 32; ++qq) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            __nv_bfloat162 h2 = __floats2bfloat162_rn(sv[32 * qq + 2 * i], sv[32 * qq + 2 * i + 1]);
            pk[i] = *reinterpret_cast<uint32_t*>(&h2);
          }
          tmem_st16(p_col + 16 * qq, pk);
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
        if (lane == 0 && ew == 0) FA_TRACE(7, x, n);
        if (j == 0) release();  // the previous item's O store has long left smem
      }
      // Epilogue: O / l -> bf16 ctx row; the next item's S_x(0) (already
      // issued) overlaps it, its PV_x(0) follows this warpgroup's next P.
      mbar_wait(&o_done[x], (n - 1) & 1);
      tc_fence_after();
      // O rows -> bf16 into this item's Q_x tile (SW128, the layout Q came
      // in; its last S is done: o_done follows it) -> TMA store of the
      // warp's 32 rows, coalesced; the buffer is released to the next Q
      // load once the store has read it (next item's first P, or the end).
      const float inv = 1.f / l;
      uint8_t* sO = sQ + (2 * qb + x) * Cfg::TILE;
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
          *reinterpret_cast<uint4*>(sO + swz(r, (c + g) >> 3)) = u;
        }
      }
      tc_fence_before();
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
#pragma unroll
        for (int a = 0; a < D / 64; ++a)
          tma_store_4d(&map_o, sO + a * ATOM + ew * 32 * 128, a * 64, it.head, qt * QT + ew * 32, it.b);
        bulk_commit();
      }
      pending = qb;
      p.lse2[(static_cast<int64_t>(it.b) * p.heads + it.head) * p.seq + q] = m_used + __log2f(l);
    }
    release();
    if (lane == 0) bulk_wait<0>();
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

int fa_poly(int d) {
  static const int v = [] {
    const char* e = std::getenv("WP_FA_POLY");
    return e ? std::atoi(e) : -1;
  }();
  return v >= 0 ? v : (d == 64 ? kFaPolyD64 : kFaPolyD128);
}

// {D, heads, seq, mbs} view of ctx [T, hidden]; box {64, 1, 32, 1}: one
// warp's 32 rows of one 64-column atom (the forward's O store).
CUtensorMap ctx_map(void* base, const AttnShape& s) {
  CUtensorMap m;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(s.head_dim), static_cast<cuuint64_t>(s.heads),
                        static_cast<cuuint64_t>(s.seq), static_cast<cuuint64_t>(s.mbs)};
  const uint64_t ld = static_cast<uint64_t>(s.hidden) * 2;
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(s.head_dim) * 2, ld, ld * s.seq};
  cuuint32_t box[4] = {64, 1, 32, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = get_encoder()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, base, dims, strides, box, estr,
                                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                   CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw std::runtime_error("attention ctx tensor map: " + std::to_string(int(r)));
  return m;
}

template <int D, int POLY>
void launch_fwd(const AttnShape& s, const void* qkv, void* ctx, float* lse2, cudaStream_t stream) {
  auto* k = flash_fwd_kernel<D, POLY>;
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
  p.n_items = p.n_pairs * s.heads * s.mbs;
  const int grid = std::min(p.n_items, num_sms());  // persistent: one CTA per SM
  const CUtensorMap mo = ctx_map(ctx, s);
  k<<<grid, FA_THREADS, FaCfg<D>::SMEM, stream>>>(mq, mk, mv, mo, p);
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
  const int poly = fa_poly(s.head_dim);
  if (s.head_dim == 128) {
    switch (poly) {
      case 0: launch_fwd<128, 0>(s, qkv, ctx, lse2, stream); break;
      case 2: launch_fwd<128, 2>(s, qkv, ctx, lse2, stream); break;
      case 4: launch_fwd<128, 4>(s, qkv, ctx, lse2, stream); break;
      case 5: launch_fwd<128, 5>(s, qkv, ctx, lse2, stream); break;
      default: launch_fwd<128, 3>(s, qkv, ctx, lse2, stream); break;
    }
  } else {
    switch (poly) {
      case 0: launch_fwd<64, 0>(s, qkv, ctx, lse2, stream); break;
      case 2: launch_fwd<64, 2>(s, qkv, ctx, lse2, stream); break;
      case 3: launch_fwd<64, 3>(s, qkv, ctx, lse2, stream); break;
      case 5: launch_fwd<64, 5>(s, qkv, ctx, lse2, stream); break;
      default: launch_fwd<64, 4>(s, qkv, ctx, lse2, stream); break;
    }
  }
  return 1;
}

}  // namespace wpk
