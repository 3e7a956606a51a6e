// Flash attention backward on the 5th-gen tensor cores (sm_100a).
//
// Work item = (128-key tile j, head, sequence): K_j and V_j stay in shared
// memory while the query tiles i (causal: i >= j) stream through.  Per q tile:
//   MMA        S^T  = K_j Q_i^T      (M=keys, N=queries, K=D)   -> TMEM
//              dP^T = V_j dO_i^T     (M=keys, N=queries, K=D)   -> TMEM
//   softmax    16 warps, one key row per thread, four 32-query quarters
//              (four warps per TMEM lane quadrant hide each other's TMEM
//              and barrier latencies): P^T = 2^(s - lse2) -> bf16 back into
//              the quarter's own S^T columns (A of dV);
//              dS^T = P^T * (dP^T - Delta) / sqrt(D)  -> bf16 -> smem (SW128)
//   MMA        dV_j += P^T dO_i (A from TMEM), dK_j += dS^T Q_i (accumulators
//              in TMEM), dQ_i = dS K_j (A = the dS^T tile read MN-major)
//   dQ warps   4 warps drain dQ_i from TMEM through their own fp32 SW128
//              slabs with TMA bulk reduce-adds into an fp32 accumulator
//              (every key tile contributes to each q tile); after an item's
//              last tile they also write its dK / dV rows
// Issue order (FA4's): S^T(i+1), dQ_i (two D halves, own commits), dK_j(i),
// dP^T(i+1) once the drain read dQ_i out of the shared columns, dV(i+1) as
// soon as P^T(i+1) is in TMEM -- the next tile's softmax overlaps this
// tile's dQ / dK and the drain.  Persistent CTAs (one per SM) walk the items
// in a grouped, heaviest-first raster (see bw_item), snake-ordered across
// CTAs; V is reloaded for the next item after the last dP^T, K after the
// last dQ; lse / Delta of each tile arrive by bulk copy off the softmax
// critical path; dK / dV leave through the drain slabs by TMA stores.
// 768 threads (80 registers each): every role works in 32-column pieces.
// Delta = rowsum(dO * O) comes from the projection GEMM's epilogue (or
// attn_bwd_prep); dq_finish converts the fp32 dQ accumulator to bf16 into dqkv.
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
#ifdef WP_BW_TRACE
// Debug timeline of CTA 0 (build with -DWP_BW_TRACE; tools/bw_trace_probe.py):
// clock64 per (event, global tile g < 32).
__device__ unsigned long long g_bwt[16 * 32];
__device__ unsigned long long g_bw_cta[2 * 160];  // per-CTA start / end (%globaltimer)
#define BWT(ev, j)                                                        \
  do {                                                                    \
    if (blockIdx.x == 0 && (j) < 32) g_bwt[(ev) * 32 + (j)] = clock64(); \
  } while (0)
#else
#define BWT(ev, j) \
  do {             \
  } while (0)
#endif
namespace {

using namespace tc;
using namespace smx;

// Of every 8 column pairs of a P^T row, this many take the FMA-pipe 2^x
// (0: measured 0 / 2 / 4 -> the backward is not SFU-bound; 0 is 1-3 %
// ahead of 2 at D 64 and even at D 128).
constexpr int kBwPoly = 0;

constexpr int T128 = 128;
constexpr int ATOM = 128 * 64 * 2;  // SW128 atom: 128 rows x 64 bf16
constexpr int SM_WARPS = 16;        // softmax warps: four per TMEM lane quadrant, 32 query columns each
constexpr int BW_THREADS = 32 * (4 + SM_WARPS + 4);  // warps 0-3 control, 4-19 softmax, 20-23 dQ drain
constexpr uint32_t kColS = 0, kColDP = 128, kColDV = 256;

template <int D>
struct BwCfg {
  static constexpr int TILE = T128 * D * 2;     // K, V, Q, dO tiles
  static constexpr int PT = T128 * T128 * 2;    // dS^T tile
  static constexpr int STAGE = 4 * 2 * SLAB_BYTES;  // dQ drain: 2 fp32 slabs per drain warp
  // K, V, Q[2], dO, dS^T, drain slabs, lse/delta (single-buffered), barriers
  static constexpr int SMEM = 5 * TILE + PT + STAGE + 2 * T128 * 4 + 1024 + 256;  // 16 barriers + TMEM slot
  static constexpr uint32_t kColDK = kColDV + D;
  // dQ: at D = 64 the accumulators leave 128 columns free, so dQ gets its
  // own (dP^T(next) need not wait for the drain); at D = 128 it reuses the
  // dP^T columns.
  static constexpr bool DQ_OWN = D == 64;
  static constexpr uint32_t kColDQ = DQ_OWN ? kColDK + D : kColDP;
};

// dV += P^T dO with P^T read from tensor memory (kind::f16, A in TMEM: lane =
// key row, 32-bit column j = queries 2j, 2j+1 packed as bf16x2).
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

// 16 consecutive 32-bit TMEM columns of this warp's 32 lanes.
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]));
}

struct BwParams {
  int batch, seq, heads, n_tiles, causal, hidden;
  int group;  // (batch, head) pairs per raster group (0: all)
  int dq_halves;  // D = 128: dQ as two N = 64 MMA groups (A/B switch)
  float scale_log2, scale;
  const float* lse2;
  const float* delta;
  float* dq_acc;                // [T, h] fp32
  __nv_bfloat16* dqkv;          // [T, 3h]
  float* dbias;                 // [3h] fp32 QKV bias gradient (+=), or null
};


__device__ __forceinline__ uint32_t swz(int r, int c) {  // 16-B chunk c of row r, SW128 K-major atoms
  const int atom = c >> 3, cc = c & 7;
  return atom * ATOM + (r >> 3) * 1024 + (r & 7) * 128 + ((cc ^ (r & 7)) << 4);
}



// One work item = (key tile kj, batch b, head).  Items in raster order:
// groups of p.group (batch, head) pairs; inside a group heaviest-first (LPT):
// every pair's key tile 0 -- the most causal query tiles -- before tile 1,
// and so on.  A group's fp32 dQ accumulator and its Q / dO stay L2-resident
// while all its key tiles reduce into / read them.
struct BwItem {
  int kj, b, head, i0, n_it;
};
__device__ __forceinline__ BwItem bw_item(const BwParams& p, int w) {
  const int bh_all = p.batch * p.heads;
  const int G = p.group > 0 && p.group < bh_all ? p.group : bh_all;
  const int grp = w / (p.n_tiles * G);
  const int gsz = min(G, bh_all - grp * G);
  const int rem = w - grp * p.n_tiles * G;
  BwItem it;
  it.kj = rem / gsz;
  const int bhi = grp * G + rem % gsz;
  it.head = bhi % p.heads;
  it.b = bhi / p.heads;
  it.i0 = p.causal ? it.kj : 0;
  it.n_it = p.n_tiles - it.i0;
  return it;
}

// Item of this CTA's k-th round: the item list in snake order across the
// CTAs (CTAs 0..G-1 on even rounds, G-1..0 on odd ones), which evens out the
// per-CTA sums of the heaviest-first item sizes.
__device__ __forceinline__ int bw_item_index(int k) {
  const int G = static_cast<int>(gridDim.x), c = static_cast<int>(blockIdx.x);
  return k * G + ((k & 1) ? G - 1 - c : c);
}

// Persistent: one CTA per SM walks its items (bw_item_index(0), (1), ...)
// Per-tile barriers run on the CTA's global tile counter g (across items),
// per-item ones on its item counter, so the next item's K/V load, S^T and
// dP^T overlap the previous item's dK / dV epilogue (done by the dQ drain
// warps), and TMEM / barriers are set up once.
template <int D>
__global__ void __launch_bounds__(BW_THREADS, 1)
    flash_bwd_kernel(const __grid_constant__ CUtensorMap map_q, const __grid_constant__ CUtensorMap map_k,
                     const __grid_constant__ CUtensorMap map_v, const __grid_constant__ CUtensorMap map_do,
                     const __grid_constant__ CUtensorMap map_dq, const __grid_constant__ CUtensorMap map_dqkv,
                     const __grid_constant__ BwParams p) {
  using Cfg = BwCfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + Cfg::TILE;
  uint8_t* sQ = sV + Cfg::TILE;       // [2]
  uint8_t* sDO = sQ + 2 * Cfg::TILE;  // single
  uint8_t* sDS = sDO + Cfg::TILE;     // dS^T [keys x queries]
  uint8_t* sStage = sDS + Cfg::PT;    // dQ drain slabs
  float* sLse = reinterpret_cast<float*>(sStage + Cfg::STAGE);  // [128]
  float* sDelta = sLse + T128;                                   // [128]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sDelta + T128);
  uint64_t* kv_full = bars + 0;
  uint64_t* q_full = bars + 1;   // [2]
  uint64_t* q_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;
  uint64_t* ds_full = bars + 6;
  uint64_t* pds_free = bars + 7;
  uint64_t* dq_full = bars + 8;
  uint64_t* dq_free = bars + 9;
  uint64_t* dkv_done = bars + 10;
  uint64_t* dp_full = bars + 11;
  uint64_t* do_full = bars + 12;
  uint64_t* do_empty = bars + 13;
  uint64_t* p_full = bars + 14;    // P^T of the tile written to TMEM (dV may start)
  uint64_t* lse_full = bars + 15;  // the tile's lse / Delta rows landed (bulk copies by warp 3)
  uint64_t* dl_full = bars + 16;
  uint64_t* kv_empty = bars + 17;  // the item's last MMA read K (its last dQ)
  uint64_t* v_empty = bars + 21;   // the item's last MMA read V (its last dP^T)
  uint64_t* dkv_free = bars + 18;  // the item's dK / dV read out of TMEM (epilogue)
  // The drain reads dQ in two D halves, each with its full / free barrier.
  uint64_t* dq_full_h[2] = {dq_full, bars + 19};
  uint64_t* dq_free_h[2] = {dq_free, bars + 20};
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 22);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_items = p.n_tiles * p.batch * p.heads;

  if (warp == 0 && lane == 0) {
    for (const CUtensorMap* m : {&map_q, &map_k, &map_v, &map_do})
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    mbar_init(kv_full, 1);
    mbar_init(kv_empty, 1);
    mbar_init(v_empty, 1);
    for (int x = 0; x < 2; ++x) {
      mbar_init(&q_full[x], 1);
      mbar_init(&q_empty[x], 1);
    }
    mbar_init(do_full, 1);
    mbar_init(do_empty, 1);
    mbar_init(s_full, 1);
    mbar_init(ds_full, SM_WARPS);
    mbar_init(pds_free, 1);  // dK and dQ MMAs done reading dS^T
    for (int h = 0; h < 2; ++h) {
      mbar_init(dq_full_h[h], 1);
      mbar_init(dq_free_h[h], 4);
    }
    mbar_init(dkv_done, 1);
    mbar_init(dkv_free, 4);
    mbar_init(dp_full, 1);
    mbar_init(p_full, SM_WARPS);
    mbar_init(lse_full, 1);
    mbar_init(dl_full, 1);
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
#ifdef WP_BW_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 160) g_bw_cta[2 * blockIdx.x] = global_ns();
#endif

  if (warp == 0) {
    if (lane == 0) {
      int g = 0;  // global tile counter
      int ip = 0;
      for (int w = bw_item_index(0); w < n_items; w = bw_item_index(ip + 1), ++ip) {
        const BwItem itm = bw_item(p, w);
        for (int t = 0; t < itm.n_it; ++t, ++g) {  // Q double-buffered (two tiles ahead), dO single
          const int qi = itm.i0 + t, x = g & 1;
          if (g >= 2) mbar_wait(&q_empty[x], ((g - 2) >> 1) & 1);
          mbar_expect_tx(&q_full[x], Cfg::TILE);
#pragma unroll
          for (int a = 0; a < D / 64; ++a)
            tma_load_4d(&map_q, &q_full[x], sQ + x * Cfg::TILE + a * ATOM, a * 64, itm.head, qi * T128, itm.b);
          // Two tiles before this item ends, warm L2 with the next item's
          // K / V (single-buffered in shared memory, they are loaded only
          // once this item's last dP^T / dQ read the current ones).
          if (t == max(0, itm.n_it - 2)) {
            const int wn = bw_item_index(ip + 1);
            if (wn < n_items) {
              const BwItem nx = bw_item(p, wn);
#pragma unroll
              for (int a = 0; a < D / 64; ++a) {
                tma_prefetch_4d(&map_k, a * 64, nx.head, nx.kj * T128, nx.b);
                tma_prefetch_4d(&map_v, a * 64, nx.head, nx.kj * T128, nx.b);
              }
            }
          }
          if (g >= 1) mbar_wait(do_empty, (g - 1) & 1);  // dV(g-1) read dO(g-1)
          mbar_expect_tx(do_full, Cfg::TILE);
#pragma unroll
          for (int a = 0; a < D / 64; ++a)
            tma_load_4d(&map_do, do_full, sDO + a * ATOM, a * 64, itm.head, qi * T128, itm.b);
          if (t == 0) {  // K / V after the first Q / dO: those buffers free up earlier
            // V as soon as the previous item's last dP^T read it, K after its
            // last dQ (the dV / dK MMAs of that tile still run)
            mbar_expect_tx(kv_full, 2 * Cfg::TILE);
            if (ip > 0) mbar_wait(v_empty, (ip - 1) & 1);
#pragma unroll
            for (int a = 0; a < D / 64; ++a)
              tma_load_4d(&map_v, kv_full, sV + a * ATOM, a * 64, itm.head, itm.kj * T128, itm.b);
            if (ip > 0) mbar_wait(kv_empty, (ip - 1) & 1);
#pragma unroll
            for (int a = 0; a < D / 64; ++a)
              tma_load_4d(&map_k, kv_full, sK + a * ATOM, a * 64, itm.head, itm.kj * T128, itm.b);
          }
        }
      }
    }
  } else if (warp == 3) {
    if (lane == 0) {
      // lse and Delta of each query tile, single-buffered: the tile's lse
      // as soon as the softmax warps finished phase A of the previous tile
      // (p_full), its Delta once they finished phase B (ds_full) -- each
      // lands while the other phase runs, off the softmax critical path.
      int g = 0;
      for (int kk = 0, w = bw_item_index(0); w < n_items; w = bw_item_index(++kk)) {
        const BwItem itm = bw_item(p, w);
        for (int t = 0; t < itm.n_it; ++t, ++g) {
          const int64_t vec = (static_cast<int64_t>(itm.b) * p.heads + itm.head) * p.seq + (itm.i0 + t) * T128;
          if (g > 0) mbar_wait(p_full, (g - 1) & 1);
          mbar_expect_tx(lse_full, T128 * 4);
          bulk_load(sLse, p.lse2 + vec, T128 * 4, lse_full);
          if (g > 0) mbar_wait(ds_full, (g - 1) & 1);
          mbar_expect_tx(dl_full, T128 * 4);
          bulk_load(sDelta, p.delta + vec, T128 * 4, dl_full);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // M=128 N=128 K-major/K-major (S^T, dP^T); M=128 N=D K-major A / MN-major B (dV, dK);
      // M=128 N=D MN-major A / MN-major B (dQ).
      constexpr uint32_t id_ss = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(T128 >> 3) << 17) |
                                 (uint32_t(T128 >> 4) << 24);
      constexpr uint32_t id_kv = (1u << 4) | (1u << 7) | (1u << 10) | (1u << 16) | (uint32_t(D >> 3) << 17) |
                                 (uint32_t(T128 >> 4) << 24);
      constexpr uint32_t id_dq = id_kv | (1u << 15);
      constexpr uint32_t id_dq_half = (id_dq & ~(0x3Fu << 17)) | (uint32_t(64 >> 3) << 17);  // N=64 (D=128 halves)
      const uint32_t aK = smem_u32(sK), aV = smem_u32(sV), aDS = smem_u32(sDS);
      // K-major (k-step offsets in-atom) and MN-major (2 KB per 16 rows) descriptors
      const uint64_t dK = make_desc(aK, 16, 1024), dV = make_desc(aV, 16, 1024), dDS = make_desc(aDS, 16, 1024);
      const uint64_t dDSm = make_desc(aDS, ATOM, 1024), dKm = make_desc(aK, ATOM, 1024);
      const uint64_t dDO = make_desc(smem_u32(sDO), 16, 1024), dDOm = make_desc(smem_u32(sDO), ATOM, 1024);
      // S^T(g) = K Q^T and dP^T(g) = V dO^T (reduction over D), committed
      // separately: the softmax turns S into P while the previous tile's dQ
      // is still being drained from the dP^T columns.
      auto issue_s = [&](int g) {
        const int x = g & 1;
        const uint64_t dQ = make_desc(smem_u32(sQ + x * Cfg::TILE), 16, 1024);
        mbar_wait(&q_full[x], (g >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * ATOM + (k & 3) * 32;
          tc_mma(tmem + kColS, desc_add(dK, off), desc_add(dQ, off), id_ss, k != 0);
        }
        tc_commit(s_full);
        BWT(3, g);
      };
      // dP^T(g) = V dO^T into the dP^T columns once the drain read dQ(g-1)
      // (both halves) out of them.
      auto issue_dp = [&](int g) {
        mbar_wait(do_full, g & 1);
        if (g > 0 && !Cfg::DQ_OWN) {
          mbar_wait(dq_free_h[0], (g - 1) & 1);
          mbar_wait(dq_free_h[1], (g - 1) & 1);
        }
        tc_fence_after();
        BWT(4, g);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * ATOM + (k & 3) * 32;
          tc_mma(tmem + kColDP, desc_add(dV, off), desc_add(dDO, off), id_ss, k != 0);
        }
        tc_commit(dp_full);
      };
      // dV += P^T(g) dO(g), P^T from TMEM (queries [0,64) at columns 0..,
      // [64,128) at 64..), as soon as the softmax warps wrote P^T -- before
      // dS^T(g) exists, so S^T(g+1) can follow right away and the next
      // tile's P^T overlaps this tile's dS^T.  first: the item's first tile
      // (overwrite the accumulator).
      auto issue_dv = [&](int g, bool first) {
        mbar_wait(p_full, g & 1);
        tc_fence_after();
        BWT(12, g);
#pragma unroll
        for (int k = 0; k < T128 / 16; ++k)
          tc_mma_ts(tmem + kColDV, tmem + kColS + (k >> 1) * 32 + (k & 1) * 8, desc_add(dDOm, k * 2048), id_kv,
                    !(first && k == 0));
        tc_commit(do_empty);
      };
      int g = 0, ip = 0;
      for (int w = bw_item_index(0); w < n_items; w = bw_item_index(ip + 1), ++ip) {
        const BwItem itm = bw_item(p, w);
        mbar_wait(kv_full, ip & 1);
        tc_fence_after();
        const int g0 = g;
        issue_s(g0);
        issue_dp(g0);
        if (itm.n_it == 1) tc_commit(v_empty);  // the item's last dP^T: V may be reloaded
        if (ip > 0) mbar_wait(dkv_free, (ip - 1) & 1);  // previous item's dK / dV read out of TMEM
        issue_dv(g0, true);
        for (int t = 0; t < itm.n_it; ++t, ++g) {
          const int x = g & 1;
          const uint64_t dQm = make_desc(smem_u32(sQ + x * Cfg::TILE), ATOM, 1024);
          // S^T(g+1) over the P^T(g) columns: in order after dV(g), which read them
          if (t + 1 < itm.n_it) issue_s(g + 1);
          mbar_wait(ds_full, g & 1);
          tc_fence_after();
          BWT(1, g);
          // dQ = dS K (reduction over the 128 keys; dS^T tile read M-major)
          // into the dP^T columns, first and in two D halves with their own
          // commits, so the drain of the first half starts while the second
          // half and dK run.
          // (Two N = 64 halves with their own commits let the drain start
          // earlier but double the MMA instructions, each of which costs
          // about as much at N = 64 as at N = 128: one N = D group by
          // default, halves with WP_BW_DQ_HALVES=1.)
          if (D == 128 && p.dq_halves) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
#pragma unroll
              for (int k = 0; k < T128 / 16; ++k)
                tc_mma(tmem + kColDP + 64 * h, desc_add(dDSm, k * 2048), desc_add(dKm, h * ATOM + k * 2048),
                       id_dq_half, k != 0);
              tc_commit(dq_full_h[h]);
              BWT(14 + h, g);
            }
          } else {  // one N = D group; the drain still reads it in two halves
            if (Cfg::DQ_OWN && g > 0) {  // own columns: the drain must have read dQ(g-1)
              mbar_wait(dq_free_h[0], (g - 1) & 1);
              mbar_wait(dq_free_h[1], (g - 1) & 1);
              tc_fence_after();
            }
#pragma unroll
            for (int k = 0; k < T128 / 16; ++k)
              tc_mma(tmem + Cfg::kColDQ, desc_add(dDSm, k * 2048), desc_add(dKm, k * 2048), id_dq, k != 0);
            tc_commit(dq_full_h[0]);
            tc_commit(dq_full_h[1]);
          }
          if (t + 1 == itm.n_it) tc_commit(kv_empty);  // the item's last dQ: K may be reloaded
          // dK += dS^T Q (reduction over the 128 queries)
#pragma unroll
          for (int k = 0; k < T128 / 16; ++k) {
            const uint32_t offa = (k >> 2) * ATOM + (k & 3) * 32;
            tc_mma(tmem + Cfg::kColDK, desc_add(dDS, offa), desc_add(dQm, k * 2048), id_kv, (t | k) != 0);
          }
          tc_commit(&q_empty[x]);
          tc_commit(pds_free);
          BWT(2, g);
          if (t + 1 < itm.n_it) {
            issue_dp(g + 1);  // after the drain read dQ(g) out of TMEM
            if (t + 2 == itm.n_it) tc_commit(v_empty);
            issue_dv(g + 1, false);
          }
        }
        tc_commit(dkv_done);
      }
    }
  } else if (warp >= 4 && warp < 4 + SM_WARPS) {
    // -------------------------------------------------- P^T / dS^T (key rows)
    // Four warps per TMEM lane quadrant: `grp` picks query columns
    // [32 grp, 32 grp + 32); its packed P^T goes to S^T columns
    // [32 grp, 32 grp + 16), inside the columns it alone reads.
    const int ew = warp & 3;
    const int grp = (warp - 4) >> 2;
    const int c0 = grp * 32;
    const int r = ew * 32 + lane;
    const uint32_t lb = static_cast<uint32_t>(ew * 32) << 16;
    int g = 0;
    for (int kk = 0, w = bw_item_index(0); w < n_items; w = bw_item_index(++kk)) {
      const BwItem itm = bw_item(p, w);
      for (int t = 0; t < itm.n_it; ++t, ++g) {
        const float* lse = sLse;
        const float* dl = sDelta;
        mbar_wait(lse_full, g & 1);
        mbar_wait(s_full, g & 1);
        tc_fence_after();
        if (warp == 4 && lane == 0) BWT(5, g);
        const bool diag = p.causal && itm.i0 + t == itm.kj;
        // Phase A: P^T = 2^(s*scale - lse) from S^T alone; kept in registers
        // for dS and written back over this warp's S^T columns (bf16x2) as
        // the A operand of dV += P^T dO.
        float pv[32];
        tmem_ld32(tmem + lb + kColS + c0, pv);
        const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
#pragma unroll
        for (int i = 0; i < 32; i += 4) {
          const float4 l4 = *reinterpret_cast<const float4*>(lse + c0 + i);  // broadcast
#pragma unroll
          for (int u = 0; u < 2; ++u) {
            float2 e = ffma2(make_float2(pv[i + 2 * u], pv[i + 2 * u + 1]), sc2,
                             u ? make_float2(-l4.z, -l4.w) : make_float2(-l4.x, -l4.y));
            if ((((i >> 1) + u) & 7) < kBwPoly) {
              e = ex2_poly2(e);
            } else {
              e.x = ex2(e.x);
              e.y = ex2(e.y);
            }
            const int c = c0 + i + 2 * u;
            pv[i + 2 * u] = (diag && c < r) ? 0.f : e.x;
            pv[i + 2 * u + 1] = (diag && c + 1 < r) ? 0.f : e.y;
          }
        }
        {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            __nv_bfloat162 hh = __floats2bfloat162_rn(pv[2 * i], pv[2 * i + 1]);
            pk[i] = *reinterpret_cast<uint32_t*>(&hh);
          }
          tmem_st16(tmem + lb + kColS + c0, pk);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) pv[i] *= p.scale;  // dS = (dP - Delta) * (P / sqrt(D))
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);  // P^T in TMEM: dV(g) may start
        if (warp == 4 && lane == 0) BWT(6, g);
        // Phase B: dS^T = P^T * (dP^T - Delta) / sqrt(D) once dP^T is in.
        mbar_wait(dp_full, g & 1);
        mbar_wait(dl_full, g & 1);
        tc_fence_after();
        if (warp == 4 && lane == 0) BWT(7, g);
        if (g > 0) mbar_wait(pds_free, (g - 1) & 1);  // dS^T buffer free (dK(g-1), dQ(g-1) read it)
        if (warp == 4 && lane == 0) BWT(8, g);
        {
          float dp[32];
          tmem_ld32(tmem + lb + kColDP + c0, dp);
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            const float4 d4 = *reinterpret_cast<const float4*>(dl + c0 + i);
            const float2 a0 = fmul2(make_float2(pv[i], pv[i + 1]), fadd2(make_float2(dp[i], dp[i + 1]),
                                                                         make_float2(-d4.x, -d4.y)));
            const float2 a1 = fmul2(make_float2(pv[i + 2], pv[i + 3]), fadd2(make_float2(dp[i + 2], dp[i + 3]),
                                                                             make_float2(-d4.z, -d4.w)));
            dp[i] = a0.x, dp[i + 1] = a0.y, dp[i + 2] = a1.x, dp[i + 3] = a1.y;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            uint4 ud;
            __nv_bfloat162* hd = reinterpret_cast<__nv_bfloat162*>(&ud);
#pragma unroll
            for (int i = 0; i < 4; ++i) hd[i] = __floats2bfloat162_rn(dp[8 * q + 2 * i], dp[8 * q + 2 * i + 1]);
            *reinterpret_cast<uint4*>(sDS + swz(r, c0 / 8 + q)) = ud;
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_full);
        if (warp == 4 && lane == 0) BWT(9, g);
      }
    }
  } else if (warp >= 4 + SM_WARPS) {
    // ----------------------------- dQ drain (query rows) and dK / dV epilogue
    // TMEM -> fp32 SW128 slabs (two per warp, in their own buffer) -> TMA
    // bulk reduce-add into dq_acc: whole 128-byte row segments reduced in L2
    // instead of per-lane atomics.  The row is read out of TMEM in two halves
    // and dq_free is raised as soon as the second half is in registers, so
    // the next dP^T overlaps the reduce-adds.  After an item's last tile the
    // same warps write its dK / dV rows (and the K / V bias-gradient column
    // sums), then free those TMEM columns for the next item.
    const int ew = warp & 3;
    const uint32_t lb = static_cast<uint32_t>(ew * 32) << 16;
    uint8_t* slabs = sStage + ew * 2 * SLAB_BYTES;
    constexpr int NCH = D / 32, HALF = NCH / 2;
    int g = 0, ip = 0;
    for (int w = bw_item_index(0); w < n_items; w = bw_item_index(ip + 1), ++ip) {
      const BwItem itm = bw_item(p, w);
      for (int t = 0; t < itm.n_it; ++t, ++g) {
        const int qi = itm.i0 + t;
        const int row0 = itm.b * p.seq + qi * T128 + ew * 32;
#pragma unroll
        for (int h = 0; h < 2; ++h) {  // D half h of dQ (its own MMA commit)
          mbar_wait(dq_full_h[h], g & 1);
          tc_fence_after();
          if (h == 0 && warp == 4 + SM_WARPS && lane == 0) BWT(10, g);
          if (h == 1 && warp == 4 + SM_WARPS && lane == 0) BWT(13, g);
          // 32 columns at a time (registers: 768 threads leave ~80 each);
          // the half's columns are free once its last chunk is in registers.
#pragma unroll
          for (int c = 0; c < HALF; ++c) {
            float v[32];
            tmem_ld32(tmem + lb + Cfg::kColDQ + (h * HALF + c) * 32, v);
            if (c == HALF - 1) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(dq_free_h[h]);  // these dQ columns read out: dP^T half h may start
              if (h == 1 && warp == 4 + SM_WARPS && lane == 0) BWT(11, g);
            }
            uint8_t* sb = slabs + ((h * HALF + c) & 1) * SLAB_BYTES;
            if (lane == 0) bulk_wait_read<1>();
            __syncwarp();
            slab_put_f32(sb, lane, v);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_reduce_add_2d(&map_dq, sb, itm.head * D + (h * HALF + c) * 32, row0);
              bulk_commit();
            }
          }
        }
      }
      // dK, dV rows of this key tile -> bf16 slabs (the drain's own, after
      // their last reduce-add read them) -> TMA stores into dqkv, whole
      // 128-byte row segments; the K / V bias-gradient column sums from the
      // fp32 values.
      mbar_wait(dkv_done, ip & 1);
      tc_fence_after();
      const int row_k = itm.b * p.seq + itm.kj * T128 + ew * 32;
#pragma unroll
      for (int part = 0; part < 2; ++part) {  // 0: dK, 1: dV
        const uint32_t col = part ? kColDV : Cfg::kColDK;
#pragma unroll
        for (int hc = 0; hc < D / 64; ++hc) {
          uint8_t* sb = slabs + ((part * (D / 64) + hc) & 1) * SLAB_BYTES;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {  // 32 columns at a time
            float v[32];
            tmem_ld32(tmem + lb + col + hc * 64 + 32 * h2, v);
#pragma unroll
            for (int cc = 0; cc < 4; ++cc) {
              uint4 u;
              __nv_bfloat162* hh = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
              for (int i = 0; i < 4; ++i) hh[i] = __floats2bfloat162_rn(v[8 * cc + 2 * i], v[8 * cc + 2 * i + 1]);
              *reinterpret_cast<uint4*>(sb + slab_off(lane, 4 * h2 + cc)) = u;
            }
            if (p.dbias) {
              // bias gradient: column sums of this warp's 32 key rows (a
              // transposing butterfly leaves column c + lane in v[0]), one
              // atomic per column per warp
#pragma unroll
              for (int sh = 16; sh >= 1; sh >>= 1) {
                const bool up = (lane & sh) != 0;
#pragma unroll
                for (int i = 0; i < sh; ++i) {
                  const float send = up ? v[i] : v[i + sh];
                  const float keep = up ? v[i + sh] : v[i];
                  v[i] = keep + __shfl_xor_sync(0xffffffffu, send, sh);
                }
              }
              atomicAdd(p.dbias + (part + 1) * p.hidden + itm.head * D + hc * 64 + 32 * h2 + lane, v[0]);
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&map_dqkv, sb, (part + 1) * p.hidden + itm.head * D + hc * 64, row_k);
            bulk_commit();
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dkv_free);
    }
    if (lane == 0) bulk_wait<0>();
  }

  tc_fence_before();
  __syncwarp();
  __syncthreads();
#ifdef WP_BW_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 160) g_bw_cta[2 * blockIdx.x + 1] = global_ns();
#endif
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

// Delta[b, h, q] = sum_d dO * O over the head's D columns: D/8 lanes per
// (token, head), one 16-byte load of each tensor per lane.
__global__ void attn_bwd_prep_k(const __nv_bfloat16* dout, const __nv_bfloat16* out, float* delta, int T, int heads,
                                int D, int seq, int hidden) {
  const int lpr = D / 8;  // lanes per (token, head): 16 (D = 128) or 8 (D = 64)
  const int gid = (blockIdx.x * blockDim.x + threadIdx.x) / lpr, sub = threadIdx.x % lpr;
  if (gid >= T * heads) return;
  const int t = gid / heads, hd = gid % heads;
  const int64_t off = static_cast<int64_t>(t) * hidden + hd * D + sub * 8;
  const uint4 ua = *reinterpret_cast<const uint4*>(dout + off), uo = *reinterpret_cast<const uint4*>(out + off);
  const __nv_bfloat162* a = reinterpret_cast<const __nv_bfloat162*>(&ua);
  const __nv_bfloat162* o = reinterpret_cast<const __nv_bfloat162*>(&uo);
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __bfloat1622float2(a[i]), y = __bfloat1622float2(o[i]);
    s += x.x * y.x + x.y * y.y;
  }
  for (int w = lpr / 2; w; w >>= 1) s += __shfl_xor_sync(0xffffffffu, s, w);
  if (sub == 0) {
    const int b = t / seq, q = t % seq;
    delta[(static_cast<int64_t>(b) * heads + hd) * seq + q] = s;
  }
}

// dqkv[:, 0:h] = bf16(dq_acc); with dbias, also += its column sums (the Q
// part of the QKV bias gradient).  Block = 64 columns x 256 rows: thread
// (x, y) converts 8 columns of rows y, y+32, ... (8 independent loads in
// flight), then the 32 row-partials of each column meet in shared memory
// and one atomic per column per block remains.
constexpr int DQ_COLS = 64, DQ_ROWS = 256;
__global__ void __launch_bounds__(256) dq_finish_k(const float* dq, __nv_bfloat16* dqkv, float* dbias, int T,
                                                   int hidden) {
  __shared__ float part[32][DQ_COLS + 1];
  const int tx = threadIdx.x & 7, ty = threadIdx.x >> 3;
  const int c = blockIdx.x * DQ_COLS + tx * 8;
  const int t0 = blockIdx.y * DQ_ROWS;
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  if (c < hidden) {
#pragma unroll
    for (int k = 0; k < DQ_ROWS / 32; ++k) {
      const int t = t0 + ty + 32 * k;
      if (t >= T) break;
      const float4 a = *reinterpret_cast<const float4*>(dq + static_cast<int64_t>(t) * hidden + c);
      const float4 b = *reinterpret_cast<const float4*>(dq + static_cast<int64_t>(t) * hidden + c + 4);
      uint4 u;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
      h[0] = __floats2bfloat162_rn(a.x, a.y);
      h[1] = __floats2bfloat162_rn(a.z, a.w);
      h[2] = __floats2bfloat162_rn(b.x, b.y);
      h[3] = __floats2bfloat162_rn(b.z, b.w);
      *reinterpret_cast<uint4*>(dqkv + static_cast<int64_t>(t) * 3 * hidden + c) = u;
      acc[0] += a.x, acc[1] += a.y, acc[2] += a.z, acc[3] += a.w;
      acc[4] += b.x, acc[5] += b.y, acc[6] += b.z, acc[7] += b.w;
    }
  }
  if (!dbias) return;
#pragma unroll
  for (int k = 0; k < 8; ++k) part[ty][tx * 8 + k] = acc[k];
  __syncthreads();
  if (threadIdx.x < DQ_COLS && blockIdx.x * DQ_COLS + threadIdx.x < hidden) {
    float sum = 0.f;
#pragma unroll 8
    for (int y = 0; y < 32; ++y) sum += part[y][threadIdx.x];
    atomicAdd(dbias + blockIdx.x * DQ_COLS + threadIdx.x, sum);
  }
}

CUtensorMap bw_map(const void* base, const AttnShape& s, int64_t ld_elems) {
  CUtensorMap m;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(s.head_dim), static_cast<cuuint64_t>(s.heads),
                        static_cast<cuuint64_t>(s.seq), static_cast<cuuint64_t>(s.mbs)};
  const uint64_t ld = ld_elems * 2;
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
void launch_bwd(const AttnShape& s, const void* qkv, const void* dout, const float* lse2, const float* delta,
                float* dq_acc, void* dqkv, float* dbias, cudaStream_t stream) {
  auto* k = flash_bwd_kernel<D>;
  static uint64_t attr_done = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_done >> (dev & 63) & 1)) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, BwCfg<D>::SMEM);
    attr_done |= 1ull << (dev & 63);
  }
  const auto* base = static_cast<const __nv_bfloat16*>(qkv);
  const int64_t ld = 3LL * s.hidden;
  const CUtensorMap mq = bw_map(base, s, ld), mk = bw_map(base + s.hidden, s, ld),
                    mv = bw_map(base + 2 * s.hidden, s, ld), mdo = bw_map(dout, s, s.hidden);
  BwParams p;
  p.batch = s.mbs;
  p.seq = s.seq;
  p.heads = s.heads;
  p.n_tiles = s.seq / T128;
  p.causal = s.causal;
  p.hidden = s.hidden;
  p.scale = 1.f / sqrtf(static_cast<float>(D));
  p.scale_log2 = 1.4426950408889634f * p.scale;
  p.lse2 = lse2;
  p.delta = delta;
  p.dq_acc = dq_acc;
  p.dqkv = static_cast<__nv_bfloat16*>(dqkv);
  p.dbias = dbias;
  static const int group = [] {
    const char* g = std::getenv("WP_BW_GROUP");  // A/B switch; 0 = one group
    return g ? std::atoi(g) : 32;
  }();
  p.group = group;
  static const int dq_halves = std::getenv("WP_BW_DQ_HALVES") ? std::atoi(std::getenv("WP_BW_DQ_HALVES")) : 0;
  p.dq_halves = dq_halves;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = std::min(p.n_tiles * s.heads * s.mbs, sms);  // persistent: one CTA per SM
  const CUtensorMap mdq = make_slab_map(dq_acc, kF32, s.hidden, int64_t(s.mbs) * s.seq, s.hidden);
  const CUtensorMap mdqkv = make_slab_map(dqkv, kBF16, 3LL * s.hidden, int64_t(s.mbs) * s.seq, 3LL * s.hidden);
  k<<<grid, BW_THREADS, BwCfg<D>::SMEM, stream>>>(mq, mk, mv, mdo, mdq, mdqkv, p);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("flash_attn_bwd: ") + cudaGetErrorString(e));
}

}  // namespace

int flash_attn_bwd(const AttnShape& s, const void* qkv, const void* out, const void* dout, const float* lse2,
                   float* delta, float* dq_acc, void* dqkv, cudaStream_t stream, float* dbias, bool delta_ready) {
  if (s.seq % 128 || (s.head_dim != 64 && s.head_dim != 128)) {
    throw std::runtime_error("flash_attn_bwd: needs seq % 128 == 0 and head_dim in {64, 128}");
  }
  const int T = s.mbs * s.seq;
  const int64_t lanes = static_cast<int64_t>(T) * s.heads * (s.head_dim / 8);
  if (!delta_ready)
    attn_bwd_prep_k<<<static_cast<int>((lanes + 255) / 256), 256, 0, stream>>>(
        static_cast<const __nv_bfloat16*>(dout), static_cast<const __nv_bfloat16*>(out), delta, T, s.heads,
        s.head_dim, s.seq, s.hidden);
  cudaMemsetAsync(dq_acc, 0, sizeof(float) * T * s.hidden, stream);
  if (s.head_dim == 128) launch_bwd<128>(s, qkv, dout, lse2, delta, dq_acc, dqkv, dbias, stream);
  else launch_bwd<64>(s, qkv, dout, lse2, delta, dq_acc, dqkv, dbias, stream);
  const dim3 fin((s.hidden + DQ_COLS - 1) / DQ_COLS, (T + DQ_ROWS - 1) / DQ_ROWS);
  dq_finish_k<<<fin, 256, 0, stream>>>(dq_acc, static_cast<__nv_bfloat16*>(dqkv), dbias, T, s.hidden);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw std::runtime_error(std::string("flash_attn_bwd: ") + cudaGetErrorString(e));
  return delta_ready ? 2 : 3;
}

}  // namespace wpk


#ifdef WP_BW_TRACE
extern "C" int wp_debug_bw_trace(unsigned long long* out, int n) {
  cudaDeviceSynchronize();
  if (n > 512) cudaMemcpyFromSymbol(out + 512, wpk::g_bw_cta, sizeof(unsigned long long) * (n - 512 < 320 ? n - 512 : 320));
  return cudaMemcpyFromSymbol(out, wpk::g_bwt, sizeof(unsigned long long) * (n < 512 ? n : 512)) == cudaSuccess ? 0 : 1;
}
#endif
