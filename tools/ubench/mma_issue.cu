// Microbenchmark: issue rate of tcgen05.mma (cta_group::1, kind::f16) for
// M=128 with N=128 / N=256, issued by one thread; clock64 around the issue
// loop and around completion (commit + mbarrier wait).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "kernels/tc_common.cuh"
using namespace wpk::tc;

template <int N>
__global__ void k_issue(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 96 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(slot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(128 >> 4) << 24);
    const uint64_t ad = make_desc(smem_u32(smem), 16, 1024), bd = make_desc(smem_u32(smem + 32768), 16, 1024);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 8; ++k) tc_mma(tmem, desc_add(ad, (k & 3) * 32), desc_add(bd, (k & 3) * 32), idesc, 1);
    }
    long long t1 = clock64();
    tc_commit(bar);
    mbar_wait(bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  long long h[2];
  const int iters = 256;  // x 8 MMAs
  for (int n : {128, 256}) {
    auto k = n == 128 ? k_issue<128> : k_issue<256>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    for (int rep = 0; rep < 2; ++rep) {
      k<<<1, 128, 100 * 1024>>>(d, iters);
      cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    }
    printf("N=%d: %d MMAs: issue %.1f clk/MMA, complete %.1f clk/MMA (%s)\n", n, iters * 8,
           double(h[0]) / (iters * 8), double(h[1]) / (iters * 8), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
