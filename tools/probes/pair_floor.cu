// probe (not product code): tcgen05.mma.cta_group::2 kind::mxf4 M256 N64 K64 (A in each CTA's TMEM,
// B in shared memory, half of the N columns in each CTA of the pair) issued lean by the leader CTA,
// with LDSW warps per sub-partition streaming LDS.128 in BOTH CTAs. Answers: what does the pair
// cost per MMA, and how much shared-memory bandwidth is left beside it (cta_group::1 at N = 64
// leaves 64 of the 128 B per cycle: mma_floor.cu -DLDSW)?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -DLDSW=2 -o pair_floor pair_floor.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#ifndef LDSW
#define LDSW 0
#endif
#ifndef PN
#define PN 64
#endif
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
// block-scaled kinds: E2M1 A/B (bits 7 / 10), N >> 3 at bit 17, UE8M0 scales (bit 23), M >> 4 at bit 24
constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | (1u << 23) | ((uint32_t(PN) >> 3) << 17) | ((256u >> 4) << 24);

__global__ void __cluster_dims__(2, 1, 1) k(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sB[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  for (int i = tid; i < 65536; i += blockDim.x) sB[i] = uint8_t(i * 7) & 0x77;
  if (tid == 0) {
    stop = 0;
    for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) {  // one warp of each CTA allocates its half of the pair's TMEM
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  if (warp < 4) {  // A columns and the (all 1.0) scale factors of this CTA's 128 lanes
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = ((tid * 7 + i) * 2654435761u) & 0x22222222u;
    for (int c = 0; c < 384; c += 16)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(tb + ((32 * warp) << 16) + c), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
    const uint32_t s = 0x7F7F7F7Fu;
    for (int c = 496; c < 512; c += 4)
      asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(tb + ((32 * warp) << 16) + c), "r"(s), "r"(s), "r"(s), "r"(s));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 1) {
    long long t0 = clock64();
    if (rank == 0) {  // the leader issues for the pair; the commit arrives on both CTAs' barriers
      const uint32_t saddr = smem_u32(sB);
      const uint64_t bdesc = uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (1ull << 46);
      uint32_t el;
      asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(el));
      if (el) {
        for (int i = 0; i < iters; i += 32) {
#pragma unroll
          for (int ks = 0; ks < 32; ++ks)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], p;\n\t}"
              :: "r"(tb + 400), "r"(tb + 8 * ks), "l"(bdesc + (PN) * (ks % 16)), "r"(IDESC), "r"(tb + 496), "r"(tb + 500) : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&bar[0])), "h"(uint16_t(3)) : "memory");
      }
      __syncwarp();
    }
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar[0])));
    long long t1 = clock64();
    if ((tid & 31) == 0) out[blockIdx.x] = t1 - t0;
    if ((tid & 31) == 0) stop = 1;
  } else if (warp >= 4 && warp < 4 + 4 * LDSW) {
    const uint4* p = reinterpret_cast<const uint4*>(sB) + (tid & 31);
    uint32_t acc = 0;
    long long n = 0, t0 = clock64();
    while (!stop) {
#pragma unroll
      for (int i = 0; i < 32; ++i) { const uint4 v = p[32 * ((i * 5 + n) & 127)]; acc ^= v.x ^ v.y ^ v.z ^ v.w; }
      ++n;
    }
    long long t1 = clock64();
    if (warp == 4 && (tid & 31) == 0) out[296 + blockIdx.x] = n ? (t1 - t0) * 100 / (n * 32) : 0;  // centi-cycles per LDS.128
    if (acc == 0x12345) out[0] = 1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
int main() {
  long long* d; cudaMalloc(&d, 8 * 600); cudaMemset(d, 0, 8 * 600);
  const int iters = 32 * 300;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  for (int rep = 0; rep < 2; ++rep) { k<<<148, 128 + 128 * LDSW, 65536>>>(d, iters); cudaError_t e = cudaDeviceSynchronize(); if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; } }
  long long h[4], hs[4];
  cudaMemcpy(h, d + 4, 32, cudaMemcpyDeviceToHost);
  cudaMemcpy(hs, d + 296 + 4, 32, cudaMemcpyDeviceToHost);
  printf("mxf4 cta_group::2 M256 N%d K64 lean issue, LDS warps/SMSP=%d: %.2f cycles per MMA (leader), %.2f (peer wait); "
         "LDS.128: %.1f / %.1f cycles per warp instruction (leader / peer CTA)\n",
         PN, LDSW, double(h[0]) / iters, double(h[1]) / iters, hs[0] / 100.0, hs[1] / 100.0);
}
