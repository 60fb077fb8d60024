// probe (not product code): tcgen05.mma kind::i8 M128 N8 K32 (A in TMEM) cost when consecutive
// MMAs alternate the instruction descriptor (u8 / s8), with 1 or 2 issuing warps and with
// concurrent tcgen05.st traffic from STW warps.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
#define KS(IA, IB) "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a], b, " IA ", p;\n\tadd.u64 b, b, 16;\n\t" \
                   "@e tcgen05.mma.cta_group::1.kind::i8 [%0], [a], b, " IB ", p;\n\tadd.u64 b, b, 16;\n\tadd.u32 a, a, 8;\n\t"
template <int MODE, int NMW, int STW>
__global__ void k(long long* out, int iters) {
  __shared__ __align__(1024) uint8_t sB[32768];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < int(sizeof(sB)); i += blockDim.x) sB[i] = uint8_t(i * 7);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  if (warp >= 4 && warp < 4 + STW) {
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = tid * 7 + i;
    const uint32_t taddr = tbase + ((32 * (warp & 3)) << 16) + 128 + 16 * ((warp >> 2) % 16);
    for (int i = 0; i < iters / 2; ++i) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
  }
  if (warp < NMW) {
    const uint32_t iu = (2u << 4) | ((8u >> 3) << 17) | ((128u >> 4) << 24);
    const uint32_t is = iu | (1u << 7) | (1u << 10);
    const uint32_t ia = MODE == 0 ? iu : iu, ib = MODE == 0 ? iu : is;
    const uint32_t saddr = smem_u32(sB);
    const uint64_t bdesc = uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (1ull << 46);
    const uint32_t d = tbase + 16 * warp;
    long long t0 = clock64();
    for (int i0 = 0; i0 < iters; i0 += 16 * NMW) {
      if (MODE == 2) {  // 8 u8 k-steps then the same 8 k-steps as s8
        asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
          "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\tmov.b32 a, %1;\n\tmov.b64 b, %2;\n\t"
          KS("%3", "%3") KS("%3", "%3") KS("%3", "%3") KS("%3", "%3")
          "mov.b32 a, %1;\n\t"
          KS("%4", "%4") KS("%4", "%4") KS("%4", "%4") KS("%4", "%4") "}"
          ::"r"(d), "r"(tbase + 256), "l"(bdesc), "r"(iu), "r"(is));
      } else {
        asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
          "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\tmov.b32 a, %1;\n\tmov.b64 b, %2;\n\t"
          KS("%3", "%4") KS("%3", "%4") KS("%3", "%4") KS("%3", "%4") KS("%3", "%4") KS("%3", "%4") KS("%3", "%4") KS("%3", "%4") "}"
          ::"r"(d), "r"(tbase + 256), "l"(bdesc), "r"(ia), "r"(ib));
      }
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar[warp])));
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar[warp])));
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}
template <int MODE, int NMW, int STW> void run() {
  long long* d; cudaMalloc(&d, 8 * 148); long long h = 0;
  const int iters = 8192;
  const int threads = 32 * (4 + STW);
  k<MODE, NMW, STW><<<148, threads>>>(d, iters); cudaDeviceSynchronize();
  k<MODE, NMW, STW><<<148, threads>>>(d, iters); cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("mode=%d (%s) issuing warps=%d st warps=%2d: %.2f cycles per MMA (%s)\n", MODE,
         MODE == 0 ? "all u8" : MODE == 1 ? "u8/s8 alternating" : "u8 block, s8 block", NMW, STW, double(h) / iters, cudaGetErrorString(e));
}
int main() {
  run<0, 1, 0>(); run<1, 1, 0>(); run<2, 1, 0>();
  run<0, 2, 0>(); run<1, 2, 0>(); run<2, 2, 0>();
  run<0, 1, 12>(); run<1, 1, 12>(); run<2, 1, 12>();
  run<1, 2, 12>(); run<2, 2, 12>();
}
