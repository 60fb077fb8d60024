// tcgen05.mma kind::i8 with A in TMEM, B in smem (no swizzle, K-major): layout probe (not product code)
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
// KS k-steps of 32 bytes; A: 128 x (32*KS) bytes row-major (global), B: 8 x (32*KS) bytes (global, row n = column n of B)
template <int KS>
__global__ void k(const uint8_t* A, const uint8_t* B, int32_t* D, int bsigned, int lbo, int sbo, int asigned) {
  __shared__ __align__(1024) uint8_t sB[KS * 256];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B into the canonical no-swizzle K-major layout: per k-step 256 B = 2 core matrices (8 rows x 16 B)
  for (int i = tid; i < KS * 256; i += blockDim.x) {
    const int ks = i / 256, r = i % 256, cm = r / 128, rr = (r % 128) / 16, bb = r % 16;
    sB[i] = B[rr * (32 * KS) + ks * 32 + cm * 16 + bb];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tbase = tmem_base;
  // A: warp w (0..3) writes lanes 32w..32w+31; columns 16.. (D at columns 0..7)
  {
    const int row = 32 * warp + lane;
    for (int ks = 0; ks < KS; ++ks) {
      uint32_t r[8];
      for (int c = 0; c < 8; ++c) r[c] = *reinterpret_cast<const uint32_t*>(A + row * (32 * KS) + ks * 32 + 4 * c);
      const uint32_t taddr = tbase + (uint32_t(32 * warp) << 16) + 16 + 8 * ks;
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};"
                   ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // sB written by threads, read by the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (tid == 0) {
    // idesc: c_format S32 (2) at [4,6), a_format [7,10), b_format [10,13), K-major, N>>3 at [17,23), M>>4 at [24,29)
    const uint32_t idesc = (2u << 4) | (uint32_t(asigned) << 7) | (uint32_t(bsigned) << 10) | ((8u >> 3) << 17) |
                           ((128u >> 4) << 24);
    for (int ks = 0; ks < KS; ++ks) {
      const uint32_t saddr = smem_u32(sB + ks * 256);
      const uint64_t desc = uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t((lbo >> 4) & 0x3FFF) << 16) |
                            (uint64_t((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
      const uint32_t a_t = tbase + 16 + 8 * ks;
      const uint32_t accum = ks > 0;
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}"
                   ::"r"(tbase), "r"(a_t), "l"(desc), "r"(idesc), "r"(accum));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  {
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}"
                 ::"r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    uint32_t d[8];
    const uint32_t taddr = tbase + (uint32_t(32 * warp) << 16);
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int c = 0; c < 8; ++c) D[(32 * warp + lane) * 8 + c] = int32_t(d[c]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tbase));
}
int main() {
  constexpr int KS = 3, KB = 32 * KS;
  std::vector<uint8_t> A(128 * KB), B(8 * KB);
  srand(1);
  for (auto& x : A) x = rand() & 0xFF;
  for (auto& x : B) x = rand() & 0xFF;
  uint8_t *dA, *dB;
  int32_t* dD;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dD, 128 * 8 * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  for (int sg = 0; sg < 4; ++sg)
    for (int v = 0; v < 2; ++v) {
      const int asg = sg & 1, bsg = sg >> 1;
      const int lbo = v == 0 ? 128 : 256, sbo = v == 0 ? 256 : 128;
      cudaMemset(dD, 0, 128 * 8 * 4);
      k<KS><<<1, 128>>>(dA, dB, dD, bsg, lbo, sbo, asg);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<int32_t> D(128 * 8);
      cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 8; ++n) {
          int32_t r = 0;
          for (int kk = 0; kk < KB; ++kk) {
            const int a = asg ? int(int8_t(A[m * KB + kk])) : int(A[m * KB + kk]);
            const int b = bsg ? int(int8_t(B[n * KB + kk])) : int(B[n * KB + kk]);
            r += a * b;
          }
          if (r != D[m * 8 + n]) {
            if (bad < 3) printf("  m%d n%d got %d want %d\n", m, n, D[m * 8 + n], r);
            ++bad;
          }
        }
      printf("a_signed %d b_signed %d lbo %d sbo %d: %s, %d mismatches of 1024\n", asg, bsg, lbo, sbo,
             cudaGetErrorString(e), bad);
      if (e != cudaSuccess) return 1;
    }
}
