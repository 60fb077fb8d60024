// probe (not product code): tcgen05.mma kind::mxf4 (block32, e2m1 x e2m1 -> f32, ue8m0 scales
// all 1.0) with A in TMEM. Checks the TMEM/smem operand layouts against a CPU product and
// measures cycles per MMA, alone and with 12 warps streaming tcgen05.st.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
#ifndef PN
#define PN 16
#endif
#ifndef BSTEP
#define BSTEP 512
#endif
#ifndef BBYTES
#define BBYTES 32768
#endif
constexpr int N = PN;
// idesc (block-scaled): a/b format E2M1 (1) at bits 7/10, scale format E8M0 (bit 23), N>>3 at 17, M>>4 at 24
constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | (1u << 23) | ((uint32_t(N) >> 3) << 17) | ((128u >> 4) << 24);
__global__ void kcheck(const uint32_t* A, const uint8_t* B, float* D) {
  __shared__ __align__(1024) uint8_t sB[N * 32];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < N * 32; i += blockDim.x) sB[i] = B[i];
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  const uint32_t lane_addr = tb + ((32 * warp) << 16);
  {  // A row m = tid: 8 columns at 256; scales (0x7F) at 384..387
    const uint32_t* a = A + tid * 8;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(lane_addr + 256),
                 "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
    const uint32_t s = 0x7F7F7F7Fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(lane_addr + 384), "r"(s), "r"(s), "r"(s), "r"(s));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp == 0) {
    const uint32_t saddr = smem_u32(sB);
    const uint64_t bdesc = uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (1ull << 46);
    asm volatile("{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                 "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], p;\n\t"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%6];\n\t}"
                 ::"r"(tb), "r"(tb + 256), "l"(bdesc), "r"(IDESC), "r"(tb + 384), "r"(tb + 386), "r"(smem_u32(&bar)));
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)));
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(lane_addr));
  asm volatile("tcgen05.wait::ld.sync.aligned;");
  for (int n = 0; n < N; ++n) D[tid * N + n] = __uint_as_float(r[n]);
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
  (void)lane;
}
template <int NMW, int STW>
__global__ void krate(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t sB[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar[4];
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < BBYTES; i += blockDim.x) {
#ifdef RANDB  // random e2m1 digit codes of both signs, as balanced base-8 centroid digits give
    uint32_t x = uint32_t(i) * 2246822519u; x ^= x >> 13; x *= 3266489917u; x ^= x >> 16;
    sB[i] = uint8_t(x);
#else
    sB[i] = uint8_t(i * 7) & 0x77;
#endif
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
#ifdef RANDA  // the A operand (TMEM columns 256..383): random HV bits as the round kernel's nibbles
  if (warp < 4) {
    for (int c = 0; c < 128; ++c) {
      uint32_t x = (tid * 2654435761u) ^ (c * 40503u) ^ 0x9E3779B9u;
      x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
      const uint32_t v = x & ((c & 1) ? 0x44444444u : 0x22222222u);
      asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(tb + ((32 * warp) << 16) + 256 + c), "r"(v));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
#endif
  if (warp < 4) {
    const uint32_t s = 0x7F7F7F7Fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(tb + ((32 * warp) << 16) + 500), "r"(s), "r"(s), "r"(s), "r"(s));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  if (warp >= 4 && warp < 4 + STW) {
    uint32_t r[16];
    for (int i = 0; i < 16; ++i) r[i] = (tid * 7 + i) & 0x66666666;
    const uint32_t taddr = tb + ((32 * (warp & 3)) << 16) + 128 + 16 * ((warp >> 2) % 16);
    for (int i = 0; i < iters / 2; ++i) {
      asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]));
      asm volatile("tcgen05.wait::st.sync.aligned;");
    }
  }
  if (warp < NMW) {
    const uint32_t saddr = smem_u32(sB);
    const uint64_t bdesc = uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (1ull << 46);
    const uint32_t d = tb + 32 * warp;
    long long t0 = clock64();
#define STR2(x) #x
#define STR(x) STR2(x)
#define MX "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [a], b, %3, [%4], [%5], p;\n\tadd.u64 b, b, " STR(BSTEP / 16) ";\n\tadd.u32 a, a, 8;\n\t"
    for (int i0 = 0; i0 < iters; i0 += 16 * NMW) {
#ifdef FENCE  // as the round kernel: mbarrier wait + fence::after_thread_sync before every 16 MMAs
      asm volatile("{\n\t.reg .pred p;\n\tWF: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 1;\n\t@!p bra WF;\n\t}" ::"r"(smem_u32(&bar[warp])));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#endif
#ifdef COMMIT  // and a commit to an mbarrier after every 16 MMAs (the A buffer release)
      if (i0) asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar[2 + warp])));
#endif
      asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
        "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\tmov.b32 a, %1;\n\tmov.b64 b, %2;\n\t"
        MX MX MX MX MX MX MX MX MX MX MX MX MX MX MX MX "}"
        ::"r"(d), "r"(tb + 256), "l"(bdesc), "r"(IDESC), "r"(tb + 500), "r"(tb + 502));
    }
    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar[warp])));
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar[warp])));
    long long t1 = clock64();
    if (tid == 0) out[blockIdx.x] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}
static float e2m1(unsigned c) {
  static const float v[8] = {0, 0.5f, 1, 1.5f, 2, 3, 4, 6};
  return (c & 8) ? -v[c & 7] : v[c & 7];
}
template <int NMW, int STW> void rate() {
  long long* d; cudaMalloc(&d, 8 * 148); long long h = 0;
  const int iters = getenv("PITERS") ? atoi(getenv("PITERS")) : 8192;
  cudaFuncSetAttribute(krate<NMW, STW>, cudaFuncAttributeMaxDynamicSharedMemorySize, BBYTES);
  krate<NMW, STW><<<148, 32 * (4 + STW), BBYTES>>>(d, iters); cudaDeviceSynchronize();
  krate<NMW, STW><<<148, 32 * (4 + STW), BBYTES>>>(d, iters); cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  printf("mxf4 N=%d issuing warps=%d st warps=%2d: %.2f cycles per MMA (%s)\n", N, NMW, STW, double(h) / iters, cudaGetErrorString(e));
}
int main() {
  uint32_t hA[128 * 8]; uint8_t hB[N * 32]; float hD[128 * N];
  srand(1);
  const unsigned avals[4] = {0, 2, 4, 0};  // the nibbles the round kernel produces: 0, 1.0, 2.0
  for (int i = 0; i < 128 * 8; ++i) { uint32_t w = 0; for (int j = 0; j < 8; ++j) w |= avals[rand() & 3] << (4 * j); hA[i] = w; }
  for (int i = 0; i < N * 32; ++i) hB[i] = uint8_t(rand() & 0xFF);
  uint32_t* dA; uint8_t* dB; float* dD;
  cudaMalloc(&dA, sizeof(hA)); cudaMalloc(&dB, sizeof(hB)); cudaMalloc(&dD, sizeof(hD));
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  kcheck<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
  printf("check kernel: %s\n", cudaGetErrorString(e));
  // CPU: A[m][k] = nibble (k % 8) of word k / 8 (low nibble first); B[n][k]: K-major core matrices of
  // 8 rows x 16 B (32 fp4), LBO 128 (next 32 k), SBO 256 (next 8 rows); low nibble = even k
  for (int order = 0; order < 2; ++order) {
    int bad = 0; double maxd = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double s = 0;
        for (int k = 0; k < 64; ++k) {
          const unsigned an = (hA[m * 8 + k / 8] >> (4 * (order ? 7 - k % 8 : k % 8))) & 15;
          const int cm = k / 32, kb = (k % 32) / 2;
          const uint8_t byte = hB[(n / 8) * 256 + cm * 128 + (n % 8) * 16 + kb];
          const unsigned bn = order ? ((k & 1) ? byte & 15 : byte >> 4) : ((k & 1) ? byte >> 4 : byte & 15);
          s += double(e2m1(an)) * e2m1(bn);
        }
        if (s != hD[m * N + n]) { ++bad; if (std::abs(s - hD[m * N + n]) > maxd) maxd = std::abs(s - hD[m * N + n]); }
      }
    printf("layout order %d: %d / %d mismatches (max |diff| %g); D[0][0..3] = %g %g %g %g\n", order, bad, 128 * N, maxd, hD[0], hD[1], hD[2], hD[3]);
  }
  rate<1, 0>(); rate<2, 0>(); rate<1, 12>(); rate<2, 12>();
}
