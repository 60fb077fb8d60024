// probe (not product code): tcgen05.st throughput per SM sub-partition, alone, with ALU work in the
// same warp (the round kernel's unpack: 4 LOP3 + 2 IMAD per stored pair of registers), with ALU
// work in sibling warps of the same sub-partition, and with a concurrent stream of mxf4 MMAs that
// read the stored columns as their A operand.
//   sttm_probe <st warps per SMSP> <alu ops per st register (0 = none)> <mma 0/1> <x: 16|32|64> <sibling ALU warps per SMSP>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
constexpr uint32_t IDESC = (1u << 7) | (1u << 10) | (1u << 23) | ((16u >> 3) << 17) | ((128u >> 4) << 24);

template <int X> __device__ __forceinline__ void st_x(uint32_t taddr, const uint32_t* r);
template <> __device__ __forceinline__ void st_x<16>(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
    ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}
template <> __device__ __forceinline__ void st_x<32>(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"
    ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]),
      "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
}
template <> __device__ __forceinline__ void st_x<64>(uint32_t taddr, const uint32_t* r) {
  st_x<32>(taddr, r);  // (two x32; a true x64 needs 64 asm operands)
  st_x<32>(taddr + 32, r + 32);
}

// warps [0, 4 STW): st warps (SMSP = warp % 4); [4 STW, 4 STW + 4 AW): sibling ALU warps; last warp: MMA
template <int X, int ALU>
__global__ void k(long long* out, int iters, int STW, int AW, int mma, int stbatch, int dcol, int nab, int a0) {
  extern __shared__ __align__(1024) uint8_t sB[];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ volatile int stop;
  const int tid = threadIdx.x, warp = __shfl_sync(0xffffffffu, tid >> 5, 0), nw = blockDim.x >> 5;
  for (int i = tid; i < 32768; i += blockDim.x) sB[i] = uint8_t(i * 7) & 0x77;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) { stop = 0; for (int i = 0; i < 2; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i]))); asm volatile("fence.mbarrier_init.release.cluster;"); }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tmem_base;
  if (warp < 4) {
    const uint32_t s = 0x7F7F7F7Fu;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(tb + ((32 * warp) << 16) + 500), "r"(s), "r"(s), "r"(s), "r"(s));
    asm volatile("tcgen05.wait::st.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  long long t0 = clock64(), t1 = t0;
  if (warp < 4 * STW) {
    uint32_t r[64];
    uint32_t w = tid * 2654435761u;
    for (int i = 0; i < 64; ++i) r[i] = (tid * 7 + i) & 0x66666666;
    const uint32_t taddr = tb + ((32 * (warp & 3)) << 16) + 128 * ((warp >> 2) % 3);
    const int per = 128 / X;  // st instructions per A buffer
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int j = 0; j < per; ++j) {
        if (ALU == 2) {  // one cheap ALU op per stored register (is the store rate data-dependent?)
#pragma unroll
          for (int q = 0; q < X; q += 2) { r[q] += w; r[q + 1] ^= w; }
          w += 0x9E3779B9u;
        } else if (ALU == 3) {  // one FMA-pipe op per stored register
#pragma unroll
          for (int q = 0; q < X; ++q) r[q] = r[q] * 3u + w;
        } else if (ALU) {  // X registers from X / 4 words: 4 LOP3 + 2 IMAD per word
#pragma unroll
          for (int q = 0; q < X / 4; ++q) {
            w = w * 1664525u + 1013904223u;
            r[4 * q + 0] = w & 0x22222222u;
            r[4 * q + 1] = w & 0x44444444u;
            r[4 * q + 2] = (w << 1) & 0x22222222u;
            r[4 * q + 3] = (w >> 1) & 0x44444444u;
          }
        }
        st_x<X>(taddr + j * X, r);
        if (stbatch == 1) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      if (stbatch != 1) asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    t1 = clock64();
    if ((tid & 31) == 0) out[blockIdx.x * 64 + warp] = t1 - t0;
    if (tid == 0) stop = 1;
  } else if (warp < 4 * STW + 4 * AW) {
    uint32_t w = tid * 2654435761u, acc = 0;
    long long n = 0;
    const int fixed = STW == 0 ? iters : (1 << 30);
    for (int i = 0; i < fixed && !stop; ++i) {
#pragma unroll
      for (int q = 0; q < 32; ++q) {
        w = w * 1664525u + 1013904223u;
        acc ^= (w & 0x22222222u) + (w & 0x44444444u);
        acc ^= ((w << 1) & 0x22222222u) ^ ((w >> 1) & 0x44444444u);
      }
      ++n;
    }
    t1 = clock64();
    if ((tid & 31) == 0) { out[blockIdx.x * 64 + warp] = n ? (t1 - t0) / n : 0; if (acc == 0x12345) out[0] = 1; }
  } else if (warp == nw - 1 && mma) {
    const uint32_t saddr = smem_u32(sB);
    const uint64_t bdesc = uint64_t((saddr >> 4) & 0x3FFF) | (uint64_t(128 >> 4) << 16) | (uint64_t(256 >> 4) << 32) | (1ull << 46);
    long long nm = 0;
    const int fixed = STW == 0 ? iters : (1 << 30);
    for (int i = 0; i < fixed && !stop; ++i) {
#ifdef LEAN
      {
        uint32_t el;
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\tselp.u32 %0, 1, 0, e;\n\t}" : "=r"(el));
        if (el) {
          const uint32_t ab = tb + a0 + 128 * (i % nab);
#pragma unroll
          for (int ks = 0; ks < 16; ++ks)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [%1], %2, %3, [%4], [%5], p;\n\t}"
              :: "r"(tb + dcol), "r"(ab + 8 * ks), "l"(bdesc + 32 * ks), "r"(IDESC), "r"(tb + 500), "r"(tb + 502) : "memory");
        }
        __syncwarp();
      }
#else
      asm volatile("{\n\t.reg .pred p, e;\n\t.reg .b32 a;\n\t.reg .b64 b;\n\t"
        "elect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, 1, 0;\n\tmov.b32 a, %1;\n\tmov.b64 b, %2;\n\t"
#define MX "@e tcgen05.mma.cta_group::1.kind::mxf4.block_scale.block32 [%0], [a], b, %3, [%4], [%5], p;\n\tadd.u64 b, b, 32;\n\tadd.u32 a, a, 8;\n\t"
        MX MX MX MX MX MX MX MX MX MX MX MX MX MX MX MX "}"
        ::"r"(tb + dcol), "r"(tb + a0 + 128 * (i % nab)), "l"(bdesc), "r"(IDESC), "r"(tb + 500), "r"(tb + 502));
#endif
      nm += 16;
      if ((i & (mma - 1)) == mma - 1) {  // bound the queue: wait for everything issued so far
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(&bar[0])));
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar[0])), "r"((i / mma) & 1));
      }
    }
    t1 = clock64();
    if ((tid & 31) == 0) out[blockIdx.x * 64 + 63] = nm ? 100 * (t1 - t0) / nm : 0;  // centi-cycles per MMA
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

template <int X, int ALU> void run(int STW, int AW, int mma, int stbatch, int dcol = 400, int nab = 3, int a0 = 0) {
  long long* d; cudaMalloc(&d, 8 * 64 * 148); cudaMemset(d, 0, 8 * 64 * 148);
  long long h[64];
  const int iters = 2048;
  const int threads = 32 * (4 * STW + 4 * AW + 1);
  cudaFuncSetAttribute(k<X, ALU>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  k<X, ALU><<<148, threads, 32768>>>(d, iters, STW, AW, mma, stbatch, dcol, nab, a0); cudaDeviceSynchronize();
  k<X, ALU><<<148, threads, 32768>>>(d, iters, STW, AW, mma, stbatch, dcol, nab, a0); cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(h, d + 64 * 5, sizeof(h), cudaMemcpyDeviceToHost);  // CTA 5
  // per A buffer of 128 columns x 32 lanes (16 KB per warp): cycles
  printf("D@%d A@%d x%d x%-2d alu=%d stw/smsp=%d sibling-alu=%d mma=%d waitEach=%d: ", dcol, a0, nab, X, ALU, STW, AW, mma, stbatch);
  if (STW) printf("%.0f cyc per 16-KB buffer per st warp (=> %.0f B/clk/SM); ", double(h[0]) / iters, 4.0 * STW * 16384.0 * iters / double(h[0]));
  if (AW) printf("sibling ALU block (192 ops): %lld cyc; ", h[4 * STW]);
  if (mma) printf("%.2f cyc per MMA; ", h[63] / 100.0);
  printf("(%s)\n", cudaGetErrorString(e));
  cudaFree(d);
}

int main(int argc, char** argv) {
  if (argc > 1 && argv[1][0] == 'r') {  // store rate with changing data: 0 no ALU, 2 one ALU op, 3 one FMA op per register
    for (int stw = 1; stw <= 4; ++stw) { run<16, 0>(stw, 0, 0, 0); run<16, 2>(stw, 0, 0, 0); run<16, 3>(stw, 0, 0, 0); }
    return 0;
  }
  if (argc > 1) {  // MMA-only placement sweep
    for (int dcol : {0, 16, 384, 400, 448}) for (int nab : {1, 3}) for (int a0 : {0, 128, 256}) {
      if (nab == 3 && a0) continue;
      if (dcol < a0 + 128 * nab && dcol + 16 > a0) continue;
      run<16, 1>(0, 0, 64, 0, dcol, nab, a0);
    }
    run<16, 0>(3, 0, 64, 0, 0, 1, 256);
    run<16, 1>(3, 0, 64, 0, 0, 1, 256);
    run<16, 0>(3, 0, 64, 0, 400, 1, 256);
    run<16, 1>(3, 0, 64, 0, 400, 1, 256);
    return 0;
  }
  for (int mma = 0; mma <= 64; mma = mma ? mma * 8 : 8) {
    for (int stw = 1; stw <= 3; ++stw) {
      run<16, 0>(stw, 0, mma, 0);
      run<16, 1>(stw, 0, mma, 0);
    }
    run<16, 0>(3, 0, mma, 1);
    run<32, 0>(3, 0, mma, 0);
    run<32, 1>(3, 0, mma, 0);
    run<64, 0>(3, 0, mma, 0);
    run<64, 1>(3, 0, mma, 0);
    run<16, 0>(1, 1, mma, 0);
    run<16, 0>(2, 1, mma, 0);
    run<16, 0>(0, 1, mma, 0);
    run<16, 1>(0, 0, mma, 0);
  }
}
