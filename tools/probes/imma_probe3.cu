// IMMA.16832 u8/s8 pair throughput (probe for the pair-packed assign kernel; not product code)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ void mma_u8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
    : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_s8(int (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
    : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// MODE 0: u8 only, 4 independent chains; 1: u8+s8 pairs into the same acc (2 chains);
// 2: u8+s8 into separate accs (4 chains); 3: mode 1 + unpack (4 LOP3 + 3 IMAD per pair) from fresh words
template <int MODE>
__global__ void k(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t w = in[threadIdx.x & 31], b0 = w ^ 0x1234, b1 = w ^ 0x777;
  uint32_t p4, p16, p64;
  asm volatile("mov.b32 %0, 4;" : "=r"(p4)); asm volatile("mov.b32 %0, 16;" : "=r"(p16)); asm volatile("mov.b32 %0, 64;" : "=r"(p64));
  int c[4][4] = {};
  for (int i = 0; i < iters; i++) {
    uint32_t x = w + i, y = w ^ i;
    if (MODE == 0) {
#pragma unroll
      for (int j = 0; j < 4; j++) mma_u8(c[j], x, y, x + j, y, b0, b1);
    } else if (MODE == 1) {
#pragma unroll
      for (int j = 0; j < 2; j++) { mma_u8(c[j], x, y, x + j, y, b0, b1); mma_s8(c[j], x, y, x + j, y, b1, b0); }
    } else if (MODE == 2) {
#pragma unroll
      for (int j = 0; j < 2; j++) { mma_u8(c[2 * j], x, y, x + j, y, b0, b1); mma_s8(c[2 * j + 1], x, y, x + j, y, b1, b0); }
    } else {
      uint32_t xs1, xs2, xs3, ys1, ys2, ys3;
      asm("mul.lo.u32 %0, %1, %2;" : "=r"(xs1) : "r"(x), "r"(p4)); asm("mul.lo.u32 %0, %1, %2;" : "=r"(xs2) : "r"(x), "r"(p16));
      asm("mul.lo.u32 %0, %1, %2;" : "=r"(xs3) : "r"(x), "r"(p64)); asm("mul.lo.u32 %0, %1, %2;" : "=r"(ys1) : "r"(y), "r"(p4));
      asm("mul.lo.u32 %0, %1, %2;" : "=r"(ys2) : "r"(y), "r"(p16)); asm("mul.lo.u32 %0, %1, %2;" : "=r"(ys3) : "r"(y), "r"(p64));
      const uint32_t M = 0xC0C0C0C0u;
      mma_u8(c[0], x & M, y & M, xs1 & M, ys1 & M, b0, b1); mma_s8(c[0], x & M, y & M, xs1 & M, ys1 & M, b1, b0);
      mma_u8(c[1], xs2 & M, ys2 & M, xs3 & M, ys3 & M, b0, b1); mma_s8(c[1], xs2 & M, ys2 & M, xs3 & M, ys3 & M, b1, b0);
    }
  }
  int s = 0;
  for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int MODE> void run(int sms, uint32_t* a, uint32_t* o, int warps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  k<MODE><<<sms, warps * 32>>>(a, o, iters);
  cudaEventRecord(e0); k<MODE><<<sms, warps * 32>>>(a, o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double per_sm = double(warps) * iters * 4;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("mode %d warps %2d: %.3f ms  %.3f IMMA/clk/SM\n", MODE, warps, ms, per_sm / (ms * 1e-3 * clk * 1e3));
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *a, *o; cudaMalloc(&a, 4096); cudaMalloc(&o, 64 << 20); cudaMemset(a, 0x5a, 4096);
  for (int w : {4, 8, 12, 16}) { run<0>(sms, a, o, w); run<1>(sms, a, o, w); run<2>(sms, a, o, w); run<3>(sms, a, o, w); }
}
