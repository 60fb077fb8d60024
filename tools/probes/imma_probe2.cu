// IMMA.16832 throughput with fresh operands (probe for the assign kernel design; not product code)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(const uint32_t* in, uint32_t* out, int iters) {
  uint32_t w = in[threadIdx.x & 31], b0 = w ^ 0x1234, b1 = w ^ 0x777;
  int c[4][4] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < 4; j++) {
      uint32_t a0, a1, a2, a3;
      if (MODE == 0) { a0 = w; a1 = w * 3; a2 = w * 5; a3 = w * 7; }
      else { uint32_t x = w + i * 4 + j; a0 = x & 0x80808080u; a1 = (x << 1) & 0x80808080u; a2 = (x << 2) & 0x80808080u; a3 = (x << 3) & 0x80808080u; }
      uint32_t bb0 = MODE == 2 ? b0 + i : b0, bb1 = MODE == 2 ? b1 ^ i : b1;
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(bb0), "r"(bb1));
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
  printf("mode %d warps %2d: %.3f ms  %.3f IMMA/clk/SM (at %.2f GHz)\n", MODE, warps, ms, per_sm / (ms * 1e-3 * clk * 1e3), clk / 1e6);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *a, *o; cudaMalloc(&a, 4096); cudaMalloc(&o, 64 << 20); cudaMemset(a, 0x5a, 4096);
  for (int w : {4, 8, 10, 16, 32}) { run<0>(sms, a, o, w); run<1>(sms, a, o, w); run<2>(sms, a, o, w); }
}
