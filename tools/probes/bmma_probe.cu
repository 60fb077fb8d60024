// b1 (AND+POPC) mma.sync throughput vs u8 IMMA (probe for the assign kernel design; not product code)
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
      uint32_t x = w + i * 4 + j;
      uint32_t a0 = x, a1 = x ^ 0x5555, a2 = x + 77, a3 = x * 3;
      if (MODE == 0) {
        asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      } else if (MODE == 1) {
        asm volatile("mma.sync.aligned.m16n8k128.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
          : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3]) : "r"(a0), "r"(a1), "r"(b0));
      } else {
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      }
    }
  }
  int s = 0;
  for (int j = 0; j < 4; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// correctness: one m16n8k256 AND.POPC against a scalar reference
__global__ void check(const uint32_t* A, const uint32_t* B, int* D) {
  int lane = threadIdx.x, g = lane >> 2, q = lane & 3;
  // A row-major 16 x 256 bits = 16 rows x 8 words; fragment: a0 (g, k 32q..), a1 (g+8, ...), a2 (g, 128+32q), a3 (g+8, 128+32q)
  uint32_t a0 = A[g * 8 + q], a1 = A[(g + 8) * 8 + q], a2 = A[g * 8 + 4 + q], a3 = A[(g + 8) * 8 + 4 + q];
  // B col-major 256 x 8: column n = g, b0 (k 32q..), b1 (k 128+32q..)
  uint32_t b0 = B[g * 8 + q], b1 = B[g * 8 + 4 + q];
  int c[4] = {0, 0, 0, 0};
  asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
    : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3]) : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  // D: c0 (g, 2q), c1 (g, 2q+1), c2 (g+8, 2q), c3 (g+8, 2q+1)
  D[g * 8 + 2 * q] = c[0]; D[g * 8 + 2 * q + 1] = c[1]; D[(g + 8) * 8 + 2 * q] = c[2]; D[(g + 8) * 8 + 2 * q + 1] = c[3];
}
template <int MODE> void run(int sms, uint32_t* a, uint32_t* o, int warps) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 4096;
  k<MODE><<<sms, warps * 32>>>(a, o, iters);
  cudaEventRecord(e0); k<MODE><<<sms, warps * 32>>>(a, o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double per_sm = double(warps) * iters * 4;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("mode %d warps %2d: %.3f ms  %.3f MMA/clk/SM (at %.2f GHz)\n", MODE, warps, ms, per_sm / (ms * 1e-3 * clk * 1e3), clk / 1e6);
}
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t *a, *o; cudaMalloc(&a, 4096); cudaMalloc(&o, 64 << 20); cudaMemset(a, 0x5a, 4096);
  for (int w : {4, 8, 16, 32}) { run<0>(sms, a, o, w); run<1>(sms, a, o, w); run<2>(sms, a, o, w); }
  uint32_t hA[128], hB[64]; int hD[128];
  uint64_t s = 88172645463325252ull;
  for (auto& x : hA) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x = uint32_t(s); }
  for (auto& x : hB) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; x = uint32_t(s); }
  uint32_t *dA, *dB; int* dD; cudaMalloc(&dA, 512); cudaMalloc(&dB, 256); cudaMalloc(&dD, 512);
  cudaMemcpy(dA, hA, 512, cudaMemcpyHostToDevice); cudaMemcpy(dB, hB, 256, cudaMemcpyHostToDevice);
  check<<<1, 32>>>(dA, dB, dD); cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 16; m++) for (int n = 0; n < 8; n++) {
    int r = 0; for (int w = 0; w < 8; w++) r += __builtin_popcount(hA[m * 8 + w] & hB[n * 8 + w]);
    if (r != hD[m * 8 + n]) bad++;
  }
  printf("b1 m16n8k256 layout check: %d mismatches of 128\n", bad);
}
