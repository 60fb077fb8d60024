// Throughput probe: legacy IMMA.16832 (u8) and ALU unpack mix on sm_100a.
// Used once to size the assign kernel; not part of the product.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void imma_tput(const uint32_t* a, uint32_t* out, int iters) {
  uint32_t a0 = a[threadIdx.x], a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 ^ 1, b1 = a0 ^ 2;
  int c[CHAINS][4] = {};
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < CHAINS; j++)
      asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+r"(c[j][0]), "+r"(c[j][1]), "+r"(c[j][2]), "+r"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  int s = 0;
#pragma unroll
  for (int j = 0; j < CHAINS; j++) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// unpack mix: per word 7 IMAD-shifts + 8 LOP3 masks, xor-folded
__global__ void unpack_tput(const uint32_t* a, uint32_t* out, int iters) {
  uint32_t w = a[threadIdx.x], acc = 0;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int s = 0; s < 8; s++) acc ^= (w << (7 - s)) & 0x80808080u;  // folded by compiler? keep w changing
    w = w * 0x9E3779B9u + acc;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  printf("device %s sms %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  uint32_t *a, *o; cudaMalloc(&a, 4096); cudaMalloc(&o, 64 << 20); cudaMemset(a, 0x5a, 4096);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int warps : {4, 8, 16, 32}) {
    int iters = 4096;
    imma_tput<4><<<sms, warps * 32>>>(a, o, iters);
    cudaEventRecord(e0);
    imma_tput<4><<<sms, warps * 32>>>(a, o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double mmas = double(sms) * warps * iters * 4;
    printf("IMMA16832 u8: warps/SM %d: %.3f ms, %.1f IMMA/clk/SM-equiv-at-1.9GHz, %.1f TMAC/s\n", warps, ms,
           mmas / sms / (ms * 1e-3 * 1.9e9), mmas * 4096 / (ms * 1e-3) / 1e12);
  }
  for (int warps : {8, 16, 32}) {
    int iters = 4096;
    unpack_tput<<<sms * 2, warps * 32>>>(a, o, iters);
    cudaEventRecord(e0);
    unpack_tput<<<sms * 2, warps * 32>>>(a, o, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double words = double(sms) * 2 * warps * 32 * iters;
    printf("unpack: warps/CTA %d x2: %.3f ms, %.2f G words/s, %.2f words/clk/SM @1.9GHz\n", warps, ms,
           words / (ms * 1e-3) / 1e9, words / sms / (ms * 1e-3 * 1.9e9));
  }
  return 0;
}
