// probe (not product code): CUDA-event time vs in-kernel %globaltimer / clock64 for a spin kernel
#include <cstdio>
#include <cuda_runtime.h>
__global__ void spin(long long cycles, unsigned long long* out) {
  unsigned long long g0, g1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  long long c0 = clock64();
  while (clock64() - c0 < cycles) {}
  long long c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[0] = g1 - g0; out[1] = c1 - c0; }
}
int main() {
  unsigned long long* d; cudaMalloc(&d, 16); unsigned long long h[2];
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (long long cyc : {20000LL, 200000LL, 2000000LL}) {
    spin<<<148, 128>>>(cyc, d); cudaDeviceSynchronize();
    cudaEventRecord(e0); spin<<<148, 128>>>(cyc, d); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("cycles %lld: events %.2f us, globaltimer %.2f us, clock64 %llu -> %.0f MHz (by globaltimer), %.0f MHz (by events)\n",
           cyc, ms * 1e3, h[0] / 1e3, h[1], h[1] / (h[0] / 1e3), h[1] / (ms * 1e3));
  }
}
