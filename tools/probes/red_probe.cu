// probe (not product code): cost of a burst of same-address reductions at kernel end.
// 148 CTAs x 10016 entries: mode 0 = atomicAdd into one shared row, mode 1 = plain stores into
// a private row per CTA, mode 2 = nothing. Events vs %globaltimer span.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long g_t[148][2];
__global__ void k(unsigned* dst, int mode, long long spin) {
  unsigned long long t0, t1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  long long c0 = clock64();
  while (clock64() - c0 < spin) {}
  const int n = 10016;
  if (mode == 0) for (int i = threadIdx.x; i < n; i += blockDim.x) atomicAdd(dst + i, 1u + (i & 7));
  if (mode == 1) for (int i = threadIdx.x; i < n; i += blockDim.x) dst[size_t(blockIdx.x) * n + i] = 1u + (i & 7);
  __syncthreads();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (threadIdx.x == 0) { g_t[blockIdx.x][0] = t0; g_t[blockIdx.x][1] = t1; }
}
__global__ void stamp(unsigned long long* out) { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); *out = t; }
int main() {
  unsigned* d; cudaMalloc(&d, 148 * 10016 * 4);
  unsigned long long* s; cudaMalloc(&s, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int mode = 0; mode < 3; ++mode)
    for (int th : {128, 512}) {
      k<<<148, th>>>(d, mode, 100000); cudaDeviceSynchronize();
      cudaEventRecord(e0); k<<<148, th>>>(d, mode, 100000); stamp<<<1, 1>>>(s); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      unsigned long long h[148][2], st; cudaMemcpyFromSymbol(h, g_t, sizeof(h)); cudaMemcpy(&st, s, 8, cudaMemcpyDeviceToHost);
      unsigned long long a = ~0ull, b = 0, m = 0; for (int i = 0; i < 148; ++i) { if (h[i][0] < a) a = h[i][0]; if (h[i][1] > b) b = h[i][1]; }
      printf("mode %d threads %3d: events %.1f us, kernel span %.1f us, last CTA end -> next kernel %.1f us\n", mode, th, ms * 1e3, (b - a) / 1e3, (double(st) - double(b)) / 1e3);
      (void)m;
    }
}
