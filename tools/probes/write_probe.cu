// probe (not product code): HBM write bandwidth of the encode's store patterns, 457 MB
// (361920 rows x 316 words). A: warp writes 128-B slices (chunk ch of 16 consecutive rows),
// chunk index fastest in the grid (the k_encode pattern). B: warp writes whole rows contiguously.
// C: plain contiguous memset-like stream. D: pattern A with rows padded to 320 words.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void kA(unsigned* g, unsigned rows, unsigned S32, unsigned rows_per_cta) {
  const unsigned ch = blockIdx.x, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned r0 = blockIdx.y * rows_per_cta;
  for (unsigned r = r0 + warp; r < min(rows, r0 + rows_per_cta); r += blockDim.x / 32)
    if (ch * 32 + lane < S32) g[size_t(r) * S32 + ch * 32 + lane] = r ^ lane;
}
__global__ void kB(unsigned* g, unsigned rows, unsigned S32) {
  const unsigned lane = threadIdx.x & 31;
  for (unsigned r = (blockIdx.x * blockDim.x + threadIdx.x) / 32; r < rows; r += gridDim.x * blockDim.x / 32)
    for (unsigned k = lane; k < S32; k += 32) g[size_t(r) * S32 + k] = r ^ k;
}
__global__ void kC(uint4* g, size_t n) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    g[i] = make_uint4(unsigned(i), 1, 2, 3);
}
int main() {
  const unsigned rows = 361920;
  unsigned* g; cudaMalloc(&g, size_t(rows) * 320 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  for (unsigned S32 : {316u, 320u}) {
    for (unsigned rpc : {64u, 256u, 1024u}) {
      dim3 grid((S32 + 31) / 32, (rows + rpc - 1) / rpc);
      kA<<<grid, 256>>>(g, rows, S32, rpc); cudaDeviceSynchronize();
      cudaEventRecord(e0); for (int i = 0; i < 5; ++i) kA<<<grid, 256>>>(g, rows, S32, rpc); cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
      printf("A slices S32=%u rows/cta=%u: %.1f us, %.2f TB/s\n", S32, rpc, ms * 1e3, rows * S32 * 4.0 / ms / 1e9);
    }
    kB<<<148 * 8, 256>>>(g, rows, S32); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int i = 0; i < 5; ++i) kB<<<148 * 8, 256>>>(g, rows, S32); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("B rows   S32=%u: %.1f us, %.2f TB/s\n", S32, ms * 1e3, rows * S32 * 4.0 / ms / 1e9);
  }
  const size_t n = size_t(rows) * 316 / 4;
  kC<<<148 * 8, 256>>>((uint4*)g, n); cudaDeviceSynchronize();
  cudaEventRecord(e0); for (int i = 0; i < 5; ++i) kC<<<148 * 8, 256>>>((uint4*)g, n); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
  printf("C stream: %.1f us, %.2f TB/s\n", ms * 1e3, n * 16.0 / ms / 1e9);
}
