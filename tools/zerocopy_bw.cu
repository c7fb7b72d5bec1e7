// Zero-copy PCIe bandwidth probe (development tool): SM kernels reading mapped pinned host
// memory (H->D), writing it (D->H), and both at once, against the copy engines.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/zc tools/zerocopy_bw.cu && /tmp/zc
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const float4* __restrict__ h, float4* __restrict__ d, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) d[i] = h[i];
}
__global__ void rdwr(const float4* __restrict__ h, float4* __restrict__ d, const float4* __restrict__ d2,
                     float4* __restrict__ h2, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    d[i] = h[i];
    h2[i] = d2[i];
  }
}

int main() {
  for (size_t mb : {1, 4, 16, 256}) {
    const size_t bytes = mb << 20, n = bytes / 16;
    float4 *h, *h2, *d, *d2;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaHostAlloc(&h2, bytes, cudaHostAllocMapped);
    cudaMalloc(&d, bytes);
    cudaMalloc(&d2, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto time = [&](auto fn) {
      for (int i = 0; i < 3; i++) fn();
      cudaEventRecord(a);
      for (int i = 0; i < 20; i++) fn();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      return ms / 20 * 1e3;
    };
    const int grid = 148 * 8;
    float t_rd = time([&] { rd<<<grid, 256>>>(h, d, n); });
    float t_wr = time([&] { rd<<<grid, 256>>>(d2, h2, n); });
    float t_both = time([&] { rdwr<<<grid, 256>>>(h, d, d2, h2, n); });
    float t_ce = time([&] {
      cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice);
      cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost);
    });
    std::printf("%4zu MB: SM read %7.1f us (%5.1f GB/s)  SM write %7.1f us (%5.1f GB/s)  SM both %7.1f us (%5.1f GB/s total)  CE H2D+D2H %7.1f us\n",
                mb, t_rd, bytes / t_rd / 1e3, t_wr, bytes / t_wr / 1e3, t_both, 2 * bytes / t_both / 1e3, t_ce);
    cudaFreeHost(h);
    cudaFreeHost(h2);
    cudaFree(d);
    cudaFree(d2);
  }
  return 0;
}
