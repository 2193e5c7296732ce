// Random row-gather bandwidth from a working set far larger than L2 (1.5 GB):
// the practical ceiling for the sampler-driven feature gathers. 16 lanes x
// float4 per 256-byte row (two half-warps per 512-byte row), rows picked
// uniformly at random; reports GB/s of row bytes read.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <random>
#include <vector>

template <int ROWB>
__global__ void k_gather(const float4* __restrict__ tab, const unsigned* __restrict__ idx, int n, float4* out) {
  constexpr int V = ROWB / 16;  // float4 per row
  const int lane = threadIdx.x % V;
  const int groups = gridDim.x * (blockDim.x / V);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = blockIdx.x * (blockDim.x / V) + threadIdx.x / V; r < n; r += groups) {
    const float4 v = tab[static_cast<size_t>(__ldg(idx + r)) * V + lane];
    acc.x += v.x;
  }
  if (acc.x == 1234.5f) out[0] = acc;
}
__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = a[i];
}

int main() {
  const size_t bytes = size_t(1536) << 20;
  float4 *tab, *out, *dst;
  cudaMalloc(&tab, bytes);
  cudaMalloc(&dst, bytes);
  cudaMalloc(&out, 64);
  cudaMemset(tab, 0, bytes);
  const int n = 1 << 22;
  std::vector<unsigned> h(n);
  std::mt19937 g(3);
  unsigned *idx256, *idx512;
  cudaMalloc(&idx256, n * 4);
  cudaMalloc(&idx512, n * 4);
  for (auto& x : h) x = g() % (bytes / 256);
  cudaMemcpy(idx256, h.data(), n * 4, cudaMemcpyHostToDevice);
  for (auto& x : h) x = g() % (bytes / 512);
  cudaMemcpy(idx512, h.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int w = 0; w < 3; ++w) k_copy<<<148 * 8, 256>>>(tab, dst, bytes / 16);
  cudaEventRecord(a);
  for (int it = 0; it < 10; ++it) k_copy<<<148 * 8, 256>>>(tab, dst, bytes / 16);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("copy (read+write)          : %7.1f GB/s\n", 2.0 * bytes * 10 / (ms * 1e6));
  for (int grid : {148 * 8, 148 * 16, 148 * 32}) {
    for (int w = 0; w < 3; ++w) k_gather<256><<<grid, 256>>>(tab, idx256, n, out);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) k_gather<256><<<grid, 256>>>(tab, idx256, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("random 256 B rows (grid %4d): %7.1f GB/s\n", grid, double(n) * 256 * 10 / (ms * 1e6));
    for (int w = 0; w < 3; ++w) k_gather<512><<<grid, 256>>>(tab, idx512, n, out);
    cudaEventRecord(a);
    for (int it = 0; it < 10; ++it) k_gather<512><<<grid, 256>>>(tab, idx512, n, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("random 512 B rows (grid %4d): %7.1f GB/s\n", grid, double(n) * 512 * 10 / (ms * 1e6));
  }
  return 0;
}
