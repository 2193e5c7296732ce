// Peer-read microbenchmark (diagnostics for the replica merge): a kernel on
// GPU 0 reads rows of a buffer resident on GPU 1 through a peer pointer, with
// the access shapes the merge uses (256 B rows, gathered by an index list, and
// a contiguous 4 B id stream). Prints GB/s per shape.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); exit(1); } } while (0)

__global__ void k_rows(const float4* __restrict__ src, const int* __restrict__ idx, int n_rows, float4* out) {
  const int hl = threadIdx.x & 15;
  const int halves = gridDim.x * (blockDim.x >> 4);
  float4 acc = make_float4(0, 0, 0, 0);
  for (int r = blockIdx.x * (blockDim.x >> 4) + (threadIdx.x >> 4); r < n_rows; r += halves) {
    const float4 v = src[static_cast<size_t>(idx[r]) * 16 + hl];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  if (acc.x == 123.f) out[0] = acc;
}
__global__ void k_ids(const unsigned* __restrict__ src, int n, unsigned* out) {
  unsigned acc = 0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) acc += src[i];
  if (acc == 0xdeadbeef) out[0] = acc;
}

int main() {
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) { printf("needs 2 GPUs\n"); return 0; }
  int can = 0;
  CK(cudaDeviceCanAccessPeer(&can, 0, 1));
  printf("canAccessPeer(0,1) = %d\n", can);
  const int rows = 1 << 18;  // 64 MB of 256 B rows
  float4 *remote, *local, *out;
  unsigned *rids, *uout;
  CK(cudaSetDevice(1));
  CK(cudaMalloc(&remote, size_t(rows) * 256));
  CK(cudaMemset(remote, 0, size_t(rows) * 256));
  CK(cudaMalloc(&rids, size_t(rows) * 4));
  CK(cudaMemset(rids, 0, size_t(rows) * 4));
  CK(cudaSetDevice(0));
  CK(cudaDeviceEnablePeerAccess(1, 0));
  CK(cudaMalloc(&local, size_t(rows) * 256));
  CK(cudaMalloc(&out, 64));
  CK(cudaMalloc(&uout, 64));
  std::vector<int> idx(rows);
  std::mt19937 g(1);
  for (int i = 0; i < rows; ++i) idx[i] = i;
  std::vector<int> shuf = idx;
  std::shuffle(shuf.begin(), shuf.end(), g);
  int *d_seq, *d_rand;
  CK(cudaMalloc(&d_seq, rows * 4));
  CK(cudaMalloc(&d_rand, rows * 4));
  CK(cudaMemcpy(d_seq, idx.data(), rows * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_rand, shuf.data(), rows * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto time_rows = [&](const float4* src, const int* id, int n, const char* what, int grid) {
    for (int w = 0; w < 3; ++w) k_rows<<<grid, 256>>>(src, id, n, out);
    CK(cudaEventRecord(a));
    for (int it = 0; it < 10; ++it) k_rows<<<grid, 256>>>(src, id, n, out);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("%-34s grid %5d rows %7d: %8.1f us  %7.1f GB/s\n", what, grid, n, ms * 100, double(n) * 256 * 10 / (ms * 1e6));
  };
  for (int grid : {148 * 8, 148 * 16}) {
    time_rows(local, d_seq, rows, "local rows, sequential", grid);
    time_rows(local, d_rand, rows, "local rows, gathered", grid);
    time_rows(remote, d_seq, rows, "peer rows, sequential", grid);
    time_rows(remote, d_rand, rows, "peer rows, gathered", grid);
    time_rows(remote, d_rand, 35000, "peer rows, gathered (35k)", grid);
  }
  for (int n : {35000, rows}) {
    for (int w = 0; w < 3; ++w) k_ids<<<296, 256>>>(rids, n, uout);
    CK(cudaEventRecord(a));
    for (int it = 0; it < 10; ++it) k_ids<<<296, 256>>>(rids, n, uout);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("peer id stream (4 B)            n %7d: %8.1f us  %7.1f GB/s\n", n, ms * 100, double(n) * 4 * 10 / (ms * 1e6));
  }
  return 0;
}
