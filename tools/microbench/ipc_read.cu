// Cross-process IPC peer-read microbenchmark: `ipc_read serve <file>` (GPU 1)
// allocates 64 MB, writes its cudaIpcMemHandle to <file> and waits;
// `ipc_read read <file>` (GPU 0) maps it with cudaIpcOpenMemHandle and times
// gathered 256 B row reads and a 4 B id stream, as the replica merge does.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <thread>
#include <chrono>
#include <vector>
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

int main(int argc, char** argv) {
  const int rows = 1 << 18;
  if (argc < 3) return 1;
  if (!strcmp(argv[1], "serve")) {
    CK(cudaSetDevice(1));
    void* p;
    CK(cudaMalloc(&p, size_t(rows) * 256 + (64 << 20)));  // an arena larger than the rows
    CK(cudaMemset(p, 0, size_t(rows) * 256 + (64 << 20)));
    cudaIpcMemHandle_t h;
    CK(cudaIpcGetMemHandle(&h, p));
    FILE* f = fopen(argv[2], "wb");
    fwrite(&h, sizeof(h), 1, f);
    fclose(f);
    std::this_thread::sleep_for(std::chrono::seconds(20));
    return 0;
  }
  for (int t = 0; t < 200; ++t) {
    FILE* f = fopen(argv[2], "rb");
    if (f) { fclose(f); break; }
    std::this_thread::sleep_for(std::chrono::milliseconds(100));
  }
  std::this_thread::sleep_for(std::chrono::milliseconds(300));
  cudaIpcMemHandle_t h;
  FILE* f = fopen(argv[2], "rb");
  if (fread(&h, sizeof(h), 1, f) != 1) return 1;
  fclose(f);
  CK(cudaSetDevice(0));
  void* rp;
  CK(cudaIpcOpenMemHandle(&rp, h, cudaIpcMemLazyEnablePeerAccess));
  const float4* remote = static_cast<const float4*>(rp) + (32 << 20) / 16;  // an offset inside the arena
  float4* out;
  CK(cudaMalloc(&out, 64));
  std::vector<int> idx(rows);
  for (int i = 0; i < rows; ++i) idx[i] = i;
  std::shuffle(idx.begin(), idx.end(), std::mt19937(1));
  int* d_rand;
  CK(cudaMalloc(&d_rand, rows * 4));
  CK(cudaMemcpy(d_rand, idx.data(), rows * 4, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int n : {35000, 100000, rows}) {
    for (int w = 0; w < 3; ++w) k_rows<<<2368, 256>>>(remote, d_rand, n, out);
    CK(cudaEventRecord(a));
    for (int it = 0; it < 10; ++it) k_rows<<<2368, 256>>>(remote, d_rand, n, out);
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("IPC peer rows gathered  n %7d: %8.1f us  %7.1f GB/s\n", n, ms * 100, double(n) * 256 * 10 / (ms * 1e6));
  }
  return 0;
}
