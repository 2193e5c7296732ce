// RNG-row microbenchmark: 38 CTAs x 256 lanes, one sampled row per lane
// (deg 125, fanout 20), with the sampler's draw code: seeding only, seeding +
// outputs, or the full draw (outputs + Fisher-Yates resolution).
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include "../../paper_2408_09697_b200/csrc/common.cuh"
using namespace hetgpu;

template <int MODE>
__global__ void __launch_bounds__(256) k_rows(std::uint64_t base, std::uint32_t* out) {
  const int lane_row = blockIdx.x * blockDim.x + threadIdx.x;
  const std::uint64_t seed = dmix_seed(base, dmix_seed(2ull << 32, lane_row));
  const std::uint64_t deg = 125;
  const int fanout = 20;
  std::uint64_t xa = seed, xa1 = Mt64::step(seed, 1), xb = xa1;
#pragma unroll 4
  for (std::uint32_t i = 2; i <= 156; ++i) xb = Mt64::step(xb, i);
  if (MODE == 0) { out[lane_row] = static_cast<std::uint32_t>(xb); return; }
  std::uint32_t jr[32];
  bool exact = true;
#pragma unroll
  for (int q = 0; q < 32; ++q) {
    jr[q] = 0xFFFFFFFFu;
    if (q < fanout) {
      const std::uint64_t t = Mt64::temper(Mt64::twist(xa, xa1, xb));
      const std::uint64_t range = deg - q;
      exact &= t * range >= range;
      jr[q] = static_cast<std::uint32_t>(q + __umul64hi(t, range));
      xa = xa1;
      xa1 = Mt64::step(xa1, q + 2u);
      xb = Mt64::step(xb, q + 157u);
    }
  }
  if (MODE == 1) { std::uint32_t s = exact; for (int q = 0; q < 32; ++q) s += jr[q]; out[lane_row] = s; return; }
  std::uint32_t* o = out + static_cast<std::size_t>(lane_row) * fanout;
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if (i < fanout) {
      std::uint32_t p = jr[i];
      int found = -1;
#pragma unroll
      for (int q = 0; q < i; ++q) if (jr[q] == p) found = q;
      while (found >= 0) {
        const int k = found; p = k; found = -1;
#pragma unroll
        for (int q = 0; q < 32; ++q) if (q < k && jr[q] == p) found = q;
      }
      o[i] = p;
    }
  }
}

int main() {
  std::uint32_t* out;
  cudaMalloc(&out, 38 * 256 * 20 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int ctas : {38, 148, 296}) {
    for (int mode = 0; mode < 3; ++mode) {
      auto run = [&] { if (mode == 0) k_rows<0><<<ctas, 256>>>(7, out); else if (mode == 1) k_rows<1><<<ctas, 256>>>(7, out); else k_rows<2><<<ctas, 256>>>(7, out); };
      if (ctas > 38 && mode == 2) continue;
      for (int w = 0; w < 20; ++w) run();
      cudaEventRecord(a);
      for (int it = 0; it < 20; ++it) run();
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("ctas %3d mode %d (%s): %.2f us per launch\n", ctas, mode, mode == 0 ? "seeding" : mode == 1 ? "+outputs" : "+resolve", ms * 1000 / 20);
    }
  }
  return 0;
}
