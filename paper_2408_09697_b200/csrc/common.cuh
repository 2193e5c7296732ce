// Shared device-side helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>

namespace hetgpu {

#define HG_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t _e = (call);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(_e) +   \
                               " at " + __FILE__ + ":" + std::to_string(__LINE__));     \
  } while (0)

constexpr int kWarp = 32;
// SM count of the current device (148 on B200), for grid sizing; queried once
// per device (cudaDevAttrMultiProcessorCount), never hard-coded
int num_sms();

// ---- programmatic dependent launch (PDL) --------------------------------------
// The step is a chain of short dependent kernels. Launched through launch_pdl, a
// kernel's CTAs become resident while its predecessor drains (once every
// predecessor CTA has passed pdl_trigger) and park in pdl_wait, which returns
// when the predecessor grid has completed and its writes are visible. Every
// kernel calls pdl_wait before touching anything an earlier kernel produced;
// outside a PDL launch both instructions are no-ops.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_enter() { pdl_wait(); }

template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, std::size_t smem, cudaStream_t st,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  // HG_NO_PDL=1: plain stream order (A/B diagnostics)
  static const bool pdl = std::getenv("HG_NO_PDL") == nullptr;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  HG_CUDA(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

__host__ __device__ inline std::uint64_t ceil_div(std::uint64_t a, std::uint64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int round_up4(int x) { return (x + 3) & ~3; }

// tf32 residual x - trunc_tf32(x): the "lo" operand of the 3xTF32 tensor-core
// products (the tensor core reads the top 19 bits of the raw fp32 as "hi")
__device__ __forceinline__ float tf32_lo(float x) { return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u); }
__device__ __forceinline__ float4 tf32_lo4(float4 v) {
  return make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
}

// ---- exact restatement of the reference's sampler arithmetic ------------------
// splitmix64 finaliser (sampling.cpp:9-15)
__device__ __forceinline__ std::uint64_t dmix_seed(std::uint64_t a, std::uint64_t b) {
  std::uint64_t z = a + 0x9e3779b97f4a7c15ULL * (b + 1);
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// std::mt19937_64 (libstdc++ 13, random.tcc:328-466): n=312, m=156, r=31.
struct Mt64 {
  static constexpr std::uint64_t kMul = 6364136223846793005ULL;
  static constexpr std::uint64_t kUpper = 0xFFFFFFFF80000000ULL;
  static constexpr std::uint64_t kLower = 0x7FFFFFFFULL;
  static constexpr std::uint64_t kA = 0xb5026f5aa96619e9ULL;

  // seeding recurrence x[i] = f*(x[i-1] ^ (x[i-1] >> 62)) + i
  __device__ __forceinline__ static std::uint64_t step(std::uint64_t x, std::uint32_t i) {
    return kMul * (x ^ (x >> 62)) + i;
  }
  __device__ __forceinline__ static std::uint64_t twist(std::uint64_t xk, std::uint64_t xk1,
                                                        std::uint64_t xm) {
    const std::uint64_t y = (xk & kUpper) | (xk1 & kLower);
    return xm ^ (y >> 1) ^ ((y & 1ULL) ? kA : 0ULL);
  }
  __device__ __forceinline__ static std::uint64_t temper(std::uint64_t z) {
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71d67fffeda60000ULL;
    z ^= (z << 37) & 0xfff7eee000000000ULL;
    z ^= (z >> 43);
    return z;
  }
};

// Full-state engine for the (rare) rows that need more than 156 outputs.
struct MtFull {
  std::uint64_t* x;  // 312 words of scratch
  std::uint32_t p;
  __device__ void seed(std::uint64_t s) {
    x[0] = s;
    for (std::uint32_t i = 1; i < 312; ++i) x[i] = Mt64::step(x[i - 1], i);
    p = 312;
  }
  __device__ void regen() {
    for (int k = 0; k < 156; ++k) x[k] = Mt64::twist(x[k], x[k + 1], x[k + 156]);
    for (int k = 156; k < 311; ++k) x[k] = Mt64::twist(x[k], x[k + 1], x[k - 156]);
    x[311] = Mt64::twist(x[311], x[0], x[155]);
    p = 0;
  }
  __device__ std::uint64_t next() {
    if (p >= 312) regen();
    return Mt64::temper(x[p++]);
  }
};

// uniform_int_distribution<uint64_t>(0, range-1) via Lemire's nearly
// divisionless method with 128-bit products (uniform_int_dist.h:255-281), on the
// full-state engine of the rows that need more than 156 outputs (the fast
// sampler path resolves its draws from the first-twist outputs in registers).
__device__ __forceinline__ bool lemire(MtFull& eng, std::uint64_t range, std::uint64_t& out) {
  std::uint64_t x = eng.next();
  std::uint64_t lo = x * range;
  std::uint64_t hi = __umul64hi(x, range);
  if (lo < range) {
    const std::uint64_t thr = (0ULL - range) % range;
    while (lo < thr) {
      x = eng.next();
      lo = x * range;
      hi = __umul64hi(x, range);
    }
  }
  out = hi;
  return true;
}

}  // namespace hetgpu
