// Adam (hgnn.cpp:364-377) shared by the dense, sparse and fused updates.
#pragma once

#include "kernels.cuh"

namespace hetgpu {

// Adam (hgnn.cpp:364-377) in fp32 with the bias corrections folded into two
// per-step scalars computed in f64: w -= a * m / (sqrt(v * b) + eps) with
// a = lr / (1 - beta1^t), b = 1 / (1 - beta2^t)
struct AdamStep {
  float a, b, c1, c2, beta1, beta2, eps;
};
__device__ __forceinline__ AdamStep adam_step_of(const AdamHyper& hp, double t) {
  AdamStep s;
  s.a = static_cast<float>(hp.lr / (1.0 - pow(hp.beta1, t)));
  s.b = static_cast<float>(1.0 / (1.0 - pow(hp.beta2, t)));
  s.beta1 = static_cast<float>(hp.beta1);
  s.beta2 = static_cast<float>(hp.beta2);
  s.c1 = static_cast<float>(1.0 - hp.beta1);
  s.c2 = static_cast<float>(1.0 - hp.beta2);
  s.eps = static_cast<float>(hp.eps);
  return s;
}
__device__ __forceinline__ void adam4(float4& w, float4& m, float4& v, const float4 g, const AdamStep& k,
                                      std::uint32_t* err) {
  float* wp = &w.x;
  float* mp = &m.x;
  float* vp = &v.x;
  const float gv[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float gi = gv[j];
    if (!isfinite(gi)) {
      atomicOr(err, 4u);
      continue;
    }
    const float md = fmaf(k.beta1, mp[j], k.c1 * gi);
    const float vd = fmaf(k.beta2, vp[j], k.c2 * gi * gi);
    mp[j] = md;
    vp[j] = vd;
    wp[j] -= k.a * md / (sqrtf(vd * k.b) + k.eps);
  }
}

// one element (the fused weight-gradient reduction)
__device__ __forceinline__ void adam1(float& w, float& m, float& v, float g, const AdamStep& k, std::uint32_t* err) {
  if (!isfinite(g)) {
    atomicOr(err, 4u);
    return;
  }
  m = fmaf(k.beta1, m, k.c1 * g);
  v = fmaf(k.beta2, v, k.c2 * g * g);
  w -= k.a * m / (sqrtf(v * k.b) + k.eps);
}

}  // namespace hetgpu
