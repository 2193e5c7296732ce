// Device self-test of the tensor-core contractions: random problems of many
// shapes run through the tcgen05 kernels and the SIMT fp32 tile kernels on
// identical device inputs; reports max|diff| / max|ref| per case. Used by the
// GPU tests to pin every tile shape / operand major / chunk count combination.
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "gemm.cuh"

namespace hetgpu {

namespace {

struct Dev {
  std::vector<void*> ptrs;
  template <typename T>
  T* up(const std::vector<T>& h) {
    void* p = nullptr;
    HG_CUDA(cudaMalloc(&p, std::max<std::size_t>(16, h.size() * sizeof(T))));
    if (!h.empty()) HG_CUDA(cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  template <typename T>
  std::vector<T> down(const T* d, std::size_t n) {
    std::vector<T> h(n);
    HG_CUDA(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost));
    return h;
  }
  ~Dev() {
    for (void* p : ptrs) cudaFree(p);
  }
};

double rel(const std::vector<float>& a, const std::vector<float>& b) {
  double m = 0, r = 1e-30;
  for (std::size_t i = 0; i < a.size(); ++i) {
    m = std::max(m, static_cast<double>(std::fabs(a[i] - b[i])));
    r = std::max(r, static_cast<double>(std::fabs(b[i])));
  }
  return m / r;
}

std::vector<float> rnd(std::mt19937& g, std::size_t n, int cols, int ld, float zero_frac = 0.f) {
  std::uniform_real_distribution<float> u(-1.f, 1.f);
  std::vector<float> v(n * ld, 0.f);
  for (std::size_t i = 0; i < n; ++i)
    for (int c = 0; c < cols; ++c) v[i * ld + c] = (zero_frac > 0 && u(g) < 2 * zero_frac - 1) ? 0.f : u(g);
  return v;
}

}  // namespace

// cases: (rows, nrel, din, dout); returns per case {project, dmean, wgrad} errors
std::vector<std::vector<double>> selftest_contractions(const std::vector<std::vector<int>>& cases) {
  std::vector<std::vector<double>> out;
  std::mt19937 gen(12345);
  cudaStream_t st = nullptr;
  for (const auto& cs : cases) {
    const int rows = cs[0], nrel = cs[1], din = cs[2], dout = cs[3];
    const int ldm = round_up4(din), ldo = round_up4(dout);
    Dev d;
    // ---- projection: out = sum_r mean_r . W_r, ReLU
    std::vector<float*> means, ws;
    for (int r = 0; r < nrel; ++r) {
      means.push_back(d.up(rnd(gen, rows, din, ldm)));
      ws.push_back(d.up(rnd(gen, din, dout, ldo)));
    }
    int* nrow = d.up(std::vector<int>{rows});
    std::vector<double> errs;
    {
      std::vector<std::vector<float>> res;
      for (int umma = 0; umma < 2; ++umma) {
        float* o = d.up(std::vector<float>(static_cast<std::size_t>(rows) * ldo, 0.f));
        ProjBatch pb{};
        pb.ng = 1;
        ProjGroup& g = pb.g[0];
        g.nrel = nrel;
        for (int r = 0; r < nrel; ++r) g.r[r] = {means[r], ldm, din, ws[r], ldo};
        g.n_rows = nrow;
        g.rows_cap = rows;
        g.out = o;
        g.ld_out = ldo;
        g.dout = dout;
        g.relu = 1;
        g.out_stride = 1;
        g.out_offset = 0;
        umma ? project_umma(pb, st) : project_tiles(pb, st);
        HG_CUDA(cudaDeviceSynchronize());
        res.push_back(d.down(o, static_cast<std::size_t>(rows) * ldo));
      }
      errs.push_back(rel(res[1], res[0]));
    }
    // ---- mean gradient: dmean = dpre . W^T / deg (dpre arrives ReLU-masked)
    {
      const auto gh = rnd(gen, rows, dout, ldo, 0.3f);
      float* g = d.up(gh);
      float* h = nullptr;
      std::vector<std::uint32_t> ip(rows + 1, 0);
      for (int i = 0; i < rows; ++i) ip[i + 1] = ip[i] + (i % 7);
      std::uint32_t* indptr = d.up(ip);
      std::vector<std::vector<float>> res;
      for (int umma = 0; umma < 2; ++umma) {
        float* o = d.up(std::vector<float>(static_cast<std::size_t>(rows) * ldm, 0.f));
        DMeanBatch db{};
        db.np = 1;
        db.p[0] = {DpreView{g, h, ldo, dout, 1, 0}, ws[0], ldo, din, indptr, nrow, rows, o, ldm};
        umma ? dmean_umma(db, st) : dmean_tiles(db, st);
        HG_CUDA(cudaDeviceSynchronize());
        res.push_back(d.down(o, static_cast<std::size_t>(rows) * ldm));
      }
      errs.push_back(rel(res[1], res[0]));
      // ---- weight gradient: dW = mean^T . dpre (split-K partials + ordered reduce)
      std::vector<std::vector<float>> resw;
      const std::size_t chunks = ceil_div(rows, kWChunkRows);
      for (int umma = 0; umma < 2; ++umma) {
        float* part = d.up(std::vector<float>(chunks * din * dout, 0.f));
        float* dw = d.up(std::vector<float>(static_cast<std::size_t>(din) * ldo, 0.f));
        WGradBatch wb{};
        wb.np = 1;
        wb.p[0] = {means[0], ldm, din, DpreView{g, h, ldo, dout, 1, 0}, nrow, rows, part, dw, ldo};
        umma ? wgrad_umma(wb, st) : wgrad_tiles(wb, st);
        HG_CUDA(cudaDeviceSynchronize());
        resw.push_back(d.down(dw, static_cast<std::size_t>(din) * ldo));
      }
      errs.push_back(rel(resw[1], resw[0]));
    }
    out.push_back(errs);
  }
  return out;
}

}  // namespace hetgpu
