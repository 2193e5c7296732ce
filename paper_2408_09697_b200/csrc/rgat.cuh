// Relational graph attention (RGAT, BASELINE configs[2] / SURVEY §8 C3) on the RAF
// blocks: the kernels around the tcgen05 projections (rgat_kernels.cu, engine side rgat.cu).
//
// The reference has no attention layer; this is the framework's
// own definition, restated in oracle/rgat.py (parity against that restatement and
// finite differences). Layer l, relation r (src type s -> dst type t), heads H,
// head width F = d_out / H, columns of head h = [h F, (h+1) F):
//   z_j      = h_j . W_r                              (per source row of the block)
//   t_j^h    = a_r^h . z_j^(h)                        (raw score)
//   alpha_e^h = softmax over the edges e of dst i of LeakyReLU_0.2(t_src(e)^h)
//   out_i    = sum_r concat_h sum_e alpha_e^h z_src(e)^(h)   (+ ReLU below the top)
// The blocks carry no destination features (the reference's frontiers do not
// contain their seeds, sampling.cpp:41-103), so the score is source-side only
// ("static" attention, the ranking GAT's own additive score gives); the top layer
// has one head.
#pragma once

#include "gemm.cuh"
#include "kernels.cuh"

namespace hetgpu {

constexpr int kAttMaxHeads = 8;
constexpr int kAttMaxCols = 512;  // row width (ld) the attention kernels hold in registers
constexpr float kAttSlope = 0.2f;

// backward through the CSC view of one hop (entries = packed (block, edge)):
// per source row j and block b of its type,
//   dz_b[j] = sum_e alpha_e^h(c) dout_dst(e)[c] + (sum_e dt_e^h(c)) a_b[c],  tsum_b[j][h] = sum_e dt_e^h
// rows [n_src, round_up(n_src, 32)) of dz are zeroed (the weight gradient's K chunks)
struct AttScatterBlock {
  const std::uint32_t* erow;  // per edge: destination row
  const float* alpha;
  const float* dt;
  const float* dout;
  const float* relu_h;
  int ld_dout;
  const float* a;
  float* dz;
  float* tsum;
  int ld, cols, heads;
  int type;  // index into the hop's CscHop::t
  int row_stride, row_offset;  // destination row -> dout row (replica shards)
};
struct AttScatter {
  AttScatterBlock b[kMaxBlocks];
  int nb;
  const std::uint32_t* offs[kMaxSegs];
  const std::uint32_t* entries[kMaxSegs];
  const int* n_src[kMaxSegs];
  int src_cap[kMaxSegs];
  int nt;
};
void att_scatter(const AttScatter& s, cudaStream_t st);

// ---- aggregate first (every layer). With q_r^h = W_r^(h) a_r^h the score is t = x_j . q^h,
// so per destination row the kernel forms agg^h = sum_e alpha_e^h x_src(e) straight from
// the input rows (the feature / learnable table by global id at layer 1, the previous
// layer's rows by source-frontier row above), and the projection reads
// agg [rows x H din_p] against the block-diagonal W_bd [H din_p x d_out]; backward:
// dagg = dout . W_bd^T, dt per edge, dq^h = sum_e dt_e^h x_src(e) (ordered partials),
// dW = diag blocks of agg^T dout + dq a^T, da = W^T dq.
struct AttLeafJob {
  const std::uint32_t* indptr;
  const std::uint32_t* keys;  // per edge: global source id
  const void* table;
  int ld_t, dtype, din, din_p;  // din_p = round_up4(din): row stride of one head's block
  const int* n_rows;
  int rows_cap;
  const float* q;    // [H x din_p]
  float* te;         // [edges x H] raw scores
  float* lse;        // [rows x H]
  float* alpha;      // [edges x H]
  float* agg;        // [rows x H din_p]; rows [n, next multiple of 32) zeroed
  const float* dagg; // backward: [rows x H din_p]
  float* dt;         // backward: [edges x H]
  float* dq_part;    // backward: [halves x H din_p]
  int heads;
};
struct AttLeafBatch {
  AttLeafJob j[kMaxBlocks];
  int n;
};
void att_leaf_forward(const AttLeafBatch& b, cudaStream_t st);
// fixed grid (att_leaf_halves() half-warps): each half-warp's dq partial is a fixed sum
void att_leaf_grad(const AttLeafBatch& b, cudaStream_t st);
int att_leaf_halves();

// per layer-1 block: q = W^(h) a^(h), W_bd and W_bd^T (prep); dW / da from the
// block-diagonal weight gradient and the reduced dq (finish)
struct AttLeafParam {
  const float* w;  // [din x ld_w]
  float* a;        // [ld_w]
  int din, din_p, dout, ld_w, heads;
  float* q;        // [H x din_p]
  float* wbd;      // [H din_p x ld_w]
  float* wbdt;     // [dout x H din_p]
  const float* dwfull;  // [H din_p x ld_w]
  const float* dq_part; // [halves x H din_p]
  float* dq;            // [att_leaf_dq_rows() x H din_p]: group sums, then dq
  float* dw;       // [din x ld_w]
  float* da;       // [ld_w]
};
struct AttLeafParams {
  AttLeafParam p[kMaxBlocks];
  int n;
};
void att_leaf_prep(const AttLeafParams& p, cudaStream_t st);
void att_leaf_finish(const AttLeafParams& p, cudaStream_t st);
int att_leaf_dq_rows();
// x[i][c] = 0 where h[i][c] <= 0 (rows < n): the ReLU mask of an inner layer's gradient
void relu_mask(float* x, const float* h, int ld, const int* n, int rows_cap, cudaStream_t st);

// W^T of every slot (the source-gradient contraction reads dz . W^T as a projection)
struct TransposeJob {
  const float* w;
  int din, dout, ld_w;
  float* wt;
  int ld_wt;
};
struct TransposeBatch {
  TransposeJob j[kMaxSlots];
  int n;
};
void transpose_slots(const TransposeBatch& b, cudaStream_t st);

}  // namespace hetgpu
