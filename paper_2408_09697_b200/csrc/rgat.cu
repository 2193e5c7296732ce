// RGAT layer type of the engine (rgat.cuh defines the layer). Every layer is aggregate
// first (the input rows are the layer-0 tables at layer 1, the previous layer's rows above):
//   forward:  q_r^h = W_r^(h) a_r^h; per destination row and head the online softmax of
//             LeakyReLU(x_j . q^h) over its edges and agg^h = sum_e alpha_e^h x_j, read by
//             global id (tables) or source-frontier row (no projected source rows); then
//             out = sum_r agg_r . W_bd,r (tcgen05 projection, relations along K, ReLU);
//   backward: dagg = dout . W_bd^T (tcgen05), per edge dt and the ordered dq^h partials,
//             dW_bd = agg^T dout (tcgen05 split-K), dW = its diagonal blocks + dq a^T,
//             da = W^T dq; sources with a gradient (inner types, learnable leaves) take the
//             transposed gather over the hop's CSC view (entries = (block, edge)) into dz and
//             dH = dz . W^T (dz carries the score term: sum_h tsum^h q^h = W (tsum a)).
// A replica's top layer trains a strided shard of the batch rows: its projection writes and
// its gradient GEMMs read the logits rows i * shards + shard (strided operands).
// Inner-layer gradients are masked by H > 0 in place before they are read.
#include <cmath>
#include <random>

#include "engine.hpp"
#include "gemm.cuh"
#include "rgat.cuh"

namespace hetgpu {

void Engine::rgat_plan(const Graph& g) {
  (void)g;
  if (o_.heads != 1 && o_.heads != 2 && o_.heads != 4 && o_.heads != 8)
    throw std::invalid_argument("RGAT heads must be 1, 2, 4 or 8");
  if (o_.hidden % o_.heads) throw std::invalid_argument("RGAT heads must divide the hidden width");
  if (replica_group_.size() > 1 && o_.k == 1)
    throw std::invalid_argument("RGAT with replica groups needs at least two layers");
  if (o_.feat_host) throw std::invalid_argument("RGAT reads its layer-0 rows from HBM tables (feat_host = 0)");
  if (round_up4(num_classes_) > kAttMaxCols || round_up4(o_.hidden) > kAttMaxCols)
    throw std::invalid_argument("RGAT layer wider than 512 columns");
  // (transposed views only where the source needs a gradient: the RGCN rule)
  for (auto& b : blocks_)
    if (b.edge_cap >= (1 << 28)) throw std::invalid_argument("RGAT block edge capacity exceeds 2^28");
}

void Engine::rgat_alloc() {
  const int k = o_.k;
  auto round32 = [](int x) { return static_cast<std::size_t>(ceil_div(std::max(1, x), 32) * 32); };
  std::size_t wpart = 0;
  const int halves = att_leaf_halves();
  for (auto& b : blocks_) {
    const int l = k - b.hop + 1;
    const int dout = out_dim(l);
    b.ld_z = round_up4(dout);
    b.heads = heads_of(l);
    b.src_cap = front(b.hop, b.src_t).cap;
    b.alpha = static_cast<float*>(alloc(static_cast<std::size_t>(b.edge_cap) * b.heads * 4));
    b.dt = static_cast<float*>(alloc(static_cast<std::size_t>(b.edge_cap) * b.heads * 4));
    b.lse = static_cast<float*>(alloc(static_cast<std::size_t>(std::max(1, b.rows_cap)) * b.heads * 4));
    if (b.din > 256) throw std::invalid_argument("RGAT input rows wider than 256 columns");
    b.din_p = round_up4(std::max(1, b.din));
    const std::size_t ldg = static_cast<std::size_t>(b.heads) * b.din_p;
    b.agg = static_cast<float*>(alloc(round32(b.rows_cap) * ldg * 4));
    b.dagg = static_cast<float*>(alloc(round32(b.rows_cap) * ldg * 4));
    b.te = static_cast<float*>(alloc(static_cast<std::size_t>(b.edge_cap) * b.heads * 4));
    b.qv = static_cast<float*>(alloc(ldg * 4));
    b.dqv = static_cast<float*>(alloc(static_cast<std::size_t>(att_leaf_dq_rows()) * ldg * 4));
    b.wbd = static_cast<float*>(alloc(ldg * b.ld_z * 4));
    b.wbdt = static_cast<float*>(alloc(static_cast<std::size_t>(dout) * ldg * 4));
    b.dwfull = static_cast<float*>(alloc(ldg * b.ld_z * 4));
    b.dq_part = static_cast<float*>(alloc(static_cast<std::size_t>(halves) * ldg * 4));
    wpart += ceil_div(round32(b.rows_cap), kWChunkRows) * ldg * dout;
    if (b.need_src_grad) {  // sources with a gradient: the transposed gather's dz rows
      const std::size_t zr = round32(b.src_cap);
      b.dz = static_cast<float*>(alloc(zr * b.ld_z * 4));
      b.tsum = static_cast<float*>(alloc(zr * b.heads * 4));
    }
  }
  rgat_wpart_floats_ = std::max<std::size_t>(1, wpart);
  rgat_wpart_ = static_cast<float*>(alloc(rgat_wpart_floats_ * 4));
  // attention vectors: U(-b, b), b = sqrt(6 / (F + 1)) (Glorot for an F x 1 vector), from
  // their own engine per (relation, layer)
  for (auto& s : slots_) {
    s.ld_wt = round_up4(std::max(1, s.din));
    s.wt = static_cast<float*>(alloc(static_cast<std::size_t>(std::max(1, s.dout)) * s.ld_wt * 4));
    s.a = static_cast<float*>(alloc(static_cast<std::size_t>(s.ld) * 4));
    s.am = static_cast<float*>(alloc(static_cast<std::size_t>(s.ld) * 4));
    s.av = static_cast<float*>(alloc(static_cast<std::size_t>(s.ld) * 4));
    s.ag = static_cast<float*>(alloc(static_cast<std::size_t>(s.ld) * 4));
    const int F = s.dout / heads_of(s.layer);
    const double bound = std::sqrt(6.0 / (F + 1.0));
    std::mt19937_64 eng(mix_seed(mix_seed(o_.model_seed, 0xa77e), static_cast<std::uint64_t>(s.rel) * 64 + s.layer));
    std::uniform_real_distribution<double> u(-bound, bound);
    std::vector<float> host(s.ld, 0.f);
    for (int c = 0; c < s.dout; ++c) host[c] = static_cast<float>(u(eng));
    HG_CUDA(cudaMemcpyAsync(s.a, host.data(), host.size() * 4, cudaMemcpyHostToDevice, st_));
    HG_CUDA(cudaStreamSynchronize(st_));
  }
}

const float* Engine::rgat_src(const BlockBuf& b, int& ld) {
  for (const auto& gr : groups_)
    if (gr.depth - 1 == b.hop && gr.type == b.src_t) {
      ld = gr.ld;
      return gr.out;
    }
  throw std::runtime_error("RGAT: no layer input for a block's source type");
}

AttLeafJob Engine::rgat_leaf_job(const BlockBuf& b) {
  // layer 1 reads the layer-0 table by global id; inner layers the previous layer's rows
  // by source-frontier row
  const void* table;
  int ld_t, dtype;
  const std::uint32_t* keys;
  if (b.hop == o_.k) {
    const TypeTable& tb = tables_[b.src_t];
    table = tb.w;
    ld_t = tb.ld;
    dtype = tb.dense ? tb.dtype : static_cast<int>(kF32);
    keys = b.src;
  } else {
    table = rgat_src(b, ld_t);
    dtype = kF32;
    keys = b.col;
  }
  return AttLeafJob{b.indptr, keys, table, ld_t, dtype, b.din, b.din_p, block_rows(b), b.rows_cap, b.qv, b.te,
                    b.lse, b.alpha, b.agg, b.dagg, b.dt, b.dq_part, b.heads};
}

namespace {
template <typename B, typename S>
AttLeafParam leaf_param(const B& b, const S& s) {
  return AttLeafParam{s.w, s.a, b.din, b.din_p, s.dout, s.ld, b.heads, b.qv, b.wbd, b.wbdt, b.dwfull, b.dq_part,
                      b.dqv, s.g, s.ag};
}
}  // namespace

void Engine::run_forward_rgat() {
  const int k = o_.k;
  HG_CUDA(cudaMemsetAsync(logits_, 0, static_cast<std::size_t>(o_.batch_cap + 1) * ldc_ * 4, st_));
  for (int l = 1; l <= k; ++l) {
    const bool top = l == k;
    std::vector<ProjBatch> pbs(1);
    // (1) q and W_bd of every relation of the layer, (2) per-head aggregates of the input rows
    //     (tables at layer 1, the previous layer's rows above)
    AttLeafParams lp{};
    AttLeafBatch lb{};
    for (const auto& gr : groups_) {
      if (gr.layer != l) continue;
      for (std::size_t q = 0; q < gr.blocks.size(); ++q) {
        const BlockBuf& b = blocks_[gr.blocks[q]];
        lp.p[lp.n++] = leaf_param(b, slots_[gr.slots[q]]);
        lb.j[lb.n++] = rgat_leaf_job(b);
      }
    }
    timed("rgat_prep", 0, [&] { att_leaf_prep(lp, st_); });
    timed(top ? "rgat_attend_top" : "rgat_attend", 0, [&] { att_leaf_forward(lb, st_); });
    // (3) out = sum_r agg_r . W_bd,r (+ReLU): the RGCN projection's shape; a replica's top
    //     layer writes its shard rows of the logits
    for (const auto& gr : groups_) {
      if (gr.layer != l) continue;
      if (gr.blocks.empty()) {
        if (!top) zero_rows(gr.out, gr.ld, front(gr.depth - 1, gr.type).count, gr.rows_cap, st_);
        continue;
      }
      const bool shard = top && replica_;
      if (pbs.back().ng == kProjGroups) pbs.emplace_back();
      ProjGroup& pg = pbs.back().g[pbs.back().ng++];
      pg.nrel = static_cast<int>(gr.blocks.size());
      pg.n_rows = shard ? shard_count_dev_ : front(gr.depth - 1, gr.type).count;
      pg.rows_cap = shard ? static_cast<int>(ceil_div(o_.batch_cap, shard_count_)) : gr.rows_cap;
      pg.out = gr.out;
      pg.ld_out = gr.ld;
      pg.dout = gr.dout;
      pg.relu = top ? 0 : 1;
      pg.out_stride = top ? shard_count_ : 1;
      pg.out_offset = top ? shard_index_ : 0;
      for (std::size_t q = 0; q < gr.blocks.size(); ++q) {
        const BlockBuf& b = blocks_[gr.blocks[q]];
        const Slot& s = slots_[gr.slots[q]];
        const int ldg = b.heads * b.din_p;
        pg.r[q] = {b.agg, ldg, ldg, b.wbd, s.ld};
      }
    }
    timed(top ? "rgat_project_top" : "rgat_project", 0, [&] {
      for (auto& pb : pbs) use_umma_ ? project_umma(pb, st_) : project_tiles(pb, st_);
    });
  }
  run_agg_all();
  if (o_.p > 1 && training_ && replica_group_.size() > 1) replica_prepare();
}

void Engine::run_backward_rgat() {
  const int k = o_.k;
  TransposeBatch tb{};
  for (auto& s : slots_) tb.j[tb.n++] = {s.w, s.din, s.dout, s.ld, s.wt, s.ld_wt};
  timed("rgat_transpose", 0, [&] { transpose_slots(tb, st_); });
  auto group_of = [&](int depth_minus_1, int t) -> const Group* {
    for (const auto& gr : groups_)
      if (gr.depth - 1 == depth_minus_1 && gr.type == t) return &gr;
    return nullptr;
  };
  for (int l = k; l >= 1; --l) {
    const int d = k - l + 1;
    const bool top = l == k;
    const CscHop ch = csc_hop(d);
    AttScatter sc{};
    sc.nt = ch.nt;
    for (int t = 0; t < ch.nt; ++t) {
      sc.offs[t] = ch.t[t].offs;
      sc.entries[t] = ch.t[t].entries;
      sc.n_src[t] = ch.t[t].n_src;
      sc.src_cap[t] = ch.t[t].src_cap;
    }
    std::vector<int> scatter_blocks;  // BlockBuf index of every CscEdges entry (csc_hop order)
    for (int bi : hop_blocks_[d]) {
      const BlockBuf& b = blocks_[bi];
      bool typed = false;
      for (const auto& c : cscs_)
        if (c.hop == d && c.src_t == b.src_t) typed = true;
      if (b.need_src_grad && typed) scatter_blocks.push_back(bi);
    }
    if (static_cast<int>(scatter_blocks.size()) != ch.nb) throw std::runtime_error("RGAT: CSC block order mismatch");
    for (int q = 0; q < ch.nb; ++q) {
      const BlockBuf& b = blocks_[scatter_blocks[q]];
      const Group* gr = group_of(d - 1, b.dst_t);
      const Slot& s = slots_[slot_of_.at(SlotId{b.rel, l})];
      if (!gr) throw std::runtime_error("RGAT: block without a destination group");
      sc.b[sc.nb++] = {b.erow, b.alpha, b.dt, gr->dout_buf, top ? nullptr : gr->out, gr->ld, s.a, b.dz, b.tsum,
                       b.ld_z, s.dout, b.heads, ch.b[q].type, top ? shard_count_ : 1, top ? shard_index_ : 0};
    }
    // dout masked in place (inner layers), dagg = dout . W_bd^T, per edge dt + dq partials,
    // dW_bd = agg^T dout, then dW / da; a replica's top layer reads its shard rows of dlogits
    if (!top)
      for (const auto& gr : groups_)
        if (gr.layer == l && !gr.blocks.empty())
          relu_mask(gr.dout_buf, gr.out, gr.ld, front(gr.depth - 1, gr.type).count, gr.rows_cap, st_);
    const int stride = top ? shard_count_ : 1, offset = top ? shard_index_ : 0;
    std::vector<ProjBatch> dbs(1);
    AttLeafBatch lb{};
    AttLeafParams lp{};
    WGradBatch wb{};
    std::size_t off = 0;
    for (const auto& gr : groups_) {
      if (gr.layer != l) continue;
      for (std::size_t q = 0; q < gr.blocks.size(); ++q) {
        const BlockBuf& b = blocks_[gr.blocks[q]];
        const Slot& s = slots_[gr.slots[q]];
        const int ldg = b.heads * b.din_p;
        if (dbs.back().ng == kProjGroups) dbs.emplace_back();
        ProjGroup& pg = dbs.back().g[dbs.back().ng++];
        pg.nrel = 1;
        pg.n_rows = block_rows(b);
        pg.rows_cap = b.rows_cap;
        pg.out = b.dagg;
        pg.ld_out = ldg;
        pg.dout = ldg;
        pg.relu = 0;
        pg.out_stride = 1;
        pg.out_offset = 0;
        pg.r[0] = {gr.dout_buf + static_cast<std::size_t>(offset) * gr.ld, gr.ld, gr.dout, b.wbdt, ldg, stride * gr.ld};
        lb.j[lb.n++] = rgat_leaf_job(b);
        lp.p[lp.n++] = leaf_param(b, s);
        if (wb.np == kMaxProblems) throw std::runtime_error("too many RGAT weight-gradient problems per layer");
        const int rows_cap = std::max(1, b.rows_cap);
        wb.p[wb.np++] = {b.agg, ldg, ldg, DpreView{gr.dout_buf, nullptr, gr.ld, gr.dout, stride, offset}, block_rows(b),
                         rows_cap, rgat_wpart_ + off, b.dwfull, s.ld, nullptr, nullptr, nullptr};
        off += ceil_div(ceil_div(rows_cap, 32) * 32, kWChunkRows) * static_cast<std::size_t>(ldg) * gr.dout;
      }
    }
    if (off > rgat_wpart_floats_) throw std::runtime_error("RGAT weight-gradient scratch too small");
    timed("rgat_dagg", 0, [&] {
      for (auto& pb : dbs) use_umma_ ? project_umma(pb, st_) : project_tiles(pb, st_);
    });
    timed("rgat_edge_grad", 0, [&] { att_leaf_grad(lb, st_); });
    timed("rgat_weight_grad", 0, [&] { use_umma_ ? wgrad_umma(wb, st_) : wgrad_tiles(wb, st_); });
    timed("rgat_att_grad", 0, [&] { att_leaf_finish(lp, st_); });
    if (sc.nb) timed(top ? "rgat_scatter_top" : "rgat_scatter", 0, [&] { att_scatter(sc, st_); });
    // source gradients dH_src = sum_b dz_b . W_r^T (inner types and learnable leaves)
    std::vector<ProjBatch> pbs(1);
    for (const auto& c : cscs_) {
      if (c.hop != d || !c.dh) continue;
      if (pbs.back().ng == kProjGroups) pbs.emplace_back();
      ProjGroup& pg = pbs.back().g[pbs.back().ng++];
      pg.nrel = 0;
      for (int bi : hop_blocks_[d]) {
        const BlockBuf& b = blocks_[bi];
        if (b.src_t != c.src_t || !b.dz) continue;
        const Slot& s = slots_[slot_of_.at(SlotId{b.rel, l})];
        if (pg.nrel == kProjRels) throw std::runtime_error("too many relations out of one source type");
        pg.r[pg.nrel++] = {b.dz, b.ld_z, s.dout, s.wt, s.ld_wt};
      }
      pg.n_rows = front(d, c.src_t).count;
      pg.rows_cap = c.src_cap;
      pg.out = c.dh;
      pg.ld_out = c.ld;
      pg.dout = c.din;
      pg.relu = 0;
      pg.out_stride = 1;
      pg.out_offset = 0;
    }
    timed("rgat_src_grad", 0, [&] {
      for (auto& pb : pbs)
        if (pb.ng) use_umma_ ? project_umma(pb, st_) : project_tiles(pb, st_);
    });
    // learnable layer-0 rows: sparse Adam (step += 1 iff the type has rows)
    if (d == k && apply_adam_) {
      AdamRowsBatch rb{};
      int base4 = 0;
      for (const auto& c : cscs_) {
        if (c.hop != k || !c.dh || !tables_[c.src_t].learnable || xchg_type(c.src_t)) continue;  // replicas: merged
        TypeTable& t = tables_[c.src_t];
        rb.t[rb.n] = {t.w, t.m, t.v, t.ld, front(k, c.src_t).list, c.dh, c.ld, front(k, c.src_t).count, t.step};
        rb.base4[rb.n] = base4;
        base4 += c.src_cap * (t.ld / 4);
        ++rb.n;
      }
      rb.total4 = base4;
      AdamHyper hp;
      timed("rgat_adam_rows", 0, [&] { adam_rows(rb, hp, err_, st_); });
    }
  }
  if (replica_group_.size() > 1) {
    join();  // the union of the replicas' leaf ids (replica_prepare, side stream)
    run_replica_merge();
  }
}

void Engine::run_update_rgat() {
  if (!apply_adam_) return;
  AdamModelBatch mb{};
  int base = 0;
  for (auto& s : slots_) {
    if (mb.n + 2 > kMaxSlots) throw std::runtime_error("too many model slots");
    mb.w[mb.n] = s.w;
    mb.m[mb.n] = s.m;
    mb.v[mb.n] = s.v;
    mb.g[mb.n] = s.g;
    mb.base4[mb.n] = base;
    base += std::max(1, s.din) * s.ld / 4;
    ++mb.n;
    mb.w[mb.n] = s.a;
    mb.m[mb.n] = s.am;
    mb.v[mb.n] = s.av;
    mb.g[mb.n] = s.ag;
    mb.base4[mb.n] = base;
    base += s.ld / 4;
    ++mb.n;
  }
  mb.total4 = base;
  AdamHyper hp;
  timed("adam", 0, [&] { adam_model(mb, &d_tsc_->model_step, hp, err_, st_); });
}

}  // namespace hetgpu
