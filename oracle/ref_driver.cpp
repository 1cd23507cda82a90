// TEST INFRASTRUCTURE ONLY. Our driver over the UNMODIFIED reference library (built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It is the reference side of
// the parity contract and the bench's CPU reference arm; the product never links it.
//
//   ref_driver golden <L> <heads> <kv> <dim> <causal> <seed> <out.bin>
//       single-device oracle, loss = sum(out * R) (mirrors report.cpp:61-85) plus the lse of
//       attn_block_forward + finalize_piece (attention.cpp:61-165)
//   ref_driver engine <engine> <sp> <L> <heads> <kv> <dim> <u> <r> <seed> <out.bin>
//       sharded run gathered to global order (mirrors report.cpp:95-133) + per-rank bytes
//   ref_driver bench <engine> <sp> <L> <heads> <kv> <dim> <steps>
//       wall time of fwd+bwd of run_attention_engine, one thread per rank (comm.cpp:197-222)
//   ref_driver batch <len> <sp> <cutoff> <pad_to_cutoff> <seed>
//       pad_batch (partition.cpp:202-215) of a random packed batch, split_position_map of its
//       image map over zigzag(sp), replicate_packing_mask over sp ranks: JSON on stdout
//   ref_driver loss
//       sequence_logprob_per_position, sft_loss_sharded and dpo_loss_sharded / the wrong-order
//       DPO (losses.cpp) on the reference's own test inputs (tests/test_losses.cpp:150-266)
//       over sp in {1, 2, 4}: JSON on stdout
//   ref_driver rope <L> <heads> <dim> <pos_scale> <pos_offset> <seed> <out.bin>
//       rope_apply (tensor.cpp:548-607) of x ~ U(-2,2) at ids i*scale+offset, loss sum(y*R)
//   ref_driver rope_engine <engine> <sp> <L> <heads> <kv> <dim> <u> <r> <pos_scale>
//                          <pos_offset> <seed> <out.bin>
//       as `engine`, with q and k rotated first by rope_apply at the GLOBAL ids of each rank's
//       rows (Model::forward, model.cpp:339-344)
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "seqpar/attention.hpp"
#include "seqpar/comm.hpp"
#include "seqpar/losses.hpp"
#include "seqpar/partition.hpp"
#include "seqpar/report.hpp"
#include "seqpar/tensor.hpp"

using namespace seqpar;

namespace {

struct Data {
  std::vector<double> q, k, v, R;
};

// Same draw order as report.cpp:42-54 (q, k, v, R; uniform(-2, 2)).
Data make_data(uint64_t seed, int64_t L, int heads, int kv, int dim) {
  Rng rng(seed);
  Data d;
  auto fill = [&](std::vector<double>& x, int64_t n) {
    x.resize(static_cast<size_t>(n));
    for (double& e : x) e = rng.uniform_range(-2.0, 2.0);
  };
  fill(d.q, L * heads * dim);
  fill(d.k, L * kv * dim);
  fill(d.v, L * kv * dim);
  fill(d.R, L * heads * dim);
  return d;
}

void put(FILE* f, const std::vector<double>& x) {
  const int64_t n = static_cast<int64_t>(x.size());
  std::fwrite(&n, sizeof(n), 1, f);
  std::fwrite(x.data(), sizeof(double), x.size(), f);
}

ShardLayout layout_for(Engine e, int64_t L, int sp, int u, int r) {
  if (e == Engine::ring) return ShardLayout::make_zigzag(L, sp);
  if (e == Engine::usp) return ShardLayout::make_usp(L, u, r);
  return ShardLayout::make_naive(L, sp);
}

int golden(int argc, char** argv) {
  if (argc != 9) return 2;
  const int64_t L = std::atoll(argv[2]);
  const int heads = std::atoi(argv[3]), kv = std::atoi(argv[4]), dim = std::atoi(argv[5]);
  const bool causal = std::atoi(argv[6]) != 0;
  const uint64_t seed = std::strtoull(argv[7], nullptr, 10);
  Data d = make_data(seed, L, heads, kv, dim);
  Tensor q = Tensor::from({1, L, heads, dim}, d.q, true);
  Tensor k = Tensor::from({1, L, kv, dim}, d.k, true);
  Tensor v = Tensor::from({1, L, kv, dim}, d.v, true);
  Tensor R = Tensor::from({1, L, heads, dim}, d.R);
  std::vector<int64_t> pos(static_cast<size_t>(L));
  std::iota(pos.begin(), pos.end(), int64_t{0});
  std::vector<double> out;
  Tape tape;
  {
    TapeScope sc(&tape);
    const int64_t rep = heads / kv;
    Tensor ke = rep > 1 ? repeat_heads(k, rep) : k;
    Tensor ve = rep > 1 ? repeat_heads(v, rep) : v;
    Tensor o = oracle_attention(q, ke, ve, pos, causal);
    tape.backward(sum_all(mul(o, R)));
    out.assign(o.values().begin(), o.values().end());
  }
  // lse through the block kernel on expanded kv
  const int64_t rep = heads / kv;
  std::vector<double> ke(static_cast<size_t>(L * heads * dim)), ve(ke.size());
  for (int64_t i = 0; i < L; ++i)
    for (int h = 0; h < heads; ++h)
      for (int c = 0; c < dim; ++c) {
        ke[(i * heads + h) * dim + c] = d.k[(i * kv + h / rep) * dim + c];
        ve[(i * heads + h) * dim + c] = d.v[(i * kv + h / rep) * dim + c];
      }
  AttnPiece p = attn_block_forward(1, heads, dim, d.q, pos, ke, ve, pos, causal,
                                   1.0 / std::sqrt(static_cast<double>(dim)));
  std::vector<double> out2, lse;
  finalize_piece(p, out2, lse);
  FILE* f = std::fopen(argv[8], "wb");
  if (!f) return 3;
  put(f, d.q); put(f, d.k); put(f, d.v); put(f, d.R);
  put(f, out); put(f, lse);
  put(f, std::vector<double>(q.grad().begin(), q.grad().end()));
  put(f, std::vector<double>(k.grad().begin(), k.grad().end()));
  put(f, std::vector<double>(v.grad().begin(), v.grad().end()));
  std::fclose(f);
  return 0;
}

int engine(int argc, char** argv, int64_t rope_scale = 0, int64_t rope_offset = 0) {
  if (argc != 12) return 2;
  const Engine e = engine_from_string(argv[2]);
  const int sp = std::atoi(argv[3]);
  const int64_t L = std::atoll(argv[4]);
  const int heads = std::atoi(argv[5]), kv = std::atoi(argv[6]), dim = std::atoi(argv[7]);
  const int u = std::atoi(argv[8]), r = std::atoi(argv[9]);
  const uint64_t seed = std::strtoull(argv[10], nullptr, 10);
  Data d = make_data(seed, L, heads, kv, dim);
  const ShardLayout layout = layout_for(e, L, sp, u, r);
  const int64_t qw = static_cast<int64_t>(heads) * dim, kw = static_cast<int64_t>(kv) * dim;
  AttentionConfig cfg{.heads = heads, .kv_heads = kv, .head_dim = dim, .causal = true,
                      .ulysses_degree = u, .ring_degree = r};
  std::vector<std::vector<double>> outs(sp), dqs(sp), dks(sp), dvs(sp);
  CommFabric fabric(sp, sp, SchedulerKind::threaded);
  fabric.run([&](RankCtx& ctx) {
    const int idx = ctx.sp_group.index_of(ctx.rank);
    const int64_t l = layout.local_len();
    Tensor ql = Tensor::from({1, l, heads, dim}, shard_rows(d.q, qw, layout, idx), true);
    Tensor kl = Tensor::from({1, l, kv, dim}, shard_rows(d.k, kw, layout, idx), true);
    Tensor vl = Tensor::from({1, l, kv, dim}, shard_rows(d.v, kw, layout, idx), true);
    Tensor Rl = Tensor::from({1, l, heads, dim}, shard_rows(d.R, qw, layout, idx));
    Tape tape;
    TapeScope sc(&tape);
    Tensor qa = ql, ka = kl;
    if (rope_scale != 0) {
      std::vector<int64_t> ids;
      for (int64_t p : layout.positions_of(idx)) ids.push_back(p * rope_scale + rope_offset);
      qa = rope_apply(ql, ids);
      ka = rope_apply(kl, ids);
    }
    Tensor out = run_attention_engine(ctx, e, cfg, layout, qa, ka, vl);
    tape.backward(sum_all(mul(out, Rl)));
    outs[idx].assign(out.values().begin(), out.values().end());
    dqs[idx].assign(ql.grad().begin(), ql.grad().end());
    dks[idx].assign(kl.grad().begin(), kl.grad().end());
    dvs[idx].assign(vl.grad().begin(), vl.grad().end());
  });
  FILE* f = std::fopen(argv[11], "wb");
  if (!f) return 3;
  put(f, gather_rows(outs, qw, layout));
  put(f, gather_rows(dqs, qw, layout));
  put(f, gather_rows(dks, kw, layout));
  put(f, gather_rows(dvs, kw, layout));
  std::vector<double> bytes, a2a, ag, p2p;
  for (int rk = 0; rk < sp; ++rk) {
    bytes.push_back(static_cast<double>(fabric.total_bytes(rk)));
    a2a.push_back(static_cast<double>(fabric.stats(rk, Primitive::all_to_all).bytes));
    ag.push_back(static_cast<double>(fabric.stats(rk, Primitive::all_gather).bytes));
    p2p.push_back(static_cast<double>(fabric.stats(rk, Primitive::p2p).bytes));
  }
  put(f, bytes); put(f, a2a); put(f, ag); put(f, p2p);
  std::fclose(f);
  return 0;
}

void put_json(const char* name, const std::vector<int64_t>& v, bool last = false) {
  std::printf("\"%s\": [", name);
  for (size_t i = 0; i < v.size(); ++i) std::printf("%s%lld", i ? ", " : "", static_cast<long long>(v[i]));
  std::printf("]%s", last ? "" : ", ");
}

int batch(int argc, char** argv) {
  if (argc != 7) return 2;
  const int64_t len = std::atoll(argv[2]);
  const int sp = std::atoi(argv[3]);
  const int64_t cutoff = std::atoll(argv[4]);
  const bool to_cutoff = std::atoi(argv[5]) != 0;
  Rng rng(std::strtoull(argv[6], nullptr, 10));
  TrainBatch b;
  int64_t seg = 0, left = 0;
  for (int64_t i = 0; i < len; ++i) {
    if (left == 0) left = rng.uniform_int(1, 9), ++seg;
    --left;
    b.tokens.push_back(rng.uniform_int(0, 1000));
    b.labels.push_back(rng.uniform_int(0, 3) == 0 ? kIgnoreLabel : b.tokens.back());
    b.position_ids.push_back(i);
    b.segment_ids.push_back(seg - 1);
    b.image_map.push_back(rng.uniform_int(0, 2) == 0 ? rng.uniform_int(0, 50) : kNoImage);
  }
  TrainBatch p = pad_batch(b, sp, /*pad_token=*/7, cutoff, to_cutoff);
  std::printf("{");
  put_json("tokens", b.tokens), put_json("labels", b.labels), put_json("segment_ids", b.segment_ids);
  put_json("image_map", b.image_map);
  put_json("p_tokens", p.tokens), put_json("p_labels", p.labels), put_json("p_position_ids", p.position_ids);
  put_json("p_segment_ids", p.segment_ids), put_json("p_image_map", p.image_map);
  const ShardLayout z = ShardLayout::make_zigzag(p.len(), sp);
  std::printf("\"split_image_map\": [");
  for (int i = 0; i < sp; ++i) {
    const auto s = split_position_map(p.image_map, z, i);
    std::printf("%s[", i ? ", " : "");
    for (size_t j = 0; j < s.size(); ++j) std::printf("%s%lld", j ? ", " : "", static_cast<long long>(s[j]));
    std::printf("]");
  }
  std::printf("], ");
  CommFabric fabric(sp, sp, SchedulerKind::threaded);
  std::vector<std::vector<uint8_t>> got(static_cast<size_t>(sp));
  fabric.run([&](RankCtx& ctx) {
    std::vector<uint8_t> mask;
    if (ctx.rank == 0)
      for (int64_t i = 0; i < p.len(); ++i) mask.push_back(static_cast<uint8_t>(p.segment_ids[static_cast<size_t>(i)] & 0xff));
    got[static_cast<size_t>(ctx.rank)] = replicate_packing_mask(ctx, ctx.sp_group, mask);
  });
  std::vector<int64_t> mask0(got[0].begin(), got[0].end()), bc;
  for (int r = 0; r < sp; ++r) bc.push_back(fabric.stats(r, Primitive::broadcast).bytes);
  put_json("mask", mask0), put_json("broadcast_bytes", bc, true);
  std::printf("}\n");
  return 0;
}

std::vector<double> rvals(int64_t n, uint64_t seed, double lo = -2.0, double hi = 2.0) {
  Rng rng(seed);
  std::vector<double> out(static_cast<size_t>(n));
  for (double& v : out) v = rng.uniform_range(lo, hi);
  return out;
}

void put_jd(const char* name, const std::vector<double>& v, bool last = false) {
  std::printf("\"%s\": [", name);
  for (size_t i = 0; i < v.size(); ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
  std::printf("]%s", last ? "" : ", ");
}

int loss(int argc, char**) {
  if (argc != 2) return 2;
  const int64_t T = 32, V = 11;
  const auto logits = rvals(T * V, 29);
  std::vector<int64_t> labels(static_cast<size_t>(T));
  Rng lr(31);
  for (auto& l : labels) l = lr.uniform() < 0.25 ? kIgnoreLabel : lr.uniform_int(0, V - 1);
  // one SFT run: loss and the logits gradient gathered to global order
  auto sft = [&](const ShardLayout& layout, ReduceMode mode, bool per_rank, std::vector<double>* grad) {
    const int sp = layout.sp;
    CommFabric fabric(sp, sp, SchedulerKind::threaded);
    std::vector<double> losses(static_cast<size_t>(sp));
    std::vector<std::vector<double>> grads(static_cast<size_t>(sp));
    fabric.run([&](RankCtx& ctx) {
      const int idx = ctx.sp_group.index_of(ctx.rank);
      Tensor lg = Tensor::from({layout.local_len(), V}, shard_rows(logits, V, layout, idx), true);
      std::vector<int64_t> lab = shard(labels, layout, idx);
      Tape tape;
      TapeScope sc(&tape);
      Tensor l = sft_loss_sharded(ctx, ctx.sp_group, lg, lab, mode, per_rank);
      tape.backward(l);
      losses[static_cast<size_t>(idx)] = l.scalar_value();
      grads[static_cast<size_t>(idx)].assign(lg.grad().begin(), lg.grad().end());
    });
    if (grad) *grad = gather_rows(grads, V, layout);
    return losses[0];
  };
  std::printf("{");
  put_jd("logits", logits);
  put_json("labels", labels);
  {
    Tensor lg = Tensor::from({T, V}, logits, false);
    Tensor pp = sequence_logprob_per_position(lg, labels);
    put_jd("per_pos", std::vector<double>(pp.values().begin(), pp.values().end()));
  }
  std::vector<double> g1, g4a, g4p;
  std::vector<double> sft_losses{sft(ShardLayout::make_naive(T, 1), ReduceMode::grad_aware, false, &g1)};
  for (int sp : {2, 4}) {
    sft_losses.push_back(sft(ShardLayout::make_naive(T, sp), ReduceMode::grad_aware, false, nullptr));
    sft_losses.push_back(sft(ShardLayout::make_zigzag(T, sp), ReduceMode::grad_aware, false, nullptr));
  }
  sft(ShardLayout::make_naive(T, 4), ReduceMode::grad_aware, false, &g4a);
  sft(ShardLayout::make_naive(T, 4), ReduceMode::plain, false, &g4p);
  put_jd("sft_losses", sft_losses);  // sp1, naive2, zigzag2, naive4, zigzag4
  put_jd("sft_per_rank_mean_sp2", {sft(ShardLayout::make_naive(T, 2), ReduceMode::grad_aware, true, nullptr)});
  put_jd("sft_grad_sp1", g1), put_jd("sft_grad_sp4_aware", g4a), put_jd("sft_grad_sp4_plain", g4p);
  // DPO (tests/test_losses.cpp:224-266)
  const int64_t TD = 24;
  const auto pc = rvals(TD, 53, -1.0, 0.0), pr = rvals(TD, 59, -2.0, -0.5), rc = rvals(TD, 61, -1.2, -0.1),
             rr = rvals(TD, 67, -1.8, -0.4);
  auto dpo = [&](const ShardLayout& layout, bool wrong, std::vector<double>* gpc) {
    const int sp = layout.sp;
    CommFabric fabric(sp, sp, SchedulerKind::threaded);
    std::vector<double> losses(static_cast<size_t>(sp));
    std::vector<std::vector<double>> grads(static_cast<size_t>(sp));
    fabric.run([&](RankCtx& ctx) {
      const int idx = ctx.sp_group.index_of(ctx.rank);
      auto t = [&](const std::vector<double>& full, bool rg) {
        return Tensor::from({layout.local_len()}, shard(full, layout, idx), rg);
      };
      Tensor a = t(pc, true), b = t(pr, true), c = t(rc, false), d = t(rr, false);
      Tape tape;
      TapeScope sc(&tape);
      Tensor l = wrong ? wrong_order_dpo_loss(ctx, ctx.sp_group, a, b, c, d, kDpoBetaDefault)
                       : dpo_loss_sharded(ctx, ctx.sp_group, a, b, c, d, kDpoBetaDefault);
      tape.backward(l);
      losses[static_cast<size_t>(idx)] = l.scalar_value();
      grads[static_cast<size_t>(idx)].assign(a.grad().begin(), a.grad().end());
    });
    if (gpc) *gpc = gather_rows(grads, 1, layout);
    return losses[0];
  };
  std::vector<double> gd1, gd2;
  std::vector<double> dl{dpo(ShardLayout::make_naive(TD, 1), false, &gd1), dpo(ShardLayout::make_naive(TD, 2), false, &gd2),
                         dpo(ShardLayout::make_zigzag(TD, 4), false, nullptr)};
  put_jd("pc", pc), put_jd("pr", pr), put_jd("rc", rc), put_jd("rr", rr);
  put_jd("dpo_losses", dl);  // sp1, naive2, zigzag4
  put_jd("dpo_wrong_sp2", {dpo(ShardLayout::make_naive(TD, 2), true, nullptr)});
  put_jd("dpo_grad_pc_sp1", gd1), put_jd("dpo_grad_pc_sp2", gd2, true);
  std::printf("}\n");
  return 0;
}

int rope(int argc, char** argv) {
  if (argc != 9) return 2;
  const int64_t L = std::atoll(argv[2]);
  const int heads = std::atoi(argv[3]), dim = std::atoi(argv[4]);
  const int64_t scale = std::atoll(argv[5]), offset = std::atoll(argv[6]);
  const uint64_t seed = std::strtoull(argv[7], nullptr, 10);
  Data d = make_data(seed, L, heads, heads, dim);
  std::vector<int64_t> ids;
  for (int64_t i = 0; i < L; ++i) ids.push_back(i * scale + offset);
  Tensor x = Tensor::from({1, L, heads, dim}, d.q, true);
  Tensor R = Tensor::from({1, L, heads, dim}, d.R);
  std::vector<double> y;
  Tape tape;
  {
    TapeScope sc(&tape);
    Tensor o = rope_apply(x, ids);
    tape.backward(sum_all(mul(o, R)));
    y.assign(o.values().begin(), o.values().end());
  }
  FILE* f = std::fopen(argv[8], "wb");
  if (!f) return 3;
  put(f, d.q); put(f, d.R); put(f, y);
  put(f, std::vector<double>(x.grad().begin(), x.grad().end()));
  std::fclose(f);
  return 0;
}

int rope_engine(int argc, char** argv) {
  if (argc != 14) return 2;
  // drop the two rope arguments and reuse the engine driver
  std::vector<char*> a(argv, argv + 10);
  a.push_back(argv[12]);
  a.push_back(argv[13]);
  return engine(12, a.data(), std::atoll(argv[10]), std::atoll(argv[11]));
}

int bench(int argc, char** argv) {
  if (argc != 9) return 2;
  const Engine e = engine_from_string(argv[2]);
  const int sp = std::atoi(argv[3]);
  const int64_t L = std::atoll(argv[4]);
  const int heads = std::atoi(argv[5]), kv = std::atoi(argv[6]), dim = std::atoi(argv[7]);
  const int steps = std::atoi(argv[8]);
  Data d = make_data(1, L, heads, kv, dim);
  const ShardLayout layout = layout_for(e, L, sp, 0, 0);
  const int64_t qw = static_cast<int64_t>(heads) * dim, kw = static_cast<int64_t>(kv) * dim;
  AttentionConfig cfg{.heads = heads, .kv_heads = kv, .head_dim = dim, .causal = true};
  CommFabric fabric(sp, sp, SchedulerKind::threaded);
  std::vector<double> secs;
  for (int s = 0; s < steps; ++s) {
    const auto t0 = std::chrono::steady_clock::now();
    fabric.run([&](RankCtx& ctx) {
      const int idx = ctx.sp_group.index_of(ctx.rank);
      const int64_t l = layout.local_len();
      Tensor ql = Tensor::from({1, l, heads, dim}, shard_rows(d.q, qw, layout, idx), true);
      Tensor kl = Tensor::from({1, l, kv, dim}, shard_rows(d.k, kw, layout, idx), true);
      Tensor vl = Tensor::from({1, l, kv, dim}, shard_rows(d.v, kw, layout, idx), true);
      Tensor Rl = Tensor::from({1, l, heads, dim}, shard_rows(d.R, qw, layout, idx));
      Tape tape;
      TapeScope sc(&tape);
      Tensor out = run_attention_engine(ctx, e, cfg, layout, ql, kl, vl);
      tape.backward(sum_all(mul(out, Rl)));
    });
    secs.push_back(std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
  }
  double tot = 0;
  for (double x : secs) tot += x;
  const double per = tot / steps;
  std::printf("{\"engine\": \"%s\", \"sp\": %d, \"L\": %lld, \"heads\": %d, \"kv\": %d, \"dim\": %d, "
              "\"steps\": %d, \"s_per_step\": %.6f, \"tokens_per_s\": %.6f, \"flops_rank0\": %lld}\n",
              argv[2], sp, static_cast<long long>(L), heads, kv, dim, steps, per,
              static_cast<double>(L) / per, static_cast<long long>(fabric.flops(0)));
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_driver golden|engine|bench ...\n");
    return 2;
  }
  try {
    const std::string mode = argv[1];
    int rc = 2;
    if (mode == "golden") rc = golden(argc, argv);
    else if (mode == "engine") rc = engine(argc, argv);
    else if (mode == "bench") rc = bench(argc, argv);
    else if (mode == "rope") rc = rope(argc, argv);
    else if (mode == "batch") rc = batch(argc, argv);
    else if (mode == "loss") rc = loss(argc, argv);
    else if (mode == "rope_engine") rc = rope_engine(argc, argv);
    if (rc == 2) std::fprintf(stderr, "bad arguments for %s\n", mode.c_str());
    return rc;
  } catch (const std::exception& ex) {
    std::fprintf(stderr, "error: %s\n", ex.what());
    return 1;
  }
}
