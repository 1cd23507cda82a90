// extern "C" boundary (include/spattn.h) over the seqpar:: C++ engines.
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "seqpar/attention.hpp"
#include "seqpar/losses.hpp"
#include "spattn.h"
#include "spattn_internal.h"

struct spattn_ctx {
  seqpar::RankCtx* rc = nullptr;
  std::unique_ptr<seqpar::RankCtx> owned;
  std::unique_ptr<seqpar::Transport> transport;
  cudaStream_t own_stream = nullptr;
};
struct spattn_fabric {
  std::unique_ptr<seqpar::LoopbackFabric> f;
  std::vector<spattn_ctx> ctxs;
};
struct spattn_saved {
  seqpar::SavedPtr s;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    return SPATTN_OK;
  } catch (const seqpar::ConfigError& e) {
    g_err = e.what();
    return SPATTN_ERR_CONFIG;
  } catch (const seqpar::ShapeError& e) {
    g_err = e.what();
    return SPATTN_ERR_SHAPE;
  } catch (const seqpar::PeerAbort& e) {
    g_err = e.what();
    return SPATTN_ERR_PEER;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SPATTN_ERR_STATE;
  } catch (...) {
    g_err = "unknown error";
    return SPATTN_ERR_STATE;
  }
}

seqpar::ShardLayout make_layout(const spattn_layout* l) {
  if (!l) throw seqpar::ConfigError("layout is null");
  switch (l->mode) {
    case SPATTN_NAIVE: return seqpar::ShardLayout::make_naive(l->global_len, l->sp);
    case SPATTN_ZIGZAG: return seqpar::ShardLayout::make_zigzag(l->global_len, l->sp);
    case SPATTN_ZIGZAG_BLOCKS: return seqpar::ShardLayout::make_zigzag_blocks(l->global_len, l->sp, l->u_degree);
    case SPATTN_SPLIT_USP: {
      auto L = seqpar::ShardLayout::make_usp(l->global_len, l->u_degree, l->r_degree);
      if (L.sp != l->sp) throw seqpar::ConfigError("usp layout: u*r != sp");
      return L;
    }
  }
  throw seqpar::ConfigError("unknown split mode " + std::to_string(l->mode));
}

seqpar::AttentionConfig make_cfg(const spattn_config* c) {
  if (!c) throw seqpar::ConfigError("config is null");
  seqpar::AttentionConfig a;
  a.heads = c->heads;
  a.kv_heads = c->kv_heads;
  a.head_dim = c->head_dim;
  a.causal = c->causal != 0;
  a.ulysses_degree = c->ulysses_degree;
  a.ring_degree = c->ring_degree;
  if (a.heads <= 0 || a.head_dim <= 0 || a.kv_heads < 0) throw seqpar::ConfigError("invalid attention config");
  return a;
}

seqpar::Engine make_engine(int e) {
  if (e < SPATTN_ORACLE || e > SPATTN_USP) throw seqpar::ConfigError("unknown engine " + std::to_string(e));
  return static_cast<seqpar::Engine>(e);
}

struct Views {
  seqpar::DeviceTensor q, k, v, o;
};
Views views(const seqpar::AttentionConfig& c, const seqpar::ShardLayout& L, int64_t bs, const void* q,
            const void* k, const void* v, const void* o) {
  const int64_t n = L.local_len();
  const int64_t kvh = c.kv_heads > 0 ? c.kv_heads : c.heads;
  Views w;
  w.q = {const_cast<void*>(q), bs, n, c.heads, c.head_dim};
  w.k = {const_cast<void*>(k), bs, n, kvh, c.head_dim};
  w.v = {const_cast<void*>(v), bs, n, kvh, c.head_dim};
  w.o = {const_cast<void*>(o), bs, n, c.heads, c.head_dim};
  if (bs <= 0) throw seqpar::ShapeError("batch size must be positive");
  if (!q || !k || !v || !o) throw seqpar::ShapeError("null tensor pointer");
  return w;
}

std::unique_ptr<seqpar::Documents> docs_of(const int64_t* d, int n) {
  if (!d || n <= 0) return nullptr;
  auto D = std::make_unique<seqpar::Documents>();
  D->lengths.assign(d, d + n);
  return D;
}

void row_moves(cudaStream_t s, const spattn_layout* layout, int index, int64_t bs, int64_t row_bytes,
               const void* src, void* dst, bool shard) {
  const auto L = make_layout(layout);
  const auto runs = seqpar::position_runs(L.positions_of(index));
  const int64_t lloc = L.local_len(), len = L.global_len;
  std::vector<spattn::CopyTask> t;
  for (int64_t b = 0; b < bs; ++b)
    for (const auto& r : runs) {
      if (shard)
        t.push_back({src, dst, row_bytes, row_bytes, b * len + r.pos0, b * lloc + r.row0, 0, 0, r.n, row_bytes, 0});
      else
        t.push_back({src, dst, row_bytes, row_bytes, b * lloc + r.row0, b * len + r.pos0, 0, 0, r.n, row_bytes, 0});
    }
  for (size_t i = 0; i < t.size(); i += spattn::kMaxCopyTasks) {
    spattn::CopyTaskSet ts{};
    ts.n = static_cast<int>(std::min<size_t>(spattn::kMaxCopyTasks, t.size() - i));
    for (int j = 0; j < ts.n; ++j) ts.t[j] = t[i + static_cast<size_t>(j)];
    spattn::launch_copy_tasks(ts, 1, s);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) throw seqpar::StateError(std::string("CUDA: ") + cudaGetErrorString(e));
}

}  // namespace

extern "C" {

const char* spattn_last_error(void) { return g_err.c_str(); }
int spattn_abi_version(void) { return 1; }

int spattn_layout_positions(const spattn_layout* layout, int index, int64_t* out) {
  return guard([&] {
    const auto L = make_layout(layout);
    const auto& p = L.positions_of(index);
    std::memcpy(out, p.data(), p.size() * sizeof(int64_t));
  });
}
int spattn_causal_pairs(const spattn_layout* layout, int index, int64_t* out) {
  return guard([&] { *out = seqpar::causal_pair_count(make_layout(layout), index); });
}
int spattn_pad_length(int64_t len, int sp, int64_t cutoff, int pad_to_cutoff, int64_t* out) {
  return guard([&] { *out = seqpar::pad_length(len, sp, cutoff, pad_to_cutoff != 0); });
}
int spattn_pick_xtuner_insp(int heads, int sp, int head_dim, int* out) {
  return guard([&] { *out = seqpar::pick_xtuner_insp(heads, sp, head_dim); });
}
int spattn_reference_bytes(int engine, int64_t bs, int64_t len, int64_t heads, int64_t d, int sp,
                           int u, int r, int64_t* out) {
  return guard([&] {
    switch (make_engine(engine)) {
      case seqpar::Engine::oracle: *out = 0; break;
      case seqpar::Engine::ulysses: *out = seqpar::ulysses_bytes(bs, len, heads, d, sp); break;
      case seqpar::Engine::dummy_head: *out = seqpar::dummy_head_bytes(bs, len, heads, d, sp); break;
      case seqpar::Engine::xtuner: *out = seqpar::xtuner_bytes(bs, len, heads, d, sp); break;
      case seqpar::Engine::ring: *out = seqpar::ring_bytes(bs, len, heads, d, sp); break;
      case seqpar::Engine::usp: *out = seqpar::usp_bytes(bs, len, heads, d, u, r); break;
    }
  });
}

int spattn_plan_heads(int heads, int kv_heads, int group, int32_t* q_lo, int32_t* q_n,
                      int32_t* kv_lo, int32_t* kv_n) {
  return guard([&] {
    std::vector<int> a, b, c, d;
    seqpar::plan_head_windows(heads, kv_heads, group, a, b, c, d);
    for (int i = 0; i < group; ++i) q_lo[i] = a[i], q_n[i] = b[i], kv_lo[i] = c[i], kv_n[i] = d[i];
  });
}

int spattn_plan_problems(const int64_t* qpos, int64_t lq, const int64_t* kpos, int64_t lk,
                         int causal, const int64_t* doc_lens, int n_docs, int32_t* out,
                         int max_problems, int* n_problems, int64_t* pairs) {
  return guard([&] {
    const auto D = docs_of(doc_lens, n_docs);
    const auto v = seqpar::plan_problems(std::vector<int64_t>(qpos, qpos + lq),
                                         std::vector<int64_t>(kpos, kpos + lk), causal != 0,
                                         D.get(), pairs);
    if (static_cast<int>(v.size()) > max_problems) throw seqpar::ConfigError("too many problems");
    for (size_t i = 0; i < v.size(); ++i)
      for (int j = 0; j < 6; ++j) out[6 * i + j] = v[i][static_cast<size_t>(j)];
    *n_problems = static_cast<int>(v.size());
  });
}

int spattn_debug_transport_selftest(spattn_ctx* ctx, int64_t bytes) {
  return guard([&] {
    if (!ctx || !ctx->rc || bytes <= 0) throw seqpar::ConfigError("transport self-test: bad arguments");
    ctx->rc->transport->self_test(ctx->rc->rank, static_cast<size_t>(bytes), ctx->rc->stream);
  });
}

int spattn_nccl_unique_id(uint8_t out[128]) {
  return guard([&] { seqpar::nccl_unique_id(out); });
}

int spattn_ctx_create_nccl(int device, int rank, int world, int sp, const uint8_t uid[128],
                           spattn_ctx** out) {
  return guard([&] {
    if (sp <= 0 || world % sp) throw seqpar::ConfigError("world must be a multiple of sp");
    auto c = std::make_unique<spattn_ctx>();
    c->transport = seqpar::make_nccl_transport(rank, world, uid, device);
    c->owned = std::make_unique<seqpar::RankCtx>();
    auto& rc = *c->owned;
    rc.transport = c->transport.get();
    rc.rank = rank;
    rc.device = device;
    for (int i = 0; i < sp; ++i) rc.sp_group.ranks.push_back(rank / sp * sp + i);
    if (cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&rc.comm_stream, cudaStreamNonBlocking) != cudaSuccess)
      throw seqpar::StateError("cannot create streams");
    rc.stream = c->own_stream;
    c->rc = &rc;
    *out = c.release();
  });
}

int spattn_ctx_destroy(spattn_ctx* c) {
  return guard([&] {
    if (!c) return;
    if (c->owned) {
      cudaStreamSynchronize(c->owned->stream);
      if (c->own_stream) cudaStreamDestroy(c->own_stream);
      if (c->owned->comm_stream) cudaStreamDestroy(c->owned->comm_stream);
    }
    delete c;
  });
}

int spattn_fabric_create(int device, int world, int sp, int force_messages, spattn_fabric** out) {
  return guard([&] {
    auto f = std::make_unique<spattn_fabric>();
    f->f = std::make_unique<seqpar::LoopbackFabric>(world, sp, device, force_messages != 0);
    f->ctxs.resize(static_cast<size_t>(world));
    for (int r = 0; r < world; ++r) {
      f->ctxs[static_cast<size_t>(r)].rc = &f->f->ctx(r);
      f->ctxs[static_cast<size_t>(r)].own_stream = f->f->ctx(r).stream;
    }
    *out = f.release();
  });
}
int spattn_fabric_destroy(spattn_fabric* f) {
  return guard([&] { delete f; });
}
int spattn_fabric_ctx(spattn_fabric* f, int rank, spattn_ctx** out) {
  return guard([&] {
    if (rank < 0 || rank >= static_cast<int>(f->ctxs.size())) throw seqpar::ConfigError("rank out of range");
    *out = &f->ctxs[static_cast<size_t>(rank)];
  });
}

int spattn_ctx_set_stream(spattn_ctx* c, void* stream) {
  return guard([&] { c->rc->stream = static_cast<cudaStream_t>(stream); });
}
int spattn_ctx_stream(spattn_ctx* c, void** stream) {
  return guard([&] { *stream = c->rc->stream; });
}
int spattn_ctx_stats(spattn_ctx* c, int primitive, int64_t* calls, int64_t* bytes) {
  return guard([&] {
    if (primitive < 0 || primitive >= seqpar::kPrimitiveCount) throw seqpar::ConfigError("bad primitive");
    *calls = c->rc->stats[static_cast<size_t>(primitive)].calls;
    *bytes = c->rc->stats[static_cast<size_t>(primitive)].bytes;
  });
}
int spattn_ctx_flops(spattn_ctx* c, int64_t* flops) {
  return guard([&] { *flops = c->rc->flops; });
}
int spattn_ctx_reset_stats(spattn_ctx* c) {
  return guard([&] { c->rc->reset_stats(); });
}
int spattn_set_kernel_family(int family) {
  return guard([&] {
    if (family < 0 || family > 4) throw seqpar::ConfigError("kernel family must be 0 .. 4");
    seqpar::set_kernel_family(static_cast<seqpar::KernelFamily>(family));
  });
}
int spattn_get_kernel_family(void) { return static_cast<int>(seqpar::kernel_family()); }

}  // extern "C"
namespace spattn {
int umma_selftest(cudaStream_t s, const void* A, const void* B, const void* Bmn, float* D1, float* D2, float* D3);
}
extern "C" {
int spattn_selftest_umma(void* stream, const void* a, const void* b, const void* b_mn, float* d1,
                         float* d2, float* d3) {
  return guard([&] {
    if (spattn::umma_selftest(static_cast<cudaStream_t>(stream), a, b, b_mn, d1, d2, d3) != 0)
      throw seqpar::StateError("umma self-test launch failed");
  });
}

}  // extern "C"
namespace spattn {
void set_bwd_trace(void* p);
void set_fwd_trace(void* p);
void set_fwd_cta_trace(void* p);
void set_pp_trace(void* p);
void set_pp_cta_trace(void* p);
}
extern "C" {
int spattn_debug_bwd_trace(void* device_buffer) {
  return guard([&] {
    spattn::set_bwd_trace(device_buffer);
    spattn::set_fwd_trace(device_buffer);
    spattn::set_pp_trace(device_buffer);
  });
}
int spattn_debug_fwd_cta_trace(void* device_buffer) {
  return guard([&] {
    spattn::set_fwd_cta_trace(device_buffer);
    spattn::set_pp_cta_trace(device_buffer);
  });
}

int64_t spattn_launch_count(void) { return spattn::launch_count(); }
int spattn_profile_enable(int on) {
  return guard([&] { seqpar::profile_enable(on != 0); });
}
int spattn_profile_read(double ms[2], int64_t n[2]) {
  return guard([&] { seqpar::profile_read(ms, n); });
}
int spattn_debug_timeline(int on) {
  return guard([&] { seqpar::timeline_enable(on != 0); });
}
int spattn_debug_timeline_read(double* start_ms, double* end_ms, int* kind, int* rank, int max, int64_t* n) {
  return guard([&] { *n = seqpar::timeline_read(start_ms, end_ms, kind, rank, max); });
}

namespace {
std::unique_ptr<seqpar::Rope> rope_of(const int64_t* position_ids, int64_t n, double base) {
  if (!position_ids) return nullptr;
  auto r = std::make_unique<seqpar::Rope>();
  r->position_ids.assign(position_ids, position_ids + n);
  r->base = base;
  return r;
}
}  // namespace

int spattn_fwd(spattn_ctx* ctx, int engine, const spattn_config* cfg, const spattn_layout* layout,
               int64_t bs, const void* q, const void* k, const void* v, void* out, float* lse,
               const int64_t* doc_lens, int n_docs, spattn_saved** saved) {
  return spattn_fwd_rope(ctx, engine, cfg, layout, bs, q, k, v, out, lse, doc_lens, n_docs, nullptr,
                         0.0, saved);
}

int spattn_fwd_rope(spattn_ctx* ctx, int engine, const spattn_config* cfg,
                    const spattn_layout* layout, int64_t bs, const void* q, const void* k,
                    const void* v, void* out, float* lse, const int64_t* doc_lens, int n_docs,
                    const int64_t* position_ids, double rope_base, spattn_saved** saved) {
  return guard([&] {
    const auto c = make_cfg(cfg);
    const auto L = make_layout(layout);
    const auto w = views(c, L, bs, q, k, v, out);
    const auto D = docs_of(doc_lens, n_docs);
    const auto R = rope_of(position_ids, w.q.len, rope_base);
    auto s = seqpar::run_attention_engine(*ctx->rc, make_engine(engine), c, L, w.q, w.k, w.v, w.o,
                                          lse, D.get(), R.get());
    if (saved) {
      *saved = new spattn_saved{std::move(s)};
    }
  });
}

int spattn_bwd(spattn_ctx* ctx, spattn_saved* saved, const void* dout, void* dq, void* dk, void* dv) {
  return guard([&] {
    if (!saved || !saved->s) throw seqpar::StateError("backward without a saved forward");
    auto& S = *saved->s;
    // views take the forward's shapes
    seqpar::run_attention_engine_backward(*ctx->rc, S, seqpar::saved_view(S, 0, const_cast<void*>(dout)),
                                          seqpar::saved_view(S, 0, dq), seqpar::saved_view(S, 1, dk),
                                          seqpar::saved_view(S, 1, dv));
  });
}

void spattn_saved_free(spattn_saved* s) { delete s; }

int spattn_fabric_fwd(spattn_fabric* f, int engine, const spattn_config* cfg,
                      const spattn_layout* layout, int64_t bs, const void* const* q,
                      const void* const* k, const void* const* v, void* const* out,
                      float* const* lse, const int64_t* doc_lens, int n_docs, spattn_saved** saved) {
  return spattn_fabric_fwd_rope(f, engine, cfg, layout, bs, q, k, v, out, lse, doc_lens, n_docs,
                                nullptr, 0.0, saved);
}

int spattn_fabric_fwd_rope(spattn_fabric* f, int engine, const spattn_config* cfg,
                           const spattn_layout* layout, int64_t bs, const void* const* q,
                           const void* const* k, const void* const* v, void* const* out,
                           float* const* lse, const int64_t* doc_lens, int n_docs,
                           const int64_t* const* position_ids, double rope_base,
                           spattn_saved** saved) {
  return guard([&] {
    const auto c = make_cfg(cfg);
    const auto L = make_layout(layout);
    const auto D = docs_of(doc_lens, n_docs);
    const auto e = make_engine(engine);
    std::vector<seqpar::SavedPtr> res(static_cast<size_t>(f->f->world_size()));
    f->f->run([&](seqpar::RankCtx& rc) {
      const size_t r = static_cast<size_t>(rc.rank);
      const auto w = views(c, L, bs, q[r], k[r], v[r], out[r]);
      const auto R = rope_of(position_ids ? position_ids[r] : nullptr, w.q.len, rope_base);
      res[r] = seqpar::run_attention_engine(rc, e, c, L, w.q, w.k, w.v, w.o, lse ? lse[r] : nullptr, D.get(),
                                            R.get());
    });
    for (size_t r = 0; r < res.size(); ++r)
      if (saved) saved[r] = new spattn_saved{std::move(res[r])};
  });
}

int spattn_fabric_bwd(spattn_fabric* f, spattn_saved* const* saved, const void* const* dout,
                      void* const* dq, void* const* dk, void* const* dv) {
  return guard([&] {
    f->f->run([&](seqpar::RankCtx& rc) {
      const size_t r = static_cast<size_t>(rc.rank);
      auto& S = *saved[r]->s;
      seqpar::run_attention_engine_backward(rc, S, seqpar::saved_view(S, 0, const_cast<void*>(dout[r])),
                                            seqpar::saved_view(S, 0, dq[r]), seqpar::saved_view(S, 1, dk[r]),
                                            seqpar::saved_view(S, 1, dv[r]));
    });
  });
}

int spattn_fabric_all_to_all(spattn_fabric* f, const void* const* local, void* const* out,
                             int64_t bs, int64_t len, int64_t heads, int64_t dim, int elem_bytes,
                             int scatter_dim, int gather_dim) {
  return guard([&] {
    f->f->run([&](seqpar::RankCtx& rc) {
      const size_t r = static_cast<size_t>(rc.rank);
      seqpar::all_to_all(rc, rc.sp_group, local[r], bs, len, heads, dim, elem_bytes, scatter_dim,
                         gather_dim, out[r]);
    });
  });
}

int spattn_all_to_all(spattn_ctx* ctx, const void* local, void* out, int64_t bs, int64_t len,
                      int64_t heads, int64_t dim, int elem_bytes, int scatter_dim, int gather_dim) {
  return guard([&] {
    seqpar::all_to_all(*ctx->rc, ctx->rc->sp_group, local, bs, len, heads, dim, elem_bytes, scatter_dim,
                       gather_dim, out);
  });
}

int spattn_all_gather(spattn_ctx* ctx, const void* local, void* out, int64_t outer, int64_t extent,
                      int64_t inner_bytes) {
  return guard([&] { seqpar::all_gather(*ctx->rc, ctx->rc->sp_group, local, outer, extent, inner_bytes, out); });
}

int spattn_all_gather_backward(spattn_ctx* ctx, const void* grad_gathered, void* parts, int64_t outer,
                               int64_t extent, int64_t inner_bytes) {
  return guard([&] {
    seqpar::all_gather_backward(*ctx->rc, ctx->rc->sp_group, grad_gathered, outer, extent, inner_bytes, parts);
  });
}

int spattn_ring_shift(spattn_ctx* ctx, const void* payload, void* out, int64_t bytes) {
  return guard([&] { seqpar::ring_shift(*ctx->rc, ctx->rc->sp_group, payload, bytes, out); });
}

int spattn_block_fwd(void* stream, int64_t bs, int heads, int kv_heads, int dim, const void* q,
                     const int64_t* qpos, int64_t lq, const void* k, const void* v,
                     const int64_t* kpos, int64_t lk, int causal, double scale, float* acc_out,
                     float* acc_lse, int64_t* pairs) {
  return guard([&] {
    std::vector<int64_t> qp(qpos, qpos + lq), kp(kpos, kpos + lk);
    seqpar::block_forward_merge(static_cast<cudaStream_t>(stream), bs, heads, kv_heads, dim, q, qp,
                                k, v, kp, causal != 0, scale, acc_out, acc_lse, pairs);
  });
}
int spattn_block_finalize(void* stream, int64_t rows, int dim, const float* acc_out, void* out) {
  return guard([&] { seqpar::block_finalize(static_cast<cudaStream_t>(stream), rows, dim, acc_out, out); });
}
int spattn_lse_merge(void* stream, float* acc_out, float* acc_lse, const float* out,
                     const float* lse, int64_t rows, int dim) {
  return guard([&] {
    spattn::launch_lse_merge(acc_out, acc_lse, out, lse, rows, dim, static_cast<cudaStream_t>(stream));
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw seqpar::StateError(std::string("CUDA: ") + cudaGetErrorString(e));
  });
}
int spattn_block_bwd(void* stream, int64_t bs, int heads, int kv_heads, int dim, const void* q,
                     const int64_t* qpos, int64_t lq, const void* k, const void* v,
                     const int64_t* kpos, int64_t lk, int causal, double scale, const void* out,
                     const float* lse, const void* dout, float* dq, float* dk, float* dv,
                     int64_t* pairs) {
  return guard([&] {
    std::vector<int64_t> qp(qpos, qpos + lq), kp(kpos, kpos + lk);
    seqpar::block_backward(static_cast<cudaStream_t>(stream), bs, heads, kv_heads, dim, q, qp, k, v,
                           kp, causal != 0, scale, out, lse, dout, dq, dk, dv, pairs);
  });
}
int spattn_shard_rows(void* stream, const spattn_layout* layout, int index, int64_t bs,
                      int64_t row_bytes, const void* full, void* local) {
  return guard([&] { row_moves(static_cast<cudaStream_t>(stream), layout, index, bs, row_bytes, full, local, true); });
}
int spattn_gather_rows(void* stream, const spattn_layout* layout, int index, int64_t bs,
                       int64_t row_bytes, const void* local, void* full) {
  return guard([&] { row_moves(static_cast<cudaStream_t>(stream), layout, index, bs, row_bytes, local, full, false); });
}

}  // extern "C"

extern "C" int spattn_rope_apply(void* stream, int64_t bs, int64_t len, int heads, int dim,
                                 const void* x, const int64_t* position_ids, double base,
                                 int inverse, void* out) {
  return guard([&] {
    if (!position_ids) throw seqpar::ShapeError("rope_apply: position ids are required");
    seqpar::rope_apply(static_cast<cudaStream_t>(stream), bs, len, heads, dim, x,
                       std::vector<int64_t>(position_ids, position_ids + len), base, inverse != 0, out);
  });
}

extern "C" int spattn_step_host(spattn_ctx* ctx, int engine, const spattn_config* cfg,
                                const spattn_layout* layout, int64_t bs, const void* q,
                                const void* k, const void* v, const void* dout, void* out,
                                float* lse, void* dq, void* dk, void* dv, const int64_t* doc_lens,
                                int n_docs, int groups) {
  return guard([&] {
    const auto c = make_cfg(cfg);
    const auto L = make_layout(layout);
    (void)views(c, L, bs, q, k, v, out ? out : dq);  // shape / config validation
    const auto D = docs_of(doc_lens, n_docs);
    seqpar::run_attention_step_host(*ctx->rc, make_engine(engine), c, L, bs, q, k, v, dout, out, lse,
                                    dq, dk, dv, D.get(), groups);
  });
}

extern "C" int spattn_pick_step_groups(int engine, const spattn_config* cfg, int sp) {
  try {
    return seqpar::pick_step_groups(make_engine(engine), make_cfg(cfg), sp);
  } catch (...) {
    return 1;
  }
}
extern "C" int spattn_pick_step_groups_len(int engine, const spattn_config* cfg, int sp, int64_t local_len) {
  try {
    return seqpar::pick_step_groups(make_engine(engine), make_cfg(cfg), sp, local_len);
  } catch (...) {
    return 1;
  }
}

extern "C" int spattn_pad_batch(const int64_t* tokens, const int64_t* labels,
                                const int64_t* position_ids, const int64_t* segment_ids,
                                const int64_t* image_map, int64_t len, int sp, int64_t pad_token,
                                int64_t cutoff_len, int pad_to_cutoff, int64_t* out_len,
                                int64_t* out_tokens, int64_t* out_labels,
                                int64_t* out_position_ids, int64_t* out_segment_ids,
                                int64_t* out_image_map) {
  return guard([&] {
    if (len < 0) throw seqpar::ConfigError("pad_batch: negative length");
    auto vec = [&](const int64_t* p) {
      return p ? std::vector<int64_t>(p, p + len) : std::vector<int64_t>();
    };
    seqpar::TrainBatch b;
    b.tokens = vec(tokens), b.labels = vec(labels), b.position_ids = vec(position_ids);
    b.segment_ids = vec(segment_ids), b.image_map = vec(image_map);
    const auto p = seqpar::pad_batch(b, sp, pad_token, cutoff_len, pad_to_cutoff != 0);
    *out_len = p.len();
    auto put = [](const std::vector<int64_t>& v, int64_t* o) {
      if (o && !v.empty()) std::memcpy(o, v.data(), v.size() * sizeof(int64_t));
    };
    put(p.tokens, out_tokens), put(p.labels, out_labels), put(p.position_ids, out_position_ids);
    put(p.segment_ids, out_segment_ids), put(p.image_map, out_image_map);
  });
}

extern "C" int spattn_split_position_map(const spattn_layout* layout, int index,
                                         const int64_t* values, int64_t* out) {
  return guard([&] {
    const auto L = make_layout(layout);
    const auto v = seqpar::split_position_map(
        std::vector<int64_t>(values, values + L.global_len), L, index);
    std::memcpy(out, v.data(), v.size() * sizeof(int64_t));
  });
}

extern "C" int spattn_documents_from_segments(const int64_t* segment_ids, int64_t len,
                                              int64_t* doc_lens, int max_docs, int* n_docs) {
  return guard([&] {
    const auto d = seqpar::documents_from_segments(std::vector<int64_t>(segment_ids, segment_ids + len));
    if (static_cast<int>(d.size()) > max_docs)
      throw seqpar::ShapeError("documents_from_segments: " + std::to_string(d.size()) +
                               " documents exceed the output capacity " + std::to_string(max_docs));
    std::memcpy(doc_lens, d.data(), d.size() * sizeof(int64_t));
    *n_docs = static_cast<int>(d.size());
  });
}

namespace {
void copy_mask(const std::vector<uint8_t>& m, uint8_t* out, int64_t cap, int64_t* out_len) {
  if (static_cast<int64_t>(m.size()) > cap)
    throw seqpar::ShapeError("packing mask of " + std::to_string(m.size()) +
                             " bytes exceeds the output capacity " + std::to_string(cap));
  if (!m.empty()) std::memcpy(out, m.data(), m.size());
  *out_len = static_cast<int64_t>(m.size());
}
}  // namespace

extern "C" int spattn_replicate_packing_mask(spattn_ctx* ctx, const uint8_t* mask, int64_t len,
                                             uint8_t* out, int64_t cap, int64_t* out_len) {
  return guard([&] {
    const std::vector<uint8_t> m = mask ? std::vector<uint8_t>(mask, mask + len) : std::vector<uint8_t>();
    copy_mask(seqpar::replicate_packing_mask(*ctx->rc, ctx->rc->sp_group, m), out, cap, out_len);
  });
}

extern "C" int spattn_broadcast_bytes(spattn_ctx* ctx, const uint8_t* payload, int64_t len, int root,
                                      uint8_t* out, int64_t cap, int64_t* out_len) {
  return guard([&] {
    const std::vector<uint8_t> m = payload ? std::vector<uint8_t>(payload, payload + len) : std::vector<uint8_t>();
    copy_mask(seqpar::broadcast_bytes(*ctx->rc, ctx->rc->sp_group, m, root), out, cap, out_len);
  });
}

extern "C" int spattn_fabric_replicate_packing_mask(spattn_fabric* f, const uint8_t* const* masks,
                                                    const int64_t* lens, uint8_t* const* outs,
                                                    int64_t cap, int64_t* out_lens) {
  return guard([&] {
    f->f->run([&](seqpar::RankCtx& rc) {
      const size_t r = static_cast<size_t>(rc.rank);
      const std::vector<uint8_t> m =
          masks && masks[r] ? std::vector<uint8_t>(masks[r], masks[r] + lens[r]) : std::vector<uint8_t>();
      copy_mask(seqpar::replicate_packing_mask(rc, rc.sp_group, m), outs[r], cap, &out_lens[r]);
    });
  });
}

// ------------------------------------------------------------------------------- losses
namespace {
seqpar::ExactSum limbs_in(const uint64_t* l) {
  std::array<uint64_t, seqpar::ExactSum::kLimbs> a{};
  std::memcpy(a.data(), l, sizeof(a));
  return seqpar::ExactSum::from_limbs(a);
}
void limbs_out(const seqpar::ExactSum& s, uint64_t* l) {
  std::memcpy(l, s.limbs().data(), sizeof(uint64_t) * seqpar::ExactSum::kLimbs);
}
}  // namespace

extern "C" int spattn_logprob_fwd(void* stream, const void* logits, int dtype, int64_t T, int64_t V,
                                  const int64_t* labels, double* out, double* lse) {
  return guard([&] {
    seqpar::logprob_forward(static_cast<cudaStream_t>(stream), logits, dtype, T, V, labels, out, lse);
  });
}
extern "C" int spattn_logprob_bwd(void* stream, const void* logits, int dtype, int64_t T, int64_t V,
                                  const int64_t* labels, const double* lse, const double* g,
                                  void* dlogits, int accumulate) {
  return guard([&] {
    seqpar::logprob_backward(static_cast<cudaStream_t>(stream), logits, dtype, T, V, labels, lse, g,
                             dlogits, accumulate != 0);
  });
}
extern "C" int spattn_exact_sum_device(void* stream, const double* values, int64_t n, uint64_t* limbs) {
  return guard([&] {
    auto acc = limbs_in(limbs);
    acc.merge(seqpar::exact_sum_device(values, n, static_cast<cudaStream_t>(stream)));
    limbs_out(acc, limbs);
  });
}
extern "C" int spattn_exact_sum_host(const double* values, int64_t n, uint64_t* limbs) {
  return guard([&] {
    auto acc = limbs_in(limbs);
    for (int64_t i = 0; i < n; ++i) acc.add(values[i]);
    limbs_out(acc, limbs);
  });
}
extern "C" int spattn_exact_merge(uint64_t* acc, const uint64_t* other) {
  return guard([&] {
    auto a = limbs_in(acc);
    a.merge(limbs_in(other));
    limbs_out(a, acc);
  });
}
extern "C" int spattn_exact_round(const uint64_t* limbs, double* out) {
  return guard([&] { *out = limbs_in(limbs).round_to_double(); });
}
extern "C" int spattn_exact_sum_all_reduce(spattn_ctx* ctx, uint64_t* limbs) {
  return guard([&] {
    limbs_out(seqpar::exact_sum_all_reduce(*ctx->rc, ctx->rc->sp_group, limbs_in(limbs)), limbs);
  });
}
extern "C" int spattn_all_reduce_count(spattn_ctx* ctx, int64_t* n) {
  return guard([&] { *n = seqpar::all_reduce_count(*ctx->rc, ctx->rc->sp_group, *n); });
}
extern "C" int spattn_all_reduce_values(spattn_ctx* ctx, double* values, int64_t n) {
  return guard([&] {
    const auto r = seqpar::all_reduce_values(*ctx->rc, ctx->rc->sp_group,
                                             std::vector<double>(values, values + n));
    std::memcpy(values, r.data(), static_cast<size_t>(n) * sizeof(double));
  });
}
