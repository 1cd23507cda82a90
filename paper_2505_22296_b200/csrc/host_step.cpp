// One training step of the SP attention layer on HOST buffers — the reference's
// run_attention_engine + tape.backward on host tensors (attention.cpp:526-574, the tape
// closures :236-258 / :290-339; the reference keeps every tensor in host memory) — with the
// host<->device traffic overlapped with compute.
//
// Attention heads are independent, so the step is cut into `groups` kv-head groups (each a
// valid engine call on heads/groups query heads and kv_heads/groups kv heads, the same math on
// a head subset). Three streams pipeline them: the H2D of group g+1 (pitched copies out of the
// [bs, len, heads, dim] host rows) and the D2H of group g-1 run on copy streams while group g's
// forward + backward run on the context's compute stream. Double-buffered device slots.
#include <cuda_runtime.h>

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "seqpar/attention.hpp"

namespace seqpar {
namespace {

#define HS_CUDA(x)                                                                            \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess) throw StateError(std::string("CUDA: ") + cudaGetErrorString(e_) + \
                                            " at " #x);                                       \
  } while (0)

struct Slot {
  void *q = nullptr, *k = nullptr, *v = nullptr, *dout = nullptr, *out = nullptr;
  void *dq = nullptr, *dk = nullptr, *dv = nullptr;
  float* lse = nullptr;
  cudaEvent_t loaded = nullptr, dout_loaded = nullptr, computed = nullptr, drained = nullptr;
};

bool group_ok(Engine e, const AttentionConfig& c, int sp, int ng) {
  const int H = c.heads, Hkv = c.kv_heads > 0 ? c.kv_heads : c.heads;
  if (ng < 1 || H % ng || Hkv % ng) return false;
  const int hg = H / ng;
  switch (e) {
    case Engine::ulysses: return hg % sp == 0;
    case Engine::dummy_head:  // no extra dummy heads: groups pad exactly as the whole would
      return static_cast<int64_t>((hg + sp - 1) / sp) * sp * ng == static_cast<int64_t>((H + sp - 1) / sp) * sp;
    case Engine::xtuner: return ng == 1;
    case Engine::usp: return c.ulysses_degree > 0 && hg % c.ulysses_degree == 0;
    default: return true;
  }
}

}  // namespace

int pick_step_groups(Engine e, const AttentionConfig& c, int sp, int64_t local_len) {
  // A ring rank's off-diagonal step block has local_len / 2 keys against local_len queries; its
  // backward launch should keep >= ~6 waves on 148 SMs even after the query-range split (at
  // most 4 pieces, engine.cpp split_query_ranges), or the step's kernels idle in their last
  // wave: at c4 SP=8 one kv head per group gives 64 key tiles x 4 = 256 CTAs, four heads 1024.
  const int Hkv = c.kv_heads > 0 ? c.kv_heads : c.heads;
  const bool ring = e == Engine::ring && sp > 1 && local_len > 0;
  int fallback = 1;
  for (int ng : {8, 4, 2}) {
    if (!group_ok(e, c, sp, ng)) continue;
    if (!ring) return ng;
    fallback = ng;  // smallest allowed so far
    const int64_t ctas = 4 * ((local_len / 2 + 127) / 128) * (Hkv / ng);
    if (ctas >= 6 * 148) return ng;
  }
  return ring ? 1 : fallback;
}

void run_attention_step_host(RankCtx& ctx, Engine engine, const AttentionConfig& cfg,
                             const ShardLayout& layout, int64_t bs, const void* hq, const void* hk,
                             const void* hv, const void* hdout, void* hout, float* hlse, void* hdq,
                             void* hdk, void* hdv, const Documents* docs, int groups) {
  const int H = cfg.heads, Hkv = cfg.kv_heads > 0 ? cfg.kv_heads : cfg.heads, d = cfg.head_dim;
  const int sp = layout.sp;
  const int ng = groups > 0 ? groups : pick_step_groups(engine, cfg, sp, layout.local_len());
  if (!group_ok(engine, cfg, sp, ng))
    throw ConfigError("host step: " + std::to_string(ng) + " head groups do not split heads=" +
                      std::to_string(H) + ", kv_heads=" + std::to_string(Hkv) + " for engine " +
                      engine_name(engine) + " at sp=" + std::to_string(sp));
  if (!hq || !hk || !hv || !hdout || !hdq || !hdk || !hdv) throw ShapeError("host step: null buffer");
  const int64_t lloc = layout.local_len();
  const int64_t rows = bs * lloc;
  const int hg = H / ng, kg = Hkv / ng;
  AttentionConfig gc = cfg;
  gc.heads = hg;
  gc.kv_heads = kg;
  const size_t qb = static_cast<size_t>(rows * hg * d * 2), kb = static_cast<size_t>(rows * kg * d * 2);
  const size_t qpitch = static_cast<size_t>(H) * d * 2, kpitch = static_cast<size_t>(Hkv) * d * 2;
  const size_t qw = static_cast<size_t>(hg) * d * 2, kw = static_cast<size_t>(kg) * d * 2;

  // Single-device steps alternate groups over two compute streams so one group's backward tail
  // overlaps the next group's forward (the last group runs after its predecessor); with
  // collectives (sp > 1) one stream keeps every rank's NCCL calls in the same order.
  cudaStream_t cs = ctx.stream, cs2 = nullptr, up = nullptr, down = nullptr;
  const bool dual = sp == 1 && ng > 1 && !getenv("SPATTN_STEP_SINGLE");  // (profiling switch)
  HS_CUDA(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
  HS_CUDA(cudaStreamCreateWithFlags(&down, cudaStreamNonBlocking));
  if (dual) HS_CUDA(cudaStreamCreateWithFlags(&cs2, cudaStreamNonBlocking));
  const int nslots = std::min(ng, dual ? 4 : 2);
  std::vector<Slot> slots(static_cast<size_t>(nslots));
  std::vector<std::pair<int64_t, cudaEvent_t>> rows_landed;  // chunked first group: (row end, event)
  auto cleanup = [&] {
    // copies in flight (also on an error path) finish before the slots go back to the pool
    cudaStreamSynchronize(up);
    cudaStreamSynchronize(down);
    if (cs2) cudaStreamSynchronize(cs2);
    for (auto& re : rows_landed) cudaEventDestroy(re.second);
    ctx.stream = cs;
    for (auto& s : slots) {
      for (void* p : {s.q, s.k, s.v, s.dout, s.out, s.dq, s.dk, s.dv, static_cast<void*>(s.lse)})
        if (p) cudaFreeAsync(p, cs);
      for (cudaEvent_t e : {s.loaded, s.dout_loaded, s.computed, s.drained})
        if (e) cudaEventDestroy(e);
    }
    cudaStreamDestroy(up);
    cudaStreamDestroy(down);
    if (cs2) cudaStreamDestroy(cs2);
  };
  try {
    for (auto& s : slots) {
      for (void** p : {&s.q, &s.dout, &s.out, &s.dq}) HS_CUDA(cudaMallocAsync(p, qb, cs));
      for (void** p : {&s.k, &s.v, &s.dk, &s.dv}) HS_CUDA(cudaMallocAsync(p, kb, cs));
      HS_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&s.lse), static_cast<size_t>(rows * hg * 4), cs));
      for (cudaEvent_t* e : {&s.loaded, &s.dout_loaded, &s.computed, &s.drained})
        HS_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    }
    // slots allocated on the compute stream must exist before the copy streams touch them
    cudaEvent_t ready;
    HS_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    HS_CUDA(cudaEventRecord(ready, cs));
    HS_CUDA(cudaStreamWaitEvent(up, ready, 0));
    HS_CUDA(cudaStreamWaitEvent(down, ready, 0));
    if (cs2) HS_CUDA(cudaStreamWaitEvent(cs2, ready, 0));
    cudaEventDestroy(ready);

    // profiling (wrong results), -DSPATTN_PROFILING builds only: SPATTN_STEP_NOCOPY=1 skips H2D
    // and D2H, 2 only D2H, 3 only H2D
#ifdef SPATTN_PROFILING
    static const int nocopy = getenv("SPATTN_STEP_NOCOPY") ? atoi(getenv("SPATTN_STEP_NOCOPY")) : 0;
#else
    constexpr int nocopy = 0;
#endif
    auto h2d = [&](void* dst, const void* src, size_t col_bytes, size_t width, size_t pitch) {
      if (nocopy == 1 || nocopy == 3) return;
      HS_CUDA(cudaMemcpy2DAsync(dst, width, static_cast<const char*>(src) + col_bytes, pitch, width,
                                static_cast<size_t>(rows), cudaMemcpyHostToDevice, up));
    };
    auto d2h = [&](void* dst, const void* src, size_t col_bytes, size_t width, size_t pitch) {
      if (nocopy == 1 || nocopy == 2) return;
      HS_CUDA(cudaMemcpy2DAsync(static_cast<char*>(dst) + col_bytes, pitch, src, width, width,
                                static_cast<size_t>(rows), cudaMemcpyDeviceToHost, down));
    };
    // row-range copies (the sequence-chunked first / last group)
    auto h2d_rows = [&](void* dst, const void* src, size_t col_bytes, size_t width, size_t pitch, int64_t r0,
                        int64_t r1) {
      if (nocopy == 1 || nocopy == 3) return;
      HS_CUDA(cudaMemcpy2DAsync(static_cast<char*>(dst) + static_cast<size_t>(r0) * width, width,
                                static_cast<const char*>(src) + static_cast<size_t>(r0) * pitch + col_bytes, pitch,
                                width, static_cast<size_t>(r1 - r0), cudaMemcpyHostToDevice, up));
    };
    auto d2h_rows = [&](void* dst, const void* src, size_t col_bytes, size_t width, size_t pitch, int64_t r0,
                        int64_t r1) {
      if (nocopy == 1 || nocopy == 2) return;
      HS_CUDA(cudaMemcpy2DAsync(static_cast<char*>(dst) + static_cast<size_t>(r0) * pitch + col_bytes, pitch,
                                static_cast<const char*>(src) + static_cast<size_t>(r0) * width, width, width,
                                static_cast<size_t>(r1 - r0), cudaMemcpyDeviceToHost, down));
    };
    // The single-device causal step can run its first group's forward on the first rows that
    // landed and copy out its last group's first final rows while the rest computes
    // (run_single_step_chunked): the step no longer waits for a whole group's H2D at the start
    // nor for a whole group's D2H at the end.
    const bool chunked = single_step_chunkable(ctx, engine, gc, layout, bs, docs) && !getenv("SPATTN_STEP_NO_CHUNKS");
    constexpr int kChunks = 4;
    auto load = [&](int g) {
      Slot& s = slots[static_cast<size_t>(g % nslots)];
      if (g >= nslots) HS_CUDA(cudaStreamWaitEvent(up, s.drained, 0));  // slot's last use done
      if (chunked && g == 0) {
        const int64_t step = std::max<int64_t>(128, (rows / kChunks + 127) / 128 * 128);
        for (int64_t r0 = 0; r0 < rows; r0 += step) {
          const int64_t r1 = std::min(rows, r0 + step);
          h2d_rows(s.q, hq, g * qw, qw, qpitch, r0, r1);
          h2d_rows(s.k, hk, g * kw, kw, kpitch, r0, r1);
          h2d_rows(s.v, hv, g * kw, kw, kpitch, r0, r1);
          cudaEvent_t e;
          HS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          HS_CUDA(cudaEventRecord(e, up));
          rows_landed.emplace_back(r1, e);
        }
      } else {
        h2d(s.q, hq, g * qw, qw, qpitch);
        h2d(s.k, hk, g * kw, kw, kpitch);
        h2d(s.v, hv, g * kw, kw, kpitch);
      }
      HS_CUDA(cudaEventRecord(s.loaded, up));  // the forward starts while dout is in flight
      h2d(s.dout, hdout, g * qw, qw, qpitch);
      HS_CUDA(cudaEventRecord(s.dout_loaded, up));
    };
    // profiling: SPATTN_STEP_TRACE=1 prints a per-group timeline (ms from the step start) to stderr
    static const bool trace = getenv("SPATTN_STEP_TRACE") != nullptr;
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t st) -> int {
      if (!trace) return -1;
      cudaEvent_t e;
      HS_CUDA(cudaEventCreate(&e));
      HS_CUDA(cudaEventRecord(e, st));
      tev.push_back(e);
      return static_cast<int>(tev.size()) - 1;
    };
    std::vector<std::array<int, 6>> tl(static_cast<size_t>(ng), {-1, -1, -1, -1, -1, -1});
    const int t0 = mark(cs);
    if (trace) HS_CUDA(cudaStreamWaitEvent(up, tev[static_cast<size_t>(t0)], 0));
    auto load_t = [&](int g) {
      tl[static_cast<size_t>(g)][0] = mark(up);
      load(g);
      tl[static_cast<size_t>(g)][1] = mark(up);
    };
    load_t(0);
    for (int g = 0; g < ng; ++g) {
      if (g + 1 < ng) load_t(g + 1);
      Slot& s = slots[static_cast<size_t>(g % nslots)];
      // the last group follows the one before it on the same stream: two groups that run side
      // by side finish together and their D2H copies would queue behind each other at the end
      // of the step (profiles/r2_s3.md: 9.6 -> ~5 ms exposed at 128K)
      cudaStream_t gs = (dual && (g & 1) && g + 1 < ng) ? cs2 : cs;
      ctx.stream = gs;
      const bool first_chunked = chunked && g == 0, last_chunked = chunked && g + 1 == ng;
      if (!first_chunked) HS_CUDA(cudaStreamWaitEvent(gs, s.loaded, 0));
      tl[static_cast<size_t>(g)][2] = mark(gs);
      const DeviceTensor tq{s.q, bs, lloc, hg, d}, tk{s.k, bs, lloc, kg, d}, tv{s.v, bs, lloc, kg, d};
      const DeviceTensor to{s.out, bs, lloc, hg, d};
      const DeviceTensor tdo{s.dout, bs, lloc, hg, d}, tdq{s.dq, bs, lloc, hg, d}, tdk{s.dk, bs, lloc, kg, d},
          tdv{s.dv, bs, lloc, kg, d};
      int64_t drained_rows = 0;  // rows of dq / dk / dv already on their way out
      if (first_chunked || last_chunked) {
        SequenceChunks hk_;
        hk_.fwd_chunks = first_chunked ? kChunks : 1;
        hk_.bwd_chunks = last_chunked ? kChunks : 1;
        hk_.before_fwd_chunk = [&](int, int64_t row_end) {
          if (!first_chunked) return;
          for (const auto& re : rows_landed)
            if (re.first >= row_end) {
              HS_CUDA(cudaStreamWaitEvent(gs, re.second, 0));
              return;
            }
          HS_CUDA(cudaStreamWaitEvent(gs, s.loaded, 0));
        };
        hk_.before_backward = [&] { HS_CUDA(cudaStreamWaitEvent(gs, s.dout_loaded, 0)); };
        hk_.after_bwd_chunk = [&](int, int64_t r0, int64_t r1) {
          if (!last_chunked || r1 == rows) return;  // the final rows go out below with the rest
          cudaEvent_t e;
          HS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          HS_CUDA(cudaEventRecord(e, gs));
          HS_CUDA(cudaStreamWaitEvent(down, e, 0));
          cudaEventDestroy(e);  // the wait is enqueued; the event can go
          d2h_rows(hdq, s.dq, g * qw, qw, qpitch, r0, r1);
          d2h_rows(hdk, s.dk, g * kw, kw, kpitch, r0, r1);
          d2h_rows(hdv, s.dv, g * kw, kw, kpitch, r0, r1);
          drained_rows = r1;
        };
        run_single_step_chunked(ctx, engine, gc, layout, tq, tk, tv, to, s.lse, tdo, tdq, tdk, tdv, hk_);
      } else {
        SavedPtr saved = run_attention_engine(ctx, engine, gc, layout, tq, tk, tv, to, s.lse, docs);
        HS_CUDA(cudaStreamWaitEvent(gs, s.dout_loaded, 0));
        run_attention_engine_backward(ctx, *saved, tdo, tdq, tdk, tdv);
        saved.reset();
      }
      ctx.stream = cs;
      tl[static_cast<size_t>(g)][3] = mark(gs);
      HS_CUDA(cudaEventRecord(s.computed, gs));
      HS_CUDA(cudaStreamWaitEvent(down, s.computed, 0));
      tl[static_cast<size_t>(g)][4] = mark(down);
      d2h_rows(hdq, s.dq, g * qw, qw, qpitch, drained_rows, rows);
      d2h_rows(hdk, s.dk, g * kw, kw, kpitch, drained_rows, rows);
      d2h_rows(hdv, s.dv, g * kw, kw, kpitch, drained_rows, rows);
      if (hout) d2h(hout, s.out, g * qw, qw, qpitch);
      if (hlse)
        HS_CUDA(cudaMemcpy2DAsync(reinterpret_cast<char*>(hlse) + static_cast<size_t>(g) * hg * 4,
                                  static_cast<size_t>(H) * 4, s.lse, static_cast<size_t>(hg) * 4,
                                  static_cast<size_t>(hg) * 4, static_cast<size_t>(rows),
                                  cudaMemcpyDeviceToHost, down));
      HS_CUDA(cudaEventRecord(s.drained, down));
      tl[static_cast<size_t>(g)][5] = mark(down);
    }
    if (trace) {
      HS_CUDA(cudaDeviceSynchronize());
      auto at = [&](int i) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, tev[static_cast<size_t>(t0)], tev[static_cast<size_t>(i)]);
        return ms;
      };
      for (int g = 0; g < ng; ++g) {
        const auto& r = tl[static_cast<size_t>(g)];
        fprintf(stderr, "step group %d: H2D %.2f-%.2f  compute %.2f-%.2f  D2H %.2f-%.2f ms\n", g, at(r[0]),
                at(r[1]), at(r[2]), at(r[3]), at(r[4]), at(r[5]));
      }
      for (cudaEvent_t e : tev) cudaEventDestroy(e);
    }
    // the step completes on the compute stream (callers time / synchronise it)
    for (int g = std::max(0, ng - nslots); g < ng; ++g)
      HS_CUDA(cudaStreamWaitEvent(cs, slots[static_cast<size_t>(g % nslots)].drained, 0));
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

}  // namespace seqpar
