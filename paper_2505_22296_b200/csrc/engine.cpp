// SP attention engines on B200: Ulysses, Dummy-Head Ulysses, XTuner hidden-split (comparator),
// zigzag Ring, USP, and the single-device oracle engine — per-rank programs over a Transport.
//
// Reference semantics (paths under /root/reference/proj/src):
//   run_attention_engine  attention.cpp:526-574   (validation, dispatch)
//   ulysses_core/engine   attention.cpp:391-410
//   dummy_head_engine     attention.cpp:412-425   (pad heads to a multiple of sp, slice back)
//   xtuner_engine         attention.cpp:427-464
//   ring_attention/engine attention.cpp:262-352, :466-472
//   usp_engine            attention.cpp:474-522
// B200 design differences (results identical up to bf16/fp32 rounding):
//   * GQA is never expanded (repeat_heads): each rank receives only the kv heads its query
//     heads read (a "kv window") and the kernels index kv head h/rep.
//   * Dummy heads are virtual: no zero head is sent or computed; a rank whose window is all
//     padding simply has zero local heads.
//   * all_to_all + pad/unpad + the layout permutation are one copy-task pass per direction
//     (peer reads on a shared-memory transport; pack -> NCCL send/recv -> unpack otherwise).
//   * Ulysses writes the gathered rows in natural position order, so the attention kernel sees
//     contiguous causal runs for any layout.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "seqpar/attention.hpp"
#ifdef SPATTN_PROFILING
#include <cstdio>

#include <nvtx3/nvToolsExt.h>
#endif
#include "spattn_internal.h"

namespace seqpar {
using spattn::AttnProblem;
using spattn::CopyTask;
using spattn::HeadMap;

#define SP_CUDA(x)                                                                              \
  do {                                                                                          \
    cudaError_t e_ = (x);                                                                       \
    if (e_ != cudaSuccess)                                                                      \
      throw StateError(std::string("CUDA: ") + cudaGetErrorString(e_) + " at " #x);            \
  } while (0)

namespace {
KernelFamily g_family = KernelFamily::tcgen05;
}
void set_kernel_family(KernelFamily f) { g_family = f; }
KernelFamily kernel_family() { return g_family; }

const char* engine_name(Engine e) {
  static const char* n[] = {"oracle", "ulysses", "dummy_head", "xtuner", "ring", "usp"};
  return n[static_cast<int>(e)];
}
Engine engine_from_string(const std::string& s) {  // attention.cpp:10-28
  for (int i = 0; i < 6; ++i)
    if (s == engine_name(static_cast<Engine>(i))) return static_cast<Engine>(i);
  throw ConfigError("unknown engine '" + s + "'");
}

// ------------------------------------------------------------------------- device buffers
namespace {

// Engine workspaces come from the device's stream-ordered pool. Its default release threshold
// (0) hands memory back to the driver at every synchronisation, so each step would re-map
// ~1.5 GB of workspace; keep it cached instead (once per device).
void keep_pool_cached() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  SP_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  for (int d : done)
    if (d == dev) return;
  cudaMemPool_t pool;
  SP_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t keep = UINT64_MAX;
  SP_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  done.push_back(dev);
}

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(size_t n, cudaStream_t st) : bytes(n), s(st) {
    keep_pool_cached();
    if (n) SP_CUDA(cudaMallocAsync(&p, n, st));
  }
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s) { o.p = nullptr; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(bytes, o.bytes);
    std::swap(s, o.s);
    return *this;
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  void zero() {
    if (bytes) SP_CUDA(cudaMemsetAsync(p, 0, bytes, s));
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

void check_launch() { SP_CUDA(cudaGetLastError()); }

// --------------------------------------------------------------------------- problem lists
int64_t admitted_pairs(const AttnProblem& p) {
  if (!p.causal) return static_cast<int64_t>(p.nq) * p.nk;
  // sum_{a=0}^{nq-1} clamp(a + off + 1, 0, nk)
  int64_t total = 0;
  const int64_t a0 = std::max<int64_t>(0, -static_cast<int64_t>(p.off));  // first a with >=1 key
  const int64_t a_full = std::max<int64_t>(a0, static_cast<int64_t>(p.nk) - 1 - p.off);  // a + off + 1 >= nk
  const int64_t a_mid_end = std::min<int64_t>(p.nq, a_full);
  if (a_mid_end > a0) {
    const int64_t lo = a0 + p.off + 1, hi = a_mid_end - 1 + p.off + 1;
    total += (lo + hi) * (a_mid_end - a0) / 2;
  }
  if (p.nq > a_full) total += (p.nq - std::max(a_full, a0)) * static_cast<int64_t>(p.nk);
  return total;
}

struct SubRun {
  int64_t row0, pos0, n;
  int64_t doc;
};

std::vector<SubRun> split_by_docs(const std::vector<PosRun>& runs, const Documents* docs) {
  std::vector<SubRun> out;
  if (!docs || docs->lengths.empty()) {
    for (const auto& r : runs) out.push_back({r.row0, r.pos0, r.n, 0});
    return out;
  }
  std::vector<int64_t> bounds{0};
  for (int64_t l : docs->lengths) bounds.push_back(bounds.back() + l);
  for (const auto& r : runs) {
    int64_t p = r.pos0, row = r.row0;
    const int64_t end = r.pos0 + r.n;
    while (p < end) {
      const auto it = std::upper_bound(bounds.begin(), bounds.end(), p);
      const int64_t doc = (it - bounds.begin()) - 1;
      const int64_t stop = std::min(end, it == bounds.end() ? end : *it);
      out.push_back({row, p, stop - p, doc});
      row += stop - p;
      p = stop;
    }
  }
  return out;
}

// Pairs every query run with every key run of the same document. A pair is skipped when no
// key is admitted, marked full when every key is admitted, else causal with c <= a + off.
// Consecutive key runs of one query run are fused when the earlier one is fully admitted
// (zigzag ring steps and Ulysses both collapse to one problem per query run this way): the
// forward's lists, one problem per query run, so the query-disjoint launches stay few.
// fuse_q (the backward's lists) fuses the other way: consecutive query runs of one key run,
// when every row of the later runs admits the whole key run — one problem per key run, so each
// key tile's backward CTA sweeps all its query tiles once (one dK / dV partial per tile).
std::vector<AttnProblem> make_problems(const std::vector<PosRun>& qruns,
                                       const std::vector<PosRun>& kruns, bool causal, int64_t bs,
                                       int64_t q_rows_b, int64_t k_rows_b, const Documents* docs,
                                       int64_t* pairs, bool fuse_q = false) {
  const auto qs = split_by_docs(qruns, docs), ks = split_by_docs(kruns, docs);
  auto pair_of = [&](const SubRun& Q, const SubRun& K, AttnProblem& p) {
    p = AttnProblem{static_cast<int>(Q.row0), static_cast<int>(Q.n), static_cast<int>(K.row0),
                    static_cast<int>(K.n), 0, 0};
    if (causal) {
      const int64_t off = Q.pos0 - K.pos0;
      if (off + Q.n - 1 < 0) return false;
      if (off < K.n - 1) {
        p.causal = 1;
        p.off = static_cast<int>(off);
      }
    }
    return true;
  };
  std::vector<AttnProblem> one;
  if (!fuse_q) {
    for (const auto& Q : qs) {
      std::vector<AttnProblem> row;
      for (const auto& K : ks) {
        AttnProblem p;
        if (K.doc == Q.doc && pair_of(Q, K, p)) row.push_back(p);
      }
      std::sort(row.begin(), row.end(),
                [](const AttnProblem& a, const AttnProblem& b) { return a.k_row0 < b.k_row0; });
      std::vector<AttnProblem> fused;
      for (const auto& p : row) {
        if (!fused.empty()) {
          AttnProblem& f = fused.back();
          const bool adjacent = f.k_row0 + f.nk == p.k_row0;
          if (adjacent && !f.causal && (!p.causal || p.off >= -1)) {
            const int shift = f.nk;
            f.nk += p.nk;
            if (p.causal) {
              f.causal = 1;
              f.off = p.off + shift;
            }
            continue;
          }
        }
        fused.push_back(p);
      }
      one.insert(one.end(), fused.begin(), fused.end());
    }
  } else {
    for (const auto& K : ks) {
      std::vector<AttnProblem> col;
      for (const auto& Q : qs) {
        AttnProblem p;
        if (K.doc == Q.doc && pair_of(Q, K, p)) col.push_back(p);
      }
      std::sort(col.begin(), col.end(),
                [](const AttnProblem& a, const AttnProblem& b) { return a.q_row0 < b.q_row0; });
      std::vector<AttnProblem> fused;
      for (const auto& p : col) {
        if (!fused.empty()) {
          AttnProblem& f = fused.back();
          // rows a >= f.nq of the fused problem admit keys c <= a + f.off: all nk of them when
          // f.nq + f.off >= nk - 1 (always when f is full)
          const bool adjacent = f.q_row0 + f.nq == p.q_row0;
          if (adjacent && !p.causal && (!f.causal || f.nq + f.off >= f.nk - 1)) {
            f.nq += p.nq;
            continue;
          }
        }
        fused.push_back(p);
      }
      one.insert(one.end(), fused.begin(), fused.end());
    }
  }
  // longest CTAs first across the whole launch (a CTA sweeps its problem's key range in the
  // forward, its query range in the backward): many short runs per rank (block-wise zigzag,
  // packed documents) would otherwise leave the heavy CTAs for the tail
  std::stable_sort(one.begin(), one.end(), [&](const AttnProblem& a, const AttnProblem& b) {
    return fuse_q ? a.nq > b.nq : a.nk > b.nk;
  });
  std::vector<AttnProblem> all;
  int64_t total = 0;
  for (int64_t b = 0; b < bs; ++b)
    for (auto p : one) {
      p.q_row0 += static_cast<int>(b * q_rows_b);
      p.k_row0 += static_cast<int>(b * k_rows_b);
      total += admitted_pairs(p);
      all.push_back(p);
    }
  if (pairs) *pairs = total;
  return all;
}

// Launch groups whose query rows are disjoint (each launch writes or merges a row once).
std::vector<std::vector<AttnProblem>> q_disjoint_waves(const std::vector<AttnProblem>& probs) {
  std::vector<std::vector<AttnProblem>> waves;
  for (const auto& p : probs) {
    bool placed = false;
    for (auto& w : waves) {
      if (static_cast<int>(w.size()) >= spattn::kMaxProblems) continue;
      bool clash = false;
      for (const auto& o : w)
        clash |= !(p.q_row0 + p.nq <= o.q_row0 || o.q_row0 + o.nq <= p.q_row0);
      if (!clash) {
        w.push_back(p);
        placed = true;
        break;
      }
    }
    if (!placed) waves.push_back({p});
  }
  return waves;
}

spattn::ProblemSet to_set(const std::vector<AttnProblem>& v, size_t from, size_t n) {
  spattn::ProblemSet ps;  // only the n problems are set (the struct is 28 KB)
  ps.n = static_cast<int>(n);
  for (size_t i = 0; i < n; ++i) ps.p[i] = v[from + i];
  return ps;
}

}  // namespace

// ---------------------------------------------------------------------- attention drivers
// Declared by the kernel translation units.
}  // namespace seqpar
namespace spattn {
void launch_attn_fwd_mma(const FwdArgs& a, const ProblemSet& ps, cudaStream_t s);
void launch_attn_bwd_mma(const BwdArgs& a, const ProblemSet& ps, cudaStream_t s);
bool tc_fwd_supported(const FwdArgs& a);
void launch_attn_fwd_tc(const FwdArgs& a, const ProblemSet& ps, cudaStream_t s);
void launch_add_tasks_f32(const CopyTaskSet& ts, cudaStream_t s);

bool tc_fwd_pp_supported(const FwdArgs& a);
void launch_attn_fwd_tc_pp(const FwdArgs& a, const ProblemSet& ps, cudaStream_t s);

bool tc_fwd_pair_supported(const FwdArgs& a);
void launch_attn_fwd_pair(const FwdArgs& a, const ProblemSet& ps, cudaStream_t s);

void launch_attn_fwd(const FwdArgs& a, const ProblemSet& ps, cudaStream_t s) {
  // the 1-tile kernel measures faster; the two-tile ping-pong forward is a selectable family
  const bool use_pp = seqpar::kernel_family() == seqpar::KernelFamily::tcgen05_pp || getenv("SPATTN_FWD_PP");
  const bool pair = seqpar::kernel_family() == seqpar::KernelFamily::tcgen05_pair || getenv("SPATTN_FWD_PAIR");
  if (use_pp && tc_fwd_pp_supported(a))
    launch_attn_fwd_tc_pp(a, ps, s);
  else if (pair && seqpar::kernel_family() != seqpar::KernelFamily::mma && tc_fwd_pair_supported(a))
    launch_attn_fwd_pair(a, ps, s);
  else if (seqpar::kernel_family() != seqpar::KernelFamily::mma && tc_fwd_supported(a))
    launch_attn_fwd_tc(a, ps, s);
  else if (seqpar::kernel_family() == seqpar::KernelFamily::mma)
    launch_attn_fwd_mma(a, ps, s);  // selected explicitly (A/B anchor), never a fallback
  else
    throw seqpar::ShapeError("attention forward: the tcgen05 kernels need 16-byte aligned q/k/v base "
                             "pointers and row strides (head_dim 64 or 128)");
}
bool tc_bwd_q64_supported(const BwdArgs& a);
void launch_attn_bwd_tc_q64(const BwdArgs& a, const ProblemSet& ps, cudaStream_t s);
bool tc_bwd_q128_supported(const BwdArgs& a);
void launch_attn_bwd_q128(const BwdArgs& a, const ProblemSet& ps, cudaStream_t s);

// The backward launch picks a tcgen05 kernel for these arguments (q128 for head_dim 128, q64
// otherwise or when selected); both can write dK / dV directly as bf16.
bool bwd_uses_tcgen05(const BwdArgs& a) {
  return seqpar::kernel_family() != seqpar::KernelFamily::mma && tc_bwd_q64_supported(a);
}

void launch_attn_bwd(const BwdArgs& a, const ProblemSet& ps, cudaStream_t s) {
  const bool tc = seqpar::kernel_family() != seqpar::KernelFamily::mma;
  if (tc && seqpar::kernel_family() != seqpar::KernelFamily::tcgen05_q64 && tc_bwd_q128_supported(a))
    launch_attn_bwd_q128(a, ps, s);
  else if (bwd_uses_tcgen05(a))
    launch_attn_bwd_tc_q64(a, ps, s);
  else if (!tc)
    launch_attn_bwd_mma(a, ps, s);  // selected explicitly (A/B anchor), never a fallback
  else
    throw seqpar::ShapeError("attention backward: the tcgen05 kernels need 16-byte aligned q/k/v/dout "
                             "base pointers and row strides (head_dim 64 or 128)");
}
}  // namespace spattn
namespace seqpar {
namespace {

// Kernel timing for bench.py's roofline: CUDA events recorded on the launching stream around
// every attention forward / backward launch group while profiling is on.
struct KernelProfiler {
  std::mutex mu;
  bool on = false;
  struct Rec {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
} g_prof;

struct ProfScope {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  int kind;
  ProfScope(cudaStream_t st, int k) : s(st), kind(k) {
    if (!g_prof.on) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  ~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(g_prof.mu);
    g_prof.recs.push_back({kind, a, b});
  }
};

// Ring-step stream timeline (spattn_debug_timeline): CUDA events around the steps' kernels,
// hops and adds on the stream each runs on.
struct Timeline {
  std::mutex mu;
  bool on = false;
  cudaEvent_t origin = nullptr;
  struct Rec {
    int kind, rank;
    cudaEvent_t a, b;
  };
  std::vector<Rec> recs;
} g_tl;

struct TlScope {
  cudaEvent_t a = nullptr, b = nullptr;
  cudaStream_t s;
  int kind, rank;
  TlScope(cudaStream_t st, int k, int r) : s(st), kind(k), rank(r) {
    if (!g_tl.on) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
  }
  ~TlScope() {
    if (!a) return;
    cudaEventRecord(b, s);
    std::lock_guard<std::mutex> lk(g_tl.mu);
    g_tl.recs.push_back({kind, rank, a, b});
  }
};

void require_dim(int d) {
  if (d != 64 && d != 128) throw ConfigError("attention kernels support head_dim 64 or 128, got " + std::to_string(d));
}

bool q_rows_disjoint(const std::vector<AttnProblem>& probs) {
  std::vector<std::pair<int64_t, int64_t>> iv;
  for (const auto& p : probs) iv.emplace_back(p.q_row0, static_cast<int64_t>(p.q_row0) + p.nq);
  std::sort(iv.begin(), iv.end());
  for (size_t i = 1; i < iv.size(); ++i)
    if (iv[i].first < iv[i - 1].second) return false;
  return true;
}

// Plain or merging forward over a problem list. Plain mode writes every query row once, so its
// problems must cover disjoint query rows (one document / one run each); any number of them is
// launched kMaxProblems at a time. Merge mode (ring steps, fused runs) groups problems into
// q-disjoint waves that merge into the running output one after another.
void attention_forward(cudaStream_t s, const spattn::FwdArgs& base,
                       const std::vector<AttnProblem>& probs, bool merge) {
  require_dim(base.d);
  ProfScope prof(s, 0);
  if (!merge) {
    if (!q_rows_disjoint(probs)) throw StateError("attention_forward: overlapping problems need merge mode");
    for (size_t i = 0; i < probs.size(); i += spattn::kMaxProblems) {
      const size_t n = std::min<size_t>(spattn::kMaxProblems, probs.size() - i);
      spattn::launch_attn_fwd(base, to_set(probs, i, n), s);
      check_launch();
    }
    return;
  }
  for (const auto& w : q_disjoint_waves(probs)) {
    spattn::launch_attn_fwd(base, to_set(w, 0, w.size()), s);
    check_launch();
  }
}

// The backward runs one CTA per (128-key tile, kv head). A launch of few, equally long CTAs (a
// ring step's off-diagonal block at SP=8: 64 key tiles x 8 kv heads = 512 CTAs = 3.46 waves on
// 148 SMs) leaves SMs idle in its last wave; when dK / dV accumulate in fp32 (no direct bf16
// rows), each fully admitted problem's query range is cut into pieces on 128-row boundaries
// (key c of query a is admitted iff c <= a + off, so the piece starting q0 rows later has
// off + q0), and the pieces' dK / dV partial sums meet in the fp32 accumulators. Measured on the
// c4 SP=8 step block (16K queries x 8K keys, tools/step_shape.py): 5.15 -> 4.74 ms.
std::vector<AttnProblem> split_query_ranges(const std::vector<AttnProblem>& probs, int hkv) {
  static const int forced = getenv("SPATTN_BWD_SPLIT") ? atoi(getenv("SPATTN_BWD_SPLIT")) : 0;
  int64_t ctas = 0;
  for (const auto& p : probs) ctas += (p.nk + 127) / 128 * static_cast<int64_t>(hkv);
  const int64_t target = 6 * 148;  // waves enough for a small last-wave share
  int parts = forced > 0 ? forced : (ctas > 0 && ctas < target ? static_cast<int>((target + ctas - 1) / ctas) : 1);
  parts = std::min(parts, 4);
  if (parts <= 1) return probs;
  std::vector<AttnProblem> out;
  for (const auto& p : probs) {
    const int tiles = (p.nq + 127) / 128;
    // only fully admitted blocks (a ring step's off-diagonal runs): causal ones already balance
    // through the heavy-first CTA order, and their pieces would be uneven
    const bool full = !p.causal || p.off >= p.nk - 1;
    const int np = full ? std::min(parts, std::max(1, tiles / 4)) : 1;  // >= 4 query tiles per piece
    if (np <= 1) {
      out.push_back(p);
      continue;
    }
    for (int i = 0; i < np; ++i) {
      const int t0 = tiles * i / np, t1 = tiles * (i + 1) / np;
      AttnProblem q = p;
      q.q_row0 = p.q_row0 + 128 * t0;
      q.nq = std::min(p.nq, 128 * t1) - 128 * t0;
      q.off = p.off + 128 * t0;
      if (q.nq > 0) out.push_back(q);
    }
  }
  return out;
}

void attention_backward(cudaStream_t s, const spattn::BwdArgs& base,
                        const std::vector<AttnProblem>& in) {
  require_dim(base.d);
  ProfScope prof(s, 1);
  const std::vector<AttnProblem> probs =
      base.dk_bf16 || getenv("SPATTN_BWD_NO_SPLIT") ? in : split_query_ranges(in, base.hm.hkv);
  for (size_t i = 0; i < probs.size(); i += spattn::kMaxProblems) {
    const size_t n = std::min<size_t>(spattn::kMaxProblems, probs.size() - i);
    spattn::launch_attn_bwd(base, to_set(probs, i, n), s);
    check_launch();
  }
}

void run_tasks(const std::vector<CopyTask>& tasks, int elem, bool add, cudaStream_t s) {
#ifdef SPATTN_PROFILING
  if (getenv("SPATTN_TRACE_COPIES")) {  // profiling builds: one line per copy launch
    int64_t bytes = 0;
    for (const auto& t : tasks) bytes += t.rows * (t.cols + t.zero_cols) * (t.elem ? t.elem : elem);
    fprintf(stderr, "copies: %zu tasks, %.1f MB, rows %lld x cols %lld (first), add %d, caller %s\n", tasks.size(),
            bytes / 1e6, tasks.empty() ? 0LL : (long long)tasks[0].rows, tasks.empty() ? 0LL : (long long)tasks[0].cols,
            (int)add, getenv("SPATTN_TRACE_TAG") ? getenv("SPATTN_TRACE_TAG") : "");
  }
  // profiling builds: the engine's own packs / unpacks under one NVTX range name, so ncu can
  // select them (--nvtx --nvtx-include "spattn_move/") apart from harness copies
  struct NvtxRange {
    NvtxRange() { nvtxRangePushA("spattn_move"); }
    ~NvtxRange() { nvtxRangePop(); }
  } nvtx_range;
#endif
  for (size_t i = 0; i < tasks.size(); i += spattn::kMaxCopyTasks) {
    spattn::CopyTaskSet ts{};
    ts.n = static_cast<int>(std::min<size_t>(spattn::kMaxCopyTasks, tasks.size() - i));
    for (int j = 0; j < ts.n; ++j) ts.t[j] = tasks[i + static_cast<size_t>(j)];
    if (add)
      spattn::launch_add_tasks_f32(ts, s);
    else
      spattn::launch_copy_tasks(ts, elem, s);
    check_launch();
  }
}

// ------------------------------------------------------------------ sequence <-> head moves
// X_i: member i's sequence shard, rows [bs * lloc], row width xw elements.
// Y_j: member j's head shard, rows [bs * lg], row width yw[j] elements.
// Forward (scatter heads, gather sequence): Y_j[b*lg + dst(i, r)] cols [ycol_j, +n_j) <-
//   X_i[b*lloc + r] cols [xcol_j, +n_j); then pad_j zero columns follow in Y_j.
// Reverse: X_i[b*lloc + r] cols [xcol_j, +n_j) (+)= Y_j[b*lg + dst(i, r)] cols [ycol_j, +n_j).
// dst(i, r) is given by runs[i] (row0 = local row, pos0 = destination row within a batch).
struct Window {
  int64_t xcol = 0, ycol = 0, n = 0, pad = 0;
};
struct MoveSpec {
  int64_t bs = 1, lloc = 0, lg = 0;
  int64_t xw = 0;
  std::vector<int64_t> yw;
  std::vector<Window> win;
  std::vector<std::vector<PosRun>> runs;
  int elem = 2;
};

// RoPE fused into a move (rope.cu): the rotating side is always the sequence-sharded X side,
// whose local row r (within a batch entry) uses row r of the owner's angle table.
struct RopeMove {
  const float2* table = nullptr;  // this rank's float2(cos, sin)[lloc][d/2]
  int dim = 0;
  int sign = 1;  // +1 forward rotation (q, k), -1 inverse (dq, dk)
};

void set_rope(CopyTask& t, const float2* table, int64_t row0, int64_t mod, int dim, int sign) {
  t.rope = table;
  t.rope_row0 = row0;
  t.rope_mod = mod;
  t.rope_dim = dim;
  t.rope_sign = sign;
}

// One forward move (sequence -> head shard) of a tensor for the message path.
struct FwdMove {
  const MoveSpec* m;
  const void* x;
  void* y;
  const RopeMove* rope;
};

// Message path of one or more forward moves over the same group: pack per destination (RoPE
// rotates while packing) -> ONE grouped send/recv carrying every move's messages (per peer in
// move order, the order NCCL matches them in) -> unpack per source. A source whose rows land as
// one contiguous block of y (bs 1, one run of all its rows, this member's window spanning y's
// rows: the natural Ulysses layout) is received in place.
void move_forward_messages(RankCtx& ctx, const CommGroup& g, const std::vector<FwdMove>& moves,
                           cudaStream_t s) {
  const int G = g.size(), me = g.index_of(ctx.rank);
  struct Plan {
    std::vector<int64_t> soff, roff;
    std::vector<char> in_place;
    DevBuf sbuf, rbuf;
  };
  std::vector<Plan> plans(moves.size());
  std::vector<CopyTask> pack_plain, pack_rope, unpack;
  int elem = 0;
  for (size_t k = 0; k < moves.size(); ++k) elem = moves[k].m->elem;
  for (size_t k = 0; k < moves.size(); ++k) {
    const MoveSpec& m = *moves[k].m;
    const RopeMove* rope = moves[k].rope;
    Plan& pl = plans[k];
    const Window& w = m.win[static_cast<size_t>(me)];
    const int64_t yw = m.yw[static_cast<size_t>(me)], rows = m.bs * m.lloc;
    int64_t sent = 0;
    for (int j = 0; j < G; ++j)
      if (j != me) sent += m.bs * m.lloc * m.win[static_cast<size_t>(j)].n * m.elem;
    ctx.count(Primitive::all_to_all, sent);
    pl.soff.assign(G + 1, 0);
    pl.roff.assign(G + 1, 0);
    pl.in_place.assign(G, 0);
    for (int i = 0; i < G; ++i) {
      const auto& ri = m.runs[static_cast<size_t>(i)];
      pl.in_place[i] = m.bs == 1 && ri.size() == 1 && ri[0].row0 == 0 && ri[0].n == m.lloc && w.ycol == 0 &&
                       w.pad == 0 && yw == w.n;
    }
    for (int j = 0; j < G; ++j) pl.soff[j + 1] = pl.soff[j] + rows * m.win[static_cast<size_t>(j)].n;
    for (int i = 0; i < G; ++i) pl.roff[i + 1] = pl.roff[i] + (pl.in_place[i] ? 0 : rows * w.n);
    pl.sbuf = DevBuf(static_cast<size_t>(pl.soff[G] * m.elem), s);
    pl.rbuf = DevBuf(static_cast<size_t>(pl.roff[G] * m.elem), s);
    std::vector<CopyTask> pack;
    for (int j = 0; j < G; ++j) {
      const Window& wj = m.win[static_cast<size_t>(j)];
      if (wj.n == 0) continue;
      pack.push_back({moves[k].x, static_cast<char*>(pl.sbuf.p) + pl.soff[j] * m.elem, m.xw, wj.n, 0, 0, wj.xcol,
                      0, rows, wj.n, 0});
      if (rope) set_rope(pack.back(), rope->table, 0, m.lloc, rope->dim, rope->sign);
    }
    for (CopyTask& t : pack) t.elem = m.elem;  // plain copies of any dtype share one launch
    if (rope)  // rotating packs share one launch of the RoPE copier
      pack_rope.insert(pack_rope.end(), pack.begin(), pack.end());
    else
      pack_plain.insert(pack_plain.end(), pack.begin(), pack.end());
    const size_t first_unpack = unpack.size();
    for (int i = 0; i < G; ++i) {
      if ((w.n == 0 && w.pad == 0) || pl.in_place[i]) continue;
      for (int64_t b = 0; b < m.bs; ++b)
        for (const auto& r : m.runs[static_cast<size_t>(i)])
          unpack.push_back({static_cast<char*>(pl.rbuf.p) + pl.roff[i] * m.elem, moves[k].y, w.n, yw,
                            b * m.lloc + r.row0, b * m.lg + r.pos0, 0, w.ycol, r.n, w.n, w.pad});
    for (size_t t = first_unpack; t < unpack.size(); ++t) unpack[t].elem = m.elem;
    }
  }
  run_tasks(pack_rope, elem, false, s);
  run_tasks(pack_plain, elem, false, s);
  std::vector<Msg> sends, recvs;
  for (int j = 0; j < G; ++j)
    for (size_t k = 0; k < moves.size(); ++k) {
      const MoveSpec& m = *moves[k].m;
      const Plan& pl = plans[k];
      const Window& w = m.win[static_cast<size_t>(me)];
      const int64_t yw = m.yw[static_cast<size_t>(me)], rows = m.bs * m.lloc;
      sends.push_back({j, static_cast<char*>(pl.sbuf.p) + pl.soff[j] * m.elem,
                       static_cast<size_t>((pl.soff[j + 1] - pl.soff[j]) * m.elem)});
      if (pl.in_place[j])
        recvs.push_back({j, static_cast<char*>(moves[k].y) + m.runs[static_cast<size_t>(j)][0].pos0 * yw * m.elem,
                         static_cast<size_t>(rows * w.n * m.elem)});
      else
        recvs.push_back({j, static_cast<char*>(pl.rbuf.p) + pl.roff[j] * m.elem,
                         static_cast<size_t>((pl.roff[j + 1] - pl.roff[j]) * m.elem)});
    }
  ctx.transport->send_recv(g, ctx.rank, sends, recvs, s);
  run_tasks(unpack, elem, false, s);  // tasks carry their element sizes
}

void move_forward(RankCtx& ctx, const CommGroup& g, const MoveSpec& m, const void* x, void* y,
                  cudaStream_t s, const RopeMove* rope = nullptr) {
  const int G = g.size(), me = g.index_of(ctx.rank);
  if (G > 1 && !ctx.transport->peer_access()) {
    move_forward_messages(ctx, g, {{&m, x, y, rope}}, s);  // counts the move itself
    return;
  }
  int64_t sent = 0;
  for (int j = 0; j < G; ++j)
    if (j != me) sent += m.bs * m.lloc * m.win[static_cast<size_t>(j)].n * m.elem;
  ctx.count(Primitive::all_to_all, sent);
  const Window& w = m.win[static_cast<size_t>(me)];
  const int64_t yw = m.yw[static_cast<size_t>(me)];
  auto unpack = [&](int i, const void* src, int64_t src_stride, int64_t src_col0,
                    const float2* table) {
    std::vector<CopyTask> t;
    for (int64_t b = 0; b < m.bs; ++b)
      for (const auto& r : m.runs[static_cast<size_t>(i)]) {
        t.push_back({src, y, src_stride, yw, b * m.lloc + r.row0, b * m.lg + r.pos0, src_col0,
                     w.ycol, r.n, w.n, w.pad});
        if (table) set_rope(t.back(), table, r.row0, m.lloc, rope->dim, rope->sign);
      }
    return t;
  };
  if (G == 1 || ctx.transport->peer_access()) {
    std::vector<void*> ptrs{const_cast<void*>(x)};
    if (G > 1) ptrs = ctx.transport->exchange_ptrs(g, ctx.rank, const_cast<void*>(x), s);
    // peer reads rotate with the SOURCE member's table (its rows' global position ids)
    std::vector<void*> tabs{rope ? const_cast<float2*>(rope->table) : nullptr};
    if (rope && G > 1) tabs = ctx.transport->exchange_ptrs(g, ctx.rank, tabs[0], s);
    std::vector<CopyTask> tasks;
    for (int i = 0; i < G; ++i) {
      auto t = unpack(i, ptrs[static_cast<size_t>(i)], m.xw, w.xcol,
                      rope ? static_cast<const float2*>(tabs[static_cast<size_t>(i)]) : nullptr);
      tasks.insert(tasks.end(), t.begin(), t.end());
    }
    run_tasks(tasks, m.elem, false, s);
    if (G > 1) ctx.transport->release(g, ctx.rank, s);
    return;
  }
}

// Several forward moves over one group: one grouped exchange on the message path, one move at
// a time on the peer-read path (each already a single copy pass).
void move_forward_many(RankCtx& ctx, const CommGroup& g, const std::vector<FwdMove>& moves, cudaStream_t s) {
  if (g.size() > 1 && !ctx.transport->peer_access() && !getenv("SPATTN_NO_GROUPED_MOVES")) {
    move_forward_messages(ctx, g, moves, s);
    return;
  }
  for (const FwdMove& mv : moves) move_forward(ctx, g, *mv.m, mv.x, mv.y, s, mv.rope);
}

void move_reverse(RankCtx& ctx, const CommGroup& g, const MoveSpec& m, const void* y, void* x,
                  bool add, cudaStream_t s, const RopeMove* rope = nullptr) {
  const int G = g.size(), me = g.index_of(ctx.rank);
  const Window& wm = m.win[static_cast<size_t>(me)];
  ctx.count(Primitive::all_to_all, (G - 1) * m.bs * m.lloc * wm.n * m.elem);
  auto gather_from = [&](int j, const void* src, int64_t src_stride, int64_t src_col0,
                         bool packed_rows) {
    const Window& wj = m.win[static_cast<size_t>(j)];
    std::vector<CopyTask> t;
    if (wj.n == 0) return t;
    if (packed_rows) {
      t.push_back({src, x, src_stride, m.xw, 0, 0, src_col0, wj.xcol, m.bs * m.lloc, wj.n, 0});
      if (rope) set_rope(t.back(), rope->table, 0, m.lloc, rope->dim, rope->sign);
      return t;
    }
    for (int64_t b = 0; b < m.bs; ++b)
      for (const auto& r : m.runs[static_cast<size_t>(me)]) {
        t.push_back({src, x, src_stride, m.xw, b * m.lg + r.pos0, b * m.lloc + r.row0, src_col0,
                     wj.xcol, r.n, wj.n, 0});
        if (rope) set_rope(t.back(), rope->table, r.row0, m.lloc, rope->dim, rope->sign);
      }
    return t;
  };
  if (G == 1 || ctx.transport->peer_access()) {
    std::vector<void*> ptrs{const_cast<void*>(y)};
    if (G > 1) ptrs = ctx.transport->exchange_ptrs(g, ctx.rank, const_cast<void*>(y), s);
    // accumulating unpacks run one source per launch: overlapping windows of different
    // members would otherwise race on the same destination elements
    std::vector<CopyTask> tasks;
    for (int j = 0; j < G; ++j) {
      auto t = gather_from(j, ptrs[static_cast<size_t>(j)], m.yw[static_cast<size_t>(j)],
                           m.win[static_cast<size_t>(j)].ycol, false);
      tasks.insert(tasks.end(), t.begin(), t.end());
      if (add) {
        run_tasks(tasks, m.elem, true, s);
        tasks.clear();
      }
    }
    run_tasks(tasks, m.elem, add, s);
    if (G > 1) ctx.transport->release(g, ctx.rank, s);
    return;
  }
  // message path: member me packs, for every destination i, its rows of i in i's local order;
  // a destination whose rows are one contiguous block of y (bs 1, one run, this member's
  // window spanning y's rows: the natural Ulysses layout) is sent in place
  const int64_t rows = m.bs * m.lloc;
  const int64_t ywm = m.yw[static_cast<size_t>(me)];
  auto in_place = [&](int i) {
    const auto& ri = m.runs[static_cast<size_t>(i)];
    return m.bs == 1 && ri.size() == 1 && ri[0].row0 == 0 && ri[0].n == m.lloc && wm.ycol == 0 && ywm == wm.n;
  };
  DevBuf sbuf(static_cast<size_t>(G * rows * wm.n * m.elem), s);
  std::vector<int64_t> roff(G + 1, 0);
  for (int j = 0; j < G; ++j) roff[j + 1] = roff[j] + rows * m.win[static_cast<size_t>(j)].n;
  DevBuf rbuf(static_cast<size_t>(roff[G] * m.elem), s);
  std::vector<CopyTask> pack;
  if (wm.n > 0)
    for (int i = 0; i < G; ++i) {
      if (in_place(i)) continue;
      char* dst = static_cast<char*>(sbuf.p) + i * rows * wm.n * m.elem;
      for (int64_t b = 0; b < m.bs; ++b)
        for (const auto& r : m.runs[static_cast<size_t>(i)])
          pack.push_back({y, dst, m.yw[static_cast<size_t>(me)], wm.n, b * m.lg + r.pos0,
                          b * m.lloc + r.row0, wm.ycol, 0, r.n, wm.n, 0});
    }
  run_tasks(pack, m.elem, false, s);
  std::vector<Msg> sends, recvs;
  for (int i = 0; i < G; ++i) {
    char* src = in_place(i) ? static_cast<char*>(const_cast<void*>(y)) +
                                  m.runs[static_cast<size_t>(i)][0].pos0 * ywm * m.elem
                            : static_cast<char*>(sbuf.p) + i * rows * wm.n * m.elem;
    sends.push_back({i, src, static_cast<size_t>(rows * wm.n * m.elem)});
    recvs.push_back({i, static_cast<char*>(rbuf.p) + roff[i] * m.elem,
                     static_cast<size_t>((roff[i + 1] - roff[i]) * m.elem)});
  }
  ctx.transport->send_recv(g, ctx.rank, sends, recvs, s);
  std::vector<CopyTask> tasks;
  for (int j = 0; j < G; ++j) {
    auto t = gather_from(j, static_cast<char*>(rbuf.p) + roff[j] * m.elem,
                         m.win[static_cast<size_t>(j)].n, 0, true);
    tasks.insert(tasks.end(), t.begin(), t.end());
    if (add) {
      run_tasks(tasks, m.elem, true, s);
      tasks.clear();
    }
  }
  run_tasks(tasks, m.elem, add, s);
}

// One reverse move (head -> sequence shard, overwrite) of a tensor for the message path.
struct RevMove {
  const MoveSpec* m;
  const void* y;
  void* x;
  const RopeMove* rope;
};

// Message path of several non-accumulating reverse moves over one group: each member packs,
// per destination, its rows of that destination (contiguous blocks of the natural Ulysses
// layout are sent in place), ONE grouped send/recv carries every move's messages (per peer in
// move order), then each move unpacks (inverse RoPE rotates while unpacking).
void move_reverse_messages(RankCtx& ctx, const CommGroup& g, const std::vector<RevMove>& moves, cudaStream_t s) {
  const int G = g.size(), me = g.index_of(ctx.rank);
  struct Plan {
    std::vector<int64_t> roff;
    std::vector<char> in_place;
    DevBuf sbuf, rbuf;
  };
  std::vector<Plan> plans(moves.size());
  std::vector<Msg> sends, recvs;
  std::vector<CopyTask> all_pack;
  for (size_t k = 0; k < moves.size(); ++k) {
    const MoveSpec& m = *moves[k].m;
    Plan& pl = plans[k];
    const Window& wm = m.win[static_cast<size_t>(me)];
    ctx.count(Primitive::all_to_all, (G - 1) * m.bs * m.lloc * wm.n * m.elem);
    const int64_t rows = m.bs * m.lloc, ywm = m.yw[static_cast<size_t>(me)];
    pl.in_place.assign(G, 0);
    for (int i = 0; i < G; ++i) {
      const auto& ri = m.runs[static_cast<size_t>(i)];
      pl.in_place[i] = m.bs == 1 && ri.size() == 1 && ri[0].row0 == 0 && ri[0].n == m.lloc && wm.ycol == 0 &&
                       ywm == wm.n;
    }
    pl.sbuf = DevBuf(static_cast<size_t>(G * rows * wm.n * m.elem), s);
    pl.roff.assign(G + 1, 0);
    for (int j = 0; j < G; ++j) pl.roff[j + 1] = pl.roff[j] + rows * m.win[static_cast<size_t>(j)].n;
    pl.rbuf = DevBuf(static_cast<size_t>(pl.roff[G] * m.elem), s);
    std::vector<CopyTask> pack;
    if (wm.n > 0)
      for (int i = 0; i < G; ++i) {
        if (pl.in_place[i]) continue;
        char* dst = static_cast<char*>(pl.sbuf.p) + i * rows * wm.n * m.elem;
        for (int64_t b = 0; b < m.bs; ++b)
          for (const auto& r : m.runs[static_cast<size_t>(i)])
            pack.push_back({moves[k].y, dst, ywm, wm.n, b * m.lg + r.pos0, b * m.lloc + r.row0, wm.ycol, 0, r.n,
                            wm.n, 0});
      }
    for (CopyTask& t : pack) t.elem = m.elem;  // every move's packs share one launch
    all_pack.insert(all_pack.end(), pack.begin(), pack.end());
  }
  run_tasks(all_pack, moves.empty() ? 2 : moves[0].m->elem, false, s);
  for (int i = 0; i < G; ++i)
    for (size_t k = 0; k < moves.size(); ++k) {
      const MoveSpec& m = *moves[k].m;
      const Plan& pl = plans[k];
      const Window& wm = m.win[static_cast<size_t>(me)];
      const int64_t rows = m.bs * m.lloc, ywm = m.yw[static_cast<size_t>(me)];
      char* src = pl.in_place[i] ? static_cast<char*>(const_cast<void*>(moves[k].y)) +
                                      m.runs[static_cast<size_t>(i)][0].pos0 * ywm * m.elem
                                : static_cast<char*>(pl.sbuf.p) + i * rows * wm.n * m.elem;
      sends.push_back({i, src, static_cast<size_t>(rows * wm.n * m.elem)});
      recvs.push_back({i, static_cast<char*>(pl.rbuf.p) + pl.roff[i] * m.elem,
                       static_cast<size_t>((pl.roff[i + 1] - pl.roff[i]) * m.elem)});
    }
  ctx.transport->send_recv(g, ctx.rank, sends, recvs, s);
  // unpacks: rotating ones share one launch, plain ones (any element sizes) another
  std::vector<CopyTask> un_rope, un_plain;
  int elem = moves.empty() ? 2 : moves[0].m->elem;
  for (size_t k = 0; k < moves.size(); ++k) {
    const MoveSpec& m = *moves[k].m;
    const RopeMove* rope = moves[k].rope;
    const Plan& pl = plans[k];
    std::vector<CopyTask> tasks;
    for (int j = 0; j < G; ++j) {
      const Window& wj = m.win[static_cast<size_t>(j)];
      if (wj.n == 0) continue;
      tasks.push_back({static_cast<char*>(pl.rbuf.p) + pl.roff[j] * m.elem, moves[k].x, wj.n, m.xw, 0, 0, 0, wj.xcol,
                       m.bs * m.lloc, wj.n, 0});
      if (rope) set_rope(tasks.back(), rope->table, 0, m.lloc, rope->dim, rope->sign);
    }
    for (CopyTask& t : tasks) t.elem = m.elem;
    if (rope && m.elem != elem) {
      run_tasks(tasks, m.elem, false, s);
      continue;
    }
    auto& dst = rope ? un_rope : un_plain;
    dst.insert(dst.end(), tasks.begin(), tasks.end());
  }
  run_tasks(un_rope, elem, false, s);
  run_tasks(un_plain, elem, false, s);
}

// Several non-accumulating reverse moves over one group (see move_forward_many).
void move_reverse_many(RankCtx& ctx, const CommGroup& g, const std::vector<RevMove>& moves, cudaStream_t s) {
  if (g.size() > 1 && !ctx.transport->peer_access() && !getenv("SPATTN_NO_GROUPED_MOVES")) {
    move_reverse_messages(ctx, g, moves, s);
    return;
  }
  for (const RevMove& mv : moves) move_reverse(ctx, g, *mv.m, mv.y, mv.x, false, s, mv.rope);
}

bool windows_overlap(const std::vector<Window>& w) {
  for (size_t a = 0; a < w.size(); ++a)
    for (size_t b = a + 1; b < w.size(); ++b)
      if (w[a].n && w[b].n && w[a].xcol < w[b].xcol + w[b].n && w[b].xcol < w[a].xcol + w[a].n)
        return true;
  return false;
}

// ---------------------------------------------------------------- head windows (Ulysses)
struct HeadPlan {
  int G = 1;
  int hp = 0;  // padded heads per member
  std::vector<int> qlo, qn, kvlo, kvn;
};

HeadPlan plan_heads(int H, int Hkv, int G) {
  HeadPlan p;
  p.G = G;
  p.hp = (H + G - 1) / G;
  const int rep = H / Hkv;
  for (int j = 0; j < G; ++j) {
    const int lo = j * p.hp;
    const int n = std::max(0, std::min(H, lo + p.hp) - lo);
    p.qlo.push_back(lo);
    p.qn.push_back(n);
    const int klo = n ? lo / rep : 0;
    p.kvlo.push_back(klo);
    p.kvn.push_back(n ? (lo + n - 1) / rep + 1 - klo : 0);
  }
  return p;
}

MoveSpec head_move(const HeadPlan& hp, bool kv, int64_t bs, int64_t lloc, int64_t heads_x, int d,
                   const std::vector<std::vector<PosRun>>& runs, int elem, int64_t unit = -1) {
  // unit: columns per head (d for tensors, 1 for lse)
  const int64_t u = unit < 0 ? d : unit;
  MoveSpec m;
  m.bs = bs;
  m.lloc = lloc;
  m.lg = lloc * hp.G;
  m.xw = heads_x * u;
  m.elem = elem;
  m.runs = runs;
  for (int j = 0; j < hp.G; ++j) {
    const int lo = kv ? hp.kvlo[static_cast<size_t>(j)] : hp.qlo[static_cast<size_t>(j)];
    const int n = kv ? hp.kvn[static_cast<size_t>(j)] : hp.qn[static_cast<size_t>(j)];
    m.win.push_back({lo * u, 0, n * u, 0});
    m.yw.push_back(n * u);
  }
  return m;
}

}  // namespace

// --------------------------------------------------------------------------- saved state
struct SavedState {
  Engine engine = Engine::oracle;
  AttentionConfig cfg;
  ShardLayout layout;
  Documents docs;
  bool has_docs = false;
  int64_t bs = 0, lloc = 0;
  cudaStream_t stream = nullptr;
  // local (sequence-sharded) views captured at forward
  DeviceTensor q, k, v, out;
  // engine workspaces
  std::vector<DevBuf> bufs;
  // ulysses/usp inner: gathered tensors and plan
  HeadPlan hplan;
  int inner_G = 1;
  std::vector<std::vector<PosRun>> inner_runs;
  // ring: local q/k/v/out (either the user views or inner-gathered), lse
  float* lse = nullptr;
  const void* rq = nullptr;
  const void* rk = nullptr;
  const void* rv = nullptr;
  const void* ro = nullptr;
  int64_t rrows = 0;
  HeadMap hm{};
  int64_t q_stride = 0, kv_stride = 0;
  std::vector<AttnProblem> plain_probs;  // single-block attention problems
  // ring
  bool ring = false;
  CommGroup ring_group;
  std::vector<std::vector<PosRun>> ring_runs;  // per ring member: local row -> position
  // xtuner
  int insp = 1;
  // rope (q, k rotated before attention; dq, dk rotated back): angle table of the local rows
  const float2* rope_table = nullptr;
};

void saved_state_free(SavedState* s) { delete s; }

void profile_enable(bool on) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  g_prof.on = on;
}

void timeline_enable(bool on) {
  std::lock_guard<std::mutex> lk(g_tl.mu);
  if (on) {
    for (auto& r : g_tl.recs) cudaEventDestroy(r.a), cudaEventDestroy(r.b);
    g_tl.recs.clear();
    if (!g_tl.origin) SP_CUDA(cudaEventCreate(&g_tl.origin));
    SP_CUDA(cudaDeviceSynchronize());
    SP_CUDA(cudaEventRecord(g_tl.origin, nullptr));
  }
  g_tl.on = on;
}

int64_t timeline_read(double* start_ms, double* end_ms, int* kind, int* rank, int max) {
  std::lock_guard<std::mutex> lk(g_tl.mu);
  SP_CUDA(cudaDeviceSynchronize());
  const int64_t n = static_cast<int64_t>(g_tl.recs.size());
  for (int64_t i = 0; i < n && i < max; ++i) {
    const auto& r = g_tl.recs[static_cast<size_t>(i)];
    float a = 0, b = 0;
    SP_CUDA(cudaEventElapsedTime(&a, g_tl.origin, r.a));
    SP_CUDA(cudaEventElapsedTime(&b, g_tl.origin, r.b));
    start_ms[i] = a, end_ms[i] = b, kind[i] = r.kind, rank[i] = r.rank;
  }
  return n;
}

void profile_read(double* ms, int64_t* n) {
  std::lock_guard<std::mutex> lk(g_prof.mu);
  ms[0] = ms[1] = 0;
  n[0] = n[1] = 0;
  for (auto& r : g_prof.recs) {
    float t = 0;
    SP_CUDA(cudaEventSynchronize(r.b));
    SP_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.kind] += t;
    n[r.kind] += 1;
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.recs.clear();
}

namespace {
// rope_apply (tensor.cpp:548-607) of a whole [bs, lloc, heads, d] bf16 tensor; src == dst is
// allowed (in place).
void rope_rows(const void* src, void* dst, int64_t bs, int64_t lloc, int64_t heads, int d,
               const float2* table, int sign, cudaStream_t s) {
  CopyTask c{src, dst, heads * d, heads * d, 0, 0, 0, 0, bs * lloc, heads * d, 0};
  set_rope(c, table, 0, lloc, d, sign);
  run_tasks({c}, 2, false, s);
}
}  // namespace

void rope_apply(cudaStream_t s, int64_t bs, int64_t len, int64_t heads, int dim, const void* x,
                const std::vector<int64_t>& position_ids, double base, bool inverse, void* out) {
  if (bs < 0 || len < 0 || heads < 0) throw ShapeError("rope_apply: negative extent");
  if (dim <= 0 || dim % 2 != 0) throw ShapeError("rope head dim must be even, got " + std::to_string(dim));
  if (static_cast<int64_t>(position_ids.size()) != len)
    throw ShapeError("position_ids length " + std::to_string(position_ids.size()) +
                     " does not match sequence extent " + std::to_string(len));
  if (bs * len * heads == 0) return;
  DevBuf table(static_cast<size_t>(len * (dim / 2) * 8), s), dpos(static_cast<size_t>(len * 8), s);
  SP_CUDA(cudaMemcpyAsync(dpos.p, position_ids.data(), static_cast<size_t>(len * 8), cudaMemcpyHostToDevice, s));
  spattn::launch_rope_table(table.as<float2>(), dpos.as<int64_t>(), len, dim, base, s);
  rope_rows(x, out, bs, len, heads, dim, table.as<float2>(), inverse ? -1 : 1, s);
  check_launch();
}

DeviceTensor saved_view(const SavedState& s, int which, void* data) {
  DeviceTensor t = which == 0 ? s.q : s.k;
  t.data = data;
  return t;
}

namespace {

struct Local {
  const void* q;
  const void* k;
  const void* v;
  int64_t rows;  // bs * local rows
  int64_t q_stride, kv_stride;
  HeadMap hm;
};

// Single-block attention (oracle_attention, attention.cpp:218-260) on local rows.
void plain_forward(RankCtx& ctx, const Local& L, int d, const std::vector<AttnProblem>& probs,
                   void* out, float* lse) {
  spattn::FwdArgs a{};
  a.q = L.q;
  a.k = L.k;
  a.v = L.v;
  a.o = out;
  a.lse = lse;
  a.acc_o = nullptr;
  a.q_row_stride = L.q_stride;
  a.kv_row_stride = L.kv_stride;
  a.o_row_stride = L.q_stride;
  a.lse_row_stride = L.hm.hq;
  a.d = d;
  a.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
  a.hm = L.hm;
  if (L.hm.hq == 0) return;
  // rows no problem covers (empty attention) carry out=0, lse=-inf (finalize_piece, :151-165);
  // the kernels write every covered row (empty ones included), so the fill is only needed when
  // some row is outside every problem
  std::vector<std::pair<int64_t, int64_t>> iv;
  for (const auto& p : probs) iv.emplace_back(p.q_row0, static_cast<int64_t>(p.q_row0) + p.nq);
  std::sort(iv.begin(), iv.end());
  int64_t reach = 0;
  for (const auto& r : iv)
    if (r.first <= reach) reach = std::max(reach, r.second);
  if (reach < L.rows) {
    SP_CUDA(cudaMemsetAsync(out, 0, static_cast<size_t>(L.rows * L.q_stride * 2), ctx.stream));
    spattn::launch_fill_f32(lse, -INFINITY, L.rows * L.hm.hq, ctx.stream);
  }
  attention_forward(ctx.stream, a, probs, false);
}

// True when every key row of the launch belongs to exactly one problem (disjoint key ranges that
// cover all rows): each (key row, kv head) is then owned by a single backward CTA.
bool keys_exclusive(const std::vector<AttnProblem>& probs, int64_t rows) {
  std::vector<std::pair<int64_t, int64_t>> iv;
  for (const auto& p : probs) iv.emplace_back(p.k_row0, static_cast<int64_t>(p.k_row0) + p.nk);
  std::sort(iv.begin(), iv.end());
  int64_t reach = 0;
  for (const auto& r : iv) {
    if (r.first != reach) return false;  // overlap or gap
    reach = r.second;
  }
  return reach == rows;
}

// dK / dV can go straight to bf16 buffers: the q64 tcgen05 kernel runs for these local tensors
// and every key row is owned by one problem.
bool direct_dkv_ok(const Local& L, int d, const std::vector<AttnProblem>& probs, const void* dk_bf16,
                   const void* dv_bf16) {
  if (!dk_bf16 || !dv_bf16 || L.hm.hq == 0) return false;
  spattn::BwdArgs probe{};
  probe.d = d;
  probe.q = L.q, probe.k = L.k, probe.v = L.v;
  probe.dout = L.q, probe.dq_acc = reinterpret_cast<float*>(const_cast<void*>(L.q));  // alignment probe only
  probe.q_row_stride = L.q_stride, probe.kv_row_stride = L.kv_stride, probe.o_row_stride = L.q_stride;
  probe.dq_row_stride = L.q_stride, probe.dkv_row_stride = L.kv_stride;
  return spattn::bwd_uses_tcgen05(probe) && keys_exclusive(probs, L.rows) &&
         reinterpret_cast<uintptr_t>(dk_bf16) % 16 == 0 && reinterpret_cast<uintptr_t>(dv_bf16) % 16 == 0 &&
         (L.kv_stride * 2) % 16 == 0;
}

// Single-block backward (attention.cpp:236-258 closure). dk_bf16 / dv_bf16 (optional): when the
// q64 tcgen05 kernel runs and the key rows are exclusive, dK / dV are written there as bf16
// (dk / dv untouched) and true is returned; otherwise dk / dv (fp32, zeroed) receive them.
bool plain_backward(RankCtx& ctx, const Local& L, int d, const std::vector<AttnProblem>& probs,
                    const void* out, const float* lse, const void* dout, float* dq, float* dk,
                    float* dv, void* dk_bf16 = nullptr, void* dv_bf16 = nullptr) {
  if (L.hm.hq == 0) return false;
  spattn::BwdArgs a{};
  a.q = L.q;
  a.k = L.k;
  a.v = L.v;
  a.o = out;
  a.dout = dout;
  a.lse = lse;
  DevBuf delta(static_cast<size_t>(L.rows * L.hm.hq * 4), ctx.stream);
  a.delta = delta.as<float>();
  a.dq_acc = dq;
  a.dk_acc = dk;
  a.dv_acc = dv;
  a.q_row_stride = L.q_stride;
  a.kv_row_stride = L.kv_stride;
  a.o_row_stride = L.q_stride;
  a.dq_row_stride = L.q_stride;
  a.dkv_row_stride = L.kv_stride;
  a.lse_row_stride = L.hm.hq;
  a.d = d;
  a.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
  a.hm = L.hm;
  const bool direct = direct_dkv_ok(L, d, probs, dk_bf16, dv_bf16) && spattn::bwd_uses_tcgen05(a);
  if (direct) {
    a.dk_bf16 = dk_bf16;
    a.dv_bf16 = dv_bf16;
    a.dkv_bf16_row_stride = L.kv_stride;
  }
  spattn::launch_attn_bwd_pre(a, static_cast<int>(L.rows), ctx.stream);
  check_launch();
  attention_backward(ctx.stream, a, probs);
  return direct;
}

// ------------------------------------------------------------------------ ring attention
// ring_attention (attention.cpp:262-352): k|v circulate sp-1 times forward (rank i receives
// from i-1), merged with the online softmax; backward circulates k|v|dk|dv sp times.
// The rotation for step s+1 runs on the comm stream while step s computes.
void ring_forward(RankCtx& ctx, const CommGroup& grp, const std::vector<std::vector<PosRun>>& runs,
                  const Local& L, int d, bool causal, int64_t bs, int64_t lrows,
                  const Documents* docs, void* out, float* lse) {
  const int G = grp.size(), me = grp.index_of(ctx.rank);
  const int64_t kv_elems = L.rows * L.kv_stride;
  const size_t kvb = static_cast<size_t>(kv_elems * 2);
  cudaStream_t s = ctx.stream, cs = ctx.comm_stream;
  DevBuf acc(static_cast<size_t>(L.rows * L.q_stride * 4), s);
  acc.zero();
  spattn::launch_fill_f32(lse, -INFINITY, L.rows * L.hm.hq, s);
  DevBuf buf[2] = {DevBuf(2 * kvb, s), DevBuf(2 * kvb, s)};
  SP_CUDA(cudaMemcpyAsync(buf[0].p, L.k, kvb, cudaMemcpyDeviceToDevice, s));
  SP_CUDA(cudaMemcpyAsync(static_cast<char*>(buf[0].p) + kvb, L.v, kvb, cudaMemcpyDeviceToDevice, s));
  cudaEvent_t ev_main, ev_comm;
  SP_CUDA(cudaEventCreateWithFlags(&ev_main, cudaEventDisableTiming));
  SP_CUDA(cudaEventCreateWithFlags(&ev_comm, cudaEventDisableTiming));
  spattn::FwdArgs a{};
  a.q = L.q;
  a.o = nullptr;
  a.acc_o = acc.as<float>();
  a.lse = lse;
  a.q_row_stride = L.q_stride;
  a.kv_row_stride = L.kv_stride;
  a.o_row_stride = L.q_stride;
  a.lse_row_stride = L.hm.hq;
  a.d = d;
  a.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
  a.hm = L.hm;
  int64_t pairs_total = 0;
  for (int step = 0; step < G; ++step) {
    DevBuf& cur = buf[step & 1];
    DevBuf& nxt = buf[(step + 1) & 1];
    if (step + 1 < G) {
      // comm stream: wait for cur to be complete and for nxt's previous readers (step-1)
      SP_CUDA(cudaEventRecord(ev_main, s));
      SP_CUDA(cudaStreamWaitEvent(cs, ev_main, 0));
      ctx.count(Primitive::p2p, static_cast<int64_t>(2 * kvb));
      const int next = (me + 1) % G, prev = (me - 1 + G) % G;
      TlScope tl(cs, 2, ctx.rank);
      if (ctx.transport->peer_access()) {
        auto ptrs = ctx.transport->exchange_ptrs(grp, ctx.rank, cur.p, cs);
        SP_CUDA(cudaMemcpyAsync(nxt.p, ptrs[static_cast<size_t>(prev)], 2 * kvb,
                                cudaMemcpyDeviceToDevice, cs));
        ctx.transport->release(grp, ctx.rank, cs);
      } else {
        ctx.transport->send_recv(grp, ctx.rank, {{next, cur.p, 2 * kvb}}, {{prev, nxt.p, 2 * kvb}}, cs);
      }
      SP_CUDA(cudaEventRecord(ev_comm, cs));
    }
    const int owner = (me - step + G) % G;
    int64_t pairs = 0;
    auto probs = make_problems(runs[static_cast<size_t>(me)], runs[static_cast<size_t>(owner)],
                               causal, bs, lrows, lrows, docs, &pairs);
    pairs_total += pairs;
    a.k = cur.p;
    a.v = static_cast<char*>(cur.p) + kvb;
    if (L.hm.hq > 0 && !probs.empty()) {
      TlScope tl(s, 0, ctx.rank);
      attention_forward(s, a, probs, true);
    }
    if (step + 1 < G) SP_CUDA(cudaStreamWaitEvent(s, ev_comm, 0));
  }
  ctx.add_flops(4 * d * pairs_total * L.hm.hq);
  spattn::launch_f32_to_bf16(out, acc.as<float>(), 1.f, L.rows * L.q_stride, s);
  check_launch();
  SP_CUDA(cudaStreamWaitEvent(s, ev_comm, 0));
  cudaEventDestroy(ev_main);
  cudaEventDestroy(ev_comm);
}

// Backward ring (attention.cpp:290-339): the block of owner (me - step) visits this rank at
// step `step` carrying the dk|dv its earlier holders accumulated; this rank adds its
// contribution and passes it on, and after G hops every block is home. The payload travels
// SPLIT so that only the short dk|dv chain stays between the steps' kernels:
//   * k|v (bf16) of step s+1 is exchanged on the comm stream WHILE step s computes (k|v do not
//     change on the way, so the hop can go early; the home-coming k|v hop is skipped);
//   * step s's kernel accumulates its contribution into a zeroed local buffer; the incoming
//     dk|dv partial sum (received on the comm stream meanwhile) is added once the kernel is
//     done, and the sum is sent on to the next rank while step s+1 computes.
// The exposed per-step cost is the fp32 add over the rank's dk|dv (an HBM pass) instead of the
// whole k|v|dk|dv hop.
void ring_backward(RankCtx& ctx, const CommGroup& grp, const std::vector<std::vector<PosRun>>& runs,
                   const Local& L, int d, bool causal, int64_t bs, int64_t lrows,
                   const Documents* docs, const void* out, const float* lse, const void* dout,
                   float* dq, void* dk_bf16, void* dv_bf16, float* dk_f32, float* dv_f32) {
  const int G = grp.size(), me = grp.index_of(ctx.rank);
  const int64_t kv_elems = L.rows * L.kv_stride;
  const size_t kvb = static_cast<size_t>(kv_elems * 2), gb = static_cast<size_t>(kv_elems * 4);
  cudaStream_t s = ctx.stream, cs = ctx.comm_stream;
  DevBuf kvbuf[2] = {DevBuf(2 * kvb, s), DevBuf(G > 1 ? 2 * kvb : 0, s)};
  DevBuf gacc[2] = {DevBuf(2 * gb, s), DevBuf(G > 1 ? 2 * gb : 0, s)};  // contribution + incoming sum
  DevBuf grecv(G > 1 ? 2 * gb : 0, s);                                  // partial sum from prev
  SP_CUDA(cudaMemcpyAsync(kvbuf[0].p, L.k, kvb, cudaMemcpyDeviceToDevice, s));
  SP_CUDA(cudaMemcpyAsync(static_cast<char*>(kvbuf[0].p) + kvb, L.v, kvb, cudaMemcpyDeviceToDevice, s));
  DevBuf delta(static_cast<size_t>(L.rows * L.hm.hq * 4), s);
  spattn::BwdArgs a{};
  a.q = L.q;
  a.o = out;
  a.dout = dout;
  a.lse = lse;
  a.delta = delta.as<float>();
  a.dq_acc = dq;
  a.q_row_stride = L.q_stride;
  a.kv_row_stride = L.kv_stride;
  a.o_row_stride = L.q_stride;
  a.dq_row_stride = L.q_stride;
  a.dkv_row_stride = L.kv_stride;
  a.lse_row_stride = L.hm.hq;
  a.d = d;
  a.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
  a.hm = L.hm;
  if (L.hm.hq > 0) {
    spattn::launch_attn_bwd_pre(a, static_cast<int>(L.rows), s);
    check_launch();
  }
  // events: ev_kv[b] = k|v of buffer b landed; ev_free[b] = step using kv/gacc buffer b done;
  // ev_add = this step's sum ready to send; ev_g = the next partial sum landed in grecv
  cudaEvent_t ev_kv[2], ev_free[2], ev_add, ev_g;
  for (int i = 0; i < 2; ++i) {
    SP_CUDA(cudaEventCreateWithFlags(&ev_kv[i], cudaEventDisableTiming));
    SP_CUDA(cudaEventCreateWithFlags(&ev_free[i], cudaEventDisableTiming));
  }
  SP_CUDA(cudaEventCreateWithFlags(&ev_add, cudaEventDisableTiming));
  SP_CUDA(cudaEventCreateWithFlags(&ev_g, cudaEventDisableTiming));
  const int next = (me + 1) % G, prev = (me - 1 + G) % G;
  // one neighbour exchange on the comm stream: `send` to next, `recv` from prev
  auto hop = [&](void* send, void* recv, size_t bytes) {
    ctx.count(Primitive::p2p, static_cast<int64_t>(bytes));
    if (ctx.transport->peer_access()) {
      auto ptrs = ctx.transport->exchange_ptrs(grp, ctx.rank, send, cs);
      SP_CUDA(cudaMemcpyAsync(recv, ptrs[static_cast<size_t>(prev)], bytes, cudaMemcpyDeviceToDevice, cs));
      ctx.transport->release(grp, ctx.rank, cs);
    } else {
      ctx.transport->send_recv(grp, ctx.rank, {{next, send, bytes}}, {{prev, recv, bytes}}, cs);
    }
  };
  SP_CUDA(cudaEventRecord(ev_free[1], s));  // buffer 1 has no earlier reader
  int64_t pairs_total = 0;
  for (int step = 0; step < G; ++step) {
    const int b = step & 1;
    char* kv = static_cast<char*>(kvbuf[b].p);
    float* acc = gacc[b].as<float>();
    if (step + 1 < G) {  // k|v of step + 1 travel while this step computes
      SP_CUDA(cudaEventRecord(ev_kv[b], s));  // kvbuf[b] complete (copied / received)
      SP_CUDA(cudaStreamWaitEvent(cs, ev_kv[b], 0));
      SP_CUDA(cudaStreamWaitEvent(cs, ev_free[b ^ 1], 0));  // step - 1 finished reading kvbuf[b^1]
      {
        TlScope tl(cs, 2, ctx.rank);
        hop(kv, kvbuf[b ^ 1].p, 2 * kvb);
      }
      SP_CUDA(cudaEventRecord(ev_kv[b ^ 1], cs));
    }
    const int owner = (me - step + G) % G;
    int64_t pairs = 0;
    auto probs = make_problems(runs[static_cast<size_t>(me)], runs[static_cast<size_t>(owner)],
                               causal, bs, lrows, lrows, docs, &pairs, /*fuse_q=*/true);
    pairs_total += pairs;
    a.k = kv;
    a.v = kv + kvb;
    a.dk_acc = acc;
    a.dv_acc = acc + kv_elems;
    SP_CUDA(cudaMemsetAsync(acc, 0, 2 * gb, s));
    if (L.hm.hq > 0 && !probs.empty()) {
      TlScope tl(s, 1, ctx.rank);
      attention_backward(s, a, probs);
    }
    if (G > 1) {
      if (step > 0) {  // + the partial sum of this block's earlier holders
        SP_CUDA(cudaStreamWaitEvent(s, ev_g, 0));
        TlScope tl(s, 3, ctx.rank);
        spattn::launch_f32_add(acc, grecv.as<float>(), 2 * kv_elems, s);
        check_launch();
      }
      SP_CUDA(cudaEventRecord(ev_add, s));
      SP_CUDA(cudaStreamWaitEvent(cs, ev_add, 0));  // the sum is final and grecv is read
      {
        TlScope tl(cs, 4, ctx.rank);
        hop(acc, grecv.p, 2 * gb);
      }
      SP_CUDA(cudaEventRecord(ev_g, cs));
      SP_CUDA(cudaEventRecord(ev_free[b], s));
      if (step + 1 < G) SP_CUDA(cudaStreamWaitEvent(s, ev_kv[b ^ 1], 0));  // next step's k|v
    }
  }
  ctx.add_flops(10 * d * pairs_total * L.hm.hq);
  // the last hop brought this rank's own block home: its dk|dv summed over every rank
  // (attention.cpp:323-324)
  const float* home = G > 1 ? grecv.as<float>() : gacc[0].as<float>();
  if (G > 1) SP_CUDA(cudaStreamWaitEvent(s, ev_g, 0));
  if (dk_f32) {
    SP_CUDA(cudaMemcpyAsync(dk_f32, home, gb, cudaMemcpyDeviceToDevice, s));
    SP_CUDA(cudaMemcpyAsync(dv_f32, home + kv_elems, gb, cudaMemcpyDeviceToDevice, s));
  } else {
    spattn::launch_f32_to_bf16(dk_bf16, home, 1.f, kv_elems, s);
    spattn::launch_f32_to_bf16(dv_bf16, home + kv_elems, 1.f, kv_elems, s);
    check_launch();
  }
  // the comm stream's last work (the home hop) is joined above; release the events
  SP_CUDA(cudaEventRecord(ev_g, cs));
  SP_CUDA(cudaStreamWaitEvent(s, ev_g, 0));
  for (int i = 0; i < 2; ++i) {
    cudaEventDestroy(ev_kv[i]);
    cudaEventDestroy(ev_free[i]);
  }
  cudaEventDestroy(ev_add);
  cudaEventDestroy(ev_g);
}

void validate(RankCtx& ctx, const AttentionConfig& cfg, const ShardLayout& layout,
              const DeviceTensor& q, const DeviceTensor& k, const DeviceTensor& v) {
  // attention.cpp:529-549
  const int kvh = cfg.kv_heads > 0 ? cfg.kv_heads : cfg.heads;
  if (q.heads != cfg.heads || q.dim != cfg.head_dim)
    throw ShapeError("attention: q shape disagrees with the config");
  if (k.bs != q.bs || k.len != q.len || k.heads != kvh || k.dim != q.dim ||
      v.bs != k.bs || v.len != k.len || v.heads != k.heads || v.dim != k.dim)
    throw ShapeError("attention: kv shape disagrees with the config");
  if (cfg.heads % kvh != 0)
    throw ConfigError("attention: heads=" + std::to_string(cfg.heads) +
                      " not a multiple of kv_heads=" + std::to_string(kvh));
  if (layout.sp != ctx.sp_group.size())
    throw ConfigError("attention: layout sp does not match the communicator size");
  if (q.len != layout.local_len())
    throw ShapeError("attention: local length " + std::to_string(q.len) +
                     " does not match layout shard length " + std::to_string(layout.local_len()));
  require_dim(cfg.head_dim);
}

std::vector<std::vector<PosRun>> runs_of(const ShardLayout& L, int from, int count) {
  std::vector<std::vector<PosRun>> r;
  for (int i = from; i < from + count; ++i) r.push_back(position_runs(L.positions_of(i)));
  return r;
}

std::vector<PosRun> concat_runs(const ShardLayout& L, int from, int count) {
  std::vector<int64_t> pos;
  for (int i = from; i < from + count; ++i) {
    const auto& o = L.positions_of(i);
    pos.insert(pos.end(), o.begin(), o.end());
  }
  return position_runs(pos);
}

CommGroup subgroup(const CommGroup& parent, int from, int count, int stride) {
  CommGroup g;
  for (int t = 0; t < count; ++t) g.ranks.push_back(parent.ranks[static_cast<size_t>(from + t * stride)]);
  return g;
}

}  // namespace

// ----------------------------------------------------------- host planners (exported)
void plan_head_windows(int heads, int kv_heads, int group, std::vector<int>& qlo,
                       std::vector<int>& qn, std::vector<int>& kvlo, std::vector<int>& kvn) {
  if (heads <= 0 || kv_heads <= 0 || heads % kv_heads || group <= 0)
    throw ConfigError("plan_head_windows: invalid heads/kv_heads/group");
  const HeadPlan p = plan_heads(heads, kv_heads, group);
  qlo = p.qlo, qn = p.qn, kvlo = p.kvlo, kvn = p.kvn;
}

std::vector<std::array<int, 6>> plan_problems(const std::vector<int64_t>& qpos,
                                              const std::vector<int64_t>& kpos, bool causal,
                                              const Documents* docs, int64_t* pairs) {
  const auto probs = make_problems(position_runs(qpos), position_runs(kpos), causal, 1,
                                   static_cast<int64_t>(qpos.size()),
                                   static_cast<int64_t>(kpos.size()), docs, pairs);
  std::vector<std::array<int, 6>> out;
  for (const auto& p : probs) out.push_back({p.q_row0, p.nq, p.k_row0, p.nk, p.off, p.causal});
  return out;
}

// =============================================================================== forward
SavedPtr run_attention_engine(RankCtx& ctx, Engine engine, const AttentionConfig& cfg,
                              const ShardLayout& layout, const DeviceTensor& q,
                              const DeviceTensor& k, const DeviceTensor& v,
                              const DeviceTensor& out, float* lse, const Documents* docs,
                              const Rope* rope) {
  validate(ctx, cfg, layout, q, k, v);
  if (docs && !docs->lengths.empty()) {
    int64_t t = 0;
    for (int64_t l : docs->lengths) {
      if (l <= 0) throw ConfigError("documents: lengths must be positive");
      t += l;
    }
    if (t != layout.global_len) throw ConfigError("documents: lengths must sum to the sequence length");
  }
  SavedPtr S(new SavedState);
  S->engine = engine;
  S->cfg = cfg;
  S->layout = layout;
  S->has_docs = docs && !docs->lengths.empty();
  if (S->has_docs) S->docs = *docs;
  const Documents* D = S->has_docs ? &S->docs : nullptr;
  S->bs = q.bs;
  S->lloc = q.len;
  S->stream = ctx.stream;
  S->q = q;
  S->k = k;
  S->v = v;
  S->out = out;
  const int H = cfg.heads, Hkv = cfg.kv_heads > 0 ? cfg.kv_heads : cfg.heads, d = cfg.head_dim;
  const int rep = H / Hkv;
  const int G = layout.sp;
  const int me = ctx.sp_group.index_of(ctx.rank);
  const int64_t bs = q.bs, lloc = q.len, L = layout.global_len;
  cudaStream_t s = ctx.stream;
  auto keep = [&](size_t bytes) -> void* {
    S->bufs.emplace_back(bytes, s);
    return S->bufs.back().p;
  };

  switch (engine) {
    case Engine::oracle: {
      if (G != 1) throw ConfigError("oracle engine runs only at sp=1");
      break;
    }
    case Engine::ulysses:
      if (H % G != 0)
        throw ConfigError("ulysses: heads=" + std::to_string(H) + " not divisible by sp=" +
                          std::to_string(G) + "; use dummy_head or xtuner");
      break;
    case Engine::ring:
      if (layout.mode != SplitMode::zigzag) throw ConfigError("ring engine requires the zigzag layout");
      break;
    case Engine::usp: {
      const int u = cfg.ulysses_degree, r = cfg.ring_degree;
      if (u <= 0 || r <= 0) throw ConfigError("usp: ulysses_degree and ring_degree must be positive");
      if (u * r != G)
        throw ConfigError("usp: ulysses_degree " + std::to_string(u) + " * ring_degree " +
                          std::to_string(r) + " != sp " + std::to_string(G));
      if (layout.mode != SplitMode::usp || layout.u_degree != u || layout.r_degree != r)
        throw ConfigError("usp: layout was not built for these degrees");
      break;
    }
    case Engine::xtuner:
    case Engine::dummy_head:
      break;
  }
  float* lse_local = lse;
  if (!lse_local) lse_local = static_cast<float*>(keep(static_cast<size_t>(bs * lloc * H * 4)));
  S->lse = lse_local;

  // one member: every engine but USP / XTuner is the single block (a one-member ring is its
  // diagonal step alone, attention.cpp:279-291), run without the ring's fp32 dK/dV accumulators,
  // rounding passes and k|v staging copy
  const bool single = engine == Engine::oracle || (engine != Engine::usp && engine != Engine::xtuner && G == 1);
  // RoPE with the caller's global position ids (Model::forward, model.cpp:342-343). Ulysses,
  // Dummy-Head and USP rotate q and k inside the sequence->head copy of the all-to-all; the
  // other engines rotate into a workspace copy first.
  const void* qd = q.data;
  const void* kd = k.data;
  RopeMove rmove;
  const RopeMove* rfwd = nullptr;
  if (rope) {
    if (d % 2 != 0) throw ShapeError("rope head dim must be even, got " + std::to_string(d));
    if (static_cast<int64_t>(rope->position_ids.size()) != lloc)
      throw ShapeError("rope: position ids length " + std::to_string(rope->position_ids.size()) +
                       " for " + std::to_string(lloc) + " tokens");
    float2* table = static_cast<float2*>(keep(static_cast<size_t>(lloc * (d / 2) * 8)));
    DevBuf dpos(static_cast<size_t>(lloc * 8), s);
    SP_CUDA(cudaMemcpyAsync(dpos.p, rope->position_ids.data(), static_cast<size_t>(lloc * 8),
                            cudaMemcpyHostToDevice, s));
    spattn::launch_rope_table(table, dpos.as<int64_t>(), lloc, d, rope->base, s);
    check_launch();
    S->rope_table = table;
    if (!single && (engine == Engine::ulysses || engine == Engine::dummy_head || engine == Engine::usp)) {
      rmove = {table, d, 1};
      rfwd = &rmove;
    } else {
      void* qr = keep(static_cast<size_t>(bs * lloc * H * d * 2));
      void* kr = keep(static_cast<size_t>(bs * lloc * Hkv * d * 2));
      rope_rows(q.data, qr, bs, lloc, H, d, table, 1, s);
      rope_rows(k.data, kr, bs, lloc, Hkv, d, table, 1, s);
      qd = qr, kd = kr;
    }
  }

  if (single) {
    // single device: one block over the full sequence (attention.cpp:559-561)
    Local Lc{qd, kd, v.data, bs * lloc, H * d, Hkv * d, {H, Hkv, 0, 0, rep}};
    auto runs = concat_runs(layout, 0, G);
    int64_t pairs = 0;
    S->plain_probs = make_problems(runs, runs, cfg.causal, bs, lloc, lloc, D, &pairs);
    ctx.add_flops(4 * d * pairs * H);
    plain_forward(ctx, Lc, d, S->plain_probs, out.data, lse_local);
    S->rq = qd, S->rk = kd, S->rv = v.data, S->ro = out.data;
    S->rrows = bs * lloc;
    S->hm = Lc.hm;
    S->q_stride = H * d, S->kv_stride = Hkv * d;
    S->engine = Engine::oracle;
    return S;
  }

  if (engine == Engine::ring) {
    Local Lc{qd, kd, v.data, bs * lloc, H * d, Hkv * d, {H, Hkv, 0, 0, rep}};
    S->ring = true;
    S->ring_group = ctx.sp_group;
    S->ring_runs = runs_of(layout, 0, G);
    ring_forward(ctx, ctx.sp_group, S->ring_runs, Lc, d, cfg.causal, bs, lloc, D, out.data, lse_local);
    S->rq = qd, S->rk = kd, S->rv = v.data, S->ro = out.data;
    S->rrows = bs * lloc;
    S->hm = Lc.hm;
    S->q_stride = H * d, S->kv_stride = Hkv * d;
    return S;
  }

  if (engine == Engine::xtuner) {
    // attention.cpp:427-464 — virtual heads of d/insp, a2a, all-gather of insp fragments into
    // hv_local full heads per rank, attention replicated insp times, virtual slice back.
    const int insp = pick_xtuner_insp(H, G, d);
    const int hv_local = H * insp / G;
    const int grp = me / insp;
    S->insp = insp;
    const int64_t lg = lloc * G;
    auto runs = runs_of(layout, 0, G);
    auto gather_spec = [&](bool kv, int elem, int64_t unit) {
      MoveSpec m;
      m.bs = bs, m.lloc = lloc, m.lg = lg, m.elem = elem, m.runs = runs;
      m.xw = (kv ? Hkv : H) * unit;
      for (int j = 0; j < G; ++j) {
        const int g = j / insp;
        int lo = g * hv_local, n = hv_local;
        if (kv) {
          const int klo = lo / rep;
          n = (lo + n - 1) / rep + 1 - klo;
          lo = klo;
        }
        m.win.push_back({lo * unit, 0, n * unit, 0});
        m.yw.push_back(n * unit);
      }
      return m;
    };
    MoveSpec mq = gather_spec(false, 2, d), mkv = gather_spec(true, 2, d);
    const int nkv = static_cast<int>(mkv.yw[static_cast<size_t>(me)] / d);
    void* qg = keep(static_cast<size_t>(bs * lg * hv_local * d * 2));
    void* kg = keep(static_cast<size_t>(bs * lg * nkv * d * 2));
    void* vg = keep(static_cast<size_t>(bs * lg * nkv * d * 2));
    void* og = keep(static_cast<size_t>(bs * lg * hv_local * d * 2));
    float* lg_lse = static_cast<float*>(keep(static_cast<size_t>(bs * lg * hv_local * 4)));
    move_forward(ctx, ctx.sp_group, mq, qd, qg, s);
    move_forward(ctx, ctx.sp_group, mkv, kd, kg, s);
    move_forward(ctx, ctx.sp_group, mkv, v.data, vg, s);
    Local Lc{qg, kg, vg, bs * lg, hv_local * d, nkv * d,
             {hv_local, nkv, grp * hv_local, static_cast<int>(mkv.win[static_cast<size_t>(me)].xcol / d), rep}};
    const std::vector<PosRun> full{{0, 0, lg}};
    int64_t pairs = 0;
    S->plain_probs = make_problems(full, full, cfg.causal, bs, lg, lg, D, &pairs);
    ctx.add_flops(4 * d * pairs * hv_local);
    plain_forward(ctx, Lc, d, S->plain_probs, og, lg_lse);
    // virtual slice of this member -> out (contiguous columns of the group's head block)
    MoveSpec mo;
    mo.bs = bs, mo.lloc = lloc, mo.lg = lg, mo.elem = 2, mo.runs = runs, mo.xw = H * d;
    MoveSpec ml = mo;
    ml.elem = 4, ml.xw = H;
    const int64_t frag = static_cast<int64_t>(hv_local) * d / insp;
    for (int j = 0; j < G; ++j) {
      const int g = j / insp, f = j - g * insp;
      mo.win.push_back({g * hv_local * d + f * frag, f * frag, frag, 0});
      mo.yw.push_back(hv_local * d);
      ml.win.push_back({g * hv_local, 0, f == 0 ? hv_local : 0, 0});
      ml.yw.push_back(hv_local);
    }
    move_reverse(ctx, ctx.sp_group, mo, og, out.data, false, s);
    move_reverse(ctx, ctx.sp_group, ml, lg_lse, lse_local, false, s);
    S->rq = qg, S->rk = kg, S->rv = vg, S->ro = og;
    S->lse = lg_lse;
    S->rrows = bs * lg;
    S->hm = Lc.hm;
    S->q_stride = hv_local * d, S->kv_stride = nkv * d;
    return S;
  }

  // ---- ulysses / dummy_head (all G members) and usp (inner u members, then ring over r)
  int u = G, r = 1, inner_from = 0, rho = 0, iota = me;
  if (engine == Engine::usp) {
    u = cfg.ulysses_degree, r = cfg.ring_degree;
    rho = me / u, iota = me % u;
    inner_from = rho * u;
  }
  const CommGroup inner = subgroup(ctx.sp_group, inner_from, u, 1);
  HeadPlan hp = plan_heads(H, Hkv, u);
  S->hplan = hp;
  S->inner_G = u;
  const int64_t lg = lloc * u;
  // destination rows: natural positions for ulysses/dummy (rows == positions); source order
  // for usp (rows follow the ring layout's positions, attention.cpp:370-378)
  std::vector<std::vector<PosRun>> runs;
  if (engine == Engine::usp) {
    for (int t = 0; t < u; ++t) runs.push_back({{0, t * lloc, lloc}});
  } else {
    runs = runs_of(layout, 0, G);
  }
  S->inner_runs = runs;
  const int nq = hp.qn[static_cast<size_t>(iota)], nkv = hp.kvn[static_cast<size_t>(iota)];
  MoveSpec mq = head_move(hp, false, bs, lloc, H, d, runs, 2);
  MoveSpec mkv = head_move(hp, true, bs, lloc, Hkv, d, runs, 2);
  void* qg = keep(static_cast<size_t>(bs * lg * nq * d * 2));
  void* kg = keep(static_cast<size_t>(bs * lg * nkv * d * 2));
  void* vg = keep(static_cast<size_t>(bs * lg * nkv * d * 2));
  void* og = keep(static_cast<size_t>(bs * lg * nq * d * 2));
  float* glse = static_cast<float*>(keep(static_cast<size_t>(bs * lg * nq * 4)));
  move_forward_many(ctx, inner, {{&mq, qd, qg, rfwd}, {&mkv, kd, kg, rfwd}, {&mkv, v.data, vg, nullptr}}, s);
  Local Lc{qg, kg, vg, bs * lg, nq * d, nkv * d,
           {nq, nkv, hp.qlo[static_cast<size_t>(iota)], hp.kvlo[static_cast<size_t>(iota)], rep}};
  if (engine == Engine::usp && r > 1) {
    const CommGroup outer = subgroup(ctx.sp_group, iota, r, u);
    const ShardLayout ring_layout = ShardLayout::make_zigzag(L, r);
    S->ring = true;
    S->ring_group = outer;
    S->ring_runs = runs_of(ring_layout, 0, r);
    ring_forward(ctx, outer, S->ring_runs, Lc, d, cfg.causal, bs, lg, D, og, glse);
  } else {
    const auto pr = engine == Engine::usp ? concat_runs(layout, rho * u, u)
                                          : std::vector<PosRun>{{0, 0, lg}};
    int64_t pairs = 0;
    S->plain_probs = make_problems(pr, pr, cfg.causal, bs, lg, lg, D, &pairs);
    ctx.add_flops(4 * d * pairs * nq);
    plain_forward(ctx, Lc, d, S->plain_probs, og, glse);
  }
  MoveSpec ml = head_move(hp, false, bs, lloc, H, d, runs, 4, 1);
  move_reverse_many(ctx, inner, {{&mq, og, out.data, nullptr}, {&ml, glse, lse_local, nullptr}}, s);
  S->rq = qg, S->rk = kg, S->rv = vg, S->ro = og;
  S->lse = glse;
  S->rrows = bs * lg;
  S->hm = Lc.hm;
  S->q_stride = nq * d, S->kv_stride = nkv * d;
  return S;
}

// ============================================================================== backward
void run_attention_engine_backward(RankCtx& ctx, SavedState& S, const DeviceTensor& dout,
                                   const DeviceTensor& dq, const DeviceTensor& dk,
                                   const DeviceTensor& dv) {
  const AttentionConfig& cfg = S.cfg;
  const int H = cfg.heads, Hkv = cfg.kv_heads > 0 ? cfg.kv_heads : cfg.heads, d = cfg.head_dim;
  const int G = S.layout.sp;
  const int me = ctx.sp_group.index_of(ctx.rank);
  const int64_t bs = S.bs, lloc = S.lloc;
  const Documents* D = S.has_docs ? &S.docs : nullptr;
  cudaStream_t s = ctx.stream;
  if (dout.bs != bs || dout.len != lloc || dout.heads != H || dout.dim != d)
    throw ShapeError("backward: dout shape disagrees with the forward output");
  Local Lc{S.rq, S.rk, S.rv, S.rrows, S.q_stride, S.kv_stride, S.hm};

  if (S.engine == Engine::oracle || (S.engine == Engine::ring)) {
    const int64_t rows = bs * lloc;
    DevBuf dqa(static_cast<size_t>(rows * H * d * 4), s);
    dqa.zero();
    if (S.engine == Engine::oracle) {
      int64_t pairs = 0;
      for (const auto& p : S.plain_probs) pairs += admitted_pairs(p);
      ctx.add_flops(10 * d * pairs * H);
      // exclusive key rows: dK / dV straight to bf16 (no fp32 accumulators, fill or rounding)
      if (direct_dkv_ok(Lc, d, S.plain_probs, dk.data, dv.data)) {
        const bool direct = plain_backward(ctx, Lc, d, S.plain_probs, S.ro, S.lse, dout.data, dqa.as<float>(),
                                           nullptr, nullptr, dk.data, dv.data);
        if (!direct) throw StateError("backward: direct dK/dV path unexpectedly unavailable");
      } else {
        DevBuf dka(static_cast<size_t>(rows * Hkv * d * 4), s), dva(static_cast<size_t>(rows * Hkv * d * 4), s);
        dka.zero();
        dva.zero();
        plain_backward(ctx, Lc, d, S.plain_probs, S.ro, S.lse, dout.data, dqa.as<float>(), dka.as<float>(),
                       dva.as<float>());
        spattn::launch_f32_to_bf16(dk.data, dka.as<float>(), 1.f, rows * Hkv * d, s);
        spattn::launch_f32_to_bf16(dv.data, dva.as<float>(), 1.f, rows * Hkv * d, s);
      }
    } else {
      ring_backward(ctx, S.ring_group, S.ring_runs, Lc, d, cfg.causal, bs, lloc, D, S.ro, S.lse,
                    dout.data, dqa.as<float>(), dk.data, dv.data, nullptr, nullptr);
    }
    spattn::launch_f32_to_bf16(dq.data, dqa.as<float>(), 1.f, rows * H * d, s);
    if (S.rope_table) {  // rope_apply backward (tensor.cpp:589-600): inverse rotation
      rope_rows(dq.data, dq.data, bs, lloc, H, d, S.rope_table, -1, s);
      rope_rows(dk.data, dk.data, bs, lloc, Hkv, d, S.rope_table, -1, s);
    }
    check_launch();
    return;
  }

  if (S.engine == Engine::xtuner) {
    const int insp = S.insp, hv_local = H * insp / G, grp = me / insp;
    const int rep = H / Hkv;
    const int64_t lg = lloc * G;
    auto runs = runs_of(S.layout, 0, G);
    // full group dout (all fragments of the group's heads): same pattern as the q gather
    MoveSpec mq;
    mq.bs = bs, mq.lloc = lloc, mq.lg = lg, mq.elem = 2, mq.runs = runs, mq.xw = H * d;
    for (int j = 0; j < G; ++j) {
      mq.win.push_back({(j / insp) * hv_local * d, 0, static_cast<int64_t>(hv_local) * d, 0});
      mq.yw.push_back(hv_local * d);
    }
    const int nkv = S.hm.hkv;
    DevBuf dog(static_cast<size_t>(bs * lg * hv_local * d * 2), s);
    move_forward(ctx, ctx.sp_group, mq, dout.data, dog.p, s);
    DevBuf dqa(static_cast<size_t>(bs * lg * hv_local * d * 4), s), dka(static_cast<size_t>(bs * lg * nkv * d * 4), s),
        dva(static_cast<size_t>(bs * lg * nkv * d * 4), s);
    dqa.zero(), dka.zero(), dva.zero();
    int64_t pairs = 0;
    for (const auto& p : S.plain_probs) pairs += admitted_pairs(p);
    ctx.add_flops(10 * d * pairs * hv_local);
    plain_backward(ctx, Lc, d, S.plain_probs, S.ro, S.lse, dog.p, dqa.as<float>(), dka.as<float>(),
                   dva.as<float>());
    DevBuf dqg(static_cast<size_t>(bs * lg * hv_local * d * 2), s);
    spattn::launch_f32_to_bf16(dqg.p, dqa.as<float>(), 1.f, bs * lg * hv_local * d, s);
    MoveSpec mo;
    mo.bs = bs, mo.lloc = lloc, mo.lg = lg, mo.elem = 2, mo.runs = runs, mo.xw = H * d;
    const int64_t frag = static_cast<int64_t>(hv_local) * d / insp;
    for (int j = 0; j < G; ++j) {
      const int g = j / insp, f = j - g * insp;
      mo.win.push_back({g * hv_local * d + f * frag, f * frag, frag, 0});
      mo.yw.push_back(hv_local * d);
    }
    move_reverse(ctx, ctx.sp_group, mo, dqg.p, dq.data, false, s);
    // kv grads: member j returns fragment f of its group's kv block; groups sharing a kv head
    // add up (the repeat_heads backward sum, tensor.cpp:437-447)
    MoveSpec mk;
    mk.bs = bs, mk.lloc = lloc, mk.lg = lg, mk.elem = 4, mk.runs = runs, mk.xw = Hkv * d;
    for (int j = 0; j < G; ++j) {
      const int g = j / insp, f = j - g * insp;
      const int lo = g * hv_local, klo = lo / rep, kn = (lo + hv_local - 1) / rep + 1 - klo;
      const int64_t kfrag = static_cast<int64_t>(kn) * d / insp;
      mk.win.push_back({klo * d + f * kfrag, f * kfrag, kfrag, 0});
      mk.yw.push_back(kn * d);
    }
    (void)grp;
    const int64_t rows = bs * lloc;
    DevBuf dkf(static_cast<size_t>(rows * Hkv * d * 4), s), dvf(static_cast<size_t>(rows * Hkv * d * 4), s);
    dkf.zero(), dvf.zero();
    move_reverse(ctx, ctx.sp_group, mk, dka.p, dkf.p, true, s);
    move_reverse(ctx, ctx.sp_group, mk, dva.p, dvf.p, true, s);
    spattn::launch_f32_to_bf16(dk.data, dkf.as<float>(), 1.f, rows * Hkv * d, s);
    spattn::launch_f32_to_bf16(dv.data, dvf.as<float>(), 1.f, rows * Hkv * d, s);
    if (S.rope_table) {
      rope_rows(dq.data, dq.data, bs, lloc, H, d, S.rope_table, -1, s);
      rope_rows(dk.data, dk.data, bs, lloc, Hkv, d, S.rope_table, -1, s);
    }
    check_launch();
    return;
  }

  // ---- ulysses / dummy_head / usp
  const HeadPlan& hp = S.hplan;
  const int u = S.inner_G;
  const int inner_from = S.engine == Engine::usp ? (me / u) * u : 0;
  const int iota = S.engine == Engine::usp ? me % u : me;
  const CommGroup inner = subgroup(ctx.sp_group, inner_from, u, 1);
  const int64_t lg = lloc * u;
  const int nq = hp.qn[static_cast<size_t>(iota)], nkv = hp.kvn[static_cast<size_t>(iota)];
  MoveSpec mq = head_move(hp, false, bs, lloc, H, d, S.inner_runs, 2);
  DevBuf dog(static_cast<size_t>(bs * lg * nq * d * 2), s);
  move_forward(ctx, inner, mq, dout.data, dog.p, s);
  MoveSpec mkv = head_move(hp, true, bs, lloc, Hkv, d, S.inner_runs, 2);
  const bool kv_overlap = windows_overlap(mkv.win);
  // the gathered dK / dV go straight to bf16 when no other member shares their kv heads and the
  // kernel owns every key row (no fp32 accumulators, fill or rounding pass)
  DevBuf dkg, dvg;
  if (!kv_overlap) {
    dkg = DevBuf(static_cast<size_t>(bs * lg * nkv * d * 2), s);
    dvg = DevBuf(static_cast<size_t>(bs * lg * nkv * d * 2), s);
  }
  const bool direct = !S.ring && !kv_overlap && direct_dkv_ok(Lc, d, S.plain_probs, dkg.p, dvg.p);
  DevBuf dqa(static_cast<size_t>(bs * lg * nq * d * 4), s), dka, dva;
  dqa.zero();
  if (!direct) {
    dka = DevBuf(static_cast<size_t>(bs * lg * nkv * d * 4), s);
    dva = DevBuf(static_cast<size_t>(bs * lg * nkv * d * 4), s);
    dka.zero(), dva.zero();
  }
  if (S.ring) {
    ring_backward(ctx, S.ring_group, S.ring_runs, Lc, d, cfg.causal, bs, lg, D, S.ro, S.lse, dog.p,
                  dqa.as<float>(), nullptr, nullptr, dka.as<float>(), dva.as<float>());
  } else {
    int64_t pairs = 0;
    for (const auto& p : S.plain_probs) pairs += admitted_pairs(p);
    ctx.add_flops(10 * d * pairs * nq);
    const bool used = plain_backward(ctx, Lc, d, S.plain_probs, S.ro, S.lse, dog.p, dqa.as<float>(),
                                     dka.as<float>(), dva.as<float>(), direct ? dkg.p : nullptr,
                                     direct ? dvg.p : nullptr);
    if (used != direct) throw StateError("backward: direct dK/dV decision changed between planning and launch");
  }
  DevBuf dqg(static_cast<size_t>(bs * lg * nq * d * 2), s);
  spattn::launch_f32_to_bf16(dqg.p, dqa.as<float>(), 1.f, bs * lg * nq * d, s);
  // the inverse rotation of dq/dk rides the head->sequence copy back (rope.cu)
  const RopeMove rinv{S.rope_table, d, -1};
  const RopeMove* rbwd = S.rope_table ? &rinv : nullptr;
  const int64_t rows = bs * lloc;
  if (!kv_overlap) {
    if (!direct) {
      spattn::launch_f32_to_bf16(dkg.p, dka.as<float>(), 1.f, bs * lg * nkv * d, s);
      spattn::launch_f32_to_bf16(dvg.p, dva.as<float>(), 1.f, bs * lg * nkv * d, s);
    }
    move_reverse_many(ctx, inner, {{&mq, dqg.p, dq.data, rbwd}, {&mkv, dkg.p, dk.data, rbwd},
                                   {&mkv, dvg.p, dv.data, nullptr}}, s);
  } else {
    move_reverse(ctx, inner, mq, dqg.p, dq.data, false, s, rbwd);
    // kv heads shared by members (Hkv % u != 0): sum fp32 partials (repeat_heads backward)
    MoveSpec mk4 = head_move(hp, true, bs, lloc, Hkv, d, S.inner_runs, 4);
    DevBuf dkf(static_cast<size_t>(rows * Hkv * d * 4), s), dvf(static_cast<size_t>(rows * Hkv * d * 4), s);
    dkf.zero(), dvf.zero();
    move_reverse(ctx, inner, mk4, dka.p, dkf.p, true, s);
    move_reverse(ctx, inner, mk4, dva.p, dvf.p, true, s);
    spattn::launch_f32_to_bf16(dk.data, dkf.as<float>(), 1.f, rows * Hkv * d, s);
    spattn::launch_f32_to_bf16(dv.data, dvf.as<float>(), 1.f, rows * Hkv * d, s);
    if (S.rope_table) rope_rows(dk.data, dk.data, bs, lloc, Hkv, d, S.rope_table, -1, s);
  }
  check_launch();
}

// ------------------------------------------- single-device step cut along the sequence
bool single_step_chunkable(RankCtx& ctx, Engine e, const AttentionConfig& cfg, const ShardLayout& layout,
                           int64_t bs, const Documents* docs) {
  if (layout.sp != 1 || e == Engine::usp || e == Engine::xtuner || !cfg.causal || bs != 1) return false;
  if (docs && docs->lengths.size() > 1) return false;
  if (ctx.sp_group.size() != 1 || kernel_family() == KernelFamily::mma) return false;
  const auto runs = concat_runs(layout, 0, 1);
  return runs.size() == 1 && runs[0].row0 == 0 && runs[0].pos0 == 0;
}

void run_single_step_chunked(RankCtx& ctx, Engine e, const AttentionConfig& cfg, const ShardLayout& layout,
                             const DeviceTensor& q, const DeviceTensor& k, const DeviceTensor& v,
                             const DeviceTensor& out, float* lse, const DeviceTensor& dout,
                             const DeviceTensor& dq, const DeviceTensor& dk, const DeviceTensor& dv,
                             const SequenceChunks& hooks) {
  validate(ctx, cfg, layout, q, k, v);
  if (!single_step_chunkable(ctx, e, cfg, layout, q.bs, nullptr))
    throw StateError("run_single_step_chunked: not a single-device causal step");
  const int H = cfg.heads, Hkv = cfg.kv_heads > 0 ? cfg.kv_heads : cfg.heads, d = cfg.head_dim;
  const int64_t L = q.len;
  cudaStream_t s = ctx.stream;
  const Local Lc{q.data, k.data, v.data, L, static_cast<int64_t>(H) * d, static_cast<int64_t>(Hkv) * d,
                 {H, Hkv, 0, 0, H / Hkv}};
  // chunk boundaries on 128-row tiles
  auto bounds = [&](int n) {
    std::vector<int64_t> b{0};
    const int64_t step = std::max<int64_t>(128, (L / std::max(1, n) + 127) / 128 * 128);
    while (b.back() < L) b.push_back(std::min(L, b.back() + step));
    return b;
  };
  // forward: query rows [r0, r1) against keys [0, r1) (causal, off = r0); the chunks cover
  // every row, so no empty-row fill is needed (plain_forward would fill the rows outside ITS
  // problems, i.e. the earlier chunks' output)
  spattn::FwdArgs fa{};
  fa.q = q.data, fa.k = k.data, fa.v = v.data, fa.o = out.data, fa.lse = lse, fa.acc_o = nullptr;
  fa.q_row_stride = Lc.q_stride, fa.kv_row_stride = Lc.kv_stride, fa.o_row_stride = Lc.q_stride;
  fa.lse_row_stride = H;
  fa.d = d;
  fa.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
  fa.hm = Lc.hm;
  const auto fb = bounds(hooks.fwd_chunks);
  int64_t pairs = 0;
  for (size_t c = 0; c + 1 < fb.size(); ++c) {
    const int64_t r0 = fb[c], r1 = fb[c + 1];
    if (hooks.before_fwd_chunk) hooks.before_fwd_chunk(static_cast<int>(c), r1);
    const std::vector<AttnProblem> probs{{static_cast<int>(r0), static_cast<int>(r1 - r0), 0, static_cast<int>(r1),
                                          static_cast<int>(r0), 1}};
    pairs += admitted_pairs(probs[0]);
    attention_forward(s, fa, probs, false);
  }
  ctx.add_flops(4 * d * pairs * H);
  if (hooks.before_backward) hooks.before_backward();
  // backward: keys [r0, r1) against queries [r0, L); dq rows [r0, r1) see no later key, so they
  // are final after chunk c, as are the chunk's dk / dv rows
  spattn::BwdArgs a{};
  DevBuf delta(static_cast<size_t>(L * H * 4), s), dqa(static_cast<size_t>(L * H * d * 4), s);
  dqa.zero();
  a.q = q.data, a.k = k.data, a.v = v.data, a.o = out.data, a.dout = dout.data, a.lse = lse;
  a.delta = delta.as<float>();
  a.dq_acc = dqa.as<float>();
  a.q_row_stride = Lc.q_stride, a.kv_row_stride = Lc.kv_stride, a.o_row_stride = Lc.q_stride;
  a.dq_row_stride = Lc.q_stride, a.dkv_row_stride = Lc.kv_stride;
  a.lse_row_stride = H;
  a.d = d;
  a.scale = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
  a.hm = Lc.hm;
  const std::vector<AttnProblem> whole{{0, static_cast<int>(L), 0, static_cast<int>(L), 0, 1}};
  const bool direct = direct_dkv_ok(Lc, d, whole, dk.data, dv.data) && spattn::bwd_uses_tcgen05(a);
  DevBuf dka, dva;
  if (direct) {
    a.dk_bf16 = dk.data, a.dv_bf16 = dv.data, a.dkv_bf16_row_stride = Lc.kv_stride;
  } else {
    dka = DevBuf(static_cast<size_t>(L * Hkv * d * 4), s), dva = DevBuf(static_cast<size_t>(L * Hkv * d * 4), s);
    dka.zero(), dva.zero();
    a.dk_acc = dka.as<float>(), a.dv_acc = dva.as<float>();
  }
  spattn::launch_attn_bwd_pre(a, static_cast<int>(L), s);
  check_launch();
  const auto bb = bounds(hooks.bwd_chunks);
  for (size_t c = 0; c + 1 < bb.size(); ++c) {
    const int64_t r0 = bb[c], r1 = bb[c + 1];
    const std::vector<AttnProblem> probs{{static_cast<int>(r0), static_cast<int>(L - r0), static_cast<int>(r0),
                                          static_cast<int>(r1 - r0), 0, 1}};
    attention_backward(s, a, probs);
    const int64_t qe = Lc.q_stride, ke = Lc.kv_stride;
    spattn::launch_f32_to_bf16(static_cast<char*>(dq.data) + r0 * qe * 2, dqa.as<float>() + r0 * qe, 1.f,
                               (r1 - r0) * qe, s);
    if (!direct) {
      spattn::launch_f32_to_bf16(static_cast<char*>(dk.data) + r0 * ke * 2, dka.as<float>() + r0 * ke, 1.f,
                                 (r1 - r0) * ke, s);
      spattn::launch_f32_to_bf16(static_cast<char*>(dv.data) + r0 * ke * 2, dva.as<float>() + r0 * ke, 1.f,
                                 (r1 - r0) * ke, s);
    }
    check_launch();
    if (hooks.after_bwd_chunk) hooks.after_bwd_chunk(static_cast<int>(c), r0, r1);
  }
  ctx.add_flops(10 * d * pairs * H);
}


// ========================================================================= kernel-level API
void block_forward_merge(cudaStream_t s, int64_t bs, int heads, int kv_heads, int dim,
                         const void* q, const std::vector<int64_t>& qpos, const void* k,
                         const void* v, const std::vector<int64_t>& kpos, bool causal,
                         double scale, float* acc_out, float* acc_lse, int64_t* pairs) {
  if (heads % kv_heads) throw ConfigError("block_forward: heads not a multiple of kv_heads");
  const int64_t lq = static_cast<int64_t>(qpos.size()), lk = static_cast<int64_t>(kpos.size());
  auto probs = make_problems(position_runs(qpos), position_runs(kpos), causal, bs, lq, lk, nullptr, pairs);
  if (pairs) *pairs *= heads;
  spattn::FwdArgs a{};
  a.q = q, a.k = k, a.v = v, a.o = nullptr, a.acc_o = acc_out, a.lse = acc_lse;
  a.q_row_stride = static_cast<int64_t>(heads) * dim;
  a.kv_row_stride = static_cast<int64_t>(kv_heads) * dim;
  a.o_row_stride = a.q_row_stride;
  a.lse_row_stride = heads;
  a.d = dim;
  a.scale = static_cast<float>(scale);
  a.hm = {heads, kv_heads, 0, 0, heads / kv_heads};
  if (!probs.empty()) attention_forward(s, a, probs, true);
}

void block_finalize(cudaStream_t s, int64_t rows, int dim, const float* acc_out, void* out_bf16) {
  spattn::launch_f32_to_bf16(out_bf16, acc_out, 1.f, rows * dim, s);
  check_launch();
}

void block_backward(cudaStream_t s, int64_t bs, int heads, int kv_heads, int dim, const void* q,
                    const std::vector<int64_t>& qpos, const void* k, const void* v,
                    const std::vector<int64_t>& kpos, bool causal, double scale, const void* out,
                    const float* lse, const void* dout, float* dq, float* dk, float* dv,
                    int64_t* pairs) {
  if (heads % kv_heads) throw ConfigError("block_backward: heads not a multiple of kv_heads");
  const int64_t lq = static_cast<int64_t>(qpos.size()), lk = static_cast<int64_t>(kpos.size());
  auto probs = make_problems(position_runs(qpos), position_runs(kpos), causal, bs, lq, lk, nullptr, pairs);
  if (pairs) *pairs *= heads;
  spattn::BwdArgs a{};
  DevBuf delta(static_cast<size_t>(bs * lq * heads * 4), s);
  a.q = q, a.k = k, a.v = v, a.o = out, a.dout = dout, a.lse = lse, a.delta = delta.as<float>();
  a.dq_acc = dq, a.dk_acc = dk, a.dv_acc = dv;
  a.q_row_stride = static_cast<int64_t>(heads) * dim;
  a.kv_row_stride = static_cast<int64_t>(kv_heads) * dim;
  a.o_row_stride = a.q_row_stride;
  a.dq_row_stride = a.q_row_stride;
  a.dkv_row_stride = a.kv_row_stride;
  a.lse_row_stride = heads;
  a.d = dim;
  a.scale = static_cast<float>(scale);
  a.hm = {heads, kv_heads, 0, 0, heads / kv_heads};
  spattn::launch_attn_bwd_pre(a, static_cast<int>(bs * lq), s);
  check_launch();
  if (!probs.empty()) attention_backward(s, a, probs);
}

void all_to_all(RankCtx& ctx, const CommGroup& group, const void* local, int64_t bs, int64_t len,
                int64_t heads, int64_t dim, int elem_bytes, int scatter_dim, int gather_dim,
                void* out) {
  const int G = group.size();
  const int me = group.index_of(ctx.rank);
  (void)me;
  MoveSpec m;
  m.bs = bs;
  m.elem = elem_bytes;
  if (scatter_dim == 2 && gather_dim == 1) {
    if (heads % G) throw ShapeError("all_to_all: extent " + std::to_string(heads) + " of axis 2 not divisible by group size " + std::to_string(G));
    const int64_t hn = heads / G;
    m.lloc = len, m.lg = len * G, m.xw = heads * dim;
    for (int j = 0; j < G; ++j) {
      m.win.push_back({j * hn * dim, 0, hn * dim, 0});
      m.yw.push_back(hn * dim);
      m.runs.push_back({{0, j * len, len}});
    }
    move_forward(ctx, group, m, local, out, ctx.stream);
  } else if (scatter_dim == 1 && gather_dim == 2) {
    if (len % G) throw ShapeError("all_to_all: extent " + std::to_string(len) + " of axis 1 not divisible by group size " + std::to_string(G));
    const int64_t lo = len / G;
    m.lloc = lo, m.lg = len, m.xw = heads * dim * G;
    for (int j = 0; j < G; ++j) {
      m.win.push_back({j * heads * dim, 0, heads * dim, 0});
      m.yw.push_back(heads * dim);
      m.runs.push_back({{0, j * lo, lo}});
    }
    move_reverse(ctx, group, m, local, out, false, ctx.stream);
  } else {
    throw ConfigError("all_to_all: only (scatter 2, gather 1) and (scatter 1, gather 2) are supported");
  }
}

void all_gather(RankCtx& ctx, const CommGroup& group, const void* local, int64_t outer, int64_t extent,
                int64_t inner_bytes, void* out) {
  if (outer < 0 || extent < 0 || inner_bytes < 0) throw ShapeError("all_gather: negative extent");
  const int G = group.size(), me = group.index_of(ctx.rank);
  const int64_t blk = extent * inner_bytes, local_bytes = outer * blk;
  ctx.count(Primitive::all_gather, local_bytes * (G - 1));
  cudaStream_t s = ctx.stream;
  if (local_bytes == 0) return;
  // member j's [outer, blk] block lands at byte column j * blk of out's [outer, G * blk] rows
  auto place = [&](int j, const void* src, std::vector<CopyTask>& t) {
    t.push_back({src, out, blk, G * blk, 0, 0, 0, j * blk, outer, blk, 0});
  };
  if (G == 1 || ctx.transport->peer_access()) {
    std::vector<void*> ptrs{const_cast<void*>(local)};
    if (G > 1) ptrs = ctx.transport->exchange_ptrs(group, ctx.rank, const_cast<void*>(local), s);
    std::vector<CopyTask> tasks;
    for (int j = 0; j < G; ++j) place(j, ptrs[static_cast<size_t>(j)], tasks);
    run_tasks(tasks, 1, false, s);
    if (G > 1) ctx.transport->release(group, ctx.rank, s);
    return;
  }
  // messages: my block to every member; a member's block is received in place when out's
  // rows are a single slice (outer == 1), else staged and placed
  DevBuf rbuf(outer == 1 ? 0 : static_cast<size_t>(G * local_bytes), s);
  std::vector<Msg> sends, recvs;
  for (int j = 0; j < G; ++j) {
    sends.push_back({j, const_cast<void*>(local), static_cast<size_t>(local_bytes)});
    char* dst = outer == 1 ? static_cast<char*>(out) + j * blk : static_cast<char*>(rbuf.p) + j * local_bytes;
    recvs.push_back({j, dst, static_cast<size_t>(local_bytes)});
  }
  ctx.transport->send_recv(group, ctx.rank, sends, recvs, s);
  if (outer > 1) {
    std::vector<CopyTask> tasks;
    for (int j = 0; j < G; ++j) place(j, static_cast<char*>(rbuf.p) + j * local_bytes, tasks);
    run_tasks(tasks, 1, false, s);
  }
  (void)me;
}

// all_gather's backward exchange (comm.cpp:415-443): member i receives block i of every member's
// gathered gradient (one all-to-all of [outer, G*extent] rows viewed as heads), counted as the
// reference counts it: a second all_gather at gather volume (comm.cpp:418-420).
void all_gather_backward(RankCtx& ctx, const CommGroup& group, const void* grad_gathered, int64_t outer,
                         int64_t extent, int64_t inner_bytes, void* parts) {
  if (outer < 0 || extent < 0 || inner_bytes < 0) throw ShapeError("all_gather: negative extent");
  const int G = group.size();
  const auto before = ctx.stats[static_cast<int>(Primitive::all_to_all)];
  all_to_all(ctx, group, grad_gathered, 1, outer, G * extent, inner_bytes, 1, 2, 1, parts);
  // the exchange above counted itself as an all_to_all; book it under all_gather instead
  ctx.stats[static_cast<int>(Primitive::all_to_all)] = before;
  ctx.count(Primitive::all_gather, outer * extent * inner_bytes * (G - 1));
}

void ring_shift(RankCtx& ctx, const CommGroup& group, const void* payload, int64_t bytes, void* out) {
  if (bytes < 0) throw ShapeError("ring_shift: negative size");
  const int G = group.size(), me = group.index_of(ctx.rank);
  ctx.count(Primitive::p2p, G == 1 ? 0 : bytes);
  cudaStream_t s = ctx.stream;
  if (bytes == 0) return;
  const int from = (me - 1 + G) % G, to = (me + 1) % G;
  if (G == 1 || ctx.transport->peer_access()) {
    std::vector<void*> ptrs{const_cast<void*>(payload)};
    if (G > 1) ptrs = ctx.transport->exchange_ptrs(group, ctx.rank, const_cast<void*>(payload), s);
    if (out != ptrs[static_cast<size_t>(from)])
      SP_CUDA(cudaMemcpyAsync(out, ptrs[static_cast<size_t>(from)], static_cast<size_t>(bytes),
                              cudaMemcpyDeviceToDevice, s));
    if (G > 1) ctx.transport->release(group, ctx.rank, s);
    return;
  }
  ctx.transport->send_recv(group, ctx.rank, {{to, const_cast<void*>(payload), static_cast<size_t>(bytes)}},
                           {{from, out, static_cast<size_t>(bytes)}}, s);
}

}  // namespace seqpar
