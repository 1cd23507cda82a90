// B200 mirror of the reference attention-engine API
// (/root/reference/proj/include/seqpar/attention.hpp). Same engine names, AttentionConfig
// fields and error behaviour; tensors are device views (bf16, [bs, len, heads, dim]
// contiguous) and the tape node becomes an explicit forward -> SavedState -> backward pair.
#pragma once
#include <cuda_runtime.h>

#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "seqpar/comm.hpp"
#include "seqpar/partition.hpp"

namespace seqpar {

enum class Engine { oracle, ulysses, dummy_head, xtuner, ring, usp };  // attention.hpp:14
const char* engine_name(Engine e);
Engine engine_from_string(const std::string& s);

struct AttentionConfig {  // attention.hpp:19-26
  int heads = 1;
  int kv_heads = 0;  // 0 = heads
  int head_dim = 1;
  bool causal = true;
  int ulysses_degree = 0;  // usp only
  int ring_degree = 0;     // usp only
};

// Non-owning device view of a [bs, len, heads, dim] bf16 tensor, contiguous.
struct DeviceTensor {
  void* data = nullptr;
  int64_t bs = 0, len = 0, heads = 0, dim = 0;
  int64_t numel() const { return bs * len * heads * dim; }
};

// Everything the backward needs (the reference's tape closure captures, attention.cpp:236-258).
// Owns the engine's device workspace; q/k/v/out views must stay valid until backward.
struct SavedState;
void saved_state_free(SavedState* s);
struct SavedDeleter {
  void operator()(SavedState* s) const { saved_state_free(s); }
};
using SavedPtr = std::unique_ptr<SavedState, SavedDeleter>;

// Neat-packed documents (varlen): consecutive global positions [0, L) are cut into documents
// of these lengths; a query only sees keys of its own document (causal by global index).
// Empty = one document. The reference has no varlen path; the composed oracle runs
// oracle_attention per document.
struct Documents {
  std::vector<int64_t> lengths;
};

// Rotary embedding of q and k ahead of attention (Model::forward's rope_apply calls,
// model.cpp:342-343) with the caller's GLOBAL position ids of its local rows — a local 0-based
// range corrupts the rotary phases when sp > 1 (model.cpp:313-318, the paper's §5.2 pitfall).
struct Rope {
  std::vector<int64_t> position_ids;  // local_len entries
  double base = 10000.0;              // kRopeBase (tensor.hpp:141-144)
};

// attention.hpp:90-92. q [bs, local_len, heads, dim], k/v [bs, local_len, kv_heads, dim];
// out has q's shape; lse (optional) is [bs, local_len, heads] fp32 natural log. With `rope`,
// q and k are rotated first (fused into the all-to-all copy for Ulysses / Dummy-Head / USP) and
// the backward returns gradients with respect to the unrotated q and k.
SavedPtr run_attention_engine(RankCtx& ctx, Engine engine, const AttentionConfig& cfg,
                              const ShardLayout& layout, const DeviceTensor& q,
                              const DeviceTensor& k, const DeviceTensor& v,
                              const DeviceTensor& out, float* lse,
                              const Documents* docs = nullptr, const Rope* rope = nullptr);

// The tape node's backward: dq/dk/dv are written (not accumulated) in q/k/v's layouts.
void run_attention_engine_backward(RankCtx& ctx, SavedState& saved, const DeviceTensor& dout,
                                   const DeviceTensor& dq, const DeviceTensor& dk,
                                   const DeviceTensor& dv);

// One fwd+bwd step of the layer on HOST buffers (host_step.cpp): the reference's
// run_attention_engine + tape.backward on host tensors, with the H2D / D2H traffic of
// independent kv-head groups overlapped with compute. All buffers are [bs, local_len, heads,
// dim] bf16 (lse fp32 [bs, local_len, heads]); out / lse may be null. groups <= 0 picks the
// largest of 8, 4, 2, 1 the engine's head constraints allow — for a multi-rank ring, the
// largest whose step kernels still fill the GPU (pick_step_groups).
void run_attention_step_host(RankCtx& ctx, Engine engine, const AttentionConfig& cfg,
                             const ShardLayout& layout, int64_t bs, const void* hq, const void* hk,
                             const void* hv, const void* hdout, void* hout, float* hlse, void* hdq,
                             void* hdk, void* hdv, const Documents* docs, int groups);
int pick_step_groups(Engine e, const AttentionConfig& cfg, int sp, int64_t local_len = 0);

// Library-internal (host_step.cpp): the single-device causal step (sp = 1, bs = 1, one
// document) cut along the sequence, so a host pipeline can start computing on the first rows
// that arrived and copy out the first rows that are final. Forward chunk c covers query rows
// [r0, r1) against keys [0, r1) and is issued after before_fwd_chunk(c, r1); backward chunk c
// covers keys [r0, r1) against queries [r0, L) — afterwards dq / dk / dv rows [r0, r1) are final
// (bf16) and after_bwd_chunk(c, r0, r1) runs. Same math as run_attention_engine + backward.
struct SequenceChunks {
  int fwd_chunks = 4, bwd_chunks = 4;
  std::function<void(int, int64_t)> before_fwd_chunk;
  std::function<void()> before_backward;
  std::function<void(int, int64_t, int64_t)> after_bwd_chunk;
};
bool single_step_chunkable(RankCtx& ctx, Engine e, const AttentionConfig& cfg, const ShardLayout& layout,
                           int64_t bs, const Documents* docs);
void run_single_step_chunked(RankCtx& ctx, Engine e, const AttentionConfig& cfg, const ShardLayout& layout,
                             const DeviceTensor& q, const DeviceTensor& k, const DeviceTensor& v,
                             const DeviceTensor& out, float* lse, const DeviceTensor& dout,
                             const DeviceTensor& dq, const DeviceTensor& dk, const DeviceTensor& dv,
                             const SequenceChunks& hooks);

// rope_apply (tensor.cpp:548-607) on a bf16 [bs, len, heads, dim] device tensor (inverse:
// the backward's rotation, tensor.cpp:589-600); out may alias x.
void rope_apply(cudaStream_t s, int64_t bs, int64_t len, int64_t heads, int dim, const void* x,
                const std::vector<int64_t>& position_ids, double base, bool inverse, void* out);

// A view shaped like the forward's q (which=0) or k/v (which=1) over `data`.
DeviceTensor saved_view(const SavedState& s, int which, void* data);

// ---- kernel-level API (attention.hpp:43-66) on device buffers ----
// attn_block_forward + merge_piece fused: merges the block's piece into the running fp32
// accumulator (acc_out [bs, lq, heads, dim], acc_lse [bs, lq, heads]; lse = -inf marks an empty
// row). finalize_piece is block_finalize. Positions are host int64 lists (run-structured).
void block_forward_merge(cudaStream_t s, int64_t bs, int heads, int kv_heads, int dim,
                         const void* q, const std::vector<int64_t>& qpos, const void* k,
                         const void* v, const std::vector<int64_t>& kpos, bool causal,
                         double scale, float* acc_out, float* acc_lse, int64_t* pairs = nullptr);
void block_finalize(cudaStream_t s, int64_t rows, int dim, const float* acc_out, void* out_bf16);
// attn_block_backward: += into fp32 dq [bs,lq,heads,dim], dk/dv [bs,lk,kv_heads,dim].
void block_backward(cudaStream_t s, int64_t bs, int heads, int kv_heads, int dim, const void* q,
                    const std::vector<int64_t>& qpos, const void* k, const void* v,
                    const std::vector<int64_t>& kpos, bool causal, double scale, const void* out,
                    const float* lse, const void* dout, float* dq, float* dk, float* dv,
                    int64_t* pairs = nullptr);

// Reference all_to_all (comm.cpp:357-379) on a [bs, len, heads, dim] tensor of any element
// size: scatter_dim/gather_dim in {1, 2}. out shape follows the reference.
void all_to_all(RankCtx& ctx, const CommGroup& group, const void* local, int64_t bs, int64_t len,
                int64_t heads, int64_t dim, int elem_bytes, int scatter_dim, int gather_dim,
                void* out);

// Reference all_gather (comm.cpp:381-447) along one axis of a tensor viewed as
// [outer, extent, inner_bytes]: out = [outer, G * extent, inner_bytes] with member j's block at
// [j * extent, (j + 1) * extent) of every outer slice (group order). Every member passes the
// same outer / extent / inner_bytes (the reference's extent check outside the axis). Counted
// as one all_gather of local_bytes * (G - 1).
void all_gather(RankCtx& ctx, const CommGroup& group, const void* local, int64_t outer, int64_t extent,
                int64_t inner_bytes, void* out);
// Backward exchange of all_gather (comm.cpp:415-443): parts [G, outer, extent, inner_bytes],
// part j = member j's gathered gradient at this member's block (the caller tree-sums them in
// group order). Counted as a second all_gather of local_bytes * (G - 1) (comm.cpp:418-420).
void all_gather_backward(RankCtx& ctx, const CommGroup& group, const void* grad_gathered, int64_t outer,
                         int64_t extent, int64_t inner_bytes, void* parts);

// Reference ring_shift (comm.cpp:449-460): group index i receives the payload of index i-1
// (`bytes` on every member). Counted as one p2p of `bytes` (0 for a single member).
void ring_shift(RankCtx& ctx, const CommGroup& group, const void* payload, int64_t bytes, void* out);

// Event timing of the attention kernels (bench.py): ms[0]/n[0] forward, ms[1]/n[1] backward.
void profile_enable(bool on);
void profile_read(double* ms, int64_t* n);
// Ring-step stream timeline (spattn_debug_timeline): kind 0 fwd kernel, 1 bwd kernel, 2 k|v hop,
// 3 dk|dv add, 4 dk|dv hop; times in ms relative to the enable call.
void timeline_enable(bool on);
int64_t timeline_read(double* start_ms, double* end_ms, int* kind, int* rank, int max);

// Host planners behind the engines (exported for multi-process tests of the N>1 logic):
// per-member query/kv head windows of the head<->sequence moves, and the problem list
// (q_row0, nq, k_row0, nk, off, causal) two position lists reduce to.
void plan_head_windows(int heads, int kv_heads, int group, std::vector<int>& qlo,
                       std::vector<int>& qn, std::vector<int>& kvlo, std::vector<int>& kvn);
std::vector<std::array<int, 6>> plan_problems(const std::vector<int64_t>& qpos,
                                              const std::vector<int64_t>& kpos, bool causal,
                                              const Documents* docs, int64_t* pairs);

// Which attention kernel family the engines launch.
// tcgen05_pp: two-tile ping-pong forward; tcgen05_pair: CTA-pair (cta_group::2) forward for d=128;
// tcgen05_q64: the 64-query-tile backward (attn_bwd_tc.cu) also for d=128, where the default
// family runs the 128-query-tile backward (attn_bwd_q128.cu)
enum class KernelFamily { tcgen05, mma, tcgen05_pp, tcgen05_pair, tcgen05_q64 };
void set_kernel_family(KernelFamily f);
KernelFamily kernel_family();

}  // namespace seqpar
