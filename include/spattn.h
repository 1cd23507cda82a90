/* spattn — C ABI of the B200 sequence-parallel attention layer (libspattn.so).
 *
 * Drop-in boundary for the reference's SP attention path
 * (/root/reference/proj, C++20 library `seqpar`). Every entry point replaces one reference
 * interface, cited below; INTEGRATION.md shows the binding a maintainer adds on the reference
 * side. Plain pointers and sizes only: device buffers are bf16 [bs, len, heads, dim]
 * contiguous (lse fp32 [bs, len, heads], natural log). Exceptions never cross this boundary:
 * every call returns a status and spattn_last_error() (thread-local) holds the message —
 * the reference throws ConfigError / ShapeError / StateError (tensor.hpp:18-26) and its
 * Python module maps them to ValueError (py_module.cpp:320-321).
 */
#ifndef SPATTN_H
#define SPATTN_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SPATTN_OK = 0,
  SPATTN_ERR_CONFIG = 1, /* seqpar::ConfigError */
  SPATTN_ERR_SHAPE = 2,  /* seqpar::ShapeError */
  SPATTN_ERR_STATE = 3,  /* seqpar::StateError, CUDA and NCCL failures */
  SPATTN_ERR_PEER = 4    /* a peer rank failed (CommFabric PeerAbort, comm.cpp:10-14) */
};

/* Engine (attention.hpp:14) and SplitMode (partition.hpp:14) enumerations, same order. */
enum { SPATTN_ORACLE = 0, SPATTN_ULYSSES, SPATTN_DUMMY_HEAD, SPATTN_XTUNER, SPATTN_RING, SPATTN_USP };
enum { SPATTN_NAIVE = 0, SPATTN_ZIGZAG, SPATTN_SPLIT_USP,
       /* extension (no reference counterpart): ShardLayout::make_zigzag_blocks with the block
          count in u_degree — zigzag within each of u_degree equal blocks (mode zigzag) */
       SPATTN_ZIGZAG_BLOCKS };
/* Primitive (comm.hpp:19) */
enum { SPATTN_ALL_TO_ALL = 0, SPATTN_ALL_GATHER, SPATTN_P2P, SPATTN_ALL_REDUCE, SPATTN_BROADCAST };

/* AttentionConfig (attention.hpp:19-26) */
typedef struct {
  int32_t heads, kv_heads, head_dim, causal, ulysses_degree, ring_degree;
} spattn_config;

/* ShardLayout::make_naive / make_zigzag / make_usp arguments (partition.hpp:29-31) */
typedef struct {
  int32_t mode, sp;
  int64_t global_len;
  int32_t u_degree, r_degree;
} spattn_layout;

typedef struct spattn_ctx spattn_ctx;       /* RankCtx (comm.hpp:63-82): one per rank */
typedef struct spattn_fabric spattn_fabric; /* CommFabric (comm.hpp:86-140): loopback ranks */
typedef struct spattn_saved spattn_saved;   /* the tape closure's captures (attention.cpp:236-258) */

const char* spattn_last_error(void);
int spattn_abi_version(void);

/* ---- partition / report host functions (pure integer, no GPU) ---- */
/* ShardLayout::positions_of (partition.cpp:105-111); out holds global_len/sp entries */
int spattn_layout_positions(const spattn_layout* layout, int index, int64_t* out);
/* causal_pair_count (partition.cpp:118-122) */
int spattn_causal_pairs(const spattn_layout* layout, int index, int64_t* out);
/* pad_length (partition.cpp:179-200) */
int spattn_pad_length(int64_t len, int sp, int64_t cutoff_len, int pad_to_cutoff, int64_t* out);
/* pick_xtuner_insp (attention.cpp:354-366) */
int spattn_pick_xtuner_insp(int heads, int sp, int head_dim, int* out);
/* ulysses/ring/dummy_head/xtuner/usp_bytes (report.cpp:906-941), reference accounting */
int spattn_reference_bytes(int engine, int64_t bs, int64_t len, int64_t heads, int64_t head_dim,
                           int sp, int u, int r, int64_t* out);

/* ---- batches, padding and neat-packing metadata (partition.hpp:92-125) ---- */
/* pad_batch (partition.cpp:202-215): every field extended to *out_len = pad_length(len, sp,
 * cutoff_len, pad_to_cutoff) entries with its sentinel (pad_token, -100, iota, -1, -1).
 * segment_ids / image_map may be NULL (then their outputs are untouched); out arrays hold
 * *out_len entries (query pad_length first). */
int spattn_pad_batch(const int64_t* tokens, const int64_t* labels, const int64_t* position_ids,
                     const int64_t* segment_ids, const int64_t* image_map, int64_t len, int sp,
                     int64_t pad_token, int64_t cutoff_len, int pad_to_cutoff, int64_t* out_len,
                     int64_t* out_tokens, int64_t* out_labels, int64_t* out_position_ids,
                     int64_t* out_segment_ids, int64_t* out_image_map);
/* split_position_map / shard (partition.cpp:217-220, :124-139) of a per-position int64 field:
 * out holds global_len/sp entries */
int spattn_split_position_map(const spattn_layout* layout, int index, const int64_t* values,
                              int64_t* out);
/* Neat-packing bridge to the varlen kernels: runs of equal segment ids -> document lengths
 * (a -1 padding tail is one more document); ConfigError when an id is not one run. */
int spattn_documents_from_segments(const int64_t* segment_ids, int64_t len, int64_t* doc_lens,
                                   int max_docs, int* n_docs);
/* broadcast_bytes (comm.hpp:159-161, comm.cpp:526-545) over a context's SP group: the bytes of
 * global rank `root` reach every member (members pass any payload); the result (at most `cap`
 * bytes) lands in out, its length in out_len. Counted as len*(g-1)/g. CONFIG error when root is
 * not in the group. */
int spattn_broadcast_bytes(spattn_ctx* ctx, const uint8_t* payload, int64_t len, int root, uint8_t* out,
                           int64_t cap, int64_t* out_len);
/* replicate_packing_mask (partition.cpp:222-227): group index 0's bytes to every member over
 * the context's transport; out holds cap bytes, *out_len receives the mask length. */
int spattn_replicate_packing_mask(spattn_ctx* ctx, const uint8_t* mask, int64_t len, uint8_t* out,
                                  int64_t cap, int64_t* out_len);
int spattn_fabric_replicate_packing_mask(spattn_fabric* f, const uint8_t* const* masks,
                                         const int64_t* lens, uint8_t* const* outs, int64_t cap,
                                         int64_t* out_lens);

/* ---- the step after the model: log-probs and sharded loss reductions (losses.cpp) ---- */
/* sequence_logprob_per_position (losses.cpp:20-72): logits [T, V] of dtype 0 fp32 / 1 bf16 /
 * 2 fp64,
 * device labels [T] int64 (-100 = ignored); out / lse device fp64 [T]. */
int spattn_logprob_fwd(void* stream, const void* logits, int dtype, int64_t T, int64_t V,
                       const int64_t* labels, double* out, double* lse);
/* its tape backward: dlogits (= or +=) g_t * (onehot(label_t) - softmax(row_t)) */
int spattn_logprob_bwd(void* stream, const void* logits, int dtype, int64_t T, int64_t V,
                       const int64_t* labels, const double* lse, const double* g, void* dlogits,
                       int accumulate);
/* ExactSum (exact_sum.hpp): 35 uint64 limbs, 2240-bit two's complement in units of 2^-1074.
 * _device adds n device doubles, _host n host doubles; limbs accumulate (+=). */
int spattn_exact_sum_device(void* stream, const double* values, int64_t n, uint64_t* limbs);
int spattn_exact_sum_host(const double* values, int64_t n, uint64_t* limbs);
int spattn_exact_merge(uint64_t* acc, const uint64_t* other);
int spattn_exact_round(const uint64_t* limbs, double* out);
/* group reductions of the context's SP group (comm.cpp:339-353, :504-524), in place */
int spattn_exact_sum_all_reduce(spattn_ctx* ctx, uint64_t* limbs);
int spattn_all_reduce_count(spattn_ctx* ctx, int64_t* n);
int spattn_all_reduce_values(spattn_ctx* ctx, double* values, int64_t n);

/* Host planners of the engines (no GPU): per-member head windows of the Ulysses
 * head<->sequence moves (query heads [q_lo, q_lo+q_n), kv heads [kv_lo, kv_lo+kv_n); dummy
 * heads are virtual), and the attention problems two position lists reduce to: rows of 6
 * int32 (q_row0, nq, k_row0, nk, off, causal) where key c is admitted for query a iff
 * !causal || c <= a + off — the kpos <= qpos rule of attention.cpp:89. */
int spattn_plan_heads(int heads, int kv_heads, int group, int32_t* q_lo, int32_t* q_n,
                      int32_t* kv_lo, int32_t* kv_n);
int spattn_plan_problems(const int64_t* qpos, int64_t lq, const int64_t* kpos, int64_t lk,
                         int causal, const int64_t* doc_lens, int n_docs, int32_t* out,
                         int max_problems, int* n_problems, int64_t* pairs);

/* ---- contexts ---- */
/* NCCL backend: one process per GPU. rank 0 creates the id, the launcher broadcasts it. */
int spattn_nccl_unique_id(uint8_t out[128]);
int spattn_ctx_create_nccl(int device, int rank, int world, int sp, const uint8_t unique_id[128],
                           spattn_ctx** out);
int spattn_ctx_destroy(spattn_ctx* ctx);
/* Diagnostics, collective over the context's transport: `bytes` sent by this rank to itself
 * through every transport entry point (NCCL: CommSplit, grouped Send/Recv on the split and the
 * world communicator, CommDestroy; loopback: send_recv). 0 when the bytes arrive intact. */
int spattn_debug_transport_selftest(spattn_ctx* ctx, int64_t bytes);
/* Loopback fabric: `world` ranks as threads sharing one device (CommFabric::run analog).
 * force_messages=1 routes collectives through the pack -> send/recv -> unpack path. */
int spattn_fabric_create(int device, int world, int sp, int force_messages, spattn_fabric** out);
int spattn_fabric_destroy(spattn_fabric* f);
int spattn_fabric_ctx(spattn_fabric* f, int rank, spattn_ctx** out);
/* Compute stream of a context (cudaStream_t; 0 is the legacy default stream). */
int spattn_ctx_set_stream(spattn_ctx* ctx, void* stream);
int spattn_ctx_stream(spattn_ctx* ctx, void** stream);
/* send-side per-primitive counters (PrimitiveStats, comm.hpp:30-33) and flop counter */
int spattn_ctx_stats(spattn_ctx* ctx, int primitive, int64_t* calls, int64_t* bytes);
int spattn_ctx_flops(spattn_ctx* ctx, int64_t* flops);
int spattn_ctx_reset_stats(spattn_ctx* ctx);
/* 0 = tcgen05/TMEM kernels (default where supported), 1 = mma.sync kernels,
 * 2 = tcgen05 with the two-tile ping-pong forward, 3 = tcgen05 with the CTA-pair
 * (cta_group::2, M=256) forward for head_dim 128, 4 = tcgen05 with the 64-query-tile
 * backward for head_dim 128 too (the default runs the 128-query-tile backward there) */
int spattn_set_kernel_family(int family);
int spattn_get_kernel_family(void);

/* Diagnostics for the bench: number of kernels this library has launched, and CUDA-event
 * timing of the attention kernels (fwd: ms[0], n[0]; bwd: ms[1], n[1]) since enabling. */
int64_t spattn_launch_count(void);
/* Profiling: per-iteration clock64 event trace of backward CTA (0,0) into a device buffer of
 * 16 int64 per iteration (NULL disables). */
int spattn_debug_bwd_trace(void* device_buffer);
/* Profiling: per-CTA globaltimer records of the forward kernel, 8 int64 per CTA (blockIdx.y-major):
 * entry, first S in TMEM, main-loop end, exit (ns), n_tiles, smid (NULL disables). */
int spattn_debug_fwd_cta_trace(void* device_buffer);
int spattn_profile_enable(int on);
int spattn_profile_read(double ms[2], int64_t n[2]);
/* Profiling: stream timeline of the ring engines. While on, every ring step records CUDA events
 * around its attention kernel (kind 0 forward, 1 backward), its k|v hop (2), the dk|dv partial-sum
 * add (3) and the dk|dv hop (4), tagged with the rank. Read returns up to `max` records as start /
 * end ms relative to the enable call, plus kind and rank; *n = records available. */
int spattn_debug_timeline(int on);
int spattn_debug_timeline_read(double* start_ms, double* end_ms, int* kind, int* rank, int max, int64_t* n);

/* Descriptor self-test of the tcgen05 path: d1 = a . b^T, d2 = a . b_mn (smem operands) and
 * d3 = a . b_mn with a read from TMEM, for 128x128 bf16 row-major tiles through TMA +
 * tcgen05.mma + TMEM (fp32 outputs, 128x128; d3 may be NULL). */
int spattn_selftest_umma(void* stream, const void* a, const void* b, const void* b_mn, float* d1,
                         float* d2, float* d3);

/* ---- engine: run_attention_engine (attention.hpp:90-92) + its tape backward ----
 * Collective over the SP group: every rank calls with its shard. q [bs, local_len, heads, d],
 * k/v [bs, local_len, kv_heads, d], out like q, lse optional. doc_lens (optional, n_docs>0)
 * cuts the global sequence into neat-packed documents (varlen). *saved must be released with
 * spattn_saved_free; q/k/v/out (and lse when given) must stay valid until spattn_bwd.
 * Stream-ordered on the context's compute stream. */
int spattn_fwd(spattn_ctx* ctx, int engine, const spattn_config* cfg, const spattn_layout* layout,
               int64_t bs, const void* q, const void* k, const void* v, void* out, float* lse,
               const int64_t* doc_lens, int n_docs, spattn_saved** saved);
/* spattn_fwd preceded by rope_apply of q and k (Model::forward, model.cpp:342-343; rope_apply,
 * tensor.cpp:548-607) with the caller's GLOBAL position ids of its local rows (host, local_len
 * entries; base = kRopeBase 10000, tensor.hpp:141-144). Ulysses / Dummy-Head / USP rotate
 * inside the all-to-all copy; spattn_bwd then returns dq, dk of the UNROTATED q, k. */
int spattn_fwd_rope(spattn_ctx* ctx, int engine, const spattn_config* cfg,
                    const spattn_layout* layout, int64_t bs, const void* q, const void* k,
                    const void* v, void* out, float* lse, const int64_t* doc_lens, int n_docs,
                    const int64_t* position_ids, double rope_base, spattn_saved** saved);
int spattn_bwd(spattn_ctx* ctx, spattn_saved* saved, const void* dout, void* dq, void* dk,
               void* dv);
void spattn_saved_free(spattn_saved* saved);

/* One training step (fwd + bwd) of the layer on HOST buffers (pinned for full overlap):
 * run_attention_engine + the tape backward on host tensors, as the reference runs them
 * (attention.cpp:526-574). The step is pipelined over `groups` independent kv-head groups
 * (0 = auto) so the H2D of q/k/v/dout and the D2H of dq/dk/dv overlap the attention kernels.
 * Shapes as spattn_fwd; out and lse may be NULL. Returns when the host results are written. */
int spattn_step_host(spattn_ctx* ctx, int engine, const spattn_config* cfg,
                     const spattn_layout* layout, int64_t bs, const void* q, const void* k,
                     const void* v, const void* dout, void* out, float* lse, void* dq, void* dk,
                     void* dv, const int64_t* doc_lens, int n_docs, int groups);

/* The head-group count spattn_step_host uses when groups = 0 (without the local length: the
 * head constraints only; with it: as spattn_step_host decides for a multi-rank ring). */
int spattn_pick_step_groups(int engine, const spattn_config* cfg, int sp);
int spattn_pick_step_groups_len(int engine, const spattn_config* cfg, int sp, int64_t local_len);

/* Loopback group drivers: one call runs every rank on its own thread (arrays of world
 * pointers), returning when all ranks' streams are idle. */
int spattn_fabric_fwd(spattn_fabric* f, int engine, const spattn_config* cfg,
                      const spattn_layout* layout, int64_t bs, const void* const* q,
                      const void* const* k, const void* const* v, void* const* out,
                      float* const* lse, const int64_t* doc_lens, int n_docs,
                      spattn_saved** saved);
int spattn_fabric_fwd_rope(spattn_fabric* f, int engine, const spattn_config* cfg,
                           const spattn_layout* layout, int64_t bs, const void* const* q,
                           const void* const* k, const void* const* v, void* const* out,
                           float* const* lse, const int64_t* doc_lens, int n_docs,
                           const int64_t* const* position_ids, double rope_base,
                           spattn_saved** saved);
int spattn_fabric_bwd(spattn_fabric* f, spattn_saved* const* saved, const void* const* dout,
                      void* const* dq, void* const* dk, void* const* dv);
/* all_to_all (comm.cpp:357-379) over a rank context's SP group (NCCL: every rank calls it);
 * device [bs, len, heads, dim] tensors of elem_bytes each, on the context's stream */
int spattn_all_to_all(spattn_ctx* ctx, const void* local, void* out, int64_t bs, int64_t len,
                      int64_t heads, int64_t dim, int elem_bytes, int scatter_dim, int gather_dim);
/* all_gather (comm.hpp:136, comm.cpp:381-447) over a rank context's SP group: the tensor is viewed
 * as [outer, extent, inner_bytes] around the gather axis; out [outer, G*extent, inner_bytes]
 * holds member j's block at [j*extent, (j+1)*extent) (group order). Every member passes the same
 * sizes. Counted as all_gather of local_bytes*(G-1). */
int spattn_all_gather(spattn_ctx* ctx, const void* local, void* out, int64_t outer, int64_t extent,
                      int64_t inner_bytes);
/* all_gather backward exchange (comm.cpp:415-443): gathered [outer, G*extent, inner_bytes]
 * gradient in; parts [G, outer, extent, inner_bytes] out, part j = member j's gradient at this
 * member's block (the caller tree-sums the parts in group order). Counted, as the reference
 * counts it (comm.cpp:418-420), as a second all_gather of local_bytes*(G-1). */
int spattn_all_gather_backward(spattn_ctx* ctx, const void* grad_gathered, void* parts, int64_t outer,
                               int64_t extent, int64_t inner_bytes);
/* ring_shift (comm.hpp:140, comm.cpp:449-460): group index i receives index i-1's payload of
 * `bytes` into out. Counted as one p2p of `bytes` (0 for a single member). */
int spattn_ring_shift(spattn_ctx* ctx, const void* payload, void* out, int64_t bytes);
/* all_to_all (comm.cpp:357-379) on [bs, len, heads, dim] tensors of elem_bytes each */
int spattn_fabric_all_to_all(spattn_fabric* f, const void* const* local, void* const* out,
                             int64_t bs, int64_t len, int64_t heads, int64_t dim, int elem_bytes,
                             int scatter_dim, int gather_dim);

/* ---- kernel-level API (attention.hpp:43-66) ---- */
/* attn_block_forward + merge_piece: merges into acc_out (fp32 [bs,lq,heads,dim]) / acc_lse
 * (fp32 [bs,lq,heads], -inf = empty row). Positions are host int64 arrays. */
int spattn_block_fwd(void* stream, int64_t bs, int heads, int kv_heads, int dim, const void* q,
                     const int64_t* qpos, int64_t lq, const void* k, const void* v,
                     const int64_t* kpos, int64_t lk, int causal, double scale, float* acc_out,
                     float* acc_lse, int64_t* pairs);
/* finalize_piece: bf16 out = acc_out (the accumulator is already normalised) */
int spattn_block_finalize(void* stream, int64_t rows, int dim, const float* acc_out, void* out);
/* merge_piece on finished pieces: acc <- LSE-merge(acc, piece) (fp32, warp per row) */
int spattn_lse_merge(void* stream, float* acc_out, float* acc_lse, const float* out,
                     const float* lse, int64_t rows, int dim);
/* attn_block_backward: += into fp32 dq [bs,lq,heads,dim], dk/dv [bs,lk,kv_heads,dim] */
int spattn_block_bwd(void* stream, int64_t bs, int heads, int kv_heads, int dim, const void* q,
                     const int64_t* qpos, int64_t lq, const void* k, const void* v,
                     const int64_t* kpos, int64_t lk, int causal, double scale, const void* out,
                     const float* lse, const void* dout, float* dq, float* dk, float* dv,
                     int64_t* pairs);
/* rope_apply (tensor.cpp:548-607) on bf16 [bs, len, heads, dim] device rows; position_ids is a
 * host array of len global ids; inverse=1 is the backward rotation (tensor.cpp:589-600);
 * out may alias x. */
int spattn_rope_apply(void* stream, int64_t bs, int64_t len, int heads, int dim, const void* x,
                      const int64_t* position_ids, double base, int inverse, void* out);
/* shard_rows / gather_rows (partition.cpp:124-158) on device rows of row_bytes each,
 * batched over bs: full [bs, L, row] <-> local [bs, L/sp, row] */
int spattn_shard_rows(void* stream, const spattn_layout* layout, int index, int64_t bs,
                      int64_t row_bytes, const void* full, void* local);
int spattn_gather_rows(void* stream, const spattn_layout* layout, int index, int64_t bs,
                       int64_t row_bytes, const void* local, void* full);

#ifdef __cplusplus
}
#endif
#endif
