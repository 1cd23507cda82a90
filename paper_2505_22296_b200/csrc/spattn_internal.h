// Internal kernel-launch interface between the C++ engines (engine.cpp) and the sm_100a
// kernels. Plain structs, device pointers, explicit streams.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace spattn {

// One rectangular attention problem in the flattened [rows, heads, dim] row space.
// Key c (0-based within the k run) is admitted for query a (0-based within the q run) iff
// !causal || c <= a + off. This is the reference's `kpos[j] <= qpos[i]` rule
// (attention.cpp:89) for contiguous position runs: off = qpos0 - kpos0.
struct AttnProblem {
  int q_row0, nq;
  int k_row0, nk;
  int off;
  int causal;
};

// Problems per launch. A problem set travels by value in the kernel parameters (CUDA 12.1+ allows
// 32764 bytes); 1000 problems keep every kernel's parameters (ProblemSet + args + up to seven
// 128-byte tensor maps) under that limit, enough for a neat-packed batch of hundreds of
// documents per launch (larger problem lists are split into several launches). The parameter
// block is copied at every launch, and 28 KB of it costs ~40 us of launch latency (measured at
// the c1 shape: 82 -> 45 us per forward launch), so every kernel is also instantiated for a
// 16-problem set, which launches with the one, two or few problems most calls carry.
#ifndef SPATTN_MAX_PROBLEMS
#define SPATTN_MAX_PROBLEMS 1000
#endif
constexpr int kMaxProblems = SPATTN_MAX_PROBLEMS;
constexpr int kSmallProblems = 16;

template <int CAP>
struct ProblemSetT {
  static constexpr int kCapacity = CAP;
  AttnProblem p[CAP];
  int tile_prefix[CAP + 1];  // cumulative q tiles (of the launching kernel's BLOCK_M)
  int n;
};
using ProblemSet = ProblemSetT<kMaxProblems>;
using SmallProblemSet = ProblemSetT<kSmallProblems>;
static_assert(sizeof(ProblemSet) + 7 * 128 + 512 <= 32764, "kernel parameter space");

// Copies the used part of a problem set (the n problems; the prefix is rebuilt by the launcher).
inline void copy_problems(ProblemSet& out, const ProblemSet& in) {
  out.n = in.n;
  for (int i = 0; i < in.n; ++i) out.p[i] = in.p[i];
}

// Calls f(set) with the smallest problem-set type that holds ps (its n problems and prefix).
template <class F>
void with_problem_set(const ProblemSet& ps, F&& f) {
  if (ps.n <= kSmallProblems) {
    SmallProblemSet sm;
    sm.n = ps.n;
    for (int i = 0; i < ps.n; ++i) sm.p[i] = ps.p[i];
    for (int i = 0; i <= ps.n; ++i) sm.tile_prefix[i] = ps.tile_prefix[i];
    f(sm);
  } else {
    f(ps);
  }
}

// Head mapping of a rank's local tensors: local q head h is global head q_head_base + h; it
// reads kv head (q_head_base + h) / rep - kv_head_base of the local kv tensor. This indexes
// GQA groups in place of repeat_heads (tensor.cpp:418-450).
struct HeadMap {
  int hq;            // local q heads computed
  int hkv;           // local kv heads stored
  int q_head_base;
  int kv_head_base;
  int rep;
};

struct FwdArgs {
  const void* q;  // bf16 [rows, q_heads_stride, d]
  const void* k;  // bf16 [rows_k, kv_heads_stride, d]
  const void* v;
  void* o;        // bf16 out (plain mode)
  float* lse;     // [rows, q_heads_stride] natural-log LSE
  float* acc_o;   // merge mode: fp32 [rows, q_heads_stride, d] running output (lse = running)
  int64_t q_row_stride, kv_row_stride, o_row_stride;  // elements between consecutive rows
  int lse_row_stride;                                 // floats between rows of lse
  int d;
  float scale;
  HeadMap hm;
};

struct BwdArgs {
  const void* q;
  const void* k;
  const void* v;
  const void* o;
  const void* dout;
  const float* lse;    // natural log
  float* delta;        // [rows, lse_row_stride] (filled by the preprocess kernel)
  float* dq_acc;       // fp32 [rows, q heads, d] (atomic)
  float* dk_acc;       // fp32 [rows_k, kv heads, d] (atomic)
  float* dv_acc;
  int64_t q_row_stride, kv_row_stride, o_row_stride;
  int64_t dq_row_stride, dkv_row_stride;  // fp32 accumulator row strides
  int lse_row_stride;
  int d;
  float scale;
  HeadMap hm;
  // optional: when every (key row, kv head) belongs to exactly one CTA of the launch (disjoint
  // key ranges), the tcgen05 kernel writes dK / dV as bf16 here instead of adding into dk_acc /
  // dv_acc (no zero fill, no atomics, no rounding pass); row stride in elements
  void* dk_bf16 = nullptr;
  void* dv_bf16 = nullptr;
  int64_t dkv_bf16_row_stride = 0;
  int debug;  // profiling switches (SPATTN_DEBUG env): 1 skip dQ atomics, 2 skip dK/dV atomics
  long long* trace;  // profiling: per-iteration clock64 events of CTA (0,0), or null
};

// Launch-side failures throw std::runtime_error (SPATTN_ERR_STATE at the C ABI): a TMA
// descriptor that does not encode or a failed shared-memory opt-in never leaves the outputs
// silently unwritten.
[[noreturn]] void launch_error(const char* kernel, const char* what);
// cudaFuncAttributeMaxDynamicSharedMemorySize for `kernel` on the CURRENT device, once per
// (kernel, device) pair (a process may drive several GPUs).
void ensure_smem(const void* kernel, int bytes);
template <class K>
void ensure_smem_for(K* kernel, int bytes) {
  ensure_smem(reinterpret_cast<const void*>(kernel), bytes);
}

// Launch accounting (bench.py's gpu_launches): every launcher in this library calls this.
void note_launch(int n = 1);
long long launch_count();

// ---- attention kernels (attn_mma.cu / attn_tc.cu) ----
void launch_attn_fwd(const FwdArgs& a, const ProblemSet& ps, cudaStream_t s);
void launch_attn_bwd_pre(const BwdArgs& a, int rows, cudaStream_t s);
void launch_attn_bwd(const BwdArgs& a, const ProblemSet& ps, cudaStream_t s);

// ---- element kernels (permute.cu) ----
// One row-run copy task of the fused pack/pad -> exchange -> unpack/unpad permutation.
// Copies `rows` rows: for r in [0, rows): dst[(dst_row0 + r) * dst_row_stride + dst_col0 ..]
// <- src[(src_row0 + r) * src_row_stride + src_col0 ..] for `cols` elements, and zero-fills
// the `zero_cols` elements that follow in dst (dummy-head padding). Strides in elements.
struct CopyTask {
  const void* src;
  void* dst;
  int64_t src_row_stride, dst_row_stride;
  int64_t src_row0, dst_row0;
  int64_t src_col0, dst_col0;
  int64_t rows, cols, zero_cols;
  // RoPE fused into the copy (rope_apply, tensor.cpp:548-607; rope.cu): bf16 payload of whole
  // heads of rope_dim columns, rotated by the float2(cos, sin) angle-table row
  // (rope_row0 + r) % rope_mod; rope_sign -1 applies the inverse rotation (the backward).
  const float2* rope = nullptr;
  int64_t rope_row0 = 0, rope_mod = 1;
  int rope_dim = 0, rope_sign = 1;
  // element size of this task in bytes (0: the launch's); tasks of different sizes share a launch
  // on the TMA copier (the warp copier splits them by size)
  int elem = 0;
};
#ifndef SPATTN_MAX_COPY_TASKS
#define SPATTN_MAX_COPY_TASKS 64
#endif
constexpr int kMaxCopyTasks = SPATTN_MAX_COPY_TASKS;
struct CopyTaskSet {
  CopyTask t[kMaxCopyTasks];
  int n;
};
void launch_copy_tasks(const CopyTaskSet& ts, int elem_bytes, cudaStream_t s);
// rope.cu: angle table float2(cos, sin)[rows][dim/2] of device position ids, and the rotating
// row copier (every task of the set carries a table)
void launch_rope_table(float2* table, const int64_t* dpos, int64_t rows, int dim, double base,
                       cudaStream_t s);
void launch_copy_tasks_rope(const CopyTaskSet& ts, cudaStream_t s);

// acc (fp32 out + lse) merge of a finished piece (fp32 out + lse) — merge_piece
// (attention.cpp:117-149) in LSE form.
void launch_lse_merge(float* acc_o, float* acc_lse, const float* o, const float* lse, int64_t rows,
                      int d, cudaStream_t s);
void launch_fill_f32(float* p, float v, int64_t n, cudaStream_t s);
// dst_bf16[i] = src_f32[i] * scale
void launch_f32_to_bf16(void* dst, const float* src, float scale, int64_t n, cudaStream_t s);
void launch_bf16_to_f32(float* dst, const void* src, int64_t n, cudaStream_t s);
// Strided variant: rows x cols block with independent row strides (elements).
void launch_f32_to_bf16_2d(void* dst, int64_t dst_stride, const float* src, int64_t src_stride,
                           int64_t rows, int64_t cols, float scale, cudaStream_t s);
void launch_f32_add_2d(float* dst, int64_t dst_stride, const float* src, int64_t src_stride,
                       int64_t rows, int64_t cols, cudaStream_t s);
// dst[i] += src[i] over n contiguous fp32 (16-byte vectors when aligned)
void launch_f32_add(float* dst, const float* src, int64_t n, cudaStream_t s);

}  // namespace spattn
